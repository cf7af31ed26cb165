"""Publish-side k-means timings on one GPU: KMeans++ seeding (per centre), one Lloyd
assignment pass and a full build_ivf, against the reference's per-centre CPU cost measured
on the same rows with the oracle (numpy, the reference's own arithmetic).

    python tools/time_kmeans.py [--n 1000000] [--dim 128] [--k 1000] [--iters 5]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2511_14881_b200 import kmeans  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    rng = np.random.default_rng(1)
    x = rng.standard_normal((a.n, a.dim)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    X = kmeans._as_device_f64(x)
    torch.cuda.synchronize()
    out = {"n": a.n, "dim": a.dim, "k": a.k}

    stats = {}
    kmeans._pp_init_device(X, 8, 0)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    chosen = kmeans._pp_init_device(X, a.k, 0, stats)
    torch.cuda.synchronize()
    t_pp = time.perf_counter() - t0
    out["pp_init_s"] = round(t_pp, 3)
    out["pp_ms_per_centre"] = round(1e3 * t_pp / a.k, 3)
    out["pp_exact_walks"] = stats.get("exact_walks")

    centers = X[chosen].to(torch.float32).to(torch.float64).contiguous()
    xx = torch.empty(a.n, dtype=torch.float64, device=X.device)
    from paper_2511_14881_b200 import _native
    _native.check(_native.lib().fb_row_sqnorm_f64(X.data_ptr(), a.n, a.dim, xx.data_ptr(),
                                                  _native.stream_ptr()))
    asg = torch.empty(a.n, dtype=torch.int64, device=X.device)
    d2 = torch.empty(a.n, dtype=torch.float64, device=X.device)
    kmeans._assign(X, xx, centers, asg, d2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        kmeans._assign(X, xx, centers, asg, d2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    out["assign_ms"] = round(ms, 2)
    out["assign_fp64_tflops"] = round(2.0 * a.n * a.k * a.dim / (ms * 1e-3) / 1e12, 2)

    t0 = time.perf_counter()
    kmeans._train_device(X, a.k, a.iters, 0.0, 0)
    torch.cuda.synchronize()
    out[f"train_{a.iters}_iters_s"] = round(time.perf_counter() - t0, 3)

    # reference arithmetic on the host (oracle), per centre, on a bounded sample of rows
    m = min(a.n, 200_000)
    xs = x[:m].astype(np.float64)
    best = ((xs - xs[0]) ** 2).sum(axis=1)
    t0 = time.perf_counter()
    reps = 5
    for r in range(reps):
        total = best.sum()
        idx = min(int(np.searchsorted(np.cumsum(best), 0.5 * total, side="right")), m - 1)
        np.minimum(best, ((xs - xs[idx]) ** 2).sum(axis=1), out=best)
    per = (time.perf_counter() - t0) / reps * (a.n / m)
    out["cpu_ref_ms_per_centre"] = round(1e3 * per, 2)
    out["cpu_ref_sample"] = f"{reps} seeding steps on {m} rows, scaled to n (1 core)"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
