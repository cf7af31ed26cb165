"""Which step of the single-request graph (fastpath.py) breaks CUDA-graph capture: captures
each step alone on a small synthetic IVF index and prints the first error per step."""
from __future__ import annotations

import sys
import traceback
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2511_14881_b200 as fb  # noqa: E402
from paper_2511_14881_b200.ivf import IvfSearchOp  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    n, dim, C = 4096, 16, 14
    emb = rng.standard_normal((n, dim)).astype(np.float32)
    qp = fb.QuantParams(float(emb.min()), float(emb.max()))
    items = fb.quantize_matrix(emb, qp).data
    offs = np.stack([np.arange(C) * (n // C) // 64 * 64, np.minimum((np.arange(C) + 1) * (n // C) // 64 * 64, n)], 1)
    offs[-1, 1] = n
    valid = np.full(n // 64, np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    cent = torch.as_tensor(rng.standard_normal((C, dim)).astype(np.float32), device="cuda")
    dix = fb.DeviceIndex.from_arrays(items, valid, np.arange(n, dtype=np.uint64), qp=qp,
                                     cluster_offsets=offs, centroids=cent)
    op = IvfSearchOp(dix, 1, 3, 10, path="probe")
    u = torch.as_tensor(emb[:1], device="cuda")
    clusters = op.probe(u)
    qq = dix.quantize_queries(u)
    op.scan(qq, clusters)
    torch.cuda.synchronize()
    steps = {
        "task_dots": lambda: fb._native.lib().fb_task_dots_f64(
            dix.centroids.data_ptr(), C, dim, op._probe_rows.data_ptr(), op._probe_cnt.data_ptr(),
            C, torch.zeros((32, dim), device="cuda").data_ptr(), 1, 32,
            torch.empty((32, C), dtype=torch.float64, device="cuda").data_ptr(),
            fb._native.stream_ptr()),
        "sort": lambda: torch.sort(torch.rand((1, C), dtype=torch.float64, device="cuda"), dim=1,
                                   descending=True, stable=True),
        "probe": lambda: op.probe(u),
        "quantize": lambda: dix.quantize_queries(u),
        "probe_words": lambda: op.probe_words(clusters),
        "scan": lambda: op.scan(qq, clusters),
    }
    for name, fn in steps.items():
        for mode in ("thread_local", "relaxed"):
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g, capture_error_mode=mode):
                    r = fn()
                g.replay()
                torch.cuda.synchronize()
                print(f"{name:12s} {mode:12s} ok ({r if isinstance(r, int) else ''})", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"{name:12s} {mode:12s} FAIL: {type(e).__name__}: {str(e).splitlines()[0]}",
                      flush=True)
                tb = traceback.format_exception(e)
                print("   " + " | ".join(x.strip().splitlines()[0] for x in tb[-6:]), flush=True)
                torch.cuda.synchronize()


if __name__ == "__main__":
    main()
