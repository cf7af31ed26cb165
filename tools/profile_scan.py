"""Profiling driver: build the config-2 workload and run the batched filtered top-k a few
times (for ``ncu`` captures; numbers printed here are not bench values).

    python tools/profile_scan.py [--items N] [--batch B] [--k K] [--iters I] [--simt]
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2511_14881_b200 import _native, workload  # noqa: E402
from paper_2511_14881_b200.engine import TopkOp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--items", type=int, default=10_000_000)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--k", type=int, default=10_000)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--simt", action="store_true")
    ap.add_argument("--unfiltered", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    wl = workload.make_workload(a.items, a.batch, filtered=not a.unfiltered)
    idx = wl.index
    op = TopkOp(idx, a.batch, a.k, np.array([[0, idx.n_slots]]),
                _native.FB_PLAN_SIMT if a.simt else 0)
    out = op.alloc_outputs()
    for i in range(a.iters):
        torch.cuda.synchronize()
        t = time.perf_counter()
        op(wl.queries_q, wl.batch, out=out)
        torch.cuda.synchronize()
        print(f"iter {i}: {1e3 * (time.perf_counter() - t):.3f} ms, "
              f"path={'tc' if _native.lib().fb_topk_scan_path(op._plan) else 'simt'}, "
              f"count[0]={int(out.count[0])}", flush=True)


if __name__ == "__main__":
    main()
