"""Median per-phase device times of the batched filtered top-k (emit pass, selection) over
many executes, optionally under several environment settings in one process.

    python tools/time_phases.py [--items N] [--batch B] [--k K] [--iters I] [--env VAR=a,b,c]

Numbers printed here are for A/B experiments; bench.py is the reported measurement.
"""

from __future__ import annotations

import argparse
import ctypes
import os
import statistics
import sys
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
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--env", default="", help="VAR=v1,v2,... (one run per value)")
    ap.add_argument("--replan", action="store_true", help="re-create the plan per --env value")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    wl = workload.make_workload(a.items, a.batch)
    idx = wl.index
    op = TopkOp(idx, a.batch, a.k, np.array([[0, idx.n_slots]]))
    out = op.alloc_outputs()
    lib = _native.lib()
    lib.fb_topk_set_timing(op._plan, 1)
    settings = [None]
    if a.env:
        var, vals = a.env.split("=", 1)
        settings = [(var, v) for v in vals.split(",")]
    for st in settings:
        if st is not None:
            os.environ[st[0]] = st[1]
            if a.replan:  # plan-time settings: a fresh plan per value
                op = TopkOp(idx, a.batch, a.k, np.array([[0, idx.n_slots]]))
                lib.fb_topk_set_timing(op._plan, 1)
        emit, sel, tot = [], [], []
        for i in range(a.iters + 3):
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            op(wl.queries_q, wl.batch, out=out)
            s1.record()
            torch.cuda.synchronize()
            e = ctypes.c_float()
            se = ctypes.c_float()
            _native.check(lib.fb_topk_last_timing(op._plan, ctypes.byref(e), ctypes.byref(se)))
            if i >= 3:
                emit.append(e.value)
                sel.append(se.value)
                tot.append(s0.elapsed_time(s1))
        med = statistics.median
        print(f"{st}: emit {med(emit):.4f} ms (min {min(emit):.4f} max {max(emit):.4f}), "
              f"select {med(sel):.4f} ms, execute {med(tot):.4f} ms", flush=True)


if __name__ == "__main__":
    main()
