"""Sampling-threshold diagnostics for one selectivity of the config-4 sweep: candidate
counts vs k and the emit buffer, and how many queries took the exact fallback.

    python tools/debug_threshold.py [--items N] [--p 0.2] [--k 10000]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))

from paper_2511_14881_b200 import workload  # noqa: E402
from paper_2511_14881_b200.bloom import BloomParams  # noqa: E402
from paper_2511_14881_b200.engine import TopkOp  # noqa: E402
from paper_2511_14881_b200.filter_query import FilterBatch, compile_filter  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--items", type=int, default=10_000_000)
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--k", type=int, default=10_000)
    a = ap.parse_args()
    import bench
    torch.cuda.set_device(0)
    B = 256
    wl = workload.make_workload(a.items, B, seed=1)
    sizes = bench.sweep_sizes(a.p)
    rng = np.random.default_rng(7)
    filters = [compile_filter(workload.four_attribute_filter(rng, sizes), BloomParams())
               for _ in range(B)]
    batch = FilterBatch.pack(filters, BloomParams()).to_device()
    op = TopkOp(wl.index, B, a.k, np.array([[0, wl.index.n_slots]]))
    for rep in range(3):
        out = op(wl.queries_q, batch)
        torch.cuda.synchronize()
        st = op.stats()
        print(f"rep {rep}: sizes={sizes} fallback_queries={st.fallback_queries} "
              f"windowed={batch.cnf_windowed} words={batch.cnf_words}", flush=True)


if __name__ == "__main__":
    main()
