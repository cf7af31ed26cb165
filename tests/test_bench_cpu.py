"""bench.py host logic without a GPU: argument defaults, workload description, the
config-4 |S| sizing and the parity comparison."""

from __future__ import annotations

import sys
from types import SimpleNamespace

import numpy as np
import torch

import bench


def test_defaults_and_workload_desc(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse_args()
    assert (a.items, a.batch, a.k, a.config, a.gpus) == (10_000_000, 256, 10_000, 2, 1)
    assert a.steps >= 3 and a.warmup >= 3
    for ex in ("owner", "pruned", "all_gather"):
        a.exchange = ex
        d1, d8 = bench.workload_desc(a, 1), bench.workload_desc(a, 8)
        assert d1["parallelism"] == "single GPU"
        assert "x8" in d8["parallelism"] and d8["items_total"] == 8 * a.items


def test_sweep_sizes_monotone():
    sizes = [bench.sweep_sizes(p) for p in bench.SWEEP if p < 1.0]
    for s0, s1 in zip(sizes, sizes[1:]):
        assert all(x <= y for x, y in zip(s0, s1))
    assert bench.sweep_sizes(0.10)[0] >= 1


def test_parity_check_counts_mismatches():
    ids = torch.tensor([[5, 7, 0], [1, 2, 3]], dtype=torch.int64)
    scores = torch.tensor([[9, 8, 0], [3, 2, 1]], dtype=torch.int32)
    out = SimpleNamespace(ids=ids, scores=scores, count=torch.tensor([2, 3], dtype=torch.int32))
    good = [(np.array([5, 7], np.uint64), np.array([9, 8], np.int32)),
            (np.array([1, 2, 3], np.uint64), np.array([3, 2, 1], np.int32))]
    assert bench.parity_check(out, good, range(2))["mismatches"] == 0
    bad = [good[0], (np.array([1, 3, 2], np.uint64), np.array([3, 2, 1], np.int32))]
    r = bench.parity_check(out, bad, range(2))
    assert r["mismatches"] == 1 and r["bad_queries"] == [1]
