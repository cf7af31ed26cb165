"""Parity at the BASELINE.json configurations (SURVEY §8(c) "how parity is checked at
scale"): the batched operator's rows vs the oracle's ``codesigned_search`` (reference
retrieval.py:110-144) on identical synthetic inputs, bit-exact ids / int32 scores / order.

* config 1 exactly: 1M items x 128-d, 64 queries, k = 1000, 4-attribute filter, every query;
* config 4 extremes: 1 % and 100 % (no filter) selectivity at 1M items, k = 10000;
* config 3 shape: 12.5M items, batch 1024, k = 20000, sampled queries (incl. the last
  256-query chunk);
* a shuffled-id variant (random 63-bit ids, so the id-rank tie-break is not the slot order).

The oracle runs in a fork pool (NumPy only in the children) so the 10M+ cases finish in
seconds per query."""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

_POOL_ARGS: dict = {}


def _one(i):
    from oracle import filtra_oracle as orc
    d = _POOL_ARGS
    q = d["queries"][i]
    prog = d["progs"][q]
    res = orc.codesigned_search(d["items"], d["valid"], d["ids"], d["offs"], d["planes"], prog,
                                d["qq"][q], [0], d["k"])
    return q, res.item_ids, res.scores


def oracle_answers(wl, k, queries, progs=None):
    from paper_2511_14881_b200._device import u64_host
    idx = wl.index
    if progs is None:
        progs = [([(int(o), int(a)) for o, a in cf.ops],
                  [(f, v, qb.set_bits) for f, v, qb in cf.leaves]) if cf is not None else None
                 for cf in wl.filters]
    _POOL_ARGS.update(items=idx.items.cpu().numpy()[:, : wl.dim], valid=u64_host(idx.valid),
                      ids=u64_host(idx.item_ids), offs=np.array([[0, idx.n_slots]]),
                      planes=idx.bloom.planes, qq=wl.queries_q.cpu().numpy()[:, : wl.dim],
                      progs=progs, k=k, queries=list(queries))
    cores = max(1, min(len(os.sched_getaffinity(0)), len(queries)))
    with mp.get_context("fork").Pool(cores) as pool:
        out = pool.map(_one, range(len(queries)), chunksize=1)
    _POOL_ARGS.clear()
    return out


def check_rows(out, answers):
    from paper_2511_14881_b200._device import u64_host
    for q, ref_ids, ref_scores in answers:
        n = int(out.count[q])
        assert n == len(ref_ids), (q, n, len(ref_ids))
        assert np.array_equal(u64_host(out.ids[q, :n]), ref_ids), q
        assert np.array_equal(out.scores[q, :n].cpu().numpy(), ref_scores), q


def run_op(wl, k, batch="workload"):
    from paper_2511_14881_b200.engine import TopkOp
    idx = wl.index
    op = TopkOp(idx, wl.queries_q.shape[0], k, np.array([[0, idx.n_slots]]))
    fb = wl.batch.to_device() if batch == "workload" else batch
    out = op(wl.queries_q, fb)
    torch.cuda.synchronize()
    return out


def test_config1_exact_all_queries(cuda):
    """BASELINE config 1: 1M x 128-d int8, 64 queries, top-k 1000, 4-attribute filter."""
    from paper_2511_14881_b200 import workload
    wl = workload.make_workload(1_000_000, 64, seed=1)
    out = run_op(wl, 1000)
    check_rows(out, oracle_answers(wl, 1000, range(64)))


@pytest.mark.parametrize("selectivity", [0.01, 1.0])
def test_config4_extremes(cuda, selectivity):
    """Config-4 sweep end points at 1M items, batch 64, k = 10000 (the bench's |S| sizing)."""
    from bench import sweep_sizes
    from paper_2511_14881_b200 import workload
    if selectivity >= 1.0:
        wl = workload.make_workload(1_000_000, 64, seed=2, filtered=False)
        out = run_op(wl, 10_000, batch=None)
    else:
        wl = workload.make_workload(1_000_000, 64, seed=2,
                                    filter_sizes=sweep_sizes(selectivity))
        out = run_op(wl, 10_000)
    qs = list(range(0, 64, 4)) + [63]
    check_rows(out, oracle_answers(wl, 10_000, qs))


def test_config3_shape_sampled(cuda):
    """Config 3 per GPU: 12.5M items, batch 1024, k = 20000; sampled queries from every
    256-query chunk of the batch."""
    from paper_2511_14881_b200 import workload
    wl = workload.make_workload(12_500_000, 1024, seed=3)
    out = run_op(wl, 20_000)
    qs = [0, 255, 256, 600, 777, 1023]
    check_rows(out, oracle_answers(wl, 20_000, qs))
    del out, wl
    torch.cuda.empty_cache()


def test_shuffled_ids_tiebreak(cuda):
    """Random 63-bit item ids (SURVEY §8(d) variant): ties must break by the u64 id, not by
    slot order; many exact duplicate rows force ties at the k-th score."""
    from paper_2511_14881_b200 import workload
    from paper_2511_14881_b200.engine import DeviceIndex
    wl = workload.make_workload(200_000, 32, seed=4)
    idx = wl.index
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    items = idx.items.clone()
    items[1::5] = items[0::5][: items[1::5].shape[0]]  # duplicate rows -> tied scores
    n = idx.n_slots
    ids = torch.randint(0, 2**63 - 1, (items.shape[0],), generator=g, device="cuda")
    ids[n:] = 0
    wl.index = DeviceIndex(items, idx.valid, ids, idx.n_slots, idx.dim, bloom=idx.bloom,
                           qp=idx.qp)
    out = run_op(wl, 3000)
    check_rows(out, oracle_answers(wl, 3000, range(0, 32, 3)))


@pytest.mark.parametrize("mode,B,v1", [("0", 40, "0"), ("1", 40, "0"), ("0", 200, "0"),
                                        ("1", 200, "0"), ("0", 200, "1"), ("1", 200, "1"),
                                        ("0", 129, "0"), ("1", 256, "0")])
def test_filter_first_and_per_hit_modes_agree(cuda, monkeypatch, mode, B, v1):
    """The window-form emit pass has two hit passes (per-hit test on item-major column bits,
    and filter-first eligibility words); the device picks one from the sampled eligibility.
    Forcing either must give the oracle's rows, at the benchmark's ~10 % selectivity and with
    explicit masks and ranges -- in the 20-warp layout (B <= 128, or FB_CNF_V1=1) and in the
    24-warp layout of two M-blocks (modes 3 and 4)."""
    from paper_2511_14881_b200 import _device, workload
    from paper_2511_14881_b200.engine import TopkOp
    monkeypatch.setenv("FB_CNF_FFIRST", mode)
    monkeypatch.setenv("FB_CNF_V1", v1)
    wl = workload.make_workload(300_000, B, seed=6)
    out = run_op(wl, 2000)
    check_rows(out, oracle_answers(wl, 2000, range(0, B, 7 if B > 64 else 3)))
    # ranges + explicit masks through the same kernel
    idx = wl.index
    rng = np.random.default_rng(5)
    ranges = np.array([[0, 64 * 700], [64 * 1500, 64 * 4000]])
    op = TopkOp(idx, B, 700, ranges)
    m = rng.integers(0, 2**63, size=(B, idx.n_words), dtype=np.int64)
    masks = torch.from_numpy(m).cuda()
    got = op(wl.queries_q, wl.batch.to_device(), masks=masks)
    torch.cuda.synchronize()
    from oracle import filtra_oracle as orc
    items = idx.items.cpu().numpy()[:, : wl.dim]
    valid, ids = _device.u64_host(idx.valid), _device.u64_host(idx.item_ids)
    qq = wl.queries_q.cpu().numpy()[:, : wl.dim]
    for q in (0, 13, 39, B - 1):
        cf = wl.filters[q]
        prog = ([(int(o), int(a)) for o, a in cf.ops], [(f, v, qb.set_bits) for f, v, qb in cf.leaves])
        full = orc.eval_compiled(prog[0], prog[1], idx.bloom.planes, valid)
        keep = full & m[q].view(np.uint64)
        ref = orc.search_clusters(items, valid, ids, ranges, qq[q], range(len(ranges)), keep, 700)
        n = int(got.count[q])
        assert np.array_equal(_device.u64_host(got.ids[q, :n]), ref.item_ids), q
        assert np.array_equal(got.scores[q, :n].cpu().numpy(), ref.scores), q
