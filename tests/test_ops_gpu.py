"""The custom ops on the B200: ``torch.library.opcheck`` (schema, fake kernel, dispatch),
bit-equality with the batched operator and the oracle, ``torch.compile(fullgraph=True)``
through the ops, and the serving pipeline's filter-batch validation."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wl(cuda):
    from paper_2511_14881_b200 import workload
    return workload.make_workload(50_000, 16, seed=5)


def test_filtered_topk_op_matches_operator_and_oracle(wl):
    from oracle import filtra_oracle as orc
    from paper_2511_14881_b200 import _device, ops
    from paper_2511_14881_b200.engine import TopkOp
    idx, k = wl.index, 700
    ids, scores, count = ops.search_batch(idx, wl.queries, k, wl.batch)
    ref = TopkOp(idx, 16, k, np.array([[0, idx.n_slots]]))(wl.queries_q, wl.batch)
    torch.cuda.synchronize()
    assert torch.equal(count, ref.count)
    for q in range(16):
        n = int(count[q])
        assert torch.equal(ids[q, :n], ref.ids[q, :n]) and torch.equal(scores[q, :n],
                                                                        ref.scores[q, :n])
    items = idx.items.cpu().numpy()[:, : wl.dim]
    valid, iid = _device.u64_host(idx.valid), _device.u64_host(idx.item_ids)
    qq = wl.queries_q.cpu().numpy()[:, : wl.dim]
    for q in (0, 7, 15):
        cf = wl.filters[q]
        prog = ([(int(o), int(a)) for o, a in cf.ops],
                [(f, v, qb.set_bits) for f, v, qb in cf.leaves])
        r = orc.codesigned_search(items, valid, iid, np.array([[0, idx.n_slots]]),
                                  idx.bloom.planes, prog, qq[q], [0], k)
        n = int(count[q])
        assert np.array_equal(_device.u64_host(ids[q, :n]), r.item_ids)
        assert np.array_equal(scores[q, :n].cpu().numpy(), r.scores)


def test_opcheck(wl):
    from paper_2511_14881_b200 import ops
    idx = wl.index
    qq = wl.queries_q
    args = (ops.index_handle(idx), qq, 50, [0, idx.n_slots], wl.batch.device_arrays(),
            wl.batch.meta(), 0)
    torch.library.opcheck(torch.ops.filtra_b200.filtered_topk.default, args,
                          test_utils=("test_schema", "test_faketensor"))
    x = wl.queries
    torch.library.opcheck(torch.ops.filtra_b200.quantize.default,
                          (x, float(idx.qp.global_min), float(idx.qp.global_max), idx.dim_pad),
                          test_utils=("test_schema", "test_faketensor"))


def test_compile_fullgraph_through_ops(wl):
    from paper_2511_14881_b200 import ops
    idx = wl.index
    h = ops.index_handle(idx)
    fa, fm = wl.batch.device_arrays(), wl.batch.meta()
    gmin, gmax = float(idx.qp.global_min), float(idx.qp.global_max)

    def f(x):
        qq = torch.ops.filtra_b200.quantize(x, gmin, gmax, idx.dim_pad)
        ids, scores, count = torch.ops.filtra_b200.filtered_topk(h, qq, 100, [], fa, fm, 0)
        return ids, scores + 0, count

    eager = f(wl.queries)
    compiled = torch.compile(f, fullgraph=True, backend="aot_eager")(wl.queries)
    for a, b in zip(eager, compiled):
        assert torch.equal(a, b)


def test_merge_op_matches_oracle(cuda):
    from oracle import filtra_oracle as orc
    rng = np.random.default_rng(3)
    S, B, k = 3, 4, 40
    scores = np.zeros((S, B, k), np.int32)
    ids = np.zeros((S, B, k), np.int64)
    cnt = rng.integers(0, k + 1, size=(S, B)).astype(np.int32)
    for s in range(S):
        for b in range(B):
            sc = rng.integers(-50, 50, size=cnt[s, b])
            ii = rng.choice(10_000, size=cnt[s, b], replace=False) + 1000 * s
            o = np.lexsort((ii, -sc))
            scores[s, b, : cnt[s, b]], ids[s, b, : cnt[s, b]] = sc[o], ii[o]
    out = torch.ops.filtra_b200.merge_topk(torch.from_numpy(scores).cuda(),
                                           torch.from_numpy(ids).cuda(),
                                           torch.from_numpy(cnt).cuda(), 60)
    for b in range(B):
        all_i = np.concatenate([ids[s, b, : cnt[s, b]] for s in range(S)]).astype(np.uint64)
        all_s = np.concatenate([scores[s, b, : cnt[s, b]] for s in range(S)])
        ri, rs = orc.reduce_topk(all_i, all_s, 60)
        n = int(out[2][b])
        assert np.array_equal(out[0][b, :n].cpu().numpy().astype(np.uint64), ri)
        assert np.array_equal(out[1][b, :n].cpu().numpy(), rs)


def test_pipeline_validates_and_repacks(wl):
    from paper_2511_14881_b200 import BloomParams, FilterBatch, compile_filter, workload
    from paper_2511_14881_b200.engine import PipelinedTopk, TopkOp
    idx, B, k = wl.index, 16, 300
    pipe = PipelinedTopk(idx, B, k, filters_template=wl.filters)
    hq = wl.queries.cpu().pin_memory()
    with pytest.raises(ValueError):
        pipe.submit(hq[:8])
    rng = np.random.default_rng(99)
    # same shape (4-attribute CNF) but other programs; then a different-shape batch
    # (two groups, a negation); then the template's own filters again
    other = [compile_filter(workload.four_attribute_filter(rng), BloomParams()) for _ in range(B)]
    from paper_2511_14881_b200.filter_query import And, Leaf, Not, Or
    odd = [compile_filter(And((Or((Leaf(1, q % 50), Leaf(2, 3))), Not(Leaf(3, q % 40)))),
                          BloomParams()) for q in range(B)]
    op = TopkOp(idx, B, k, np.array([[0, idx.n_slots]]))
    for cfs in (other, odd, wl.filters, other):
        fb = FilterBatch.pack(cfs, BloomParams()).pin()
        ids, scores, count = pipe.result(pipe.submit(hq, fb))
        ref = op(wl.queries_q, FilterBatch.pack(cfs, BloomParams()).to_device())
        torch.cuda.synchronize()
        assert torch.equal(count, ref.count.cpu())
        for q in range(B):
            n = int(count[q])
            assert torch.equal(ids[q, :n], ref.ids[q, :n].cpu())
            assert torch.equal(scores[q, :n], ref.scores[q, :n].cpu())
