"""The C++ batch packer on the GPU path: request filter texts packed by
``FilterBatch.from_text`` (C++ parse + compile + pack) drive the fused scan to the oracle's
``codesigned_search`` answers (reference retrieval.py:110-144 over compile_filter of the
same texts); fresh batches of another shape go through ``PipelinedTopk.submit``; and
``eval_compiled`` works beyond int16 plane ids (reference test_evaluation.py:132 uses
M = 1 << 16)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wl(cuda):
    from paper_2511_14881_b200 import workload
    return workload.make_workload(60_000, 24, seed=11)


def _texts(n, seed):
    from paper_2511_14881_b200 import workload
    from paper_2511_14881_b200.filter_query import And, Leaf, Not, Or, format_filter
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        if i % 6 == 5:
            out.append("")  # unfiltered
        elif i % 6 == 4:  # negations / nesting: the non-windowed or bytecode forms
            e = And((Or((Leaf(1, int(rng.integers(50))), Not(Leaf(2, int(rng.integers(50)))))),
                     Not(And((Leaf(3, int(rng.integers(40))), Leaf(4, int(rng.integers(30))))))))
            out.append(format_filter(e))
        else:
            out.append(format_filter(workload.four_attribute_filter(rng)))
    return out


def _oracle(wl, texts, q, k):
    from oracle import filtra_oracle as orc
    from paper_2511_14881_b200 import _device
    from paper_2511_14881_b200.bloom import BloomParams
    from paper_2511_14881_b200.filter_query import compile_filter, parse_filter
    idx = wl.index
    items = idx.items.cpu().numpy()[:, : wl.dim]
    valid, iid = _device.u64_host(idx.valid), _device.u64_host(idx.item_ids)
    qq = wl.queries_q.cpu().numpy()[:, : wl.dim]
    prog = None
    if texts[q]:
        cf = compile_filter(parse_filter(texts[q]), BloomParams())
        prog = ([(int(o), int(a)) for o, a in cf.ops], [(f, v, qb.set_bits) for f, v, qb in cf.leaves])
    return orc.codesigned_search(items, valid, iid, np.array([[0, idx.n_slots]]), idx.bloom.planes,
                                 prog, qq[q], [0], k)


@pytest.mark.parametrize("seed", [1, 2])
def test_text_batch_scan_vs_oracle(wl, seed):
    from paper_2511_14881_b200 import _device
    from paper_2511_14881_b200.bloom import BloomParams
    from paper_2511_14881_b200.engine import TopkOp
    from paper_2511_14881_b200.filter_query import FilterBatch
    texts = _texts(24, seed)
    batch = FilterBatch.from_text(texts, None, BloomParams())
    k = 400
    out = TopkOp(wl.index, 24, k, np.array([[0, wl.index.n_slots]]))(wl.queries_q, batch)
    torch.cuda.synchronize()
    for q in range(24):
        ref = _oracle(wl, texts, q, k)
        n = int(out.count[q])
        assert np.array_equal(_device.u64_host(out.ids[q, :n]), ref.item_ids), q
        assert np.array_equal(out.scores[q, :n].cpu().numpy(), ref.scores), q


def test_pipelined_fresh_text_batches(wl):
    """Every step a new batch of texts (differently shaped packed arrays): uploaded on the
    copy stream, results equal the oracle's."""
    from paper_2511_14881_b200 import _device
    from paper_2511_14881_b200.bloom import BloomParams
    from paper_2511_14881_b200.engine import PipelinedTopk
    from paper_2511_14881_b200.filter_query import FilterBatch
    k = 300
    pipe = PipelinedTopk(wl.index, 24, k, filters_template=wl.filters)
    host_q = wl.queries.cpu().pin_memory()
    batches = [_texts(24, 40 + s) for s in range(4)]
    tickets = [pipe.submit(host_q, FilterBatch.from_text(t, None, BloomParams())) for t in batches[:2]]
    got = {}
    for j, t in enumerate(tickets):
        ids, sc, cnt = pipe.result(t)
        got[j] = (ids.clone(), sc.clone(), cnt.clone())
    for j in range(2):
        ids, sc, cnt = got[j]
        for q in (0, 4, 5, 11, 23):
            ref = _oracle(wl, batches[j], q, k)
            n = int(cnt[q])
            assert np.array_equal(_device.u64_host(ids[q, :n]), ref.item_ids), (j, q)
            assert np.array_equal(sc[q, :n].numpy(), ref.scores), (j, q)


def test_eval_compiled_large_m_bits(cuda):
    from oracle import filtra_oracle as orc
    from paper_2511_14881_b200.bloom import BloomParams, build_bloom
    from paper_2511_14881_b200.filter_query import And, Leaf, Not, Or, compile_filter, eval_compiled
    rng = np.random.default_rng(6)
    feats = [[(int(rng.integers(100)), int(rng.integers(100)))] for _ in range(700)]
    p = BloomParams(m_bits=1 << 16, k_hashes=5)
    bl = build_bloom(feats, p)
    n_words = (len(feats) + 63) // 64
    valid = np.full(n_words, np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    valid[-1] = np.uint64((1 << (len(feats) % 64)) - 1)
    for e in (Leaf(*feats[3][0]), Or((Leaf(*feats[5][0]), Not(Leaf(*feats[9][0])))),
              And((Leaf(10_000, 1), Leaf(10_001, 2)))):
        cf = compile_filter(e, p)
        got = eval_compiled(cf, bl, valid)
        want = orc.eval_compiled([(int(o), int(a)) for o, a in cf.ops],
                                 [(f, v, qb.set_bits) for f, v, qb in cf.leaves], bl.planes, valid)
        assert np.array_equal(got, want)
