"""CPU-only checks: the C-ABI library loads and exports every declared symbol; host-side
hashing / compilation / packing / parsing match the reference golden vectors."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, json_to_expr, load_json, load_npz
from paper_2511_14881_b200 import _native, bitset
from paper_2511_14881_b200.bloom import BloomParams, hash_positions, hash_positions_batch, \
    hash_seed, positions_from_seed
from paper_2511_14881_b200.errors import FilterSyntaxError, UnknownFeature, UnknownValue
from paper_2511_14881_b200.filter_query import (And, FilterBatch, Leaf, Not, OpCode, Or,
                                                Vocabulary, compile_filter, format_filter,
                                                parse_filter)


def header_symbols() -> set[str]:
    text = (ROOT / "include" / "filtra_b200.h").read_text()
    return set(re.findall(r"^\s*(?:int|int64_t|const char\*|uint64_t|void)\s+(fb_\w+)\(", text, flags=re.M))


def test_library_exports_every_header_symbol():
    lib = _native.load_library()
    declared = header_symbols()
    assert declared, "no declarations parsed"
    assert declared == set(_native.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.fb_abi_version() == _native.ABI_VERSION == 5


def test_library_is_sm100a_only():
    so = _native.library_path()
    data = so.read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


def test_c_hash_matches_reference_kats():
    for case in load_json("hash_kats.json"):
        fid, val = int(case["fid"]), int(case["value"])
        p = BloomParams(case["m_bits"], case["k_hashes"])
        assert list(hash_positions(fid, val, p).set_bits) == case["positions"]
        assert hash_seed(fid, val) == int(case["seed"])
        assert list(positions_from_seed(int(case["seed"]), p)) == case["positions"]


def test_c_hash_batch_padding():
    pos, cnt = hash_positions_batch([1, 2], [2, 3], BloomParams(8, 6))
    for row, c in zip(pos, cnt):
        assert list(row[c:]) == [-1] * (6 - c)
        assert list(row[:c]) == sorted(set(row[:c]))


def test_compile_matches_reference_golden():
    for e in load_json("filter_exprs.json"):
        cf = compile_filter(json_to_expr(e["expr"]), BloomParams(64, 3))
        assert [[int(o), int(a)] for o, a in cf.ops] == e["ops"]
        assert [[str(f), str(v), list(q.set_bits)] for f, v, q in cf.leaves] == e["leaves"]
        assert cf.max_stack_depth() == e["max_stack"]


VOCAB = Vocabulary(feature_ids={"country": 1, "lang": 2, "topic": 3},
                   values={"US": 10, "EN": 20, "ES": 21, "sports": 30})


def test_parser_grammar():
    assert parse_filter('country = "US" AND (lang = "EN" OR lang = "ES")', VOCAB) == \
        And((Leaf(1, 10), Or((Leaf(2, 20), Leaf(2, 21)))))
    assert parse_filter("1 = 1 OR 1 = 2 AND 2 = 3") == And((Or((Leaf(1, 1), Leaf(1, 2))), Leaf(2, 3)))
    assert parse_filter("NOT 1 = 1 AND 2 = 2") == And((Not(Leaf(1, 1)), Leaf(2, 2)))
    assert parse_filter("1 = 1 and not 2 = 2") == And((Leaf(1, 1), Not(Leaf(2, 2))))
    for bad in ("1 = ", "(1 = 2", "1 = 2 2 = 3"):
        with pytest.raises(FilterSyntaxError):
            parse_filter(bad, VOCAB)
    with pytest.raises(UnknownFeature):
        parse_filter('bogus = "US"', VOCAB)
    with pytest.raises(UnknownValue):
        parse_filter('country = "XX"', VOCAB)


def test_format_roundtrip():
    for e in load_json("filter_exprs.json"):
        expr = json_to_expr(e["expr"])
        assert parse_filter(format_filter(expr)) == expr


def test_filter_batch_packing_dedupes_across_queries():
    p = BloomParams()
    a = compile_filter(And((Leaf(1, 1), Or((Leaf(2, 2), Leaf(1, 1))))), p)
    b = compile_filter(Or((Leaf(2, 2), Leaf(3, 3))), p)
    batch = FilterBatch.pack([a, None, b], p)
    assert batch.n_queries == 3 and batch.n_leaves == 3
    assert list(batch.host_op_offset) == [0, len(a.ops), len(a.ops), len(a.ops) + len(b.ops)]
    ops = batch.host_ops
    # query b's first push refers to the shared (2, 2) leaf index 1
    assert int(ops[len(a.ops)]) == 1
    assert int(ops[2]) >> 14 == 0 and int(ops[3]) >> 14 == int(OpCode.OR)
    assert batch.push_leaf_bits[1] == 0
    row = batch.host_leaf_pos[0]
    assert list(row[row >= 0]) == list(hash_positions(1, 1, p).set_bits)


def test_bitset_helpers_match_reference_layout():
    flags = np.zeros(130, dtype=bool)
    flags[[0, 63, 64, 129]] = True
    w = bitset.from_bool(flags)
    assert list(w) == [(1 | (1 << 63)), 1, 2]
    assert np.array_equal(bitset.to_bool(w, 130), flags)
    assert list(bitset.indices(w, 130)) == [0, 63, 64, 129]
    assert bitset.popcount(bitset.ones(70)) == 70


def _numpy_pairwise(p):
    """Restatement of the summation order fb_dot_rows_f64 implements."""
    n = len(p)
    if n < 8:
        r = 0.0
        for x in p:
            r += x
        return r
    if n <= 128:
        r = list(p[:8])
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += p[i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += p[i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return _numpy_pairwise(p[:n2]) + _numpy_pairwise(p[n2:])


@pytest.mark.parametrize("d", [2, 7, 8, 12, 16, 24, 32, 128, 129, 300])
def test_pairwise_order_reproduces_numpy_dot_rows(d):
    rng = np.random.default_rng(d)
    rows = rng.standard_normal((50, d)).astype(np.float32)
    v = rng.standard_normal(d).astype(np.float32)
    ref = np.sum(rows.astype(np.float64) * v.astype(np.float64), axis=1)
    for i in range(50):
        p = rows[i].astype(np.float64) * v.astype(np.float64)
        assert 0.0 + _numpy_pairwise(list(p)) == ref[i]


def test_header_documents_reference_interfaces():
    text = (ROOT / "include" / "filtra_b200.h").read_text()
    for cite in ("bloom.py:114-144", "filter_query.py:314-356", "ivf.py:272-334",
                 "serve.py:98-121", "quantize.py:64-76"):
        assert cite in text


def test_golden_fixtures_present():
    for name in ("hash_kats.json", "bloom_cases.npz", "filter_cases.npz", "scan_cases.npz",
                 "four_attr.npz", "topk20000.npz", "merge_cases.npz", "quantize_cases.npz"):
        assert (Path(ROOT) / "tests" / "golden" / name).exists()
    assert load_npz("merge_cases.npz")["n_cases"][0] == 5


def _cnf_eval(batch, planes, q):
    """The scan's CNF semantics on the host: column bits = AND of the literal's planes
    (complemented when negated); query q passes a slot iff each of its groups shares a
    column with it. Returns u64 words (validity not applied)."""
    nw = planes.shape[1]
    cols = []
    for cl in batch.host_col_leaf:
        leaf = int(cl) if cl >= 0 else ~int(cl)
        m = np.full(nw, ~np.uint64(0), dtype=np.uint64)
        for pos in batch.host_leaf_pos[leaf]:
            if pos >= 0:
                m &= planes[pos]
        cols.append(~m if cl < 0 else m)
    out = np.full(nw, ~np.uint64(0), dtype=np.uint64)
    for g in range(int(batch.host_qgroups[q])):
        acc = np.zeros(nw, dtype=np.uint64)
        for c in range(len(cols)):
            if (int(batch.host_qmask[q, g, c >> 5]) >> (c & 31)) & 1:
                acc |= cols[c]
        out &= acc
    return out


@pytest.mark.parametrize("n_feat,n_vals,windowed", [(3, 12, 1), (4, 50, 1), (6, 12, 0)])
def test_cnf_packing_matches_compiled_programs(n_feat, n_vals, windowed):
    """FilterBatch.pack's CNF form (feature-binned 64-column windows) evaluates exactly like
    the compiled postfix programs (oracle eval_compiled) on random planes; batches whose
    groups each sit in one aligned u32 pair with <= 4 groups are flagged windowed."""
    from oracle import filtra_oracle as orc
    rng = np.random.default_rng(n_feat * 100 + n_vals)
    p = BloomParams()
    exprs = []
    for q in range(24):
        groups = []
        for f in range(1, n_feat + 1):
            k = int(rng.integers(1, 6))
            lits = [Leaf(f, int(v)) for v in rng.choice(n_vals, size=k, replace=False)]
            if rng.random() < 0.3:
                lits[0] = Not(lits[0])
            groups.append(Or(tuple(lits)) if len(lits) > 1 else lits[0])
        exprs.append(And(tuple(groups)))
    filters = [compile_filter(e, p) for e in exprs]
    filters[5] = None
    batch = FilterBatch.pack(filters, p)
    assert batch.is_cnf and batch.cnf_windowed == windowed
    planes = rng.integers(0, 2**63, size=(p.m_bits, 3), dtype=np.int64).astype(np.uint64)
    planes |= rng.integers(0, 2**63, size=(p.m_bits, 3), dtype=np.int64).astype(np.uint64)
    valid = np.full(3, ~np.uint64(0), dtype=np.uint64)
    for q, cf in enumerate(filters):
        got = _cnf_eval(batch, planes, q)
        if cf is None:
            assert int(batch.host_qgroups[q]) == 0
            continue
        ref = orc.eval_compiled([(int(o), int(a)) for o, a in cf.ops],
                                [(f, v, qb.set_bits) for f, v, qb in cf.leaves], planes, valid)
        assert np.array_equal(got, ref), q
    if windowed:
        nz = batch.host_qmask != 0
        for q in range(batch.n_queries):
            for g in range(int(batch.host_qgroups[q])):
                w = np.nonzero(nz[q, g])[0]
                assert len(w) and w.min() // 2 == w.max() // 2


def test_compile_filter_cache_returns_identical_program():
    """Repeated expressions hit the compile cache; the cached program equals a fresh one."""
    from paper_2511_14881_b200 import filter_query as fq
    expr = And((Or((Leaf(1, 2), Leaf(1, 3))), Not(Leaf(2, 7))))
    a = compile_filter(expr, BloomParams())
    b = compile_filter(And((Or((Leaf(1, 2), Leaf(1, 3))), Not(Leaf(2, 7)))), BloomParams())
    assert a is b
    fresh = fq._compile_filter(expr, BloomParams())
    assert fresh.ops == a.ops and fresh.leaves == a.leaves
    assert compile_filter(expr, BloomParams(m_bits=512)) is not a   # params are in the key
