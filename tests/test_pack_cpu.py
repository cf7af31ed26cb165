"""The C++ batch packer (csrc/fb_pack.cpp: ``fb_pack_postfix`` / ``fb_pack_text``) against
the Python restatement of the batch device form (tests/pack_restatement.py) -- byte-equal
arrays and scalars -- and its text path against the reference grammar (parse_filter +
compile_filter, reference filter_query.py:82-311). CPU only: the packer is host code."""

from __future__ import annotations

import time

import numpy as np
import pytest

from paper_2511_14881_b200 import errors
from paper_2511_14881_b200.bloom import BloomParams
from paper_2511_14881_b200.filter_query import (And, FilterBatch, Leaf, Not, Or, Vocabulary,
                                                compile_filter, format_filter, parse_filter)
from pack_restatement import pack_py

FIELDS = ("host_leaf_pos", "host_op_offset", "host_ops", "host_plane_list", "host_leaf_slot",
          "host_rop_offset", "host_rops", "host_col_leaf", "host_qmask", "host_qgroups")
SCALARS = ("n_queries", "n_leaves", "k_max", "max_stack", "rmax_stack", "cnf_words", "cnf_gmax",
           "cnf_windowed")


def assert_same(a: FilterBatch, b: FilterBatch):
    for f in FIELDS:
        x, y = getattr(a, f), getattr(b, f)
        assert (x is None) == (y is None), f
        if x is not None:
            assert x.dtype == y.dtype and x.shape == y.shape, (f, x.dtype, y.dtype, x.shape, y.shape)
            assert np.array_equal(x, y), f
    for f in SCALARS:
        assert getattr(a, f) == getattr(b, f), f
    assert a.meta() == b.meta()
    assert np.array_equal(np.asarray(a.push_leaf_bits), np.asarray(b.push_leaf_bits))


def rand_expr(rng, depth, feats, vals, p_not=0.15):
    r = rng.random()
    if depth == 0 or r < 0.3:
        e = Leaf(int(rng.choice(feats)), int(rng.integers(vals)))
    elif r < 0.65:
        e = And(tuple(rand_expr(rng, depth - 1, feats, vals, p_not)
                      for _ in range(int(rng.integers(2, 4)))))
    else:
        e = Or(tuple(rand_expr(rng, depth - 1, feats, vals, p_not)
                     for _ in range(int(rng.integers(2, 5)))))
    return Not(e) if rng.random() < p_not else e


def cnf_expr(rng, n_groups, sizes, feats, card):
    groups = []
    for g in range(n_groups):
        f = feats[g % len(feats)]
        vs = rng.choice(card, size=min(sizes, card), replace=False)
        lits = [Leaf(f, int(v)) if rng.random() > 0.1 else Not(Leaf(f, int(v))) for v in vs]
        groups.append(Or(tuple(lits)) if len(lits) > 1 else lits[0])
    return And(tuple(groups)) if len(groups) > 1 else groups[0]


def check_batch(exprs, params=BloomParams()):
    cfs = [None if e is None else compile_filter(e, params) for e in exprs]
    got = FilterBatch.pack(cfs, params)
    want = FilterBatch(**pack_py(cfs, params))
    assert_same(got, want)
    return got


@pytest.mark.parametrize("seed", range(12))
def test_random_programs_match_restatement(seed):
    rng = np.random.default_rng(seed)
    exprs = [None if rng.random() < 0.1 else rand_expr(rng, 3, [1, 2, 3, 7], 20)
             for _ in range(int(rng.integers(1, 40)))]
    check_batch(exprs)


@pytest.mark.parametrize("seed", range(8))
def test_cnf_batches_match_restatement(seed):
    rng = np.random.default_rng(100 + seed)
    n_groups = int(rng.integers(1, 10))      # > 8 groups: not CNF-packable
    size = int(rng.integers(1, 40))
    feats = [1, 2, 3, 4, 5, 6][: int(rng.integers(1, 7))]
    card = int(rng.integers(2, 90))          # > 64 literals of one feature: first-seen columns
    exprs = [cnf_expr(rng, n_groups, size, feats, card) if rng.random() > 0.05 else None
             for _ in range(int(rng.integers(1, 64)))]
    b = check_batch(exprs)
    assert b.n_queries == len(exprs)


def test_four_attribute_batch_is_windowed():
    from paper_2511_14881_b200.workload import four_attribute_filter
    rng = np.random.default_rng(7)
    b = check_batch([four_attribute_filter(rng) for _ in range(256)])
    assert b.is_cnf and b.cnf_windowed == 1 and b.cnf_gmax == 4


def test_unfiltered_and_empty_batches():
    check_batch([None, None, None])
    check_batch([])
    check_batch([Leaf(1, 2)])
    check_batch([Not(Leaf(1, 2)), None])


def test_large_m_bits():
    """m_bits beyond int16 (reference test_evaluation.py:132 uses 1 << 16)."""
    p = BloomParams(m_bits=1 << 16, k_hashes=5)
    b = check_batch([And((Leaf(10_000, 1), Leaf(10_001, 2))), Leaf(5, 5)], p)
    assert int(b.host_leaf_pos.max()) >= 32768 or int(b.host_plane_list.max()) < 1 << 16


VOCAB = Vocabulary(feature_ids={"country": 1, "lang": 2, "cat.sub": 3},
                   values={"US": 7, "DE": 8, "en": 9, "a b": 10})


@pytest.mark.parametrize("seed", range(6))
def test_text_path_matches_reference_grammar(seed):
    rng = np.random.default_rng(300 + seed)
    exprs = [rand_expr(rng, 3, [1, 2, 3, 11], 12) for _ in range(30)]
    texts = [format_filter(e, VOCAB) for e in exprs] + ["", None]
    got = FilterBatch.from_text(texts, VOCAB, BloomParams())
    want_cfs = [compile_filter(parse_filter(t, VOCAB), BloomParams()) if t else None for t in texts]
    assert_same(got, FilterBatch(**pack_py(want_cfs, BloomParams())))


def test_text_keywords_whitespace_and_names():
    texts = ['country = "US" and NOT (lang = "en" Or 3=4)', '\t1=2\nAND\r\x1c2 = 3',
             'cat.sub = "a b"', 'NOT NOT 5 = 6', '(((1 = 1)))']
    got = FilterBatch.from_text(texts, VOCAB, BloomParams())
    cfs = [compile_filter(parse_filter(t, VOCAB), BloomParams()) for t in texts]
    assert_same(got, FilterBatch(**pack_py(cfs, BloomParams())))


@pytest.mark.parametrize("text,exc", [
    ("country = ", errors.FilterSyntaxError),
    ("(1 = 2", errors.FilterSyntaxError),
    ("1 = 2)", errors.FilterSyntaxError),
    ("1 = 2 AND", errors.FilterSyntaxError),
    ('1 = "unterminated', errors.FilterSyntaxError),
    ("1 == 2", errors.FilterSyntaxError),
    ("1 = 2 # x", errors.FilterSyntaxError),
    ("nosuch = 1", errors.UnknownFeature),
    ('country = "XX"', errors.UnknownValue),
])
def test_text_errors_are_the_reference_exceptions(text, exc):
    with pytest.raises(exc) as got:
        FilterBatch.from_text(["1 = 1", text], VOCAB, BloomParams())
    with pytest.raises(exc) as want:
        parse_filter(text, VOCAB)
    assert str(got.value) == str(want.value)


def test_unicode_whitespace_takes_the_python_tokenizer():
    t = "1 = 2 AND 3 = 4"
    got = FilterBatch.from_text([t], VOCAB, BloomParams())
    cf = compile_filter(parse_filter(t, VOCAB), BloomParams())
    assert_same(got, FilterBatch(**pack_py([cf], BloomParams())))


def test_cold_text_pack_time():
    """Cold parse + compile + pack of 256 fresh four-attribute filter texts (reported; the
    assertion is loose so a loaded CI host does not flake)."""
    from paper_2511_14881_b200.workload import four_attribute_filter
    rng = np.random.default_rng(int(time.time()) & 0xFFFF)
    texts = [format_filter(four_attribute_filter(rng)) for _ in range(256)]
    t0 = time.perf_counter()
    b = FilterBatch.from_text(texts, None, BloomParams(m_bits=1024 + int(rng.integers(1, 999))))
    dt = (time.perf_counter() - t0) * 1e3
    print(f"cold text parse+compile+pack, 256 four-attribute filters: {dt:.2f} ms")
    assert b.is_cnf and dt < 200


def test_explicit_leaf_positions_are_kept():
    """A compiled filter's own leaf positions (bloom_eval_leaf's QueryBloom) win over
    hashing its (fid, value) placeholder."""
    from paper_2511_14881_b200.bloom import QueryBloom
    from paper_2511_14881_b200.filter_query import CompiledFilter, OpCode
    qb = QueryBloom((3, 700, 1023))
    b = FilterBatch.from_leaf(qb, BloomParams())
    assert b.host_leaf_pos[0].tolist() == [3, 700, 1023]
    cf = CompiledFilter(ops=((OpCode.PUSH_LEAF, 0),), leaves=((0, 0, qb),))
    assert_same(b, FilterBatch(**pack_py([cf], BloomParams())))
    with pytest.raises(ValueError):
        FilterBatch.from_leaf(QueryBloom((5, 2048)), BloomParams())
