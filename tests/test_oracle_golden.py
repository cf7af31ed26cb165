"""Pin the CPU oracle (oracle/filtra_oracle.py) against vectors produced by the real
reference package (tests/golden/make_golden.py). CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import json_to_oracle_expr, load_json, load_npz
from oracle import filtra_oracle as orc


def test_hash_kats_match_reference():
    for case in load_json("hash_kats.json"):
        fid, val = int(case["fid"]), int(case["value"])
        assert orc.fnv1a64_pair(fid, val) == int(case["seed"])
        got = orc.hash_positions(fid, val, case["m_bits"], case["k_hashes"])
        assert list(got) == case["positions"], case


def test_hash_vectorised_matches_scalar():
    cases = load_json("hash_kats.json")
    by_mk: dict = {}
    for c in cases:
        by_mk.setdefault((c["m_bits"], c["k_hashes"]), []).append(c)
    for (m, k), group in by_mk.items():
        fids = np.array([int(c["fid"]) for c in group], dtype=np.uint64)
        vals = np.array([int(c["value"]) for c in group], dtype=np.uint64)
        pos = orc.hash_positions_np(fids, vals, m, k)
        for row, c in zip(pos, group):
            assert [int(p) for p in row if p >= 0] == c["positions"]


def test_survey_kats():
    # SURVEY.md §8(c) known answers generated from the reference
    assert orc.fnv1a64_pair(1, 2) == 0x7717980363C8E066
    assert orc.hash_positions(1, 2, 1024, 5) == (199, 486, 770, 853, 906)
    assert orc.hash_positions(2**64 - 1, 2**63, 512, 7) == (20, 172, 278, 289, 347, 354, 478)
    assert orc.hash_positions(1, 2, 1800, 5) == (733, 778, 962, 1023, 1342)


def test_bloom_build_matches_reference():
    z = load_npz("bloom_cases.npz")
    for i in range(int(z["n_cases"][0])):
        m, k, n_slots = (int(x) for x in z[f"c{i}_meta"])
        planes = orc.build_bloom_pairs(z[f"c{i}_fid"], z[f"c{i}_val"], z[f"c{i}_slot"],
                                       n_slots, m, k)
        assert np.array_equal(planes, z[f"c{i}_planes"]), i
    # SURVEY KAT: nonzero words of the 4-slot M=64 K=3 case
    p = z["c0_planes"]
    nz = {int(r): int(p[r, 0]) for r in np.flatnonzero(p[:, 0])}
    assert nz == {2: 0x2, 11: 0x8, 19: 0x8, 21: 0x9, 26: 0x2, 33: 0x9, 44: 0x9, 54: 0xA}


def test_eval_compiled_matches_reference():
    z = load_npz("filter_cases.npz")
    exprs = load_json("filter_exprs.json")
    m, k, n = (int(x) for x in z["meta"])
    ranges = [tuple(int(v) for v in r) for r in z["ranges"]]
    for i, e in enumerate(exprs):
        ops, leaves = orc.compile_expr(json_to_oracle_expr(e["expr"]), m, k)
        assert [list(o) for o in ops] == e["ops"]
        assert [[str(f), str(v), list(p)] for f, v, p in leaves] == e["leaves"]
        full = orc.eval_compiled(ops, leaves, z["planes"], z["valid"])
        assert np.array_equal(full, z["fulls"][i])
        ranged = np.concatenate([orc.eval_compiled(ops, leaves, z["planes"], z["valid"], r)
                                 for r in ranges])
        assert np.array_equal(ranged, z["ranged"][i])
    with pytest.raises(ValueError):
        orc.eval_compiled([(0, 0)], [(1, 1, (1,))], z["planes"], z["valid"], (10, 64))


def test_quantize_matches_reference():
    z = load_npz("quantize_cases.npz")
    for x, q, (lo, hi) in zip(z["x"], z["q"], z["params"]):
        assert np.array_equal(orc.quantize(x, lo, hi), q)
    assert list(z["kat"]) == [-128, 127, 0]


def test_scan_cases_match_reference():
    z = load_npz("scan_cases.npz")
    meta = load_json("scan_meta.json")
    for ci, m in enumerate(meta):
        pre = f"s{ci}_"
        items_q, valid, ids, offs = (z[pre + "items_q"], z[pre + "valid"], z[pre + "item_ids"],
                                     z[pre + "offsets"])
        planes = z[pre + "planes"]
        lo, hi = z[pre + "qp"]
        for q in m["queries"]:
            t = q["t"]
            qq = z[pre + f"q{t}_q"]
            assert np.array_equal(orc.quantize(z[pre + f"q{t}_f"], lo, hi), qq)
            probed = orc.probe_centroids(z[pre + "centroids"], z[pre + f"q{t}_f"], q["nprobe"])
            assert probed.tolist() == q["clusters"]
            if q["kind"] == 0:
                res = orc.search_clusters(items_q, valid, ids, offs, qq, q["clusters"],
                                          z[pre + f"q{t}_mask"], q["topk"])
            elif q["kind"] == 1:
                prog = orc.compile_expr(json_to_oracle_expr(q["expr"]), 1024, 5)
                res = orc.codesigned_search(items_q, valid, ids, offs, planes, prog, qq,
                                            q["clusters"], q["topk"])
            else:
                res = orc.search_clusters(items_q, valid, ids, offs, qq, q["clusters"], None,
                                          q["topk"])
            assert np.array_equal(res.item_ids, z[pre + f"q{t}_ids"])
            assert np.array_equal(res.scores, z[pre + f"q{t}_scores"])
        bf = orc.brute_force_int8(items_q, ids, orc.quantize(z[pre + "bf_q"], lo, hi), 64,
                                  keep=orc.to_bool(valid, items_q.shape[0]))
        assert np.array_equal(bf.item_ids, z[pre + "bf_ids"])
        assert np.array_equal(bf.scores, z[pre + "bf_scores"])


def test_ties_ascending_id():
    z = load_npz("scan_cases.npz")
    lo, hi = z["tie_qp"]
    qq = orc.quantize(np.array([1.0, 0.0], dtype=np.float32), lo, hi)
    res = orc.search_clusters(z["tie_items_q"], z["tie_valid"], z["tie_item_ids"],
                              z["tie_offsets"], qq, [0], None, 4)
    assert res.item_ids.tolist() == [1, 3, 7, 9] == z["tie_ids"].tolist()


def test_four_attribute_and_topk20000():
    z = load_npz("four_attr.npz")
    cases = load_json("four_attr.json")
    lo, hi = z["qp"]
    for t, c in enumerate(cases):
        prog = orc.compile_expr(json_to_oracle_expr(c["expr"]), 1024, 5)
        assert len(prog[1]) == c["n_leaves"] and len(prog[0]) == c["n_ops"]
        res = orc.codesigned_search(z["items_q"], z["valid"], z["item_ids"], z["offsets"],
                                    z["planes"], prog, orc.quantize(z[f"q{t}_f"], lo, hi),
                                    [0], c["k"])
        assert np.array_equal(res.item_ids, z[f"q{t}_ids"])
        assert np.array_equal(res.scores, z[f"q{t}_scores"])
    y = load_npz("topk20000.npz")
    lo, hi = y["qp"]
    res = orc.search_clusters(y["items_q"], y["valid"], y["item_ids"], y["offsets"],
                              orc.quantize(y["q"], lo, hi), range(len(y["offsets"])), None, 20000)
    assert np.array_equal(res.item_ids, y["ids"]) and np.array_equal(res.scores, y["scores"])


def test_reduce_topk_matches_reference():
    z = load_npz("merge_cases.npz")
    for c in range(int(z["n_cases"][0])):
        ids, sc = orc.reduce_topk(z[f"c{c}_ids"], z[f"c{c}_scores"], int(z[f"c{c}_k"][0]))
        assert np.array_equal(ids, z[f"c{c}_rids"]) and np.array_equal(sc, z[f"c{c}_rscores"])


def _retrieve_fixture():
    z = load_npz("retrieve_cases.npz")
    meta = load_json("retrieve_meta.json")
    return z, meta


def oracle_score_fn(z, scorer):
    if scorer == "dot":
        return lambda t, u, v: orc.score_dot(u, v)
    if scorer == "mlp":
        hidden = [(z["mlp_w"], z["mlp_b"])]
        heads = {f"t{i}": (z[f"mlp_head{i}_w"], float(z[f"mlp_head{i}_b"][0])) for i in range(4)}
        return lambda t, u, v: orc.score_mlp(hidden, heads, t, u, v)
    comps = [(z[f"mol_u{j}"], z[f"mol_i{j}"]) for j in range(3)]
    return lambda t, u, v: orc.score_mol(comps, z["mol_gw"], z["mol_gb"], u, v)


def test_oracle_retrieve_matches_reference():
    """Config-5 pipeline: per-task exhaustive co-designed search, merge, re-score, value
    model, final top-k -- the oracle reproduces the reference's ids and floats exactly."""
    z, meta = _retrieve_fixture()
    items = z["items_q"]
    qp = (float(z["qp"][0]), float(z["qp"][1]))
    for m in meta:
        pre = f"r{m['r']}_"
        users = z[pre + "users"]
        prog = orc.compile_expr(json_to_oracle_expr(m["expr"]), 1024, 5)
        per_task = []
        for j in range(4):
            qq = orc.quantize(users[j], *qp)
            res = orc.codesigned_search(items, z["valid"], z["item_ids"], z["offsets"], z["planes"],
                                        prog, qq, [0], m["k0"])
            per_task.append(res.item_ids)
        ids, final, ts = orc.retrieve(per_task, m["merge"], z["cache_ids"], z["cache_vectors"],
                                      oracle_score_fn(z, m["scorer"]), [f"t{i}" for i in range(4)],
                                      users, m["vm"], m["topk"])
        assert np.array_equal(ids, z[pre + "ids"]), m["r"]
        assert np.array_equal(final, z[pre + "scores"]), m["r"]
        assert np.array_equal(ts, z[pre + "task_scores"]), m["r"]


def test_oracle_merge_candidates_matches_reference():
    z = load_npz("retrieve_cases.npz")
    for c in range(4):
        lists = [z[f"m{c}_l{i}"] for i in range(int(z[f"m{c}_n"][0]))]
        assert np.array_equal(orc.merge_candidates(lists, "union"), z[f"m{c}_union"])
        assert np.array_equal(orc.merge_candidates(lists, "intersection"), z[f"m{c}_inter"])


def test_oracle_kmeans_matches_reference():
    """KMeans++ seeding, Lloyd and the IVF slot layout (ref ivf.py:76-258)."""
    z = load_npz("kmeans_cases.npz")
    meta = load_json("kmeans_meta.json")
    for m in meta["pp"]:
        x = z[f"pp_{m['name']}_x"]
        got = np.asarray(x, dtype=np.float64)[orc.kmeans_pp_init(x, m["k"], m["seed"])]
        assert np.array_equal(got.astype(np.float32), z[f"pp_{m['name']}_c"]), m["name"]
    for m in meta["train"]:
        c, a = orc.kmeans_train(z[f"tr_{m['name']}_x"], m["k"], m["max_iters"], m["tol"], m["seed"])
        assert np.array_equal(c, z[f"tr_{m['name']}_c"]), m["name"]
        assert np.array_equal(a, z[f"tr_{m['name']}_a"]), m["name"]
    k, seed = meta["ivf"]["k"], meta["ivf"]["seed"]
    c, a = orc.kmeans_train(z["ivf_emb"], k, seed=seed)
    assert np.array_equal(c, z["ivf_centroids"])
    perm, offs = orc.ivf_layout(a, z["ivf_ids"], k)
    assert np.array_equal(perm, z["ivf_perm"])
    assert np.array_equal(offs, z["ivf_offsets"])
