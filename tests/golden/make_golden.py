"""Generate golden vectors by running the REAL reference package.

Run in the build container (where ``/root/reference`` exists)::

    python tests/golden/make_golden.py

It imports ``filtra`` from ``/root/reference/pkg/src`` (read-only), runs the
reference's own hot-path functions on seed-pinned inputs, and writes small
``.npz`` / ``.json`` fixtures next to this script. The fixtures are committed;
nothing on the GPU box reads ``/root/reference``.

Functions exercised (reference ``pkg/src/filtra``):
  bloom.hash_seed / hash_positions (bloom.py:65-88), build_bloom (114-144),
  bloom_eval_leaf (160-181), filter_query.compile_filter / eval_compiled
  (280-356), quantize.quantize_vector (72-76), ivf.build_ivf / probe_centroids /
  search_clusters / search (207-343), retrieval.codesigned_search (110-144),
  serve._reduce_topk (98-100), evaluation.brute_force_topk (45-69),
  retrieval.merge_candidates / retrieve (147-199), scoring (61-130),
  value_model (97-221).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _import_reference():
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(REF.parent / "tests"))
    import filtra  # noqa: F401
    return filtra


def expr_to_json(expr):
    from filtra.filter_query import And, Leaf, Not, Or
    if isinstance(expr, Leaf):
        return ["leaf", int(expr.feature_id), int(expr.value)]
    if isinstance(expr, Not):
        return ["not", expr_to_json(expr.child)]
    if isinstance(expr, And):
        return ["and", [expr_to_json(c) for c in expr.children]]
    if isinstance(expr, Or):
        return ["or", [expr_to_json(c) for c in expr.children]]
    raise TypeError(expr)


def random_expr(rng, depth=0, max_depth=3, n_features=5, n_values=5):
    """Same generator shape as the reference's tests/conftest.py:37-47."""
    from filtra.filter_query import And, Leaf, Not, Or
    if depth >= max_depth or rng.random() < 0.35:
        return Leaf(int(rng.integers(1, n_features + 1)), int(rng.integers(1, n_values + 1)))
    roll = rng.random()
    if roll < 0.18:
        return Not(random_expr(rng, depth + 1, max_depth, n_features, n_values))
    cls = And if roll < 0.6 else Or
    return cls(tuple(random_expr(rng, depth + 1, max_depth, n_features, n_values)
                     for _ in range(int(rng.integers(2, 4)))))


def four_attribute_expr(rng, sizes=(17, 17, 14, 11), cards=(50, 50, 40, 30)):
    """AND of four per-feature OR groups."""
    from filtra.filter_query import And, Leaf, Or
    groups = []
    for fid, (size, card) in enumerate(zip(sizes, cards), start=1):
        vals = rng.choice(card, size=min(size, card), replace=False)
        groups.append(Or(tuple(Leaf(fid, int(v)) for v in vals)))
    return And(tuple(groups))


def flat_pairs(slot_features):
    f, v, s = [], [], []
    for slot, pairs in enumerate(slot_features):
        for fid, val in pairs:
            f.append(fid)
            v.append(val)
            s.append(slot)
    return (np.array(f, dtype=np.uint64), np.array(v, dtype=np.uint64),
            np.array(s, dtype=np.int64))


def gen_hash(filtra):
    from filtra.bloom import BloomParams, hash_positions, hash_seed
    rng = np.random.default_rng(5)
    cases = [(1, 2, 1024, 5), (0, 0, 512, 7), (2**64 - 1, 2**63, 512, 7), (6, 9, 1024, 5),
             (1, 2, 1800, 5), (5, 6, 128, 1), (1, 1, 1 << 16, 8), (42, 42, 8, 2)]
    for _ in range(200):
        fid = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        val = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        m = int(rng.choice([8, 64, 100, 512, 1024, 1800, 4096]))
        k = int(rng.integers(1, 9))
        cases.append((fid, val, m, k))
    for fid in range(1, 7):
        for val in range(50):
            cases.append((fid, val, 1024, 5))
    out = []
    for fid, val, m, k in cases:
        out.append({"fid": str(fid), "value": str(val), "m_bits": m, "k_hashes": k,
                    "seed": str(hash_seed(fid, val)),
                    "positions": list(hash_positions(fid, val, BloomParams(m, k)).set_bits)})
    (OUT / "hash_kats.json").write_text(json.dumps(out))
    print("hash_kats.json", len(out))


def gen_bloom(filtra):
    from filtra.bloom import BloomParams, build_bloom
    rng = np.random.default_rng(11)
    arrays = {}
    specs = [(64, 3, 4, None), (128, 4, 30, None), (1024, 5, 300, 320), (512, 5, 1000, None),
             (1800, 5, 200, None), (8, 2, 70, 128)]
    for i, (m, k, n, n_slots) in enumerate(specs):
        sf = [[(int(rng.integers(0, 12)), int(rng.integers(0, 40)))
               for _ in range(int(rng.integers(0, 6)))] for _ in range(n)]
        if i == 0:
            sf = [[(1, 1)], [(2, 2)], [], [(1, 1), (3, 7)]]
        idx = build_bloom(sf, BloomParams(m_bits=m, k_hashes=k), n_slots=n_slots)
        f, v, s = flat_pairs(sf)
        arrays[f"c{i}_fid"], arrays[f"c{i}_val"], arrays[f"c{i}_slot"] = f, v, s
        arrays[f"c{i}_meta"] = np.array([m, k, idx.n_slots], dtype=np.int64)
        arrays[f"c{i}_planes"] = idx.planes
    arrays["n_cases"] = np.array([len(specs)])
    np.savez_compressed(OUT / "bloom_cases.npz", **arrays)
    print("bloom_cases.npz")


def gen_filter(filtra):
    from filtra import bitset
    from filtra.bloom import BloomParams, FilterStats, bloom_eval_leaf, build_bloom
    from filtra.filter_query import compile_filter, eval_compiled
    rng = np.random.default_rng(1234)
    params = BloomParams(m_bits=64, k_hashes=3)
    n = 320
    sf = [[(int(rng.integers(1, 6)), int(rng.integers(1, 6)))
           for _ in range(int(rng.integers(0, 6)))] for _ in range(n)]
    index = build_bloom(sf, params)
    valid_bool = rng.random(n) < 0.9
    valid = bitset.from_bool(valid_bool)
    exprs, fulls, ranged = [], [], []
    ranges = [(0, 64), (64, 192), (256, 320), (0, 320), (128, 130)]
    for t in range(80):
        expr = random_expr(rng)
        cf = compile_filter(expr, params)
        exprs.append({"expr": expr_to_json(expr),
                      "ops": [[int(o), int(a)] for o, a in cf.ops],
                      "leaves": [[str(f), str(v), list(qb.set_bits)] for f, v, qb in cf.leaves],
                      "max_stack": cf.max_stack_depth()})
        fulls.append(eval_compiled(cf, index, valid))
        ranged.append(np.concatenate([eval_compiled(cf, index, valid, slot_range=r)
                                      for r in ranges]))
    # leaf word-budget counters (ref tests/test_bloom.py:136-145)
    leaf_budget = []
    for fid, val in [(1, 1), (2, 3), (5, 5)]:
        qb = filtra.bloom.hash_positions(fid, val, params)
        st = FilterStats()
        m = bloom_eval_leaf(index, qb, word_range=(1, 4), stats=st)
        leaf_budget.append([fid, val, st.words_read] + [int(x) for x in m])
    f, v, s = flat_pairs(sf)
    np.savez_compressed(OUT / "filter_cases.npz", planes=index.planes, valid=valid,
                        fulls=np.stack(fulls), ranged=np.stack(ranged),
                        ranges=np.array(ranges), leaf_budget=np.array(leaf_budget, dtype=np.uint64),
                        fid=f, val=v, slot=s, meta=np.array([64, 3, n]))
    (OUT / "filter_exprs.json").write_text(json.dumps(exprs))
    print("filter_cases.npz", len(exprs))


def gen_quantize(filtra):
    from filtra.quantize import QuantParams, quantize_vector, quantize_value
    rng = np.random.default_rng(3)
    rows = []
    params = []
    for i in range(20):
        lo = float(rng.uniform(-3, 0))
        hi = lo + float(rng.uniform(0.01, 5))
        p = QuantParams(lo, hi)
        x = rng.uniform(lo - 0.5, hi + 0.5, size=64).astype(np.float32)
        # exact bucket midpoints exercise round-half-to-even
        mids = (np.arange(-128, 128, 8) + 128 + 0.5) / p.scale + lo
        x[:32] = mids.astype(np.float32)
        rows.append((x, quantize_vector(x, p)))
        params.append((lo, hi))
    kat = [quantize_value(v, QuantParams(-1.0, 1.0)) for v in (-1.0, 1.0, 0.0)]
    np.savez_compressed(OUT / "quantize_cases.npz", x=np.stack([r[0] for r in rows]),
                        q=np.stack([r[1] for r in rows]), params=np.array(params),
                        kat=np.array(kat))
    print("quantize_cases.npz")


def gen_scan(filtra):
    from conftest import catalog_from_rows, make_catalog
    from filtra import bitset
    from filtra.evaluation import brute_force_topk
    from filtra.filter_query import compile_filter
    from filtra.ivf import build_ivf, probe_centroids, search, search_clusters
    from filtra.quantize import quantize_vector
    from filtra.retrieval import codesigned_search
    from filtra.snapshot import PublishConfig, build_engine

    arrays = {}
    meta = []
    # (a) restricted scans with random masks (ref tests/test_ivf.py:242-255)
    cases = [(2000, 12, 20, 6), (400, 8, 5, 11), (1500, 12, 10, 20), (3000, 24, 30, 7)]
    for ci, (n, dim, ncl, seed) in enumerate(cases):
        cat = make_catalog(n_items=n, dim=dim, n_clusters=ncl, seed=seed)
        eng = build_engine(cat, PublishConfig(n_clusters=ncl, seed=seed))
        ivf = eng.ivf
        rng = np.random.default_rng(77 + ci)
        pre = f"s{ci}_"
        arrays[pre + "items_q"] = ivf.items_q.data
        arrays[pre + "valid"] = ivf.valid_mask
        arrays[pre + "item_ids"] = ivf.item_ids
        arrays[pre + "offsets"] = ivf.cluster_offsets
        arrays[pre + "centroids"] = ivf.centroids.vectors
        arrays[pre + "qp"] = np.array([ivf.items_q.params.global_min, ivf.items_q.params.global_max])
        arrays[pre + "planes"] = eng.bloom.planes
        arrays[pre + "emb"] = cat.embeddings
        qlist = []
        for t in range(12):
            qf = cat.embeddings[int(rng.integers(len(cat)))]
            nprobe = int(rng.integers(1, ncl + 1))
            qq = quantize_vector(qf, ivf.items_q.params)
            clusters = probe_centroids(ivf, qf, nprobe)
            kind = t % 3
            topk = [10, 50, 200, 1000][t % 4]
            entry = {"case": ci, "t": t, "nprobe": nprobe, "topk": topk, "kind": kind,
                     "clusters": clusters.tolist()}
            arrays[pre + f"q{t}_f"] = qf
            arrays[pre + f"q{t}_q"] = qq
            if kind == 0:      # random mask scan
                mask = bitset.from_bool(rng.random(ivf.n_slots) < 0.6)
                res = search_clusters(ivf, qq, clusters, mask, topk)
                arrays[pre + f"q{t}_mask"] = mask
            elif kind == 1:    # co-designed filtered search
                expr = random_expr(rng, n_features=6, n_values=10)
                cf = compile_filter(expr, eng.bloom.params)
                res = codesigned_search(ivf, eng.bloom, cf, qf, nprobe, topk)
                entry["expr"] = expr_to_json(expr)
            else:              # unfiltered search
                res = search(ivf, qf, nprobe, topk)
            arrays[pre + f"q{t}_ids"] = res.item_ids
            arrays[pre + f"q{t}_scores"] = res.scores
            qlist.append(entry)
        # exhaustive == int8 brute force (ref tests/test_ivf.py:287-294)
        qf = cat.embeddings[42]
        bf = brute_force_topk(cat, qf, 64, score="int8_dot")
        arrays[pre + "bf_q"] = qf
        arrays[pre + "bf_ids"] = bf.item_ids
        arrays[pre + "bf_scores"] = bf.scores
        meta.append({"n": n, "dim": dim, "n_clusters": ncl, "seed": seed, "queries": qlist})

    # (b) ties -> ascending item id (ref tests/test_ivf.py:312-320)
    rows = [(i, [1.0, 0.0], []) for i in (9, 3, 7, 1)]
    tcat = catalog_from_rows(rows, dim=2)
    tidx = build_ivf(tcat, k=1, seed=0)
    tres = search(tidx, np.array([1.0, 0.0], dtype=np.float32), nprobe=1, topk=4)
    arrays["tie_items_q"] = tidx.items_q.data
    arrays["tie_valid"] = tidx.valid_mask
    arrays["tie_item_ids"] = tidx.item_ids
    arrays["tie_offsets"] = tidx.cluster_offsets
    arrays["tie_qp"] = np.array([tidx.items_q.params.global_min, tidx.items_q.params.global_max])
    arrays["tie_ids"] = tres.item_ids
    arrays["tie_scores"] = tres.scores

    np.savez_compressed(OUT / "scan_cases.npz", **arrays)
    (OUT / "scan_meta.json").write_text(json.dumps(meta))
    print("scan_cases.npz", len(meta))


def gen_four_attr(filtra):
    """1 cluster, 20k items, the canonical 4-attribute filter + large k."""
    from filtra.bloom import BloomParams
    from filtra.catalog import default_features_spec, synth_catalog
    from filtra.filter_query import compile_filter
    from filtra.retrieval import codesigned_search
    from filtra.snapshot import PublishConfig, build_engine
    cat = synth_catalog(20000, 32, 20, default_features_spec(), seed=24, blob_std=0.08)
    eng = build_engine(cat, PublishConfig(n_clusters=1, seed=24, bloom=BloomParams()))
    rng = np.random.default_rng(7)
    arrays = {"items_q": eng.ivf.items_q.data, "valid": eng.ivf.valid_mask,
              "item_ids": eng.ivf.item_ids, "offsets": eng.ivf.cluster_offsets,
              "planes": eng.bloom.planes,
              "qp": np.array([eng.ivf.items_q.params.global_min, eng.ivf.items_q.params.global_max])}
    exprs = []
    for t in range(4):
        expr = four_attribute_expr(rng)
        cf = compile_filter(expr, eng.bloom.params)
        qf = cat.embeddings[int(rng.integers(len(cat)))]
        k = [1000, 3000, 50, 20000][t]
        res = codesigned_search(eng.ivf, eng.bloom, cf, qf, 1, k)
        arrays[f"q{t}_f"] = qf
        arrays[f"q{t}_ids"] = res.item_ids
        arrays[f"q{t}_scores"] = res.scores
        exprs.append({"expr": expr_to_json(expr), "k": k, "n_leaves": len(cf.leaves),
                      "n_ops": len(cf.ops)})
    np.savez_compressed(OUT / "four_attr.npz", **arrays)
    (OUT / "four_attr.json").write_text(json.dumps(exprs))
    print("four_attr.npz")


def gen_topk20000(filtra):
    """Acceptance #8 analogue: exhaustive top-20000 exact (ref tests/test_acceptance.py:250-258)."""
    from filtra.catalog import default_features_spec, synth_catalog
    from filtra.evaluation import brute_force_topk
    from filtra.ivf import build_ivf, search
    cat = synth_catalog(60000, 16, 100, default_features_spec()[:1], seed=24, blob_std=0.08)
    index = build_ivf(cat, k=4, seed=24, max_iters=4)
    q = cat.embeddings[4242]
    res = search(index, q, nprobe=index.n_clusters, topk=20000)
    oracle = brute_force_topk(cat, q, 20000, score="int8_dot")
    assert np.array_equal(res.item_ids, oracle.item_ids)
    np.savez_compressed(OUT / "topk20000.npz", items_q=index.items_q.data, valid=index.valid_mask,
                        item_ids=index.item_ids, offsets=index.cluster_offsets,
                        qp=np.array([index.items_q.params.global_min, index.items_q.params.global_max]),
                        q=q, ids=res.item_ids, scores=res.scores)
    print("topk20000.npz")


def gen_merge(filtra):
    from filtra.serve import _reduce_topk
    rng = np.random.default_rng(9)
    arrays = {}
    for c in range(5):
        s = int(rng.integers(1, 9))
        k = int(rng.integers(1, 300))
        ids, scores = [], []
        for sh in range(s):
            n = int(rng.integers(0, k + 1))
            i = rng.choice(100000, size=n, replace=False).astype(np.uint64) * np.uint64(8) + np.uint64(sh)
            sc = rng.integers(-50, 50, size=n).astype(np.int32)
            o = np.lexsort((i, -sc.astype(np.int64)))
            ids.append(i[o])
            scores.append(sc[o])
        cat_ids = np.concatenate(ids)
        cat_scores = np.concatenate(scores)
        rid, rsc = _reduce_topk(cat_ids, cat_scores, k)
        arrays[f"c{c}_ids"] = cat_ids
        arrays[f"c{c}_scores"] = cat_scores
        arrays[f"c{c}_lens"] = np.array([len(x) for x in ids])
        arrays[f"c{c}_k"] = np.array([k])
        arrays[f"c{c}_rids"] = rid
        arrays[f"c{c}_rscores"] = rsc
    arrays["n_cases"] = np.array([5])
    np.savez_compressed(OUT / "merge_cases.npz", **arrays)
    print("merge_cases.npz")


VM_SPECS = [
    None,  # per-request mean of the task scores (ref/value_model.py:216-221)
    {"op": "add", "args": [
        {"op": "mul", "args": [{"op": "const", "value": 0.5}, {"op": "task", "task": "t0"}]},
        {"op": "mul", "args": [{"op": "const", "value": 0.3}, {"op": "task", "task": "t1"}]},
        {"op": "clamp", "lo": -0.1, "hi": 0.4, "args": [{"op": "task", "task": "t2"}]},
        {"op": "if", "cond": {"left": {"op": "task", "task": "t3"}, "cmp": ">",
                              "right": {"op": "const", "value": 0.2}},
         "then": {"op": "max", "args": [{"op": "task", "task": "t0"},
                                        {"op": "task", "task": "t3"}]},
         "else": {"op": "div", "args": [{"op": "sub", "args": [{"op": "task", "task": "t1"},
                                                               {"op": "const", "value": 1.0}]},
                                        {"op": "const", "value": 4.0}]}}]},
]


def gen_retrieve(filtra):
    """Config-5 shape: multi-task requests (4 towers sharing one filter), exhaustive
    co-designed search per task, merge, identity-MoL (f64 dot) / MLP / MoL re-scoring,
    value-model aggregation, final (score desc, id asc) top-k
    (ref/retrieval.py:147-199, scoring.py:61-130, value_model.py:164-221)."""
    from filtra.catalog import default_features_spec, synth_catalog
    from filtra.retrieval import (MERGE_INTERSECTION, MERGE_UNION, RetrievalRequest,
                                  TaskQuery, merge_candidates, retrieve)
    from filtra.scoring import LinearHead, MlpScorer, MolScorer
    from filtra.snapshot import PublishConfig, build_engine
    from filtra.value_model import parse_value_model
    dim = 32
    cat = synth_catalog(6000, dim, 12, default_features_spec(), seed=31, blob_std=0.08)
    rng = np.random.default_rng(5)
    mlp = MlpScorer(hidden=((rng.standard_normal((16, 2 * dim)).astype(np.float32) * 0.2,
                             rng.standard_normal(16).astype(np.float32) * 0.1),),
                    heads={f"t{i}": LinearHead(rng.standard_normal(16).astype(np.float32),
                                               float(rng.standard_normal())) for i in range(4)})
    mol = MolScorer(components=tuple((rng.standard_normal((8, dim)).astype(np.float32) * 0.3,
                                      rng.standard_normal((8, dim)).astype(np.float32) * 0.3)
                                     for _ in range(3)),
                    gate_weight=rng.standard_normal((3, 2 * dim)).astype(np.float32) * 0.2,
                    gate_bias=rng.standard_normal(3).astype(np.float32) * 0.1)
    arrays, meta = {}, []
    base = build_engine(cat, PublishConfig(n_clusters=1, seed=31))
    arrays["items_q"] = base.ivf.items_q.data
    arrays["valid"] = base.ivf.valid_mask
    arrays["item_ids"] = base.ivf.item_ids
    arrays["offsets"] = base.ivf.cluster_offsets
    arrays["planes"] = base.bloom.planes
    arrays["qp"] = np.array([base.ivf.items_q.params.global_min,
                             base.ivf.items_q.params.global_max])
    arrays["cache_ids"] = base.cache.item_ids
    arrays["cache_vectors"] = base.cache.vectors
    arrays["mlp_w"] = mlp.hidden[0][0]
    arrays["mlp_b"] = mlp.hidden[0][1]
    for i in range(4):
        arrays[f"mlp_head{i}_w"] = mlp.heads[f"t{i}"].weight
        arrays[f"mlp_head{i}_b"] = np.array([mlp.heads[f"t{i}"].bias])
    for j, (u, it) in enumerate(mol.components):
        arrays[f"mol_u{j}"] = u
        arrays[f"mol_i{j}"] = it
    arrays["mol_gw"] = mol.gate_weight
    arrays["mol_gb"] = mol.gate_bias
    engines = {"dot": base}
    for name, sc in (("mlp", mlp), ("mol", mol)):
        e = build_engine(cat, PublishConfig(n_clusters=1, seed=31, scorer=sc))
        assert np.array_equal(e.ivf.items_q.data, base.ivf.items_q.data)
        engines[name] = e
    r = 0
    for scorer_name in ("dot", "mlp", "mol"):
        for vi, spec in enumerate(VM_SPECS):
            for merge in (MERGE_UNION, MERGE_INTERSECTION):
                if scorer_name != "dot" and merge == MERGE_INTERSECTION:
                    continue
                expr = four_attribute_expr(rng)
                tasks = tuple(TaskQuery(f"t{i}", cat.embeddings[int(rng.integers(len(cat)))])
                              for i in range(4))
                vm = parse_value_model(spec) if spec is not None else None
                req = RetrievalRequest(tasks=tasks, filter=expr, nprobe=1, k0=300, topk=100,
                                       merge=merge, value_model=vm)
                res = retrieve(engines[scorer_name], req)
                pre = f"r{r}_"
                arrays[pre + "users"] = np.stack([t.user_embedding for t in tasks])
                arrays[pre + "ids"] = np.array([it.item_id for it in res.items], dtype=np.uint64)
                arrays[pre + "scores"] = np.array([it.score for it in res.items])
                arrays[pre + "task_scores"] = np.array(
                    [[it.task_scores[f"t{i}"] for i in range(4)] for it in res.items])
                meta.append({"r": r, "scorer": scorer_name, "vm": spec, "merge": merge,
                             "expr": expr_to_json(expr), "k0": 300, "topk": 100})
                r += 1
    # merge_candidates algebra
    for c in range(4):
        lists = [np.sort(rng.choice(500, size=int(rng.integers(0, 80)), replace=False)).astype(np.uint64)
                 for _ in range(int(rng.integers(1, 5)))]
        for li, x in enumerate(lists):
            arrays[f"m{c}_l{li}"] = x
        arrays[f"m{c}_union"] = merge_candidates(lists, MERGE_UNION)
        arrays[f"m{c}_inter"] = merge_candidates(lists, MERGE_INTERSECTION)
        arrays[f"m{c}_n"] = np.array([len(lists)])
    np.savez_compressed(OUT / "retrieve_cases.npz", **arrays)
    (OUT / "retrieve_meta.json").write_text(json.dumps(meta))
    print("retrieve_cases.npz", len(meta))


def gen_snapshot(filtra):
    """A reference-published FLTRSNP1 file (ref/snapshot.py:157-174) plus its describe()
    and, for two multi-task requests over all clusters, the reference retrieve() output."""
    from filtra.catalog import default_features_spec, synth_catalog
    from filtra.retrieval import RetrievalRequest, TaskQuery, retrieve
    from filtra.snapshot import PublishConfig, describe, load, publish
    cat = synth_catalog(3000, 32, 12, default_features_spec(), seed=44, blob_std=0.08)
    vm = {"op": "add", "args": [{"op": "task", "task": "a"},
                                {"op": "mul", "args": [{"op": "const", "value": 0.5},
                                                       {"op": "task", "task": "b"}]}]}
    path = OUT / "snapshot_small.fsnap"
    publish(cat, path, version=7, config=PublishConfig(n_clusters=8, seed=44, value_model=vm))
    engine = load(path)
    rng = np.random.default_rng(12)
    out = {"describe": describe(path), "requests": []}
    for r in range(2):
        expr = four_attribute_expr(rng, sizes=(20, 20, 16, 12))
        tasks = [cat.embeddings[int(rng.integers(len(cat)))] for _ in range(2)]
        req = RetrievalRequest(tasks=(TaskQuery("a", tasks[0]), TaskQuery("b", tasks[1])),
                               filter=expr, nprobe=8, k0=200, topk=50)
        res = retrieve(engine, req)
        out["requests"].append({"expr": expr_to_json(expr),
                                "users": [t.tolist() for t in tasks],
                                "ids": [int(it.item_id) for it in res.items],
                                "scores": [float(it.score).hex() for it in res.items]})
    (OUT / "snapshot_small.json").write_text(json.dumps(out))
    print("snapshot_small.fsnap", path.stat().st_size)


def _blobs(n_per=50, dim=4, gap=10.0, seed=0):
    """The reference's tests/test_ivf.py:14-18 data shape."""
    rng = np.random.default_rng(seed)
    return np.vstack([rng.standard_normal((n_per, dim)) * 0.1,
                      rng.standard_normal((n_per, dim)) * 0.1 + gap])


def gen_kmeans(filtra):
    """KMeans++ seeding, Lloyd and the build_ivf layout (ref ivf.py:76-258)."""
    from filtra.catalog import default_features_spec, synth_catalog
    from filtra.ivf import build_ivf, kmeans_pp_init, kmeans_train
    rng = np.random.default_rng(77)
    pp = {
        "normal128": (rng.standard_normal((1500, 128)), 40, 3),
        "unit_f32": (None, 30, 11),
        "blobs": (_blobs(), 5, 9),
        "dups": (np.repeat(_blobs(n_per=10), 10, axis=0), 8, 21),
        "zero_mass": (np.repeat(rng.standard_normal((3, 8)), 5, axis=0), 6, 4),
        "k_eq_n": (np.arange(12, dtype=np.float64).reshape(6, 2), 6, 5),
        "dim13": (rng.standard_normal((500, 13)), 20, 6),
        "dim200": (rng.standard_normal((300, 200)), 10, 7),
    }
    e = rng.standard_normal((2000, 64)).astype(np.float32)
    pp["unit_f32"] = ((e / np.linalg.norm(e, axis=1, keepdims=True)).astype(np.float32), 30, 11)
    arrays, meta = {}, {"pp": [], "train": []}
    for name, (x, k, seed) in pp.items():
        arrays[f"pp_{name}_x"] = x
        arrays[f"pp_{name}_c"] = kmeans_pp_init(x, k, seed).vectors
        meta["pp"].append({"name": name, "k": k, "seed": seed})
    centres4 = np.array([[0, 0], [0, 8], [8, 0], [8, 8]], dtype=np.float64)
    r2 = np.random.default_rng(2)
    train = {
        "four_blobs": (np.vstack([r2.standard_normal((100, 2)) * 0.5 + c for c in centres4]),
                       4, 0, 25, 1e-4),
        "two_blobs6": (_blobs(n_per=100, dim=6, gap=3.0, seed=8), 5, 13, 12, 0.0),
        "dups": (np.repeat(_blobs(n_per=10), 10, axis=0), 8, 21, 25, 1e-4),
        "normal16": (rng.standard_normal((2000, 16)), 12, 2, 25, 1e-4),
    }
    for name, (x, k, seed, iters, tol) in train.items():
        c, a = kmeans_train(x, k, max_iters=iters, tol=tol, seed=seed)
        arrays[f"tr_{name}_x"] = x
        arrays[f"tr_{name}_c"] = c.vectors
        arrays[f"tr_{name}_a"] = a
        meta["train"].append({"name": name, "k": k, "seed": seed, "max_iters": iters, "tol": tol})
    cat = synth_catalog(3000, 16, 30, default_features_spec()[:2], seed=5, blob_std=0.08)
    index = build_ivf(cat, k=7, seed=3)
    arrays.update(ivf_emb=cat.embeddings, ivf_ids=cat.item_ids, ivf_perm=index.perm,
                  ivf_inv_perm=index.inv_perm, ivf_offsets=index.cluster_offsets,
                  ivf_items_q=index.items_q.data, ivf_valid=index.valid_mask,
                  ivf_slot_ids=index.item_ids, ivf_centroids=index.centroids.vectors,
                  ivf_qp=np.array([index.items_q.params.global_min, index.items_q.params.global_max]))
    meta["ivf"] = {"k": 7, "seed": 3}
    np.savez_compressed(OUT / "kmeans_cases.npz", **arrays)
    (OUT / "kmeans_meta.json").write_text(json.dumps(meta))
    print("kmeans_cases.npz")


def main():
    filtra = _import_reference()
    gen_hash(filtra)
    gen_bloom(filtra)
    gen_filter(filtra)
    gen_quantize(filtra)
    gen_scan(filtra)
    gen_four_attr(filtra)
    gen_topk20000(filtra)
    gen_merge(filtra)
    gen_retrieve(filtra)
    gen_snapshot(filtra)
    gen_kmeans(filtra)


if __name__ == "__main__":
    main()
