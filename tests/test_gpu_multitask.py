"""Config 5 on the GPU: multi-task requests (4 towers sharing one filter) through the
batched filtered top-k, device merge, re-scoring, value model and final top-k -- against
golden outputs of the reference's ``retrieval.retrieve`` (tests/golden/retrieve_*), and
against the CPU oracle on a larger batched workload."""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from conftest import json_to_expr, load_json, load_npz
from oracle import filtra_oracle as orc

pytestmark = pytest.mark.gpu
TASKS = [f"t{i}" for i in range(4)]


@pytest.fixture(scope="module")
def golden(cuda):
    import paper_2511_14881_b200 as fb
    z = load_npz("retrieve_cases.npz")
    meta = load_json("retrieve_meta.json")
    bloom = fb.BloomIndex(fb.BloomParams(), z["planes"], z["items_q"].shape[0])
    dix = fb.DeviceIndex.from_arrays(z["items_q"], z["valid"], z["item_ids"], bloom=bloom,
                                     qp=fb.QuantParams(float(z["qp"][0]), float(z["qp"][1])))
    cache = fb.DeviceCache(z["cache_ids"], z["cache_vectors"])
    return fb, z, meta, dix, cache


def ref_scorer(z, kind):
    if kind == "mlp":
        heads = {f"t{i}": SimpleNamespace(weight=z[f"mlp_head{i}_w"], bias=float(z[f"mlp_head{i}_b"][0]))
                 for i in range(4)}
        return SimpleNamespace(hidden=[(z["mlp_w"], z["mlp_b"])], heads=heads, shared_head=None)
    if kind == "mol":
        return SimpleNamespace(components=[(z[f"mol_u{j}"], z[f"mol_i{j}"]) for j in range(3)],
                               gate_weight=z["mol_gw"], gate_bias=z["mol_gb"])
    eye = np.eye(z["cache_vectors"].shape[1], dtype=np.float32)
    return SimpleNamespace(components=[(eye, eye)], gate_weight=np.zeros((1, 2 * eye.shape[0]), np.float32),
                           gate_bias=np.zeros(1, np.float32))


def assert_close_order(got_ids, got_scores, want_ids, want_scores):
    """Float scorers: scores within 1e-5 relative position by position; ids equal except
    inside runs of near-tied scores (ordering by float64 noise)."""
    assert len(got_ids) == len(want_ids)
    tol = 1e-5 * np.maximum(np.abs(want_scores), 1e-3)
    assert np.all(np.abs(got_scores - want_scores) <= tol)
    for i in range(len(want_ids)):
        if got_ids[i] != want_ids[i]:
            near = np.abs(want_scores - want_scores[i]) <= 1e-9 * max(abs(want_scores[i]), 1e-3)
            assert got_ids[i] in set(want_ids[near].tolist()), i


def test_multitask_op_matches_reference_retrieve(golden):
    fb, z, meta, dix, cache = golden
    for m in meta:
        pre = f"r{m['r']}_"
        scorer = fb.DeviceScorer.from_reference(ref_scorer(z, m["scorer"]))
        assert scorer.kind == m["scorer"]
        op = fb.MultiTaskOp(dix, cache, 1, TASKS, m["k0"], m["topk"], merge=m["merge"],
                            scorer=scorer, value_model=m["vm"])
        cf = fb.compile_filter(json_to_expr(m["expr"]), fb.BloomParams())
        users = torch.as_tensor(z[pre + "users"][None], device="cuda")
        out = op(users, op.pack_filters([cf]).to_device())
        torch.cuda.synchronize()
        ids, scores, ts = out.host(0)
        want_ids, want_scores, want_ts = z[pre + "ids"], z[pre + "scores"], z[pre + "task_scores"]
        if m["scorer"] == "dot":  # exact: pairwise-order float64 dots, IEEE value model
            assert np.array_equal(ids, want_ids), m["r"]
            assert np.array_equal(scores, want_scores), m["r"]
            assert np.array_equal(ts, want_ts), m["r"]
        else:
            assert_close_order(ids, scores, want_ids, want_scores)
            tol = 1e-5 * np.maximum(np.abs(want_ts), 1e-3)
            same = ids == want_ids
            assert np.all(np.abs(ts[same] - want_ts[same]) <= tol[same])


def test_retrieve_drop_in_matches_reference(golden):
    """``retrieve(engine, req)`` with a reference-shaped engine (duck-typed) and request."""
    fb, z, meta, dix, cache = golden
    ivf = SimpleNamespace(items_q=SimpleNamespace(data=z["items_q"],
                                                  params=fb.QuantParams(float(z["qp"][0]), float(z["qp"][1]))),
                          valid_mask=z["valid"], item_ids=z["item_ids"],
                          cluster_offsets=z["offsets"], centroids=None,
                          n_slots=z["items_q"].shape[0], dim=z["items_q"].shape[1])
    bloom = fb.BloomIndex(fb.BloomParams(), z["planes"], z["items_q"].shape[0])
    ref_cache = SimpleNamespace(item_ids=z["cache_ids"], vectors=z["cache_vectors"])
    for m in meta:
        if m["scorer"] != "dot":
            continue
        pre = f"r{m['r']}_"
        engine = SimpleNamespace(ivf=ivf, bloom=bloom, cache=ref_cache, scorer=ref_scorer(z, "dot"),
                                 default_value_model=None,
                                 compile=lambda e: fb.compile_filter(e, fb.BloomParams()))
        tasks = tuple(SimpleNamespace(task_name=t, user_embedding=z[pre + "users"][j])
                      for j, t in enumerate(TASKS))
        req = SimpleNamespace(tasks=tasks, filter=json_to_expr(m["expr"]), nprobe=1, k0=m["k0"],
                              topk=m["topk"], merge=m["merge"], value_model=m["vm"])
        res = fb.retrieve(engine, req)
        assert [it.item_id for it in res.items] == [int(x) for x in z[pre + "ids"]], m["r"]
        assert np.array_equal(np.array([it.score for it in res.items]), z[pre + "scores"])


def test_multitask_batched_vs_oracle(cuda):
    """16 requests x 4 towers over 60k items at dim 128 (tensor-core scan), the
    4-attribute filter per request, k0=500, topk=100, a formula value model."""
    import paper_2511_14881_b200 as fb
    from paper_2511_14881_b200 import _device, workload
    B, T, k0, topk = 16, 4, 500, 100
    wl = workload.make_workload(60_000, B * T, dim=128, seed=41)
    idx = wl.index
    rng = np.random.default_rng(3)
    vecs = rng.standard_normal((idx.n_slots, 128)).astype(np.float32)
    cache = fb.DeviceCache(_device.u64_host(idx.item_ids)[: idx.n_slots], vecs)
    spec = {"op": "sub", "args": [{"op": "max", "args": [{"op": "task", "task": "t0"},
                                                          {"op": "task", "task": "t2"}]},
                                  {"op": "mul", "args": [{"op": "const", "value": 0.25},
                                                         {"op": "task", "task": "t3"}]}]}
    op = fb.MultiTaskOp(idx, cache, B, TASKS, k0, topk, value_model=spec)
    filters = [wl.filters[b * T] for b in range(B)]
    users = wl.queries.view(B, T, -1)
    out = op(users, op.pack_filters(filters).to_device())
    torch.cuda.synchronize()
    items = idx.items.cpu().numpy()[:, :128]
    valid = _device.u64_host(idx.valid)
    ids_all = _device.u64_host(idx.item_ids)
    offs = np.array([[0, idx.n_slots]])
    qq = wl.queries_q.cpu().numpy()[:, :128]
    uf = users.cpu().numpy()
    for b in range(B):
        cf = filters[b]
        prog = ([(int(o), int(a)) for o, a in cf.ops], [(f, v, q.set_bits) for f, v, q in cf.leaves])
        per_task = [orc.codesigned_search(items, valid, ids_all, offs, idx.bloom.planes, prog,
                                          qq[b * T + t], [0], k0).item_ids for t in range(T)]
        want = orc.retrieve(per_task, "union", ids_all[: idx.n_slots], vecs,
                            lambda t, u, v: orc.score_dot(u, v), TASKS, uf[b], spec, topk)
        ids, scores, ts = out.host(b)
        assert np.array_equal(ids, want[0]), b
        assert np.array_equal(scores, want[1]), b
        assert np.array_equal(ts, want[2]), b


def test_multitask_missing_cache_item_raises(cuda):
    """A merged candidate absent from the embedding cache raises MissingItem (reference
    EmbeddingCache.batch, scoring.py:45-52), on the rank-table path."""
    import paper_2511_14881_b200 as fb
    from paper_2511_14881_b200 import _device, workload
    from paper_2511_14881_b200.errors import MissingItem
    B, T = 2, 4
    wl = workload.make_workload(20_000, B * T, dim=128, seed=43, filtered=False)
    idx = wl.index
    ids = _device.u64_host(idx.item_ids)[: idx.n_slots]
    vecs = np.random.default_rng(1).standard_normal((idx.n_slots, 128)).astype(np.float32)
    op = fb.MultiTaskOp(idx, fb.DeviceCache(ids, vecs), B, TASKS, 50, 10)
    out = op(wl.queries.view(B, T, -1), None)
    torch.cuda.synchronize()
    victim = out.host(0)[0][0]
    keep = ids != victim
    op2 = fb.MultiTaskOp(idx, fb.DeviceCache(ids[keep], vecs[keep]), B, TASKS, 50, 10)
    with pytest.raises(MissingItem):
        op2(wl.queries.view(B, T, -1), None)


def test_retrieve_graph_path_equals_eager(golden, monkeypatch):
    """The CUDA-graph single-request path (fastpath.py) returns exactly what the
    step-by-step path returns -- ids, scores, task scores, scan and filter counters --
    for every golden request shape, and it is the path taken."""
    from paper_2511_14881_b200 import fastpath
    fb, z, meta, dix, cache = golden
    ivf = SimpleNamespace(items_q=SimpleNamespace(data=z["items_q"],
                                                  params=fb.QuantParams(float(z["qp"][0]), float(z["qp"][1]))),
                          valid_mask=z["valid"], item_ids=z["item_ids"],
                          cluster_offsets=z["offsets"], centroids=None,
                          n_slots=z["items_q"].shape[0], dim=z["items_q"].shape[1])
    bloom = fb.BloomIndex(fb.BloomParams(), z["planes"], z["items_q"].shape[0])
    ref_cache = SimpleNamespace(item_ids=z["cache_ids"], vectors=z["cache_vectors"])
    monkeypatch.setenv("FB_GRAPH_STRICT", "1")
    for m in meta:
        pre = f"r{m['r']}_"
        engine = SimpleNamespace(ivf=ivf, bloom=bloom, cache=ref_cache,
                                 scorer=ref_scorer(z, m["scorer"]), default_value_model=None,
                                 compile=lambda e: fb.compile_filter(e, fb.BloomParams()))
        tasks = tuple(SimpleNamespace(task_name=t, user_embedding=z[pre + "users"][j])
                      for j, t in enumerate(TASKS))
        req = SimpleNamespace(tasks=tasks, filter=json_to_expr(m["expr"]), nprobe=1, k0=m["k0"],
                              topk=m["topk"], merge=m["merge"], value_model=m["vm"])
        before = fastpath.graph_count()
        fast = fb.retrieve(engine, req)
        assert fastpath.graph_count() >= before and fastpath.graph_count() > 0
        monkeypatch.setenv("FB_EAGER_B1", "1")
        slow = fb.retrieve(engine, req)
        monkeypatch.delenv("FB_EAGER_B1")
        assert [(i.item_id, i.score, i.task_scores) for i in fast.items] == \
            [(i.item_id, i.score, i.task_scores) for i in slow.items], m["r"]
        assert vars(fast.scan) == vars(slow.scan) and vars(fast.filter_stats) == vars(slow.filter_stats)


@pytest.mark.gpu
@pytest.mark.parametrize("C,topk", [(20000, 5000), (37, 5), (1000, 1000), (24576, 8192)])
def test_final_topk_kernel_numpy_order(C, topk):
    """fb_final_topk == np.lexsort((positions, -final))[:topk] per request (ref
    retrieval.py:190) on values with heavy ties, NaN, +-0.0, +-inf and short counts."""
    import numpy as np
    import torch

    from paper_2511_14881_b200.overarch import final_topk_device
    rng = np.random.default_rng(C + topk)
    B = 6
    vals = rng.integers(-50, 50, size=(B, C)).astype(np.float64) / 8.0
    specials = np.array([np.nan, 0.0, -0.0, np.inf, -np.inf])
    hit = rng.random((B, C)) < 0.02
    vals[hit] = specials[rng.integers(0, len(specials), size=int(hit.sum()))]
    counts = np.array([C, C - 1, topk // 2, 0, 1, max(1, C // 3)], dtype=np.int32)
    order, n = final_topk_device(torch.as_tensor(vals, device="cuda"),
                                 torch.as_tensor(counts, device="cuda"), topk)
    order, n = order.cpu().numpy(), n.cpu().numpy()
    for b in range(B):
        m = int(counts[b])
        want = np.lexsort((np.arange(m), -vals[b, :m]))[:topk]
        assert n[b] == len(want)
        assert np.array_equal(order[b, : n[b]], want), f"request {b}"


@pytest.mark.gpu
def test_value_model_kernel_matches_numpy():
    """fb_value_model == the reference's NumPy evaluation (ref value_model.py:75-124)
    bit for bit: n-ary folds, sub/div, min/max with NaN, clip, if with both branches,
    and the zero-divisor flag only for valid candidates."""
    import numpy as np
    import torch

    from paper_2511_14881_b200.overarch import value_model_kernel
    rng = np.random.default_rng(11)
    B, T, C = 3, 3, 1000
    ts = rng.standard_normal((B, T, C))
    ts[rng.random((B, T, C)) < 0.01] = np.nan
    ts[rng.random((B, T, C)) < 0.01] = 0.0
    names = ["a", "b", "c"]
    t = {"op": "task"}
    A, Bt, Ct = ({**t, "task": n} for n in names)
    specs = [
        {"op": "mul", "args": [{"op": "const", "value": 1 / 3}, {"op": "add", "args": [A, Bt, Ct]}]},
        {"op": "sub", "args": [{"op": "max", "args": [A, Bt, {"op": "const", "value": 0.25}]},
                               {"op": "min", "args": [Ct, A]}]},
        {"op": "clamp", "args": [{"op": "add", "args": [A, Ct]}], "lo": -0.5, "hi": 0.75},
        {"op": "if", "cond": {"left": A, "cmp": ">=", "right": Bt},
         "then": {"op": "mul", "args": [A, {"op": "const", "value": 3.0}]}, "else": Ct},
        {"op": "div", "args": [A, {"op": "add", "args": [Bt, {"op": "const", "value": 10.0}]}]},
    ]

    def ref(spec, s):
        op = spec["op"]
        if op == "const":
            return spec["value"]
        if op == "task":
            return s[names.index(spec["task"])]
        if op in ("add", "mul", "min", "max"):
            acc = ref(spec["args"][0], s)
            f = {"add": np.add, "mul": np.multiply, "min": np.minimum, "max": np.maximum}[op]
            for x in spec["args"][1:]:
                acc = f(acc, ref(x, s))
            return acc
        if op == "sub":
            return ref(spec["args"][0], s) - ref(spec["args"][1], s)
        if op == "div":
            return ref(spec["args"][0], s) / ref(spec["args"][1], s)
        if op == "clamp":
            return np.clip(ref(spec["args"][0], s), spec["lo"], spec["hi"])
        c = spec["cond"]
        cmp = {"<": np.less, "<=": np.less_equal, ">": np.greater, ">=": np.greater_equal,
               "==": np.equal}[c["cmp"]]
        return np.where(cmp(ref(c["left"], s), ref(c["right"], s)), ref(spec["then"], s),
                        ref(spec["else"], s))

    counts = np.array([C, 600, 0], dtype=np.int32)
    for spec in specs:
        out, zero = value_model_kernel(spec, names, torch.as_tensor(ts, device="cuda"),
                                       torch.as_tensor(counts, device="cuda"))
        got = out.cpu().numpy()
        for b in range(B):
            m = int(counts[b])
            with np.errstate(all="ignore"):
                want = np.broadcast_to(ref(spec, ts[b]), (C,))
            assert np.array_equal(got[b, :m], want[:m], equal_nan=True), (spec["op"], b)
        assert int(zero.item()) == 0
    # a zero divisor inside a valid candidate sets the flag; past the count it does not
    z = ts.copy()
    z[1, 1, 700] = 0.0
    z[1, 1, 10] = 1.0
    div = {"op": "div", "args": [A, Bt]}
    zt = np.where(np.isnan(z), 1.0, z)
    zt[:, 1, :] = np.where(zt[:, 1, :] == 0.0, 2.0, zt[:, 1, :])
    zt[1, 1, 700] = 0.0
    _, zero = value_model_kernel(div, names, torch.as_tensor(zt, device="cuda"),
                                 torch.as_tensor(np.array([C, 600, 0], dtype=np.int32), device="cuda"))
    assert int(zero.item()) == 0
    zt[1, 1, 10] = 0.0
    _, zero = value_model_kernel(div, names, torch.as_tensor(zt, device="cuda"),
                                 torch.as_tensor(np.array([C, 600, 0], dtype=np.int32), device="cuda"))
    assert int(zero.item()) == 1
