"""GPU parity: every drop-in entry point vs the reference golden vectors and the CPU
oracle, bit-exact (ids, int32 scores, Bloom masks); float64 dequantised scores within
1e-5 relative. Runs through the C-ABI library on a B200."""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from conftest import json_to_expr, json_to_oracle_expr, load_json, load_npz
from oracle import filtra_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fb(cuda):
    import paper_2511_14881_b200 as fb
    return fb


def ref_index(z, pre, fb):
    lo, hi = (float(x) for x in z[pre + "qp"])
    ns = SimpleNamespace
    cent = z[pre + "centroids"] if (pre + "centroids") in z.files else None
    return ns(items_q=ns(data=z[pre + "items_q"], params=fb.QuantParams(lo, hi)),
              valid_mask=z[pre + "valid"], item_ids=z[pre + "item_ids"],
              cluster_offsets=z[pre + "offsets"],
              centroids=ns(vectors=cent) if cent is not None else None,
              n_slots=z[pre + "items_q"].shape[0], dim=z[pre + "items_q"].shape[1])


def test_bloom_build_golden(fb):
    z = load_npz("bloom_cases.npz")
    for i in range(int(z["n_cases"][0])):
        m, k, n_slots = (int(x) for x in z[f"c{i}_meta"])
        idx = fb.build_bloom_arrays(z[f"c{i}_fid"], z[f"c{i}_val"], z[f"c{i}_slot"], n_slots,
                                    fb.BloomParams(m, k))
        assert np.array_equal(idx.planes, z[f"c{i}_planes"]), i
        assert idx.plane_bytes == m * ((n_slots + 63) // 64) * 8


def test_build_bloom_list_front_end(fb):
    idx = fb.build_bloom([[(1, 1)], [(2, 2)], [], [(1, 1), (3, 7)]], fb.BloomParams(64, 3))
    p = idx.planes
    nz = {int(r): int(p[r, 0]) for r in np.flatnonzero(p[:, 0])}
    assert nz == {2: 0x2, 11: 0x8, 19: 0x8, 21: 0x9, 26: 0x2, 33: 0x9, 44: 0x9, 54: 0xA}
    padded = fb.build_bloom([[(1, 1)], [(2, 2)]], fb.BloomParams(64, 3), n_slots=128)
    for slot in range(2, 128):
        assert not padded.signature(slot).any()


def test_eval_compiled_golden(fb):
    z = load_npz("filter_cases.npz")
    exprs = load_json("filter_exprs.json")
    m, k, n = (int(x) for x in z["meta"])
    params = fb.BloomParams(m, k)
    bloom = fb.BloomIndex(params, z["planes"], n)
    ranges = [tuple(int(v) for v in r) for r in z["ranges"]]
    for i, e in enumerate(exprs):
        cf = fb.compile_filter(json_to_expr(e["expr"]), params)
        full = fb.eval_compiled(cf, bloom, z["valid"])
        assert np.array_equal(full, z["fulls"][i]), i
        ranged = np.concatenate([fb.eval_compiled(cf, bloom, z["valid"], r) for r in ranges])
        assert np.array_equal(ranged, z["ranged"][i]), i
    cf = fb.compile_filter(fb.Leaf(1, 1), params)
    with pytest.raises(ValueError):
        fb.eval_compiled(cf, bloom, z["valid"], slot_range=(10, 64))
    for row in z["leaf_budget"]:
        fid, val, words_read = (int(x) for x in row[:3])
        st = fb.FilterStats()
        got = fb.bloom_eval_leaf(bloom, fb.hash_positions(fid, val, params), word_range=(1, 4),
                                 stats=st)
        assert st.words_read == words_read
        assert np.array_equal(got, row[3:].astype(np.uint64))


def test_eval_not_is_valid_complement(fb, rng):
    params = fb.BloomParams(64, 3)
    sf = [[(int(rng.integers(1, 6)), int(rng.integers(1, 6))) for _ in range(int(rng.integers(0, 6)))]
          for _ in range(200)]
    bloom = fb.build_bloom(sf, params)
    valid = orc.from_bool(np.ones(200, dtype=bool))
    leaf = fb.Leaf(1, 1)
    a = fb.eval_compiled(fb.compile_filter(leaf, params), bloom, valid)
    b = fb.eval_compiled(fb.compile_filter(fb.Not(leaf), params), bloom, valid)
    assert not np.any(a & b)
    assert np.array_equal(a | b, valid)


def test_quantize_golden(fb):
    z = load_npz("quantize_cases.npz")
    for x, q, (lo, hi) in zip(z["x"], z["q"], z["params"]):
        p = fb.QuantParams(float(lo), float(hi))
        assert np.array_equal(fb.quantize_vector(x, p), q)
        assert np.array_equal(fb.quantize_vector(x.astype(np.float64), p), q)
    p = fb.QuantParams(-1.0, 1.0)
    assert [fb.quantize_value(v, p) for v in (-1.0, 1.0, 0.0)] == [-128, 127, 0]
    assert fb.quantize_value(-5.0, fb.QuantParams(0.0, 1.0)) == -128


def test_int8_dot_kats(fb, rng):
    v = np.array([127, 127, 127, 127], dtype=np.int8)
    assert fb.int8_dot(v, v) == 64516
    a = np.full(4096, 127, dtype=np.int8)
    b = np.full(4096, -128, dtype=np.int8)
    assert fb.int8_dot(a, b) == 127 * -128 * 4096
    x = rng.integers(-128, 128, size=128).astype(np.int8)
    y = rng.integers(-128, 128, size=128).astype(np.int8)
    assert fb.int8_dot(x, y) == sum(int(p) * int(q) for p, q in zip(x, y))
    from paper_2511_14881_b200.errors import LengthMismatch
    with pytest.raises(LengthMismatch):
        fb.int8_dot(np.zeros(3, dtype=np.int8), np.zeros(4, dtype=np.int8))


def test_scan_golden(fb):
    z = load_npz("scan_cases.npz")
    meta = load_json("scan_meta.json")
    for ci, m in enumerate(meta):
        pre = f"s{ci}_"
        ivf = ref_index(z, pre, fb)
        bloom = fb.BloomIndex(fb.BloomParams(), z[pre + "planes"], ivf.n_slots)
        for q in m["queries"]:
            t = q["t"]
            qf = z[pre + f"q{t}_f"]
            assert fb.probe_centroids(ivf, qf, q["nprobe"]).tolist() == q["clusters"]
            if q["kind"] == 0:
                res = fb.search_clusters(ivf, z[pre + f"q{t}_q"], np.array(q["clusters"]),
                                         z[pre + f"q{t}_mask"], q["topk"])
            elif q["kind"] == 1:
                cf = fb.compile_filter(json_to_expr(q["expr"]), fb.BloomParams())
                res = fb.codesigned_search(ivf, bloom, cf, qf, q["nprobe"], q["topk"])
            else:
                res = fb.search(ivf, qf, q["nprobe"], q["topk"])
            assert np.array_equal(res.item_ids, z[pre + f"q{t}_ids"]), (ci, t)
            assert np.array_equal(res.scores, z[pre + f"q{t}_scores"]), (ci, t)
            assert res.scores.dtype == np.int32 and res.item_ids.dtype == np.uint64
        # exhaustive search == int8 brute force (reference tests/test_ivf.py:287-294)
        res = fb.search(ivf, z[pre + "bf_q"], nprobe=len(z[pre + "offsets"]), topk=64)
        assert np.array_equal(res.item_ids, z[pre + "bf_ids"])
        assert np.array_equal(res.scores, z[pre + "bf_scores"])


def test_ties_ascending_item_id(fb):
    z = load_npz("scan_cases.npz")
    ivf = ref_index(z, "tie_", fb)
    res = fb.search_clusters(ivf, fb.quantize_vector(np.array([1.0, 0.0], np.float32),
                                                     ivf.items_q.params), [0], None, 4)
    assert res.item_ids.tolist() == [1, 3, 7, 9] == z["tie_ids"].tolist()
    assert len(set(res.scores.tolist())) == 1


def test_four_attribute_and_topk20000(fb):
    z = load_npz("four_attr.npz")
    ivf = ref_index(z, "", fb)
    bloom = fb.BloomIndex(fb.BloomParams(), z["planes"], ivf.n_slots)
    for t, c in enumerate(load_json("four_attr.json")):
        cf = fb.compile_filter(json_to_expr(c["expr"]), fb.BloomParams())
        res = fb.codesigned_search(ivf, bloom, cf, z[f"q{t}_f"], 1, c["k"])
        assert np.array_equal(res.item_ids, z[f"q{t}_ids"]), t
        assert np.array_equal(res.scores, z[f"q{t}_scores"]), t
    y = load_npz("topk20000.npz")
    ivf = ref_index(y, "", fb)
    q = fb.quantize_vector(y["q"], ivf.items_q.params)
    res = fb.search_clusters(ivf, q, np.arange(len(y["offsets"])), None, 20000)
    assert len(res) == 20000
    assert np.array_equal(res.item_ids, y["ids"]) and np.array_equal(res.scores, y["scores"])


def test_reduce_topk_golden(fb):
    z = load_npz("merge_cases.npz")
    for c in range(int(z["n_cases"][0])):
        ids, sc = fb._reduce_topk(z[f"c{c}_ids"], z[f"c{c}_scores"], int(z[f"c{c}_k"][0]))
        assert np.array_equal(ids, z[f"c{c}_rids"]) and np.array_equal(sc, z[f"c{c}_rscores"])


def test_scan_edge_cases(fb):
    z = load_npz("scan_cases.npz")
    ivf = ref_index(z, "s1_", fb)
    q = z["s1_q0_q"]
    n_cl = len(z["s1_offsets"])
    res = fb.search_clusters(ivf, q, np.arange(n_cl), np.zeros_like(z["s1_valid"]), 10)
    assert len(res) == 0
    res = fb.search_clusters(ivf, q, np.arange(n_cl), None, 10 ** 6)
    assert len(res) == 400
    pairs = list(zip(res.scores.tolist(), res.item_ids.tolist()))
    assert pairs == sorted(pairs, key=lambda t: (-t[0], t[1]))
    assert len(fb.search_clusters(ivf, q, np.arange(n_cl), None, 0)) == 0
    assert len(fb.search_clusters(ivf, q, np.array([], dtype=np.int64), None, 5)) == 0
    from paper_2511_14881_b200.errors import DimMismatch
    with pytest.raises(DimMismatch):
        fb.search_clusters(ivf, np.zeros(ivf.dim + 1, np.int8), [0], None, 5)
    with pytest.raises(DimMismatch):
        fb.probe_centroids(ivf, np.zeros(ivf.dim + 1, np.float32), 1)


def test_scan_stats_and_codesign_accounting(fb):
    z = load_npz("scan_cases.npz")
    ivf = ref_index(z, "s2_", fb)
    bloom = fb.BloomIndex(fb.BloomParams(), z["s2_planes"], ivf.n_slots)
    cf = fb.compile_filter(fb.Or((fb.Leaf(1, 1), fb.Leaf(2, 2))), fb.BloomParams())
    scan, filt = fb.ScanStats(), fb.FilterStats()
    qf = z["s2_q0_f"]
    fb.codesigned_search(ivf, bloom, cf, qf, 3, 10, scan_stats=scan, filter_stats=filt)
    probed = fb.probe_centroids(ivf, qf, 3)
    expected = sum(int(e - s) for s, e in (z["s2_offsets"][int(c)] for c in probed))
    assert scan.slots_scanned == expected and filt.slots_evaluated == expected
    sizes = [int(e - s) for s, e in (z["s2_offsets"][int(c)] for c in probed)]
    assert scan.tiles == sum((n + 4095) // 4096 for n in sizes if n > 0)  # ref ivf.py:311-327
    assert scan.max_tile_rows == max([min(n, 4096) for n in sizes if n > 0] or [0])
    assert filt.words_read == sum(len(qb.set_bits) for _, _, qb in cf.leaves) * expected // 64


# --- batched path vs the oracle -------------------------------------------------------

def oracle_batch(wl, idx, k, ranges=None, masks=None, filtered=True):
    from paper_2511_14881_b200 import _device
    items = idx.items.cpu().numpy()[:, : wl.dim]
    valid = _device.u64_host(idx.valid)
    ids = _device.u64_host(idx.item_ids)
    offs = np.array([[0, idx.n_slots]] if ranges is None else ranges)
    qq = wl.queries_q.cpu().numpy()[:, : wl.dim]
    out = []
    for q in range(qq.shape[0]):
        cf = wl.filters[q] if filtered else None
        prog = None
        if cf is not None:
            prog = ([(int(o), int(a)) for o, a in cf.ops],
                    [(f, v, qb.set_bits) for f, v, qb in cf.leaves])
        clusters = list(range(len(offs)))
        if masks is not None:
            mask = masks[q]
            if prog is not None:
                mask = mask & orc.eval_compiled(prog[0], prog[1], idx.bloom.planes, valid)
            out.append(orc.search_clusters(items, valid, ids, offs, qq[q], clusters, mask, k))
        else:
            out.append(orc.codesigned_search(items, valid, ids, offs, idx.bloom.planes, prog,
                                             qq[q], clusters, k))
    return out


@pytest.fixture(scope="module")
def wl_small(fb):
    from paper_2511_14881_b200 import workload
    return workload.make_workload(50_000, 24, dim=128, seed=11)


@pytest.mark.parametrize("k", [1, 100, 5000])
@pytest.mark.parametrize("flags", [0, 1])  # 1 = FB_PLAN_FORCE_FALLBACK
def test_batched_filtered_vs_oracle(fb, wl_small, k, flags):
    wl = wl_small
    idx = wl.index
    op = fb.TopkOp(idx, 24, k, np.array([[0, idx.n_slots]]), flags)
    out = op(wl.queries_q, wl.batch)
    torch.cuda.synchronize()
    ref = oracle_batch(wl, idx, k)
    for q in range(24):
        ids, scores = out.host(q)
        assert np.array_equal(ids, ref[q].item_ids), q
        assert np.array_equal(scores, ref[q].scores), q


def test_batched_ranges_masks_unfiltered(fb, wl_small, rng):
    wl = wl_small
    idx = wl.index
    ranges = np.array([[0, 640], [6400, 20000], [30016, 30080], [49984, 50048]])
    k = 700
    masks_np = np.stack([orc.from_bool(rng.random(idx.n_slots) < 0.5) for _ in range(24)])
    from paper_2511_14881_b200 import _device
    masks = _device.to_dev_u64(masks_np).view(24, -1)
    for filtered in (False, True):
        op = fb.TopkOp(idx, 24, k, ranges)
        out = op(wl.queries_q, wl.batch if filtered else None, masks=masks)
        torch.cuda.synchronize()
        ref = oracle_batch(wl, idx, k, ranges=ranges, masks=masks_np, filtered=filtered)
        for q in range(24):
            ids, scores = out.host(q)
            assert np.array_equal(ids, ref[q].item_ids), (filtered, q)
            assert np.array_equal(scores, ref[q].scores), (filtered, q)


def test_dequantised_scores_within_1e5(fb, wl_small):
    wl = wl_small
    idx = wl.index
    op = fb.TopkOp(idx, 24, 300, np.array([[0, idx.n_slots]]))
    out = op(wl.queries_q, wl.batch, fscores=True)
    torch.cuda.synchronize()
    items = idx.items.cpu().numpy()[:, : wl.dim]
    qq = wl.queries_q.cpu().numpy()[:, : wl.dim]
    lo, hi = wl.qp.global_min, wl.qp.global_max
    for q in range(0, 24, 5):
        ids, _ = out.host(q)
        n = len(ids)
        got = out.fscores[q, :n].cpu().numpy()
        want = (orc.dequantize(items[ids.astype(np.int64)], lo, hi) *
                orc.dequantize(qq[q], lo, hi)).sum(axis=1)
        scale = np.abs(orc.dequantize(items[ids.astype(np.int64)], lo, hi) *
                       orc.dequantize(qq[q], lo, hi)).sum(axis=1)
        assert np.all(np.abs(got - want) <= 1e-5 * np.maximum(np.abs(want), scale * 1e-3))


def test_sampling_path_large_k(fb):
    """Candidate buffer smaller than the scanned set: the sampled threshold path must
    stay exact (vs brute force), with and without the forced fallback."""
    from paper_2511_14881_b200 import _device, workload
    wl = workload.make_workload(400_000, 6, dim=128, seed=5)
    idx = wl.index
    items = idx.items.cpu().numpy()[:, : wl.dim]
    valid = _device.u64_host(idx.valid)
    planes = idx.bloom.planes
    for flags in (0, 1):
        op = fb.TopkOp(idx, 6, 3000, np.array([[0, idx.n_slots]]), flags)
        out = op(wl.queries_q, wl.batch)
        torch.cuda.synchronize()
        for q in range(6):
            cf = wl.filters[q]
            mask = orc.eval_compiled([(int(o), int(a)) for o, a in cf.ops],
                                     [(f, v, qb.set_bits) for f, v, qb in cf.leaves], planes, valid)
            ref = orc.brute_force_int8(items, np.arange(idx.n_slots, dtype=np.uint64),
                                       wl.queries_q[q, : wl.dim].cpu().numpy(), 3000,
                                       keep=orc.to_bool(mask, idx.n_slots))
            ids, scores = out.host(q)
            assert np.array_equal(ids, ref.item_ids), (flags, q)
            assert np.array_equal(scores, ref.scores), (flags, q)


def test_config3_shape_batch1024_k20000(fb):
    """Config-3 shape at 2M items: 1024 queries (four 256-query chunks of the scan kernel),
    top-k 20000, the 4-attribute filter; sampled queries from every chunk vs brute force."""
    from paper_2511_14881_b200 import _device, workload
    wl = workload.make_workload(2_000_000, 1024, dim=128, seed=17)
    idx = wl.index
    op = fb.TopkOp(idx, 1024, 20000, np.array([[0, idx.n_slots]]))
    out = op(wl.queries_q, wl.batch)
    torch.cuda.synchronize()
    assert _device is not None and out.count.shape[0] == 1024
    items = idx.items.cpu().numpy()[:, : wl.dim]
    valid = _device.u64_host(idx.valid)
    ids_all = _device.u64_host(idx.item_ids)
    planes = idx.bloom.planes
    for q in (0, 255, 256, 600, 1023):
        cf = wl.filters[q]
        mask = orc.eval_compiled([(int(o), int(a)) for o, a in cf.ops],
                                 [(f, v, qb.set_bits) for f, v, qb in cf.leaves], planes, valid)
        ref = orc.brute_force_int8(items, ids_all, wl.queries_q[q, : wl.dim].cpu().numpy(),
                                   20000, keep=orc.to_bool(mask, idx.n_slots))
        ids, scores = out.host(q)
        assert np.array_equal(ids, ref.item_ids), q
        assert np.array_equal(scores, ref.scores), q


@pytest.mark.parametrize("filtered", [False, True])
def test_bytecode_kernel_multi_tile_per_cta(fb, filtered):
    """Enough tiles that every CTA cycles through all item stages (the per-stage id-rank
    area is found at the right offset), unfiltered (no program) and with a non-CNF
    program batch; vs brute force."""
    from paper_2511_14881_b200 import _device, workload
    from paper_2511_14881_b200.filter_query import FilterBatch
    wl = workload.make_workload(300_000, 16, dim=128, seed=23, filtered=False)
    idx = wl.index
    batch = None
    filters = [None] * 16
    if filtered:
        rng = np.random.default_rng(8)
        filters = [fb.compile_filter(_to_expr(fb, _random_filter(rng)), fb.BloomParams())
                   for _ in range(16)]
        batch = FilterBatch.pack(filters, fb.BloomParams())
        assert not batch.is_cnf
    op = fb.TopkOp(idx, 16, 2000, np.array([[0, idx.n_slots]]))
    out = op(wl.queries_q, batch)
    torch.cuda.synchronize()
    items = idx.items.cpu().numpy()[:, :128]
    valid = _device.u64_host(idx.valid)
    ids_all = _device.u64_host(idx.item_ids)
    for q in range(16):
        keep = orc.to_bool(valid, idx.n_slots)
        if filters[q] is not None:
            cf = filters[q]
            m = orc.eval_compiled([(int(o), int(a)) for o, a in cf.ops],
                                  [(f, v, b.set_bits) for f, v, b in cf.leaves], idx.bloom.planes, valid)
            keep = orc.to_bool(m, idx.n_slots)
        ref = orc.brute_force_int8(items, ids_all, wl.queries_q[q, :128].cpu().numpy(), 2000, keep=keep)
        ids, scores = out.host(q)
        assert np.array_equal(ids, ref.item_ids), q
        assert np.array_equal(scores, ref.scores), q


def test_pipelined_topk_matches_batched_op(fb, wl_small):
    """The serving pipeline (copies overlapped on a second stream, two slots) returns the
    batched operator's results for every submitted batch, including alternating inputs."""
    wl = wl_small
    idx = wl.index
    k = 400
    op = fb.TopkOp(idx, 24, k, np.array([[0, idx.n_slots]]))
    want = op(wl.queries_q, wl.batch)
    want_ids = want.ids.cpu().numpy().copy()
    want_sc = want.scores.cpu().numpy().copy()
    pipe = fb.PipelinedTopk(idx, 24, k, filters_template=wl.filters)
    hq = wl.queries.cpu().pin_memory()
    hq2 = (wl.queries.flip(0)).cpu().pin_memory()
    h_batch = fb.FilterBatch.pack(wl.filters, fb.BloomParams()).pin()
    tickets = [pipe.submit(hq if t % 2 == 0 else hq2, h_batch) for t in range(2)]
    for t in tickets:
        ids, sc, cnt = pipe.result(t)
        src = hq if t % 2 == 0 else hq2
        if t % 2 == 0:
            assert np.array_equal(ids.numpy(), want_ids)
            assert np.array_equal(sc.numpy(), want_sc)
        else:
            qq = idx.quantize_queries(src.cuda())
            ref = op(qq, wl.batch)
            assert np.array_equal(ids.numpy(), ref.ids.cpu().numpy())
            assert np.array_equal(sc.numpy(), ref.scores.cpu().numpy())


@pytest.mark.parametrize("path", ["probe", "masked"])
@pytest.mark.parametrize("case,nprobe,filtered", [(0, 3, True), (3, 7, True), (2, 1, False),
                                                (1, 5, True), (3, 30, True), (0, 20, False)])
def test_ivf_batched_probe_vs_oracle(fb, case, nprobe, filtered, path):
    """Batched IVF-probed co-designed search (IvfSearchOp): per-query centroid probe on the
    GPU (numpy-order float64 dots, ties by cluster id) + per-query probe masks + one
    batched filtered top-k == the oracle's codesigned_search with nprobe, per query."""
    from paper_2511_14881_b200.filter_query import FilterBatch
    z = load_npz("scan_cases.npz")
    pre = f"s{case}_"
    idx = ref_index(z, pre, fb)
    dix = fb.device_index_for(idx, bloom=fb.BloomIndex(fb.BloomParams(), z[pre + "planes"],
                                                        z[pre + "items_q"].shape[0]))
    qs = np.stack([z[pre + f"q{t}_f"] for t in range(12)])
    rng = np.random.default_rng(case * 10 + nprobe)
    filters = [fb.compile_filter(_to_expr(fb, _random_filter(rng)), fb.BloomParams())
               if filtered else None for _ in range(12)]
    batch = FilterBatch.pack(filters, fb.BloomParams()) if filtered else None
    k = 60
    op = fb.IvfSearchOp(dix, 12, nprobe, k, path=path)
    out, clusters = op(torch.as_tensor(qs, device="cuda"), batch)
    torch.cuda.synchronize()
    lo, hi = (float(x) for x in z[pre + "qp"])
    for t in range(12):
        cl = orc.probe_centroids(z[pre + "centroids"], qs[t], nprobe)
        assert np.array_equal(np.sort(clusters[t].cpu().numpy()), np.sort(cl)), t
        prog = None
        if filters[t] is not None:
            cf = filters[t]
            prog = ([(int(o), int(a)) for o, a in cf.ops], [(f, v, b.set_bits) for f, v, b in cf.leaves])
        ref = orc.codesigned_search(z[pre + "items_q"], z[pre + "valid"], z[pre + "item_ids"],
                                    z[pre + "offsets"], z[pre + "planes"], prog,
                                    orc.quantize(qs[t], lo, hi), cl, k)
        ids, scores = out.host(t)
        assert np.array_equal(ids, ref.item_ids), t
        assert np.array_equal(scores, ref.scores), t


@pytest.mark.parametrize("filtered,k", [(True, 1000), (False, 2000), (True, 30000)])
def test_ivf_grouped_scan_at_scale_vs_oracle(fb, filtered, k):
    """The grouped IVF scan (fb_ivf_topk) over a GPU-built IVF index (200k items, 400
    k-means clusters, 64 queries x 8 probes, the 4-attribute filter) == the oracle's
    codesigned_search per query; k = 30000 exceeds what one query can probe (all kept) and
    takes the slot-carrying selection."""
    from paper_2511_14881_b200 import kmeans, workload
    from paper_2511_14881_b200.filter_query import FilterBatch
    n, B, nprobe = 200_000, 64, 8
    wl = workload.make_workload(20_000, B, dim=128, seed=5)  # for its 4-attribute filters
    rng = np.random.default_rng(9)
    centres = rng.standard_normal((500, 128)).astype(np.float32)
    emb = centres[rng.integers(500, size=n)] + rng.standard_normal((n, 128)).astype(np.float32) * 0.3
    emb /= np.linalg.norm(emb, axis=1, keepdims=True)
    ids = rng.permutation(np.arange(1, n + 1, dtype=np.uint64) * 7919)
    cat = type("Cat", (), {"embeddings": emb, "item_ids": ids, "__len__": lambda self: n})()
    ivf = kmeans.build_ivf(cat, k=400, seed=1, max_iters=3)
    feats = [[(1, int(rng.integers(50))), (2, int(rng.integers(50))), (3, int(rng.integers(40))),
              (4, int(rng.integers(30)))] for _ in range(n)]
    bloom = fb.build_bloom(ivf.slot_features(feats), fb.BloomParams(), ivf.n_slots)
    dix = fb.device_index_for(ivf, bloom=bloom)
    qs = emb[rng.integers(n, size=B)] + rng.standard_normal((B, 128)).astype(np.float32) * 0.05
    filters = [wl.filters[b] if filtered else None for b in range(B)]
    batch = FilterBatch.pack(filters, fb.BloomParams()) if filtered else None
    op = fb.IvfSearchOp(dix, B, nprobe, k)
    out, clusters = op(torch.as_tensor(qs, device="cuda"), batch)
    torch.cuda.synchronize()
    qp = ivf.items_q.params
    planes = bloom.planes if isinstance(bloom.planes, np.ndarray) else bloom.planes.cpu().numpy()
    for t in range(0, B, 4):
        cl = clusters[t].cpu().numpy()
        prog = None
        if filters[t] is not None:
            cf = filters[t]
            prog = ([(int(o), int(a)) for o, a in cf.ops], [(f, v, b.set_bits) for f, v, b in cf.leaves])
        ref = orc.codesigned_search(ivf.items_q.data, ivf.valid_mask, ivf.item_ids,
                                    ivf.cluster_offsets, planes, prog,
                                    orc.quantize(qs[t], qp.global_min, qp.global_max), cl, k)
        got_ids, got_scores = out.host(t)
        assert np.array_equal(got_ids, ref.item_ids), t
        assert np.array_equal(got_scores, ref.scores), t


def test_merge_topk_device(fb, rng):
    n_lists, B, k = 5, 3, 50
    scores = np.zeros((n_lists, B, k), np.int32)
    ids = np.zeros((n_lists, B, k), np.uint64)
    cnt = rng.integers(0, k + 1, size=(n_lists, B)).astype(np.int32)
    for l in range(n_lists):
        for b in range(B):
            s = rng.integers(-5, 5, size=cnt[l, b]).astype(np.int32)
            i = rng.choice(10_000, size=cnt[l, b], replace=False).astype(np.uint64) * 8 + l
            o = np.lexsort((i, -s.astype(np.int64)))
            scores[l, b, : cnt[l, b]] = s[o]
            ids[l, b, : cnt[l, b]] = i[o]
    from paper_2511_14881_b200 import _device
    out = fb.merge_topk(_device.to_dev(scores, torch.int32),
                        _device.to_dev_u64(ids).view(n_lists, B, k),
                        _device.to_dev(cnt, torch.int32), 60)
    for b in range(B):
        all_i = np.concatenate([ids[l, b, : cnt[l, b]] for l in range(n_lists)])
        all_s = np.concatenate([scores[l, b, : cnt[l, b]] for l in range(n_lists)])
        ri, rs = orc.reduce_topk(all_i, all_s, 60)
        gi, gs = out.host(b)
        assert np.array_equal(gi, ri) and np.array_equal(gs, rs)


# --- tensor-core scan ---------------------------------------------------------------

def test_tc_raw_scores_match_int32_matmul(fb, rng):
    """The tcgen05 kind::i8 path (TMA SWIZZLE_128B tiles, UMMA descriptors, TMEM reads)
    reproduces the exact int32 dot of every (query, slot)."""
    from paper_2511_14881_b200 import _device, _native
    for n, nq in ((512, 5), (1024, 130), (2304, 256)):
        items = rng.integers(-128, 128, size=(n, 128)).astype(np.int8)
        items[: n // 8] = 127  # saturated rows: |dot| up to 128*128*128
        q = rng.integers(-128, 128, size=(nq, 128)).astype(np.int8)
        q[0] = -128
        dix = fb.DeviceIndex.from_arrays(items, orc.from_bool(np.ones(n, bool)),
                                         np.arange(n, dtype=np.uint64))
        qd = _device.to_dev(q, torch.int8)
        out = torch.empty((nq, dix.n_slots_pad), dtype=torch.int32, device=qd.device)
        _native.check(_native.lib().fb_debug_tc_scores(dix.struct(), qd.data_ptr(), nq,
                                                       out.data_ptr(), _native.stream_ptr()))
        want = q.astype(np.int64) @ items.astype(np.int64).T
        assert np.array_equal(out.cpu().numpy()[:, :n], want), (n, nq)


@pytest.mark.parametrize("k", [1, 777, 10000])
def test_tc_vs_simt_vs_oracle(fb, wl_small, k):
    from paper_2511_14881_b200 import _native
    wl = wl_small
    idx = wl.index
    ref = oracle_batch(wl, idx, k)
    for flags in (0, _native.FB_PLAN_SIMT, _native.FB_PLAN_FORCE_FALLBACK):
        op = fb.TopkOp(idx, 24, k, np.array([[0, idx.n_slots]]), flags)
        out = op(wl.queries_q, wl.batch)
        torch.cuda.synchronize()
        path = _native.lib().fb_topk_scan_path(op._plan)
        assert path == (0 if flags == _native.FB_PLAN_SIMT else 1)
        for q in range(24):
            ids, scores = out.host(q)
            assert np.array_equal(ids, ref[q].item_ids), (flags, q)
            assert np.array_equal(scores, ref[q].scores), (flags, q)


def _random_filter(rng, depth=0):
    if depth >= 3 or rng.random() < 0.3:
        return ("leaf", int(rng.integers(1, 5)), int(rng.integers(0, 12)))
    roll = rng.random()
    if roll < 0.2:
        return ("not", _random_filter(rng, depth + 1))
    kind = "and" if roll < 0.6 else "or"
    return (kind, [_random_filter(rng, depth + 1) for _ in range(int(rng.integers(2, 4)))])


def _to_expr(fb, t):
    if t[0] == "leaf":
        return fb.Leaf(t[1], t[2])
    if t[0] == "not":
        return fb.Not(_to_expr(fb, t[1]))
    cls = fb.And if t[0] == "and" else fb.Or
    return cls(tuple(_to_expr(fb, c) for c in t[1]))


@pytest.mark.parametrize("shape,nq", [("cnf_neg", 40), ("cnf_neg", 200), ("cnf_bins", 40),
                                      ("cnf_bins", 256), ("cnf_bins", 300), ("cnf_wide", 40),
                                      ("cnf_wide", 150), ("random_mixed", 40)])
def test_tc_filter_modes_vs_oracle(fb, shape, nq):
    """CNF batches (with negated literals / NOT over groups) take the per-hit tensor-core
    epilogue: the fast form (<= 64 literal columns, <= 4 groups) or the general form (wide
    batches); batches with any non-CNF program take the bytecode epilogue. All must match
    the oracle exactly, with one or two 128-query M-blocks."""
    from paper_2511_14881_b200 import _device, _native, workload
    from paper_2511_14881_b200.filter_query import FilterBatch
    wl = workload.make_workload(30_000, nq, dim=128, seed=21, filtered=False)
    idx = wl.index
    rng = np.random.default_rng(5)
    p = fb.BloomParams()
    exprs = []
    for q in range(nq):
        if shape == "cnf_bins":  # 4 features x up to 40 values: windowed, 8 column words
            groups = []
            for f in range(1, 5):
                lits = [fb.Leaf(f, int(v)) for v in rng.choice(40, size=6, replace=False)]
                groups.append(fb.Or(tuple(lits)))
            exprs.append(fb.And(tuple(groups)))
        elif shape == "cnf_wide":
            groups = []
            for f in range(1, 7):
                lits = [fb.Leaf(f, int(v)) for v in rng.choice(12, size=4, replace=False)]
                if rng.random() < 0.2:
                    lits[1] = fb.Not(lits[1])
                groups.append(fb.Or(tuple(lits)))
            exprs.append(fb.And(tuple(groups)))
        elif shape == "cnf_neg":
            groups = []
            for f in range(1, 4):
                lits = [fb.Leaf(f, int(v)) for v in rng.choice(12, size=3, replace=False)]
                if rng.random() < 0.4:
                    lits[0] = fb.Not(lits[0])
                groups.append(fb.Or(tuple(lits)))
            e = fb.And(tuple(groups))
            if rng.random() < 0.2:
                e = fb.Not(fb.Or((fb.Leaf(5, int(rng.integers(0, 20))), fb.Leaf(6, 1))))
            exprs.append(e)
        else:
            exprs.append(_to_expr(fb, _random_filter(rng)))
    filters = [fb.compile_filter(e, p) for e in exprs]
    filters[3] = None
    batch = FilterBatch.pack(filters, p)
    assert batch.is_cnf == shape.startswith("cnf")
    if shape.startswith("cnf"):
        assert batch.cnf_windowed == (shape != "cnf_wide")
    if shape == "cnf_bins":
        assert batch.cnf_words > 2
    items = idx.items.cpu().numpy()[:, :128]
    valid = _device.u64_host(idx.valid)
    ids = _device.u64_host(idx.item_ids)
    offs = np.array([[0, idx.n_slots]])
    qq = wl.queries_q.cpu().numpy()[:, :128]
    for k in (50, 3000):
        op = fb.TopkOp(idx, nq, k, offs)
        out = op(wl.queries_q, batch)
        torch.cuda.synchronize()
        assert _native.lib().fb_topk_scan_path(op._plan) == 1
        for q in range(nq):
            cf = filters[q]
            prog = None if cf is None else ([(int(o), int(a)) for o, a in cf.ops],
                                            [(f, v, b.set_bits) for f, v, b in cf.leaves])
            ref = orc.codesigned_search(items, valid, ids, offs, idx.bloom.planes, prog, qq[q],
                                        [0], k)
            got_ids, got_scores = out.host(q)
            assert np.array_equal(got_ids, ref.item_ids), (shape, k, q)
            assert np.array_equal(got_scores, ref.scores), (shape, k, q)


@pytest.mark.parametrize("k", [1, 777, 5000])
def test_select_paths_agree_with_oracle(fb, wl_small, k):
    """Key-only radix selection (index with a rank -> slot table) and the chunked
    bitonic selection (no table) give the oracle's order."""
    wl = wl_small
    idx = wl.index
    ref = oracle_batch(wl, idx, k)
    saved = idx.slot_of_rank
    assert saved is not None
    try:
        for table in (saved, None):
            idx.slot_of_rank = table
            op = fb.TopkOp(idx, 24, k, np.array([[0, idx.n_slots]]))
            out = op(wl.queries_q, wl.batch, keys=True)
            torch.cuda.synchronize()
            for q in range(24):
                ids, scores = out.host(q)
                assert np.array_equal(ids, ref[q].item_ids), (table is None, q)
                assert np.array_equal(scores, ref[q].scores), (table is None, q)
    finally:
        idx.slot_of_rank = saved


def test_select_heavy_ties(fb, rng):
    """Few distinct scores (items in {-1, 0, 1}): order by (score desc, id asc) through
    the radix selection, against brute force; ids deliberately not in slot order."""
    from paper_2511_14881_b200 import _device, _native
    n = 30_000
    items = rng.integers(-1, 2, size=(n, 128)).astype(np.int8)
    ids = rng.permutation(n * 3)[:n].astype(np.uint64) + np.uint64(1 << 40)
    valid = rng.random(n) < 0.9
    dix = fb.DeviceIndex.from_arrays(items, orc.from_bool(valid), ids)
    assert dix.slot_of_rank is not None
    q = rng.integers(-1, 2, size=(4, 128)).astype(np.int8)
    for k in (100, 4000, 10_000):
        op = fb.TopkOp(dix, 4, k, np.array([[0, n]]), _native.FB_PLAN_NO_SAMPLE)
        out = op(_device.to_dev(q, torch.int8), None)
        torch.cuda.synchronize()
        for b in range(4):
            ref = orc.brute_force_int8(items, ids, q[b], k, keep=valid)
            gi, gs = out.host(b)
            assert np.array_equal(gi, ref.item_ids), (k, b)
            assert np.array_equal(gs, ref.scores), (k, b)


def test_select_dense_ids(fb, rng):
    """Shards whose valid ids are one contiguous run (in rank order) take the computed-id
    selection (fb_index_t.id_dense: id = base + rank, no id_of_rank gather); any other id
    set keeps the table. Both agree with brute force, and forcing the table on a dense
    shard gives identical outputs. Invalid slots hold ids outside the run; the base sits
    above 2^63 so the u64 arithmetic is exercised."""
    from paper_2511_14881_b200 import _device, _native
    n = 40_000
    items = rng.integers(-3, 4, size=(n, 128)).astype(np.int8)
    valid = rng.random(n) < 0.85
    base = np.uint64((1 << 63) + 12345)
    ids = np.full(n, np.uint64(7), dtype=np.uint64)
    order = rng.permutation(int(valid.sum()))
    ids[valid] = base + order.astype(np.uint64)
    q = rng.integers(-3, 4, size=(4, 128)).astype(np.int8)
    broken = ids.copy()
    broken[np.flatnonzero(valid)[0]] = base + np.uint64(n * 2)  # a gap: not dense
    for id_set, dense in ((ids, 1), (broken, 0)):
        dix = fb.DeviceIndex.from_arrays(items, orc.from_bool(valid), id_set)
        assert dix.id_dense == dense
        if dense:
            assert dix.id_base == int(base)
        for k in (100, 10_000):
            outs = []
            for force_table in ((False, True) if dense else (False,)):
                if force_table:
                    dix.id_dense = 0
                op = fb.TopkOp(dix, 4, k, np.array([[0, n]]), _native.FB_PLAN_NO_SAMPLE)
                out = op(_device.to_dev(q, torch.int8), None)
                torch.cuda.synchronize()
                outs.append([out.host(b) for b in range(4)])
                dix.id_dense = dense
            for b in range(4):
                ref = orc.brute_force_int8(items, id_set, q[b], k, keep=valid)
                for o in outs:
                    assert np.array_equal(o[b][0], ref.item_ids), (dense, k, b)
                    assert np.array_equal(o[b][1], ref.scores), (dense, k, b)


@pytest.mark.parametrize("depth", [2, 3])
def test_pipelined_topk_overlapped_plans(fb, wl_small, depth):
    """Per-slot plans on per-slot compute streams (overlap=True: batch i+1's sample pass
    and threshold run beside batch i's selection) return, for a stream of alternating
    batches kept ``depth`` deep in flight, exactly the single-plan results."""
    wl = wl_small
    idx = wl.index
    k = 400
    op = fb.TopkOp(idx, 24, k, np.array([[0, idx.n_slots]]))
    srcs = [wl.queries, wl.queries.flip(0), wl.queries.roll(5, 0)]
    want = []
    for q in srcs:
        r = op(idx.quantize_queries(q), wl.batch)
        want.append((r.ids.cpu().numpy().copy(), r.scores.cpu().numpy().copy(),
                     r.count.cpu().numpy().copy()))
    hq = [q.cpu().pin_memory() for q in srcs]
    h_batch = fb.FilterBatch.pack(wl.filters, fb.BloomParams()).pin()
    pipe = fb.PipelinedTopk(idx, 24, k, depth=depth, filters_template=wl.filters)
    assert len(pipe.ops) == depth and len(set(id(s) for s in pipe.streams)) == depth
    n = 9
    for t in range(n + depth - 1):
        if t < n:
            pipe.submit(hq[t % 3], h_batch)
        c = t - depth + 1
        if c >= 0:
            ids, sc, cnt = pipe.result(c)
            w = want[c % 3]
            assert np.array_equal(ids.numpy(), w[0]), (depth, c)
            assert np.array_equal(sc.numpy(), w[1]), (depth, c)
            assert np.array_equal(cnt.numpy(), w[2]), (depth, c)
