"""Publish-side k-means on the GPU (paper_2511_14881_b200.kmeans) against the reference's
outputs (tests/golden/kmeans_cases.npz, made by running ref ivf.py) and the reference's own
property tests for this code (ref tests/test_ivf.py:20-150)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import load_json, load_npz
from oracle import filtra_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def km(cuda):
    from paper_2511_14881_b200 import kmeans
    return kmeans


@pytest.fixture(scope="module")
def golden():
    return load_npz("kmeans_cases.npz"), load_json("kmeans_meta.json")


def test_pp_init_matches_reference(km, golden):
    z, meta = golden
    for m in meta["pp"]:
        got = km.kmeans_pp_init(z[f"pp_{m['name']}_x"], m["k"], m["seed"]).vectors
        assert np.array_equal(got, z[f"pp_{m['name']}_c"]), m["name"]


def test_train_matches_reference(km, golden):
    z, meta = golden
    for m in meta["train"]:
        c, a = km.kmeans_train(z[f"tr_{m['name']}_x"], m["k"], max_iters=m["max_iters"],
                               tol=m["tol"], seed=m["seed"])
        assert np.array_equal(a, z[f"tr_{m['name']}_a"]), m["name"]
        assert np.array_equal(c.vectors, z[f"tr_{m['name']}_c"]), m["name"]


def test_build_ivf_matches_reference(km, golden):
    z, meta = golden
    cat = type("Cat", (), {"embeddings": z["ivf_emb"], "item_ids": z["ivf_ids"],
                           "__len__": lambda self: len(z["ivf_emb"])})()
    idx = km.build_ivf(cat, k=meta["ivf"]["k"], seed=meta["ivf"]["seed"])
    assert np.array_equal(idx.centroids.vectors, z["ivf_centroids"])
    assert np.array_equal(idx.perm, z["ivf_perm"])
    assert np.array_equal(idx.inv_perm, z["ivf_inv_perm"])
    assert np.array_equal(idx.cluster_offsets, z["ivf_offsets"])
    assert np.array_equal(idx.items_q.data, z["ivf_items_q"])
    assert np.array_equal(idx.valid_mask, z["ivf_valid"])
    assert np.array_equal(idx.item_ids, z["ivf_slot_ids"])
    qp = z["ivf_qp"]
    assert (idx.items_q.params.global_min, idx.items_q.params.global_max) == (qp[0], qp[1])


def test_pairwise_sum_bit_exact(km):
    rng = np.random.default_rng(5)
    for n in [0, 1, 7, 8, 127, 128, 129, 1000, 4097, 65536, 100_003, 2_500_017]:
        x = rng.random(n) * rng.random(n) ** 12 * 1e6
        assert km.pairwise_sum(torch.as_tensor(x, device="cuda")) == x.sum(), n


def test_draw_exact_including_ambiguous_crossings(km):
    """The D^2 draw equals searchsorted(cumsum(best), u * total, 'right') (ref ivf.py:94-96),
    also when the parallel prefix cannot decide the crossing (huge dynamic range)."""
    from paper_2511_14881_b200 import _native
    lib = _native.lib()
    rng = np.random.default_rng(8)
    walked = 0
    for case in range(40):
        n = int(rng.integers(1, 300_000))
        best = rng.random(n) ** 4
        if case % 2:
            best[int(rng.integers(n))] = 1e22  # forces an error window wider than the steps
        if case % 5 == 0:
            best[: n // 2] = 0.0
        x = torch.as_tensor(best, device="cuda")
        sc = km._Scratch(n, x.device)
        total = sc.pairwise_sum(x)
        prefix = torch.cumsum(x, 0)
        for u in (0.0, float(rng.random()), 0.999999999):
            _native.check(lib.fb_kmeans_draw(x.data_ptr(), prefix.data_ptr(), n, total.data_ptr(), u,
                                             sc.idx.data_ptr(), sc.lo.data_ptr(),
                                             sc.walks.data_ptr(), _native.stream_ptr()))
            want = min(int(np.searchsorted(np.cumsum(best), u * best.sum(), side="right")), n - 1)
            assert int(sc.idx.item()) == want, (case, n, u)
        walked += int(sc.walks.item())
    assert walked > 0  # the exact sequential walk was exercised


def test_kmeans_at_scale_matches_oracle_seeding(km):
    """64k points x 128 dims, k = 256: seeding chosen rows identical to the oracle's."""
    rng = np.random.default_rng(12)
    x = rng.standard_normal((65_536, 128)).astype(np.float32)
    X = km._as_device_f64(x)
    got = km._pp_init_device(X, 256, 3).cpu().numpy()
    want = orc.kmeans_pp_init(x, 256, 3)
    assert np.array_equal(got, want)


# ---- the reference's property tests (ref tests/test_ivf.py:20-150) -------------------

def two_blobs(n_per=50, dim=4, gap=10.0, seed=0):
    rng = np.random.default_rng(seed)
    return np.vstack([rng.standard_normal((n_per, dim)) * 0.1,
                      rng.standard_normal((n_per, dim)) * 0.1 + gap])


def test_k_too_large(km):
    from paper_2511_14881_b200.errors import KTooLarge
    with pytest.raises(KTooLarge):
        km.kmeans_pp_init(np.zeros((3, 2)), 4, seed=0)
    with pytest.raises(KTooLarge):
        km.kmeans_train(np.zeros((3, 2)), 4)


def test_k_equals_n_every_point_is_center(km):
    data = np.arange(12, dtype=np.float64).reshape(6, 2)
    got = {tuple(r) for r in km.kmeans_pp_init(data, 6, seed=5).vectors}
    assert got == {tuple(r) for r in data.astype(np.float32)}


def test_two_blobs_one_center_each(km):
    data = two_blobs()
    for seed in range(10):
        c = km.kmeans_pp_init(data, 2, seed=seed).vectors
        assert c[0, 0] * c[1, 0] < 20.0
        split = km.kmeans_inertia(data, c)
        assert split < 0.1 * km.kmeans_inertia(data, np.tile(data.mean(0), (2, 1)))


def test_train_k1_closed_form_and_deterministic(km):
    data = two_blobs()
    c, a = km.kmeans_train(data, 1, seed=0)
    assert np.allclose(c.vectors[0], data.mean(axis=0), atol=1e-5)
    assert np.all(a == 0)
    d = two_blobs(seed=4)
    c1, a1 = km.kmeans_train(d, 4, seed=17)
    c2, a2 = km.kmeans_train(d, 4, seed=17)
    assert np.array_equal(c1.vectors, c2.vectors) and np.array_equal(a1, a2)


def test_inertia_non_increasing_and_no_empty_clusters(km):
    data = two_blobs(n_per=100, dim=6, gap=3.0, seed=8)
    prev = np.inf
    for iters in (1, 2, 3, 5, 8, 12):
        c, _ = km.kmeans_train(data, 5, max_iters=iters, tol=0.0, seed=13)
        inertia = km.kmeans_inertia(data, c.vectors)
        assert inertia <= prev + 1e-9
        prev = inertia
    _, a = km.kmeans_train(np.repeat(two_blobs(n_per=10), 10, axis=0), 8, seed=21)
    assert len(np.unique(a)) == 8


def test_inertia_matches_oracle(km):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((5000, 32))
    c = rng.standard_normal((50, 32))
    want = float(orc.sq_dists(x, c).min(axis=1).sum())
    assert abs(km.kmeans_inertia(x, c) - want) <= 1e-9 * want
