"""Publish-side IVF build on the GPU: KMeans++ seeding, Lloyd iterations and the
cluster-major slot layout (reference ivf.py:68-258), behind the reference signatures.

What is bit-identical to the reference (same seed, same float64 data):
  * ``kmeans_pp_init``: the D^2 distances, their totals and the cumsum/searchsorted draw
    follow numpy's exact summation orders (``fb_kmeans_min_sqdist``,
    ``fb_pairwise_sum_f64``, ``fb_kmeans_draw``), and the random stream is numpy's own
    ``default_rng(seed)`` drawn on the host in the reference's order -- so the chosen
    centres are the reference's;
  * cluster means (``fb_kmeans_means``) and inertia totals, given the same assignment;
  * the ``build_ivf`` layout (cluster-major, 64-aligned, ascending item id inside a cluster,
    quantised rows, validity, slot ids) given the same assignment.
Lloyd assignment distances come from a BLAS GEMM in the reference (unspecified summation
order), so assignments agree except where two centres are within fp64 rounding of a tie;
the reference's own tests for this code are property tests (determinism, inertia bounds,
no empty clusters), which ``tests/test_gpu_kmeans.py`` runs against this module.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from ._device import device
from .errors import KTooLarge
from .quantize import QuantizedMatrix, QuantParams, compute_quant_params, quantize_device

DEFAULT_MAX_ITERS = 25  # ivf.py:26-27
DEFAULT_TOL = 1e-4
WORD_BITS = 64


@dataclass(frozen=True)
class Centroids:
    """ivf.py:30-40."""
    vectors: np.ndarray  # float32 (n_clusters, dim)

    @property
    def n_clusters(self) -> int:
        return int(self.vectors.shape[0])

    @property
    def dim(self) -> int:
        return int(self.vectors.shape[1])


@dataclass(eq=False)
class IvfIndex:
    """Reference-shaped IVF index (ivf.py:154-204): host arrays in slot order."""
    centroids: Centroids
    perm: np.ndarray             # i64 slot -> item index, -1 padding
    inv_perm: np.ndarray         # i64 item index -> slot
    cluster_offsets: np.ndarray  # u64 (n_clusters, 2)
    items_q: QuantizedMatrix     # int8 rows in slot order
    valid_mask: np.ndarray       # packed u64 words
    item_ids: np.ndarray         # u64 per slot (0 on padding)
    _valid_bool: np.ndarray | None = field(default=None, repr=False)

    @property
    def n_slots(self) -> int:
        return int(self.perm.shape[0])

    @property
    def n_clusters(self) -> int:
        return self.centroids.n_clusters

    @property
    def dim(self) -> int:
        return self.centroids.dim

    @property
    def n_items(self) -> int:
        return int((self.perm >= 0).sum())

    @property
    def valid_bool(self) -> np.ndarray:
        if self._valid_bool is None:
            bits = np.unpackbits(self.valid_mask.view(np.uint8), bitorder="little")
            self._valid_bool = bits[: self.n_slots].astype(bool)
        return self._valid_bool

    def slot_features(self, feature_lists):
        return [feature_lists[p] if p >= 0 else [] for p in self.perm]

    def cluster_sizes(self) -> np.ndarray:
        return (self.cluster_offsets[:, 1] - self.cluster_offsets[:, 0]).astype(np.int64)


class _Scratch:
    """Device buffers reused across the per-centre steps of one training run."""

    def __init__(self, n: int, dev):
        lib = _native.lib()
        self.sum_buf = torch.empty(max(1, int(lib.fb_pairwise_sum_scratch(n))), dtype=torch.float64,
                                   device=dev)
        self.total = torch.empty(1, dtype=torch.float64, device=dev)
        self.idx = torch.empty(1, dtype=torch.int64, device=dev)
        self.lo = torch.empty(1, dtype=torch.int64, device=dev)
        self.walks = torch.zeros(1, dtype=torch.int32, device=dev)

    def pairwise_sum(self, x: torch.Tensor) -> torch.Tensor:
        _native.check(_native.lib().fb_pairwise_sum_f64(
            x.data_ptr(), x.numel(), self.total.data_ptr(), self.sum_buf.data_ptr(),
            self.sum_buf.numel(), _native.stream_ptr()))
        return self.total


def _as_device_f64(data) -> torch.Tensor:
    if isinstance(data, torch.Tensor):
        t = data.to(device=device(), dtype=torch.float64)
    else:
        t = torch.as_tensor(np.ascontiguousarray(np.asarray(data, dtype=np.float64)), device=device())
    if t.dim() != 2:
        t = t.reshape(t.shape[0], -1)
    return t.contiguous()


def pairwise_sum(x: torch.Tensor) -> float:
    """numpy's ``x.sum()`` for a float64 CUDA vector, bit-identical."""
    x = x.contiguous()
    return float(_Scratch(x.numel(), x.device).pairwise_sum(x).item())


def _pp_init_device(X: torch.Tensor, k: int, seed: int, stats: dict | None = None) -> torch.Tensor:
    """kmeans_pp_init (ivf.py:76-101) over float64 CUDA rows; returns the chosen row
    indices (int64 CUDA [k])."""
    lib = _native.lib()
    n, dim = X.shape
    if k > n:
        raise KTooLarge(k, n)
    st = _native.stream_ptr()
    rng = np.random.default_rng(seed)
    sc = _Scratch(n, X.device)
    chosen = torch.empty(k, dtype=torch.int64, device=X.device)
    first = int(rng.integers(n))
    chosen[0] = first
    best = torch.empty(n, dtype=torch.float64, device=X.device)
    _native.check(lib.fb_kmeans_min_sqdist(X.data_ptr(), n, dim, first, best.data_ptr(), 1, st))
    taken = torch.zeros(n, dtype=torch.bool, device=X.device)
    taken[first] = True
    prefix = torch.empty_like(best)
    for i in range(1, k):
        total = float(sc.pairwise_sum(best).item())
        if total <= 0.0:
            # remaining points duplicate chosen centres: uniform over the untaken ones
            pool = torch.nonzero(~taken).view(-1)
            idx = int(pool[int(rng.integers(pool.numel()))].item())
        else:
            u = float(rng.random())
            torch.cumsum(best, 0, out=prefix)
            _native.check(lib.fb_kmeans_draw(best.data_ptr(), prefix.data_ptr(), n,
                                             sc.total.data_ptr(), u, sc.idx.data_ptr(),
                                             sc.lo.data_ptr(), sc.walks.data_ptr(), st))
            idx = int(sc.idx.item())
        chosen[i] = idx
        taken[idx] = True
        _native.check(lib.fb_kmeans_min_sqdist(X.data_ptr(), n, dim, idx, best.data_ptr(), 0, st))
    if stats is not None:
        stats["exact_walks"] = int(sc.walks.item())
    return chosen


def kmeans_pp_init(data, k: int, seed: int) -> Centroids:
    """ivf.py:76-101 on the GPU; the chosen rows are the reference's."""
    X = _as_device_f64(data)
    chosen = _pp_init_device(X, k, seed)
    return Centroids(vectors=X[chosen].to(torch.float32).cpu().numpy())


def _assign(X, xx, centers, out_assign, out_d2):
    lib = _native.lib()
    n, dim = X.shape
    k = centers.shape[0]
    cc = torch.empty(k, dtype=torch.float64, device=X.device)
    st = _native.stream_ptr()
    _native.check(lib.fb_row_sqnorm_f64(centers.data_ptr(), k, dim, cc.data_ptr(), st))
    _native.check(lib.fb_kmeans_assign(X.data_ptr(), n, dim, centers.data_ptr(), k, xx.data_ptr(),
                                       cc.data_ptr(), out_assign.data_ptr(), out_d2.data_ptr(), st))


def _refill_empty(assign: torch.Tensor, point_cost: torch.Tensor, k: int) -> None:
    """ivf.py:123-130: each empty cluster takes the farthest point of the (first) largest."""
    sizes = torch.bincount(assign, minlength=k)
    empties = torch.nonzero(sizes == 0).view(-1).tolist()
    for c in empties:
        donor = int(torch.argmax(sizes).item())  # first maximum, as np.argmax
        cost = torch.where(assign == donor, point_cost, torch.full_like(point_cost, -np.inf))
        far = int(torch.argmax(cost).item())     # first maximum in ascending member order
        assign[far] = c
        point_cost[far] = 0.0
        sizes[donor] -= 1
        sizes[c] += 1


def _means(X, assign, k, centers):
    lib = _native.lib()
    order = torch.sort(assign, stable=True).indices  # members in ascending row order
    count = torch.bincount(assign, minlength=k)
    start = torch.cumsum(count, 0) - count
    _native.check(lib.fb_kmeans_means(X.data_ptr(), X.shape[1], order.data_ptr(), start.data_ptr(),
                                      count.data_ptr(), k, centers.data_ptr(),
                                      _native.stream_ptr()))


def _train_device(X: torch.Tensor, k: int, max_iters: int, tol: float, seed: int):
    n, dim = X.shape
    if k > n:
        raise KTooLarge(k, n)
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    lib = _native.lib()
    chosen = _pp_init_device(X, k, seed)
    centers = X[chosen].to(torch.float32).to(torch.float64).contiguous()
    xx = torch.empty(n, dtype=torch.float64, device=X.device)
    _native.check(lib.fb_row_sqnorm_f64(X.data_ptr(), n, dim, xx.data_ptr(), _native.stream_ptr()))
    assign = torch.zeros(n, dtype=torch.int64, device=X.device)
    d2 = torch.empty(n, dtype=torch.float64, device=X.device)
    sc = _Scratch(n, X.device)
    prev = None
    for _ in range(max_iters):
        _assign(X, xx, centers, assign, d2)
        _refill_empty(assign, d2, k)
        _means(X, assign, k, centers)
        _assign(X, xx, centers, assign, d2)
        inertia = float(sc.pairwise_sum(d2).item())
        if prev is not None and prev - inertia <= tol * prev:
            break
        prev = inertia
    return centers, assign


def kmeans_train(data, k: int, max_iters: int = DEFAULT_MAX_ITERS, tol: float = DEFAULT_TOL,
                 seed: int = 0) -> tuple[Centroids, np.ndarray]:
    """ivf.py:104-145 on the GPU: Lloyd from KMeans++ seeding, empty clusters re-seeded
    from the farthest point of the largest cluster."""
    X = _as_device_f64(data)
    centers, assign = _train_device(X, k, max_iters, tol, seed)
    return Centroids(vectors=centers.to(torch.float32).cpu().numpy()), assign.cpu().numpy()


def kmeans_inertia(data, centers) -> float:
    """ivf.py:148-151: sum over points of the squared distance to the nearest centre."""
    X = _as_device_f64(data)
    C = _as_device_f64(centers)
    n, dim = X.shape
    lib = _native.lib()
    xx = torch.empty(n, dtype=torch.float64, device=X.device)
    _native.check(lib.fb_row_sqnorm_f64(X.data_ptr(), n, dim, xx.data_ptr(), _native.stream_ptr()))
    assign = torch.empty(n, dtype=torch.int64, device=X.device)
    d2 = torch.empty(n, dtype=torch.float64, device=X.device)
    _assign(X, xx, C, assign, d2)
    return pairwise_sum(d2)


def ivf_layout(assign: torch.Tensor, item_ids_u64: torch.Tensor, k: int):
    """Cluster-major slot layout (ivf.py:229-249): per cluster, members by ascending item
    id, range padded to a multiple of 64. Returns (perm [n_slots] i64 CUDA, offsets
    [k, 2] i64 CUDA)."""
    dev = assign.device
    n = assign.numel()
    key = torch.bitwise_xor(item_ids_u64, -(1 << 63))                # u64 order as int64
    o1 = torch.sort(key, stable=True).indices
    o2 = torch.sort(assign[o1], stable=True).indices
    order = o1[o2]                                                   # by (cluster, item id)
    count = torch.bincount(assign, minlength=k)
    padded = (count + WORD_BITS - 1) // WORD_BITS * WORD_BITS
    end = torch.cumsum(padded, 0)
    start = end - padded
    n_slots = int(end[-1].item()) if k > 0 else 0
    cstart = torch.cumsum(count, 0) - count
    cl = assign[order]
    slot = start[cl] + (torch.arange(n, device=dev) - cstart[cl])
    perm = torch.full((n_slots,), -1, dtype=torch.int64, device=dev)
    perm[slot] = order
    return perm, torch.stack([start, end], dim=1)


def build_ivf(catalog, k: int | None = None, qp: QuantParams | None = None, seed: int = 0,
              max_iters: int = DEFAULT_MAX_ITERS, tol: float = DEFAULT_TOL) -> IvfIndex:
    """ivf.py:207-258 on the GPU: cluster the catalog, lay it out cluster-major with int8
    rows. ``k`` defaults to ceil(sqrt(n)); ``qp`` to the global min/max of the embeddings."""
    emb = np.asarray(catalog.embeddings, dtype=np.float32)
    n = len(catalog)
    if k is None:
        k = int(np.ceil(np.sqrt(n)))
    if k < 1:
        raise KTooLarge(k, n)
    dev = device()
    E = torch.as_tensor(np.ascontiguousarray(emb), device=dev)
    X = E.to(torch.float64).contiguous()
    centers, assign = _train_device(X, k, max_iters, tol, seed)
    if qp is None:
        qp = compute_quant_params(E)
    ids_np = np.asarray(catalog.item_ids, dtype=np.uint64)
    ids = torch.as_tensor(ids_np.view(np.int64), device=dev)
    perm, offsets = ivf_layout(assign, ids, k)
    n_slots = perm.numel()
    real = perm >= 0
    rows = torch.zeros((n_slots, emb.shape[1]), dtype=torch.float32, device=dev)
    rows[real] = E[perm[real]]
    items_q = quantize_device(rows, qp) if n_slots else torch.zeros((0, emb.shape[1]),
                                                                    dtype=torch.int8, device=dev)
    items_q[~real] = 0
    inv_perm = torch.full((n,), -1, dtype=torch.int64, device=dev)
    inv_perm[perm[real]] = torch.nonzero(real).view(-1)
    slot_ids = torch.zeros(n_slots, dtype=torch.int64, device=dev)
    slot_ids[real] = ids[perm[real]]
    n_words = (n_slots + WORD_BITS - 1) // WORD_BITS
    bits = torch.zeros(n_words * WORD_BITS, dtype=torch.int64, device=dev)
    bits[:n_slots] = real.to(torch.int64)
    shifts = torch.arange(WORD_BITS, dtype=torch.int64, device=dev)
    words = (bits.view(n_words, WORD_BITS) << shifts).sum(dim=1)     # disjoint bits: sum == OR
    return IvfIndex(centroids=Centroids(vectors=centers.to(torch.float32).cpu().numpy()),
                    perm=perm.cpu().numpy(), inv_perm=inv_perm.cpu().numpy(),
                    cluster_offsets=offsets.cpu().numpy().astype(np.uint64),
                    items_q=QuantizedMatrix(data=items_q.cpu().numpy(), params=qp),
                    valid_mask=words.cpu().numpy().view(np.uint64),
                    item_ids=slot_ids.cpu().numpy().view(np.uint64))
