"""Drop-in shims for the reference IVF scan API (ivf.py:43-343).

``search_clusters`` / ``search`` / ``probe_centroids`` keep the reference signatures and
return the reference result types; they accept either a ``DeviceIndex`` or a
reference-shaped ``IvfIndex`` (uploaded to HBM once and cached). Compute runs through
``fb_topk_execute`` (masked exact scan + exact (score desc, item_id asc) top-k) and
``fb_dot_rows_f64`` (numpy-order float64 centroid dots).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._device import device, to_dev, to_dev_u64
from .engine import DeviceIndex, TopkOp, TopkOutput, cached_op, device_index_for
from .errors import DimMismatch

TILE_ROWS = 4096  # reference tile contract (ivf.py:24); GPU tiles are 128 rows


@dataclass(frozen=True)
class TopkResult:
    """Scores sorted descending, ties by ascending item id (reference ivf.py:43-56)."""

    item_ids: np.ndarray
    scores: np.ndarray
    k_requested: int

    def __len__(self) -> int:
        return len(self.item_ids)

    @property
    def entries(self) -> list[tuple[int, float]]:
        return [(int(i), s.item()) for i, s in zip(self.item_ids, self.scores)]


@dataclass
class ScanStats:
    """Work counters (reference ivf.py:59-65), filled analytically from the plan."""

    slots_scanned: int = 0
    max_tile_rows: int = 0
    tiles: int = 0


def _empty(topk: int) -> TopkResult:
    return TopkResult(item_ids=np.empty(0, dtype=np.uint64), scores=np.empty(0, dtype=np.int32),
                      k_requested=topk)


def cluster_ranges(dix: DeviceIndex, clusters) -> np.ndarray:
    offs = dix.cluster_offsets
    cl = np.asarray(clusters, dtype=np.int64).reshape(-1)
    if cl.size == 0:
        return np.zeros((0, 2), dtype=np.int64)
    return np.ascontiguousarray(offs[cl].astype(np.int64))


def count_scan(ranges, stats: ScanStats) -> None:
    """``search_clusters``' counters for slot ranges, in the reference's tile contract (ref
    ivf.py:311-327: slots per range, ``TILE_ROWS``-row tiles, the largest tile) -- the
    GPU's own 256-item tiles are an implementation detail the counters do not expose."""
    for s, e in ranges:
        n = int(e) - int(s)
        stats.slots_scanned += n
        if n > 0:
            stats.tiles += (n + TILE_ROWS - 1) // TILE_ROWS
            stats.max_tile_rows = max(stats.max_tile_rows, min(n, TILE_ROWS))


def run_scan(dix: DeviceIndex, query_q: np.ndarray, ranges: np.ndarray, mask, topk: int,
             filters=None, stats: ScanStats | None = None, flags: int = 0) -> TopkResult:
    """B = 1 view of the batched operator."""
    total = int(sum(int(e) - int(s) for s, e in ranges))
    if stats is not None:
        count_scan(ranges, stats)
    if topk <= 0 or total == 0:
        return _empty(topk)
    k_eff = min(int(topk), total)
    op = cached_op(dix, 1, k_eff, ranges, flags)
    q = dix.pad_queries(query_q)
    masks = None
    if mask is not None:
        m = to_dev_u64(mask)
        if m.numel() < dix.n_words:
            m = torch.cat([m, torch.zeros(dix.n_words - m.numel(), dtype=torch.int64,
                                          device=m.device)])
        masks = m.view(1, -1)
    out = op(q, filters, masks=masks)
    ids, scores = out.host(0)
    return TopkResult(item_ids=ids, scores=scores.astype(np.int32), k_requested=topk)


def search_clusters(index, query_q: np.ndarray, clusters, mask: np.ndarray | None, topk: int,
                    stats: ScanStats | None = None) -> TopkResult:
    """Exact integer top-k over the valid, mask-admitted slots of ``clusters``
    (reference ivf.py:285-334), on the GPU."""
    dix = device_index_for(index)
    query_q = np.asarray(query_q, dtype=np.int8)
    if query_q.shape[0] != dix.dim:
        raise DimMismatch(dix.dim, query_q.shape[0])
    return run_scan(dix, query_q, cluster_ranges(dix, clusters), mask, topk, stats=stats)


def probe_centroids(index, query: np.ndarray, nprobe: int) -> np.ndarray:
    """Ids of the nprobe highest float64-dot centroids, ties by ascending id
    (reference ivf.py:261-269); dots in numpy's pairwise order on the GPU."""
    dix = device_index_for(index)
    query = np.asarray(query, dtype=np.float32)
    if query.shape[0] != dix.dim:
        raise DimMismatch(dix.dim, query.shape[0])
    n_clusters = dix.cluster_offsets.shape[0]
    nprobe = min(max(int(nprobe), 1), n_clusters)
    if dix.centroids is None:
        if n_clusters != 1:
            raise ValueError("index has no centroids")
        return np.zeros(1, dtype=np.int64)
    scores = torch.empty(n_clusters, dtype=torch.float64, device=device())
    qv = to_dev(query, torch.float32)
    _native.check(_native.lib().fb_dot_rows_f64(dix.centroids.data_ptr(), n_clusters, dix.dim,
                                                qv.data_ptr(), scores.data_ptr(),
                                                _native.stream_ptr()))
    order = torch.sort(scores, descending=True, stable=True).indices
    return order[:nprobe].cpu().numpy().astype(np.int64)


def quantize_query(dix: DeviceIndex, query) -> torch.Tensor:
    """The query's int8 codes exactly as reference ``quantize_vector`` (quantize.py:72-76)
    computes them: from the float64 value of the caller's array (a float32 array widens
    exactly, so it takes the float32 kernel; anything else is quantised from float64,
    never rounded through float32 first)."""
    x = np.asarray(query)
    if x.dtype != np.float32:
        x = x.astype(np.float64)
    dt = torch.float32 if x.dtype == np.float32 else torch.float64
    return dix.quantize_queries(to_dev(x.reshape(1, -1), dt))


def search(index, query: np.ndarray, nprobe: int, topk: int, mask: np.ndarray | None = None,
           stats: ScanStats | None = None) -> TopkResult:
    """Quantise with the index params, probe, fused scan (reference ivf.py:337-343)."""
    dix = device_index_for(index)
    if np.asarray(query).shape[0] != dix.dim:
        raise DimMismatch(dix.dim, np.asarray(query).shape[0])
    qq = quantize_query(dix, query)
    clusters = probe_centroids(dix, query, nprobe)
    return run_scan(dix, qq, cluster_ranges(dix, clusters), mask, topk, stats=stats)


class IvfSearchOp:
    """Batched IVF-probed co-designed search (reference ``retrieval.codesigned_search`` with
    ``nprobe < n_clusters``, ref/retrieval.py:110-144, for B queries at once).

    On the device: every query's centroid dots (``fb_task_dots_f64``, numpy's pairwise
    order, so probe ties resolve as in ``probe_centroids``) and its top-``nprobe`` clusters
    (stable sort: ties by ascending cluster id). Then, by default (``path="probe"``), the
    grouped scan ``fb_ivf_topk``: one CTA per (query, probed cluster) evaluates the query's
    filter on that cluster's words only and scores its eligible slots -- work proportional
    to nprobe, not to the index -- followed by the exact top-k selection. ``path="masked"``
    runs the exhaustive tensor-core scan with per-query probe masks instead (same results);
    ``"auto"`` (default) takes the grouped scan unless its candidate buffer would pass 8 GB.
    """

    def __init__(self, index, n_queries: int, nprobe: int, k0: int, flags: int = 0,
                 path: str = "auto"):
        if path not in ("probe", "masked", "auto"):
            raise ValueError(f"unknown path {path!r}")
        self.dix = device_index_for(index)
        if self.dix.centroids is None and self.dix.cluster_offsets.shape[0] != 1:
            raise ValueError("index has no centroids")
        self.B = int(n_queries)
        self.C = int(self.dix.cluster_offsets.shape[0])
        self.nprobe = min(max(int(nprobe), 1), self.C)
        self.k0 = int(k0)
        dev = device()
        offs = torch.as_tensor(self.dix.cluster_offsets, dtype=torch.int64, device=dev)
        self._w0 = offs[:, 0] >> 6
        self._w1 = (offs[:, 1] + 63) >> 6
        # the most slots one query can probe: its nprobe largest clusters
        sizes = np.sort(np.asarray(self.dix.cluster_offsets[:, 1] - self.dix.cluster_offsets[:, 0],
                                   dtype=np.int64))[::-1]
        self.cap = int(max(1, sizes[: self.nprobe].sum()))
        if path == "auto":
            # the grouped scan keeps every probed eligible pair: past ~8 GB of candidate
            # keys (nprobe close to the cluster count) the exhaustive masked scan is used
            path = "probe" if self.B * self.cap * 8 <= (8 << 30) else "masked"
        self.path = path
        if path == "masked":
            self.op = TopkOp(self.dix, self.B, self.k0,
                             np.array([[0, self.dix.n_slots]], dtype=np.int64), flags)
            return
        if self.cap >= 1 << 31:
            raise ValueError("probed slot count exceeds the 32-bit candidate buffer")
        need_slot = self.dix.slot_of_rank is None or self.k0 > 24576
        self._cand_key = torch.empty((self.B, self.cap), dtype=torch.int64, device=dev)
        self._cand_slot = (torch.empty((self.B, self.cap), dtype=torch.int32, device=dev)
                           if need_slot else None)
        self._cand_cnt = torch.empty(self.B, dtype=torch.int32, device=dev)
        self._idx_struct = self.dix.struct()

    def probe(self, queries: torch.Tensor) -> torch.Tensor:
        """int64 [B, nprobe] probed cluster ids per query."""
        if self.dix.centroids is None:
            return torch.zeros((self.B, 1), dtype=torch.int64, device=queries.device)
        # the batch as groups of 32 "tasks" over one shared row list (every centroid), so a
        # CTA's staged centroid rows serve 32 queries (fb_task_dots_f64, numpy pairwise order)
        G = 32
        ng = (self.B + G - 1) // G
        u = torch.zeros((ng * G, self.dix.dim), dtype=torch.float32, device=queries.device)
        u[: self.B] = queries.to(torch.float32)
        if getattr(self, "_probe_rows", None) is None:
            self._probe_rows = torch.arange(self.C, dtype=torch.int64,
                                            device=queries.device).repeat(ng, 1)
            self._probe_cnt = torch.full((ng,), self.C, dtype=torch.int32, device=queries.device)
        dots = torch.empty((ng * G, self.C), dtype=torch.float64, device=queries.device)
        _native.check(_native.lib().fb_task_dots_f64(
            self.dix.centroids.data_ptr(), self.C, self.dix.dim, self._probe_rows.data_ptr(),
            self._probe_cnt.data_ptr(), self.C, u.data_ptr(), ng, G, dots.data_ptr(),
            _native.stream_ptr()))
        order = torch.sort(dots[: self.B], dim=1, descending=True, stable=True).indices
        return order[:, : self.nprobe]

    def masks(self, clusters: torch.Tensor) -> torch.Tensor:
        """Per-query probe masks int64 [B, n_words] (u64 bits)."""
        W = self.dix.n_words
        diff = torch.zeros((self.B, W + 1), dtype=torch.int32, device=clusters.device)
        ones = torch.ones_like(clusters, dtype=torch.int32)
        diff.scatter_add_(1, self._w0[clusters], ones)
        diff.scatter_add_(1, self._w1[clusters], -ones)
        cover = torch.cumsum(diff, dim=1)[:, :W] > 0
        return torch.where(cover, torch.full_like(cover, -1, dtype=torch.int64),
                           torch.zeros_like(cover, dtype=torch.int64))

    def probe_words(self, clusters: torch.Tensor) -> torch.Tensor:
        """int64 [B, nprobe, 2] word ranges of the probed clusters."""
        return torch.stack([self._w0[clusters], self._w1[clusters]], dim=2).contiguous()

    def __call__(self, queries: torch.Tensor, filters=None):
        """queries float32 [B, dim] (device) -> TopkOutput; also returns the probed ids."""
        if queries.shape != (self.B, self.dix.dim):
            raise DimMismatch(self.dix.dim, int(queries.shape[-1]))
        clusters = self.probe(queries)
        qq = self.dix.quantize_queries(queries)
        return self.scan(qq, clusters, filters), clusters

    def scan(self, qq: torch.Tensor, clusters: torch.Tensor, filters=None) -> TopkOutput:
        """The filtered top-k of int8 queries ``qq`` [B, dim_pad] over their probed
        ``clusters`` [B, nprobe] (device-resident probe lists: no host round trip, so the
        whole probe + scan can be captured in a CUDA graph)."""
        if self.path == "masked":
            return self.op(qq, filters, masks=self.masks(clusters))
        words = self.probe_words(clusters)
        dev = qq.device
        k = max(self.k0, 1)
        out = TopkOutput(ids=torch.empty((self.B, k), dtype=torch.int64, device=dev),
                         scores=torch.empty((self.B, k), dtype=torch.int32, device=dev),
                         count=torch.empty((self.B,), dtype=torch.int32, device=dev),
                         keys=None, fscores=None)
        prog = filters.struct() if filters is not None else None
        qp = self.dix.qp
        _native.check(_native.lib().fb_ivf_topk(
            ctypes.byref(self._idx_struct), qq.data_ptr(), self.B,
            ctypes.byref(prog) if prog is not None else None, words.data_ptr(), self.nprobe,
            self.k0, self.cap, self._cand_key.data_ptr(),
            self._cand_slot.data_ptr() if self._cand_slot is not None else None,
            self._cand_cnt.data_ptr(), out.ids.data_ptr(), out.scores.data_ptr(),
            out.count.data_ptr(), None, None,
            float(qp.global_min) if qp else 0.0, float(qp.global_max) if qp else 1.0,
            _native.stream_ptr()))
        self._keep = (qq, filters, words)
        return out


# result / counter types: the reference's classes when it is importable (see _refapi)
from ._refapi import bind as _bind  # noqa: E402

_bind(globals(), "ivf", ["TopkResult","ScanStats"])
