"""Device-resident index and the batched filtered top-k operator.

``DeviceIndex`` holds one shard's slot space in HBM in the layout the kernels read
(include/filtra_b200.h ``fb_index_t``): int8 rows padded to a 32-byte multiple, the
transposed Bloom planes ``[M, W]``, validity words, per-slot item ids, the global
id rank (tie-break key) and per-row code sums (dequantised-score term).

``TopkOp`` wraps a ``fb_topk_plan`` (scratch allocated once per shape) and runs the
hot path -- sample -> threshold -> fused filter+scan emit -> exactness check ->
select -- on the current CUDA stream with no host synchronisation.
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._device import IdentityCache, device, round_up, to_dev, to_dev_u64, u64_host
from .bloom import BloomIndex, BloomParams
from .filter_query import FilterBatch
from .quantize import QuantParams, quantize_device


def _u64_order_key(ids: torch.Tensor) -> torch.Tensor:
    """int64 tensor holding uint64 bits -> int64 with the same order as the unsigned ids."""
    return torch.bitwise_xor(ids, -(1 << 63))


@dataclass
class TopkOutput:
    """Device outputs of one batched call: rows sorted by (score desc, item_id asc)."""

    ids: torch.Tensor       # int64 [B, k] holding uint64 item ids
    scores: torch.Tensor    # int32 [B, k]
    count: torch.Tensor     # int32 [B]
    keys: torch.Tensor | None = None      # int64 [B, k] merge keys
    fscores: torch.Tensor | None = None   # float64 [B, k] dequantised scores

    def host(self, q: int) -> tuple[np.ndarray, np.ndarray]:
        n = int(self.count[q])
        return u64_host(self.ids[q, :n]), self.scores[q, :n].cpu().numpy()


class DeviceIndex:
    """One shard of the catalog, resident in HBM."""

    def __init__(self, items: torch.Tensor, valid: torch.Tensor, item_ids: torch.Tensor,
                 n_slots: int, dim: int, bloom: BloomIndex | None = None,
                 qp: QuantParams | None = None, cluster_offsets: np.ndarray | None = None,
                 centroids: torch.Tensor | None = None, id_rank: torch.Tensor | None = None,
                 row_sum: torch.Tensor | None = None):
        self.items = items            # int8 [n_slots_pad, dim_pad]
        self.valid = valid            # int64 [W] (uint64 bits)
        self.item_ids = item_ids      # int64 [n_slots_pad] (uint64 bits)
        self.n_slots = int(n_slots)   # logical (reference) slot count
        self.dim = int(dim)
        self.dim_pad = int(items.shape[1])
        self.bloom = bloom
        self.qp = qp
        self.cluster_offsets = (np.asarray(cluster_offsets, dtype=np.int64)
                                if cluster_offsets is not None
                                else np.array([[0, self.n_slots]], dtype=np.int64))
        self.centroids = centroids
        if id_rank is None:
            id_rank = self._ranks_from_ids()
        self.id_rank = id_rank        # int32 [n_slots_pad] (uint32 bits)
        self.slot_of_rank = self._inverse_ranks(id_rank)  # int32 [n_slots_pad] or None
        self.id_of_rank = (self.item_ids[self.slot_of_rank.long()]  # int64 (u64 bits) or None
                           if self.slot_of_rank is not None else None)
        self.id_dense, self.id_base = self._dense_ids()
        if row_sum is None:
            row_sum = torch.empty(items.shape[0], dtype=torch.int32, device=items.device)
            _native.check(_native.lib().fb_row_sums(items.data_ptr(), items.shape[0], self.dim,
                                                    self.dim_pad, row_sum.data_ptr(),
                                                    _native.stream_ptr()))
        self.row_sum = row_sum
        if bloom is None:
            planes = torch.zeros((1, self.n_words), dtype=torch.int64, device=items.device)
            self._planes = planes
            self.m_bits, self.k_hashes = 1, 1
        else:
            self._planes = bloom.planes_dev
            self.m_bits, self.k_hashes = bloom.params.m_bits, bloom.params.k_hashes
            if bloom.n_words < self.n_words:
                # tile padding (slot space rounded up to 256): zero planes for padded words
                pad = torch.zeros((self.m_bits, self.n_words), dtype=torch.int64,
                                  device=items.device)
                pad[:, : bloom.n_words] = bloom.planes_dev
                self._planes = pad

    @property
    def n_words(self) -> int:
        return int(self.valid.shape[0])

    @property
    def n_slots_pad(self) -> int:
        return int(self.items.shape[0])

    def _valid_slots(self) -> torch.Tensor:
        """bool [n_slots_pad]: the validity bitmap unpacked."""
        bits = torch.arange(64, device=self.items.device, dtype=torch.int64)
        words = self.valid.view(-1, 1)
        return ((words >> bits) & 1).view(-1)[: self.n_slots_pad].bool()

    def _dense_ids(self) -> tuple[int, int]:
        """(1, base) when every valid slot's id is base + its rank (mod 2^64), i.e. the
        valid ids are one contiguous run in rank order; (0, 0) otherwise. With it the
        selection computes output ids instead of gathering them (fb_index_t.id_dense)."""
        if self.id_of_rank is None:
            return 0, 0
        ranks = self.id_rank[self._valid_slots()].to(torch.int64)
        if ranks.numel() == 0:
            return 0, 0
        base = self.id_of_rank[ranks] - ranks  # int64 arithmetic wraps like u64
        b0 = base[:1]
        if not bool((base == b0).all()):
            return 0, 0
        return 1, int(b0.item()) & 0xFFFFFFFFFFFFFFFF

    def _ranks_from_ids(self) -> torch.Tensor:
        """Rank of each valid slot's id among the valid ids (ascending u64)."""
        n = self.n_slots_pad
        vbool = self._valid_slots()
        key = _u64_order_key(self.item_ids)
        key = torch.where(vbool, key, torch.full_like(key, (1 << 63) - 1))
        order = torch.argsort(key, stable=True)
        rank = torch.empty(n, dtype=torch.int64, device=key.device)
        rank[order] = torch.arange(n, device=key.device, dtype=torch.int64)
        return rank.to(torch.int32)

    @staticmethod
    def _inverse_ranks(rank: torch.Tensor) -> torch.Tensor | None:
        """slot_of_rank[id_rank[s]] = s when the ranks are a permutation of the slots
        (always for ranks computed here); None otherwise."""
        n = int(rank.numel())
        r = rank.to(torch.int64)
        if n == 0 or int(r.min()) < 0 or int(r.max()) >= n:
            return None
        inv = torch.full((n,), -1, dtype=torch.int64, device=rank.device)
        inv[r] = torch.arange(n, device=rank.device, dtype=torch.int64)
        if bool((inv < 0).any()):
            return None
        return inv.to(torch.int32)

    @classmethod
    def from_arrays(cls, items_q, valid, item_ids, *, bloom: BloomIndex | None = None,
                    qp: QuantParams | None = None, cluster_offsets=None, centroids=None,
                    id_rank=None) -> "DeviceIndex":
        """Upload reference-layout arrays (int8 rows in slot order, packed validity,
        per-slot u64 ids) -- numpy or CUDA tensors."""
        dev = device()
        items = to_dev(items_q, torch.int8, dev)
        n_slots, dim = int(items.shape[0]), int(items.shape[1])
        dim_pad = round_up(max(dim, 1), 32)
        n_pad = round_up(max(n_slots, 1), 256)  # whole 256-slot tensor-core tiles
        if dim_pad != dim or n_pad != n_slots:
            padded = torch.zeros((n_pad, dim_pad), dtype=torch.int8, device=dev)
            padded[:n_slots, :dim] = items
            items = padded
        v = to_dev_u64(valid, dev)
        if v.numel() < n_pad // 64:
            v = torch.cat([v, torch.zeros(n_pad // 64 - v.numel(), dtype=torch.int64, device=dev)])
        ids = to_dev_u64(item_ids, dev)
        if ids.numel() < n_pad:
            ids = torch.cat([ids, torch.zeros(n_pad - ids.numel(), dtype=torch.int64, device=dev)])
        cent = to_dev(centroids, torch.float32, dev) if centroids is not None else None
        rank = to_dev(id_rank, torch.int32, dev) if id_rank is not None else None
        return cls(items, v, ids, n_slots, dim, bloom=bloom, qp=qp,
                   cluster_offsets=cluster_offsets, centroids=cent, id_rank=rank)

    def struct(self) -> _native.FbIndex:
        return _native.FbIndex(self.items.data_ptr(), self._planes.data_ptr(),
                               self.valid.data_ptr(), self.id_rank.data_ptr(),
                               self.item_ids.data_ptr(), self.row_sum.data_ptr(),
                               self.n_slots_pad, self.n_words, self.dim, self.dim_pad,
                               self.m_bits, self.k_hashes,
                               self.slot_of_rank.data_ptr() if self.slot_of_rank is not None
                               else None,
                               self.id_of_rank.data_ptr() if self.id_of_rank is not None
                               else None, self.id_dense, self.id_base)

    def quantize_queries(self, queries: torch.Tensor) -> torch.Tensor:
        if self.qp is None:
            raise ValueError("index has no quantisation parameters")
        return quantize_device(queries, self.qp, out_stride=self.dim_pad)

    def pad_queries(self, query_q) -> torch.Tensor:
        q = to_dev(query_q, torch.int8)
        if q.dim() == 1:
            q = q.view(1, -1)
        if q.shape[1] == self.dim_pad:
            return q
        out = torch.zeros((q.shape[0], self.dim_pad), dtype=torch.int8, device=q.device)
        out[:, : q.shape[1]] = q
        return out


_REF_CACHE = IdentityCache()


def device_index_for(index, bloom=None) -> DeviceIndex:
    """A ``DeviceIndex`` for either our own index or a reference-shaped ``IvfIndex``
    (duck-typed: ``items_q.data``, ``valid_mask``, ``item_ids``, ``cluster_offsets``),
    uploaded once and cached on the object."""
    if isinstance(index, DeviceIndex):
        return index
    cached = _REF_CACHE.get(index)
    if cached is not None and (bloom is None or cached.bloom is not None):
        return cached
    if bloom is not None and not isinstance(bloom, BloomIndex):
        bloom = BloomIndex(BloomParams(bloom.params.m_bits, bloom.params.k_hashes),
                           bloom.planes, bloom.n_slots)
    qp = index.items_q.params
    dix = DeviceIndex.from_arrays(
        index.items_q.data, index.valid_mask, index.item_ids, bloom=bloom,
        qp=QuantParams(float(qp.global_min), float(qp.global_max)),
        cluster_offsets=np.asarray(index.cluster_offsets, dtype=np.int64),
        centroids=getattr(getattr(index, "centroids", None), "vectors", None))
    _REF_CACHE.put(index, dix)
    return dix


# Plans whose owner was collected while this thread was capturing a CUDA graph: a plan
# destroy is a cudaFree, which would invalidate the capture, so it waits for the next plan
# create (fastpath.py captures single-request graphs; the GC can run a finalizer anywhere).
_DEFERRED_PLANS: list = []
_DEFERRED_LOCK = threading.Lock()


def _capturing() -> bool:
    try:
        import torch
        return torch.cuda.is_current_stream_capturing()
    except Exception:  # noqa: BLE001 -- interpreter shutdown
        return False


def _destroy_plan(plan) -> None:
    if _capturing():
        with _DEFERRED_LOCK:
            _DEFERRED_PLANS.append(plan)
        return
    try:
        _native.load_library().fb_topk_plan_destroy(plan)
    except Exception:  # noqa: BLE001 -- interpreter shutdown
        pass


def _drain_deferred_plans() -> None:
    if not _DEFERRED_PLANS or _capturing():
        return
    with _DEFERRED_LOCK:
        plans, _DEFERRED_PLANS[:] = list(_DEFERRED_PLANS), []
    for p in plans:
        _destroy_plan(p)


class TopkOp:
    """A planned batched filtered top-k over fixed slot ranges."""

    def __init__(self, index: DeviceIndex, n_queries: int, k: int, ranges: np.ndarray,
                 flags: int = 0):
        self.index = index
        self.n_queries = int(n_queries)
        self.k = int(k)
        self.flags = int(flags)
        r = np.ascontiguousarray(np.asarray(ranges, dtype=np.int64).reshape(-1, 2))
        self.ranges = r
        self._idx_struct = index.struct()
        _drain_deferred_plans()
        plan = ctypes.c_void_p()
        _native.check(_native.lib().fb_topk_plan_create(
            ctypes.byref(self._idx_struct), self.n_queries, self.k, r.ctypes.data, r.shape[0],
            self.flags, ctypes.byref(plan)))
        self._plan = plan

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            _destroy_plan(plan)
            self._plan = None

    def _unfiltered_batch(self) -> FilterBatch:
        """A batch of unfiltered queries as a zero-group CNF program (cached): same results
        as no program, but the scan takes the per-hit CNF kernel instead of the bytecode one."""
        if getattr(self, "_null_batch", None) is None:
            from .bloom import BloomParams
            params = BloomParams(self.index.m_bits, self.index.k_hashes)
            self._null_batch = FilterBatch.pack([None] * self.n_queries, params).to_device()
        return self._null_batch

    def stats(self) -> _native.FbStats:
        st = _native.FbStats()
        _native.check(_native.load_library().fb_topk_plan_stats(self._plan, ctypes.byref(st)))
        return st

    def alloc_outputs(self, keys: bool = False, fscores: bool = False) -> TopkOutput:
        dev = self.index.items.device
        B, k = self.n_queries, max(self.k, 1)
        return TopkOutput(
            ids=torch.empty((B, k), dtype=torch.int64, device=dev),
            scores=torch.empty((B, k), dtype=torch.int32, device=dev),
            count=torch.empty((B,), dtype=torch.int32, device=dev),
            keys=torch.empty((B, k), dtype=torch.int64, device=dev) if keys else None,
            fscores=torch.empty((B, k), dtype=torch.float64, device=dev) if fscores else None)

    def __call__(self, queries_q: torch.Tensor, filters: FilterBatch | None = None,
                 masks: torch.Tensor | None = None, out: TopkOutput | None = None,
                 keys: bool = False, fscores: bool = False, stream=None) -> TopkOutput:
        if queries_q.dtype != torch.int8 or queries_q.shape != (self.n_queries, self.index.dim_pad):
            raise ValueError(f"queries_q must be int8 [{self.n_queries}, {self.index.dim_pad}]")
        if out is None:
            out = self.alloc_outputs(keys=keys, fscores=fscores)
        if filters is None:
            filters = self._unfiltered_batch()
        prog = filters.struct()
        qp = self.index.qp
        _native.check(_native.lib().fb_topk_execute(
            self._plan, queries_q.data_ptr(), ctypes.byref(prog) if prog is not None else None,
            masks.data_ptr() if masks is not None else None,
            out.ids.data_ptr(), out.scores.data_ptr(), out.count.data_ptr(),
            out.keys.data_ptr() if out.keys is not None else None,
            out.fscores.data_ptr() if out.fscores is not None else None,
            float(qp.global_min) if qp else 0.0, float(qp.global_max) if qp else 1.0,
            _native.stream_ptr(stream)))
        self._keep = (queries_q, filters, masks)  # keep inputs alive until the next call
        return out


_PLAN_LOCK = threading.Lock()
PLAN_CACHE_SIZE = 64


def cached_op(index: DeviceIndex, n_queries: int, k: int, ranges, flags: int = 0) -> TopkOp:
    """A ``TopkOp`` for (B, k, ranges, flags) from a small per-index LRU, so per-call entry
    points (the B = 1 reference shims, the custom op) do not pay plan creation -- device
    scratch allocation and uploads -- on every call. Plans are per thread: a plan's
    scratch is reused call after call on the calling thread's stream, and the reference's
    ``BatchingServer`` calls concurrently from several threads."""
    r = np.ascontiguousarray(np.asarray(ranges, dtype=np.int64).reshape(-1, 2))
    key = (threading.get_ident(), int(n_queries), int(k), r.tobytes(), int(flags))
    with _PLAN_LOCK:
        cache = index.__dict__.setdefault("_plans", OrderedDict())
        op = cache.get(key)
        if op is not None:
            cache.move_to_end(key)
            return op
    op = TopkOp(index, n_queries, k, r, flags)
    with _PLAN_LOCK:
        cache[key] = op
        while len(cache) > PLAN_CACHE_SIZE:
            cache.popitem(last=False)
    return op


def filtered_topk(index: DeviceIndex, queries_q: torch.Tensor, k: int,
                  filters: FilterBatch | None = None, ranges=None, flags: int = 0,
                  masks: torch.Tensor | None = None, keys: bool = False,
                  fscores: bool = False) -> TopkOutput:
    """One-shot batched filtered top-k (plans and runs)."""
    if ranges is None:
        ranges = np.array([[0, index.n_slots]], dtype=np.int64)
    op = TopkOp(index, queries_q.shape[0], k, ranges, flags)
    res = op(queries_q, filters, masks=masks, keys=keys, fscores=fscores)
    torch.cuda.current_stream().synchronize()
    return res


def merge_topk(scores: torch.Tensor, ids: torch.Tensor, count: torch.Tensor, k_out: int,
               fscores: torch.Tensor | None = None) -> TopkOutput:
    """GPU merge of ``n_lists`` per-query lists sorted by (score desc, item_id asc)
    (``_reduce_topk`` semantics). scores int32 / ids int64(u64 bits) [n_lists, B, k_in];
    count int32 [n_lists, B]."""
    n_lists, B, k_in = scores.shape
    dev = scores.device
    k_out = max(int(k_out), 1)
    out = TopkOutput(ids=torch.empty((B, k_out), dtype=torch.int64, device=dev),
                     scores=torch.empty((B, k_out), dtype=torch.int32, device=dev),
                     count=torch.empty((B,), dtype=torch.int32, device=dev),
                     fscores=(torch.empty((B, k_out), dtype=torch.float64, device=dev)
                              if fscores is not None else None))
    scores = scores.to(torch.int32).contiguous()
    ids = ids.contiguous()
    count = count.to(torch.int32).contiguous()
    fs = fscores.contiguous() if fscores is not None else None
    _native.check(_native.lib().fb_merge_topk(
        scores.data_ptr(), ids.data_ptr(), fs.data_ptr() if fs is not None else None,
        count.data_ptr(), n_lists, B, k_in, k_out, out.ids.data_ptr(), out.scores.data_ptr(),
        out.count.data_ptr(), out.fscores.data_ptr() if out.fscores is not None else None,
        _native.stream_ptr()))
    return out


class PipelinedTopk:
    """Host-in / host-out batched filtered top-k for serving: batch i's scan runs on the
    compute stream while batch i+1's queries and filter arrays are copied in on one copy
    stream and batch i-1's ids / scores are copied out on another (``depth`` slots of
    device and pinned host buffers, ordered by CUDA events; separate streams so a copy-out
    waiting for its scan never holds up the next copy-in).

    With ``overlap`` (default) every slot also has its own plan and compute stream, so batch
    i+1's sampling pass and threshold (about 0.1 ms, two partial waves) fill the SMs that
    batch i's selection leaves idle in its second wave, instead of waiting behind it."""

    def __init__(self, index: DeviceIndex, n_queries: int, k: int, ranges=None,
                 flags: int = 0, depth: int = 2, filters_template=None, overlap: bool = True):
        if ranges is None:
            ranges = np.array([[0, index.n_slots]], dtype=np.int64)
        self.index, self.B, self.k = index, int(n_queries), max(int(k), 1)
        n_ops = depth if overlap else 1
        self.ops = [TopkOp(index, n_queries, k, ranges, flags) for _ in range(n_ops)]
        self.op = self.ops[0]
        self.compute = torch.cuda.current_stream()
        self.streams = [self.compute] + [torch.cuda.Stream() for _ in range(n_ops - 1)]
        self.copy_in = torch.cuda.Stream()
        self.copy_out = torch.cuda.Stream()
        dev = index.items.device
        self.slots = []
        for _ in range(depth):
            batch = None
            if filters_template is not None:
                batch = FilterBatch.pack(filters_template, index.bloom.params).to_device()
                for d in batch._dev:  # read on the slot's compute stream
                    d.record_stream(self.streams[len(self.slots) % len(self.streams)])
            self.slots.append({
                "q": torch.empty((self.B, index.dim), dtype=torch.float32, device=dev),
                "qq": torch.empty((self.B, index.dim_pad), dtype=torch.int8, device=dev),
                "batch": batch, "out": self.op.alloc_outputs(),
                "ids": torch.empty((self.B, self.k), dtype=torch.int64).pin_memory(),
                "scores": torch.empty((self.B, self.k), dtype=torch.int32).pin_memory(),
                "count": torch.empty((self.B,), dtype=torch.int32).pin_memory(),
                "h2d": torch.cuda.Event(), "comp": torch.cuda.Event(), "d2h": torch.cuda.Event(),
            })
        self._n = 0

    @staticmethod
    def _same_shape(batch: FilterBatch, filters: FilterBatch) -> bool:
        """True when ``filters`` can be copied into ``batch``'s device arrays: the same
        scalar metadata (program form, leaf/plane/column counts, CNF layout) and the same
        count, shape and dtype of every array."""
        if batch is None or batch.meta() != filters.meta():
            return False
        dev, host = batch._dev, filters.host_arrays()
        return len(dev) == len(host) and all(
            tuple(d.shape) == tuple(h.shape) and d.element_size() == h.itemsize
            for d, h in zip(dev, host))

    def submit(self, host_queries: torch.Tensor, filters: FilterBatch | None = None) -> int:
        """Enqueue one batch: float32 queries [B, dim] (pinned for an asynchronous copy) and
        the batch's packed filters (``FilterBatch.pack``; ``.pin()`` it for asynchronous
        copies), or None to reuse the slot's filters. A batch with the slot's shape is
        copied into the slot's device arrays on the copy stream; any other batch replaces
        the slot's (one upload). Returns a ticket for ``result``."""
        if tuple(host_queries.shape) != (self.B, self.index.dim):
            raise ValueError(f"queries must be [{self.B}, {self.index.dim}], got "
                             f"{tuple(host_queries.shape)}")
        if filters is not None and filters.n_queries != self.B:
            raise ValueError(f"filter batch holds {filters.n_queries} programs, expected {self.B}")
        t = self._n
        s = self.slots[t % len(self.slots)]
        op, cs = self.ops[t % len(self.ops)], self.streams[t % len(self.streams)]
        self._n += 1
        self.copy_in.wait_event(s["comp"])       # the slot's inputs are no longer read
        if filters is not None and not self._same_shape(s["batch"], filters):
            # another shape (e.g. a fresh batch of request filters): new device arrays for
            # the slot, allocated and filled on the copy stream from pinned staging so the
            # host never waits for the scan in flight
            fresh = filters.clone_host()
            with torch.cuda.stream(self.copy_in):
                dev = []
                for h in filters.pin().pinned_arrays():
                    d = torch.empty(h.shape, dtype=h.dtype, device=s["q"].device)
                    d.copy_(h, non_blocking=True)
                    d.record_stream(cs)
                    dev.append(d)
            fresh._dev = tuple(dev)
            s["batch"] = fresh
            filters = None
        with torch.cuda.stream(self.copy_in):
            s["q"].copy_(host_queries, non_blocking=True)
            if filters is not None:
                for d, h in zip(s["batch"]._dev, filters.pinned_arrays()):
                    d.copy_(h, non_blocking=True)
            s["h2d"].record(self.copy_in)
        cs.wait_event(s["h2d"])
        cs.wait_event(s["d2h"])                  # the slot's outputs were copied out
        with torch.cuda.stream(cs):
            quantize_device(s["q"], self.index.qp, out_stride=self.index.dim_pad, out=s["qq"])
            res = op(s["qq"], s["batch"], out=s["out"])
        s["comp"].record(cs)
        self.copy_out.wait_event(s["comp"])
        with torch.cuda.stream(self.copy_out):
            s["ids"].copy_(res.ids, non_blocking=True)
            s["scores"].copy_(res.scores, non_blocking=True)
            s["count"].copy_(res.count, non_blocking=True)
            s["d2h"].record(self.copy_out)
        return t

    def result(self, ticket: int):
        """Host (ids u64-bits int64 [B, k], int32 scores [B, k], int32 counts [B]) of a
        submitted batch (waits for its copy-out; valid until the slot is reused)."""
        s = self.slots[ticket % len(self.slots)]
        s["d2h"].synchronize()
        return s["ids"], s["scores"], s["count"]

    def done_event(self, ticket: int):
        return self.slots[ticket % len(self.slots)]["d2h"]
