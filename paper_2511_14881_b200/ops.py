"""PyTorch custom operators for the hot path (``torch.ops.filtra_b200.*``).

north_star asks for the new path to be "a drop-in PyTorch custom op"; these are registered
with ``torch.library.custom_op`` and carry ``register_fake`` kernels, so they trace under
FakeTensor / ``torch.compile`` / ``torch.export`` as opaque ops with known output shapes,
and dispatch to the C-ABI library (``include/filtra_b200.h``) on CUDA tensors:

* ``filtra_b200::filtered_topk(index, queries_q, k, ranges, filter_arrays, filter_meta,
  flags) -> (ids, scores, count)`` -- the batched co-designed search (reference
  retrieval.py:110-144 / ivf.py:285-334 for B queries): ``fb_topk_execute`` with a cached
  per-thread plan. ``index`` is a handle from ``index_handle(DeviceIndex)`` (the index is
  device-resident state, like a weight); ``filter_arrays`` / ``filter_meta`` are
  ``FilterBatch.device_arrays()`` / ``FilterBatch.meta()`` (empty = unfiltered).
* ``filtra_b200::merge_topk(scores, ids, count, k) -> (ids, scores, count)`` -- the shard
  merge (reference serve.py:98-100 ``_reduce_topk``), ``fb_merge_topk``.
* ``filtra_b200::quantize(x, gmin, gmax, out_stride) -> int8`` -- ``quantize_vector``
  (reference quantize.py:72-76) for a batch, ``fb_quantize(_f64)``.

ids are int64 tensors holding the u64 item ids' bits; rows are sorted by (score desc,
item_id asc); ``count[b]`` < k when fewer items are eligible.
"""

from __future__ import annotations

import itertools
import threading
import weakref

import numpy as np
import torch

from . import _native
from .engine import DeviceIndex, cached_op, merge_topk as _merge_topk
from .filter_query import FilterBatch
from .quantize import QuantParams, quantize_device

_HANDLES: dict[int, "weakref.ref[DeviceIndex]"] = {}
_NEXT = itertools.count(1)
_LOCK = threading.Lock()


def index_handle(index: DeviceIndex) -> int:
    """Stable integer handle of a device index for the custom op (held weakly)."""
    h = index.__dict__.get("_op_handle")
    if h is None:
        with _LOCK:
            h = next(_NEXT)
            _HANDLES[h] = weakref.ref(index)
            index._op_handle = h
    return h


def _index(h: int) -> DeviceIndex:
    ref = _HANDLES.get(int(h))
    dix = ref() if ref is not None else None
    if dix is None:
        raise ValueError(f"unknown or released device index handle {h}")
    return dix


@torch.library.custom_op("filtra_b200::filtered_topk", mutates_args=(), device_types="cuda")
def filtered_topk(index: int, queries_q: torch.Tensor, k: int, ranges: list[int],
                  filter_arrays: list[torch.Tensor], filter_meta: list[int],
                  flags: int = 0) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    dix = _index(index)
    B = int(queries_q.shape[0])
    r = np.asarray(ranges, dtype=np.int64).reshape(-1, 2) if len(ranges) else \
        np.array([[0, dix.n_slots]], dtype=np.int64)
    op = cached_op(dix, B, k, r, flags)
    batch = None
    if len(filter_arrays):
        batch = _DeviceFilters(list(filter_arrays), list(filter_meta))
    out = op(queries_q.contiguous(), batch)
    return out.ids, out.scores, out.count


@filtered_topk.register_fake
def _(index, queries_q, k, ranges, filter_arrays, filter_meta, flags=0):
    B, kk = queries_q.shape[0], max(int(k), 1)
    return (queries_q.new_empty((B, kk), dtype=torch.int64),
            queries_q.new_empty((B, kk), dtype=torch.int32),
            queries_q.new_empty((B,), dtype=torch.int32))


class _DeviceFilters:
    """A FilterBatch view over arrays that already live on the device (op boundary)."""

    def __init__(self, arrays, meta):
        if len(meta) != len(FilterBatch.META_FIELDS):
            raise ValueError(f"filter_meta needs {len(FilterBatch.META_FIELDS)} fields")
        self._arrays, self._meta = arrays, meta
        self.n_queries = int(meta[0])

    def struct(self):
        return FilterBatch.struct_from(self._arrays, self._meta)


@torch.library.custom_op("filtra_b200::merge_topk", mutates_args=(), device_types="cuda")
def merge_topk(scores: torch.Tensor, ids: torch.Tensor, count: torch.Tensor,
               k: int) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    out = _merge_topk(scores, ids, count, k)
    return out.ids, out.scores, out.count


@merge_topk.register_fake
def _(scores, ids, count, k):
    B, kk = scores.shape[1], max(int(k), 1)
    return (ids.new_empty((B, kk)), scores.new_empty((B, kk), dtype=torch.int32),
            count.new_empty((B,), dtype=torch.int32))


@torch.library.custom_op("filtra_b200::quantize", mutates_args=(), device_types="cuda")
def quantize(x: torch.Tensor, gmin: float, gmax: float, out_stride: int) -> torch.Tensor:
    return quantize_device(x, QuantParams(gmin, gmax), out_stride=out_stride)


@quantize.register_fake
def _(x, gmin, gmax, out_stride):
    rows = x.shape[0] if x.dim() == 2 else 1
    return x.new_empty((rows, out_stride), dtype=torch.int8)


def search_batch(index: DeviceIndex, queries: torch.Tensor, k: int,
                 filters: FilterBatch | None = None, ranges=None, flags: int = 0):
    """Float queries [B, dim] (CUDA) -> (ids, scores, count) through the custom ops."""
    qp = index.qp
    qq = torch.ops.filtra_b200.quantize(queries, float(qp.global_min), float(qp.global_max),
                                        index.dim_pad)
    rl = [] if ranges is None else [int(x) for x in np.asarray(ranges).reshape(-1)]
    fa, fm = ([], []) if filters is None else (filters.device_arrays(), filters.meta())
    return torch.ops.filtra_b200.filtered_topk(index_handle(index), qq, int(k), rl, fa, fm,
                                               int(flags))


__all__ = ["filtered_topk", "merge_topk", "quantize", "index_handle", "search_batch"]
_ = _native  # the ops dispatch through the C-ABI library
