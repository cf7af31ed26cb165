"""Transposed Bloom-signature index, resident in HBM.

Same API and bit layout as the reference (bloom.py:1-192): plane ``p`` is a packed
bit vector over all slots, ``planes`` is ``uint64[M, ceil(n_slots/64)]``. Hashing
runs in the C library (host), plane construction and leaf evaluation run as
sm_100a kernels (``fb_bloom_build`` / ``fb_filter_eval``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._device import device, to_dev, to_dev_u64, u64_host

HASH_SCHEME_FNV1A_SPLITMIX = 1
_FNV_OFFSET = 0xCBF29CE484222325
_FNV_PRIME = 0x100000001B3
_U64 = 0xFFFFFFFFFFFFFFFF
_GAMMA = 0x9E3779B97F4A7C15


@dataclass(frozen=True)
class BloomParams:
    """Signature width M, hash count K, pinned hash recipe (reference bloom.py:26-38)."""

    m_bits: int = 1024
    k_hashes: int = 5
    hash_scheme_id: int = HASH_SCHEME_FNV1A_SPLITMIX

    def __post_init__(self):
        if self.m_bits < 1 or self.k_hashes < 1:
            raise ValueError("m_bits and k_hashes must be >= 1")
        if self.hash_scheme_id != HASH_SCHEME_FNV1A_SPLITMIX:
            raise ValueError(f"unknown hash_scheme_id {self.hash_scheme_id}")


@dataclass(frozen=True)
class QueryBloom:
    """Sorted, de-duplicated hash positions of one (feature, value) leaf."""

    set_bits: tuple[int, ...]


@dataclass
class FilterStats:
    """Filter work counters (reference bloom.py:147-157), filled analytically."""

    words_read: int = 0
    slots_evaluated: int = 0


def hash_seed(feature_id: int, value: int) -> int:
    """FNV-1a-64 of the 16-byte little-endian ``feature_id || value`` (reference
    bloom.py:65-68). Host scalar helper; the batched path hashes in C."""
    h = _FNV_OFFSET
    for byte in int(feature_id).to_bytes(8, "little") + int(value).to_bytes(8, "little"):
        h = ((h ^ byte) * _FNV_PRIME) & _U64
    return h


def hash_positions_batch(fids, values, params: BloomParams) -> tuple[np.ndarray, np.ndarray]:
    """Positions of many leaves via ``fb_hash_leaves``: int32 ``[n, K]`` (-1 padded) and
    the per-leaf count."""
    fids = np.ascontiguousarray(np.asarray(fids, dtype=np.uint64))
    values = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
    n = len(fids)
    k = params.k_hashes
    pos = np.empty((n, k), dtype=np.int32)
    cnt = np.empty(n, dtype=np.int32)
    lib = _native.load_library()
    _native.check(lib.fb_hash_leaves(fids.ctypes.data, values.ctypes.data, n, params.m_bits, k,
                                     pos.ctypes.data, cnt.ctypes.data))
    return pos, cnt


def hash_positions(feature_id: int, value: int, params: BloomParams) -> QueryBloom:
    """Bit positions selected by one (feature, value) leaf (reference bloom.py:86-88)."""
    pos, cnt = hash_positions_batch([feature_id], [value], params)
    return QueryBloom(set_bits=tuple(int(p) for p in pos[0, : cnt[0]]))


class BloomIndex:
    """M transposed bit planes over the slot space (reference bloom.py:91-111).

    ``planes_dev`` is the HBM copy (int64-typed tensor holding the uint64 words);
    ``planes`` is a lazily downloaded numpy view for drop-in callers.
    """

    def __init__(self, params: BloomParams, planes, n_slots: int):
        self.params = params
        self.n_slots = int(n_slots)
        if isinstance(planes, torch.Tensor):
            self.planes_dev = planes if planes.dtype == torch.int64 else planes.view(torch.int64)
            self._planes_host = None
        else:
            self._planes_host = np.ascontiguousarray(np.asarray(planes, dtype=np.uint64))
            self.planes_dev = to_dev_u64(self._planes_host)

    @property
    def planes(self) -> np.ndarray:
        if self._planes_host is None:
            self._planes_host = u64_host(self.planes_dev)
        return self._planes_host

    @property
    def n_words(self) -> int:
        return int(self.planes_dev.shape[1])

    @property
    def plane_bytes(self) -> int:
        return int(self.planes_dev.numel() * 8)

    def signature(self, slot: int) -> np.ndarray:
        word = self.planes[:, slot >> 6]
        return ((word >> np.uint64(slot & 63)) & np.uint64(1)).astype(bool)


def build_bloom_arrays(fids, values, slots, n_slots: int, params: BloomParams) -> BloomIndex:
    """Planes from flat (fid, value, slot) arrays (host numpy or CUDA tensors) with the
    ``fb_bloom_build`` kernel: one thread per pair, 64-bit atomicOr per position."""
    lib = _native.lib()
    dev = device()
    f = to_dev_u64(fids, dev)
    v = to_dev_u64(values, dev)
    s = to_dev(slots, torch.int64, dev)
    nw = (int(n_slots) + 63) // 64
    planes = torch.empty((params.m_bits, nw), dtype=torch.int64, device=dev)
    _native.check(lib.fb_bloom_build(f.data_ptr(), v.data_ptr(), s.data_ptr(), int(f.numel()),
                                     int(n_slots), params.m_bits, params.k_hashes,
                                     planes.data_ptr(), _native.stream_ptr()))
    return BloomIndex(params=params, planes=planes, n_slots=n_slots)


def build_bloom(slot_features, params: BloomParams, n_slots: int | None = None) -> BloomIndex:
    """Populate planes from per-slot feature pairs in the caller's slot order
    (reference bloom.py:114-144)."""
    if n_slots is None:
        n_slots = len(slot_features)
    if len(slot_features) > n_slots:
        raise ValueError("more feature lists than slots")
    counts = np.fromiter((len(p) for p in slot_features), dtype=np.int64, count=len(slot_features))
    total = int(counts.sum())
    fids = np.empty(total, dtype=np.uint64)
    vals = np.empty(total, dtype=np.uint64)
    i = 0
    for pairs in slot_features:
        for fid, val in pairs:
            fids[i] = fid
            vals[i] = val
            i += 1
    slots = np.repeat(np.arange(len(slot_features), dtype=np.int64), counts)
    return build_bloom_arrays(fids, vals, slots, n_slots, params)


def bloom_eval_leaf(index: BloomIndex, qb: QueryBloom, out: np.ndarray | None = None,
                    word_range: tuple[int, int] | None = None,
                    stats: FilterStats | None = None) -> np.ndarray:
    """AND of the leaf's planes over a word range on the GPU (reference bloom.py:160-181);
    empty leaf -> all ones; reads ``len(set_bits) * width`` words."""
    from .filter_query import FilterBatch  # local: avoids an import cycle
    w0, w1 = word_range if word_range is not None else (0, index.n_words)
    width = w1 - w0
    if out is None:
        out = np.empty(width, dtype=np.uint64)
    if width <= 0:
        return out
    batch = FilterBatch.from_leaf(qb, index.params)
    res = batch.evaluate(index, None, w0, w1, apply_valid=False)
    out[:] = res[0]
    if stats is not None and qb.set_bits:
        stats.words_read += len(qb.set_bits) * width
    return out


def bloom_fpr_theoretical(params: BloomParams, n_inserted: int) -> float:
    """(1 - (1 - 1/M)^(K n))^K (reference bloom.py:184-187)."""
    m, k = params.m_bits, params.k_hashes
    return float((1.0 - (1.0 - 1.0 / m) ** (k * n_inserted)) ** k)


def heuristic_bits(max_feature_values: int, k_hashes: int, collision_buffer: int = 3) -> int:
    """max values per item x K x safety buffer (reference bloom.py:190-192)."""
    return max_feature_values * k_hashes * collision_buffer


def positions_from_seed(seed: int, params: BloomParams) -> tuple[int, ...]:
    """``sorted({splitmix64(seed ^ i*GAMMA) mod M})`` (reference bloom.py:71-83)."""
    out = set()
    for i in range(params.k_hashes):
        z = seed ^ ((i * _GAMMA) & _U64)
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _U64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _U64
        out.add((z ^ (z >> 31)) % params.m_bits)
    return tuple(sorted(out))



# result / counter types: the reference's classes when it is importable (see _refapi)
from ._refapi import bind as _bind  # noqa: E402

_bind(globals(), "bloom", ["FilterStats"])
