"""Co-designed filtered search (reference retrieval.py:57-144).

``codesigned_search`` keeps the reference signature. The reference probes, evaluates
the compiled filter over each probed cluster's 64-aligned range into a zero mask,
quantises, then scans. Here the filter program is evaluated *inside* the scan
kernel on the probed ranges only, so the Bloom mask never leaves the SM; the result
is identical because a range-restricted evaluation equals the restriction of the
full one (reference filter_query.py:319-323).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, bitset
from ._device import to_dev
from .bloom import FilterStats
from .engine import device_index_for
from .errors import DimMismatch
from .filter_query import CompiledFilter, FilterBatch
from .ivf import (ScanStats, TopkResult, cluster_ranges, probe_centroids, quantize_query,
                  run_scan)


@dataclass
class StageTimings:
    probe_us: int = 0
    filter_us: int = 0
    scan_us: int = 0
    overarch_us: int = 0
    total_us: int = 0

    def as_dict(self) -> dict[str, int]:
        return {"probe_us": self.probe_us, "filter_us": self.filter_us,
                "scan_us": self.scan_us, "overarch_us": self.overarch_us,
                "total_us": self.total_us}


def codesigned_search(ivf, bloom_index, cf: CompiledFilter | None, query: np.ndarray,
                      nprobe: int, k0: int, scan_stats: ScanStats | None = None,
                      filter_stats: FilterStats | None = None,
                      timings: StageTimings | None = None) -> TopkResult:
    """Probe, then one fused filter+scan launch sequence over the probed clusters (one
    CUDA-graph replay per call, fastpath.py; ``FB_EAGER_B1=1`` launches step by step)."""
    if not _native.env_flag("FB_EAGER_B1"):
        from . import fastpath
        t0 = time.perf_counter()
        r = fastpath.codesigned_search(ivf, bloom_index, cf, query, nprobe, k0,
                                       scan_stats=scan_stats, filter_stats=filter_stats)
        if r is not None:
            if timings is not None:
                timings.scan_us += int((time.perf_counter() - t0) * 1e6)
            return r
    dix = device_index_for(ivf, bloom=bloom_index if cf is not None else None)
    raw_query = query
    query = np.asarray(query, dtype=np.float32)  # probing is float32 (ref ivf.py:263)
    if query.shape[0] != dix.dim:
        raise DimMismatch(dix.dim, query.shape[0])
    t0 = time.perf_counter()
    clusters = probe_centroids(dix, query, nprobe)
    t1 = time.perf_counter()
    ranges = cluster_ranges(dix, clusters)
    ranges = ranges[ranges[:, 1] > ranges[:, 0]] if len(ranges) else ranges
    filters = None
    if cf is not None:
        if dix.bloom is None:
            if bloom_index is None:
                raise ValueError("a filter needs the Bloom index")
            dix = device_index_for(ivf, bloom=bloom_index)
        filters = FilterBatch.pack([cf], dix.bloom.params)
        if filter_stats is not None:
            words = int(sum(((int(e) + 63) >> 6) - (int(s) >> 6) for s, e in ranges))
            filter_stats.slots_evaluated += words * bitset.WORD_BITS
            filter_stats.words_read += int(filters.push_leaf_bits[0]) * words
    qq = quantize_query(dix, raw_query)  # quantised from float64 (ref quantize.py:73)
    result = run_scan(dix, qq, ranges, None, k0, filters=filters, stats=scan_stats)
    t2 = time.perf_counter()
    if timings is not None:
        timings.probe_us += int((t1 - t0) * 1e6)
        timings.scan_us += int((t2 - t1) * 1e6)
    return result


# result / counter types: the reference's classes when it is importable (see _refapi)
from ._refapi import bind as _bind  # noqa: E402

_bind(globals(), "retrieval", ["StageTimings"])
