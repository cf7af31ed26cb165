"""Synthetic workload of BASELINE.json / SURVEY.md §8(d), generated on the GPU.

Items follow the reference generator's semantics (catalog.py:184-218): ``N/1000``
Gaussian centres, L2-normalised; uniform blob ids; N(0, 0.08^2) noise; L2-normalised
float32 rows; ``item_id = index``. Features follow ``default_features_spec``
(catalog.py:221-223): six features, ten distinct values per item. One global
min/max quantisation; Bloom M=1024, K=5. The "4-attribute" filter is
``AND(OR(f1 in S1), OR(f2 in S2), OR(f3 in S3), OR(f4 in S4))`` with
|S| = (17, 17, 14, 11) drawn without replacement (PAPER.md:175-185 shape, ~10%
selectivity). Queries are catalogue rows plus N(0, 0.05^2) noise (cli.py:160-162).

This is bench/test input generation, not part of the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .bloom import BloomParams, build_bloom_arrays
from .engine import DeviceIndex
from .filter_query import And, CompiledFilter, FilterBatch, Leaf, Or, compile_filter
from .quantize import QuantParams, quantize_device

DEFAULT_FEATURES = [(1, 50, 2), (2, 50, 2), (3, 40, 2), (4, 30, 2), (5, 20, 1), (6, 10, 1)]
FOUR_ATTR_SIZES = (17, 17, 14, 11)


@dataclass
class Workload:
    index: DeviceIndex
    queries: torch.Tensor            # float32 [B, dim] (CUDA)
    queries_q: torch.Tensor          # int8 [B, dim_pad] (CUDA)
    filters: list[CompiledFilter | None]
    batch: FilterBatch | None
    qp: QuantParams
    n_items: int
    dim: int


def _normalize(x: torch.Tensor) -> torch.Tensor:
    n = torch.linalg.vector_norm(x.double(), dim=1, keepdim=True)
    n[n == 0] = 1.0
    return (x / n.float()).float()


def make_items(n_items: int, dim: int, seed: int, dev, blob_std: float = 0.08,
               chunk: int = 1 << 22) -> torch.Tensor:
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    n_clusters = max(1, n_items // 1000)
    centers = _normalize(torch.randn((n_clusters, dim), generator=g, device=dev))
    out = torch.empty((n_items, dim), dtype=torch.float32, device=dev)
    for s in range(0, n_items, chunk):
        e = min(n_items, s + chunk)
        blob = torch.randint(0, n_clusters, (e - s,), generator=g, device=dev)
        noise = torch.randn((e - s, dim), generator=g, device=dev) * blob_std
        out[s:e] = _normalize(centers[blob] + noise)
    return out


def make_feature_pairs(n_items: int, seed: int, dev, spec=DEFAULT_FEATURES):
    """(fid, value, slot) arrays: per feature, ``vpi`` distinct uniform values."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed + 1)
    fids, vals, slots = [], [], []
    ar = torch.arange(n_items, device=dev, dtype=torch.int64)
    for fid, card, vpi in spec:
        take = min(vpi, card)
        if take >= 1:
            a = torch.randint(0, card, (n_items,), generator=g, device=dev)
            fids.append(torch.full((n_items,), fid, dtype=torch.int64, device=dev))
            vals.append(a)
            slots.append(ar)
        if take >= 2:
            b = (a + 1 + torch.randint(0, card - 1, (n_items,), generator=g, device=dev)) % card
            fids.append(torch.full((n_items,), fid, dtype=torch.int64, device=dev))
            vals.append(b)
            slots.append(ar)
        if take > 2:
            raise NotImplementedError("values_per_item > 2 is not used by the default spec")
    return torch.cat(fids), torch.cat(vals), torch.cat(slots)


def four_attribute_filter(rng: np.random.Generator, sizes=FOUR_ATTR_SIZES, spec=DEFAULT_FEATURES):
    groups = []
    for (fid, card, _), size in zip(spec, sizes):
        vals = rng.choice(card, size=min(size, card), replace=False)
        groups.append(Or(tuple(Leaf(fid, int(v)) for v in vals)))
    return And(tuple(groups))


def make_workload(n_items: int, n_queries: int, dim: int = 128, seed: int = 1,
                  filter_seed: int = 7, filter_sizes=FOUR_ATTR_SIZES, filtered: bool = True,
                  params: BloomParams = BloomParams(), id_base: int = 0,
                  reduce_minmax=None, share_queries=None) -> Workload:
    """One shard of the synthetic catalogue.

    Sharded use: ``reduce_minmax(lo, hi) -> (lo, hi)`` turns the
    shard's min/max into the catalogue's (e.g. an all-reduce MIN/MAX), so every shard
    quantises with ONE global ``QuantParams``; ``id_base`` offsets this shard's item ids
    (global ids are fixed before the device index derives its rank tables);
    ``share_queries(q) -> q`` replaces the float queries (e.g. a broadcast from rank 0)
    before they are quantised."""
    dev = torch.device("cuda", torch.cuda.current_device())
    emb = make_items(n_items, dim, seed, dev)
    lo, hi = float(emb.min()), float(emb.max())
    if reduce_minmax is not None:
        lo, hi = reduce_minmax(lo, hi)
    qp = QuantParams(lo, hi)
    dim_pad = (dim + 31) // 32 * 32
    n_pad = (n_items + 255) // 256 * 256  # whole 256-slot tensor-core tiles
    items = torch.zeros((n_pad, dim_pad), dtype=torch.int8, device=dev)
    chunk = 1 << 22
    for s in range(0, n_items, chunk):
        e = min(n_items, s + chunk)
        quantize_device(emb[s:e], qp, out_stride=dim_pad, out=items[s:e])
    # queries: catalogue rows + noise
    g = torch.Generator(device=dev)
    g.manual_seed(seed + 2)
    rows = torch.randint(0, n_items, (n_queries,), generator=g, device=dev)
    queries = emb[rows] + torch.randn((n_queries, dim), generator=g, device=dev) * 0.05
    queries = queries.float().contiguous()
    if share_queries is not None:
        queries = share_queries(queries).float().contiguous()
    del emb
    # validity: all real items; padding cleared
    n_words = n_pad // 64
    valid = torch.zeros((n_words,), dtype=torch.int64, device=dev)
    valid[: n_items // 64] = -1
    rem = n_items % 64
    if rem:
        valid[n_items // 64] = (1 << rem) - 1
    ids = torch.arange(n_pad, dtype=torch.int64, device=dev) + int(id_base)
    ids[n_items:] = 0
    rank = torch.arange(n_pad, dtype=torch.int32, device=dev)
    fid, val, slot = make_feature_pairs(n_items, seed, dev)
    bloom = build_bloom_arrays(fid, val, slot, n_pad, params)
    del fid, val, slot
    index = DeviceIndex(items, valid, ids, n_pad, dim, bloom=bloom, qp=qp, id_rank=rank)
    queries_q = quantize_device(queries, qp, out_stride=dim_pad)
    filters: list[CompiledFilter | None]
    if filtered:
        rng = np.random.default_rng(filter_seed)
        filters = [compile_filter(four_attribute_filter(rng, filter_sizes), params)
                   for _ in range(n_queries)]
        batch = FilterBatch.pack(filters, params)
    else:
        filters = [None] * n_queries
        batch = None
    torch.cuda.synchronize()
    return Workload(index=index, queries=queries, queries_q=queries_q, filters=filters,
                    batch=batch, qp=qp, n_items=n_items, dim=dim)
