"""Item-sharded search across GPUs and the shard merge (reference serve.py:58-145).

The reference fans a request out to in-process shards, concatenates their local
top-k lists and reduces them with ``_reduce_topk`` (a global
``lexsort((ids, -scores))[:k]``, serve.py:98-100). Here one process drives one GPU
and one shard: every rank runs the fused filtered top-k on its own slot range, the
per-rank (score, id) lists are exchanged with one NCCL ``all_gather`` over NVLink, and
``fb_merge_topk`` merges them on the GPU. Quantisation parameters are global (shared
by all shards), so the merged answer is bit-identical to the unsharded search.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from ._device import to_dev, to_dev_u64, u64_host
from .engine import DeviceIndex, TopkOp, TopkOutput, merge_topk


def _reduce_topk(ids: np.ndarray, scores: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """Drop-in for the reference shard reduce: the concatenation of per-shard lists
    (each sorted by (score desc, id asc)) is split into its sorted runs and merged on
    the GPU. Any input order is accepted (a run may have length 1)."""
    ids = np.asarray(ids, dtype=np.uint64)
    scores = np.asarray(scores).astype(np.int64)
    n = len(ids)
    if n == 0 or k <= 0:
        return ids[:0], scores[:0].astype(np.int32)
    # run boundaries: position i starts a new run when pair i is not after pair i-1
    breaks = np.flatnonzero((scores[1:] > scores[:-1]) |
                            ((scores[1:] == scores[:-1]) & (ids[1:] <= ids[:-1]))) + 1
    starts = np.concatenate([[0], breaks])
    ends = np.concatenate([breaks, [n]])
    lens = ends - starts
    n_lists, k_in = len(starts), int(lens.max())
    sc = np.zeros((n_lists, 1, k_in), dtype=np.int32)
    iv = np.zeros((n_lists, 1, k_in), dtype=np.uint64)
    for li, (s, e) in enumerate(zip(starts, ends)):
        sc[li, 0, : e - s] = scores[s:e]
        iv[li, 0, : e - s] = ids[s:e]
    out = merge_topk(to_dev(sc, torch.int32), to_dev_u64(iv).view(n_lists, 1, k_in),
                     to_dev(lens.reshape(n_lists, 1), torch.int32), min(k, n))
    cnt = int(out.count[0])
    return u64_host(out.ids[0, :cnt]), out.scores[0, :cnt].cpu().numpy()


def shard_ranges(n_items: int, world: int) -> list[tuple[int, int]]:
    """Contiguous 64-aligned item partition, one shard per rank."""
    words = (n_items + 63) // 64
    per = (words + world - 1) // world
    out = []
    for r in range(world):
        w0, w1 = min(r * per, words), min((r + 1) * per, words)
        out.append((min(w0 * 64, n_items), min(w1 * 64, n_items)))
    return out


def exchange_topk(local_scores: torch.Tensor, local_ids: torch.Tensor, local_count: torch.Tensor,
                  group=None) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """All-gather the per-rank (scores, ids, count) lists: [world, B, k] / [world, B]."""
    world = dist.get_world_size(group)
    gs = [torch.empty_like(local_scores) for _ in range(world)]
    gi = [torch.empty_like(local_ids) for _ in range(world)]
    gc = [torch.empty_like(local_count) for _ in range(world)]
    dist.all_gather(gs, local_scores.contiguous(), group=group)
    dist.all_gather(gi, local_ids.contiguous(), group=group)
    dist.all_gather(gc, local_count.contiguous(), group=group)
    return torch.stack(gs), torch.stack(gi), torch.stack(gc)


@dataclass
class ShardedSearch:
    """One rank's part of an item-sharded filtered top-k.

    ``op`` is this rank's planned ``TopkOp`` over its local shard (ids are the global
    item ids). ``__call__`` returns the global top-k on every rank.
    """

    op: TopkOp
    group: object = None
    merge: object = None  # injectable merge (tests on CPU/gloo); default: fb_merge_topk

    def __call__(self, queries_q: torch.Tensor, filters=None, k: int | None = None) -> TopkOutput:
        local = self.op(queries_q, filters)
        k = self.op.k if k is None else k
        s, i, c = exchange_topk(local.scores, local.ids, local.count, self.group)
        merge = self.merge or merge_topk
        return merge(s, i, c, k)


__all__ = ["_reduce_topk", "shard_ranges", "exchange_topk", "ShardedSearch", "DeviceIndex"]
