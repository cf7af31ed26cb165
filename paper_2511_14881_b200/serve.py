"""Item-sharded search across GPUs and the shard merge (reference serve.py:58-145).

The reference fans a request out to in-process shards, concatenates their local
top-k lists and reduces them with ``_reduce_topk`` (a global
``lexsort((ids, -scores))[:k]``, serve.py:98-100). Here one process drives one GPU
and one shard: every rank runs the fused filtered top-k on its own slot range, the
per-rank (score, id) lists are exchanged over NVLink (by default one NCCL all-to-all
to the rank owning each query slice; ``all_gather`` and a pruned variant are kept), and
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
    raw = np.asarray(scores)
    scores = raw.astype(np.int64)
    if raw.dtype.kind == "f" and raw.size and not np.array_equal(scores, raw):
        # the GPU merge ranks exact int32 scores (every shard result of the int8 path);
        # fractional scores would be truncated and re-ordered, so refuse them loudly
        raise NotImplementedError("_reduce_topk: the GPU shard merge takes integral int32 "
                                  "scores; got fractional float scores")
    if raw.size and (scores.min() < -2**31 or scores.max() >= 2**31):
        raise NotImplementedError("_reduce_topk: scores outside the int32 range")
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


def query_owner_slices(n_queries: int, world: int) -> list[tuple[int, int]]:
    """Contiguous query slice each rank merges in the owner-partitioned exchange."""
    return [(r * n_queries // world, (r + 1) * n_queries // world) for r in range(world)]


def exchange_owner(local_scores: torch.Tensor, local_ids: torch.Tensor,
                   local_count: torch.Tensor, group=None):
    """Owner-partitioned exchange with static sizes (the default): every rank sends each
    query's local list to the rank owning the query (``query_owner_slices``) in ONE
    ``all_to_all_single`` of a packed [B, 3k + 1] int32 payload (ids as two int32 words,
    scores, count). All split sizes follow from (B, world), so there is no device->host
    synchronisation and the step can be captured in a CUDA graph. Per rank the traffic is
    B * k pairs (the all-gather moves (world - 1) * B * k).

    Returns (q0, q1, scores [world, q1-q0, k], ids [...], counts [world, q1-q0])."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B, k = local_scores.shape
    payload = torch.cat([local_ids.contiguous().view(torch.int32).view(B, 2 * k),
                         local_scores.to(torch.int32), local_count.to(torch.int32).view(B, 1)],
                        dim=1)
    slices = query_owner_slices(B, world)
    q0, q1 = slices[rank]
    nq = q1 - q0
    recv = torch.empty((world * nq, 3 * k + 1), dtype=torch.int32, device=payload.device)
    dist.all_to_all_single(recv, payload, output_split_sizes=[nq] * world,
                           input_split_sizes=[b - a for a, b in slices], group=group)
    recv = recv.view(world, nq, 3 * k + 1)
    ids = recv[:, :, : 2 * k].contiguous().view(torch.int64).view(world, nq, k)
    scores = recv[:, :, 2 * k: 3 * k].contiguous()
    count = recv[:, :, 3 * k].contiguous()
    return q0, q1, scores, ids, count


def exchange_pruned(local_scores: torch.Tensor, local_ids: torch.Tensor,
                    local_count: torch.Tensor, k: int, group=None):
    """Owner-partitioned, pruned exchange (SURVEY §8(e) "optimised"): one all-reduce(MAX)
    of every query's local k-th score gives a bound tau* the global k-th score cannot fall
    below (the union of the ranks' lists holds >= k pairs scoring >= it), so each rank
    ships only its pairs with score >= tau*, and only to the rank owning the query
    (all-to-all). Per rank the traffic drops from (world - 1) * B * k pairs (all-gather) to
    about B * k / world.

    Returns (q0, q1, scores [world, q1-q0, kmax], ids [...], counts [world, q1-q0]): the
    lists of this rank's query slice, ready for the merge (ties at tau* are all kept, so
    the merge of the pruned lists equals the merge of the full ones)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B, kin = local_scores.shape
    dev = local_scores.device
    cnt = local_count.to(torch.int64).clamp(max=kin)
    pos = torch.arange(kin, device=dev)[None, :]
    # local k-th score (INT32_MIN when a rank holds fewer than k pairs for the query)
    kth = torch.where(cnt >= k, local_scores.gather(1, (cnt.clamp(min=1) - 1)[:, None]
                                                    .clamp(max=k - 1))[:, 0].to(torch.int64),
                      torch.full((B,), -2**31, dtype=torch.int64, device=dev))
    tau = kth.clone()
    dist.all_reduce(tau, op=dist.ReduceOp.MAX, group=group)
    keep = (pos < cnt[:, None]) & (local_scores.to(torch.int64) >= tau[:, None])
    n_keep = keep.sum(dim=1)                                        # lists are sorted: a prefix
    slices = query_owner_slices(B, world)
    send_counts = torch.stack([n_keep[a:b].sum() for a, b in slices]).to(torch.int64)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    q0, q1 = slices[rank]
    nq = q1 - q0
    # per-query kept counts for the owner
    send_nk = torch.cat([n_keep[a:b] for a, b in slices]).to(torch.int64)
    recv_nk = torch.empty((world * nq,), dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv_nk, send_nk, output_split_sizes=[nq] * world,
                           input_split_sizes=[b - a for a, b in slices], group=group)
    flat_s = local_scores[keep]
    flat_i = local_ids[keep]
    sc = send_counts.tolist()
    rc = recv_counts.tolist()
    rs = torch.empty((sum(rc),), dtype=local_scores.dtype, device=dev)
    ri = torch.empty((sum(rc),), dtype=local_ids.dtype, device=dev)
    dist.all_to_all_single(rs, flat_s, output_split_sizes=rc, input_split_sizes=sc, group=group)
    dist.all_to_all_single(ri, flat_i, output_split_sizes=rc, input_split_sizes=sc, group=group)
    nk = recv_nk.view(world, nq)
    kmax = max(1, int(nk.max().item()) if nk.numel() else 1)
    out_s = torch.full((world * nq, kmax), -2**31, dtype=local_scores.dtype, device=dev)
    out_i = torch.zeros((world * nq, kmax), dtype=local_ids.dtype, device=dev)
    flat = recv_nk                                   # received in (source rank, query) order
    if rs.numel():
        seg = torch.repeat_interleave(torch.arange(world * nq, device=dev), flat)
        start = torch.cumsum(flat, 0) - flat
        slot = torch.arange(rs.numel(), device=dev) - start[seg]
        out_s[seg, slot] = rs
        out_i[seg, slot] = ri
    return (q0, q1, out_s.view(world, nq, kmax), out_i.view(world, nq, kmax),
            nk.to(torch.int32))


@dataclass
class ShardedSearch:
    """One rank's part of an item-sharded filtered top-k.

    ``op`` is this rank's planned ``TopkOp`` over its local shard (ids are the global
    item ids). ``__call__`` returns the global top-k on every rank.
    """

    op: TopkOp
    group: object = None
    merge: object = None  # injectable merge (tests on CPU/gloo); default: fb_merge_topk
    exchange: str = "owner"  # "owner" (exchange_owner), "pruned" or "all_gather"

    def __call__(self, queries_q: torch.Tensor, filters=None, k: int | None = None) -> TopkOutput:
        """Global top-k: every query on every rank ("all_gather"), or with ``exchange=
        "owner"`` / ``"pruned"`` the rows of this rank's query slice (``query_owner_slices``)."""
        local = self.op(queries_q, filters)
        k = self.op.k if k is None else k
        merge = self.merge or merge_topk
        if self.exchange == "owner":
            _, _, s, i, c = exchange_owner(local.scores, local.ids, local.count, self.group)
            return merge(s, i, c, k)
        if self.exchange == "pruned":
            _, _, s, i, c = exchange_pruned(local.scores, local.ids, local.count, k, self.group)
            return merge(s, i, c, k)
        s, i, c = exchange_topk(local.scores, local.ids, local.count, self.group)
        return merge(s, i, c, k)


__all__ = ["_reduce_topk", "shard_ranges", "exchange_topk", "exchange_owner", "exchange_pruned",
           "query_owner_slices", "ShardedSearch", "DeviceIndex"]
