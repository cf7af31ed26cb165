"""Item-sharded search across ranks (serve.ShardedSearch / exchange_topk / shard_ranges),
exercised with world_size 2 on the gloo backend (CPU). The per-rank local top-k and the
merge are injected from the oracle here; on GPUs they are fb_topk_execute and
fb_merge_topk over NCCL (covered by the -m gpu tests on one device)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import filtra_oracle as orc


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _OracleOp:
    """Stands in for TopkOp on one shard: local exact top-k per query."""

    def __init__(self, items, ids, queries, k):
        self.items, self.ids, self.queries, self.k = items, ids, queries, k

    def __call__(self, queries_q, filters=None):
        from paper_2511_14881_b200.engine import TopkOutput
        B = self.queries.shape[0]
        scores = torch.full((B, self.k), -2**31, dtype=torch.int32)
        out_ids = torch.zeros((B, self.k), dtype=torch.int64)
        count = torch.zeros(B, dtype=torch.int32)
        for q in range(B):
            res = orc.brute_force_int8(self.items, self.ids, self.queries[q], self.k)
            n = len(res.item_ids)
            scores[q, :n] = torch.from_numpy(res.scores.astype(np.int32))
            out_ids[q, :n] = torch.from_numpy(res.item_ids.view(np.int64))
            count[q] = n
        return TopkOutput(ids=out_ids, scores=scores, count=count)


def _oracle_merge(scores, ids, count, k):
    from paper_2511_14881_b200.engine import TopkOutput
    n_lists, B, _ = scores.shape
    out_s = torch.full((B, k), -2**31, dtype=torch.int32)
    out_i = torch.zeros((B, k), dtype=torch.int64)
    out_c = torch.zeros(B, dtype=torch.int32)
    for q in range(B):
        all_i = np.concatenate([ids[l, q, : count[l, q]].numpy().view(np.uint64)
                                for l in range(n_lists)])
        all_s = np.concatenate([scores[l, q, : count[l, q]].numpy() for l in range(n_lists)])
        ri, rs = orc.reduce_topk(all_i, all_s, k)
        out_i[q, : len(ri)] = torch.from_numpy(ri.view(np.int64))
        out_s[q, : len(rs)] = torch.from_numpy(rs.astype(np.int32))
        out_c[q] = len(ri)
    return TopkOutput(ids=out_i, scores=out_s, count=out_c)


def _worker(rank, world, port, n_items, k, result_q, exchange="all_gather"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_14881_b200.serve import ShardedSearch, shard_ranges
        rng = np.random.default_rng(3)
        items = rng.integers(-128, 128, size=(n_items, 16)).astype(np.int8)
        items[::7] = items[0]  # many exact ties across shards
        ids = rng.permutation(n_items).astype(np.uint64) * np.uint64(3) + np.uint64(11)
        queries = rng.integers(-128, 128, size=(5, 16)).astype(np.int8)
        s0, s1 = shard_ranges(n_items, world)[rank]
        op = _OracleOp(items[s0:s1], ids[s0:s1], queries, k)
        op.k = k
        search = ShardedSearch(op=op, merge=_oracle_merge, exchange=exchange)
        out = search(torch.from_numpy(queries), None, k)
        if exchange == "pruned":
            from paper_2511_14881_b200.serve import query_owner_slices
            q0, q1 = query_owner_slices(5, world)[rank]
        else:
            q0, q1 = 0, 5
        got = {q0 + j: (out.ids[j, : out.count[j]].numpy().view(np.uint64).tolist(),
                        out.scores[j, : out.count[j]].tolist()) for j in range(q1 - q0)}
        result_q.put((rank, got, (s0, s1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_items,k,exchange", [(1000, 50, "all_gather"), (130, 200, "all_gather"),
                                                (1000, 50, "pruned"), (130, 200, "pruned"),
                                                (3000, 40, "pruned")])
def test_sharded_search_equals_unsharded(n_items, k, exchange):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_items, k, q, exchange))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(3)
    items = rng.integers(-128, 128, size=(n_items, 16)).astype(np.int8)
    items[::7] = items[0]
    ids = rng.permutation(n_items).astype(np.uint64) * np.uint64(3) + np.uint64(11)
    queries = rng.integers(-128, 128, size=(5, 16)).astype(np.int8)
    ranges = sorted(r[2] for r in results)
    assert ranges[0][0] == 0 and ranges[-1][1] == n_items and ranges[0][1] == ranges[1][0]
    seen = set()
    for rank, got, _ in results:
        for qi, (gi, gs) in got.items():
            ref = orc.brute_force_int8(items, ids, queries[qi], k)
            assert gi == ref.item_ids.tolist(), (rank, qi)
            assert gs == ref.scores.tolist(), (rank, qi)
            seen.add(qi)
    assert seen == set(range(5))


def test_shard_ranges_partition():
    from paper_2511_14881_b200.serve import shard_ranges
    for n, w in [(1, 1), (100, 3), (12_500_000, 8), (64 * 8 + 5, 8)]:
        r = shard_ranges(n, w)
        assert r[0][0] == 0 and r[-1][1] == n
        for (a0, a1), (b0, b1) in zip(r, r[1:]):
            assert a1 == b0 and (a0 % 64 == 0 or a0 == n) and a0 <= a1
