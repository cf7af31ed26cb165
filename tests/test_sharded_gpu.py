"""Item-sharded search through the REAL kernels, world_size 2 on one GPU.

Both ranks run on ``cuda:0``: each builds its shard with the catalogue's global
quantisation parameters (all-reduce MIN/MAX) and global item ids, runs the fused
filtered top-k (``TopkOp`` -> ``fb_topk_execute``), exchanges its local lists over gloo
(tensors staged through host memory, since both ranks share one device) with each of
the three exchanges, and merges with ``fb_merge_topk``. The merged rows must equal the
oracle's unsharded ``codesigned_search`` over the concatenated catalogue bit for bit
(reference serve.py:103-121 ``sharded_retrieve`` -> ``_reduce_topk``)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_items, B, k, exchange, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2511_14881_b200 import _device, workload
        from paper_2511_14881_b200.engine import TopkOp, TopkOutput, merge_topk
        from paper_2511_14881_b200.serve import (exchange_owner, exchange_pruned,
                                                 exchange_topk)

        def reduce_minmax(lo, hi):
            t = torch.tensor([-lo, hi], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return -float(t[0]), float(t[1])

        def share_queries(q):
            h = q.cpu()
            dist.broadcast(h, 0)
            return h.to(q.device)

        wl = workload.make_workload(n_items, B, seed=11 + rank, id_base=rank * n_items,
                                    reduce_minmax=reduce_minmax, share_queries=share_queries)
        idx = wl.index
        op = TopkOp(idx, B, k, np.array([[0, idx.n_slots]]))
        local = op(wl.queries_q, wl.batch.to_device())
        torch.cuda.synchronize()
        ls, li, lc = local.scores.cpu(), local.ids.cpu(), local.count.cpu()
        if exchange == "owner":
            q0, q1, s, i, c = exchange_owner(ls, li, lc)
        elif exchange == "pruned":
            q0, q1, s, i, c = exchange_pruned(ls, li, lc, k)
        else:
            q0, q1 = 0, B
            s, i, c = exchange_topk(ls, li, lc)
        out: TopkOutput = merge_topk(s.cuda(), i.cuda(), c.cuda(), k)
        torch.cuda.synchronize()
        got = {}
        for j in range(q1 - q0):
            n = int(out.count[j])
            got[q0 + j] = (_device.u64_host(out.ids[j, :n]), out.scores[j, :n].cpu().numpy())
        shard = (idx.items.cpu().numpy()[:, : wl.dim], _device.u64_host(idx.valid),
                 _device.u64_host(idx.item_ids), idx.bloom.planes)
        progs = [([(int(o), int(a)) for o, a in cf.ops],
                  [(f, v, qb.set_bits) for f, v, qb in cf.leaves]) for cf in wl.filters]
        result_q.put((rank, got, shard, wl.queries_q.cpu().numpy()[:, : wl.dim], progs,
                      (wl.qp.global_min, wl.qp.global_max)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_items,B,k,exchange", [(20_000, 6, 300, "owner"),
                                                  (20_000, 6, 300, "pruned"),
                                                  (20_000, 5, 300, "all_gather"),
                                                  (6_000, 4, 2_000, "owner")])
def test_sharded_real_kernels_equal_unsharded(cuda, n_items, B, k, exchange):
    from oracle import filtra_oracle as orc
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_items, B, k, exchange, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # one global quantisation and one query batch on both ranks
    assert results[0][5] == results[1][5]
    assert np.array_equal(results[0][3], results[1][3])
    items = np.concatenate([r[2][0] for r in results])
    valid = np.concatenate([r[2][1] for r in results])
    ids = np.concatenate([r[2][2] for r in results])
    planes = np.concatenate([r[2][3] for r in results], axis=1)
    assert len(np.unique(ids[np.unpackbits(valid.view(np.uint8), bitorder="little")
                             .astype(bool)])) == world * n_items  # global ids, no collisions
    qq, progs = results[0][3], results[0][4]
    offs = np.array([[0, items.shape[0]]])
    seen = set()
    for _, got, *_ in results:
        for qi, (gi, gs) in got.items():
            ref = orc.codesigned_search(items, valid, ids, offs, planes, progs[qi], qq[qi], [0], k)
            assert np.array_equal(gi, ref.item_ids), (exchange, qi)
            assert np.array_equal(gs, ref.scores), (exchange, qi)
            seen.add(qi)
    assert seen == set(range(B))


def _graph_worker(port, exchange, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        from paper_2511_14881_b200 import _device, workload
        from paper_2511_14881_b200.engine import TopkOp
        from paper_2511_14881_b200.serve import ShardedSearch
        wl = workload.make_workload(40_000, 16, seed=5)
        idx = wl.index
        op = TopkOp(idx, 16, 500, np.array([[0, idx.n_slots]]))
        ss = ShardedSearch(op, exchange=exchange)
        batch = wl.batch.to_device()
        want = ss(wl.queries_q, batch)  # eager (also the warm-up)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            ss(wl.queries_q, batch)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            got = ss(wl.queries_q, batch)
        g.replay()
        torch.cuda.synchronize()
        ok = True
        for q in range(16):
            n = int(want.count[q])
            ok &= int(got.count[q]) == n
            ok &= np.array_equal(_device.u64_host(got.ids[q, :n]), _device.u64_host(want.ids[q, :n]))
            ok &= np.array_equal(got.scores[q, :n].cpu().numpy(), want.scores[q, :n].cpu().numpy())
        result_q.put(("ok" if ok else "mismatch", None))
    except Exception as e:  # noqa: BLE001
        result_q.put(("error", f"{type(e).__name__}: {e}"))
    # no NCCL teardown: the process ends here (a communicator destroy can block at exit)
    result_q.close()
    result_q.join_thread()
    os._exit(0)


@pytest.mark.parametrize("exchange", ["owner", "all_gather"])
def test_sharded_step_captures_in_cuda_graph(cuda, exchange):
    """The sharded step (local filtered top-k -> NCCL exchange -> GPU merge) has no
    device->host synchronisation, so it captures in one CUDA graph; the replay returns the
    eager step's rows (world size 1 on the one GPU: the collectives are real NCCL calls)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_graph_worker, args=(_free_port(), exchange, q))
    p.start()
    try:
        status, msg = q.get(timeout=600)
    finally:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
            p.join(timeout=30)
    assert status == "ok", msg
