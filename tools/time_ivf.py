"""IVF-probed batched search on one GPU: a k-means-clustered index of N items
(GPU k-means, k = ceil(sqrt(N)) unless given), B queries x nprobe probes with the
4-attribute filter; times IvfSearchOp's grouped scan (path="probe") and the exhaustive masked
scan (path="masked") with CUDA events, and the oracle's codesigned_search per query on the host
for a bounded sample.

    python tools/time_ivf.py [--n 10000000] [--batch 256] [--nprobe 24] [--k 1000]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2511_14881_b200 import kmeans, workload  # noqa: E402
from paper_2511_14881_b200.bloom import BloomParams, build_bloom_arrays  # noqa: E402
from paper_2511_14881_b200.engine import DeviceIndex  # noqa: E402
from paper_2511_14881_b200.ivf import IvfSearchOp  # noqa: E402
from paper_2511_14881_b200.quantize import QuantParams, quantize_device  # noqa: E402


def build(n, dim, n_clusters, iters, seed=1):
    dev = torch.device("cuda", 0)
    emb = workload.make_items(n, dim, seed, dev)
    X = emb.to(torch.float64)
    t0 = time.perf_counter()
    centers, assign = kmeans._train_device(X, n_clusters, iters, 0.0, seed)
    torch.cuda.synchronize()
    t_km = time.perf_counter() - t0
    del X
    ids = torch.arange(n, dtype=torch.int64, device=dev)
    perm, offs = kmeans.ivf_layout(assign, ids, n_clusters)
    n_slots = perm.numel()
    n_pad = (n_slots + 255) // 256 * 256
    real = perm >= 0
    qp = QuantParams(float(emb.min()), float(emb.max()))
    dim_pad = (dim + 31) // 32 * 32
    rows = torch.zeros((n_pad, dim), dtype=torch.float32, device=dev)
    rows[:n_slots][real] = emb[perm[real]]
    items = quantize_device(rows, qp, out_stride=dim_pad)
    items[:n_slots][~real] = 0
    items[n_slots:] = 0
    del rows
    slot_of_item = torch.empty(n, dtype=torch.int64, device=dev)
    slot_of_item[perm[real]] = torch.nonzero(real).view(-1)
    fid, val, it = workload.make_feature_pairs(n, seed, dev)
    bloom = build_bloom_arrays(fid, val, slot_of_item[it], n_pad, BloomParams())
    bits = torch.zeros(n_pad, dtype=torch.int64, device=dev)
    bits[:n_slots] = real.to(torch.int64)
    valid = (bits.view(-1, 64) << torch.arange(64, device=dev)).sum(dim=1)
    slot_ids = torch.zeros(n_pad, dtype=torch.int64, device=dev)
    slot_ids[:n_slots][real] = ids[perm[real]]
    dix = DeviceIndex(items, valid, slot_ids, n_pad, dim, bloom=bloom, qp=qp,
                      cluster_offsets=offs.cpu().numpy(), centroids=centers.to(torch.float32))
    return dix, emb, t_km


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--clusters", type=int, default=0)
    ap.add_argument("--kmeans-iters", type=int, default=2)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--nprobe", type=int, default=24)
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cpu-queries", type=int, default=4)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    C = a.clusters or int(np.ceil(np.sqrt(a.n)))
    dix, emb, t_km = build(a.n, a.dim, C, a.kmeans_iters)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    rows = torch.randint(0, a.n, (a.batch,), generator=g, device="cuda")
    queries = (emb[rows] + torch.randn((a.batch, a.dim), generator=g, device="cuda") * 0.05).float()
    del emb
    rng = np.random.default_rng(7)
    from paper_2511_14881_b200.filter_query import FilterBatch, compile_filter
    filters = [compile_filter(workload.four_attribute_filter(rng), BloomParams())
               for _ in range(a.batch)]
    batch = FilterBatch.pack(filters, BloomParams()).to_device()
    out = {"n": a.n, "clusters": C, "kmeans_iters": a.kmeans_iters, "kmeans_s": round(t_km, 2),
           "batch": a.batch, "nprobe": a.nprobe, "k": a.k}
    res = {}
    for path in ("probe", "masked"):
        op = IvfSearchOp(dix, a.batch, a.nprobe, a.k, path=path)
        for _ in range(3):
            r, cl = op(queries, batch)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            r, cl = op(queries, batch)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        out[f"{path}_ms_per_batch"] = round(ms, 3)
        out[f"{path}_qps"] = round(a.batch / (ms * 1e-3), 1)
        res[path] = (r.ids.clone(), r.scores.clone(), r.count.clone())
        del op
    # phases of the grouped path
    op = IvfSearchOp(dix, a.batch, a.nprobe, a.k, path="probe")
    op(queries, batch)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    acc = [0.0, 0.0, 0.0]
    for _ in range(a.iters):
        ev[0].record()
        cl = op.probe(queries)
        ev[1].record()
        words = op.probe_words(cl)
        qq = dix.quantize_queries(queries)
        ev[2].record()
        op(queries, batch)
        ev[3].record()
        torch.cuda.synchronize()
        for i in range(3):
            acc[i] += ev[i].elapsed_time(ev[i + 1])
    out["phase_probe_ms"] = round(acc[0] / a.iters, 3)
    out["phase_words_quant_ms"] = round(acc[1] / a.iters, 3)
    out["phase_full_call_ms"] = round(acc[2] / a.iters, 3)
    del op
    same = all(torch.equal(x, y) for x, y in zip(res["probe"], res["masked"]))
    out["probe_equals_masked"] = bool(same)
    out["mean_results"] = float(res["probe"][2].float().mean())
    # host reference arithmetic (oracle) on a bounded sample of queries
    from oracle import filtra_oracle as orc
    items = dix.items.cpu().numpy()[:, : a.dim]
    valid = dix.valid.cpu().numpy().view(np.uint64)
    ids = dix.item_ids.cpu().numpy().view(np.uint64)
    planes = dix.bloom.planes
    offs = dix.cluster_offsets
    qf = queries.cpu().numpy()
    qp = dix.qp
    t0 = time.perf_counter()
    for t in range(a.cpu_queries):
        cf = filters[t]
        prog = ([(int(o), int(x)) for o, x in cf.ops], [(f, v, b.set_bits) for f, v, b in cf.leaves])
        cl = orc.probe_centroids(dix.centroids.cpu().numpy(), qf[t], a.nprobe)
        ref = orc.codesigned_search(items, valid, ids, offs, planes, prog,
                                    orc.quantize(qf[t], qp.global_min, qp.global_max), cl, a.k)
        got = res["probe"][0][t, : int(res["probe"][2][t])].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, ref.item_ids), t
    if a.cpu_queries > 0:
        per = (time.perf_counter() - t0) / a.cpu_queries
        out["cpu_oracle_ms_per_query"] = round(1e3 * per, 1)
        out["cpu_oracle_qps_1core"] = round(1.0 / per, 2)
    out["oracle_checked_queries"] = a.cpu_queries
    print(json.dumps(out))


if __name__ == "__main__":
    main()
