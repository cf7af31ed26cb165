"""Single-request serving on CUDA graphs (the reference's per-request entry points,
``retrieval.retrieve`` -- ref/retrieval.py:163-199 -- and ``retrieval.codesigned_search``
-- ref/retrieval.py:110-144 -- called once per request from N server threads).

A request runs a fixed sequence of small device steps: per task the centroid probe
(numpy-order float64 dots + stable top-nprobe), the query quantisation, the grouped
filtered scan over the probed clusters with exact top-k (``fb_ivf_topk``, device-resident
probe lists), then the merge across tasks, cache-row lookup, re-scoring, value model and
final (score desc, id asc) top-k. Launched one by one from Python that is ~30 launches,
several host round trips and ~1 ms per request; here the whole sequence is captured ONCE
per request shape into a CUDA graph (static input / output buffers, results copied into
pinned host memory inside the graph) and every request is: copy the task vectors (and the
packed filter, if any) into the static buffers, one graph launch, one stream sync. Errors
the eager path raises mid-way (a candidate missing from the embedding cache, a zero
divisor in the value model) become device flags tested after the replay, in the same
order. Graphs are per thread (the reference server calls from a thread pool) and keyed on
everything that fixes the sequence: engine objects, task names, nprobe, k0, topk, merge,
value model, query dtype and the packed filter's shape.
"""

from __future__ import annotations

import gc
import json
import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _native
from ._device import device
from .bloom import FilterStats
from .engine import device_index_for
from .errors import DivByZero, MissingItem
from .filter_query import FilterBatch
from .ivf import IvfSearchOp, ScanStats, TopkResult, count_scan

GRAPHS_PER_THREAD = 16
_local = threading.local()


class _CaptureLock:
    """Captures run alone (exclusive); replays run concurrently (shared), each thread on
    its own stream, so the small single-request graphs of N server threads overlap on the
    device instead of queueing behind one lock and one stream."""

    def __init__(self):
        self._cv = threading.Condition()
        self._readers = 0
        self._writer = False

    def shared(self):
        lock = self

        class _S:
            def __enter__(self):
                with lock._cv:
                    while lock._writer:
                        lock._cv.wait()
                    lock._readers += 1

            def __exit__(self, *exc):
                with lock._cv:
                    lock._readers -= 1
                    if lock._readers == 0:
                        lock._cv.notify_all()
        return _S()

    def exclusive(self):
        lock = self

        class _X:
            def __enter__(self):
                with lock._cv:
                    while lock._writer or lock._readers:
                        lock._cv.wait()
                    lock._writer = True

            def __exit__(self, *exc):
                with lock._cv:
                    lock._writer = False
                    lock._cv.notify_all()
        return _X()


_GPU_LOCK = _CaptureLock()


def _stream() -> torch.cuda.Stream:
    """The calling thread's stream for captures and replays."""
    s = getattr(_local, "stream", None)
    if s is None:
        s = _local.stream = torch.cuda.Stream()
    return s


def _ck(tag: str) -> None:
    """FB_CAPTURE_TRACE=1: print the current stream's capture status after a step (finds
    the step that invalidates a capture)."""
    if not _native.env_flag("FB_CAPTURE_TRACE"):
        return
    from cuda.bindings import runtime as rt
    err, st = rt.cudaStreamIsCapturing(torch.cuda.current_stream().cuda_stream)
    print(f"[capture] {tag}: {st}", flush=True)


def _graphs() -> OrderedDict:
    g = getattr(_local, "graphs", None)
    if g is None:
        g = _local.graphs = OrderedDict()
    return g


def _batch_sig(batch: FilterBatch | None):
    if batch is None:
        return None
    return (tuple(batch.meta()), tuple((a.shape, a.dtype.str) for a in batch.host_arrays()))


def scan_stats_for(cluster_offsets: np.ndarray, clusters: np.ndarray, stats: ScanStats) -> None:
    """``search_clusters``' counters for the probed clusters (ivf.count_scan)."""
    count_scan([cluster_offsets[int(c)] for c in clusters], stats)


def filter_stats_for(cluster_offsets: np.ndarray, clusters: np.ndarray, push_bits: int,
                     stats: FilterStats) -> None:
    """``eval_compiled``'s counters over the probed, non-empty clusters (ref
    retrieval.py:127-133, filter_query.py:333-334, bloom.py:180)."""
    for c in clusters:
        s, e = (int(x) for x in cluster_offsets[int(c)])
        if s == e:
            continue
        words = ((e + 63) >> 6) - (s >> 6)
        stats.slots_evaluated += words * 64
        stats.words_read += push_bits * words


class _Graph:
    """One captured request shape: T task vectors -> probe + filtered scan (+ the
    multi-task tail when ``tail`` is set) -> pinned host outputs."""

    def __init__(self, dix, T: int, nprobe: int, k0: int, qdtype, batch: FilterBatch | None,
                 tail=None):
        dev = device()
        self.dix, self.T, self.k0 = dix, T, k0
        self.op = IvfSearchOp(dix, T, nprobe, k0, path="probe")
        # inputs: the task vectors as float32 (probe) and in the caller's dtype (quantise),
        # staged in one pinned buffer and sent by ONE copy per request
        nq = T * dix.dim * torch.empty((), dtype=qdtype).element_size()
        n32 = T * dix.dim * 4
        self.h_in = torch.zeros(n32 + nq, dtype=torch.uint8, pin_memory=True)
        self.d_in = torch.zeros(n32 + nq, dtype=torch.uint8, device=dev)
        self.u32 = self.d_in[:n32].view(torch.float32).view(T, dix.dim)
        self.uq = self.d_in[n32:].view(qdtype).view(T, dix.dim)
        self.h_u32 = self.h_in[:n32].view(torch.float32).view(T, dix.dim).numpy()
        self.h_uq = self.h_in[n32:].view(qdtype).view(T, dix.dim).numpy()
        self.batch = None
        self.h_batch = []
        if batch is not None:
            self.batch = batch.clone_host().to_device()
            self.h_batch = [torch.zeros(d.shape, dtype=d.dtype, pin_memory=True)
                            for d in self.batch._dev]
        self.tail = tail
        # every output lives in one flat device buffer written inside the graph and copied
        # to pinned host memory by ONE copy after the replay (no pinned-memory copies inside
        # the capture: torch's host allocator polls events, which a capture forbids)
        P = self.op.nprobe
        K = max(k0, 1)
        spec = [("clusters", (T, P), torch.int64), ("count", (T,), torch.int32),
                ("ids", (T, K), torch.int64), ("scores", (T, K), torch.int32)]
        if tail is not None:
            topk = tail["topk"]
            spec += [("out_ids", (1, topk), torch.int64), ("final", (1, topk), torch.float64),
                     ("ts", (1, T, topk), torch.float64), ("n", (1,), torch.int32),
                     ("missing", (2,), torch.int64), ("zero", (1,), torch.int32)]
        offs, off = {}, 0
        for name, shape, dt in spec:
            nbytes = int(np.prod(shape)) * torch.empty((), dtype=dt).element_size()
            offs[name] = (off, shape, dt)
            off += (nbytes + 15) // 16 * 16
        self.d_out = torch.zeros(max(off, 16), dtype=torch.uint8, device=dev)
        self.h_out = torch.zeros(max(off, 16), dtype=torch.uint8, pin_memory=True)

        def views(buf):
            return {n: buf[o: o + int(np.prod(sh)) * torch.empty((), dtype=dt).element_size()]
                    .view(dt).view(sh) for n, (o, sh, dt) in offs.items()}
        self.d = views(self.d_out)
        self.h = views(self.h_out)
        # eager warm-up (allocates lazily built state, raises the eager path's errors for
        # a malformed request shape before anything is captured), then the capture
        self._run()
        torch.cuda.current_stream().synchronize()
        self.graph = torch.cuda.CUDAGraph()
        # no collector pass inside the capture: a finalizer that frees device memory (a
        # collected TopkOp's plan) would invalidate it (engine._destroy_plan defers those too)
        gc.collect()
        gc_was = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
                self._run()
        finally:
            if gc_was:
                gc.enable()

    def _run(self):
        clusters = self.op.probe(self.u32)
        _ck("probe")
        qq = self.dix.quantize_queries(self.uq)
        _ck("quantize")
        out = self.op.scan(qq, clusters, self.batch)
        _ck("scan")
        d = self.d
        d["clusters"].copy_(clusters)
        d["count"].copy_(out.count)
        d["ids"].copy_(out.ids)
        d["scores"].copy_(out.scores)
        if self.tail is not None:
            self._run_tail(out)

    def _run_tail(self, out):
        from .overarch import (final_topk_device, merge_device, value_model_device,
                               value_model_kernel)
        t = self.tail
        T, k = self.T, self.k0
        merged, mcount = merge_device(out.ids.view(1, T, k), out.count.view(1, T), t["merge"])
        _ck("merge")
        valid = torch.arange(merged.shape[1], device=merged.device)[None, :] < mcount[:, None]
        rows, bad = t["cache"].rows_and_missing(merged, valid)
        badc = bad.reshape(-1)
        first = torch.argmax(badc.to(torch.int32)).view(1)   # device-only indexing below
        d = self.d
        d["missing"][0:1].copy_(badc.any().to(torch.int64).view(1))
        d["missing"][1:2].copy_(merged.reshape(-1).index_select(0, first))
        _ck("rows")
        ts = t["scorer"].score(t["cache"], rows, mcount, self.u32[None], t["names"])
        _ck("score")
        zero = []
        if getattr(self, "_vm_zero", None) is None:
            self._vm_zero = torch.zeros(1, dtype=torch.int32, device=ts.device)
        vm = value_model_kernel(t["spec"], t["names"], ts, mcount, zero=self._vm_zero)
        if vm is None:
            final = value_model_device(t["spec"], {n: ts[:, j, :] for j, n in enumerate(t["names"])},
                                       valid, zero_flags=zero)
        else:
            final, zf = vm
            zero.append(zf != 0)
        _ck("value_model")
        anyz = torch.zeros((1,), dtype=torch.bool, device=merged.device)
        for z in zero:
            anyz |= z.view(1)
        d["zero"].copy_(anyz.to(torch.int32))
        topk = t["topk"]
        order, n = final_topk_device(final, mcount, topk)
        d["out_ids"].copy_(torch.gather(merged, 1, order))
        d["final"].copy_(torch.gather(final, 1, order))
        d["ts"].copy_(torch.gather(ts, 2, order[:, None, :].expand(1, T, -1)))
        d["n"].copy_(n.to(torch.int32))

    def replay(self, users: np.ndarray, batch: FilterBatch | None):
        """users float [T, dim] (the caller's dtype) -> run; host outputs valid after."""
        # the previous replay on this thread's stream ended with a synchronize, so the
        # pinned staging buffers are free to overwrite
        np.copyto(self.h_u32, users, casting="unsafe")
        np.copyto(self.h_uq, users, casting="unsafe")
        st = _stream()
        with _GPU_LOCK.shared(), torch.cuda.stream(st):
            self.d_in.copy_(self.h_in, non_blocking=True)
            if batch is not None:
                for d, hp, h in zip(self.batch._dev, self.h_batch, batch.host_arrays()):
                    hp.numpy()[...] = h
                    d.copy_(hp, non_blocking=True)
            self.graph.replay()
            self.h_out.copy_(self.d_out, non_blocking=True)
            st.synchronize()


def _get_graph(key, make):
    """The thread's graph for ``key`` (LRU), or None when the shape cannot be captured or
    its eager warm-up raised -- the caller then runs the eager path, which raises the same
    request error or serves the request step by step."""
    g = _graphs()
    if key in g:
        g.move_to_end(key)
        return g[key]
    try:
        with _GPU_LOCK.exclusive(), torch.cuda.stream(_stream()):
            hit = make()
            torch.cuda.current_stream().synchronize()
    except Exception:  # noqa: BLE001 -- remembered as "eager only" for this shape
        if _native.env_flag("FB_GRAPH_STRICT"):  # tests: a capture failure is a failure
            raise
        hit = None
    g[key] = hit
    while len(g) > GRAPHS_PER_THREAD:
        g.popitem(last=False)
    return hit


def _eligible(dix, nprobe, k0) -> bool:
    return int(k0) >= 1 and int(nprobe) >= 1 and (
        dix.centroids is not None or dix.cluster_offsets.shape[0] == 1)


def _qdtype(x: np.ndarray):
    # reference quantize_vector quantises the caller's float64 value (a float32 array widens
    # exactly, so it takes the float32 kernel)
    return torch.float32 if x.dtype == np.float32 else torch.float64


def codesigned_search(ivf, bloom_index, cf, query, nprobe: int, k0: int, scan_stats=None,
                      filter_stats=None, timings=None):
    """Graph-replayed ``codesigned_search`` for one query, or None when the request shape
    is not covered (the caller then runs the eager path)."""
    dix = device_index_for(ivf, bloom=bloom_index if cf is not None else None)
    raw = np.asarray(query)
    if raw.ndim != 1 or raw.shape[0] != dix.dim or not _eligible(dix, nprobe, k0):
        return None
    if cf is not None and dix.bloom is None:
        return None
    batch = FilterBatch.pack([cf], dix.bloom.params) if cf is not None else None
    if raw.dtype != np.float32:
        raw = raw.astype(np.float64)
    key = ("cs", id(dix), int(nprobe), int(k0), raw.dtype.str, _batch_sig(batch))
    g = _get_graph(key, lambda: _Graph(dix, 1, int(nprobe), int(k0), _qdtype(raw), batch))
    if g is None:
        return None
    g.replay(raw[None], batch)
    h = g.h
    clusters = h["clusters"][0].numpy().copy()
    if scan_stats is not None:
        scan_stats_for(dix.cluster_offsets, clusters, scan_stats)
    if filter_stats is not None and cf is not None:
        filter_stats_for(dix.cluster_offsets, clusters, int(batch.push_leaf_bits[0]), filter_stats)
    n = int(h["count"][0])
    return TopkResult(item_ids=h["ids"][0, :n].numpy().view(np.uint64).copy(),
                      scores=h["scores"][0, :n].numpy().copy(), k_requested=int(k0))


def retrieve_fast(engine, req, cache_factory, scorer_factory, spec, names):
    """Graph-replayed ``retrieve`` for one request: returns (ids u64 [n], final f64 [n],
    task scores f64 [T, n], clusters per task, per-task counts) or None when not covered."""
    if len(req.tasks) == 0:
        return None
    dix = device_index_for(engine.ivf, bloom=engine.bloom if req.filter is not None else None)
    users = [np.asarray(t.user_embedding) for t in req.tasks]
    if any(u.ndim != 1 or u.shape[0] != dix.dim for u in users):
        return None
    if not _eligible(dix, req.nprobe, req.k0) or int(req.topk) < 1:
        return None
    cf = engine.compile(req.filter) if req.filter is not None else None
    if cf is not None and dix.bloom is None:
        return None
    batch = FilterBatch.pack([cf] * len(users), dix.bloom.params) if cf is not None else None
    f64 = any(u.dtype != np.float32 for u in users)
    U = np.stack([u.astype(np.float64 if f64 else np.float32) for u in users])
    cache = cache_factory(engine.cache)
    scorer = scorer_factory(engine.scorer)
    topk = min(int(req.topk), len(users) * int(req.k0))
    key = ("rt", id(dix), id(cache), id(scorer), tuple(names), int(req.nprobe), int(req.k0),
           topk, req.merge, json.dumps(spec, sort_keys=True, default=str), U.dtype.str,
           _batch_sig(batch))
    tail = {"cache": cache, "scorer": scorer, "names": list(names), "spec": spec,
            "merge": req.merge, "topk": topk}
    g = _get_graph(key, lambda: _Graph(dix, len(users), int(req.nprobe), int(req.k0),
                                       torch.float64 if f64 else torch.float32, batch, tail))
    if g is None:
        return None
    g.replay(U, batch)
    h = g.h
    if int(h["missing"][0]):
        raise MissingItem(int(h["missing"][1]) & 0xFFFFFFFFFFFFFFFF)
    if int(h["zero"][0]):
        raise DivByZero("division by zero in value model")
    n = int(h["n"][0])
    return (h["out_ids"][0, :n].numpy().view(np.uint64).copy(), h["final"][0, :n].numpy().copy(),
            h["ts"][0, :, :n].numpy().copy(), h["clusters"].numpy().copy(),
            int(batch.push_leaf_bits[0]) if batch is not None else 0, dix)


def graph_count() -> int:
    """Captured graphs of the calling thread (tests check the fast path was taken)."""
    return sum(1 for v in _graphs().values() if v is not None)
