"""Per-request latency of the B = 1 drop-in path (reference handle_request -> retrieve ->
codesigned_search), the workload of reference acceptance test #11 (2000 items, dim 16,
14 clusters; nprobe 2, k0 16, topk 4, one task): single-thread time per request, 4-thread
throughput, and a cProfile of the single-thread loop. Needs baseline/_ref (the installed
reference + its tests) and a GPU.

    python tools/time_b1.py [--n 2000] [--profile]
"""
from __future__ import annotations

import argparse
import cProfile
import pstats
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT / "baseline" / "_ref"), str(ROOT / "baseline" / "_ref" / "tests"),
                str(ROOT)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--reference", action="store_true", help="unpatched reference (numpy)")
    a = ap.parse_args()
    from conftest import make_catalog
    from filtra.serve import handle_request
    from filtra.snapshot import PublishConfig, build_engine
    if not a.reference:
        from paper_2511_14881_b200 import integration
        integration.install()
    cat = make_catalog(n_items=2000, dim=16, n_clusters=14, seed=70)
    engine = build_engine(cat, PublishConfig(n_clusters=14, seed=70), snapshot_version=5)
    req = {"id": "swap", "mode": "retrieve", "nprobe": 2, "k0": 16, "topk": 4,
           "tasks": [{"name": "m", "user_embedding": cat.embeddings[3].tolist()}]}
    for _ in range(50):
        handle_request(engine, req)
    t0 = time.perf_counter()
    for _ in range(a.n):
        handle_request(engine, req)
    dt = time.perf_counter() - t0
    print(f"single thread: {1e6 * dt / a.n:.1f} us/request ({a.n / dt:.0f} req/s)")
    stop = threading.Event()
    counts = [0] * 4

    def hammer(j):
        while not stop.is_set():
            handle_request(engine, req)
            counts[j] += 1

    th = [threading.Thread(target=hammer, args=(j,)) for j in range(4)]
    for t in th:
        t.start()
    time.sleep(2.8)
    stop.set()
    for t in th:
        t.join()
    print(f"4 threads, 2.8 s: {sum(counts)} responses (reference acceptance #11 needs >= 10000)")
    if a.profile:
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(500):
            handle_request(engine, req)
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
