"""End-to-end serving throughput of engine.PipelinedTopk (host queries + packed filters in,
ids / scores / counts out) for several pipeline shapes on config 2.

    python tools/time_pipeline.py [--items N] [--batch B] [--k K] [--steps S]

A/B numbers for DESIGN.md; bench.py's ``e2e`` is the reported measurement.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2511_14881_b200 import workload  # noqa: E402
from paper_2511_14881_b200.bloom import BloomParams  # noqa: E402
from paper_2511_14881_b200.engine import PipelinedTopk  # noqa: E402
from paper_2511_14881_b200.filter_query import FilterBatch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--items", type=int, default=10_000_000)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--k", type=int, default=10_000)
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    wl = workload.make_workload(a.items, a.batch)
    idx = wl.index
    host_q = wl.queries.cpu().pin_memory()
    h_batch = FilterBatch.pack(wl.filters, BloomParams()).pin()
    stream = torch.cuda.current_stream()
    for depth, overlap in ((2, False), (2, True), (3, False), (3, True), (4, True)):
        pipe = PipelinedTopk(idx, a.batch, a.k, depth=depth, overlap=overlap,
                             filters_template=wl.filters)
        for _ in range(4):
            pipe.result(pipe.submit(host_q, h_batch))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        last = None
        for _ in range(a.steps):
            last = pipe.submit(host_q, h_batch)
        stream.wait_event(pipe.done_event(last))
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        print(json.dumps({"depth": depth, "overlap": overlap, "ms_per_step": round(ms, 4),
                          "queries_per_s": round(a.batch / ms * 1e3, 1)}), flush=True)
        del pipe
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
