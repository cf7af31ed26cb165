"""Per-stage device times of the config-5 multi-task operator (for A/B work only).

    python tools/time_multitask.py [--items N] [--requests R] [--k K]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2511_14881_b200 import _device, workload  # noqa: E402
from paper_2511_14881_b200.overarch import (DeviceCache, MultiTaskOp, merge_device,  # noqa: E402
                                            value_model_device, final_topk_device,
                                            value_model_kernel)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--items", type=int, default=10_000_000)
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--k", type=int, default=5000)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    R, T = a.requests, 4
    tasks = [f"t{i}" for i in range(T)]
    wl = workload.make_workload(a.items, R * T, seed=1)
    idx = wl.index
    cache = DeviceCache(_device.u64_host(idx.item_ids)[: a.items],
                        workload.make_items(a.items, 128, 1, idx.items.device))
    op = MultiTaskOp(idx, cache, R, tasks, a.k, a.k)
    batch = op.pack_filters([wl.filters[r * T] for r in range(R)]).to_device()
    users = wl.queries.view(R, T, -1)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for it in range(4):
        e = [ev() for _ in range(7)]
        e[0].record()
        qq = idx.quantize_queries(users.reshape(R * T, -1))
        res = op.op(qq, batch, keys=True)
        e[1].record()
        merged, ranks, mcount = op._merge_union(res)
        e[2].record()
        C = merged.shape[1]
        valid = torch.arange(C, device=merged.device)[None, :] < mcount[:, None]
        rows = op._rows_of_ranks(merged, ranks, valid)
        e[3].record()
        ts = op.scorer.score(cache, rows, mcount, users, tasks)
        e[4].record()
        final, _ = value_model_kernel(op.spec, tasks, ts, mcount)
        e[5].record()
        order, _ = final_topk_device(final, mcount, a.k)
        torch.gather(merged, 1, order)
        e[6].record()
        torch.cuda.synchronize()
        names = ["scan", "merge", "cache rows", "re-score", "value model", "final top-k"]
        if it >= 1:
            print(" ".join(f"{n} {e[i].elapsed_time(e[i + 1]):.3f}" for i, n in enumerate(names)),
                  f"| total {e[0].elapsed_time(e[6]):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
