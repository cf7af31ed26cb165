"""A/B: an all-unfiltered batch through the bytecode kernel (prog = NULL) vs the CNF kernel
(zero-group CNF program); checks identical outputs and times both with CUDA events."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2511_14881_b200 import workload  # noqa: E402
from paper_2511_14881_b200.bloom import BloomParams  # noqa: E402
from paper_2511_14881_b200.engine import TopkOp  # noqa: E402
from paper_2511_14881_b200.filter_query import FilterBatch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
B, k = 256, 10000
wl = workload.make_workload(n, B, filtered=False)
idx = wl.index
op = TopkOp(idx, B, k, np.array([[0, idx.n_slots]]))
null = FilterBatch.pack([None] * B, BloomParams()).to_device()
res = {}
for name, batch in (("prog=NULL", None), ("cnf-null", null)):
    out = op.alloc_outputs()
    for _ in range(3):
        op(wl.queries_q, batch, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        op(wl.queries_q, batch, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res[name] = (out.ids.clone(), out.scores.clone(), out.count.clone())
    print(f"{name}: {ms:.3f} ms/batch  {B / ms * 1e3:.0f} q/s  fallback={op.stats().fallback_queries}")
print("identical:", all(torch.equal(a, b) for a, b in zip(res["prog=NULL"], res["cnf-null"])))
