"""Run one batched filtered top-k on a small workload (hang triage for kernel changes).

    python tools/hang_probe.py ITEMS BATCH K
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2511_14881_b200 import workload  # noqa: E402
from paper_2511_14881_b200.engine import TopkOp  # noqa: E402

n, b, k = (int(x) for x in sys.argv[1:4])
wl = workload.make_workload(n, b, seed=11)
op = TopkOp(wl.index, b, k, np.array([[0, wl.index.n_slots]]))
out = op(wl.queries_q, wl.batch)
torch.cuda.synchronize()
print("ok", n, b, k, int(out.count.sum()))
