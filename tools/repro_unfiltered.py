import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_14881_b200 import workload, _native
from paper_2511_14881_b200.engine import TopkOp
torch.cuda.set_device(0)
wl = workload.make_workload(int(sys.argv[1]), 256, filtered=False)
idx = wl.index
for k in [int(x) for x in sys.argv[2].split(',')]:
    op = TopkOp(idx, 256, k, np.array([[0, idx.n_slots]]))
    out = op(wl.queries_q, None)
    torch.cuda.synchronize()
    st = op.stats()
    print(k, "ok", int(out.count.min()), int(out.count.max()), flush=True)
