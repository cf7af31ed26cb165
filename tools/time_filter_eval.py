"""fb_filter_eval (the batched eval_compiled, ref filter_query.py:314-356) at 10M slots for a
256-query 4-attribute batch: device time per batch with CUDA events."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2511_14881_b200 import _native, workload  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
B = 256
wl = workload.make_workload(n, B)
idx = wl.index
batch = wl.batch.to_device()
prog = batch.struct()
s = idx.struct()
W = idx.n_words
out = torch.empty((B, W), dtype=torch.int64, device="cuda")
lib = _native.lib()
import ctypes
for _ in range(2):
    _native.check(lib.fb_filter_eval(ctypes.byref(s), ctypes.byref(prog), 0, W, 1, out.data_ptr(),
                                     _native.stream_ptr()))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    _native.check(lib.fb_filter_eval(ctypes.byref(s), ctypes.byref(prog), 0, W, 1, out.data_ptr(),
                                     _native.stream_ptr()))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"fb_filter_eval: {B} queries x {W} words: {ms:.3f} ms per batch "
      f"({ms / B * 1e3:.1f} us per query mask of {n} slots); checksum {int(out.sum().item())}")
