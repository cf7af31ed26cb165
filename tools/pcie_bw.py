import torch, time
x = torch.empty(30_721_024 // 4, dtype=torch.int32, device='cuda')
h = torch.empty_like(x, device='cpu').pin_memory()
for _ in range(3): h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): h.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"D2H {x.numel()*4/1e6:.1f} MB: {ms:.3f} ms -> {x.numel()*4/ms/1e6:.1f} GB/s")
e0.record()
for _ in range(20): x.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"H2D: {ms:.3f} ms -> {x.numel()*4/ms/1e6:.1f} GB/s")
