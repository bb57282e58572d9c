import torch, time
n = 1920*1080*3
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device='cuda')
s = torch.cuda.Stream()
for _ in range(5): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
print(f"H2D {n*4/1e6:.1f} MB: {ms:.3f} ms, {n*4/ms/1e6:.1f} GB/s")
