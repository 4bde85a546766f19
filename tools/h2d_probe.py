"""Host<->device copy bandwidth from pinned memory on this box (context for e2e)."""
import time, torch
x = torch.empty(800_000_000 // 4, dtype=torch.float32, pin_memory=True)
d = torch.empty_like(x, device="cuda")
for _ in range(3):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"H2D pinned 800 MB: {dt*1e3:.2f} ms = {0.8/dt:.1f} GB/s")
t = time.perf_counter()
for _ in range(5):
    x.copy_(d, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"D2H pinned 800 MB: {dt*1e3:.2f} ms = {0.8/dt:.1f} GB/s")
