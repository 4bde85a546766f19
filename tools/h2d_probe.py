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
# 128 MB chunks back to back (the obt_predict_host pipeline's copy pattern)
chunk = 128 << 20
n = x.numel() * 4
t = time.perf_counter()
for _ in range(5):
    off = 0
    while off < n:
        ln = min(chunk, n - off)
        d.view(torch.uint8)[off:off + ln].copy_(x.view(torch.uint8)[off:off + ln], non_blocking=True)
        off += ln
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"H2D pinned 800 MB in 128 MB chunks: {dt*1e3:.2f} ms = {0.8/dt:.1f} GB/s")
# two copy streams, alternating 64 MB chunks (do two DMA engines beat one?)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
chunk = 64 << 20
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    off, i = 0, 0
    while off < n:
        ln = min(chunk, n - off)
        with torch.cuda.stream(s1 if i % 2 == 0 else s2):
            d.view(torch.uint8)[off:off + ln].copy_(x.view(torch.uint8)[off:off + ln], non_blocking=True)
        off += ln
        i += 1
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"H2D pinned 800 MB on two streams: {dt*1e3:.2f} ms = {0.8/dt:.1f} GB/s")
