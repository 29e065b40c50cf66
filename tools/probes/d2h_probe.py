"""D2H bandwidth of one (1080, 1920, 3) f32 frame image into pinned host memory (the e2e copy)."""
import time

import torch

h, w = 1080, 1920
dev = torch.rand((h, w, 3), device="cuda")
host = [torch.empty((h, w, 3)).pin_memory() for _ in range(2)]
s = torch.cuda.Stream()
for n in (10, 90):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for i in range(n):
            host[i % 2].copy_(dev, non_blocking=True)
    s.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{n} copies: {dt * 1e3:.3f} ms per frame image = {dev.numel() * 4 / dt / 1e9:.1f} GB/s")
# D2H while a compute stream keeps the GPU busy with HBM-bound work
a = torch.empty(1 << 28, device="cuda")
b = torch.empty_like(a)
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s):
    for i in range(90):
        host[i % 2].copy_(dev, non_blocking=True)
for _ in range(200):
    b.copy_(a)
s.synchronize()
torch.cuda.synchronize()
print(f"with concurrent HBM copies: {(time.perf_counter() - t0) * 1e3 / 90:.3f} ms per frame image (wall incl. compute)")
