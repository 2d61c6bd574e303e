"""Pinned host -> device copy bandwidth, repeated (host-side PCIe / memory contention probe)."""
import time

import torch

n = 400 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
o = torch.empty(n, dtype=torch.uint8).pin_memory()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
gbs = []
for _ in range(20):
    t0 = time.perf_counter()
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    gbs.append(n / (time.perf_counter() - t0) / 1e9)
print("h2d GB/s", [round(x, 1) for x in gbs])
s2 = torch.cuda.Stream()
bi = []
for _ in range(10):
    t0 = time.perf_counter()
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        o.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    bi.append(2 * n / (time.perf_counter() - t0) / 1e9)
print("h2d+d2h concurrent GB/s", [round(x, 1) for x in bi])
