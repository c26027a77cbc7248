#!/usr/bin/env python3
"""PCIe copy characteristics on the GPU box: latency/bandwidth vs size, H2D,
D2H, and both directions at once (pinned host memory)."""
import time

import torch

torch.cuda.init()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=50):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps * 1e6


for size in (4 << 10, 64 << 10, 512 << 10, 2 << 20, 4 << 20, 32 << 20):
    h = torch.empty(size, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(size, dtype=torch.uint8).pin_memory()
    d = torch.empty(size, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(size, dtype=torch.uint8, device="cuda")
    h2d = t(lambda: d.copy_(h, non_blocking=True))
    d2h = t(lambda: h.copy_(d, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    bi = t(both)
    print(f"{size >> 10:7d} KiB  h2d {h2d:8.1f} us ({size / h2d / 1e3:5.1f} GB/s)  d2h {d2h:8.1f} us "
          f"({size / d2h / 1e3:5.1f} GB/s)  both {bi:8.1f} us ({2 * size / bi / 1e3:5.1f} GB/s)")
x = torch.zeros(1, device="cuda")
print("empty sync round trip", t(lambda: x.add_(1)) , "us")
