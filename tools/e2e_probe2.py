#!/usr/bin/env python3
"""Where does the end-to-end step go?  Device-timeline (events) vs wall time
of parva_plan_host_packed for chunk counts / record formats."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2409_14447_b200 import _native as N
from paper_2409_14447_b200 import batch as B
from paper_2409_14447_b200 import workloads as W

fx = W.load_fixtures()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
sb = W.scenario_batch(fx, n, seed=0)
M = 11
off = np.arange(n + 1, dtype=np.int32) * M
tab = np.tile(np.arange(M, dtype=np.int32), n)
rate, bound = sb.rate.ravel().copy(), sb.bound.ravel().copy()
dt = N.device_tables_for(fx.tables)
s = torch.cuda.current_stream()
for chunks in (1, 2, 3, 4):
    for fmt, pbytes in ((1, 128), (2, 64)):
        pb = B.PackedHostBatch(off, tab, rate, bound, n_chunks=chunks, cfg_format=fmt, plan_bytes=pbytes)
        for _ in range(10):
            pb.run(dt)
        wall, dev = [], []
        for _ in range(50):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record(s)
            pb.run(dt)
            b.record(s)
            torch.cuda.synchronize()
            wall.append((time.perf_counter() - t0) * 1e6)
            dev.append(a.elapsed_time(b) * 1e3)
        print(f"chunks={chunks} cfg={fmt} plan={pbytes}: wall {np.median(wall):7.1f} us  device {np.median(dev):7.1f} us"
              f"  in {pb.h2d_bytes / 1e6:.2f} MB out {pb.d2h_bytes / 1e6:.2f} MB", flush=True)
# raw copy speed of the same byte counts with one stream, pinned
h = torch.empty(2_020_096, dtype=torch.uint8).pin_memory(); d = torch.empty_like(h, device="cuda")
h2 = torch.empty(1_600_000, dtype=torch.uint8).pin_memory(); d2 = torch.empty_like(h2, device="cuda")
for _ in range(5):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"serial H2D 2.02 MB + D2H 1.6 MB: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us")
