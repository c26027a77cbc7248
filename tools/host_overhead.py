#!/usr/bin/env python3
"""Host-side overhead of the e2e entries: wall per call for tiny batches, and
the empty-kernel round trip for comparison."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from bench import c2_inputs
from paper_2409_14447_b200 import _native as N
from paper_2409_14447_b200 import batch as B
from paper_2409_14447_b200 import workloads as W

fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)


def timeit(f, reps=500):
    for _ in range(50):
        f()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    return (time.perf_counter() - t0) / reps * 1e6


x = torch.zeros(1, device="cuda")
print(f"torch tiny op + sync: {timeit(lambda: (x.add_(1), torch.cuda.synchronize())):.1f} us")
for n in (1, 16, 1000, 10000):
    off, tab, rate, bound = c2_inputs(fx, n, 0)
    mb = B.MappedHostBatch(off, tab, rate, bound, cfg_format=2, plan_bytes=64)
    pb = B.PackedHostBatch(off, tab, rate, bound, n_chunks=3 if n >= 3 else 1, cfg_format=2, plan_bytes=64)
    print(f"n={n:6d}: mapped {timeit(lambda: mb.run(dt)):7.1f} us   packed {timeit(lambda: pb.run(dt)):7.1f} us")
