#!/usr/bin/env python3
"""Zero-copy entry: synchronous calls vs pipelined submit/wait (depth D),
wall time per call and parity with the device path.

    python tools/e2e_async.py [n] [steps]
"""
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 400
fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)
off, tab, rate, bound = c2_inputs(fx, n, 0)
ref = B.MappedHostBatch(off, tab, rate, bound, cfg_format=2, plan_bytes=64)
ref.run(dt)
_, eplan = ref.outputs()
for _ in range(20):
    ref.run(dt)
t0 = time.perf_counter()
for _ in range(steps):
    ref.run(dt)
sync_us = (time.perf_counter() - t0) / steps * 1e6
print(f"sync        : {sync_us:7.1f} us/call  {n / sync_us * 1e6:.3e} scen/s")
for D in (int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["2", "3", "4"])):
    mb = B.MappedHostBatch(off, tab, rate, bound, cfg_format=2, plan_bytes=64, depth=D)

    def go(k):
        for i in range(k):
            mb.submit(dt, i % D)
            if i >= D - 1:
                mb.wait((i - D + 1) % D)
        for i in range(max(0, k - D + 1), k):
            mb.wait(i % D)
    go(20)
    t0 = time.perf_counter()
    go(steps)
    us = (time.perf_counter() - t0) / steps * 1e6
    ok = all(mb.outputs(s)[1].tobytes() == eplan.tobytes() for s in range(D))
    print(f"depth {D}     : {us:7.1f} us/call  {n / us * 1e6:.3e} scen/s  parity {ok}")
