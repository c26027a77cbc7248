#!/usr/bin/env python3
"""Zero-copy host entry vs the packed copy pipeline: parity and wall time.

    python tools/e2e_mapped.py [n]
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
fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)
off, tab, rate, bound = c2_inputs(fx, n, 0)
ref = B.plan_batch(dt, off, tab, rate, bound, cfg_format=2)
torch.cuda.synchronize()
rcfg, rplan = ref.cfg.cpu().numpy().view(np.uint8), ref.host()[1]


def timeit(f, reps=200):
    for _ in range(20):
        f()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    return (time.perf_counter() - t0) / reps * 1e6


pb = B.PackedHostBatch(off, tab, rate, bound, n_chunks=3, cfg_format=2, plan_bytes=64)
us = timeit(lambda: pb.run(dt))
c, p = pb.outputs()
print(f"packed 3-chunk: {us:7.1f} us/step  {n / us * 1e6:.3e} scen/s  plan==device {p.tobytes() == rplan.tobytes()}")
import os
mb = B.MappedHostBatch(off, tab, rate, bound, cfg_format=2, plan_bytes=64, chunk_scen=int(os.environ.get("CHUNK", "64")))
us = timeit(lambda: mb.run(dt))
c, p = mb.outputs()
print(f"mapped:         {us:7.1f} us/step  {n / us * 1e6:.3e} scen/s  plan==device {p.tobytes() == rplan.tobytes()}"
      f"  cfg==device {c.view(np.uint8).tobytes() == ref.cfg.cpu().numpy().reshape(-1)[:8 * len(c)].tobytes()}  in {mb.h2d_bytes} out {mb.d2h_bytes}")
# device-side timing of the mapped launch with host/device-resident blocks
s = torch.cuda.current_stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
hin, hout = mb.h_in, mb.h_out
din, dout = hin.cuda(), hout.cuda()
for name, i_, o_ in (("in host, out host", hin, hout), ("in host, out dev", hin, dout)):
    mb.h_in, mb.h_out = i_, o_
    ts = []
    for _ in range(30):
        a.record(s)
        mb.run(dt)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"mapped entry, {name}: span p50 {np.median(ts):.1f} us")
mb.h_in, mb.h_out = hin, hout
