#!/usr/bin/env python3
"""C5 on the general kernels: wall time of plan_general with and without the
optimize pass (the serial chain = the difference), device time by events."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import dataclasses

import numpy as np
import torch

from paper_2409_14447_b200 import _native as N
from paper_2409_14447_b200 import batch as B
from paper_2409_14447_b200 import workloads as W

fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)
rates = W.c5_rates()
n = rates.shape[0]
t = dt.packed.index_of()[W.C5_MODEL]
cfg, _ = B.plan_batch(dt, np.array([0, n], dtype=np.int32), np.full(n, t, dtype=np.int32), rates,
                      np.full(n, W.C5_SLO / 2.0)).host()
a = time.perf_counter()
g = B.general_from_configs(dt.packed, np.full(n, t), cfg, True, 4)
print(f"general_from_configs {(time.perf_counter() - a) * 1e3:.1f} ms")
g0 = dataclasses.replace(g, optimize=False)
for name, gg in (("relocate only", g0), ("relocate + optimize", g)):
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        out = B.plan_general(gg)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name}: wall {(time.perf_counter() - t0) * 1e3:.1f} ms  events {e0.elapsed_time(e1):.1f} ms  "
              f"gpus {len(out.gpu_id)}")
