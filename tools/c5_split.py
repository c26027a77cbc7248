#!/usr/bin/env python3
"""C5 wall-time split of batch.plan_general: host -> device inputs, output
allocations, the two kernels (events), device -> host reads."""
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
dt = N.device_tables_for(fx.tables)
rates = W.c5_rates()
n = rates.shape[0]
t = dt.packed.index_of()[W.C5_MODEL]
cfg, _ = B.plan_batch(dt, np.array([0, n], dtype=np.int32), np.full(n, t, dtype=np.int32), rates,
                      np.full(n, W.C5_SLO / 2.0)).host()
g = B.general_from_configs(dt.packed, np.full(n, t), cfg, True, 4)
print("services", g.n_services, "cats", len(g.cat_size), "names", len(g.names))
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = B.plan_general(g)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"plan_general wall {(t1 - t0) * 1e3:.1f} ms, gpus {len(out.gpu_id)} unopt {out.n_gpus_unopt} "
          f"diags {len(out.diags)} fallback {out.fallback}")
# kernel-only: profile the C call with events
import cProfile
import pstats
pr = cProfile.Profile()
pr.enable()
out = B.plan_general(g)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
