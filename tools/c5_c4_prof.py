#!/usr/bin/env python3
"""Profiling driver (run under ncu): `c5` runs the C5 allocation 3 times on
the general kernels; `c4` runs 3 K2 launches over the 10^6-scenario C4
batch (the steady-state occupancy picture of the thread planner)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2409_14447_b200 import _native as N
from paper_2409_14447_b200 import batch as B
from paper_2409_14447_b200 import workloads as W

fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)
what = sys.argv[1] if len(sys.argv) > 1 else "c5"
if what == "c5":
    rates = W.c5_rates()
    n = rates.shape[0]
    t = dt.packed.index_of()[W.C5_MODEL]
    cfg, _ = B.plan_batch(dt, np.array([0, n], dtype=np.int32), np.full(n, t, dtype=np.int32), rates,
                          np.full(n, W.C5_SLO / 2.0)).host()
    g = B.general_from_configs(dt.packed, np.full(n, t), cfg, True, 4)
    for _ in range(3):
        out = B.plan_general(g)
    torch.cuda.synchronize()
    print("c5 gpus", len(out.gpu_id), "unopt", out.n_gpus_unopt)
else:
    n = 1_000_000
    sb = W.scenario_batch(fx, n, seed=1)
    M = sb.rate.shape[1]
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    d = [N.to_device(a) for a in (off, tab, sb.rate.ravel().copy(), sb.bound.ravel().copy())]
    res = B.plan_batch(dt, *d)
    for _ in range(2):
        B.plan_batch(dt, *d, out=res)
    torch.cuda.synchronize()
    print("c4 done")
