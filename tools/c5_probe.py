#!/usr/bin/env python3
"""Time the C5 large-cluster allocation (10^5 segments) on the general kernel
and the CPU oracle."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2409_14447_b200 as P
from paper_2409_14447_b200 import batch as B
from paper_2409_14447_b200 import workloads as W

fx = W.load_fixtures()
rates = W.c5_rates()
svcs = [P.make_service(f"d121#{i}", W.C5_MODEL, float(r), W.C5_SLO) for i, r in enumerate(rates)]
t0 = time.perf_counter()
res = P.plan_services(svcs, fx.tables)
t1 = time.perf_counter()
print(f"plan_services C5 (host decode incl.): {t1 - t0:.3f} s, planning_ms {res.planning_ms:.1f}, "
      f"gpus {res.gpu_count} unopt {res.unoptimized_gpu_count}")
# kernel-only timing of the general kernel on the same problem
from paper_2409_14447_b200.tables import pack_tables
from paper_2409_14447_b200 import _native as N
dt = N.device_tables_for(fx.tables)
n = len(svcs)
off = np.array([0, n], dtype=np.int32)
t = dt.packed.index_of()[W.C5_MODEL]
r = B.plan_batch(dt, off, np.full(n, t, dtype=np.int32), rates, np.full(n, W.C5_SLO / 2.0))
cfg, plan = r.host()
g = B.general_from_configs(dt.packed, np.full(n, t), cfg, True, 4)
for _ in range(2):
    torch.cuda.synchronize()
    a = time.perf_counter()
    out = B.plan_general(g)
    torch.cuda.synchronize()
    b = time.perf_counter()
    print(f"plan_general (upload+kernel+download): {(b - a) * 1000:.1f} ms, gpus {len(out.gpu_id)}")
import oracle
pt = pack_tables(fx.tables)
a = time.perf_counter()
cfg_o, res_o = oracle.plan_scenario(pt, np.full(n, t), rates, np.full(n, W.C5_SLO / 2.0), True, 4, gcap=200_000)
print(f"oracle C5: {time.perf_counter() - a:.3f} s, gpus {len(res_o['gpus'])}")
