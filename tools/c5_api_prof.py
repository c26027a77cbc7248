#!/usr/bin/env python3
"""C5 through the public API (plan_services on 49,612 Service objects):
wall time and a cProfile of where the host time goes."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_14447_b200 as P
from paper_2409_14447_b200 import workloads as W

fx = W.load_fixtures()
rates = W.c5_rates()
svcs = [P.make_service(f"d121#{i}", W.C5_MODEL, float(r), W.C5_SLO) for i, r in enumerate(rates)]
P.plan_services(svcs[:100], fx.tables)
for _ in range(2):
    t0 = time.perf_counter()
    res = P.plan_services(svcs, fx.tables)
    n = res.gpu_count
    t1 = time.perf_counter()
    res.services, res.deployment
    t2 = time.perf_counter()
    res.deployment.to_json()
    t3 = time.perf_counter()
    print(f"plan_services C5: {(t1 - t0) * 1e3:.0f} ms (gpus {n}, planning_ms {res.planning_ms:.1f}); "
          f"decode {(t2 - t1) * 1e3:.0f} ms; to_json {(t3 - t2) * 1e3:.0f} ms")
pr = cProfile.Profile()
pr.enable()
res = P.plan_services(svcs, fx.tables)
res.deployment.to_json()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
