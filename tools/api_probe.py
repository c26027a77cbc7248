#!/usr/bin/env python3
"""Throughput of the drop-in Python API: plan_many over C2 scenarios (build
Service objects, one fused launch, decode PlanResults) vs plan_services in a loop."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_14447_b200 as P
from paper_2409_14447_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
fx = W.load_fixtures()
sb = W.scenario_batch(fx, n, seed=0)
sets = [[P.make_service(m, m, float(sb.rate[k, j]), float(sb.slo[k, j])) for j, m in enumerate(sb.models)]
        for k in range(n)]
P.plan_many(sets[:100], fx.tables)
t0 = time.perf_counter()
res = P.plan_many(sets, fx.tables)
t1 = time.perf_counter()
print(f"plan_many {n}: {(t1 - t0) * 1e3:.1f} ms -> {n / (t1 - t0):.0f} scenarios/s")
t0 = time.perf_counter()
for ss in sets[:200]:
    try:
        P.plan_services(ss, fx.tables)
    except P.MigplanError:
        pass
t1 = time.perf_counter()
print(f"plan_services loop: {(t1 - t0) / 200 * 1e6:.0f} us per scenario")
