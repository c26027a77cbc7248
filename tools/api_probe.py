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
for rep in range(3):
    t0 = time.perf_counter()
    res = P.plan_many(sets, fx.tables)
    t1 = time.perf_counter()
    gpus = sum(r.gpu_count for r in res if not isinstance(r, Exception))
    t2 = time.perf_counter()
    for r in res:                       # force every lazy result's decode
        if not isinstance(r, Exception):
            r.services, r.deployment
    t3 = time.perf_counter()
    print(f"plan_many {n}: {(t1 - t0) * 1e3:.1f} ms -> {n / (t1 - t0):.0f} scenarios/s returned "
          f"(gpu_count of all: {(t2 - t1) * 1e3:.1f} ms, {gpus} GPUs); full decode of every result "
          f"{(t3 - t2) * 1e3:.0f} ms -> {n / (t3 - t0):.0f} scenarios/s end to end")
t0 = time.perf_counter()
for ss in sets[:200]:
    try:
        P.plan_services(ss, fx.tables)
    except P.MigplanError:
        pass
t1 = time.perf_counter()
print(f"plan_services loop: {(t1 - t0) / 200 * 1e6:.0f} us per scenario")
