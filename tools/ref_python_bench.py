#!/usr/bin/env python3
"""Time the reference itself (`migplan`, pure Python, installed unmodified
into baseline/_ref by `pip install --no-deps --target baseline/_ref`) on the
bench's workloads, on this host's cores.  Used by bench.py's cpu_baseline
leg; prints one JSON object.

    python tools/ref_python_bench.py c2 --n 2000 --procs 1
    python tools/ref_python_bench.py c1
    python tools/ref_python_bench.py c3 --n 200
    python tools/ref_python_bench.py c4 --n 2000     (C4 generator = C2 with seed 1)
    python tools/ref_python_bench.py c5

Timed region per scenario = the reference's own (pipeline.py:95-103):
configure_service for every service, relocate_segments, optimize_allocation;
tables are prepared once outside it (pipeline.py:94).  C2 inputs come from
the same generator as the GPU arm (seed 0); an infeasible
scenario raises InfeasibleSLOError inside configure, as in plan_services.
--procs > 1: a fork Pool over strided scenario chunks, wall time of the pool.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
REF = REPO / "baseline" / "_ref"
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REF))

import migplan  # noqa: E402  (the reference, unmodified)
from migplan import allocator as RA  # noqa: E402
from migplan import configurator as RC  # noqa: E402
from migplan import pipeline as RP  # noqa: E402

from paper_2409_14447_b200 import workloads as W  # noqa: E402  (input generator only)

_STATE = {}


def ref_tables(fx):
    tables = {}
    for m, t in fx.tables.items():
        pts = tuple(migplan.ProfilePoint(m, p.instance_size, p.batch_size, p.process_count, p.throughput, p.latency,
                                         p.memory_required) for p in t.points)
        tables[m] = migplan.ProfileTable(m, pts)
    return RP.prepare_tables(tables, RP.PlanOptions())


def plan_one(services, prepared):
    """configure -> relocate -> optimize, as plan_services' timed region."""
    configured = [RC.configure_service(s, prepared[s.model_id]) for s in services]
    dmap = RA.relocate_segments(configured)
    return RA.optimize_allocation(dmap, configured, threshold=4)


def _c2_chunk(args):
    lo, hi, step = args
    sb, prepared = _STATE["sb"], _STATE["prepared"]
    done = infeasible = 0
    t0 = time.perf_counter()
    for k in range(lo, hi, step):
        services = [RC.make_service(f"{m}", m, float(sb.rate[k, j]), float(sb.slo[k, j]))
                    for j, m in enumerate(sb.models)]
        try:
            plan_one(services, prepared)
        except migplan.InfeasibleSLOError:
            infeasible += 1
        done += 1
    return done, infeasible, time.perf_counter() - t0


def run_c1(reps=20):
    """S1-S6 (Table IV fixtures), the plan region per scenario, median of reps."""
    fx = W.load_fixtures()
    prepared = ref_tables(fx)
    out = {}
    for name, svcs in fx.scenarios.items():
        services = [RC.make_service(f"{m}#{i}", m, float(r), float(l)) for i, (m, r, l) in enumerate(svcs)]
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            res = plan_one(services, prepared)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        out[name] = {"ms": ts[len(ts) // 2] * 1e3, "gpus": res.gpu_count, "services": len(services)}
    return {"config": "C1", "scenarios": out, "procs": 1}


def run_c2(n, procs, seed=0):
    fx = W.load_fixtures()
    _STATE["prepared"] = ref_tables(fx)
    _STATE["sb"] = W.scenario_batch(fx, n, seed=seed)
    if procs <= 1:
        done, inf, el = _c2_chunk((0, n, 1))
    else:
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        with ctx.Pool(procs) as pool:
            pool.map(_c2_chunk, [(r, min(n, 64 * procs), procs) for r in range(procs)])   # warm the workers
            t0 = time.perf_counter()
            parts = pool.map(_c2_chunk, [(r, n, procs) for r in range(procs)])
            el = time.perf_counter() - t0
        done, inf = sum(p[0] for p in parts), sum(p[1] for p in parts)
    return {"config": "C2" if seed == 0 else f"C2 generator, seed {seed}", "scenarios": done, "infeasible": inf,
            "seconds": el, "scenarios_per_s": done / el, "procs": procs}


def run_c5():
    fx = W.load_fixtures()
    prepared = ref_tables(fx)
    rates = W.c5_rates()
    services = [RC.make_service(f"d121#{i}", W.C5_MODEL, float(r), W.C5_SLO) for i, r in enumerate(rates)]
    t0 = time.perf_counter()
    configured = [RC.configure_service(s, prepared[s.model_id]) for s in services]
    t1 = time.perf_counter()
    dmap = RA.relocate_segments(configured)
    t2 = time.perf_counter()
    unopt = dmap.gpu_count
    out = RA.optimize_allocation(dmap, configured, threshold=4)
    t3 = time.perf_counter()
    return {"config": "C5", "services": len(services), "gpus_before_optimize": unopt, "gpus": out.gpu_count,
            "configure_s": t1 - t0, "relocate_s": t2 - t1, "optimize_s": t3 - t2, "seconds": t3 - t0}


def run_c3(n):
    """configure_service (configurator.py:189-191) for the first n C3
    workloads, one query each; ProfileTables built outside the timer."""
    INSTANCE_SIZES = (1, 2, 3, 4, 7)
    dth = W.dense_tables(n, seed=3)
    tables = []
    for w in range(n):
        pts = []
        for c, size in enumerate(INSTANCE_SIZES):
            a = int(dth.seg_start[w * 5 + c])
            for i in range(a, a + int(dth.seg_count[w * 5 + c])):
                pts.append(migplan.ProfilePoint(f"w{w:05d}", size, int(dth.batch[i]), int(dth.procs[i]),
                                                float(dth.tp[i]), float(dth.lat[i])))
        tables.append(migplan.ProfileTable(f"w{w:05d}", tuple(pts)))
    services = [RC.make_service(f"w{w:05d}", f"w{w:05d}", float(dth.rate[w]), float(dth.slo[w])) for w in range(n)]
    done = infeasible = 0
    t0 = time.perf_counter()
    for s, t in zip(services, tables):
        try:
            RC.configure_service(s, t)
        except migplan.MigplanError:
            infeasible += 1
        done += 1
    el = time.perf_counter() - t0
    points = int(dth.seg_count.sum())
    return {"config": "C3", "workloads": done, "infeasible_or_uncoverable": infeasible, "points": points,
            "seconds": el, "workloads_per_s": done / el, "points_per_s": points / el, "procs": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--procs", type=int, default=1)
    a = ap.parse_args()
    if a.config == "c1":
        res = run_c1()
    elif a.config in ("c2", "c4"):
        res = run_c2(a.n, a.procs, seed=0 if a.config == "c2" else 1)
    elif a.config == "c3":
        res = run_c3(a.n)
    else:
        res = run_c5()
    res["python"] = sys.version.split()[0]
    res["reference"] = "migplan (baseline/_ref, unmodified)"
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
