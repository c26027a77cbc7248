#!/usr/bin/env python3
"""Render golden fixtures from the REFERENCE planner (`migplan`).

Runs only in the build container, where the read-only reference lives at
/root/reference (override with MIGPLAN_SRC).  Everything it writes is a
small committed JSON file under tests/golden/; nothing at test, smoke or
bench time reads /root/reference.

    python tests/golden/make_golden.py            # everything but C5
    python tests/golden/make_golden.py --c5       # + the 10^5-segment case (~90 s)

Files:
  fixture_tables.json   11 fixture tables (fixtures.py:241-249 with calibration.json)
                        and the Table IV scenarios (fixtures.py:155-229)
  fixture_plans.json    S1-S6 x {default, --no-optimize, --single-process}
  fuzz_plans.json       random plan_services cases (SURVEY App. B #5 mix + options)
  unit_cases.json       configure / select_optimal_segment / propose_small_segments
                        fuzz incl. near-ties (App. A F1-F5, F10)
  alloc_cases.json      relocate_segments and optimize_allocation on crafted and
                        random maps (App. B #3, #4)
  reconfigure_cases.json  reconfigure_service + diff_maps on planned maps (§8f row 1)
  c2_digests.json       digest of every C2 scenario plan (seed 0, 10^4) + 200 full plans
  c3_sample.json        200 C3 dense workloads: table digest + configure result
  c5_summary.json       C5 large-cluster allocation summary (with --c5)
  sim_cases.json        run_simulation (evaluation.py:286-464) reports on the S1-S6
                        plans: arrival kinds, rate scales, horizons, seeds (§8f row 4)
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import random
import sys
import time
from dataclasses import replace
from pathlib import Path

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF_SRC = os.environ.get("MIGPLAN_SRC", "/root/reference/pkg/src")
REF_CAL = Path(REF_SRC).parent / "fixtures" / "calibration.json"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(HERE))

import migplan as R                                   # noqa: E402  the reference
from migplan import fixtures as RF                    # noqa: E402
from migplan.allocator import DeploymentMap as RDeploymentMap   # noqa: E402
from migplan.mig import GpuState as RGpuState, Placement as RPlacement  # noqa: E402

import canon                                          # noqa: E402
from paper_2409_14447_b200 import workloads as W      # noqa: E402


def write(name, obj):
    path = HERE / name
    path.write_text(json.dumps(obj, separators=(",", ":")) + "\n")
    print(f"wrote {path.name}: {path.stat().st_size / 1024:.0f} KiB")


def ref_tables():
    return RF.build_tables(RF.load_calibration(REF_CAL))


# ------------------------------------------------------------------ C1
def gen_fixture_tables(tables):
    obj = {
        "source": "migplan.fixtures.build_tables(load_calibration('pkg/fixtures/calibration.json'))",
        "models": list(RF.MODEL_IDS),
        "tables": {m: [[p.instance_size, p.batch_size, p.process_count, p.throughput,
                        p.latency, p.memory_required] for p in tables[m].points]
                   for m in RF.MODEL_IDS},
        "scenarios": {name: [[m, float(r), float(s)] for m, (r, s) in RF.SCENARIOS[name].items()]
                      for name in RF.SCENARIO_NAMES},
        "csv_sha256": {m: hashlib.sha256(R.serialize_profile_table(tables[m], "csv").encode()).hexdigest()[:16]
                       for m in RF.MODEL_IDS},
    }
    write("fixture_tables.json", obj)


OPTION_SETS = {
    "default": {},
    "noopt": {"optimize": False},
    "single": {"single_process": True},
}


def gen_fixture_plans(tables):
    out = []
    for name in RF.SCENARIO_NAMES:
        sc = RF.make_scenario(name)
        for oname, kw in OPTION_SETS.items():
            res = R.plan_scenario(sc, tables, R.PlanOptions(**kw))
            summ = res.summary()
            summ.pop("planning_ms")
            out.append({"scenario": name, "options": oname,
                        "inputs": [[s.model, float(s.request_rate), float(s.slo_latency_ms)] for s in sc.services],
                        "plan": canon.plan(res), "summary": summ,
                        "json_sha256": hashlib.sha256(res.deployment.to_json().encode()).hexdigest()[:16]})
    write("fixture_plans.json", out)


# ---------------------------------------------------------------- fuzz
def gen_fuzz_plans(tables, n=400, seed=12345):
    rng = random.Random(seed)
    cases = []
    lo_r, hi_r, lo_s, hi_s = math.log(5), math.log(8000), math.log(20), math.log(3000)
    for i in range(n):
        k = rng.randint(1, 11)
        models = rng.sample(list(RF.MODEL_IDS), k)
        inputs = []
        for m in models:
            rate = math.exp(rng.uniform(lo_r, hi_r))
            if rng.random() < 0.04:
                rate = 0.0
            slo = math.exp(rng.uniform(lo_s, hi_s))
            inputs.append([m, rate, slo])
        opts = {"optimize": rng.random() < 0.85, "single_process": rng.random() < 0.25,
                "threshold": rng.choice([4, 4, 4, 4, 4, 0, 1, 2, 3, 5, 6, 7])}
        if rng.random() < 0.1:
            opts["memory_map"] = {1: 5.0, 2: 10.0, 3: 20.0, 4: 20.0, 7: 40.0}
        services = [R.make_service(m, m, r, s) for m, r, s in inputs]
        popts = R.PlanOptions(**{k: (v if k != "memory_map" else dict(v)) for k, v in opts.items()})
        try:
            res = R.plan_services(services, tables, popts)
            out = canon.plan(res)
        except R.MigplanError as exc:
            out = canon.error(exc)
        if "memory_map" in opts:
            opts["memory_map"] = [[s, v] for s, v in opts["memory_map"].items()]
        cases.append({"inputs": [[m, m, r, s] for m, r, s in inputs], "options": opts, "result": out})
    # size-4-heavy mix (SURVEY App. B #5 / C5 generator, small): many services on one model
    for i in range(120):
        k = rng.randint(2, 45)
        inputs = [[f"d121#{j}", W.C5_MODEL, rng.uniform(100, 3 * 2183.7), W.C5_SLO] for j in range(k)]
        opts = {"threshold": rng.choice([4, 4, 4, 3, 5])}
        services = [R.make_service(a, m, r, s) for a, m, r, s in inputs]
        try:
            out = canon.plan(R.plan_services(services, tables, R.PlanOptions(**opts)))
        except R.MigplanError as exc:
            out = canon.error(exc)
        cases.append({"inputs": inputs, "options": opts, "result": out})
    write("fuzz_plans.json", cases)


def _rand_tp(rng, ties):
    if ties:
        return float(rng.choice([100.0, 150.0, 200.0, 250.0, 300.0, 400.0, 600.0, 700.0]))
    return math.exp(rng.uniform(math.log(20), math.log(3000)))


def gen_unit_cases(seed=777):
    rng = random.Random(seed)
    configure = []
    for i in range(600):
        ties = rng.random() < 0.5
        sizes = rng.sample(list(R.INSTANCE_SIZES), rng.randint(1, 5))
        pts = []
        for s in sizes:
            for b in rng.sample([1, 2, 4, 8, 16], rng.randint(1, 5)):
                for p in rng.sample([1, 2, 3], rng.randint(1, 3)):
                    tp = _rand_tp(rng, ties) * (s if rng.random() < 0.5 else 1)
                    lat = float(rng.randint(1, 30)) if ties else rng.uniform(0.5, 30)
                    pts.append([s, b, p, tp, lat])
        table = R.ProfileTable("m", tuple(R.ProfilePoint("m", s, b, p, tp, lat) for s, b, p, tp, lat in pts))
        bound = float(rng.randint(0, 32)) if rng.random() < 0.5 else rng.uniform(0, 35)
        mode = rng.random()
        if mode < 0.1:
            rate = 0.0
        elif mode < 0.4:
            # exact multiple of some throughput -> residual exactly zero or float dust
            rate = rng.randint(1, 12) * rng.choice([p[3] for p in pts])
        else:
            rate = math.exp(rng.uniform(math.log(1), math.log(20000)))
        svc = R.make_service("s", "m", rate, 1.0, internal_latency=bound)
        try:
            out = canon.service(R.configure_service(svc, table))
        except R.MigplanError as exc:
            out = canon.error(exc)
        configure.append({"points": pts, "bound": bound, "rate": rate, "result": out})

    select = []
    for i in range(2000):
        n = rng.randint(1, 5)
        base_tp = math.exp(rng.uniform(math.log(50), math.log(5000)))
        trips = []
        for j in range(n):
            s = rng.choice(R.INSTANCE_SIZES)
            if rng.random() < 0.6:
                tp = base_tp * s / 1.0            # same efficiency up to rounding
                k = rng.randint(-3, 3)
                for _ in range(abs(k)):
                    tp = math.nextafter(tp, math.inf if k > 0 else -math.inf)
            else:
                tp = math.exp(rng.uniform(math.log(50), math.log(5000)))
            trips.append([s, rng.choice([1, 2, 4]), rng.choice([1, 2, 3]), tp, float(rng.randint(1, 50))])
        tobj = [R.Triplet(*t) for t in trips]
        best = R.select_optimal_segment(tobj)
        idx = next(k for k, t in enumerate(tobj) if t is best)
        select.append({"triplets": trips, "index": idx})

    propose = []
    for i in range(3000):
        tp1 = _rand_tp(rng, False) if rng.random() < 0.85 else None
        tp2 = _rand_tp(rng, False) * rng.uniform(1.0, 2.2) if rng.random() < 0.85 else None
        mode = rng.random()
        if mode < 0.1:
            freed = -rng.uniform(0, 500) if rng.random() < 0.5 else 0.0
        elif mode < 0.4:
            unit = rng.choice([t for t in (tp1, tp2) if t is not None] or [100.0])
            freed = rng.randint(1, 9) * unit
            if rng.random() < 0.5:
                freed = math.nextafter(freed, math.inf if rng.random() < 0.5 else -math.inf)
        else:
            freed = rng.uniform(0, 5000)
        best = []
        if tp1 is not None:
            best.append(R.Triplet(1, 2, 1, tp1, 5.0))
        if tp2 is not None:
            best.append(R.Triplet(2, 4, 2, tp2, 6.0))
        svc = replace(R.make_service("p", "m", 1.0, 10.0), best_triplets=tuple(best))
        try:
            segs = R.propose_small_segments(svc, freed)
            k2 = sum(1 for t in segs if t.instance_size == 2)
            out = [k2, len(segs) - k2]
        except R.MigplanError as exc:
            out = canon.error(exc)
        propose.append({"tp1": tp1, "tp2": tp2, "freed": freed, "result": out})
    write("unit_cases.json", {"configure": configure, "select": select, "propose": propose})


# ------------------------------------------------------------ allocator
def _canon_map_in(d):
    return canon.dmap(d)


def _configured_services(rng, tables, k):
    out = []
    models = rng.sample(list(RF.MODEL_IDS), k)
    for m in models:
        for _ in range(20):
            svc = R.make_service(m, m, math.exp(rng.uniform(math.log(5), math.log(6000))),
                                 math.exp(rng.uniform(math.log(60), math.log(3000))))
            try:
                out.append(R.configure_service(svc, tables[m]))
                break
            except R.InfeasibleSLOError:
                continue
    return out


def gen_alloc_cases(tables, seed=4242):
    rng = random.Random(seed)
    relocate = []
    for i in range(200):
        svcs = _configured_services(rng, tables, rng.randint(1, 11))
        d = R.relocate_segments(svcs)
        relocate.append({"services": [canon.service(s) for s in svcs], "result": canon.dmap(d)})

    optimize = []
    # drained-GPU refill into an already-emptied GPU.
    def T(s, tp):
        return R.Triplet(s, 1, 1, tp, 1.0)

    def svc(name, trips, rate=1.0):
        return replace(R.make_service(name, name, rate, 10.0), best_triplets=tuple(trips))

    A = svc("A", [T(7, 700.0)]); B = svc("B", [T(1, 120.0), T(2, 200.0)]); C = svc("C", [T(1, 120.0), T(2, 200.0)])
    d = RDeploymentMap(gpus=[RGpuState(0, [RPlacement("A", 7, 1, 1, 700.0, 0)]),
                             RGpuState(1, [RPlacement("B", 2, 1, 1, 200.0, 0)]),
                             RGpuState(2, [RPlacement("C", 1, 1, 1, 120.0, 0)])])
    crafted = [(d, [A, B, C], 4, "appB3_drained_refill")]
    # regression fallback.
    A4 = svc("A", [T(1, 150.0), T(4, 100.0)]); X = svc("X", [T(1, 50.0)])
    d4 = RDeploymentMap(gpus=[RGpuState(0, [RPlacement("X", 1, 1, 1, 50.0, 0)]),
                              RGpuState(1, [RPlacement("A", 4, 1, 1, 100.0, 0)])])
    crafted.append((d4, [A4, X], 4, "appB4_regression_fallback"))
    for d, svcs, thr, tag in crafted:
        res = R.optimize_allocation(d, svcs, thr)
        optimize.append({"tag": tag, "services": [canon.service(s) for s in svcs],
                         "map": canon.dmap(d), "threshold": thr, "result": canon.dmap(res)})

    for i in range(300):
        svcs = _configured_services(rng, tables, rng.randint(1, 8))
        if not svcs:
            continue
        if rng.random() < 0.5:
            d = R.relocate_segments(svcs)
            # perturb: drop a few placements, shuffle GPU order and ids
            for g in d.gpus:
                g.placements = [p for p in g.placements if rng.random() < 0.8]
            d.gpus = [g for g in d.gpus if g.placements or rng.random() < 0.2]
            rng.shuffle(d.gpus)
            for g in d.gpus:
                g.id = g.id * 3 + rng.randint(0, 2)
        else:
            gpus = []
            ids = rng.sample(range(100), rng.randint(1, 7))
            for gid in ids:
                g = RGpuState(gid)
                for _ in range(rng.randint(0, 6)):
                    s = rng.choice(svcs)
                    t = rng.choice(s.best_triplets)
                    sid = s.id if rng.random() > 0.03 else "ghost"
                    g.place(sid, t.instance_size, t.batch_size, t.process_count, t.throughput)
                gpus.append(g)
            d = RDeploymentMap(gpus=gpus)
        if rng.random() < 0.9:
            # keep optimize's coverage assert (allocator.py:437-442) satisfiable
            cov = {}
            for g in d.gpus:
                for p in g.placements:
                    cov[p.service_id] = cov.get(p.service_id, 0.0) + p.throughput
            svcs = [replace(s, request_rate=min(s.request_rate, 0.5 * cov.get(s.id, 0.0))) for s in svcs]
        if rng.random() < 0.3:
            for s in rng.sample(svcs, rng.randint(1, len(svcs))):
                d.freed_rate[s.id] = rng.uniform(-300, 300)
        if rng.random() < 0.2:
            d.diagnostics.append("earlier note")
        thr = rng.choice([4, 4, 4, 2, 3, 5, 7])
        try:
            res = canon.dmap(R.optimize_allocation(d, svcs, thr))
        except (R.MigplanError, AssertionError) as exc:
            res = canon.error(exc)
        optimize.append({"tag": f"random{i}", "services": [canon.service(s) for s in svcs],
                         "map": canon.dmap(d), "threshold": thr, "result": res})
    write("alloc_cases.json", {"relocate": relocate, "optimize": optimize})


# ------------------------------------------------------- reconfigure (§8f-1)
def gen_reconfigure(tables, n=120, seed=31337):
    rng = random.Random(seed)
    cases = []
    for i in range(n):
        k = rng.randint(2, 9)
        models = rng.sample(list(RF.MODEL_IDS), k)
        inputs = [[m, m, math.exp(rng.uniform(math.log(20), math.log(6000))),
                   math.exp(rng.uniform(math.log(100), math.log(3000)))] for m in models]
        services = [R.make_service(a, m, r, s) for a, m, r, s in inputs]
        try:
            res = R.plan_services(services, tables)
        except R.MigplanError:
            continue
        target = rng.randrange(k)
        mode = rng.random()
        old = res.services[target]
        if mode < 0.15:
            new_rate, new_slo = old.request_rate, old.slo_latency          # unchanged demand
        elif mode < 0.25:
            new_rate, new_slo = old.request_rate, 1.0                      # infeasible SLO
        else:
            new_rate = old.request_rate * rng.choice([0.3, 0.7, 1.5, 2.0, 3.0])
            new_slo = old.slo_latency * rng.choice([0.6, 1.0, 1.4])
        updated = R.make_service(old.id, old.model_id, new_rate, new_slo)
        thr = rng.choice([4, 4, 3, 5])
        table = R.filter_feasible(tables[old.model_id])
        try:
            dmap, changes, new_services = R.reconfigure_service(res.deployment, res.services, updated, table, thr)
            out = {"map": canon.dmap(dmap), "changes": [c.to_json_obj() for c in changes],
                   "services": [canon.service(s) for s in new_services]}
        except R.MigplanError as exc:
            out = canon.error(exc)
        cases.append({"inputs": inputs, "target": target, "new_rate": new_rate, "new_slo": new_slo,
                      "threshold": thr, "base": canon.plan(res), "result": out})
    write("reconfigure_cases.json", cases)


# ------------------------------------------------------------------ C2
def gen_c2(tables, n=10_000, full=200):
    fx = W.load_fixtures()
    sb = W.scenario_batch(fx, n, seed=0)
    digests, fulls = [], []
    t0 = time.perf_counter()
    n_infeasible = 0
    for k in range(n):
        services = [R.make_service(m, m, float(sb.rate[k, j]), float(sb.slo[k, j]))
                    for j, m in enumerate(sb.models)]
        try:
            out = canon.plan(R.plan_services(services, tables))
        except R.MigplanError as exc:
            out = canon.error(exc)
            n_infeasible += 1
        digests.append(canon.digest(out))
        if k < full:
            fulls.append(out)
    dt = time.perf_counter() - t0
    inp = hashlib.sha256(sb.rate.tobytes() + sb.slo.tobytes()).hexdigest()[:16]
    write("c2_digests.json", {"n": n, "seed": 0, "input_sha256": inp, "digests": digests,
                              "full": fulls, "n_infeasible": n_infeasible,
                              "reference_seconds_1core": dt})
    print(f"C2: {n} scenarios in {dt:.1f}s on 1 core ({n / dt:.0f} scen/s), infeasible {n_infeasible}")


# ------------------------------------------------------------------ C3
def gen_c3(n=200):
    dt = W.dense_tables(n, seed=3)
    prm = W.dense_params(n, seed=3)
    rows = []
    t_cfg = 0.0
    npts = 0
    for w in range(n):
        params = R.SyntheticModelParams(
            model_id=f"w{w:05d}", base_throughput=float(prm["base"][w]),
            gpc_exponent=float(prm["gexp"][w]), sat_work=float(prm["sat"][w]),
            sat_exponent=float(prm["sexp"][w]), weight_memory_gb=float(prm["wmem"][w]),
            activation_memory_gb=float(prm["amem"][w]), jitter=0.0)
        table = R.filter_feasible(R.synthesize_profile(params, seed=w, batch_sizes=range(1, 129),
                                                       process_counts=range(1, 9)))
        mine = W.dense_table_objects(dt, w)
        ref_pts = [(p.instance_size, p.batch_size, p.process_count, p.throughput, p.latency) for p in table.points]
        my_pts = [(p.instance_size, p.batch_size, p.process_count, p.throughput, p.latency) for p in mine.points]
        assert ref_pts == my_pts, f"C3 generator mismatch at workload {w}"
        svc = R.make_service(f"w{w:05d}", f"w{w:05d}", float(prm["rate"][w]), float(prm["slo"][w]))
        t0 = time.perf_counter()
        try:
            out = canon.service(R.configure_service(svc, table))
        except R.MigplanError as exc:
            out = canon.error(exc)
        t_cfg += time.perf_counter() - t0
        npts += len(table)
        rows.append({"points": len(table), "table_sha": hashlib.sha256(repr(ref_pts).encode()).hexdigest()[:16],
                     "result": out})
    write("c3_sample.json", {"n": n, "seed": 3, "rows": rows,
                             "reference_points_per_s_1core": npts / t_cfg})
    print(f"C3: {n} workloads, {npts} points, configure {npts / t_cfg / 1e6:.2f} M pts/s/core")


# ------------------------------------------------------------------ C5
def gen_c5(tables):
    table = tables[W.C5_MODEL]
    rates = W.c5_rates(W.C5_SERVICES + 50)
    svcs, nseg = [], 0
    for i, r in enumerate(rates.tolist()):
        s = R.configure_service(R.make_service(f"d121#{i}", W.C5_MODEL, r, W.C5_SLO), table)
        svcs.append(s)
        nseg += len(s.segments())
        if nseg >= 100_000:
            break
    assert len(svcs) == W.C5_SERVICES, (len(svcs), nseg)
    t0 = time.perf_counter()
    d = R.relocate_segments(svcs)
    t1 = time.perf_counter()
    o = R.optimize_allocation(d, svcs)
    t2 = time.perf_counter()
    sizes = {}
    for s in svcs:
        for t in s.segments():
            sizes[t.instance_size] = sizes.get(t.instance_size, 0) + 1
    write("c5_summary.json", {
        "services": len(svcs), "segments": nseg, "segments_by_size": sizes,
        "unopt_gpus": d.gpu_count, "gpus": o.gpu_count, "total_gpcs": o.total_gpcs,
        "relocate_sha256": canon.digest(canon.dmap(d)), "optimized_sha256": canon.digest(canon.dmap(o)),
        "json_sha256": hashlib.sha256(o.to_json().encode()).hexdigest()[:16],
        "n_diags": len(o.diagnostics), "freed_sha256": canon.digest([[k, v] for k, v in o.freed_rate.items()]),
        "reference_relocate_s": t1 - t0, "reference_optimize_s": t2 - t1})
    print(f"C5: {len(svcs)} services {nseg} segments {d.gpu_count} -> {o.gpu_count} GPUs "
          f"(relocate {t1 - t0:.1f}s optimize {t2 - t1:.1f}s)")


# ------------------------------------------------------------ simulator
SIM_SETS = [
    # (scenario, plan options, arrivals, rate scale, horizon s, seed)
    *[(name, "default", "poisson", 1.0, 3.0, 0) for name in ("S1", "S2", "S3", "S4", "S5", "S6")],
    *[(name, "default", "deterministic", 1.0, 3.0, 1) for name in ("S1", "S3", "S6")],
    ("S2", "default", "poisson", 1.6, 4.0, 7), ("S6", "default", "poisson", 1.4, 2.0, 3),
    ("S4", "default", "poisson", 0.3, 5.0, 11), ("S5", "single", "poisson", 1.0, 2.5, 5),
    ("S6", "default", "deterministic", 1.7, 2.0, 2), ("S1", "default", "poisson", 2.5, 6.0, 13),
    ("S6", "default", "poisson", 1.0, 10.0, 21),
]


def gen_sim(tables):
    out = []
    for name, oname, kind, scale, horizon, seed in SIM_SETS:
        sc = RF.make_scenario(name)
        opts = R.PlanOptions(**OPTION_SETS[oname])
        res = R.plan_scenario(sc, tables, opts)
        from migplan.pipeline import prepare_tables as _prep
        prepared = _prep(tables, opts)
        wl = R.Workload.from_services(R.scenario_services(sc), kind=kind, scale=scale)
        t0 = time.perf_counter()
        rep = R.run_simulation(res.deployment, prepared, res.services, workload=wl, horizon_s=horizon, seed=seed)
        dt = time.perf_counter() - t0
        obj = rep.to_json_obj()
        obj["metrics"] = {"internal_slack": R.internal_slack(rep.activity) if rep.activity.segments else None,
                          "slo_compliance": R.slo_compliance(rep)}
        out.append({"scenario": name, "options": oname, "arrivals": kind, "rate_scale": scale,
                    "horizon_s": horizon, "seed": seed, "map": res.deployment.to_json(), "report": obj,
                    "reference_s": dt})
        print(f"  sim {name} {oname} {kind} x{scale} {horizon}s seed {seed}: {dt:.2f} s")
    # explicit-input cases: an extra service that is defined but never placed,
    # zero rates, both arrival kinds
    sc = RF.make_scenario("S3")
    res = R.plan_scenario(sc, tables, R.PlanOptions())
    services = list(res.services) + [R.make_service("idle", res.services[0].model_id, 50.0, 500.0)]
    rates = [(s.id, 0.0 if i % 3 == 0 else s.request_rate) for i, s in enumerate(res.services)] + [("idle", 50.0)]
    for kind in ("poisson", "deterministic"):
        rep = R.run_simulation(res.deployment, tables, services, workload=R.Workload(tuple(rates), kind),
                               horizon_s=1.5, seed=3)
        obj = rep.to_json_obj()
        obj["metrics"] = {"internal_slack": R.internal_slack(rep.activity) if rep.activity.segments else None,
                          "slo_compliance": R.slo_compliance(rep)}
        out.append({"scenario": "S3", "options": "default", "arrivals": kind, "rate_scale": 1.0, "horizon_s": 1.5,
                    "seed": 3, "map": res.deployment.to_json(), "report": obj, "reference_s": None,
                    "services": [[s.id, s.model_id, s.request_rate, s.slo_latency] for s in services],
                    "rates": [[sid, r] for sid, r in rates]})
    write("sim_cases.json", out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    tables = ref_tables()
    steps = {"tables": lambda: gen_fixture_tables(tables), "fixture": lambda: gen_fixture_plans(tables),
             "fuzz": lambda: gen_fuzz_plans(tables), "unit": gen_unit_cases,
             "alloc": lambda: gen_alloc_cases(tables), "reconf": lambda: gen_reconfigure(tables),
             "c2": lambda: gen_c2(tables), "c3": gen_c3, "sim": lambda: gen_sim(tables)}
    if a.c5:
        steps["c5"] = lambda: gen_c5(tables)
    for name, fn in steps.items():
        if a.only and name not in a.only.split(","):
            continue
        fn()


if __name__ == "__main__":
    main()
