"""Pin the C oracle against golden vectors rendered from the reference.

CPU-only: these tests never touch CUDA.  They are what makes the oracle a
trustworthy checker for the GPU parity tests (tests/test_gpu_parity.py).
"""

import hashlib
import math
import random

import numpy as np
import pytest

import oracle
from helpers import canon, golden, oracle_plan_canon, map_canon, service_canon
from paper_2409_14447_b200 import workloads as W
from paper_2409_14447_b200.profiles import ProfilePoint, ProfileTable, serialize_profile_table
from paper_2409_14447_b200.tables import pack_tables, pack_dense


@pytest.fixture(scope="module")
def fx():
    return W.load_fixtures()


def _pack(fx, options):
    mm = options.get("memory_map")
    if mm is not None:
        mm = {int(s): float(v) for s, v in mm}
    return pack_tables(fx.tables, memory_map=mm, single_process=options.get("single_process", False))


def test_fixture_tables_match_reference_csv(fx):
    g = golden("fixture_tables.json")
    for m in fx.models:
        sha = hashlib.sha256(serialize_profile_table(fx.tables[m], "csv").encode()).hexdigest()[:16]
        assert sha == g["csv_sha256"][m]
    assert g["csv_sha256"]["inceptionv3"] == "a34f57a6f81f9392"
    assert g["csv_sha256"]["resnet50"] == "c5082c21144f5b1b"


def test_pysum_is_python312_sum():
    rng = random.Random(5)
    for _ in range(3000):
        n = rng.randint(0, 40)
        xs = [rng.choice([0.1, 1e16, -1e16, 3.3, rng.uniform(-1e6, 1e6), 1e-9]) for _ in range(n)]
        assert oracle.pysum(xs) == sum(xs), xs
    assert oracle.pysum([0.1] * 10) == 1.0


OPTS = {"default": {}, "noopt": {"optimize": False}, "single": {"single_process": True}}


def test_fixture_plans(fx):
    for case in golden("fixture_plans.json"):
        opts = OPTS[case["options"]]
        pt = _pack(fx, opts)
        inputs = [[m, m, r, s] for m, r, s in case["inputs"]]
        got = oracle_plan_canon(oracle, pt, inputs, opts)
        assert got == case["plan"], (case["scenario"], case["options"])


def test_fixture_gpu_counts(fx):
    counts = {(c["scenario"], c["options"]): len(c["plan"]["gpus"]) for c in golden("fixture_plans.json")}
    assert [counts[(f"S{i}", "default")] for i in range(1, 7)] == [1, 2, 3, 4, 8, 9]
    assert [counts[(f"S{i}", "single")] for i in range(1, 7)] == [1, 2, 3, 4, 8, 10]


def test_fuzz_plans(fx):
    packs = {}
    for i, case in enumerate(golden("fuzz_plans.json")):
        opts = case["options"]
        key = (repr(opts.get("memory_map")), opts.get("single_process", False))
        if key not in packs:
            packs[key] = _pack(fx, opts)
        got = oracle_plan_canon(oracle, packs[key], case["inputs"], opts)
        assert got == case["result"], i


def _single_table(points):
    t = ProfileTable("m", tuple(ProfilePoint("m", s, b, p, tp, lat) for s, b, p, tp, lat in points))
    return pack_tables([t], prepared=True)


def test_unit_configure():
    for i, case in enumerate(golden("unit_cases.json")["configure"]):
        pt = _single_table(case["points"])
        rec = oracle.configure_batch(pt, [0], [case["rate"]], [case["bound"]])[0]
        res = case["result"]
        if "error" in res:
            assert rec["status"] == 1 and res["error"] == "InfeasibleSLOError", i
            continue
        got = service_canon("s", "m", case["rate"], 1.0, case["bound"], pt, 0, rec)
        assert got == res, i


def test_unit_select_optimal():
    for case in golden("unit_cases.json")["select"]:
        trips = [(t[0], t[3]) for t in case["triplets"]]
        assert oracle.select_optimal(trips) == case["index"], case


def test_unit_propose():
    for case in golden("unit_cases.json")["propose"]:
        got = oracle.propose(case["tp1"], case["tp2"], case["freed"])
        res = case["result"]
        if isinstance(res, dict):
            assert got is None and res["error"] == "SmallSegmentsUnavailableError", case
        else:
            assert list(got) == res, case


def _services_general(svcs):
    out = []
    for s in svcs:
        out.append({"best": {t[0]: t[:4] + [0.0] for t in s["best"]}, "opt": s["opt"], "count": s["count"],
                    "last": s["last"], "rate": s["rate"]})
    return out


def _general_case(svcs, dmap_in, relocate, optimize, threshold):
    names = [s["id"] for s in svcs]
    extra = []
    for _, pls in (dmap_in["gpus"] if dmap_in else []):
        for p in pls:
            if p[0] not in names and p[0] not in extra:
                extra.append(p[0])
    for k, _ in (dmap_in["freed"] if dmap_in else []):
        if k not in names and k not in extra:
            extra.append(k)
    allnames = names + extra
    nid = {n: i for i, n in enumerate(allnames)}
    gpus = [(gid, [(nid[p[0]], p[1:5], p[5]) for p in pls]) for gid, pls in (dmap_in["gpus"] if dmap_in else [])]
    ledger = {nid[k]: (v, r + 1) for r, (k, v) in enumerate(dmap_in["freed"] if dmap_in else [])}
    res = oracle.plan_general(len(allnames), _services_general(svcs), gpus, ledger, relocate, optimize, threshold)
    return res, allnames


def test_alloc_relocate():
    for i, case in enumerate(golden("alloc_cases.json")["relocate"]):
        res, names = _general_case(case["services"], None, 1, 0, 4)
        assert map_canon(res, names) == case["result"], i


def test_alloc_optimize():
    for i, case in enumerate(golden("alloc_cases.json")["optimize"]):
        res, names = _general_case(case["services"], case["map"], 0, 1, case["threshold"])
        exp = case["result"]
        if "error" in exp:
            assert exp["error"] == "AssertionError" and res["status"] == 6, (i, case["tag"])
            continue
        assert res["status"] == 0, (i, case["tag"])
        got = map_canon(res, names, prior_diags=case["map"]["diags"])
        if res["fallback"]:
            # fallback returns the input clone: its ledger, not the optimize pass's
            got["freed"] = case["map"]["freed"]
        assert got == exp, (i, case["tag"])


def test_c2_digests(fx):
    g = golden("c2_digests.json")
    sb = W.scenario_batch(fx, g["n"], seed=g["seed"])
    assert hashlib.sha256(sb.rate.tobytes() + sb.slo.tobytes()).hexdigest()[:16] == g["input_sha256"]
    pt = pack_tables(fx.tables)
    bad = []
    for k in range(g["n"]):
        inputs = [[m, m, float(sb.rate[k, j]), float(sb.slo[k, j])] for j, m in enumerate(sb.models)]
        got = oracle_plan_canon(oracle, pt, inputs, {})
        if k < len(g["full"]):
            assert got == g["full"][k], k
        if canon.digest(got) != g["digests"][k]:
            bad.append(k)
    assert not bad, bad[:10]


def test_c3_sample():
    g = golden("c3_sample.json")
    dt = W.dense_tables(g["n"], seed=g["seed"])
    pt = pack_dense(dt)
    n = g["n"]
    recs = oracle.configure_batch(pt, np.arange(n), dt.rate, dt.slo / 2.0)
    for w in range(n):
        row = g["rows"][w]
        assert int(dt.seg_count[w * 5:(w + 1) * 5].sum()) == row["points"]
        if "error" in row["result"]:
            assert recs[w]["status"] == 1
            continue
        sid = f"w{w:05d}"
        got = service_canon(sid, sid, dt.rate[w], dt.slo[w], dt.slo[w] / 2.0, pt, w, recs[w])
        assert got == row["result"], w


@pytest.mark.slow
def test_c5_large_cluster(fx):
    g = golden("c5_summary.json")
    pt = pack_tables(fx.tables)
    t = pt.index_of()[W.C5_MODEL]
    rates = W.c5_rates()
    n = rates.shape[0]
    cfg, res = oracle.plan_scenario(pt, np.full(n, t), rates, np.full(n, W.C5_SLO / 2.0), True, 4,
                                    gcap=200_000)
    assert res["unopt"] == g["unopt_gpus"] and len(res["gpus"]) == g["gpus"]
    names = [f"d121#{i}" for i in range(n)]
    assert canon.digest(map_canon(res, names)) == g["optimized_sha256"]


def test_record_format_decodes_to_reference_plans(fx):
    """Oracle -> 128-byte plan records -> this package's decoder -> canonical
    plans == the reference's digests.  Pins the record format and the decoder
    (used on the GPU path) without a GPU."""
    from paper_2409_14447_b200.configurator import make_service, raise_for_record, service_from_record
    from paper_2409_14447_b200.errors import MigplanError
    from paper_2409_14447_b200.pipeline import PlanResult, _decode_record
    g = golden("c2_digests.json")
    n = 3000
    sb = W.scenario_batch(fx, n, seed=g["seed"])
    pt = pack_tables(fx.tables)
    M = len(sb.models)
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    cfg, plan = oracle.plan_batch_records(pt, off, tab, sb.rate.ravel(), sb.bound.ravel())
    for k in range(n):
        svcs = [make_service(m, m, float(sb.rate[k, j]), float(sb.slo[k, j])) for j, m in enumerate(sb.models)]
        try:
            conf = []
            for j, s in enumerate(svcs):
                raise_for_record(s, cfg[k * M + j])
                conf.append(service_from_record(s, pt, j, cfg[k * M + j]))
            assert plan[k]["status"] == 0
            res = PlanResult("", conf, _decode_record(conf, plan[k]), 0.0, int(plan[k]["n_gpus_unopt"]))
            got = canon.plan(res)
        except MigplanError as exc:
            got = canon.error(exc)
        assert canon.digest(got) == g["digests"][k], k


def test_plan_metrics_from_records(fx):
    """§8f row 3: fragmentation / allocated fraction from the plan records equal
    the reference's summary() values on S1-S6 (evaluation.py:65-82)."""
    from paper_2409_14447_b200.evaluation import plan_metrics
    cases = [c for c in golden("fixture_plans.json") if c["options"] == "default"]
    pt = pack_tables(fx.tables)
    idx = pt.index_of()
    off = [0]
    tab, rate, bound = [], [], []
    for c in cases:
        for m, r, s in c["inputs"]:
            tab.append(idx[m]); rate.append(r); bound.append(s / 2.0)
        off.append(len(tab))
    _, plan = oracle.plan_batch_records(pt, np.array(off), np.array(tab), np.array(rate), np.array(bound))
    met = plan_metrics(plan)
    for k, c in enumerate(cases):
        assert met["gpu_count"][k] == c["summary"]["gpu_count"]
        assert met["total_gpcs"][k] == c["summary"]["total_gpcs"]
        assert met["allocated_fraction"][k] == c["summary"]["allocated_fraction"]
        assert met["external_fragmentation"][k] == c["summary"]["external_fragmentation"]


def test_sim_oracle_vs_reference_reports():
    """run_simulation (evaluation.py:286-464) with the C event loop: every
    report of tests/golden/sim_cases.json (rendered by the reference) is
    reproduced exactly -- JSON, internal slack and SLO compliance."""
    import json
    from helpers import sim_report_with_oracle, sim_scenario_inputs
    from paper_2409_14447_b200 import simulation as S
    from paper_2409_14447_b200 import workloads as W
    fx = W.load_fixtures()
    cases = golden("sim_cases.json")
    assert len(cases) >= 16
    for case in cases:
        dmap, services, wl = sim_scenario_inputs(case, fx)
        job = S.SimJob(dmap, fx.tables, services, wl, case["horizon_s"], case["seed"])
        rep, _, _ = sim_report_with_oracle(oracle, job)
        obj = rep.to_json_obj()
        obj["metrics"] = {"internal_slack": S.internal_slack(rep.activity) if rep.activity.segments else None,
                          "slo_compliance": S.slo_compliance(rep)}
        assert json.loads(json.dumps(obj)) == case["report"], (case["scenario"], case["arrivals"], case["seed"])


def test_plan_many_lazy_results_decode_to_reference_plans(fx, monkeypatch):
    """plan_many's lazy results (LazyPlanResult) and its vectorized error
    path, with the oracle standing in for the device (CPU): every one of the
    first 3000 C2 scenarios decodes to the reference's digest; gpu_count is
    answered from the record before any decode; results compare equal to the
    eagerly decoded PlanResult."""
    import types
    import paper_2409_14447_b200 as P
    from paper_2409_14447_b200 import _native as Nm
    from paper_2409_14447_b200 import pipeline as PL
    from paper_2409_14447_b200.records import CONFIG_DTYPE, PLAN_DTYPE
    g = golden("c2_digests.json")
    n = 3000
    sb = W.scenario_batch(fx, n, seed=g["seed"])
    pt = pack_tables(fx.tables)

    def fake_plan_batch(dt, off, tab, rate, bound, optimize=True, threshold=4, **kw):
        cfg, plan = oracle.plan_batch_records(pt, off, tab, rate, bound, optimize=optimize, threshold=threshold)
        return types.SimpleNamespace(host=lambda: (cfg.view(CONFIG_DTYPE), plan.view(PLAN_DTYPE)))

    monkeypatch.setattr(PL, "plan_batch", fake_plan_batch)
    monkeypatch.setattr(PL, "resolve_capacity", lambda *a, **k: {})
    monkeypatch.setattr(Nm, "device_tables_for", lambda *a, **k: types.SimpleNamespace(packed=pt, index_struct=None))
    monkeypatch.setattr(Nm, "require_cuda", lambda: types.SimpleNamespace(
        cuda=types.SimpleNamespace(synchronize=lambda: None)))
    sets = [[P.make_service(m, m, float(sb.rate[k, j]), float(sb.slo[k, j])) for j, m in enumerate(sb.models)]
            for k in range(n)]
    res = P.plan_many(sets, fx.tables)
    n_err = 0
    for k, r in enumerate(res):
        if isinstance(r, Exception):
            n_err += 1
            got = canon.error(r)
        else:
            assert isinstance(r, PL.PlanResult) and r._dec is None
            cnt = r.gpu_count                     # from the record, no decode
            assert r._dec is None
            got = canon.plan(r)
            assert r.gpu_count == cnt == r.deployment.gpu_count
        assert canon.digest(got) == g["digests"][k], k
    assert n_err == 30
    # a lazy result equals the eager one and survives dataclasses.replace / summary
    import dataclasses
    k = next(i for i, r in enumerate(res) if not isinstance(r, Exception))
    lazy = P.plan_many([sets[k]], fx.tables)[0]
    eager = PL.PlanResult(lazy.scenario_name, lazy.services, lazy.deployment, lazy.planning_ms,
                          lazy.unoptimized_gpu_count)
    assert lazy == eager
    assert dataclasses.replace(lazy, scenario_name="x").deployment.to_json() == eager.deployment.to_json()
    assert lazy.summary() == eager.summary()
    with pytest.raises(P.InfeasibleSLOError):
        P.plan_services(sets[next(i for i, r in enumerate(res) if isinstance(r, Exception))], fx.tables)
    # repeated service ids: rejected (a documented deviation)
    dup = [dataclasses.replace(s, id="same") for s in sets[k][:3]]
    got = P.plan_many([sets[k], dup], fx.tables)
    assert isinstance(got[1], P.ValidationError) and not isinstance(got[0], Exception)
