"""Shared test helpers: canonical dicts (tests/golden/canon.py) from the C
oracle's outputs and from this package's records."""

from __future__ import annotations

import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
for p in (str(REPO), str(GOLDEN)):
    if p not in sys.path:
        sys.path.insert(0, p)

import json  # noqa: E402

import canon  # noqa: E402,F401
from paper_2409_14447_b200 import errors  # noqa: E402
from paper_2409_14447_b200.records import format_diag  # noqa: E402

SIZES = (1, 2, 3, 4, 7)
_cache = {}


def golden(name):
    if name not in _cache:
        _cache[name] = json.loads((GOLDEN / name).read_text())
    return _cache[name]


def trip_from(pt, t, c, j):
    i = pt.point(t, c, j)
    return [SIZES[c], int(pt.batch[i]), int(pt.procs[i]), float(pt.tp[i]), float(pt.lat[i])]


def service_canon(sid, model, rate, slo, internal, pt, t, rec):
    best = [trip_from(pt, t, c, int(rec["best"][c])) for c in range(5) if rec["best"][c] >= 0]
    o, l = int(rec["opt_sc"]), int(rec["last_sc"])
    return {"id": sid, "model": model, "rate": float(rate), "slo": float(slo), "internal": float(internal),
            "best": best, "opt": trip_from(pt, t, o, int(rec["best"][o])) if o >= 0 else None,
            "count": int(rec["count"]),
            "last": trip_from(pt, t, l, int(rec["best"][l])) if l >= 0 else None,
            "coverage": float(rec["coverage"])}


def config_error(rec, sid, bound):
    st = int(rec["status"])
    if st == 1:
        return canon.error(errors.InfeasibleSLOError(sid, bound))
    raise AssertionError(f"unexpected config status {st}")


def oracle_plan_canon(oracle, pt, inputs, options):
    """inputs: [[sid, model, rate, slo], ...] -> canonical plan dict or error dict."""
    idx = pt.index_of()
    tab = [idx[m] for _, m, _, _ in inputs]
    rate = [float(r) for _, _, r, _ in inputs]
    slo = [float(s) for _, _, _, s in inputs]
    bound = [s / 2.0 for s in slo]
    cfg, res = oracle.plan_scenario(pt, tab, rate, bound, options.get("optimize", True),
                                    options.get("threshold", 4))
    for k, (sid, m, r, s) in enumerate(inputs):
        if cfg[k]["status"]:
            return config_error(cfg[k], sid, bound[k])
    names = [sid for sid, _, _, _ in inputs]
    out = {"services": [service_canon(sid, m, r, s, b, pt, t, cfg[k])
                        for k, ((sid, m, r, s), t, b) in enumerate(zip(inputs, tab, bound))],
           "unopt": res["unopt"]}
    out.update(map_canon(res, names))
    return out


def map_canon(res, names, prior_diags=()):
    gpus = [[gid, [[names[n], sz, b, p, tp, slot] for n, sz, b, p, tp, slot in pls]] for gid, pls in res["gpus"]]
    diags = list(prior_diags) + [format_diag(r, g, names[n] if n >= 0 else None) for r, g, n in res["diags"]]
    return {"gpus": gpus, "freed": [[names[k], v] for k, v in res["ledger"]], "diags": diags}


def sim_scenario_inputs(case, fixtures):
    """(DeploymentMap, services, Workload) of a tests/golden/sim_cases.json case."""
    import paper_2409_14447_b200 as P
    from paper_2409_14447_b200.scenario import ScenarioService
    from paper_2409_14447_b200.simulation import Workload
    dmap = P.DeploymentMap.from_json(case["map"])
    if "services" in case:        # explicit inputs
        services = [P.make_service(sid, model, rate, slo) for sid, model, rate, slo in case["services"]]
        wl = Workload(tuple((sid, r) for sid, r in case["rates"]), case["arrivals"])
        return dmap, services, wl
    sc = P.Scenario(case["scenario"], tuple(ScenarioService(m, r, s) for m, r, s in fixtures.scenarios[case["scenario"]]))
    services = P.scenario_services(sc)
    wl = Workload.from_services(services, kind=case["arrivals"], scale=case["rate_scale"])
    return dmap, services, wl


def sim_report_with_oracle(oracle, job):
    """run_simulation with numpy arrivals on the host and the C oracle as the
    event loop (CPU; test only) -- an independent path from the GPU's."""
    import numpy as np
    from paper_2409_14447_b200 import simulation as S
    pr = S._Prepared(job)
    per = [[] for _ in pr.ids]
    for gi, (si, p, gid, ms) in enumerate(pr.segments):
        per[si].append(gi)
    arrived, served, batches, viol, lats, busy = [], [], [], [], [], {}
    for si in range(len(pr.ids)):
        segs = [pr.segments[g] for g in per[si]]
        arr = pr.host_arrivals(si)
        sv, nb, nv, lat, bz = oracle.simulate_service(arr, [x[3] for x in segs], [x[1].batch_size for x in segs],
                                                      [x[1].process_count for x in segs],
                                                      pr.svc[si].slo_latency, pr.horizon_ms)
        arrived.append(arr.shape[0]); served.append(sv); batches.append(nb); viol.append(nv); lats.append(lat)
        for k, g in enumerate(per[si]):
            busy[g] = bz[k]
    rep = S._report(pr, [(x, None) for x in lats], np.array(arrived), np.array(served), np.array(batches),
                    np.array(viol), busy)
    return rep, lats, busy
