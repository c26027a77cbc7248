"""GPU parity: the sm_100a kernels vs the reference goldens and the C oracle.

Bar (BASELINE.json north_star): integer decisions bit-exact, floats within
1e-9 relative — in practice every float here is compared bit-exactly
(tolerance 0), because the kernels reproduce CPython's operation order.
"""

import hashlib

import numpy as np
import pytest

import oracle
from helpers import canon, golden, map_canon, service_canon

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2409_14447_b200 as P  # noqa: E402
from paper_2409_14447_b200 import _native as N  # noqa: E402
from paper_2409_14447_b200 import batch as B  # noqa: E402
from paper_2409_14447_b200 import workloads as W  # noqa: E402
from paper_2409_14447_b200.configurator import Service, Triplet  # noqa: E402
from paper_2409_14447_b200.records import (CFG_COMPACT, CFG_TINY, CONFIG_DTYPE, PLAN_DTYPE, TINY_DTYPE,  # noqa: E402
                                           compact_config)
from paper_2409_14447_b200.tables import pack_dense, pack_tables  # noqa: E402


@pytest.fixture(scope="module")
def fx():
    return W.load_fixtures()


def _opts(o):
    kw = {k: v for k, v in o.items() if k != "memory_map"}
    if "memory_map" in o:
        kw["memory_map"] = {int(s): float(v) for s, v in o["memory_map"]}
    return P.PlanOptions(**kw)


def _canon_result(r):
    return canon.error(r) if isinstance(r, Exception) else canon.plan(r)


def test_library_is_loaded_from_tree():
    lib = N.lib()
    assert "paper_2409_14447_b200/_build/libparva_b200.so" in lib._name


def test_fixture_plans(fx):
    for case in golden("fixture_plans.json"):
        opts = {"default": {}, "noopt": {"optimize": False}, "single": {"single_process": True}}[case["options"]]
        sc = P.Scenario(case["scenario"], tuple(P.scenario.ScenarioService(m, r, s) for m, r, s in case["inputs"]))
        res = P.plan_scenario(sc, fx.tables, P.PlanOptions(**opts))
        assert canon.plan(res) == case["plan"], (case["scenario"], case["options"])
        assert hashlib.sha256(res.deployment.to_json().encode()).hexdigest()[:16] == case["json_sha256"]
        summ = res.summary()
        summ.pop("planning_ms")
        assert summ == case["summary"]


def test_fuzz_plans_batched(fx):
    cases = golden("fuzz_plans.json")
    groups = {}
    for i, c in enumerate(cases):
        groups.setdefault(repr(sorted(c["options"].items())), []).append(i)
    for _, idxs in groups.items():
        opts = _opts(cases[idxs[0]]["options"])
        sets = [[P.make_service(a, m, r, s) for a, m, r, s in cases[i]["inputs"]] for i in idxs]
        results = P.plan_many(sets, fx.tables, opts)
        for i, r in zip(idxs, results):
            assert _canon_result(r) == cases[i]["result"], i


def test_unit_configure_sweep():
    cases = golden("unit_cases.json")["configure"]
    tables = [P.ProfileTable(f"t{i}", tuple(P.ProfilePoint(f"t{i}", s, b, p, tp, lat)
                                            for s, b, p, tp, lat in c["points"])) for i, c in enumerate(cases)]
    pt = pack_tables(tables, prepared=True)
    dt = N.DeviceTables(pt)
    out = B.configure_sweep(dt, np.arange(len(cases)), [c["rate"] for c in cases], [c["bound"] for c in cases])
    recs = N.records_to_numpy(out, len(cases), CONFIG_DTYPE)
    for i, c in enumerate(cases):
        if "error" in c["result"]:
            assert recs[i]["status"] == 1, i
        else:
            got = service_canon("s", "m", c["rate"], 1.0, c["bound"], pt, i, recs[i])
            assert got == c["result"], i
    # the K2 indexed path must agree with the streaming sweep on the same tables
    res = B.plan_batch(dt, np.arange(len(cases) + 1), np.arange(len(cases)), [c["rate"] for c in cases],
                       [c["bound"] for c in cases])
    cfg2, _ = res.host()
    assert cfg2.tobytes() == recs.tobytes()


def test_unit_configure_object_api():
    for c in golden("unit_cases.json")["configure"][:60]:
        table = P.ProfileTable("m", tuple(P.ProfilePoint("m", s, b, p, tp, lat) for s, b, p, tp, lat in c["points"]))
        svc = P.make_service("s", "m", c["rate"], 1.0, internal_latency=c["bound"])
        try:
            got = canon.service(P.configure_service(svc, table))
        except P.MigplanError as exc:
            got = canon.error(exc)
        assert got == c["result"]


def test_unit_select_optimal():
    for c in golden("unit_cases.json")["select"][:300]:
        trips = [Triplet(*t) for t in c["triplets"]]
        assert P.select_optimal_segment(trips) is trips[c["index"]]


def test_unit_propose_batched():
    cases = golden("unit_cases.json")["propose"]
    n = len(cases)
    tp1 = N.to_device(np.array([c["tp1"] or 0.0 for c in cases]))
    tp2 = N.to_device(np.array([c["tp2"] or 0.0 for c in cases]))
    fr = N.to_device(np.array([c["freed"] for c in cases]))
    k2 = torch.empty(n, dtype=torch.int64, device="cuda")
    k1 = torch.empty(n, dtype=torch.int64, device="cuda")
    ok = torch.empty(n, dtype=torch.uint8, device="cuda")
    import ctypes as C
    N.check(N.lib().parva_propose_small_batch(C.c_int32(n), N.ptr(tp1), N.ptr(tp2), N.ptr(fr), N.ptr(k2), N.ptr(k1),
                                              N.ptr(ok), N.stream_handle()), "propose")
    k2, k1, ok = k2.cpu().numpy(), k1.cpu().numpy(), ok.cpu().numpy()
    for i, c in enumerate(cases):
        if isinstance(c["result"], dict):
            assert ok[i] == 0, i
        else:
            assert ok[i] == 1 and [k2[i], k1[i]] == c["result"], i


def test_unit_propose_object_api():
    for c in golden("unit_cases.json")["propose"][:100]:
        best = []
        if c["tp1"] is not None:
            best.append(Triplet(1, 2, 1, c["tp1"], 5.0))
        if c["tp2"] is not None:
            best.append(Triplet(2, 4, 2, c["tp2"], 6.0))
        svc = Service("p", "m", 1.0, 10.0, 5.0, best_triplets=tuple(best))
        try:
            segs = P.propose_small_segments(svc, c["freed"])
            k2 = sum(1 for t in segs if t.instance_size == 2)
            got = [k2, len(segs) - k2]
        except P.MigplanError as exc:
            got = canon.error(exc)
        assert got == c["result"]


def _svc_from_canon(d):
    t = lambda x: Triplet(*x) if x is not None else None  # noqa: E731
    return Service(d["id"], d["model"], d["rate"], d["slo"], d["internal"],
                   best_triplets=tuple(Triplet(*b) for b in d["best"]), optimal_segment=t(d["opt"]),
                   optimal_segment_count=d["count"], last_segment=t(d["last"]))


def _map_from_canon(d):
    gpus = [P.GpuState(gid, [P.Placement(*p) for p in pls]) for gid, pls in d["gpus"]]
    return P.DeploymentMap(gpus=gpus, freed_rate={k: v for k, v in d["freed"]}, diagnostics=list(d["diags"]))


def test_alloc_relocate():
    for i, c in enumerate(golden("alloc_cases.json")["relocate"]):
        d = P.relocate_segments([_svc_from_canon(s) for s in c["services"]])
        assert canon.dmap(d) == c["result"], i


def test_alloc_optimize():
    for i, c in enumerate(golden("alloc_cases.json")["optimize"]):
        svcs = [_svc_from_canon(s) for s in c["services"]]
        dm = _map_from_canon(c["map"])
        try:
            got = canon.dmap(P.optimize_allocation(dm, svcs, c["threshold"]))
        except (P.MigplanError, AssertionError) as exc:
            got = canon.error(exc)
        exp = c["result"]
        if "error" in exp:
            assert got.get("error") == exp["error"], (i, c["tag"])
        else:
            assert got == exp, (i, c["tag"])


def test_empty_plan(fx):
    r = P.plan_services([], fx.tables)
    assert r.deployment.gpus == [] and r.unoptimized_gpu_count == 0 and r.deployment.diagnostics == []


def test_c2_records_vs_oracle_and_goldens(fx):
    g = golden("c2_digests.json")
    sb = W.scenario_batch(fx, g["n"], seed=g["seed"])
    assert hashlib.sha256(sb.rate.tobytes() + sb.slo.tobytes()).hexdigest()[:16] == g["input_sha256"]
    pt = pack_tables(fx.tables)
    dt = N.device_tables_for(fx.tables)
    n, M = sb.rate.shape
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    rate, bound = sb.rate.ravel(), sb.bound.ravel()
    res = B.plan_batch(dt, off, tab, rate, bound)
    cfg, plan = res.host()
    ocfg, oplan = oracle.plan_batch_records(pt, off, tab, rate, bound)
    assert cfg.tobytes() == ocfg.tobytes()
    assert plan.tobytes() == oplan.tobytes()
    # compact config records for host transfers
    resc = B.plan_batch(dt, off, tab, rate, bound, cfg_format=CFG_COMPACT)
    ccfg, cplan = resc.host()
    assert ccfg.tobytes() == compact_config(ocfg).tobytes() and cplan.tobytes() == oplan.tobytes()
    # and through the object decode, against the reference's own digests
    sets = [[P.make_service(m, m, float(sb.rate[k, j]), float(sb.slo[k, j])) for j, m in enumerate(sb.models)]
            for k in range(n)]
    results = P.plan_many(sets, fx.tables)
    bad = [k for k, r in enumerate(results) if canon.digest(_canon_result(r)) != g["digests"][k]]
    assert not bad, bad[:10]


def test_plan_batch_overlapped_back_to_back(fx):
    """parva_plan_batch_overlapped: 24 back-to-back programmatic dependent
    launches over 6 different batches into 3 rotating output blocks (and a
    plain launch in between); every block holds exactly the oracle's records
    of the batch planned into it last."""
    from paper_2409_14447_b200.records import tiny_config
    pt = pack_tables(fx.tables)
    dt = N.device_tables_for(fx.tables)
    ins, exp = [], []
    for b in range(6):
        sb = W.scenario_batch(fx, 3_001 + 500 * b, seed=40 + b)
        n, M = sb.rate.shape
        off = np.arange(n + 1, dtype=np.int32) * M
        tab = np.tile(np.arange(M, dtype=np.int32), n)
        rate, bound = sb.rate.ravel().copy(), sb.bound.ravel().copy()
        ocfg, oplan = oracle.plan_batch_records(pt, off, tab, rate, bound)
        ins.append(tuple(N.to_device(a) for a in (off, tab, rate, bound)))
        exp.append((tiny_config(ocfg).tobytes(), oplan.tobytes()))
    big = max(int(x[0].shape[0]) - 1 for x in ins), max(int(x[1].shape[0]) for x in ins)
    outs = [B.BatchResult(N.empty_records(big[1], TINY_DTYPE), N.empty_records(big[0], PLAN_DTYPE), big[0], big[1],
                          CFG_TINY) for _ in range(3)]
    last = {}
    ring = B.SlotRing(3)
    for i in range(24):
        b, r = (5 * i + 1) % 6, i % 3
        o = outs[r]
        k, m = int(ins[b][0].shape[0]) - 1, int(ins[b][1].shape[0])
        view = B.BatchResult(o.cfg[:m], o.plan[:k], k, m, CFG_TINY)
        if i == 11:
            torch.cuda.synchronize()     # a plain launch: every earlier launch into the slot is done
            B.plan_batch(dt, *ins[b], cfg_format=CFG_TINY, out=view)
        else:
            B.plan_batch(dt, *ins[b], cfg_format=CFG_TINY, out=view, overlap=True, ticket=ring.ticket(r, k))
        last[r] = (b, view)
    torch.cuda.synchronize()
    ring.check()
    for r, (b, view) in last.items():
        cfg, plan = view.host()
        assert plan.tobytes() == exp[b][1], (r, b)
        assert cfg.tobytes() == exp[b][0], (r, b)


def test_c4_sample_vs_oracle(fx):
    sb = W.scenario_batch(fx, 100_000, seed=1)
    pt = pack_tables(fx.tables)
    dt = N.device_tables_for(fx.tables)
    n, M = sb.rate.shape
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    for optimize, thr in ((True, 4), (False, 4), (True, 6)):
        res = B.plan_batch(dt, off, tab, sb.rate.ravel(), sb.bound.ravel(), optimize=optimize, threshold=thr)
        cfg, plan = res.host()
        ocfg, oplan = oracle.plan_batch_records(pt, off, tab, sb.rate.ravel(), sb.bound.ravel(),
                                                optimize=optimize, threshold=thr)
        assert cfg.tobytes() == ocfg.tobytes()
        assert plan.tobytes() == oplan.tobytes()


def test_c4_full_vs_oracle(fx):
    """All 10^6 C4 scenarios (seed 1) in one K2 launch, byte for
    byte against the oracle (every host thread)."""
    sb = W.scenario_batch(fx, 1_000_000, seed=1)
    pt = pack_tables(fx.tables)
    dt = N.device_tables_for(fx.tables)
    n, M = sb.rate.shape
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    rate, bound = sb.rate.ravel(), sb.bound.ravel()
    res = B.plan_batch(dt, off, tab, rate, bound, cfg_format=CFG_TINY)
    cfg, plan = res.host()
    ocfg, oplan = oracle.plan_batch_records(pt, off, tab, rate, bound)
    from paper_2409_14447_b200.records import tiny_config
    assert plan.tobytes() == oplan.tobytes()
    assert cfg.tobytes() == tiny_config(ocfg).tobytes()


def test_c3_sweep_vs_goldens_and_oracle():
    g = golden("c3_sample.json")
    dt_h = W.dense_tables(2000, seed=3)
    pt = pack_dense(dt_h)
    dt = N.DeviceTables(pt, build_index=False)
    n = dt_h.n_workloads
    out = B.configure_sweep(dt, np.arange(n), dt_h.rate, dt_h.slo / 2.0)
    recs = N.records_to_numpy(out, n, CONFIG_DTYPE)
    for w in range(g["n"]):
        row = g["rows"][w]
        if "error" in row["result"]:
            assert recs[w]["status"] == 1
            continue
        sid = f"w{w:05d}"
        got = service_canon(sid, sid, dt_h.rate[w], dt_h.slo[w], dt_h.slo[w] / 2.0, pt, w, recs[w])
        assert got == row["result"], w
    orec = oracle.configure_batch(pt, np.arange(n), dt_h.rate, dt_h.slo / 2.0)
    assert recs.tobytes() == orec.tobytes()
    # same queries, shuffled order and repeated tables: still per-row exact
    perm = np.random.default_rng(0).permutation(n)
    out2 = B.configure_sweep(dt, perm, dt_h.rate[perm], dt_h.slo[perm] / 2.0)
    recs2 = N.records_to_numpy(out2, n, CONFIG_DTYPE)
    assert recs2.tobytes() == orec[perm].tobytes()


def test_c5_large_cluster(fx):
    g = golden("c5_summary.json")
    rates = W.c5_rates()
    svcs = [P.make_service(f"d121#{i}", W.C5_MODEL, float(r), W.C5_SLO) for i, r in enumerate(rates)]
    res = P.plan_services(svcs, fx.tables)
    assert res.unoptimized_gpu_count == g["unopt_gpus"]
    assert res.gpu_count == g["gpus"] and res.deployment.total_gpcs == g["total_gpcs"]
    assert canon.digest(canon.dmap(res.deployment)) == g["optimized_sha256"]
    assert hashlib.sha256(res.deployment.to_json().encode()).hexdigest()[:16] == g["json_sha256"]


def test_host_entry_pipelined_vs_oracle(fx):
    """parva_plan_host (chunked H2D / plan / D2H pipeline) == oracle records."""
    import ctypes as C
    sb = W.scenario_batch(fx, 9_001, seed=5)
    n, M = sb.rate.shape
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    rate, bound = sb.rate.ravel().copy(), sb.bound.ravel().copy()
    dt = N.device_tables_for(fx.tables)
    L = N.lib()
    for fmt in (0, 1, 1, 0):   # repeated calls exercise the cached pipeline graph
        h_cfg = np.zeros(n * M * (32 if fmt == 0 else 16), dtype=np.uint8)
        h_plan = np.zeros(n * 128, dtype=np.uint8)
        nb = int(L.parva_plan_host_scratch(C.c_int32(n), C.c_int32(n * M)))
        scratch = torch.empty(nb, dtype=torch.uint8, device="cuda")
        vp = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
        rc = L.parva_plan_host(C.byref(dt.struct), C.byref(dt.index_struct), C.c_int32(n), vp(off), vp(tab),
                               vp(rate), vp(bound), C.c_int32(1), C.c_int32(4), vp(h_cfg), C.c_int32(fmt),
                               vp(h_plan), N.ptr(scratch), C.c_size_t(nb), N.stream_handle())
        assert rc == 0
        ocfg, oplan = oracle.plan_batch_records(pack_tables(fx.tables), off, tab, rate, bound)
        exp_cfg = ocfg if fmt == 0 else compact_config(ocfg)
        assert h_cfg.tobytes() == exp_cfg.tobytes()
        assert h_plan.tobytes() == oplan.tobytes()


def test_host_entry_packed_vs_oracle(fx):
    """parva_plan_host_packed (one H2D + one D2H per chunk, cached graph) == oracle."""
    sb = W.scenario_batch(fx, 7_003, seed=9)
    n, M = sb.rate.shape
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    rate, bound = sb.rate.ravel().copy(), sb.bound.ravel().copy()
    dt = N.device_tables_for(fx.tables)
    ocfg, oplan = oracle.plan_batch_records(pack_tables(fx.tables), off, tab, rate, bound)
    from paper_2409_14447_b200.records import tiny_config
    conv = {0: lambda c: c, 1: compact_config, 2: tiny_config}
    for chunks, fmt, pbytes in ((1, 1, 128), (3, 1, 128), (3, 0, 128), (4, 1, 128), (3, 2, 64), (1, 2, 64)):
        pb = B.PackedHostBatch(off, tab, rate, bound, n_chunks=chunks, cfg_format=fmt, plan_bytes=pbytes)
        for _ in range(2):
            pb.run(dt)
            cfg, plan = pb.outputs()
            assert plan.tobytes() == oplan.tobytes()
            assert cfg.tobytes() == conv[fmt](ocfg).tobytes()
            if pbytes == 64:   # the 64-byte records themselves, and the spill list as a set
                from paper_2409_14447_b200.records import plan64_view
                for c, (ccfg, p64, spills) in enumerate(pb.raw_outputs()):
                    a, b = pb.bounds[c]
                    exp64, exp_sp = plan64_view(oplan[a:b], pb.layouts[c].spill_cap)
                    assert p64.tobytes() == exp64.tobytes()
                    assert sorted(int(x) for x in spills["scenario"]) == exp_sp


def _mapped_raw(mb):
    """(config records, plan records as written) of a MappedHostBatch."""
    from paper_2409_14447_b200.records import PLAN64_DTYPE, PLAN_DTYPE
    lay, buf = mb.layout, mb.h_out.numpy()
    pdt = PLAN64_DTYPE if mb.plan_bytes == 64 else PLAN_DTYPE
    return buf[lay.out_plan:lay.out_plan + mb.plan_bytes * mb.n_scen].view(pdt)


def test_host_entry_mapped_vs_oracle(fx):
    """parva_plan_host_mapped (in-kernel PCIe streaming, records written to
    mapped host memory) == oracle, for every record format and chunking;
    repeated calls reuse the scratch (slice-flag epochs)."""
    from paper_2409_14447_b200.records import plan64_view, tiny_config
    sb = W.scenario_batch(fx, 7_003, seed=11)
    n, M = sb.rate.shape
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    rate, bound = sb.rate.ravel().copy(), sb.bound.ravel().copy()
    dt = N.device_tables_for(fx.tables)
    ocfg, oplan = oracle.plan_batch_records(pack_tables(fx.tables), off, tab, rate, bound)
    conv = {0: lambda c: c, 1: compact_config, 2: tiny_config}
    for fmt, pbytes, chunk in ((2, 64, 64), (1, 128, 16), (0, 128, 1000), (2, 64, 1), (2, 128, 7003)):
        mb = B.MappedHostBatch(off, tab, rate, bound, cfg_format=fmt, plan_bytes=pbytes, chunk_scen=chunk)
        for _ in range(3):
            mb.h_out.zero_()
            mb.run(dt)
            cfg, plan = mb.outputs()
            assert plan.tobytes() == oplan.tobytes(), (fmt, pbytes, chunk)
            assert cfg.tobytes() == conv[fmt](ocfg).tobytes(), (fmt, pbytes, chunk)
            if pbytes == 64:
                exp64, _ = plan64_view(oplan, n)
                assert _mapped_raw(mb).tobytes() == exp64.tobytes()


def test_host_entry_mapped_fuzz(fx):
    """Mapped entry on ragged batches: empty scenarios, >32 services
    (CAPACITY), zero rates, infeasible SLOs, options; and 0 / 1 scenarios."""
    import random
    from paper_2409_14447_b200.records import tiny_config
    rng = random.Random(77)
    dt = N.device_tables_for(fx.tables)
    pt = pack_tables(fx.tables)
    nm = len(fx.models)
    for trial, n_scen in enumerate((0, 1, 2, 500, 2500)):
        sizes = [rng.choice([0, 1, 3, 11, 11, 20, 33, 40]) for _ in range(n_scen)]
        total = int(sum(sizes))
        tab = np.array([rng.randrange(nm) for _ in range(total)], dtype=np.int32)
        rate = np.array([0.0 if rng.random() < 0.05 else math_exp(rng.uniform(1.0, 9.0)) for _ in range(total)])
        bound = np.array([math_exp(rng.uniform(2.5, 8.0)) / 2.0 for _ in range(total)])
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        optimize, threshold = rng.random() < 0.8, rng.choice([2, 4, 5])
        ocfg, oplan = oracle.plan_batch_records(pt, off, tab, rate, bound, optimize=optimize, threshold=threshold)
        mb = B.MappedHostBatch(off, tab, rate, bound, cfg_format=2, plan_bytes=64, chunk_scen=rng.choice([1, 5, 64]))
        mb.run(dt, optimize=optimize, threshold=threshold)
        cfg, plan = mb.outputs()
        assert plan.tobytes() == oplan.tobytes(), trial
        assert cfg.tobytes() == tiny_config(ocfg).tobytes(), trial


def test_host_entry_mapped_few_scenarios_many_services(fx):
    """More input slices than scenarios-per-16: every loader CTA must be
    launched (the grid covers the loaders), else the slices never land."""
    from paper_2409_14447_b200.records import tiny_config
    rng = np.random.default_rng(5)
    nm = len(fx.models)
    dt = N.device_tables_for(fx.tables)
    for sizes in ((700, 650, 720), (1, 2000), (3000,)):
        total = int(sum(sizes))
        tab = rng.integers(0, nm, total).astype(np.int32)
        rate = np.exp(rng.uniform(1.0, 9.0, total))
        bound = np.exp(rng.uniform(2.5, 8.0, total)) / 2.0
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        ocfg, oplan = oracle.plan_batch_records(pack_tables(fx.tables), off, tab, rate, bound)
        mb = B.MappedHostBatch(off, tab, rate, bound, cfg_format=2, plan_bytes=64, chunk_scen=1)
        assert mb.in_bytes > 8192 * len(sizes)
        mb.run(dt)
        cfg, plan = mb.outputs()
        assert plan.tobytes() == oplan.tobytes(), sizes
        assert cfg.tobytes() == tiny_config(ocfg).tobytes(), sizes


def test_host_entry_mapped_async_overlap(fx):
    """parva_plan_host_mapped_submit / _wait: calls of two batches
    interleaved on one stream, two slots each (overlapping programmatic
    dependent launches), a synchronous call and an empty batch in between;
    every slot's records == oracle."""
    from paper_2409_14447_b200.records import tiny_config
    dt = N.device_tables_for(fx.tables)
    pt = pack_tables(fx.tables)
    batches = []
    for n, seed in ((6_001, 21), (2_500, 22)):
        sb = W.scenario_batch(fx, n, seed=seed)
        k, M = sb.rate.shape
        off = np.arange(k + 1, dtype=np.int32) * M
        tab = np.tile(np.arange(M, dtype=np.int32), k)
        rate, bound = sb.rate.ravel().copy(), sb.bound.ravel().copy()
        ocfg, oplan = oracle.plan_batch_records(pt, off, tab, rate, bound)
        mb = B.MappedHostBatch(off, tab, rate, bound, cfg_format=2, plan_bytes=64, depth=2)
        batches.append((mb, tiny_config(ocfg).tobytes(), oplan.tobytes()))
    empty = B.MappedHostBatch(np.zeros(1, dtype=np.int32), np.zeros(0, np.int32), np.zeros(0), np.zeros(0),
                              depth=2)
    for rnd in range(3):
        for slot in (0, 1):
            for mb, _, _ in batches:
                mb.h_outs[slot].zero_()
        for slot in (0, 1):
            for mb, _, _ in batches:
                mb.submit(dt, slot)
            empty.submit(dt, slot)
        if rnd == 1:
            batches[1][0].wait(0)
            batches[1][0].run(dt)      # synchronous call on a slot with a finished async call
        for slot in (0, 1):
            empty.wait(slot)
            for i, (mb, ecfg, eplan) in enumerate(batches):
                mb.wait(slot)
                cfg, plan = mb.outputs(slot)
                assert plan.tobytes() == eplan, (rnd, slot, i)
                assert cfg.tobytes() == ecfg, (rnd, slot, i)
    # a second submit on a busy slot waits for the first (one call per scratch)
    mb, ecfg, eplan = batches[0]
    for _ in range(4):
        mb.submit(dt, 0)
    mb.wait(0)
    assert mb.outputs(0)[1].tobytes() == eplan


def test_reconfigure_service(fx):
    """§III-F re-planning (allocator.py:494-537) + diff_maps (:484-491) vs reference goldens."""
    for i, c in enumerate(golden("reconfigure_cases.json")):
        base = c["base"]
        svcs = [_svc_from_canon(s) for s in base["services"]]
        dm = _map_from_canon({"gpus": base["gpus"], "freed": base["freed"], "diags": base["diags"]})
        old = svcs[c["target"]]
        upd = P.make_service(old.id, old.model_id, c["new_rate"], c["new_slo"])
        table = P.filter_feasible(fx.tables[old.model_id])
        try:
            dmap, changes, new_services = P.reconfigure_service(dm, svcs, upd, table, c["threshold"])
            got = {"map": canon.dmap(dmap), "changes": [ch.to_json_obj() for ch in changes],
                   "services": [canon.service(s) for s in new_services]}
        except P.MigplanError as exc:
            got = canon.error(exc)
        assert got == c["result"], i


def test_prepare_tables_on_device(fx):
    """§8f row 2: filter_feasible + restrict as kernel predicates == the host
    preparation (profiles.py:260-271, pipeline.py:70-80), including memory
    values exactly at, just below and just above the caps."""
    import math
    import random
    from paper_2409_14447_b200.tables import pack_raw
    rng = random.Random(3)
    caps = {1: 10.0, 2: 20.0, 3: 40.0, 4: 40.0, 7: 80.0}
    rand_tables = []
    for t in range(40):
        pts = []
        for s in (1, 2, 3, 4, 7):
            for b in rng.sample(range(1, 65), rng.randint(0, 40)):
                for p in rng.sample([1, 2, 3, 4], rng.randint(1, 4)):
                    c = caps[s]
                    mem = rng.choice([c, math.nextafter(c, 0), math.nextafter(c, 99), rng.uniform(0, 2 * c), 0.0])
                    pts.append(P.ProfilePoint(f"r{t}", s, b, p, rng.uniform(1, 999), rng.uniform(1, 99), mem))
        rand_tables.append(P.ProfileTable(f"r{t}", tuple(pts)))
    cases = [(fx.tables, None, False), (fx.tables, None, True),
             (fx.tables, {1: 5.0, 2: 10.0, 3: 20.0, 4: 20.0, 7: 40.0}, False),
             (rand_tables, None, False), (rand_tables, None, True), (rand_tables, {1: 3, 2: 7, 3: 11, 4: 11, 7: 30}, True)]
    for tables, mm, single in cases:
        host = pack_tables(tables, memory_map=mm, single_process=single)
        dev = N.DeviceTables.prepare_on_device(pack_raw(tables), mm, single)
        hp = dev.packed
        for f in ("tp", "lat", "batch", "procs", "seg_start", "seg_count"):
            assert np.asarray(getattr(hp, f)).tobytes() == np.asarray(getattr(host, f)).astype(
                np.asarray(getattr(hp, f)).dtype).tobytes(), f
        pts = dev.pts[:2 * host.n_points].cpu().numpy()
        assert pts[0::2].tobytes() == host.tp.tobytes() and pts[1::2].tobytes() == host.lat.tobytes()


def test_broad_fuzz_vs_oracle(fx):
    """Random scenario sizes (0..40 services, so empty scenarios and the
    CAPACITY path included), random options; K2 records == oracle records and
    the decoded objects == the oracle's plans (capacity scenarios through KG)."""
    import random
    from helpers import oracle_plan_canon
    rng = random.Random(2024)
    models = list(fx.models)
    for trial in range(6):
        opts = {"optimize": rng.random() < 0.8, "threshold": rng.choice([0, 2, 3, 4, 4, 5, 7]),
                "single_process": rng.random() < 0.3}
        mm = {1: 6.0, 2: 12.0, 3: 24.0, 4: 24.0, 7: 60.0} if rng.random() < 0.3 else None
        pt = pack_tables(fx.tables, memory_map=mm, single_process=opts["single_process"])
        dt = N.device_tables_for(fx.tables, mm, opts["single_process"])
        n_scen = 3000
        sizes = [rng.choice([0, 1, 2, 5, 11, 11, 11, 17, 25, 33, 40]) for _ in range(n_scen)]
        tab, rate, bound, names = [], [], [], []
        for k, sz in enumerate(sizes):
            row = []
            for j in range(sz):
                m = rng.randrange(len(models))
                r = 0.0 if rng.random() < 0.03 else math_exp(rng.uniform(1.0, 9.5))
                slo = math_exp(rng.uniform(3.0, 8.0))
                tab.append(m); rate.append(r); bound.append(slo / 2.0)
                row.append([f"s{j}", models[m], r, slo])
            names.append(row)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        tab = np.array(tab, dtype=np.int32)
        res = B.plan_batch(dt, off, tab, np.array(rate), np.array(bound), optimize=opts["optimize"],
                           threshold=opts["threshold"])
        cfg, plan = res.host()
        ocfg, oplan = oracle.plan_batch_records(pt, off, tab, rate, bound, optimize=opts["optimize"],
                                                threshold=opts["threshold"])
        assert cfg.tobytes() == ocfg.tobytes(), trial
        assert plan.tobytes() == oplan.tobytes(), trial
        # objects, incl. CAPACITY scenarios re-planned by the general kernel
        sets = [[P.make_service(a, m, r, s) for a, m, r, s in row] for row in names[:400]]
        popts = P.PlanOptions(optimize=opts["optimize"], threshold=opts["threshold"],
                              single_process=opts["single_process"], **({"memory_map": mm} if mm else {}))
        got = P.plan_many(sets, fx.tables, popts)
        for k in range(400):
            exp = oracle_plan_canon(oracle, pt, names[k], opts)
            assert _canon_result(got[k]) == exp, (trial, k)


def math_exp(x):
    import math
    return math.exp(x)


def test_simulation_reports_vs_reference(fx):
    """run_simulation / run_simulations (event loops on the GPU) reproduce every
    reference report of tests/golden/sim_cases.json exactly; the batched call
    gives the same reports as one call per job."""
    import json
    from helpers import sim_scenario_inputs
    from paper_2409_14447_b200 import simulation as S
    cases = golden("sim_cases.json")
    jobs = []
    for case in cases:
        dmap, services, wl = sim_scenario_inputs(case, fx)
        jobs.append(S.SimJob(dmap, fx.tables, services, wl, case["horizon_s"], case["seed"]))
    batched = S.run_simulations(jobs)
    for case, job, rep in zip(cases, jobs, batched):
        for r in (rep, S.run_simulation(job.dmap, job.tables, job.services, job.workload, job.horizon_s, job.seed)):
            obj = r.to_json_obj()
            obj["metrics"] = {"internal_slack": S.internal_slack(r.activity) if r.activity.segments else None,
                              "slo_compliance": S.slo_compliance(r)}
            assert json.loads(json.dumps(obj)) == case["report"], (case["scenario"], case["arrivals"], case["seed"])


def test_simulation_event_loop_vs_oracle(fx):
    """Raw event-loop outputs (every batch latency, busy time per segment,
    counters) bit-identical to the C oracle on random maps, overloads,
    horizons and seeds -- including services without segments or arrivals."""
    import random
    from helpers import sim_report_with_oracle
    from paper_2409_14447_b200 import simulation as S
    rng = random.Random(99)
    names = list(fx.scenarios)
    jobs = []
    for i in range(40):
        sc = P.Scenario(f"r{i}", tuple(P.scenario.ScenarioService(m, r, s) for m, r, s in fx.scenarios[rng.choice(names)]))
        res = P.plan_scenario(sc, fx.tables)
        services = list(res.services)
        wl = S.Workload.from_services(services, kind=rng.choice(["poisson", "poisson", "deterministic"]),
                                      scale=rng.choice([0.0, 0.2, 1.0, 1.5, 3.0]))
        jobs.append(S.SimJob(res.deployment, fx.tables, services, wl, rng.choice([0.5, 1.0, 2.0]), rng.randrange(1000)))
    gpu = S.run_simulations(jobs)
    for job, rep in zip(jobs, gpu):
        orep, _, _ = sim_report_with_oracle(oracle, job)
        assert rep.to_json_obj() == orep.to_json_obj()
        assert [s.activity for s in rep.activity.segments] == [s.activity for s in orep.activity.segments]
        for sid in rep.services:
            a, b = rep.services[sid], orep.services[sid]
            assert (a.served, a.batches, a.violations, a.latency_ms) == (b.served, b.batches, b.violations, b.latency_ms)


def test_simulator_log1p_matches_host_libm():
    """The exponential tail's log1p on the GPU equals the host libm's (glibc)
    on random arguments in (-1, 0], incl. the branch boundaries."""
    import ctypes as C
    import math
    rng = np.random.default_rng(4)
    u = rng.random(2_000_000)
    u[:4] = [0.0, 2.0 ** -60, 2.0 ** -30, 1.0 - 2.0 ** -53]
    x = np.concatenate([-u, -np.array([0.29289321881345254, 0.2928932188134524, 0.29289321881345265])])
    d_x = N.to_device(x)
    d_o = torch.empty_like(d_x)
    N.check(N.lib().parva_sim_log1p(N.ptr(d_x), N.ptr(d_o), C.c_int64(x.shape[0]), N.stream_handle()),
            "parva_sim_log1p")
    got = d_o.cpu().numpy()
    exp = np.array([math.log1p(v) for v in x])
    assert got.tobytes() == exp.tobytes()


def test_simulator_exponential_matches_numpy():
    """numpy Generator.exponential reproduced draw for draw on the GPU
    (PCG64 + ziggurat incl. the wedge and tail paths)."""
    import ctypes as C
    for seed, scale in ((0, 1.0), (7, 1.0 / 1234.5), (12345, 3.0)):
        rng = np.random.default_rng(np.random.SeedSequence(seed).spawn(2)[1])
        st = rng.bit_generator.state["state"]
        m = (1 << 64) - 1
        pcg = np.array([st["state"] >> 64, st["state"] & m, st["inc"] >> 64, st["inc"] & m], dtype=np.uint64)
        n = 200_000
        ref = rng.exponential(scale, size=n)
        d_p = N.to_device(pcg)
        d_o = torch.empty(n, dtype=torch.float64, device="cuda")
        N.check(N.lib().parva_sim_exponential(N.ptr(d_p), C.c_double(scale), C.c_int64(n), N.ptr(d_o),
                                              N.stream_handle()), "parva_sim_exponential")
        assert d_o.cpu().numpy().tobytes() == ref.tobytes(), seed


def test_simulation_edge_cases(fx):
    """Unplaced services (no segments), services with zero rate, a service
    missing from the definitions, a non-positive horizon: the reference's
    reports / errors (checked against the C-oracle path, which is pinned on
    the reference's reports)."""
    import json
    from helpers import sim_report_with_oracle
    from paper_2409_14447_b200 import simulation as S
    sc = P.Scenario("S3", tuple(P.scenario.ScenarioService(m, r, s) for m, r, s in fx.scenarios["S3"]))
    res = P.plan_scenario(sc, fx.tables)
    services = list(res.services)
    extra = P.make_service("idle", services[0].model_id, 50.0, 500.0)      # defined, never placed
    rates = tuple((s.id, 0.0 if i % 3 == 0 else s.request_rate) for i, s in enumerate(services)) + (("idle", 50.0),)
    for kind in ("poisson", "deterministic"):
        wl = S.Workload(rates, kind)
        job = S.SimJob(res.deployment, fx.tables, services + [extra], wl, 1.5, 3)
        rep = S.run_simulation(job.dmap, job.tables, job.services, job.workload, job.horizon_s, job.seed)
        orep, _, _ = sim_report_with_oracle(oracle, job)
        assert json.dumps(rep.to_json_obj()) == json.dumps(orep.to_json_obj())
        assert rep.services["idle"].batches == 0 and rep.services["idle"].arrived > 0
    with pytest.raises(P.SimulationConfigError):
        S.run_simulation(res.deployment, fx.tables, services[1:], S.Workload.from_services(services), 1.0, 0)
    with pytest.raises(P.SimulationConfigError):
        S.run_simulation(res.deployment, fx.tables, services, None, 0.0, 0)


def test_mapped_entry_rejects_pageable_memory(fx):
    """The zero-copy entry refuses pageable host blocks (status BAD_INPUT)
    instead of letting the kernel fault on an unmapped address."""
    import ctypes as C
    sb = W.scenario_batch(fx, 16, seed=1)
    n, M = sb.rate.shape
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    mb = B.MappedHostBatch(off, tab, sb.rate.ravel(), sb.bound.ravel())
    dt = N.device_tables_for(fx.tables)
    pageable_in = np.frombuffer(mb.h_in.numpy().tobytes(), dtype=np.uint8).copy()
    rc = N.lib().parva_plan_host_mapped(
        C.byref(dt.struct), C.byref(dt.index_struct), C.c_int32(mb.n_scen), C.c_int32(mb.n_svc),
        C.c_void_p(pageable_in.ctypes.data), C.c_int64(mb.in_bytes), C.c_void_p(mb.h_out.data_ptr()),
        C.c_int32(1), C.c_int32(4), C.c_int32(2), C.c_int32(64), N.ptr(mb.scratch), C.c_size_t(mb.scratch_bytes),
        N.stream_handle())
    assert rc == 5          # PARVA_BAD_INPUT
    mb.run(dt)              # and the pinned path still works afterwards
    ocfg, oplan = oracle.plan_batch_records(pack_tables(fx.tables), off, tab, sb.rate.ravel(), sb.bound.ravel())
    assert mb.outputs()[1].tobytes() == oplan.tobytes()


def test_host_entry_mapped_pack_every_step(fx):
    """The e2e pipeline of bench.py: every step packs a different batch of
    plain host arrays into its slot's pinned block (parva_stream_pack_arrays)
    and submits it, 3 calls in flight; every step's records == oracle."""
    from paper_2409_14447_b200.records import tiny_config
    dt = N.device_tables_for(fx.tables)
    pt = pack_tables(fx.tables)
    batches = []
    for seed in range(60, 66):
        sb = W.scenario_batch(fx, 4_000, seed=seed)
        k, M = sb.rate.shape
        off = np.arange(k + 1, dtype=np.int32) * M
        tab = np.tile(np.arange(M, dtype=np.int32), k)
        batches.append((off, tab, sb.rate.ravel().copy(), sb.bound.ravel().copy()))
    exp = []
    for b in batches:
        ocfg, oplan = oracle.plan_batch_records(pt, *b)
        exp.append((tiny_config(ocfg).tobytes(), oplan.tobytes()))
    D = 3
    mb = B.MappedHostBatch(*batches[0], cfg_format=2, plan_bytes=64, depth=D)
    inflight = {}
    for i in range(20):
        slot = i % D
        if slot in inflight:
            mb.wait(slot)
            cfg, plan = mb.outputs(slot)
            j = inflight.pop(slot)
            assert plan.tobytes() == exp[j][1] and cfg.tobytes() == exp[j][0], (i, j)
        j = (7 * i) % len(batches)
        mb.fill(*batches[j], slot=slot)
        mb.submit(dt, slot)
        inflight[slot] = j
    for slot, j in inflight.items():
        mb.wait(slot)
        cfg, plan = mb.outputs(slot)
        assert plan.tobytes() == exp[j][1] and cfg.tobytes() == exp[j][0], j


def test_tiny_records_rejected_for_tables_over_254_points():
    """the 8-byte config record stores a point position in a byte;
    tables with more than 254 points in one (table, size) segment make every
    entry reject PARVA_CFG_TINY (the device planner itself is exact there:
    the full records equal the oracle's)."""
    from paper_2409_14447_b200.tables import pack_dense
    dth = W.dense_tables(6, seed=3)
    pt = pack_dense(dth)
    assert int(pt.seg_count.max()) > 254
    dt = N.DeviceTables(pt)
    off = np.array([0, 3, 6], dtype=np.int32)
    tab = np.arange(6, dtype=np.int32)
    rate, bound = dth.rate, dth.slo / 2.0
    with pytest.raises(Exception, match="parva_plan_batch"):
        B.plan_batch(dt, off, tab, rate, bound, cfg_format=CFG_TINY)
    with pytest.raises(Exception):
        B.MappedHostBatch(off, tab, rate, bound, cfg_format=CFG_TINY).run(dt)
    cfg, plan = B.plan_batch(dt, off, tab, rate, bound).host()
    ocfg, oplan = oracle.plan_batch_records(pt, off, tab, rate, bound)
    assert cfg.tobytes() == ocfg.tobytes() and plan.tobytes() == oplan.tobytes()


def test_host_entry_mapped_stream_producer_thread(fx):
    """MappedHostBatch.stream: a producer thread packs batch i+1 while the
    caller submits batch i; every batch's records (checked in consume,
    before its slot is reused) == oracle."""
    from paper_2409_14447_b200.records import tiny_config
    dt = N.device_tables_for(fx.tables)
    pt = pack_tables(fx.tables)
    batches, exp = [], []
    for seed in range(70, 75):
        sb = W.scenario_batch(fx, 3_000, seed=seed)
        k, M = sb.rate.shape
        b = (np.arange(k + 1, dtype=np.int32) * M, np.tile(np.arange(M, dtype=np.int32), k),
             sb.rate.ravel().copy(), sb.bound.ravel().copy())
        ocfg, oplan = oracle.plan_batch_records(pt, *b)
        batches.append(b)
        exp.append((tiny_config(ocfg).tobytes(), oplan.tobytes()))
    mb = B.MappedHostBatch(*batches[0], cfg_format=2, plan_bytes=64, depth=3)
    order = [(3 * i) % 5 for i in range(17)]
    seen = []

    def consume(i, slot):
        cfg, plan = mb.outputs(slot)
        j = order[i]
        assert plan.tobytes() == exp[j][1] and cfg.tobytes() == exp[j][0], (i, j)
        seen.append(i)

    assert mb.stream(dt, (batches[j] for j in order), consume=consume) == len(order)
    assert sorted(seen) == list(range(len(order)))


def test_host_entry_arrays_submit(fx):
    """parva_plan_host_arrays_submit (wait for the slot, pack the plain
    arrays, submit -- one C call per step), 3 slots, 14 steps over 5
    batches: every step's records == oracle."""
    from paper_2409_14447_b200.records import tiny_config
    dt = N.device_tables_for(fx.tables)
    pt = pack_tables(fx.tables)
    batches, exp = [], []
    for seed in range(90, 95):
        sb = W.scenario_batch(fx, 2_500, seed=seed)
        k, M = sb.rate.shape
        b = (np.arange(k + 1, dtype=np.int32) * M, np.tile(np.arange(M, dtype=np.int32), k),
             sb.rate.ravel().copy(), sb.bound.ravel().copy())
        ocfg, oplan = oracle.plan_batch_records(pt, *b)
        batches.append(b)
        exp.append((tiny_config(ocfg).tobytes(), oplan.tobytes()))
    mb = B.MappedHostBatch(*batches[0], cfg_format=2, plan_bytes=64, depth=3)
    last = {}
    for i in range(14):
        slot, j = i % 3, (2 * i + 1) % 5
        if slot in last:
            mb.wait(slot)
            cfg, plan = mb.outputs(slot)
            assert plan.tobytes() == exp[last[slot]][1] and cfg.tobytes() == exp[last[slot]][0], i
        mb.submit_arrays(dt, slot, *batches[j])
        last[slot] = j
    for slot, j in last.items():
        mb.wait(slot)
        cfg, plan = mb.outputs(slot)
        assert plan.tobytes() == exp[j][1] and cfg.tobytes() == exp[j][0]


def test_plan_many_zero_copy_and_copy_paths(fx):
    """plan_many below pipeline._ZERO_COPY_MAX scenarios runs K2 straight on
    pinned host buffers (no copies); above it, on device copies.  Both give
    the reference's C2 digests (first 1,500 scenarios: one call of 1,000 on
    the zero-copy path, then 1,500 on the copy path, then single scenarios)."""
    from paper_2409_14447_b200 import pipeline as PL
    g = golden("c2_digests.json")
    n = 1500
    sb = W.scenario_batch(fx, n, seed=g["seed"])
    sets = [[P.make_service(m, m, float(sb.rate[k, j]), float(sb.slo[k, j])) for j, m in enumerate(sb.models)]
            for k in range(n)]
    assert 1000 <= PL._ZERO_COPY_MAX < n
    for lo, hi in ((0, 1000), (0, n)):
        res = P.plan_many(sets[lo:hi], fx.tables)
        for k, r in enumerate(res, start=lo):
            assert canon.digest(_canon_result(r)) == g["digests"][k], (lo, hi, k)
    for k in (0, 99, 777):
        r = P.plan_many([sets[k]], fx.tables)[0]
        assert canon.digest(_canon_result(r)) == g["digests"][k], k


def test_general_kernel_global_memory_chain(fx):
    """A C5-like allocation too large for KG's shared-memory GPU state
    (> ~110k GPUs before optimize): the optimize chain runs on global memory
    (opt_chain<false>).  Same deployment map, ledger and diagnostics as the
    oracle (the C restatement with the reference's cursors)."""
    from helpers import map_canon
    rates = W.c5_rates(n=120_000, seed=7)
    n = len(rates)
    svcs = [P.make_service(f"d121#{i}", W.C5_MODEL, float(r), W.C5_SLO) for i, r in enumerate(rates)]
    res = P.plan_services(svcs, fx.tables)
    pt = pack_tables(fx.tables)
    t = pt.index_of()[W.C5_MODEL]
    _, ores = oracle.plan_scenario(pt, np.full(n, t), rates, np.full(n, W.C5_SLO / 2.0), True, 4, gcap=400_000)
    assert res.unoptimized_gpu_count == ores["unopt"] > 115_000
    assert canon.dmap(res.deployment) == map_canon(ores, [s.id for s in svcs])


@pytest.mark.parametrize("with_index", [False, True])
def test_plan_batch_dense_tables_vs_oracle(with_index):
    """Scenarios over the C3 dense tables (up to 1,024 points per size):
    without the prefix-argmax index K1 configures and the tile kernel plans
    (parva_plan_batch_preconfigured); with it, the thread kernel searches the
    index through L1.  Records byte-equal to the oracle's."""
    dt_h = W.dense_tables(300, seed=3)
    pt = pack_dense(dt_h)
    dt = N.DeviceTables(pt, build_index=with_index)
    assert (dt.index_struct is not None) == with_index
    rng = np.random.default_rng(11)
    n = 600
    sizes = rng.integers(1, 9, n)
    off = np.zeros(n + 1, dtype=np.int32)
    off[1:] = np.cumsum(sizes)
    m = int(off[-1])
    tab = rng.integers(0, dt_h.n_workloads, m).astype(np.int32)
    rate = np.exp(rng.uniform(np.log(10.0), np.log(3000.0), m))
    bound = np.exp(rng.uniform(np.log(20.0), np.log(2000.0), m)) / 2.0
    cfg, plan = B.plan_batch(dt, off, tab, rate, bound).host()
    ocfg, oplan = oracle.plan_batch_records(pt, off, tab, rate, bound)
    assert cfg.tobytes() == ocfg.tobytes()
    assert plan.tobytes() == oplan.tobytes()
    assert (plan["status"] == 0).sum() > n // 4          # mostly real plans, not errors


@pytest.mark.parametrize("threshold", [0, 1, 3, 6, 7, 9])
def test_general_kernel_thresholds_vs_oracle(fx, threshold):
    """KG's optimize chain across drain thresholds (0: nothing drains; >= 7:
    every non-empty GPU is a candidate) on a C5-like allocation with mixed
    models, against the oracle: maps, ledger and diagnostics equal."""
    from helpers import map_canon
    rng = np.random.default_rng(threshold)
    models = list(fx.models)
    n = 3000
    pick = rng.integers(0, len(models), n)
    svcs, tab, rates, bounds = [], [], [], []
    pt = pack_tables(fx.tables)
    idx = pt.index_of()
    for i in range(n):
        m = models[pick[i]]
        lat = [p.latency for p in fx.tables[m].points]
        slo = float(rng.uniform(2.5 * min(lat), 2.5 * max(lat)))
        rate = float(rng.uniform(10.0, 3000.0))
        svcs.append(P.make_service(f"s{i}", m, rate, slo))
        tab.append(idx[m]); rates.append(rate); bounds.append(slo / 2.0)
    ocfg, ores = oracle.plan_scenario(pt, np.array(tab), np.array(rates), np.array(bounds), True, threshold,
                                      gcap=100_000)
    if (ocfg["status"] != 0).any():
        pytest.skip("an infeasible service in this draw")
    res = P.plan_services(svcs, fx.tables, P.PlanOptions(threshold=threshold))
    assert res.unoptimized_gpu_count == ores["unopt"]
    assert canon.dmap(res.deployment) == map_canon(ores, [s.id for s in svcs])


def test_concurrent_planning_threads(fx):
    """Disjoint runs may execute concurrently: four host
    threads plan different scenario sets at once through the public API
    (small calls on the zero-copy path, larger ones on device copies); every
    result equals the single-threaded one."""
    import threading
    g = golden("c2_digests.json")
    sb = W.scenario_batch(fx, 1600, seed=g["seed"])
    sets = [[P.make_service(m, m, float(sb.rate[k, j]), float(sb.slo[k, j])) for j, m in enumerate(sb.models)]
            for k in range(1600)]
    jobs = [(0, 1), (1, 300), (300, 301), (301, 1600), (5, 6), (6, 1100)]
    errors = []

    def worker(t):
        try:
            for rep in range(3):
                for a, b in jobs[t::4] if t < 4 else []:
                    for k, r in enumerate(P.plan_many(sets[a:b], fx.tables), start=a):
                        if canon.digest(_canon_result(r)) != g["digests"][k]:
                            errors.append((t, rep, k))
        except Exception as exc:  # noqa: BLE001
            errors.append((t, repr(exc)))
    th = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors[:5]
