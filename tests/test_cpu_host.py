"""CPU-only checks: the C ABI library loads and exports every declared
symbol; host-side data model mirrors the reference; no silent CPU path."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2409_14447_b200 as P
from paper_2409_14447_b200 import _native as N
from paper_2409_14447_b200 import workloads as W
from paper_2409_14447_b200.records import CONFIG_DTYPE, PLAN_DTYPE
from paper_2409_14447_b200.tables import pack_tables

REPO = Path(__file__).resolve().parent.parent


def _declared():
    text = (REPO / "include" / "parva_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|int64_t|size_t|void)\s+(parva_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.load_library()
    declared = _declared()
    assert len(declared) >= 13
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(N.EXPORTS)
    assert lib.parva_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(N.lib_path())],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sim_seed_states_match_numpy():
    """parva_sim_seed_states (host C) == default_rng(SeedSequence(seed).spawn(n)[i])
    PCG64 states, for small, 32-bit-boundary and multi-word seeds."""
    from paper_2409_14447_b200.simulation import _spawn_states
    m = (1 << 64) - 1
    for seed in (0, 1, 7, 2**32 - 1, 2**32, 2**40 + 7, 2**70 + 3, 2**200 + 5):
        got = _spawn_states(seed, 40)
        exp = []
        for ss in np.random.SeedSequence(seed).spawn(40):
            st = np.random.default_rng(ss).bit_generator.state["state"]
            exp.append((st["state"] >> 64, st["state"] & m, st["inc"] >> 64, st["inc"] & m))
        assert got == exp, seed


def test_batched_percentiles_match_numpy():
    """Simulator statistics: the batched linear percentiles equal
    np.percentile bit for bit (sizes 0-1000, ties, exact index hits)."""
    from paper_2409_14447_b200 import simulation as S
    rng = np.random.default_rng(3)
    sizes = [1, 2, 3, 4, 5, 7, 10, 19, 20, 21, 100, 101, 1000, 0, 13] + list(rng.integers(1, 300, 40))
    samples = [np.sort(rng.exponential(5, size=int(n))) for n in sizes] + [np.ones(3), np.array([2.0, 2.0])]
    cnt = np.array([len(x) for x in samples])
    off = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    got = S._percentiles_batch(np.concatenate(samples), off, cnt)
    for x, g in zip(samples, got):
        if len(x) == 0:
            assert g is None
            continue
        assert g == tuple(float(np.percentile(x, 100 * q)) for q in S._Q) + (float(x.max()),)


def test_service_from_record_with_empty_size_classes():
    """Record decoding (host): a table with only size-7 points (size classes
    0-3 empty, so their segments start where size 7's does) decodes to
    size-7 triplets, from a numpy record and from its tuple form."""
    from paper_2409_14447_b200.configurator import service_from_record
    pts = tuple(P.ProfilePoint("m", 7, b, p, 100.0 * b + p, 10.0 + b) for b in (1, 2, 4) for p in (1, 2))
    pt = pack_tables([P.ProfileTable("m", pts)], prepared=True)
    rec = np.zeros(1, dtype=CONFIG_DTYPE)[0]
    rec["best"] = [-1, -1, -1, -1, 0]
    rec["opt_sc"], rec["last_sc"], rec["count"] = 4, -1, 2
    svc = P.make_service("s", "m", 500.0, 100.0)
    for r in (rec, rec.tolist()):
        got = service_from_record(svc, pt, 0, r)
        assert [t.instance_size for t in got.best_triplets] == [7]
        assert got.optimal_segment.instance_size == 7 and got.optimal_segment_count == 2
        assert got.last_segment is None


def test_c_abi_rejects_bad_arguments_before_touching_the_device():
    """Argument checks of the C entries run before any CUDA call, so they
    return PARVA_BAD_INPUT (5) here, on a host without a GPU."""
    import ctypes as C
    L = N.load_library()
    BAD = 5
    m = N.Mirror()
    m.n = 0
    dummy = C.c_void_p(16)
    assert L.parva_plan_batch_fused(None, None, 0, 0, None, None, None, None, 1, 4, None, 2, None,
                                    C.byref(m), None) == BAD
    # a well-formed mirror whose sections are too small for the records
    # (the copy would run past the config section into the next
    # rank's part): rejected before any launch
    tab, idx = N.ParvaTables(), N.ParvaIndex()
    m = N.Mirror()
    m.n, m.plan_bytes = 1, 128
    m.plan[0] = m.cfg[0] = m.flag[0] = m.d_acks = m.d_done = 16
    m.epoch = 1
    m.ticket = N.SlotTicket(16, 0, None)
    m.plan_capacity, m.cfg_capacity = 10 * 128, 110 * 8
    args = (C.byref(tab), C.byref(idx), 10, 110, dummy, dummy, dummy, dummy, 1, 4, dummy)
    assert L.parva_plan_batch_fused(*args, 0, dummy, C.byref(m), None) == BAD     # 32-B records > 8-B section
    m.plan_capacity = 9 * 128
    assert L.parva_plan_batch_fused(*args, 2, dummy, C.byref(m), None) == BAD     # plan section too small
    m.plan_capacity, m.plan_bytes = 10 * 128, 64
    assert L.parva_plan_batch_fused(*args, 2, dummy, C.byref(m), None) == BAD     # 64-B records need overflow
    m.plan_bytes = 128
    m.prev_epoch = 1
    assert L.parva_plan_batch_fused(*args, 2, dummy, C.byref(m), None) == BAD     # epoch == prev_epoch
    m.prev_epoch, m.d_done = 0, None
    assert L.parva_plan_batch_fused(*args, 2, dummy, C.byref(m), None) == BAD     # no CTA counter
    # overlapped launches need a ticket
    assert L.parva_plan_batch_overlapped(*args, 2, dummy, None, None) == BAD
    t = N.SlotTicket(None, 0, None)
    assert L.parva_plan_batch_overlapped(*args, 2, dummy, C.byref(t), None) == BAD
    g = N.GatherSlot()
    g.n = 1
    assert L.parva_gather_wait(None, 1, 1, 0, None, None) == BAD
    assert L.parva_gather_wait(C.byref(g), 1, 1, 0, dummy, None) == BAD            # no flag row
    g.d_flags = 16
    assert L.parva_gather_wait(C.byref(g), 0, 0, 0, dummy, None) == BAD            # epoch 0
    assert L.parva_gather_wait(C.byref(g), 1, 1, 0, dummy, None) == BAD            # release without ack words
    g.n = 9
    assert L.parva_gather_wait(C.byref(g), 1, 0, 0, dummy, None) == BAD
    assert L.parva_gather_release(None, 1, None) == BAD
    assert L.parva_ipc_handle(None, None) == BAD
    assert L.parva_ipc_open(None, None) == BAD
    assert L.parva_ipc_alloc(C.c_size_t(0), C.byref(C.c_void_p())) == BAD
    assert L.parva_plan_host_mapped_submit(None, None, 0, 0, None, C.c_int64(0), None, 1, 4, 2, 64, None,
                                           C.c_size_t(0), None, None) == BAD
    assert L.parva_plan_host_mapped(None, None, 0, 0, None, C.c_int64(0), None, 1, 4, 2, 64, None,
                                    C.c_size_t(0), None) == BAD
    assert L.parva_plan_host_mapped_wait(C.c_uint64(0)) == 0          # the empty call's ticket
    assert L.parva_sim_seed_states(None, 1, C.c_int64(0), C.c_int64(1), None) == BAD
    assert L.parva_ipc_handle_bytes() == 64


def test_record_layouts():
    assert CONFIG_DTYPE.itemsize == 32 and PLAN_DTYPE.itemsize == 128


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    fx = W.load_fixtures()
    with pytest.raises(P.NativeLibraryError):
        P.plan_services([P.make_service("resnet50", "resnet50", 100.0, 200.0)], fx.tables)
    with pytest.raises(P.NativeLibraryError):
        P.configure_service(P.make_service("resnet50", "resnet50", 100.0, 200.0), fx.tables["resnet50"])


def test_enumerate_full_configs_is_19():
    cfgs = P.enumerate_full_configs()
    assert len(cfgs) == 19
    assert ((0, 1), (1, 1), (2, 1), (3, 1), (4, 1), (5, 1), (6, 1)) in cfgs


def test_greedy_copies_on_empty_gpu():
    for size, n in ((1, 7), (2, 3), (3, 2), (4, 1), (7, 1)):
        g = P.GpuState(0)
        k = 0
        while g.place("s", size, 1, 1, 1.0) is not None:
            k += 1
        assert k == n
    g = P.GpuState(0)
    assert g.place("s", 3, 1, 1, 1.0).start_slot == 4
    assert g.place("s", 3, 1, 1, 1.0).start_slot == 0
    assert g.find_start(1) is None            # slot 3 blocked


def test_make_service_and_errors():
    s = P.make_service("a", "m", 10, 200)
    assert s.internal_latency == 100.0 and isinstance(s.request_rate, float)
    with pytest.raises(P.MigplanError):
        P.make_service("a", "m", -1, 200)
    with pytest.raises(P.MigplanError):
        P.make_service("a", "m", 1, 0)
    e = P.InfeasibleSLOError("x", 12.5)
    assert str(e) == "service 'x': no profile point has latency below 12.5 ms"
    assert str(P.SmallSegmentsUnavailableError("y")) == "service 'y' has no size-1 or size-2 triplet"


def test_profile_csv_round_trip():
    fx = W.load_fixtures()
    for m in fx.models:
        t = fx.tables[m]
        assert P.load_profile_table(P.serialize_profile_table(t, "csv")) == t
        assert P.load_profile_table(P.serialize_profile_table(t, "json"), format="json") == t
    with pytest.raises(P.ValidationError):
        P.ProfileTable("m", (P.ProfilePoint("m", 1, 1, 1, 1.0, 1.0), P.ProfilePoint("m", 1, 1, 1, 2.0, 1.0)))


def test_pack_tables_layout():
    fx = W.load_fixtures()
    pt = pack_tables(fx.tables)
    assert pt.n_tables == 11 and pt.n_points == 1311
    single = pack_tables(fx.tables, single_process=True)
    assert (single.procs == 1).all()
    # segments in key order: batch asc then procs asc within each size class
    for t in range(pt.n_tables):
        for c in range(5):
            a, n = int(pt.seg_start[t * 5 + c]), int(pt.seg_count[t * 5 + c])
            keys = list(zip(pt.batch[a:a + n], pt.procs[a:a + n]))
            assert keys == sorted(keys)


def test_workload_generators_deterministic():
    fx = W.load_fixtures()
    a = W.scenario_batch(fx, 300, seed=0)
    b = W.scenario_batch(fx, 300, seed=0)
    assert a.rate.tobytes() == b.rate.tobytes() and a.slo.tobytes() == b.slo.tobytes()
    d1 = W.dense_tables(5, seed=3)
    d2 = W.dense_tables(3, seed=3, first=2)
    s1 = int(d1.seg_start[10])
    assert d1.tp[s1:].tobytes() == d2.tp.tobytes()
    assert d1.rate[2:].tobytes() == d2.rate.tobytes() and d1.slo[2:].tobytes() == d2.slo.tobytes()
    assert W.c5_rates(3).tolist() == W.c5_rates(5)[:3].tolist()


def test_deployment_map_json_round_trip():
    d = P.DeploymentMap(gpus=[P.GpuState(3, [P.Placement("a", 4, 8, 2, 1695.0, 0), P.Placement("b", 3, 1, 1, 9.5, 4)])])
    e = P.DeploymentMap.from_json(d.to_json())
    assert e.to_json() == d.to_json()
    with pytest.raises(P.ValidationError):
        P.DeploymentMap.from_json('{"gpus":[{"id":0,"segments":[{"service":"a","instance_size":2,'
                                  '"batch_size":1,"process_count":1,"start_slot":5,"throughput_rps":1.0}]}]}')


def test_stream_pack_arrays_matches_the_u16_pack():
    """parva_stream_pack_arrays (plain int32 arrays, host thread pool) writes
    exactly the block parva_stream_pack writes from u16 table ids; ids
    outside [0, 65535) become 0xFFFF; bad offsets / capacity give -1."""
    import ctypes as C
    from paper_2409_14447_b200 import workloads as W
    L = N.load_library()
    fx = W.load_fixtures()
    sb = W.scenario_batch(fx, 3_000, seed=4)
    n, M = sb.rate.shape
    rng = np.random.default_rng(9)
    cnt = rng.integers(0, 30, 2_000)
    cases = [(np.arange(n + 1, dtype=np.int32) * M, np.tile(np.arange(M, dtype=np.int32), n),
              sb.rate.ravel().copy(), sb.bound.ravel().copy()),
             (np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32),
              rng.integers(-3, 70_000, int(cnt.sum())).astype(np.int32),
              rng.random(int(cnt.sum())), rng.random(int(cnt.sum())))]
    for off, tab, rate, bound in cases:
        k = len(off) - 1
        for chunk in (1, 7, 32):
            cap = int(L.parva_stream_bytes(C.c_int32(k), N.np_ptr(off), C.c_int32(chunk)))
            t16 = np.where((tab < 0) | (tab >= 65535), 65535, tab).astype(np.uint16)
            a = np.zeros(cap, np.uint8)
            na = L.parva_stream_pack(C.c_int32(k), N.np_ptr(off), N.np_ptr(t16), N.np_ptr(rate), N.np_ptr(bound),
                                     C.c_int32(chunk), N.np_ptr(a), C.c_int64(cap))
            for threads in (1, 3, 0):
                b = np.full(cap, 0xCD, np.uint8)
                nb = L.parva_stream_pack_arrays(C.c_int32(k), N.np_ptr(off), N.np_ptr(tab), N.np_ptr(rate),
                                                N.np_ptr(bound), C.c_int32(chunk), N.np_ptr(b), C.c_int64(cap),
                                                C.c_int32(threads))
                assert na == nb > 0 and a[:na].tobytes() == b[:nb].tobytes(), (k, chunk, threads)
            assert L.parva_stream_pack_arrays(C.c_int32(k), N.np_ptr(off), N.np_ptr(tab), N.np_ptr(rate),
                                              N.np_ptr(bound), C.c_int32(chunk), N.np_ptr(b),
                                              C.c_int64(na - 16), C.c_int32(0)) == -1
    bad = np.array([0, 5, 3, 8], dtype=np.int32)
    z = np.zeros(8)
    buf = np.zeros(4096, np.uint8)
    assert L.parva_stream_pack_arrays(C.c_int32(3), N.np_ptr(bad), N.np_ptr(np.zeros(8, np.int32)), N.np_ptr(z),
                                      N.np_ptr(z), C.c_int32(2), N.np_ptr(buf), C.c_int64(4096), C.c_int32(0)) == -1


def test_deployment_json_matches_json_dumps():
    """DeploymentMap.to_json writes the reference's json.dumps(indent=2)
    text directly; byte-equal on random maps (escapes, non-finite floats,
    ints, empty lists, slot order)."""
    import json
    import random

    from paper_2409_14447_b200.allocator import DeploymentMap
    from paper_2409_14447_b200.mig import GpuState, Placement
    rng = random.Random(7)
    for trial in range(400):
        gpus = []
        for g in range(rng.randint(0, 6)):
            gs = GpuState(id=rng.choice([g, 7 * g, -3, 10 ** 12]))
            for _ in range(rng.randint(0, 4)):
                tp = rng.choice([1.5, 0.1 + 0.2, 1e-300, 123456789.123, float("inf"), float("nan"), 3.0, 1e22,
                                 5e-324, -0.0, 7])
                sid = rng.choice(["a", "d121#3", 'q"uo\\te', "ünï", "tab\t", ""])
                gs.placements.append(Placement(sid, rng.choice([1, 2, 3, 4, 7]), rng.randint(1, 128),
                                               rng.randint(1, 8), tp, rng.randint(0, 6)))
            gpus.append(gs)
        d = DeploymentMap(gpus=gpus)
        assert d.to_json() == json.dumps(d.to_json_obj(), indent=2) + "\n", trial
