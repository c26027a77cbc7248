"""ctypes wrapper of the CPU oracle (oracle/migplan_oracle.c).

TEST INFRASTRUCTURE ONLY — a plain-C restatement of the reference planner
(`migplan`, /root/reference/pkg/src/migplan) used as the parity checker.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.  The product package
(paper_2409_14447_b200) never imports it.

Parity of the oracle itself is pinned against golden vectors rendered from
the reference (tests/golden/make_golden.py, checked by
tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libmigplan_oracle.so"

OTRIP = np.dtype([("size", "<i4"), ("batch", "<i4"), ("procs", "<i4"), ("tp", "<f8"),
                  ("lat", "<f8"), ("valid", "<i4")], align=True)
assert OTRIP.itemsize == 40

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = C.CDLL(str(LIB_PATH))
        _lib.oracle_pysum.restype = C.c_double
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else C.c_void_p(0)


class _OResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("n_gpus", C.c_int32), ("n_gpus_unopt", C.c_int32),
                ("n_place", C.c_int32), ("n_diag", C.c_int32), ("fallback", C.c_int32),
                ("gpu_cap", C.c_int32), ("place_cap", C.c_int32), ("diag_cap", C.c_int32),
                ("gpu_id", C.c_void_p), ("pl_off", C.c_void_p), ("pl_name", C.c_void_p),
                ("pl_trip", C.c_void_p), ("pl_slot", C.c_void_p), ("diag", C.c_void_p),
                ("ledger_val", C.c_void_p), ("ledger_order", C.c_void_p), ("unopt_place", C.c_int32)]


class _OProblem(C.Structure):
    _fields_ = [("n_names", C.c_int32), ("n_services", C.c_int32),
                ("svc_best", C.c_void_p), ("svc_opt", C.c_void_p), ("svc_count", C.c_void_p),
                ("svc_last", C.c_void_p), ("svc_rate", C.c_void_p), ("n_gpus", C.c_int32),
                ("gpu_id", C.c_void_p), ("pl_off", C.c_void_p), ("pl_name", C.c_void_p),
                ("pl_trip", C.c_void_p), ("pl_slot", C.c_void_p), ("ledger_val", C.c_void_p),
                ("ledger_order", C.c_void_p), ("relocate", C.c_int32), ("optimize", C.c_int32),
                ("threshold", C.c_int32)]


def _records():
    from paper_2409_14447_b200.records import CONFIG_DTYPE, PLAN_DTYPE
    return CONFIG_DTYPE, PLAN_DTYPE


def pysum(xs) -> float:
    a = np.ascontiguousarray(xs, dtype=np.float64)
    return lib().oracle_pysum(_p(a), C.c_int64(a.shape[0]))


def select_optimal(trips) -> int:
    """trips: list of (size, tp)."""
    a = np.zeros(len(trips), dtype=OTRIP)
    for i, (s, tp) in enumerate(trips):
        a[i]["size"] = s; a[i]["tp"] = tp; a[i]["valid"] = 1
    return lib().oracle_select_optimal(_p(a), C.c_int32(len(trips)))


def propose(tp1, tp2, freed):
    """-> (k2, k1) or None for SmallSegmentsUnavailableError."""
    t = np.zeros(2, dtype=OTRIP)
    p1 = p2 = C.c_void_p(0)
    if tp1 is not None:
        t[0]["size"] = 1; t[0]["tp"] = tp1; t[0]["valid"] = 1; p1 = C.c_void_p(t.ctypes.data)
    if tp2 is not None:
        t[1]["size"] = 2; t[1]["tp"] = tp2; t[1]["valid"] = 1; p2 = C.c_void_p(t.ctypes.data + OTRIP.itemsize)
    k2 = C.c_int64(); k1 = C.c_int64()
    rc = lib().oracle_propose(p1, p2, C.c_double(freed), C.byref(k2), C.byref(k1))
    return None if rc else (k2.value, k1.value)


def configure_batch(pt, q_table, q_rate, q_bound, threads: int = 0) -> np.ndarray:
    CONFIG, _ = _records()
    q_table = np.ascontiguousarray(q_table, dtype=np.int32)
    q_rate = np.ascontiguousarray(q_rate, dtype=np.float64)
    q_bound = np.ascontiguousarray(q_bound, dtype=np.float64)
    out = np.zeros(q_table.shape[0], dtype=CONFIG)
    lib().oracle_configure_batch(_p(pt.tp), _p(pt.lat), _p(pt.batch), _p(pt.procs), _p(pt.seg_start),
                                 _p(pt.seg_count), C.c_int32(q_table.shape[0]), _p(q_table), _p(q_rate),
                                 _p(q_bound), _p(out), C.c_int32(threads))
    return out


def plan_batch_records(pt, scen_off, svc_table, svc_rate, svc_bound, optimize=True, threshold=4,
                       threads: int = 0):
    """Batched plan_services in the parva record format -> (config records, plan records)."""
    CONFIG, PLAN = _records()
    scen_off = np.ascontiguousarray(scen_off, dtype=np.int32)
    svc_table = np.ascontiguousarray(svc_table, dtype=np.int32)
    svc_rate = np.ascontiguousarray(svc_rate, dtype=np.float64)
    svc_bound = np.ascontiguousarray(svc_bound, dtype=np.float64)
    n_scen = scen_off.shape[0] - 1
    n_svc = svc_table.shape[0]
    cfg = np.zeros(n_svc, dtype=CONFIG)
    plan = np.zeros(n_scen, dtype=PLAN)
    lib().oracle_plan_batch_records(_p(pt.tp), _p(pt.lat), _p(pt.batch), _p(pt.procs), _p(pt.seg_start),
                                    _p(pt.seg_count), C.c_int32(n_scen), _p(scen_off), _p(svc_table),
                                    _p(svc_rate), _p(svc_bound), C.c_int32(int(optimize)),
                                    C.c_int32(int(threshold)), _p(cfg), _p(plan), C.c_int32(threads))
    return cfg, plan


class _ResultBuf:
    def __init__(self, n_names, gcap=4096, dcap=4096):
        self.gpu_id = np.zeros(gcap, dtype=np.int64)
        self.pl_off = np.zeros(gcap + 1, dtype=np.int32)
        pcap = gcap * 7
        self.pl_name = np.zeros(pcap, dtype=np.int32)
        self.pl_trip = np.zeros(pcap, dtype=OTRIP)
        self.pl_slot = np.zeros(pcap, dtype=np.int32)
        self.diag = np.zeros(dcap * 3, dtype=np.int64)
        self.lv = np.zeros(max(n_names, 1), dtype=np.float64)
        self.lo = np.zeros(max(n_names, 1), dtype=np.int32)
        self.s = _OResult(gpu_cap=gcap, place_cap=pcap, diag_cap=dcap,
                          gpu_id=self.gpu_id.ctypes.data, pl_off=self.pl_off.ctypes.data,
                          pl_name=self.pl_name.ctypes.data, pl_trip=self.pl_trip.ctypes.data,
                          pl_slot=self.pl_slot.ctypes.data, diag=self.diag.ctypes.data,
                          ledger_val=self.lv.ctypes.data, ledger_order=self.lo.ctypes.data)

    def decode(self, n_names):
        s = self.s
        gpus = []
        for g in range(s.n_gpus):
            pls = []
            for k in range(self.pl_off[g], self.pl_off[g + 1]):
                t = self.pl_trip[k]
                pls.append((int(self.pl_name[k]), int(t["size"]), int(t["batch"]), int(t["procs"]),
                            float(t["tp"]), int(self.pl_slot[k])))
            gpus.append((int(self.gpu_id[g]), pls))
        diags = [tuple(int(v) for v in self.diag[3 * k:3 * k + 3]) for k in range(s.n_diag)]
        ledger = sorted(((int(self.lo[k]), k, float(self.lv[k])) for k in range(n_names) if self.lo[k]))
        return {"status": s.status, "gpus": gpus, "unopt": s.n_gpus_unopt, "diags": diags,
                "fallback": bool(s.fallback), "ledger": [(k, v) for _, k, v in ledger]}


def plan_scenario(pt, svc_table, svc_rate, svc_bound, optimize=True, threshold=4, gcap=4096):
    CONFIG, _ = _records()
    svc_table = np.ascontiguousarray(svc_table, dtype=np.int32)
    svc_rate = np.ascontiguousarray(svc_rate, dtype=np.float64)
    svc_bound = np.ascontiguousarray(svc_bound, dtype=np.float64)
    n = svc_table.shape[0]
    cfg = np.zeros(n, dtype=CONFIG)
    buf = _ResultBuf(n, gcap=gcap)
    lib().oracle_plan_scenario(_p(pt.tp), _p(pt.lat), _p(pt.batch), _p(pt.procs), _p(pt.seg_start),
                               _p(pt.seg_count), C.c_int32(n), _p(svc_table), _p(svc_rate), _p(svc_bound),
                               C.c_int32(int(optimize)), C.c_int32(int(threshold)), _p(cfg), C.byref(buf.s))
    return cfg, buf.decode(n)


def trips_array(rows):
    """rows: list of (size, batch, procs, tp, lat) or None -> OTRIP array."""
    a = np.zeros(len(rows), dtype=OTRIP)
    for i, r in enumerate(rows):
        if r is None:
            continue
        a[i]["size"], a[i]["batch"], a[i]["procs"], a[i]["tp"], a[i]["lat"] = r[0], r[1], r[2], r[3], r[4]
        a[i]["valid"] = 1
    return a


def plan_general(n_names, services, gpus, ledger, relocate, optimize, threshold, gcap=None):
    """services: list of dict(best={size: trip}, opt=trip|None, count=int, last=trip|None, rate=float);
    gpus: list of (id, [(name, (size, batch, procs, tp), slot), ...]); ledger: {name: (val, order)}."""
    S = len(services)
    best = trips_array([s["best"].get(sz) for s in services for sz in (1, 2, 3, 4, 7)] or [None])
    opt = trips_array([s["opt"] for s in services] or [None])
    last = trips_array([s["last"] for s in services] or [None])
    count = np.array([s["count"] for s in services] or [0], dtype=np.int64)
    rate = np.array([s["rate"] for s in services] or [0.0], dtype=np.float64)
    gid = np.array([g[0] for g in gpus] or [0], dtype=np.int64)
    off = np.zeros(len(gpus) + 1, dtype=np.int32)
    names, trips, slots = [], [], []
    for i, (_, pls) in enumerate(gpus):
        for name, t, slot in pls:
            names.append(name); trips.append(tuple(t) + (0.0,)); slots.append(slot)
        off[i + 1] = len(names)
    pl_name = np.array(names or [0], dtype=np.int32)
    pl_trip = trips_array(trips or [None])
    pl_slot = np.array(slots or [0], dtype=np.int32)
    lv = np.zeros(max(n_names, 1)); lo = np.zeros(max(n_names, 1), dtype=np.int32)
    for k, (v, o) in ledger.items():
        lv[k] = v; lo[k] = o
    P = _OProblem(n_names=n_names, n_services=S, svc_best=best.ctypes.data, svc_opt=opt.ctypes.data,
                  svc_count=count.ctypes.data, svc_last=last.ctypes.data, svc_rate=rate.ctypes.data,
                  n_gpus=len(gpus), gpu_id=gid.ctypes.data, pl_off=off.ctypes.data,
                  pl_name=pl_name.ctypes.data, pl_trip=pl_trip.ctypes.data, pl_slot=pl_slot.ctypes.data,
                  ledger_val=lv.ctypes.data, ledger_order=lo.ctypes.data, relocate=int(relocate),
                  optimize=int(optimize), threshold=int(threshold))
    total_pl = len(names) + sum(int(s["count"]) + (1 if s["last"] else 0) for s in services)
    buf = _ResultBuf(n_names, gcap=gcap or max(64, len(gpus) + total_pl + 1))
    lib().oracle_plan_general(C.byref(P), C.byref(buf.s))
    return buf.decode(n_names)


def simulate_service(arr_ms, seg_ms, seg_batch, seg_lanes, slo, horizon_ms):
    """One service of run_simulation's event loop -> (served, batches, violations,
    latencies[batches], busy_ms per segment)."""
    arr = np.ascontiguousarray(arr_ms, dtype=np.float64)
    ms = np.ascontiguousarray(seg_ms, dtype=np.float64)
    b = np.ascontiguousarray(seg_batch, dtype=np.int32)
    ln = np.ascontiguousarray(seg_lanes, dtype=np.int32)
    lat = np.zeros(max(arr.shape[0], 1), dtype=np.float64)
    busy = np.zeros(max(ms.shape[0], 1), dtype=np.float64)
    out = np.zeros(3, dtype=np.int64)
    lib().oracle_simulate_service(C.c_int64(arr.shape[0]), _p(arr), C.c_int32(ms.shape[0]), _p(ms), _p(b), _p(ln),
                                  C.c_double(slo), C.c_double(horizon_ms), _p(out[0:1]), _p(out[1:2]),
                                  _p(out[2:3]), _p(lat), _p(busy))
    return int(out[0]), int(out[1]), int(out[2]), lat[:out[1]].copy(), busy[:ms.shape[0]].copy()
