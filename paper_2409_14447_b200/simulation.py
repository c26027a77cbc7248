"""Discrete-event request simulator, batched on the GPU.

Mirrors the reference's simulator API (migplan evaluation.py:85-464):
`Workload`, `ServiceSimStats`, `SimReport`, `SegmentActivity`,
`ActivityReport`, `run_simulation`, `slo_compliance`, `internal_slack` --
same names, signatures, report fields and JSON.  `run_simulations` runs any
number of (deployment, services, workload, horizon, seed) jobs in ONE kernel
launch.

Split of the work:
  * seeding on the host: SeedSequence(seed).spawn over the sorted service
    ids and default_rng(child), exactly as the reference (evaluation.py:
    327-335); only each generator's 256-bit PCG64 state goes to the GPU;
  * arrivals on the GPU (parva_simulate, csrc/simulate.cu): numpy's
    Generator.exponential (PCG64 + ziggurat, tables from numpy itself) with
    the reference's chunked cumsum (evaluation.py:207-226), bit-identical;
  * the event loop (evaluation.py:337-416) -- completions and arrival
    wakeups in (time, seq) order, FIFO batching, lane accounting, busy time --
    on the GPU, one thread per service: services never interact in that
    loop, so each is an independent simulation;
  * statistics (numpy mean / percentile / max, rounding) on the host, with
    the reference's calls (evaluation.py:436-456).
There is no CPU event loop here: without the CUDA library this raises
NativeLibraryError.
"""

from __future__ import annotations

import copy
import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Mapping, Optional, Sequence

import numpy as np

from . import _native as N
from .errors import SimulationConfigError, UndefinedMetricError, ValidationError
from .evaluation import DEFAULT_SMS_PER_GPC
from .mig import SLOT_COUNT

ARRIVAL_KINDS = ("poisson", "deterministic")


@dataclass(frozen=True)
class SegmentActivity:
    service_id: str
    gpu: int
    start_slot: int
    instance_size: int
    sm_count: int
    activity: float


@dataclass(frozen=True)
class ActivityReport:
    """Per-segment SM activity plus the provisioned totals (evaluation.py:46-52)."""

    segments: tuple
    gpu_count: int
    sms_per_gpu: int


def internal_slack(report: ActivityReport) -> float:
    """One minus SM-weighted activity over all allocated SMs (evaluation.py:55-62)."""
    if not report.segments:
        raise UndefinedMetricError("internal slack is undefined for an empty report")
    weighted = sum(s.sm_count * s.activity for s in report.segments)
    total = sum(s.sm_count for s in report.segments)
    return 1.0 - weighted / total


@dataclass(frozen=True)
class Workload:
    """Arrival process: per-service rates in requests/s (evaluation.py:85-109)."""

    rates: tuple
    kind: str = "poisson"

    def __post_init__(self) -> None:
        if self.kind not in ARRIVAL_KINDS:
            raise ValidationError(f"arrival kind {self.kind!r} not in {ARRIVAL_KINDS}")
        for sid, rate in self.rates:
            if rate < 0:
                raise ValidationError(f"negative arrival rate for {sid!r}")

    @classmethod
    def from_services(cls, services, kind: str = "poisson", scale: float = 1.0) -> "Workload":
        return cls(rates=tuple((s.id, s.request_rate * scale) for s in services), kind=kind)

    def rate_map(self) -> dict:
        return dict(self.rates)


@dataclass
class ServiceSimStats:
    service_id: str
    arrived: int = 0
    served: int = 0
    queued_at_end: int = 0
    batches: int = 0
    violations: int = 0
    achieved_rps: float = 0.0
    latency_ms: dict = field(default_factory=dict)

    @property
    def slo_compliance(self) -> float:
        """Share of batches within the SLO; 1.0 with no batches (evaluation.py:122-127)."""
        if self.batches == 0:
            return 1.0
        return 1.0 - self.violations / self.batches


@dataclass
class SimReport:
    horizon_s: float
    seed: int
    kind: str
    services: dict
    activity: ActivityReport

    def to_json_obj(self) -> dict:
        """The reference's report JSON (evaluation.py:138-169)."""
        return {
            "horizon_s": self.horizon_s,
            "seed": self.seed,
            "arrivals": self.kind,
            "services": {
                sid: {"arrived": st.arrived, "served": st.served, "queued_at_end": st.queued_at_end,
                      "batches": st.batches, "violations": st.violations, "slo_compliance": st.slo_compliance,
                      "achieved_rps": round(st.achieved_rps, 6), "latency_ms": st.latency_ms}
                for sid, st in sorted(self.services.items())
            },
            "segments": [
                {"service": s.service_id, "gpu": s.gpu, "start_slot": s.start_slot,
                 "instance_size": s.instance_size, "sm_count": s.sm_count, "activity": round(s.activity, 9)}
                for s in self.activity.segments
            ],
        }

    def csv_rows(self, run_label: str = "") -> list:
        """One flat row per service (evaluation.py:171-192)."""
        rows = []
        for sid, st in sorted(self.services.items()):
            rows.append({
                "run": run_label, "seed": self.seed, "horizon_s": self.horizon_s, "arrivals": self.kind,
                "service": sid, "arrived": st.arrived, "served": st.served, "queued_at_end": st.queued_at_end,
                "batches": st.batches, "violations": st.violations, "slo_compliance": st.slo_compliance,
                "achieved_rps": round(st.achieved_rps, 6), "latency_mean_ms": st.latency_ms.get("mean", ""),
                "latency_p95_ms": st.latency_ms.get("p95", ""), "latency_max_ms": st.latency_ms.get("max", ""),
            })
        return rows


def slo_compliance(report: SimReport) -> dict:
    """Per-service share of batches meeting the SLO; None without batches (evaluation.py:195-204)."""
    return {sid: (None if st.batches == 0 else 1.0 - st.violations / st.batches)
            for sid, st in report.services.items()}


def _arrival_times(kind: str, rate: float, horizon: float, rng: np.random.Generator) -> np.ndarray:
    """All arrival instants in [0, horizon), seconds (evaluation.py:207-226).

    The same numpy calls in the same order as the reference, so the stream
    of each service's generator is consumed identically."""
    if rate <= 0:
        return np.empty(0)
    if kind == "deterministic":
        step = 1.0 / rate
        n = int(math.floor(horizon / step))
        times = np.arange(1, n + 1, dtype=np.float64) * step
        return times[times < horizon]
    chunks = []
    total = 0.0
    expected = max(int(rate * horizon * 1.2) + 16, 64)
    while total < horizon:
        gaps = rng.exponential(1.0 / rate, size=expected)
        chunk = np.cumsum(gaps) + total
        total = float(chunk[-1])
        chunks.append(chunk)
    times = np.concatenate(chunks)
    return times[times < horizon]


@dataclass
class SimJob:
    """One run_simulation call of a batch."""

    dmap: object
    tables: Mapping
    services: Sequence
    workload: Optional[Workload] = None
    horizon_s: float = 60.0
    seed: int = 0
    sms_per_gpc: int = DEFAULT_SMS_PER_GPC


def _spawn_states(seed, n: int) -> list:
    """PCG64 states (state hi, lo, inc hi, lo) of default_rng(child) for the
    children of SeedSequence(seed).spawn(n): the library's restatement for
    non-negative integer seeds, numpy itself otherwise."""
    if isinstance(seed, (int, np.integer)) and not isinstance(seed, bool) and int(seed) >= 0 and n > 0:
        v, words = int(seed), []
        while True:
            words.append(v & 0xFFFFFFFF)
            v >>= 32
            if not v:
                break
        if len(words) <= 64:
            w = np.asarray(words, dtype=np.uint32)
            out = np.zeros(4 * n, dtype=np.uint64)
            N.check(N.lib().parva_sim_seed_states(N.np_ptr(w), C.c_int32(len(words)), C.c_int64(0), C.c_int64(n),
                                                  N.np_ptr(out)), "parva_sim_seed_states")
            return [tuple(int(x) for x in out[4 * i:4 * i + 4]) for i in range(n)]
    m = (1 << 64) - 1
    states = []
    for ss in np.random.SeedSequence(seed).spawn(n):
        st = np.random.default_rng(ss).bit_generator.state["state"]
        states.append((st["state"] >> 64, st["state"] & m, st["inc"] >> 64, st["inc"] & m))
    return states


class _Prepared:
    """Host-side layout of one job: service order, per-service generator
    state and arrival parameters, segments (evaluation.py:311-345)."""

    def __init__(self, job: SimJob):
        if job.horizon_s <= 0:
            raise SimulationConfigError("horizon must be positive")
        self.job = job
        services_by_id = {s.id: s for s in job.services}
        workload = job.workload or Workload.from_services(job.services)
        self.kind = workload.kind
        rates = workload.rate_map()
        dmap = job.dmap
        ordered = sorted({p.service_id for _, p in dmap.placements()} | set(rates) | set(services_by_id))
        self.ids = ordered
        self.svc, self.rates = [], []
        # per service: arrival kind (0 none, 1 poisson, 2 deterministic), PCG64
        # state, scale / step, chunk size / count
        self.akind, self.pcg, self.scale, self.count = [], [], [], []
        self.pcg = _spawn_states(job.seed, len(ordered))      # evaluation.py:308-315
        for sid in ordered:
            svc = services_by_id.get(sid)
            if svc is None:
                raise SimulationConfigError(f"no service definition for {sid!r}")
            rate = rates.get(sid, 0.0)
            self.svc.append(svc)
            self.rates.append(rate)
            if rate <= 0:
                self.akind.append(0); self.scale.append(0.0); self.count.append(0)
            elif workload.kind == "deterministic":
                step = 1.0 / rate
                self.akind.append(2); self.scale.append(step); self.count.append(int(math.floor(job.horizon_s / step)))
            else:
                self.akind.append(1); self.scale.append(1.0 / rate)
                self.count.append(max(int(rate * job.horizon_s * 1.2) + 16, 64))
        # segments in deployment-map order; per service in that order too (dispatch order)
        index = {sid: i for i, sid in enumerate(ordered)}
        self.segments = []            # (service position, placement, gpu id, service_ms)
        for gpu in dmap.gpus:
            for p in sorted(gpu.placements, key=lambda p: p.start_slot):
                svc = services_by_id.get(p.service_id)
                if svc is None:
                    raise SimulationConfigError(f"no service definition for {p.service_id!r}")
                table = job.tables.get(svc.model_id)
                if table is None:
                    raise SimulationConfigError(f"no profile table for model {svc.model_id!r}")
                try:
                    point = table.get(p.instance_size, p.batch_size, p.process_count)
                except KeyError:
                    raise SimulationConfigError(
                        f"segment {p.service_id!r} ({p.instance_size},{p.batch_size},"
                        f"{p.process_count}) has no matching profile point") from None
                self.segments.append((index[p.service_id], p, gpu.id, point.latency))
        self.horizon_ms = job.horizon_s * 1000.0
        self.gpu_count = len(dmap.gpus)

    def buffer_len(self, si: int) -> int:
        """Arrival buffer of service si: two chunks (a third is needed with
        vanishing probability and is reported as capacity) or the grid."""
        k = self.akind[si]
        return 0 if k == 0 else 2 * self.count[si] if k == 1 else self.count[si]

    def host_arrivals(self, si: int) -> np.ndarray:
        """Arrivals (ms) of service si with numpy on the host -- the reference's
        own generator calls (for the CPU oracle in the tests)."""
        rng = np.random.default_rng(np.random.SeedSequence(self.job.seed).spawn(len(self.ids))[si])
        return _arrival_times(self.kind, self.rates[si], self.job.horizon_s, rng) * 1000.0


def _prepare_all(jobs: Sequence[SimJob]) -> list:
    """_Prepared per job; jobs that share the deployment, tables, services,
    workload and horizon (e.g. many seeds of one plan) share everything but
    the generator states."""
    memo, out = {}, []
    for j in jobs:
        key = (id(j.dmap), id(j.tables), id(j.services), id(j.workload), j.horizon_s)
        t = memo.get(key)
        if t is None:
            t = memo[key] = _Prepared(j)
            out.append(t)
        else:
            p = copy.copy(t)
            p.job = j
            p.pcg = _spawn_states(j.seed, len(t.ids))
            out.append(p)
    return out


def run_simulations(jobs: Sequence[SimJob], stream=None) -> list:
    """Batched run_simulation: every job's services simulated in one launch
    (arrivals generated on the GPU from each service's numpy generator state)."""
    torch = N.require_cuda()
    preps = _prepare_all(jobs)
    kind, pcg, scale, count, hs, buf_off = [], [], [], [], [], [0]
    seg_off, seg_ms, seg_batch, seg_lanes, slo, horizon = [0], [], [], [], [], []
    seg_rows = []                      # flat segment row -> (job, segment index)
    for pi, pr in enumerate(preps):
        per_svc = [[] for _ in pr.ids]
        for gi, (si, p, gid, ms) in enumerate(pr.segments):
            per_svc[si].append(gi)
        for si in range(len(pr.ids)):
            kind.append(pr.akind[si]); pcg.extend(pr.pcg[si]); scale.append(pr.scale[si]); count.append(pr.count[si])
            hs.append(pr.job.horizon_s)
            buf_off.append(buf_off[-1] + pr.buffer_len(si))
            for gi in per_svc[si]:
                _, p, _, ms = pr.segments[gi]
                seg_ms.append(ms); seg_batch.append(p.batch_size); seg_lanes.append(p.process_count)
                seg_rows.append((pi, gi))
            seg_off.append(len(seg_ms))
            slo.append(pr.svc[si].slo_latency)
            horizon.append(pr.horizon_ms)
    n = len(slo)
    if n == 0:
        return [_report(pr, [], [], [], [], [], {}) for pr in preps]
    dev = lambda a, dt: N.to_device(np.ascontiguousarray(a if len(a) else [0], dtype=dt))  # noqa: E731
    d = {"kind": dev(kind, np.int32), "pcg": dev(pcg, np.uint64), "scale": dev(scale, np.float64),
         "count": dev(count, np.int64), "hs": dev(hs, np.float64), "buf_off": dev(buf_off, np.int64),
         "seg_off": dev(seg_off, np.int32), "seg_ms": dev(seg_ms, np.float64), "seg_batch": dev(seg_batch, np.int32),
         "seg_lanes": dev(seg_lanes, np.int32), "slo": dev(slo, np.float64), "h": dev(horizon, np.float64)}
    o = {k: torch.zeros(n, dtype=torch.int64, device="cuda") for k in ("arrived", "served", "batches", "viol")}
    o_buf = torch.empty(max(buf_off[-1], 1), dtype=torch.float64, device="cuda")
    o_busy = torch.zeros(max(len(seg_ms), 1), dtype=torch.float64, device="cuda")
    o_status = torch.zeros(n, dtype=torch.int32, device="cuda")
    v = lambda t: N.ptr(t).value  # noqa: E731
    P = N.SimProblem(n, v(d["kind"]), v(d["pcg"]), v(d["scale"]), v(d["count"]), v(d["hs"]), v(d["buf_off"]),
                     v(d["seg_off"]), v(d["seg_ms"]), v(d["seg_batch"]), v(d["seg_lanes"]), v(d["slo"]), v(d["h"]))
    R = N.SimResult(v(o["arrived"]), v(o["served"]), v(o["batches"]), v(o["viol"]), v(o_buf), v(o_busy), v(o_status))
    N.check(N.lib().parva_simulate(C.byref(P), C.byref(R), N.stream_handle(stream)), "parva_simulate")
    if bool((o_status != 0).any()):
        raise SimulationConfigError("simulator capacity exceeded (> 32 segments or > 64 lanes for a service, "
                                    "or more than two arrival chunks)")
    # gather every service's batch latencies into one array (device), one copy back
    b_dev = o["batches"]
    starts = torch.as_tensor(np.asarray(buf_off[:-1], dtype=np.int64), device="cuda")
    tot = int(b_dev.sum().item())
    if tot:
        within = torch.arange(tot, device="cuda") - torch.repeat_interleave(torch.cumsum(b_dev, 0) - b_dev, b_dev)
        idx = torch.repeat_interleave(starts, b_dev) + within
        lat_dev = o_buf[idx]
        # per-service sorted samples for the percentiles: one segmented sort
        # on the device (values, then service id, both stable)
        seg = torch.repeat_interleave(torch.arange(n, device="cuda"), b_dev)
        v_sorted, perm = torch.sort(lat_dev, stable=True)
        _, perm2 = torch.sort(seg[perm], stable=True)
        srt_all = v_sorted[perm2].cpu().numpy()
        lat_all = lat_dev.cpu().numpy()
    else:
        lat_all = srt_all = np.zeros(0)
    arrived, served, batches, viol = (o[k].cpu().numpy() for k in ("arrived", "served", "batches", "viol"))
    busy = o_busy.cpu().numpy()
    lat_off = np.concatenate([[0], np.cumsum(batches)])
    pct = _percentiles_batch(srt_all, lat_off[:-1], batches)
    reports, k = [], 0
    for pi, pr in enumerate(preps):
        m = len(pr.ids)
        busy_by_seg = {}
        for si in range(m):
            for r in range(seg_off[k + si], seg_off[k + si + 1]):
                busy_by_seg[seg_rows[r][1]] = busy[r]
        lats = [(lat_all[lat_off[k + si]:lat_off[k + si + 1]], pct[k + si]) for si in range(m)]
        reports.append(_report(pr, lats, arrived[k:k + m], served[k:k + m], batches[k:k + m], viol[k:k + m],
                               busy_by_seg))
        k += m
    return reports


_Q = (np.true_divide(50, 100), np.true_divide(95, 100), np.true_divide(99, 100))


def _percentile_sorted(srt: np.ndarray, q) -> float:
    """np.percentile(a, 100*q) (method "linear") from the sorted sample, with
    numpy's own operations (_quantile: virtual index (n-1)*q, floor, clip to
    the last element, _lerp), so the value is bit-identical."""
    n = srt.shape[0]
    v = (n - 1) * q
    prev = math.floor(v)
    if v >= n - 1:
        return float(srt[-1])
    a, b = srt[prev], srt[prev + 1]
    gamma = np.float64(v - prev)
    diff = b - a
    if gamma >= 0.5:
        return float(b - diff * (1 - gamma))
    return float(a + diff * gamma)


def _percentiles_batch(srt_all: np.ndarray, off: np.ndarray, cnt: np.ndarray) -> list:
    """_percentile_sorted for many sorted samples at once (sample i =
    srt_all[off[i]:off[i] + cnt[i]]), elementwise with the same float64
    operations, so every value is bit-identical: per sample (p50, p95, p99, max),
    or None for an empty sample."""
    cnt = np.asarray(cnt, dtype=np.int64)
    off = np.asarray(off, dtype=np.int64)
    ok = cnt > 0
    res = np.zeros((cnt.shape[0], 4))
    if ok.any():
        o, n = off[ok], cnt[ok]
        last = o + n - 1
        cols = []
        for q in _Q:
            v = (n - 1).astype(np.float64) * q
            prev = np.floor(v)
            at_end = v >= (n - 1)
            pi = np.minimum(prev.astype(np.int64), n - 2).clip(min=0)
            a = srt_all[o + pi]
            b = srt_all[np.minimum(o + pi + 1, last)]
            gamma = v - prev
            diff = b - a
            val = np.where(gamma >= 0.5, b - diff * (1 - gamma), a + diff * gamma)
            cols.append(np.where(at_end, srt_all[last], val))
        cols.append(srt_all[last])
        res[ok] = np.stack(cols, axis=1)
    return [tuple(float(x) for x in r) if k else None for r, k in zip(res, ok)]


def _latency_stats(lat: np.ndarray, srt=None) -> dict:
    """The reference's latency summary (evaluation.py:436-456): numpy mean
    (pairwise sum, in batch order), linear-interpolated percentiles, max;
    rounded to 6 dp.  `srt` = the sample sorted (else sorted here), or the
    precomputed (p50, p95, p99, max)."""
    if isinstance(srt, tuple):
        p50, p95, p99, mx = srt
    else:
        if srt is None:
            srt = np.sort(lat)
        p50, p95, p99 = (_percentile_sorted(srt, q) for q in _Q)
        mx = float(srt[-1])
    return {"mean": round(float(lat.mean()), 6), "p50": round(p50, 6), "p95": round(p95, 6),
            "p99": round(p99, 6), "max": round(mx, 6)}


def _report(pr: _Prepared, lats, arrived, served, batches, viol, busy_by_seg) -> SimReport:
    job = pr.job
    activity = ActivityReport(
        segments=tuple(
            SegmentActivity(service_id=p.service_id, gpu=gid, start_slot=p.start_slot, instance_size=p.instance_size,
                            sm_count=p.instance_size * job.sms_per_gpc,
                            # Python floats, as in the reference: sum() compensates only exact floats
                            activity=min(1.0, float(busy_by_seg.get(gi, 0.0)) / (p.process_count * pr.horizon_ms)))
            for gi, (si, p, gid, ms) in enumerate(pr.segments)),
        gpu_count=pr.gpu_count,
        sms_per_gpu=SLOT_COUNT * job.sms_per_gpc,
    )
    out = {}
    for si, sid in enumerate(pr.ids):
        na = int(arrived[si]) if len(arrived) else 0
        nb = int(batches[si]) if len(batches) else 0
        sv = int(served[si]) if len(served) else 0
        lat, srt = lats[si] if nb else (None, None)
        out[sid] = ServiceSimStats(
            service_id=sid, arrived=na, served=sv, queued_at_end=na - sv, batches=nb,
            violations=int(viol[si]) if len(viol) else 0, achieved_rps=sv / job.horizon_s,
            latency_ms=({} if lat is None else _latency_stats(lat, srt)),
        )
    return SimReport(horizon_s=job.horizon_s, seed=job.seed, kind=pr.kind, services=out, activity=activity)


def run_simulation(dmap, tables: Mapping, services: Sequence, workload: Workload | None = None,
                   horizon_s: float = 60.0, seed: int = 0, sms_per_gpc: int = DEFAULT_SMS_PER_GPC) -> SimReport:
    """Simulate request service against a deployment map (evaluation.py:286-464)."""
    return run_simulations([SimJob(dmap, tables, services, workload, horizon_s, seed, sms_per_gpc)])[0]
