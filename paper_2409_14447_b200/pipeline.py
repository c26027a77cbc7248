"""End-to-end planning — drop-in for reference pipeline.py (:21-123).

plan_services runs the reference's timed region (pipeline.py:95-103:
configure -> relocate -> optimize) as ONE fused K2 launch
(csrc/plan_batch.cu) and decodes the 128-byte plan record into the same
PlanResult / Service / DeploymentMap objects.  Scenarios beyond the fast
path's record limits are re-planned by the general kernel on the GPU.
`plan_many` plans a list of independent service sets in a single launch.
"""

from __future__ import annotations

import struct
import time
from dataclasses import dataclass, field
from typing import Mapping, Optional, Sequence

import numpy as np

from . import _native as N
from .allocator import DEFAULT_OPTIMIZATION_THRESHOLD, DUPLICATE_IDS, DeploymentMap
from .batch import plan_batch, resolve_capacity
from .configurator import Service, raise_for_record, service_from_record
from .errors import MigplanError, ValidationError
from .evaluation import DEFAULT_SMS_PER_GPC, allocated_fraction, external_fragmentation
from .mig import INSTANCE_SIZES, GpuState, Placement
from .profiles import DEFAULT_MEMORY_MAP, ProfileTable, filter_feasible
from .records import BAD_INPUT, CAPACITY, DIAG_REGRESSED, FLAG_FALLBACK, OK, format_diag, plan_payload, unpack_diag, unpack_place
from .scenario import Scenario, load_tables_for, scenario_services


@dataclass(frozen=True)
class PlanOptions:
    optimize: bool = True
    single_process: bool = False
    threshold: int = DEFAULT_OPTIMIZATION_THRESHOLD
    sms_per_gpc: int = DEFAULT_SMS_PER_GPC
    memory_map: Mapping[int, float] = field(default_factory=lambda: dict(DEFAULT_MEMORY_MAP))


@dataclass
class PlanResult:
    scenario_name: str
    services: list[Service]
    deployment: DeploymentMap
    planning_ms: float
    unoptimized_gpu_count: int

    @property
    def gpu_count(self) -> int:
        return self.deployment.gpu_count

    def summary(self, sms_per_gpc: int = DEFAULT_SMS_PER_GPC) -> dict:
        frag: Optional[float] = None
        alloc: Optional[float] = None
        if self.deployment.gpus:
            frag = external_fragmentation(self.deployment, sms_per_gpc)
            alloc = allocated_fraction(self.deployment, sms_per_gpc)
        return {
            "scenario": self.scenario_name, "gpu_count": self.gpu_count,
            "total_gpcs": self.deployment.total_gpcs, "external_fragmentation": frag,
            "allocated_fraction": alloc, "planning_ms": round(self.planning_ms, 3),
            "services": {s.id: {"request_rate": s.request_rate, "coverage_rps": round(s.coverage, 6),
                                "segments": len(s.segments()), "gpcs": s.total_gpcs} for s in self.services},
            "diagnostics": list(self.deployment.diagnostics),
        }


def prepare_tables(tables: Mapping[str, ProfileTable], options: PlanOptions) -> dict[str, ProfileTable]:
    """Memory filter + optional single-process restriction (pipeline.py:70-80)."""
    prepared = {}
    for model, table in tables.items():
        table = filter_feasible(table, options.memory_map)
        if options.single_process:
            table = table.restrict(process_counts=(1,))
        prepared[model] = table
    return prepared


def _decode_record(services: list[Service], rec) -> DeploymentMap:
    """DeploymentMap from a 128-byte plan record (include/parva_b200.h):
    `rec` is the record (numpy) or its 128 bytes."""
    buf = rec.tobytes() if hasattr(rec, "tobytes") else rec
    n_place, n_diag, n_ledger, flags = buf[4], buf[5], buf[6], buf[7]
    u16 = struct.unpack_from(f"<{n_place + n_diag}H", buf, 8)
    off = 8 + ((2 * (n_place + n_diag) + 7) & ~7)
    vals = struct.unpack_from(f"<{n_ledger}d", buf, off)
    keys = struct.unpack_from(f"<{n_ledger}H", buf, off + 8 * n_ledger)
    gpus: list[GpuState] = []
    kinds: dict = {}
    new_p = object.__new__
    cur = None
    for v in u16[:n_place]:
        g, cat, slot = v >> 11, (v >> 3) & 0xFF, v & 7
        if cur is None or cur.id != g:
            cur = GpuState(id=g)
            gpus.append(cur)
        k = kinds.get(cat)
        if k is None:
            s, c = divmod(cat, 5)
            size = INSTANCE_SIZES[c]
            t = next(x for x in services[s].best_triplets if x.instance_size == size)
            k = kinds[cat] = (services[s].id, size, t.batch_size, t.process_count, t.throughput)
        p = new_p(Placement)              # frozen dataclass: fill its __dict__ directly
        p.__dict__.update(service_id=k[0], instance_size=k[1], batch_size=k[2], process_count=k[3],
                          throughput=k[4], start_slot=slot)
        cur.placements.append(p)
    freed = {services[kk & 0xFF].id: v for kk, v in zip(keys, vals)}
    if flags & FLAG_FALLBACK:
        diags = [format_diag(DIAG_REGRESSED, -1, None)]
    else:
        diags = []
        for v in u16[n_place:]:
            g, reason, s = unpack_diag(v)
            diags.append(format_diag(reason, g, services[s].id))
    return DeploymentMap(gpus=gpus, freed_rate=freed, diagnostics=diags)


def _decode_general(services: list[Service], g, out) -> DeploymentMap:
    """DeploymentMap from the general kernel's outputs (GPU ids, placement
    lists as catalogue indices + start slots, ledger, diagnostics)."""
    cat_key = g.cat_key
    proto: dict = {}          # catalogue entry -> (service id, triplet fields)
    by_size: dict = {}        # service -> {instance size: triplet}

    def kind(cat):
        v = proto.get(cat)
        if v is None:
            s, c = cat_key[cat]
            d = by_size.get(s)
            if d is None:
                d = by_size[s] = {x.instance_size: x for x in services[s].best_triplets}
            t = d[INSTANCE_SIZES[c]]
            v = proto[cat] = (services[s].id, t.instance_size, t.batch_size, t.process_count, t.throughput)
        return v

    pl_cat, pl_slot, pl_off = out.pl_cat.tolist(), out.pl_slot.tolist(), out.pl_off.tolist()
    new_o = object.__new__
    _fields = ("service_id", "instance_size", "batch_size", "process_count", "throughput", "start_slot")

    def placement(cat, slot):       # frozen dataclass: fill its __dict__ directly (what __init__ stores)
        p = new_o(Placement)
        p.__dict__.update(zip(_fields, (*kind(cat), slot)))
        return p

    gpus = []
    for k, gid in enumerate(out.gpu_id.tolist()):
        g = new_o(GpuState)
        g.__dict__.update(id=gid, placements=[placement(pl_cat[j], pl_slot[j]) for j in range(pl_off[k], pl_off[k + 1])])
        gpus.append(g)
    order = out.ledger_order
    live = np.flatnonzero(order[:len(services)])
    ranks = live[np.argsort(order[live], kind="stable")].tolist()
    vals = out.ledger_val
    freed = {services[s].id: float(vals[s]) for s in ranks}
    diags = [format_diag(r, gid, services[n].id if n >= 0 else None) for r, gid, n in out.diags]
    return DeploymentMap(gpus=gpus, freed_rate=freed, diagnostics=diags)


class _BatchRecords:
    """The records of one plan_many call, shared by its lazy results: config
    records (numpy), plan records, and the general kernel's outputs for the
    scenarios it re-planned."""

    __slots__ = ("pt", "off", "tab", "cfg", "plan", "general")

    def __init__(self, pt, off, tab, cfg, plan, general):
        self.pt, self.off, self.tab, self.cfg, self.plan, self.general = pt, off, tab, cfg, plan, general

    def decode(self, k: int, ss) -> tuple[list[Service], DeploymentMap]:
        a = int(self.off[k])
        recs = self.cfg[a:a + len(ss)].tolist()
        configured = [service_from_record(s, self.pt, self.tab[a + i], recs[i]) for i, s in enumerate(ss)]
        if k in self.general:
            g, go = self.general[k]
            dmap = _decode_general(configured, g, go)
            if go.fallback:
                dmap.diagnostics = [format_diag(DIAG_REGRESSED, -1, None)]
        else:
            dmap = _decode_record(configured, self.plan[k])
        return configured, dmap


class LazyPlanResult(PlanResult):
    """A PlanResult of plan_many whose configured services and deployment map
    are built from the batch's records on first access (the scenario-level
    fields -- gpu_count, unoptimized_gpu_count -- come straight from the plan
    record).  It is a PlanResult in every other respect: same fields,
    equality, repr, summary()."""

    def __init__(self, scenario_name="", services=None, deployment=None, planning_ms=0.0, unoptimized_gpu_count=0,
                 *, _src=None, _k=0, _ss=None, _n_gpus=0):
        self.scenario_name = scenario_name
        self.planning_ms = planning_ms
        self.unoptimized_gpu_count = unoptimized_gpu_count
        self._src, self._k, self._ss, self._n_gpus = _src, _k, _ss, _n_gpus
        self._dec = None if _src is not None else [services, deployment]

    def _decoded(self):
        if self._dec is None:
            self._dec = list(self._src.decode(self._k, self._ss))
            self._src = self._ss = None
        return self._dec

    @property
    def services(self) -> list[Service]:
        return self._decoded()[0]

    @services.setter
    def services(self, v):
        self._decoded()[0] = v

    @property
    def deployment(self) -> DeploymentMap:
        return self._decoded()[1]

    @deployment.setter
    def deployment(self, v):
        self._decoded()[1] = v

    @property
    def gpu_count(self) -> int:
        return self._n_gpus if self._dec is None else self._dec[1].gpu_count

    def __eq__(self, other):
        if not isinstance(other, PlanResult):
            return NotImplemented
        f = lambda r: (r.scenario_name, r.services, r.deployment, r.planning_ms, r.unoptimized_gpu_count)  # noqa: E731
        return f(self) == f(other)

    __hash__ = None


def _first_errors(cfg, plan, off, general) -> dict:
    """Scenario -> index of its first non-OK config record (input order), or
    -1 when every service is OK but the plan record failed (vectorized)."""
    st = cfg["status"]
    bad = np.flatnonzero(st != OK)
    out = {}
    if len(bad):
        ks = np.searchsorted(off, bad, side="right") - 1
        first = np.ones(len(bad), dtype=bool)
        first[1:] = ks[1:] != ks[:-1]
        out = {int(k): int(i) for k, i in zip(ks[first], bad[first])}
    for k in np.flatnonzero(plan["status"] != OK).tolist():
        if k not in out and k not in general:
            out[k] = -1
    return out


_ZERO_COPY_MAX = 1024        # scenarios: smaller plan_many calls run zero-copy from pinned host memory


class _PinnedArena:
    """Pinned host memory of the small-batch path (one per process, grown on
    demand, one call at a time).  With unified addressing a pinned host
    pointer is also a device pointer, so K2 reads the inputs and writes its
    records over PCIe: no copies, one launch and one synchronize per call."""

    def __init__(self):
        import threading
        self.lock = threading.Lock()
        self.buf = None

    def views(self, n: int, m: int):
        torch = N.require_cuda()
        up = lambda x: (x + 255) & ~255  # noqa: E731
        sizes = [4 * (n + 1), 4 * m, 8 * m, 8 * m, 32 * max(m, 1), 128 * max(n, 1)]   # >= 1 record each
        offs, tot = [], 0
        for b in sizes:
            offs.append(tot)
            tot += up(max(b, 1))
        if self.buf is None or self.buf.numel() < tot:
            self.buf = torch.empty(max(tot, 1 << 20), dtype=torch.uint8).pin_memory()
        v = [self.buf[o:o + b] for o, b in zip(offs, sizes)]
        return (v[0].view(torch.int32), v[1].view(torch.int32), v[2].view(torch.float64), v[3].view(torch.float64),
                v[4].view(-1, 32), v[5].view(-1, 128))


_ARENA = _PinnedArena()


def _plan_zero_copy(dt, off, tab, rate, bound, options):
    """One K2 launch over pinned host buffers; (config, plan) record copies."""
    from .batch import BatchResult
    from .records import CFG_FULL, CONFIG_DTYPE, PLAN_DTYPE
    torch = N.require_cuda()
    n, m = len(off) - 1, len(tab)
    with _ARENA.lock:
        t_off, t_tab, t_rate, t_bound, o_cfg, o_plan = _ARENA.views(n, m)
        t_off.numpy()[:] = off
        if m:
            t_tab.numpy()[:] = tab
            t_rate.numpy()[:] = rate
            t_bound.numpy()[:] = bound
        out = BatchResult(o_cfg, o_plan, n, m, CFG_FULL)
        plan_batch(dt, t_off, t_tab, t_rate, t_bound, optimize=options.optimize, threshold=options.threshold,
                   out=out)
        torch.cuda.current_stream().synchronize()
        cfg = o_cfg.numpy()[:m].copy().view(CONFIG_DTYPE).reshape(m)
        plan = o_plan.numpy()[:n].copy().view(PLAN_DTYPE).reshape(n)
    return cfg, plan


def plan_many(service_sets: Sequence[Sequence[Service]], tables: Mapping[str, ProfileTable],
              options: PlanOptions = PlanOptions(), names: Sequence[str] | None = None,
              raise_errors: bool = False) -> list:
    """Plan independent service sets in one fused launch.

    Returns one PlanResult per set (a LazyPlanResult: its services and
    deployment are decoded from the records on first access), or the
    exception the reference would raise for that set (raised instead when
    raise_errors)."""
    dt = N.device_tables_for(tables, options.memory_map, options.single_process)
    pt = dt.packed
    idx = pt.index_of()
    n = len(service_sets)
    counts = np.fromiter((len(ss) for ss in service_sets), dtype=np.int64, count=n)
    off = np.zeros(n + 1, dtype=np.int32)
    np.cumsum(counts, out=off[1:])
    flat = [s for ss in service_sets for s in ss]
    tab = np.fromiter((idx.get(s.model_id, -1) for s in flat), dtype=np.int32, count=len(flat))
    rate = np.fromiter((s.request_rate for s in flat), dtype=np.float64, count=len(flat))
    bound = np.fromiter((s.internal_latency for s in flat), dtype=np.float64, count=len(flat))
    torch = N.require_cuda()
    t0 = time.perf_counter()
    if n <= _ZERO_COPY_MAX and dt.index_struct is not None:
        cfg, plan = _plan_zero_copy(dt, off, tab, rate, bound, options)
    else:
        res = plan_batch(dt, off, tab, rate, bound, optimize=options.optimize, threshold=options.threshold)
        cfg, plan = res.host()
    general = resolve_capacity(pt, off, tab, cfg, plan, options.optimize, options.threshold)
    torch.cuda.synchronize()
    elapsed_ms = (time.perf_counter() - t0) * 1000.0
    errors = _first_errors(cfg, plan, off, general)
    for k, ss in enumerate(service_sets):             # repeated ids: rejected (see allocator.DUPLICATE_IDS)
        if len(ss) > 1 and len({s.id for s in ss}) != len(ss) and k not in errors:
            errors[k] = -2
    src = _BatchRecords(pt, off, tab.tolist(), cfg, plan, general)
    n_gpus = plan["n_gpus"].tolist()
    unopt = plan["n_gpus_unopt"].tolist()
    out = []
    for k, ss in enumerate(service_sets):
        name = names[k] if names else ""
        if k in errors:
            try:
                i = errors[k]
                if i == -2:
                    raise ValidationError(DUPLICATE_IDS)
                if i < 0:
                    raise MigplanError(f"device planner status {int(plan[k]['status'])}")
                a = int(off[k])
                rec = cfg[i]
                if int(rec["status"]) == BAD_INPUT:
                    raise KeyError(ss[i - a].model_id)
                raise_for_record(ss[i - a], rec)
                raise MigplanError(f"device planner status {int(rec['status'])}")
            except (MigplanError, KeyError, OverflowError) as exc:
                if raise_errors:
                    raise
                out.append(exc)
            continue
        if k in general:
            g, go = general[k]
            if go.status != OK:
                exc = MigplanError(f"device planner status {go.status}")
                if raise_errors:
                    raise exc
                out.append(exc)
                continue
            out.append(LazyPlanResult(name, planning_ms=elapsed_ms, unoptimized_gpu_count=int(go.n_gpus_unopt),
                                      _src=src, _k=k, _ss=ss, _n_gpus=int(len(go.gpu_id))))
            continue
        out.append(LazyPlanResult(name, planning_ms=elapsed_ms, unoptimized_gpu_count=unopt[k], _src=src, _k=k,
                                  _ss=ss, _n_gpus=n_gpus[k]))
    return out


def plan_services(services: Sequence[Service], tables: Mapping[str, ProfileTable],
                  options: PlanOptions = PlanOptions(), scenario_name: str = "") -> PlanResult:
    """Configure, relocate and (optionally) optimize (pipeline.py:83-111)."""
    return plan_many([list(services)], tables, options, names=[scenario_name], raise_errors=True)[0]


def plan_scenario(scenario: Scenario, tables: Mapping[str, ProfileTable] | None = None,
                  options: PlanOptions = PlanOptions(), profiles_override=None) -> PlanResult:
    if tables is None:
        tables = load_tables_for(scenario, profiles_override)
    return plan_services(scenario_services(scenario), tables, options, scenario_name=scenario.name)
