"""End-to-end planning — drop-in for reference pipeline.py (:21-123).

plan_services runs the reference's timed region (pipeline.py:95-103:
configure -> relocate -> optimize) as ONE fused K2 launch
(csrc/plan_batch.cu) and decodes the 128-byte plan record into the same
PlanResult / Service / DeploymentMap objects.  Scenarios beyond the fast
path's record limits are re-planned by the general kernel on the GPU.
`plan_many` plans a list of independent service sets in a single launch.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Mapping, Optional, Sequence

import numpy as np

from . import _native as N
from .allocator import DEFAULT_OPTIMIZATION_THRESHOLD, DeploymentMap
from .batch import plan_batch, resolve_capacity
from .configurator import Service, raise_for_record, service_from_record
from .errors import MigplanError
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
    """DeploymentMap from a 128-byte plan record (include/parva_b200.h)."""
    places, diag_codes, ledger = plan_payload(rec)
    gpus: list[GpuState] = []
    by_size = [{t.instance_size: t for t in s.best_triplets} for s in services]
    for v in places:
        g, cat, slot = unpack_place(v)
        s, c = divmod(cat, 5)
        if not gpus or gpus[-1].id != g:
            gpus.append(GpuState(id=g))
        t = by_size[s][INSTANCE_SIZES[c]]
        gpus[-1].placements.append(Placement(services[s].id, t.instance_size, t.batch_size,
                                             t.process_count, t.throughput, slot))
    freed = {services[s].id: v for s, v in ledger}
    if int(rec["flags"]) & FLAG_FALLBACK:
        diags = [format_diag(DIAG_REGRESSED, -1, None)]
    else:
        diags = []
        for v in diag_codes:
            g, reason, s = unpack_diag(v)
            diags.append(format_diag(reason, g, services[s].id))
    return DeploymentMap(gpus=gpus, freed_rate=freed, diagnostics=diags)


def _decode_general(services: list[Service], g, out) -> DeploymentMap:
    gpus = []
    for k in range(len(out.gpu_id)):
        gs = GpuState(id=int(out.gpu_id[k]))
        for j in range(int(out.pl_off[k]), int(out.pl_off[k + 1])):
            s, c = g.cat_key[int(out.pl_cat[j])]
            t = {INSTANCE_SIZES.index(x.instance_size): x for x in services[s].best_triplets}[c]
            gs.placements.append(Placement(services[s].id, t.instance_size, t.batch_size, t.process_count,
                                           t.throughput, int(out.pl_slot[j])))
        gpus.append(gs)
    ranks = sorted((int(out.ledger_order[s]), s) for s in range(len(services)) if out.ledger_order[s])
    freed = {services[s].id: float(out.ledger_val[s]) for _, s in ranks}
    diags = [format_diag(r, gid, services[n].id if n >= 0 else None) for r, gid, n in out.diags]
    return DeploymentMap(gpus=gpus, freed_rate=freed, diagnostics=diags)


def plan_many(service_sets: Sequence[Sequence[Service]], tables: Mapping[str, ProfileTable],
              options: PlanOptions = PlanOptions(), names: Sequence[str] | None = None,
              raise_errors: bool = False) -> list:
    """Plan independent service sets in one fused launch.

    Returns one PlanResult per set, or the exception the reference would
    raise for that set (raised instead when raise_errors)."""
    dt = N.device_tables_for(tables, options.memory_map, options.single_process)
    pt = dt.packed
    idx = pt.index_of()
    off = np.zeros(len(service_sets) + 1, dtype=np.int32)
    tab, rate, bound = [], [], []
    for k, ss in enumerate(service_sets):
        for s in ss:
            tab.append(idx.get(s.model_id, -1)); rate.append(s.request_rate); bound.append(s.internal_latency)
        off[k + 1] = len(tab)
    torch = N.require_cuda()
    t0 = time.perf_counter()
    res = plan_batch(dt, off, np.asarray(tab, dtype=np.int32), np.asarray(rate), np.asarray(bound),
                     optimize=options.optimize, threshold=options.threshold)
    cfg, plan = res.host()
    general = resolve_capacity(pt, off, np.asarray(tab, dtype=np.int32), cfg, plan, options.optimize,
                               options.threshold)
    torch.cuda.synchronize()
    elapsed_ms = (time.perf_counter() - t0) * 1000.0
    out = []
    cfg_t = cfg.tolist()                   # records as tuples: plain attribute-free access below
    for k, ss in enumerate(service_sets):
        a = int(off[k])
        try:
            configured = []
            for i, s in enumerate(ss):
                rec = cfg_t[a + i]
                if rec[3] == BAD_INPUT:
                    raise KeyError(s.model_id)
                raise_for_record(s, rec)
                configured.append(service_from_record(s, pt, tab[a + i], rec))
            rec = plan[k]
            if k in general:
                g, go = general[k]
                if go.status != OK:
                    raise MigplanError(f"device planner status {go.status}")
                dmap = _decode_general(configured, g, go)
                unopt = go.n_gpus_unopt
                if go.fallback:
                    dmap.diagnostics = [format_diag(DIAG_REGRESSED, -1, None)]
            else:
                if int(rec["status"]) != OK:
                    raise MigplanError(f"device planner status {int(rec['status'])}")
                dmap = _decode_record(configured, rec)
                unopt = int(rec["n_gpus_unopt"])
            out.append(PlanResult(scenario_name=(names[k] if names else ""), services=configured,
                                  deployment=dmap, planning_ms=elapsed_ms, unoptimized_gpu_count=unopt))
        except (MigplanError, KeyError, OverflowError) as exc:
            if raise_errors:
                raise
            out.append(exc)
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
