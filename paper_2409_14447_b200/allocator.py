"""Segment Allocator (Alg. 2) — drop-in for reference allocator.py.

Same names, signatures and results as `migplan.allocator`
(allocator.py:26-537).  DeploymentMap is the host-side container (JSON I/O,
metrics); relocate_segments, propose_small_segments, optimize_allocation
and reconfigure_service run on the GPU (csrc/plan_general.cu,
csrc/unit_ops.cu).  The batched fast path is pipeline.plan_services /
batch.plan_batch.
"""

from __future__ import annotations

import ctypes as C
import json
from collections import deque
from dataclasses import dataclass, field
from typing import Iterator, Optional, Sequence

import numpy as np

from . import _native as N
from .batch import GeneralInput, GeneralOutput, plan_general
from .configurator import Service, Triplet, configure_service
from .errors import MigplanError, SmallSegmentsUnavailableError, ValidationError
from .mig import SLOT_COUNT, GpuState, Placement, allowed_start_slots
from .records import COVERAGE_ASSERT, DIAG_REGRESSED, OK, format_diag

SIZE_ORDER = (7, 4, 3, 2, 1)
DEFAULT_OPTIMIZATION_THRESHOLD = 4


class SegmentQueues:
    """Per-size FIFO queues of (service id, triplet) (allocator.py:32-51)."""

    def __init__(self) -> None:
        self._queues: dict[int, deque] = {size: deque() for size in SIZE_ORDER}

    def enqueue(self, service_id: str, triplet: Triplet) -> None:
        self._queues[triplet.instance_size].append((service_id, triplet))

    def __len__(self) -> int:
        return sum(len(q) for q in self._queues.values())

    def drain(self) -> Iterator[tuple[str, Triplet]]:
        for size in SIZE_ORDER:
            q = self._queues[size]
            while q:
                yield q.popleft()


@dataclass
class DeploymentMap:
    """Ordered GPUs (stable ids) + freed_rate ledger + diagnostics (allocator.py:54-165).

    placement_log is kept for API compatibility; the device planner does not
    record the reference's internal per-placement log (it is never serialized).
    """

    gpus: list[GpuState] = field(default_factory=list)
    freed_rate: dict[str, float] = field(default_factory=dict)
    placement_log: list[dict] = field(default_factory=list)
    diagnostics: list[str] = field(default_factory=list)

    @property
    def gpu_count(self) -> int:
        return len(self.gpus)

    @property
    def total_gpcs(self) -> int:
        return sum(g.num_gpcs for g in self.gpus)

    def unallocated_fraction(self) -> float:
        if not self.gpus:
            return 0.0
        return 1.0 - self.total_gpcs / (SLOT_COUNT * len(self.gpus))

    def placements(self) -> Iterator[tuple[GpuState, Placement]]:
        for gpu in self.gpus:
            for p in gpu.placements:
                yield gpu, p

    def service_throughput(self) -> dict[str, float]:
        totals: dict[str, float] = {}
        for _, p in self.placements():
            totals[p.service_id] = totals.get(p.service_id, 0.0) + p.throughput
        return totals

    def clone(self) -> "DeploymentMap":
        return DeploymentMap(gpus=[g.clone() for g in self.gpus], freed_rate=dict(self.freed_rate),
                             placement_log=list(self.placement_log), diagnostics=list(self.diagnostics))

    def validate(self) -> None:
        for gpu in self.gpus:
            used: set[int] = set()
            for p in gpu.placements:
                cells = p.option.occupied + p.option.blocked
                overlap = used.intersection(cells)
                if overlap:
                    raise ValidationError(f"GPU {gpu.id}: slot overlap at {sorted(overlap)}")
                used.update(cells)
            if gpu.num_gpcs > SLOT_COUNT:
                raise ValidationError(f"GPU {gpu.id}: {gpu.num_gpcs} GPCs > 7")

    def to_json_obj(self) -> dict:
        return {"gpus": [{"id": gpu.id, "segments": [
            {"service": p.service_id, "instance_size": p.instance_size, "batch_size": p.batch_size,
             "process_count": p.process_count, "start_slot": p.start_slot, "throughput_rps": p.throughput}
            for p in sorted(gpu.placements, key=lambda p: p.start_slot)]} for gpu in self.gpus]}

    def to_json(self) -> str:
        """json.dumps(self.to_json_obj(), indent=2) + "\\n", byte for byte
        (the reference's to_json), written directly: one string template per
        segment, each distinct placement formatted once."""
        return _map_json(self.gpus)

    @classmethod
    def from_json(cls, text: str) -> "DeploymentMap":
        try:
            obj = json.loads(text)
        except json.JSONDecodeError as exc:
            raise ValidationError(f"deployment map: {exc}") from exc
        gpus = []
        for gpu_obj in obj.get("gpus", []):
            gpu = GpuState(id=int(gpu_obj["id"]))
            for seg in gpu_obj.get("segments", []):
                p = Placement(service_id=seg["service"], instance_size=int(seg["instance_size"]),
                              batch_size=int(seg["batch_size"]), process_count=int(seg["process_count"]),
                              throughput=float(seg["throughput_rps"]), start_slot=int(seg["start_slot"]))
                if p.start_slot not in [o.start for o in allowed_start_slots(p.instance_size)]:
                    raise ValidationError(f"GPU {gpu.id}: size {p.instance_size} cannot start at slot {p.start_slot}")
                gpu.placements.append(p)
            gpus.append(gpu)
        dmap = cls(gpus=gpus)
        dmap.validate()
        return dmap


_INF = (float("inf"), float("-inf"))


def _json_scalar(x) -> str:
    """json.dumps of one scalar: ints by int.__repr__, finite floats by
    float.__repr__ (what json's encoder does), anything else through json."""
    t = type(x)
    if t is int:
        return int.__repr__(x)
    if t is float and x == x and x not in _INF:
        return float.__repr__(x)
    return json.dumps(x)


_SEGMENT_JSON = ('        {{\n          "service": {},\n          "instance_size": {},\n          "batch_size": {},\n'
                 '          "process_count": {},\n          "start_slot": {},\n          "throughput_rps": {}\n        }}')


def _map_json(gpus) -> str:
    if not gpus:
        return '{\n  "gpus": []\n}\n'
    ids: dict = {}
    fmt, js = _SEGMENT_JSON.format, _json_scalar

    def seg(p):
        sid = ids.get(p.service_id)
        if sid is None:
            sid = ids[p.service_id] = json.dumps(p.service_id)
        return fmt(sid, js(p.instance_size), js(p.batch_size), js(p.process_count), js(p.start_slot), js(p.throughput))

    parts = []
    for gpu in gpus:
        pl = gpu.placements
        if len(pl) > 1:
            pl = sorted(pl, key=lambda p: p.start_slot)
        head = '    {\n      "id": ' + js(gpu.id) + ',\n      "segments": '
        parts.append(head + ("[\n" + ",\n".join([seg(p) for p in pl]) + "\n      ]\n    }" if pl else "[]\n    }"))
    return '{\n  "gpus": [\n' + ",\n".join(parts) + '\n  ]\n}\n'


# ---------------------------------------------------- general-problem glue
# Deliberate deviation: the reference accepts repeated
# service ids -- optimize_allocation then proposes from the last service of
# an id and merges their freed_rate entries (allocator.py:377-404) -- while
# the device planners keep one ledger entry per service.  Rather than return
# a silently different plan, every planning entry rejects repeated ids.
DUPLICATE_IDS = "service ids must be unique (the device planners keep one freed_rate entry per service)"


class _Builder:
    """Flattens (map, services) into the general kernel's catalogue form."""

    def __init__(self, services: Sequence[Service]):
        ids = [s.id for s in services]
        if len(set(ids)) != len(ids):
            raise ValidationError(DUPLICATE_IDS)
        self.services = list(services)
        self.names = list(ids)
        self.name_idx = {n: i for i, n in enumerate(ids)}
        self.g = GeneralInput(names=self.names, n_services=len(ids))
        self.memo: dict = {}
        self.cat_trip: list = []   # cat -> (name, size, batch, procs, tp)

    def name(self, sid: str) -> int:
        if sid not in self.name_idx:
            self.name_idx[sid] = len(self.names)
            self.names.append(sid)
        return self.name_idx[sid]

    def cat(self, sid: str, size: int, batch: int, procs: int, tp: float) -> int:
        key = (sid, size, batch, procs, tp)
        if key not in self.memo:
            self.cat_trip.append(key)
        return self.g.add_cat(size, tp, self.name(sid), self.memo, key)

    def trip_cat(self, sid: str, t: Optional[Triplet]) -> int:
        return -1 if t is None else self.cat(sid, t.instance_size, t.batch_size, t.process_count, t.throughput)

    def add_services(self, relocate_ids: Optional[set] = None):
        for s in self.services:
            by_size = {t.instance_size: t for t in s.best_triplets}
            self.g.svc_t1.append(self.trip_cat(s.id, by_size.get(1)))
            self.g.svc_t2.append(self.trip_cat(s.id, by_size.get(2)))
            take = relocate_ids is None or s.id in relocate_ids
            self.g.svc_opt.append(self.trip_cat(s.id, s.optimal_segment) if take else -1)
            self.g.svc_count.append(int(s.optimal_segment_count) if take and s.optimal_segment is not None else 0)
            self.g.svc_last.append(self.trip_cat(s.id, s.last_segment) if take else -1)
            self.g.svc_rate.append(float(s.request_rate))

    def add_map(self, dmap: DeploymentMap):
        for gpu in dmap.gpus:
            self.g.gpu_id.append(int(gpu.id))
            for p in gpu.placements:
                self.g.pl_cat.append(self.cat(p.service_id, p.instance_size, p.batch_size, p.process_count,
                                              p.throughput))
                self.g.pl_slot.append(int(p.start_slot))
            self.g.pl_off.append(len(self.g.pl_cat))
        for rank, (sid, v) in enumerate(dmap.freed_rate.items()):
            k = self.name(sid)
            while len(self.g.ledger_val) <= k:
                self.g.ledger_val.append(0.0); self.g.ledger_order.append(0)
            self.g.ledger_val[k] = float(v); self.g.ledger_order[k] = rank + 1

    def decode(self, out: GeneralOutput, base: DeploymentMap) -> DeploymentMap:
        gpus = []
        for g in range(len(out.gpu_id)):
            gs = GpuState(id=int(out.gpu_id[g]))
            for k in range(int(out.pl_off[g]), int(out.pl_off[g + 1])):
                sid, size, batch, procs, tp = self.cat_trip[int(out.pl_cat[k])]
                gs.placements.append(Placement(sid, size, batch, procs, tp, int(out.pl_slot[k])))
            gpus.append(gs)
        ledger = sorted((int(out.ledger_order[k]), k) for k in range(len(self.names)) if out.ledger_order[k])
        freed = {self.names[k]: float(out.ledger_val[k]) for _, k in ledger}
        diags = list(base.diagnostics)
        for reason, gid, name in out.diags:
            if reason == DIAG_REGRESSED:
                diags.append(format_diag(reason, -1, None))
            else:
                diags.append(format_diag(reason, gid, self.names[name] if name >= 0 else None))
        return DeploymentMap(gpus=gpus, freed_rate=freed, placement_log=list(base.placement_log), diagnostics=diags)


def _check_status(out: GeneralOutput, what: str, services=(), dmap=None):
    if out.status == OK:
        return
    if out.status == COVERAGE_ASSERT and dmap is not None:
        after = dmap.service_throughput()
        for svc in services:
            if svc.request_rate > 0 and svc.id in after and not after[svc.id] >= svc.request_rate * (1 - 1e-9):
                raise AssertionError(f"coverage for {svc.id} dropped below its request rate")
        raise AssertionError("coverage dropped below a request rate")
    raise MigplanError(f"{what}: device planner status {out.status}")


def relocate_segments(services: Sequence[Service]) -> DeploymentMap:
    """Queue all segments by size, first-fit onto fresh GPUs (allocator.py:292-316)."""
    for svc in services:
        if svc.optimal_segment is None and svc.request_rate > 0:
            raise MigplanError(f"service {svc.id!r} is not configured; run match_demand first")
    b = _Builder(services)
    b.add_services()
    b.g.relocate = True
    out = plan_general(b.g)
    _check_status(out, "relocate_segments")
    return b.decode(out, DeploymentMap())


def propose_small_segments(service: Service, freed_rate: float) -> list[Triplet]:
    """Min-GPC, then min-count size-1/2 cover of a freed rate (allocator.py:319-359)."""
    torch = N.require_cuda()
    by_size = {t.instance_size: t for t in service.best_triplets}
    t1, t2 = by_size.get(1), by_size.get(2)
    tp1 = N.to_device(np.array([t1.throughput if t1 else 0.0]))
    tp2 = N.to_device(np.array([t2.throughput if t2 else 0.0]))
    fr = N.to_device(np.array([float(freed_rate)]))
    k2 = torch.empty(1, dtype=torch.int64, device="cuda")
    k1 = torch.empty(1, dtype=torch.int64, device="cuda")
    ok = torch.empty(1, dtype=torch.uint8, device="cuda")
    N.check(N.lib().parva_propose_small_batch(C.c_int32(1), N.ptr(tp1), N.ptr(tp2), N.ptr(fr), N.ptr(k2), N.ptr(k1),
                                              N.ptr(ok), N.stream_handle()), "parva_propose_small_batch")
    if not int(ok.item()):
        raise SmallSegmentsUnavailableError(service.id)
    return [t2] * int(k2.item()) + [t1] * int(k1.item())


def optimize_allocation(dmap: DeploymentMap, services: Sequence[Service],
                        threshold: int = DEFAULT_OPTIMIZATION_THRESHOLD) -> DeploymentMap:
    """Split lightly loaded GPUs into size-1/2 segments and refill forward (allocator.py:362-443)."""
    b = _Builder(services)
    b.add_services(relocate_ids=set())
    b.add_map(dmap)
    b.g.optimize = True
    b.g.threshold = int(threshold)
    out = plan_general(b.g)
    res = b.decode(out, dmap)
    if out.fallback:
        res = dmap.clone()
        res.diagnostics.append(format_diag(DIAG_REGRESSED, -1, None))
        return res
    _check_status(out, "optimize_allocation", services, res)
    return res


@dataclass(frozen=True)
class PlacementChange:
    """One placement added to or removed from a map (allocator.py:446-467)."""

    action: str
    gpu: int
    service: str
    instance_size: int
    batch_size: int
    process_count: int
    start_slot: int

    def to_json_obj(self) -> dict:
        return {"action": self.action, "gpu": self.gpu, "service": self.service,
                "instance_size": self.instance_size, "batch_size": self.batch_size,
                "process_count": self.process_count, "start_slot": self.start_slot}


def _placement_set(dmap: DeploymentMap) -> set[tuple]:
    return {(gpu.id, p.service_id, p.instance_size, p.batch_size, p.process_count, p.start_slot)
            for gpu, p in dmap.placements()}


def diff_maps(before: DeploymentMap, after: DeploymentMap) -> list[PlacementChange]:
    """Placements that differ, removed first (allocator.py:484-491)."""
    old, new = _placement_set(before), _placement_set(after)
    return ([PlacementChange("removed", *e) for e in sorted(old - new)]
            + [PlacementChange("added", *e) for e in sorted(new - old)])


def reconfigure_service(dmap: DeploymentMap, services: Sequence[Service], updated: Service, table,
                        threshold: int = DEFAULT_OPTIMIZATION_THRESHOLD):
    """Re-plan one service against an existing map (allocator.py:494-537)."""
    ids = [s.id for s in services]
    if updated.id not in ids:
        raise ValidationError(f"service {updated.id!r} not present in the deployment")
    old = services[ids.index(updated.id)]
    new_service = configure_service(updated, table)
    unchanged = (new_service.optimal_segment == old.optimal_segment
                 and new_service.optimal_segment_count == old.optimal_segment_count
                 and new_service.last_segment == old.last_segment)
    new_services = [new_service if s.id == updated.id else s for s in services]
    if unchanged:
        return dmap, [], new_services
    working = dmap.clone()
    for gpu in working.gpus:
        gpu.placements = [p for p in gpu.placements if p.service_id != updated.id]
    working.gpus = [g for g in working.gpus if g.placements]
    b = _Builder(new_services)
    b.add_services(relocate_ids={updated.id})
    b.add_map(working)
    b.g.relocate = True
    b.g.optimize = True
    b.g.threshold = int(threshold)
    out = plan_general(b.g)
    optimized = b.decode(out, working)   # on fallback: the relocated working map + note
    if not out.fallback:
        _check_status(out, "reconfigure_service", new_services, optimized)
    return optimized, diff_maps(dmap, optimized), new_services
