"""Segment Configurator (Alg. 1) — drop-in for reference configurator.py.

Same names, signatures, value types and exceptions as
`migplan.configurator` (configurator.py:23-191).  The decisions are made on
the GPU: decide_best_triplets / configure_service run the K1 sweep kernel
(csrc/configure.cu), select_optimal_segment / match_demand run the list
kernels (csrc/unit_ops.cu).  For many services at once use
`pipeline.plan_services` or `batch.plan_batch`, which fuse everything into
one launch.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .errors import (InfeasibleSLOError, MigplanError, ResidualUncoverableError)
from .mig import INSTANCE_SIZES
from .profiles import ProfileTable
from .records import COUNT_OVERFLOW, INFEASIBLE_SLO, OK, RESIDUAL_UNCOVERABLE

_RESIDUAL_EPS = 1e-9


@dataclass(frozen=True)
class Triplet:
    """An operating point: instance size, batch size, process count (configurator.py:23-36)."""

    instance_size: int
    batch_size: int
    process_count: int
    throughput: float
    latency: float

    @property
    def efficiency(self) -> float:
        return self.throughput / self.instance_size


@dataclass(frozen=True)
class Service:
    """One inference service and its configuration (configurator.py:39-66)."""

    id: str
    model_id: str
    request_rate: float
    slo_latency: float
    internal_latency: float
    best_triplets: tuple[Triplet, ...] = ()
    optimal_segment: Optional[Triplet] = None
    optimal_segment_count: int = 0
    last_segment: Optional[Triplet] = None

    def segments(self) -> tuple[Triplet, ...]:
        segs = (self.optimal_segment,) * self.optimal_segment_count
        if self.last_segment is not None:
            segs = segs + (self.last_segment,)
        return segs

    @property
    def coverage(self) -> float:
        return sum(t.throughput for t in self.segments())

    @property
    def total_gpcs(self) -> int:
        return sum(t.instance_size for t in self.segments())


def make_service(service_id: str, model_id: str, request_rate: float, slo_latency: float,
                 internal_latency: float | None = None) -> Service:
    """Unconfigured service; planning bound defaults to slo / 2 (configurator.py:69-90)."""
    if slo_latency <= 0:
        raise MigplanError(f"service {service_id!r}: slo_latency must be > 0")
    if request_rate < 0:
        raise MigplanError(f"service {service_id!r}: request_rate must be >= 0")
    return Service(id=service_id, model_id=model_id, request_rate=float(request_rate),
                   slo_latency=float(slo_latency),
                   internal_latency=(float(slo_latency) / 2.0 if internal_latency is None
                                     else float(internal_latency)))


# ------------------------------------------------------------ decoding
def _triplet_cache(pt):
    """(point index -> Triplet cache, segment starts as Python ints) of a
    PackedTables, created on first use."""
    d = pt.__dict__
    cache = d.get("_triplet_cache")
    if cache is None:
        cache = d["_triplet_cache"] = {}
        d["_seg_start_py"] = [int(x) for x in pt.seg_start]
    return cache, d["_seg_start_py"]


def triplet_at(pt, t: int, c: int, j: int) -> Triplet:
    """The Triplet of point j of table t, size class c (one shared, immutable
    instance per point, built on first use)."""
    cache, seg = _triplet_cache(pt)
    i = seg[t * 5 + c] + j
    tr = cache.get(i)
    if tr is None:
        tr = cache[i] = Triplet(INSTANCE_SIZES[c], int(pt.batch[i]), int(pt.procs[i]), float(pt.tp[i]),
                                float(pt.lat[i]))
    return tr




def service_from_record(svc: Service, pt, t: int, rec) -> Service:
    """Configured Service from a config record (status must be OK): a numpy
    record, or the same record as a tuple (records.tolist()).  The triplet
    part (best per size, optimal, last) is shared by every service of table
    t with the same record positions (Triplets are immutable)."""
    if isinstance(rec, tuple):
        bests, o, l, count = rec[0], rec[1], rec[2], rec[6]
    else:
        bests, o, l, count = rec["best"].tolist(), int(rec["opt_sc"]), int(rec["last_sc"]), int(rec["count"])
    d = pt.__dict__
    kinds = d.get("_service_kinds")
    if kinds is None:
        kinds = d["_service_kinds"] = {}
    key = (t, *bests, o, l)
    v = kinds.get(key)
    if v is None:
        best = [None] * 5
        cache, seg = _triplet_cache(pt)
        for c in range(5):
            j = bests[c]
            if j >= 0:
                tr = cache.get(seg[t * 5 + c] + j)
                best[c] = tr if tr is not None else triplet_at(pt, t, c, j)
        v = kinds[key] = (tuple([b for b in best if b is not None]), best[o] if o >= 0 else None,
                          best[l] if l >= 0 else None)
    out = object.__new__(Service)     # frozen dataclass: fill its __dict__ directly (what __init__ stores)
    out.__dict__.update(id=svc.id, model_id=svc.model_id, request_rate=svc.request_rate,
                        slo_latency=svc.slo_latency, internal_latency=svc.internal_latency, best_triplets=v[0],
                        optimal_segment=v[1], optimal_segment_count=int(count), last_segment=v[2])
    return out


def raise_for_record(svc: Service, rec) -> None:
    st = rec[3] if isinstance(rec, tuple) else int(rec["status"])
    if st == OK:
        return
    if st == INFEASIBLE_SLO:
        raise InfeasibleSLOError(svc.id, svc.internal_latency)
    if st == COUNT_OVERFLOW:
        raise OverflowError(f"service {svc.id!r}: request rate / throughput is not a representable "
                            f"segment count (limit 2**40)")
    if st == RESIDUAL_UNCOVERABLE:
        raise ResidualUncoverableError(f"service {svc.id!r}: residual exceeds every triplet's throughput")
    raise MigplanError(f"service {svc.id!r}: configuration failed with status {st}")


def _sweep_one(service: Service, table: ProfileTable):
    from .batch import configure_sweep
    dt = N.device_tables_for([table], prepared=True)
    out = configure_sweep(dt, [0], [service.request_rate], [service.internal_latency])
    rec = N.records_to_numpy(out, 1, N.CONFIG_DTYPE)[0]
    return dt.packed, rec


def decide_best_triplets(service: Service, table: ProfileTable) -> Service:
    """Max-throughput point per size with latency < internal bound (configurator.py:93-113)."""
    pt, rec = _sweep_one(service, table)
    if int(rec["status"]) == INFEASIBLE_SLO:
        raise InfeasibleSLOError(service.id, service.internal_latency)
    best = [triplet_at(pt, 0, c, int(rec["best"][c])) for c in range(5) if rec["best"][c] >= 0]
    return replace(service, best_triplets=tuple(best))


def _lists(lists: Sequence[Sequence[Triplet]]):
    off = np.zeros(len(lists) + 1, dtype=np.int32)
    sizes, tps = [], []
    for k, ts in enumerate(lists):
        for t in ts:
            sizes.append(t.instance_size); tps.append(t.throughput)
        off[k + 1] = len(sizes)
    return (N.to_device(off), N.to_device(np.asarray(sizes or [0], dtype=np.int32)),
            N.to_device(np.asarray(tps or [0.0], dtype=np.float64)))


def select_optimal_segment(triplets: Sequence[Triplet]) -> Triplet:
    """Max throughput per GPC, ties to the larger instance (configurator.py:127-139)."""
    if not triplets:
        raise MigplanError("select_optimal_segment needs a non-empty triplet array")
    torch = N.require_cuda()
    off, size, tp = _lists([list(triplets)])
    out = torch.empty(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().parva_select_optimal_lists(C.c_int32(1), N.ptr(off), N.ptr(size), N.ptr(tp), N.ptr(out),
                                               N.stream_handle()), "parva_select_optimal_lists")
    return triplets[int(out.item())]


def match_demand(service: Service) -> Service:
    """Optimal segments x floor(rate/tp) plus a last segment (configurator.py:142-186)."""
    if not service.best_triplets:
        raise MigplanError(f"service {service.id!r} has no best_triplets; "
                           "decide_best_triplets must run first")
    torch = N.require_cuda()
    trips = list(service.best_triplets)
    off, size, tp = _lists([trips])
    rate = N.to_device(np.array([service.request_rate], dtype=np.float64))
    o_opt = torch.empty(1, dtype=torch.int32, device="cuda")
    o_last = torch.empty(1, dtype=torch.int32, device="cuda")
    o_count = torch.empty(1, dtype=torch.int64, device="cuda")
    o_cov = torch.empty(1, dtype=torch.float64, device="cuda")
    o_st = torch.empty(1, dtype=torch.uint8, device="cuda")
    N.check(N.lib().parva_match_demand_lists(C.c_int32(1), N.ptr(off), N.ptr(size), N.ptr(tp), N.ptr(rate),
                                             N.ptr(o_opt), N.ptr(o_last), N.ptr(o_count), N.ptr(o_cov),
                                             N.ptr(o_st), N.stream_handle()), "parva_match_demand_lists")
    st = int(o_st.item())
    if st != OK:
        raise_for_record(service, {"status": st})
    last = int(o_last.item())
    return replace(service, optimal_segment=trips[int(o_opt.item())],
                   optimal_segment_count=int(o_count.item()),
                   last_segment=trips[last] if last >= 0 else None)


def configure_service(service: Service, table: ProfileTable) -> Service:
    """Both configuration stages in one K1 launch (configurator.py:189-191)."""
    pt, rec = _sweep_one(service, table)
    raise_for_record(service, rec)
    return service_from_record(service, pt, 0, rec)
