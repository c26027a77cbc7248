"""Batched device entry points (the product's hot path).

    configure_sweep(dt, q_table, q_rate, q_bound)       K1, HBM-bound sweep
    plan_batch(dt, scen_off, svc_table, rate, bound)    K2, fused planner
    plan_general(GeneralInput)                          KG, unbounded problems

All of them enqueue sm_100a kernels on the current torch CUDA stream through
the C ABI (include/parva_b200.h); nothing here computes a plan on the host.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .records import (CAPACITY, CFG_COMPACT, CFG_FULL, CFG_TINY, COMPACT_DTYPE, CONFIG_DTYPE, PLAN64_DTYPE, PLAN_DTYPE,
                      SPILL_DTYPE, SPILLED, TINY_DTYPE)
from .tables import PackedTables


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def configure_sweep(dt: N.DeviceTables, q_table, q_rate, q_bound, out=None, stream=None):
    """Device config records (uint8 [nq, 32]) for one query per row."""
    torch = N.require_cuda()
    q_table = q_table if isinstance(q_table, torch.Tensor) else N.to_device(_i32(q_table))
    q_rate = q_rate if isinstance(q_rate, torch.Tensor) else N.to_device(_f64(q_rate))
    q_bound = q_bound if isinstance(q_bound, torch.Tensor) else N.to_device(_f64(q_bound))
    nq = int(q_table.shape[0])
    if out is None:
        out = N.empty_records(nq, CONFIG_DTYPE)
    N.check(N.lib().parva_configure_sweep(C.byref(dt.struct), C.c_int32(nq), N.ptr(q_table), N.ptr(q_rate),
                                          N.ptr(q_bound), N.ptr(out), N.stream_handle(stream)),
            "parva_configure_sweep")
    return out


@dataclass
class BatchResult:
    cfg: object            # device uint8 config records (32, 16 or 8 bytes each, cfg_format)
    plan: object           # device uint8 plan records: 128 bytes each, or 64 with `spill`
    n_scenarios: int
    n_services: int
    cfg_format: int = CFG_FULL
    spill: object = None   # 64-byte records: full records of spilled scenarios (same index, 128 B each)

    def host(self):
        """(config records, 128-byte plan records) on the host."""
        cfg = N.records_to_numpy(self.cfg, self.n_services, _CFG_DT[self.cfg_format])
        if self.spill is None:
            return cfg, N.records_to_numpy(self.plan, self.n_scenarios, PLAN_DTYPE)
        p64 = N.records_to_numpy(self.plan, self.n_scenarios, PLAN64_DTYPE)
        plan = np.zeros(self.n_scenarios, dtype=PLAN_DTYPE)
        plan.view(np.uint8).reshape(-1, 128)[:, :64] = p64.view(np.uint8).reshape(-1, 64)
        sp = np.nonzero(p64["status"] == SPILLED)[0]
        if len(sp):
            plan[sp] = N.records_to_numpy(self.spill, self.n_scenarios, PLAN_DTYPE)[sp]
        return cfg, plan


class SlotRing:
    """Output slots of overlapped launches (parva_slot_ticket): `n_slots`
    slots, each with a u64 completion counter on the device.  ticket(slot,
    n_scenarios) is the ticket of the next launch into `slot`: its CTAs
    store nothing until every scenario of the slot's earlier launches is
    done, so overlapped launches that share a slot never overlap each other
    -- safe by construction, however many grids are in flight."""

    def __init__(self, n_slots: int):
        torch = N.require_cuda()
        if n_slots < 1:
            raise ValueError("n_slots must be >= 1")
        self.n_slots = int(n_slots)
        self.counts = torch.zeros(self.n_slots, dtype=torch.int64, device="cuda")
        self.err = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.issued = [0] * self.n_slots       # scenarios launched into each slot so far

    def ticket(self, slot: int, n_scenarios: int) -> N.SlotTicket:
        t = N.SlotTicket(self.counts.data_ptr() + 8 * slot, self.issued[slot], self.err.data_ptr())
        self.issued[slot] += int(n_scenarios)
        return t

    def check(self):
        """Raise if a ticket wait timed out (the launch stored nothing)."""
        if int(self.err.item()) != 0:
            raise RuntimeError("overlapped launch: a slot ticket wait timed out (its records were not written)")


def plan_batch(dt: N.DeviceTables, scen_off, svc_table, svc_rate, svc_bound, optimize: bool = True,
               threshold: int = 4, cfg_format: int = CFG_FULL, stream=None,
               out: BatchResult | None = None, overlap: bool = False, ticket: N.SlotTicket | None = None,
               mirror=None) -> BatchResult:
    """Plan independent scenarios; scenario k owns services [scen_off[k], scen_off[k+1]).

    overlap=True launches the kernel as a programmatic dependent launch
    (parva_plan_batch_overlapped): it may start while the previous planning
    call on the stream is still running.  It needs the `ticket` of `out`'s
    slot (SlotRing.ticket): launches into one slot are serialized on the
    device.  mirror (an N.Mirror, from distributed.PeerGather.mirror) adds
    the fused all-gather (parva_plan_batch_fused); it carries its own ticket.
    A ticket is issued for exactly one launch of its n_scenarios."""
    torch = N.require_cuda()
    if overlap and mirror is None and ticket is None:
        raise ValueError("overlap=True needs the slot ticket of `out` (SlotRing.ticket)")
    if mirror is not None and dt.index_struct is None:
        raise ValueError("the fused all-gather needs tables small enough for the shared-memory index "
                         "(parva_plan_batch_preconfigured has no peer stores)")
    dev = lambda a, f: a if isinstance(a, torch.Tensor) else N.to_device(f(a))  # noqa: E731
    scen_off = dev(scen_off, _i32)
    svc_table = dev(svc_table, _i32)
    svc_rate = dev(svc_rate, _f64)
    svc_bound = dev(svc_bound, _f64)
    n_scen = int(scen_off.shape[0]) - 1
    n_svc = int(svc_table.shape[0])
    if dt.index_struct is None:
        cfg_format = CFG_FULL
    if out is None:
        plan_dt = PLAN64_DTYPE if mirror is not None and mirror.plan_bytes == 64 else PLAN_DTYPE
        out = BatchResult(N.empty_records(n_svc, _CFG_DT[cfg_format]),
                          N.empty_records(n_scen, plan_dt), n_scen, n_svc, cfg_format)
    s = N.stream_handle(stream)
    L = N.lib()
    if dt.index_struct is not None:
        args = (C.byref(dt.struct), C.byref(dt.index_struct), C.c_int32(n_scen), C.c_int32(n_svc), N.ptr(scen_off),
                N.ptr(svc_table), N.ptr(svc_rate), N.ptr(svc_bound), C.c_int32(int(optimize)),
                C.c_int32(int(threshold)), N.ptr(out.cfg), C.c_int32(out.cfg_format), N.ptr(out.plan))
        if mirror is not None:
            rc = L.parva_plan_batch_fused(*args, C.byref(mirror), s)
        elif overlap:
            rc = L.parva_plan_batch_overlapped(*args, C.byref(ticket), s)
        else:
            rc = L.parva_plan_batch(*args, s)
        N.check(rc, "parva_plan_batch")
    else:
        configure_sweep(dt, svc_table, svc_rate, svc_bound, out=out.cfg, stream=stream)
        rc = L.parva_plan_batch_preconfigured(C.byref(dt.struct), C.c_int32(n_scen), C.c_int32(n_svc), N.ptr(scen_off),
                                              N.ptr(svc_table), C.c_int32(int(optimize)), C.c_int32(int(threshold)),
                                              N.ptr(out.cfg), N.ptr(out.plan), s)
        N.check(rc, "parva_plan_batch_preconfigured")
    return out


# ----------------------------------------------------------------- general
@dataclass
class GeneralInput:
    """One allocator problem for the general kernel (see parva_general_problem).

    names: service ids first (n_services of them), then other ids that occur
    only in placements or the initial ledger."""

    names: list
    n_services: int
    cat_size: list = field(default_factory=list)
    cat_tp: list = field(default_factory=list)
    cat_name: list = field(default_factory=list)
    svc_t1: list = field(default_factory=list)
    svc_t2: list = field(default_factory=list)
    svc_opt: list = field(default_factory=list)
    svc_count: list = field(default_factory=list)
    svc_last: list = field(default_factory=list)
    svc_rate: list = field(default_factory=list)
    gpu_id: list = field(default_factory=list)
    pl_off: list = field(default_factory=lambda: [0])
    pl_cat: list = field(default_factory=list)
    pl_slot: list = field(default_factory=list)
    ledger_val: list = field(default_factory=list)
    ledger_order: list = field(default_factory=list)
    relocate: bool = False
    optimize: bool = False
    threshold: int = 4
    cat_key: list = field(default_factory=list)   # host-side decode key per catalogue entry

    def add_cat(self, size: int, tp: float, name: int, memo: dict, key) -> int:
        if key in memo:
            return memo[key]
        self.cat_size.append(size); self.cat_tp.append(tp); self.cat_name.append(name)
        self.cat_key.append(key)
        memo[key] = len(self.cat_size) - 1
        return memo[key]


@dataclass
class GeneralOutput:
    status: int
    gpu_id: np.ndarray
    pl_off: np.ndarray
    pl_cat: np.ndarray
    pl_slot: np.ndarray
    diags: list            # (reason, gpu id, name index)
    ledger_val: np.ndarray
    ledger_order: np.ndarray
    fallback: bool
    n_gpus_unopt: int


def plan_general(g: GeneralInput, stream=None) -> GeneralOutput:
    torch = N.require_cuda()
    n_names = max(len(g.names), 1)
    total_new = (int(np.asarray(g.svc_count, dtype=np.int64).sum()) +
                 int((np.asarray(g.svc_last, dtype=np.int64) >= 0).sum())) if g.relocate else 0
    gpu_cap = len(g.gpu_id) + total_new + 1
    place_cap = gpu_cap * 7
    diag_cap = gpu_cap + 1

    def d(a, dt, n=1):
        arr = np.asarray(a, dtype=dt) if len(a) else np.zeros(n, dtype=dt)
        return N.to_device(arr)

    cat_size = d(g.cat_size, np.uint8); cat_tp = d(g.cat_tp, np.float64); cat_name = d(g.cat_name, np.int32)
    svc_t1 = d(g.svc_t1, np.int32); svc_t2 = d(g.svc_t2, np.int32); svc_opt = d(g.svc_opt, np.int32)
    svc_count = d(g.svc_count, np.int64); svc_last = d(g.svc_last, np.int32); svc_rate = d(g.svc_rate, np.float64)
    gpu_id = d(g.gpu_id, np.int64); pl_off = d(g.pl_off, np.int32); pl_cat = d(g.pl_cat, np.int32)
    pl_slot = d(g.pl_slot, np.uint8)
    lv = np.zeros(n_names); lo = np.zeros(n_names, dtype=np.int32)
    lv[:len(g.ledger_val)] = g.ledger_val
    lo[:len(g.ledger_order)] = g.ledger_order
    ledger_val = N.to_device(lv); ledger_order = N.to_device(lo)
    P = N.GeneralProblem(len(g.cat_size), cat_size.data_ptr(), cat_tp.data_ptr(), cat_name.data_ptr(),
                         g.n_services, len(g.names), svc_t1.data_ptr(), svc_t2.data_ptr(), svc_opt.data_ptr(),
                         svc_count.data_ptr(), svc_last.data_ptr(), svc_rate.data_ptr(), len(g.gpu_id),
                         gpu_id.data_ptr(), pl_off.data_ptr(), pl_cat.data_ptr(), pl_slot.data_ptr(),
                         ledger_val.data_ptr(), ledger_order.data_ptr(), int(g.relocate), int(g.optimize),
                         int(g.threshold))
    o_status = torch.zeros(1, dtype=torch.int32, device="cuda")
    o_counts = torch.zeros(4, dtype=torch.int32, device="cuda")
    o_gid = torch.zeros(gpu_cap, dtype=torch.int64, device="cuda")
    o_off = torch.zeros(gpu_cap + 1, dtype=torch.int32, device="cuda")
    o_cat = torch.zeros(place_cap, dtype=torch.int32, device="cuda")
    o_slot = torch.zeros(place_cap, dtype=torch.uint8, device="cuda")
    o_diag = torch.zeros(diag_cap * 3, dtype=torch.int64, device="cuda")
    o_lv = torch.zeros(n_names, dtype=torch.float64, device="cuda")
    o_lo = torch.zeros(n_names, dtype=torch.int32, device="cuda")
    o_fb = torch.zeros(1, dtype=torch.int32, device="cuda")
    R = N.GeneralResult(gpu_cap, place_cap, diag_cap, o_status.data_ptr(), o_counts.data_ptr(), o_gid.data_ptr(),
                        o_off.data_ptr(), o_cat.data_ptr(), o_slot.data_ptr(), o_diag.data_ptr(), o_lv.data_ptr(),
                        o_lo.data_ptr(), o_fb.data_ptr())
    L = N.lib()
    ws_bytes = L.parva_plan_general_workspace(C.byref(P), C.c_int32(gpu_cap))
    ws = torch.empty(max(int(ws_bytes), 1), dtype=torch.uint8, device="cuda")
    N.check(L.parva_plan_general(C.byref(P), C.byref(R), N.ptr(ws), C.c_size_t(ws_bytes), N.stream_handle(stream)),
            "parva_plan_general")
    counts = o_counts.cpu().numpy()
    ng, npl, nd, nun = (int(x) for x in counts)
    diag = o_diag.cpu().numpy()[:3 * min(nd, diag_cap)].reshape(-1, 3)
    return GeneralOutput(
        status=int(o_status.item()), gpu_id=o_gid[:ng].cpu().numpy(), pl_off=o_off[:ng + 1].cpu().numpy(),
        pl_cat=o_cat[:npl].cpu().numpy(), pl_slot=o_slot[:npl].cpu().numpy(),
        diags=[tuple(int(v) for v in row) for row in diag], ledger_val=o_lv.cpu().numpy(),
        ledger_order=o_lo.cpu().numpy(), fallback=bool(o_fb.item()), n_gpus_unopt=nun)


def general_from_configs(pt: PackedTables, svc_table, cfg, optimize: bool, threshold: int) -> GeneralInput:
    """General problem for one scenario from its config records (CAPACITY path).

    Vectorized: the catalogue is every (service, size class) with a best
    point, in service-major order (the order the reference enqueues them)."""
    n = len(svc_table)
    t = np.asarray(svc_table, dtype=np.int64)
    best = np.asarray(cfg["best"], dtype=np.int64).reshape(n, 5)
    valid = best >= 0
    cat = np.where(valid, np.cumsum(valid.ravel()).reshape(n, 5) - 1, -1)
    s_idx, c_idx = np.nonzero(valid)
    pts = pt.seg_start.astype(np.int64)[t[s_idx] * 5 + c_idx] + best[s_idx, c_idx]
    sizes = np.array((1, 2, 3, 4, 7), dtype=np.uint8)
    rows = np.arange(n)
    opt = np.asarray(cfg["opt_sc"], dtype=np.int64)
    last = np.asarray(cfg["last_sc"], dtype=np.int64)
    return GeneralInput(
        names=list(range(n)), n_services=n, relocate=True, optimize=optimize, threshold=threshold,
        cat_size=sizes[c_idx], cat_tp=np.asarray(pt.tp, dtype=np.float64)[pts], cat_name=s_idx.astype(np.int32),
        svc_t1=cat[:, 0].astype(np.int32), svc_t2=cat[:, 1].astype(np.int32),
        svc_opt=np.where(opt >= 0, cat[rows, np.maximum(opt, 0)], -1).astype(np.int32),
        svc_count=np.asarray(cfg["count"], dtype=np.int64),
        svc_last=np.where(last >= 0, cat[rows, np.maximum(last, 0)], -1).astype(np.int32),
        svc_rate=np.zeros(n), cat_key=list(zip(s_idx.tolist(), c_idx.tolist())))


def resolve_capacity(pt: PackedTables, scen_off, svc_table, cfg, plan, optimize=True, threshold=4) -> dict:
    """Re-plan every PARVA_CAPACITY scenario with the general kernel.

    Returns {scenario index: (GeneralInput, GeneralOutput)}; config records
    are valid for all scenarios."""
    out = {}
    for k in np.nonzero(plan["status"] == CAPACITY)[0].tolist():
        a, b = int(scen_off[k]), int(scen_off[k + 1])
        recs = cfg[a:b]
        if (recs["status"] != 0).any():
            continue  # configuration error: reported from the config records
        g = general_from_configs(pt, svc_table[a:b], recs, optimize, threshold)
        out[k] = (g, plan_general(g))
    return out


# ------------------------------------------------------------ packed host
class ChunkLayout(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("in_scen_off", "in_rate", "in_bound", "in_table", "in_bytes",
                                         "out_plan", "out_cfg", "out_spill", "out_bytes")] + \
               [("plan_bytes", C.c_int32), ("spill_cap", C.c_int32)]


_CFG_DT = {CFG_FULL: CONFIG_DTYPE, CFG_COMPACT: COMPACT_DTYPE, CFG_TINY: TINY_DTYPE}


class PackedHostBatch:
    """A batch in the packed host format of parva_plan_host_packed.

    The scenarios are cut into `n_chunks` contiguous ranges; each chunk owns
    one pinned input block (offsets, rates, bounds, u16 table ids) and one
    pinned output block (plan records, then config records), so a chunk
    costs one H2D and one D2H copy.  `fill` packs inputs (host side, done
    once per batch by whoever produces the queries); `run` is the timed
    end-to-end call: copies in, plans, copies out, synchronizes."""

    def __init__(self, scen_off, svc_table, svc_rate, svc_bound, n_chunks: int = 2, cfg_format: int = CFG_COMPACT,
                 plan_bytes: int = 128):
        torch = N.require_cuda()
        L = N.lib()
        scen_off = np.asarray(scen_off, dtype=np.int64)
        n = len(scen_off) - 1
        n_chunks = max(1, min(n_chunks, max(n, 1)))
        self.cfg_format = cfg_format
        self.plan_bytes = plan_bytes
        self.bounds = [(n * c // n_chunks, n * (c + 1) // n_chunks) for c in range(n_chunks)]
        self.k = np.array([b - a for a, b in self.bounds], dtype=np.int32)
        self.m = np.array([scen_off[b] - scen_off[a] for a, b in self.bounds], dtype=np.int32)
        self.layouts, self.h_in, self.h_out = [], [], []
        for c, (a, b) in enumerate(self.bounds):
            lay = ChunkLayout()
            N.check(L.parva_packed_layout(C.c_int32(int(self.k[c])), C.c_int32(int(self.m[c])),
                                          C.c_int32(cfg_format), C.c_int32(plan_bytes), C.byref(lay)),
                    "parva_packed_layout")
            self.layouts.append(lay)
            self.h_in.append(torch.zeros(lay.in_bytes, dtype=torch.uint8).pin_memory())
            self.h_out.append(torch.zeros(lay.out_bytes, dtype=torch.uint8).pin_memory())
        self.n_scen, self.n_svc = n, int(scen_off[-1])
        self.fill(scen_off, svc_table, svc_rate, svc_bound)
        self.in_ptrs = (C.c_void_p * n_chunks)(*[t.data_ptr() for t in self.h_in])
        self.out_ptrs = (C.c_void_p * n_chunks)(*[t.data_ptr() for t in self.h_out])
        self.k_c = (C.c_int32 * n_chunks)(*self.k.tolist())
        self.m_c = (C.c_int32 * n_chunks)(*self.m.tolist())
        self.scratch_bytes = int(L.parva_plan_host_packed_scratch(C.c_int32(n_chunks), self.k_c, self.m_c,
                                                                 C.c_int32(cfg_format), C.c_int32(plan_bytes)))
        self.scratch = torch.empty(self.scratch_bytes, dtype=torch.uint8, device="cuda")

    def fill(self, scen_off, svc_table, svc_rate, svc_bound):
        scen_off = np.asarray(scen_off, dtype=np.int64)
        for c, (a, b) in enumerate(self.bounds):
            lay, buf = self.layouts[c], self.h_in[c].numpy()
            sa, sb = int(scen_off[a]), int(scen_off[b])
            k, m = b - a, sb - sa
            buf[lay.in_scen_off:lay.in_scen_off + 4 * (k + 1)].view(np.int32)[:] = scen_off[a:b + 1] - sa
            buf[lay.in_rate:lay.in_rate + 8 * m].view(np.float64)[:] = np.asarray(svc_rate)[sa:sb]
            buf[lay.in_bound:lay.in_bound + 8 * m].view(np.float64)[:] = np.asarray(svc_bound)[sa:sb]
            buf[lay.in_table:lay.in_table + 2 * m].view(np.uint16)[:] = np.asarray(svc_table)[sa:sb]

    def run(self, dt: N.DeviceTables, optimize: bool = True, threshold: int = 4, stream=None):
        rc = N.lib().parva_plan_host_packed(
            C.byref(dt.struct), C.byref(dt.index_struct), C.c_int32(len(self.bounds)), self.k_c, self.m_c,
            self.in_ptrs, self.out_ptrs, C.c_int32(int(optimize)), C.c_int32(int(threshold)),
            C.c_int32(self.cfg_format), C.c_int32(self.plan_bytes), N.ptr(self.scratch), C.c_size_t(self.scratch_bytes),
            N.stream_handle(stream))
        N.check(rc, "parva_plan_host_packed")

    @property
    def h2d_bytes(self) -> int:
        return int(sum(l.in_bytes for l in self.layouts))

    @property
    def d2h_bytes(self) -> int:
        return int(sum(l.out_bytes for l in self.layouts))

    def raw_outputs(self):
        """Per chunk: (config records, plan records as written, spill entries)."""
        cdt = _CFG_DT[self.cfg_format]
        pdt = PLAN64_DTYPE if self.plan_bytes == 64 else PLAN_DTYPE
        out = []
        for c, lay in enumerate(self.layouts):
            buf = self.h_out[c].numpy()
            k, m = int(self.k[c]), int(self.m[c])
            plan = buf[lay.out_plan:lay.out_plan + self.plan_bytes * k].view(pdt)
            cfg = buf[lay.out_cfg:lay.out_cfg + cdt.itemsize * m].view(cdt)
            spills = np.zeros(0, dtype=SPILL_DTYPE)
            if self.plan_bytes == 64:
                cnt = int(buf[lay.out_spill:lay.out_spill + 4].view(np.int32)[0])
                cnt = min(cnt, lay.spill_cap)
                spills = buf[lay.out_spill + 16:lay.out_spill + 16 + SPILL_DTYPE.itemsize * cnt].view(SPILL_DTYPE)
            out.append((cfg, plan, spills))
        return out

    def outputs(self):
        """(config records, 128-byte plan records) of the whole batch; 64-byte
        records are widened and spilled scenarios restored from the spill list."""
        cfgs, plans = [], []
        for cfg, plan, spills in self.raw_outputs():
            if self.plan_bytes == 64:
                wide = np.zeros(plan.shape[0], dtype=PLAN_DTYPE)
                wide.view(np.uint8).reshape(-1, 128)[:, :64] = plan.view(np.uint8).reshape(-1, 64)
                for e in spills:
                    wide[int(e["scenario"])] = e["record"]
                plan = wide
            cfgs.append(cfg)
            plans.append(plan)
        return np.concatenate(cfgs), np.concatenate(plans)


# ------------------------------------------------------------ mapped host
class MappedHostBatch:
    """Batches for the zero-copy host entry parva_plan_host_mapped (the
    end-to-end path).

    Per slot one pinned input block in the streamed layout (a chunk table,
    then one packed block per `chunk_scen` consecutive scenarios) and one
    pinned output block (plan records, config records, and for 64-byte plan
    records an overflow area of full records).  fill() packs a caller's
    plain arrays (scenario offsets, int32 table ids, rates, bounds -- any
    host memory) into a slot's input block on the library's host threads
    (parva_stream_pack_arrays).  Inside one kernel, loader warps stream the
    input block over PCIe in order while the other warps plan each scenario
    as soon as its chunk has landed and write its records straight into the
    output block; `run` is one launch plus a stream synchronize.

    depth > 1 keeps that many calls in flight (one input block, scratch and
    output block per slot): `submit(dt, slot)` enqueues a call without
    waiting, `wait(slot)` spins on its completion word; consecutive submits
    on a stream overlap (the next call's input stream starts while the
    previous call finishes planning).  Every batch must have the offsets'
    shape the object was built with (same scenario and service counts)."""

    def __init__(self, scen_off, svc_table, svc_rate, svc_bound, cfg_format: int = CFG_TINY, plan_bytes: int = 64,
                 chunk_scen: int = 32, depth: int = 1):
        torch = N.require_cuda()
        L = N.lib()
        scen_off = np.asarray(scen_off, dtype=np.int64)
        self.n_scen, self.n_svc = len(scen_off) - 1, int(scen_off[-1] - scen_off[0])
        self.cfg_format, self.plan_bytes, self.chunk_scen = cfg_format, plan_bytes, chunk_scen
        self.layout = ChunkLayout()
        N.check(L.parva_mapped_layout(C.c_int32(self.n_scen), C.c_int32(self.n_svc), C.c_int32(cfg_format),
                                      C.c_int32(plan_bytes), C.byref(self.layout)), "parva_mapped_layout")
        off32 = np.ascontiguousarray(scen_off - scen_off[0], dtype=np.int32)
        cap = int(L.parva_stream_bytes(C.c_int32(self.n_scen), N.np_ptr(off32), C.c_int32(chunk_scen)))
        if cap < 0:
            raise ValueError("invalid scenario offsets")
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.depth = depth
        self.in_capacity = cap              # upper bound; fill() records each slot's packed size
        self.in_sizes = [cap] * depth
        self.h_ins = [torch.zeros(max(cap, 256), dtype=torch.uint8).pin_memory() for _ in range(depth)]
        self.h_outs = [torch.zeros(max(self.layout.out_bytes, 256), dtype=torch.uint8).pin_memory()
                       for _ in range(depth)]
        self.scratch_bytes = int(L.parva_plan_host_mapped_scratch(C.c_int64(cap)))
        self.scratches = [torch.empty(self.scratch_bytes, dtype=torch.uint8, device="cuda") for _ in range(depth)]
        self._tickets = [0] * depth
        self._ticket = C.c_uint64(0)
        self._args = {}
        for slot in range(depth):
            self.fill(scen_off, svc_table, svc_rate, svc_bound, slot=slot)

    @property
    def h_in(self):
        return self.h_ins[0]

    @property
    def in_bytes(self):
        return self.in_sizes[0]

    @property
    def h_out(self):
        return self.h_outs[0]

    @property
    def scratch(self):
        return self.scratches[0]

    def fill(self, scen_off, svc_table, svc_rate, svc_bound, slot: int = 0, threads: int = 0):
        """Pack a batch into `slot`'s input block (the slot's previous call
        must have completed: wait(slot))."""
        if self._tickets[slot]:
            raise RuntimeError("fill(): the slot's previous call is still in flight (wait(slot) first)")
        scen_off = np.asarray(scen_off)
        sa = int(scen_off[0])
        if sa != 0 or scen_off.dtype != np.int32:
            scen_off = np.ascontiguousarray(scen_off - sa, dtype=np.int32)
        sb = sa + int(scen_off[-1])

        def arr(x, dt):
            x = np.asarray(x)
            if sa or len(x) != sb - sa:
                x = x[sa:sb]
            return x if x.dtype == dt and x.flags.c_contiguous else np.ascontiguousarray(x, dtype=dt)

        tab, rate, bound = arr(svc_table, np.int32), arr(svc_rate, np.float64), arr(svc_bound, np.float64)
        if len(scen_off) - 1 != self.n_scen or int(scen_off[-1]) != self.n_svc:
            raise ValueError("batch shape differs from the one this MappedHostBatch was built for")
        n = N.lib().parva_stream_pack_arrays(C.c_int32(self.n_scen), N.np_ptr(scen_off), N.np_ptr(tab),
                                             N.np_ptr(rate), N.np_ptr(bound), C.c_int32(self.chunk_scen),
                                             C.c_void_p(self.h_ins[slot].data_ptr()), C.c_int64(self.in_capacity),
                                             C.c_int32(threads))
        if n < 0:
            raise ValueError("parva_stream_pack_arrays failed (offsets not non-decreasing?)")
        self.in_sizes[slot] = int(n)    # chunks that repeat one table-id sequence store it once

    def _call_args(self, dt, optimize, threshold, stream, slot):
        sh = N.stream_handle(stream)
        key = (id(dt), bool(optimize), int(threshold), sh.value, slot, self.in_sizes[slot])
        hit = self._args.get(key)
        if hit is None:   # the argument tuple is built once per (tables, options, stream, slot, size)
            args = (C.byref(dt.struct), C.byref(dt.index_struct), C.c_int32(self.n_scen), C.c_int32(self.n_svc),
                    C.c_void_p(self.h_ins[slot].data_ptr()), C.c_int64(self.in_sizes[slot]),
                    C.c_void_p(self.h_outs[slot].data_ptr()), C.c_int32(int(optimize)), C.c_int32(int(threshold)),
                    C.c_int32(self.cfg_format), C.c_int32(self.plan_bytes), N.ptr(self.scratches[slot]),
                    C.c_size_t(self.scratch_bytes), sh)
            self._args[key] = (args, dt)
            return args
        return hit[0]

    def run(self, dt: N.DeviceTables, optimize: bool = True, threshold: int = 4, stream=None, slot: int = 0):
        """One synchronous call on `slot`."""
        self.wait(slot)
        N.check(N.lib().parva_plan_host_mapped(*self._call_args(dt, optimize, threshold, stream, slot)),
                "parva_plan_host_mapped")

    def submit(self, dt: N.DeviceTables, slot: int = 0, optimize: bool = True, threshold: int = 4, stream=None):
        """Enqueue a call on `slot` (its input block -> its output block); returns at once."""
        N.check(N.lib().parva_plan_host_mapped_submit(*self._call_args(dt, optimize, threshold, stream, slot),
                                                      C.byref(self._ticket)), "parva_plan_host_mapped_submit")
        self._tickets[slot] = self._ticket.value

    def submit_arrays(self, dt: N.DeviceTables, slot, scen_off, svc_table, svc_rate, svc_bound,
                      optimize: bool = True, threshold: int = 4, stream=None):
        """The e2e step in one C call (parva_plan_host_arrays_submit): wait
        for the slot's previous call, pack the plain arrays (int32 offsets
        starting at 0 and table ids, f64 rates and bounds -- any host memory,
        the shape this object was built for) into the slot's pinned block on
        the library's host threads, and submit.  Returns at once; wait(slot)
        before reading the slot's outputs."""
        for a, dt_ in ((scen_off, np.int32), (svc_table, np.int32), (svc_rate, np.float64), (svc_bound, np.float64)):
            if a.dtype != dt_ or not a.flags.c_contiguous:
                raise ValueError("submit_arrays: int32 / float64 C-contiguous arrays expected")
        if len(scen_off) != self.n_scen + 1 or len(svc_table) < self.n_svc:
            raise ValueError("batch shape differs from the one this MappedHostBatch was built for")
        key = ("arrays", id(dt), bool(optimize), int(threshold), slot, N.stream_handle(stream).value)
        hit = self._args.get(key)
        if hit is None:
            sh = N.stream_handle(stream)
            pre = (C.byref(dt.struct), C.byref(dt.index_struct), C.c_int32(self.n_scen))
            post = (C.c_int32(self.chunk_scen), C.c_void_p(self.h_ins[slot].data_ptr()), C.c_int64(self.in_capacity),
                    C.c_void_p(self.h_outs[slot].data_ptr()), C.c_int32(int(optimize)), C.c_int32(int(threshold)),
                    C.c_int32(self.cfg_format), C.c_int32(self.plan_bytes), N.ptr(self.scratches[slot]),
                    C.c_size_t(self.scratch_bytes), sh, C.byref(self._ticket))
            hit = self._args[key] = ((pre, post), dt)
        pre, post = hit[0]
        N.check(N.lib().parva_plan_host_arrays_submit(*pre, scen_off.ctypes.data, svc_table.ctypes.data,
                                                      svc_rate.ctypes.data, svc_bound.ctypes.data, *post),
                "parva_plan_host_arrays_submit")
        self._tickets[slot] = self._ticket.value

    def wait(self, slot: int = 0):
        """Wait until slot `slot`'s last submitted call has written its records."""
        t = self._tickets[slot]
        if t:
            self._tickets[slot] = 0
            N.check(N.lib().parva_plan_host_mapped_wait(C.c_uint64(t)), "parva_plan_host_mapped_wait")

    def stream(self, dt: N.DeviceTables, batches, consume=None, optimize: bool = True, threshold: int = 4,
               stream=None, threads: int = 0) -> int:
        """Plan an iterable of host batches (scen_off, table ids, rates, bounds)
        through the slots with a producer thread: while the calling thread
        submits batch i and waits for earlier ones, the producer packs batch
        i + 1 into a free slot (the pack and the waits release the GIL), so
        the host work of a step overlaps the GPU work of the steps in flight.
        depth - 1 calls are in flight, one slot is being packed.
        consume(i, slot), if given, runs after batch i's records have landed
        (read them with outputs(slot)) and before the slot is reused.
        Returns the number of batches planned."""
        import queue
        import threading
        if self.depth < 2:
            raise ValueError("stream() needs depth >= 2")
        for s in range(self.depth):
            self.wait(s)
        free, packed = queue.Queue(), queue.Queue()
        for s in range(self.depth):
            free.put(s)
        failure = []

        def produce():
            try:
                for i, b in enumerate(batches):
                    slot = free.get()
                    if slot is None:
                        return
                    self.fill(*b, slot=slot, threads=threads)
                    packed.put((i, slot))
            except BaseException as exc:  # noqa: BLE001 -- re-raised by the caller
                failure.append(exc)
            packed.put(None)

        th = threading.Thread(target=produce, daemon=True)
        th.start()
        inflight = []
        done = 0
        try:
            while True:
                item = packed.get()
                if item is None:
                    break
                self.submit(dt, item[1], optimize, threshold, stream)
                inflight.append(item)
                if len(inflight) == self.depth - 1:
                    i, slot = inflight.pop(0)
                    self.wait(slot)
                    if consume is not None:
                        consume(i, slot)
                    done += 1
                    free.put(slot)
            for i, slot in inflight:
                self.wait(slot)
                if consume is not None:
                    consume(i, slot)
                done += 1
        finally:
            free.put(None)
            th.join()
        if failure:
            raise failure[0]
        return done

    def __del__(self):
        try:
            for s in range(self.depth):
                self.wait(s)
            L = N.lib()
            for h in self.h_ins + self.h_outs:
                L.parva_forget_block(C.c_void_p(h.data_ptr()))
            for d in self.scratches:
                L.parva_forget_block(C.c_void_p(d.data_ptr()))
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass

    @property
    def h2d_bytes(self) -> int:
        """Bytes the kernel streams from the host input block per call (mean over slots)."""
        return int(sum(self.in_sizes) / len(self.in_sizes))

    @property
    def d2h_bytes(self) -> int:
        """Record bytes the kernel writes into the host output block per call
        (plan + config records; the overflow area only for spilled scenarios)."""
        lay = self.layout
        return int(lay.out_cfg + _CFG_DT[self.cfg_format].itemsize * self.n_svc)

    def outputs(self, slot: int = 0):
        """(config records, 128-byte plan records) of slot `slot`; spilled
        scenarios are restored from the overflow area."""
        lay, buf = self.layout, self.h_outs[slot].numpy()
        cdt = _CFG_DT[self.cfg_format]
        pdt = PLAN64_DTYPE if self.plan_bytes == 64 else PLAN_DTYPE
        k, m = self.n_scen, self.n_svc
        plan = buf[lay.out_plan:lay.out_plan + self.plan_bytes * k].view(pdt)
        cfg = buf[lay.out_cfg:lay.out_cfg + cdt.itemsize * m].view(cdt)
        if self.plan_bytes == 64:
            wide = np.zeros(k, dtype=PLAN_DTYPE)
            wide.view(np.uint8).reshape(-1, 128)[:, :64] = plan.view(np.uint8).reshape(-1, 64)
            sp = np.nonzero(plan["status"] == SPILLED)[0]
            if len(sp):
                full = buf[lay.out_spill:lay.out_spill + 128 * k].view(PLAN_DTYPE)
                wide[sp] = full[sp]
            plan = wide
        return cfg.copy(), plan
