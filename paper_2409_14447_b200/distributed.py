"""Scenario sharding across GPUs: one process per GPU, torch.distributed.

Scenarios are independent, so a batch shards into contiguous
scenario blocks, one per rank, with no exchange during planning.  The only
collective is the gather of the fixed-size results at the end:
one all-gather of the 128-byte plan records and one of the 32-byte config
records, each padded to the largest shard so every rank contributes the
same byte count (NCCL over NVLink on the GPU box; gloo in the CPU tests).
`gather_packed` is the one-collective form the benchmark step uses: every
rank's plan records and 8-byte tiny config records in one block.

`plan_fn(off, tab, rate, bound) -> (cfg_u8[n_svc,32], plan_u8[n_scen,128])`
is the per-rank planner: batch.plan_batch on the GPU; the tests inject the
CPU oracle to check the sharding/gather logic without a GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [a, b) of n items for `rank` (sizes differ by at most 1)."""
    base, extra = divmod(n, world)
    a = rank * base + min(rank, extra)
    return a, a + base + (1 if rank < extra else 0)


@dataclass
class Shard:
    scen_a: int
    scen_b: int
    off: np.ndarray     # local scenario offsets (start at 0)
    svc_a: int
    svc_b: int


def make_shard(scen_off: np.ndarray, rank: int, world: int) -> Shard:
    n = len(scen_off) - 1
    a, b = shard_bounds(n, rank, world)
    sa, sb = int(scen_off[a]), int(scen_off[b])
    return Shard(a, b, (scen_off[a:b + 1] - sa).astype(np.int32), sa, sb)


def gather_records(local_cfg, local_plan, shard: Shard, scen_off, group=None, device=None):
    """All-gather padded per-rank record blocks and reassemble in global order.

    local_cfg / local_plan: torch uint8 tensors [n, 32] / [n, 128] on the
    collective's device.  Returns (cfg [N_svc, 32], plan [N_scen, 128]) as
    torch tensors on that device."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n_scen = len(scen_off) - 1
    sizes_s = [shard_bounds(n_scen, r, world) for r in range(world)]
    max_s = max(b - a for a, b in sizes_s)
    sizes_v = [(int(scen_off[a]), int(scen_off[b])) for a, b in sizes_s]
    max_v = max(b - a for a, b in sizes_v)
    dev = local_plan.device if device is None else device

    def padded(t, rows, width):
        out = torch.zeros((max(rows, 1), width), dtype=torch.uint8, device=dev)
        out[:t.shape[0]] = t
        return out

    pl = padded(local_plan[:shard.scen_b - shard.scen_a], max_s, 128)
    cf = padded(local_cfg[:shard.svc_b - shard.svc_a], max_v, 32)
    all_pl = torch.empty((world * max(max_s, 1), 128), dtype=torch.uint8, device=dev)
    all_cf = torch.empty((world * max(max_v, 1), 32), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(all_pl, pl, group=group)
    dist.all_gather_into_tensor(all_cf, cf, group=group)
    plan = torch.cat([all_pl[r * max(max_s, 1): r * max(max_s, 1) + (b - a)] for r, (a, b) in enumerate(sizes_s)])
    cfg = torch.cat([all_cf[r * max(max_v, 1): r * max(max_v, 1) + (b - a)] for r, (a, b) in enumerate(sizes_v)])
    return cfg, plan


def packed_block(scen_off, world: int, plan_bytes: int = 128, cfg_bytes: int = 8) -> tuple[int, int, int]:
    """Per-rank block of the packed gather: [plan records | config records],
    each section padded to the largest shard.  Returns (plan section bytes,
    config section bytes, block bytes)."""
    n_scen = len(scen_off) - 1
    spans = [shard_bounds(n_scen, r, world) for r in range(world)]
    max_s = max(max(b - a for a, b in spans), 1)
    max_v = max(max(int(scen_off[b]) - int(scen_off[a]) for a, b in spans), 1)
    ps = max_s * plan_bytes
    cs = (max_v * cfg_bytes + 15) & ~15
    return ps, cs, ps + cs


def gather_packed(block, scen_off, plan_bytes: int = 128, cfg_bytes: int = 8, group=None):
    """ONE all-gather of every rank's packed [plan | config] block (the only
    collective of a sharded step; 8-byte tiny config records keep it at
    ~216 B per scenario).  `block` is this rank's uint8 tensor of
    packed_block(...)[2] bytes, plan records first.  Returns (cfg, plan) in
    global scenario / service order as uint8 tensors [N_svc, cfg_bytes],
    [N_scen, plan_bytes]."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n_scen = len(scen_off) - 1
    ps, cs, blk = packed_block(scen_off, world, plan_bytes, cfg_bytes)
    everything = torch.empty(world * blk, dtype=torch.uint8, device=block.device)
    dist.all_gather_into_tensor(everything, block, group=group)
    rows = everything.view(world, blk)
    spans = [shard_bounds(n_scen, r, world) for r in range(world)]
    plans = [rows[r, :(b - a) * plan_bytes].view(-1, plan_bytes) for r, (a, b) in enumerate(spans)]
    cfgs = [rows[r, ps:ps + (int(scen_off[b]) - int(scen_off[a])) * cfg_bytes].view(-1, cfg_bytes)
            for r, (a, b) in enumerate(spans)]
    return torch.cat(cfgs), torch.cat(plans)


def plan_sharded(scen_off, svc_table, svc_rate, svc_bound, plan_fn, group=None, device=None):
    """Plan this rank's contiguous shard with plan_fn, then all-gather every
    rank's records.  All ranks return the full (cfg, plan) record arrays."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    scen_off = np.asarray(scen_off, dtype=np.int32)
    sh = make_shard(scen_off, rank, world)
    cfg, plan = plan_fn(sh.off, np.asarray(svc_table)[sh.svc_a:sh.svc_b],
                        np.asarray(svc_rate)[sh.svc_a:sh.svc_b], np.asarray(svc_bound)[sh.svc_a:sh.svc_b])
    return gather_records(cfg, plan, sh, scen_off, group=group, device=device)


# --------------------------------------------------- fused all-gather (peer memory)
@dataclass
class GatherLayout:
    """Per-rank part of a gathered slot: [plan section | config section |
    overflow section], each padded to the largest shard (16-byte aligned).
    plan_bytes 64: 64-byte plan records, a spilled scenario's full 128-byte
    record at the same index of the overflow section; 128: no overflow."""
    plan_bytes: int
    cfg_bytes: int
    ps: int
    cs: int
    os: int
    blk: int
    spans: list          # scenario span [a, b) of every rank
    svc_spans: list      # service span [sa, sb) of every rank


def gather_layout(scen_off, world: int, plan_bytes: int = 64, cfg_bytes: int = 8) -> GatherLayout:
    if plan_bytes not in (64, 128):
        raise ValueError("plan_bytes must be 64 or 128")
    n_scen = len(scen_off) - 1
    spans = [shard_bounds(n_scen, r, world) for r in range(world)]
    svc = [(int(scen_off[a]), int(scen_off[b])) for a, b in spans]
    max_s = max(max(b - a for a, b in spans), 1)
    max_v = max(max(b - a for a, b in svc), 1)
    ps = (max_s * plan_bytes + 15) & ~15
    cs = (max_v * cfg_bytes + 15) & ~15
    os_ = max_s * 128 if plan_bytes == 64 else 0
    return GatherLayout(plan_bytes, cfg_bytes, ps, cs, os_, ps + cs + os_, spans, svc)


def decode_gathered(rows: np.ndarray, lay: GatherLayout):
    """(config records [N_svc] (uint8 rows of cfg_bytes), 128-byte plan
    records [N_scen]) in global order from a gathered slot (uint8 [world,
    blk]); spilled 64-byte records are restored from the overflow section."""
    from .records import PLAN64_DTYPE, PLAN_DTYPE, SPILLED
    plans, cfgs = [], []
    for r, ((a, b), (sa, sb)) in enumerate(zip(lay.spans, lay.svc_spans)):
        k = b - a
        row = rows[r]
        if lay.plan_bytes == 128:
            plan = row[:k * 128].view(PLAN_DTYPE).copy()
        else:
            p64 = row[:k * 64].view(PLAN64_DTYPE)
            plan = np.zeros(k, dtype=PLAN_DTYPE)
            plan.view(np.uint8).reshape(-1, 128)[:, :64] = p64.view(np.uint8).reshape(-1, 64)
            sp = np.nonzero(p64["status"] == SPILLED)[0]
            if len(sp):
                full = row[lay.ps + lay.cs:lay.ps + lay.cs + 128 * k].view(PLAN_DTYPE)
                plan[sp] = full[sp]
        plans.append(plan)
        cfgs.append(row[lay.ps:lay.ps + (sb - sa) * lay.cfg_bytes].reshape(-1, lay.cfg_bytes).copy())
    return np.concatenate(cfgs), np.concatenate(plans)


class PeerGather:
    """Gathered slots in peer memory for the fused all-gather.

    Every rank allocates one exportable device buffer: a header (per slot a
    flag row -- rank r's last landed epoch -- an ack row -- rank r's last
    released epoch -- and the slot's ticket words), then `n_slots` slots of
    world x layout.blk bytes (rank r's part at r * blk).  The CUDA IPC
    handles are exchanged with one all_gather_object and every process maps
    its peers' buffers.  A launch into slot s (mirror(s), then
    batch.plan_batch(..., out=local(s), mirror=...)) plans this rank's shard
    straight into its own part of slot s and stores each tile's records into
    its part of slot s on every rank (K2, parva_plan_batch_fused); its CTAs
    first wait until every rank released the slot's previous epoch.
    wait(s) makes the stream wait until every rank's records of the slot's
    last epoch have landed here and releases the slot.  All ranks must call
    mirror() in the same order (the epochs agree).  One process per GPU
    (peers on other GPUs of the NVLink domain; the tests also run several
    processes on one GPU)."""

    def __init__(self, layout: GatherLayout, n_slots: int = 3, group=None):
        import ctypes as C
        import torch
        import torch.distributed as dist
        self.torch = torch
        L = N.lib()
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        if self.world > 8:
            raise ValueError("the fused all-gather spans at most 8 ranks (one NVLink domain)")
        if len(layout.spans) != self.world:
            raise ValueError("layout was built for another world size")
        self.layout, self.n_slots = layout, int(n_slots)
        self.blk = layout.blk
        self.slot_bytes = self.world * self.blk
        self.head = (80 * self.n_slots + 255) & ~255   # flags, acks (8 u32 each), CTA counter + u64 count
        size = self.head + self.n_slots * self.slot_bytes
        p = C.c_void_p()
        N.check(L.parva_ipc_alloc(C.c_size_t(size), C.byref(p)), "parva_ipc_alloc")
        self.base = p.value
        hb = int(L.parva_ipc_handle_bytes())
        h = (C.c_uint8 * hb)()
        N.check(L.parva_ipc_handle(C.c_void_p(self.base), h), "parva_ipc_handle")
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h), group=group)
        self.peers, self.opened = [], []
        for m, hm in enumerate(handles):
            if m == self.rank:
                self.peers.append(self.base)
                continue
            q = C.c_void_p()
            N.check(L.parva_ipc_open((C.c_uint8 * hb).from_buffer_copy(hm), C.byref(q)), "parva_ipc_open")
            self.peers.append(q.value)
            self.opened.append(q.value)
        self.status = torch.zeros(2, dtype=torch.int32, device="cuda")   # [0] gather waits, [1] tickets
        self.epoch = 0
        self.last = [0] * self.n_slots
        self.issued = [0] * self.n_slots
        dist.barrier(group=group)

    # header addresses
    def _flag(self, base, slot, r):
        return base + 4 * (8 * slot + r)

    def _ack(self, base, slot, r):
        return base + 32 * self.n_slots + 4 * (8 * slot + r)

    def _part(self, base, slot, r):
        return base + self.head + slot * self.slot_bytes + r * self.blk

    def slot_view(self, slot: int):
        """This process's gathered slot as a uint8 tensor view (world x blk)."""
        return _device_view(self._part(self.base, slot, 0), self.slot_bytes)

    def local(self, slot: int, cfg_format: int):
        """This rank's part of its own slot as the launch's output (a
        batch.BatchResult over the plan / config / overflow sections)."""
        from .batch import BatchResult
        lay = self.layout
        a, b = lay.spans[self.rank]
        sa, sb = lay.svc_spans[self.rank]
        part = self._part(self.base, slot, self.rank)
        if cfg_format != {8: 2, 16: 1, 32: 0}[lay.cfg_bytes]:
            raise ValueError("cfg_format does not match the layout's config record width")
        plan = _device_view(part, lay.ps).view(-1, lay.plan_bytes)
        cfg = _device_view(part + lay.ps, lay.cs)[:(sb - sa) * lay.cfg_bytes].view(-1, lay.cfg_bytes)
        spill = _device_view(part + lay.ps + lay.cs, lay.os).view(-1, 128) if lay.os else None
        return BatchResult(cfg, plan, b - a, sb - sa, cfg_format, spill)

    def mirror(self, slot: int, overlap: bool = False):
        """parva_mirror of the next launch into `slot` (the next epoch): this
        rank's sections of the slot on every rank, the slot's ack row and
        ticket."""
        lay = self.layout
        self.epoch = self.epoch % 0xFFFFFFFF + 1
        m = N.Mirror()
        m.n = self.world
        m.overlap = 1 if overlap else 0
        for r, b in enumerate(self.peers):
            part = self._part(b, slot, self.rank)
            m.plan[r] = part
            m.cfg[r] = part + lay.ps
            m.spill[r] = part + lay.ps + lay.cs if lay.os else None
            m.flag[r] = self._flag(b, slot, self.rank)
        m.d_acks = self._ack(self.base, slot, 0)
        m.d_done = self.base + 64 * self.n_slots + 4 * slot
        m.d_spill = self._part(self.base, slot, self.rank) + lay.ps + lay.cs if lay.os else None
        m.plan_capacity, m.cfg_capacity, m.spill_capacity = lay.ps, lay.cs, lay.os
        m.plan_bytes = lay.plan_bytes
        m.epoch, m.prev_epoch = self.epoch, self.last[slot]
        a, b = lay.spans[self.rank]
        cnt = self.base + 64 * self.n_slots + 4 * self.n_slots
        cnt = (cnt + 7) & ~7
        m.ticket = N.SlotTicket(cnt + 8 * slot, self.issued[slot], self.status.data_ptr() + 4)
        self.issued[slot] += b - a
        self.last[slot] = self.epoch
        return m

    def gather_slot(self, slot: int, pdl: bool = False):
        g = N.GatherSlot()
        g.n, g.pdl = self.world, 1 if pdl else 0
        g.d_flags = self._flag(self.base, slot, 0)
        for r, b in enumerate(self.peers):
            g.ack[r] = self._ack(b, slot, self.rank)
        return g

    def wait(self, slot: int, release: bool = True, pdl: bool = False, timeout_s: float = 60.0, stream=None,
             gslot=None):
        """Stream-ordered: wait until every rank's records of the slot's last
        epoch have landed here; release=True also releases the slot to every
        producer (nothing later on the stream may read it -- else call
        release() after the reader).  A timeout is reported by check()."""
        import ctypes as C
        g = gslot if gslot is not None else self.gather_slot(slot, pdl)
        N.check(N.lib().parva_gather_wait(C.byref(g), C.c_uint32(self.last[slot]), C.c_int32(int(release)),
                                          C.c_int64(int(timeout_s * 1e9)), N.ptr(self.status),
                                          N.stream_handle(stream)), "parva_gather_wait")

    def release(self, slot: int, stream=None):
        import ctypes as C
        g = self.gather_slot(slot)
        N.check(N.lib().parva_gather_release(C.byref(g), C.c_uint32(self.last[slot]), N.stream_handle(stream)),
                "parva_gather_release")

    def records(self, slot: int):
        """(config records, 128-byte plan records) of every rank in global order, from this process's copy."""
        rows = self.slot_view(slot).view(self.world, self.blk).cpu().numpy()
        return decode_gathered(rows, self.layout)

    def check(self):
        st = self.status.cpu().tolist()
        if st[0] != 0:
            raise RuntimeError("fused all-gather: a peer's records did not arrive (timeout)")
        if st[1] != 0:
            raise RuntimeError("fused all-gather: a slot was not released in time (its launch stored nothing)")

    def close(self):
        import ctypes as C
        L = N.lib()
        self.torch.cuda.synchronize()
        for q in self.opened:
            L.parva_ipc_close(C.c_void_p(q))
        self.opened = []
        if self.base:
            L.parva_ipc_free(C.c_void_p(self.base))
            self.base = 0


def _device_view(addr: int, nbytes: int):
    """uint8 CUDA tensor over raw device memory owned elsewhere (no copy)."""
    import torch

    class _Holder:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (addr, False), "version": 3}

    return torch.as_tensor(_Holder(), device="cuda")
