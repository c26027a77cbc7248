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
class PeerGather:
    """Gathered blocks in peer memory for the fused all-gather.

    Every rank allocates one exportable device buffer: a flag array (one u32
    per source rank) followed by `n_slots` gathered blocks of world x blk
    bytes (the packed_block layout, rank r's block at r * blk).  The CUDA IPC
    handles are exchanged with one all_gather_object, every process maps its
    peers' buffers, and K2 (parva_plan_batch_fused) stores each record into
    this rank's block of slot s on every rank while it plans, then raises its
    flag word on every rank to the launch's epoch.  wait(epoch) makes the
    stream wait until every rank's records of that epoch have landed here.
    One process per GPU (peers on other GPUs of the NVLink domain; the tests
    also run two processes on one GPU)."""

    FLAG_BYTES = 256

    def __init__(self, blk_bytes: int, n_slots: int = 3, group=None):
        import ctypes as C
        import torch
        import torch.distributed as dist
        self.torch = torch
        L = N.lib()
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        if self.world > 8:
            raise ValueError("the fused all-gather spans at most 8 ranks (one NVLink domain)")
        self.blk, self.n_slots = int(blk_bytes), int(n_slots)
        self.slot_bytes = self.world * self.blk
        size = self.FLAG_BYTES + self.n_slots * self.slot_bytes
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
        self.done = torch.zeros(self.n_slots, dtype=torch.int32, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.epoch = 0
        dist.barrier(group=group)

    def slot_view(self, slot: int):
        """This process's gathered block of `slot` as a uint8 tensor view
        (world x blk), for reading the results."""
        n = self.slot_bytes
        return _device_view(self.base + self.FLAG_BYTES + slot * n, n)

    def mirror(self, slot: int, ps: int, overlap: bool = False):
        """parva_mirror for a launch into `slot` (next epoch): this rank's
        plan / config sections on every rank."""
        import ctypes as C
        self.epoch += 1
        m = N.Mirror()
        m.n = self.world
        m.overlap = 1 if overlap else 0
        off = self.FLAG_BYTES + slot * self.slot_bytes + self.rank * self.blk
        for r, b in enumerate(self.peers):
            m.plan[r] = b + off
            m.cfg[r] = b + off + ps
            m.flag[r] = b + 4 * self.rank
        m.d_done = self.done.data_ptr() + 4 * slot
        m.epoch = self.epoch
        return m

    def wait(self, epoch: int | None = None, timeout_s: float = 60.0, stream=None):
        """Stream-ordered wait until every rank's flag reached `epoch` (default:
        the last launch's); raises later via check() if a peer timed out."""
        import ctypes as C
        e = self.epoch if epoch is None else int(epoch)
        N.check(N.lib().parva_gather_wait(C.c_void_p(self.base), C.c_int32(self.world), C.c_uint32(e),
                                          C.c_int64(int(timeout_s * 1e9)), N.ptr(self.status),
                                          N.stream_handle(stream)), "parva_gather_wait")

    def check(self):
        if int(self.status.item()) != 0:
            raise RuntimeError("fused all-gather: a peer's records did not arrive (timeout)")

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
