"""Fused all-gather (parva_plan_batch_fused + PeerGather): K2
stores every tile's records into this rank's part of a slot on every rank
over CUDA-IPC mapped peer memory, then raises its flag word of the slot on
every rank; consumers wait for the exact epoch and release the slot.
Checked end to end against the oracle, in one process (world 1) and with
two processes sharing the one GPU (real IPC mappings between processes; on
a multi-GPU box the same mappings are NVLink peer memory):
  * several fused launches in flight before any wait (one slot each),
  * slot reuse across ranks (tickets + acks: a producer never overwrites a
    slot a peer has not released),
  * 64-byte plan records with the overflow section, and 128-byte records."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(fx, n, seed):
    from paper_2409_14447_b200 import workloads as W
    sb = W.scenario_batch(fx, n, seed=seed)
    M = len(sb.models)
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    return off, tab, sb.rate.ravel().copy(), sb.bound.ravel().copy()


def _run_rank(rank, world, port, n, seeds, plan_bytes, n_slots):
    import torch.distributed as dist

    import oracle
    from paper_2409_14447_b200 import _native as N
    from paper_2409_14447_b200 import batch as B
    from paper_2409_14447_b200 import distributed as D
    from paper_2409_14447_b200 import workloads as W
    from paper_2409_14447_b200.records import CFG_TINY, tiny_config
    from paper_2409_14447_b200.tables import pack_tables
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        fx = W.load_fixtures()
        dt = N.device_tables_for(fx.tables)
        pt = pack_tables(fx.tables)
        off0 = _batch(fx, n, seeds[0])[0]
        lay = D.gather_layout(off0, world, plan_bytes=plan_bytes, cfg_bytes=8)
        pg = D.PeerGather(lay, n_slots=n_slots)
        pending = []                       # (slot, seed) launched, not yet checked
        keep = []                          # launch inputs stay alive until the end
        n_spilled = 0

        def check(slot, seed):
            nonlocal n_spilled
            pg.wait(slot, release=False)
            torch.cuda.synchronize()
            pg.check()
            cfg, plan = pg.records(slot)
            off, tab, rate, bound = _batch(fx, n, seed)
            ocfg, oplan = oracle.plan_batch_records(pt, off, tab, rate, bound)
            assert plan.tobytes() == oplan.tobytes(), (rank, slot, seed)
            assert cfg.tobytes() == tiny_config(ocfg).tobytes(), (rank, slot, seed)
            a, b = lay.spans[rank]
            lc, lp = pg.local(slot, CFG_TINY).host()
            assert lp.tobytes() == oplan[a:b].tobytes(), (rank, slot, seed)
            if plan_bytes == 64:
                p64 = pg.slot_view(slot).view(world, lay.blk).cpu().numpy()
                n_spilled += int(sum((p64[r, :(y - x) * 64:64] == 8).sum() for r, (x, y) in enumerate(lay.spans)))
            pg.release(slot)           # a peer may now reuse the slot

        for step, seed in enumerate(seeds):
            off, tab, rate, bound = _batch(fx, n, seed)
            sh = D.make_shard(off, rank, world)
            ins = [N.to_device(a) for a in (sh.off, tab[sh.svc_a:sh.svc_b], rate[sh.svc_a:sh.svc_b],
                                            bound[sh.svc_a:sh.svc_b])]
            slot = step % n_slots
            if len(pending) == n_slots:    # every slot is in flight: check them all, then reuse
                for s_, sd in pending:
                    check(s_, sd)
                pending = []
            B.plan_batch(dt, *ins, cfg_format=CFG_TINY, out=pg.local(slot, CFG_TINY),
                         mirror=pg.mirror(slot, overlap=step > 0))
            pending.append((slot, seed))
            keep.append(ins)
        for s_, sd in pending:
            check(s_, sd)
        if plan_bytes == 64:
            assert n_spilled > 0           # the overflow section was exercised
        pg.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("plan_bytes", [64, 128])
def test_fused_gather_one_rank(plan_bytes):
    _run_rank(0, 1, _free_port(), 3_001, [5, 6, 7, 8, 9, 10, 11, 12, 13], plan_bytes, 4)


@pytest.mark.parametrize("plan_bytes", [64, 128])
def test_fused_gather_two_processes_one_gpu(plan_bytes):
    import torch.multiprocessing as mp
    mp.spawn(_run_rank, args=(2, _free_port(), 2_501, list(range(11, 22)), plan_bytes, 5), nprocs=2, join=True)
