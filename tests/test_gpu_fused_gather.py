"""Fused all-gather (parva_plan_batch_fused + PeerGather): K2 stores every
record into this rank's slot of every rank's gathered block over CUDA-IPC
mapped peer memory and raises its flag on every rank.  Checked end to end
against the oracle: in one process (world 1) and with two processes sharing
the one GPU (real IPC mappings between processes; on a multi-GPU box the
same mappings are NVLink peer memory)."""

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


def _run_rank(rank, world, port, n, seeds):
    import torch.distributed as dist

    import oracle
    from paper_2409_14447_b200 import _native as N
    from paper_2409_14447_b200 import batch as B
    from paper_2409_14447_b200 import distributed as D
    from paper_2409_14447_b200 import workloads as W
    from paper_2409_14447_b200.records import CFG_TINY, PLAN_DTYPE, TINY_DTYPE, tiny_config
    from paper_2409_14447_b200.tables import pack_tables
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        fx = W.load_fixtures()
        dt = N.device_tables_for(fx.tables)
        pt = pack_tables(fx.tables)
        off0 = _batch(fx, n, seeds[0])[0]
        ps, cs, blk = D.packed_block(off0, world)
        pg = D.PeerGather(blk, n_slots=3)
        spans = [D.shard_bounds(n, r, world) for r in range(world)]
        for step, seed in enumerate(seeds):
            off, tab, rate, bound = _batch(fx, n, seed)
            sh = D.make_shard(off, rank, world)
            ins = [N.to_device(a) for a in (sh.off, tab[sh.svc_a:sh.svc_b], rate[sh.svc_a:sh.svc_b],
                                            bound[sh.svc_a:sh.svc_b])]
            slot = step % 3
            local = B.plan_batch(dt, *ins, cfg_format=CFG_TINY, mirror=pg.mirror(slot, ps, overlap=step > 0))
            pg.wait()
            torch.cuda.synchronize()
            pg.check()
            rows = pg.slot_view(slot).view(world, blk).cpu().numpy()
            plan = np.concatenate([rows[r, :(b - a) * 128].view(PLAN_DTYPE) for r, (a, b) in enumerate(spans)])
            cfg = np.concatenate([rows[r, ps:ps + (int(off[b]) - int(off[a])) * 8].view(TINY_DTYPE)
                                  for r, (a, b) in enumerate(spans)])
            ocfg, oplan = oracle.plan_batch_records(pt, off, tab, rate, bound)
            assert plan.tobytes() == oplan.tobytes(), (rank, step)
            assert cfg.tobytes() == tiny_config(ocfg).tobytes(), (rank, step)
            lc, lp = local.host()
            a, b = spans[rank]
            assert lp.tobytes() == oplan[a:b].tobytes(), (rank, step)
            dist.barrier()             # every rank has read this slot before it is rewritten
        pg.close()
    finally:
        dist.destroy_process_group()


def test_fused_gather_one_rank():
    _run_rank(0, 1, _free_port(), 3_001, [5, 6, 7, 8])


def test_fused_gather_two_processes_one_gpu():
    import torch.multiprocessing as mp
    mp.spawn(_run_rank, args=(2, _free_port(), 2_501, [11, 12, 13, 14, 15]), nprocs=2, join=True)
