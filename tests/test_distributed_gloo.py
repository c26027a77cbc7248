"""world_size-2 gloo test of the scenario-sharding + all-gather logic.

The per-rank planner is the CPU oracle here (the checker), so this runs
without a GPU; on the GPU box the same code path runs with batch.plan_batch
and NCCL (bench.py --gpus N)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_14447_b200.distributed import gather_packed, make_shard, packed_block, plan_sharded, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(n):
    from paper_2409_14447_b200 import workloads as W
    fx = W.load_fixtures()
    sb = W.scenario_batch(fx, n, seed=7)
    M = len(sb.models)
    off = np.arange(n + 1, dtype=np.int32) * M
    # ragged: drop the last service of every third scenario
    keep = np.ones(n * M, dtype=bool)
    keep[[k * M + M - 1 for k in range(0, n, 3)]] = False
    tab = np.tile(np.arange(M, dtype=np.int32), n)[keep]
    rate, bound = sb.rate.ravel()[keep], sb.bound.ravel()[keep]
    counts = np.full(n, M) - np.array([1 if k % 3 == 0 else 0 for k in range(n)])
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    return fx, off, tab, rate, bound


def _oracle_fn(fx):
    import oracle
    from paper_2409_14447_b200.tables import pack_tables
    pt = pack_tables(fx.tables)

    def fn(off, tab, rate, bound):
        cfg, plan = oracle.plan_batch_records(pt, off, tab, rate, bound, threads=1)
        return (torch.from_numpy(cfg.view(np.uint8).reshape(-1, 32).copy()),
                torch.from_numpy(plan.view(np.uint8).reshape(-1, 128).copy()))
    return fn


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fx, off, tab, rate, bound = _inputs(n)
        cfg, plan = plan_sharded(off, tab, rate, bound, _oracle_fn(fx))
        # the packed one-collective form: [plan records | tiny config records] per rank
        from paper_2409_14447_b200.records import tiny_config
        from paper_2409_14447_b200.records import CONFIG_DTYPE
        sh = make_shard(off, rank, world)
        lcfg, lplan = _oracle_fn(fx)(sh.off, tab[sh.svc_a:sh.svc_b], rate[sh.svc_a:sh.svc_b], bound[sh.svc_a:sh.svc_b])
        ps, cs, blk = packed_block(off, world)
        block = torch.zeros(blk, dtype=torch.uint8)
        block[:lplan.numel()] = lplan.reshape(-1)
        tiny = tiny_config(lcfg.numpy().reshape(-1).view(CONFIG_DTYPE)).view(np.uint8)
        block[ps:ps + tiny.shape[0]] = torch.from_numpy(tiny.copy())
        pcfg, pplan = gather_packed(block, off)
        q.put((rank, cfg.numpy().tobytes(), plan.numpy().tobytes(), pcfg.numpy().tobytes(), pplan.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover():
    for n in (0, 1, 7, 10, 101):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


@pytest.mark.parametrize("n", [37, 2])
def test_two_rank_gather_matches_single_process(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    fx, off, tab, rate, bound = _inputs(n)
    cfg, plan = _oracle_fn(fx)(off, tab, rate, bound)
    from paper_2409_14447_b200.records import CONFIG_DTYPE, tiny_config
    tiny = tiny_config(cfg.numpy().reshape(-1).view(CONFIG_DTYPE)).view(np.uint8)
    for rank, c, pl, pc, ppl in out:
        assert c == cfg.numpy().tobytes(), rank
        assert pl == plan.numpy().tobytes(), rank
        assert pc == tiny.tobytes(), rank
        assert ppl == plan.numpy().tobytes(), rank


def test_make_shard_offsets():
    off = np.array([0, 3, 3, 8, 9, 15], dtype=np.int32)
    sh = make_shard(off, 1, 2)
    assert (sh.scen_a, sh.scen_b) == (3, 5)
    assert sh.off.tolist() == [0, 1, 7] and (sh.svc_a, sh.svc_b) == (8, 15)
