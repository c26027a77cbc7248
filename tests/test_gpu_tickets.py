"""Bounded overlap of parva_plan_batch_overlapped (parva_slot_ticket): the
launches that share an output slot are serialized on the device however
many programmatic dependent launches are in flight."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]


def _inputs(fx, n, seed):
    from paper_2409_14447_b200 import workloads as W
    sb = W.scenario_batch(fx, n, seed=seed)
    M = len(sb.models)
    off = np.arange(n + 1, dtype=np.int32) * M
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    return off, tab, sb.rate.ravel().copy(), sb.bound.ravel().copy()


def test_slow_first_launch_then_queued_launches_into_the_same_slots():
    """A long launch (200k scenarios) into slot 0, then 6 short overlapped
    launches alternating slots 1, 0, 1, 0, 1, 0 before any synchronization:
    the short launches into slot 0 write its first records while the long
    one may still be writing its tail.  The ticket makes them wait, so slot 0
    ends as [last short batch | rest of the long batch] exactly."""
    import oracle
    from paper_2409_14447_b200 import _native as N
    from paper_2409_14447_b200 import batch as B
    from paper_2409_14447_b200 import workloads as W
    from paper_2409_14447_b200.records import CFG_TINY, PLAN_DTYPE, TINY_DTYPE, tiny_config
    from paper_2409_14447_b200.tables import pack_tables
    fx = W.load_fixtures()
    dt = N.device_tables_for(fx.tables)
    pt = pack_tables(fx.tables)
    big = _inputs(fx, 200_000, 71)
    small = [_inputs(fx, 1_500 + 250 * j, 80 + j) for j in range(6)]
    nb, mb = 200_000, int(big[0][-1])
    outs = [B.BatchResult(N.empty_records(mb, TINY_DTYPE), N.empty_records(nb, PLAN_DTYPE), nb, mb, CFG_TINY)
            for _ in range(2)]
    ring = B.SlotRing(2)
    d_big = [N.to_device(a) for a in big]
    d_small = [[N.to_device(a) for a in s] for s in small]
    torch.cuda.synchronize()
    B.plan_batch(dt, *d_big, cfg_format=CFG_TINY, out=outs[0], overlap=True, ticket=ring.ticket(0, nb))
    for j in range(6):
        r = (j + 1) % 2
        k, m = len(small[j][0]) - 1, int(small[j][0][-1])
        view = B.BatchResult(outs[r].cfg[:m], outs[r].plan[:k], k, m, CFG_TINY)
        B.plan_batch(dt, *d_small[j], cfg_format=CFG_TINY, out=view, overlap=True, ticket=ring.ticket(r, k))
    torch.cuda.synchronize()
    ring.check()
    bc, bp = oracle.plan_batch_records(pt, *big)
    bc = tiny_config(bc)
    for r, j in ((0, 5), (1, 4)):
        sc, sp = oracle.plan_batch_records(pt, *small[j])
        sc = tiny_config(sc)
        cfg, plan = outs[r].host()
        k, m = len(small[j][0]) - 1, int(small[j][0][-1])
        assert plan[:k].tobytes() == sp.tobytes() and cfg[:m].tobytes() == sc.tobytes(), r
        if r == 0:   # the rest of slot 0 is the long batch's, untouched by the short launches
            assert plan[k:].tobytes() == bp[k:].tobytes() and cfg[m:].tobytes() == bc[m:].tobytes()


_TIMEOUT_CHILD = r"""
import numpy as np, torch, sys
sys.path.insert(0, sys.argv[1])
from paper_2409_14447_b200 import _native as N, batch as B, workloads as W
from paper_2409_14447_b200.records import CFG_TINY, PLAN_DTYPE, TINY_DTYPE
fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)
sb = W.scenario_batch(fx, 500, seed=3)
off = np.arange(501, dtype=np.int32) * 11
tab = np.tile(np.arange(11, dtype=np.int32), 500)
out = B.BatchResult(N.empty_records(5500, TINY_DTYPE), N.empty_records(500, PLAN_DTYPE), 500, 5500, CFG_TINY)
out.plan.fill_(0xAB)
ring = B.SlotRing(1)
bad = N.SlotTicket(ring.counts.data_ptr(), 7, ring.err.data_ptr())   # 7 scenarios never complete
B.plan_batch(dt, off, tab, sb.rate.ravel(), sb.bound.ravel(), cfg_format=CFG_TINY, out=out, overlap=True, ticket=bad)
torch.cuda.synchronize()
assert int(ring.err.item()) == 7, ring.err            # PARVA_LAUNCH_ERROR
assert bool((out.plan == 0xAB).all()), "a timed-out launch stored records"
assert int(ring.counts[0].item()) == 0                 # the slot's counter did not advance
ring.err.zero_()
B.plan_batch(dt, off, tab, sb.rate.ravel(), sb.bound.ravel(), cfg_format=CFG_TINY, out=out, overlap=True,
             ticket=ring.ticket(0, 500))
torch.cuda.synchronize()
ring.check()
assert int(ring.counts[0].item()) == 500
print("ok")
"""


def test_ticket_wait_times_out_without_storing():
    env = dict(os.environ, PARVA_TICKET_TIMEOUT_MS="300")
    r = subprocess.run([sys.executable, "-c", _TIMEOUT_CHILD, str(REPO)], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
