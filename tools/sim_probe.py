#!/usr/bin/env python3
"""Where does batched run_simulations time go?  host prep (seeding),
GPU kernel, gather, host statistics."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2409_14447_b200 as P
from paper_2409_14447_b200 import simulation as S
from paper_2409_14447_b200 import workloads as W

fx = W.load_fixtures()
sc = P.Scenario("S6", tuple(P.scenario.ScenarioService(m, r, l) for m, r, l in fx.scenarios["S6"]))
res = P.plan_scenario(sc, fx.tables)
services = list(res.services)
wl = S.Workload.from_services(services)
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 256
jobs = [S.SimJob(res.deployment, fx.tables, services, wl, 10.0, seed) for seed in range(runs)]
S.run_simulations(jobs[:4])
t0 = time.perf_counter()
preps = S._prepare_all(jobs)
t1 = time.perf_counter()
print(f"host prep (seeding, {sum(len(p.ids) for p in preps)} services): {(t1 - t0) * 1e3:.1f} ms")
orig = S._report
tr = [0.0]


def timed_report(*a, **k):
    s = time.perf_counter()
    r = orig(*a, **k)
    tr[0] += time.perf_counter() - s
    return r


S._report = timed_report
ev = [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
_lib = S.N.lib


class _Timed:
    def __getattr__(self, k):
        return getattr(_lib(), k)

    def parva_simulate(self, *a):
        ev[0].record()
        r = _lib().parva_simulate(*a)
        ev[1].record()
        return r


S.N.lib = lambda: _Timed()
s = torch.cuda.current_stream()
t0 = time.perf_counter()
S.run_simulations(jobs)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"run_simulations total {(t1 - t0) * 1e3:.1f} ms, of which host stats {tr[0] * 1e3:.1f} ms, "
      f"simulate kernel {ev[0].elapsed_time(ev[1]):.1f} ms")
