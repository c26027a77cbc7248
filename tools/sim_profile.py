#!/usr/bin/env python3
"""cProfile of one batched run_simulations call (S6 x N seeds)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
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
pr = cProfile.Profile()
pr.enable()
S.run_simulations(jobs)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
