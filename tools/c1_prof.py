#!/usr/bin/env python3
"""Where the time of one small plan_scenario call goes (C1, S6): cProfile
of 200 calls through the public API (launch + synchronize + full decode)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_14447_b200 as P
from paper_2409_14447_b200 import workloads as W

fx = W.load_fixtures()
sc = P.Scenario("S6", tuple(P.scenario.ScenarioService(m, r, l) for m, r, l in fx.scenarios["S6"]))
for _ in range(20):
    res = P.plan_scenario(sc, fx.tables)
    res.services, res.deployment
t0 = time.perf_counter()
for _ in range(200):
    res = P.plan_scenario(sc, fx.tables)
    res.services, res.deployment
print(f"plan_scenario S6: {(time.perf_counter() - t0) / 200 * 1e6:.0f} us per call")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    res = P.plan_scenario(sc, fx.tables)
    res.services, res.deployment
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
