#!/usr/bin/env python3
"""Back-to-back K2 launches over rotating resident batches: plain stream
order vs programmatic dependent launches (parva_plan_batch_overlapped, three
rotating output blocks).  Span per step and parity of the last outputs.

    python tools/k2_overlap.py [n] [steps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from bench import c2_inputs
from paper_2409_14447_b200 import _native as N
from paper_2409_14447_b200 import batch as B
from paper_2409_14447_b200 import workloads as W
from paper_2409_14447_b200.records import CFG_TINY

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)
P = 64
batches = []
for p in range(P):
    off, tab, rate, bound = c2_inputs(fx, n, 0 if p == 0 else 1000 + p)
    batches.append(tuple(N.to_device(a) for a in (off, tab, rate, bound)))
R = 3
outs = [B.plan_batch(dt, *batches[0], cfg_format=CFG_TINY) for _ in range(R)]
expect = {}
for p in range(P):
    r = B.plan_batch(dt, *batches[p], cfg_format=CFG_TINY)
    expect[p] = (r.plan.cpu().numpy().tobytes(), r.cfg.cpu().numpy().tobytes())


def run(overlap, k):
    for i in range(k):
        B.plan_batch(dt, *batches[i % P], cfg_format=CFG_TINY, out=outs[i % R], overlap=overlap)


for overlap in (False, True, False, True):
    run(overlap, 20)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run(overlap, steps)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / steps
    ok = all((outs[i % R].plan.cpu().numpy().tobytes(), outs[i % R].cfg.cpu().numpy().tobytes()) == expect[i % P]
             for i in range(steps - R, steps))
    print(f"overlap={overlap!s:5}: {us:6.1f} us/step  {n / us * 1e6:.3e} scen/s  parity {ok}")
