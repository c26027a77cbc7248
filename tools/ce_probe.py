#!/usr/bin/env python3
"""Copy-engine e2e pipeline probe: per step H2D of a C2-sized input block,
(optionally) one K2 launch on the slot's stream, D2H of the records; D slots
on D streams, the host waits on the slot's event before reusing it.
Prints us/step for copies only, copies + K2, and with a host pack (np.copyto)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_14447_b200 import _native as N  # noqa: E402
from paper_2409_14447_b200 import batch as B  # noqa: E402
from paper_2409_14447_b200 import workloads as W  # noqa: E402
from paper_2409_14447_b200.records import CFG_TINY  # noqa: E402

fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)
n = 10_000
sb = W.scenario_batch(fx, n, seed=0)
M = sb.rate.shape[1]
off = np.arange(n + 1, dtype=np.int32) * M
tab = np.tile(np.arange(M, dtype=np.int32), n)
rate, bound = sb.rate.ravel().copy(), sb.bound.ravel().copy()
IN = [off, tab, rate, bound]
in_bytes = sum(a.nbytes for a in IN)


def run(D, steps, kernel, pack, in_mb=None, out_mb=None):
    streams = [torch.cuda.Stream() for _ in range(D)]
    ev = [None] * D
    hin = [[torch.from_numpy(a.copy()).pin_memory() for a in IN] for _ in range(D)]
    din = [[torch.empty_like(h, device="cuda") for h in hs] for hs in hin]
    res = [B.plan_batch(dt, *[d for d in ds], cfg_format=CFG_TINY) for ds in din]
    torch.cuda.synchronize()
    hout = [(torch.empty(r.cfg.numel(), dtype=torch.uint8).pin_memory(),
             torch.empty(r.plan.numel(), dtype=torch.uint8).pin_memory()) for r in res]
    if in_mb:   # raw copy sizes instead
        hin = [[torch.empty(int(in_mb * 2**20), dtype=torch.uint8).pin_memory()] for _ in range(D)]
        din = [[torch.empty_like(h[0], device="cuda")] for h in hin]
    if out_mb:
        hout = [(torch.empty(int(out_mb * 2**20), dtype=torch.uint8).pin_memory(),) for _ in range(D)]
        dout = [torch.empty(int(out_mb * 2**20), dtype=torch.uint8, device="cuda") for _ in range(D)]

    def step(i):
        s = i % D
        if ev[s] is not None:
            ev[s].synchronize()
        if pack and not in_mb:
            for h, a in zip(hin[s], IN):
                np.copyto(h.numpy(), a)
        with torch.cuda.stream(streams[s]):
            for d, h in zip(din[s], hin[s]):
                d.copy_(h, non_blocking=True)
            if kernel:
                B.plan_batch(dt, *din[s], cfg_format=CFG_TINY, out=res[s], stream=streams[s])
            if out_mb:
                hout[s][0].copy_(dout[s], non_blocking=True)
            else:
                hout[s][0].copy_(res[s].cfg, non_blocking=True)
                hout[s][1].copy_(res[s].plan, non_blocking=True)
            e = torch.cuda.Event()
            e.record(streams[s])
            ev[s] = e
    for i in range(2 * D):
        step(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        step(i)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps * 1e6


print(f"input {in_bytes / 1e6:.2f} MB, output {(10_000 * 128 + M * n * 8) / 1e6:.2f} MB per step")
for mb_in, mb_out in ((2.0, 1.5), (2.0, 0.01), (0.01, 1.5)):
    for D in (3, 6):
        print(f"raw copies in {mb_in} MB out {mb_out} MB D={D}: {run(D, 300, False, False, mb_in, mb_out):.1f} us/step")
for D in (3, 4, 6, 8):
    print(f"D={D}: copies {run(D, 300, False, False):.1f}  +K2 {run(D, 300, True, False):.1f}  "
          f"+K2+pack {run(D, 300, True, True):.1f} us/step")
for D in (4,):
    for steps in (20, 200):
        print(f"D={D} steps {steps}: +K2+pack {run(D, steps, True, True):.1f} us/step")
