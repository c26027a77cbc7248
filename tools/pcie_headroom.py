#!/usr/bin/env python3
"""Is the e2e step bound by the PCIe link?  Run the bench's e2e pipeline
(parva_plan_host_arrays_submit, 5 calls in flight) alone, then again with an
extra copy-engine H2D (or D2H) copy of X MB per step on another stream.  If
the step time stays flat while the copy engine moves X more MB per step, the
link has headroom the zero-copy kernel does not use."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import c2_inputs  # noqa: E402
from paper_2409_14447_b200 import _native as N  # noqa: E402
from paper_2409_14447_b200 import batch as B  # noqa: E402
from paper_2409_14447_b200 import workloads as W  # noqa: E402

fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)
host = [c2_inputs(fx, 10_000, 0 if p == 0 else 1000 + p) for p in range(8)]
D = 5
mb = B.MappedHostBatch(*host[0], cfg_format=2, plan_bytes=64, depth=D)
side = torch.cuda.Stream()


def run(steps, extra_mb=0.0, direction="h2d"):
    n = int(extra_mb * 2**20)
    if n:
        h = torch.empty(n, dtype=torch.uint8).pin_memory()
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for i in range(steps):
        slot = i % D
        mb.submit_arrays(dt, slot, *host[i % 8])
        if n:
            with torch.cuda.stream(side):
                if direction == "h2d":
                    d.copy_(h, non_blocking=True)
                else:
                    h.copy_(d, non_blocking=True)
    for slot in range(D):
        mb.wait(slot)
    torch.cuda.synchronize()


for extra, dr in ((0.0, "h2d"), (0.5, "h2d"), (1.0, "h2d"), (2.0, "h2d"), (1.0, "d2h"), (2.0, "d2h"), (0.0, "h2d")):
    run(20, extra, dr)
    t0 = time.perf_counter()
    run(300, extra, dr)
    us = (time.perf_counter() - t0) / 300 * 1e6
    print(f"extra {dr} {extra:.1f} MB/step: {us:6.1f} us/step  (e2e {10_000 / us * 1e6:.3e} scenarios/s)")
