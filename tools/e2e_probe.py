#!/usr/bin/env python3
"""Breakdown of the host-buffer path: H2D / kernel / D2H times and the
pipelined parva_plan_host, for the C2 batch (1 GPU)."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2409_14447_b200 import _native as N
from paper_2409_14447_b200 import batch as B
from paper_2409_14447_b200 import workloads as W

fx = W.load_fixtures()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
sb = W.scenario_batch(fx, n, seed=0)
M = 11
off = np.arange(n + 1, dtype=np.int32) * M
tab = np.tile(np.arange(M, dtype=np.int32), n)
rate, bound = sb.rate.ravel().copy(), sb.bound.ravel().copy()
dt = N.device_tables_for(fx.tables)
L = N.lib()
pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
h_off, h_tab, h_rate, h_bound = pin(off), pin(tab), pin(rate), pin(bound)
h_cfg = torch.empty((n * M, 16), dtype=torch.uint8).pin_memory()
h_plan = torch.empty((n, 128), dtype=torch.uint8).pin_memory()
d_off, d_tab, d_rate, d_bound = (torch.empty_like(x, device="cuda") for x in (h_off, h_tab, h_rate, h_bound))
res = B.plan_batch(dt, d_off.copy_(h_off), d_tab.copy_(h_tab), d_rate.copy_(h_rate), d_bound.copy_(h_bound),
                   cfg_format=1)
torch.cuda.synchronize()


def timeit(f, reps=50):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e6


def h2d():
    d_off.copy_(h_off, non_blocking=True); d_tab.copy_(h_tab, non_blocking=True)
    d_rate.copy_(h_rate, non_blocking=True); d_bound.copy_(h_bound, non_blocking=True)


def d2h():
    h_cfg.copy_(res.cfg[:n * M], non_blocking=True); h_plan.copy_(res.plan[:n], non_blocking=True)


def kern():
    B.plan_batch(dt, d_off, d_tab, d_rate, d_bound, cfg_format=1, out=res)


def serial():
    h2d(); kern(); d2h(); torch.cuda.synchronize()


nb = int(L.parva_plan_host_scratch(C.c_int32(n), C.c_int32(n * M)))
scratch = torch.empty(nb, dtype=torch.uint8, device="cuda")


def host():
    rc = L.parva_plan_host(C.byref(dt.struct), C.byref(dt.index_struct), C.c_int32(n), N.ptr(h_off), N.ptr(h_tab),
                           N.ptr(h_rate), N.ptr(h_bound), C.c_int32(1), C.c_int32(4), N.ptr(h_cfg), C.c_int32(1),
                           N.ptr(h_plan), N.ptr(scratch), C.c_size_t(nb), N.stream_handle())
    assert rc == 0


ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
devt = []
for _ in range(30):
    ev0.record(); host(); ev1.record(); torch.cuda.synchronize(); devt.append(ev0.elapsed_time(ev1) * 1000)
print(f"parva_plan_host device-timeline (events) median {sorted(devt)[15]:.1f} us")
for chunks in (1, 2, 3, 4, 6):
    pb = B.PackedHostBatch(off, tab, rate, bound, n_chunks=chunks)
    f = lambda: pb.run(dt)  # noqa: E731
    print(f"packed chunks={chunks}: {timeit(f):.1f} us  (h2d {pb.h2d_bytes} B, d2h {pb.d2h_bytes} B)")
print(f"n={n}: h2d {timeit(h2d):.1f} us  kernel {timeit(kern):.1f} us  d2h {timeit(d2h):.1f} us  "
      f"serial {timeit(serial):.1f} us  parva_plan_host {timeit(host):.1f} us")
