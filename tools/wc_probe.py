#!/usr/bin/env python3
"""Write-combined vs cached pinned input blocks for the e2e path, A/B inside
one process (the e2e level differs between processes on the GPU box): the
bench's e2e loop (parva_plan_host_arrays_submit, 5 calls in flight) over the
same C2 batches with the slots' input blocks in (a) torch pinned memory,
(b) cudaHostAlloc(WriteCombined | Mapped | Portable) memory, alternating."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from cuda.bindings import runtime as rt  # noqa: E402

from bench import c2_inputs  # noqa: E402
from paper_2409_14447_b200 import _native as N  # noqa: E402
from paper_2409_14447_b200 import batch as B  # noqa: E402
from paper_2409_14447_b200 import workloads as W  # noqa: E402


class HostBlock:
    """cudaHostAlloc'd bytes with the two methods MappedHostBatch uses."""

    def __init__(self, n, flags):
        err, self.p = rt.cudaHostAlloc(n, flags)
        assert err == rt.cudaError_t.cudaSuccess, err
        self.n = n

    def data_ptr(self):
        return int(self.p)

    def numpy(self):
        return np.ctypeslib.as_array((C.c_uint8 * self.n).from_address(int(self.p)))


fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)
host = [c2_inputs(fx, 10_000, 0 if p == 0 else 1000 + p) for p in range(8)]
D = 5
mb = B.MappedHostBatch(*host[0], cfg_format=2, plan_bytes=64, depth=D)
cached = list(mb.h_ins)
flags = rt.cudaHostAllocWriteCombined | rt.cudaHostAllocMapped | rt.cudaHostAllocPortable
wc = [HostBlock(b.numel(), flags) for b in cached]


def loop(a, k):
    for i in range(a, a + k):
        mb.submit_arrays(dt, i % D, *host[i % 8])
    for s in range(D):
        mb.wait(s)


def span(bufs, steps=300):
    mb.h_ins[:] = bufs
    loop(0, 2 * D)
    t0 = time.perf_counter()
    loop(0, steps)
    return (time.perf_counter() - t0) / steps * 1e6


res = {"cached": [], "wc": []}
for rep in range(6):
    res["cached"].append(span(cached))
    res["wc"].append(span(wc))
for k, v in res.items():
    print(f"{k:7s} us/step: " + " ".join(f"{x:5.1f}" for x in v) + f"   median {np.median(v):5.1f}  "
          f"-> {1e10 / np.median(v) / 1e6:.3e} scenarios/s")
# records still right with WC inputs
import oracle  # noqa: E402
from paper_2409_14447_b200.records import tiny_config  # noqa: E402
from paper_2409_14447_b200.tables import pack_tables  # noqa: E402
mb.h_ins[:] = wc
loop(0, D)
ok = True
for s in range(D):
    ocfg, oplan = oracle.plan_batch_records(pack_tables(fx.tables), *host[s])
    cfg, plan = mb.outputs(s)
    ok = ok and plan.tobytes() == oplan.tobytes() and cfg.tobytes() == tiny_config(ocfg).tobytes()
print("records equal oracle with WC inputs:", ok)
mb.h_ins[:] = cached
