#!/usr/bin/env python3
"""Development probe for K2 (plan_batch_kernel): builds a variant of the
library with -DPARVA_PHASE_TIMING into tools/_variants/ and prints per-CTA
phase times (index load, configure, plan) and per-warp finish times for the
C2 batch.  Not part of the product.

    python tools/k2_probe.py build        # here (nvcc)
    python tools/k2_probe.py run [n]      # on the GPU box
"""
import ctypes as C
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
OUT = REPO / "tools" / "_variants"
LIB = OUT / "libparva_phase.so"


def build(extra=()):
    from paper_2409_14447_b200 import build as b
    OUT.mkdir(parents=True, exist_ok=True)
    cmd = [b.NVCC, *[f for f in b.FLAGS if f not in ("-v", "-Xptxas")], "-DPARVA_PHASE_TIMING", *extra,
           "-o", str(LIB), *[str(b.CSRC / s) for s in b.SOURCES], "-lcudart"]
    subprocess.run(cmd, check=True)
    print("built", LIB)


def run(n=10_000, fmt=0):
    import numpy as np
    import torch
    from paper_2409_14447_b200 import _native as N
    N._LIB = None
    lib = C.CDLL(str(LIB))
    for name in N.EXPORTS:
        getattr(lib, name)
    for name in ("parva_plan_batch_workspace", "parva_plan_host_scratch", "parva_plan_general_workspace",
                 "parva_plan_host_packed_scratch"):
        getattr(lib, name).restype = C.c_size_t
    N._LIB = lib
    from paper_2409_14447_b200 import batch as B
    from paper_2409_14447_b200 import workloads as W
    sys.path.insert(0, str(REPO))
    from bench import c2_inputs
    fx = W.load_fixtures()
    dt = N.device_tables_for(fx.tables)
    off, tab, rate, bound = c2_inputs(fx, n, 0)
    d = [N.to_device(a) for a in (off, tab, rate, bound)]
    res = B.plan_batch(dt, *d, cfg_format=fmt)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        flush.zero_()
        B.plan_batch(dt, *d, out=res, cfg_format=fmt)
    torch.cuda.synchronize()
    flush.zero_()
    B.plan_batch(dt, *d, out=res, cfg_format=fmt)
    torch.cuda.synchronize()
    ph = np.zeros((1024, 4), dtype=np.uint64)
    we = np.zeros((1024, 16, 2), dtype=np.uint64)
    cyc = np.zeros((1024, 16, 4), dtype=np.uint64)
    lib.parva_dbg_phase(ph.ctypes.data_as(C.c_void_p), we.ctypes.data_as(C.c_void_p), cyc.ctypes.data_as(C.c_void_p))

    used = ph[:, 0] > 0
    ph = ph[used].astype(np.int64)
    we = we[used].astype(np.int64)
    t0 = ph[:, 0].min()
    rel = (ph - t0) / 1000.0
    print(f"CTAs {used.sum()}  kernel span {rel[:, 3].max():.2f} us")
    for i, name in enumerate(["start", "index", "configured", "end"]):
        c = rel[:, i]
        print(f"  {name:11s} min {c.min():7.2f}  p50 {np.median(c):7.2f}  max {c.max():7.2f} us")
    wend = (we[:, :, 0] - t0) / 1000.0
    wn = we[:, :, 1]
    print(f"  warp end    min {wend.min():7.2f}  p50 {np.median(wend):7.2f}  max {wend.max():7.2f} us")
    print(f"  scen/warp   hist {np.bincount(wn.ravel())}")
    plan_span = wend - rel[:, 2:3]
    print(f"  plan span per warp: p50 {np.median(plan_span):.2f} max {plan_span.max():.2f} us; "
          f"per scenario p50 {np.median(plan_span / np.maximum(wn, 1)):.2f} us")
    tot = cyc.sum(axis=(0, 1)).astype(np.float64) / (6.0 * n)
    print("  warp cycles per scenario: cfgload %.0f relocate %.0f optimize %.0f emit %.0f" % tuple(tot))


def run_mapped(n=10_000):
    """Streamed zero-copy entry: loader finish times vs warp finish times."""
    import numpy as np
    import torch
    from paper_2409_14447_b200 import _native as N
    lib = C.CDLL(str(LIB))
    for name in ("parva_plan_batch_workspace", "parva_plan_host_scratch", "parva_plan_general_workspace",
                 "parva_plan_host_packed_scratch", "parva_plan_host_mapped_scratch"):
        getattr(lib, name).restype = C.c_size_t
    lib.parva_stream_bytes.restype = C.c_int64
    lib.parva_stream_pack.restype = C.c_int64
    N._LIB = lib
    from paper_2409_14447_b200 import batch as B
    from paper_2409_14447_b200 import workloads as W
    from bench import c2_inputs
    fx = W.load_fixtures()
    dt = N.device_tables_for(fx.tables)
    off, tab, rate, bound = c2_inputs(fx, n, 0)
    mb = B.MappedHostBatch(off, tab, rate, bound, cfg_format=2, plan_bytes=64)
    for _ in range(10):
        mb.run(dt)
    torch.cuda.synchronize()
    ph = np.zeros((1024, 4), dtype=np.uint64)
    we = np.zeros((1024, 16, 2), dtype=np.uint64)
    cyc = np.zeros((1024, 16, 4), dtype=np.uint64)
    lib.parva_dbg_phase(ph.ctypes.data_as(C.c_void_p), we.ctypes.data_as(C.c_void_p), cyc.ctypes.data_as(C.c_void_p))
    used = ph[:, 0] > 0
    ph = ph[used].astype(np.int64)
    we = we[used].astype(np.int64)
    t0 = ph[:, 0].min()
    load_end = (ph[:, 1] - t0) / 1e3
    wend = (we[:, :, 0] - t0) / 1e3
    print(f"CTAs {used.sum()}  start spread {(ph[:, 0].max() - t0) / 1e3:.2f} us")
    print(f"  loader CTAs phase-1 end: min {load_end.min():.2f} p50 {np.median(load_end):.2f} max {load_end.max():.2f} us")
    pub = ph[:, 2][ph[:, 2] > 0]
    if pub.size:
        pub = (pub - t0) / 1e3
        print(f"  last slice published: min {pub.min():.2f} p50 {np.median(pub):.2f} max {pub.max():.2f} us")
    print(f"  warp end: min {wend.min():.2f} p50 {np.median(wend):.2f} p90 {np.percentile(wend, 90):.2f} max {wend.max():.2f} us")
    cy = cyc[used].astype(np.float64)
    nsc = cy[:, :, 3].sum()
    print(f"  per scenario (group cycles, 10 runs): locate+wait {cy[:, :, 0].sum() / nsc:.0f}  configure {cy[:, :, 1].sum() / nsc:.0f}"
          f"  plan {cy[:, :, 2].sum() / nsc:.0f}   scenarios counted {nsc:.0f}")


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    elif sys.argv[1] == "mapped":
        run_mapped(int(sys.argv[2]) if len(sys.argv) > 2 else 10_000)
    else:
        run(int(sys.argv[2]) if len(sys.argv) > 2 else 10_000, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
