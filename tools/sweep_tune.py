#!/usr/bin/env python3
"""Tuning harness for the K1 sweep: build variants (warps, chunk, stages) of
the library into tools/_variants/ and time configure_sweep on C3 with each.

    python tools/sweep_tune.py build      # here (nvcc)
    python tools/sweep_tune.py run        # on the GPU box
"""
import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
OUT = REPO / "tools" / "_variants"
VARIANTS = [(12, 384, 3), (9, 512, 3), (14, 256, 4), (7, 512, 4), (6, 768, 3), (18, 256, 3), (24, 192, 3),
            (6, 384, 3), (8, 256, 3), (4, 512, 3)]


def build():
    from paper_2409_14447_b200 import build as b
    OUT.mkdir(parents=True, exist_ok=True)
    for w, ch, st in VARIANTS:
        lib = OUT / f"lib_{w}_{ch}_{st}.so"
        cmd = [b.NVCC, *[f for f in b.FLAGS if f != "-v" and f != "-Xptxas"], f"-DPARVA_SW_WARPS={w}",
               f"-DPARVA_SW_CH={ch}", f"-DPARVA_SW_STAGES={st}", "-o", str(lib),
               *[str(b.CSRC / s) for s in b.SOURCES], "-lcudart"]
        subprocess.run(cmd, check=True)
        print("built", lib.name)


def run():
    import numpy as np
    import torch
    from paper_2409_14447_b200 import _native as N
    from paper_2409_14447_b200 import workloads as W
    from paper_2409_14447_b200.tables import pack_dense
    dth = W.dense_tables(10_000, seed=3)
    pt = pack_dense(dth)
    dt = N.DeviceTables(pt, build_index=False)
    nq = dth.n_workloads
    qt = N.to_device(np.arange(nq, dtype=np.int32)); qr = N.to_device(dth.rate); qb = N.to_device(dth.slo / 2.0)
    out = torch.empty((nq, 32), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    alg = pt.n_points * 16 + nq * 52
    res = {}
    for w, ch, st in VARIANTS:
        lib = C.CDLL(str(OUT / f"lib_{w}_{ch}_{st}.so"))
        f = lambda: lib.parva_configure_sweep(C.byref(dt.struct), C.c_int32(nq), N.ptr(qt), N.ptr(qr), N.ptr(qb),  # noqa
                                              N.ptr(out), N.stream_handle())
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = sorted(ts)[len(ts) // 2]
        res[f"{w}x{ch}x{st}"] = (ms * 1000, alg / (ms / 1000) / 1e9 / 6547.5)
        print(f"{w:3d} warps ch {ch:4d} st {st}: {ms * 1000:7.1f} us  frac {res[f'{w}x{ch}x{st}'][1]:.3f}", flush=True)
    json.dump(res, open(REPO / "gpurun_out" / "sweep_tune.json", "w"), indent=1)


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
