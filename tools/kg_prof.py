#!/usr/bin/env python3
"""Build libparva with -DPARVA_KG_PROF into tools/_variants and run C5 on it
(device printf of the optimize chain's phase cycles).  usage: build | run"""
import ctypes as C
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
LIB = REPO / "tools" / "_variants" / "libkg_prof.so"
if sys.argv[1] == "build":
    from paper_2409_14447_b200 import build as b
    LIB.parent.mkdir(parents=True, exist_ok=True)
    r = subprocess.run([b.NVCC, *b.FLAGS, "-DPARVA_KG_PROF", "-o", str(LIB), *[str(b.CSRC / s) for s in b.SOURCES],
                        "-lcudart"], capture_output=True, text=True)
    print("build", r.returncode, r.stderr[-500:] if r.returncode else "")
else:
    import numpy as np
    import torch
    from paper_2409_14447_b200 import _native as N
    lib = C.CDLL(str(LIB))
    for fn in ("parva_plan_batch_workspace", "parva_plan_host_scratch", "parva_plan_general_workspace",
               "parva_plan_host_packed_scratch", "parva_plan_host_mapped_scratch"):
        getattr(lib, fn).restype = C.c_size_t
    lib.parva_stream_bytes.restype = C.c_int64
    lib.parva_stream_pack.restype = C.c_int64
    N._LIB = lib
    from paper_2409_14447_b200 import batch as B
    from paper_2409_14447_b200 import workloads as W
    fx = W.load_fixtures()
    dt = N.device_tables_for(fx.tables)
    rates = W.c5_rates()
    n = rates.shape[0]
    t = dt.packed.index_of()[W.C5_MODEL]
    cfg, _ = B.plan_batch(dt, np.array([0, n], dtype=np.int32), np.full(n, t, dtype=np.int32), rates,
                          np.full(n, W.C5_SLO / 2.0)).host()
    g = B.general_from_configs(dt.packed, np.full(n, t), cfg, True, 4)
    for _ in range(2):
        out = B.plan_general(g)
        torch.cuda.synchronize()
    print("gpus", len(out.gpu_id))
