#!/usr/bin/env python3
"""A/B of K2 builds on one box, each through its own C ABI: the committed
library of a git ref (old ABI: no slot ticket) against the working tree and
flag variants of it.  Times one launch alone (L2 flushed) and 200
back-to-back overlapped launches (16 resident C2 batches, 3 output slots).

    python tools/k2_ab.py build [REF]      # default REF f4dad16 (round 1)
    python tools/k2_ab.py run
"""
import ctypes as C
import os
import shutil
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
OUT = REPO / "tools" / "_variants" / "ab"

# name -> (git ref or None for the working tree, extra nvcc flags)
VARIANTS = {
    "ref": ("REF", []),
    "tree": (None, []),
    "tree_binsearch": (None, ["-DPARVA_BINARY_SEARCH"]),
    "tree_fltreg": (None, ["-DPARVA_FLOAT_REGRESSION"]),
}


def build(ref="f4dad16"):
    from paper_2409_14447_b200 import build as b
    OUT.mkdir(parents=True, exist_ok=True)
    for name, (src, flags) in VARIANTS.items():
        root = OUT / name
        if root.exists():
            shutil.rmtree(root)
        (root / "pkg").mkdir(parents=True)
        (root / "include").mkdir()
        shutil.copytree(b.CSRC, root / "pkg" / "csrc")
        shutil.copy(REPO / "include" / "parva_b200.h", root / "include")
        if src == "REF":
            for f in (root / "pkg" / "csrc").iterdir():
                r = subprocess.run(["git", "show", f"{ref}:paper_2409_14447_b200/csrc/{f.name}"], cwd=REPO,
                                   capture_output=True)
                if r.returncode == 0:
                    f.write_bytes(r.stdout)
            r = subprocess.run(["git", "show", f"{ref}:include/parva_b200.h"], cwd=REPO, capture_output=True)
            (root / "include" / "parva_b200.h").write_bytes(r.stdout)
        srcs = [str(root / "pkg" / "csrc" / s) for s in b.SOURCES if (root / "pkg" / "csrc" / s).exists()]
        lib = OUT / f"lib_{name}.so"
        r = subprocess.run([b.NVCC, *b.FLAGS, *flags, "-o", str(lib), *srcs, "-lcudart"], capture_output=True,
                           text=True)
        i = r.stderr.find("_ZN5parva17plan_batch_kernelILb0")
        print(name, r.returncode, r.stderr[i:i + 300].split("\n")[1:2], r.stderr[-500:] if r.returncode else "")


class Ticket(C.Structure):
    _fields_ = [("d_count", C.c_void_p), ("wait_count", C.c_uint64), ("d_err", C.c_void_p)]


def run():
    import numpy as np
    import torch
    from bench import batch_seed, c2_inputs
    from paper_2409_14447_b200 import _native as N
    from paper_2409_14447_b200 import workloads as W
    fx = W.load_fixtures()
    dt = N.device_tables_for(fx.tables)          # tables + index built by the tree's library
    bats = [[N.to_device(a) for a in c2_inputs(fx, 10_000, batch_seed(p))] for p in range(16)]
    n, m = 10_000, 110_000
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    outs = [(torch.empty((m, 8), dtype=torch.uint8, device="cuda"), torch.empty((n, 128), dtype=torch.uint8,
                                                                                  device="cuda")) for _ in range(3)]
    words = torch.zeros(3, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    sh = N.stream_handle(s)
    ref_plan = None
    for rnd in range(2):
        for name in VARIANTS:
            lib = C.CDLL(str(OUT / f"lib_{name}.so"))
            new_abi = hasattr(lib, "parva_gather_release")

            def args(p, r):
                d = bats[p]
                return (C.byref(dt.struct), C.byref(dt.index_struct), C.c_int32(n), C.c_int32(m), N.ptr(d[0]),
                        N.ptr(d[1]), N.ptr(d[2]), N.ptr(d[3]), C.c_int32(1), C.c_int32(4), N.ptr(outs[r][0]),
                        C.c_int32(2), N.ptr(outs[r][1]))
            ts = []
            for i in range(60):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                lib.parva_plan_batch(*args(i % 16, 0), sh)
                b.record(s)
                torch.cuda.synchronize()
                if i >= 10:
                    ts.append(a.elapsed_time(b) * 1e3)
            words.zero_()
            issued = [0, 0, 0]
            tick = []
            for i in range(220):
                r = i % 3
                if new_abi:
                    tick.append(Ticket(words.data_ptr() + 8 * r, 0 if "nodone" in name else issued[r],
                                       err.data_ptr()))
                    issued[r] += n
            torch.cuda.synchronize()
            for i in range(220):
                if i == 20:
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(s)
                if new_abi:
                    lib.parva_plan_batch_overlapped(*args(i % 16, i % 3), C.byref(tick[i]), sh)
                else:
                    lib.parva_plan_batch_overlapped(*args(i % 16, i % 3), sh)
            b.record(s)
            torch.cuda.synchronize()
            ov = a.elapsed_time(b) * 1e3 / 200
            plan = outs[219 % 3][1].cpu().numpy()
            lib.parva_plan_batch(*args(219 % 16, 0), sh)
            torch.cuda.synchronize()
            ok = plan.tobytes() == outs[0][1].cpu().numpy().tobytes()
            print(f"round {rnd} {name:16s}: solo p50 {np.median(ts):6.1f} us  min {min(ts):6.1f}   overlapped "
                  f"{ov:6.2f} us/step  ok {ok}  err {int(err.item())}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(*(sys.argv[2:3] or []))
    else:
        run()
