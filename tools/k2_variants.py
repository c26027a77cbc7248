#!/usr/bin/env python3
"""A/B harness for K2 source variants: each variant is a set of text patches
applied to a copy of csrc/; every variant is built into tools/_variants/ and
timed on the C2 batch (device path + zero-copy e2e), with a parity check.

    python tools/k2_variants.py build
    python tools/k2_variants.py run
"""
import ctypes as C
import os
import shutil
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
OUT = REPO / "tools" / "_variants"
PATCH_DIR = REPO / "tools" / "k2_patches"


def variants():
    """name -> (patch list, extra flags).  A patch file holds OLD/NEW blocks
    separated by lines '<<<<' / '====' / '>>>>'.  "head" is the committed
    csrc/ (git HEAD), "base" the working tree."""
    vs = {"base": ([], [])} if os.environ.get("K2_NO_HEAD") else {"head": (["HEAD"], []), "base": ([], [])}
    for w, mb in ():   # launch-shape variants, e.g. ((17, 2), (12, 3), (24, 1))
        vs[f"w{w}_b{mb}"] = ([], [f"-DPARVA_PB_WARPS={w}", f"-DPARVA_PB_MINB={mb}"])
    # flag variants, e.g. ("-DPARVA_PB_WARPS=12", "-DPARVA_TILE_MINB=3", "-DPARVA_TILE_SVC=256"),
    # ("-DPARVA_STREAM_SLICE=16384",), ("-DPARVA_NO_OUT",) (K2s without its record writes)
    for flags in (tuple(f.split()) for f in os.environ.get("K2_FLAGS", "").split(",") if f):
        vs["_".join(f[8:].replace("=", "") for f in flags)] = ([], list(flags))
    if PATCH_DIR.exists():
        for f in sorted(PATCH_DIR.glob("*.patch")):
            vs[f.stem] = ([f], [])
    return vs


def apply(src: str, patch: Path) -> str:
    text = patch.read_text()
    for block in text.split("<<<<\n")[1:]:
        old, rest = block.split("====\n", 1)
        new = rest.split(">>>>\n", 1)[0]
        assert old in src, (patch, old[:80])
        src = src.replace(old, new)
    return src


def build():
    from paper_2409_14447_b200 import build as b
    OUT.mkdir(parents=True, exist_ok=True)
    for name, (patches, flags) in variants().items():
        d = OUT / f"v_{name}" / "csrc"      # csrc/../../include -> OUT/include
        if d.exists():
            shutil.rmtree(d)
        shutil.copytree(b.CSRC, d)
        if not (OUT / "include").exists():
            (OUT / "include").symlink_to(REPO / "include")
        sources = list(b.SOURCES)
        if patches == ["HEAD"]:            # the committed csrc/ at K2_REF (default HEAD)
            ref = os.environ.get("K2_REF", "HEAD")
            for f in d.iterdir():
                r = subprocess.run(["git", "show", f"{ref}:paper_2409_14447_b200/csrc/{f.name}"], cwd=REPO,
                                   capture_output=True)
                if r.returncode == 0:
                    f.write_bytes(r.stdout)
                elif f.name in sources:
                    sources.remove(f.name)
            patches = []
        for p in patches:                    # each block applies to the csrc file that holds its OLD text
            for block in p.read_text().split("<<<<\n")[1:]:
                old, rest = block.split("====\n", 1)
                hit = [f for f in sorted(d.iterdir()) if f.suffix in (".cu", ".cuh") and old in f.read_text()]
                assert hit, (p, old[:80])
                hit[0].write_text(hit[0].read_text().replace(old, rest.split(">>>>\n", 1)[0]))
        lib = OUT / f"libk2_{name}.so"
        inc = str(REPO / "include")
        cmd = [b.NVCC, *b.FLAGS, *flags, "-o", str(lib), *[str(d / s) for s in sources], "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        i = r.stderr.find(os.environ.get("K2_FN", "_ZN5parva18plan_thread_kernelILb0"))
        print(name, r.returncode, r.stderr[i:i + 400].split("\n")[1:4], r.stderr[:300] if r.returncode else "")


def run():
    import time
    import numpy as np
    import torch
    from paper_2409_14447_b200 import _native as N
    from bench import c2_inputs
    from paper_2409_14447_b200 import workloads as W
    from paper_2409_14447_b200.tables import pack_tables
    fx = W.load_fixtures()
    off, tab, rate, bound = c2_inputs(fx, 10_000, 0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ref = None
    for name in variants():
        lib = C.CDLL(str(OUT / f"libk2_{name}.so"))
        for fn in ("parva_plan_batch_workspace", "parva_plan_host_scratch", "parva_plan_general_workspace",
                   "parva_plan_host_packed_scratch", "parva_plan_host_mapped_scratch"):
            getattr(lib, fn).restype = C.c_size_t
        lib.parva_stream_bytes.restype = C.c_int64
        lib.parva_stream_pack.restype = C.c_int64
        N._LIB = lib
        from paper_2409_14447_b200 import batch as B
        dt = N.DeviceTables(pack_tables(fx.tables))
        d = [N.to_device(a) for a in (off, tab, rate, bound)]
        res = B.plan_batch(dt, *d)
        got = res.host()[1].copy()
        ref = got if ref is None else ref
        s = torch.cuda.current_stream()
        ts = []
        for i in range(80):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            B.plan_batch(dt, *d, out=res)
            b.record(s)
            torch.cuda.synchronize()
            if i >= 10:
                ts.append(a.elapsed_time(b) * 1e3)
        # back-to-back overlapped launches over 16 resident batches, 3 output blocks
        if not hasattr(run, "_batches"):
            run._batches = [c2_inputs(fx, 10_000, 0 if p == 0 else 1000 + p) for p in range(16)]
        dbat = [[N.to_device(a) for a in bt] for bt in run._batches]
        outs = [B.plan_batch(dt, *dbat[0]) for _ in range(16)]
        ring = B.SlotRing(16)
        gate = torch.zeros(1, dtype=torch.int32).pin_memory()
        gerr = torch.zeros(1, dtype=torch.int32, device="cuda")
        sh = N.stream_handle(s)
        for rep in range(2):
            torch.cuda.synchronize()
            gate.zero_()
            lib.parva_host_gate(C.c_void_p(gate.data_ptr()), C.c_uint32(1), C.c_int64(int(30e9)), N.ptr(gerr), sh)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for i in range(200):
                B.plan_batch(dt, *dbat[i % 16], out=outs[i % 16], overlap=True, ticket=ring.ticket(i % 16, 10_000))
            b.record(s)
            gate.numpy()[0] = 1
        torch.cuda.synchronize()
        ring.check()
        ov = a.elapsed_time(b) * 1e3 / 200
        ok_ov = outs[199 % 16].host()[1].tobytes() == B.plan_batch(dt, *dbat[199 % 16]).host()[1].tobytes()
        # C4-like: 2 x 10^5 scenarios in one launch (many tiles per CTA)
        if not hasattr(run, "_c4"):
            run._c4 = [N.to_device(a) for a in c2_inputs(fx, 200_000, 1)]
        r4 = B.plan_batch(dt, *run._c4)
        t4 = []
        for i in range(6):
            a4, b4 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a4.record(s)
            B.plan_batch(dt, *run._c4, out=r4)
            b4.record(s)
            torch.cuda.synchronize()
            t4.append(a4.elapsed_time(b4) * 1e3 / 20)
        p4 = r4.host()[1]
        if not hasattr(run, "_c4ref"):
            run._c4ref = p4.tobytes()
        ok4 = p4.tobytes() == run._c4ref
        mb = B.MappedHostBatch(off, tab, rate, bound, cfg_format=2, plan_bytes=64, depth=4)
        for k in range(2):
            if k:
                t0 = time.perf_counter()
            for i in range(300 if k else 20):
                mb.submit(dt, i % 4)
                if i >= 3:
                    mb.wait((i - 3) % 4)
            for sl in range(4):
                mb.wait(sl)
        e2e = (time.perf_counter() - t0) / 300 * 1e6
        ok = got.tobytes() == ref.tobytes() and mb.outputs(0)[1].tobytes() == ref.tobytes() and ok_ov
        print(f"{name:24s}: device K2 p50 {np.median(ts):6.1f} us  min {min(ts):6.1f}  overlapped {ov:6.1f} us/step"
              f"  c4 {np.median(t4):6.1f} us/10^4  e2e(depth 4) {e2e:6.1f} us  ok {ok} {ok4}")


if __name__ == "__main__":
    build() if sys.argv[1] == "build" else run()
