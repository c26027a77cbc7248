"""Build the sm_100a CUDA library (nvcc, in-tree) -> _build/libparva_b200.so.

    python -m paper_2409_14447_b200.build
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_build"
LIB = OUT_DIR / "libparva_b200.so"
SOURCES = ["configure.cu", "plan_batch.cu", "plan_general.cu", "unit_ops.cu", "prepare.cu", "capi.cu",
           "simulate.cu", "gather.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",                  # no FMA contraction: bit-exact with CPython
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def _deps():
    return sorted(CSRC.glob("*")) + [PKG.parent / "include" / "parva_b200.h"]


def source_hash() -> str:
    """Content hash of every source, the header and the compiler flags: a
    library is current iff it was built from exactly these (mtimes are not
    trusted -- copies of the tree, e.g. onto a GPU box, do not keep them)."""
    import hashlib
    h = hashlib.sha256()
    for p in _deps():
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    h.update(" ".join(FLAGS + SOURCES).encode())
    return h.hexdigest()


HASH_FILE = OUT_DIR / "libparva_b200.sha256"


def stale() -> bool:
    if not LIB.exists() or not HASH_FILE.exists():
        return True
    return HASH_FILE.read_text().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> Path:
    """nvcc into a temporary file, then an atomic rename, under a file lock:
    several processes (e.g. one per rank) may call this at once."""
    import fcntl
    if not force and not stale():
        return LIB
    OUT_DIR.mkdir(exist_ok=True)
    with open(OUT_DIR / ".build.lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        try:
            if not force and not stale():        # another process built it meanwhile
                return LIB
            digest = source_hash()
            tmp = OUT_DIR / f".libparva_b200.{os.getpid()}.so"
            cmd = [NVCC, *FLAGS, "-o", str(tmp), *[str(CSRC / s) for s in SOURCES], "-lcudart"]
            res = subprocess.run(cmd, capture_output=True, text=True)
            (OUT_DIR / "ptxas.log").write_text(res.stdout + res.stderr)
            if res.returncode != 0:
                tmp.unlink(missing_ok=True)
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError("nvcc failed building libparva_b200.so")
            os.replace(tmp, LIB)
            HASH_FILE.write_text(digest + "\n")
            if verbose:
                print(res.stderr)
        finally:
            fcntl.flock(lock, fcntl.LOCK_UN)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
