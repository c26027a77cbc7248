"""Host pack throughput on this box: parva_stream_pack_arrays (C2 batch,
plain int32/f64 arrays -> pinned streamed block) vs thread count, a plain
memcpy of the same bytes into pinned memory, and the pool's fixed cost."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_14447_b200 import _native as N  # noqa: E402
from paper_2409_14447_b200 import workloads as W  # noqa: E402

L = N.load_library()
fx = W.load_fixtures()
sb = W.scenario_batch(fx, 10_000, seed=0)
n, M = sb.rate.shape
off = np.arange(n + 1, dtype=np.int32) * M
tab = np.tile(np.arange(M, dtype=np.int32), n)
rate, bound = sb.rate.ravel().copy(), sb.bound.ravel().copy()
cap = int(L.parva_stream_bytes(C.c_int32(n), N.np_ptr(off), C.c_int32(32)))
pin = torch.zeros(cap, dtype=torch.uint8).pin_memory()
reg = np.zeros(cap, np.uint8)


def t(fn, reps=50):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6, min(ts) * 1e6


for dst, name in ((pin.data_ptr(), "pinned"), (reg.ctypes.data, "pageable")):
    for th in (1, 2, 4, 8, 12, 16, 0):
        f = lambda: L.parva_stream_pack_arrays(C.c_int32(n), N.np_ptr(off), N.np_ptr(tab), N.np_ptr(rate),  # noqa
                                               N.np_ptr(bound), C.c_int32(32), C.c_void_p(dst), C.c_int64(cap),
                                               C.c_int32(th))
        print(f"pack {name:8s} threads {th:2d}: median {t(f)[0]:7.1f} us  min {t(f)[1]:7.1f} us")
pn = pin.numpy()
src = np.concatenate([rate.view(np.uint8), bound.view(np.uint8)])[:cap]
print("np.copyto 1.78 MB -> pinned: median %.1f us" % t(lambda: np.copyto(pn[:len(src)], src))[0])
o1, t1 = np.array([0, 11], np.int32), np.arange(11, dtype=np.int32)
r1 = np.ones(11)
f = lambda: L.parva_stream_pack_arrays(C.c_int32(1), N.np_ptr(o1), N.np_ptr(t1), N.np_ptr(r1), N.np_ptr(r1),  # noqa
                                       C.c_int32(32), C.c_void_p(pin.data_ptr()), C.c_int64(cap), C.c_int32(0))
print("pack of 1 scenario (pool fixed cost): median %.1f us" % t(f)[0])
