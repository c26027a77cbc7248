"""Per-step host timeline of the e2e loop (wait slot / pack / submit) over
K-step runs, to see where a short run loses time."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import batch_seed, c2_inputs  # noqa: E402
from paper_2409_14447_b200 import _native as N  # noqa: E402
from paper_2409_14447_b200 import batch as B  # noqa: E402
from paper_2409_14447_b200 import workloads as W  # noqa: E402

fx = W.load_fixtures()
dt = N.device_tables_for(fx.tables)
host = [c2_inputs(fx, 10_000, batch_seed(p)) for p in range(8)]
D = int(sys.argv[1]) if len(sys.argv) > 1 else 5
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
mb = B.MappedHostBatch(*host[0], cfg_format=2, plan_bytes=64, depth=D)


def loop(a, k, rec=None):
    for i in range(a, a + k):
        s = i % D
        t0 = time.perf_counter()
        mb.wait(s)
        t1 = time.perf_counter()
        mb.fill(*host[i % 8], slot=s)
        t2 = time.perf_counter()
        mb.submit(dt, s)
        t3 = time.perf_counter()
        if rec is not None:
            rec.append((t1 - t0, t2 - t1, t3 - t2))
    t0 = time.perf_counter()
    for s in range(D):
        mb.wait(s)
    return time.perf_counter() - t0


def loop2(a, k):
    for i in range(a, a + k):
        mb.submit_arrays(dt, i % D, *host[i % 8])
    for s in range(D):
        mb.wait(s)


loop2(0, 10)
for rep in range(4):
    t0 = time.perf_counter()
    loop2(10, K)
    el = time.perf_counter() - t0
    print(f"submit_arrays K={K} D={D}: {el / K * 1e6:6.1f} us/step ({10_000 * K / el:.3e} scen/s)")
loop(0, 10)
for rep in range(3):
    rec = []
    t0 = time.perf_counter()
    tail = loop(10, K, rec)
    el = time.perf_counter() - t0
    r = np.array(rec) * 1e6
    print(f"K={K} D={D}: {el / K * 1e6:6.1f} us/step ({10_000 * K / el:.3e} scen/s)  drain {tail * 1e6:5.0f} us | "
          f"wait med {np.median(r[:, 0]):5.1f} max {r[:, 0].max():6.1f}  pack med {np.median(r[:, 1]):5.1f} "
          f"max {r[:, 1].max():6.1f}  submit med {np.median(r[:, 2]):5.1f} max {r[:, 2].max():6.1f}")
