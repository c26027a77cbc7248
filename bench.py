#!/usr/bin/env python3
"""Benchmark: scenarios scheduled/sec (configurator + allocator) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1], "C2"): the 11 fixture models x 10^4
synthetic (SLO, request-rate) scenarios per GPU (SURVEY §8d C2 generator).
One step = one pass of the hot path over one batch: one K2 launch that
configures every service, relocates and optimizes every scenario
(pipeline.py:95-103 semantics) with its inputs resident in HBM.  Steps cycle
through ~70 resident input batches (more than the 126 MB L2 in total, so no
flush is needed) and write into one output slot per step; consecutive steps
are programmatic dependent launches whose slot tickets serialize launches
that share a slot.  N > 1 (torchrun, one process per GPU): every rank plans
its contiguous shard of each global batch (weak scaling: 10^4 scenarios per
GPU) and the step ends when every rank holds every rank's records: by
default K2 itself stores them into every rank's slot over NVLink peer
memory (fused all-gather, 64-byte plan records + 8-byte config records),
with one exact-epoch wait + release per step; --gather nccl uses one NCCL
all-gather of the packed 128-byte records instead.  After the timed region
every rank checks its gathered copy of every timed step against the CPU
oracle (digests of each rank's own shard, exchanged once).

Also reported: e2e through the C-ABI host entry from plain host arrays
(median of five 300-step spans, with the PCIe floor of its bytes), the C3
configurator sweep (the HBM-roofline kernel; sharded across ranks at N > 1
with one all-gather of config records), C4 (10^6 scenarios; sharded at
N > 1), C5, C1 (the fixture scenarios through the public API), the batched
simulator, and the CPU baselines (the C oracle = a port of the reference,
and the reference's own Python planner when baseline/_ref is installed).
"""

from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

PEAKS_PATH = REPO / "MEASURED_PEAKS.json"
METRIC = "scenarios scheduled/sec (configurator+allocator)"
# K2 on device-resident batches: the thread-per-scenario kernel (csrc/plan_thread.cuh)
K2_KERNEL = "plan_thread_kernel"
UNIT = "scenarios/s"


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu
    --set full capture (profiles/ncu_traffic.json), or None."""
    try:
        t = json.loads((REPO / "profiles" / "ncu_traffic.json").read_text())
        k = t[kernel]
        return int(k["dram_read"] + k["dram_write"])
    except Exception:  # noqa: BLE001
        return None


def ncu_inst(kernel):
    """Warp instructions per launch of `kernel` (smsp__inst_executed.sum of the
    committed ncu capture), or None."""
    try:
        return int(json.loads((REPO / "profiles" / "ncu_traffic.json").read_text())[kernel]["warp_inst"])
    except Exception:  # noqa: BLE001
        return None


def issue_roofline(kernel, kern_s, sm_mhz):
    """Instruction-issue roofline of a latency/issue-bound kernel: warp
    instructions per launch (ncu) / launch time, against one instruction per
    SM sub-partition per clock (148 SMs x 4 SMSPs x the sampled SM clock)."""
    inst = ncu_inst(kernel)
    if inst is None or not sm_mhz:
        return None
    peak = 148 * 4 * sm_mhz * 1e6
    ach = inst / kern_s
    return {"achieved": ach, "peak": peak, "unit": "warp-instructions/s", "frac": ach / peak,
            "warp_inst_per_launch": inst, "source": "profiles/ncu_traffic.json warp_inst; peak at the sampled SM clock"}


def peaks():
    try:
        p = json.loads(PEAKS_PATH.read_text())
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons.  nvidia-smi runs in its own loop
    mode (-lms) as ONE child process started before the warm-up, so nothing
    forks while the timed region runs (a fork per sample had stalled the
    launching thread); mark() brackets the spans whose samples count."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 20):
        self.samples = []          # (monotonic time, fields)
        self.spans = []
        self._p = None
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", str(period_ms)],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001
            self._p = None

    def _read(self):
        for line in self._p.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 6:
                self.samples.append((time.monotonic(), f))

    def begin(self):
        self._t0 = time.monotonic()

    def end(self):
        self.spans.append((self._t0, time.monotonic()))

    def close(self):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self._p.kill()

    def summary(self):
        pad = 0.025
        sel = [f for t, f in self.samples if any(a - pad <= t <= b + pad for a, b in self.spans)]
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        num = lambda x: x.replace(".", "").isdigit()  # noqa: E731
        sm = [float(s[0]) for s in sel if num(s[0])]
        mx = [float(s[1]) for s in sel if num(s[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in sel for i in range(4) if s[2 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sel)}


def c2_inputs(fx, n, seed):
    from paper_2409_14447_b200 import workloads as W
    sb = W.scenario_batch(fx, n, seed=seed)
    M = len(sb.models)
    off = (np.arange(n + 1, dtype=np.int32) * M)
    tab = np.tile(np.arange(M, dtype=np.int32), n)
    return off, tab, np.ascontiguousarray(sb.rate.ravel()), np.ascontiguousarray(sb.bound.ravel())


def batch_seed(p):
    """Seed of resident input batch p: batch 0 is C2 itself (seed 0)."""
    return 0 if p == 0 else 1000 + p


def n_resident_batches(n_svc_local, n_local):
    """P resident input batches of one shard's shape, cycled so that every
    step reads inputs that are not in L2 (P x ~2.2 MB > 126 MB)."""
    per_batch = n_svc_local * 20 + (n_local + 1) * 4
    return int(min(256, max(2, -(-160_000_000 // max(per_batch, 1)))))


def lscpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return None


def digest(cfg_bytes: bytes, plan_bytes: bytes) -> str:
    return hashlib.sha256(cfg_bytes + plan_bytes).hexdigest()[:32]


def ref_python(*argv, timeout=900):
    """tools/ref_python_bench.py: the reference itself (migplan from
    baseline/_ref, unmodified) on this host; None if it is not installed."""
    if not (REPO / "baseline" / "_ref" / "migplan").is_dir():
        return None
    try:
        r = subprocess.run([sys.executable, str(REPO / "tools" / "ref_python_bench.py"), *map(str, argv)],
                           capture_output=True, text=True, timeout=timeout,
                           env=dict(os.environ, PYTHONDONTWRITEBYTECODE="1"))
        return json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-300:]}
    except Exception as exc:  # noqa: BLE001
        return {"error": str(exc)}


def cpu_baselines(fx, n, min_seconds=10.0):
    """BASELINE.md §3 on this host: the oracle (C port of the reference) on
    all host threads (the headline CPU number, the reference arm's) and on
    one; the reference itself (pure Python migplan) on one core over a
    bounded C2 sample and on every core (fork Pool) over the full C2 batch."""
    import oracle
    from paper_2409_14447_b200.tables import pack_tables
    pt = pack_tables(fx.tables)
    off, tab, rate, bound = c2_inputs(fx, n, 0)
    threads = os.cpu_count() or 1

    def port(th, budget):
        oracle.plan_batch_records(pt, off, tab, rate, bound, threads=th)  # warm
        done, t0 = 0, time.perf_counter()
        while True:
            oracle.plan_batch_records(pt, off, tab, rate, bound, threads=th)
            done += n
            el = time.perf_counter() - t0
            if el >= budget:
                return done / el, done // n, el

    v, reps, el = port(threads, min_seconds)
    v1, reps1, el1 = port(1, min_seconds / 2)
    out = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": lscpu_model(),
           "sample": f"C2 batch of {n} scenarios x 11 services, repeated {reps}x ({el:.1f} s), "
                     f"oracle/migplan_oracle.c via OpenMP on {threads} threads",
           "port_1core": {"value": v1, "unit": UNIT, "cores": 1,
                          "sample": f"C2 batch repeated {reps1}x ({el1:.1f} s) on one thread"}}
    r1 = ref_python("c2", "--n", n, "--procs", 1)
    ra = ref_python("c2", "--n", n, "--procs", threads)
    if r1 is not None:
        out["reference_python_1core"] = {"value": r1.get("scenarios_per_s"), "unit": UNIT, "cores": 1,
                                         "sample": f"full C2 batch ({n} scenarios, seed 0), configure + relocate + "
                                                   "optimize per scenario (pipeline.py:95-103)", "raw": r1}
        out["reference_python_all_cores"] = {"value": ra.get("scenarios_per_s"), "unit": UNIT, "cores": threads,
                                             "sample": f"full C2 batch ({n} scenarios), fork Pool of {threads} "
                                                       "over strided chunks", "raw": ra}
    return out


def c5_cpu(fx):
    """C5 on this host's CPU: the oracle (C port with the reference's
    cursors, one thread) and the reference itself (migplan, one core)."""
    import oracle
    from paper_2409_14447_b200 import workloads as Wm
    from paper_2409_14447_b200.tables import pack_tables
    pt = pack_tables(fx.tables)
    t = pt.index_of()[Wm.C5_MODEL]
    rates = Wm.c5_rates()
    k = rates.shape[0]
    t0 = time.perf_counter()
    _, res = oracle.plan_scenario(pt, np.full(k, t), rates, np.full(k, Wm.C5_SLO / 2.0), True, 4, gcap=200_000)
    port_s = time.perf_counter() - t0
    out = {"port_1core_s": port_s, "port_gpus": len(res["gpus"])}
    r = ref_python("c5", timeout=900)
    if r is not None:
        out["reference_python"] = r
    return out


def run_reference(args, rank, world):
    """The reference arm: the CPU oracle (C restatement of the reference's
    planner; the reference itself is pure Python) on all host threads, over
    the same resident batches in the same order as the repo arm."""
    if rank != 0:
        return
    from paper_2409_14447_b200 import workloads as W
    fx = W.load_fixtures()
    import oracle
    from paper_2409_14447_b200.tables import pack_tables
    pt = pack_tables(fx.tables)
    n = args.scenarios
    P = n_resident_batches(n * 11, n)
    calls = args.warmup + args.steps
    need = sorted({c % P for c in range(calls)})
    ins = {p: c2_inputs(fx, n, batch_seed(p)) for p in need}
    threads = os.cpu_count() or 1
    for c in range(args.warmup):
        oracle.plan_batch_records(pt, *ins[c % P], threads=threads)
    t0 = time.perf_counter()
    for c in range(args.warmup, calls):
        oracle.plan_batch_records(pt, *ins[c % P], threads=threads)
    el = time.perf_counter() - t0
    v = n * args.steps / el
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1000 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (C2 generator; the repo arm's resident batches in the same order: batch 0 = seed 0, "
                    "batch p = seed 1000 + p)",
            "config": {"workload": "C2: 11 fixture workloads x 10^4 synthetic SLO/rate scenarios per GPU",
                       "scenarios_per_gpu": n, "services_per_scenario": 11, "global_batch": n,
                       "input_batches": P, "optimize": True, "threshold": 4},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "cpu_model": lscpu_model(),
                             "sample": f"one full C2 batch ({n} scenarios) per step on {threads} host threads; "
                                       "the reference itself is pure Python (its own timing: cpu_baseline."
                                       "reference_python in the repo arm's line)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def dist_max(dist, torch, world, vals):
    t = torch.tensor(vals, dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def dist_all(dist, torch, world, ok: bool) -> bool:
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(int(t.item()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scenarios", type=int, default=10_000,
                    help="scenarios per GPU per step (weak) or in total (strong)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--gather", default="fused", choices=["fused", "nccl"],
                    help="N > 1: K2 stores its records into every rank's slot over peer memory (fused), "
                         "or one NCCL all-gather per step")
    ap.add_argument("--slots", type=int, default=0,
                    help="output slots (0: one per timed step up to 64, at least 3)")
    ap.add_argument("--lag", type=int, default=2,
                    help="fused gather: step i waits for (and releases) step i - lag's slot")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C3 configurator-sweep measurement")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the C4 / C5 / simulator side measurements")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end host-entry measurement")
    ap.add_argument("--no-gate", action="store_true",
                    help="enqueue the timed steps without the host gate (needed under ncu, which serializes "
                         "launches: the gate kernel would never see its word written)")
    ap.add_argument("--sweep-workloads", type=int, default=10_000)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    # one process per GPU; PARVA_DIST_BACKEND=gloo lets the multi-rank path be
    # smoke-tested with several ranks on one device (NCCL refuses that)
    backend = os.environ.get("PARVA_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    clk = ClockSampler(local)

    from paper_2409_14447_b200 import _native as N
    from paper_2409_14447_b200 import batch as B
    from paper_2409_14447_b200 import distributed as D
    from paper_2409_14447_b200 import workloads as W
    from paper_2409_14447_b200.records import CFG_TINY, PLAN_DTYPE

    fx = W.load_fixtures()
    dt = N.device_tables_for(fx.tables)
    n_global = args.scenarios * (world if args.scaling == "weak" else 1)
    g_off, g_tab, _, _ = c2_inputs(fx, n_global, 0)          # every batch has this shape
    shard = D.make_shard(g_off, rank, world)
    off = shard.off
    tab = np.ascontiguousarray(g_tab[shard.svc_a:shard.svc_b])
    n = shard.scen_b - shard.scen_a
    n_svc_local = int(off[-1])
    P = n_resident_batches(n_svc_local, n)

    def shard_inputs(p):
        _, _, r, b = c2_inputs(fx, n_global, batch_seed(p))
        return (off, tab, np.ascontiguousarray(r[shard.svc_a:shard.svc_b]),
                np.ascontiguousarray(b[shard.svc_a:shard.svc_b]))

    batches = []
    for p in range(P):
        _, _, r, b = shard_inputs(p)
        batches.append((N.to_device(off), N.to_device(tab), N.to_device(r), N.to_device(b)))
    stream = torch.cuda.current_stream()
    sh = N.stream_handle(stream)
    L = N.lib()

    # output slots: one per timed step (up to 64), so every timed step's
    # records survive for the parity check; a slot's ticket serializes the
    # launches that share it
    S = args.slots if args.slots > 0 else max(3, min(args.steps, 64))

    def base_args(p, res):
        d_off, d_tab, d_rate, d_bound = batches[p]
        return (C.byref(dt.struct), C.byref(dt.index_struct), C.c_int32(n), C.c_int32(n_svc_local),
                N.ptr(d_off), N.ptr(d_tab), N.ptr(d_rate), N.ptr(d_bound), C.c_int32(1), C.c_int32(4),
                N.ptr(res.cfg), C.c_int32(CFG_TINY), N.ptr(res.plan))

    class Steps:
        """The sharded step: an overlapped K2 launch into output slot c % S
        (batch c % P), then the gather -- fused (K2's own peer stores + one
        exact-epoch wait/release, step c - lag), NCCL (one async all-gather of
        the slot), or none (N = 1)."""

        def __init__(self, mode):
            self.mode, self.peer, self.unwaited = mode, None, []
            if mode == "fused":
                self.lay = D.gather_layout(g_off, world, plan_bytes=64, cfg_bytes=8)
                self.peer = D.PeerGather(self.lay, n_slots=S)
                self.results = [self.peer.local(s, CFG_TINY) for s in range(S)]
                self.gslots = [self.peer.gather_slot(s, pdl=True) for s in range(S)]
                return
            lay = self.lay = D.gather_layout(g_off, world, plan_bytes=128, cfg_bytes=8)   # = packed_block's
            self.blocks = [torch.zeros(lay.blk, dtype=torch.uint8, device="cuda") for _ in range(S)]
            self.results = [B.BatchResult(bk[lay.ps:lay.ps + 8 * n_svc_local].view(-1, 8),
                                          bk[:lay.ps].view(-1, 128), n, n_svc_local, CFG_TINY) for bk in self.blocks]
            self.ring = B.SlotRing(S)
            self.gathered = ([torch.empty(world * lay.blk, dtype=torch.uint8, device="cuda") for _ in range(S)]
                             if world > 1 else None)
            self.works = [None] * S

        def prepare(self, c0, c1):
            """C-ABI arguments of calls [c0, c1), built before the timed
            region (tickets and mirrors carry sequential epochs)."""
            out = []
            for c in range(c0, c1):
                s = c % S
                a = base_args(c % P, self.results[s])
                t = self.peer.mirror(s, overlap=True) if self.peer is not None else self.ring.ticket(s, n)
                out.append((s, a + (C.byref(t), sh), t))
            return out

        def launch(self, item, timeout_s=60.0):
            s, a, _keep = item
            if self.peer is not None:
                N.check(L.parva_plan_batch_fused(*a), "parva_plan_batch_fused")
                self.unwaited.append(s)
                while len(self.unwaited) > args.lag:
                    w = self.unwaited.pop(0)
                    self.peer.wait(w, release=True, pdl=True, gslot=self.gslots[w], timeout_s=timeout_s)
                return
            if self.works[s] is not None:
                self.works[s].wait()     # the slot's previous all-gather has read it (a stream wait under NCCL)
                self.works[s] = None
            N.check(L.parva_plan_batch_overlapped(*a), "parva_plan_batch_overlapped")
            if world > 1:
                self.works[s] = dist.all_gather_into_tensor(self.gathered[s], self.blocks[s], async_op=True)

        def drain(self, timeout_s=60.0):
            if self.peer is not None:
                while self.unwaited:
                    s = self.unwaited.pop(0)
                    self.peer.wait(s, release=True, pdl=True, gslot=self.gslots[s], timeout_s=timeout_s)
                return
            for s in range(S):
                if self.works[s] is not None:
                    self.works[s].wait()
                    self.works[s] = None

        def healthy(self):
            if self.peer is not None:
                return int(self.peer.status.abs().sum().item()) == 0
            return int(self.ring.err.item()) == 0

        def check(self):
            if self.peer is not None:
                self.peer.check()
            else:
                self.ring.check()

        def rows(self, s):
            v = self.peer.slot_view(s) if self.peer is not None else self.gathered[s]
            return v.view(world, self.lay.blk).cpu().numpy()

        def close(self):
            if self.peer is not None:
                self.peer.close()
                self.peer = None

    gather_mode = "none" if world == 1 else args.gather
    st = None
    if gather_mode == "fused":
        try:
            st = Steps("fused")
        except Exception as exc:  # noqa: BLE001 -- no peer access: the NCCL collective instead
            print(f"fused all-gather unavailable ({exc}); using NCCL", file=sys.stderr)
            gather_mode = "nccl"
    if st is None:
        st = Steps(gather_mode)

    # ---- warm-up, then the timed steps
    if world > 1:
        dist.barrier()                   # every rank's inputs are resident before anyone waits on flags
    for item in st.prepare(0, args.warmup):
        st.launch(item, timeout_s=10.0)
    st.drain(timeout_s=10.0)
    torch.cuda.synchronize()
    if gather_mode == "fused" and not dist_all(dist, torch, world, st.healthy()):
        # no working peer stores on this box: time the NCCL collective instead
        print("fused all-gather: peer records did not arrive in the warm-up; using NCCL", file=sys.stderr)
        st.close()
        gather_mode = "nccl"
        st = Steps("nccl")
        for item in st.prepare(0, args.warmup):
            st.launch(item)
        st.drain()
        torch.cuda.synchronize()
    timed = st.prepare(args.warmup, args.warmup + args.steps)
    if world > 1:
        dist.barrier()
    t_start, t_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the K steps are queued behind a gate (one thread spinning on a pinned
    # host word) and the gate is opened once they are all enqueued: the
    # events then time device execution only, with no host launch gaps
    # a host-blocking collective (gloo copies CUDA tensors to the host) would
    # wait behind the gate forever: no gate for the gloo test path either
    use_gate = not args.no_gate and not (world > 1 and gather_mode == "nccl" and backend != "nccl")
    gate = torch.zeros(1, dtype=torch.int32).pin_memory()
    gate_err = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    clk.begin()
    if use_gate:
        N.check(L.parva_host_gate(C.c_void_p(gate.data_ptr()), C.c_uint32(1), C.c_int64(int(30e9)), N.ptr(gate_err),
                                  sh), "parva_host_gate")
    t_start.record(stream)
    for item in timed:
        st.launch(item)
    st.drain()
    t_stop.record(stream)
    gate.numpy()[0] = 1
    torch.cuda.synchronize()
    if int(gate_err.item()):
        raise RuntimeError("timed region: the gate timed out before the steps were enqueued")
    step_ms = t_start.elapsed_time(t_stop)
    st.check()

    # ---- parity of every timed step that survives in its slot: every rank
    # checks its copy of every rank's records against the oracle (digests of
    # each rank's own shard, computed here and exchanged once)
    import oracle
    from paper_2409_14447_b200.records import tiny_config
    from paper_2409_14447_b200.tables import pack_tables
    pt = pack_tables(fx.tables)
    first = max(args.warmup, args.warmup + args.steps - S)
    checked = list(range(first, args.warmup + args.steps))
    threads = max(1, (os.cpu_count() or 1) // world)
    own = {}
    for c in checked:
        p = c % P
        if p not in own:
            ocfg, oplan = oracle.plan_batch_records(pt, *shard_inputs(p), threads=threads)
            own[p] = digest(tiny_config(ocfg).tobytes(), oplan.tobytes())
    if world > 1:
        every = [None] * world
        dist.all_gather_object(every, own)
    else:
        every = [own]
    ok = True
    for c in checked:
        s, p = c % S, c % P
        if world == 1:
            cfg, plan = st.results[s].host()
            ok = ok and digest(cfg.tobytes(), plan.tobytes()) == every[0][p]
            continue
        cfg, plan = D.decode_gathered(st.rows(s), st.lay)
        for r, ((a, b), (sa, sb)) in enumerate(zip(st.lay.spans, st.lay.svc_spans)):
            ok = ok and digest(cfg[sa:sb].tobytes(), plan[a:b].tobytes()) == every[r][p]
    parity = dist_all(dist, torch, world, ok)
    parity_info = {"equal": parity, "steps_checked": len(checked), "ranks": world,
                   "scope": ("every rank's gathered copy of every rank's config + plan records of each timed step"
                             if world > 1 else "the config + plan records of each timed step"),
                   "checker": "oracle/migplan_oracle.c (C restatement of the reference), sha256 digests"}

    # ---- K2's own launch duration (roofline): the timed batches one launch
    # at a time into a scratch output, each bracketed by events on the
    # launching stream (not overlapped)
    scratch = B.BatchResult(torch.empty((n_svc_local, 8), dtype=torch.uint8, device="cuda"),
                            torch.empty((n, 128), dtype=torch.uint8, device="cuda"), n, n_svc_local, CFG_TINY)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        kev[i][0].record(stream)
        N.check(L.parva_plan_batch(*base_args((args.warmup + i) % P, scratch), sh), "parva_plan_batch")
        kev[i][1].record(stream)
    torch.cuda.synchronize()
    kern_ms = sum(a.elapsed_time(b) for a, b in kev)
    # keep the GPU busy a little longer so the sampler sees the loaded clocks
    t_end = time.perf_counter() + 1.0
    while time.perf_counter() < t_end:
        for j in range(50):
            L.parva_plan_batch(*base_args(j % P, scratch), sh)
        torch.cuda.synchronize()
    clk.end()
    step_ms, kern_ms = dist_max(dist, torch, world, [step_ms, kern_ms])

    n_svc = int(off[-1])
    hbm, peak_src = peaks()
    # algorithmic bytes per K2 launch: per service 20 B in
    # (table id, rate, bound) + 8 B tiny config record out; per scenario 4 B
    # offset + 128 B plan record; tables+index once (18 B / point).
    bytes_per_launch = n_svc * (20 + 8) + n * (4 + 128) + dt.packed.n_points * 18
    kern_s = kern_ms / 1000.0 / args.steps
    step_s = step_ms / 1000.0 / args.steps
    # back-to-back launches overlap, so a launch's average duration over the
    # timed region is the step time; one launch alone is reported beside it
    achieved = bytes_per_launch / step_s / 1e9
    value = n_global * args.steps / (step_ms / 1000.0)
    if gather_mode == "fused":
        par = (" + fused all-gather: K2 stores each tile's 64-B plan + 8-B config records (full records of "
               "spilled scenarios in an overflow section) into every rank's slot over peer memory; per step one "
               f"exact-epoch wait + release of step i-{args.lag}'s slot")
    elif gather_mode == "nccl":
        par = " + one NCCL all-gather of the packed 128-B plan + 8-B config records per step"
    else:
        par = ""
    launches_per_step = 2 if gather_mode == "fused" else 1

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY C2 generator: batch 0 is C2 seed 0, the other resident batches seeds 1001.., "
                "sharded contiguously; fixture tables rendered from the reference)",
        "config": {"workload": "C2: 11 fixture workloads x 10^4 synthetic SLO/rate scenarios per GPU"
                               if args.scaling == "weak" else f"C2/C4 generator, {n_global} scenarios total",
                   "scenarios_per_gpu": n, "services_per_scenario": 11, "global_batch": n_global,
                   "l2": "not reused: steps cycle through resident input batches larger than L2 in total",
                   "input_batches": P, "output_slots": S,
                   "launch": ("parva_plan_batch_overlapped / _fused per step (programmatic dependent launches; "
                              "slot tickets serialize launches sharing an output slot), "
                              + ("all K steps enqueued behind a gate kernel that is opened once they are queued "
                                 "(device time, no host launch gaps); " if use_gate
                                 else "no gate (host launch gaps included); ")
                              + "kernel_ms_per_step from separate one-at-a-time launches"),
                   "parallelism": f"scenario-sharded x{world}" + par,
                   "gather": gather_mode, "optimize": True, "threshold": 4},
        "gpu_launches": args.steps * launches_per_step + (1 if use_gate else 0),
        "kernel_ms_per_step": kern_ms / args.steps,
        "roofline": {"bound": "hbm", "kernel": f"{K2_KERNEL} (fused configure + relocate + optimize, thread per scenario)",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "duration": "average launch duration over the timed region (= ms_per_step: the launches overlap)",
                     "traffic": ncu_traffic(K2_KERNEL),
                     "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read+write per launch)",
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": bytes_per_launch,
                     "alone": {"achieved": bytes_per_launch / kern_s / 1e9,
                               "frac": bytes_per_launch / kern_s / 1e9 / hbm,
                               "duration": "one launch at a time (kernel_ms_per_step)"},
                     "note": "latency-bound sequential allocator (dependency chains per scenario, register-limited "
                             "occupancy); HBM fraction reported, not targeted"},
        "parity_timed_steps": parity_info,
    }
    clk_summary = clk.summary()
    line["clocks"] = clk_summary
    line["roofline"]["issue"] = issue_roofline(K2_KERNEL, step_s, clk_summary.get("sm_mhz"))
    line["roofline"]["issue_alone"] = issue_roofline(K2_KERNEL, kern_s, clk_summary.get("sm_mhz"))
    st.close()

    if not args.no_e2e:
        line["e2e"] = e2e_measure(args, torch, dist, world, N, B, fx, dt, shard_inputs, P, n_global, pt)
    if not args.no_sweep:
        line["configurator_sweep"] = sweep_measure(args, torch, dist, world, rank, N, B, W, hbm, peak_src)
    if not args.no_extra:
        if world > 1:
            line["c4_sharded"] = c4_sharded_measure(torch, dist, world, rank, N, B, D, fx, dt)
        elif rank == 0:
            line["c4_single_gpu"] = c4_measure(torch, N, B, W, fx, dt, local)
        if rank == 0:
            line["large_cluster"] = c5_measure(torch, fx)
            line["simulation"] = sim_measure(torch, fx)
    if not args.no_extra and rank == 0:
        line["c1_fixtures"] = c1_measure(fx)
    if not args.no_cpu and rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baselines(fx, n)
        if "large_cluster" in line:
            line["large_cluster"]["cpu"] = c5_cpu(fx)
        if "c1_fixtures" in line:
            r = ref_python("c1")
            if r:
                line["c1_fixtures"]["reference_python_1core"] = r
        if "c4_single_gpu" in line:
            r = ref_python("c4", "--n", 2000, "--procs", 1)
            if r:
                r["extrapolated_s_for_10^6"] = r["seconds"] * 1e6 / r["scenarios"]
                line["c4_single_gpu"].setdefault("cpu", {})["reference_python_1core"] = r
    clk.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_measure(args, torch, dist, world, N, B, fx, dt, shard_inputs, P, n_global, pt):
    """End to end through the C ABI, starting every step from a caller's
    plain host arrays (scenario offsets, int32 table ids, f64 rates and
    bounds in pageable numpy memory; 8 different C2 batches in rotation).
    Per step: pack the batch into a pinned input block on the library's host
    threads (parva_stream_pack_arrays), submit one K2s launch
    (parva_plan_host_mapped_submit) that streams the block over PCIe and
    writes its config + plan records (ledger included) into pinned host
    memory; E2E_DEPTH steps in flight, the host waits for every step's
    completion word (parva_plan_host_mapped_wait) before reusing its slot.
    The packing of step i overlaps the GPU work of steps i-3..i-1.  Reported
    beside it: the same pipeline with inputs packed once outside the loop
    (prepacked), and one synchronous call per step."""
    import oracle
    from paper_2409_14447_b200.records import tiny_config
    E2E_DEPTH, E2E_BATCHES, E2E_SPANS = int(os.environ.get("PARVA_E2E_DEPTH", 5)), 8, 5
    span_s = []
    # a throughput over at least 300 steps: a 20-step run would mostly time
    # the pipeline's fill and drain (5 calls in flight)
    steps = max(args.steps, 300)
    host = [shard_inputs(p) for p in range(E2E_BATCHES)]      # the caller's arrays (pageable)
    mb = B.MappedHostBatch(*host[0], cfg_format=2, plan_bytes=64, depth=E2E_DEPTH)
    pack_s = []

    def batches(c0, k):
        for i in range(c0, c0 + k):
            yield host[i % E2E_BATCHES]

    mode = os.environ.get("PARVA_E2E_MODE", "loop")
    c0 = max(args.warmup, E2E_DEPTH)
    last = {}
    if mode == "stream":
        mb.stream(dt, batches(0, c0))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        mb.stream(dt, batches(c0, steps), consume=lambda i, slot: last.__setitem__(slot, c0 + i))
        e2e_s = time.perf_counter() - t0
    else:   # one C call per step: wait for the slot's previous call, pack into its block, submit
        def loop(a, k):
            for i in range(a, a + k):
                slot = i % E2E_DEPTH
                mb.submit_arrays(dt, slot, *host[i % E2E_BATCHES])
                last[slot] = i
            for slot in range(E2E_DEPTH):
                mb.wait(slot)
        loop(0, c0)
        if world > 1:
            dist.barrier()
        # E2E_SPANS spans of `steps` steps each (the pipeline drains between
        # spans); the median span is the value: one host scheduling hiccup of
        # a few ms inside a ~15 ms span would otherwise move it by 10-20%
        for r in range(E2E_SPANS):
            t0 = time.perf_counter()
            loop(c0 + r * steps, steps)
            span_s.append(time.perf_counter() - t0)
        e2e_s = statistics.median(span_s)
    h2d = mb.h2d_bytes
    # the records of the last batch planned in every slot against the oracle
    ok = True
    for slot, i in last.items():
        ocfg, oplan = oracle.plan_batch_records(pt, *host[i % E2E_BATCHES])
        cfg, plan = mb.outputs(slot)
        ok = ok and plan.tobytes() == oplan.tobytes() and cfg.tobytes() == tiny_config(ocfg).tobytes()
    # the host pack alone (the producer's share of a step)
    for i in range(20):
        t = time.perf_counter()
        mb.fill(*host[i % E2E_BATCHES], slot=0)
        pack_s.append(time.perf_counter() - t)

    def run_steps(c0, k, pack=True):
        for i in range(c0, c0 + k):
            slot = i % E2E_DEPTH
            mb.wait(slot)
            if pack:
                mb.fill(*host[i % E2E_BATCHES], slot=slot)
            mb.submit(dt, slot)
        for slot in range(E2E_DEPTH):
            mb.wait(slot)

    # the same pipeline with the inputs packed outside the loop (one batch per slot)
    for slot in range(E2E_DEPTH):
        mb.fill(*host[slot], slot=slot)
    run_steps(0, args.warmup, pack=False)
    t0 = time.perf_counter()
    run_steps(0, steps, pack=False)
    pre_s = time.perf_counter() - t0
    # one synchronous call per step (pack + launch + stream synchronize)
    for i in range(args.warmup):
        mb.fill(*host[i % E2E_BATCHES], slot=0)
        mb.run(dt)
    t0 = time.perf_counter()
    for i in range(steps):
        mb.fill(*host[i % E2E_BATCHES], slot=0)
        mb.run(dt)
    sync_s = time.perf_counter() - t0
    p_h2d, p_d2h, p_bi = pcie_peaks(torch)
    ok = dist_all(dist, torch, world, ok)
    e2e_s, pre_s, sync_s = dist_max(dist, torch, world, [e2e_s, pre_s, sync_s])
    K = n_global * steps
    step_us = e2e_s / steps * 1e6
    floor_us = max(mb.h2d_bytes / p_h2d, mb.d2h_bytes / p_d2h, (mb.h2d_bytes + mb.d2h_bytes) / p_bi) / 1e3
    return {"value": K / e2e_s, "unit": UNIT, "steps": steps,
            "spans": {"n": len(span_s), "steps_each": steps, "value_per_span": [n_global * steps / x for x in span_s],
                      "value": "the median span"} if span_s else None,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": mb.d2h_bytes,
            "api": "per step one C call, parva_plan_host_arrays_submit: wait for the slot's previous call, pack the "
                   "plain host arrays into the slot's pinned streamed block (parva_stream_pack_arrays, on the "
                   f"library's host threads), submit the K2s launch; {E2E_DEPTH} calls in flight; the host waits "
                   "for every call's completion word (a producer-thread variant, MappedHostBatch.stream, measured "
                   "slower: PARVA_E2E_MODE=stream)",
            "inputs": f"{E2E_BATCHES} different C2 batches in rotation, plain pageable numpy arrays "
                      "(int32 offsets and table ids, f64 rates and bounds)",
            "pipeline_depth": E2E_DEPTH,
            "host_pack_us_median": statistics.median(pack_s) * 1e6 if pack_s else None,
            "pcie_roofline": {
                "bound": "pcie", "achieved": (mb.h2d_bytes + mb.d2h_bytes) / (step_us * 1e3), "peak": p_bi,
                "unit": "GB/s", "frac": floor_us / step_us, "step_us": step_us, "floor_us": floor_us,
                "peaks_gbs": {"h2d": p_h2d, "d2h": p_d2h, "both": p_bi},
                "floor": "max(H2D bytes / H2D peak, D2H bytes / D2H peak, all bytes / both-direction peak), "
                         "peaks measured here with 32 MB copy-engine copies from/to pinned memory: the bus time "
                         "a step's transfers cannot go below; frac = floor / step"},
            "records_equal_oracle_last_steps": ok,
            "prepacked": {"value": K / pre_s, "unit": UNIT,
                          "api": "the same pipeline with every slot's input block packed once outside the loop"},
            "synchronous": {"value": K / sync_s, "unit": UNIT,
                            "api": "pack + parva_plan_host_mapped (one launch + stream synchronize) per step"}}


def pcie_peaks(torch, mb=32, reps=10):
    """Measured PCIe peaks (GB/s) of this box: copy-engine copies of `mb` MB
    from/to pinned memory -- H2D alone, D2H alone, and both at once on two
    streams (the bus is full duplex)."""
    n = mb << 20
    h1, h2 = (torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2))
    d1, d2 = (torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    def both():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    h2d = n / timed(lambda: d1.copy_(h1, non_blocking=True)) / 1e9
    d2h = n / timed(lambda: h2.copy_(d2, non_blocking=True)) / 1e9
    bi = 2 * n / timed(both) / 1e9
    return h2d, d2h, bi


def sim_measure(torch, fx, runs=256, horizon=10.0):
    """Batched run_simulation: the S6 plan under `runs`
    seeds, 10 s of Poisson arrivals each, in one call (host seeding + GPU
    arrivals and event loops + host statistics, all inside the wall time).
    CPU comparison on the box: numpy arrivals + the C oracle event loop on
    one core for a sample; the Python reference's time per run was measured
    in the build container (tests/golden/sim_cases.json)."""
    import paper_2409_14447_b200 as P
    from paper_2409_14447_b200 import simulation as S
    sc = P.Scenario("S6", tuple(P.scenario.ScenarioService(m, r, l) for m, r, l in fx.scenarios["S6"]))
    res = P.plan_scenario(sc, fx.tables)
    services = list(res.services)
    wl = S.Workload.from_services(services)
    jobs = [S.SimJob(res.deployment, fx.tables, services, wl, horizon, seed) for seed in range(runs)]
    S.run_simulations(jobs)              # warm-up at full size (device buffers cached)
    torch.cuda.synchronize()
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        reps = S.run_simulations(jobs)
        walls.append(time.perf_counter() - t0)
    wall = statistics.median(walls)
    arrivals = sum(st.arrived for r in reps for st in r.services.values())
    # CPU path on the box (test infrastructure as the checker/baseline): a sample of runs
    import oracle
    sys.path.insert(0, str(REPO / "tests"))
    from helpers import sim_report_with_oracle
    k = 8
    t0 = time.perf_counter()
    for j in jobs[:k]:
        orep, _, _ = sim_report_with_oracle(oracle, j)
    cpu = (time.perf_counter() - t0) / k
    ok = all(sim_report_with_oracle(oracle, j)[0].to_json_obj() == r.to_json_obj() for j, r in zip(jobs[:4], reps[:4]))
    ref = None
    try:
        cases = json.loads((REPO / "tests" / "golden" / "sim_cases.json").read_text())
        ref = [c["reference_s"] for c in cases if c["scenario"] == "S6" and c["horizon_s"] == 10.0][0]
    except Exception:  # noqa: BLE001
        pass
    return {"workload": f"S6 plan x {runs} seeds x {horizon:g} s Poisson arrivals, one batched run_simulations call "
                        "(median of 3 after a full-size warm-up)",
            "runs": runs, "arrivals": int(arrivals), "wall_s": wall, "runs_per_s": runs / wall,
            "arrivals_per_s": arrivals / wall, "cpu_c_oracle_s_per_run": cpu,
            "reference_python_s_per_run": ref, "reports_equal_cpu_path_first_4": ok}


def c5_measure(torch, fx):
    """C5: one allocation of 100,002 segments (49,612 services) -- general
    kernels (parallel relocation + warp-cooperative optimize), device time."""
    from paper_2409_14447_b200 import batch as Bm
    from paper_2409_14447_b200 import _native as Nm
    from paper_2409_14447_b200 import workloads as Wm
    dt = Nm.device_tables_for(fx.tables)
    rates = Wm.c5_rates()
    n = rates.shape[0]
    t = dt.packed.index_of()[Wm.C5_MODEL]
    cfg, _ = Bm.plan_batch(dt, np.array([0, n], dtype=np.int32), np.full(n, t, dtype=np.int32), rates,
                           np.full(n, Wm.C5_SLO / 2.0)).host()
    g = Bm.general_from_configs(dt.packed, np.full(n, t), cfg, True, 4)
    out = Bm.plan_general(g)          # warm-up
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ms = []
    for _ in range(3):
        t0 = time.perf_counter()
        ev[0].record()
        out = Bm.plan_general(g)
        ev[1].record()
        torch.cuda.synchronize()
        ms.append(((time.perf_counter() - t0) * 1000, ev[0].elapsed_time(ev[1])))
    return {"workload": "C5: 49,612 densenet121 services, 100,002 segments, one allocation",
            "gpus_before_optimize": out.n_gpus_unopt, "gpus": int(len(out.gpu_id)),
            "ms_wall_incl_transfers": min(m[0] for m in ms), "ms_stream": min(m[1] for m in ms),
            "note": "CPU times on this host in large_cluster.cpu (cpu leg)"}


def c1_measure(fx, reps=20):
    """C1: the Table IV fixture scenarios S1-S6 through the public API
    (plan_scenario: one fused launch + decode of every object), wall time per
    scenario (median of reps), GPU counts checked against the reference's."""
    import paper_2409_14447_b200 as P
    want = {"S1": 1, "S2": 2, "S3": 3, "S4": 4, "S5": 8, "S6": 9}     # SURVEY 8c / BASELINE 2
    out = {}
    for name, svcs in fx.scenarios.items():
        sc = P.Scenario(name, tuple(P.scenario.ScenarioService(m, r, l) for m, r, l in svcs))
        P.plan_scenario(sc, fx.tables)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            res = P.plan_scenario(sc, fx.tables)
            res.services, res.deployment
            ts.append(time.perf_counter() - t0)
        ts.sort()
        out[name] = {"ms": ts[len(ts) // 2] * 1e3, "gpus": res.gpu_count,
                     "gpus_equal_reference": res.gpu_count == want.get(name)}
    return {"workload": "C1: S1-S6 through plan_scenario (one launch + synchronize + full decode per scenario)",
            "scenarios": out}


def c4_measure(torch, N, B, W, fx, dt, local):
    """C4 on one GPU: 10^6 scenarios in one K2 launch (the strong-scaling unit)."""
    n = 1_000_000
    off, tab, rate, bound = c2_inputs(fx, n, 1)
    d = [N.to_device(a) for a in (off, tab, rate, bound)]
    res = B.plan_batch(dt, *d)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    times = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        B.plan_batch(dt, *d, out=res)
        b.record(s)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    ms = sorted(times)[len(times) // 2]
    line = {"workload": "C4 generator (seed 1), 10^6 scenarios x 11 services, one GPU", "ms_per_launch": ms,
            "value": n / (ms / 1000.0), "unit": UNIT, "l2": "inputs 17.6 MB + outputs 480 MB exceed L2 reuse"}
    # the first 10^4 scenarios on the CPU: the port's time (one thread) and a parity check of those records
    import oracle
    from paper_2409_14447_b200.tables import pack_tables
    k = 10_000
    cfg = N.records_to_numpy(res.cfg, 11 * k, N.CONFIG_DTYPE)
    plan = N.records_to_numpy(res.plan, k, B.PLAN_DTYPE)
    tc = time.perf_counter()
    ocfg, oplan = oracle.plan_batch_records(pack_tables(fx.tables), off[:k + 1], tab[:11 * k], rate[:11 * k],
                                            bound[:11 * k], threads=1)
    port_s = time.perf_counter() - tc
    line["parity_vs_oracle_first_10000"] = bool(cfg[:11 * k].tobytes() == ocfg.tobytes() and
                                                plan[:k].tobytes() == oplan.tobytes())
    line["cpu"] = {"port_1core": {"scenarios": k, "seconds": port_s, "value": k / port_s, "unit": UNIT,
                                  "extrapolated_s_for_10^6": port_s * n / k}}
    return line


def c4_sharded_measure(torch, dist, world, rank, N, B, D, fx, dt, reps=5):
    """C4 strong-scaled (BASELINE configs[3]): 10^6 scenarios sharded
    contiguously across the ranks; the step is done when every rank holds
    every rank's records.  Reported: this shard's K2 alone (compute), one
    NCCL all-gather of the packed 128-B records (collective only), and the
    fused K2 + peer-store all-gather with 64-B records + one exact-epoch wait
    (the product path); each the median of `reps`, max over ranks.  Every
    rank checks its gathered copy against the oracle (digests per shard)."""
    import oracle
    from paper_2409_14447_b200.records import CFG_TINY, tiny_config
    from paper_2409_14447_b200.tables import pack_tables
    n = 1_000_000
    off, tab, rate, bound = c2_inputs(fx, n, 1)
    sh = D.make_shard(off, rank, world)
    ins = (sh.off, tab[sh.svc_a:sh.svc_b], rate[sh.svc_a:sh.svc_b], bound[sh.svc_a:sh.svc_b])
    d = [N.to_device(np.ascontiguousarray(a)) for a in ins]
    k, m = sh.scen_b - sh.scen_a, sh.svc_b - sh.svc_a
    s = torch.cuda.current_stream()

    def timed(fn):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return sorted(ts)[len(ts) // 2]

    lay128 = D.gather_layout(off, world, plan_bytes=128, cfg_bytes=8)
    blk = torch.zeros(lay128.blk, dtype=torch.uint8, device="cuda")
    res = B.BatchResult(blk[lay128.ps:lay128.ps + 8 * m].view(-1, 8), blk[:lay128.ps].view(-1, 128), k, m, CFG_TINY)
    gat = torch.empty(world * lay128.blk, dtype=torch.uint8, device="cuda")
    ms_compute = timed(lambda: B.plan_batch(dt, *d, cfg_format=CFG_TINY, out=res))
    ms_nccl = timed(lambda: dist.all_gather_into_tensor(gat, blk))
    lay = D.gather_layout(off, world, plan_bytes=64, cfg_bytes=8)
    pg = D.PeerGather(lay, n_slots=2)
    state = {"i": 0}

    def fused():
        slot = state["i"] % 2
        state["i"] += 1
        B.plan_batch(dt, *d, cfg_format=CFG_TINY, out=pg.local(slot, CFG_TINY), mirror=pg.mirror(slot))
        pg.wait(slot, release=True)

    fused()
    ms_fused = timed(fused)
    torch.cuda.synchronize()
    pg.check()
    last = (state["i"] - 1) % 2
    ocfg, oplan = oracle.plan_batch_records(pack_tables(fx.tables), *ins, threads=max(1, (os.cpu_count() or 1) // world))
    mine = digest(tiny_config(ocfg).tobytes(), oplan.tobytes())
    every = [None] * world
    dist.all_gather_object(every, mine)
    cfg, plan = pg.records(last)
    ok = all(digest(cfg[sa:sb].tobytes(), plan[a:b].tobytes()) == every[r]
             for r, ((a, b), (sa, sb)) in enumerate(zip(lay.spans, lay.svc_spans)))
    ok = dist_all(dist, torch, world, ok)
    pg.close()
    ms_compute, ms_nccl, ms_fused = dist_max(dist, torch, world, [ms_compute, ms_nccl, ms_fused])
    return {"workload": f"C4 generator (seed 1), 10^6 scenarios x 11 services sharded over {world} GPUs (strong)",
            "scenarios": n, "scenarios_per_gpu": k, "value": n / (ms_fused / 1000.0), "unit": UNIT,
            "ms_fused_plan_and_gather": ms_fused, "ms_compute_only": ms_compute,
            "ms_nccl_allgather_only": ms_nccl,
            "gathered_bytes_per_scenario": {"fused": 64 + 8 * 11, "nccl": 128 + 8 * 11},
            "value_compute_plus_nccl": n / ((ms_compute + ms_nccl) / 1000.0),
            "parity_gathered": ok, "timing": "median of 5 after a barrier, CUDA events, max over ranks"}


def sweep_measure(args, torch, dist, world, rank, N, B, W, hbm, peak_src):
    """C3 configurator sweep (K1, the HBM-roofline kernel).  N > 1: the 10^4
    workloads shard contiguously (each rank generates and sweeps only its
    tables), then ONE all-gather of the 32-B config records; every rank
    checks the gathered records of every shard (digests vs the oracle on a
    sample of each shard)."""
    import oracle
    from paper_2409_14447_b200 import distributed as D
    from paper_2409_14447_b200.tables import pack_dense
    nw = args.sweep_workloads
    a, b = D.shard_bounds(nw, rank, world)
    t0 = time.perf_counter()
    dth = W.dense_tables(b - a, seed=3, first=a)
    gen_s = time.perf_counter() - t0
    pt = pack_dense(dth)
    dt = N.DeviceTables(pt, build_index=False)
    nl = b - a
    q_table = N.to_device(np.arange(nl, dtype=np.int32))
    q_rate = N.to_device(dth.rate)
    q_bound = N.to_device(dth.slo / 2.0)
    max_l = max(y - x for x, y in (D.shard_bounds(nw, r, world) for r in range(world)))
    out = torch.zeros((max_l, 32), dtype=torch.uint8, device="cuda")
    B.configure_sweep(dt, q_table, q_rate, q_bound, out=out)
    steps = max(10, min(args.steps, 50))
    for _ in range(5):
        B.configure_sweep(dt, q_table, q_rate, q_bound, out=out)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        ev[i][0].record(s)
        B.configure_sweep(dt, q_table, q_rate, q_bound, out=out)
        ev[i][1].record(s)
    torch.cuda.synchronize()
    ms = sum(x.elapsed_time(y) for x, y in ev) / steps
    points = pt.n_points
    alg = points * 16 + nl * (4 + 8 + 8) + nl * 32
    achieved = alg / (ms / 1000.0) / 1e9
    k = min(nl, 1000)
    recs = N.records_to_numpy(out, nl, N.CONFIG_DTYPE)
    tc = time.perf_counter()
    orec = oracle.configure_batch(pt, np.arange(k), dth.rate[:k], dth.slo[:k] / 2.0, threads=1)
    port_s = time.perf_counter() - tc
    local_ok = bool(recs[:k].tobytes() == orec.tobytes())
    port_points = int(np.asarray(pt.seg_count)[:5 * k].sum())
    line = {"workload": "C3: 10^4 dense tables (5 sizes x batch 1-128 x procs 1-8), 1 query each",
            "workloads": nw, "points": points, "ms_per_launch": ms, "value": nw / (ms / 1000.0) if world == 1 else None,
            "unit": "workloads/s", "points_per_s": points / (ms / 1000.0),
            "roofline": {"bound": "hbm", "kernel": "configure_sweep_kernel", "achieved": achieved, "peak": hbm,
                         "unit": "GB/s", "frac": achieved / hbm, "traffic": ncu_traffic("configure_sweep_kernel"),
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": alg},
            "parity_vs_oracle_first_1000": local_ok,
            "l2": "no flush: the profile points per launch exceed the 126 MB L2",
            "generation_s": gen_s,
            "cpu": {"port_1core": {"workloads": k, "points": port_points, "seconds": port_s,
                                   "workloads_per_s": k / port_s, "points_per_s": port_points / port_s,
                                   "what": "oracle/migplan_oracle.c configure for the first workloads, one thread"}}}
    if world == 1:
        if not args.no_cpu:
            r = ref_python("c3", "--n", 200)
            if r:
                line["cpu"]["reference_python_1core"] = r
        return line
    # one all-gather of the config records (padded to the largest shard)
    gat = torch.empty((world * max_l, 32), dtype=torch.uint8, device="cuda")
    gts = []
    for _ in range(5):
        torch.cuda.synchronize()
        dist.barrier()
        x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x.record(s)
        dist.all_gather_into_tensor(gat, out)
        y.record(s)
        torch.cuda.synchronize()
        gts.append(x.elapsed_time(y))
    ms_g = sorted(gts)[2]
    mine = hashlib.sha256(recs[:k].tobytes()).hexdigest() if local_ok else "local-mismatch"
    every = [None] * world
    dist.all_gather_object(every, mine)
    rows = gat.view(world, max_l, 32).cpu().numpy()
    ok = all(hashlib.sha256(rows[r, :min(1000, y - x)].tobytes()).hexdigest() == every[r]
             for r, (x, y) in enumerate(D.shard_bounds(nw, r2, world) for r2 in range(world)))
    ok = dist_all(dist, torch, world, ok)
    ms_max, ms_g, frac_min = dist_max(dist, torch, world, [ms, ms_g, -achieved / hbm])
    line.update({"value": nw / ((ms_max + ms_g) / 1000.0), "ms_sweep_max_over_ranks": ms_max,
                 "ms_allgather_config_records": ms_g, "workloads_per_gpu": nl,
                 "roofline_frac_min_over_ranks": -frac_min, "parity_gathered_sample": ok,
                 "note": "value = all workloads / (slowest rank's sweep + one NCCL all-gather of 32-B records)"})
    return line


if __name__ == "__main__":
    main()
