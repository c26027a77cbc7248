"""The bench's sharded (N > 1) flow end to end: two ranks on the one GPU over
gloo (PARVA_DIST_BACKEND=gloo), fused all-gather and the NCCL-style
collective path, one JSON line each with the driver-contract fields."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REPO = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("gather", ["fused", "nccl"])
def test_bench_two_ranks(gather):
    env = dict(os.environ, PARVA_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(REPO / "bench.py"),
           "--gpus", "2", "--steps", "5", "--warmup", "3", "--no-cpu", "--no-extra", "--sweep-workloads", "500",
           "--gather", gather]
    r = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["gather"] == gather
    sw = line["configurator_sweep"]      # sharded C3: one all-gather of config records
    assert sw["parity_vs_oracle_first_1000"] is True and sw["parity_gathered_sample"] is True
    par = line["parity_timed_steps"]
    assert par["equal"] is True and par["steps_checked"] == 5 and par["ranks"] == 2
    assert line["e2e"]["records_equal_oracle_last_steps"] is True
    # + the host gate kernel (not used on this gloo test path for the NCCL-style
    # gather, whose host-side collective would wait behind it)
    assert line["value"] > 0 and line["gpu_launches"] == (5 * 2 + 1 if gather == "fused" else 5)


def test_bench_two_ranks_extra_legs():
    """The N > 1 side measurements: C4 sharded over the ranks (fused plan +
    gather, checked on every rank), C5 / simulation / C1 on rank 0."""
    env = dict(os.environ, PARVA_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(REPO / "bench.py"),
           "--gpus", "2", "--steps", "5", "--warmup", "3", "--no-cpu", "--no-e2e", "--no-sweep"]
    r = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["parity_timed_steps"]["equal"] is True
    c4 = line["c4_sharded"]
    assert c4["parity_gathered"] is True and c4["scenarios"] == 1_000_000
    assert line["large_cluster"]["gpus"] == 51364
    assert all(s["gpus_equal_reference"] for s in line["c1_fixtures"]["scenarios"].values())
