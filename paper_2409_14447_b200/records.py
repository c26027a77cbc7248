"""numpy views of the C-ABI records (include/parva_b200.h)."""

from __future__ import annotations

import numpy as np

CONFIG_DTYPE = np.dtype([
    ("best", "<i2", (5,)), ("opt_sc", "i1"), ("last_sc", "i1"), ("status", "u1"),
    ("flags", "u1"), ("reserved", "<i2"), ("count", "<i8"), ("coverage", "<f8"),
])
COMPACT_DTYPE = np.dtype([
    ("best", "<i2", (5,)), ("opt_sc", "i1"), ("last_sc", "i1"), ("status", "u1"),
    ("flags", "u1"), ("count", "<u2"),
])
PLAN_DTYPE = np.dtype([
    ("status", "u1"), ("err_service", "u1"), ("n_gpus", "u1"), ("n_gpus_unopt", "u1"),
    ("n_place", "u1"), ("n_diag", "u1"), ("n_ledger", "u1"), ("flags", "u1"),
    ("payload", "u1", (120,)),
])
assert CONFIG_DTYPE.itemsize == 32 and PLAN_DTYPE.itemsize == 128 and COMPACT_DTYPE.itemsize == 16
CFG_FULL, CFG_COMPACT = 0, 1

# parva_status
OK, INFEASIBLE_SLO, RESIDUAL_UNCOVERABLE, COUNT_OVERFLOW, CAPACITY, BAD_INPUT, COVERAGE_ASSERT, LAUNCH_ERROR = range(8)
# parva_diag_reason
DIAG_SMALL_UNAVAILABLE, DIAG_NEED_NEW_GPU, DIAG_UNKNOWN_SERVICE, DIAG_REGRESSED = range(4)
FLAG_FALLBACK = 1
MAX_GPUS, MAX_SERVICES, PAYLOAD = 32, 32, 120


def plan_payload(rec):
    """(places, diags, ledger) of a plan record; ledger = [(service, value)] in rank order."""
    pay = np.asarray(rec["payload"], dtype=np.uint8)
    np_, nd, nl = int(rec["n_place"]), int(rec["n_diag"]), int(rec["n_ledger"])
    u16 = pay[:2 * (np_ + nd)].view("<u2")
    places = [int(v) for v in u16[:np_]]
    diags = [int(v) for v in u16[np_:]]
    off = (2 * (np_ + nd) + 7) & ~7
    vals = pay[off:off + 8 * nl].view("<f8")
    keys = pay[off + 8 * nl:off + 10 * nl].view("<u2")
    ledger = [(int(k) & 0xFF, float(v)) for k, v in zip(keys, vals)]
    return places, diags, ledger


def compact_config(full: np.ndarray) -> np.ndarray:
    """Full 32-byte config records -> 16-byte compact records (parva_config_compact)."""
    out = np.zeros(full.shape[0], dtype=COMPACT_DTYPE)
    for f in ("best", "opt_sc", "last_sc", "status"):
        out[f] = full[f]
    sat = full["count"] > 65535
    out["flags"] = sat.astype(np.uint8)
    out["count"] = np.where(sat, 65535, full["count"]).astype(np.uint16)
    return out


def unpack_place(v: int) -> tuple[int, int, int]:
    """place[i] = gpu << 11 | cat << 3 | slot."""
    return v >> 11, (v >> 3) & 0xFF, v & 7


def unpack_diag(v: int) -> tuple[int, int, int]:
    """diag[i] = gpu << 7 | reason << 5 | service -> (gpu, reason, service)."""
    return v >> 7, (v >> 5) & 3, v & 31


def format_diag(reason: int, gpu_id: int, name: str | None) -> str:
    """Diagnostic strings of optimize_allocation (allocator.py:394,401,410-412,421,432-434)."""
    if reason == DIAG_REGRESSED:
        return "optimization regressed GPU count or fragmentation; input kept"
    if reason == DIAG_SMALL_UNAVAILABLE:
        failure = f"service {name!r} has no size-1 or size-2 triplet"
    elif reason == DIAG_NEED_NEW_GPU:
        failure = f"replacements for GPU {gpu_id} would need a new GPU; kept as is"
    elif reason == DIAG_UNKNOWN_SERVICE:
        failure = f"unknown service {name!r}"
    else:
        raise ValueError(f"unknown diagnostic reason {reason}")
    return f"GPU {gpu_id}: optimization skipped: {failure}"
