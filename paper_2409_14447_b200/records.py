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
TINY_DTYPE = np.dtype([("best", "u1", (5,)), ("opt_last", "u1"), ("status_flags", "u1"), ("count", "u1")])
PLAN64_DTYPE = np.dtype([
    ("status", "u1"), ("err_service", "u1"), ("n_gpus", "u1"), ("n_gpus_unopt", "u1"),
    ("n_place", "u1"), ("n_diag", "u1"), ("n_ledger", "u1"), ("flags", "u1"),
    ("payload", "u1", (56,)),
])
SPILL_DTYPE = np.dtype([("scenario", "<i4"), ("pad", "<i4", (3,)), ("record", PLAN_DTYPE)])
assert CONFIG_DTYPE.itemsize == 32 and PLAN_DTYPE.itemsize == 128 and COMPACT_DTYPE.itemsize == 16
assert TINY_DTYPE.itemsize == 8 and PLAN64_DTYPE.itemsize == 64 and SPILL_DTYPE.itemsize == 144
CFG_FULL, CFG_COMPACT, CFG_TINY = 0, 1, 2

# parva_status
OK, INFEASIBLE_SLO, RESIDUAL_UNCOVERABLE, COUNT_OVERFLOW, CAPACITY, BAD_INPUT, COVERAGE_ASSERT, LAUNCH_ERROR, SPILLED = range(9)
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


def tiny_config(full: np.ndarray) -> np.ndarray:
    """Full 32-byte config records -> 8-byte tiny records (parva_config_tiny).
    A point position >= 255 does not fit the byte (the device entries reject
    PARVA_CFG_TINY for such tables): ValueError."""
    if full.shape[0] and int(full["best"].max(initial=-1)) >= 255:
        raise ValueError("tiny config records hold point positions < 255 (a table has > 254 points per size)")
    out = np.zeros(full.shape[0], dtype=TINY_DTYPE)
    out["best"] = np.where(full["best"] < 0, 255, full["best"]).astype(np.uint8)
    opt = np.where(full["opt_sc"] < 0, 15, full["opt_sc"]).astype(np.uint8)
    last = np.where(full["last_sc"] < 0, 15, full["last_sc"]).astype(np.uint8)
    out["opt_last"] = opt | (last << 4)
    sat = full["count"] > 255
    out["status_flags"] = full["status"].astype(np.uint8) | np.where(sat, 0x80, 0).astype(np.uint8)
    out["count"] = np.where(sat, 255, full["count"]).astype(np.uint8)
    return out


def expand_config(cfg: np.ndarray) -> np.ndarray:
    """Any config record format -> COMPACT_DTYPE fields (best i16, opt/last, status, count)."""
    if cfg.dtype == COMPACT_DTYPE:
        return cfg
    out = np.zeros(cfg.shape[0], dtype=COMPACT_DTYPE)
    if cfg.dtype == TINY_DTYPE:
        out["best"] = np.where(cfg["best"] == 255, -1, cfg["best"]).astype(np.int16)
        o, l = cfg["opt_last"] & 15, cfg["opt_last"] >> 4
        out["opt_sc"] = np.where(o == 15, -1, o).astype(np.int8)
        out["last_sc"] = np.where(l == 15, -1, l).astype(np.int8)
        out["status"] = cfg["status_flags"] & 0x7F
        out["flags"] = (cfg["status_flags"] >> 7).astype(np.uint8)
        out["count"] = cfg["count"]
        return out
    for f in ("best", "opt_sc", "last_sc", "status"):
        out[f] = cfg[f]
    out["count"] = np.minimum(cfg["count"], 65535)
    out["flags"] = (cfg["count"] > 65535).astype(np.uint8)
    return out


def plan64_view(plan128: np.ndarray, spill_cap: int):
    """Expected 64-byte records + spill list for given 128-byte records
    (what parva_plan_host_packed returns with plan_bytes = 64)."""
    p64 = np.zeros(plan128.shape[0], dtype=PLAN64_DTYPE)
    raw = plan128.view(np.uint8).reshape(-1, 128)
    p64.view(np.uint8).reshape(-1, 64)[:] = raw[:, :64]
    spills = []
    for k in range(plan128.shape[0]):
        r = plan128[k]
        if r["status"] != OK:
            continue
        need = ((2 * (int(r["n_place"]) + int(r["n_diag"])) + 7) & ~7) + 10 * int(r["n_ledger"])
        if need > 56:
            p64.view(np.uint8).reshape(-1, 64)[k] = 0
            if len(spills) < spill_cap:
                p64[k]["status"] = SPILLED
                spills.append(k)
            else:
                p64[k]["status"] = CAPACITY
    return p64, spills
