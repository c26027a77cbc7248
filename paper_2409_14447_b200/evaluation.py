"""Deployment metrics used by PlanResult.summary (reference evaluation.py:56-82).

Post-processing of a DeploymentMap (SURVEY §8f "next" row 3).  The
discrete-event simulator of the reference (evaluation.py:85-464) is in
simulation.py (§8f row 4, event loops on the GPU).
"""

from __future__ import annotations

from .errors import UndefinedMetricError
from .mig import SLOT_COUNT

DEFAULT_SMS_PER_GPC = 14


def allocated_fraction(dmap, sms_per_gpc: int = DEFAULT_SMS_PER_GPC) -> float:
    """Share of provisioned GPU SMs covered by allocated segments (evaluation.py:65-72)."""
    if not dmap.gpus:
        raise UndefinedMetricError("allocated fraction is undefined for an empty map")
    allocated = sum(p.instance_size for _, p in dmap.placements()) * sms_per_gpc
    provisioned = len(dmap.gpus) * SLOT_COUNT * sms_per_gpc
    return allocated / provisioned


def external_fragmentation(dmap, sms_per_gpc: int = DEFAULT_SMS_PER_GPC) -> float:
    """Unallocated share of provisioned GPU SMs (evaluation.py:75-82)."""
    return 1.0 - allocated_fraction(dmap, sms_per_gpc)


def plan_metrics(plan, sms_per_gpc: int = DEFAULT_SMS_PER_GPC) -> dict:
    """Per-scenario deployment metrics straight from 128-byte plan records
    (SURVEY §8f row 3), vectorised: the same integer counts and the same
    correctly rounded int/int division as allocated_fraction /
    external_fragmentation (evaluation.py:65-82).  Rows whose status is not
    OK (or whose map is empty) get NaN fractions."""
    import numpy as np
    from .records import OK, PLAN_DTYPE
    plan = np.asarray(plan)
    n = plan.shape[0]
    pay = plan["payload"].astype(np.uint16)
    words = pay[:, 0::2] | (pay[:, 1::2] << 8)            # u16 little endian, 60 per record
    idx = np.arange(words.shape[1])[None, :]
    is_place = idx < plan["n_place"][:, None]
    cls = ((words >> 3) & 0xFF) % 5
    sizes = np.array([1, 2, 3, 4, 7], dtype=np.int64)[cls]
    total = np.where(is_place, sizes, 0).sum(axis=1)
    gpus = plan["n_gpus"].astype(np.int64)
    ok = (plan["status"] == OK) & (gpus > 0)
    alloc = np.full(n, np.nan)
    alloc[ok] = (total[ok] * sms_per_gpc).astype(np.float64) / (gpus[ok] * SLOT_COUNT * sms_per_gpc).astype(np.float64)
    return {"gpu_count": gpus, "total_gpcs": total, "allocated_fraction": alloc,
            "external_fragmentation": 1.0 - alloc, "unoptimized_gpu_count": plan["n_gpus_unopt"].astype(np.int64)}
