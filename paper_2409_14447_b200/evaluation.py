"""Deployment metrics used by PlanResult.summary (reference evaluation.py:56-82).

Post-processing of a DeploymentMap (SURVEY §8f "next" row 3); the
discrete-event simulator of the reference (evaluation.py:85-464) is out of
scope for this build.
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
