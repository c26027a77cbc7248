"""Canonical plain-dict form of planner results, shared by the golden
generator (fed by the reference `migplan`) and the tests (fed by the C
oracle or by this package's CUDA path).  Floats stay Python floats, so
`json.dumps` writes them with repr and a hash of the dump is bit-exact.
"""

from __future__ import annotations

import hashlib
import json


def triplet(t):
    if t is None:
        return None
    return [int(t.instance_size), int(t.batch_size), int(t.process_count),
            float(t.throughput), float(t.latency)]


def service(s):
    return {
        "id": s.id, "model": s.model_id, "rate": float(s.request_rate),
        "slo": float(s.slo_latency), "internal": float(s.internal_latency),
        "best": [triplet(t) for t in s.best_triplets],
        "opt": triplet(s.optimal_segment), "count": int(s.optimal_segment_count),
        "last": triplet(s.last_segment),
        "coverage": float(s.coverage),
    }


def dmap(d):
    return {
        "gpus": [[int(g.id), [[p.service_id, int(p.instance_size), int(p.batch_size),
                               int(p.process_count), float(p.throughput), int(p.start_slot)]
                              for p in g.placements]] for g in d.gpus],
        "freed": [[k, float(v)] for k, v in d.freed_rate.items()],
        "diags": list(d.diagnostics),
    }


def plan(result):
    out = {"services": [service(s) for s in result.services],
           "unopt": int(result.unoptimized_gpu_count)}
    out.update(dmap(result.deployment))
    return out


def error(exc):
    return {"error": type(exc).__name__, "service": getattr(exc, "service_id", None),
            "message": str(exc)}


def dumps(obj) -> str:
    return json.dumps(obj, separators=(",", ":"))


def digest(obj) -> str:
    return hashlib.sha256(dumps(obj).encode()).hexdigest()[:16]
