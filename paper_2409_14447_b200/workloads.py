"""Seeded synthetic inputs for the BASELINE.json configurations.

These generate planner INPUTS only (profile tables, (rate, SLO) demands);
they never plan anything.  Transcendentals go through Python's `math`
(glibc) element by element instead of numpy's SIMD ufuncs so that the same
seed gives bit-identical inputs on this container and on the GPU box.

C1  fixture tables + Table IV scenarios S1-S6 (reference fixtures.py:28-229),
    loaded from tests/golden/fixture_tables.json (rendered from the
    reference by tests/golden/make_golden.py).
C2  11 fixture models x 10^4 log-uniform (rate, SLO) scenarios, seed 0;
    every 100th scenario forces one InfeasibleSLOError.
C3  10^4 dense synthetic tables (5 sizes x batch 1..128 x procs 1..8),
    the jitter-free `synthesize_profile` surface (profiles.py:319-469),
    one query per table, seed 3.
C4  the C2 generator with seed 1 and 10^6 scenarios.
C5  one scenario of 49,612 densenet121 services (random.Random(1)),
    100,002 segments after configuration.
"""

from __future__ import annotations

import json
import math
import os
import random
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .mig import INSTANCE_SIZES
from .profiles import DEFAULT_MEMORY_MAP, ProfilePoint, ProfileTable

REPO_ROOT = Path(__file__).resolve().parent.parent
FIXTURE_JSON = REPO_ROOT / "tests" / "golden" / "fixture_tables.json"


def _exp(a: np.ndarray) -> np.ndarray:
    flat = np.asarray(a, dtype=np.float64).ravel().tolist()
    return np.fromiter(map(math.exp, flat), dtype=np.float64, count=len(flat)).reshape(np.shape(a))


# --------------------------------------------------------------------- C1
@dataclass
class Fixtures:
    models: list[str]
    tables: dict[str, ProfileTable]
    scenarios: dict[str, list[tuple[str, float, float]]]


def load_fixtures(path: str | os.PathLike | None = None) -> Fixtures:
    obj = json.loads(Path(path or FIXTURE_JSON).read_text())
    tables = {}
    for m in obj["models"]:
        pts = tuple(ProfilePoint(m, int(s), int(b), int(p), float(tp), float(lat), float(mem))
                    for s, b, p, tp, lat, mem in obj["tables"][m])
        tables[m] = ProfileTable(m, pts)
    scen = {k: [(m, float(r), float(l)) for m, r, l in v] for k, v in obj["scenarios"].items()}
    return Fixtures(list(obj["models"]), tables, scen)


# ------------------------------------------------------------ C2 / C4
@dataclass
class ScenarioBatch:
    """n_scen scenarios x n_models services; service j of every scenario is model j."""

    models: list[str]
    rate: np.ndarray   # f64 [n_scen, n_models]
    slo: np.ndarray    # f64 [n_scen, n_models]

    @property
    def n_scenarios(self) -> int:
        return self.rate.shape[0]

    @property
    def bound(self) -> np.ndarray:
        return self.slo / 2.0   # make_service: internal_latency = slo / 2.0 (configurator.py:87-89)


def scenario_batch(fx: Fixtures, n: int, seed: int, inject_infeasible: bool = True) -> ScenarioBatch:
    models = fx.models
    M = len(models)
    lo_r = np.empty(M); hi_r = np.empty(M); lo_l = np.empty(M); hi_l = np.empty(M)
    for j, m in enumerate(models):
        rs = [r for sc in fx.scenarios.values() for mm, r, _ in sc if mm == m]
        ls = [l for sc in fx.scenarios.values() for mm, _, l in sc if mm == m]
        lo_r[j], hi_r[j] = math.log(0.5 * min(rs)), math.log(1.5 * max(rs))
        lo_l[j], hi_l[j] = math.log(0.75 * min(ls)), math.log(1.25 * max(ls))
    rng = np.random.default_rng(seed)
    u = rng.random((n, M, 2))
    rate = _exp(lo_r + (hi_r - lo_r) * u[:, :, 0])
    slo = _exp(lo_l + (hi_l - lo_l) * u[:, :, 1])
    if inject_infeasible:
        min_lat = [min(p.latency for p in fx.tables[m].points
                       if p.memory_required <= DEFAULT_MEMORY_MAP[p.instance_size]) for m in models]
        for k in range(99, n, 100):
            j = (k // 100) % M
            slo[k, j] = min_lat[j]
    return ScenarioBatch(list(models), rate, slo)


# ------------------------------------------------------------------ C3
@dataclass
class DenseTables:
    """Prepared (memory-filtered) dense tables in key order, concatenated.

    seg_start[w*5+c] .. seg_start[w*5+c] + seg_count[w*5+c] are the points of
    workload w, size class c (instance size INSTANCE_SIZES[c]).
    """

    tp: np.ndarray
    lat: np.ndarray
    batch: np.ndarray
    procs: np.ndarray
    seg_start: np.ndarray   # i64 [W*5]
    seg_count: np.ndarray   # i32 [W*5]
    rate: np.ndarray        # one query per workload
    slo: np.ndarray

    @property
    def n_workloads(self) -> int:
        return self.rate.shape[0]

    @property
    def n_points(self) -> int:
        return int(self.seg_count.sum())


def _round3_exact(x: np.ndarray) -> np.ndarray:
    """Python's correctly rounded round(x, 3), vectorised; near-ties via round()."""
    y = x * 1000.0
    r = np.rint(y) / 1000.0
    frac = np.abs(y - np.floor(y) - 0.5)
    risky = np.nonzero(frac < 1e-6)[0]
    for i in risky.tolist():
        r[i] = round(float(x[i]), 3)
    return r


def dense_params(n_workloads: int, seed: int = 3, first: int = 0) -> dict[str, np.ndarray]:
    """Per-workload SyntheticModelParams fields and the query, C3 stream."""
    W_all = first + n_workloads
    rng = np.random.default_rng(seed)
    u = rng.random((W_all, 8))[first:]     # one row per workload: 6 params + query
    q = u[:, 6:8]
    ln = math.log
    gexp = 0.95 + (1.4 - 0.95) * u[:, 1]
    return {
        "base": _exp(ln(100.0) + (ln(5000.0) - ln(100.0)) * u[:, 0]),
        "gexp": gexp,
        "sexp": 0.5 + (np.minimum(0.9, gexp) - 0.5) * u[:, 2],
        "sat": 5.0 + (15.0 - 5.0) * u[:, 3],
        "wmem": _exp(ln(0.01) + (ln(1.5) - ln(0.01)) * u[:, 4]),
        "amem": _exp(ln(0.005) + (ln(0.06) - ln(0.005)) * u[:, 5]),
        "slo": _exp(ln(20.0) + (ln(2000.0) - ln(20.0)) * q[:, 0]),
        "rate": _exp(ln(10.0) + (ln(20000.0) - ln(10.0)) * q[:, 1]),
    }


def dense_tables(n_workloads: int, seed: int = 3, batch_max: int = 128, procs_max: int = 8,
                 first: int = 0) -> DenseTables:
    """C3 tables: jitter-free synthesize_profile (profiles.py:319-322,443-466) + filter_feasible.

    Workload parameters: base_throughput logU(100, 5000),
    gpc_exponent U(0.95, 1.4), sat_exponent U(0.5, min(0.9, gpc)), sat_work
    U(5, 15), weight_memory logU(0.01, 1.5), activation_memory logU(0.005, 0.06);
    query slo logU(20, 2000) ms, rate logU(10, 20000) rps.  `first` skips the
    first workloads (same stream) so bounded samples can be regenerated.
    """
    prm = dense_params(n_workloads, seed, first)
    base, gexp, sexp, sat, wmem, amem = (prm[k] for k in ("base", "gexp", "sexp", "sat", "wmem", "amem"))
    slo, rate = prm["slo"], prm["rate"]
    W = n_workloads

    B = np.arange(1, batch_max + 1, dtype=np.int64)
    P = np.arange(1, procs_max + 1, dtype=np.int64)
    bb, pp = np.meshgrid(B, P, indexing="ij")           # key order within a size: batch, procs
    bb = bb.ravel(); pp = pp.ravel()
    work = (bb * pp).astype(np.float64)                  # float(b * pr)
    ncell = work.shape[0]

    tps, lats, mems = [], [], []
    for s in INSTANCE_SIZES:
        # Python float ** (libm pow) per workload, exactly as _raw_throughput does.
        cap = np.array([b * float(s) ** g for b, g in zip(base.tolist(), gexp.tolist())])
        half = np.array([w * float(s) ** e for w, e in zip(sat.tolist(), sexp.tolist())])
        tp = cap[:, None] * work[None, :] / (work[None, :] + half[:, None])
        tp = tp * 1.0                                    # anchor-free scale factor
        lat = np.maximum(1.0, np.rint(1000.0 * work[None, :] / tp))
        mem = pp[None, :].astype(np.float64) * (wmem[:, None] + bb[None, :].astype(np.float64) * amem[:, None])
        tps.append(tp); lats.append(lat); mems.append(_round3_exact(mem.ravel()).reshape(W, ncell))
    tp = np.stack(tps, axis=1)      # [W, 5, ncell]
    lat = np.stack(lats, axis=1)
    mem = np.stack(mems, axis=1)
    caps = np.array([DEFAULT_MEMORY_MAP[s] for s in INSTANCE_SIZES])
    keep = mem <= caps[None, :, None]
    seg_count = keep.sum(axis=2).astype(np.int32).ravel()
    seg_start = np.zeros(W * 5, dtype=np.int64)
    seg_start[1:] = np.cumsum(seg_count.astype(np.int64))[:-1]
    flat_keep = keep.ravel()
    return DenseTables(
        tp=np.ascontiguousarray(tp.ravel()[flat_keep]),
        lat=np.ascontiguousarray(lat.ravel()[flat_keep]),
        batch=np.ascontiguousarray(np.broadcast_to(bb, (W, 5, ncell)).ravel()[flat_keep].astype(np.int32)),
        procs=np.ascontiguousarray(np.broadcast_to(pp, (W, 5, ncell)).ravel()[flat_keep].astype(np.int32)),
        seg_start=seg_start, seg_count=seg_count, rate=rate, slo=slo)


def dense_table_objects(dt: DenseTables, w: int, model_id: str | None = None) -> ProfileTable:
    """Workload w of a DenseTables as a (prepared) ProfileTable."""
    mid = model_id or f"w{w:05d}"
    pts = []
    for c, s in enumerate(INSTANCE_SIZES):
        a = int(dt.seg_start[w * 5 + c]); n = int(dt.seg_count[w * 5 + c])
        for i in range(a, a + n):
            pts.append(ProfilePoint(mid, s, int(dt.batch[i]), int(dt.procs[i]),
                                    float(dt.tp[i]), float(dt.lat[i]), 0.0))
    return ProfileTable(mid, tuple(pts))


# ------------------------------------------------------------------ C5
C5_SERVICES = 49_612          # first count reaching >= 10^5 segments (re-checked by make_golden)
C5_MODEL = "densenet121"
C5_SLO = 183.0


def c5_rates(n: int = C5_SERVICES, seed: int = 1) -> np.ndarray:
    rng = random.Random(seed)
    return np.array([rng.uniform(100, 3 * 2183.7) for _ in range(n)], dtype=np.float64)
