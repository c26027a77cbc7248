"""Device layout of prepared profile tables.

`pack_tables` applies the preparation the reference does outside its timed
region (pipeline.py:70-80: filter_feasible with the memory map, then
restrict(process_counts=(1,)) for --single-process) and lays the surviving
points out as structure-of-arrays grouped by (table, size class):

    segment s = t*5 + c  ->  points [seg_start[s], seg_start[s] + seg_count[s])

in key order (batch asc, procs asc).  A point's position inside its segment
is its tie-break rank for _better_triplet (configurator.py:116-124), so the
kernels read 16 bytes per point (tp f64, lat f64) and never a key.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from .errors import ValidationError
from .mig import INSTANCE_SIZES, SIZE_CLASS
from .profiles import ProfileTable, check_memory_map


@dataclass
class PackedTables:
    names: list[str]
    tp: np.ndarray          # f64 [P]
    lat: np.ndarray         # f64 [P]
    batch: np.ndarray       # i32 [P]
    procs: np.ndarray       # i32 [P]
    seg_start: np.ndarray   # i64 [T*5]
    seg_count: np.ndarray   # i32 [T*5]
    mem: np.ndarray | None = None   # f64 [P] memory_required (raw tables only)

    @property
    def n_tables(self) -> int:
        return len(self.names)

    @property
    def n_points(self) -> int:
        return int(self.tp.shape[0])

    def index_of(self) -> dict[str, int]:
        return {n: i for i, n in enumerate(self.names)}

    def point(self, t: int, c: int, j: int) -> int:
        return int(self.seg_start[t * 5 + c]) + int(j)


def pack_tables(tables: Mapping[str, ProfileTable] | Sequence[ProfileTable],
                memory_map: Mapping[int, float] | None = None,
                single_process: bool = False, prepared: bool = False) -> PackedTables:
    """Prepare and pack tables; `prepared=True` skips the memory filter."""
    if isinstance(tables, Mapping):
        items = list(tables.items())
    else:
        items = [(t.model_id, t) for t in tables]
    mm = check_memory_map(memory_map)
    tp, lat, batch, procs, mem = [], [], [], [], []
    seg_start = np.zeros(len(items) * 5, dtype=np.int64)
    seg_count = np.zeros(len(items) * 5, dtype=np.int32)
    pos = 0
    for t, (_, table) in enumerate(items):
        per = [[] for _ in INSTANCE_SIZES]
        for p in table.points:
            if not prepared and not p.memory_required <= mm[p.instance_size]:
                continue
            if single_process and p.process_count != 1:
                continue
            per[SIZE_CLASS[p.instance_size]].append(p)
        for c, pts in enumerate(per):
            if len(pts) > 32767:
                raise ValidationError("more than 32767 points of one instance size in a table")
            seg_start[t * 5 + c] = pos
            seg_count[t * 5 + c] = len(pts)
            pos += len(pts)
            for p in pts:
                tp.append(p.throughput); lat.append(p.latency)
                batch.append(p.batch_size); procs.append(p.process_count); mem.append(p.memory_required)
    return PackedTables(
        names=[n for n, _ in items],
        tp=np.asarray(tp, dtype=np.float64), lat=np.asarray(lat, dtype=np.float64),
        batch=np.asarray(batch, dtype=np.int32), procs=np.asarray(procs, dtype=np.int32),
        seg_start=seg_start, seg_count=seg_count, mem=np.asarray(mem, dtype=np.float64))


def pack_raw(tables) -> PackedTables:
    """Every point of the tables, unfiltered, in the device grouping (input of
    the device-side preparation, csrc/prepare.cu)."""
    return pack_tables(tables, prepared=True)


def pack_dense(dt) -> PackedTables:
    """workloads.DenseTables (already prepared, contiguous) as PackedTables."""
    W = dt.n_workloads
    return PackedTables(names=[f"w{w:05d}" for w in range(W)], tp=dt.tp, lat=dt.lat,
                        batch=dt.batch, procs=dt.procs,
                        seg_start=dt.seg_start.astype(np.int64), seg_count=dt.seg_count.astype(np.int32))
