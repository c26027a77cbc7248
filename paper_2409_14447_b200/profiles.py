"""Profile tables: the planner's input data model.

Mirrors reference `pkg/src/migplan/profiles.py:25-271` (ProfilePoint,
ProfileTable, CSV/JSON I/O, filter_feasible).  These are host-side value
types; the planning kernels never see them.  `batch.TableSet` packs them
into the device layout (structure-of-arrays grouped by (table, instance
size)).
"""

from __future__ import annotations

import csv
import io
import json
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Iterator, Mapping

from .errors import ProfileParseError, ValidationError
from .mig import INSTANCE_SIZES

DEFAULT_BATCH_SIZES = (1, 2, 4, 8, 16, 32, 64, 128)
DEFAULT_PROCESS_COUNTS = (1, 2, 3)
DEFAULT_MEMORY_MAP: dict[int, float] = {1: 10.0, 2: 20.0, 3: 40.0, 4: 40.0, 7: 80.0}

CSV_HEADER = ("model_id", "instance_size", "batch_size", "process_count",
              "throughput_rps", "latency_ms", "memory_gb")

ProfileKey = tuple[int, int, int]


@dataclass(frozen=True)
class ProfilePoint:
    """One (instance size, batch, procs) operating point (profiles.py:44-76)."""

    model_id: str
    instance_size: int
    batch_size: int
    process_count: int
    throughput: float
    latency: float
    memory_required: float = 0.0

    def __post_init__(self) -> None:
        if self.instance_size not in INSTANCE_SIZES:
            raise ValidationError(f"instance_size {self.instance_size} not in {INSTANCE_SIZES}")
        if self.batch_size < 1:
            raise ValidationError(f"batch_size must be positive, got {self.batch_size}")
        if self.process_count < 1:
            raise ValidationError(f"process_count must be positive, got {self.process_count}")
        if not self.throughput > 0:
            raise ValidationError(f"throughput must be > 0, got {self.throughput}")
        if not self.latency > 0:
            raise ValidationError(f"latency must be > 0, got {self.latency}")
        if self.memory_required < 0:
            raise ValidationError(f"memory_required must be >= 0, got {self.memory_required}")

    @property
    def key(self) -> ProfileKey:
        return (self.instance_size, self.batch_size, self.process_count)


@dataclass(frozen=True)
class ProfileTable:
    """Immutable, key-unique, key-sorted points of one model (profiles.py:79-129)."""

    model_id: str
    points: tuple[ProfilePoint, ...] = field(default=())

    def __post_init__(self) -> None:
        seen: set[ProfileKey] = set()
        for p in self.points:
            if p.model_id != self.model_id:
                raise ValidationError(f"point for model {p.model_id!r} in table {self.model_id!r}")
            if p.key in seen:
                raise ValidationError(f"duplicate profile key {p.key} for model {self.model_id!r}")
            seen.add(p.key)
        object.__setattr__(self, "points", tuple(sorted(self.points, key=lambda p: p.key)))

    def __len__(self) -> int:
        return len(self.points)

    def __iter__(self) -> Iterator[ProfilePoint]:
        return iter(self.points)

    def get(self, instance_size: int, batch_size: int, process_count: int) -> ProfilePoint:
        key = (instance_size, batch_size, process_count)
        for p in self.points:
            if p.key == key:
                return p
        raise KeyError(key)

    def restrict(self, process_counts: Iterable[int] | None = None,
                 batch_sizes: Iterable[int] | None = None) -> "ProfileTable":
        procs = set(process_counts) if process_counts is not None else None
        batches = set(batch_sizes) if batch_sizes is not None else None
        kept = tuple(p for p in self.points
                     if (procs is None or p.process_count in procs)
                     and (batches is None or p.batch_size in batches))
        return ProfileTable(self.model_id, kept)


def _parse_row(fields: Mapping[str, str], row: int) -> ProfilePoint:
    try:
        return ProfilePoint(
            model_id=fields["model_id"],
            instance_size=int(fields["instance_size"]),
            batch_size=int(fields["batch_size"]),
            process_count=int(fields["process_count"]),
            throughput=float(fields["throughput_rps"]),
            latency=float(fields["latency_ms"]),
            memory_required=float(fields["memory_gb"]),
        )
    except (KeyError, TypeError, ValueError) as exc:
        raise ProfileParseError(str(exc), row=row) from exc


def _as_text(source) -> str:
    if isinstance(source, (str, Path)) and "\n" not in str(source):
        return Path(source).read_text(encoding="utf-8")
    if isinstance(source, str):
        return source
    if isinstance(source, bytes):
        return source.decode("utf-8")
    data = source.read()
    return data.decode("utf-8") if isinstance(data, bytes) else data


def load_profile_table(source, format: str = "csv") -> ProfileTable:
    """Load one model's table from CSV or JSON (profiles.py:160-198)."""
    text = _as_text(source)
    points: list[ProfilePoint] = []
    if format == "csv":
        reader = csv.DictReader(io.StringIO(text))
        if reader.fieldnames is None or tuple(reader.fieldnames) != CSV_HEADER:
            raise ProfileParseError(f"expected header {','.join(CSV_HEADER)}, got {reader.fieldnames}")
        for i, row in enumerate(reader, start=2):
            if None in row or None in row.values():
                raise ProfileParseError("wrong field count", row=i)
            points.append(_parse_row(row, i))
    elif format == "json":
        try:
            rows = json.loads(text)
        except json.JSONDecodeError as exc:
            raise ProfileParseError(str(exc)) from exc
        if not isinstance(rows, list):
            raise ProfileParseError("top-level JSON value must be an array")
        for i, row in enumerate(rows):
            if not isinstance(row, dict):
                raise ProfileParseError("array element is not an object", row=i)
            points.append(_parse_row({k: str(v) for k, v in row.items()}, i))
    else:
        raise ValidationError(f"unknown profile format {format!r}")
    model_ids = {p.model_id for p in points}
    if len(model_ids) > 1:
        raise ValidationError(f"profile source mixes models {sorted(model_ids)}; one model per table")
    return ProfileTable(model_id=points[0].model_id if points else "", points=tuple(points))


def _format_number(x: float) -> str:
    return str(int(x)) if float(x).is_integer() else repr(float(x))


def serialize_profile_table(table: ProfileTable, format: str = "csv") -> str:
    """Inverse of load_profile_table (profiles.py:207-240)."""
    if format == "csv":
        out = io.StringIO()
        w = csv.writer(out, lineterminator="\n")
        w.writerow(CSV_HEADER)
        for p in table.points:
            w.writerow([p.model_id, p.instance_size, p.batch_size, p.process_count,
                        _format_number(p.throughput), _format_number(p.latency),
                        _format_number(p.memory_required)])
        return out.getvalue()
    if format == "json":
        rows = [{"model_id": p.model_id, "instance_size": p.instance_size,
                 "batch_size": p.batch_size, "process_count": p.process_count,
                 "throughput_rps": p.throughput, "latency_ms": p.latency,
                 "memory_gb": p.memory_required} for p in table.points]
        return json.dumps(rows, indent=2) + "\n"
    raise ValidationError(f"unknown profile format {format!r}")


def load_profile_tables(directory: str | Path) -> dict[str, ProfileTable]:
    """Every <model>.csv / .json table in a directory (profiles.py:243-257)."""
    directory = Path(directory)
    tables: dict[str, ProfileTable] = {}
    for path in sorted(directory.iterdir()):
        if path.suffix == ".csv":
            table = load_profile_table(path, format="csv")
        elif path.suffix == ".json":
            table = load_profile_table(path, format="json")
        else:
            continue
        if table.model_id in tables:
            raise ValidationError(f"model {table.model_id!r} appears twice in {directory}")
        tables[table.model_id] = table
    return tables


def check_memory_map(memory_map: Mapping[int, float] | None) -> dict[int, float]:
    mm = DEFAULT_MEMORY_MAP if memory_map is None else dict(memory_map)
    missing = [s for s in INSTANCE_SIZES if s not in mm]
    if missing:
        raise ValidationError(f"memory_map missing instance sizes {missing}")
    return {s: float(mm[s]) for s in INSTANCE_SIZES}


def filter_feasible(table: ProfileTable, memory_map: Mapping[int, float] | None = None) -> ProfileTable:
    """Drop points whose memory demand exceeds the instance capacity (profiles.py:260-271).

    Table preparation, outside the planner's timed region in the reference
    (pipeline.py:94); the device path applies the same predicate while
    packing (batch.TableSet).
    """
    mm = check_memory_map(memory_map)
    return ProfileTable(table.model_id,
                        tuple(p for p in table.points if p.memory_required <= mm[p.instance_size]))
