"""Benchmark rows and their CSV form (reference: bench.py:1-130; SURVEY next-3).

RunSpec describes a run (app, input id, partitions, farm width, deployment
mode, seed), BenchRow its outcome -- the LoopReport's iteration count and
final reduce plus the copy ledger's fill / halo / readback counts -- and
emit_csv writes rows sorted by their identifying columns, header first,
floats with six significant digits, RFC 4180 quoting.  Column set and order
are the reference's, so CSVs from either package line up.
"""

from __future__ import annotations

import csv
import io
import os
from dataclasses import astuple, dataclass, fields
from typing import Iterable, Union

from .grid import GridError
from .partition import DeploymentMode

COLUMNS = ("app", "input_id", "partitions", "width", "mode", "seed", "iterations", "wall_ms",
           "fill_events", "halo_elems", "readback_events", "reduce_final")
_KEY = COLUMNS[:6]  # rows sort on their identifying columns


@dataclass(frozen=True)
class RunSpec:
    """What ran: app, problem id and the deployment shape (bench.py:36-57)."""

    app: str
    input_id: str
    partitions: int = 1
    width: int = 1
    mode: DeploymentMode = DeploymentMode.ONE_TO_ONE
    seed: int = 42

    def __post_init__(self):
        problems = []
        if not self.app:
            problems.append("app name must be non-empty")
        if self.partitions < 1:
            problems.append(f"partitions must be >= 1, got {self.partitions}")
        if self.width < 1:
            problems.append(f"width must be >= 1, got {self.width}")
        if problems:
            raise GridError(problems[0])
        m = DeploymentMode.parse(self.mode)
        object.__setattr__(self, "mode", m)
        if m is DeploymentMode.ONE_TO_N and self.partitions < 2:
            raise GridError("1:n deployment needs at least 2 partitions")


@dataclass(frozen=True)
class BenchRow:
    """One CSV line (bench.py:60-94)."""

    app: str
    input_id: str
    partitions: int
    width: int
    mode: str
    seed: int
    iterations: int
    wall_ms: float
    fill_events: int
    halo_elems: int
    readback_events: int
    reduce_final: float

    @classmethod
    def from_run(cls, spec: RunSpec, report, wall_ms: float) -> "BenchRow":
        led = report.copies
        return cls(spec.app, spec.input_id, spec.partitions, spec.width, spec.mode.value,
                   spec.seed, report.iterations, wall_ms, led.fill_events, led.halo_elems,
                   led.readback_events, report.final_reduce)


if tuple(f.name for f in fields(BenchRow)) != COLUMNS:  # keep the two in step
    raise ImportError("BenchRow fields drifted from COLUMNS")


def _fmt(v) -> str:
    if isinstance(v, bool):
        raise GridError("bool has no CSV representation here")
    return format(v, ".6g") if isinstance(v, float) else str(v)


def emit_csv(rows: Iterable[BenchRow],
             out: Union[str, os.PathLike, io.TextIOBase, None] = None) -> str:
    """CSV text of `rows` (sorted, header first), also written to `out` (a
    path or an open text file) when given (bench.py:112-130)."""
    ordered = sorted(rows, key=lambda r: astuple(r)[:len(_KEY)])
    text = io.StringIO()
    w = csv.writer(text)
    w.writerow(COLUMNS)
    w.writerows([_fmt(v) for v in astuple(r)] for r in ordered)
    s = text.getvalue()
    if isinstance(out, (str, os.PathLike)):
        with open(out, "w", newline="", encoding="ascii") as fh:
            fh.write(s)
    elif out is not None:
        out.write(s)
    return s
