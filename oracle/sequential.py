"""CPU oracle for user elemental functions: the reference's sequential route.

TEST INFRASTRUCTURE ONLY (like oracle/stencil_oracle.py): imported by
`tests/` only, as the checker for the run-time compiled kernels
(paper_1609_04567_b200/jit.py).  It runs the user's own Python point
function on every element, which is the reference's semantic definition:

  * SequentialExecutor.step (loop.py:154-191): row-major visit, window of
    radius k with ABSENT off the grid (neighborhood_at /
    indexed_neighborhood_at, grid.py:270-324), `new = point(nb, env)`,
    `acc = op(acc, delta(new, old))` (or `op(acc, new)`) from the identity;
    an exception becomes StencilError at that index (loop.py:178-181);
  * _drive (loop.py:198-224): at least one iteration, cond(value, it, state)
    after each, the cap sets `exhausted`, final_reduce = last value;
  * the reduce is the ParallelExecutor's (parallel_loop's executor): each of
    the P row blocks folded from the identity, then the partials folded in
    ascending order from the identity (partition.py:642-646, 319-366).

Windows are built with small local classes that honour the reference's
Neighborhood interface (at, center, center_index, values, pairs, k, len,
iteration); the ABSENT marker is passed in, so a function written against
either package's ABSENT sees its own marker.  Sizes are kept small in the
tests: this is Python per element.
"""

from __future__ import annotations

from typing import Any, Callable, Optional

import numpy as np


class _Nb:
    __slots__ = ("k", "center_index", "entries", "_absent")

    def __init__(self, k, center_index, entries, absent):
        self.k = k
        self.center_index = center_index
        self.entries = entries
        self._absent = absent

    @property
    def center(self):
        if len(self.center_index) == 1:
            return self.entries[self.k]
        w = 2 * self.k + 1
        return self.entries[self.k * w + self.k]

    def at(self, *delta):
        k, w = self.k, 2 * self.k + 1
        if len(delta) == 1:
            return self.entries[k + delta[0]]
        return self.entries[(k + delta[0]) * w + (k + delta[1])]

    def values(self):
        return [v for v in self.entries if v is not self._absent]

    def __iter__(self):
        return iter(self.entries)

    def __len__(self):
        return len(self.entries)


class _IndexedNb(_Nb):
    __slots__ = ()

    def pairs(self):
        return [p for p in self.entries if p is not self._absent]

    def values(self):
        return [p[0] for p in self.entries if p is not self._absent]


class OracleError(RuntimeError):
    """The user function raised: (index, cause) like the reference's StencilError."""

    def __init__(self, index, cause):
        self.index = index
        self.cause = cause
        super().__init__(f"failed at {index}: {cause!r}")


def _windows_1d(front, n, k, indexed, absent):
    cls = _IndexedNb if indexed else _Nb
    for i in range(n):
        entries = []
        for a in range(2 * k + 1):
            gi = i - k + a
            if 0 <= gi < n:
                entries.append((front[gi], (gi,)) if indexed else front[gi])
            else:
                entries.append(absent)
        yield (i,), cls(k, (i,), tuple(entries), absent)


def _windows(front, rows, cols, k, indexed, absent):
    w = 2 * k + 1
    cls = _IndexedNb if indexed else _Nb
    for i in range(rows):
        for j in range(cols):
            entries = []
            for a in range(w):
                gi = i - k + a
                for b in range(w):
                    gj = j - k + b
                    if 0 <= gi < rows and 0 <= gj < cols:
                        v = front[gi][gj]
                        entries.append((v, (gi, gj)) if indexed else v)
                    else:
                        entries.append(absent)
            yield (i, j), cls(k, (i, j), tuple(entries), absent)


def sequential_loop(point: Callable, k: int, op: Callable, identity: Any,
                    cond: Callable, grid, env=None, delta: Optional[Callable] = None,
                    indexed: bool = False, max_iterations: int = 10_000, absent=None,
                    partitions: int = 1, state=None):
    """Run the loop; returns (rows of values, iterations, final_reduce, exhausted).
    A flat sequence is a rank-1 grid (the reference's 1D route,
    partition.py:369-404).

    `grid` is a 2D sequence of Python values (numpy scalars keep their type,
    as in a reference Grid built from an array's elements); `cond(value, it,
    state)` as the reference's Condition.fn."""
    if absent is None:
        from paper_1609_04567_b200.grid import ABSENT as absent  # the product's marker
    one_d = not isinstance(grid[0], (list, tuple, np.ndarray))
    front = list(grid) if one_d else [list(r) for r in grid]
    rows = len(front)
    cols = 1 if one_d else len(front[0])
    bounds = [(0, rows)]
    if partitions > 1:
        from oracle.stencil_oracle import split_ranges

        bounds = split_ranges(rows, partitions)
    s = state.init() if state is not None else None
    it = 0
    stopped = False
    value = None
    while True:
        it += 1
        back = [None] * rows if one_d else [[None] * cols for _ in range(rows)]
        part_acc = [identity for _ in bounds]
        wins = _windows_1d(front, rows, k, indexed, absent) if one_d else \
            _windows(front, rows, cols, k, indexed, absent)
        for idx, nb in wins:
            try:
                new = point(nb, env)
            except Exception as e:
                raise OracleError(idx, e) from e
            i = idx[0]
            old = front[i] if one_d else front[i][idx[1]]
            if one_d:
                back[i] = new
            else:
                back[i][idx[1]] = new
            p = next(q for q, (lo, hi) in enumerate(bounds) if lo <= i < hi)
            part_acc[p] = op(part_acc[p], new if delta is None else delta(new, old))
        value = identity  # host combine of the partials (partition.py:642-646)
        for a in part_acc:
            value = op(value, a)
        front = back
        if state is not None:
            s = state.update(s, it, value)
        if cond(value, it, s):
            stopped = True
            break
        if it >= max_iterations:
            break
    return front, it, value, not stopped
