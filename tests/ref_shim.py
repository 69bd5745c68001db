"""Test-only stand-in for the reference's loop front end (stencilkit/loop.py,
grid.py, patterns.py) -- what a `stencilkit` user's call goes through when
they keep `stencilkit` and pass our DeviceExecutor as `executor=`
(INTEGRATION.md section 2).  /root/reference does not exist on the GPU box,
so this restates, for the tests, the reference's observable host protocol:

* its value types with the reference's field names: a list-backed `Grid`
  (`dims`, `data`), `ElementalFn(point, k, block, pad_mode, pad_value)`,
  `Combinator(fn, identity, on_array)`, `Delta(fn, on_arrays)`,
  `LoopPlan`, `Condition(fn, max_iterations)`, `LoopState`, `LoopReport`
  (grid.py:47-176, patterns.py:41-122, loop.py:43-110);
* `_as_plan` wrapping a bare callable / our ElementalFn as the `point` of
  its own ElementalFn (loop.py:113-121);
* `_drive` (loop.py:198-224): begin; repeat { step; state.update; cond }
  with at least one iteration, the cap setting `exhausted`, the last value
  as `final_reduce`; finish; abort on any exception -- host-driven, no
  device loop.

tests/test_ref_shim.py pins this stand-in against the real reference in
the build container (same executor call sequence, same reports).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Callable, Optional


class Grid:
    def __init__(self, dims, data):
        self.dims = tuple(dims)
        self.data = list(data)


@dataclass(frozen=True)
class ElementalFn:
    point: Callable
    k: int
    block: Optional[Callable] = None
    pad_mode: str = "constant"
    pad_value: Any = 0


@dataclass(frozen=True)
class Combinator:
    fn: Callable
    identity: Any
    on_array: Optional[Callable] = None


@dataclass(frozen=True)
class Delta:
    fn: Callable
    on_arrays: Optional[Callable] = None


@dataclass(frozen=True)
class Condition:
    fn: Callable
    max_iterations: int = 10_000


@dataclass(frozen=True)
class LoopState:
    init: Callable
    update: Callable


@dataclass
class LoopReport:
    iterations: int
    final_reduce: Any
    copies: Any
    exhausted: bool = False


@dataclass(frozen=True)
class LoopPlan:
    fn: ElementalFn
    k: int
    op: Combinator
    env: Any = None
    indexed: bool = False
    delta: Optional[Delta] = None


def max_combinator(identity):
    return Combinator(lambda a, b: a if b < a else b, identity)


def sum_combinator(identity=0):
    return Combinator(lambda a, b: a + b, identity)


def _as_plan(f, k, op, env, indexed, delta):
    if isinstance(f, ElementalFn):
        if k is not None and k != f.k:
            raise ValueError(f"explicit radius {k} disagrees with kernel radius {f.k}")
        k = f.k
    elif k is None:
        raise ValueError("radius required for a bare callable")
    else:
        f = ElementalFn(point=f, k=k)  # a foreign kernel object becomes the point
    if not isinstance(op, Combinator):
        raise TypeError("op must be a Combinator (it carries the identity)")
    if delta is not None and not isinstance(delta, Delta):
        delta = Delta(delta)
    return LoopPlan(fn=f, k=k, op=op, env=env, indexed=indexed, delta=delta)


def _drive(plan, cond, state, grid, executor, max_iterations):
    if not isinstance(cond, Condition):
        cond = Condition(cond) if max_iterations is None else Condition(cond, max_iterations)
    elif max_iterations is not None:
        cond = Condition(cond.fn, max_iterations)
    run = executor.begin(plan, grid)
    s = state.init() if state is not None else None
    try:
        it, value, stopped = 0, None, False
        while not stopped:
            it += 1
            value = executor.step(run)
            if state is not None:
                s = state.update(s, it, value)
            stopped = bool(cond.fn(value, it, s))
            if not stopped and it >= cond.max_iterations:
                break
        out, copies = executor.finish(run)
    except BaseException:
        executor.abort(run)
        raise
    return out, LoopReport(iterations=it, final_reduce=value, copies=copies,
                           exhausted=not stopped)


def loop_stencil_reduce(k, f, op, cond, a, env=None, executor=None, max_iterations=None):
    return _drive(_as_plan(f, k, op, env, False, None), cond, None, a, executor, max_iterations)


def loop_stencil_reduce_d(k, f, delta, op, cond, a, env=None, executor=None, indexed=False,
                          max_iterations=None):
    return _drive(_as_plan(f, k, op, env, indexed, delta), cond, None, a, executor,
                  max_iterations)


def loop_stencil_reduce_s(k, f, op, cond, state, a, env=None, executor=None, delta=None,
                          indexed=False, max_iterations=None):
    return _drive(_as_plan(f, k, op, env, indexed, delta), cond, state, a, executor,
                  max_iterations)
