"""Kernel descriptors and the map/reduce/stencil vocabulary.

Mirrors the reference's patterns module (patterns.py:29-211): StencilError,
ElementalFn, Combinator, Delta, apply_to_all/map_pattern, reduce_all/
reduce_pattern, stencil_apply(_indexed), sum_combinator, max_combinator.

What changes is what a descriptor carries.  In the reference an
ElementalFn is a Python callable (+ an optional numpy block form) that the
runtime calls per element or per block.  Here an ElementalFn may carry a
`device` descriptor naming one of the engine's hand-written sm_100a kernels
and its dtype-rounded constants; without one, its Python `point` function
(and the plan's Combinator / Delta callables) are translated and compiled
for the device at run time (jit.py).  Sum / max combinators and abs /
square deltas are recognised (declared `kind`, or by probing the callable)
and map onto the engine's reduce / delta enums.  Anything that cannot be
compiled is rejected with DeviceUnsupported -- there is no host path.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Callable, Optional

from .grid import Grid, GridError


class StencilError(RuntimeError):
    """Elemental-function failure, tagged with the element (patterns.py:29-38)."""

    def __init__(self, index, cause, partition: Optional[int] = None):
        self.index = tuple(index) if index is not None else None
        self.partition = partition
        where = f"index {self.index}" if self.index is not None else "block kernel"
        if partition is not None:
            where += f" (partition {partition})"
        super().__init__(f"elemental function failed at {where}: {cause!r}")


class DeviceUnsupported(NotImplementedError):
    """The operation has no sm_100a kernel in this engine (and no host fallback)."""


@dataclass(frozen=True)
class DeviceKernel:
    """Names an engine kernel plus its parameters (see include/stencilkit_b200.h).

    name     'helmholtz' | 'sobel' | 'amf' | 'restore' | 'life'
    params   kernel constants as Python floats (rounded to the grid dtype by
             the engine, like numpy's NEP 50 weak scalars)
    """

    name: str
    params: tuple = ()


@dataclass(frozen=True)
class ElementalFn:
    """Stencil kernel: per-element function, radius, optional block form,
    pad semantics (patterns.py:41-68), plus the device descriptor."""

    point: Callable[[Any, Any], Any]
    k: int
    block: Optional[Callable] = None
    pad_mode: str = "constant"
    pad_value: Any = 0
    device: Optional[DeviceKernel] = field(default=None, compare=False)

    def __post_init__(self):
        if self.k < 0:
            raise ValueError(f"radius must be >= 0, got {self.k}")
        if self.pad_mode not in ("constant", "edge"):
            raise ValueError(f"unknown pad mode {self.pad_mode!r}")

    def __call__(self, nb, env: Any = None) -> Any:
        return self.point(nb, env)


def _radius(f, k: Optional[int]) -> int:
    if isinstance(f, ElementalFn):
        if k is not None and k != f.k:
            raise ValueError(f"explicit radius {k} disagrees with kernel radius {f.k}")
        return f.k
    if k is None:
        raise ValueError("radius required for a bare callable")
    return k


@dataclass(frozen=True)
class Combinator:
    """Associative combiner with identity (patterns.py:85-107).  `kind`
    ('sum' | 'max') is the device reduce; None means "probe fn"."""

    fn: Callable[[Any, Any], Any]
    identity: Any
    on_array: Optional[Callable] = None
    kind: Optional[str] = field(default=None, compare=False)

    def __call__(self, a: Any, b: Any) -> Any:
        return self.fn(a, b)

    def fold(self, values) -> Any:
        acc = self.identity
        for v in values:
            acc = self.fn(acc, v)
        return acc


@dataclass(frozen=True)
class Delta:
    """Per-element change measure (patterns.py:110-122).  `kind`
    ('abs' | 'square') is the device delta; None means "probe fn"."""

    fn: Callable[[Any, Any], Any]
    on_arrays: Optional[Callable] = None
    kind: Optional[str] = field(default=None, compare=False)

    def __call__(self, new: Any, old: Any) -> Any:
        return self.fn(new, old)


# ---------------------------------------------------------------- recognition

_PAIRS = ((1.5, 2.25), (2.25, 1.5), (-3.0, 0.5), (0.0, 7.0), (5.0, 3.0), (-2.0, -9.5))


def _probe(fn, expect) -> bool:
    try:
        return all(fn(a, b) == expect(a, b) for a, b in _PAIRS)
    except Exception:
        return False


def combinator_kind(op: Combinator) -> str:
    """'sum' or 'max' for the device reduce, else DeviceUnsupported."""
    if getattr(op, "kind", None) is not None:
        return op.kind
    if _probe(op.fn, lambda a, b: a + b):
        return "sum"
    if _probe(op.fn, lambda a, b: a if b < a else b):
        return "max"
    raise DeviceUnsupported("combinator is neither a sum nor a max; no device reduce for it")


def delta_kind(d: Optional[Delta]) -> str:
    """'none', 'abs' or 'square' for the device delta, else DeviceUnsupported."""
    if d is None:
        return "none"
    if getattr(d, "kind", None) is not None:
        return d.kind
    if _probe(d.fn, lambda n, o: abs(n - o)):
        return "abs"
    if _probe(d.fn, lambda n, o: (n - o) ** 2):
        return "square"
    raise DeviceUnsupported("delta is neither |new-old| nor (new-old)**2; no device delta for it")


def abs_change() -> Delta:
    """|new - old| (apps/denoise.py:252-254)."""
    import numpy as np

    return Delta(lambda new, old: abs(new - old), on_arrays=lambda n, o: np.abs(n - o), kind="abs")


def sq_change() -> Delta:
    """(new - old)**2 (apps/helmholtz.py:98-100)."""
    return Delta(lambda new, old: (new - old) ** 2, on_arrays=lambda n, o: (n - o) ** 2,
                 kind="square")


def _check_env(env: Any, dims) -> None:
    """env grids must match the loop grid's dims (patterns.py:125-135)."""
    if env is None:
        return
    grids = (env,) if isinstance(env, Grid) else tuple(g for g in env if isinstance(g, Grid)) \
        if isinstance(env, tuple) else ()
    for g in grids:
        if g.dims != tuple(dims):
            raise GridError(f"env dims {g.dims} do not match grid dims {tuple(dims)}")


# ---------------------------------------------------------------- functionals


def stencil_apply(f, k: Optional[int], a: Grid, env: Any = None) -> Grid:
    """One stencil application into a fresh grid (patterns.py:161-177), run on
    the device: a single-iteration loop of the kernel."""
    from .loop import stop_after, loop_stencil_reduce

    k = _radius(f, k)
    _check_env(env, a.dims)
    out, _ = loop_stencil_reduce(k, f, sum_combinator(0), stop_after(1), a, env=env)
    return out


def stencil_apply_indexed(f, k: Optional[int], a: Grid, env: Any = None) -> Grid:
    """Indexed stencil application (patterns.py:180-192): window entries are
    (value, index) pairs."""
    from .loop import stop_after, loop_stencil_reduce_i

    k = _radius(f, k)
    _check_env(env, a.dims)
    out, _ = loop_stencil_reduce_i(k, f, sum_combinator(0), stop_after(1), a, env=env)
    return out


def apply_to_all(f: Callable[[Any], Any], a: Grid) -> Grid:
    """Elementwise map (patterns.py:138-140) on the device: a radius-0
    stencil.  A plain Python `f(x)` is compiled for the device (jit.py); a
    radius-0 ElementalFn is applied as is."""
    if isinstance(f, ElementalFn):
        return stencil_apply(f, f.k, a)
    return stencil_apply(ElementalFn(point=lambda nb, env: f(nb.center), k=0), 0, a)


def reduce_all(op: Combinator, a: Grid) -> Any:
    """Left fold of all elements from the identity (patterns.py:143-147) on
    the device: SUM / MAX directly; any other combinator as a one-iteration
    loop of the identity stencil whose reduce is the compiled combinator."""
    from . import _native

    _native.require_cuda()
    import torch

    try:
        kind = combinator_kind(op)
    except DeviceUnsupported:
        kind = None
    if kind is None:
        from .loop import loop_stencil_reduce, stop_after

        _, rep = loop_stencil_reduce(0, ElementalFn(point=lambda nb, env: nb.center, k=0), op,
                                     stop_after(1), a)
        return rep.final_reduce
    t = a.tensor(device="cuda")
    if t.numel() == 0:
        return op.identity
    v = (t.sum(dtype=torch.float64) if t.is_floating_point() else t.sum()).item() \
        if kind == "sum" else t.max().item()
    return op.fn(op.identity, v)


def map_pattern(f, a: Grid) -> Grid:
    return apply_to_all(f, a)


def reduce_pattern(op: Combinator, a: Grid) -> Any:
    return reduce_all(op, a)


def sum_combinator(identity: Any = 0) -> Combinator:
    """Addition with identity (patterns.py:195-202)."""
    import numpy as np

    return Combinator(lambda a, b: a + b, identity, on_array=lambda arr: np.sum(arr).item(),
                      kind="sum")


def max_combinator(identity: Any) -> Combinator:
    """Maximum with identity (patterns.py:205-211)."""
    import numpy as np

    return Combinator(lambda a, b: a if b < a else b, identity,
                      on_array=lambda arr: np.max(arr).item() if arr.size else identity,
                      kind="max")
