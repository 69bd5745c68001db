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
square deltas are recognised (declared `kind`, or an exact AST match)
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
    ('sum' | 'max') is the device reduce; None means "look at fn's source"."""

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
    ('abs' | 'square') is the device delta; None means "look at fn's source"."""

    fn: Callable[[Any, Any], Any]
    on_arrays: Optional[Callable] = None
    kind: Optional[str] = field(default=None, compare=False)

    def __call__(self, new: Any, old: Any) -> Any:
        return self.fn(new, old)


# ---------------------------------------------------------------- recognition
#
# A user Combinator / Delta maps onto the engine's SUM / MAX reduce and
# |new-old| / (new-old)**2 delta enums only when it says so (`kind`) or when
# its source IS one of those expressions (checked on the AST, names resolved
# to the builtins).  Anything else -- including functions that agree with a
# built-in on many inputs but not on all -- is compiled as written (jit.py)
# or, for the hand-written kernels, rejected with DeviceUnsupported.  No
# classification by sampling: a near-miss would silently diverge from the
# reference's fold of op.fn (patterns.py:85-122, loop.py:163-191).


def _lambda_expr(fn):
    """(param names, returned expression) of a one-expression function, or None."""
    import ast

    try:
        from .jit import _func_node

        node = _func_node(fn)
    except Exception:
        return None
    a = node.args
    if a.vararg or a.kwarg or a.kwonlyargs or a.defaults or len(a.args) != 2:
        return None
    if isinstance(node, ast.Lambda):
        body = node.body
    else:
        stmts = [st for st in node.body
                 if not (isinstance(st, ast.Expr) and isinstance(st.value, ast.Constant))]
        if len(stmts) != 1 or not isinstance(stmts[0], ast.Return) or stmts[0].value is None:
            return None
        body = stmts[0].value
    return [x.arg for x in a.args], body


def _resolves_to(fn, name: str, target) -> bool:
    """`name` inside fn means the builtin / module object `target`."""
    import builtins
    import inspect

    try:
        cv = inspect.getclosurevars(fn)
    except Exception:
        return False
    for scope in (cv.nonlocals, cv.globals):
        if name in scope:
            return scope[name] is target
    return getattr(builtins, name, None) is target


def _is_name(node, name) -> bool:
    import ast

    return isinstance(node, ast.Name) and node.id == name


def _is_diff(node, x, y) -> bool:
    import ast

    return (isinstance(node, ast.BinOp) and isinstance(node.op, ast.Sub)
            and _is_name(node.left, x) and _is_name(node.right, y))


def _ast_combinator(fn) -> Optional[str]:
    import ast

    le = _lambda_expr(fn)
    if le is None:
        return None
    (a, b), e = le
    if isinstance(e, ast.BinOp) and isinstance(e.op, ast.Add):  # a + b / b + a
        if {getattr(e.left, "id", None), getattr(e.right, "id", None)} == {a, b} \
                and isinstance(e.left, ast.Name) and isinstance(e.right, ast.Name):
            return "sum"
    if isinstance(e, ast.IfExp) and _is_name(e.body, a) and _is_name(e.orelse, b) \
            and isinstance(e.test, ast.Compare) and len(e.test.ops) == 1:
        t, op, r = e.test.left, e.test.ops[0], e.test.comparators[0]
        # the reference's max: `a if b < a else b` (patterns.py:205-211), or `a if a > b else b`
        if (isinstance(op, ast.Lt) and _is_name(t, b) and _is_name(r, a)) or \
                (isinstance(op, ast.Gt) and _is_name(t, a) and _is_name(r, b)):
            return "max"
    if isinstance(e, ast.Call) and isinstance(e.func, ast.Name) and not e.keywords \
            and len(e.args) == 2 and _is_name(e.args[0], a) and _is_name(e.args[1], b) \
            and _resolves_to(fn, e.func.id, max):
        return "max"
    return None


def _ast_delta(fn) -> Optional[str]:
    import ast

    le = _lambda_expr(fn)
    if le is None:
        return None
    (n, o), e = le
    diff = lambda d: _is_diff(d, n, o) or _is_diff(d, o, n)  # noqa: E731
    if isinstance(e, ast.Call) and not e.keywords and len(e.args) == 1 and diff(e.args[0]):
        f = e.func
        if isinstance(f, ast.Name) and _resolves_to(fn, f.id, abs):
            return "abs"
    if isinstance(e, ast.BinOp) and isinstance(e.op, ast.Pow) and diff(e.left) \
            and isinstance(e.right, ast.Constant) and type(e.right.value) is int \
            and e.right.value == 2:
        return "square"
    return None


def combinator_kind(op: Combinator) -> str:
    """'sum' or 'max' for the device reduce, else DeviceUnsupported (the
    JIT then compiles op.fn itself)."""
    if getattr(op, "kind", None) is not None:
        return op.kind
    import operator

    k = "sum" if op.fn is operator.add else "max" if op.fn is max else _ast_combinator(op.fn)
    if k is None:
        raise DeviceUnsupported("combinator is not exactly `a + b` or `a if b < a else b`; "
                                "no built-in device reduce for it")
    return k


def delta_kind(d: Optional[Delta]) -> str:
    """'none', 'abs' or 'square' for the device delta, else DeviceUnsupported."""
    if d is None:
        return "none"
    if getattr(d, "kind", None) is not None:
        return d.kind
    k = _ast_delta(d.fn)
    if k is None:
        raise DeviceUnsupported("delta is not exactly `abs(new - old)` or `(new - old) ** 2`; "
                                "no built-in device delta for it")
    return k


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
    """Left fold of all elements from the identity, row-major
    (patterns.py:143-147), on the device.  SUM / MAX combinators
    (declared or recognised exactly, combinator_kind) run sk_reduce_fold:
    bit-identical to the sequential fold -- integer sums are order-free,
    float MAX keeps `a if b < a else b`'s NaN / tie behaviour, float SUM is
    folded sequentially in the element type (numpy NEP 50).  Any other
    combinator, or an identity whose type would change the arithmetic
    (a float identity on integers, a numpy scalar of another width), runs
    as a one-iteration loop of the identity stencil whose reduce is the
    compiled combinator."""
    import ctypes as C

    from . import _native

    lib = _native.require_cuda()
    import numpy as np
    import torch

    try:
        kind = combinator_kind(op)
    except DeviceUnsupported:
        kind = None
    t = a.tensor(device="cuda") if kind is not None else None
    plan = None if t is None else _fold_plan(kind, t.dtype, op.identity)
    if plan is not None and kind == "max" and t.is_floating_point() and not _is_ifexp_max(op):
        plan = None  # builtin max() keeps the first of equal values and skips NaN: fold it as written
    if plan is None:
        from .loop import loop_stencil_reduce, stop_after

        _, rep = loop_stencil_reduce(0, ElementalFn(point=lambda nb, env: nb.center, k=0), op,
                                     stop_after(1), a)
        return rep.final_reduce
    dt, ident_bytes, host_post = plan
    t = t.contiguous().reshape(-1)
    out = torch.zeros(1, dtype=torch.float64, device=t.device)
    buf = C.create_string_buffer(ident_bytes, 8)
    _native.check(lib.sk_reduce_fold(C.c_void_p(t.data_ptr()), t.numel(), dt,
                                     _native.SK_REDUCE_SUM if kind == "sum" else _native.SK_REDUCE_MAX,
                                     buf, C.c_void_p(out.data_ptr()),
                                     _native.stream_handle(torch.cuda.current_stream(t.device))))
    raw = out.cpu().numpy().view(np.uint8)
    return host_post(raw)


def _fold_plan(kind, tdtype, ident):
    """(sk dtype, identity bytes, result decoder) for sk_reduce_fold, or None
    when the reference's arithmetic would differ from the kernel's."""
    import numpy as np
    import torch

    from . import _native

    ints = {torch.uint8: _native.SK_U8, torch.int32: _native.SK_I32, torch.int64: _native.SK_I64}
    if tdtype in ints:
        if isinstance(ident, (bool, np.bool_)):
            return None
        if isinstance(ident, (int, np.integer)):
            iv = int(ident)
            if not -(1 << 63) <= iv < (1 << 63):
                return None
            if kind == "sum":
                return ints[tdtype], np.int64(iv).tobytes(), lambda r: int(r[:8].view(np.int64)[0])
            # MAX: the kernel folds from int64's minimum; the identity joins last
            # (integers: no NaN, equal values are equal)
            return (ints[tdtype], np.int64(np.iinfo(np.int64).min).tobytes(),
                    lambda r: _max_join(iv, int(r[:8].view(np.int64)[0])))
        if kind == "max" and isinstance(ident, float):
            return (ints[tdtype], np.int64(np.iinfo(np.int64).min).tobytes(),
                    lambda r: _max_join(ident, int(r[:8].view(np.int64)[0])))
        return None  # a float identity makes the reference's sum float arithmetic
    if tdtype not in (torch.float32, torch.float64):
        return None
    npdt = np.float32 if tdtype == torch.float32 else np.float64
    weak = isinstance(ident, (int, float)) and not isinstance(ident, bool)
    if not weak and not (isinstance(ident, np.floating) and ident.dtype == npdt):
        return None
    iv = npdt(ident)  # NEP 50: a Python scalar takes the array's type
    if npdt == np.float32:
        dec = lambda r: np.float32(r[:4].view(np.float32)[0])  # noqa: E731
    else:
        dec = lambda r: float(r[:8].view(np.float64)[0])  # noqa: E731
    return (_native.SK_F32 if npdt == np.float32 else _native.SK_F64, iv.tobytes(), dec)


def _is_ifexp_max(op) -> bool:
    """The reference's `a if b < a else b` (declared by max_combinator, or
    that exact expression), as opposed to the builtin max()."""
    import ast

    if getattr(op, "kind", None) == "max" and op.fn is not max:
        le = _lambda_expr(op.fn)
        return le is None or not isinstance(le[1], ast.Call)
    le = _lambda_expr(op.fn)
    return le is not None and isinstance(le[1], ast.IfExp) and _ast_combinator(op.fn) == "max"


def _max_join(ident, m):
    """`a if b < a else b` of the identity and the data's maximum (ints)."""
    return ident if m < ident else m


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
