"""User elemental functions on the device.

The reference's pattern API takes *user* functions: the elemental function
(ElementalFn.point, patterns.py:41-68 -- a Python callable over a
Neighborhood, grid.py:201-324), the combinator (Combinator.fn,
patterns.py:85-107) and the delta (Delta.fn, patterns.py:110-122).  The
paper's own API takes the same three as kernel source strings
(Fig. 1).  Both become one CUDA program
here, compiled at run time with NVRTC for sm_100a (csrc/sk_jit.cu) into the
fused sweep of csrc/sk_jit_kernel.cuh -- the same device-resident loop,
deterministic reduce fold and loop test as the built-in kernels.  There is
no host fallback: a function this module cannot translate raises
DeviceUnsupported.

Two ways in:

* `cuda_elemental(body, k, ...)` -- the paper's form: the body of
  `sk_val_t f(const SkNb<V>& nb, const SkEnv& env, SkErr& err)` written
  against csrc/sk_jit_prelude.cuh (`nb.at(di, dj)`, `nb.ok(di, dj)`,
  `nb.center()`, `nb.i`, `nb.j`, `env.get<T>(slot, i, j)`).  Off-grid slots
  read the pad value (block-route semantics, partition.py:551-581).
* any `ElementalFn` whose `point` is a plain Python function: translated from
  its source (a subset of Python: arithmetic, comparisons, if/elif/else,
  for over range / constant tuples / the window, while, break/continue,
  the window API incl. ABSENT tests and indexed pairs, env.at, math /
  builtins).  Semantics follow the reference's point route
  (partition.py:319-366): ABSENT outside the grid, Python int/float
  arithmetic (numpy float32 rules, NEP 50, for float32 grids), and Python's
  exceptions become a StencilError at the lowest failing index.
  Documented differences: ints are 64-bit (Python's are unbounded), and
  transcendental math functions (exp, log, sin, ...) come from CUDA's libm
  (within 2 ulp of glibc's; +, -, *, /, sqrt are exact).
"""

from __future__ import annotations

import ast
import builtins
import ctypes as C
import inspect
import re
import linecache
import math
import os
import threading
from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

from . import _native as N
from .patterns import DeviceUnsupported

# ----------------------------------------------------------------------------- types

BOOL, INT, F32, F64 = "bool", "int", "f32", "f64"
# join order: a numpy float32 value meeting a Python float (F64 here is always
# a Python float: f64 grids hold Python floats, as in the reference's list
# Grid) stays float32 (NEP 50), so F32 ranks above F64
_RANK = {BOOL: 0, INT: 1, F64: 2, F32: 3}
CTYPE = {BOOL: "bool", INT: "long long", F32: "float", F64: "double"}
NP_OF = {BOOL: np.dtype(np.bool_), INT: np.dtype(np.int64), F32: np.dtype(np.float32),
         F64: np.dtype(np.float64)}

# storage dtype -> (C storage type, semantic type)
_STORAGE = {
    np.dtype(np.bool_): ("bool", BOOL), np.dtype(np.int8): ("signed char", INT),
    np.dtype(np.uint8): ("unsigned char", INT), np.dtype(np.int16): ("short", INT),
    np.dtype(np.uint16): ("unsigned short", INT), np.dtype(np.int32): ("int", INT),
    np.dtype(np.uint32): ("unsigned int", INT), np.dtype(np.int64): ("long long", INT),
    np.dtype(np.float32): ("float", F32), np.dtype(np.float64): ("double", F64),
}

# device error codes (csrc/sk_jit_prelude.cuh) -> the exception Python raises
ERR_ABSENT, ERR_ZERODIV, ERR_DOMAIN, ERR_OVERFLOW, ERR_NONE_RET, ERR_GRID, ERR_INDEX, ERR_NEGPOW = \
    1, 2, 3, 4, 5, 6, 7, 8


def error_cause(code: int) -> BaseException:
    from .grid import GridError

    return {
        ERR_ABSENT: TypeError("unsupported operand: ABSENT (off-grid window slot) used as a number"),
        ERR_ZERODIV: ZeroDivisionError("division by zero"),
        ERR_DOMAIN: ValueError("math domain error"),
        ERR_OVERFLOW: ValueError("cannot convert float infinity or NaN to integer"),
        ERR_NONE_RET: TypeError("elemental function returned None"),
        ERR_GRID: GridError("env index out of range"),
        ERR_INDEX: IndexError("window offset outside the radius"),
        ERR_NEGPOW: ValueError("integer power with a negative exponent"),
        9: IndexError("env row beyond this rank's row block and halo"),
    }.get(code, RuntimeError(f"device error code {code}"))


def storage_of(dtype) -> tuple:
    dt = np.dtype(dtype)
    if dt not in _STORAGE:
        raise DeviceUnsupported(f"grid element type {dt} has no device form")
    return _STORAGE[dt]


def _arith(a: str, b: str) -> str:
    """Result type of +, -, *, //, %, ** (Python ints/floats; numpy float32
    scalars with Python-scalar operands stay float32, NEP 50)."""
    if F32 in (a, b):
        return F32  # the other operand is a Python int/float (weak) here
    if F64 in (a, b):
        return F64
    return INT


def _join(a: Optional[str], b: Optional[str]) -> Optional[str]:
    if a is None:
        return b
    if b is None:
        return a
    return a if _RANK[a] >= _RANK[b] else b


class TranslateError(DeviceUnsupported):
    """The Python function uses something with no device translation."""


def _lit(v, t: str) -> str:
    if t == BOOL:
        return "true" if v else "false"
    if t == INT:
        v = int(v)
        if not -(1 << 63) <= v < (1 << 63):
            raise TranslateError(f"integer constant {v} does not fit 64 bits")
        if v == -(1 << 63):
            return "(-9223372036854775807LL-1)"
        return f"({v}LL)" if v >= 0 else f"(-{-v}LL)"
    f = float(v)
    if math.isnan(f):
        s = "__longlong_as_double(0x7ff8000000000000LL)"
        return f"((float){s})" if t == F32 else s
    if math.isinf(f):
        s = "(double)INFINITY" if f > 0 else "(-(double)INFINITY)"
        return f"((float){s})" if t == F32 else s
    if t == F32:
        return f"({float(np.float32(f)).hex()}f)"
    return f"({f.hex()})"


# ----------------------------------------------------------------------------- values


@dataclass
class Val:
    """A translated Python value.

    kind  'num'    a number: C expression `c` of type `t`; `ok` is a C bool
                   expression when it may be ABSENT (None = always present)
          'tuple'  `items` (Vals); `ok` as above for window pairs
          'absent' the ABSENT marker
          'none'   None
          'nb'     the window;  'env' the env argument;  'envgrid' env slot
          'obj'    a translate-time Python object (constants, modules, ...)
    """

    kind: str
    c: str = ""
    t: str = ""
    ok: Optional[str] = None
    items: tuple = ()
    obj: Any = None
    const: Any = None  # Python value when known at translate time
    slot: int = 0      # envgrid slot


def num(c: str, t: str, ok=None, const=None) -> Val:
    return Val("num", c=c, t=t, ok=ok, const=const)


def const_val(v) -> Val:
    if isinstance(v, (bool, np.bool_)):
        return num(_lit(bool(v), BOOL), BOOL, const=bool(v))
    if isinstance(v, (int, np.integer)) and not isinstance(v, bool):
        return num(_lit(int(v), INT), INT, const=int(v))
    if isinstance(v, np.float32):
        return num(_lit(float(v), F32), F32, const=float(v))
    if isinstance(v, (float, np.floating)):
        return num(_lit(float(v), F64), F64, const=float(v))
    return Val("obj", obj=v)


def _is_absent_obj(o) -> bool:
    return type(o).__name__ in ("_Absent", "_AbsentType") and repr(o) == "ABSENT"


# ----------------------------------------------------------------------------- source


_file_cache: dict = {}


_node_cache: dict = {}


def _func_node(fn):
    """AST of a function or lambda, located in its source file (memoised per
    code object: the drop-in loop calls classify the same combinator / delta
    on every call, and locating it walks the whole file's AST)."""
    code = getattr(fn, "__code__", None)
    if code is None:
        raise TranslateError(f"{fn!r} is not a Python function")
    hit = _node_cache.get(code)
    if hit is not None:
        return hit
    node = _func_node_uncached(fn, code)
    if len(_node_cache) > 256:
        _node_cache.clear()
    _node_cache[code] = node
    return node


def _func_node_uncached(fn, code):
    fname = code.co_filename
    lines = linecache.getlines(fname)
    if not lines:
        try:
            lines = inspect.getsourcelines(fn)[0]
            src = "".join(lines)
            tree = ast.parse(_dedent(src))
            base = code.co_firstlineno - 1
        except (OSError, TypeError, SyntaxError) as e:
            raise TranslateError(f"source of {getattr(fn, '__name__', fn)} unavailable: {e}")
    else:
        src = "".join(lines)
        key = (fname, hash(src))
        tree = _file_cache.get(key)
        if tree is None:
            try:
                tree = ast.parse(src)
            except SyntaxError as e:
                raise TranslateError(f"cannot parse {fname}: {e}")
            _file_cache.clear() if len(_file_cache) > 64 else None
            _file_cache[key] = tree
        base = 0
    want_line = code.co_firstlineno - base
    cands = []
    for node in ast.walk(tree):
        if isinstance(node, (ast.Lambda, ast.FunctionDef)):
            line = node.lineno if isinstance(node, ast.Lambda) else (
                node.decorator_list[0].lineno if node.decorator_list else node.lineno)
            if line == want_line or (isinstance(node, ast.FunctionDef) and node.lineno == want_line):
                names = [a.arg for a in node.args.args]
                if names == list(code.co_varnames[:code.co_argcount]):
                    if isinstance(node, ast.FunctionDef) and node.name != code.co_name:
                        continue
                    cands.append(node)
    if not cands:
        raise TranslateError(f"cannot locate the source of {getattr(fn, '__name__', fn)}")
    if len(cands) > 1:  # several lambdas on one line: match source columns
        pos = [(ln, col) for ln, _e, col, ec in code.co_positions()
               if ln is not None and col is not None and ec is not None and ec > col]
        pos = [(ln - base, col) for ln, col in pos]

        def contains(node):
            lo = (node.lineno, node.col_offset)
            hi = (node.end_lineno, node.end_col_offset)
            return bool(pos) and all(lo <= q < hi for q in pos)

        inside = [n for n in cands if contains(n)]
        # nested lambdas also contain the positions: take the innermost
        inside.sort(key=lambda n: (n.end_lineno - n.lineno, n.end_col_offset - n.col_offset))
        if not inside:
            raise TranslateError(f"cannot tell which lambda on line {code.co_firstlineno} "
                                 f"is {getattr(fn, '__qualname__', fn)}")
        return inside[0]
    return cands[0]


def _dedent(src: str) -> str:
    import textwrap

    return textwrap.dedent(src)


# ----------------------------------------------------------------------------- translator


@dataclass
class WindowSpec:
    """What the elemental sees: window radius and element types."""

    k: int
    in_c: str       # C storage type of the window elements
    in_t: str       # semantic type
    indexed: bool
    env: list = field(default_factory=list)   # per slot (C storage type, semantic type)
    env_kind: str = "none"                    # 'none' | 'grid' | 'tuple' | 'obj'
    env_obj: Any = None
    ndim: int = 2                             # 1: a rank-1 grid, run as an (n, 1) column
    dims: tuple = ()                          # the grid's dims (env grids share them)


class Translator:
    """Python function AST -> a C++ __device__ function body.

    Types are inferred by re-running the translation until every local's type
    is stable (a join over its assignments); the final pass emits code."""

    def __init__(self, fn, params: list, role: str, win: Optional[WindowSpec] = None,
                 ctx: Optional["HelperCtx"] = None):
        self.fn = fn
        self.role = role  # 'elemental' | 'delta' | 'combine' | 'helper'
        self.win = win
        self.ctx = ctx if ctx is not None else HelperCtx()
        self.node = _func_node(fn)
        self.params = params  # list of (name -> Val) in order, for non-window roles
        try:
            cv = inspect.getclosurevars(fn)
            self.nonlocals = dict(cv.nonlocals)
            self.globals = dict(cv.globals)
        except Exception:
            self.nonlocals, self.globals = {}, {}
        self.fglobals = getattr(fn, "__globals__", {})
        self.types: dict = {}  # local name -> shape (type str or tuple of shapes)
        self.absentable: set = set()

    # -- driver ---------------------------------------------------------------
    def translate(self):
        """Returns (C body lines, return type)."""
        prev = None
        for _ in range(8):
            self.lines, self.ret_t, self.new_types, self.new_abs = [], None, {}, set()
            self.tmp = 0
            self.depth = 1
            self._bind_params()
            self._body()
            state = (dict(self.new_types), set(self.new_abs))
            if state == prev:
                break
            prev = state
            self.types = {k: v for k, v in self.new_types.items()}
            self.absentable = set(self.new_abs)
        else:
            raise TranslateError("types of the function's locals do not settle")
        if self.ret_t is None:
            raise TranslateError("the function never returns a number")
        decls = []
        for name, shape in sorted(self.types.items()):
            for cname, t in self._flat(f"v_{name}", shape):
                decls.append(f"  {CTYPE[t]} {cname} = 0;")
            if name in self.absentable:
                decls.append(f"  bool v_{name}_ok = true;")
        return decls + self.lines, self.ret_t

    def _flat(self, base, shape):
        if isinstance(shape, tuple):
            out = []
            for i, s in enumerate(shape):
                out += self._flat(f"{base}__{i}", s)
            return out
        return [(base, shape)]

    def _bind_params(self):
        node = self.node
        args = [a.arg for a in node.args.args]
        self.local_vals = {}
        if node.args.vararg or node.args.kwarg or node.args.kwonlyargs or node.args.defaults:
            raise TranslateError(f"{getattr(self.fn, '__qualname__', self.fn)}: only plain "
                                 "positional parameters are supported")
        if self.role == "elemental":
            if len(args) != 2:
                raise TranslateError("an elemental function takes (nb, env)")
            self.local_vals[args[0]] = Val("nb")
            self.local_vals[args[1]] = self._env_val()
        else:
            if len(args) != len(self.params):
                raise TranslateError(f"{self.role} takes {len(self.params)} arguments")
            for a, v in zip(args, self.params):
                self.local_vals[a] = v

    def _env_val(self):
        w = self.win
        if w.env_kind == "grid":
            return Val("envgrid", slot=0)
        if w.env_kind == "tuple":
            return Val("env")
        if w.env_kind == "none":
            return Val("none")
        return self._pyval(w.env_obj)

    def _body(self):
        node = self.node
        if isinstance(node, ast.Lambda):
            v = self.expr(node.body)
            self._return(v)
        else:
            for s in node.body:
                self.stmt(s)
            self.emit("err.set(5); return (RET_T)0;  // fell off the end: returns None")

    # -- emission helpers ------------------------------------------------------
    def emit(self, line: str):
        self.lines.append("  " * self.depth + line)

    def fresh(self, t: str, init: str) -> str:
        self.tmp += 1
        name = f"t{self.tmp}"
        self.emit(f"const {CTYPE[t]} {name} = {init};")
        return name

    def fail(self, node, msg):
        line = getattr(node, "lineno", "?")
        raise TranslateError(f"{getattr(self.fn, '__qualname__', self.fn)} line {line}: {msg}")

    # -- values ---------------------------------------------------------------
    def _pyval(self, o) -> Val:
        if _is_absent_obj(o):
            return Val("absent")
        if o is None:
            return Val("none")
        if isinstance(o, (bool, int, float, np.number, np.bool_)):
            return const_val(o)
        return Val("obj", obj=o)

    def present(self, v: Val, node) -> Val:
        """Numeric value with Python's check that it is not ABSENT."""
        if v.kind == "absent":
            return num("(err.set(1), 0LL)", INT)
        if v.kind != "num":
            self.fail(node, f"expected a number, got {v.kind}")
        if v.ok is None:
            return v
        return num(f"py_val({v.c}, {v.ok}, err)", v.t)

    def cast(self, v: Val, t: str) -> str:
        if v.t == t:
            return v.c
        if v.const is not None and t in (F32, F64) and v.t in (INT, BOOL, F64, F32):
            return _lit(float(v.const), t)
        return f"(({CTYPE[t]})({v.c}))"

    def truth(self, v: Val, node) -> str:
        if v.kind == "absent" or v.kind == "none":
            return "false"
        if v.kind == "tuple":
            return "true" if v.ok is None else v.ok
        if v.kind == "obj":
            return "true" if v.obj else "false"
        if v.kind != "num":
            self.fail(node, "truth value of a non-number")
        b = v.c if v.t == BOOL else f"(({v.c}) != 0)"
        return b if v.ok is None else f"(({v.ok}) && {b})"

    # -- statements -----------------------------------------------------------
    def stmt(self, s):
        if isinstance(s, ast.Expr):
            if isinstance(s.value, ast.Constant) and isinstance(s.value.value, str):
                return  # docstring
            self.fail(s, "expression statements (calls with side effects) are not supported")
        if isinstance(s, ast.Pass):
            return
        if isinstance(s, ast.Return):
            if s.value is None:
                self.emit("err.set(5); return (RET_T)0;")
                return
            self._return(self.expr(s.value), s)
            return
        if isinstance(s, ast.Assign):
            v = self.expr(s.value)
            for tgt in s.targets:
                self.assign(tgt, v)
            return
        if isinstance(s, ast.AnnAssign) and s.value is not None:
            self.assign(s.target, self.expr(s.value))
            return
        if isinstance(s, ast.AugAssign):
            cur = self.expr(ast.Name(id=s.target.id, ctx=ast.Load())) \
                if isinstance(s.target, ast.Name) else self.fail(s, "augmented assignment target")
            v = self.binop(s.op, cur, self.expr(s.value), s)
            self.assign(s.target, v)
            return
        if isinstance(s, ast.If):
            c = self.truth(self.expr(s.test), s)
            self.emit(f"if ({c}) {{")
            self.depth += 1
            for b in s.body:
                self.stmt(b)
            self.depth -= 1
            if s.orelse:
                self.emit("} else {")
                self.depth += 1
                for b in s.orelse:
                    self.stmt(b)
                self.depth -= 1
            self.emit("}")
            return
        if isinstance(s, ast.For):
            self.for_loop(s)
            return
        if isinstance(s, ast.While):
            if s.orelse:
                self.fail(s, "while/else is not supported")
            self.emit("while (true) {")
            self.depth += 1
            c = self.truth(self.expr(s.test), s)
            self.emit(f"if (!({c})) break;")
            for b in s.body:
                self.stmt(b)
            self.depth -= 1
            self.emit("}")
            return
        if isinstance(s, ast.Break):
            self.emit("break;")
            return
        if isinstance(s, ast.Continue):
            self.emit("continue;")
            return
        self.fail(s, f"{type(s).__name__} statements are not supported")

    def _return(self, v: Val, node=None):
        v = self.present(v, node or self.node)
        if v.kind != "num":
            self.fail(node or self.node, "the elemental must return a number")
        self.ret_t = _join(self.ret_t, v.t)
        self.emit(f"return (RET_T)({v.c});")

    def shape_of(self, v: Val, node):
        if v.kind == "num":
            return v.t
        if v.kind == "tuple":
            return tuple(self.shape_of(x, node) for x in v.items)
        self.fail(node, f"cannot store a {v.kind} in a variable")

    def assign(self, tgt, v: Val):
        if isinstance(tgt, ast.Name):
            name = tgt.id
            if v.kind in ("nb", "env", "envgrid", "obj", "none", "array"):
                # translate-time alias (e.g. e = env[0], tbl = _RING)
                self.local_vals[name] = v
                return
            if v.kind == "absent":
                shape = self.types.get(name)
                if shape is None:
                    shape = INT
                self.new_types[name] = self._join_shape(self.new_types.get(name), shape, tgt)
                self.new_abs.add(name)
                if name in self.absentable:
                    self.emit(f"v_{name}_ok = false;")
                self.local_vals.pop(name, None)
                return
            shape = self.shape_of(v, tgt)
            old = self.types.get(name)
            joined = self._join_shape(self.new_types.get(name), shape, tgt)
            self.new_types[name] = joined
            if v.ok is not None:
                self.new_abs.add(name)
            self.local_vals.pop(name, None)
            if old is None:
                return  # first typing pass: no code yet
            self._store(f"v_{name}", old, v)
            if name in self.absentable:
                self.emit(f"v_{name}_ok = {v.ok if v.ok is not None else 'true'};")
            return
        if isinstance(tgt, (ast.Tuple, ast.List)):
            if v.kind == "tuple":
                if len(v.items) != len(tgt.elts):
                    self.fail(tgt, "tuple unpacking length mismatch")
                if v.ok is not None:
                    # unpacking ABSENT raises TypeError
                    self.emit(f"if (!({v.ok})) err.set(1);")
                items = v.items
            elif v.kind == "obj" and isinstance(v.obj, (tuple, list)):
                if len(v.obj) != len(tgt.elts):
                    self.fail(tgt, "tuple unpacking length mismatch")
                items = tuple(self._pyval(x) for x in v.obj)
            elif v.kind == "env":  # a, b = env (a tuple of grids)
                if len(self.win.env) != len(tgt.elts):
                    self.fail(tgt, "env unpacking length mismatch")
                items = tuple(Val("envgrid", slot=i) for i in range(len(tgt.elts)))
            else:
                self.fail(tgt, "unpacking a non-tuple")
            # evaluate all components before storing (a, b = b, a)
            held = []
            for it in items:
                if it.kind == "num" and it.const is None:
                    held.append(num(self.fresh(it.t, it.c), it.t, ok=it.ok))
                else:
                    held.append(it)
            for t, it in zip(tgt.elts, held):
                self.assign(t, it)
            return
        self.fail(tgt, "assignment target")

    def _join_shape(self, a, b, node):
        if a is None:
            return b
        if isinstance(a, tuple) or isinstance(b, tuple):
            if not (isinstance(a, tuple) and isinstance(b, tuple) and len(a) == len(b)):
                self.fail(node, "a variable changes between a tuple and a number")
            return tuple(self._join_shape(x, y, node) for x, y in zip(a, b))
        return _join(a, b)

    def _store(self, base, shape, v: Val):
        if isinstance(shape, tuple):
            for i, (s, it) in enumerate(zip(shape, v.items)):
                self._store(f"{base}__{i}", s, it)
            return
        self.emit(f"{base} = {self.cast(v, shape)};")

    def _load(self, name, shape, ok) -> Val:
        base = f"v_{name}"
        if isinstance(shape, tuple):
            return Val("tuple", items=tuple(self._load_sub(f"{base}__{i}", s)
                                            for i, s in enumerate(shape)), ok=ok)
        return num(base, shape, ok=ok)

    def _load_sub(self, base, shape):
        if isinstance(shape, tuple):
            return Val("tuple", items=tuple(self._load_sub(f"{base}__{i}", s)
                                            for i, s in enumerate(shape)))
        return num(base, shape)

    # -- loops ----------------------------------------------------------------
    def for_loop(self, s: ast.For):
        if s.orelse:
            self.fail(s, "for/else is not supported")
        it = s.iter
        # range(...)
        if isinstance(it, ast.Call) and isinstance(it.func, ast.Name) and it.func.id == "range" \
                and it.func.id not in self.local_vals:
            args = [self.present(self.expr(a), s) for a in it.args]
            if not 1 <= len(args) <= 3 or any(a.t not in (INT, BOOL) for a in args):
                self.fail(s, "range() takes 1-3 integer arguments")
            lo, hi, st = ("0LL", args[0].c, "1LL") if len(args) == 1 else \
                (args[0].c, args[1].c, "1LL") if len(args) == 2 else (args[0].c, args[1].c, args[2].c)
            self.tmp += 1
            i, e, d = f"r{self.tmp}", f"re{self.tmp}", f"rs{self.tmp}"
            self.emit(f"{{ const long long {e} = {hi}, {d} = {st};")
            self.emit(f"if ({d} == 0) err.set(3);")
            self.emit(f"for (long long {i} = {lo}; {d} > 0 ? {i} < {e} : ({d} < 0 && {i} > {e}); {i} += {d}) {{")
            self.depth += 1
            self.assign(s.target, num(i, INT))
            for b in s.body:
                self.stmt(b)
            self.depth -= 1
            self.emit("} }")
            return
        src = self.expr(it)
        # the window: nb.values() / nb.pairs() / iter(nb)
        if src.kind == "array":
            self.tmp += 1
            i = f"ai{self.tmp}"
            self.emit(f"for (int {i} = 0; {i} < {src.obj}; ++{i}) {{")
            self.depth += 1
            self.assign(s.target, num(f"{src.c}[{i}]", src.t))
            for b in s.body:
                self.stmt(b)
            self.depth -= 1
            self.emit("}")
            return
        if src.kind == "obj" and isinstance(src.obj, _WindowIter):
            self._window_loop(s, src.obj)
            return
        if src.kind == "nb":
            self._window_loop(s, _WindowIter("entries"))
            return
        # a constant table (closure / global tuple or list)
        if src.kind == "obj" and isinstance(src.obj, (tuple, list)):
            self._table_loop(s, list(src.obj))
            return
        if src.kind == "tuple":  # a small tuple of values: unrolled
            for item in src.items:
                self.emit("do {")
                self.depth += 1
                self.assign(s.target, item)
                for b in s.body:
                    self.stmt(b)
                self.depth -= 1
                self.emit("} while (0);")
            if any(isinstance(n, ast.Break) for n in ast.walk(s)):
                self.fail(s, "break inside a loop over a tuple of values")
            return
        self.fail(s, "for-loop over this iterable is not supported")

    def _table_loop(self, s, items):
        """for x in <constant table>: one C array per leaf position of the
        (uniformly nested) items; the loop target gets the same nesting."""
        if not items:
            return

        def shape(x):
            if isinstance(x, (tuple, list)):
                return tuple(shape(y) for y in x)
            if isinstance(x, (int, float, bool, np.number)):
                return None
            self.fail(s, "constant table must hold numbers or tuples of numbers")

        sh = shape(items[0])
        if any(shape(x) != sh for x in items):
            self.fail(s, "constant table items differ in structure")

        def leaves(x):
            if isinstance(x, (tuple, list)):
                out = []
                for y in x:
                    out += leaves(y)
                return out
            return [x]

        cols = list(zip(*[leaves(x) for x in items]))
        self.tmp += 1
        name = f"tab{self.tmp}"
        types = []
        self.emit("{")
        for j, col in enumerate(cols):
            t = None
            for x in col:
                t = _join(t, const_val(x).t)
            types.append(t)
            vals = ", ".join(self.cast(const_val(x), t) for x in col)
            self.emit(f"const {CTYPE[t]} {name}_{j}[{len(items)}] = {{{vals}}};")
        self.emit(f"for (int {name}_i = 0; {name}_i < {len(items)}; ++{name}_i) {{")
        self.depth += 1
        pos = [0]

        def build(shp):
            if shp is None:
                j = pos[0]
                pos[0] += 1
                return num(f"{name}_{j}[{name}_i]", types[j])
            return Val("tuple", items=tuple(build(x) for x in shp))

        self.assign(s.target, build(sh))
        for b in s.body:
            self.stmt(b)
        self.depth -= 1
        self.emit("} }")

    def _win_slots(self, i: str):
        """(slot count, row-offset expr, column-offset expr) of a window walk
        in row-major order (rank-1 grids: one offset, the column stays 0)."""
        k = self.win.k
        n = 2 * k + 1
        if self.win.ndim == 1:
            return n, f"({i} - {k})", "0"
        return n * n, f"({i} / {n} - {k})", f"({i} % {n} - {k})"

    def _idx_tuple(self, a: str, b: str) -> Val:
        if self.win.ndim == 1:
            return Val("tuple", items=(num(f"((long long)nb.i + {a})", INT),))
        return Val("tuple", items=(num(f"((long long)nb.i + {a})", INT),
                                   num(f"((long long)nb.j + {b})", INT)))

    def _window_loop(self, s, w: "_WindowIter"):
        self.tmp += 1
        i = f"w{self.tmp}"
        cnt, ea, eb = self._win_slots(i)
        self.emit(f"for (int {i} = 0; {i} < {cnt}; ++{i}) {{")
        self.depth += 1
        self.emit(f"const int {i}a = {ea}, {i}b = {eb};")
        okc = f"nb.ok({i}a, {i}b)"
        val = self._win_value(f"{i}a", f"{i}b")
        if w.what == "entries":
            item = self._win_entry(f"{i}a", f"{i}b", okc)
        else:
            self.emit(f"if (!{okc}) continue;")
            if w.what == "values":
                item = val
            else:  # pairs
                item = Val("tuple", items=(val, self._idx_tuple(f"{i}a", f"{i}b")))
        self.assign(s.target, item)
        for b in s.body:
            self.stmt(b)
        self.depth -= 1
        self.emit("}")

    def _win_value(self, a, b) -> Val:
        w = self.win
        c = f"nb.at({a}, {b})"
        if w.in_c != CTYPE[w.in_t]:
            c = f"(({CTYPE[w.in_t]}){c})"
        return num(c, w.in_t)

    def _win_entry(self, a, b, okc) -> Val:
        val = self._win_value(a, b)
        if self.win.indexed:
            return Val("tuple", items=(val, self._idx_tuple(a, b)), ok=okc)
        val.ok = okc
        return val

    # -- expressions ----------------------------------------------------------
    def expr(self, e) -> Val:
        m = getattr(self, "x_" + type(e).__name__, None)
        if m is None:
            self.fail(e, f"{type(e).__name__} expressions are not supported")
        return m(e)

    def x_Constant(self, e):
        return self._pyval(e.value)

    def x_Name(self, e):
        name = e.id
        if name in self.local_vals:
            return self.local_vals[name]
        if name in self.types or name in self.new_types:
            # (first typing pass: the type seen so far; its code is discarded)
            shape = self.types.get(name) or self.new_types.get(name)
            ok = f"v_{name}_ok" if name in self.absentable else None
            return self._load(name, shape, ok)
        if name in self.nonlocals:
            _record_dep(self, "nonlocal", name, self.nonlocals[name])
            return self._pyval(self.nonlocals[name])
        if name in self.fglobals:
            _record_dep(self, "global", name, self.fglobals[name])
            return self._pyval(self.fglobals[name])
        if hasattr(builtins, name):
            return Val("obj", obj=getattr(builtins, name))
        self.fail(e, f"unknown name {name!r}")

    def x_Tuple(self, e):
        return Val("tuple", items=tuple(self.expr(x) for x in e.elts))

    x_List = x_Tuple

    def x_Attribute(self, e):
        base = self.expr(e.value)
        a = e.attr
        if base.kind == "nb":
            w = self.win
            if a == "center":
                v = self._win_value("0", "0")
                if w.indexed:
                    return Val("tuple", items=(v, self._idx_tuple("0", "0")))
                return v
            if a == "center_index":
                return self._idx_tuple("0", "0")
            if a == "k":
                return const_val(w.k)
            if a in ("at", "values", "pairs"):
                return Val("obj", obj=_NbMethod(a))
            self.fail(e, f"Neighborhood has no device attribute {a!r}")
        if base.kind in ("envgrid", "env"):
            if a in ("at", "in_range"):
                return Val("obj", obj=_EnvMethod(a, base))
            if a == "dims":
                return Val("obj", obj=tuple(int(d) for d in self.win.dims))
            if a == "ndim":
                return const_val(self.win.ndim)
            self.fail(e, f"env attribute {a!r} is not supported on the device")
        if base.kind == "obj":
            try:
                return self._pyval(getattr(base.obj, a))
            except AttributeError:
                self.fail(e, f"{base.obj!r} has no attribute {a!r}")
        self.fail(e, f"attribute {a!r} of a {base.kind}")

    def x_Subscript(self, e):
        base = self.expr(e.value)
        idx = e.slice
        if base.kind == "obj" and isinstance(base.obj, _WindowIter) and base.obj.what == "values":
            base = self._materialize(base.obj, sort=False, node=e)
        if base.kind == "array":
            if isinstance(idx, ast.Slice):
                self.fail(e, "slices of window values are not supported")
            i = self.present(self.expr(idx), e)
            if i.t not in (INT, BOOL):
                self.fail(e, "list indices must be integers")
            ii = self.fresh(INT, self.cast(i, INT))
            n = base.obj
            self.emit(f"if ({ii} < -(long long){n} || {ii} >= (long long){n}) err.set(7);")
            return num(f"{base.c}[{ii} < 0 ? ({ii} + {n} < 0 ? 0 : {ii} + {n}) : "
                       f"({ii} >= {n} ? 0 : {ii})]", base.t)
        if base.kind == "env":
            i = self.expr(idx)
            if i.const is None:
                self.fail(e, "env[...] needs a constant slot")
            if not 0 <= i.const < len(self.win.env):
                self.fail(e, f"env slot {i.const} out of range")
            return Val("envgrid", slot=int(i.const))
        if base.kind == "envgrid":
            if isinstance(idx, ast.Tuple) and len(idx.elts) == 2:
                return self._env_at(base, [self.expr(x) for x in idx.elts], e)
            self.fail(e, "env grids are indexed with [i, j]")
        if base.kind == "tuple":
            i = self.expr(idx)
            if i.const is None:
                self.fail(e, "tuple index must be a constant")
            if base.ok is not None:
                self.emit(f"if (!({base.ok})) err.set(1);")
            return base.items[int(i.const)]
        if base.kind == "obj" and isinstance(base.obj, (tuple, list)):
            i = self.expr(idx)
            if i.const is not None:
                return self._pyval(base.obj[int(i.const)])
            items = base.obj
            if all(isinstance(x, (int, float, bool, np.number)) for x in items):
                vals = [const_val(x) for x in items]
                t = None
                for v in vals:
                    t = _join(t, v.t)
                self.tmp += 1
                name = f"ctab{self.tmp}"
                self.emit(f"const {CTYPE[t]} {name}[{len(vals)}] = {{{', '.join(self.cast(v, t) for v in vals)}}};")
                ii = self.present(i, e)
                n = len(vals)
                self.emit(f"if ({ii.c} < -{n} || {ii.c} >= {n}) err.set(7);")
                return num(f"{name}[(({ii.c}) % {n} + {n}) % {n}]", t)
            self.fail(e, "dynamic index into a table of tuples")
        self.fail(e, f"subscript of a {base.kind}")

    def _env_at(self, g: Val, idx, node):
        if self.win.ndim == 1:
            if len(idx) != 1:
                self.fail(node, "env.at takes (i) on a rank-1 grid")
            idx = [idx[0], const_val(0)]
        if len(idx) != 2:
            self.fail(node, "env.at takes (i, j)")
        i, j = (self.present(x, node) for x in idx)
        if i.t not in (INT, BOOL) or j.t not in (INT, BOOL):
            self.fail(node, "env indices must be integers")
        slot = g.slot
        cst, sem = self.win.env[slot]
        if _centre_offset(i.c, "i") == 0 and _centre_offset(j.c, "j") == 0:
            # the centre's own env element: on the grid and resident
            return num(f"(({CTYPE[sem]})nb.template centre_env<{cst}>(env, {slot}))", sem)
        ii = self.fresh(INT, i.c)
        jj = self.fresh(INT, j.c)
        # Within the radius of the centre an env element is on the grid and
        # resident whenever the window is (interior tiles).  `near` is a
        # run-time test that the C compiler folds to a constant when the
        # index is the centre index plus literals (the usual case, however
        # the Python code names it), so the checks compile away there.
        near = f"sk_env_near(nb, {ii}, {jj})"
        self.emit(f"const bool {ii}_near = {near};")
        self.emit(f"if (!{ii}_near && !env.ok({ii}, {jj})) err.set(6); "
                  f"else if (!{ii}_near && !env.resident({ii})) err.set(9);")
        okc = f"({ii}_near || (env.ok({ii}, {jj}) && env.resident({ii})))"
        c = (f"({okc} ? ({CTYPE[sem]})env.get<{cst}>({slot}, {ii}, {jj}) : ({CTYPE[sem]})0)")
        return num(c, sem)

    def _args(self, e):
        out = []
        for a in e.args:
            if isinstance(a, ast.Starred):
                v = self.expr(a.value)
                if v.kind == "tuple":
                    if v.ok is not None:
                        self.emit(f"if (!({v.ok})) err.set(1);")
                    out += list(v.items)
                elif v.kind == "obj" and isinstance(v.obj, (tuple, list)):
                    out += [self._pyval(x) for x in v.obj]
                else:
                    self.fail(e, "*args needs a tuple")
            else:
                out.append(self.expr(a))
        return out

    def x_Call(self, e):
        f = self.expr(e.func)
        if e.keywords:
            self.fail(e, "keyword arguments are not supported")
        if f.kind != "obj":
            self.fail(e, "call of a non-function")
        fo = f.obj
        if isinstance(fo, _NbMethod):
            return self._nb_call(fo.name, e)
        if isinstance(fo, _EnvMethod):
            args = self._args(e)
            if fo.name == "at":
                return self._env_at(fo.grid if fo.grid.kind == "envgrid" else Val("envgrid", slot=0),
                                    args, e)
            a = [self.present(x, e) for x in args]
            if self.win.ndim == 1:
                return num(f"env.ok({a[0].c}, 0)", BOOL) if len(a) == 1 else const_val(False)
            return num(f"env.ok({a[0].c}, {a[1].c})", BOOL) if len(a) == 2 else const_val(False)
        return self._builtin_call(fo, e)

    def _nb_call(self, name, e):
        w = self.win
        if name == "at":
            args = self._args(e)
            if w.ndim == 1 and len(args) == 1:
                args = [args[0], const_val(0)]
            if len(args) != 2:
                self.fail(e, f"nb.at takes {w.ndim} offset(s) on a rank-{w.ndim} grid")
            a, b = (self.present(x, e) for x in args)
            for v in (a, b):
                if v.t not in (INT, BOOL):
                    self.fail(e, "window offsets must be integers")
                if v.const is not None and abs(v.const) > w.k:
                    self.fail(e, f"window offset {v.const} outside radius {w.k}")
            ac, bc = a.c, b.c
            if a.const is None or b.const is None:
                ac, bc = self.fresh(INT, a.c), self.fresh(INT, b.c)
                self.emit(f"if ({ac} < -{w.k} || {ac} > {w.k} || {bc} < -{w.k} || {bc} > {w.k}) err.set(7);")
                ac = f"(int)({ac} < -{w.k} || {ac} > {w.k} ? 0 : {ac})"
                bc = f"(int)({bc} < -{w.k} || {bc} > {w.k} ? 0 : {bc})"
            else:
                ac, bc = str(int(a.const)), str(int(b.const))
            return self._win_entry(ac, bc, f"nb.ok({ac}, {bc})")
        if name in ("values", "pairs"):
            if e.args:
                self.fail(e, f"nb.{name}() takes no arguments")
            return Val("obj", obj=_WindowIter(name))
        self.fail(e, f"nb.{name}")

    def _materialize(self, w: "_WindowIter", sort: bool, node) -> Val:
        """The window's in-grid values as a local array (`sorted(nb.values())`,
        `list(nb.values())`, `nb.values()[i]`): row-major, then an insertion
        sort -- Python's sort of numbers is that order too (stable, `<`)."""
        win = self.win
        t = win.in_t
        self.tmp += 1
        arr, i = f"arr{self.tmp}", f"wa{self.tmp}"
        cnt, ea, eb = self._win_slots(i)
        self.emit(f"{CTYPE[t]} {arr}[{cnt}]; int {arr}_n = 0;")
        self.emit(f"for (int {i} = 0; {i} < {cnt}; ++{i}) {{")
        self.emit(f"  const int {i}a = {ea}, {i}b = {eb};")
        self.emit(f"  if (nb.ok({i}a, {i}b)) {arr}[{arr}_n++] = {self._win_value(f'{i}a', f'{i}b').c};")
        self.emit("}")
        val = Val("array", c=arr, t=t, obj=f"{arr}_n")
        if sort:
            self._sort_array(val)
        return val

    def _copy_array(self, a: Val) -> Val:
        self.tmp += 1
        arr = f"arr{self.tmp}"
        self.emit(f"{CTYPE[a.t]} {arr}[sizeof({a.c}) / sizeof({a.c}[0])]; const int {arr}_n = {a.obj};")
        self.emit(f"for (int q = 0; q < {arr}_n; ++q) {arr}[q] = {a.c}[q];")
        return Val("array", c=arr, t=a.t, obj=f"{arr}_n")

    def _sort_array(self, a: Val) -> None:
        self.tmp += 1
        i, j, x = f"si{self.tmp}", f"sj{self.tmp}", f"sx{self.tmp}"
        self.emit(f"for (int {i} = 1; {i} < {a.obj}; ++{i}) {{")
        self.emit(f"  const {CTYPE[a.t]} {x} = {a.c}[{i}]; int {j} = {i} - 1;")
        self.emit(f"  while ({j} >= 0 && {x} < {a.c}[{j}]) {{ {a.c}[{j} + 1] = {a.c}[{j}]; --{j}; }}")
        self.emit(f"  {a.c}[{j} + 1] = {x};")
        self.emit("}")

    def _reduce_array(self, how: str, a: Val) -> Val:
        t = INT if (how == "sum" and a.t == BOOL) else a.t
        if how == "len":
            return num(f"((long long){a.obj})", INT)
        self.tmp += 1
        acc = f"ra{self.tmp}"
        self.emit(f"{CTYPE[t]} {acc} = 0;")
        if how == "sum":
            if t == F64:  # CPython >= 3.12 sum(): Neumaier compensation
                self.emit(f"{{ double c_ = 0.0; for (int q = 0; q < {a.obj}; ++q) {{ "
                          f"const double x_ = {a.c}[q], t_ = {acc} + x_; "
                          f"c_ += (fabs({acc}) >= fabs(x_)) ? ({acc} - t_) + x_ : (x_ - t_) + {acc}; "
                          f"{acc} = t_; }} if (c_ != 0.0 && isfinite(c_)) {acc} += c_; }}")
            else:
                self.emit(f"for (int q = 0; q < {a.obj}; ++q) {acc} = {acc} + ({CTYPE[t]}){a.c}[q];")
            return num(acc, t)
        fn = "py_max" if how == "max" else "py_min"
        self.emit(f"if ({a.obj} == 0) err.set(3); else {{ {acc} = {a.c}[0]; "
                  f"for (int q = 1; q < {a.obj}; ++q) {acc} = {fn}({acc}, ({CTYPE[t]}){a.c}[q]); }}")
        return num(acc, t)

    def _reduce_window(self, how, w: "_WindowIter", e):
        """sum / max / min / len over nb.values() as an inline loop."""
        win = self.win
        k, n = win.k, 2 * win.k + 1
        t = win.in_t
        if how == "sum" and t == BOOL:
            t = INT
        self.tmp += 1
        acc, cnt, i = f"acc{self.tmp}", f"cnt{self.tmp}", f"q{self.tmp}"
        self.emit(f"{CTYPE[t] if how != 'len' else 'long long'} {acc} = 0; long long {cnt} = 0;")
        if how == "sum" and t == F64:
            self.emit(f"double {acc}c = 0.0;")
        cntw, ea, eb = self._win_slots(i)
        self.emit(f"for (int {i} = 0; {i} < {cntw}; ++{i}) {{")
        self.emit(f"  const int {i}a = {ea}, {i}b = {eb};")
        self.emit(f"  if (!nb.ok({i}a, {i}b)) continue;")
        v = self._win_value(f"{i}a", f"{i}b")
        vc = self.cast(v, t) if how != "len" else "0"
        neumaier = how == "sum" and t == F64
        if neumaier:
            # CPython >= 3.12 sums exact floats with Neumaier compensation
            # (bltinmodule.c builtin_sum_impl)
            self.emit(f"  const double {i}x = {vc}, {i}t = {acc} + {i}x;")
            self.emit(f"  {acc}c += (fabs({acc}) >= fabs({i}x)) ? ({acc} - {i}t) + {i}x : ({i}x - {i}t) + {acc};")
            self.emit(f"  {acc} = {i}t;")
        elif how == "sum":
            self.emit(f"  {acc} = {acc} + {vc};")
        elif how == "max":
            self.emit(f"  {acc} = {cnt} == 0 ? {vc} : py_max({acc}, ({CTYPE[t]}){vc});")
        elif how == "min":
            self.emit(f"  {acc} = {cnt} == 0 ? {vc} : py_min({acc}, ({CTYPE[t]}){vc});")
        self.emit(f"  ++{cnt};")
        self.emit("}")
        if how == "sum" and t == F64:
            self.emit(f"if ({acc}c != 0.0 && isfinite({acc}c)) {acc} += {acc}c;")
        if how == "len":
            return num(cnt, INT)
        if how in ("max", "min"):
            self.emit(f"if ({cnt} == 0) err.set(3);  // max()/min() of an empty sequence")
        return num(acc, t)

    def _builtin_call(self, fo, e):
        args = self._args(e)
        mod = getattr(fo, "__module__", None) or ""
        name = getattr(fo, "__name__", "")
        # window aggregates
        if fo in (sorted, list) and len(args) == 1 and args[0].kind == "obj" \
                and isinstance(args[0].obj, _WindowIter) and args[0].obj.what == "values":
            return self._materialize(args[0].obj, sort=fo is sorted, node=e)
        if fo is sorted and len(args) == 1 and args[0].kind == "array":
            arr = self._copy_array(args[0])
            self._sort_array(arr)
            return arr
        if fo in (sum, max, min, len) and len(args) == 1 and args[0].kind == "array":
            return self._reduce_array(fo.__name__, args[0])
        if fo in (sum, max, min, len) and len(args) == 1 and args[0].kind == "obj" \
                and isinstance(args[0].obj, _WindowIter) and args[0].obj.what == "values":
            return self._reduce_window(fo.__name__, args[0].obj, e)
        if fo is len and len(args) == 1 and args[0].kind == "nb":
            return const_val((2 * self.win.k + 1) ** self.win.ndim)
        if fo is len and len(args) == 1 and args[0].kind == "obj" and isinstance(args[0].obj, (tuple, list)):
            return const_val(len(args[0].obj))
        if fo is len and len(args) == 1 and args[0].kind == "tuple":
            return const_val(len(args[0].items))
        # all remaining builtins take numbers
        if fo in (abs, min, max, round, int, float, bool, pow, divmod) or mod in ("math", "numpy") \
                or fo in (np.float32, np.float64, np.int64, np.int32):
            if fo in (min, max) and len(args) == 1 and args[0].kind == "tuple":
                args = list(args[0].items)
            if fo in (min, max) and len(args) == 1 and args[0].kind == "obj" \
                    and isinstance(args[0].obj, (tuple, list)):
                args = [self._pyval(x) for x in args[0].obj]
            if fo is bool:
                return num(self.truth(args[0], e), BOOL) if args else const_val(False)
            nums = [self.present(a, e) for a in args]
            return self._numeric_call(fo, name, mod, nums, e)
        if inspect.isfunction(fo):
            if self.role in ("delta", "combine"):
                self.fail(e, "deltas and combinators cannot call other Python functions")
            return self._helper_call(fo, args, e)
        self.fail(e, f"call of {getattr(fo, '__qualname__', fo)!r} is not supported on the device")

    def _helper_call(self, fo, args, e):
        """A call of another plain Python function: translated once per
        argument signature into its own __device__ function (which receives
        the window, env and error state too, so it may use them)."""
        sig, cparams, cargs, pvals = [], [], [], []
        for i, a in enumerate(args):
            if a.kind == "num":
                sig.append(("num", a.t, a.ok is not None))
                cparams.append(f"{CTYPE[a.t]} p{i}")
                cargs.append(a.c)
                ok = None
                if a.ok is not None:
                    cparams.append(f"bool p{i}_ok")
                    cargs.append(a.ok)
                    ok = f"p{i}_ok"
                pvals.append(num(f"p{i}", a.t, ok=ok))
            elif a.kind in ("nb", "env", "envgrid", "absent", "none"):
                sig.append((a.kind, a.slot))
                pvals.append(a)
            elif a.kind == "obj":
                sig.append(("obj", id(a.obj)))
                pvals.append(a)
            elif a.kind == "tuple" and all(x.kind == "num" and x.ok is None for x in a.items) \
                    and a.ok is None:
                sig.append(("tuple", tuple(x.t for x in a.items)))
                items = []
                for j, x in enumerate(a.items):
                    cparams.append(f"{CTYPE[x.t]} p{i}_{j}")
                    cargs.append(x.c)
                    items.append(num(f"p{i}_{j}", x.t))
                pvals.append(Val("tuple", items=tuple(items)))
            else:
                self.fail(e, f"cannot pass a {a.kind} to {fo.__qualname__}")
        win_t = (self.win.in_c, self.win.in_t) if self.win is not None else None
        name, ret_t = self.ctx.helper(fo, tuple(sig), win_t, cparams, pvals, self.win)
        return num(f"{name}(nb, env, err{''.join(', ' + c for c in cargs)})", ret_t)

    def _numeric_call(self, fo, name, mod, a, e):
        def f64(v):
            return self.cast(v, F64)

        if fo is abs:
            t = INT if a[0].t == BOOL else a[0].t
            return num(f"py_abs({self.cast(a[0], t)})", t)
        if fo in (min, max):
            if len(a) < 2:
                self.fail(e, f"{name}() needs at least two numbers")
            t = None
            for v in a:
                t = _join(t, INT if v.t == BOOL else v.t)
            acc = self.cast(a[0], t)
            for v in a[1:]:
                acc = f"py_{name}<{CTYPE[t]}>({acc}, {self.cast(v, t)})"
            return num(acc, t)
        if fo is round:
            if len(a) != 1:
                self.fail(e, "round(x, n) is not supported")
            if a[0].t in (INT, BOOL):
                return num(self.cast(a[0], INT), INT)
            return num(f"py_round({f64(a[0])}, err)", INT)
        if fo is int or fo in (np.int64, np.int32):
            if a[0].t in (INT, BOOL):
                return num(self.cast(a[0], INT), INT)
            return num(f"py_int({f64(a[0])}, err)", INT)
        if fo is float or fo is np.float64:
            return num(f64(a[0]), F64)
        if fo is np.float32:
            return num(self.cast(a[0], F32), F32)
        if fo is pow:
            return self.binop(ast.Pow(), a[0], a[1], e)
        if mod == "math":
            simple = {"exp": "exp", "sin": "sin", "cos": "cos", "tan": "tan", "atan": "atan",
                      "asin": "asin", "acos": "acos", "sinh": "sinh", "cosh": "cosh", "tanh": "tanh",
                      "fabs": "fabs", "trunc": None, "expm1": "expm1", "cbrt": "cbrt",
                      "erf": "erf", "erfc": "erfc"}
            if name == "sqrt":
                return num(f"py_sqrt({f64(a[0])}, err)", F64)
            if name == "log" and len(a) == 1:
                return num(f"py_log({f64(a[0])}, err)", F64)
            if name in ("log2", "log10", "log1p"):
                return num(f"{name}({f64(a[0])})", F64)
            if name in ("floor", "ceil"):
                if a[0].t in (INT, BOOL):
                    return num(self.cast(a[0], INT), INT)
                return num(f"py_{name}_int({f64(a[0])}, err)", INT)
            if name == "trunc":
                return num(f"py_int({f64(a[0])}, err)", INT) if a[0].t not in (INT, BOOL) else \
                    num(self.cast(a[0], INT), INT)
            if name in simple and simple[name]:
                return num(f"{simple[name]}({f64(a[0])})", F64)
            if name in ("atan2", "hypot", "copysign", "fmod", "pow") and len(a) == 2:
                fn = {"pow": "pow"}.get(name, name)
                return num(f"{fn}({f64(a[0])}, {f64(a[1])})", F64)
            if name in ("isnan", "isinf", "isfinite"):
                return num(f"{name}({f64(a[0])})", BOOL)
        if mod == "numpy":
            t = F32 if a and a[0].t == F32 else F64
            un = {"sqrt": "sqrt", "exp": "exp", "log": "log", "sin": "sin", "cos": "cos",
                  "tan": "tan", "abs": "fabs", "absolute": "fabs", "fabs": "fabs", "floor": "floor",
                  "ceil": "ceil", "trunc": "trunc", "rint": "rint", "tanh": "tanh"}
            if name in un and len(a) == 1:
                if a[0].t in (INT, BOOL) and name in ("abs", "absolute"):
                    return num(f"py_abs({self.cast(a[0], INT)})", INT)
                fn = un[name] + ("f" if t == F32 else "")
                return num(f"{fn}({self.cast(a[0], t)})", t)
            if name in ("maximum", "minimum", "fmax", "fmin") and len(a) == 2:
                t = _join(_join(a[0].t, a[1].t), F64 if F32 not in (a[0].t, a[1].t) else F32)
                fn = {"maximum": "fmax", "minimum": "fmin", "fmax": "fmax", "fmin": "fmin"}[name]
                return num(f"{fn}({self.cast(a[0], t)}, {self.cast(a[1], t)})", t)
        self.fail(e, f"{mod}.{name} is not supported on the device")

    def x_BinOp(self, e):
        return self.binop(e.op, self.expr(e.left), self.expr(e.right), e)

    def binop(self, op, a: Val, b: Val, node):
        a, b = self.present(a, node), self.present(b, node)
        if a.kind != "num" or b.kind != "num":
            self.fail(node, "arithmetic on non-numbers")
        if a.const is not None and b.const is not None and not isinstance(op, (ast.Div, ast.FloorDiv, ast.Mod, ast.Pow)):
            try:
                r = _PYOPS[type(op)](a.const, b.const)
                t = _arith(a.t, b.t) if not isinstance(op, (ast.BitAnd, ast.BitOr, ast.BitXor)) \
                    or not (a.t == BOOL and b.t == BOOL) else BOOL
                if t == F32:
                    r = float(np.float32(r))
                return num(_lit(r, t), t, const=r)
            except Exception:
                pass
        ta, tb = a.t, b.t
        if isinstance(op, (ast.Add, ast.Sub, ast.Mult)):
            t = _arith(ta, tb)
            sym = {ast.Add: "+", ast.Sub: "-", ast.Mult: "*"}[type(op)]
            return num(f"({self.cast(a, t)} {sym} {self.cast(b, t)})", t)
        if isinstance(op, ast.Div):
            if F32 in (ta, tb):
                return num(f"py_truediv({self.cast(a, F32)}, {self.cast(b, F32)}, err)", F32)
            if F64 in (ta, tb):
                return num(f"py_truediv({self.cast(a, F64)}, {self.cast(b, F64)}, err)", F64)
            return num(f"py_truediv({self.cast(a, INT)}, {self.cast(b, INT)}, err)", F64)
        if isinstance(op, (ast.FloorDiv, ast.Mod)):
            t = _arith(ta, tb)
            fn = "py_floordiv" if isinstance(op, ast.FloorDiv) else "py_mod"
            return num(f"{fn}({self.cast(a, t)}, {self.cast(b, t)}, err)", t)
        if isinstance(op, ast.Pow):
            if ta in (INT, BOOL) and tb in (INT, BOOL):
                if b.const is not None and b.const < 0:
                    return num(f"py_pow({self.cast(a, F64)}, {self.cast(b, F64)}, err)", F64)
                bb = self.fresh(INT, self.cast(b, INT))
                self.emit(f"if ({bb} < 0) err.set(8);")
                return num(f"py_ipow({self.cast(a, INT)}, {bb})", INT)
            t = F32 if F32 in (ta, tb) else F64
            return num(f"py_pow({self.cast(a, t)}, {self.cast(b, t)}, err)", t)
        if isinstance(op, (ast.BitAnd, ast.BitOr, ast.BitXor, ast.LShift, ast.RShift)):
            if ta not in (INT, BOOL) or tb not in (INT, BOOL):
                self.fail(node, "bitwise operators need integers")
            sym = {ast.BitAnd: "&", ast.BitOr: "|", ast.BitXor: "^", ast.LShift: "<<",
                   ast.RShift: ">>"}[type(op)]
            if ta == BOOL and tb == BOOL and sym in "&|^":
                return num(f"(bool)({a.c} {sym} {b.c})", BOOL)
            return num(f"({self.cast(a, INT)} {sym} {self.cast(b, INT)})", INT)
        self.fail(node, f"operator {type(op).__name__}")

    def x_UnaryOp(self, e):
        v = self.expr(e.operand)
        if isinstance(e.op, ast.Not):
            return num(f"(!{self.truth(v, e)})", BOOL)
        v = self.present(v, e)
        if isinstance(e.op, ast.USub):
            if v.const is not None:
                t = INT if v.t == BOOL else v.t
                return num(_lit(-v.const, t), t, const=-v.const)
            t = INT if v.t == BOOL else v.t
            return num(f"(-{self.cast(v, t)})", t)
        if isinstance(e.op, ast.UAdd):
            t = INT if v.t == BOOL else v.t
            return num(self.cast(v, t), t, const=v.const)
        if isinstance(e.op, ast.Invert):
            if v.t not in (INT, BOOL):
                self.fail(e, "~ needs an integer")
            return num(f"(~{self.cast(v, INT)})", INT)
        self.fail(e, "unary operator")

    def x_BoolOp(self, e):
        vals = [self.expr(x) for x in e.values]
        is_and = isinstance(e.op, ast.And)
        # pure truth-value use (the common case): C short-circuit
        if all(v.kind == "num" and v.t == BOOL and v.ok is None for v in vals):
            sym = " && " if is_and else " || "
            return num("(" + sym.join(v.c for v in vals) + ")", BOOL)
        # value semantics: a and b -> b if a else a; a or b -> a if a else b
        acc = vals[-1]
        for v in reversed(vals[:-1]):
            acc = self._select(self.truth(v, e), acc if is_and else v, v if is_and else acc, e)
        return acc

    def _select(self, cond: str, a: Val, b: Val, node) -> Val:
        if a.kind == "absent" and b.kind == "num":
            return num(b.c, b.t, ok=f"(!({cond}) && {b.ok or 'true'})")
        if b.kind == "absent" and a.kind == "num":
            return num(a.c, a.t, ok=f"(({cond}) && {a.ok or 'true'})")
        if a.kind == "num" and b.kind == "num":
            t = _join(a.t, b.t)
            ok = None
            if a.ok is not None or b.ok is not None:
                ok = f"(({cond}) ? {a.ok or 'true'} : {b.ok or 'true'})"
            return num(f"(({cond}) ? {self.cast(a, t)} : {self.cast(b, t)})", t, ok=ok)
        if a.kind == "tuple" and b.kind == "tuple" and len(a.items) == len(b.items):
            return Val("tuple", items=tuple(self._select(cond, x, y, node) for x, y in zip(a.items, b.items)))
        self.fail(node, "conditional expression mixes incompatible values")

    def x_IfExp(self, e):
        c = self.truth(self.expr(e.test), e)
        # evaluate each branch's code unconditionally only if it has no side
        # effects on the error state: branch values are C expressions, and
        # C's ?: evaluates one of them
        return self._select(c, self.expr(e.body), self.expr(e.orelse), e)

    def x_Compare(self, e):
        left = self.expr(e.left)
        parts = []
        for op, rnode in zip(e.ops, e.comparators):
            right = self.expr(rnode)
            parts.append(self._compare(op, left, right, e))
            left = right
        if len(parts) == 1:
            return num(parts[0], BOOL)
        return num("(" + " && ".join(parts) + ")", BOOL)

    def _compare(self, op, a: Val, b: Val, node) -> str:
        if isinstance(op, (ast.Is, ast.IsNot)):
            neg = isinstance(op, ast.IsNot)
            for x, y in ((a, b), (b, a)):
                if y.kind == "absent":
                    if x.kind == "absent":
                        r = "true"
                    elif x.kind in ("num", "tuple"):
                        r = "false" if x.ok is None else f"(!({x.ok}))"
                    else:
                        r = "false"
                    return f"(!{r})" if neg else r
                if y.kind == "none":
                    r = "true" if x.kind == "none" else "false"
                    return f"(!{r})" if neg else r
            self.fail(node, "`is` is supported only against ABSENT / None")
        if isinstance(op, (ast.In, ast.NotIn)):
            if b.kind == "obj" and isinstance(b.obj, (tuple, list)):
                items = [self._pyval(x) for x in b.obj]
            elif b.kind == "tuple":
                items = list(b.items)
            else:
                self.fail(node, "`in` needs a constant tuple")
            r = "(" + " || ".join(self._compare(ast.Eq(), a, x, node) for x in items) + ")" if items else "false"
            return f"(!{r})" if isinstance(op, ast.NotIn) else r
        if isinstance(op, (ast.Eq, ast.NotEq)):
            eq = isinstance(op, ast.Eq)
            if a.kind == "absent" or b.kind == "absent":
                x = b if a.kind == "absent" else a
                if x.kind == "absent":
                    r = "true"
                else:
                    r = "false" if x.ok is None else f"(!({x.ok}))"
                return r if eq else f"(!{r})"
            if a.kind == "num" and b.kind == "num":
                t = _join(a.t, b.t)
                cmp = f"({self.cast(a, t)} == {self.cast(b, t)})"
                oks = [o for o in (a.ok, b.ok) if o is not None]
                if oks:  # ABSENT == number is False (no exception)
                    cmp = "(" + " && ".join(oks) + f" && {cmp})"
                return cmp if eq else f"(!{cmp})"
            self.fail(node, "comparison of non-numbers")
        a, b = self.present(a, node), self.present(b, node)
        if a.kind != "num" or b.kind != "num":
            self.fail(node, "ordering comparison of non-numbers")
        t = _join(a.t, b.t)
        sym = {ast.Lt: "<", ast.LtE: "<=", ast.Gt: ">", ast.GtE: ">="}[type(op)]
        return f"({self.cast(a, t)} {sym} {self.cast(b, t)})"


import operator as _op  # noqa: E402

_PYOPS = {ast.Add: _op.add, ast.Sub: _op.sub, ast.Mult: _op.mul, ast.BitAnd: _op.and_,
          ast.BitOr: _op.or_, ast.BitXor: _op.xor, ast.LShift: _op.lshift, ast.RShift: _op.rshift}


class HelperCtx:
    """Helper functions called by the translated code, shared by every
    translation of one program (emitted before their callers)."""

    def __init__(self):
        self.funcs = {}      # key -> (name, ret type)
        self.sources = []    # C definitions in dependency order
        self.active = set()

    def helper(self, fo, sig, win_t, cparams, pvals, win):
        key = (fo.__code__, sig, win_t)
        if key in self.funcs:
            return self.funcs[key]
        if key in self.active:
            raise TranslateError(f"recursive call of {fo.__qualname__} is not supported")
        self.active.add(key)
        try:
            tr = Translator(fo, pvals, "helper", win, ctx=self)
            body, ret_t = tr.translate()
        finally:
            self.active.discard(key)
        import re

        name = f"sk_h{len(self.funcs)}_" + re.sub(r"\W", "_", fo.__name__)
        rt = CTYPE[ret_t]
        head = ", ".join(["const NBT& nb", "const SkEnv& env", "SkErr& err"] + cparams)
        src = [f"template <class NBT>", f"__device__ {rt} {name}({head}) {{"]
        src += [ln.replace("RET_T", rt) for ln in body]
        src.append("}")
        self.sources.append("\n".join(src))
        self.funcs[key] = (name, ret_t)
        return name, ret_t


@dataclass(frozen=True)
class _NbMethod:
    name: str


@dataclass(frozen=True)
class _EnvMethod:
    name: str
    grid: Any


@dataclass(frozen=True)
class _WindowIter:
    what: str  # 'values' | 'pairs' | 'entries'


# ----------------------------------------------------------------------------- programs


@dataclass(frozen=True)
class JitKernel:
    """Device descriptor of a user elemental written as CUDA source (the
    paper's API).  `body` is the body of
    `template <class NB> sk_val_t f(const NB& nb, const SkEnv& env, SkErr& err)`;
    `out_dtype` is the element type of the result grid (default: the input's)."""

    body: str
    out_dtype: Any = None
    name: str = "jit"
    params: tuple = ()


def cuda_elemental(body: str, k: int, out_dtype=None, pad_mode: str = "constant",
                   pad_value: Any = 0):
    """ElementalFn from CUDA source (the paper's elemental-function-as-kernel-
    source API).  Window slots off the grid read `pad_value`
    (or the nearest border element with pad_mode="edge"), as in the
    reference's block route; `nb.ok(di, dj)` tells them apart."""
    from .patterns import ElementalFn

    def point(nb, env):
        raise DeviceUnsupported("this elemental function exists only as device source")

    return ElementalFn(point=point, k=k, block=None, pad_mode=pad_mode, pad_value=pad_value,
                       device=JitKernel(body=body, out_dtype=None if out_dtype is None
                                        else np.dtype(out_dtype)))


@dataclass(frozen=True)
class CudaDelta:
    """Delta as CUDA source: body of `double f(V nw, V old, SkErr& err)`."""

    body: str


@dataclass(frozen=True)
class CudaCombine:
    """Combinator as CUDA source: body of `double f(double a, double b)`."""

    body: str


@dataclass
class Program:
    handle: Any
    source: str
    in_dtype: np.dtype
    out_dtype: np.dtype
    env_dtypes: tuple
    reduce: int
    int_value: bool
    tile_rows: int = 16


_prog_lock = threading.Lock()
_prog_cache: dict = {}


def compile_source(source: str) -> C.c_void_p:
    """NVRTC-compile a full program (cached by text)."""
    with _prog_lock:
        h = _prog_cache.get(source)
        if h is not None:
            return h
        lib = N.load()
        h = C.c_void_p()
        rc = lib.sk_jit_compile(source.encode(), b"sk_user_elemental.cu", C.byref(h))
        if rc != N.SK_OK:
            msg = lib.sk_last_error().decode(errors="replace")
            raise DeviceUnsupported(f"device compile of the elemental failed:\n{msg}\n--- source ---\n{source}")
        _prog_cache[source] = h
        return h


def cubin_of(prog: "Program") -> bytes:
    """The program's sm_100a cubin (inspect with cuobjdump -sass)."""
    lib = N.load()
    n = lib.sk_jit_cubin_size(prog.handle)
    buf = C.create_string_buffer(n)
    N.check(lib.sk_jit_cubin(prog.handle, buf))
    return buf.raw


def _reduce_parts(op, delta, val_t: str, in_t: str, val_c: str, in_c: str):
    """C definitions of sk_delta_1/_n and SkComb, the reduce id, int-ness."""
    from .patterns import combinator_kind

    lines = []
    dt = None
    if delta is None:
        dt = val_t
        for suffix, ot in (("1", in_c), ("n", val_c)):
            lines.append(f"__device__ __forceinline__ sk_delta_t sk_delta_{suffix}(sk_val_t nw, {ot} old, SkErr& err) "
                         f"{{ return (sk_delta_t)nw; }}")
    elif isinstance(getattr(delta, "fn", None), CudaDelta) or isinstance(delta, CudaDelta):
        body = (delta if isinstance(delta, CudaDelta) else delta.fn).body
        dt = F64
        for suffix, ot in (("1", in_c), ("n", val_c)):
            lines.append(f"__device__ __forceinline__ sk_delta_t sk_delta_{suffix}(sk_val_t nw, {ot} old, SkErr& err) "
                         f"{{ {body} }}")
    else:
        bodies = []
        for suffix, ot, os_ in (("1", in_t, in_c), ("n", val_t, val_c)):
            tr = Translator(delta.fn, [num("nw", val_t), num(f"(({CTYPE[ot]})old)", ot)], "delta")
            body, rt = tr.translate()
            dt = _join(dt, rt)
            bodies.append((suffix, os_, body))
        for suffix, os_, body in bodies:
            lines.append(f"__device__ __forceinline__ sk_delta_t sk_delta_{suffix}(sk_val_t nw, {os_} old, SkErr& err) {{")
            lines += [ln.replace("RET_T", "sk_delta_t") for ln in body]
            lines.append("}")
    lines.insert(0, f"typedef {CTYPE[dt]} sk_delta_t;")
    kind = None
    if isinstance(getattr(op, "fn", None), CudaCombine):
        comb_body = op.fn.body
    else:
        try:
            kind = combinator_kind(op)
        except DeviceUnsupported:
            kind = None
        comb_body = None
    if kind == "sum":
        lines.append("typedef SkSum SkComb;")
        reduce = N.SK_REDUCE_SUM
    elif kind == "max":
        lines.append("typedef SkMax SkComb;")
        # per-thread max in the delta's own type, converted once (exact:
        # conversion to double is monotonic)
        lines.append("#define SK_LOCAL_MAX 1")
        reduce = N.SK_REDUCE_MAX
    else:
        if comb_body is None:
            tr = Translator(op.fn, [num("a", F64), num("b", F64)], "combine")
            body, _ = tr.translate()
            inner = "\n".join(ln.replace("RET_T", "double") for ln in body)
        else:
            inner = comb_body
        lines.append("struct SkComb {")
        lines.append("  __device__ double operator()(double a, double b) const {")
        lines.append("    SkErr err;")
        lines.append(inner)
        lines.append("  }")
        lines.append("  __device__ __forceinline__ double fold(double acc, double v) const { return (*this)(acc, v); }")
        lines.append("  __device__ __forceinline__ double neutral(double id) const { return id; }")
        lines.append("};")
        reduce = N.SK_REDUCE_CUSTOM
    ident = op.identity
    int_value = dt in (INT, BOOL) and isinstance(ident, (int, np.integer, bool))
    return lines, reduce, int_value


def _env_spec(env):
    from .grid import Grid

    if env is None:
        return "none", [], None
    if isinstance(env, Grid):
        return "grid", [env], None
    if isinstance(env, tuple) and env and all(isinstance(g, Grid) for g in env):
        if len(env) > 4:
            raise DeviceUnsupported("at most 4 env grids on the device")
        return "tuple", list(env), None
    return "obj", [], env


def grid_dtype(g) -> np.dtype:
    sd = g.storage_dtype()
    if g._src == "list":  # a list-backed grid: the whole list decides
        sd = g._host().dtype
    return np.dtype(sd)


_CENTRE_RE = {ax: re.compile(r"^\(\(long long\)nb\.%s(?: ([+-]) (\d+))?\)$" % ax) for ax in "ij"}


def _centre_offset(c: str, ax: str):
    """d when the C expression `c` is nb.<ax> + d (d a literal), else None."""
    m = _CENTRE_RE[ax].match(c)
    if not m:
        return None
    return 0 if m.group(1) is None else (int(m.group(2)) if m.group(1) == "+" else -int(m.group(2)))


# ---------------------------------------------------------------- translation cache
# Translating an elemental takes ~2 ms of Python per loop call; a drop-in
# user calling the loop again with the same functions gets the Program back
# from this cache.  Every global / nonlocal value the translation read is
# recorded and re-checked on a hit (same object, or an equal immutable
# scalar), so a rebound constant or helper re-translates; programs that read
# any mutable value (lists, arrays, objects) are never cached.
_dep_rec = threading.local()
_tr_cache: dict = {}
_IMMUT = (bool, int, float, complex, str, bytes, type(None), np.number, np.bool_, np.dtype)


def _record_dep(tr, scope: str, name: str, value) -> None:
    deps = getattr(_dep_rec, "deps", None)
    if deps is not None:
        deps.append((tr.role, tr.fn if tr.role == "helper" else None, scope, name, value))


def _stable(v) -> bool:
    import types

    if isinstance(v, _IMMUT):
        return True
    if isinstance(v, (types.ModuleType, types.FunctionType, types.BuiltinFunctionType, type, np.ufunc)):
        return True
    from .grid import ABSENT

    if v is ABSENT:  # the reference's out-of-grid sentinel (a singleton)
        return True
    return isinstance(v, tuple) and all(_stable(x) for x in v)


def _same(cur, v) -> bool:
    if cur is v:
        return True
    if type(cur) is not type(v):
        return False
    if isinstance(v, tuple):
        return len(cur) == len(v) and all(_same(a, b) for a, b in zip(cur, v))
    if isinstance(v, (float, complex, np.inexact)):
        return repr(cur) == repr(v)  # -0.0 vs 0.0, NaN
    if isinstance(v, _IMMUT):
        return bool(cur == v)
    return False


def _program_key(plan, grid, dims):
    from .patterns import combinator_kind, delta_kind

    fn = plan.fn
    if getattr(fn, "device", None) is not None:
        return None
    point = getattr(fn, "point", None)
    code = getattr(point, "__code__", None)
    if code is None:
        return None
    env_kind, env_grids, env_obj = _env_spec(plan.env)
    if env_obj is not None:
        return None
    op, delta = plan.op, plan.delta
    try:
        opk = combinator_kind(op)
    except DeviceUnsupported:
        opk = getattr(getattr(op, "fn", None), "__code__", None)
        if opk is None:
            return None
    if delta is None:
        dk = None
    else:
        try:
            dk = delta_kind(delta)
        except DeviceUnsupported:
            dk = getattr(getattr(delta, "fn", None), "__code__", None)
            if dk is None:
                return None
    pad, ident = fn.pad_value, op.identity
    if not (_stable(pad) and _stable(ident)):
        return None
    return (code, plan.k, bool(plan.indexed), fn.pad_mode, type(pad), repr(pad), grid_dtype(grid),
            tuple(grid_dtype(g) for g in env_grids), env_kind, grid.ndim, tuple(grid.dims),
            tuple(dims) if dims is not None else None, opk, dk, type(ident), repr(ident),
            os.environ.get("SK_JIT_MINB"), os.environ.get("SK_JIT_SMEM_KB"))


def _deps_valid(deps, plan) -> bool:
    roles = {"elemental": plan.fn.point, "combine": getattr(plan.op, "fn", None),
             "delta": getattr(plan.delta, "fn", None)}
    for role, fobj, scope, name, val in deps:
        f = fobj if role == "helper" else roles.get(role)
        if f is None:
            return False
        if scope == "global":
            g = getattr(f, "__globals__", None)
            if g is None or name not in g:
                return False
            cur = g[name]
        else:
            code = getattr(f, "__code__", None)
            if code is None or name not in code.co_freevars or f.__closure__ is None:
                return False
            try:
                cur = f.__closure__[code.co_freevars.index(name)].cell_contents
            except ValueError:  # an empty cell
                return False
        if not _same(cur, val):
            return False
    return True


def build_program(plan, grid, dims=None) -> Program:
    """The CUDA program of a plan whose elemental has no built-in kernel
    (translated by _build_program, or from the translation cache)."""
    key = _program_key(plan, grid, dims)
    if key is not None:
        hit = _tr_cache.get(key)
        if hit is not None and _deps_valid(hit[0], plan):
            return hit[1]
    _dep_rec.deps = []
    try:
        prog = _build_program(plan, grid, dims)
        deps = _dep_rec.deps
    finally:
        _dep_rec.deps = None
    if key is not None and all(_stable(d[4]) for d in deps):
        if len(_tr_cache) > 256:
            _tr_cache.clear()
        _tr_cache[key] = (deps, prog)
    return prog


def _build_program(plan, grid, dims=None) -> Program:
    """The CUDA program of a plan whose elemental has no built-in kernel.
    `dims`: the global grid dims when `grid` is one rank's row block."""
    fn = plan.fn
    k = plan.k
    if k > 8:
        raise DeviceUnsupported(f"device stencils support radius <= 8 (got {k})")
    in_dtype = grid_dtype(grid)
    in_c, in_t = storage_of(in_dtype)
    env_kind, env_grids, env_obj = _env_spec(plan.env)
    env_types = [storage_of(grid_dtype(g)) for g in env_grids]
    win = WindowSpec(k=k, in_c=in_c, in_t=in_t, indexed=bool(plan.indexed), env=env_types,
                     env_kind=env_kind, env_obj=env_obj, ndim=grid.ndim,
                     dims=tuple(dims if dims is not None else grid.dims))
    dk = getattr(fn, "device", None)
    pad_edge = 1 if fn.pad_mode == "edge" else 0
    pad = fn.pad_value
    parts = []
    ctx = HelperCtx()
    if isinstance(dk, JitKernel):
        out_dtype = dk.out_dtype if dk.out_dtype is not None else in_dtype
        val_c, val_t = storage_of(out_dtype)
        body = dk.body
        parts.append("template <class NB>")
        parts.append("__device__ __forceinline__ sk_val_t sk_user(const NB& nb, const SkEnv& env, SkErr& err) {")
        parts.append(body)
        parts.append("}")
        parts.append("template <class NB> __device__ __forceinline__ sk_val_t sk_elemental_1(const NB& nb, const SkEnv& env, SkErr& err) { return sk_user(nb, env, err); }")
        parts.append("template <class NB> __device__ __forceinline__ sk_val_t sk_elemental_n(const NB& nb, const SkEnv& env, SkErr& err) { return sk_user(nb, env, err); }")
    else:
        point = fn.point
        tr1 = Translator(point, [], "elemental", win, ctx=ctx)
        body1, t1 = tr1.translate()
        # later iterations see the first iteration's output type
        val_c, val_t = CTYPE[t1], t1
        win_n = WindowSpec(k=k, in_c=val_c, in_t=val_t, indexed=win.indexed, env=env_types,
                           env_kind=env_kind, env_obj=env_obj, ndim=win.ndim, dims=win.dims)
        trn = Translator(point, [], "elemental", win_n, ctx=ctx)
        bodyn, tn = trn.translate()
        if tn != t1:
            raise DeviceUnsupported(
                f"the elemental's result type changes across iterations ({t1} then {tn})")
        out_dtype = NP_OF[t1]
        for suffix, vt, body in (("1", "sk_in_t", body1), ("n", "sk_val_t", bodyn)):
            # templated on the window type: SkNb<V, true> (interior tiles)
            # folds every ABSENT test away
            parts.append(f"template <class NB> __device__ sk_val_t sk_elemental_{suffix}(const NB& nb, const SkEnv& env, SkErr& err) {{")
            parts += [ln.replace("RET_T", "sk_val_t") for ln in body]
            parts.append("}")
    red, reduce, int_value = _reduce_parts(plan.op, plan.delta, val_t, in_t, val_c, in_c)
    if pad is None or pad is not None and not isinstance(pad, (int, float, bool, np.number)):
        pad_lit = "0"
    else:
        pad_lit = _lit(pad, val_t if isinstance(pad, float) or val_t == F32 else INT) \
            if val_t != BOOL else _lit(bool(pad), BOOL)
    # env slot 0 staged in shared memory: measured faster for 4-byte grids and
    # env (f32 Jacobi 16384^2: 0.75 -> 0.69 ms with 32-row tiles at 72 KB),
    # slower for 8-byte ones (fewer CTAs per SM), which keep the L1 prefetch
    esize = max(np.dtype(in_dtype).itemsize, np.dtype(out_dtype).itemsize)
    env0_size = np.dtype(grid_dtype(env_grids[0])).itemsize if env_grids else 0
    env0_stage = win.ndim == 2 and env0_size == 4 and esize == 4
    th = tile_rows(k, esize, env0_size if env0_stage else 0,
                   budget_kb=72 if env0_stage else 40)
    head = [
        '#include "sk_jit_prelude.cuh"',
        "namespace sk {",
        f"typedef {in_c} sk_in_t;",
        f"typedef {val_c} sk_val_t;",
        f"#define SK_K {k}",
        f"#define SK_TH {th}",
        # CTAs per SM the registers are sized for: 4 with the env tile staged
        # (3 fit by shared memory; measured 0.69 -> 0.64 ms for the f32
        # Jacobi against 6), else 6
        f"#define SK_MINB {int(os.environ.get('SK_JIT_MINB', '0')) or (4 if env0_stage else 6)}",
        f"#define SK_PAD_EDGE {pad_edge}",
        f"#define SK_PAD_VALUE {pad_lit}",
        f"#define SK_NENV {len(env_types)}",
        # env slot 0 is staged per tile in shared memory next to the grid
        # tile (2D sweeps; 4- or 8-byte elements)
        f"#define SK_ENV0_STAGE {1 if env0_stage else 0}",
        f"typedef {env_types[0][0] if env_types else 'float'} sk_env0_t;",
        # rank-1 grids: contiguous element tiles (sk_jit_kernel.cuh jit_sweep1)
        f"#define SK_NDIM {1 if win.ndim == 1 else 2}",
        # byte address of env element `eidx` of slot s (the sweep prefetches
        # a tile's env rows into L1 before computing it)
        "__device__ __forceinline__ const void* sk_env_elem(const SkEnv& e, int s, long long eidx) {",
        "  switch (s) {",
    ] + [f"    case {i}: return static_cast<const {cst}*>(e.p[{i}]) + eidx;"
         for i, (cst, _sem) in enumerate(env_types)] + [
        "    default: return nullptr;",
        "  }",
        "}",
    ]
    src = "\n".join(head + ctx.sources + parts + red +
                    ["}  // namespace sk", '#include "sk_jit_kernel.cuh"', ""])
    handle = compile_source(src)
    return Program(handle=handle, source=src, in_dtype=in_dtype, out_dtype=np.dtype(out_dtype),
                   env_dtypes=tuple(grid_dtype(g) for g in env_grids), reduce=reduce,
                   int_value=int_value, tile_rows=th)


def tile_rows(k: int, esize: int, env0: int = 0, budget_kb: int = 40) -> int:
    """Rows per staged tile: the tallest of 32 / 16 / 8 whose two buffers of
    the window (+ radius frame, 128 columns wide) -- and of env slot 0's
    tile, `env0` bytes per element, when it is staged -- fit the
    shared-memory budget (dynamic shared memory; taller tiles spread the
    per-tile staging and setup over more cells, at the price of CTAs per
    SM)."""
    ka = (k + 3) // 4 * 4
    budget = int(os.environ.get("SK_JIT_SMEM_KB", str(budget_kb))) * 1024
    for th in (32, 16):
        if 2 * (th + 2 * k) * (128 + 2 * ka) * esize + 2 * th * 128 * env0 <= budget:
            return th
    return 8
