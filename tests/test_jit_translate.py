"""User elemental functions -> device programs, checked without a GPU.

* the sequential oracle (oracle/sequential.py) reproduces the REAL
  reference's outputs for every case (golden_jit.*, made by
  tests/golden/make_golden_jit.py with /root/reference): pins the oracle;
* every case translates and compiles with NVRTC for sm_100a (no device
  needed), in both element types it meets;
* functions outside the supported subset are rejected with
  DeviceUnsupported (no host fallback), and the paper-style CUDA-source
  elemental compiles.
"""

import numpy as np
import pytest

import jit_cases as J
import paper_1609_04567_b200 as sk
from jit_common import env_grids, golden, inputs, op_of, py_rows
from oracle.sequential import OracleError, sequential_loop
from paper_1609_04567_b200 import jit
from paper_1609_04567_b200.loop import LoopPlan


class _HostGrid:
    """env for the oracle: the reference Grid's at / in_range over an array."""

    def __init__(self, a):
        self.a = np.asarray(a)
        self.dims = self.a.shape

    def at(self, *idx):
        if len(idx) != len(self.dims) or not all(0 <= i < d for i, d in zip(idx, self.dims)):
            raise sk.GridError("out of range")
        v = self.a[idx]
        return v if self.a.dtype == np.float32 else v.item()

    def in_range(self, *idx):
        return len(idx) == len(self.dims) and all(0 <= i < d for i, d in zip(idx, self.dims))


def _oracle(spec):
    g, env = inputs(spec)
    oenv = tuple(_HostGrid(e) for e in env) if isinstance(env, tuple) else (
        _HostGrid(env) if env is not None else None)
    kind, fn = spec["op"]
    op = (lambda a, b: a + b) if kind == "sum" else (lambda a, b: a if b < a else b) \
        if kind == "max" else fn
    return sequential_loop(spec["point"], spec["k"], op, spec["identity"], J.cond_fn(spec),
                           py_rows(g), env=oenv, delta=spec["delta"],
                           indexed=spec.get("indexed", False), max_iterations=spec.get("max_it", 10_000))


@pytest.mark.parametrize("name", sorted({**J.CASES, **J.CASES_1D}))
def test_oracle_matches_reference(name):
    meta, arrays = golden()
    rows, it, val, ex = _oracle({**J.CASES, **J.CASES_1D}[name])
    m = meta[name]
    assert it == m["iterations"] and ex == m["exhausted"]
    assert float(val) == m["final_reduce"]
    got = np.asarray(rows)
    want = arrays[name]
    assert got.shape == want.shape
    assert np.array_equal(got.astype(want.dtype).view(np.uint8), want.view(np.uint8))


@pytest.mark.parametrize("name", sorted(J.ERROR_CASES))
def test_oracle_errors_match_reference(name):
    meta, _ = golden()
    with pytest.raises(OracleError) as ei:
        _oracle(J.ERROR_CASES[name])
    assert list(ei.value.index) == meta[name]["index"]
    assert type(ei.value.cause).__name__ == meta[name]["error"]


@pytest.mark.parametrize("name", sorted({**J.CASES, **J.ERROR_CASES, **J.CASES_1D}))
def test_case_compiles(name):
    spec = {**J.CASES, **J.ERROR_CASES, **J.CASES_1D}[name]
    g, env = inputs(spec)
    plan = LoopPlan(fn=sk.ElementalFn(point=spec["point"], k=spec["k"]), k=spec["k"],
                    op=op_of(spec), env=env_grids(env),
                    indexed=spec.get("indexed", False),
                    delta=sk.Delta(spec["delta"]) if spec["delta"] is not None else None)
    prog = jit.build_program(plan, sk.Grid(g.shape, g))
    assert prog.handle
    assert prog.in_dtype == g.dtype
    assert prog.out_dtype == {np.float32: np.float32}.get(g.dtype.type, prog.out_dtype)
    assert "sk_elemental_1" in prog.source and "sk_elemental_n" in prog.source


def test_reference_apps_point_functions_compile():
    """The reference's own app point functions, as written (life, sobel)."""
    import sys

    ref = "/root/reference/pkg/src"
    import os

    if not os.path.isdir(ref):
        pytest.skip("reference not present")
    sys.path.insert(0, ref)
    try:
        from stencilkit.apps import helmholtz as rh, life as rl, sobel as rs
        import stencilkit as R
    finally:
        sys.path.remove(ref)
    gi = sk.Grid((8, 9), np.zeros((8, 9), np.int64))
    for f, op in ((rl.life_kernel, rl.liveness_op()), (R.ElementalFn(rs._sobel_point, 1), rs._pixel_sum())):
        jit.build_program(LoopPlan(fn=f, k=1, op=op), gi)
    gf = sk.Grid((8, 9), np.zeros((8, 9)))
    jit.build_program(LoopPlan(fn=rh.helmholtz_kernel(rh.HelmholtzConfig(8, 9)), k=1,
                               op=R.max_combinator(0.0), env=gf, delta=sk.abs_change()), gf)


def _nested(nb, env):
    def helper(x):
        return x + 1

    return helper(nb.center)


def _listy(nb, env):
    terms = []
    for v in nb.values():
        terms.append(v)
    return len(terms)


@pytest.mark.parametrize("fn", [_nested, _listy, lambda nb, env: str(nb.center)])
def test_untranslatable_is_rejected(fn):
    g = sk.Grid((4, 4), np.zeros((4, 4)))
    plan = LoopPlan(fn=sk.ElementalFn(point=fn, k=1), k=1, op=sk.sum_combinator(0.0))
    with pytest.raises(sk.DeviceUnsupported):
        jit.build_program(plan, g)


def test_cuda_source_elemental_compiles():
    f = jit.cuda_elemental(
        "return 0.25 * (nb.at(-1, 0) + nb.at(1, 0) + nb.at(0, -1) + nb.at(0, 1));", k=1)
    g = sk.Grid((5, 7), np.zeros((5, 7)))
    prog = jit.build_program(LoopPlan(fn=f, k=1, op=sk.max_combinator(0.0),
                                      delta=sk.abs_change()), g)
    assert prog.out_dtype == np.float64 and prog.reduce == 2


def test_compile_error_reports_log():
    f = jit.cuda_elemental("return undefined_symbol;", k=1)
    g = sk.Grid((5, 7), np.zeros((5, 7)))
    with pytest.raises(sk.DeviceUnsupported) as ei:
        jit.build_program(LoopPlan(fn=f, k=1, op=sk.sum_combinator(0.0)), g)
    assert "undefined_symbol" in str(ei.value)


def test_pattern_wrappers_compile():
    """apply_to_all's wrapper (a lambda calling the user's lambda) and an
    indexed identity stencil compile."""
    g = sk.Grid((6, 9), np.arange(54, dtype=np.int64).reshape(6, 9))
    f = lambda x: x * x - 3 * x if x > 0 else -x  # noqa: E731
    wrap = sk.ElementalFn(point=lambda nb, env: f(nb.center), k=0)
    prog = jit.build_program(LoopPlan(fn=wrap, k=0, op=sk.sum_combinator(0)), g)
    assert prog.out_dtype == np.int64
    idx = sk.ElementalFn(point=lambda nb, env: nb.center[0] + nb.center[1][0], k=0)
    jit.build_program(LoopPlan(fn=idx, k=0, op=sk.sum_combinator(0), indexed=True), g)
    mn = sk.Combinator(lambda p, q: p if p < q else q, 10 ** 6)
    jit.build_program(LoopPlan(fn=sk.ElementalFn(point=lambda nb, env: nb.center, k=0), k=0,
                               op=mn), g)


def test_interior_window_specialisation():
    """Elementals are templated on the window type (interior tiles fold the
    ABSENT tests away); env reads at the centre use the unchecked centre
    access, env reads within the radius are guarded by nb.inner()."""
    assert jit._centre_offset("((long long)nb.i)", "i") == 0
    assert jit._centre_offset("((long long)nb.i + 0)", "i") == 0
    assert jit._centre_offset("((long long)nb.j - 2)", "j") == -2
    assert jit._centre_offset("((long long)nb.j + v)", "j") is None
    assert jit._centre_offset("((long long)nb.i + 1)", "j") is None

    def near(nb, env):
        i, j = nb.center_index
        return nb.center + env.at(i, j) + env.at(i - 1, j + 1) + env.at(i + 3, j)

    g = np.random.default_rng(1).random((20, 140))
    e = np.random.default_rng(2).random((20, 140))
    plan = LoopPlan(fn=sk.ElementalFn(point=near, k=1), k=1, op=sk.sum_combinator(0.0),
                    env=sk.Grid(e.shape, e))
    src = jit.build_program(plan, sk.Grid(g.shape, g)).source
    assert "template <class NB> __device__ sk_val_t sk_elemental_1(const NB& nb" in src
    # every env read carries the window-radius test (the C compiler folds it
    # for centre-plus-literal indices); the bounds checks stay behind it
    body1 = src[src.index("sk_elemental_1"):src.index("sk_elemental_n")]
    assert body1.count("sk_env_near(nb, ") == 3
    assert body1.count("_near && !env.ok(") == 3

    def centre(nb, env):
        return nb.center + env.at(*nb.center_index)

    plan = LoopPlan(fn=sk.ElementalFn(point=centre, k=1), k=1, op=sk.sum_combinator(0.0),
                    env=sk.Grid(e.shape, e))
    src = jit.build_program(plan, sk.Grid(g.shape, g)).source
    assert "nb.template centre_env<double>(env, 0)" in src and "env.ok(" not in src
