"""User elemental functions compiled at run time (NVRTC, sm_100a) vs the
REAL reference's outputs (golden_jit.*, tests/golden/make_golden_jit.py)
and the sequential oracle (oracle/sequential.py).

Bar: identical iteration counts and exhaustion flags; grids bit-identical
(the cases use only +, -, *, /, //, %, ** and sqrt, which the device
evaluates exactly like Python / numpy float32); MAX and integer reduces
bit-equal; float SUM reduces within rel 1e-12 (fp64 tree vs the reference's
left fold).  Elemental failures raise StencilError at the same index with
the same exception type as the reference.
"""

import math

import numpy as np
import pytest

import jit_cases as J
import paper_1609_04567_b200 as sk
from jit_common import as_grid, golden, host_cond, inputs, op_of, py_rows, run_device
from oracle.sequential import sequential_loop
from paper_1609_04567_b200 import jit

pytestmark = pytest.mark.gpu

SUM_RTOL = 1e-12


def _check(name, out, rep):
    meta, arrays = golden()
    m = meta[name]
    want = arrays[name]
    assert rep.iterations == m["iterations"], (rep.iterations, m["iterations"])
    assert rep.exhausted == m["exhausted"]
    got = out.to_array()
    assert got.dtype == want.dtype, (got.dtype, want.dtype)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), \
        f"{name}: {np.count_nonzero(got != want)} elements differ"
    kind = {**J.CASES, **J.CASES_1D}[name]["op"][0]
    fr = float(rep.final_reduce)
    if kind == "sum" and not m["final_is_int"]:
        assert math.isclose(fr, m["final_reduce"], rel_tol=SUM_RTOL, abs_tol=1e-300)
    else:
        assert fr == m["final_reduce"]
    if m["final_is_int"]:
        assert isinstance(rep.final_reduce, int)


@pytest.mark.parametrize("name", sorted(J.CASES))
def test_case_device_loop(name):
    out, rep = run_device(J.CASES[name])
    _check(name, out, rep)


@pytest.mark.parametrize("name", sorted(J.CASES_1D))
def test_rank1_grid(name):
    """Rank-1 grids (the reference's 1D route, partition.py:369-404)."""
    out, rep = run_device(J.CASES_1D[name])
    assert out.dims == J.CASES_1D[name]["grid"]().shape
    _check(name, out, rep)
    out3, rep3 = run_device(J.CASES_1D[name], P=3)
    _check(name, out3, rep3)


@pytest.mark.parametrize("name", ["jacobi_f64", "life_glider", "int_mix", "f32_relax"])
def test_case_host_condition(name):
    """A Python condition + LoopState: host-driven steps with lag-1
    speculation; state.update then cond once per iteration (loop.py:209-218)."""
    spec = J.CASES[name]
    seen = []
    state = sk.LoopState(init=lambda: 0, update=lambda s, it, v: (seen.append(it), s + 1)[1])
    out, rep = run_device(spec, cond=host_cond(spec), state=state)
    _check(name, out, rep)
    assert seen == list(range(1, rep.iterations + 1))


@pytest.mark.parametrize("name,P", [("jacobi_f64", 3), ("life_glider", 4), ("median3_int", 2)])
def test_case_partitions(name, P):
    """1:n partitions: same grid, same reduce (MAX / int SUM are order-free)."""
    out, rep = run_device(J.CASES[name], P=P)
    _check(name, out, rep)


@pytest.mark.parametrize("name", sorted(J.ERROR_CASES))
def test_error_cases_raise_stencil_error(name):
    meta, _ = golden()
    with pytest.raises(sk.StencilError) as ei:
        run_device(J.ERROR_CASES[name])
    assert list(ei.value.index) == meta[name]["index"]
    assert meta[name]["error"] in str(ei.value)


def test_error_after_host_condition_stop_is_not_raised():
    """A failure only in the speculative iteration past the stop is not an
    error: the loop had already ended (lag-1 speculation must not leak)."""
    calls = []

    def fails_late(nb, env):
        c = nb.center
        return c + 1.0 if c < 1.5 else 1.0 / (c - c)

    g = sk.Grid((6, 40), np.zeros((6, 40)))
    cond = sk.Condition(lambda v, it, s: (calls.append(it), it >= 2)[1])
    out, rep = sk.loop_stencil_reduce(1, sk.ElementalFn(fails_late, 1), sk.sum_combinator(0.0),
                                      cond, g)
    assert rep.iterations == 2 and calls == [1, 2]
    assert np.all(out.to_array() == 2.0)


def test_cuda_source_elemental_matches_python_form():
    """The paper's API (kernel source) and the Python point form of the same
    Jacobi update give bit-identical loops."""
    spec = J.CASES["jacobi_f64"]
    body = f"""
      const double c = nb.center();
      const double f = env.get<double>(0, nb.i, nb.j);
      return (1.0 - {J._RELAX!r}) * c + {J._RELAX!r} * (f + {J._AX!r} * (nb.at(0, -1) + nb.at(0, 1))
             + {J._AY!r} * (nb.at(-1, 0) + nb.at(1, 0))) / {J._B!r};
    """
    f = jit.cuda_elemental(body, k=1, pad_value=0.0)
    g, env = inputs(spec)
    out, rep = sk.loop_stencil_reduce_d(1, f, sk.abs_change(), sk.max_combinator(0.0),
                                        sk.Condition.below(spec["cond"][1], spec["max_it"]),
                                        as_grid(g), env=as_grid(env))
    _check("jacobi_f64", out, rep)


def test_custom_delta_and_combinator_vs_oracle():
    """Python delta + custom combinator on a larger grid (several tiles and
    partitions) against the oracle run on the box."""
    def pt(nb, env):
        c = nb.center
        s = 0
        for v in nb.values():
            s += v % 7
        return (c * 3 + s) % 101

    rng = np.random.default_rng(21)
    a = rng.integers(0, 101, (70, 300)).astype(np.int64)
    op = sk.Combinator(lambda x, y: x if x > y else y, -1)
    delta = sk.Delta(lambda new, old: (new - old) % 13)
    out, rep = sk.parallel_loop("1:n", 3, 1, sk.ElementalFn(pt, 1), op, sk.stop_after(3),
                                as_grid(a), delta=delta)
    rows, it, val, ex = sequential_loop(pt, 1, op.fn, -1, lambda v, i, s: i >= 3, a.tolist(),
                                        delta=delta.fn, partitions=3)
    assert rep.iterations == it == 3
    assert rep.final_reduce == val and isinstance(rep.final_reduce, int)
    assert np.array_equal(out.to_array(), np.asarray(rows))


def test_reference_executor_protocol_drop_in():
    """The reference loop API shape: our DeviceExecutor passed as the
    executor of loop_stencil_reduce with a plain Python point function."""
    spec = J.CASES["sobel_int"]
    g, _ = inputs(spec)
    ex = sk.DeviceExecutor(1)
    out, rep = sk.loop_stencil_reduce(1, J.sobel, sk.sum_combinator(0), sk.stop_after(1),
                                      as_grid(g), executor=ex)
    _check("sobel_int", out, rep)


def test_map_and_reduce_patterns_compile_python_functions():
    """apply_to_all / reduce_all / stencil_apply_indexed with plain Python
    callables (patterns.py:138-192) run as compiled device programs."""
    a = np.random.default_rng(30).integers(-50, 50, (40, 200)).astype(np.int64)
    g = as_grid(a)
    out = sk.apply_to_all(lambda x: x * x - 3 * x if x > 0 else -x, g)
    want = np.where(a > 0, a * a - 3 * a, -a)
    assert np.array_equal(out.to_array(), want)
    mn = sk.reduce_all(sk.Combinator(lambda p, q: p if p < q else q, 10 ** 6), g)
    assert mn == int(a.min()) and isinstance(mn, int)
    assert sk.reduce_all(sk.sum_combinator(0), g) == int(a.sum())

    def idx_pt(nb, env):
        v, (i, j) = nb.center
        return v + 1000 * i + j

    out = sk.stencil_apply_indexed(idx_pt, 0, g)
    ii, jj = np.indices(a.shape)
    assert np.array_equal(out.to_array(), a + 1000 * ii + jj)


def test_cuda_source_delta_and_combinator():
    spec = J.CASES["box_mean_r2"]
    g, _ = inputs(spec)
    d = sk.Delta(sk.CudaDelta("const double t = nw - old; return t * t;"))
    op = sk.Combinator(sk.CudaCombine("return a + b;"), 0.0)
    out, rep = sk.loop_stencil_reduce_d(2, sk.ElementalFn(J.box_mean, 2), d, op, sk.stop_after(4),
                                        as_grid(g))
    meta, arrays = golden()
    assert np.array_equal(out.to_array(), arrays["box_mean_r2"])
    assert math.isclose(rep.final_reduce, meta["box_mean_r2"]["final_reduce"], rel_tol=1e-12)


def test_plain_lambda_condition_runs_on_the_device():
    """A threshold lambda (`v < tol`) is recognised and the loop runs on the
    device (one persistent launch), with the host-driven loop's result."""
    spec = J.CASES["jacobi_f64"]
    g, env = inputs(spec)
    ex = sk.DeviceExecutor(1)
    tol = spec["cond"][1]
    out, rep = sk.loop_stencil_reduce_d(1, sk.ElementalFn(J.jacobi, 1), sk.abs_change(),
                                        sk.max_combinator(0.0),
                                        sk.Condition(lambda v, it, s: v < tol, spec["max_it"]),
                                        as_grid(g), env=as_grid(env), executor=ex)
    assert ex.launches == 1
    _check("jacobi_f64", out, rep)


def _wide1d(nb, env):
    """radius-2 rank-1 smoothing with ABSENT edges (many tiles of the 1D sweep)"""
    c = nb.center
    s = c
    n = 1
    for d in (-2, -1, 1, 2):
        v = nb.at(d)
        if v is not ABSENT_1D:
            s = s + v
            n += 1
    (i,) = nb.center_index
    return 0.25 * c + 0.75 * (s / n) + 0.001 * env.at(i)


ABSENT_1D = J.ABSENT


@pytest.mark.parametrize("n,P", [(10007, 1), (20011, 3)])
def test_rank1_multi_tile_matches_oracle(n, P):
    """Rank-1 grids run as contiguous element tiles (2048 + radius per tile):
    several tiles and partitions against the sequential oracle."""
    g = np.random.default_rng(21).random(n)
    e = np.random.default_rng(22).random(n)
    f = sk.ElementalFn(point=_wide1d, k=2)
    out, rep = sk.parallel_loop("1:n" if P > 1 else "1:1", P, 2, f, sk.max_combinator(0.0),
                                sk.stop_after(4), sk.Grid((n,), g), env=sk.Grid((n,), e),
                                delta=sk.Delta(lambda a, b: abs(a - b)))

    class _E:
        def __init__(self, a):
            self.a, self.dims = a, a.shape

        def at(self, *idx):
            return self.a[idx].item()

        def in_range(self, *idx):
            return 0 <= idx[0] < self.a.shape[0]

    ref, it, val, ex = sequential_loop(_wide1d, 2, lambda a, b: a if b < a else b, 0.0,
                                       lambda v, i, s: i >= 4, [float(x) for x in g],
                                       env=_E(e), delta=lambda a, b: abs(a - b))
    assert rep.iterations == it == 4
    assert np.array_equal(out.to_array(), np.asarray(ref))
    assert float(rep.final_reduce) == val


def _near_sum(a, b):
    return a + b if b < 50 else a  # == a + b on small partials only


def _near_abs(n, o):
    return abs(n - o) if abs(n - o) < 100 else 0.0


def test_near_miss_combinator_and_delta_compile_as_written():
    """A combinator / delta that agree with SUM / |new-old| on small inputs
    but not everywhere: before round 2 they were classified by sampling and
    ran as the built-in reduce; now they are compiled as written, and the
    device matches the reference's sequential fold of op.fn
    (loop.py:163-191, partition.py:642-646) exactly."""
    def pt(nb, env):
        s = 0.0
        for v in nb.values():
            s += v
        return s * 0.25 + 7.0

    rng = np.random.default_rng(5)
    a = rng.random((67, 301)) * 200.0
    for P in (1, 3):
        op = sk.Combinator(_near_sum, 0.0)
        delta = sk.Delta(_near_abs)
        out, rep = sk.parallel_loop("1:n" if P > 1 else "1:1", P, 1, sk.ElementalFn(pt, 1), op,
                                    sk.stop_after(4), as_grid(a), delta=delta)
        rows, it, val, ex = sequential_loop(pt, 1, _near_sum, 0.0, lambda v, i, s: i >= 4,
                                            a.tolist(), delta=_near_abs, partitions=P)
        assert rep.iterations == it == 4
        assert rep.final_reduce == val, (P, rep.final_reduce, val)
        assert np.array_equal(out.to_array(), np.asarray(rows))
        # the plain SUM of |delta| differs: the near-miss really is exercised
        plain = sk.parallel_loop("1:n" if P > 1 else "1:1", P, 1, sk.ElementalFn(pt, 1),
                                 sk.sum_combinator(0.0), sk.stop_after(4), as_grid(a),
                                 delta=sk.abs_change())[1].final_reduce
        assert plain != val


def test_builtin_kernel_rejects_unrecognised_reduce():
    """The hand-written kernels only have the SUM / MAX reduce and abs /
    square deltas: anything else is refused loudly, never approximated."""
    from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

    rhs = np.ones((40, 40), np.float32)
    with pytest.raises(sk.DeviceUnsupported):
        sk.parallel_loop("1:1", 1, 1, helmholtz_kernel(HelmholtzConfig(40, 40)),
                         sk.Combinator(_near_sum, 0.0), sk.Condition.below(1e-4),
                         sk.Grid(rhs.shape, np.zeros_like(rhs)), env=sk.Grid(rhs.shape, rhs),
                         delta=sk.abs_change())
    with pytest.raises(sk.DeviceUnsupported):
        sk.parallel_loop("1:1", 1, 1, helmholtz_kernel(HelmholtzConfig(40, 40)),
                         sk.max_combinator(0.0), sk.Condition.below(1e-4),
                         sk.Grid(rhs.shape, np.zeros_like(rhs)), env=sk.Grid(rhs.shape, rhs),
                         delta=sk.Delta(_near_abs))
