"""reduce_all on the device (csrc/sk_reduce.cu) against the reference's
definition itself: Combinator.fold, the sequential left fold of op.fn from
the identity over the row-major elements (reference patterns.py:103-108,
143-147), evaluated here in Python with numpy scalars as the reference's
elements are.  Bit-exact, NaN / +-0 / identity cases included."""

import math

import numpy as np
import pytest

import paper_1609_04567_b200 as sk

pytestmark = pytest.mark.gpu


def ref_fold(op, arr):
    """The reference grid's elements: Python ints for integer grids
    (Grid.from_array -> tolist), numpy float32 scalars for float32 grids (the
    fixtures' convention), Python floats for float64."""
    acc = op.identity
    vals = arr.reshape(-1).tolist() if arr.dtype.kind in "iu" else arr.reshape(-1)
    for v in vals:
        acc = op.fn(acc, v)
    return acc


def same(a, b):
    if isinstance(a, float) or isinstance(b, float) or isinstance(a, np.floating):
        fa, fb = float(a), float(b)
        if math.isnan(fa) or math.isnan(fb):
            return math.isnan(fa) and math.isnan(fb)
        return np.float64(fa).tobytes() == np.float64(fb).tobytes()
    return a == b


def grid(a):
    return sk.Grid(a.shape, a)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("ident", [0, 0.0, 1.5])
def test_float_sum_is_the_sequential_fold(dt, ident):
    rng = np.random.default_rng(1)
    a = (rng.standard_normal((123, 457)) * 10.0 ** rng.integers(-3, 6, (123, 457))).astype(dt)
    op = sk.sum_combinator(ident)
    got = sk.reduce_all(op, grid(a))
    want = ref_fold(op, a)
    assert same(got, want), (got, want)
    assert type(got) is type(want) or (dt == np.float64 and isinstance(got, float))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_float_max_nan_and_signed_zero_rules(dt):
    op = sk.max_combinator(0.0)
    nan = float("nan")
    cases = [
        [1.0, 3.0, 2.0], [-1.0, -3.0], [nan, 1.0, 5.0, 2.0], [1.0, 5.0, nan, 2.0, 0.5],
        [1.0, 5.0, nan], [nan], [0.0, -0.0], [-0.0, 0.0, -0.0], [-5.0, -0.0],
        [float("-inf"), -1e300 if dt == np.float64 else -1e30], [nan, nan, -0.0],
        [3.0, 3.0, nan, 3.0, -0.0, 3.0],
    ]
    for c in cases:
        a = np.array(c, dtype=dt).reshape(1, -1)
        for o in (op, sk.max_combinator(float("nan")), sk.max_combinator(-1.0)):
            got = sk.reduce_all(o, grid(a))
            want = ref_fold(o, a)
            if not (isinstance(want, float) and math.isnan(want)):
                assert np.asarray(got, dtype=dt).tobytes() == np.asarray(want, dtype=dt).tobytes(), \
                    (c, o.identity, got, want)
            else:
                assert math.isnan(float(got)), (c, o.identity, got)
    rng = np.random.default_rng(2)
    a = rng.standard_normal((300, 301)).astype(dt)
    a[rng.random(a.shape) < 0.001] = np.nan
    a[5, 7] = 50.0
    assert same(sk.reduce_all(op, grid(a)), ref_fold(op, a))


@pytest.mark.parametrize("dt", [np.uint8, np.int32, np.int64])
def test_integer_sum_and_max(dt):
    rng = np.random.default_rng(3)
    hi = 255 if dt == np.uint8 else 10 ** 6
    a = rng.integers(0 if dt == np.uint8 else -hi, hi, (211, 97)).astype(dt)
    for op in (sk.sum_combinator(0), sk.sum_combinator(7), sk.max_combinator(0),
               sk.max_combinator(10 ** 7), sk.max_combinator(-2.5)):
        got = sk.reduce_all(op, grid(a))
        want = ref_fold(op, a)
        assert got == want and type(got) in (int, float), (op.identity, got, want)


def test_builtin_max_and_other_combinators_fold_as_written():
    a = np.array([[1.0, 4.0, 2.0], [4.0, -1.0, 3.0]])
    assert sk.reduce_all(sk.Combinator(max, 0.0), grid(a)) == 4.0
    mn = sk.reduce_all(sk.Combinator(lambda p, q: p if p < q else q, 10.0), grid(a))
    assert mn == -1.0
