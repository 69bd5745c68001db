"""Helmholtz loops on grids that fit on chip (the register-resident
whole-loop kernel, helm_resident) at widths that are not a multiple of a
thread's vector, against the oracle bit for bit, beside the batched
(timing) loop form on the same inputs.  Regression: a lane whose vector
straddled the last column once wrote its f tail over the next row's head in
shared memory, a race the aligned BASELINE widths never showed."""

import numpy as np
import pytest

import paper_1609_04567_b200 as sk

pytestmark = pytest.mark.gpu

SHAPES = [(515, 777), (300, 1023), (1100, 2047), (37, 5), (600, 1538), (64, 130), (9, 2041)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dtype,op,delta", [(np.float32, "max", "abs"), (np.float64, "sum", "sq"),
                                            (np.float32, "sum", "abs")])
def test_resident_loop_odd_widths_match_oracle(shape, dtype, op, delta):
    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

    n, m = shape
    rng = np.random.default_rng(n * 7 + m)
    u0 = rng.random((n, m)).astype(dtype)
    f = rng.random((n, m)).astype(dtype)
    cfg = HelmholtzConfig(rows=n, cols=m, alpha=0.5, dx=0.5, dy=0.25, relax=0.9)
    tol = 1e-4 if op == "max" else 1e-3
    want, it, v, _ = O.helmholtz_loop(u0, f, O.helmholtz_consts(0.5, 0.5, 0.25, 0.9),
                                      delta=delta, op=op, cond=lambda val, i: val < tol,
                                      max_iterations=60)
    comb = sk.max_combinator(0.0) if op == "max" else sk.sum_combinator(0.0)
    dl = sk.abs_change() if delta == "abs" else sk.Delta(lambda a, b: (a - b) ** 2, kind="square")
    for ex in (None, sk.DeviceExecutor(1, timing=True)):
        out, rep = sk.loop_stencil_reduce_d(1, helmholtz_kernel(cfg), dl, comb,
                                            sk.Condition.below(tol, max_iterations=60),
                                            sk.Grid(u0.shape, u0), env=sk.Grid(f.shape, f),
                                            executor=ex)
        got = out.to_array()
        assert rep.iterations == it, (shape, ex)
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (shape, ex)
        if op == "max":
            assert rep.final_reduce == v
        else:
            assert rep.final_reduce == pytest.approx(v, rel=1e-12 if dtype == np.float64 else 1e-5)
