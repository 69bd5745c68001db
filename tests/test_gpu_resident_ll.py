"""The barrier-free resident Helmholtz loop (helm_resident_ll: halo rows and
reduce partials exchanged as iteration-tagged 8-byte words, the loop
decision taken one iteration late) against the oracle bit for bit, and
against the barrier form (SK_RES_LL=0) on the same inputs.

Covers every band height 1..8 (rows up to 8 x 148), both MAX deltas, odd
widths, the iteration cap landing on the speculative iteration, and many
back-to-back solves on one stream with different caps (the per-stream
exchange buffer is never cleared: stale words from earlier solves must
never match a new solve's tags)."""

import os

import numpy as np
import pytest

import paper_1609_04567_b200 as sk

pytestmark = pytest.mark.gpu


def _solve(u0, f, cfg, delta, tol, max_it, ll=True, op="max"):
    from paper_1609_04567_b200.apps import helmholtz_kernel

    old = os.environ.get("SK_RES_LL")
    os.environ["SK_RES_LL"] = "1" if ll else "0"
    try:
        dl = sk.abs_change() if delta == "abs" else sk.Delta(lambda a, b: (a - b) ** 2, kind="square")
        comb = sk.max_combinator(0.0) if op == "max" else sk.sum_combinator(0.0)
        out, rep = sk.loop_stencil_reduce_d(1, helmholtz_kernel(cfg), dl, comb,
                                            sk.Condition.below(tol, max_iterations=max_it),
                                            sk.Grid(u0.shape, u0), env=sk.Grid(f.shape, f))
    finally:
        if old is None:
            del os.environ["SK_RES_LL"]
        else:
            os.environ["SK_RES_LL"] = old
    return out.to_array(), rep


# band = ceil(rows / 148): 1 (100 rows) .. 8 (1100 rows), odd widths
SHAPES = [(100, 64), (250, 333), (400, 1024), (520, 77), (700, 1000), (800, 515), (1024, 1024),
          (1100, 1023)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("delta", ["abs", "sq"])
def test_ll_resident_matches_oracle(shape, delta):
    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import HelmholtzConfig

    n, m = shape
    rng = np.random.default_rng(n * 31 + m)
    u0 = rng.random((n, m)).astype(np.float32)
    f = rng.random((n, m)).astype(np.float32)
    cfg = HelmholtzConfig(rows=n, cols=m, alpha=0.5, dx=0.5, dy=0.25, relax=0.9)
    tol = 1e-4 if delta == "abs" else 1e-8
    want, it, v, ex = O.helmholtz_loop(u0, f, O.helmholtz_consts(0.5, 0.5, 0.25, 0.9), delta=delta,
                                       op="max", cond=lambda val, i: val < tol, max_iterations=80)
    got, rep = _solve(u0, f, cfg, delta, tol, 80)
    assert rep.iterations == it and rep.exhausted == ex
    assert rep.final_reduce == v
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    got0, rep0 = _solve(u0, f, cfg, delta, tol, 80, ll=False)
    assert rep0.iterations == it and np.array_equal(got0.view(np.uint32), got.view(np.uint32))


def test_ll_resident_back_to_back_caps():
    """Many solves on one stream, caps 1..12 and a converging one: every
    result equals the oracle's (the cap stops the loop at the iteration the
    kernel computes speculatively past)."""
    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import HelmholtzConfig

    n, m = 1024, 1024
    rng = np.random.default_rng(5)
    u0 = rng.random((n, m)).astype(np.float32)
    f = rng.random((n, m)).astype(np.float32)
    cfg = HelmholtzConfig(rows=n, cols=m, alpha=0.5, dx=0.5, dy=0.25, relax=0.9)
    consts = O.helmholtz_consts(0.5, 0.5, 0.25, 0.9)
    ref = {}
    u = u0
    for k in range(1, 13):  # the oracle's iterate after k sweeps
        u, _, v, _ = O.helmholtz_loop(u, f, consts, delta="abs", op="max",
                                      cond=lambda val, i: False, max_iterations=1)
        ref[k] = (u.copy(), v)
    for rep_i in range(3):
        for cap in [1, 2, 3, 7, 12, 5, 1]:
            got, rep = _solve(u0, f, cfg, "abs", 1e-30, cap)
            assert rep.iterations == cap and rep.exhausted, (rep_i, cap)
            assert rep.final_reduce == ref[cap][1]
            assert np.array_equal(got.view(np.uint32), ref[cap][0].view(np.uint32)), (rep_i, cap)


def test_ll_resident_many_streams():
    """Solves issued from 40 different CUDA streams (the exchange buffer is
    cached per stream, the cache dropped past 32 streams): every result
    equals the default-stream one."""
    import torch
    from paper_1609_04567_b200.apps import HelmholtzConfig

    n, m = 512, 640
    rng = np.random.default_rng(11)
    u0 = rng.random((n, m)).astype(np.float32)
    f = rng.random((n, m)).astype(np.float32)
    cfg = HelmholtzConfig(rows=n, cols=m, alpha=0.5, dx=0.5, dy=0.25, relax=0.9)
    want, rep0 = _solve(u0, f, cfg, "abs", 1e-4, 60)
    for _ in range(40):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            got, rep = _solve(u0, f, cfg, "abs", 1e-4, 60)
        assert rep.iterations == rep0.iterations and rep.final_reduce == rep0.final_reduce
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("delta", ["abs", "sq"])
def test_ll_resident_sum_matches_barrier_form(shape, delta):
    """SUM reduces: the barrier-free loop folds the bands' partials in the
    engine's fixed tree, so grid, iteration count and final value are
    bit-identical to the barrier form (and within the fp32-sum tolerance of
    the oracle's pairwise sum)."""
    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import HelmholtzConfig

    n, m = shape
    rng = np.random.default_rng(n * 13 + m)
    u0 = rng.random((n, m)).astype(np.float32)
    f = rng.random((n, m)).astype(np.float32)
    cfg = HelmholtzConfig(rows=n, cols=m, alpha=0.5, dx=0.5, dy=0.25, relax=0.9)
    tol = 1e-3 * n * m if delta == "abs" else 1e-6 * n * m
    got, rep = _solve(u0, f, cfg, delta, tol, 60, op="sum")
    ref, rep0 = _solve(u0, f, cfg, delta, tol, 60, ll=False, op="sum")
    assert (rep.iterations, rep.exhausted) == (rep0.iterations, rep0.exhausted)
    assert np.float64(rep.final_reduce).tobytes() == np.float64(rep0.final_reduce).tobytes()
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    want, it, v, _ = O.helmholtz_loop(u0, f, O.helmholtz_consts(0.5, 0.5, 0.25, 0.9), delta=delta,
                                      op="sum", cond=lambda val, i: val < tol, max_iterations=60)
    assert rep.iterations == it
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert rep.final_reduce == pytest.approx(v, rel=1e-5)


def test_ll_resident_seeded_sweep():
    """40 seeded random geometries (rows 1..1184, cols 1..1024), MAX/SUM x
    |d| / d^2, random caps and tolerances: the barrier-free loop equals the
    barrier form bit for bit (grid, iterations, exhaustion, final value)."""
    from paper_1609_04567_b200.apps import HelmholtzConfig

    rng = np.random.default_rng(2024)
    for case in range(40):
        n = int(rng.integers(1, 1185))
        m = int(rng.integers(1, 1025))
        op = ("max", "sum")[case % 2]
        delta = ("abs", "sq")[(case // 2) % 2]
        u0 = rng.random((n, m)).astype(np.float32)
        f = rng.random((n, m)).astype(np.float32)
        cfg = HelmholtzConfig(rows=n, cols=m, alpha=float(rng.uniform(0.2, 2.0)), dx=0.5, dy=0.25,
                              relax=float(rng.uniform(0.5, 1.0)))
        tol = float(10 ** rng.uniform(-6, -2)) * (n * m if op == "sum" else 1)
        cap = int(rng.integers(1, 50))
        got, rep = _solve(u0, f, cfg, delta, tol, cap, op=op)
        ref, rep0 = _solve(u0, f, cfg, delta, tol, cap, ll=False, op=op)
        what = (case, n, m, op, delta, cap)
        assert (rep.iterations, rep.exhausted) == (rep0.iterations, rep0.exhausted), what
        assert np.float64(rep.final_reduce).tobytes() == np.float64(rep0.final_reduce).tobytes(), what
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), what
