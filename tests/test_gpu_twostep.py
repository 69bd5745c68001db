"""Two loop iterations per kernel launch (helmholtz_sweep2, temporal
blocking; opt-in with SK_TWOSTEP=1) against one iteration per launch: identical grids, iteration
counts, final values (MAX and SUM) and exhaustion flags, for stops on the
first (fix-up sweep) and second iteration of a pair, partial vectors and
several column blocks, fp32 and fp64, P = 1 and 3 partitions."""

import numpy as np
import pytest

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

pytestmark = pytest.mark.gpu


def _run(monkeypatch, twostep, n, m, dtype, cond, reduce, P, executor=None):
    monkeypatch.setenv("SK_NO_PERSIST", "1")  # the graph / batched device loop
    monkeypatch.setenv("SK_TWOSTEP", "1" if twostep else "0")
    rhs = np.random.default_rng(n * 7 + m).random((n, m)).astype(dtype)
    cfg = HelmholtzConfig(n, m, alpha=0.5, dx=0.5, dy=0.25, relax=0.8)
    op, delta = (sk.max_combinator(0.0), sk.abs_change()) if reduce == "max" else \
        (sk.sum_combinator(0.0), sk.sq_change())
    out, rep = sk.parallel_loop("1:n" if P > 1 else "1:1", P, 1, helmholtz_kernel(cfg), op, cond,
                                sk.Grid(rhs.shape, np.zeros_like(rhs)), env=sk.Grid(rhs.shape, rhs),
                                delta=delta)
    return out.to_array(), rep


CASES = [
    (200, 136, np.float32, "below", "max", 3),
    (1000, 1300, np.float32, "below", "max", 1),
    (257, 700, np.float64, "below", "sum", 1),
    (300, 520, np.float32, "after5", "max", 1),   # stops on the first of a pair
    (300, 520, np.float32, "after6", "sum", 2),   # stops on the second
    (129, 515, np.float64, "cap7", "max", 1),     # exhausted on an odd iteration
    (129, 515, np.float32, "cap8", "sum", 3),     # exhausted on an even one
]


def _cond(kind):
    if kind == "below":
        return sk.Condition.below(1e-4)
    if kind.startswith("after"):
        return sk.stop_after(int(kind[5:]))
    return sk.Condition.below(1e-30, max_iterations=int(kind[3:]))


@pytest.mark.parametrize("n,m,dtype,cond,reduce,P", CASES)
def test_two_iterations_per_launch_match_one(monkeypatch, n, m, dtype, cond, reduce, P):
    a, ra = _run(monkeypatch, True, n, m, dtype, _cond(cond), reduce, P)
    b, rb = _run(monkeypatch, False, n, m, dtype, _cond(cond), reduce, P)
    assert (ra.iterations, ra.exhausted) == (rb.iterations, rb.exhausted)
    assert ra.final_reduce == rb.final_reduce
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_batched_timing_mode_two_step(monkeypatch):
    """The bench's timed mode (batched launches, device-decided stop)."""
    monkeypatch.setenv("SK_TWOSTEP", "1")
    n = 1024
    u0 = sk.Grid((n, n), np.zeros((n, n), np.float32))
    f = sk.Grid((n, n), np.ones((n, n), np.float32))
    ex = sk.DeviceExecutor(1, timing=True)
    out, rep = sk.loop_stencil_reduce_d(1, helmholtz_kernel(HelmholtzConfig(n, n)),
                                        sk.abs_change(), sk.max_combinator(0.0),
                                        sk.Condition.below(1e-4), u0, env=f, executor=ex)
    assert rep.iterations == 36
    ms, launches = ex.last_kernel_time
    assert launches == 18  # two iterations per timed launch
    monkeypatch.setenv("SK_TWOSTEP", "0")
    out2, rep2 = sk.loop_stencil_reduce_d(1, helmholtz_kernel(HelmholtzConfig(n, n)),
                                          sk.abs_change(), sk.max_combinator(0.0),
                                          sk.Condition.below(1e-4), u0, env=f,
                                          executor=sk.DeviceExecutor(1, timing=True))
    assert rep2.final_reduce == rep.final_reduce
    assert np.array_equal(out.to_array().view(np.uint32), out2.to_array().view(np.uint32))
