"""The documented plugin route on the GPU: the
reference's own host loop -- `loop_stencil_reduce*` -> `_as_plan` ->
`_drive` (loop.py:113-121, 198-268), here through tests/ref_shim.py, its
restatement pinned against the real reference by tests/test_ref_shim.py --
driving our DeviceExecutor with the reference's own value types
(list-backed Grid, its ElementalFn / Combinator / Delta / Condition).
`_drive` is host-driven, so this exercises begin -> step x N (lag-1) ->
finish, not our device loop."""

import math

import numpy as np
import pytest

import jit_cases as J
import paper_1609_04567_b200 as sk
import ref_shim as S
from jit_common import golden as jit_golden
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

pytestmark = pytest.mark.gpu


def test_helmholtz_through_reference_drive(golden):
    """helmholtz_solve's loop (apps/helmholtz.py:108-135), called the way a
    stencilkit user would with our kernel + executor: fp64 rhs as a list
    Grid, RMS condition as a Python lambda, delta / combinator as the
    reference's objects.  Grid bit-identical to the reference's fixture."""
    name = "helm_f64_rand_64x48_P1"
    m = golden.meta[name]
    rhs = golden[name + "/rhs"]
    n, c = rhs.shape
    nm = n * c
    tol = m["tol"]
    for P in (1, 2):
        ex = sk.DeviceExecutor(P)
        out, rep = S.loop_stencil_reduce_d(
            1, helmholtz_kernel(HelmholtzConfig(n, c, tol=tol)),
            S.Delta(lambda a, b: (a - b) ** 2), S.sum_combinator(0.0),
            lambda v, it, s: math.sqrt(v / nm) < tol,
            S.Grid((n, c), [0.0] * nm), env=S.Grid((n, c), rhs.ravel().tolist()),
            executor=ex)
        assert rep.iterations == m["iterations"] and rep.exhausted == m["exhausted"]
        assert rep.final_reduce == pytest.approx(m["final_reduce"], rel=1e-12)
        assert np.array_equal(out.to_array(), golden[name + "/out"])
        assert ex.launches >= rep.iterations  # the host loop: one launch per step


@pytest.mark.parametrize("name", ["life_glider", "sobel_int", "median3_int"])
def test_user_elemental_through_reference_drive(name):
    """A plain Python point function handed to the reference's
    loop_stencil_reduce with our executor: compiled for the device by the
    executor, driven by the reference's host loop; grid and report equal
    the reference's own run of the same call (golden_jit)."""
    meta, arrays = jit_golden()
    spec = J.CASES[name]
    g = spec["grid"]()
    kind = spec["op"][0]
    op = S.sum_combinator(spec["identity"]) if kind == "sum" else S.max_combinator(
        spec["identity"])
    cond = S.Condition(J.cond_fn(spec), spec.get("max_it", 10_000))
    grid = S.Grid(g.shape, np.asarray(g).ravel().tolist())
    if spec["delta"] is None:
        out, rep = S.loop_stencil_reduce(spec["k"], spec["point"], op, cond, grid,
                                         executor=sk.DeviceExecutor(1))
    else:
        out, rep = S.loop_stencil_reduce_d(spec["k"], spec["point"], S.Delta(spec["delta"]), op,
                                           cond, grid, executor=sk.DeviceExecutor(1))
    m = meta[name]
    assert rep.iterations == m["iterations"] and rep.exhausted == m["exhausted"]
    assert rep.final_reduce == m["final_reduce"]
    assert np.array_equal(out.to_array(), arrays[name])
