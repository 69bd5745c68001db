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


def test_app_kernels_through_reference_drive():
    """The hand-written app kernels (Sobel, adaptive-median detection,
    variational restore) behind the reference's own host loop with our
    executor: each equals the oracle's restatement of the reference, with
    the reference's iteration count for the restore loop."""
    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import RestoreConfig, detect_kernel, restore_kernel, sobel_kernel

    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (61, 93))
    grid = S.Grid(img.shape, img.ravel().tolist())
    out, rep = S.loop_stencil_reduce(1, sobel_kernel, S.sum_combinator(0),
                                     S.Condition(lambda v, it, s: it >= 1), grid,
                                     executor=sk.DeviceExecutor(2))
    want = O.sobel(img)
    assert np.array_equal(np.asarray(out.to_array()).astype(np.uint8), want)
    assert rep.iterations == 1 and rep.final_reduce == int(want.astype(np.int64).sum())

    base = ((np.arange(48)[:, None] * 3 + np.arange(70)[None, :] * 2) % 200 + 20)
    noisy, _ = O.salt_pepper(base, 0.3, seed=9)
    g = S.Grid(noisy.shape, noisy.ravel().tolist())
    mask, mrep = S.loop_stencil_reduce(3, detect_kernel(7), S.sum_combinator(0),
                                       S.Condition(lambda v, it, s: it >= 1), g,
                                       executor=sk.DeviceExecutor(1))
    wm = O.amf_detect(noisy)
    assert np.array_equal(np.asarray(mask.to_array()).astype(np.uint8), wm)
    cfg = RestoreConfig()
    denom = max(int(wm.sum()), 1)
    mg = S.Grid(wm.shape, wm.astype(np.int64).ravel().tolist())
    out, rep = S.loop_stencil_reduce_d(
        1, restore_kernel(cfg), S.Delta(lambda a, b: abs(a - b)), S.sum_combinator(0.0),
        S.Condition(lambda v, it, s: v / denom < cfg.tol, cfg.max_iterations),
        S.Grid(noisy.shape, [float(v) for v in noisy.ravel()]), env=mg, indexed=True,
        executor=sk.DeviceExecutor(2))
    wo, it, v, ex = O.restore_loop(noisy, wm, P=2)
    assert rep.iterations == it and rep.exhausted == ex
    assert rep.final_reduce == pytest.approx(v, rel=1e-12)
    assert np.array_equal(np.asarray(out.to_array(), dtype=np.float64).view(np.uint64),
                          wo.view(np.uint64))
