"""Parity at the PRODUCTION geometry of the Helmholtz sweep.

golden_large's C1 cases fit one 512-column block or take the resident
whole-loop kernel; the kernel BASELINE C4 runs -- the non-resident
`helmholtz_sweep<T>` (csrc/sk_helmholtz.cu) with many column blocks,
>= 64-row work chunks, a ragged last column block and a padded pitch -- is
pinned here against tests/golden/golden_prod.json (make_golden_prod.py:
the REAL reference for the 4099 x 4133 and 2500 x 3000 cases, the pinned
oracle for 32768^2), in every device-loop form the engine has:

  graph      CUDA graph with a WHILE node (default above 2^24 cells)
  persistent one cooperative launch (default at or below 2^24 cells)
  batched    SK_NO_GRAPH / SK_NO_PERSIST: 8 launches per host status check
  timing     DeviceExecutor(timing=True), the bench's measured form
  host       a LoopState forces the host-driven lag-1 loop (one launch per
             iteration, the value read back per iteration)

Reference: apps/helmholtz.py:85-92 (block), :98-105 (delta/reduce),
:108-135 (helmholtz_solve), partition.py:596-664 (the partitioned loop).
"""

import hashlib
import json
import math
import os

import numpy as np
import pytest

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel, helmholtz_solve

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_prod.json")


@pytest.fixture(scope="module")
def prod():
    return json.load(open(GOLD))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rhs_for(n, m, seed):
    return np.random.default_rng(seed).random((n, m)).astype(np.float32)


FORMS = ["default", "batched", "timing", "host"]


def _env_for(form, monkeypatch):
    if form == "batched":
        monkeypatch.setenv("SK_NO_GRAPH", "1")
        monkeypatch.setenv("SK_NO_PERSIST", "1")
    else:
        monkeypatch.delenv("SK_NO_GRAPH", raising=False)
        monkeypatch.delenv("SK_NO_PERSIST", raising=False)


def _f32_run(m, form):
    import torch

    n, c, P, tol = m["rows"], m["cols"], m["P"], m["tol"]
    rhs = np.ones((n, c), np.float32) if m.get("rhs") == "ones" else rhs_for(n, c, m["seed"])
    f = torch.from_numpy(rhs).cuda()
    u0 = torch.zeros_like(f)
    kern = helmholtz_kernel(HelmholtzConfig(n, c, tol=tol))
    ex = sk.DeviceExecutor(P, timing=(form == "timing"))
    if form == "host":
        st = sk.LoopState(init=lambda: 0, update=lambda s, it, v: s + 1)
        out, rep = sk.loop_stencil_reduce_s(1, kern, sk.max_combinator(0.0),
                                            lambda v, it, s: v < tol, st, sk.Grid.from_tensor(u0),
                                            env=sk.Grid.from_tensor(f), executor=ex,
                                            delta=sk.abs_change())
    else:
        out, rep = sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0),
                                            sk.Condition.below(tol), sk.Grid.from_tensor(u0),
                                            env=sk.Grid.from_tensor(f), executor=ex)
    return out, rep, ex


@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("case", ["prod_f32_max_rand7_4099x4133_P1",
                                  "prod_f32_max_rand7_4099x4133_P3",
                                  "prod_f32_max_rand8_2500x3000_P2"])
def test_f32_sweep_production_geometry(prod, case, form, monkeypatch):
    m = prod[case]
    _env_for(form, monkeypatch)
    out, rep, ex = _f32_run(m, form)
    assert rep.iterations == m["iterations"] and rep.exhausted == m["exhausted"]
    assert rep.final_reduce == m["final_reduce"]
    assert sha(out.to_array()) == m["sha"], (case, form)
    if form == "timing":
        assert ex.last_kernel_time[1] >= m["iterations"]


@pytest.mark.parametrize("form", ["default", "batched", "timing"])
@pytest.mark.parametrize("P", [1, 3])
def test_f64_solve_production_geometry(prod, P, form, monkeypatch):
    """fp64 `helmholtz_solve` route (RMS of the squared change, SUM reduce):
    grid bit-identical, iteration count identical, the SUM within rel 1e-12
    (device partials accumulate in fp64 in a different tree than numpy's
    pairwise sum)."""
    import torch

    m = prod[f"prod_f64_solve_rand7_4099x4133_P{P}"]
    _env_for(form, monkeypatch)
    n, c, tol = m["rows"], m["cols"], m["tol"]
    rhs = rhs_for(n, c, m["seed"]).astype(np.float64)
    cfg = HelmholtzConfig(n, c, tol=tol)
    if form == "timing":
        f = torch.from_numpy(rhs).cuda()
        out, rep = sk.loop_stencil_reduce_d(
            1, helmholtz_kernel(cfg), sk.sq_change(), sk.sum_combinator(0.0),
            sk.Condition.rms_below(tol, n * c), sk.Grid.from_tensor(torch.zeros_like(f)),
            env=sk.Grid.from_tensor(f), executor=sk.DeviceExecutor(P, timing=True))
    else:
        out, rep = helmholtz_solve(cfg, sk.Grid.from_array(rhs), partitions=P,
                                   mode="1:n" if P > 1 else "1:1")
    assert rep.iterations == m["iterations"] and rep.exhausted == m["exhausted"]
    assert rep.final_reduce == pytest.approx(m["final_reduce"], rel=1e-12)
    a = out.to_array()
    assert a.dtype == np.float64
    assert sha(a) == m["sha"]


@pytest.mark.parametrize("form", ["default", "timing"])
def test_c4_32768_unit_rhs(prod, form, monkeypatch):
    """BASELINE C4 exactly (32768^2 fp32, rhs = 1, MAX |delta| < 1e-4), in
    the graph form (the default production loop) and the bench's timing
    form: 36 iterations, final max|delta| bit-equal, output grid SHA-256
    equal to the pinned oracle's."""
    m = prod["prod_C4_f32_max_unit_32768"]
    _env_for(form, monkeypatch)
    out, rep, _ = _f32_run(m, form)
    assert rep.iterations == m["iterations"] == 36
    assert rep.final_reduce == m["final_reduce"]
    t = out.tensor()
    assert t.is_cuda
    assert sha(t.cpu().numpy()) == m["sha"]
