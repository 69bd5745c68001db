"""Plain Python loop conditions recognised as device-evaluable threshold
forms (loop.device_form), and same-line lambdas told apart by their source
columns (the translator must never compile the wrong one)."""

import math

import numpy as np
import pytest

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200 import jit
from paper_1609_04567_b200.loop import DeviceCond, LoopPlan, device_form

TOL, N = 1e-4, 100


class _Cfg:
    tol = 2e-3


CFG = _Cfg()


@pytest.mark.parametrize("fn,want", [
    (lambda v, it, s: v < 1e-4, DeviceCond("lt", 1e-4)),
    (lambda v, it, s: v < TOL, DeviceCond("lt", TOL)),
    (lambda v, it, s: v <= TOL, DeviceCond("lt", math.nextafter(TOL, math.inf))),
    (lambda v, it, s: TOL > v, DeviceCond("lt", TOL)),
    (lambda v, it, s: it >= 5, DeviceCond("iter_ge", 0.0, 5.0)),
    (lambda v, it, s: it > 5, DeviceCond("iter_ge", 0.0, 6.0)),
    (lambda v, it, s: it == 7, DeviceCond("iter_ge", 0.0, 7.0)),
    (lambda v, it, s: v / N < TOL, DeviceCond("mean_lt", TOL, 100.0)),
    (lambda v, it, s: math.sqrt(v / N) < CFG.tol, DeviceCond("rms_lt", 2e-3, 100.0)),
])
def test_recognised(fn, want):
    assert device_form(fn) == want


@pytest.mark.parametrize("fn", [
    lambda v, it, s: v < TOL or it > 3,        # compound
    lambda v, it, s: print(v) or False,        # side effect
    lambda v, it, s: v / 0 < 1.0,              # Python would raise
    lambda v, it, s: s is not None and v < 1,  # uses the state
])
def test_not_recognised(fn):
    assert device_form(fn) is None


def test_same_line_lambdas_are_told_apart():
    a, b = 3.0, 5.0
    fs = [lambda nb, env: nb.center * a, lambda nb, env: nb.center * b]  # one line, closures
    g = sk.Grid((4, 4), np.zeros((4, 4)))
    srcs = [jit.build_program(LoopPlan(fn=sk.ElementalFn(f, 0), k=0, op=sk.sum_combinator(0.0)),
                              g).source for f in fs]
    assert float(3.0).hex() in srcs[0] and float(5.0).hex() not in srcs[0]
    assert float(5.0).hex() in srcs[1] and float(3.0).hex() not in srcs[1]
    conds = [lambda v, it, s: it >= 2, lambda v, it, s: v < a]  # noqa: E731
    assert device_form(conds[0]) == DeviceCond("iter_ge", 0.0, 2.0)
    assert device_form(conds[1]) == DeviceCond("lt", 3.0)
