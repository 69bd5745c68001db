"""The JIT translation cache (jit.build_program): a repeated loop call with
the same functions reuses the translated program, and every global /
nonlocal value the translation read is re-checked, so rebinding a constant
or a helper re-translates and a mutable value is never cached.  No GPU
needed (NVRTC compiles for sm_100a on the host)."""

import numpy as np

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200 import jit
from paper_1609_04567_b200.grid import ABSENT
from paper_1609_04567_b200.loop import LoopPlan

SCALE = 2.0
WEIGHTS = [1.0, 2.0]


def _scaled(nb, env):
    left = nb.at(0, -1)
    left = 0.0 if left is ABSENT else left
    return SCALE * nb.center + left


def _helper(x):
    return x * SCALE


def _uses_helper(nb, env):
    return _helper(nb.center)


def _uses_list(nb, env):
    return nb.center * WEIGHTS[1]


def _plan(point):
    return LoopPlan(fn=sk.ElementalFn(point=point, k=1), k=1, op=sk.max_combinator(0.0), env=None,
                    indexed=False, delta=sk.abs_change())


def _grid():
    return sk.Grid((8, 8), np.zeros((8, 8), np.float64))


def test_repeat_call_hits_the_cache():
    p1 = jit.build_program(_plan(_scaled), _grid())
    p2 = jit.build_program(_plan(_scaled), _grid())
    assert p1 is p2


def test_rebound_global_retranslates():
    global SCALE
    p1 = jit.build_program(_plan(_scaled), _grid())
    old = SCALE
    try:
        SCALE = 3.0
        p2 = jit.build_program(_plan(_scaled), _grid())
        assert p2 is not p1 and p2.source != p1.source
        SCALE = -0.0 if old == 0 else old  # back to an equal value: a hit again
        p3 = jit.build_program(_plan(_scaled), _grid())
        assert p3.source == p1.source
    finally:
        SCALE = old


def test_rebound_value_read_by_a_helper_retranslates():
    global SCALE
    p1 = jit.build_program(_plan(_uses_helper), _grid())
    old = SCALE
    try:
        SCALE = 5.0
        p2 = jit.build_program(_plan(_uses_helper), _grid())
        assert p2.source != p1.source
    finally:
        SCALE = old


def test_closure_values_are_checked():
    def make(c):
        def point(nb, env):
            return nb.center + c
        return point

    a = jit.build_program(_plan(make(1.0)), _grid())
    b = jit.build_program(_plan(make(2.0)), _grid())  # same code, another closure value
    assert a.source != b.source
    c = jit.build_program(_plan(make(1.0)), _grid())
    assert c.source == a.source


def test_mutable_values_are_never_cached():
    p1 = jit.build_program(_plan(_uses_list), _grid())
    WEIGHTS[1] = 7.0
    try:
        p2 = jit.build_program(_plan(_uses_list), _grid())
        assert p2 is not p1 and p2.source != p1.source
    finally:
        WEIGHTS[1] = 2.0


def test_grid_dtype_is_part_of_the_key():
    p1 = jit.build_program(_plan(_scaled), _grid())
    p2 = jit.build_program(_plan(_scaled), sk.Grid.from_tensor(__import__("torch").zeros((8, 8))))
    assert p1.in_dtype != p2.in_dtype
