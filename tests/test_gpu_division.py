"""The engine's 3-op division by a run constant equals IEEE division.

fp32: exhaustive over every numerator in the fast path's range, for a set
of divisors (the engine also re-runs this check for each new divisor before
using the fast path).  fp64 is covered by the bit-exact Helmholtz fp64 grids.
"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("b", [5.0, 40.5, 3.0, 7.0, 0.1, 1.2345, 6.0001, 1e-5, 12345.678,
                               float(np.float32(2.0) ** 20 - 1)])
def test_div_const_exhaustive_fp32(b):
    from paper_1609_04567_b200 import _native

    lib = _native.require_cuda()
    bad = lib.sk_verify_div_f32(C.c_float(b), None)
    assert bad == 0, f"b={b}: {bad} mismatches"
