"""User elemental functions for the run-time compiled (JIT) path.

Plain Python point functions of the kind a `stencilkit` user writes against
the reference's Neighborhood API (grid.py:201-324) -- no package imports
besides the ABSENT marker, which `tests/golden/make_golden_jit.py` rebinds to
the reference's own marker when it runs these through the real reference to
produce the golden fixtures (tests/golden/golden_jit.*).

Each case: point function, radius, combinator (fn, identity), delta, loop
condition, input / env generators (seeded), indexed flag.
"""

from __future__ import annotations

import math

import numpy as np

from paper_1609_04567_b200.grid import ABSENT  # rebound by make_golden_jit.py

_RING = ((-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1))
_GX = (((-1, -1), -1), ((-1, 1), 1), ((0, -1), -2), ((0, 1), 2), ((1, -1), -1), ((1, 1), 1))
_GY = (((-1, -1), -1), ((-1, 0), -2), ((-1, 1), -1), ((1, -1), 1), ((1, 0), 2), ((1, 1), 1))
_AX, _AY, _B, _RELAX = 4.0, 16.0, 60.5, 0.8


def jacobi(nb, env):
    """Relaxed 5-point Helmholtz update, Dirichlet-0 (apps/helmholtz.py:72-83 form)."""
    c = nb.center
    left = nb.at(0, -1)
    right = nb.at(0, 1)
    up = nb.at(-1, 0)
    down = nb.at(1, 0)
    left = 0.0 if left is ABSENT else left
    right = 0.0 if right is ABSENT else right
    up = 0.0 if up is ABSENT else up
    down = 0.0 if down is ABSENT else down
    f = env.at(*nb.center_index)
    return (1.0 - _RELAX) * c + _RELAX * (f + _AX * (left + right) + _AY * (up + down)) / _B


def life(nb, env):
    """B3/S23 (apps/life.py:24-32 form)."""
    alive = 0
    for di, dj in _RING:
        v = nb.at(di, dj)
        if v is not ABSENT and v:
            alive += 1
    if alive == 3:
        return 1
    return 1 if (nb.center and alive == 2) else 0


def sobel(nb, env):
    """Sobel magnitude, off-grid slots read as the centre (apps/sobel.py:33-44 form)."""
    c = nb.center
    gx = 0
    for (di, dj), w in _GX:
        v = nb.at(di, dj)
        gx += w * (c if v is ABSENT else v)
    gy = 0
    for (di, dj), w in _GY:
        v = nb.at(di, dj)
        gy += w * (c if v is ABSENT else v)
    mag = round(math.sqrt(gx * gx + gy * gy))
    return 0 if mag < 0 else (255 if mag > 255 else mag)


def box_mean(nb, env):
    """Mean over the in-grid part of a radius-2 window."""
    vals = nb.values()
    return sum(vals) / len(vals)


def median3(nb, env):
    """Median of the in-grid 3x3 values by counting (integer, while loop)."""
    best = nb.center
    n = len(nb.values())
    for v in nb.values():
        lower = 0
        higher = 0
        for w in nb.values():
            if w < v:
                lower += 1
            elif w > v:
                higher += 1
        if lower <= n // 2 and higher <= n // 2:
            best = v
            break
    return best


def int_mix(nb, env):
    """Python integer semantics: floor division / modulo of negatives, powers."""
    c = nb.center
    s = 0
    for di in range(-1, 2):
        v = nb.at(di, 0)
        if v is ABSENT:
            continue
        s += (v - 7) // 3 + (v - 5) % 4 - (v % 11) ** 2 // 5
    k = 0
    while s > 40:
        s -= 13
        k += 1
    return s + k + (c % 2)


def f32_relax(nb, env):
    """float32 grid: numpy scalar arithmetic (NEP 50) with Python constants."""
    c = nb.center
    s = c
    n = 1
    for di, dj in ((0, 1), (0, -1), (1, 0), (-1, 0)):
        v = nb.at(di, dj)
        if v is not ABSENT:
            s = s + v
            n += 1
    return 0.5 * c + 0.5 * (s / n) - 0.125 * c


def indexed_weighted(nb, env):
    """Indexed window: neighbour values weighted by an env grid at their index."""
    z, (i, j) = nb.center
    acc = 0.0
    wsum = 0.0
    for p in nb.pairs():
        v, (ni, nj) = p
        w = 1.0 + env.at(ni, nj)
        acc += w * v
        wsum += w
    return 0.5 * z + 0.5 * acc / wsum


def tuple_env(nb, env):
    """Two env grids: a source term and a mask."""
    a, m = env
    c = nb.center
    up = nb.at(-1, 0)
    up = c if up is ABSENT else up
    i, j = nb.center_index
    if m.at(i, j):
        return c
    return 0.75 * c + 0.25 * up + 0.1 * a.at(i, j)


def absent_bug(nb, env):
    """Uses a right neighbour without checking for ABSENT: TypeError at the
    last column (the reference raises StencilError there)."""
    return nb.center + nb.at(0, 1)


def div_bug(nb, env):
    """ZeroDivisionError where the centre is 0."""
    return 10.0 / nb.center


def _lt(tol):
    return lambda v, it, s: v < tol


def _after(n):
    return lambda v, it, s: it >= n


def _min(a, b):
    return a if a < b else b


def _rng_f64(seed, shape, lo=0.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, shape)


# name -> spec
CASES = {
    "jacobi_f64": dict(point=jacobi, k=1, op=("max", None), identity=0.0,
                       delta=lambda new, old: abs(new - old), cond=("below", 1e-9), max_it=300,
                       grid=lambda: np.zeros((37, 141)), env=lambda: _rng_f64(1, (37, 141))),
    "life_glider": dict(point=life, k=1, op=("sum", None), identity=0, delta=None,
                        cond=("after", 9), grid=lambda: (np.random.default_rng(2).random((45, 133)) < 0.3).astype(np.int64),
                        env=None),
    "sobel_int": dict(point=sobel, k=1, op=("sum", None), identity=0, delta=None, cond=("after", 1),
                      grid=lambda: np.random.default_rng(3).integers(0, 256, (33, 150)).astype(np.int64),
                      env=None),
    "box_mean_r2": dict(point=box_mean, k=2, op=("sum", None), identity=0.0,
                        delta=lambda new, old: (new - old) ** 2, cond=("after", 4),
                        grid=lambda: _rng_f64(4, (29, 131), -5, 5), env=None),
    "median3_int": dict(point=median3, k=1, op=("max", None), identity=0,
                        delta=lambda new, old: abs(new - old), cond=("after", 3),
                        grid=lambda: np.random.default_rng(5).integers(0, 100, (21, 130)).astype(np.int64),
                        env=None),
    "int_mix": dict(point=int_mix, k=1, op=("custom", _min), identity=10 ** 9,
                    delta=lambda new, old: new - old, cond=("after", 5),
                    grid=lambda: np.random.default_rng(6).integers(-60, 60, (19, 135)).astype(np.int64),
                    env=None),
    "f32_relax": dict(point=f32_relax, k=1, op=("max", None), identity=0.0,
                      delta=lambda new, old: abs(new - old), cond=("below", 1e-5), max_it=300,
                      grid=lambda: _rng_f64(7, (40, 129)).astype(np.float32), env=None),
    "indexed_weighted": dict(point=indexed_weighted, k=1, op=("sum", None), identity=0.0,
                             delta=lambda new, old: abs(new - old), cond=("after", 6),
                             grid=lambda: _rng_f64(8, (26, 140)), env=lambda: _rng_f64(9, (26, 140)),
                             indexed=True),
    "tuple_env": dict(point=tuple_env, k=1, op=("sum", None), identity=0.0,
                      delta=lambda new, old: abs(new - old), cond=("after", 5),
                      grid=lambda: _rng_f64(10, (31, 130)),
                      env=lambda: (_rng_f64(11, (31, 130)),
                                   (np.random.default_rng(12).random((31, 130)) < 0.2).astype(np.int64))),
}

# cases whose reference run raises StencilError (index recorded in the golden)
ERROR_CASES = {
    "absent_bug": dict(point=absent_bug, k=1, op=("sum", None), identity=0.0, delta=None,
                       cond=("after", 1), grid=lambda: _rng_f64(13, (9, 17)), env=None),
    "div_bug": dict(point=div_bug, k=0, op=("sum", None), identity=0.0, delta=None,
                    cond=("after", 1),
                    grid=lambda: np.where(np.arange(9 * 17).reshape(9, 17) == 77, 0.0, 1.5),
                    env=None),
}


def cond_fn(spec):
    kind, x = spec["cond"]
    return _lt(x) if kind == "below" else _after(x)


def _clip(x, lo, hi):
    if x < lo:
        return lo
    return hi if x > hi else x


def _weight(v, c):
    d = v - c
    return 1.0 / (1.0 + d * d)


def bilateral(nb, env):
    """Helper functions (plain Python, called per window slot)."""
    c = nb.center
    acc = 0.0
    ws = 0.0
    for v in nb.values():
        w = _weight(v, c)
        acc += w * v
        ws += w
    return _clip(acc / ws, -1.0, 1.0)


CASES["bilateral_helpers"] = dict(point=bilateral, k=1, op=("sum", None), identity=0.0,
                                  delta=lambda new, old: abs(new - old), cond=("after", 4),
                                  grid=lambda: _rng_f64(14, (23, 135), -2, 2), env=None)


def smooth1d(nb, env):
    """Rank-1 grid: 3-point relaxation with one offset per slot."""
    c = nb.center
    l = nb.at(-1)
    r = nb.at(1)
    l = c if l is ABSENT else l
    r = c if r is ABSENT else r
    (i,) = nb.center_index
    return 0.5 * c + 0.25 * (l + r) + 0.01 * env.at(i)


CASES_1D = {
    "smooth1d": dict(point=smooth1d, k=1, op=("max", None), identity=0.0,
                     delta=lambda new, old: abs(new - old), cond=("after", 7),
                     grid=lambda: _rng_f64(15, (517,)), env=lambda: _rng_f64(16, (517,))),
}


def median_filter(nb, env):
    """Median of the in-grid window values (radius 2), by sorting them."""
    vals = sorted(nb.values())
    n = len(vals)
    if n % 2:
        return vals[n // 2]
    return (vals[n // 2 - 1] + vals[n // 2]) / 2


def trimmed_mean(nb, env):
    """Mean of the window without its extremes (negative indices, sum of a list)."""
    vals = sorted(nb.values())
    inner = 0.0
    for v in vals:
        inner += v
    return (inner - vals[0] - vals[-1]) / (len(vals) - 2)


CASES["median_filter"] = dict(point=median_filter, k=2, op=("sum", None), identity=0,
                              delta=None, cond=("after", 2),
                              grid=lambda: np.random.default_rng(17).integers(0, 50, (27, 133)).astype(np.int64),
                              env=None)
CASES["trimmed_mean"] = dict(point=trimmed_mean, k=1, op=("max", None), identity=0.0,
                             delta=lambda new, old: abs(new - old), cond=("after", 3),
                             grid=lambda: _rng_f64(18, (25, 131), -3, 3), env=None)
