"""Shared helpers for the JIT (user elemental) tests."""

from __future__ import annotations

import json
import os

import numpy as np

import jit_cases as J
import paper_1609_04567_b200 as sk

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden():
    meta = json.load(open(os.path.join(GOLDEN, "golden_jit.json")))
    arrays = np.load(os.path.join(GOLDEN, "golden_jit.npz"))
    return meta, arrays


def op_of(spec):
    kind, fn = spec["op"]
    if kind == "sum":
        return sk.sum_combinator(spec["identity"])
    if kind == "max":
        return sk.max_combinator(spec["identity"])
    return sk.Combinator(fn, spec["identity"])


def device_cond(spec):
    kind, x = spec["cond"]
    mi = spec.get("max_it", 10_000)
    return sk.Condition.below(x, mi) if kind == "below" else sk.stop_after(x)


def host_cond(spec):
    return sk.Condition(J.cond_fn(spec), spec.get("max_it", 10_000))


def inputs(spec):
    g = spec["grid"]()
    env = spec["env"]() if spec["env"] is not None else None
    return g, env


def as_grid(a):
    return sk.Grid(a.shape, np.asarray(a))


def env_grids(env):
    if env is None:
        return None
    if isinstance(env, tuple):
        return tuple(as_grid(e) for e in env)
    return as_grid(env)


def py_rows(a):
    """Rows of Python scalars as a reference Grid built from `.tolist()`
    holds them (numpy float32 scalars for float32 grids)."""
    a = np.asarray(a)
    if a.dtype == np.float32:
        return [list(r) for r in a]
    return a.tolist()


def run_device(spec, P=1, cond=None, state=None):
    g, env = inputs(spec)
    delta = sk.Delta(spec["delta"]) if spec["delta"] is not None else None
    f = sk.ElementalFn(point=spec["point"], k=spec["k"])
    out, rep = sk.parallel_loop("1:n" if P > 1 else "1:1", P, spec["k"], f, op_of(spec),
                                cond if cond is not None else device_cond(spec), as_grid(g),
                                env=env_grids(env), delta=delta,
                                indexed=spec.get("indexed", False), state=state)
    return out, rep
