"""Golden fixtures for the run-time compiled elemental path (tests/jit_cases.py),
produced by the REAL reference package's own loop (build container only):

    python tests/golden/make_golden_jit.py

Each case runs through stencilkit.parallel_loop("1:1", 1, ...) with the
case's plain Python point function, combinator and delta; the reference has
no block form for them, so it takes its point route (partition.py:319-366).
Grids are built from Python scalars (`.tolist()`), float32 cases from numpy
float32 scalars, exactly as a reference user would.  Writes
tests/golden/golden_jit.npz (outputs) and golden_jit.json (iterations,
final_reduce, exhausted; for ERROR_CASES the failing index and exception).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def as_ref_grid(Grid, a):
    a = np.asarray(a)
    data = list(a.ravel()) if a.dtype == np.float32 else a.ravel().tolist()
    return Grid(a.shape, data)


def main():
    sys.path.insert(0, REF)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import stencilkit as ref
    import jit_cases as J

    J.ABSENT = ref.ABSENT  # the functions test against the reference's marker
    arrays, meta = {}, {}
    for name, spec in {**J.CASES, **J.ERROR_CASES, **J.CASES_1D}.items():
        g = spec["grid"]()
        env = spec["env"]() if spec["env"] is not None else None
        if isinstance(env, tuple):
            renv = tuple(as_ref_grid(ref.Grid, e) for e in env)
        elif env is not None:
            renv = as_ref_grid(ref.Grid, env)
        else:
            renv = None
        kind, fn = spec["op"]
        op = ref.sum_combinator(spec["identity"]) if kind == "sum" else (
            ref.max_combinator(spec["identity"]) if kind == "max" else ref.Combinator(fn, spec["identity"]))
        delta = ref.Delta(spec["delta"]) if spec["delta"] is not None else None
        cond = ref.Condition(J.cond_fn(spec), max_iterations=spec.get("max_it", 10_000))
        f = ref.ElementalFn(point=spec["point"], k=spec["k"])
        try:
            out, rep = ref.parallel_loop("1:1", 1, spec["k"], f, op, cond, as_ref_grid(ref.Grid, g),
                                         env=renv, delta=delta, indexed=spec.get("indexed", False))
        except ref.StencilError as e:
            meta[name] = {"error": type(e.__cause__).__name__, "index": list(e.index)}
            print(name, "StencilError", e.index, type(e.__cause__).__name__)
            continue
        arr = np.asarray(out.data).reshape(out.dims)
        arrays[name] = arr
        fr = rep.final_reduce
        meta[name] = {"iterations": rep.iterations, "final_reduce": float(fr),
                      "final_is_int": isinstance(fr, (int, np.integer)) and not isinstance(fr, bool),
                      "exhausted": rep.exhausted, "dtype": str(arr.dtype)}
        print(name, rep.iterations, fr, arr.dtype)
    np.savez_compressed(os.path.join(HERE, "golden_jit.npz"), **arrays)
    with open(os.path.join(HERE, "golden_jit.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
