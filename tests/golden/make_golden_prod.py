"""Golden fixtures for the PRODUCTION geometry of the Helmholtz sweep.

Run in the build container only (the reference is not present on the GPU box):

    python tests/golden/make_golden_prod.py            # reference-run cases (~3 min)
    python tests/golden/make_golden_prod.py --c4       # + 32768^2 via the pinned oracle (~5 min, 30 GB)

Why: the C1-sized fixtures in golden_large.json all fit one 512-column
block (or take the register-resident whole-loop kernel), so they never
reach the code that BASELINE C4 runs -- the non-resident
`helmholtz_sweep<T>` with many column blocks, >= 64-row work chunks and a
ragged last column block.  These cases do:

* 4099 x 4133 random rhs (16.9 M cells > 2^24: the graph / batched loop
  forms, 9 column blocks, a ragged last block, an odd pitch), fp32 MAX
  |delta| and fp64 `helmholtz_solve` (RMS), P = 1 and 3 -- run by the REAL
  reference (`stencilkit` from /root/reference/pkg/src) and cross-checked
  against the numpy oracle (oracle/stencil_oracle.py) bit for bit;
* 2500 x 3000 (7.5 M cells: the persistent non-resident form) fp32, P = 2;
* 32768^2 unit rhs fp32 MAX |delta| < 1e-4 (BASELINE C4 exactly, P = 1):
  the reference cannot hold it in Python lists, so the pinned oracle
  (`helmholtz_loop_max_banded`, bit-identical to the reference at every
  size it was compared at, tests/test_oracle_golden.py) produces it.

Writes tests/golden/golden_prod.json (SHA-256 of the output grid bytes,
iteration count, final reduce).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "golden_prod.json")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rhs_for(n, m, seed):
    return np.random.default_rng(seed).random((n, m)).astype(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c4", action="store_true", help="also the 32768^2 oracle case")
    ap.add_argument("--only-c4", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, ROOT)
    from oracle import stencil_oracle as O

    meta = json.load(open(OUT)) if os.path.exists(OUT) else {}

    if not args.only_c4:
        sys.path.insert(0, REF)
        from stencilkit import Condition, Delta, Grid, max_combinator, parallel_loop
        from stencilkit.apps import HelmholtzConfig, helmholtz_solve
        from stencilkit.apps.helmholtz import helmholtz_kernel

        def mode(P):
            return "1:n" if P > 1 else "1:1"

        def f32_case(name, n, m, seed, P, tol=1e-4):
            rhs = rhs_for(n, m, seed)
            cfg = HelmholtzConfig(rows=n, cols=m, tol=tol)
            u0 = Grid((n, m), list(np.zeros((n, m), np.float32).ravel()))
            f = Grid((n, m), list(rhs.ravel()))
            delta = Delta(lambda a, b: abs(a - b), on_arrays=lambda a, b: np.abs(a - b))
            cond = Condition(lambda v, it, s: v < tol, max_iterations=10_000)
            t0 = time.perf_counter()
            out, rep = parallel_loop(mode(P), P, 1, helmholtz_kernel(cfg), max_combinator(0.0),
                                     cond, u0, env=f, delta=delta)
            dt = time.perf_counter() - t0
            a = out.to_array().astype(np.float32)
            # the pinned oracle must agree bit for bit (grid, count, value)
            u, it, v, ex = O.helmholtz_loop(np.zeros((n, m), np.float32), rhs,
                                            O.helmholtz_consts(), delta="abs", op="max",
                                            cond=lambda val, i: val < tol, P=P)
            assert it == rep.iterations and v == rep.final_reduce and ex == rep.exhausted
            assert np.array_equal(u.view(np.uint32), a.view(np.uint32)), name
            meta[name] = dict(kind="helmholtz", dtype="f32", rows=n, cols=m, seed=seed, P=P,
                              tol=tol, reduce="max", iterations=rep.iterations,
                              final_reduce=rep.final_reduce, exhausted=rep.exhausted,
                              sha=sha(a), source="reference", wall_s=dt)
            print(name, rep.iterations, rep.final_reduce, f"{dt:.1f}s", flush=True)

        def f64_case(name, n, m, seed, P, tol=1e-4):
            rhs = rhs_for(n, m, seed).astype(np.float64)
            cfg = HelmholtzConfig(rows=n, cols=m, tol=tol)
            t0 = time.perf_counter()
            out, rep = helmholtz_solve(cfg, Grid.from_array(rhs), partitions=P, mode=mode(P))
            dt = time.perf_counter() - t0
            a = out.to_array()
            assert a.dtype == np.float64
            nm = n * m
            u, it, v, ex = O.helmholtz_loop(np.zeros((n, m)), rhs, O.helmholtz_consts(),
                                            delta="sq", op="sum",
                                            cond=lambda val, i: math.sqrt(val / nm) < tol, P=P)
            assert it == rep.iterations and ex == rep.exhausted
            assert v == rep.final_reduce, (v, rep.final_reduce)
            assert np.array_equal(u.view(np.uint64), a.view(np.uint64)), name
            meta[name] = dict(kind="helmholtz_solve", dtype="f64", rows=n, cols=m, seed=seed,
                              P=P, tol=tol, reduce="sum", iterations=rep.iterations,
                              final_reduce=rep.final_reduce, exhausted=rep.exhausted,
                              sha=sha(a), source="reference", wall_s=dt)
            print(name, rep.iterations, rep.final_reduce, f"{dt:.1f}s", flush=True)

        for P in (1, 3):
            f32_case(f"prod_f32_max_rand7_4099x4133_P{P}", 4099, 4133, 7, P)
        f32_case("prod_f32_max_rand8_2500x3000_P2", 2500, 3000, 8, 2)
        for P in (1, 3):
            f64_case(f"prod_f64_solve_rand7_4099x4133_P{P}", 4099, 4133, 7, P)

    if args.c4 or args.only_c4:
        n = 32768
        t0 = time.perf_counter()
        u, it, v, ex = O.helmholtz_loop_max_banded(np.zeros((n, n), np.float32),
                                                   np.ones((n, n), np.float32),
                                                   O.helmholtz_consts(), tol=1e-4,
                                                   threads=os.cpu_count() or 8)
        dt = time.perf_counter() - t0
        meta["prod_C4_f32_max_unit_32768"] = dict(
            kind="helmholtz", dtype="f32", rows=n, cols=n, seed=None, rhs="ones", P=1, tol=1e-4,
            reduce="max", iterations=it, final_reduce=v, exhausted=ex, sha=sha(u),
            source="oracle (helmholtz_loop_max_banded)", wall_s=dt)
        print("C4", it, v, f"{dt:.1f}s", flush=True)

    with open(OUT, "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
