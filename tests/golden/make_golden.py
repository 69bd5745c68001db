"""Generate the golden fixtures from the REAL reference package.

Run in the build container only (the reference is not present on the GPU box):

    python tests/golden/make_golden.py            # small + medium cases
    python tests/golden/make_golden.py --large    # adds C1 1024^2, C5 frames, C3-like 512^2

Imports `stencilkit` from /root/reference/pkg/src and records, per case, the
reference's own outputs: iteration counts, final reduce values, full output
arrays for small grids and SHA-256 digests for large ones.  The fixtures are
committed (small) so the GPU-box tests never need the reference.
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


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, REF)
    from stencilkit import Condition, Delta, Grid, max_combinator, parallel_loop, sum_combinator
    from stencilkit.apps import (HelmholtzConfig, amf_detect, game_of_life, GolConfig,
                                 helmholtz_solve, restore_regularize, salt_pepper, sobel_filter)
    from stencilkit.apps.helmholtz import helmholtz_kernel
    from stencilkit.cli import _synthetic_frame

    arrays: dict[str, np.ndarray] = {}
    meta: dict[str, dict] = {}

    def mode(P):
        return "1:n" if P > 1 else "1:1"

    # ---------------- Helmholtz, fp32 block route, MAX |delta| (config C1 form)
    def helm_f32(name, n, m, rhs, tol, P, alpha=1.0, dx=1.0, dy=1.0, relax=1.0,
                 keep_full=True, reduce="max"):
        cfg = HelmholtzConfig(rows=n, cols=m, alpha=alpha, dx=dx, dy=dy, relax=relax, tol=tol)
        u0 = Grid((n, m), list(np.zeros((n, m), np.float32).ravel()))
        f = Grid((n, m), list(rhs.astype(np.float32).ravel()))
        if reduce == "max":
            delta = Delta(lambda a, b: abs(a - b), on_arrays=lambda a, b: np.abs(a - b))
            op = max_combinator(0.0)
            cond = Condition(lambda v, it, s: v < tol, max_iterations=10_000)
        else:
            delta = Delta(lambda a, b: (a - b) ** 2, on_arrays=lambda a, b: (a - b) ** 2)
            op = sum_combinator(0.0)
            nm = n * m
            cond = Condition(lambda v, it, s: math.sqrt(v / nm) < tol, max_iterations=10_000)
        t0 = time.perf_counter()
        out, rep = parallel_loop(mode(P), P, 1, helmholtz_kernel(cfg), op, cond, u0, env=f,
                                 delta=delta)
        dt = time.perf_counter() - t0
        a64 = out.to_array()
        a = a64.astype(np.float32)  # gather() widens to Python floats; values are fp32-exact
        assert np.array_equal(a.astype(np.float64), a64)
        meta[name] = dict(kind="helmholtz", dtype="f32", rows=n, cols=m, alpha=alpha, dx=dx,
                          dy=dy, relax=relax, tol=tol, P=P, reduce=reduce,
                          iterations=rep.iterations, final_reduce=rep.final_reduce,
                          exhausted=rep.exhausted, sha=sha(a), wall_s=dt,
                          ledger=vars(rep.copies))
        if keep_full:
            arrays[name + "/out"] = a
            arrays[name + "/rhs"] = rhs.astype(np.float32)
        print(name, rep.iterations, rep.final_reduce, f"{dt:.2f}s", flush=True)

    one = lambda n, m: np.ones((n, m))
    helm_f32("helm_f32_max_unit_64", 64, 64, one(64, 64), 1e-4, 1)
    helm_f32("helm_f32_max_unit_64_P3", 64, 64, one(64, 64), 1e-4, 3)
    rr = np.random.default_rng(0).random((96, 80))
    helm_f32("helm_f32_max_rand_96x80", 96, 80, rr, 1e-4, 1, alpha=0.5, dx=0.5, dy=0.25, relax=0.8)
    helm_f32("helm_f32_max_rand_96x80_P4", 96, 80, rr, 1e-4, 4, alpha=0.5, dx=0.5, dy=0.25, relax=0.8)
    helm_f32("helm_f32_sum_rand_50x70", 50, 70, np.random.default_rng(5).random((50, 70)), 1e-4, 1,
             reduce="sum")
    helm_f32("helm_f32_max_odd_37x13", 37, 13, np.random.default_rng(6).random((37, 13)), 1e-3, 2,
             relax=0.9)

    # ---------------- Helmholtz fp64 via helmholtz_solve (RMS criterion)
    def helm_f64(name, n, m, rhs, tol, P, alpha=1.0, dx=1.0, dy=1.0, relax=1.0, u0=None,
                 keep_full=True):
        cfg = HelmholtzConfig(rows=n, cols=m, alpha=alpha, dx=dx, dy=dy, relax=relax, tol=tol)
        t0 = time.perf_counter()
        g0 = None if u0 is None else Grid.from_array(u0)
        out, rep = helmholtz_solve(cfg, Grid.from_array(rhs), g0, partitions=P, mode=mode(P))
        dt = time.perf_counter() - t0
        a = out.to_array()
        assert a.dtype == np.float64
        meta[name] = dict(kind="helmholtz_solve", dtype="f64", rows=n, cols=m, alpha=alpha, dx=dx,
                          dy=dy, relax=relax, tol=tol, P=P, iterations=rep.iterations,
                          final_reduce=rep.final_reduce, exhausted=rep.exhausted, sha=sha(a),
                          wall_s=dt, ledger=vars(rep.copies))
        if keep_full:
            arrays[name + "/out"] = a
            arrays[name + "/rhs"] = np.asarray(rhs, np.float64)
            if u0 is not None:
                arrays[name + "/u0"] = np.asarray(u0, np.float64)
        print(name, rep.iterations, rep.final_reduce, f"{dt:.2f}s", flush=True)

    helm_f64("helm_f64_unit_16", 16, 16, one(16, 16), 1e-6, 1)
    r40 = np.random.default_rng(40).random((12, 10))
    helm_f64("helm_f64_rand_12x10", 12, 10, r40, 1e-5, 1, alpha=0.5, dx=0.5, dy=0.25, relax=0.8)
    r64 = np.random.default_rng(1).random((64, 48))
    for P in (1, 2, 3):
        helm_f64(f"helm_f64_rand_64x48_P{P}", 64, 48, r64, 1e-6, P)
    helm_f64("helm_f64_unit_32x48_P3", 32, 48, one(32, 48), 1e-5, 3)
    warm = np.random.default_rng(9).random((20, 24))
    helm_f64("helm_f64_warm_20x24", 20, 24, one(20, 24), 1e-5, 1, u0=warm)

    # ---------------- Sobel
    def sob(name, img, P=1, keep_full=True):
        g = Grid.from_array(img.astype(np.int64))
        t0 = time.perf_counter()
        out, rep = sobel_filter(g, partitions=P, mode=mode(P), with_report=True)
        dt = time.perf_counter() - t0
        a = out.to_array().astype(np.uint8)
        meta[name] = dict(kind="sobel", rows=img.shape[0], cols=img.shape[1], P=P,
                          iterations=rep.iterations, final_reduce=rep.final_reduce, sha=sha(a),
                          wall_s=dt, ledger=vars(rep.copies))
        if keep_full:
            arrays[name + "/in"] = img.astype(np.uint8)
            arrays[name + "/out"] = a
        print(name, rep.final_reduce, f"{dt:.2f}s", flush=True)

    rs = np.random.default_rng(12)
    for shp in ((5, 5), (9, 4), (1, 6), (7, 1), (1, 1), (2, 3)):
        sob(f"sobel_{shp[0]}x{shp[1]}", rs.integers(0, 256, shp))
    sob("sobel_step_4x4", np.array([[0, 0, 255, 255]] * 4))
    sob("sobel_64x48_P3", np.random.default_rng(77).integers(0, 256, (64, 48)), P=3)
    sob("sobel_130x259", np.random.default_rng(78).integers(0, 256, (130, 259)))

    # ---------------- AMF detection
    def grad(n, m, lo=20, span=200):
        r = np.arange(n)[:, None]
        c = np.arange(m)[None, :]
        return ((r * 3 + c * 2) % span + lo).astype(np.int64)

    def amf(name, img, wmax=7, P=1, keep_full=True):
        t0 = time.perf_counter()
        mask = amf_detect(Grid.from_array(img.astype(np.int64)), wmax=wmax, partitions=P,
                          mode=mode(P))
        dt = time.perf_counter() - t0
        a = mask.to_array().astype(np.uint8)
        meta[name] = dict(kind="amf", rows=img.shape[0], cols=img.shape[1], wmax=wmax, P=P,
                          flagged=int(a.sum()), sha=sha(a), wall_s=dt)
        if keep_full:
            arrays[name + "/in"] = img.astype(np.uint8)
            arrays[name + "/out"] = a
        print(name, int(a.sum()), f"{dt:.2f}s", flush=True)

    amf("amf_rand_14x11", np.random.default_rng(30).integers(0, 256, (14, 11)))
    imp = np.zeros((9, 9), np.int64)
    imp[4, 5] = 255
    amf("amf_impulse_9x9", imp)
    amf("amf_rand_12x10_w5", np.random.default_rng(31).integers(0, 256, (12, 10)), wmax=5)
    amf("amf_rand_12x10_w3", np.random.default_rng(31).integers(0, 256, (12, 10)), wmax=3)
    noisy20 = salt_pepper(Grid.from_array(grad(20, 16)), 0.2, seed=9)[0].to_array()
    amf("amf_grad_20x16_P4", noisy20, P=4)
    noisy50 = salt_pepper(Grid.from_array(grad(96, 96)), 0.5, seed=42)[0].to_array()
    amf("amf_grad50_96", noisy50)
    amf("amf_w9_40x33", salt_pepper(Grid.from_array(grad(40, 33)), 0.4, seed=3)[0].to_array(),
        wmax=9)

    # ---------------- restoration
    def rest(name, img, mask, P=1, keep_full=True, cfg=None):
        from stencilkit.apps import RestoreConfig
        cfg = cfg or RestoreConfig()
        t0 = time.perf_counter()
        out, rep = restore_regularize(Grid.from_array(img.astype(np.int64)),
                                      Grid.from_array(mask.astype(np.int64)), cfg,
                                      partitions=P, mode=mode(P))
        dt = time.perf_counter() - t0
        a = out.to_array().astype(np.float64)
        u8 = np.clip(np.rint(a), 0, 255).astype(np.uint8)
        meta[name] = dict(kind="restore", rows=img.shape[0], cols=img.shape[1], P=P,
                          iterations=rep.iterations, final_reduce=rep.final_reduce,
                          exhausted=rep.exhausted, flagged=int(mask.sum()), sha=sha(a),
                          sha_u8=sha(u8), wall_s=dt, max_iterations=cfg.max_iterations,
                          ledger=vars(rep.copies))
        if keep_full:
            arrays[name + "/in"] = img.astype(np.uint8)
            arrays[name + "/mask"] = mask.astype(np.uint8)
            arrays[name + "/out"] = a
        print(name, rep.iterations, rep.final_reduce, rep.exhausted, f"{dt:.2f}s", flush=True)

    for (n, m, lvl, seed, P) in ((24, 24, 0.3, 42, 1), (18, 14, 0.25, 11, 3), (48, 40, 0.5, 42, 1),
                                 (48, 40, 0.5, 42, 2), (64, 64, 0.5, 42, 1)):
        noisy = salt_pepper(Grid.from_array(grad(n, m)), lvl, seed=seed)[0]
        mask = amf_detect(noisy).to_array()
        rest(f"restore_grad{int(lvl*100)}_{n}x{m}_P{P}", noisy.to_array(), mask, P=P)
    rows = np.array([[12, 240, 33], [91, 255, 18], [77, 160, 204]])
    nz = np.array([[0, 1, 0], [0, 1, 0], [1, 0, 0]])
    from stencilkit.apps import RestoreConfig
    rest("restore_3x3_one_sweep", rows, nz, cfg=RestoreConfig(max_iterations=1))
    # full two-phase on the 256^2 standard image (acceptance criterion 6 input)
    noisy = salt_pepper(Grid.from_array(grad(256, 256)), 0.3, seed=42)[0]
    mask = amf_detect(noisy).to_array()
    rest("restore_grad30_256", noisy.to_array(), mask, keep_full=False)

    # ---------------- Game of Life
    def life(name, board, steps, P=1):
        out, rep = game_of_life(Grid.from_array(board), config=GolConfig(*board.shape, steps=steps),
                                partitions=P, mode=mode(P))
        a = out.to_array().astype(np.uint8)
        meta[name] = dict(kind="life", rows=board.shape[0], cols=board.shape[1], steps=steps,
                          P=P, final_reduce=rep.final_reduce, sha=sha(a))
        arrays[name + "/in"] = board.astype(np.uint8)
        arrays[name + "/out"] = a

    soup = (np.random.default_rng(1).random((64, 64)) < 0.3).astype(np.int64)
    life("life_soup_64_100", soup, 100)
    life("life_soup_64_100_P4", soup, 100, P=4)

    if args.large:
        # C1 exactly: 1024^2 fp32, rhs=1, MAX|delta| < 1e-4
        helm_f32("C1_helm_f32_max_unit_1024", 1024, 1024, one(1024, 1024), 1e-4, 8, keep_full=False)
        helm_f32("C1_helm_f32_max_rand0_1024", 1024, 1024,
                 np.random.default_rng(0).random((1024, 1024)), 1e-4, 8, keep_full=False)
        helm_f64("C1_helm_f64_solve_unit_1024", 1024, 1024, one(1024, 1024), 1e-4, 8,
                 keep_full=False)
        # Sobel 2048^2 random (config C2 frame form)
        sob("C2_sobel_rng0_2048", np.random.default_rng(0).integers(0, 256, (2048, 2048)), P=8,
            keep_full=False)
        for i in range(2):
            sob(f"C2_sobel_rng{42 + i}_2048",
                np.random.default_rng(42 + i).integers(0, 256, (2048, 2048)), P=8, keep_full=False)
        # C3-like at 512^2 (50% noise, expect the 100-iteration cap)
        noisy = salt_pepper(Grid.from_array(grad(512, 512)), 0.5, seed=42)[0]
        a = noisy.to_array()
        amf("C3_amf_grad50_512", a, P=8, keep_full=False)
        mask = amf_detect(noisy, partitions=8).to_array()
        rest("C3_restore_grad50_512_P8", a, mask, P=8, keep_full=False)
        # C5 frames 0..3: 1080x1920, 10% noise, seed 42+i
        for i in range(4):
            noisy = salt_pepper(_synthetic_frame(1080, 1920, i), 0.1, seed=42 + i)[0]
            a = noisy.to_array()
            amf(f"C5_amf_frame{i}", a, P=8, keep_full=False)
            mask = amf_detect(noisy, partitions=8).to_array()
            rest(f"C5_restore_frame{i}_P8", a, mask, P=8, keep_full=False)

    tag = "large" if args.large else "small"
    np.savez_compressed(os.path.join(HERE, f"golden_{tag}.npz"), **arrays)
    with open(os.path.join(HERE, f"golden_{tag}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(meta), "cases")


if __name__ == "__main__":
    main()
