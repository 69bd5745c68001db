"""Seeded differential sweep: random shapes (including 1-row, 1-column and
odd widths), partitions, dtypes, reduces, deltas and loop forms through the
public API, each against the oracle's restatement of the reference
(oracle/stencil_oracle.py, pinned to real reference runs by
test_oracle_golden.py).  Bit-exact grids, masks and iteration counts;
MAX reduces bit-exact, fp64 SUM reduces within 1e-12.  Regression net for
geometry-dependent kernel paths (resident loop, column blocks, chunk
tails, warp-edge lanes, TMA boxes)."""

import numpy as np
import pytest

import paper_1609_04567_b200 as sk

pytestmark = pytest.mark.gpu


def _shape(rng, rmax, cmax):
    r = int(np.exp(rng.uniform(0, np.log(rmax))))
    c = int(np.exp(rng.uniform(0, np.log(cmax))))
    return max(r, 1), max(c, 1)


@pytest.mark.parametrize("seed", range(10))
def test_helmholtz_random_geometries(seed):
    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

    rng = np.random.default_rng(1000 + seed)
    for case in range(12):
        n, m = _shape(rng, 700, 1500)
        dt = np.float32 if rng.random() < 0.6 else np.float64
        op = "max" if dt == np.float32 or rng.random() < 0.5 else "sum"
        delta = "abs" if rng.random() < 0.6 else "sq"
        P = int(rng.integers(1, min(n, 5) + 1))
        relax = float(rng.choice([0.6, 0.9, 1.0]))
        u0 = rng.random((n, m)).astype(dt)
        f = rng.random((n, m)).astype(dt)
        tol = float(rng.choice([1e-2, 1e-3])) if op == "max" else 1e-3 * n * m
        cfg = HelmholtzConfig(rows=n, cols=m, alpha=0.5, dx=0.5, dy=0.25, relax=relax)
        want, it, v, ex = O.helmholtz_loop(u0, f, O.helmholtz_consts(0.5, 0.5, 0.25, relax),
                                           delta=delta, op=op, cond=lambda val, i: val < tol,
                                           P=P, max_iterations=40)
        comb = sk.max_combinator(0.0) if op == "max" else sk.sum_combinator(0.0)
        dl = sk.abs_change() if delta == "abs" else sk.sq_change()
        ex_dev = None if rng.random() < 0.6 else sk.DeviceExecutor(P, timing=True)
        out, rep = sk.loop_stencil_reduce_d(1, helmholtz_kernel(cfg), dl, comb,
                                            sk.Condition.below(tol, max_iterations=40),
                                            sk.Grid(u0.shape, u0), env=sk.Grid(f.shape, f),
                                            executor=ex_dev) if ex_dev is not None else \
            sk.parallel_loop("1:n" if P > 1 else "1:1", P, 1, helmholtz_kernel(cfg), comb,
                             sk.Condition.below(tol, max_iterations=40), sk.Grid(u0.shape, u0),
                             env=sk.Grid(f.shape, f), delta=dl)
        tag = (seed, case, n, m, dt.__name__, op, delta, P, ex_dev is not None)
        assert rep.iterations == it and rep.exhausted == ex, tag
        got = out.to_array()
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), tag
        if op == "max":
            assert rep.final_reduce == v, tag
        else:
            assert rep.final_reduce == pytest.approx(v, rel=1e-12), tag


def test_sobel_every_tiny_shape_and_random_ones():
    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import sobel_filter, sobel_frames

    rng = np.random.default_rng(7)
    shapes = [(r, c) for r in range(1, 6) for c in range(1, 6)]
    shapes += [_shape(rng, 400, 2600) for _ in range(12)]
    for n, m in shapes:
        img = rng.integers(0, 256, (n, m)).astype(np.int64)
        want = O.sobel(img)
        P = int(rng.integers(1, min(n, 4) + 1))
        out, rep = sobel_filter(sk.Grid.from_array(img), partitions=P, with_report=True)
        assert np.array_equal(out.to_array().astype(np.uint8), want), (n, m, P)
        assert rep.final_reduce == int(want.astype(np.int64).sum()), (n, m, P)
    import torch

    for _ in range(8):
        F = int(rng.integers(1, 6))
        n, m = _shape(rng, 300, 2300)
        pitch = -(-m // 16) * 16 + 16 * int(rng.integers(0, 3))
        imgs = rng.integers(0, 256, (F, n, m)).astype(np.uint8)
        buf = torch.zeros((F, n, pitch), dtype=torch.uint8, device="cuda")
        buf[:, :, :m] = torch.from_numpy(imgs).cuda()
        edges, sums = sobel_frames(buf[:, :, :m])
        e = edges.cpu().numpy()
        s = sums.cpu().numpy()
        for k in range(F):
            w = O.sobel(imgs[k])
            assert np.array_equal(e[k], w), (F, n, m, pitch, k)
            assert int(s[k]) == int(w.astype(np.int64).sum())


def test_life_amf_restore_random():
    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import GolConfig, amf_detect, game_of_life, restore_regularize

    rng = np.random.default_rng(11)
    for _ in range(8):
        n, m = _shape(rng, 120, 300)
        board = (rng.random((n, m)) < 0.35).astype(np.int64)
        steps = int(rng.integers(1, 6))
        P = int(rng.integers(1, min(n, 3) + 1))
        out, rep = game_of_life(sk.Grid.from_array(board), config=GolConfig(n, m, steps=steps),
                                partitions=P)
        w = board.astype(np.uint8)
        for _s in range(steps):
            w = O.life_step(w)
        assert np.array_equal(out.to_array().astype(np.uint8), w), (n, m, steps, P)
    for _ in range(6):
        n, m = _shape(rng, 90, 160)
        base = ((np.arange(n)[:, None] * 3 + np.arange(m)[None, :] * 2) % 200 + 20)
        noisy, _ = O.salt_pepper(base, float(rng.choice([0.1, 0.3, 0.6])),
                                 seed=int(rng.integers(1 << 30)))
        img = sk.Grid.from_array(noisy.astype(np.int64))
        mask = amf_detect(img)
        wm = O.amf_detect(noisy)
        assert np.array_equal(mask.to_array().astype(np.uint8), wm), (n, m)
        P = int(rng.integers(1, min(n, 3) + 1))
        out, rep = restore_regularize(img, mask, partitions=P)
        wo, it, v, ex = O.restore_loop(noisy, wm, P=P)
        assert rep.iterations == it and rep.exhausted == ex, (n, m, P)
        assert np.array_equal(out.to_array().view(np.uint64), wo.view(np.uint64)), (n, m, P)
