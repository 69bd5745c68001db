"""The reference's host building blocks on device buffers: partition,
halo_exchange, parallel_step, PartitionSet.gather (partition.py:60-262,
415-432) -- split arithmetic, halo contents, ledger counts, and steps that
reproduce the whole-grid stencil (the reference's test_partition.py cases)."""

import numpy as np
import pytest

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200 import ABSENT, Grid, GridError

pytestmark = pytest.mark.gpu


def life_point(nb, env):
    alive = 0
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            if di == 0 and dj == 0:
                continue
            v = nb.at(di, dj)
            if v is not ABSENT and v:
                alive += 1
    return 1 if alive == 3 or (nb.center and alive == 2) else 0


def grid_8x4():
    return Grid.from_rows([[r * 4 + c for c in range(4)] for r in range(8)])


def test_split_and_seeded_halos():
    ps = sk.partition(grid_8x4(), 2, 1)
    p0, p1 = ps.parts
    assert (p0.r_begin, p0.r_end, p1.r_begin, p1.r_end) == (0, 4, 4, 8)
    assert (p0.top_halo, p0.bottom_halo, p1.top_halo, p1.bottom_halo) == (0, 1, 1, 0)
    assert p0.front[p0.top_halo + p0.rows] == [16, 17, 18, 19]
    assert p1.front[0] == [12, 13, 14, 15]
    assert [p.rows for p in sk.partition(Grid.filled((10, 3), 0), 4, 1).parts] == [3, 3, 2, 2]
    assert ps.ledger.full_fill_elems == 32 and ps.ledger.fill_events == 2
    assert ps.buffer_allocations == 4


def test_preconditions():
    with pytest.raises(GridError):
        sk.partition(Grid.filled((3, 3), 0), 4, 1)
    with pytest.raises(GridError):
        sk.partition(Grid.filled((8, 3), 0), 4, 3)
    sk.partition(Grid.filled((2, 3), 0), 1, 3)


def test_1d_split():
    ps = sk.partition(Grid((10,), list(range(10))), 3, 1)
    assert [(p.r_begin, p.r_end) for p in ps.parts] == [(0, 4), (4, 7), (7, 10)]
    assert ps.parts[1].front == [3, 4, 5, 6, 7]


def test_gather_and_readback_count():
    g = grid_8x4()
    ps = sk.partition(g, 3, 1)
    for p in ps.parts:
        p.back = [list(r) for r in p.front]
    out = ps.gather("back")
    assert out == g
    assert ps.ledger.readback_elems == 32 and ps.ledger.readback_events == 3


def test_halo_exchange_moves_rows_and_counts():
    ps = sk.partition(grid_8x4(), 2, 1)
    ps.parts[0].front[ps.parts[0].top_halo + 3] = [90, 91, 92, 93]
    sk.halo_exchange(ps)
    assert ps.parts[1].front[0] == [90, 91, 92, 93]
    assert ps.parts[0].front[4] == [16, 17, 18, 19]
    assert ps.ledger.halo_elems == 8 and ps.ledger.halo_events == 2
    one = sk.partition(grid_8x4(), 1, 1)
    sk.halo_exchange(one)
    assert one.ledger.halo_elems == 0


def test_steps_match_the_whole_grid_stencil():
    rng = np.random.default_rng(21)
    g = Grid.from_array(rng.integers(0, 2, (9, 5)))
    expected = sk.stencil_apply(life_point, 1, g)
    for P in (1, 2, 3, 4):
        ps = sk.partition(g, P, 1)
        sk.halo_exchange(ps)
        sk.parallel_step(ps, life_point, 1, sk.sum_combinator(0))
        ps.swap_all()
        assert ps.gather("front") == expected, P


def test_partials_combine_to_the_whole_grid_value():
    rng = np.random.default_rng(33)
    g = Grid.from_array(rng.integers(0, 2, (32, 32)))
    expected = int(sk.stencil_apply(life_point, 1, g).to_array().sum())
    for P in (1, 2, 3, 4):
        ps = sk.partition(g, P, 1)
        partials, combined = sk.parallel_step(ps, life_point, 1, sk.sum_combinator(0))
        assert len(partials) == P and combined == expected


def test_helmholtz_steps_with_env_slices():
    """A built-in kernel with an env grid, stepped partition by partition."""
    from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

    n, m = 37, 64
    rhs = np.random.default_rng(5).random((n, m))
    f = Grid.from_array(rhs)
    kern = helmholtz_kernel(HelmholtzConfig(rows=n, cols=m, relax=0.8))
    u = Grid.from_array(np.zeros((n, m)))
    want = u
    for _ in range(3):
        want = sk.stencil_apply(kern, 1, want, env=f)
    ps = sk.partition(u, 3, 1)
    for _ in range(3):
        sk.halo_exchange(ps)
        sk.parallel_step(ps, kern, 1, sk.max_combinator(0.0), env=f)
        ps.swap_all()
    assert np.array_equal(ps.gather("front").to_array(), want.to_array())
