"""Host-side logic of the drop-in API (CPU): grid container, partition
geometry and preconditions, copy-ledger model, reduce/delta/condition
recognition, worker groups, and that the product path refuses to run
without the GPU engine (no CPU fallback)."""

import math

import numpy as np
import pytest

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200 import _native
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel
from paper_1609_04567_b200.grid import ABSENT, GridError
from paper_1609_04567_b200.partition import _check_partitioning, _split_ranges, model_ledger
from paper_1609_04567_b200.patterns import (DeviceUnsupported, combinator_kind, delta_kind)


# --------------------------------------------------------------- grid

def test_grid_construction_and_access():
    g = sk.Grid((2, 3), [1, 2, 3, 4, 5, 6])
    assert g.at(1, 2) == 6 and g[0, 1] == 2 and g.size == 6 and g.ndim == 2
    assert g.to_rows() == [[1, 2, 3], [4, 5, 6]]
    assert g.to_array().dtype == np.int64
    with pytest.raises(GridError):
        sk.Grid((2, 2), [1, 2, 3])
    with pytest.raises(GridError):
        sk.Grid((0, 2), [])
    with pytest.raises(GridError):
        sk.Grid((1, 1, 1), [1])
    with pytest.raises(GridError):
        g.at(2, 0)
    with pytest.raises(GridError):
        sk.Grid.from_rows([[1, 2], [3]])


def test_grid_equality_and_storage_kinds():
    a = sk.Grid((2, 2), [1.0, 2.0, 3.0, 4.0])
    b = sk.Grid.from_array(np.array([[1, 2], [3, 4]], dtype=np.int64))
    assert a == b  # value equality, like the reference's list comparison
    assert sk.Grid.filled((3, 3), 0.0).storage_dtype() == np.float64
    f32 = sk.Grid((2, 2), list(np.zeros(4, np.float32)))
    assert f32.storage_dtype() == np.float32
    c = a.copy()
    c.data[0] = 99.0
    assert a.at(0, 0) == 1.0 and c.at(0, 0) == 99.0


def test_windows_and_absent():
    g = sk.Grid.from_rows([[1, 2, 3], [4, 5, 6], [7, 8, 9]])
    nb = sk.neighborhood_at(g, (0, 0), 1)
    assert nb.center == 1 and nb.at(-1, -1) is ABSENT and nb.at(1, 1) == 5
    assert nb.values() == [1, 2, 4, 5]
    inb = sk.indexed_neighborhood_at(g, (2, 2), 1)
    assert inb.center == (9, (2, 2)) and inb.at(0, 1) is ABSENT
    assert sk.grid_get_padded(g, (5, 5)) is ABSENT
    assert not ABSENT and repr(ABSENT) == "ABSENT"


# --------------------------------------------------------------- partitions

def test_split_ranges_remainder_to_lowest():
    assert _split_ranges(8, 2) == [(0, 4), (4, 8)]
    assert _split_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert _split_ranges(5, 5) == [(i, i + 1) for i in range(5)]


def test_partitioning_preconditions():
    with pytest.raises(GridError):
        _check_partitioning(3, 4, 1)
    with pytest.raises(GridError):
        _check_partitioning(8, 4, 3)  # 2 rows per partition < halo 3
    with pytest.raises(GridError):
        _check_partitioning(8, 0, 1)
    _check_partitioning(8, 1, 5)  # a single partition needs no halo


def test_model_ledger_matches_reference_fixtures(golden):
    checked = 0
    for name, m in golden.meta.items():
        if "ledger" not in m:
            continue
        k = 1
        led = model_ledger((m["rows"], m["cols"]), m.get("P", 1), k, m.get("iterations", 1))
        assert vars(led) == m["ledger"], name
        checked += 1
    assert checked >= 20


def test_deployment_mode_parse():
    assert sk.DeploymentMode.parse("1:n") is sk.DeploymentMode.ONE_TO_N
    with pytest.raises(GridError):
        sk.DeploymentMode.parse("2:3")


# --------------------------------------------------------------- recognition

def test_combinator_and_delta_recognition():
    assert combinator_kind(sk.sum_combinator(0.0)) == "sum"
    assert combinator_kind(sk.Combinator(lambda a, b: a + b, 0)) == "sum"
    assert combinator_kind(sk.Combinator(lambda a, b: a if b < a else b, 0.0)) == "max"
    assert combinator_kind(sk.Combinator(lambda a, b: max(a, b), 0.0)) == "max"
    with pytest.raises(DeviceUnsupported):
        combinator_kind(sk.Combinator(lambda a, b: a * b, 1))
    assert delta_kind(None) == "none"
    assert delta_kind(sk.Delta(lambda n, o: abs(n - o))) == "abs"
    assert delta_kind(sk.Delta(lambda n, o: (n - o) ** 2)) == "square"
    with pytest.raises(DeviceUnsupported):
        delta_kind(sk.Delta(lambda n, o: n - o))


def _shadow_abs(x):
    return 0.0


@pytest.mark.parametrize("fn", [
    lambda a, b: a + b if b < 50 else a,       # agrees with a + b on small values only
    lambda a, b: min(a + b, 100.0),
    lambda a, b: a + b + 0.0 * a,
    lambda a, b: a - b,
    lambda a, b: b if b < a else a,            # min, not max
    lambda a, b: a if b <= a else b,
])
def test_near_miss_combinators_are_not_builtin_reduces(fn):
    """no classification by sampling -- a function that
    matches SUM / MAX on probe pairs but not everywhere must not run as the
    built-in reduce (the JIT compiles it instead)."""
    with pytest.raises(DeviceUnsupported):
        combinator_kind(sk.Combinator(fn, 0.0))


@pytest.mark.parametrize("fn", [
    lambda n, o: abs(n - o) if abs(n - o) < 100 else 0.0,
    lambda n, o: min(abs(n - o), 10.0),
    lambda n, o: (n - o) ** 3,
    lambda n, o: abs(n + o),
    lambda n, o: _shadow_abs(n - o),
])
def test_near_miss_deltas_are_not_builtin_deltas(fn):
    with pytest.raises(DeviceUnsupported):
        delta_kind(sk.Delta(fn))


def test_exact_forms_and_shadowed_names():
    import operator

    assert combinator_kind(sk.Combinator(operator.add, 0)) == "sum"
    assert combinator_kind(sk.Combinator(lambda x, y: y + x, 0)) == "sum"
    assert combinator_kind(sk.Combinator(lambda a, b: a if a > b else b, 0.0)) == "max"

    def mx(a, b):
        """docstring is fine"""
        return a if b < a else b

    assert combinator_kind(sk.Combinator(mx, 0.0)) == "max"
    assert delta_kind(sk.Delta(lambda new, old: abs(old - new))) == "abs"
    assert delta_kind(sk.Delta(lambda new, old: (old - new) ** 2)) == "square"


def test_shadowed_abs_is_not_the_builtin():
    abs = _shadow_abs  # noqa: A001 -- a local `abs` that is not the builtin
    with pytest.raises(DeviceUnsupported):
        delta_kind(sk.Delta(lambda n, o: abs(n - o)))


@pytest.mark.parametrize("cond", [sk.Condition.below(1e-4), sk.Condition.rms_below(1e-6, 256),
                                  sk.Condition.mean_below(0.02, 1234), sk.stop_after(7)])
def test_device_conditions_equal_their_python_predicates(cond):
    # the device evaluates the same fp64 expression; check the host form here
    dc = cond.device
    rng = np.random.default_rng(0)
    for v in list(rng.random(200) * 1e-3) + [0.0, 1e-4, 2.56e-10, 24.68]:
        for it in (1, 6, 7, 8):
            if dc.kind == "lt":
                dev = v < dc.a
            elif dc.kind == "rms_lt":
                dev = math.sqrt(v / dc.n) < dc.a
            elif dc.kind == "mean_lt":
                dev = v / dc.n < dc.a
            else:
                dev = it >= dc.n
            assert dev == cond.fn(v, it, None)


def test_condition_validation():
    with pytest.raises(ValueError):
        sk.Condition(lambda v, i, s: True, max_iterations=0)
    with pytest.raises(ValueError):
        sk.stop_after(0)


# --------------------------------------------------------------- groups

def test_worker_group_single_run_and_close():
    g = sk.WorkerGroup(2)
    g.start_run()
    with pytest.raises(RuntimeError):
        g.start_run()
    with pytest.raises(RuntimeError):
        g.close()
    g.end_run()
    g.close()
    with pytest.raises(RuntimeError):
        g.start_run()
    with pytest.raises(ValueError):
        sk.WorkerGroup(0)
    with pytest.raises(ValueError):
        sk.DeviceExecutor(3, sk.WorkerGroup(2))


def test_parallel_loop_argument_validation():
    g = sk.Grid.filled((4, 4), 0.0)
    k = helmholtz_kernel(HelmholtzConfig(4, 4))
    with pytest.raises(GridError):
        sk.parallel_loop("1:n", 1, 1, k, sk.sum_combinator(0.0), sk.stop_after(1), g, env=g)
    with pytest.raises(GridError):
        sk.parallel_loop("1:1", 0, 1, k, sk.sum_combinator(0.0), sk.stop_after(1), g, env=g)
    with pytest.raises(GridError):
        sk.parallel_loop("1:1", 1, 1, k, sk.sum_combinator(0.0), sk.stop_after(1), g, env=g,
                         group=sk.WorkerGroup(2))


def test_product_path_has_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = sk.Grid.filled((8, 8), 0.0)
    with pytest.raises(_native.DeviceUnavailable):
        sk.parallel_loop("1:1", 1, 1, helmholtz_kernel(HelmholtzConfig(8, 8)),
                         sk.max_combinator(0.0), sk.Condition.below(1e-4), g, env=g,
                         delta=sk.abs_change())
    with pytest.raises(_native.DeviceUnavailable):
        sk.loop_stencil_reduce(1, lambda nb, env: nb.center, sk.sum_combinator(0),
                               sk.stop_after(1), g)


def test_adapts_reference_plan_objects():
    """The executor accepts the reference's own LoopPlan/Grid shapes (plugin route)."""
    from types import SimpleNamespace

    from paper_1609_04567_b200.partition import _adapt

    ours = helmholtz_kernel(HelmholtzConfig(4, 4))
    ref_fn = SimpleNamespace(point=ours, k=1, device=None)  # stencilkit wraps bare callables
    ref_grid = SimpleNamespace(dims=(4, 4), data=[0.0] * 16)
    ref_env = SimpleNamespace(dims=(4, 4), data=[1.0] * 16)
    ref_plan = SimpleNamespace(fn=ref_fn, k=1, op=SimpleNamespace(fn=lambda a, b: a + b,
                                                                   identity=0.0),
                               env=ref_env, indexed=False, delta=None)
    plan, grid = _adapt(ref_plan, ref_grid)
    assert plan.fn is ours and isinstance(grid, sk.Grid) and isinstance(plan.env, sk.Grid)
    assert combinator_kind(plan.op) == "sum"


def test_from_array_widens_floats_like_the_reference():
    """the reference's Grid.from_array stores
    arr.tolist() -- Python floats -- so a float32 array computes in fp64;
    Grid(dims, float32 elements) and from_tensor keep float32."""
    import torch

    a = np.arange(6, dtype=np.float32).reshape(2, 3) / 3
    g = sk.Grid.from_array(a)
    assert g.storage_dtype() == np.float64
    assert np.array_equal(g.to_array(), a.astype(np.float64))
    assert sk.Grid(a.shape, a).storage_dtype() == np.float32
    assert sk.Grid.from_tensor(torch.from_numpy(a)).storage_dtype() == np.float32
    assert sk.Grid.from_array(np.arange(4, dtype=np.uint8)).storage_dtype() == np.uint8
