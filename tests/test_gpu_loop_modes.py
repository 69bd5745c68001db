"""Every device-loop mode gives the same bits: persistent cooperative launch
(default), CUDA-graph WHILE loop (SK_NO_PERSIST=1), batched launches with a
device-decided stop (SK_NO_PERSIST=1 SK_NO_GRAPH=1), and the host-driven
lag-1 loop (a plain Python condition)."""

import numpy as np
import pytest

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import (HelmholtzConfig, amf_detect, helmholtz_kernel,
                                        restore_regularize)
from oracle import stencil_oracle as O

pytestmark = pytest.mark.gpu

MODES = [{}, {"SK_NO_PERSIST": "1"}, {"SK_NO_PERSIST": "1", "SK_NO_GRAPH": "1"}]


def _helm():
    n, m = 200, 136
    rhs = np.random.default_rng(3).random((n, m)).astype(np.float32)
    cfg = HelmholtzConfig(n, m, alpha=0.5, dx=0.5, dy=0.25, relax=0.8)
    out, rep = sk.parallel_loop("1:n", 3, 1, helmholtz_kernel(cfg), sk.max_combinator(0.0),
                                sk.Condition.below(1e-4), sk.Grid(rhs.shape, np.zeros_like(rhs)),
                                env=sk.Grid(rhs.shape, rhs), delta=sk.abs_change())
    return out.to_array(), rep.iterations, rep.final_reduce


def _denoise():
    noisy, _ = O.salt_pepper(O.gradient_image(96, 80), 0.5, seed=42)
    g = sk.Grid.from_array(noisy)
    mask = amf_detect(g)
    out, rep = restore_regularize(g, mask, partitions=2)
    return out.to_array(), rep.iterations, rep.final_reduce, mask.to_array()


@pytest.mark.parametrize("env", MODES)
def test_modes_agree(monkeypatch, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    u, it, v = _helm()
    n, m = u.shape
    rhs = np.random.default_rng(3).random((n, m)).astype(np.float32)
    ref_u, ref_it, ref_v, _ = O.helmholtz_loop(np.zeros_like(rhs), rhs,
                                               O.helmholtz_consts(0.5, 0.5, 0.25, 0.8),
                                               delta="abs", op="max",
                                               cond=lambda val, i: val < 1e-4, P=3)
    assert (it, v) == (ref_it, ref_v)
    assert np.array_equal(u.view(np.uint32), ref_u.view(np.uint32))
    out, it2, v2, mask = _denoise()
    noisy, _ = O.salt_pepper(O.gradient_image(96, 80), 0.5, seed=42)
    assert np.array_equal(mask.astype(np.uint8), O.amf_detect(noisy))
    ref_o, ref_it2, ref_v2, _ = O.restore_loop(noisy, O.amf_detect(noisy), P=2)
    assert it2 == ref_it2 and np.array_equal(out, ref_o)
    assert v2 == pytest.approx(ref_v2, rel=1e-12)


def test_host_driven_loop_with_state_matches_device_loop():
    rhs = np.ones((64, 64), np.float32)
    cfg = HelmholtzConfig(64, 64)
    seen = []
    state = sk.LoopState(init=lambda: 0, update=lambda s, it, v: (seen.append(v), s + 1)[1])
    out, rep = sk.loop_stencil_reduce_s(1, helmholtz_kernel(cfg), sk.max_combinator(0.0),
                                        lambda v, it, s: v < 1e-4, state,
                                        sk.Grid(rhs.shape, np.zeros_like(rhs)),
                                        env=sk.Grid(rhs.shape, rhs), delta=sk.abs_change())
    out2, rep2 = sk.loop_stencil_reduce_d(1, helmholtz_kernel(cfg), sk.abs_change(),
                                          sk.max_combinator(0.0), sk.Condition.below(1e-4),
                                          sk.Grid(rhs.shape, np.zeros_like(rhs)),
                                          env=sk.Grid(rhs.shape, rhs))
    assert rep.iterations == rep2.iterations == len(seen) == 36
    assert rep.final_reduce == rep2.final_reduce == seen[-1]
    assert out == out2
    assert all(b <= a for a, b in zip(seen[1:], seen[2:]))
