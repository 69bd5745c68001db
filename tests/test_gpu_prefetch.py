"""Grid.prefetch_device / prefetch_host(out=): the asynchronous copies a
host pipeline of drop-in calls uses (bench.py's pipelined e2e).  Results
must equal the synchronous path bit for bit."""

import numpy as np
import pytest

import paper_1609_04567_b200 as sk

pytestmark = pytest.mark.gpu


def test_prefetched_inputs_and_async_readback_equal_sync_path():
    import torch

    from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

    n, m = 515, 777
    rng = np.random.default_rng(4)
    u0 = rng.random((n, m)).astype(np.float32)
    f = rng.random((n, m)).astype(np.float32)
    kern = helmholtz_kernel(HelmholtzConfig(rows=n, cols=m, relax=0.9))
    cond = sk.Condition.below(1e-4)

    def solve(gu, gf):
        return sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0), cond,
                                        gu, env=gf)

    ref, rrep = solve(sk.Grid(u0.shape, u0), sk.Grid(f.shape, f))
    want = ref.to_array()
    hu = torch.from_numpy(u0).pin_memory()
    hf = torch.from_numpy(f).pin_memory()
    outs = [torch.empty((n, m), dtype=torch.float32).pin_memory() for _ in range(2)]
    prev = None
    nxt = (sk.Grid.from_tensor(hu).prefetch_device(), sk.Grid(f.shape, f).prefetch_device())
    for k in range(4):
        gu, gf = nxt
        o, rep = solve(gu, gf)
        assert rep.iterations == rrep.iterations and rep.final_reduce == rrep.final_reduce
        nxt = (sk.Grid.from_tensor(hu).prefetch_device(), sk.Grid.from_tensor(hf).prefetch_device())
        o.prefetch_host(out=outs[k % 2].numpy())
        if prev is not None:
            assert np.array_equal(prev.to_array().view(np.uint32), want.view(np.uint32))
        prev = o
    got = prev.to_array()
    assert got is not None and np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # a host grid that was prefetched and then read on the host is unchanged
    g = sk.Grid(u0.shape, u0.copy()).prefetch_device()
    assert np.array_equal(g.to_array(), u0)
    assert np.array_equal(g.tensor(device="cuda").cpu().numpy(), u0)
