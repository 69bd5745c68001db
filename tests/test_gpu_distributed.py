"""The multi-GPU rank-block engine on one B200: two ranks (processes) share
cuda:0 over gloo (halo rows and partials staged through the host -- NCCL
refuses two ranks per GPU), each running the native DeviceBlock (fused sweep
with real halo rows + device-side rank-ordered combine).  The gathered grid
must equal the single-GPU solve of the same global grid bit for bit, with the
same iteration count and final MAX value."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, n, m, q, transport="collective"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1609_04567_b200.distributed import DeviceBlock, make_cond, run_block_loop
        from paper_1609_04567_b200.partition import _split_ranges

        torch.cuda.set_device(0)
        rhs = np.random.default_rng(5).random((n, m)).astype(np.float32)
        lo, hi = _split_ranges(n, world)[rank]
        u0 = torch.zeros((hi - lo, m), dtype=torch.float32, device="cuda")
        f = torch.from_numpy(rhs[lo:hi]).cuda()
        consts = (4.0, 16.0, 40.5, 1.0 - 0.8, 0.8)  # alpha .5, dx .5, dy .25, relax .8
        blk = DeviceBlock(u0, f, consts, rank=rank, world=world, transport=transport)
        res = run_block_loop(blk, make_cond("lt", 1e-4), batch=3)
        out = res.out.contiguous().cpu()
        blk.close()
        parts = [torch.zeros((b - a, m), dtype=torch.float32) for a, b in _split_ranges(n, world)]
        for r in range(world):
            dist.broadcast(out if r == rank else parts[r], src=r)
        parts[rank] = out
        if rank == 0:
            q.put((res.iterations, res.final_reduce, torch.cat(parts).numpy()))
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,n,transport", [(2, 200, "collective"), (3, 131, "collective"),
                                               (2, 200, "peer"), (3, 131, "peer"),
                                               (4, 97, "peer")])
def test_two_ranks_one_gpu_equal_single_gpu(world, n, transport):
    """transport="peer": the sweep kernel stores boundary rows into the
    neighbours' halo rows and publishes its partial + flag into every rank's
    mailbox (CUDA IPC mappings of the other processes' memory on the same
    device); the stream waits on the flags; no collective on the path."""
    import paper_1609_04567_b200 as sk
    from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

    m = 160
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, m, q, transport))
          for r in range(world)]
    for p in ps:
        p.start()
    try:
        it, val, grid = q.get(timeout=300)
        for p in ps:
            p.join(timeout=120)
            assert p.exitcode == 0
    finally:
        for p in ps:  # a rank stuck on a stream wait must not outlive the test
            if p.is_alive():
                p.kill()
    rhs = np.random.default_rng(5).random((n, m)).astype(np.float32)
    cfg = HelmholtzConfig(n, m, alpha=0.5, dx=0.5, dy=0.25, relax=0.8)
    out, rep = sk.parallel_loop("1:1", 1, 1, helmholtz_kernel(cfg), sk.max_combinator(0.0),
                                sk.Condition.below(1e-4), sk.Grid(rhs.shape, np.zeros_like(rhs)),
                                env=sk.Grid(rhs.shape, rhs), delta=sk.abs_change())
    assert it == rep.iterations and val == rep.final_reduce
    assert np.array_equal(grid.view(np.uint32), out.to_array().view(np.uint32))


def _worker2(rank, world, port, n, m, q, transport):
    """fp64, SUM of squared deltas (the RMS form of helmholtz_solve)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1609_04567_b200.distributed import DeviceBlock, make_cond, run_block_loop
        from paper_1609_04567_b200.partition import _split_ranges

        torch.cuda.set_device(0)
        rhs = np.random.default_rng(9).random((n, m))
        lo, hi = _split_ranges(n, world)[rank]
        u0 = torch.zeros((hi - lo, m), dtype=torch.float64, device="cuda")
        f = torch.from_numpy(rhs[lo:hi]).cuda()
        consts = (1.0, 1.0, 5.0, 0.0, 1.0)
        blk = DeviceBlock(u0, f, consts, rank=rank, world=world, reduce="sum", delta="square",
                          transport=transport)
        res = run_block_loop(blk, make_cond("rms_lt", 1e-6, float(n * m)), batch=4)
        out = res.out.contiguous().cpu()
        blk.close()
        parts = [torch.zeros((b - a, m), dtype=torch.float64) for a, b in _split_ranges(n, world)]
        for r in range(world):
            dist.broadcast(out if r == rank else parts[r], src=r)
        parts[rank] = out
        if rank == 0:
            q.put((res.iterations, res.final_reduce, torch.cat(parts).numpy()))
    finally:
        dist.destroy_process_group()


def test_peer_transport_fp64_sum_matches_collective():
    """The two transports give the same grid, iteration count and final SUM
    (fp64, RMS condition, 3 ranks on one GPU)."""
    outs = {}
    for transport in ("collective", "peer"):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _port()
        ps = [ctx.Process(target=_worker2, args=(r, 3, port, 61, 70, q, transport))
              for r in range(3)]
        for p in ps:
            p.start()
        try:
            outs[transport] = q.get(timeout=300)
            for p in ps:
                p.join(timeout=120)
                assert p.exitcode == 0
        finally:
            for p in ps:
                if p.is_alive():
                    p.kill()
    (i1, v1, g1), (i2, v2, g2) = outs["collective"], outs["peer"]
    assert i1 == i2 and i1 > 1 and v1 == v2
    assert np.array_equal(g1.view(np.uint64), g2.view(np.uint64))
