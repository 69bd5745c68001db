"""Multi-rank driver logic on CPU (gloo, world_size 2 and 3).

The rank-block driver of paper_1609_04567_b200.distributed (halo exchange
of boundary rows, all-gather of per-rank partials, rank-ordered combine,
batched stepping with a device-decided stop) is run with a CPU test double
of the per-rank engine whose sweep is the oracle's restatement of the
reference block kernel.  The gathered result must equal the single-process
oracle run bit for bit, with the same iteration count and final value.
The GPU path replaces only the sweep/combine engine (DeviceBlock).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import stencil_oracle as O
from paper_1609_04567_b200.distributed import exchange_halos, gather_partials, run_block_loop
from paper_1609_04567_b200.partition import _split_ranges


class OracleBlock:
    """CPU stand-in for DeviceBlock: same buffers/halo layout and protocol."""

    def __init__(self, u0, f, consts, rank, world, tol, max_it):
        self.rank, self.world = rank, world
        self.rows, self.cols = u0.shape
        self.ht = 1 if rank > 0 else 0
        self.hb = 1 if rank < world - 1 else 0
        R = self.ht + self.rows + self.hb
        self.src = torch.zeros((R, self.cols), dtype=torch.float32)
        self.src[self.ht:self.ht + self.rows] = torch.from_numpy(u0)
        self.f = f
        self.consts = consts
        self.bufs = [torch.zeros_like(self.src) for _ in range(2)]
        exchange_halos(self.src, rank, world, self.ht, self.rows)
        self.it = self.launched = self.decided = 0
        self.stopped = self.exhausted = False
        self.partial = torch.zeros(1, dtype=torch.float64)
        self.gathered = torch.zeros(world, dtype=torch.float64)
        self.gvalue = None
        self.tol, self.max_it = tol, max_it

    def buffer_of(self, t):
        return self.bufs[t & 1]

    def step(self, cond):
        self.launched += 1
        if not self.stopped:
            t = self.it + 1
            front = self.src if t == 1 else self.bufs[(t - 1) & 1]
            slab = front.numpy()
            new = O.helmholtz_sweep(slab, np.pad(self.f, ((self.ht, self.hb), (0, 0))),
                                    self.consts)[self.ht:self.ht + self.rows]
            # rows next to a halo saw the halo; rows next to the slab edge saw 0 = global edge
            old = slab[self.ht:self.ht + self.rows]
            self.buffer_of(t)[self.ht:self.ht + self.rows] = torch.from_numpy(new)
            self.partial[0] = float(np.max(np.abs(new - old)))
            self.it = t
        exchange_halos(self.buffer_of(self.launched), self.rank, self.world, self.ht, self.rows)
        gather_partials(self.partial, self.gathered)
        if not self.stopped and self.it > self.decided:
            acc = 0.0
            for v in self.gathered.tolist():
                acc = acc if v < acc else v
            self.gvalue, self.decided = acc, self.it
            c = acc < self.tol
            self.exhausted = not c and self.it >= self.max_it
            self.stopped = c or self.it >= self.max_it

    def status(self):
        return self.it, self.gvalue, self.stopped, self.exhausted


def _worker(rank, world, port, n, m, tol, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rhs = np.random.default_rng(3).random((n, m)).astype(np.float32)
        lo, hi = _split_ranges(n, world)[rank]
        consts = O.helmholtz_consts(0.5, 0.5, 0.25, 0.8)
        blk = OracleBlock(np.zeros((hi - lo, m), np.float32), rhs[lo:hi], consts, rank, world,
                          tol, 10_000)
        res = run_block_loop(blk, cond=None, batch=3)
        out = res.out.contiguous()
        parts = [torch.zeros((b - a, m), dtype=torch.float32) for a, b in _split_ranges(n, world)]
        dist.all_gather(parts, out) if all(p.shape == out.shape for p in parts) else \
            [dist.broadcast(p if r != rank else out, src=r) for r, p in enumerate(parts)]
        if rank == 0:
            parts[0] = out
            q.put((res.iterations, res.final_reduce, torch.cat(parts).numpy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,n", [(2, 48), (3, 37)])
def test_rank_blocks_match_single_process_oracle(world, n):
    m, tol = 40, 1e-4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, tol, q)) for r in range(world)]
    for p in procs:
        p.start()
    it, val, grid = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rhs = np.random.default_rng(3).random((n, m)).astype(np.float32)
    u, it_ref, v_ref, _ = O.helmholtz_loop(np.zeros_like(rhs), rhs,
                                           O.helmholtz_consts(0.5, 0.5, 0.25, 0.8), delta="abs",
                                           op="max", cond=lambda v, i: v < tol)
    assert it == it_ref and val == v_ref
    assert np.array_equal(grid.view(np.uint32), u.view(np.uint32))
