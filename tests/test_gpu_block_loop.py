"""Multi-rank loops of user elemental functions (distributed.block_loop) on
one B200: 2-3 ranks share cuda:0 over gloo (NCCL refuses two ranks per GPU),
each sweeping its row block with k-deep halo rows exchanged every iteration
and the partials folded in rank order on the device.  The gathered grid must
equal the REAL reference's single-process result bit for bit (golden_jit),
with the same iteration count and final value."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _worker(rank, world, port, name, q):
    sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import jit_cases as J
        import paper_1609_04567_b200 as sk
        from jit_common import device_cond, op_of
        from paper_1609_04567_b200.distributed import block_loop
        from paper_1609_04567_b200.partition import _split_ranges

        torch.cuda.set_device(0)
        spec = {**J.CASES, **J.CASES_1D}[name]
        g = spec["grid"]()
        env = spec["env"]() if spec["env"] is not None else None
        lo, hi = _split_ranges(g.shape[0], world)[rank]

        def blk(a):
            # Grid(dims, array) keeps the element dtype (the fixture's f32 grid
            # was built from np.float32 values); from_array widens like the reference
            b = np.ascontiguousarray(a[lo:hi])
            return sk.Grid(b.shape, b)

        benv = None if env is None else (tuple(blk(e) for e in env) if isinstance(env, tuple)
                                         else blk(env))
        delta = sk.Delta(spec["delta"]) if spec["delta"] is not None else None
        out, rep = block_loop(sk.ElementalFn(spec["point"], spec["k"]), spec["k"], op_of(spec),
                              device_cond(spec), blk(g), env=benv, delta=delta,
                              indexed=spec.get("indexed", False), rank=rank, world=world)
        mine = torch.from_numpy(out.to_array())
        parts = [torch.zeros((b - a,) + tuple(mine.shape[1:]), dtype=mine.dtype)
                 for a, b in _split_ranges(g.shape[0], world)]
        for r in range(world):
            dist.broadcast(mine if r == rank else parts[r], src=r)
        parts[rank] = mine
        if rank == 0:
            q.put((rep.iterations, rep.final_reduce, rep.exhausted, torch.cat(parts).numpy()))
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,world", [("jacobi_f64", 2), ("jacobi_f64", 3),
                                        ("box_mean_r2", 3), ("life_glider", 2),
                                        ("tuple_env", 2), ("f32_relax", 3)])
def test_block_loop_equals_reference(name, world):
    sys.path.insert(0, HERE)
    from jit_common import golden

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in ps:
        p.start()
    it, val, ex, grid = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    meta, arrays = golden()
    m = meta[name]
    assert it == m["iterations"] and ex == m["exhausted"]
    want = arrays[name]
    assert grid.dtype == want.dtype
    assert np.array_equal(grid.view(np.uint8), want.view(np.uint8))
    if m["final_is_int"] or name in ("jacobi_f64", "f32_relax"):  # exact reduces
        assert float(val) == m["final_reduce"]
    else:
        assert abs(float(val) - m["final_reduce"]) <= 1e-12 * abs(m["final_reduce"])
