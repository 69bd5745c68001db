"""Multi-GPU 1:n deployment: one process per GPU, one row block per rank.

The reference models "1:n multi-device" with threads over row partitions
(partition.py:187-262, 596-664).  Here every rank is a real device:

  * rank r owns a contiguous block of rows of the global grid, stored with
    one halo row above (r > 0) and below (r < P-1) in both iteration
    buffers (the engine's halo_top / halo_bottom layout);
  * per iteration: the fused sweep (stencil + delta + this rank's reduce)
    -> halo exchange of the freshly written boundary rows with the two
    neighbours (NCCL send/recv over NVLink, halo_exchange partition.py:
    247-262) -> all-gather of the per-rank partials -> a one-thread device
    kernel folds them in rank order from the identity (partition.py:642-646)
    and evaluates the loop condition (loop.py:209-218) on every rank, so
    all ranks stop on the same iteration without any host round trip;
  * the host enqueues `batch` iterations ahead and reads the status once
    per batch; sweeps after the device-decided stop are no-ops.

The exchange and gather work on any torch.distributed backend: device
tensors go straight to NCCL; with gloo (CPU tests, or several ranks sharing
one GPU) rows are staged through host memory.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from .partition import _split_ranges


def _dist():
    import torch.distributed as dist

    return dist


def _direct(t) -> bool:
    """True when the backend can move `t` itself (NCCL + CUDA tensor)."""
    dist = _dist()
    return t.is_cuda and dist.get_backend() == "nccl"


def exchange_halos(buf, rank: int, world: int, halo_top: int, rows: int, group=None) -> None:
    """Refresh buf's halo rows from the neighbours' boundary rows.

    buf: [halo_top + rows + halo_bottom, pitch]; owned rows start at halo_top.
    Sends the first owned row up and the last owned row down; receives the
    neighbours' rows into the top/bottom halo rows (partition.py:247-262).
    """
    import torch

    dist = _dist()
    first, last = buf[halo_top], buf[halo_top + rows - 1]
    top = buf[0] if halo_top else None
    bot = buf[halo_top + rows] if rank < world - 1 else None
    direct = _direct(buf)
    stage = (lambda t: t) if direct else (lambda t: t.detach().cpu())
    ops, recvs = [], []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, stage(first).contiguous(), rank - 1, group))
        r = top if direct else torch.empty_like(top, device="cpu")
        ops.append(dist.P2POp(dist.irecv, r, rank - 1, group))
        recvs.append((r, top))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, stage(last).contiguous(), rank + 1, group))
        r = bot if direct else torch.empty_like(bot, device="cpu")
        ops.append(dist.P2POp(dist.irecv, r, rank + 1, group))
        recvs.append((r, bot))
    if not ops:
        return
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    if not direct:
        for r, dst in recvs:
            dst.copy_(r)


def gather_partials(value, out, group=None) -> None:
    """All-gather one double per rank into out[world] (rank order)."""
    dist = _dist()
    if _direct(value):
        dist.all_gather_into_tensor(out, value, group=group)
        return
    import torch

    parts = [torch.empty(1, dtype=torch.float64) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, value.detach().cpu().reshape(1), group=group)
    out.copy_(torch.cat(parts))


class _DevPtr:
    """A raw device pointer as a CUDA array (zero-copy torch view)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


@dataclass
class BlockResult:
    iterations: int
    final_reduce: float
    exhausted: bool
    out: object  # this rank's owned rows (device tensor view)


class DeviceBlock:
    """One rank's Helmholtz row block on its GPU, driven through the C-ABI.

    u0 / f: [rows, cols] device tensors of this rank's owned rows (fp32 or
    fp64).  The initial halo rows are exchanged at construction.
    """

    def __init__(self, u0, f, consts, *, rank: int, world: int, reduce: str = "max",
                 delta: str = "abs", identity: float = 0.0, timing: bool = False, group=None):
        import torch

        lib = N.require_cuda()
        self.lib, self.rank, self.world, self.group = lib, rank, world, group
        rows, cols = u0.shape
        self.rows, self.cols = rows, cols
        self.ht = 1 if rank > 0 else 0
        self.hb = 1 if rank < world - 1 else 0
        R = self.ht + rows + self.hb
        dt = u0.dtype
        vec = max(16 // u0.element_size(), 4)  # whole 4-element thread vectors
        pitch = -(-cols // vec) * vec
        self.pitch = pitch
        dev = u0.device
        self.src = torch.zeros((R, pitch), dtype=dt, device=dev)
        self.src[self.ht:self.ht + rows, :cols] = u0
        self.env = torch.zeros((R, pitch), dtype=dt, device=dev)
        self.env[self.ht:self.ht + rows, :cols] = f
        self.bufs = [torch.zeros((R, pitch), dtype=dt, device=dev) for _ in range(2)]
        exchange_halos(self.src, rank, world, self.ht, rows, group)
        p = N.sk_plan()
        p.kernel = N.SK_KERNEL_HELMHOLTZ
        p.dtype = N.SK_F32 if dt == torch.float32 else N.SK_F64
        p.rows, p.cols = rows, cols
        p.partitions = 1
        p.reduce_op = N.SK_REDUCE_MAX if reduce == "max" else N.SK_REDUCE_SUM
        p.delta_op = {"none": N.SK_DELTA_NONE, "abs": N.SK_DELTA_ABS,
                      "square": N.SK_DELTA_SQUARE}[delta]
        p.halo_top, p.halo_bottom = self.ht, self.hb
        p.flags = N.SK_FLAG_TIMING if timing else 0
        p.identity = identity
        for i, v in enumerate(consts):
            p.params[i] = float(v)
        h = C.c_void_p()
        st = torch.cuda.current_stream()
        N.check(lib.sk_run_begin(C.byref(p), C.c_void_p(self.src.data_ptr()), pitch,
                                 C.c_void_p(self.env.data_ptr()), pitch,
                                 C.c_void_p(self.bufs[0].data_ptr()),
                                 C.c_void_p(self.bufs[1].data_ptr()), pitch,
                                 N.stream_handle(st), C.byref(h)))
        self.h = h
        vp = C.c_void_p()
        N.check(lib.sk_run_value_ptr(h, C.byref(vp)))
        self._vptr = _DevPtr(vp.value, 1)
        self.partial = torch.as_tensor(self._vptr, device=dev)
        self.gathered = torch.zeros(world, dtype=torch.float64, device=dev)
        self.launched = 0

    def buffer_of(self, t: int):
        return self.bufs[t & 1]

    def step(self, cond: "N.sk_cond") -> None:
        """Enqueue one iteration: sweep -> halo exchange -> gather -> combine."""
        N.check(self.lib.sk_run_launch(self.h, 1))
        self.launched += 1
        exchange_halos(self.buffer_of(self.launched), self.rank, self.world, self.ht, self.rows,
                       self.group)
        gather_partials(self.partial, self.gathered, self.group)
        N.check(self.lib.sk_run_combine(self.h, C.c_void_p(self.gathered.data_ptr()), self.world,
                                        C.byref(cond)))

    def status(self):
        it, val, stp, ex = C.c_int64(), C.c_double(), C.c_int32(), C.c_int32()
        N.check(self.lib.sk_run_status(self.h, C.byref(it), C.byref(val), C.byref(stp),
                                       C.byref(ex)))
        return it.value, val.value, bool(stp.value), bool(ex.value)

    def kernel_time(self):
        ms, n = C.c_double(), C.c_int64()
        N.check(self.lib.sk_run_kernel_time(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def launches(self) -> int:
        n = C.c_int64()
        N.check(self.lib.sk_run_launches(self.h, C.byref(n)))
        return n.value

    def close(self):
        if self.h is not None:
            N.check(self.lib.sk_run_destroy(self.h))
            self.h = None


def make_cond(kind: str, a: float = 0.0, n: float = 0.0, max_iterations: int = 10_000):
    c = N.sk_cond()
    c.kind = {"lt": N.SK_COND_LT, "rms_lt": N.SK_COND_RMS_LT, "mean_lt": N.SK_COND_MEAN_LT,
              "iter_ge": N.SK_COND_ITER_GE}[kind]
    c.a, c.n, c.max_iterations = a, n, max_iterations
    return c


def run_block_loop(block, cond, batch: int = 4) -> BlockResult:
    """Drive a block (DeviceBlock or a test double) to the device-decided stop."""
    while True:
        for _ in range(batch):
            block.step(cond)
        it, val, stopped, ex = block.status()
        if stopped:
            break
    out = block.buffer_of(it)[block.ht:block.ht + block.rows, :block.cols]
    return BlockResult(iterations=it, final_reduce=val, exhausted=ex, out=out)


# ---------------------------------------------------------------- bench driver


def bench_weak_scaling(args, world: int, rank: int, local: int, ClockSampler, measured_peaks):
    """C4 weak scaling: every rank a 32768 x 32768 fp32 block of a (32768*P) x
    32768 grid; returns rank 0's JSON line (None on other ranks)."""
    import torch

    dist = _dist()
    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    n = args.n
    consts = (1.0, 1.0, 5.0, 0.0, 1.0)
    cond = make_cond("lt", 1e-4, 0.0, 10_000)
    u0 = torch.zeros((n, n), dtype=torch.float32, device="cuda")
    f = torch.ones((n, n), dtype=torch.float32, device="cuda")

    def solve(timing=False):
        blk = DeviceBlock(u0, f, consts, rank=rank, world=world, timing=timing)
        res = run_block_loop(blk, cond)
        kt = blk.kernel_time() if timing else (0.0, 0)
        nl = blk.launches()
        blk.close()
        return res, kt, nl

    for _ in range(args.warmup):
        res, _, _ = solve()
    torch.cuda.synchronize()
    dist.barrier()
    kms, kn, launches = 0.0, 0, 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        s.record()
        for _ in range(args.steps):
            res, kt, nl = solve(timing=True)
            kms += kt[0]
            kn += kt[1]
            launches += nl
            del res
        e.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([s.elapsed_time(e) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    res, _, _ = solve()
    iters = res.iterations
    cells = float(world) * n * n * iters
    peak, peak_kind = measured_peaks()
    avg = kms / max(kn, 1)
    alg = 12.0 * n * n
    if rank != 0:
        return None
    return {
        "metric": "stencil cell-updates/s", "value": cells / (ms / 1e3),
        "unit": "cell-updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (rhs=1, u0=0)",
        "config": {"workload": f"C4 Helmholtz/Jacobi ({n}*{world})x{n} fp32, MAX|delta|<1e-4",
                   "rows_per_gpu": n, "cols": n, "iterations_per_step": iters,
                   "final_reduce": res.final_reduce, "parallelism": f"row blocks x{world}, "
                   "NCCL halo rows + device-side rank-ordered combine",
                   "l2": "inputs 4.3 GB/array > 126 MB L2 (no flush needed)"},
        "gpu_launches": launches,
        "e2e": None,
        "roofline": {"bound": "hbm", "achieved": alg / (avg / 1e3) / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": alg / (avg / 1e3) / 1e9 / peak, "traffic": None,
                     "kernel": "helmholtz_sweep<float> (rank 0)", "avg_kernel_ms": avg,
                     "peak_source": peak_kind},
        "cpu_baseline": None,
        "clocks": clk.summary(),
    }
