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


def exchange_halos(buf, rank: int, world: int, halo_top: int, rows: int, group=None,
                   k: int = 1) -> None:
    """Refresh buf's halo rows from the neighbours' boundary rows.

    buf: [halo_top + rows + halo_bottom, pitch]; owned rows start at halo_top.
    Sends the first k owned rows up and the last k down; receives the
    neighbours' rows into the top/bottom k halo rows (partition.py:247-262).
    """
    import torch

    dist = _dist()
    first, last = buf[halo_top:halo_top + k], buf[halo_top + rows - k:halo_top + rows]
    top = buf[0:k] if halo_top else None
    bot = buf[halo_top + rows:halo_top + rows + k] if rank < world - 1 else None
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


class PeerUnavailable(RuntimeError):
    """The peer transport cannot be set up on these ranks (raised on all)."""


class PeerRegion:
    """This rank's share of the peer transport, and every rank's as mapped here.

    One device allocation per rank (cudaMalloc, exported by CUDA IPC):
    [buf0 | buf1 | mailbox double[2][world] | flag words uint32[world]],
    the same layout on every rank (buffers sized for the largest block).
    Other ranks' regions are mapped with cudaIpcOpenMemHandle -- over
    NVLink on a multi-GPU node, or the same device when ranks share a GPU.
    """

    def __init__(self, buf_bytes: int, rank: int, world: int, group=None):
        lib = N.require_cuda()
        self.lib, self.rank, self.world, self.group = lib, rank, world, group
        al = lambda x: -(-x // 256) * 256
        self.off_buf = (0, al(buf_bytes))
        self.off_mail = 2 * al(buf_bytes)
        self.off_flag = self.off_mail + al(16 * world)
        total = self.off_flag + al(4 * world)
        # every step is agreed across ranks, so a failure anywhere (no IPC in
        # the container, no peer access) makes every rank raise PeerUnavailable
        # together instead of leaving the others in a collective
        self.own, mine = None, None
        try:
            ptr = C.c_void_p()
            N.check(lib.sk_ipc_alloc(total, C.byref(ptr)))
            self.own = ptr.value
            h = C.create_string_buffer(64)
            N.check(lib.sk_ipc_handle(C.c_void_p(self.own), h))
            mine = bytes(h.raw)
        except N.NativeError as e:
            mine = f"error: {e}"
        handles = _all_objects(mine, group)
        bad = [x for x in handles if not isinstance(x, bytes)]
        if bad:
            self._free_own()
            raise PeerUnavailable(bad[0])
        self.base, err = [], None
        for p, hb in enumerate(handles):
            if p == rank:
                self.base.append(self.own)
                continue
            q = C.c_void_p()
            try:
                N.check(lib.sk_ipc_open(C.create_string_buffer(hb, 64), C.byref(q)))
                self.base.append(q.value)
            except N.NativeError as e:
                err = err or f"rank {rank} cannot map rank {p}: {e}"
        errs = [x for x in _all_objects(err, group) if x]
        if errs:
            for p, b in enumerate(self.base):
                if p != rank:
                    self.lib.sk_ipc_close(C.c_void_p(b))
            self._free_own()
            raise PeerUnavailable(errs[0])

    def _free_own(self):
        if self.own is not None:
            self.lib.sk_ipc_free(C.c_void_p(self.own))
            self.own = None

    def buf(self, p: int, j: int) -> int:
        return self.base[p] + self.off_buf[j]

    def mail(self, p: int) -> int:
        return self.base[p] + self.off_mail

    def flags(self, p: int) -> int:
        return self.base[p] + self.off_flag

    def close(self) -> None:
        """Collective: no rank may still write into a region being freed."""
        if self.own is None:
            return
        _dist().barrier(group=self.group)
        for p, b in enumerate(self.base):
            if p != self.rank:
                N.check(self.lib.sk_ipc_close(C.c_void_p(b)))
        N.check(self.lib.sk_ipc_free(C.c_void_p(self.own)))
        self.own = None


def _all_objects(obj, group=None):
    dist = _dist()
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


class DeviceBlock:
    """One rank's Helmholtz row block on its GPU, driven through the C-ABI.

    u0 / f: [rows, cols] device tensors of this rank's owned rows (fp32 or
    fp64).  The initial halo rows are exchanged at construction.

    transport: "collective" -- halo rows by send/recv and the partials by an
    all-gather over the process group (NCCL, or gloo staged through the
    host); "peer" -- the sweep kernel itself stores its boundary rows into
    the neighbours' halo rows and publishes its partial and a flag into
    every rank's mailbox (PeerRegion), the stream waits on the flags with
    no SM involvement, then the rank-ordered combine runs (no collective
    library on the iteration path; ranks on one node).
    """

    def __init__(self, u0, f, consts, *, rank: int, world: int, reduce: str = "max",
                 delta: str = "abs", identity: float = 0.0, timing: bool = False, group=None,
                 transport: str = "collective"):
        import torch

        if transport not in ("collective", "peer"):
            raise ValueError(f"unknown transport {transport!r}")
        if transport == "peer" and not 2 <= world <= N.SK_MAX_PEERS:
            transport = "collective"  # one rank: nothing to exchange
        lib = N.require_cuda()
        self.lib, self.rank, self.world, self.group = lib, rank, world, group
        self.transport = transport
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
        self.region = None
        if transport == "peer":
            es = u0.element_size()
            shapes = [v[0] for v in _all_ints([rows], group)]  # every rank's owned rows
            Rmax = max(shapes) + 2
            try:
                self.region = PeerRegion(Rmax * pitch * es, rank, world, group)
            except PeerUnavailable:
                transport = self.transport = "collective"  # every rank falls back together
        if transport == "peer":
            typestr = "<f4" if dt == torch.float32 else "<f8"
            self.bufs = [torch.as_tensor(_DevPtr(self.region.buf(rank, j), R * pitch, typestr),
                                         device=dev).view(R, pitch) for j in range(2)]
            pe = N.sk_peers()
            pe.rank, pe.world = rank, world
            for j in range(2):
                if rank > 0:  # rank-1's bottom halo row: after its ht + rows rows
                    ht_up = 1 if rank - 1 > 0 else 0
                    pe.up_rows[j] = self.region.buf(rank - 1, j) + (ht_up + shapes[rank - 1]) * pitch * es
                if rank < world - 1:  # rank+1's top halo row is its row 0
                    pe.down_rows[j] = self.region.buf(rank + 1, j)
            for p in range(world):
                pe.mail[p] = self.region.mail(p)
                pe.flags[p] = self.region.flags(p)
            self._peers = pe
        else:
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
        if transport == "peer":
            N.check(lib.sk_run_set_peers(h, C.byref(self._peers)))
            # every rank's buffers exist and are zeroed before anyone's first
            # sweep stores into them
            torch.cuda.synchronize()
            _dist().barrier(group=group)

    def buffer_of(self, t: int):
        return self.bufs[t & 1]

    def step(self, cond: "N.sk_cond") -> None:
        """Enqueue one iteration: sweep -> halo exchange -> gather -> combine
        (peer transport: sweep with fused halo/partial stores -> stream wait
        on the peers' flags -> combine)."""
        N.check(self.lib.sk_run_launch(self.h, 1))
        self.launched += 1
        if self.transport == "peer":
            q = self.launched
            N.check(self.lib.sk_run_peer_wait(self.h, q))
            row = self.region.mail(self.rank) + (q & 1) * self.world * 8
            N.check(self.lib.sk_run_combine(self.h, C.c_void_p(row), self.world, C.byref(cond)))
            return
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
        """Collective when the peer transport is on (the region is freed
        only after every rank's last sweep)."""
        if self.h is not None:
            N.check(self.lib.sk_run_destroy(self.h))
            self.h = None
        if self.region is not None:
            self.bufs = None
            self.region.close()
            self.region = None


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


# ---------------------------------------------------------------- any elemental


def _all_ints(vals, group=None):
    """All-gather small ints on any backend (host round trip)."""
    import torch

    dist = _dist()
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    mine = torch.tensor(vals, dtype=torch.int64, device=dev)
    out = [torch.zeros_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, mine, group=group)
    return [t.tolist() for t in out]


def block_loop(f, k, op, cond, block, *, env=None, delta=None, indexed: bool = False,
               rank: int, world: int, group=None, max_iterations=None, batch: int = 4):
    """parallel_loop over a grid split across ranks: this rank holds `block`,
    its contiguous rows of the global grid (ranks in row order), and `env`,
    the same rows of each env grid.  Any elemental function -- a built-in
    Helmholtz kernel or a user function compiled for the device (jit.py) --
    with a recognised sum / max combinator.  Per iteration: the sweep on the
    block (k-deep halo rows in its buffers), the k boundary rows to each
    neighbour (NCCL / gloo), the partials all-gathered and folded in rank
    order on the device, the loop condition evaluated there (or, for a
    Python condition, on the host from that same value on every rank).
    Returns (this rank's owned rows as a device Grid, LoopReport)."""
    import torch

    from .grid import Grid
    from .jit import JitKernel, build_program
    from .loop import LoopReport, _as_plan, as_condition
    from .partition import _TORCH_DT, model_ledger
    from .patterns import DeviceUnsupported, StencilError, _check_env, combinator_kind

    lib = N.require_cuda()
    dist = _dist()
    block = block if isinstance(block, Grid) else Grid.from_tensor(block)
    if block.ndim != 2:
        raise DeviceUnsupported("rank blocks are 2D row blocks")
    rows, cols = block.dims
    plan = _as_plan(f, k, op, env, indexed=indexed, delta=delta)
    k = plan.k
    _check_env(plan.env, block.dims)
    counts = [c[0] for c in _all_ints([rows], group)]
    if any(c < max(k, 1) for c in counts) and world > 1:
        raise ValueError(f"every rank needs at least {max(k, 1)} rows, got {counts}")
    row0, grows = sum(counts[:rank]), sum(counts)
    cond = as_condition(cond, max_iterations)
    reduce = combinator_kind(plan.op)  # sum / max: the device's cross-rank fold
    dk = getattr(plan.fn, "device", None)
    if dk is not None and not isinstance(dk, JitKernel):
        raise DeviceUnsupported("block_loop runs compiled elementals; use DeviceBlock for "
                                "the Helmholtz kernel")
    prog = build_program(plan, block, dims=(grows, cols))
    dev = torch.device("cuda", torch.cuda.current_device())
    ht = k if rank > 0 else 0
    hb = k if rank < world - 1 else 0
    R = ht + rows + hb

    def with_halos(g, dtype):
        t = g.tensor(device=dev)
        if t.dtype != _TORCH_DT[dtype]:
            t = t.to(_TORCH_DT[dtype])
        buf = torch.zeros((R, cols), dtype=t.dtype, device=dev)
        buf[ht:ht + rows] = t.reshape(rows, cols)
        exchange_halos(buf, rank, world, ht, rows, group, k=k) if k else None
        return buf

    src = with_halos(block, prog.in_dtype)
    env_grids = plan.env if isinstance(plan.env, tuple) else (
        (plan.env,) if isinstance(plan.env, Grid) else ())
    envs = [with_halos(g, d) for g, d in zip(env_grids, prog.env_dtypes)]
    bufs = [torch.zeros((R, cols), dtype=_TORCH_DT[prog.out_dtype], device=dev) for _ in range(2)]
    p = N.sk_plan()
    p.kernel, p.dtype = N.SK_KERNEL_JIT, 0
    p.rows, p.cols, p.partitions = rows, cols, 1
    p.reduce_op, p.delta_op = prog.reduce, N.SK_DELTA_NONE
    p.halo_top, p.halo_bottom = ht, hb
    p.identity = float(plan.op.identity)
    p.params[0], p.params[1], p.params[2] = float(prog.tile_rows), float(row0), float(grows)
    n = len(envs)
    eptr = (C.c_void_p * 4)(*[C.c_void_p(t[ht].data_ptr()) for t in envs])
    epitch = (C.c_int64 * 4)(*[t.stride(0) for t in envs])
    h = C.c_void_p()
    N.check(lib.sk_run_begin_jit(C.byref(p), prog.handle, C.c_void_p(src.data_ptr()), cols,
                                 eptr, epitch, n, C.c_void_p(bufs[0].data_ptr()),
                                 C.c_void_p(bufs[1].data_ptr()), cols,
                                 N.stream_handle(torch.cuda.current_stream()), C.byref(h)))
    try:
        vp = C.c_void_p()
        N.check(lib.sk_run_value_ptr(h, C.byref(vp)))
        partial = torch.as_tensor(_DevPtr(vp.value, 1), device=dev)
        gathered = torch.zeros(world, dtype=torch.float64, device=dev)
        dc = cond.device
        c = N.sk_cond()
        if dc is not None:
            c.kind = {"lt": N.SK_COND_LT, "rms_lt": N.SK_COND_RMS_LT, "mean_lt": N.SK_COND_MEAN_LT,
                      "iter_ge": N.SK_COND_ITER_GE}[dc.kind]
            c.a, c.n = dc.a, dc.n
        else:
            c.kind = N.SK_COND_HOST
        c.max_iterations = cond.max_iterations
        launched = 0
        step_batch = batch if dc is not None else 1

        def status():
            it, val, stp, ex = C.c_int64(), C.c_double(), C.c_int32(), C.c_int32()
            N.check(lib.sk_run_status(h, C.byref(it), C.byref(val), C.byref(stp), C.byref(ex)))
            code, index, eit = C.c_int32(), C.c_int64(), C.c_int64()
            N.check(lib.sk_run_error(h, C.byref(code), C.byref(index), C.byref(eit)))
            return it.value, val.value, bool(stp.value), bool(ex.value), code.value, index.value

        while True:
            for _ in range(step_batch):
                N.check(lib.sk_run_launch(h, 1))
                launched += 1
                if k:
                    exchange_halos(bufs[launched & 1], rank, world, ht, rows, group, k=k)
                gather_partials(partial, gathered, group)
                N.check(lib.sk_run_combine(h, C.c_void_p(gathered.data_ptr()), world, C.byref(c)))
            it, val, stopped, ex, code, index = status()
            host_stop = False
            if dc is None and not stopped and code == 0:
                host_stop = bool(cond.fn(val, it, None))
            # one decision for every rank: stop if any rank stopped or failed
            flags = _all_ints([int(stopped or host_stop), int(code != 0), int(ex)], group)
            if any(fl[1] for fl in flags):
                if code:
                    from .jit import error_cause

                    i, j = divmod(index, cols)
                    raise StencilError((i, j), error_cause(code), partition=rank)
                raise StencilError(None, RuntimeError("an elemental failed on another rank"),
                                   partition=rank)
            if all(fl[0] for fl in flags) or it >= cond.max_iterations:
                exhausted = not (stopped and not ex) and not host_stop
                break
        which = bufs[it & 1]
        out = Grid.from_tensor(which[ht:ht + rows].contiguous(), logical_dtype=prog.out_dtype)
        value = int(val) if prog.int_value else val
        rep = LoopReport(iterations=it, final_reduce=value,
                         copies=model_ledger((grows, cols), world, k, it), exhausted=exhausted)
        return out, rep
    finally:
        N.check(lib.sk_run_destroy(h))
