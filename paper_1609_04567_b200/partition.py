"""Partitioned loop runtime on the GPU (reference: partition.py:1-692).

Public surface mirrors the reference: DeploymentMode, WorkerGroup,
parallel_loop, partition/_split_ranges geometry, PartitionSet, halo_exchange,
parallel_step -- plus `DeviceExecutor`, the Executor-protocol implementation
(loop.py:124-137) over the native engine (include/stencilkit_b200.h).

Mapping of the reference's model onto one GPU:
  * partitions  -> contiguous row blocks exactly as _split_ranges
                   (partition.py:187-195).  On one device the blocks share one
                   pair of iteration buffers, so a "halo exchange" is a read of
                   the neighbour's rows in place; the engine keeps the
                   per-partition reduce structure (CTA work chunks never span
                   a partition; partials are folded per partition, then in
                   ascending partition order from the identity,
                   partition.py:642-646).  The CopyLedger reports the
                   reference's traffic model from the committed iteration
                   count (fill/readback per partition, 2*k*d2 per boundary per
                   exchanged iteration, none after the last).
  * WorkerGroup -> a reusable device context: one CUDA stream, one active run
                   at a time, size = partitions it serves (partition.py:451-532).
  * multi-GPU   -> one process per GPU (see distributed.py): each rank owns one
                   row block with real halo rows moved over NCCL/NVLink.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from enum import Enum
from typing import Any, Optional

import numpy as np

from . import _native as N
from .grid import Grid, GridError
from .ledger import CopyLedger
from .loop import Executor, LoopPlan, LoopState, _as_plan, _drive
from .jit import JitKernel, build_program
from .patterns import (Combinator, DeviceUnsupported, StencilError, _check_env, combinator_kind,
                       delta_kind)


class DeploymentMode(Enum):
    """ONE_TO_ONE: each loop on one partition; ONE_TO_N: split across P >= 2
    partitions (partition.py:39-57)."""

    ONE_TO_ONE = "1:1"
    ONE_TO_N = "1:n"

    @classmethod
    def parse(cls, text) -> "DeploymentMode":
        if isinstance(text, cls):
            return text
        for m in cls:
            if m.value == text:
                return m
        raise GridError(f"unknown deployment mode {text!r} (expected 1:1 or 1:n)")


def _split_ranges(d1: int, P: int) -> list:
    """Row ranges, remainder to the lowest partitions (partition.py:187-195)."""
    base, rem = divmod(d1, P)
    out, b = [], 0
    for i in range(P):
        s = base + (1 if i < rem else 0)
        out.append((b, b + s))
        b += s
    return out


def _check_partitioning(d1: int, P: int, k: int) -> None:
    """Preconditions of partition() (partition.py:205-215)."""
    if P < 1:
        raise GridError(f"partition count must be >= 1, got {P}")
    if k < 0:
        raise GridError(f"halo depth must be >= 0, got {k}")
    if d1 < P:
        raise GridError(f"cannot split {d1} rows across {P} partitions")
    if P > 1 and d1 // P < k:
        raise GridError(f"partitions of {d1} rows across {P} are shallower than halo depth {k}")


def model_ledger(dims, P: int, k: int, iterations: int) -> CopyLedger:
    """The reference's copy-traffic model for a committed run (partition.py:
    225-262, 170-184; halo skipped after the final iteration, :629-635)."""
    led = CopyLedger()
    width = dims[1] if len(dims) == 2 else 1
    for lo, hi in _split_ranges(dims[0], P):
        led.record_fill((hi - lo) * width)
    if k > 0 and P > 1:
        for _ in range(max(iterations - 1, 0)):
            for _b in range(P - 1):
                led.record_halo(2 * k * width, 2)
    for lo, hi in _split_ranges(dims[0], P):
        led.record_readback((hi - lo) * width)
    return led


# ---------------------------------------------------------------- partition sets
# The reference's host-side building blocks (partition.py:60-262, 415-432):
# split a grid into row partitions with k-deep halos, exchange halos, run one
# step per partition, gather.  Here every partition buffer lives in device
# memory; rows read and write as Python lists like the reference's list
# storage, so code poking at `part.front[i]` keeps working.


class DeviceRows:
    """A partition buffer (rows incl. halos) in device memory, indexed by
    local row: `rows[i]` -> list (scalar for 1D), `rows[i] = list`."""

    def __init__(self, t):
        self.t = t

    def __len__(self):
        return int(self.t.shape[0])

    def __getitem__(self, i):
        v = self.t[i]
        return v.tolist()

    def __setitem__(self, i, value):
        torch = _torch()
        self.t[i] = torch.as_tensor(value, dtype=self.t.dtype, device=self.t.device)

    def __iter__(self):
        return iter(self.t.tolist())

    def __eq__(self, other):
        if isinstance(other, DeviceRows):
            other = other.t.tolist()
        return self.t.tolist() == list(other)

    __hash__ = None

    def __repr__(self):
        return f"DeviceRows({tuple(self.t.shape)}, {self.t.dtype})"


def _as_rows(buf, like) -> "DeviceRows":
    """Whatever a caller stored in front/back (DeviceRows, tensor, lists) as
    device rows shaped like `like`."""
    if isinstance(buf, DeviceRows):
        return buf
    torch = _torch()
    if torch.is_tensor(buf):
        return DeviceRows(buf)
    return DeviceRows(torch.as_tensor(buf, dtype=like.t.dtype, device=like.t.device))


class Partition:
    """One partition: owned rows [r_begin, r_end) plus k-deep halos, double
    buffered in device memory (partition.py:76-148)."""

    def __init__(self, index, r_begin, r_end, top_halo, bottom_halo, width):
        self.index = index
        self.r_begin, self.r_end = r_begin, r_end
        self.top_halo, self.bottom_halo = top_halo, bottom_halo
        self.width = width  # None for 1D grids
        self.front = None
        self.back = None

    @property
    def rows(self) -> int:
        return self.r_end - self.r_begin

    @property
    def owned_elems(self) -> int:
        return self.rows * (self.width or 1)

    def _t(self, which):
        b = _as_rows(self.front if which == "front" else self.back, self.front)
        if which == "front":
            self.front = b
        else:
            self.back = b
        return b.t

    def owned_view(self, which):
        return self._t(which)[self.top_halo:self.top_halo + self.rows]

    def owned_head(self, which, k):
        lo = self.top_halo
        return self._t(which)[lo:lo + k].clone()

    def owned_tail(self, which, k):
        hi = self.top_halo + self.rows
        return self._t(which)[hi - k:hi].clone()

    def set_top_halo(self, which, rows) -> None:
        self._t(which)[0:self.top_halo] = rows

    def set_bottom_halo(self, which, rows) -> None:
        lo = self.top_halo + self.rows
        self._t(which)[lo:lo + self.bottom_halo] = rows

    def swap(self) -> None:
        self.front, self.back = self.back, self.front


class PartitionSet:
    """All partitions of one grid plus the copy ledger (partition.py:151-184)."""

    def __init__(self, dims, k, parts, storage):
        self.dims = tuple(dims)
        self.k = k
        self.parts = parts
        self.storage = storage
        self.ledger = CopyLedger()

    @property
    def buffer_allocations(self) -> int:
        return 2 * len(self.parts)  # front + back per partition (partition.py:160)

    @property
    def P(self) -> int:
        return len(self.parts)

    def swap_all(self) -> None:
        for p in self.parts:
            p.swap()

    def gather(self, which: str = "back") -> Grid:
        """The owned rows back as one (device) grid; one readback per partition."""
        torch = _torch()
        pieces = []
        for p in self.parts:
            pieces.append(p.owned_view(which))
            self.ledger.record_readback(p.owned_elems)
        return Grid.from_tensor(torch.cat(pieces).reshape(self.dims).contiguous())


def partition(a: Grid, P: int, k: int, storage: str = "list") -> PartitionSet:
    """Split into P row partitions with k-deep halos and load them into device
    memory (one fill per partition; partition.py:198-244).  `storage` is kept
    for the signature: the buffers are device tensors either way."""
    torch = _torch()
    N.require_cuda()
    _check_partitioning(a.dims[0], P, k)
    width = a.dims[1] if a.ndim == 2 else None
    full = a.tensor(device=torch.device("cuda", torch.cuda.current_device()))
    parts = []
    ranges = _split_ranges(a.dims[0], P)
    ps = PartitionSet(a.dims, k, parts, storage)
    for i, (lo, hi) in enumerate(ranges):
        p = Partition(i, lo, hi, k if i > 0 else 0, k if i < P - 1 else 0, width)
        p.front = DeviceRows(full[lo - p.top_halo:hi + p.bottom_halo].clone())
        p.back = DeviceRows(torch.empty_like(p.front.t))
        parts.append(p)
        ps.ledger.record_fill(p.owned_elems)
    return ps


def halo_exchange(ps: PartitionSet, which: str = "front") -> None:
    """Refresh every halo from the neighbouring partition's owned rows, device
    to device; 2*k*width elements and two events per boundary
    (partition.py:247-262)."""
    k = ps.k
    if k == 0 or ps.P == 1:
        return
    per_row = ps.parts[0].width or 1
    for a, b in zip(ps.parts, ps.parts[1:]):
        b.set_top_halo(which, a.owned_tail(which, k))
        a.set_bottom_halo(which, b.owned_head(which, k))
        ps.ledger.record_halo(2 * k * per_row, 2)


def parallel_step(ps: PartitionSet, f, k, op: Combinator, env: Any = None):
    """One stencil step over every partition plus the combined reduce
    (partition.py:415-432): each partition's buffer (owned rows + halos) is
    swept on the device, its owned outputs land in the back buffer, its
    partial is the device reduce of those outputs; the partials are folded
    in ascending partition order from the identity, on the host as in the
    reference."""
    from .loop import loop_stencil_reduce, stop_after
    from .patterns import _radius, reduce_all

    kk = _radius(f, k)
    if kk != ps.k:
        raise GridError(f"stencil radius {kk} does not match halo depth {ps.k}")
    _check_env(env, ps.dims)
    partials = []
    for p in ps.parts:
        buf = _as_rows(p.front, p.front).t
        lo, hi = p.r_begin - p.top_halo, p.r_end + p.bottom_halo
        penv = _slice_env(env, lo, hi)
        out, _ = loop_stencil_reduce(kk, f, op, stop_after(1), Grid.from_tensor(buf), env=penv)
        owned = out.tensor()[p.top_halo:p.top_halo + p.rows]
        if p.back is None or not isinstance(p.back, DeviceRows) or p.back.t.dtype != owned.dtype:
            p.back = DeviceRows(_torch().empty((hi - lo,) + tuple(owned.shape[1:]),
                                               dtype=owned.dtype, device=owned.device))
        p.back.t[p.top_halo:p.top_halo + p.rows] = owned
        partials.append(reduce_all(op, Grid.from_tensor(owned.contiguous())))
    combined = op.identity
    for v in partials:
        combined = op.fn(combined, v)
    return partials, combined


def _slice_env(env, lo, hi):
    if env is None:
        return None
    if isinstance(env, Grid):
        return Grid.from_tensor(env.tensor(device="cuda")[lo:hi])
    if isinstance(env, tuple):
        return tuple(_slice_env(e, lo, hi) if isinstance(e, Grid) else e for e in env)
    return env


# ---------------------------------------------------------------- worker group


class WorkerGroup:
    """Reusable device context for loop runs (partition.py:451-532).

    Owns one CUDA stream; serves one run at a time; `size` is the partition
    count of the runs it serves.  Stream-farm replicas keep one each so their
    runs overlap on the GPU.
    """

    def __init__(self, size: int, device: Optional[int] = None):
        if size < 1:
            raise ValueError(f"worker group size must be >= 1, got {size}")
        self.size = size
        self.device = device
        self._stream = None
        self._busy = False
        self._closed = False
        self._lock = threading.Lock()

    @property
    def stream(self):
        if self._stream is None:
            import torch

            dev = self.device if self.device is not None else torch.cuda.current_device()
            self._stream = torch.cuda.Stream(device=dev)
        return self._stream

    def start_run(self) -> None:
        with self._lock:
            if self._closed:
                raise RuntimeError("worker group is closed")
            if self._busy:
                raise RuntimeError("worker group already has an active run")
            self._busy = True

    def end_run(self) -> None:
        with self._lock:
            self._busy = False

    def close(self) -> None:
        with self._lock:
            if self._closed:
                return
            if self._busy:
                raise RuntimeError("cannot close a worker group with an active run")
            self._closed = True
            if self._stream is not None:
                self._stream.synchronize()

    def __enter__(self) -> "WorkerGroup":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


# ---------------------------------------------------------------- executor

_KERNEL_IDS = {"helmholtz": N.SK_KERNEL_HELMHOLTZ, "sobel": N.SK_KERNEL_SOBEL,
               "amf": N.SK_KERNEL_AMF, "restore": N.SK_KERNEL_RESTORE,
               "life": N.SK_KERNEL_LIFE}
_REDUCE = {"sum": N.SK_REDUCE_SUM, "max": N.SK_REDUCE_MAX}
_DELTA = {"none": N.SK_DELTA_NONE, "abs": N.SK_DELTA_ABS, "square": N.SK_DELTA_SQUARE}
_COND = {"lt": N.SK_COND_LT, "rms_lt": N.SK_COND_RMS_LT, "mean_lt": N.SK_COND_MEAN_LT,
         "iter_ge": N.SK_COND_ITER_GE, "mean_flagged_lt": N.SK_COND_MEAN_FLAGGED_LT}
# value range every output pixel of a u8 kernel lies in (tags the result grid
# so the next device stage can skip re-validating it)
_OUT_RANGE = {"sobel": (0, 255), "amf": (0, 1), "life": (0, 1)}


def _torch():
    import torch

    return torch


class _TorchDtypes(dict):
    def __missing__(self, key):
        torch = _torch()
        table = {np.dtype(np.bool_): torch.bool, np.dtype(np.int8): torch.int8,
                 np.dtype(np.uint8): torch.uint8, np.dtype(np.int16): torch.int16,
                 np.dtype(np.uint16): torch.uint16, np.dtype(np.int32): torch.int32,
                 np.dtype(np.uint32): torch.uint32, np.dtype(np.int64): torch.int64,
                 np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}
        self.update(table)
        return table[np.dtype(key)]


_TORCH_DT = _TorchDtypes()


@dataclass
class _DevRun:
    plan: LoopPlan
    dims: tuple
    P: int
    handle: Any
    bufs: list
    src: Any
    env: Any
    pitch: int
    cols: int
    out_dtype: Any        # numpy logical dtype of the result grid
    int_value: bool       # reduce value reported as int
    stream: Any
    group: Optional[WorkerGroup]
    owns_group: bool
    steps: int = 0        # committed (host-observed) iterations
    launched: int = 0     # iterations enqueued on the device
    committed: Optional[int] = None
    released: bool = False
    jit: Any = None       # jit.Program of a user elemental


def _u8_from(grid: Grid, what: str, lo: int, hi: int, dev):
    """Integer image -> device uint8 tensor, values checked in [lo, hi].

    Host grids are checked and narrowed to uint8 on the host (1 byte per
    pixel crosses PCIe); device grids tagged with a known value range by the
    kernel that produced them skip the check (no host synchronisation)."""
    torch = _torch()
    sd = grid.storage_dtype()
    if sd.kind not in "iub":
        raise GridError(f"{what} expects integer pixels, got dtype {sd}")
    rng = grid.value_range
    known = rng is not None and rng[0] >= lo and rng[1] <= hi
    if getattr(grid, "_pending", None) is not None:  # a prefetched upload
        t = grid.tensor(device=dev)
        if t.dtype == torch.uint8 and hi >= 255:
            return t
    t0 = grid._t if grid._src == "t" else None
    if t0 is not None and not t0.is_cuda and t0.dtype == torch.uint8 and hi >= 255:
        # a uint8 host tensor needs no range check; from pinned memory the
        # upload is asynchronous on the current stream
        return t0.to(dev, non_blocking=t0.is_pinned())
    if not grid.is_device:
        a = grid._host()
        if not known and sd != np.uint8 or (sd == np.uint8 and hi < 255 and not known):
            mn, mx = (int(a.min()), int(a.max())) if a.size else (lo, lo)
            if mn < lo or mx > hi:
                raise GridError(
                    f"{what}: pixel values must lie in [{lo}, {hi}], found [{mn}, {mx}]")
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).to(dev)
    t = grid.tensor(device=dev)
    if not known and (t.dtype != torch.uint8 or hi < 255):
        mn, mx = int(t.min().item()), int(t.max().item())
        if mn < lo or mx > hi:
            raise GridError(f"{what}: pixel values must lie in [{lo}, {hi}], found [{mn}, {mx}]")
    return t if t.dtype == torch.uint8 else t.to(torch.uint8)


def _our_grid(g):
    if g is None or isinstance(g, Grid):
        return g
    if hasattr(g, "dims") and hasattr(g, "data"):  # the reference's list-backed Grid
        return Grid(g.dims, g.data)
    if isinstance(g, tuple):
        return tuple(_our_grid(x) for x in g)
    return g


def _adapt(plan, grid):
    """Accept the reference package's own LoopPlan/Grid objects (when this
    executor is passed to stencilkit's loop_stencil_reduce*): its _as_plan
    wraps our ElementalFn as the `point` of its own ElementalFn."""
    fn = plan.fn
    if getattr(fn, "device", None) is None and getattr(getattr(fn, "point", None), "device", None):
        fn = fn.point
    env = _our_grid(plan.env)
    if fn is not plan.fn or env is not plan.env or not isinstance(plan, LoopPlan):
        plan = LoopPlan(fn=fn, k=plan.k, op=plan.op, env=env, indexed=plan.indexed,
                        delta=plan.delta)
    return plan, _our_grid(grid)


class DeviceExecutor(Executor):
    """Executor over the native engine: `partitions` row partitions on one GPU."""

    device_loop = True

    def __init__(self, partitions: int = 1, group: Optional[WorkerGroup] = None,
                 timing: bool = False):
        if group is not None and group.size != partitions:
            raise ValueError(
                f"worker group size {group.size} does not match partitions {partitions}")
        self.partitions = partitions
        self._group = group
        self.timing = timing
        self.last_kernel_time = None
        self.launches = 0  # native sweep launches over this executor's runs

    # -- begin -----------------------------------------------------------
    def begin(self, plan: LoopPlan, grid: Grid) -> _DevRun:
        lib = N.require_cuda()
        torch = _torch()
        plan, grid = _adapt(plan, grid)
        _check_env(plan.env, grid.dims)
        dk = plan.fn.device if hasattr(plan.fn, "device") else None
        jit_fn = dk is None or isinstance(dk, JitKernel)
        if grid.ndim == 1 and jit_fn:
            rows, cols = grid.dims[0], 1  # a rank-1 grid runs as an (n, 1) column
        elif grid.ndim != 2:
            raise DeviceUnsupported("the built-in device kernels run on 2D grids")
        else:
            rows, cols = grid.dims
        P = self.partitions
        _check_partitioning(rows, P, plan.k)
        prog = None
        if jit_fn:
            # a user elemental: compiled for the device at run time (jit.py);
            # raises DeviceUnsupported if it cannot be translated
            prog = build_program(plan, grid)
            reduce = delta = None
        else:
            reduce = combinator_kind(plan.op)
            delta = delta_kind(plan.delta)
        group = self._group
        owns = group is None
        cur = torch.cuda.current_stream()
        stream = group.stream if group is not None else cur
        if group is not None:
            # the run's stream starts after whatever the caller enqueued on
            # its current stream (e.g. a non-blocking upload of the inputs)
            stream.wait_stream(cur)
            group.start_run()
        try:
            if stream == cur:  # (the stream context costs several us per loop)
                if prog is not None:
                    return self._begin_jit(lib, plan, grid, prog, rows, cols, P, stream, group, owns)
                return self._begin_on(lib, plan, grid, dk, rows, cols, P, reduce, delta,
                                      stream, group, owns)
            with torch.cuda.stream(stream):
                if prog is not None:
                    return self._begin_jit(lib, plan, grid, prog, rows, cols, P, stream, group, owns)
                return self._begin_on(lib, plan, grid, dk, rows, cols, P, reduce, delta,
                                      stream, group, owns)
        except BaseException:
            if group is not None:
                group.end_run()
            raise

    def _begin_jit(self, lib, plan, grid, prog, rows, cols, P, stream, group, owns):
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device())
        tin = _TORCH_DT[prog.in_dtype]
        src = grid.tensor(device=dev)
        if src.dtype != tin:
            src = src.to(tin)
        src = src.reshape(rows, cols).contiguous()
        env_grids = plan.env if isinstance(plan.env, tuple) else (
            (plan.env,) if isinstance(plan.env, Grid) else ())
        envs = []
        for g, edt in zip(env_grids, prog.env_dtypes):
            t = g.tensor(device=dev)
            if t.dtype != _TORCH_DT[edt]:
                t = t.to(_TORCH_DT[edt])
            envs.append(t.reshape(rows, cols).contiguous())
        tout = _TORCH_DT[prog.out_dtype]
        bufs = [torch.empty((rows, cols), dtype=tout, device=dev) for _ in range(2)]
        p = N.sk_plan()
        p.kernel = N.SK_KERNEL_JIT
        p.dtype = 0
        p.rows, p.cols = rows, cols
        p.partitions = P
        p.reduce_op = prog.reduce
        p.delta_op = N.SK_DELTA_NONE
        p.halo_top = p.halo_bottom = 0
        p.flags = N.SK_FLAG_TIMING if self.timing else 0
        ident = plan.op.identity
        p.identity = float(ident) if isinstance(ident, (int, float, bool, np.number)) else 0.0
        p.params[0] = float(prog.tile_rows)  # the program's SK_TH (rows per work tile)
        p.params[3] = 1.0 if grid.ndim == 1 else 0.0  # rank 1: contiguous element tiles
        n = len(envs)
        eptr = (C.c_void_p * 4)(*[C.c_void_p(t.data_ptr()) for t in envs])
        epitch = (C.c_int64 * 4)(*[t.stride(0) for t in envs])
        h = C.c_void_p()
        N.check(lib.sk_run_begin_jit(C.byref(p), prog.handle, C.c_void_p(src.data_ptr()),
                                     src.stride(0), eptr, epitch, n,
                                     C.c_void_p(bufs[0].data_ptr()), C.c_void_p(bufs[1].data_ptr()),
                                     cols, N.stream_handle(stream), C.byref(h)))
        return _DevRun(plan=plan, dims=tuple(grid.dims), P=P, handle=h, bufs=bufs, src=src,
                       env=envs, pitch=cols, cols=cols, out_dtype=prog.out_dtype,
                       int_value=prog.int_value, stream=stream, group=group, owns_group=owns,
                       jit=prog)

    def _raise_if_failed(self, run: "_DevRun", upto: Optional[int] = None) -> None:
        """A recorded elemental failure becomes the reference's StencilError
        (partition.py:357-360, 638-641) for the lowest failing index."""
        if run.jit is None:
            return
        lib = N.load()
        code, index, it = C.c_int32(), C.c_int64(), C.c_int64()
        N.check(lib.sk_run_error(run.handle, C.byref(code), C.byref(index), C.byref(it)))
        if code.value == 0 or (upto is not None and it.value > upto):
            return
        from .jit import error_cause

        i, j = divmod(index.value, run.cols)
        where = (i,) if len(run.dims) == 1 else (i, j)
        part = None
        if run.P > 1:
            for pi, (lo, hi) in enumerate(_split_ranges(run.dims[0], run.P)):
                if lo <= i < hi:
                    part = pi
        raise StencilError(where, error_cause(code.value), partition=part)

    def _begin_on(self, lib, plan, grid, dk, rows, cols, P, reduce, delta, stream, group, owns):
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device())
        name = dk.name
        env_t = None
        int_value = False
        if name == "helmholtz":
            sd = grid.storage_dtype()
            if sd not in (np.float32, np.float64):
                raise DeviceUnsupported(f"helmholtz runs on float32/float64 grids, got {sd}")
            dtype = N.SK_F32 if sd == np.float32 else N.SK_F64
            tdt = torch.float32 if sd == np.float32 else torch.float64
            src = grid.tensor(device=dev)
            if src.dtype != tdt:
                src = src.to(tdt)
            if plan.env is None or not isinstance(plan.env, Grid):
                raise GridError("helmholtz needs the right-hand side grid as env")
            ed = plan.env.storage_dtype()
            if ed != sd:
                raise DeviceUnsupported(
                    f"env dtype {ed} differs from grid dtype {sd}: the reference would mix "
                    "precisions; pass both grids in the same dtype")
            env_t = plan.env.tensor(device=dev)
            out_dtype = sd
        elif name in ("sobel", "amf", "life"):
            hi = 1 if name == "life" else 255
            src = _u8_from(grid, name, 0, hi, dev)
            dtype = N.SK_U8
            out_dtype = np.dtype(np.int64)
            int_value = True
            if delta != "none":
                raise DeviceUnsupported(f"{name}: delta reduces are not supported")
        elif name == "restore":
            sd = grid.storage_dtype()
            if sd.kind not in "fiu":
                raise DeviceUnsupported(f"restore needs a numeric grid, got {sd}")
            src = grid.tensor(device=dev)
            if src.dtype != torch.float64:
                src = src.to(torch.float64)
            if plan.env is None or not isinstance(plan.env, Grid):
                raise GridError("restore needs the noise map grid as env")
            env_t = _u8_from(plan.env, "noise map", 0, 1, dev)
            dtype = N.SK_F64
            out_dtype = np.dtype(np.float64)
        else:
            raise DeviceUnsupported(f"unknown device kernel {name!r}")

        esize = src.element_size()
        # row pitch: whole 16-byte vectors, and whole 4-element thread vectors
        # for the Helmholtz sweep (fp64 threads load 2 x 16 B)
        vec = max(16 // esize, 4) if name == "helmholtz" else 16 // esize
        pitch = -(-cols // vec) * vec
        staged = pitch != cols or src.data_ptr() % 16 != 0
        if staged:
            s2 = torch.zeros((rows, pitch), dtype=src.dtype, device=dev)
            s2[:, :cols] = src.reshape(rows, cols)
            src = s2
            bufs = [torch.zeros((rows, pitch), dtype=src.dtype, device=dev) for _ in range(2)]
        else:
            src = src.reshape(rows, cols)
            bufs = [torch.empty((rows, pitch), dtype=src.dtype, device=dev) for _ in range(2)]
        env_pitch = 0
        env_ptr = None
        if env_t is not None:
            ev = 16 // env_t.element_size()
            ep = -(-cols // ev) * ev
            if ep != cols or env_t.data_ptr() % 16 != 0:
                e2 = torch.zeros((rows, ep), dtype=env_t.dtype, device=dev)
                e2[:, :cols] = env_t.reshape(rows, cols)
                env_t = e2
            env_pitch = ep
            env_ptr = env_t.data_ptr()

        p = N.sk_plan()
        p.kernel = _KERNEL_IDS[name]
        p.dtype = dtype
        p.rows, p.cols = rows, cols
        p.partitions = P
        p.reduce_op = _REDUCE[reduce]
        p.delta_op = _DELTA[delta]
        p.halo_top = p.halo_bottom = 0
        p.flags = N.SK_FLAG_TIMING if self.timing else 0
        ident = plan.op.identity
        p.identity = float(ident) if ident is not None else 0.0
        for i, v in enumerate(dk.params[:8]):
            p.params[i] = float(v)
        h = C.c_void_p()
        N.check(lib.sk_run_begin(C.byref(p), C.c_void_p(src.data_ptr()), pitch if staged else cols,
                                 C.c_void_p(env_ptr), env_pitch,
                                 C.c_void_p(bufs[0].data_ptr()), C.c_void_p(bufs[1].data_ptr()),
                                 pitch, N.stream_handle(stream), C.byref(h)))
        return _DevRun(plan=plan, dims=(rows, cols), P=P, handle=h, bufs=bufs, src=src, env=env_t,
                       pitch=pitch, cols=cols, out_dtype=out_dtype, int_value=int_value,
                       stream=stream, group=group, owns_group=owns)

    # -- host-driven steps (generic Python condition / LoopState) ----------
    def step(self, run: _DevRun) -> Any:
        lib = N.load()
        t = run.steps + 1
        while run.launched < t + 1:  # keep one speculative iteration in flight (lag-1)
            N.check(lib.sk_run_launch(run.handle, 1))
            run.launched += 1
        v = C.c_double()
        N.check(lib.sk_run_value(run.handle, t, C.byref(v)))
        if run.jit is not None and v.value != v.value:  # NaN: maybe a failed iteration
            self._raise_if_failed(run, upto=t)
        run.steps = t
        return self._value(run, v.value)

    def _value(self, run: _DevRun, v: float):
        if run.int_value:
            return int(v)
        return v

    # -- whole loop on the device --------------------------------------------
    def run_loop(self, run: _DevRun, cond):
        lib = N.load()
        dc = cond.device
        c = N.sk_cond()
        c.kind = _COND[dc.kind]
        c.a = dc.a
        c.n = dc.n
        c.max_iterations = cond.max_iterations
        it, val, ex = C.c_int64(), C.c_double(), C.c_int32()
        N.check(lib.sk_run_loop(run.handle, C.byref(c), C.byref(it), C.byref(val), C.byref(ex)))
        self._raise_if_failed(run)
        run.steps = run.launched = it.value
        return it.value, self._value(run, val.value), bool(ex.value)

    # -- finish / abort ------------------------------------------------------
    def finish(self, run: _DevRun):
        lib = N.load()
        torch = _torch()
        it = run.steps
        which = C.c_int32()
        N.check(lib.sk_run_result(run.handle, it, C.byref(which)))
        nl = C.c_int64()
        N.check(lib.sk_run_launches(run.handle, C.byref(nl)))
        self.launches += nl.value
        if self.timing:
            ms, n = C.c_double(), C.c_int64()
            N.check(lib.sk_run_kernel_time(run.handle, C.byref(ms), C.byref(n)))
            self.last_kernel_time = (ms.value, n.value)
        buf = run.bufs[which.value] if which.value >= 0 else run.src
        self._release(run)
        out = buf[:, :run.cols]
        if run.pitch != run.cols:
            out = out.contiguous()
        if len(run.dims) == 1:
            out = out.reshape(run.dims)
        led = model_ledger(run.dims, run.P, run.plan.k, it)
        g = Grid.from_tensor(out, logical_dtype=run.out_dtype)
        g.value_range = _OUT_RANGE.get(getattr(getattr(run.plan.fn, "device", None), "name", None))
        return g, led

    def abort(self, run: _DevRun) -> None:
        self._release(run)

    def _release(self, run: _DevRun) -> None:
        if run.released:
            return
        run.released = True
        lib = N.load()
        rc = lib.sk_run_destroy(run.handle)
        if run.group is not None:
            run.group.end_run()
        N.check(rc)


class ParallelExecutor(DeviceExecutor):
    """The reference's partitioned executor (partition.py:596-664) by name:
    `partitions` row partitions on the GPU (a DeviceExecutor)."""

    def __init__(self, partitions: int, group: Optional[WorkerGroup] = None):
        super().__init__(partitions, group)


@dataclass(frozen=True)
class BlockInfo:
    """Geometry of a padded block handed to a numpy block kernel
    (partition.py:60-73): block[k + r, k + c] is global element (row0 + r, c);
    `valid` marks the block cells inside the grid.  Kept for code that builds
    or inspects block-kernel inputs; the device engine never calls numpy
    block forms."""

    row0: int
    rows: int
    cols: int
    dims: tuple
    k: int
    valid: Any


def parallel_loop(mode, partitions: int, k, f, op: Combinator, cond, a: Grid,
                  env: Any = None, *, delta=None, indexed: bool = False,
                  state: Optional[LoopState] = None,
                  group: Optional[WorkerGroup] = None,
                  max_iterations: Optional[int] = None):
    """Partitioned stencil-reduce loop (partition.py:667-692) on the GPU."""
    mode = DeploymentMode.parse(mode)
    if partitions < 1:
        raise GridError(f"partition count must be >= 1, got {partitions}")
    if mode is DeploymentMode.ONE_TO_N and partitions < 2:
        raise GridError("1:n deployment needs at least 2 partitions")
    eff = partitions if mode is DeploymentMode.ONE_TO_N else 1
    if group is not None and group.size != eff:
        raise GridError(f"worker group size {group.size} does not match {eff} partitions")
    plan = _as_plan(f, k, op, env, indexed=indexed, delta=delta)
    return _drive(plan, cond, state, a, DeviceExecutor(eff, group), max_iterations)
