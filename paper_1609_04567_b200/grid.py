"""Dense rank-1/2 grids, the ABSENT marker and window views.

Same public surface as the reference's grid module (grid.py:15-324): Grid,
GridError, ABSENT/is_absent, grid_new, grid_get_padded, Neighborhood,
IndexedNeighborhood, neighborhood_at, indexed_neighborhood_at.

The difference is storage.  The reference keeps a Python list (32 B per
element, grid.py:47-76); here a Grid holds a numpy array (host) or a torch
tensor (device, possibly the output buffer of a device run) and only builds
the Python list when `.data` is read.  A device-resident result therefore
costs nothing until someone looks at it, and `Grid.tensor()` hands it to
the next device run without a copy.
"""

from __future__ import annotations

from typing import Any, Iterator, Sequence

import os

import numpy as np


class GridError(ValueError):
    """Invalid grid construction or out-of-contract access (grid.py:15-16)."""


class _Absent:
    """Singleton for window slots outside the grid (grid.py:19-44)."""

    __slots__ = ()
    _one = None

    def __new__(cls):
        if cls._one is None:
            cls._one = super().__new__(cls)
        return cls._one

    def __repr__(self) -> str:
        return "ABSENT"

    def __bool__(self) -> bool:
        return False

    def __reduce__(self):
        return (_Absent, ())


ABSENT = _Absent()


def is_absent(value: Any) -> bool:
    return value is ABSENT


def _check_dims(dims) -> tuple:
    dims = tuple(int(d) for d in dims)
    if len(dims) not in (1, 2):
        raise GridError(f"grid rank must be 1 or 2, got {len(dims)}")
    if any(d <= 0 for d in dims):
        raise GridError(f"grid dims must be positive, got {dims}")
    return dims


def _torch():
    import torch

    return torch


class Grid:
    """Dense row-major grid of rank 1 or 2.

    Construct from any sequence (like the reference), a numpy array, or a
    torch tensor (`Grid.from_tensor`).  `logical_dtype` is the numpy dtype
    `to_array()` reports; device results of integer kernels are stored as
    uint8 but read back as int64, exactly as the reference's grids of Python
    ints do.
    """

    __slots__ = ("dims", "_list", "_arr", "_t", "_ldtype", "_src", "value_range", "_fresh",
                 "_pending")

    def __init__(self, dims: Sequence[int], data: Sequence[Any]):
        dims = _check_dims(dims)
        size = 1
        for d in dims:
            size *= d
        self._list = self._arr = self._t = None
        self._ldtype = None
        self.value_range = None  # (lo, hi) known bound of every element, if any
        if isinstance(data, np.ndarray):
            if data.size != size:
                raise GridError(
                    f"data length {data.size} does not match dims {dims} (expected {size})")
            self._arr = np.ascontiguousarray(data).reshape(dims)
            self._src = "arr"
        elif type(data).__module__.startswith("torch"):
            if data.numel() != size:
                raise GridError(
                    f"data length {data.numel()} does not match dims {dims} (expected {size})")
            self._t = data.contiguous().reshape(dims)
            self._src = "t"
        else:
            data = list(data)
            if len(data) != size:
                raise GridError(
                    f"data length {len(data)} does not match dims {dims} (expected {size})")
            self._list = data
            self._src = "list"
        self.dims = dims

    # -- constructors -----------------------------------------------------

    @classmethod
    def filled(cls, dims: Sequence[int], fill: Any) -> "Grid":
        dims = _check_dims(dims)
        size = int(np.prod(dims))
        if isinstance(fill, (bool, int, float, np.generic)) and not isinstance(fill, np.object_):
            a = np.full(dims, fill, dtype=np.asarray([fill]).dtype)
            return cls(dims, a)
        return cls(dims, [fill] * size)

    @classmethod
    def from_rows(cls, rows: Sequence[Sequence[Any]]) -> "Grid":
        rows = [list(r) for r in rows]
        if not rows:
            raise GridError("no rows")
        width = len(rows[0])
        if any(len(r) != width for r in rows):
            raise GridError("ragged rows")
        flat: list = []
        for r in rows:
            flat.extend(r)
        return cls((len(rows), width), flat)

    @classmethod
    def from_array(cls, arr) -> "Grid":
        a = np.asarray(arr)
        if a.ndim not in (1, 2):
            raise GridError(f"array rank must be 1 or 2, got {a.ndim}")
        if a.dtype.kind == "f" and a.dtype != np.float64:
            # the reference stores arr.tolist() (grid.py:100-107): Python
            # floats, so every computation on the grid is fp64
            return cls(a.shape, a.astype(np.float64))
        return cls(a.shape, a.copy())

    @classmethod
    def from_tensor(cls, t, logical_dtype=None) -> "Grid":
        """Wrap a (device) tensor without copying."""
        if t.dim() not in (1, 2):
            raise GridError(f"tensor rank must be 1 or 2, got {t.dim()}")
        g = cls(tuple(t.shape), t)
        g._ldtype = np.dtype(logical_dtype) if logical_dtype is not None else None
        return g

    # -- properties -------------------------------------------------------

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def size(self) -> int:
        n = 1
        for d in self.dims:
            n *= d
        return n

    @property
    def data(self) -> list:
        """The elements as a flat Python list (built on first use)."""
        if self._list is None:
            self._list = self._host().ravel().tolist()
        return self._list

    @data.setter
    def data(self, value) -> None:
        self._list = list(value)
        self._arr = self._t = self._fresh = None
        self._src = "list"
        self.value_range = None

    @property
    def is_device(self) -> bool:
        return self._t is not None and self._t.is_cuda

    def storage_dtype(self):
        """numpy dtype of the backing store, or None for a generic list."""
        if self._src == "t":
            return _numpy_dtype_of(self._t.dtype)
        if self._src == "arr":
            return self._arr.dtype
        a = self._probe()
        return a.dtype

    def _probe(self):
        return np.asarray(self._list[:1]) if self._list else np.asarray([])

    # -- access -----------------------------------------------------------

    def at(self, *index: int) -> Any:
        if len(index) != len(self.dims):
            raise GridError(f"index arity {len(index)} vs rank {len(self.dims)}")
        for i, d in zip(index, self.dims):
            if not 0 <= i < d:
                raise GridError(f"index {index} out of range for dims {self.dims}")
        flat = index[0] if len(index) == 1 else index[0] * self.dims[1] + index[1]
        if self._src == "list":
            return self._list[flat]
        return self._host().ravel()[flat].item()

    def __getitem__(self, index) -> Any:
        if isinstance(index, tuple):
            return self.at(*index)
        return self.at(index)

    def in_range(self, *index: int) -> bool:
        if len(index) != len(self.dims):
            return False
        return all(0 <= i < d for i, d in zip(index, self.dims))

    def indices(self) -> Iterator[tuple]:
        if len(self.dims) == 1:
            for i in range(self.dims[0]):
                yield (i,)
        else:
            d1, d2 = self.dims
            for i in range(d1):
                for j in range(d2):
                    yield (i, j)

    def to_rows(self) -> list:
        data = self.data
        if len(self.dims) == 1:
            return list(data)
        d1, d2 = self.dims
        return [data[i * d2:(i + 1) * d2] for i in range(d1)]

    def _host(self) -> np.ndarray:
        """Cached host array (one device->host copy at most)."""
        if self._src == "list":
            # the list is the source of truth (callers may mutate .data)
            return np.asarray(self._list).reshape(self.dims)
        if self._arr is None:
            if self._t is not None:
                a = _to_host(self._t).reshape(self.dims)
                if self._ldtype is not None and a.dtype != self._ldtype:
                    a = a.astype(self._ldtype)
                self._arr = a
            else:
                self._arr = np.asarray(self._list).reshape(self.dims)
        return self._arr

    def prefetch_host(self, out: np.ndarray = None) -> None:
        """Read a device grid back ahead of to_array().

        Without `out`: now, on the calling thread (stream replicas call this
        so the D2H copies of many frames run in parallel rather than in the
        ordered writer).  With `out` (a host array of the grid's shape and
        dtype, ideally over pinned memory): asynchronously, one DMA on a copy
        stream ordered after the work that produced the grid; the next
        to_array() waits for it and returns `out`.  No effect on host grids."""
        if not (self._src == "t" and self._arr is None and self._t is not None and self._t.is_cuda):
            return
        if out is None:
            self._fresh = self.to_array()
            return
        torch = _torch()
        t = self._t
        if tuple(out.shape) != tuple(self.dims) or out.dtype != _numpy_dtype_of(t.dtype):
            raise GridError(f"prefetch_host: out must be {self.dims} {_numpy_dtype_of(t.dtype)}")
        cs = _copy_stream(t.device, "down")
        cs.wait_stream(torch.cuda.current_stream(t.device))
        with torch.cuda.stream(cs):
            torch.from_numpy(out).copy_(t if t.is_contiguous() else t.contiguous(),
                                        non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        t.record_stream(cs)
        self._fresh = (out, ev)

    def prefetch_device(self, device="cuda") -> "Grid":
        """Start uploading a host grid to `device` now, asynchronously, on a
        copy stream; the kernels that consume the grid later wait for the
        copy on their own stream (no host synchronisation).  A host grid over
        a pinned tensor is one DMA; other host storage streams through the
        pinned staging chunks.  Returns self."""
        torch = _torch()
        dev = torch.device(device)
        if dev.type != "cuda" or self.is_device or getattr(self, "_pending", None) is not None:
            return self
        if self._src == "t" and self._t is not None and self._t.is_pinned():
            src = self._t.contiguous()
        else:
            a = self._host()
            if a.dtype == object:
                raise GridError("grid elements are not numeric")
            src = torch.from_numpy(np.ascontiguousarray(a))
            if src.numel() * src.element_size() >= (8 << 20):
                src = src.pin_memory()  # one pinned copy, then the DMA is asynchronous
        cs = _copy_stream(dev, "up")
        with torch.cuda.stream(cs):
            d = src.to(dev, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        self._pending = (d, ev, src)
        return self

    def to_array(self, dtype=None) -> np.ndarray:
        """Fresh host numpy array of the elements (grid.py:158-162)."""
        fresh = getattr(self, "_fresh", None)
        if fresh is not None:
            # a prefetched copy nobody else holds: hand it over (once)
            self._fresh = None
            if isinstance(fresh, tuple):  # asynchronous read into the caller's array
                fresh, ev = fresh
                ev.synchronize()
            if self._ldtype is not None and fresh.dtype != self._ldtype:
                return fresh.astype(self._ldtype if dtype is None else dtype)
            return fresh.astype(dtype) if dtype is not None else fresh
        if self._src == "t" and self._arr is None and self._t is not None and self._t.is_cuda:
            # read straight from the device into a fresh array (no cached
            # copy to copy again)
            a = _to_host(self._t).reshape(self.dims)
            if self._ldtype is not None and a.dtype != self._ldtype:
                return a.astype(self._ldtype if dtype is None else dtype)
            return a.astype(dtype) if dtype is not None else a
        a = self._host()
        return a.astype(dtype) if dtype is not None else a.copy()

    def tensor(self, device=None, dtype=None):
        """The grid as a torch tensor (on `device` if given), cached; no copy
        when it already lives there."""
        torch = _torch()
        pend = getattr(self, "_pending", None)
        if pend is not None and device is not None and torch.device(device).type == "cuda":
            d, ev, _src = pend
            if d.device == _cuda_index(torch, device):
                # a prefetched upload: the consuming stream waits for the copy
                cur = torch.cuda.current_stream(d.device)
                cur.wait_event(ev)
                d.record_stream(cur)
                self._pending = None
                self._t = d
                if self._src != "list":
                    self._src = "t"
                return d.to(dtype) if dtype is not None and d.dtype != dtype else d
        t = self._t
        if t is None:
            a = self._host()
            if a.dtype == object:
                raise GridError("grid elements are not numeric")
            t = torch.from_numpy(np.ascontiguousarray(a))
            if self._src != "list":
                self._t = t
        if device is not None and t.device != torch.device(device):
            dev = torch.device(device)
            if t.device.type == "cpu" and dev.type == "cuda" and not t.is_pinned():
                t = _to_device(t.numpy(), dev)  # pageable host memory: staged
            else:
                t = t.to(device, non_blocking=False)
            if self._src != "list":
                self._t = t
        if dtype is not None and t.dtype != dtype:
            return t.to(dtype)
        return t

    def copy(self) -> "Grid":
        if self._src == "list":
            return Grid(self.dims, list(self._list))
        if self._t is not None:
            g = Grid(self.dims, self._t.clone())
            g._ldtype = self._ldtype
            return g
        return Grid(self.dims, self._arr.copy())

    def __eq__(self, other) -> bool:
        if not isinstance(other, Grid):
            return NotImplemented
        if self.dims != other.dims:
            return False
        if self._src == "list" and other._src == "list":
            return self._list == other._list
        a, b = self._host(), other._host()
        if a.dtype == object or b.dtype == object:
            return self.data == other.data
        return bool(np.array_equal(a, b))

    __hash__ = None

    def __repr__(self) -> str:
        where = "device" if self.is_device else "host"
        return f"Grid(dims={self.dims}, {where})"

    def __getstate__(self):
        return {"dims": self.dims, "data": self._host()}

    def __setstate__(self, st):
        self.dims = st["dims"]
        self._arr = st["data"]
        self._list = self._t = None
        self._ldtype = None
        self._src = "arr"
        self.value_range = None


_COPY_POOL = None
_STAGE_LOCK = None
_STAGE_FREE: list = []
_CHUNK = 32 << 20  # bytes per pinned staging chunk
_NSTAGE = 3        # chunks in flight per transfer


def _copy_pool():
    global _COPY_POOL
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _COPY_POOL = ThreadPoolExecutor(8, thread_name_prefix="sk-hostcopy")
    return _COPY_POOL


_COPY_STREAMS = {}


def _copy_stream(device, kind):
    """Side streams per device: "up" for prefetch_device, "down" for
    prefetch_host (separate, so uploads and read-backs use both PCIe
    directions at once)."""
    torch = _torch()
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    s = _COPY_STREAMS.get((idx, kind))
    if s is None:
        s = _COPY_STREAMS.setdefault((idx, kind), torch.cuda.Stream(device=idx))
    return s


def _cuda_index(torch, device):
    dev = torch.device(device)
    return dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())


def _host_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src (1-D uint8 views) with 8 threads: large copies are bound
    by first-touch page faults of fresh memory, which parallelise (numpy
    releases the GIL in copyto)."""
    n = src.size
    if n < (4 << 20):
        np.copyto(dst, src)
        return
    k = 8
    step = -(-n // k)
    list(_copy_pool().map(
        lambda i: np.copyto(dst[i * step:(i + 1) * step], src[i * step:(i + 1) * step]),
        range(k)))


def _par_copy(src: np.ndarray) -> np.ndarray:
    out = np.empty_like(src)
    _host_copy(out.reshape(-1).view(np.uint8), src.reshape(-1).view(np.uint8))
    return out


class _Stage:
    """_NSTAGE pinned host chunks + one event each: a transfer of any size
    streams through them, the host copy of chunk k overlapping the DMA of
    chunk k+1 (pageable <-> pinned <-> device)."""

    def __init__(self):
        torch = _torch()
        self.bufs = [torch.empty(_CHUNK, dtype=torch.uint8, pin_memory=True)
                     for _ in range(_NSTAGE)]
        self.views = [b.numpy() for b in self.bufs]
        self.events = [None] * _NSTAGE


def _stage_get() -> _Stage:
    import threading

    global _STAGE_LOCK
    if _STAGE_LOCK is None:
        _STAGE_LOCK = threading.Lock()
    with _STAGE_LOCK:
        if _STAGE_FREE:
            return _STAGE_FREE.pop()
    return _Stage()


def _stage_put(st: _Stage) -> None:
    with _STAGE_LOCK:
        _STAGE_FREE.append(st)


def _to_device(a: np.ndarray, device):
    """Host array -> new device tensor.  Large arrays stream through pinned
    chunks on the current stream (pageable memory crosses PCIe at a fraction
    of the pinned rate); the call returns once the data is on the device."""
    torch = _torch()
    a = np.ascontiguousarray(a)
    if a.nbytes < (8 << 20):
        return torch.from_numpy(a).to(device)
    out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device=device)
    src = a.reshape(-1).view(np.uint8)
    dst = out.view(-1).view(torch.uint8)
    stream = torch.cuda.current_stream(out.device)
    st = _stage_get()
    try:
        for k, off in enumerate(range(0, src.size, _CHUNK)):
            j = k % _NSTAGE
            m = min(_CHUNK, src.size - off)
            if st.events[j] is not None:
                st.events[j].synchronize()  # chunk k - _NSTAGE has left this buffer
            _host_copy(st.views[j][:m], src[off:off + m])
            dst[off:off + m].copy_(st.bufs[j][:m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            st.events[j] = ev
        for ev in st.events:
            if ev is not None:
                ev.synchronize()
    finally:
        st.events = [None] * _NSTAGE
        _stage_put(st)
    return out


def _to_host(t) -> np.ndarray:
    """Device tensor -> fresh numpy array.  Large tensors stream through
    pinned chunks: the DMA of chunk k+1.. runs while chunk k is copied out
    into the fresh array."""
    torch = _torch()
    if not t.is_cuda or t.numel() * t.element_size() < (1 << 20):
        return t.detach().cpu().numpy()
    if os.environ.get("SK_D2H", "pinned") == "direct":
        # the driver's own staged copy straight into the fresh array
        out = np.empty(tuple(t.shape), dtype=_numpy_dtype_of(t.dtype))
        src = t.detach() if t.is_contiguous() else t.detach().contiguous()
        torch.from_numpy(out).copy_(src)
        return out
    out = np.empty(tuple(t.shape), dtype=_numpy_dtype_of(t.dtype))
    src = (t.detach() if t.is_contiguous() else t.detach().contiguous()).reshape(-1)
    src = src.view(torch.uint8)
    dst = out.reshape(-1).view(np.uint8)
    stream = torch.cuda.current_stream(t.device)
    st = _stage_get()
    offs = list(range(0, dst.size, _CHUNK))
    try:
        def issue(k):
            j = k % _NSTAGE
            m = min(_CHUNK, dst.size - offs[k])
            st.bufs[j][:m].copy_(src[offs[k]:offs[k] + m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            st.events[j] = ev

        for k in range(min(_NSTAGE, len(offs))):
            issue(k)
        for k in range(len(offs)):
            j = k % _NSTAGE
            m = min(_CHUNK, dst.size - offs[k])
            st.events[j].synchronize()
            _host_copy(dst[offs[k]:offs[k] + m], st.views[j][:m])
            if k + _NSTAGE < len(offs):
                issue(k + _NSTAGE)
    finally:
        st.events = [None] * _NSTAGE
        _stage_put(st)
    return out


def _numpy_dtype_of(tdtype):
    torch = _torch()
    return {
        torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64),
        torch.uint8: np.dtype(np.uint8), torch.int64: np.dtype(np.int64),
        torch.int32: np.dtype(np.int32), torch.bool: np.dtype(bool),
    }[tdtype]


def grid_new(dims: Sequence[int], fill: Any) -> Grid:
    """A grid of the given shape with every element set to fill."""
    return Grid.filled(dims, fill)


def grid_get_padded(g: Grid, index: Sequence[int]) -> Any:
    """Element read returning ABSENT outside the grid (grid.py:184-198)."""
    index = tuple(index)
    if len(index) != g.ndim:
        raise GridError(f"index arity {len(index)} vs rank {g.ndim}")
    if not g.in_range(*index):
        return ABSENT
    return g.at(*index)


class Neighborhood:
    """(2k+1)^n window centred on one element; ABSENT outside (grid.py:201-240)."""

    __slots__ = ("k", "center_index", "entries")

    def __init__(self, k: int, center_index: tuple, entries: tuple):
        self.k = k
        self.center_index = center_index
        self.entries = entries

    def _slot(self, offs) -> int:
        w = 2 * self.k + 1
        if len(offs) == 1:
            return self.k + offs[0]
        return (self.k + offs[0]) * w + self.k + offs[1]

    @property
    def center(self) -> Any:
        return self.entries[self._slot((0,) * len(self.center_index))]

    def at(self, *delta: int) -> Any:
        return self.entries[self._slot(delta)]

    def values(self) -> list:
        return [v for v in self.entries if v is not ABSENT]

    def __iter__(self):
        return iter(self.entries)

    def __len__(self) -> int:
        return len(self.entries)

    def __repr__(self) -> str:
        return f"Neighborhood(k={self.k}, center={self.center_index})"


class IndexedNeighborhood(Neighborhood):
    """Window of (value, global index) pairs (grid.py:243-256)."""

    __slots__ = ()

    def pairs(self) -> list:
        return [p for p in self.entries if p is not ABSENT]

    def values(self) -> list:
        return [p[0] for p in self.entries if p is not ABSENT]


def _window(g: Grid, center, k: int, indexed: bool):
    if k < 0:
        raise GridError(f"window radius must be >= 0, got {k}")
    center = tuple(center)
    if len(center) != g.ndim:
        raise GridError(f"center arity {len(center)} vs rank {g.ndim}")
    if not g.in_range(*center):
        raise GridError(f"center {center} out of range for dims {g.dims}")
    data = g.data
    span = range(-k, k + 1)
    if g.ndim == 1:
        (i,) = center
        idx = [(i + a,) for a in span]
    else:
        i, j = center
        idx = [(i + a, j + b) for a in span for b in span]
    out = []
    d2 = g.dims[1] if g.ndim == 2 else 1
    for ix in idx:
        if not g.in_range(*ix):
            out.append(ABSENT)
            continue
        v = data[ix[0] * d2 + ix[1]] if g.ndim == 2 else data[ix[0]]
        out.append((v, ix) if indexed else v)
    cls = IndexedNeighborhood if indexed else Neighborhood
    return cls(k, center, tuple(out))


def neighborhood_at(g: Grid, center: Sequence[int], k: int) -> Neighborhood:
    return _window(g, center, k, False)


def indexed_neighborhood_at(g: Grid, center: Sequence[int], k: int) -> IndexedNeighborhood:
    return _window(g, center, k, True)
