"""Two-phase impulse-noise removal for 8-bit images (reference: apps/denoise.py).

Phase one flags suspect pixels with the adaptive median test (sm_100a
kernel csrc/sk_amf.cu); phase two restores only the flagged pixels by
minimising a local edge-preserving functional with an 18-step ternary
search in fp64, iterated until the mean change per flagged pixel drops
below tolerance (csrc/sk_restore.cu; the loop and its stopping test run on
the device).  The video entry point is the reference's

    pipeline(read, detect, ordered_farm(restore, W), write)

where every restore replica owns a WorkerGroup -- its own CUDA stream -- so
W restoration loops are in flight on the GPU at once.
"""

from __future__ import annotations

import os
import threading
import time

import ctypes as C
import math
from dataclasses import dataclass
from typing import Callable, Iterable, Optional

import numpy as np

from .. import _native as N
from ..grid import Grid, GridError
from ..loop import Condition, DeviceCond, stop_after
from ..partition import DeploymentMode, WorkerGroup, parallel_loop
from ..patterns import Combinator, DeviceKernel, DeviceUnsupported, ElementalFn, abs_change
from ..streams import (Stage, StreamReport, _host_ring, batch_farm, ordered_farm, pipeline,
                       run_stream)

_SEARCH_STEPS = math.ceil(math.log((255.0 - 0.0) / 0.25) / math.log(1.5))  # 18, as the reference


@dataclass(frozen=True)
class RestoreConfig:
    """Knobs for both phases (apps/denoise.py:48-72)."""

    amf_wmax: int = 7
    phi_eps: float = 1e-2
    beta: float = 2.0
    tol: float = 0.02
    max_iterations: int = 100

    def __post_init__(self):
        if self.amf_wmax < 3 or self.amf_wmax % 2 == 0:
            raise GridError(f"amf_wmax must be odd and >= 3, got {self.amf_wmax}")
        if self.phi_eps <= 0 or self.beta <= 0 or self.tol <= 0:
            raise GridError("phi_eps, beta and tol must all be positive")


def _device_only(nb, env):
    raise DeviceUnsupported("denoise kernels run only on the device")


# ---------------------------------------------------------------- phase one


def detect_kernel(wmax: int = 7) -> ElementalFn:
    """Adaptive-median classifier of radius wmax//2 (apps/denoise.py:79-138)."""
    if wmax < 3 or wmax % 2 == 0:
        raise GridError(f"wmax must be odd and >= 3, got {wmax}")
    if wmax > 15:
        raise DeviceUnsupported("the device detector supports windows up to 15x15")
    return ElementalFn(point=_device_only, k=wmax // 2, block=None, pad_mode="constant",
                       pad_value=0, device=DeviceKernel("amf", (float(wmax),)))


def _mask_sum() -> Combinator:
    return Combinator(lambda a, b: a + b, 0, on_array=lambda arr: int(np.sum(arr)), kind="sum")


def amf_detect(img: Grid, wmax: int = 7, *, partitions: int = 1,
               mode=DeploymentMode.ONE_TO_N, group: Optional[WorkerGroup] = None) -> Grid:
    """0/1 impulse map (apps/denoise.py:145-157)."""
    if img.ndim != 2:
        raise GridError("detection expects a 2D image")
    if partitions == 1:
        mode = DeploymentMode.ONE_TO_ONE
    out, _ = parallel_loop(mode, partitions, wmax // 2, detect_kernel(wmax), _mask_sum(),
                           stop_after(1), img, group=group)
    return out


def _detect_frame(img: Grid, wmax: int, stream) -> Grid:
    """amf_detect of one frame through the batched detector, on `stream`.
    Same kernel and bit-exact result as amf_detect; the mask comes back as a
    device Grid tagged with its (0, 1) range."""
    import torch

    from ..partition import _u8_from

    N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.stream(stream):
        t = _u8_from(img, "amf", 0, 255, dev).reshape(1, *img.dims)
        masks, _ = amf_frames(t, wmax, stream=stream)
    stream.synchronize()
    g = Grid.from_tensor(masks[0], logical_dtype=np.int64)
    g.value_range = (0, 1)
    return g


def amf_frames(frames, wmax: int = 7, out=None, stream=None):
    """Batched detection over a [F, H, W] uint8 CUDA tensor (one launch).
    Returns (masks [F, H, W] uint8 0/1, flagged counts [F] int64)."""
    import torch

    lib = N.require_cuda()
    if frames.dtype != torch.uint8 or frames.dim() != 3 or not frames.is_cuda:
        raise GridError("amf_frames expects a [F, H, W] uint8 CUDA tensor")
    F, H, W = frames.shape
    if out is None:  # rows padded to 16 bytes (the kernels' pitch rule)
        Wp = -(-frames.shape[2] // 16) * 16
        out = torch.empty((frames.shape[0], frames.shape[1], Wp), dtype=torch.uint8,
                          device=frames.device)[:, :, :frames.shape[2]]
    counts = torch.empty(F, dtype=torch.int64, device=frames.device)
    st = stream if stream is not None else torch.cuda.current_stream()
    N.check(lib.sk_amf_frames(C.c_void_p(frames.data_ptr()), frames.stride(1), frames.stride(0),
                              C.c_void_p(out.data_ptr()), out.stride(1), out.stride(0), F, H, W,
                              wmax, C.c_void_p(counts.data_ptr()), N.stream_handle(st)))
    return out, counts


# ---------------------------------------------------------------- phase two


def restore_kernel(cfg: RestoreConfig) -> ElementalFn:
    """Ternary-search restoration of flagged pixels (apps/denoise.py:164-249)."""
    return ElementalFn(point=_device_only, k=1, block=None, pad_mode="constant", pad_value=0.0,
                       device=DeviceKernel("restore", (cfg.beta, cfg.phi_eps)))


def _float_sum() -> Combinator:
    return Combinator(lambda a, b: a + b, 0.0, on_array=lambda arr: float(np.sum(arr)), kind="sum")


def _check_mask(noise: Grid) -> None:
    """The reference rejects anything but 0/1 (apps/denoise.py:276-278).  Host
    masks are checked on the host; detector outputs carry a (0, 1) range tag;
    other device masks are checked on the device."""
    sd = noise.storage_dtype()
    if sd.kind not in "iub":
        raise GridError(f"noise map must be 0/1, found dtype {sd}")
    rng = noise.value_range
    if rng is not None and rng[0] >= 0 and rng[1] <= 1:
        return
    if noise.is_device:
        t = noise.tensor()
        mn, mx = int(t.min().item()), int(t.max().item())
        if mn < 0 or mx > 1:
            raise GridError(f"noise map must be 0/1, found values in [{mn}, {mx}]")
        return
    a = noise._host()
    bad = (a != 0) & (a != 1)
    if bad.any():
        raise GridError(f"noise map must be 0/1, found {a[bad].ravel()[0]!r}")


def _flagged_count(noise: Grid) -> int:
    sd = noise.storage_dtype()
    if sd.kind not in "iub":
        raise GridError(f"noise map must be 0/1, found dtype {sd}")
    if noise.is_device:
        t = noise.tensor()
        mn, mx = int(t.min().item()), int(t.max().item())
        if mn < 0 or mx > 1:
            raise GridError(f"noise map must be 0/1, found values in [{mn}, {mx}]")
        return int(t.sum().item())
    a = noise.to_array()
    bad = (a != 0) & (a != 1)
    if bad.any():
        raise GridError(f"noise map must be 0/1, found {a[bad].ravel()[0]!r}")
    return int(a.sum())


def restore_regularize(img: Grid, noise: Grid, cfg: Optional[RestoreConfig] = None,
                       *, partitions: int = 1, mode=DeploymentMode.ONE_TO_N,
                       group: Optional[WorkerGroup] = None, devices: Optional[list] = None):
    """Restore the flagged pixels; returns (fp64 grid, LoopReport)
    (apps/denoise.py:262-288).

    `devices` (several GPUs, 1:n): the `partitions` row blocks are spread
    over these GPUs (contiguous blocks per GPU) and restored together, the
    boundary rows exchanged every iteration (_restore_split)."""
    cfg = cfg or RestoreConfig()
    if img.ndim != 2:
        raise GridError("restoration expects a 2D image")
    if noise.dims != img.dims:
        raise GridError(f"noise map dims {noise.dims} do not match image {img.dims}")
    _check_mask(noise)
    if devices is not None and len(devices) > 1:
        if partitions < len(devices):
            raise GridError(f"{len(devices)} GPUs need at least as many partitions, got {partitions}")
        return _restore_split(img, noise, cfg, partitions, [int(getattr(d, "index", d))
                                                             for d in devices])
    # value / max(flagged, 1) < tol: on the device the run counts the flagged
    # pixels itself; a host-evaluated loop counts them once, on first use
    denom = []

    def stop(value, it, state):
        if not denom:
            denom.append(max(_flagged_count(noise), 1))
        return value / denom[0] < cfg.tol

    cond = Condition(stop, cfg.max_iterations, DeviceCond("mean_flagged_lt", float(cfg.tol)))
    if partitions == 1:
        mode = DeploymentMode.ONE_TO_ONE
    return parallel_loop(mode, partitions, 1, restore_kernel(cfg), _float_sum(), cond, img,
                         env=noise, delta=abs_change(), indexed=True, group=group)


def _restore_split(img: Grid, noise: Grid, cfg: RestoreConfig, P: int, devices: list):
    """restore_regularize with its P row partitions spread over several GPUs
    (the paper's 1:n deployment of one frame across a GPU pair, Table 3).

    One run per partition, on devices[p * len(devices) // P], each over a
    full-size replica of the frame but computing only its own partition
    (SK_KERNEL_RESTORE params pa, pb).  After every iteration the rows at
    each partition boundary (values and change flags) are copied to the
    neighbouring partition's run (sk_run_exchange_rows: a peer copy,
    stream-ordered before the neighbour's next sweep) -- the reference's
    halo_exchange (partition.py:247-262).  Each run's value is its own
    partition's sum; the host folds them in partition order from 0.0 and
    applies value / max(flagged, 1) < tol (apps/denoise.py:262-288), exactly
    the single-GPU engine's fold, so grids, iteration counts and values are
    bit-identical to a one-GPU restore with the same partitions."""
    import torch

    from ..loop import LoopReport
    from ..partition import _split_ranges, _u8_from, model_ledger

    lib = N.require_cuda()
    H, W = img.dims
    if P > H or P > 64:
        raise GridError(f"cannot split {H} rows across {P} partitions")
    ranges = _split_ranges(H, P)
    denom = max(_flagged_count(noise), 1)
    Wp = -(-W // 2) * 2  # fp64 rows in whole 16-byte vectors
    runs = []
    try:
        for p in range(P):
            dev = devices[p * len(devices) // P]
            with torch.cuda.device(dev):
                st = torch.cuda.Stream(device=dev)
                with torch.cuda.stream(st):
                    d = torch.device("cuda", dev)
                    src = torch.zeros((H, Wp), dtype=torch.float64, device=d)
                    src[:, :W] = img.tensor(device=d).to(torch.float64)
                    env = torch.zeros((H, -(-W // 16) * 16), dtype=torch.uint8, device=d)
                    env[:, :W] = _u8_from(noise, "noise map", 0, 1, d)
                    bufs = [torch.empty((H, Wp), dtype=torch.float64, device=d) for _ in range(2)]
                    pl = N.sk_plan()
                    pl.kernel, pl.dtype = N.SK_KERNEL_RESTORE, N.SK_F64
                    pl.rows, pl.cols, pl.partitions = H, W, P
                    pl.reduce_op, pl.delta_op = N.SK_REDUCE_SUM, N.SK_DELTA_ABS
                    pl.identity = 0.0
                    pl.params[0], pl.params[1] = cfg.beta, cfg.phi_eps
                    pl.params[2], pl.params[3] = float(p), float(p + 1)
                    h = C.c_void_p()
                    N.check(lib.sk_run_begin(C.byref(pl), C.c_void_p(src.data_ptr()), Wp,
                                             C.c_void_p(env.data_ptr()), env.stride(0),
                                             C.c_void_p(bufs[0].data_ptr()),
                                             C.c_void_p(bufs[1].data_ptr()), Wp,
                                             N.stream_handle(st), C.byref(h)))
                    runs.append({"h": h, "dev": dev, "stream": st, "keep": (src, env),
                                 "bufs": bufs})
        t, value, stopped = 0, 0.0, False
        v = C.c_double()
        while True:
            t += 1
            for r in runs:
                N.check(lib.sk_run_launch(r["h"], 1))
            for p in range(P - 1):  # boundary rows of iteration t, both ways
                lo_next = ranges[p + 1][0]
                N.check(lib.sk_run_exchange_rows(runs[p + 1]["h"], runs[p]["h"], lo_next - 1,
                                                 lo_next, t))
                N.check(lib.sk_run_exchange_rows(runs[p]["h"], runs[p + 1]["h"], lo_next,
                                                 lo_next + 1, t))
            value = 0.0
            for r in runs:  # partition order, from the identity
                N.check(lib.sk_run_value(r["h"], t, C.byref(v)))
                value = value + v.value
            if value / denom < cfg.tol:
                stopped = True
                break
            if t >= cfg.max_iterations:
                break
        home = torch.device("cuda", devices[0])
        out = torch.empty((H, W), dtype=torch.float64, device=home)
        for (lo, hi), r in zip(ranges, runs):
            r["stream"].synchronize()
            out[lo:hi].copy_(r["bufs"][t & 1][lo:hi, :W])
    finally:
        for r in runs:
            N.check(lib.sk_run_destroy(r["h"]))
    g = Grid.from_tensor(out, logical_dtype=np.float64)
    return g, LoopReport(iterations=t, final_reduce=value, copies=model_ledger((H, W), P, 1, t),
                         exhausted=not stopped)


def restore_frames(frames, masks, cfg: Optional[RestoreConfig] = None, stream=None):
    """restore_regularize over a batch of up to 64 frames in ONE persistent
    launch: a device-side farm of loops.  Every frame keeps its own stopping
    test, iteration count and final value (bit-identical to restoring it
    alone); the grid barrier of the loop ends when the last frame stops.

    frames: [F, H, W] CUDA tensor (uint8 or float64); masks: [F, H, W] uint8
    0/1 CUDA tensor (e.g. from amf_frames).  Returns (outputs, reports): F
    float64 [H, W] device views and F LoopReports.
    """
    import torch

    from ..loop import LoopReport
    from ..partition import model_ledger

    lib = N.require_cuda()
    cfg = cfg or RestoreConfig()
    if frames.dim() != 3 or masks.shape != frames.shape or not frames.is_cuda:
        raise GridError("restore_frames expects [F, H, W] CUDA frames and masks of that shape")
    F, H, W = frames.shape
    if not 1 <= F <= 64:
        raise GridError("restore_frames takes 1..64 frames per batch")
    st = stream if stream is not None else torch.cuda.current_stream()
    with torch.cuda.stream(st):
        src = frames.reshape(F * H, W).to(torch.float64).contiguous()
        env = masks.reshape(F * H, W).to(torch.uint8).contiguous()
        bufs = [torch.empty((F * H, W), dtype=torch.float64, device=frames.device)
                for _ in range(2)]
        p = N.sk_plan()
        p.kernel, p.dtype = N.SK_KERNEL_RESTORE, N.SK_F64
        p.rows, p.cols, p.partitions = F * H, W, F
        p.reduce_op, p.delta_op = N.SK_REDUCE_SUM, N.SK_DELTA_ABS
        p.flags = N.SK_FLAG_FRAMES
        p.identity = 0.0
        p.params[0], p.params[1] = cfg.beta, cfg.phi_eps
        h = C.c_void_p()
        N.check(lib.sk_run_begin(C.byref(p), C.c_void_p(src.data_ptr()), W,
                                 C.c_void_p(env.data_ptr()), W, C.c_void_p(bufs[0].data_ptr()),
                                 C.c_void_p(bufs[1].data_ptr()), W, N.stream_handle(st),
                                 C.byref(h)))
        try:
            c = N.sk_cond()
            c.kind, c.a, c.max_iterations = N.SK_COND_MEAN_FLAGGED_LT, cfg.tol, cfg.max_iterations
            it, val, ex = C.c_int64(), C.c_double(), C.c_int32()
            N.check(lib.sk_run_loop(h, C.byref(c), C.byref(it), C.byref(val), C.byref(ex)))
            its = (C.c_int64 * F)()
            vals = (C.c_double * F)()
            exh = (C.c_int32 * F)()
            N.check(lib.sk_run_frame_status(h, its, vals, exh))
        finally:
            N.check(lib.sk_run_destroy(h))
    outs, reps = [], []
    for f in range(F):
        k = int(its[f])
        outs.append(bufs[k & 1][f * H:(f + 1) * H])
        reps.append(LoopReport(iterations=k, final_reduce=float(vals[f]),
                               copies=model_ledger((H, W), 1, 1, k), exhausted=bool(exh[f])))
    return outs, reps


# ---------------------------------------------------------------- inputs, video


def salt_pepper_array(a: np.ndarray, level: float, seed: int = 42):
    """numpy form of `salt_pepper` (same PCG64 stream): (noisy, hit) arrays."""
    if not 0 <= level <= 1:
        raise GridError(f"noise level must be in [0, 1], got {level}")
    rng = np.random.default_rng(seed)
    hit = rng.random(a.shape) < level
    salt = rng.random(a.shape) < 0.5
    return np.where(hit, np.where(salt, 255, 0), a), hit


def salt_pepper(img: Grid, level: float, seed: int = 42):
    """Corrupt a fraction of pixels to 0/255 with numpy's PCG64, exactly as the
    reference (apps/denoise.py:295-304); returns (noisy, mask).  Host-side
    input synthesis: identical streams of random numbers require numpy."""
    noisy, hit = salt_pepper_array(img.to_array(), level, seed)
    return Grid.from_array(noisy), Grid.from_array(hit.astype(np.int64))


class _RestoreBatcher:
    """Coalesces the restore farm's frames on ONE GPU into device batches.

    Every farm lane still hands in one frame at a time (the reference's
    ordered farm, apps/denoise.py:338-356); what the lanes of one GPU hand in
    concurrently is restored together by `restore_frames` -- one persistent
    launch in which every frame runs its own loop to its own stop, each
    bit-identical to restoring it alone.  A batch is closed when it is full,
    or when no further frame arrives within `linger_s`.  The batch waits for
    each submitting lane's stream (its upload) and the lane waits for the
    batch's completion event, so no host synchronisation sits between them."""

    def __init__(self, cfg: RestoreConfig, max_batch: int, linger_s: float = 2e-4,
                 detect: bool = False, device: Optional[int] = None):
        import torch

        self.cfg = cfg
        self.max_batch = max(1, min(64, max_batch))
        self.linger_s = linger_s
        self.cv = threading.Condition()
        self.pending = []
        self.closed = False
        self.detect = detect  # run the detector on each batch first (masks not given)
        self.device = torch.cuda.current_device() if device is None else device
        self.stream = torch.cuda.Stream(device=self.device)
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def submit(self, frame, mask, after=None):
        """frame / mask: [H, W] uint8 tensors on this batcher's GPU, ready
        after the event `after` (None: already complete); returns
        (out, report, done_event)."""
        slot = {"done": threading.Event(), "after": after}
        with self.cv:
            if self.closed:
                raise RuntimeError("restore batcher is closed")
            self.pending.append((frame, mask, slot))
            self.cv.notify_all()
        slot["done"].wait()
        if "error" in slot:
            raise slot["error"]
        return slot["result"]

    def _take(self):
        with self.cv:
            while not self.pending and not self.closed:
                self.cv.wait()
            if not self.pending:
                return None
            deadline = time.perf_counter() + self.linger_s
            while len(self.pending) < self.max_batch:
                left = deadline - time.perf_counter()
                if left <= 0 or self.closed:
                    break
                self.cv.wait(left)
            shape = self.pending[0][0].shape
            batch = [x for x in self.pending if x[0].shape == shape][:self.max_batch]
            for x in batch:
                self.pending.remove(x)
            return batch

    def _run(self):
        import torch

        torch.cuda.set_device(self.device)
        while True:
            batch = self._take()
            if batch is None:
                return
            try:
                with torch.cuda.stream(self.stream):
                    for _f, _m, slot in batch:
                        if slot["after"] is not None:
                            self.stream.wait_event(slot["after"])
                    frames = torch.stack([b[0] for b in batch])
                    if self.detect:
                        masks, _ = amf_frames(frames, self.cfg.amf_wmax, stream=self.stream)
                    else:
                        masks = torch.stack([b[1] for b in batch])
                    outs, reps = restore_frames(frames, masks, self.cfg, stream=self.stream)
                    done = torch.cuda.Event()
                    done.record(self.stream)
                for (_f, _m, slot), o, r in zip(batch, outs, reps):
                    g = Grid.from_tensor(o, logical_dtype=np.float64)
                    slot["result"] = (g, r, done)
                    slot["done"].set()
            except Exception as e:  # the batch's frames all fail with it
                for _f, _m, slot in batch:
                    slot["error"] = e
                    slot["done"].set()

    def close(self):
        with self.cv:
            self.closed = True
            self.cv.notify_all()
        self.thread.join(timeout=30)


def _host_u8(img):
    """A frame for the batched farm: a uint8 torch tensor (host or device),
    range-checked like amf_detect's input (no copy for uint8 tensors)."""
    import torch

    from ..partition import _u8_from

    if not isinstance(img, Grid):
        raise GridError(f"frames must be grids, got {type(img).__name__}")
    if img.ndim != 2:
        raise GridError("detection expects a 2D image")
    t0 = img._t if img._src == "t" else None
    if t0 is not None and t0.dtype == torch.uint8:
        return t0
    if img.is_device:
        return _u8_from(img, "amf", 0, 255, img._t.device)
    return _u8_from(img, "amf", 0, 255, torch.device("cpu"))


def _batched_restore_stream(frames, cfg, writer, loader, devices, host_buffers,
                            batch) -> StreamReport:
    """read -> detect -> ordered_farm(restore) -> write for the 1:1 case with
    fused detection, farmed at batch granularity (streams.batch_farm): each
    batch is detected (amf_frames) and restored (restore_frames: every frame
    its own loop in one persistent launch) on one GPU."""
    import numpy as np

    def run_batch(d, stream):
        masks, _ = amf_frames(d, cfg.amf_wmax, stream=stream)
        outs, _reps = restore_frames(d, masks, cfg, stream=stream)
        return outs

    return batch_farm(frames, _host_u8, run_batch, writer=writer, loader=loader,
                      devices=devices, batch=batch, host_buffers=host_buffers,
                      logical_dtype=np.float64, compute_name="restore")


def video_restore_pipeline(frames: Iterable, *, width: int = 1, partitions: int = 1,
                           mode=DeploymentMode.ONE_TO_ONE, cfg: Optional[RestoreConfig] = None,
                           writer: Optional[Callable] = None, loader: Optional[Callable] = None,
                           mask_writer: Optional[Callable] = None,
                           devices: Optional[list] = None,
                           host_buffers: bool = False,
                           gpus_per_frame: int = 1) -> StreamReport:
    """read -> detect -> ordered_farm(restore, width) -> write
    (apps/denoise.py:307-368), over one GPU or several.

    `devices` (default: the caller's GPU): the restore farm's `width` lanes
    are spread round-robin over these GPUs (streams.ordered_farm), each lane
    with its own CUDA stream; frames keep stream order end to end.

    1:1 deployment: each lane uploads its frame (uint8) on its own stream and
    hands it to its GPU's batcher, which detects and restores whatever that
    GPU's lanes have in flight together in a single persistent launch (a
    device-side farm of loops, restore_frames).  With a `mask_writer` the
    detector runs per frame in the detect stage instead, so masks are written
    in stream order.  1:n deployment: each lane runs restore_regularize over
    `partitions` row blocks of its frame on its GPU -- or, with
    `gpus_per_frame=g` > 1, across a group of g GPUs (`devices` cut into
    consecutive groups, lanes round-robin over the groups; boundary rows
    exchanged over NVLink every iteration): the paper's "2xGPUs 1:2"
    deployment (Table 3).

    `host_buffers=True` (with a `writer`): each restored frame is read back by
    one DMA into a recycled pinned host frame and handed to the writer as a
    host Grid over it (`g.tensor()` is that pinned tensor, no copy); the
    buffer is reused once the writer returns, so a writer that keeps a frame
    must copy it (`g.to_array()`).  Default: every frame is a fresh grid, as
    in the reference."""
    import torch

    from ..partition import _u8_from
    from ..streams import current_lane

    mode = DeploymentMode.parse(mode)
    if mode is DeploymentMode.ONE_TO_N and partitions < 2:
        raise GridError("1:n deployment needs at least 2 partitions")
    eff = partitions if mode is DeploymentMode.ONE_TO_N else 1
    cfg = cfg or RestoreConfig()
    N.require_cuda()
    if devices is None:
        devices = [torch.cuda.current_device()]
    devices = [int(getattr(d, "index", d)) for d in devices]
    groups = None
    if gpus_per_frame > 1:
        if mode is not DeploymentMode.ONE_TO_N or eff < gpus_per_frame:
            raise GridError("gpus_per_frame > 1 needs 1:n mode with at least that many partitions")
        if len(devices) % gpus_per_frame:
            raise GridError(f"{len(devices)} devices do not split into groups of {gpus_per_frame}")
        groups = [devices[i:i + gpus_per_frame] for i in range(0, len(devices), gpus_per_frame)]
        devices = [g[0] for g in groups]  # a lane runs on its group's first GPU
        group_of = {k: groups[k % len(groups)] for k in range(width)}
    batched = eff == 1
    fused_detect = batched and mask_writer is None
    if fused_detect and not os.environ.get("SK_LANE_FARM"):
        # the farm at batch granularity: the device-side farm of loops
        # (restore_frames) fed by two workers per GPU, frames written in order
        per_dev = -(-width // len(devices))
        cap = int(os.environ.get("SK_BATCH_CAP", "0")) or max(1, min(64, -(-per_dev // 2)))
        return _batched_restore_stream(frames, cfg, writer, loader, devices, host_buffers, cap)
    per_dev = -(-width // len(devices))
    # a GPU's lanes fill two batches: one restores while the other's frames
    # are read back and the next frames uploaded (SK_BATCH_CAP overrides)
    cap = int(os.environ.get("SK_BATCH_CAP", "0")) or max(1, -(-per_dev // 2))
    batchers = ({d: _RestoreBatcher(cfg, cap, detect=fused_detect, device=d)
                 for d in dict.fromkeys(devices)} if batched else {})
    ring = _host_ring() if (host_buffers and writer is not None) else None
    held, held_lock = {}, threading.Lock()  # id(grid handed on) -> its pinned frame

    def detect_fn(img: Grid):
        if img.ndim != 2:
            raise GridError("detection expects a 2D image")
        if fused_detect:
            return img, None  # the restore lane uploads it; its batcher detects
        lane = current_lane()
        if not batched:
            mask = _detect_frame(img, cfg.amf_wmax, lane.stream)
            if mask_writer is not None:
                mask_writer(mask)
            return img, mask
        dev = torch.device("cuda", lane.device)
        t = _u8_from(img, "amf", 0, 255, dev)
        masks, _ = amf_frames(t.reshape(1, *img.dims), cfg.amf_wmax, stream=lane.stream)
        if mask_writer is not None:
            lane.stream.synchronize()
            mg = Grid.from_tensor(masks[0], logical_dtype=np.int64)
            mg.value_range = (0, 1)
            mask_writer(mg)
        return t, masks[0]

    def make_restorer():
        lane = current_lane()
        dev = torch.device("cuda", lane.device)
        grp = None if batched else WorkerGroup(eff)

        class _Restorer:
            def __call__(self, pair):
                img, mask = pair
                if batched:
                    # on the lane's stream (current): the frame's upload, and
                    # the mask's move when detect ran on another GPU
                    if isinstance(img, Grid):
                        img = _u8_from(img, "amf", 0, 255, dev)
                    elif img.device != dev:
                        img = img.to(dev, non_blocking=True)
                    if mask is not None and mask.device != dev:
                        mask = mask.to(dev, non_blocking=True)
                    up = torch.cuda.Event()
                    up.record(lane.stream)
                    out, _rep, done = batchers[lane.device].submit(img, mask, after=up)
                    lane.stream.wait_event(done)
                elif groups is not None:  # the frame split across the lane's GPU group
                    out, _rep = restore_regularize(img, mask, cfg, partitions=eff, mode=mode,
                                                   devices=group_of[lane.index])
                else:
                    out, _rep = restore_regularize(
                        img, mask, cfg, partitions=eff,
                        mode=mode if eff > 1 else DeploymentMode.ONE_TO_ONE, group=grp)
                if ring is not None:
                    # one DMA into a recycled pinned frame, on the lane's stream
                    t = out.tensor()
                    h = ring.get(t.shape, t.dtype)
                    h.copy_(t, non_blocking=True)
                    lane.stream.synchronize()
                    g = Grid.from_tensor(h, logical_dtype=np.float64)
                    with held_lock:
                        held[id(g)] = h
                    return g
                if writer is not None:
                    # read the frame back here, in parallel across lanes; the
                    # ordered writer's to_array() then takes it over
                    out.prefetch_host()
                return out

            def close(self):
                if grp is not None:
                    grp.close()

        return _Restorer()

    read = Stage(loader or (lambda f: f), name="read")
    detect = Stage(detect_fn, name="detect")
    restore = Stage(factory=make_restorer, name="restore")
    if writer is None:
        write = Stage(lambda g: g, name="write")
    else:
        def write_fn(g):
            writer(g)
            if ring is not None:  # the writer is done with the pinned frame
                with held_lock:
                    h = held.pop(id(g), None)
                if h is not None:
                    ring.put(h)
            return g

        write = Stage(write_fn, name="write")
    top = pipeline(read, detect, ordered_farm(restore, width, devices=devices), write)
    try:
        return run_stream(frames, top, sink=lambda _item: None)
    finally:
        for b in batchers.values():
            b.close()
