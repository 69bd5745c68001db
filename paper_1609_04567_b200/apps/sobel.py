"""Sobel edge magnitude over 8-bit images (reference: apps/sobel.py).

One stencil pass: magnitude of the two 3x3 Sobel gradients, rounded half to
even and clipped to [0, 255]; off-image window slots read as the centre
pixel.  Runs as the u8 sm_100a kernel in csrc/sk_u8stencil.cu, either as a
single-iteration loop behind the pattern API (`sobel_filter`) or batched
over a stack of frames (`sobel_frames`, the stream-mode entry point).
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

from .. import _native as N
from ..grid import Grid, GridError
from ..streams import StreamReport, batch_farm
from ..loop import stop_after
from ..partition import DeploymentMode, WorkerGroup, parallel_loop
from ..patterns import Combinator, DeviceKernel, DeviceUnsupported, ElementalFn


def _device_only(nb, env):
    raise DeviceUnsupported("sobel_kernel runs only as the sm_100a u8 stencil")


sobel_kernel = ElementalFn(point=_device_only, k=1, block=None, pad_mode="constant", pad_value=0,
                           device=DeviceKernel("sobel"))


def _pixel_sum() -> Combinator:
    """Sum of output magnitudes (apps/sobel.py:73-74)."""
    import numpy as np

    return Combinator(lambda a, b: a + b, 0, on_array=lambda arr: int(np.sum(arr)), kind="sum")


def sobel_filter(img: Grid, *, partitions: int = 1, mode=DeploymentMode.ONE_TO_N,
                 group: Optional[WorkerGroup] = None, with_report: bool = False):
    """Edge-magnitude image of an 8-bit grid (apps/sobel.py:77-94)."""
    if img.ndim != 2:
        raise GridError("sobel expects a 2D image")
    if partitions == 1:
        mode = DeploymentMode.ONE_TO_ONE
    # pixel range is validated on the device copy (GridError outside [0, 255])
    out, report = parallel_loop(mode, partitions, 1, sobel_kernel, _pixel_sum(), stop_after(1),
                                img, group=group)
    return (out, report) if with_report else out


def sobel_frames(frames, out=None, stream=None):
    """Batched Sobel over a [F, H, W] uint8 CUDA tensor (one launch).

    Returns (edges [F, H, W] uint8, per-frame pixel sums [F] int64), both on
    the device.  Row pitch and frame stride must be multiples of 8 bytes.
    """
    import torch

    lib = N.require_cuda()
    if frames.dtype != torch.uint8 or frames.dim() != 3 or not frames.is_cuda:
        raise GridError("sobel_frames expects a [F, H, W] uint8 CUDA tensor")
    F, H, W = frames.shape
    if out is None:  # rows padded to 16 bytes (the kernels' pitch rule)
        Wp = -(-frames.shape[2] // 16) * 16
        out = torch.empty((frames.shape[0], frames.shape[1], Wp), dtype=torch.uint8,
                          device=frames.device)[:, :, :frames.shape[2]]
    sums = torch.empty(F, dtype=torch.int64, device=frames.device)
    st = stream if stream is not None else torch.cuda.current_stream()
    N.check(lib.sk_sobel_frames(C.c_void_p(frames.data_ptr()), frames.stride(1),
                                frames.stride(0), C.c_void_p(out.data_ptr()), out.stride(1),
                                out.stride(0), F, H, W, C.c_void_p(sums.data_ptr()),
                                N.stream_handle(st)))
    return out, sums


def _frame_u8(img):
    """One stream frame as a uint8 tensor (host or device), values checked
    in [0, 255] like sobel_filter's input."""
    import torch

    from ..partition import _u8_from

    if not isinstance(img, Grid):
        raise GridError(f"frames must be grids, got {type(img).__name__}")
    if img.ndim != 2:
        raise GridError("sobel expects a 2D image")
    t0 = img._t if img._src == "t" else None
    if t0 is not None and t0.dtype == torch.uint8:
        return t0
    dev = img._t.device if img.is_device else torch.device("cpu")
    return _u8_from(img, "sobel", 0, 255, dev)


def sobel_stream(frames, *, writer=None, loader=None, width: int = 32, devices=None,
                 host_buffers: bool = False, workers_per_device: int = 2) -> StreamReport:
    """Stream mode of the Sobel filter (BASELINE C2): read -> ordered farm of
    the batched Sobel (sobel_frames, one launch per batch of width/2 frames;
    `workers_per_device` batches in flight per GPU, so uploads, launches and
    read-backs overlap on both PCIe directions) -> write, in stream order
    (streams.batch_farm).  Each frame is an 8-bit image Grid; the writer
    receives its edge image (the same values sobel_filter returns) as a Grid
    -- with host_buffers=True over a recycled pinned host frame filled by
    one DMA (`g.tensor()` is that uint8 tensor, valid during the call)."""
    import numpy as np
    import torch

    N.require_cuda()

    def run_batch(d, stream):
        n, h, w = d.shape
        if w % 16:  # sobel_frames' row pitch: whole 16-byte vectors
            p = torch.zeros((n, h, -(-w // 16) * 16), dtype=torch.uint8, device=d.device)
            p[:, :, :w] = d
            d = p[:, :, :w]
        out, _sums = sobel_frames(d, stream=stream)
        return [out[i] for i in range(n)]

    return batch_farm(frames, _frame_u8, run_batch, writer=writer, loader=loader,
                      devices=devices, batch=max(1, min(512, width // 2)),
                      host_buffers=host_buffers, logical_dtype=np.int64, compute_name="sobel",
                      workers_per_device=workers_per_device)
