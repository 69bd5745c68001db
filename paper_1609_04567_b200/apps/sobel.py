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
