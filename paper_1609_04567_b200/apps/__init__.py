"""The paper's workloads on the device engine (reference: apps/__init__.py)."""

from .denoise import (RestoreConfig, amf_detect, amf_frames, detect_kernel, restore_kernel,
                      restore_frames, restore_regularize, salt_pepper, video_restore_pipeline)
from .helmholtz import HelmholtzConfig, helmholtz_kernel, helmholtz_solve
from .life import GolConfig, game_of_life, life_kernel, liveness_op
from .sobel import sobel_filter, sobel_frames, sobel_kernel, sobel_stream

__all__ = [
    "GolConfig", "game_of_life", "life_kernel", "liveness_op",
    "HelmholtzConfig", "helmholtz_solve", "helmholtz_kernel",
    "sobel_filter", "sobel_kernel", "sobel_frames", "sobel_stream",
    "RestoreConfig", "amf_detect", "amf_frames", "detect_kernel", "restore_kernel",
    "restore_regularize", "restore_frames", "salt_pepper", "video_restore_pipeline",
]
