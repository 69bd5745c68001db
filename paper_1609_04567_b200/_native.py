"""ctypes binding of the native engine (include/stencilkit_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
device entry point raises `DeviceUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import _build

SK_OK, SK_ERR_ARG, SK_ERR_CUDA, SK_ERR_STATE, SK_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
SK_U8, SK_F32, SK_F64 = 1, 3, 4
SK_I32, SK_I64 = 2, 5  # sk_reduce_fold only
SK_KERNEL_HELMHOLTZ, SK_KERNEL_SOBEL, SK_KERNEL_AMF, SK_KERNEL_RESTORE, SK_KERNEL_LIFE = 1, 2, 3, 4, 5
SK_KERNEL_JIT = 6
SK_REDUCE_SUM, SK_REDUCE_MAX, SK_REDUCE_CUSTOM = 1, 2, 3
SK_DELTA_NONE, SK_DELTA_ABS, SK_DELTA_SQUARE = 0, 1, 2
SK_COND_HOST, SK_COND_LT, SK_COND_RMS_LT, SK_COND_MEAN_LT, SK_COND_ITER_GE = 0, 1, 2, 3, 4
SK_COND_MEAN_FLAGGED_LT = 5
SK_FLAG_TIMING = 1
SK_FLAG_FRAMES = 2

# every symbol include/stencilkit_b200.h declares
EXPORTS = (
    "sk_last_error", "sk_abi_version", "sk_run_begin", "sk_run_launch", "sk_run_value",
    "sk_run_loop", "sk_run_result", "sk_run_value_ptr", "sk_run_combine", "sk_run_status",
    "sk_run_frame_status",
    "sk_run_kernel_time",
    "sk_run_launches", "sk_run_destroy", "sk_verify_div_f32", "sk_sobel_frames",
    "sk_amf_frames", "sk_jit_compile", "sk_jit_log", "sk_jit_cubin_size", "sk_jit_cubin", "sk_jit_destroy",
    "sk_run_begin_jit", "sk_run_error",
    "sk_run_set_peers", "sk_run_peer_wait", "sk_run_exchange_rows", "sk_ipc_alloc", "sk_ipc_handle", "sk_ipc_open",
    "sk_ipc_close", "sk_ipc_free", "sk_reduce_fold",
)

SK_MAX_PEERS = 8


class DeviceUnavailable(RuntimeError):
    """The native library or a CUDA device is missing; there is no fallback."""


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"stencilkit_b200 error {code}: {msg}")


class sk_plan(C.Structure):
    _fields_ = [
        ("kernel", C.c_int32), ("dtype", C.c_int32),
        ("rows", C.c_int64), ("cols", C.c_int64),
        ("partitions", C.c_int32), ("reduce_op", C.c_int32), ("delta_op", C.c_int32),
        ("halo_top", C.c_int32), ("halo_bottom", C.c_int32), ("flags", C.c_int32),
        ("identity", C.c_double), ("params", C.c_double * 8),
    ]


class sk_cond(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad", C.c_int32), ("a", C.c_double), ("n", C.c_double),
                ("max_iterations", C.c_int64)]


class sk_peers(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32),
                ("up_rows", C.c_void_p * 2), ("down_rows", C.c_void_p * 2),
                ("mail", C.c_void_p * SK_MAX_PEERS), ("flags", C.c_void_p * SK_MAX_PEERS)]


_lock = threading.Lock()
_lib = None


def lib_path() -> str:
    # SK_LIB_PATH: load an alternative build (kernel-variant experiments)
    return os.environ.get("SK_LIB_PATH") or _build.lib_path()


def load(build_if_missing: bool = True):
    """Load (building in-tree first if needed) and return the ctypes CDLL."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if build_if_missing and path == _build.lib_path() and _build.needs_build():
            try:
                _build.build()
            except Exception as e:  # no toolkit here: only a prebuilt .so can work
                if not os.path.exists(path):
                    raise DeviceUnavailable(f"cannot build {path}: {e}") from e
        if not os.path.exists(path):
            raise DeviceUnavailable(f"native library missing: {path}")
        lib = C.CDLL(path)
        _declare(lib)
        _lib = lib
        return lib


def _declare(lib):
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    lib.sk_last_error.restype = C.c_char_p
    lib.sk_abi_version.restype = C.c_int
    sig = {
        "sk_run_begin": [C.POINTER(sk_plan), P, I64, P, I64, P, P, I64, P, C.POINTER(P)],
        "sk_run_launch": [P, I32],
        "sk_run_value": [P, I64, C.POINTER(D)],
        "sk_run_loop": [P, C.POINTER(sk_cond), C.POINTER(I64), C.POINTER(D), C.POINTER(I32)],
        "sk_run_result": [P, I64, C.POINTER(I32)],
        "sk_run_value_ptr": [P, C.POINTER(P)],
        "sk_run_combine": [P, P, I32, C.POINTER(sk_cond)],
        "sk_run_status": [P, C.POINTER(I64), C.POINTER(D), C.POINTER(I32), C.POINTER(I32)],
        "sk_run_frame_status": [P, C.POINTER(I64), C.POINTER(D), C.POINTER(I32)],
        "sk_run_kernel_time": [P, C.POINTER(D), C.POINTER(I64)],
        "sk_run_launches": [P, C.POINTER(I64)],
        "sk_run_destroy": [P],
        "sk_sobel_frames": [P, I64, I64, P, I64, I64, I32, I64, I64, P, P],
        "sk_amf_frames": [P, I64, I64, P, I64, I64, I32, I64, I64, I32, P, P],
        "sk_jit_compile": [C.c_char_p, C.c_char_p, C.POINTER(P)],
        "sk_jit_destroy": [P],
        "sk_jit_cubin": [P, P],
        "sk_run_begin_jit": [C.POINTER(sk_plan), P, P, I64, C.POINTER(P), C.POINTER(I64), I32, P, P,
                             I64, P, C.POINTER(P)],
        "sk_run_error": [P, C.POINTER(I32), C.POINTER(I64), C.POINTER(I64)],
        "sk_run_set_peers": [P, C.POINTER(sk_peers)],
        "sk_run_peer_wait": [P, I64],
        "sk_run_exchange_rows": [P, P, I64, I64, I64],
        "sk_reduce_fold": [P, I64, I32, I32, P, P, P],
        "sk_ipc_alloc": [I64, C.POINTER(P)],
        "sk_ipc_handle": [P, C.c_char_p],
        "sk_ipc_open": [C.c_char_p, C.POINTER(P)],
        "sk_ipc_close": [P],
        "sk_ipc_free": [P],
    }
    lib.sk_jit_log.argtypes = [P]
    lib.sk_jit_log.restype = C.c_char_p
    lib.sk_jit_cubin_size.argtypes = [P]
    lib.sk_jit_cubin_size.restype = C.c_int64
    lib.sk_verify_div_f32.argtypes = [C.c_float, P]
    lib.sk_verify_div_f32.restype = C.c_longlong
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int


def check(rc: int):
    if rc != SK_OK:
        msg = _lib.sk_last_error().decode(errors="replace") if _lib is not None else "?"
        raise NativeError(rc, msg)


_cuda_ok = False


def require_cuda():
    """Raise DeviceUnavailable unless a CUDA device and the library are present
    (the device check runs until it first succeeds: it is per-call overhead
    on every loop)."""
    global _cuda_ok
    if not _cuda_ok:
        import torch

        if not torch.cuda.is_available():
            raise DeviceUnavailable("no CUDA device: stencilkit_b200 runs only on the GPU")
        _cuda_ok = True
    return load()


def stream_handle(stream) -> C.c_void_p:
    return C.c_void_p(stream.cuda_stream if stream is not None else 0)
