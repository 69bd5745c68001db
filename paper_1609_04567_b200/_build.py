"""Build the native library in-tree with nvcc for sm_100a.

    python -m paper_1609_04567_b200._build

Produces paper_1609_04567_b200/_lib/libstencilkit_b200.so.  Plain nvcc (no
torch extension machinery): the library's ABI is the C header in
include/stencilkit_b200.h, with no torch types in any signature.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIBNAME = "libstencilkit_b200.so"

SOURCES = [
    "sk_runtime.cu",
    "sk_helmholtz.cu",
    "sk_verify.cu",
    "sk_u8stencil.cu",
    "sk_amf.cu",
    "sk_restore.cu",
    "sk_dispatch.cu",
]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # the reference's arithmetic is op-by-op (no FMA); kernels also use
    # explicit _rn intrinsics, this keeps any stray expression honest
    "-fmad=false",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build")
    return cand


def lib_path() -> str:
    return os.path.join(LIBDIR, LIBNAME)


def needs_build() -> bool:
    out = lib_path()
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "stencilkit_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose: bool = False, force: bool = False) -> str:
    out = lib_path()
    if not force and not needs_build():
        return out
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = out + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, "-shared", "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building " + LIBNAME)
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as fh:
        fh.write(res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
