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
    "sk_sobel_tma.cu",
    "sk_reduce.cu",
    "sk_amf.cu",
    "sk_restore.cu",
    "sk_dispatch.cu",
    "sk_jit.cu",
]

# Headers NVRTC compiles user elemental programs against (embedded in the
# library, see sk_jit.cu), with the include names the sources use.
JIT_HEADERS = [
    ("../../include/stencilkit_b200.h", os.path.join(ROOT, "include", "stencilkit_b200.h")),
    ("sk_common.cuh", os.path.join(CSRC, "sk_common.cuh")),
    ("sk_sweep.cuh", os.path.join(CSRC, "sk_sweep.cuh")),
    ("sk_jit_prelude.cuh", os.path.join(CSRC, "sk_jit_prelude.cuh")),
    ("sk_jit_kernel.cuh", os.path.join(CSRC, "sk_jit_kernel.cuh")),
]
GEN = os.path.join(LIBDIR, "gen")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # the reference's arithmetic is op-by-op (no FMA); kernels also use
    # explicit _rn intrinsics, this keeps any stray expression honest
    "-fmad=false",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
    "-ldl",
]


def write_jit_headers() -> str:
    """Render JIT_HEADERS as C string tables (sk_jit_headers.inc)."""
    os.makedirs(GEN, exist_ok=True)
    names, srcs = [], []
    for name, path in JIT_HEADERS:
        with open(path) as fh:
            text = fh.read()
        delim = "SKJIT"
        assert f"){delim}\"" not in text
        names.append(f'"{name}"')
        # split into <= 8 KB raw-string pieces (compiler literal limits)
        parts = [text[i:i + 8000] for i in range(0, len(text), 8000)] or [""]
        srcs.append("\n".join(f'R"{delim}({p}){delim}"' for p in parts))
    out = os.path.join(GEN, "sk_jit_headers.inc")
    body = (f"static const int kJitHeaderCount = {len(names)};\n"
            f"static const char* const kJitHeaderNames[] = {{{', '.join(names)}}};\n"
            f"static const char* const kJitHeaderSrcs[] = {{\n" + ",\n".join(srcs) + "};\n")
    if not os.path.exists(out) or open(out).read() != body:
        with open(out, "w") as fh:
            fh.write(body)
    return out


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
    write_jit_headers()
    tmp = out + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, "-I", GEN, "-shared", "-o", tmp,
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
