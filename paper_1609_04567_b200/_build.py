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


def _compile(src: str, obj: str) -> subprocess.CompletedProcess:
    cmd = [nvcc(), *NVCC_FLAGS, "-I", GEN, "-c", "-o", obj, os.path.join(CSRC, src)]
    return subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)


def build(verbose: bool = False, force: bool = False) -> str:
    """Compile every source to an object in parallel (no cross-file device
    symbols, so no relocatable device code), then link the shared library."""
    from concurrent.futures import ThreadPoolExecutor

    out = lib_path()
    if not force and not needs_build():
        return out
    os.makedirs(LIBDIR, exist_ok=True)
    write_jit_headers()
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in SOURCES]
    # an object is reused only when it is newer than its source and every
    # header (force rebuilds everything)
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".cu")]
    hdrs += [os.path.join(ROOT, "include", "stencilkit_b200.h"), os.path.abspath(__file__)]
    newest_hdr = max(os.path.getmtime(h) for h in hdrs if os.path.exists(h))
    todo = [(s, o) for s, o in zip(SOURCES, objs)
            if force or not os.path.exists(o)
            or os.path.getmtime(o) < max(newest_hdr, os.path.getmtime(os.path.join(CSRC, s)))]
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as pool:
        results = list(pool.map(lambda so: _compile(*so), todo))
    log = "".join(r.stdout + r.stderr for r in results)
    bad = [so[0] for so, r in zip(todo, results) if r.returncode != 0]
    if bad:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed building {LIBNAME} ({', '.join(bad)})")
    tmp = out + ".tmp"
    res = subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                          "-o", tmp, *objs, "-ldl"],
                         cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking " + LIBNAME)
    if verbose:
        sys.stderr.write(log)
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as fh:
        fh.write(log)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
