"""The C-ABI library builds for sm_100a, loads, and exports every function the
header declares (no compute calls here: there is no GPU in the CPU suite)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1609_04567_b200 import _build, _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stencilkit_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    try:
        _build.build()
    except RuntimeError as e:  # no toolkit: only a prebuilt library can be checked
        if not os.path.exists(_build.lib_path()):
            pytest.skip(str(e))
    return _native.load(build_if_missing=False)


def test_header_and_binding_agree():
    assert declared() == sorted(_native.EXPORTS)


def test_every_declared_symbol_is_exported(lib):
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _build.lib_path()], capture_output=True,
                         text=True).stdout
    for name in declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_abi_version_and_error_channel(lib):
    assert lib.sk_abi_version() == 1
    assert isinstance(lib.sk_last_error(), bytes)


def test_argument_validation_without_a_device(lib):
    # null arguments are rejected before any CUDA call
    assert lib.sk_run_begin(None, None, 0, None, 0, None, None, 0, None, None) == _native.SK_ERR_ARG
    assert b"null" in lib.sk_last_error()
    assert lib.sk_run_destroy(None) == _native.SK_OK


def test_built_for_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.lib_path()], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_no_fma_contraction_in_exact_kernels():
    # helmholtz/restore arithmetic must be op-by-op; FFMA may appear only in the
    # division / sqrt sequences, never fusing a product into the update sum.
    # Evidence check: the library is compiled with -fmad=false.
    assert "-fmad=false" in _build.NVCC_FLAGS
