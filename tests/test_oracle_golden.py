"""The CPU oracle (oracle/stencil_oracle.py) reproduces the reference's own
outputs bit-for-bit on every committed fixture: this is what pins the oracle
(the fixtures come from running the real reference, tests/golden/make_golden.py)."""

import hashlib
import math

import numpy as np
import pytest

from oracle import stencil_oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_helmholtz_fp32(golden):
    for name in golden.cases("helmholtz"):
        m = golden.meta[name]
        f = golden[name + "/rhs"]
        c = O.helmholtz_consts(m["alpha"], m["dx"], m["dy"], m["relax"])
        tol, nm = m["tol"], f.size
        if m["reduce"] == "max":
            u, it, v, ex = O.helmholtz_loop(np.zeros_like(f), f, c, delta="abs", op="max",
                                            cond=lambda val, i: val < tol, P=m["P"])
        else:
            u, it, v, ex = O.helmholtz_loop(np.zeros_like(f), f, c, delta="sq", op="sum",
                                            cond=lambda val, i: math.sqrt(val / nm) < tol,
                                            P=m["P"])
        assert it == m["iterations"] and v == m["final_reduce"], name
        assert np.array_equal(u.view(np.uint32), golden[name + "/out"].view(np.uint32)), name


def test_helmholtz_fp64(golden):
    for name in golden.cases("helmholtz_solve"):
        m = golden.meta[name]
        f = golden[name + "/rhs"]
        u0 = golden[name + "/u0"] if golden.has(name + "/u0") else np.zeros_like(f)
        c = O.helmholtz_consts(m["alpha"], m["dx"], m["dy"], m["relax"])
        tol, nm = m["tol"], f.size
        u, it, v, ex = O.helmholtz_loop(u0, f, c, delta="sq", op="sum",
                                        cond=lambda val, i: math.sqrt(val / nm) < tol, P=m["P"])
        assert it == m["iterations"] and v == m["final_reduce"], name
        assert np.array_equal(u, golden[name + "/out"]), name


def test_sobel_amf_life(golden):
    for name in golden.cases("sobel"):
        o = O.sobel(golden[name + "/in"])
        assert np.array_equal(o, golden[name + "/out"]), name
        assert int(o.astype(np.int64).sum()) == golden.meta[name]["final_reduce"]
    for name in golden.cases("amf"):
        o = O.amf_detect(golden[name + "/in"], golden.meta[name]["wmax"])
        assert np.array_equal(o, golden[name + "/out"]), name
    for name in golden.cases("life"):
        a = golden[name + "/in"]
        for _ in range(golden.meta[name]["steps"]):
            a = O.life_step(a)
        assert np.array_equal(a, golden[name + "/out"]), name


def test_restore(golden):
    for name in golden.cases("restore"):
        m = golden.meta[name]
        if not golden.has(name + "/in"):
            continue
        u, it, v, ex = O.restore_loop(golden[name + "/in"], golden[name + "/mask"], P=m["P"],
                                      max_iterations=m["max_iterations"])
        assert (it, v, ex) == (m["iterations"], m["final_reduce"], m["exhausted"]), name
        assert np.array_equal(u, golden[name + "/out"]), name


def test_large_configs(golden_large):
    m = golden_large.meta["C1_helm_f32_max_unit_1024"]
    f = np.ones((1024, 1024), np.float32)
    u, it, v, _ = O.helmholtz_loop(np.zeros_like(f), f, O.helmholtz_consts(), delta="abs",
                                   op="max", cond=lambda val, i: val < 1e-4, P=8, threads=4)
    assert (it, v, sha(u)) == (m["iterations"], m["final_reduce"], m["sha"])
    img = np.random.default_rng(0).integers(0, 256, (2048, 2048))
    s = O.sobel(img)
    mm = golden_large.meta["C2_sobel_rng0_2048"]
    assert sha(s) == mm["sha"] and int(s.astype(np.int64).sum()) == mm["final_reduce"]
    noisy, _ = O.salt_pepper(O.gradient_image(512, 512), 0.5, seed=42)
    assert sha(O.amf_detect(noisy)) == golden_large.meta["C3_amf_grad50_512"]["sha"]


def test_input_generators_match_reference(golden):
    # the restore fixtures were built from salt_pepper(gradient_image(...)); the
    # oracle's generators must reproduce them exactly (same PCG64 stream)
    noisy, mask = O.salt_pepper(O.gradient_image(48, 40), 0.5, seed=42)
    assert np.array_equal(noisy.astype(np.uint8), golden["restore_grad50_48x40_P1/in"])
