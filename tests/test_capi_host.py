"""CPU tests of the C-ABI library (no GPU needed): it loads, exports every
entry point include/sglgpu.h declares, validates arguments like the reference
(sgl_transform.cpp:18-35) and reports the missing device loudly (no CPU
fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1604_05140_b200 as sgl
from conftest import gpu_available

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(REPO, "include", "sglgpu.h")).read()
    return sorted(set(re.findall(r"\b(sglgpu_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("sglgpu_plan_create", "sglgpu_plan_destroy", "sglgpu_forward", "sglgpu_inverse",
                 "sglgpu_last_error", "sglgpu_spherical_forward", "sglgpu_radial_forward"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    L = sgl.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", sgl.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", sgl.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", sgl.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # fp64 tensor-core contractions
    assert "LDGSTS" in sass       # cp.async staging
    assert "UTMALDG" in sass      # TMA tensor loads (the Legendre forward's B tiles)


def test_cpp_api_symbols_exported():
    out = subprocess.run(["nm", "-DC", "--defined-only", sgl.LIB_PATH], capture_output=True, text=True).stdout
    for sym in ("sgl::fsglft(", "sgl::ifsglft(", "sgl::TransformPlan::compute(", "sgl::TransformPlan::from_tables(",
                "sgl::roundtrip_error("):
        assert sym in out, sym


@pytest.mark.skipif(gpu_available(), reason="checks the no-device error path")
def test_no_device_fails_loudly():
    plan = sgl.TransformPlan.compute(4)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        plan.handle


def test_plan_argument_validation():
    L = sgl.lib()
    d = sgl._PlanDesc(0, None, None, None, -1)
    h = ctypes.c_void_p()
    assert L.sglgpu_plan_create(ctypes.byref(d), ctypes.byref(h)) == sgl.SGLGPU_EINVAL
    r = np.array([0.5, 0.4, 1.0, 2.0])  # not increasing
    am = np.ones(4)
    d = sgl._PlanDesc(2, r.ctypes.data, am.ctypes.data, None, -1)
    assert L.sglgpu_plan_create(ctypes.byref(d), ctypes.byref(h)) == sgl.SGLGPU_EINVAL
    assert b"increasing" in L.sglgpu_last_error()
    assert L.sglgpu_forward(None, None, None, 1, 0, None) == sgl.SGLGPU_EINVAL
    # the fused-exchange entry points validate before touching a device
    assert L.sglgpu_radial_forward_to(None, None, 0, 1, 1, 1, 1, None, None) == sgl.SGLGPU_EINVAL
    assert L.sglgpu_radial_inverse_to(None, None, 0, 1, 1, 1, 1, None, None) == sgl.SGLGPU_EINVAL


def test_transform_shape_errors_match_reference_messages():
    plan = sgl.TransformPlan.compute(2)
    with pytest.raises(ValueError, match="sample grid must have length 8B\\^3"):
        sgl.fsglft(sgl.SampleGrid(2, np.zeros(10, complex)), plan)
    with pytest.raises(ValueError, match="coefficient and plan bandlimits disagree"):
        sgl.ifsglft(sgl.SglCoefficients(3, np.zeros(sgl.coefficient_count(3), complex)), plan)
    with pytest.raises(ValueError, match="grid and plan bandlimits disagree"):
        sgl.fsglft(sgl.SampleGrid(3, np.zeros(sgl.sample_count(3), complex)), plan)


def test_layout_helpers():
    assert sgl.sample_count(64) == 8 * 64 ** 3
    assert sgl.coefficient_count(64) == 89440  # test_indexing.cpp:11-20
    assert sgl.omega_index(1, 0, 0) == 0
    assert sgl.omega_index(2, 1, 1) == 4
    seen = set()
    for n in range(1, 5):
        for l in range(n):
            for m in range(-l, l + 1):
                seen.add(sgl.omega_index(n, l, m))
    assert seen == set(range(sgl.coefficient_count(4)))


def test_roundtrip_error_semantics():
    e = sgl.roundtrip_error(np.array([1.0 + 0j]), np.array([1.5 + 0j]))
    assert e.max_abs == pytest.approx(0.5) and e.max_rel == pytest.approx(0.5) and e.skipped_zero == 0
    e = sgl.roundtrip_error(np.array([0.0, 2.0]), np.array([1e-3, 2.0]))
    assert e.skipped_zero == 1 and e.max_rel == 0.0
    e = sgl.roundtrip_error(np.array([1.0, 1.0]), np.array([np.nan, 1.0]))
    assert e.nonfinite == 1  # the reference's std::max is NaN-blind (sgl_transform.cpp:355-363)
    with pytest.raises(ValueError):
        sgl.roundtrip_error(np.zeros(3), np.zeros(2))
