"""CPU tests: pin the oracle (oracle/sgl_oracle.c) before trusting it.

1. Against the committed golden fixtures produced by the reference itself
   (tests/golden/make_golden.py).
2. Against the reference's own known-answer tests, restated:
   exactness on sampled basis functions (test_sgl_transform.cpp:176-191,
   acceptance criterion 1), unit coefficient -> pi^{-3/4} grid (:127-146),
   unit omega(2,1,0) inverse = sampled basis (:205-214), linearity (:238-255),
   Parseval (:257-279), zero -> zero (:216-236), matrix semantics at B = 2
   (:303-346), the acceptance suite's round-trip bounds (criterion 3).
3. Live against the reference library when oracle/_ref was built here.
4. The oracle stays valid where the reference breaks (B = 128, 256; SURVEY.md
   section 0): finite outputs and a round trip at fp64 accuracy.
"""
import json
import os

import numpy as np
import pytest

from oracle_bindings import (Oracle, Reference, coefficient_count, normwise, omega_index, per_shell, psi_index,
                             sample_count)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.fromfile(os.path.join(GOLDEN, name), dtype="<f8").view(np.complex128)


_orc = {}


def orc(B):
    if B not in _orc:
        _orc[B] = Oracle(B)
    return _orc[B]


def test_golden_manifest_integrity():
    import hashlib

    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        man = json.load(f)
    for name, meta in man.items():
        if not name.endswith(".bin"):
            continue
        with open(os.path.join(GOLDEN, name), "rb") as f:
            assert hashlib.sha256(f.read()).hexdigest() == meta["sha256"], name


@pytest.mark.parametrize("B", [2, 4, 8, 16])
def test_oracle_matches_reference_golden(B):
    c = load(f"rt_B{B}_coeffs.bin")
    g_ref = load(f"rt_B{B}_grid.bin")
    back_ref = load(f"rt_B{B}_back.bin")
    # the golden coefficients are the acceptance suite's draw
    assert np.array_equal(c, Oracle.random_coefficients(B, 1000 + 10 * B))
    o = orc(B)
    g = o.inverse(c, threads=1)
    assert per_shell(g, g_ref, B) < 1e-13
    assert normwise(o.forward(g_ref, threads=1), back_ref) < 1e-13
    assert normwise(back_ref, c) < 1e-12  # the reference's own round trip


def test_oracle_matrix_semantics_golden_b2():
    B = 2
    o = orc(B)
    mat = load("mat_B2_forward.bin").reshape(sample_count(B), coefficient_count(B))
    for p in range(sample_count(B)):
        e = np.zeros(sample_count(B), dtype=np.complex128)
        e[p] = 1.0
        assert np.abs(o.forward(e) - mat[p]).max() < 1e-12


def test_oracle_matrix_semantics_closed_form_b2():
    """fsglft == explicit matrix conj(H) e^{-r^2} a_mod b_cal (test_sgl_transform.cpp:303-330)."""
    B = 2
    o = orc(B)
    for p in range(sample_count(B)):
        e = np.zeros(sample_count(B), dtype=np.complex128)
        e[p] = 1.0
        col = o.forward(e)
        i, rest = divmod(p, 4 * B * B)
        j, k = divmod(rest, 2 * B)
        w = np.exp(-o.r[i] ** 2) * o.a_mod[i] * o.b_cal[j]
        for n in range(1, B + 1):
            for l in range(n):
                for m in range(-l, l + 1):
                    h = Oracle.sgl_basis(n, l, m, o.r[i], o.theta[j], o.phi[k])
                    assert abs(col[omega_index(n, l, m)] - np.conj(h) * w) < 1e-12


def test_oracle_unit_basis_b3_golden():
    B = 3
    u = np.zeros(coefficient_count(B), dtype=np.complex128)
    u[omega_index(2, 1, 0)] = 1.0
    g = orc(B).inverse(u)
    assert np.abs(g - load("basis_B3_210.bin")).max() < 1e-11
    assert np.abs(g - orc(B).sample_basis(2, 1, 0)).max() < 1e-11


@pytest.mark.parametrize("B", [2, 4])
def test_oracle_exact_on_sampled_basis(B):
    o = orc(B)
    for n in range(1, B + 1):
        for l in range(n):
            for m in range(-l, l + 1):
                c = o.forward(o.sample_basis(n, l, m))
                target = np.zeros_like(c)
                target[omega_index(n, l, m)] = 1.0
                assert np.abs(c - target).max() < 1e-10


def test_oracle_unit_coefficient_is_constant_grid():
    B = 2
    u = np.zeros(coefficient_count(B), dtype=np.complex128)
    u[0] = 1.0
    g = orc(B).inverse(u)
    assert np.abs(g - np.pi ** -0.75).max() < 1e-12


def test_oracle_zero_and_linearity():
    B = 4
    o = orc(B)
    assert not np.abs(o.forward(np.zeros(sample_count(B), complex))).any()
    assert not np.abs(o.inverse(np.zeros(coefficient_count(B), complex))).any()
    rng = np.random.default_rng(41)
    g1 = rng.uniform(-1, 1, sample_count(B)) + 1j * rng.uniform(-1, 1, sample_count(B))
    g2 = rng.uniform(-1, 1, sample_count(B)) + 1j * rng.uniform(-1, 1, sample_count(B))
    alpha = 1.4 - 0.3j
    assert np.abs(o.forward(alpha * g1 + g2) - (alpha * o.forward(g1) + o.forward(g2))).max() < 1e-11


@pytest.mark.parametrize("B", [2, 4, 8])
def test_oracle_parseval(B):
    o = orc(B)
    c = Oracle.random_coefficients(B, 600 + B)
    g = o.inverse(c).reshape(2 * B, 2 * B, 2 * B)
    w = (o.a * o.r ** 2)[:, None, None] * o.b_cal[None, :, None]
    assert abs((w * np.abs(g) ** 2).sum() / (np.abs(c) ** 2).sum() - 1.0) < 1e-9


@pytest.mark.parametrize("B", [2, 4, 8, 16, 32])
def test_oracle_roundtrip_protocol(B):
    """Acceptance criterion 3 (acceptance_main.cpp:184-205): mean max-abs < 1e-8, max-rel < 1e-6."""
    o = orc(B)
    abs_err, rel_err = [], []
    for rep in range(3):
        c = Oracle.random_coefficients(B, 4200 + B + rep)
        back = o.forward(o.inverse(c))
        abs_err.append(np.abs(back - c).max())
        rel_err.append((np.abs(back - c) / np.abs(c)).max())
    assert np.mean(abs_err) < 1e-8 and np.mean(rel_err) < 1e-6


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("B", [1, 2, 3, 5, 8, 16, 32, 64])
def test_oracle_matches_reference_live(B):
    ref, o = Reference(B), orc(B)
    assert np.array_equal(ref.b_cal, o.b_cal)
    rng = np.random.default_rng(B)
    n = coefficient_count(B)
    c = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2)
    g_ref = ref.inverse(c)
    assert per_shell(o.inverse(c), g_ref, B) < 1e-13
    assert normwise(o.forward(g_ref), ref.forward(g_ref)) < 1e-13


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_stage_functions_match_reference():
    B = 8
    ref, o = Reference(B), orc(B)
    rng = np.random.default_rng(3)
    for l in (0, 3, B - 1):
        s = rng.standard_normal(2 * B) + 1j * rng.standard_normal(2 * B)
        assert np.abs(o.drt_forward(l, s) - ref.drt_forward(l, s)).max() < 1e-13 * max(1, np.abs(ref.drt_forward(l, s)).max())
        t = rng.standard_normal(B - l) + 1j * rng.standard_normal(B - l)
        r_inv = ref.drt_inverse(l, t)
        assert np.abs(o.drt_inverse(l, t) - r_inv).max() < 1e-13 * np.abs(r_inv).max()
    samples = rng.standard_normal(4 * B * B) + 1j * rng.standard_normal(4 * B * B)
    assert normwise(o.sft_forward(samples), ref.sft_forward(samples)) < 1e-13


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built (needs /root/reference)")
def test_reference_breaks_at_b128_but_oracle_does_not():
    """the reference loses coefficients with l+|m| >~ 172 at B = 128."""
    B = 128
    ref, o = Reference(B), orc(B)
    rng = np.random.default_rng(0)
    n = coefficient_count(B)
    c = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2)
    g = o.inverse(c)
    assert np.isfinite(g).all()
    assert normwise(o.forward(g), c) < 1e-13
    bad = np.abs(ref.forward(g) - c) > 1e-6
    assert bad.sum() > 10000  # the reference's M_lm underflow (special_functions.cpp:81-88)


def test_oracle_valid_at_b128():
    B = 128
    o = orc(B)
    rng = np.random.default_rng(1)
    n = coefficient_count(B)
    c = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2)
    g = o.inverse(c)
    assert np.isfinite(g).all()
    assert normwise(o.forward(g), c) < 1e-12


def _lm_of_omega(B):
    """(l, |m|) of every omega-order entry (indexing.cpp:50-78)."""
    ls, ms = [], []
    for n in range(1, B + 1):
        for l in range(n):
            ls += [l] * (2 * l + 1)
            ms += list(range(-l, l + 1))
    return np.array(ls), np.abs(np.array(ms))


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_pinned_to_reference_b128_representable_subset():
    """Pins the oracle to the reference itself at B = 128 where the reference is
    valid: M_lm (special_functions.cpp:81-88) stays representable for
    l + |m| <~ 172, so on entries with l + |m| <= 160 the reference's fsglft /
    ifsglft (sgl_transform.cpp:274-348) are exact and must agree with the
    restatement.  Forward: every output coefficient depends only on its own
    (l, m) row, so the valid rows are compared on a full random grid.  Inverse:
    inputs supported on the valid rows only (the reference's underflowed rows are
    zero, not NaN, at B = 128)."""
    B = 128
    ref, o = Reference(B), orc(B)
    assert np.array_equal(ref.b_cal, o.b_cal)
    l, am = _lm_of_omega(B)
    ok = l + am <= 160
    assert ok.sum() > 0.85 * ok.size  # 633,568 of 707,264
    rng = np.random.default_rng(128)
    n = coefficient_count(B)
    c = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2)
    g = o.inverse(c)
    f_ref = ref.forward(g)
    f_orc = o.forward(g)
    assert np.isfinite(f_ref[ok]).all()
    assert normwise(f_orc[ok], f_ref[ok]) <= 1e-12
    c_ok = np.where(ok, c, 0)
    g_ref = ref.inverse(c_ok)
    assert np.isfinite(g_ref).all()
    assert per_shell(o.inverse(c_ok), g_ref, B) <= 1e-12
