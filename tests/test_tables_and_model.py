"""CPU tests of the plan-time data and of the device algorithm's math.

* Radial rules (paper_1604_05140_b200/tables/*.sglt, mpmath restatement of
  quadrature.cpp:133-227): CRC, pinned N = 1 values (test_quadrature.cpp:85-92),
  moment exactness (:94-106), interlacing-free monotone nodes, a_mod consistency
  (:142-155), reproducibility of the generator.
* Device tables (libsglb200 host generator, long double): normalized Legendre
  rows against the oracle's closed-form basis; radial rows against the closed-form
  Laguerre route; no overflow/NaN at B = 256.
* The numpy model of the CUDA algorithm (tests/device_model.py: equatorial fold,
  (|m|, parity) grouping, nu-major S, per-l radial GEMMs) against the oracle.
"""
import os

import mpmath as mp
from scipy.special import sph_harm_y
import numpy as np
import pytest

import paper_1604_05140_b200 as sgl
from device_model import DeviceModel, host_tables
from oracle_bindings import Oracle, Reference, coefficient_count, normwise, per_shell, sample_count

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

TABLES = os.path.join(os.path.dirname(sgl.__file__), "tables")
ALL_B = sorted(int(f[len("radial_rule_B"):-5]) for f in os.listdir(TABLES) if f.startswith("radial_rule_B"))


def test_committed_rules_cover_the_configs():
    for B in (1, 2, 3, 4, 8, 16, 32, 64, 128, 256):
        assert B in ALL_B


def test_rule_n1_pinned_values():
    rr = sgl.load_radial_rule(os.path.join(TABLES, "radial_rule_B1.sglt"))
    r, a, am = rr.r, rr.a, rr.a_mod
    # the committed files hold even orders 2B; pin the N = 1 rule through the generator
    from paper_1604_05140_b200.tables.gen_radial_rules import rule as gen
    r1, a1, _ = gen(1)
    assert r1[0] == pytest.approx(1 / np.sqrt(np.pi), rel=1e-15)
    assert a1[0] == pytest.approx(np.sqrt(np.pi) / 2, rel=1e-15)
    assert r.size == 2 and np.all(np.diff(r) > 0) and np.all(a > 0) and np.all(am > 0)


@pytest.mark.parametrize("B", [1, 4, 16, 32])
def test_rule_moments(B):
    """sum a_i r_i^k = Gamma((k+1)/2)/2 for k < 4B (Gaussian exactness, 2N-1 = 4B-1)."""
    rr = sgl.load_radial_rule(os.path.join(TABLES, f"radial_rule_B{B}.sglt"))
    for k in range(0, 4 * B, max(1, B // 2)):
        s = mp.fsum(mp.mpf(ai) * mp.mpf(ri) ** k for ri, ai in zip(rr.r, rr.a))
        assert float(s / (mp.gamma((k + 1) / 2.0) / 2)) == pytest.approx(1.0, abs=1e-13)


@pytest.mark.parametrize("B", [8, 64, 256])
def test_rule_files_are_consistent(B):
    rr = sgl.load_radial_rule(os.path.join(TABLES, f"radial_rule_B{B}.sglt"))
    assert rr.order == 2 * B and np.all(np.diff(rr.r) > 0) and np.all(rr.a_mod > 0)
    # a_mod = a e^{r^2} r^2 where a is representable (quadrature.cpp:176, :229-235)
    ok = rr.a > 1e-280
    lhs = np.log(rr.a_mod[ok])
    rhs = np.log(rr.a[ok]) + rr.r[ok] ** 2 + 2 * np.log(rr.r[ok])
    assert np.abs(lhs - rhs).max() < 1e-12 * np.abs(rhs).max() + 1e-13


def test_generator_reproduces_committed_file():
    from paper_1604_05140_b200.tables.gen_radial_rules import rule as gen
    r, a, am = gen(2 * 6)
    rr = sgl.load_radial_rule(os.path.join(TABLES, "radial_rule_B6.sglt"))
    assert np.array_equal(np.array(r), rr.r) and np.array_equal(np.array(a), rr.a)
    assert np.array_equal(np.array(am), rr.a_mod)


def test_sglt_crc_is_checked(tmp_path):
    src = os.path.join(TABLES, "radial_rule_B4.sglt")
    data = bytearray(open(src, "rb").read())
    data[20] ^= 0xFF
    bad = tmp_path / "radial_rule_B4.sglt"
    bad.write_bytes(bytes(data))
    with pytest.raises(RuntimeError, match="checksum"):
        sgl.load_radial_rule(str(bad))


@pytest.mark.parametrize("B", [4, 7, 16])
def test_device_legendre_table_matches_closed_form(B):
    o = Oracle(B)
    t = host_tables(B, o.r, o.a_mod, o.b_cal)
    theta = o.theta
    ls = B + (B & 1)  # rows padded to an even length, pad entry 0
    for am in range(B):
        for p in range(2):
            rows = max(0, (B - am - p + 1) // 2)
            assert t["leg_off"][2 * am + p] % 2 == 0  # 16-byte aligned rows
            blk = t["leg"][t["leg_off"][2 * am + p]:][:rows * ls].reshape(rows, ls)
            assert not blk[:, B:].any()
            blk = blk[:, :B]
            for row in range(rows):
                l = am + p + 2 * row
                # Y_l^am(theta, 0) = Pbar_l^am(cos theta), Condon-Shortley phase included
                ref = sph_harm_y(l, am, theta[:B], 0.0).real
                assert np.abs(blk[row] - ref).max() < 1e-13


@pytest.mark.parametrize("B", [1, 2, 7, 16, 33])
def test_table_offsets_closed_form(B):
    # the GEMM kernels compute these offsets in closed form instead of loading them
    # (sgl_kernels.cu leg_table_off / rad_table_off)
    o = Oracle(B)
    t = host_tables(B, o.r, o.a_mod, o.b_cal)
    ls = B + (B & 1)
    for pid in range(2 * B):
        am, p = pid >> 1, pid & 1
        assert t["leg_off"][pid] == ls * (am * B - am * (am - 1) // 2 + p * ((B - am + 1) // 2))
    for l in range(B):
        off = 2 * B * (l * B - l * (l - 1) // 2)
        assert t["W_off"][l] == off and t["V_off"][l] == off


def test_device_tables_finite_at_b256():
    o = Oracle(256)
    t = host_tables(256, o.r, o.a_mod, o.b_cal)
    for k in ("leg", "W", "V"):
        assert np.isfinite(t[k]).all(), k
    assert np.abs(t["V"]).max() < 1e300


@pytest.mark.parametrize("B", [1, 2, 3, 4, 8, 16])
def test_device_model_matches_oracle(B):
    o = Oracle(B)
    d = DeviceModel(B, o.r, o.a_mod, o.b_cal)
    rng = np.random.default_rng(B)
    n = coefficient_count(B)
    c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    g = o.inverse(c)
    assert per_shell(d.inverse(c), g, B) < 1e-13
    assert normwise(d.forward(g), o.forward(g)) < 1e-13
    x = rng.standard_normal(sample_count(B)) + 1j * rng.standard_normal(sample_count(B))
    assert normwise(d.forward(x), o.forward(x)) < 1e-13


@pytest.mark.parametrize("B", [4, 8])
def test_device_radial_tables_match_closed_form(B):
    """W_l[n][i] = N_nl R_nl(r_i) e^{-r_i^2} a_mod_i and V_l[n][i] = N_nl R_nl(r_i)
    (radial_transform.cpp:75-133) against the closed-form Laguerre route
    (special_functions.cpp:110-127)."""
    o = Oracle(B)
    t = host_tables(B, o.r, o.a_mod, o.b_cal)
    for l in range(B):
        W = t["W"][t["W_off"][l]:t["W_off"][l + 1]].reshape(B - l, 2 * B)
        V = t["V"][t["V_off"][l]:t["V_off"][l + 1]].reshape(B - l, 2 * B)
        y0 = np.sqrt((2 * l + 1) / (4 * np.pi))
        for q in range(B - l):
            n = l + 1 + q
            rad = np.array([Oracle.sgl_basis(n, l, 0, ri, 0.0, 0.0).real / y0 for ri in o.r])
            assert np.abs(V[q] - rad).max() < 1e-12 * max(1.0, np.abs(rad).max())
            w = rad * np.exp(-o.r ** 2) * o.a_mod
            assert np.abs(W[q] - w).max() < 1e-12 * max(1.0, np.abs(w).max())


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("B", [2, 7, 16, 64])
def test_cpp_mirror_plan_tables_against_reference_store(B, tmp_path):
    """TransformPlan::from_tables reads the SGLT kinds 1-3 the REFERENCE writes
    (precompute_store.cpp:160-237); the 4-argument assemble validates orders
    (sgl_transform.cpp:52-63); LegendreDctTable::build reproduces the
    reference's rows (spherical_transform.cpp:31-86); and the mirror's writers
    are byte-identical to the reference's.  Host only (no device plan)."""
    import filecmp
    import subprocess

    ref_dir, out_dir = tmp_path / "ref", tmp_path / "mirror"
    ref_dir.mkdir()
    Reference(B).save_tables(str(ref_dir))
    exe = tmp_path / "test_tables_mirror"
    lib = os.path.join(REPO, "paper_1604_05140_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(REPO, "include"),
                    os.path.join(REPO, "tests", "cpp", "test_tables_mirror.cpp"), "-L", lib, "-lsglb200",
                    "-Wl,-rpath," + lib, "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), str(ref_dir), str(B), str(out_dir)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    err = float(out.stdout.split("max_row_err")[1].split()[0])
    assert err < 1e-12, err  # the reference's own double recurrence: 1.7e-13 at B = 64
    for name in (f"radial_rule_B{B}.sglt", f"sphere_rule_B{B}.sglt", f"legendre_dct_B{B}.sglt"):
        assert filecmp.cmp(ref_dir / name, out_dir / name, shallow=False), name
