"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (fp64, normwise as SURVEY.md section 8(d) recommends):
  coefficients: max|d| / max|ref| <= 1e-12
  grids:        max over shells of max|d| / max|ref| on that shell <= 1e-12
plus an explicit isfinite check (the reference's roundtrip_error is NaN-blind,
sgl_transform.cpp:355-363).
"""
import numpy as np
import pytest

import paper_1604_05140_b200 as sgl
from oracle_bindings import Oracle, coefficient_count, normwise, per_shell, sample_count

pytestmark = pytest.mark.gpu
TOL = 1e-12


def complex_normal(rng, n):
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2)


_plans = {}


def plan_for(B):
    if B not in _plans:
        _plans[B] = (sgl.TransformPlan.compute(B), Oracle(B))
    return _plans[B]


@pytest.mark.parametrize("B", [1, 2, 3, 4, 5, 8, 12, 16, 32, 64, 128])
def test_inverse_and_forward_match_oracle(B):
    plan, orc = plan_for(B)
    rng = np.random.default_rng(1000 + B)
    c = complex_normal(rng, coefficient_count(B))
    g_ref = orc.inverse(c)
    g = sgl.ifsglft(sgl.SglCoefficients(B, c), plan).values
    assert np.isfinite(g).all()
    assert per_shell(g, g_ref, B) <= TOL
    f_ref = orc.forward(g_ref)
    f = sgl.fsglft(sgl.SampleGrid(B, g_ref), plan).values
    assert np.isfinite(f).all()
    assert normwise(f, f_ref) <= TOL
    assert normwise(f, c) <= TOL  # round trip through the oracle grid


@pytest.mark.parametrize("B", [7, 9, 33])
def test_odd_bandlimit_batch_matches_oracle(B):
    # odd B: Legendre table rows padded to an even length (16-byte A units), the
    # naive DFT azimuthal kernels for non-power-of-two 2B, and a batch of three
    import torch

    plan, orc = plan_for(B)
    rng = np.random.default_rng(3000 + B)
    n, ns = coefficient_count(B), sample_count(B)
    c = np.stack([complex_normal(rng, n) for _ in range(3)])
    x = np.stack([complex_normal(rng, ns) for _ in range(3)])
    g = sgl.ifsglft_batch(plan, torch.from_numpy(c).cuda()).cpu().numpy()
    f = sgl.fsglft_batch(plan, torch.from_numpy(x).cuda()).cpu().numpy()
    for b in range(3):
        assert np.isfinite(g[b]).all() and np.isfinite(f[b]).all()
        assert per_shell(g[b], orc.inverse(c[b]), B) <= TOL
        assert normwise(f[b], orc.forward(x[b])) <= TOL


def test_forward_random_grid_matches_oracle():
    # a non-bandlimited input: every stage contributes
    for B in (4, 16, 32):
        plan, orc = plan_for(B)
        rng = np.random.default_rng(7 + B)
        g = complex_normal(rng, sample_count(B))
        assert normwise(sgl.fsglft(sgl.SampleGrid(B, g), plan).values, orc.forward(g)) <= TOL


@pytest.mark.parametrize("B", [16, 64])
def test_batched_device_matches_single(B):
    import torch

    plan, orc = plan_for(B)
    rng = np.random.default_rng(B)
    nb = 5
    c = complex_normal(rng, nb * coefficient_count(B)).reshape(nb, -1)
    dc = torch.from_numpy(c).cuda()
    dg = sgl.ifsglft_batch(plan, dc)
    db = sgl.fsglft_batch(plan, dg)
    torch.cuda.synchronize()
    g = dg.cpu().numpy()
    back = db.cpu().numpy()
    for b in range(nb):
        assert per_shell(g[b], orc.inverse(c[b]), B) <= TOL
        assert normwise(back[b], c[b]) <= TOL


def test_batched_b128_matches_single_function():
    # B = 128: the TMA-fed Legendre forward with several functions in G (the group
    # coordinate runs over the batch) against one-function calls
    import torch

    B = 128
    plan, _ = plan_for(B)
    rng = np.random.default_rng(128)
    nb = 3
    c = complex_normal(rng, nb * coefficient_count(B)).reshape(nb, -1)
    dg = sgl.ifsglft_batch(plan, torch.from_numpy(c).cuda())
    db = sgl.fsglft_batch(plan, dg).cpu().numpy()
    g = dg.cpu().numpy()
    for b in range(nb):
        g1 = sgl.ifsglft(sgl.SglCoefficients(B, c[b]), plan).values
        f1 = sgl.fsglft(sgl.SampleGrid(B, g[b]), plan).values
        assert per_shell(g[b], g1, B) <= 1e-14
        assert normwise(db[b], f1) <= 1e-14
        assert normwise(db[b], c[b]) <= TOL


def _c4_coefficients(B, seed, count=1):
    """BASELINE config C4: iid complex normal scaled by (1 + l)^-1."""
    rng = np.random.default_rng(seed)
    l = np.zeros(coefficient_count(B), dtype=int)
    for n in range(1, B + 1):
        for ll in range(n):
            s = sgl.omega_index(n, ll, -ll)
            l[s:s + 2 * ll + 1] = ll
    return np.stack([complex_normal(rng, coefficient_count(B)) / (1.0 + l) for _ in range(count)])


def test_b256_matches_oracle_both_directions():
    """Config C4 (B = 256) against the CPU oracle in each direction separately
    (a round trip alone would cancel an error common to both directions: a
    permuted omega / nu index, a conjugation, an odd-m sign).  Covers the
    paths only B = 256 takes: FFTShape<512> with doubled azimuthal CTAs and
    4-shell G groups, the Legendre inverse's K = 128 row-table limit and the
    radial forward's 512-row table."""
    B = 256
    plan, orc = plan_for(B)
    c = _c4_coefficients(B, 2560)[0]
    g_ref = orc.inverse(c)
    assert np.isfinite(g_ref).all()
    g = sgl.ifsglft(sgl.SglCoefficients(B, c), plan).values
    assert np.isfinite(g).all()
    assert per_shell(g, g_ref, B) <= TOL
    f_ref = orc.forward(g_ref)
    f = sgl.fsglft(sgl.SampleGrid(B, g_ref), plan).values
    assert np.isfinite(f).all()
    assert normwise(f, f_ref) <= TOL
    assert normwise(f, c) <= TOL
    # a non-bandlimited input (every row of every stage contributes)
    rng = np.random.default_rng(2561)
    x = complex_normal(rng, sample_count(B))
    assert normwise(sgl.fsglft(sgl.SampleGrid(B, x), plan).values, orc.forward(x)) <= TOL


def test_b256_batch_of_two_matches_oracle():
    import torch

    B = 256
    plan, orc = plan_for(B)
    c = _c4_coefficients(B, 2562, count=2)
    dg = sgl.ifsglft_batch(plan, torch.from_numpy(c).cuda())
    df = sgl.fsglft_batch(plan, dg)
    g = dg.cpu().numpy()
    f = df.cpu().numpy()
    del dg, df
    for b in range(2):
        g_ref = orc.inverse(c[b])
        assert np.isfinite(g[b]).all() and np.isfinite(f[b]).all()
        assert per_shell(g[b], g_ref, B) <= TOL
        assert normwise(f[b], orc.forward(g[b])) <= TOL
        assert normwise(f[b], c[b]) <= TOL


def test_roundtrip_b256():
    B = 256
    plan, orc = plan_for(B)
    rng = np.random.default_rng(256)
    l = np.zeros(coefficient_count(B), dtype=int)
    for n in range(1, B + 1):
        for ll in range(n):
            s = sgl.omega_index(n, ll, -ll)
            l[s:s + 2 * ll + 1] = ll
    c = complex_normal(rng, coefficient_count(B)) / (1.0 + l)  # BASELINE config C4 scaling
    g = sgl.ifsglft(sgl.SglCoefficients(B, c), plan).values
    assert np.isfinite(g).all()
    back = sgl.fsglft(sgl.SampleGrid(B, g), plan).values
    assert normwise(back, c) <= TOL


# ----------------------------------------------------------------- golden fixtures (reference outputs)
import os  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _gold(name):
    return np.fromfile(os.path.join(GOLDEN, name), dtype="<f8").view(np.complex128)


@pytest.mark.parametrize("B", [2, 4, 8, 16])
def test_gpu_matches_reference_golden(B):
    plan, _ = plan_for(B)
    c = _gold(f"rt_B{B}_coeffs.bin")
    g = sgl.ifsglft(sgl.SglCoefficients(B, c), plan).values
    assert per_shell(g, _gold(f"rt_B{B}_grid.bin"), B) <= 1e-13
    f = sgl.fsglft(sgl.SampleGrid(B, _gold(f"rt_B{B}_grid.bin")), plan).values
    assert normwise(f, _gold(f"rt_B{B}_back.bin")) <= 1e-13


def test_gpu_matrix_semantics_b2():
    """fsglft is the reference's matrix (test_sgl_transform.cpp:303-330), and ifsglft is
    the conjugate transpose of the weight-stripped forward (:332-345)."""
    import torch

    B = 2
    plan, orc = plan_for(B)
    mat = _gold("mat_B2_forward.bin").reshape(sgl.sample_count(B), sgl.coefficient_count(B))
    eye = torch.eye(sgl.sample_count(B), dtype=torch.complex128).cuda().contiguous()
    cols = sgl.fsglft_batch(plan, eye).cpu().numpy()
    assert np.abs(cols - mat).max() < 1e-12
    eye_c = torch.eye(sgl.coefficient_count(B), dtype=torch.complex128).cuda().contiguous()
    inv_cols = sgl.ifsglft_batch(plan, eye_c).cpu().numpy()  # [omega][psi]
    w = (np.exp(-orc.r ** 2) * orc.a_mod)[:, None, None] * orc.b_cal[None, :, None]
    w = np.broadcast_to(w, (2 * B, 2 * B, 2 * B)).reshape(-1)
    stripped = mat / w[:, None]
    assert np.abs(inv_cols - np.conj(stripped).T).max() < 1e-12


def test_gpu_exact_on_sampled_basis():
    """test_sgl_transform.cpp:176-191: fsglft(sampled H_nlm) = unit vector, B = 4."""
    import torch

    B = 4
    plan, orc = plan_for(B)
    grids, targets = [], []
    for n in range(1, B + 1):
        for l in range(n):
            for m in range(-l, l + 1):
                grids.append(orc.sample_basis(n, l, m))
                t = np.zeros(sgl.coefficient_count(B), dtype=np.complex128)
                t[sgl.omega_index(n, l, m)] = 1.0
                targets.append(t)
    out = sgl.fsglft_batch(plan, torch.from_numpy(np.stack(grids)).cuda()).cpu().numpy()
    assert np.abs(out - np.stack(targets)).max() < 1e-10


def test_gpu_unit_coefficient_b3_golden():
    B = 3
    plan, _ = plan_for(B)
    u = np.zeros(sgl.coefficient_count(B), dtype=np.complex128)
    u[sgl.omega_index(2, 1, 0)] = 1.0
    g = sgl.ifsglft(sgl.SglCoefficients(B, u), plan).values
    assert np.abs(g - _gold("basis_B3_210.bin")).max() < 1e-11


def test_gpu_zero_and_linearity():
    B = 8
    plan, _ = plan_for(B)
    z = sgl.fsglft(sgl.SampleGrid(B, np.zeros(sgl.sample_count(B), complex)), plan).values
    assert not np.abs(z).any()
    z = sgl.ifsglft(sgl.SglCoefficients(B, np.zeros(sgl.coefficient_count(B), complex)), plan).values
    assert not np.abs(z).any()
    rng = np.random.default_rng(3)
    g1, g2 = (complex_normal(rng, sgl.sample_count(B)) for _ in range(2))
    a = 1.4 - 0.3j
    f = lambda g: sgl.fsglft(sgl.SampleGrid(B, g), plan).values  # noqa: E731
    assert np.abs(f(a * g1 + g2) - (a * f(g1) + f(g2))).max() < 1e-11


def test_gpu_deterministic():
    B = 16
    plan, _ = plan_for(B)
    g = complex_normal(np.random.default_rng(5), sgl.sample_count(B))
    a = sgl.fsglft(sgl.SampleGrid(B, g), plan).values
    b = sgl.fsglft(sgl.SampleGrid(B, g), plan).values
    assert np.array_equal(a, b)


# ----------------------------------------------------------------- BASELINE configs (reduced batch)
def test_config_c2_batch_b64():
    """C2: B = 64, coefficients x exp(-n/16), batched (here 4 functions)."""
    import torch

    B = 64
    plan, orc = plan_for(B)
    n_of = np.concatenate([[n] * (n * n) for n in range(1, B + 1)])
    rng = np.random.default_rng(64)
    c = complex_normal(rng, (4, sgl.coefficient_count(B))) * np.exp(-n_of / 16.0)
    g = sgl.ifsglft_batch(plan, torch.from_numpy(c).cuda())
    back = sgl.fsglft_batch(plan, g).cpu().numpy()
    g = g.cpu().numpy()
    for f in range(4):
        assert per_shell(g[f], orc.inverse(c[f]), B) <= TOL
        assert normwise(back[f], c[f]) <= TOL


def test_config_c5_real_valued_b32():
    """C5: B = 32 real-valued functions, f_{nl,-m} = (-1)^m conj(f_nlm): samples are
    real to roundoff and the round trip holds (here 8 functions)."""
    import torch

    B = 32
    plan, _ = plan_for(B)
    rng = np.random.default_rng(32)
    nb = 8
    c = np.zeros((nb, sgl.coefficient_count(B)), dtype=np.complex128)
    for n in range(1, B + 1):
        for l in range(n):
            for m in range(0, l + 1):
                w = sgl.omega_index(n, l, m)
                if m == 0:
                    c[:, w] = rng.standard_normal(nb) * np.exp(-n / 8.0)
                else:
                    v = complex_normal(rng, nb) * np.exp(-n / 8.0)
                    c[:, w] = v
                    c[:, sgl.omega_index(n, l, -m)] = (-1) ** m * np.conj(v)
    g = sgl.ifsglft_batch(plan, torch.from_numpy(c).cuda())
    gi = g.imag.abs().max().item() / g.abs().max().item()
    assert gi < 1e-13
    back = sgl.fsglft_batch(plan, g).cpu().numpy()
    assert normwise(back, c) <= TOL


# ----------------------------------------------------------------- multi-GPU stage entry points
@pytest.mark.parametrize("B,W,batch", [(16, 2, 1), (16, 4, 3), (64, 8, 1), (128, 8, 1)])
def test_stage_entry_points_emulated_split(B, W, batch):
    """The shell / (l, m) decomposition of paper_1604_05140_b200.distributed with the
    CUDA stages, all ranks emulated one after another on one GPU (the all-to-all
    becomes tensor slicing; nothing waits on another rank)."""
    import torch

    from paper_1604_05140_b200.distributed import CudaStages, Partition

    plan, orc = plan_for(B)
    st = CudaStages(plan)
    part = Partition.make(B, W)
    rng = np.random.default_rng(B + W)
    c = complex_normal(rng, (batch, sgl.coefficient_count(B)))
    g_full = np.stack([orc.inverse(c[f]) for f in range(batch)])
    sc, n_sh = part.shells_per_rank, 4 * B * B
    dg = torch.from_numpy(g_full).cuda()
    S_loc = []
    for r in range(W):
        s0, s1 = part.shell_range(r)
        S_loc.append(st.spherical_forward(dg[:, s0 * n_sh:s1 * n_sh].contiguous(), s0, sc, batch)
                     .view(B * B, batch * sc))
    coeffs = torch.zeros((batch, sgl.coefficient_count(B)), dtype=torch.complex128, device="cuda")
    for q in range(W):
        nu0, nu1 = part.nu_range(q)
        l0, l1 = part.l_ranges[q]
        if l1 == l0:
            continue
        blocks = torch.cat([S_loc[r][nu0:nu1].reshape(-1) for r in range(W)])
        part_c = torch.zeros_like(coeffs)
        st.radial_forward(blocks, l0, l1, sc, batch, part_c)
        coeffs += part_c
    ref = np.stack([orc.forward(g_full[f]) for f in range(batch)])
    assert normwise(coeffs.cpu().numpy(), ref) <= TOL
    # inverse
    dc = torch.from_numpy(c).cuda()
    sent = []
    for q in range(W):
        l0, l1 = part.l_ranges[q]
        nu0, nu1 = part.nu_range(q)
        blk = st.radial_inverse(dc, l0, l1, sc, batch) if l1 > l0 else torch.zeros(0, dtype=torch.complex128, device="cuda")
        sent.append(blk.view(W, -1))
    for r in range(W):
        S_r = torch.cat([sent[q][r] for q in range(W)])
        s0, s1 = part.shell_range(r)
        x = st.spherical_inverse(S_r.contiguous(), s0, sc, batch).view(batch, -1).cpu().numpy()
        for f in range(batch):
            assert normwise(x[f], g_full[f, s0 * n_sh:s1 * n_sh]) <= 1e-12


# ----------------------------------------------------------------- C++ API (the drop-in surface)
def test_cpp_api_driver():
    import subprocess

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join("/tmp", "sgl_b200_test_sgl_api")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(repo, "include"),
                    os.path.join(repo, "tests", "cpp", "test_sgl_api.cpp"),
                    "-L", os.path.join(repo, "paper_1604_05140_b200"), "-lsglb200",
                    "-Wl,-rpath," + os.path.join(repo, "paper_1604_05140_b200"), "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "[FAIL]" not in out.stdout


def test_graph_replay_matches_eager():
    """Device-memory calls are captured into a CUDA graph from the second call on
    (small transforms); replays must give bit-identical results, also after the
    workspace grows for a bigger batch."""
    import torch

    B = 16
    plan, _ = plan_for(B)
    rng = np.random.default_rng(11)
    c = torch.from_numpy(complex_normal(rng, (1, sgl.coefficient_count(B)))).cuda()
    s = torch.cuda.Stream()
    outs = []
    with torch.cuda.stream(s):
        g = torch.empty((1, sgl.sample_count(B)), dtype=torch.complex128, device="cuda")
        for it in range(4):
            sgl.ifsglft_batch(plan, c, out=g)
            outs.append(g.clone())
            if it == 1:  # grow the workspaces with a larger batch in between
                big = torch.from_numpy(complex_normal(rng, (8, sgl.coefficient_count(B)))).cuda()
                sgl.ifsglft_batch(plan, big)
    s.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_cli_roundtrip_and_transform(tmp_path):
    """The CLI front end (reference formats) on the GPU: roundtrip CSV row and a
    fwd/inv file transform that reproduces the reference's golden grid."""
    from paper_1604_05140_b200 import cli

    csv = tmp_path / "bench.csv"
    assert cli.main(["bench", "--bandlimits", "4,16", "--repetitions", "3", "--csv", str(csv)]) == 0
    rows = cli.read_csv(str(csv))
    assert [r["B"] for r in rows] == [4, 16]
    assert all(r["mean_max_abs_err"] < 1e-10 and r["mean_max_rel_err"] < 1e-6 for r in rows)
    src = os.path.join(GOLDEN, "rt_B8_coeffs.bin")
    out = tmp_path / "grid.bin"
    assert cli.main(["transform", "--direction", "inv", "--bandlimit", "8", "--in", src, "--out", str(out)]) == 0
    g = np.fromfile(out, dtype="<f8").view(np.complex128)
    assert per_shell(g, _gold("rt_B8_grid.bin"), 8) <= 1e-13


# ----------------------------------------------------------------- real-valued fast path (C5)
def _real_coeffs(B, nb, rng, decay=8.0):
    c = np.zeros((nb, sgl.coefficient_count(B)), dtype=np.complex128)
    for n in range(1, B + 1):
        for l in range(n):
            for m in range(0, l + 1):
                w = sgl.omega_index(n, l, m)
                if m == 0:
                    c[:, w] = rng.standard_normal(nb) * np.exp(-n / decay)
                else:
                    v = complex_normal(rng, nb) * np.exp(-n / decay)
                    c[:, w] = v
                    c[:, sgl.omega_index(n, l, -m)] = (-1) ** m * np.conj(v)
    return c


@pytest.mark.parametrize("B", [2, 4, 8, 16, 32, 64])
def test_real_path_matches_oracle(B):
    import torch

    plan, orc = plan_for(B)
    rng = np.random.default_rng(500 + B)
    nb = 3
    c = _real_coeffs(B, nb, rng)
    g_ref = np.stack([orc.inverse(c[f]) for f in range(nb)])
    assert np.abs(g_ref.imag).max() <= 1e-13 * np.abs(g_ref).max()
    g = sgl.ifsglft_real_batch(plan, torch.from_numpy(c).cuda())
    assert g.dtype == torch.float64
    back = sgl.fsglft_real_batch(plan, g).cpu().numpy()
    g = g.cpu().numpy()
    for f in range(nb):
        assert per_shell(g[f] + 0j, g_ref[f].real + 0j, B) <= TOL
        assert normwise(back[f], orc.forward(g_ref[f].real + 0j)) <= TOL
        assert normwise(back[f], c[f]) <= TOL
    # host-memory variant and agreement with the complex path on the same real samples
    h = sgl.fsglft_real_batch(plan, g)
    assert normwise(h, back) <= 1e-15
    cplx = sgl.fsglft_batch(plan, torch.from_numpy(g + 0j).cuda()).cpu().numpy()
    assert normwise(back, cplx) <= 1e-13


def test_real_path_rejects_unsupported_bandlimit():
    plan, _ = plan_for(3)
    with pytest.raises(ValueError, match="power of two"):
        sgl.fsglft_real_batch(plan, np.zeros(sgl.sample_count(3)))


def test_nccl_split_path_single_rank():
    """The distributed path end to end over NCCL (torchrun, one rank on this GPU)."""
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                          "--master-addr", "127.0.0.1", "--master-port", "29561",
                          os.path.join(here, "dist_split_check.py"), "16", "2"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "NCCL split path OK" in out.stdout


def test_full_size_properties_b128():
    """Size-independent checks at the headline size: Parseval (quadrature norm of
    the synthesis = coefficient norm, test_sgl_transform.cpp:257-279), linearity
    and zero -> zero, all on the GPU path."""
    import torch

    B = 128
    plan, orc = plan_for(B)
    rng = np.random.default_rng(128)
    n = sgl.coefficient_count(B)
    c = torch.from_numpy(complex_normal(rng, (2, n))).cuda()
    g = sgl.ifsglft_batch(plan, c)
    w = torch.from_numpy((orc.a * orc.r ** 2)[:, None, None] * orc.b_cal[None, :, None]).cuda()
    gn = (w * g.view(2, 2 * B, 2 * B, 2 * B).abs() ** 2).sum(dim=(1, 2, 3))
    cn = (c.abs() ** 2).sum(dim=1)
    assert torch.allclose(gn / cn, torch.ones_like(cn), rtol=1e-9, atol=0)
    a = 0.3 - 1.1j
    lin = sgl.ifsglft_batch(plan, (a * c[0] + c[1]).unsqueeze(0).contiguous())[0]
    ref = a * g[0] + g[1]
    assert float((lin - ref).abs().max() / ref.abs().max()) < 1e-13
    z = sgl.fsglft_batch(plan, torch.zeros((1, sgl.sample_count(B)), dtype=torch.complex128, device="cuda"))
    assert not bool(z.abs().max())


# ---------------------------------------------------------------- on-device cross-oracle
@pytest.mark.parametrize("B", [1, 2, 3, 5, 8, 16, 32])
def test_separated_cross_oracle_matches_fast_path_and_oracle(B):
    """dsglft_separated / idsglft_separated on the GPU (closed-form basis values, direct
    quadratures: sgl_transform.cpp:189-272) agree with the fast GPU path and the CPU oracle."""
    plan, orc = plan_for(B)
    rng = np.random.default_rng(4000 + B)
    c = complex_normal(rng, coefficient_count(B))
    g_sep = sgl.idsglft_separated(sgl.SglCoefficients(B, c), plan).values
    g_fast = sgl.ifsglft(sgl.SglCoefficients(B, c), plan).values
    assert np.isfinite(g_sep).all()
    assert per_shell(g_sep, g_fast, B) <= TOL
    assert per_shell(g_sep, orc.inverse(c), B) <= TOL
    g = complex_normal(rng, sample_count(B))  # not bandlimited: every term of the quadrature counts
    f_sep = sgl.dsglft_separated(sgl.SampleGrid(B, g), plan).values
    assert normwise(f_sep, sgl.fsglft(sgl.SampleGrid(B, g), plan).values) <= TOL
    assert normwise(f_sep, orc.forward(g)) <= TOL


@pytest.mark.parametrize("B", [2, 4, 8, 16])
def test_separated_cross_oracle_on_reference_golden(B):
    """The reference's own round trip (tests/golden, made by oracle/_ref) through the separated rung."""
    import os

    golden = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    load = lambda n: np.fromfile(os.path.join(golden, n), dtype="<f8").view(np.complex128)
    plan, _ = plan_for(B)
    g_ref, back_ref = load(f"rt_B{B}_grid.bin"), load(f"rt_B{B}_back.bin")
    assert normwise(sgl.dsglft_separated(sgl.SampleGrid(B, g_ref), plan).values, back_ref) <= 1e-13
    assert per_shell(sgl.idsglft_separated(sgl.SglCoefficients(B, load(f"rt_B{B}_coeffs.bin")), plan).values,
                     g_ref, B) <= 1e-13


def test_separated_cross_oracle_rejects_large_bandlimit():
    plan, _ = plan_for(128)
    with pytest.raises(ValueError, match="<= 64"):
        sgl.dsglft_separated(sgl.SampleGrid(128, np.zeros(sample_count(128), complex)), plan)


# ---------------------------------------------------------------- fused exchange (peer stores instead of all-to-all)
@pytest.mark.parametrize("B,W,nb", [(8, 2, 1), (16, 4, 2), (32, 8, 1), (128, 8, 1)])
def test_fused_exchange_emulated_ranks(B, W, nb):
    """The peer-store epilogues with W virtual ranks on one device (receive buffers
    as local allocations): every rank's spherical stage writes its S rows into the
    owners' buffers, every rank's radial stage reads its own in place -- and the
    mirror for the inverse.  Ranks run one after another; nothing waits on a peer."""
    import torch

    from paper_1604_05140_b200.distributed import (CudaStages, Partition, PeerBuffers, fused_forward_radial,
                                                   fused_forward_radial_bcast, fused_forward_spherical,
                                                   fused_inverse_radial, fused_inverse_spherical)

    plan, orc = plan_for(B)
    part = Partition.make(B, W)
    st = CudaStages(plan)
    peers = PeerBuffers.local(part, nb)
    try:
        rng = np.random.default_rng(77 + B)
        n = coefficient_count(B)
        c = complex_normal(rng, nb * n).reshape(nb, n)
        dc = torch.from_numpy(c).cuda()
        for r in range(W):
            fused_inverse_radial(dc, part, st, peers, r)
        torch.cuda.synchronize()
        sc, nsh = part.shells_per_rank, 4 * B * B
        slices = [fused_inverse_spherical(part, st, peers, r, dc.device).view(nb, -1) for r in range(W)]
        torch.cuda.synchronize()
        for r in range(W):
            for f in range(nb):
                g_ref = orc.inverse(c[f])[r * sc * nsh:(r + 1) * sc * nsh]
                assert per_shell(slices[r][f].cpu().numpy(), g_ref, B, shells=sc) <= TOL
        for r in range(W):
            fused_forward_spherical(slices[r].contiguous(), part, st, peers, r, nb)
        torch.cuda.synchronize()
        coeffs = torch.zeros((nb, n), dtype=torch.complex128, device="cuda")
        for r in range(W):
            fused_forward_radial(part, st, peers, r, coeffs)
        back = coeffs.cpu().numpy()
        for f in range(nb):
            assert normwise(back[f], c[f]) <= TOL
        # the fused assembly: each rank's radial stage stores into every rank's vectors
        for r in range(W):
            fused_forward_radial_bcast(part, st, peers, r)
        torch.cuda.synchronize()
        for q in range(W):
            assert np.array_equal(peers.coef_tensor(q).cpu().numpy(), back)
    finally:
        peers.close()


def test_fused_exchange_ipc_two_processes():
    """CUDA IPC mapping of the receive buffers + peer-store epilogues across two
    processes (both on this box's GPU; CPU barriers between the steps)."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, SGL_FUSED_DEVICE="0")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29563",
                          os.path.join(here, "dist_fused_check.py"), "16", "2"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "fused exchange OK" in out.stdout


def test_large_batch_crosses_workspace_chunks():
    """B = 32, 1200 functions: more than one ~6 GiB workspace chunk (batch_chunk in
    sgl_capi.cpp) and several 1 GiB function slices inside each -- every function
    must still match its own single-function transform."""
    import torch

    B, nb = 32, 1200
    plan, orc = plan_for(B)
    rng = np.random.default_rng(1200)
    n = coefficient_count(B)
    c = torch.from_numpy(complex_normal(rng, nb * n).reshape(nb, n)).cuda()
    g = sgl.ifsglft_batch(plan, c)
    back = sgl.fsglft_batch(plan, g)
    torch.cuda.synchronize()
    assert float((back - c).abs().max() / c.abs().max()) <= TOL
    for f in (0, 599, 1143, 1144, 1145, nb - 1):
        gf = sgl.ifsglft_batch(plan, c[f:f + 1].contiguous())
        assert float((g[f] - gf[0]).abs().max() / gf.abs().max()) <= 1e-14
    assert per_shell(g[nb - 1].cpu().numpy(), orc.inverse(c[nb - 1].cpu().numpy()), B) <= TOL


def test_empty_batch_and_zero_bandlimit_errors():
    """batch = 0 is a no-op; malformed calls fail with the reference's exception type."""
    plan, _ = plan_for(4)
    out = np.zeros((0, coefficient_count(4)), dtype=np.complex128)
    assert sgl.fsglft_batch(plan, np.zeros((0, sample_count(4)), dtype=np.complex128), out=out).shape[0] == 0
    with pytest.raises(ValueError):
        sgl.fsglft(sgl.SampleGrid(4, np.zeros(10, complex)), plan)
    with pytest.raises(ValueError):
        sgl.ifsglft(sgl.SglCoefficients(5, np.zeros(coefficient_count(5), complex)), plan)


def test_two_plans_from_two_threads():
    """Plans used concurrently from two host threads (kernel attributes are set
    once per kernel AND device under a lock; results must equal single-thread
    calls bit for bit)."""
    import threading

    cases = {}
    for B in (64, 256):
        rng = np.random.default_rng(B + 9)
        c = complex_normal(rng, coefficient_count(B))
        plan = sgl.TransformPlan.compute(B, device=0)
        cases[B] = (plan, c)
    results, errors = {}, []

    def run(B):
        try:
            plan, c = cases[B]
            out = []
            for _ in range(3):
                g = sgl.ifsglft(sgl.SglCoefficients(B, c), plan).values
                out.append((g, sgl.fsglft(sgl.SampleGrid(B, g), plan).values))
            results[B] = out
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=run, args=(B,)) for B in cases]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for B, (plan, c) in cases.items():
        g1 = sgl.ifsglft(sgl.SglCoefficients(B, c), plan).values
        f1 = sgl.fsglft(sgl.SampleGrid(B, g1), plan).values
        for g, f in results[B]:
            assert np.array_equal(g, g1) and np.array_equal(f, f1)
        assert normwise(f1, c) <= TOL


def test_reference_sgl_transform_unit_tests_pass_against_the_mirror():
    """/root/reference/proj/tests/test_sgl_transform.cpp -- all 16 of the
    reference's own test cases (naive / separated / fast transforms, KATs on
    sampled basis functions, matrix semantics at B = 2, Parseval, linearity,
    thread-count independence, error semantics) -- compiled UNMODIFIED against
    the sgl:: mirror (tests/cpp/Makefile, doctest shim) and run on the GPU."""
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "ref_test_sgl_transform")
    if not os.path.exists(exe):
        pytest.skip("ref_test_sgl_transform not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "16 passed, 0 failed" in out.stdout


@pytest.mark.parametrize("B", [2, 4, 8])
def test_naive_rung_matches_oracle(B):
    """dsglft_naive / idsglft_naive (sgl_transform.cpp:122-187) on the device
    against the CPU oracle: the third rung of the reference's oracle chain."""
    plan, orc = plan_for(B)
    rng = np.random.default_rng(80 + B)
    x = complex_normal(rng, sample_count(B))
    c = complex_normal(rng, coefficient_count(B))
    assert normwise(sgl.dsglft_naive(sgl.SampleGrid(B, x), plan).values, orc.forward(x)) <= 1e-12
    assert per_shell(sgl.idsglft_naive(sgl.SglCoefficients(B, c), plan).values, orc.inverse(c), B) <= 1e-12


@pytest.mark.parametrize("B", [4, 16])
def test_sample_sgl_basis_matches_oracle(B):
    plan, orc = plan_for(B)
    for (n, l, m) in [(1, 0, 0), (2, 1, -1), (B, B - 1, B - 1), (B, B - 1, -(B - 2)), (B - 1, 1, 0)]:
        assert per_shell(sgl.sample_sgl_basis(n, l, m, plan).values, orc.sample_basis(n, l, m), B) <= 1e-12


@pytest.mark.parametrize("B", [128, 256])
def test_fast_transform_exact_on_sampled_basis_at_large_b(B):
    """The reference's exactness KAT (test_sgl_transform.cpp:176-191: fsglft of a
    sampled H_nlm is the unit vector) at B = 128 / 256, where the reference's own
    basis sampler underflows: sample_sgl_basis uses normalized recurrences.
    Includes the extreme corners l + |m| = 2B - 2 and the radial edge n = B."""
    plan, _ = plan_for(B)
    for (n, l, m) in [(B, B - 1, B - 1), (B, B - 1, -(B - 1)), (B, 0, 0), (B // 2, B // 2 - 1, -(B // 4)), (3, 2, 1)]:
        g = sgl.sample_sgl_basis(n, l, m, plan).values
        assert np.isfinite(g).all()
        f = sgl.fsglft(sgl.SampleGrid(B, g), plan).values
        target = np.zeros_like(f)
        target[sgl.omega_index(n, l, m)] = 1.0
        assert np.abs(f - target).max() <= 1e-10, (n, l, m, np.abs(f - target).max())


@pytest.mark.parametrize("B", [16, 64, 128])
def test_fused_spherical_forward_matches_oracle(B, monkeypatch):
    """The opt-in persistent fused spherical forward (SGL_FUSED=1: azimuthal items
    and straddling Legendre slice tiles in one launch) gives
    the same coefficients as the oracle, also for a batch."""
    import torch

    monkeypatch.setenv("SGL_FUSED", "1")
    plan, orc = plan_for(B)
    rng = np.random.default_rng(500 + B)
    x = complex_normal(rng, (2, sample_count(B)))
    f = sgl.fsglft_batch(plan, torch.from_numpy(x).cuda()).cpu().numpy()
    for b in range(2):
        assert normwise(f[b], orc.forward(x[b])) <= TOL


@pytest.mark.parametrize("mode", ["leginv", "ws"])
@pytest.mark.parametrize("B", [3, 16, 64, 128, 256])
def test_int8_tensor_core_legendre_inverse_matches_oracle(B, mode, monkeypatch):
    """The opt-in INT8 tensor-core Legendre inverse (SGL_I8=leginv: fp64 by
    7-byte fixed-point slices, 28 tcgen05 kind::i8 GEMMs per 32-deep k step,
    DESIGN.md section 4) matches the oracle per shell, for one function and a
    batch of two (columns spanning functions), with every output finite."""
    import torch

    monkeypatch.setenv("SGL_I8", mode)
    plan, orc = plan_for(B) if B <= 128 else (sgl.TransformPlan.compute(B), Oracle(B))
    rng = np.random.default_rng(700 + B)
    c = complex_normal(rng, (2, coefficient_count(B)))
    if B == 256:  # C4's scaling, as in test_b256_matches_oracle_both_directions
        c = _c4_coefficients(B, 700 + B, 2)
    g = sgl.ifsglft_batch(plan, torch.from_numpy(c).cuda()).cpu().numpy()
    assert np.isfinite(g).all()
    for b in range(2 if B <= 64 else 1):
        assert per_shell(g[b], orc.inverse(c[b]), B) <= TOL
    monkeypatch.setenv("SGL_I8", "0")
    g0 = sgl.ifsglft_batch(plan, torch.from_numpy(c).cuda()).cpu().numpy()
    for b in range(2):
        assert per_shell(g[b], g0[b], B) <= TOL


@pytest.mark.parametrize("B,nb", [(1, 1), (2, 3), (4, 1), (8, 2), (16, 1), (16, 8)])
def test_fused_small_bandlimit_path_matches_general_path_and_oracle(B, nb, monkeypatch):
    """The one-launch-per-direction small-bandlimit kernels (2B <= 32, sgl_small.cu,
    the default there) against the oracle and against the general staged path
    (SGL_SMALL=0) on the same batch (up to the path's batch cap of 8 functions)."""
    import torch

    plan, orc = plan_for(B)
    rng = np.random.default_rng(900 + 10 * B + nb)
    c = torch.from_numpy(complex_normal(rng, (nb, coefficient_count(B)))).cuda()
    x = torch.from_numpy(complex_normal(rng, (nb, sample_count(B)))).cuda()
    g = sgl.ifsglft_batch(plan, c).cpu().numpy()
    f = sgl.fsglft_batch(plan, x).cpu().numpy()
    monkeypatch.setenv("SGL_SMALL", "0")
    g0 = sgl.ifsglft_batch(plan, c).cpu().numpy()
    f0 = sgl.fsglft_batch(plan, x).cpu().numpy()
    cn, xn = c.cpu().numpy(), x.cpu().numpy()
    for b in range(nb):
        assert per_shell(g[b], orc.inverse(cn[b]), B) <= TOL
        assert normwise(f[b], orc.forward(xn[b])) <= TOL
        assert normwise(g[b], g0[b]) <= 1e-14 and normwise(f[b], f0[b]) <= 1e-14


@pytest.mark.parametrize("B,nb", [(64, 2), (128, 1), (256, 1)])
def test_warp_private_legendre_inverse_matches_general_engine_and_oracle(B, nb, monkeypatch):
    """The default Legendre inverse for 64 <= B <= 256 (leginv_wp_kernel: A panel once per
    CTA, warp-private cp.async rings) against the general GEMM engine
    (SGL_LEGINV_WP=0) on the same coefficients, and against the oracle per shell."""
    import torch

    plan, orc = plan_for(B) if B <= 128 else (sgl.TransformPlan.compute(B), Oracle(B))
    c = _c4_coefficients(B, 1100 + B, nb) if B == 256 else complex_normal(np.random.default_rng(1100 + B),
                                                                          (nb, coefficient_count(B)))
    ct = torch.from_numpy(c).cuda()
    g = sgl.ifsglft_batch(plan, ct).cpu().numpy()
    assert np.isfinite(g).all()
    monkeypatch.setenv("SGL_LEGINV_WP", "0")
    g0 = sgl.ifsglft_batch(plan, ct).cpu().numpy()
    for b in range(nb):
        assert per_shell(g[b], g0[b], B) <= 1e-13
    assert per_shell(g[0], orc.inverse(c[0]), B) <= TOL


def test_real_path_with_sample_buffers_that_are_not_32_byte_aligned():
    """At B = 32 the real-valued azimuthal kernels use 256-bit sample loads / stores when
    the sample pointer is 32-byte aligned; a buffer at a 16-byte offset takes the 16-byte
    kernels and must give the same samples and coefficients."""
    import torch

    B, nb = 32, 3
    plan, orc = plan_for(B)
    rng = np.random.default_rng(1200)
    c = torch.from_numpy(_real_coeffs(B, nb, rng)).cuda()
    x = sgl.ifsglft_real_batch(plan, c)
    assert x.data_ptr() % 32 == 0
    big = torch.empty(x.numel() + 2, dtype=x.dtype, device=x.device)
    x_off = big[2:].view_as(x)
    assert x_off.data_ptr() % 32 == 16
    sgl.ifsglft_real_batch(plan, c, out=x_off)
    assert torch.equal(x, x_off) or normwise(x_off.cpu().numpy().ravel(), x.cpu().numpy().ravel()) <= 1e-14
    f = sgl.fsglft_real_batch(plan, x).cpu().numpy()
    f_off = sgl.fsglft_real_batch(plan, x_off).cpu().numpy()
    cn = c.cpu().numpy()
    for b in range(nb):
        assert normwise(f_off[b], f[b]) <= 1e-14
        assert normwise(f[b], cn[b]) <= TOL
