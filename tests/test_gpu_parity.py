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
