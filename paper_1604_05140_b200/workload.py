"""Algorithmic work per stage (the fixed roofline numerators of SURVEY.md section 8(d)).

All counts are per function and per direction, for the reference algorithm
(implementation-independent: a kernel that does extra flops gets no credit).

  F_az  = (2B)^2 * 5 * (2B) * log2(2B)           azimuthal FFT of 4B^2 rings
  F_w   = (2B) * (2B-1) * (2B) * 2               b_j weighting
  F_dct = (2B)(2B-1) * [5 (2B) log2(2B) + 6 (2B)] DCT/DST per (shell, m)
  F_dlt = (2B) * sum_{l<B} (2l+1)(l+1) * 4        truncated Legendre dots
  F_drt = sum_{l<B} (2l+1)(B-l) * (2B) * 4        discrete R transform
  F_fwd = F_az + F_w + F_dct + F_dlt + F_drt      (= F_inv)

Compulsory bytes: per direction
  stage 1 (spherical):  Q1 = 16*8B^3 (samples) + 16*2B^3 (S, the per-shell coefficients)
  stage 2 (radial):     Q2 = 16*2B^3 + 16*Omega + 8*sum_l (B-l)*2B (radial table)
Per-stage roofline time = max(F_s / P_fp64, Q_s / BW_hbm); the transform's
roofline time is the sum over both stages and both directions.

Stage mapping of the CUDA path: the spherical stage is two
kernels joined by the intermediate G (16*(2B)^2*(2B-1) bytes, written by one and
read by the other).  G is NOT compulsory: it is booked separately
(`intermediate_bytes`) so the kernels' HBM fractions count only Q1's share:
  az kernel        <- F_az + F_w        compulsory: samples (16*8B^3)     + G (intermediate)
  legendre kernel  <- F_dct + F_dlt     compulsory: S (16*2B^3)           + G (intermediate)
  radial kernel    <- F_drt             compulsory: Q2
"""
from __future__ import annotations

import math


def omega(B: int) -> int:
    return B * (B + 1) * (2 * B + 1) // 6


def f_az(B):
    n = 2 * B
    return n * n * 5 * n * math.log2(n)


def f_w(B):
    n = 2 * B
    return n * (n - 1) * n * 2


def f_dct(B):
    n = 2 * B
    return n * (n - 1) * (5 * n * math.log2(n) + 6 * n)


def f_dlt(B):
    return 2 * B * sum((2 * l + 1) * (l + 1) for l in range(B)) * 4


def f_drt(B):
    return sum((2 * l + 1) * (B - l) for l in range(B)) * 2 * B * 4


def f_fwd(B):
    return f_az(B) + f_w(B) + f_dct(B) + f_dlt(B) + f_drt(B)


def q_io(B):
    """Compulsory bytes of one direction: samples + coefficients."""
    return 16 * (8 * B ** 3 + omega(B))


def g_bytes(B):
    """The azimuthal -> polar intermediate G of one function (one direction)."""
    return 16 * (2 * B) ** 2 * (2 * B - 1)


def q1(B):
    return 16 * 8 * B ** 3 + 16 * 2 * B ** 3


def q2(B):
    return 16 * 2 * B ** 3 + 16 * omega(B) + 8 * sum(B - l for l in range(B)) * 2 * B


def stage_work(B: int):
    """{stage: (flops, compulsory bytes, intermediate bytes)} per function, stages as
    in sglgpu.h (0..5)."""
    g = g_bytes(B)
    az = (f_az(B) + f_w(B), 16 * 8 * B ** 3, g)
    leg = (f_dct(B) + f_dlt(B), 16 * 2 * B ** 3, g)
    rad = (f_drt(B), q2(B), 0)
    sph = (az[0] + leg[0], q1(B), g)  # the fused persistent spherical kernels (G through L2)
    return {0: az, 1: leg, 2: rad, 3: rad, 4: leg, 5: az, 6: sph, 7: sph}


def roofline_time(B: int, fp64_flops: float, hbm_bytes_s: float) -> float:
    """Seconds of one fwd+inv round trip of one function at the per-stage roofline."""
    sph = max((f_az(B) + f_w(B) + f_dct(B) + f_dlt(B)) / fp64_flops, q1(B) / hbm_bytes_s)
    rad = max(f_drt(B) / fp64_flops, q2(B) / hbm_bytes_s)
    return 2 * (sph + rad)


STAGE_NAMES = ["az_forward", "legendre_forward", "radial_forward", "radial_inverse", "legendre_inverse",
               "az_inverse", "spherical_forward_fused", "spherical_inverse_fused"]
