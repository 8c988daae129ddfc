"""Algorithmic work per stage (the fixed roofline numerators of SURVEY.md section 8(d)).

All counts are per function and per direction, for the reference algorithm
(implementation-independent: a kernel that does extra flops gets no credit).

  F_az  = (2B)^2 * 5 * (2B) * log2(2B)           azimuthal FFT of 4B^2 rings
  F_w   = (2B) * (2B-1) * (2B) * 2               b_j weighting
  F_dct = (2B)(2B-1) * [5 (2B) log2(2B) + 6 (2B)] DCT/DST per (shell, m)
  F_dlt = (2B) * sum_{l<B} (2l+1)(l+1) * 4        truncated Legendre dots
  F_drt = sum_{l<B} (2l+1)(B-l) * (2B) * 4        discrete R transform
  F_fwd = F_az + F_w + F_dct + F_dlt + F_drt      (= F_inv)

Stage mapping of the CUDA path:
  az kernel        <- F_az + F_w        bytes: samples in (16*8B^3) + G out (16*(2B)^2*(2B-1))
  legendre kernel  <- F_dct + F_dlt     bytes: G in + S out (16*2B^3)
  radial kernel    <- F_drt             bytes: S in + coefficients out (16*Omega)
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


def stage_work(B: int):
    """{stage: (flops, bytes)} per function, stages as in sglgpu.h (0..5)."""
    g_bytes = 16 * (2 * B) ** 2 * (2 * B - 1)
    s_bytes = 16 * 2 * B ** 3
    az = (f_az(B) + f_w(B), 16 * 8 * B ** 3 + g_bytes)
    leg = (f_dct(B) + f_dlt(B), g_bytes + s_bytes)
    rad = (f_drt(B), s_bytes + 16 * omega(B))
    return {0: az, 1: leg, 2: rad, 3: rad, 4: leg, 5: az}


STAGE_NAMES = ["az_forward", "legendre_forward", "radial_forward", "radial_inverse", "legendre_inverse",
               "az_inverse"]
