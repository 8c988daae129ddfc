"""Half-range Gauss-Hermite radial rules, persisted as SGLT kind-1 table files.

Plan-time data generator (not a hot-path component). It restates the
reference's rule construction, which lives in
/root/reference/proj/core/src/quadrature.cpp:

* moments m_k = Gamma((k+1)/2)/2, via m_k = ((k-1)/2) m_{k-2}     (quadrature.cpp:135-145)
* monic recurrence (alpha_k, beta_k) from the moments by the
  Chebyshev "sigma table" algorithm, beta_0 = m_0               (quadrature.cpp:30-62)
* nodes = eigenvalues of the Jacobi matrix, weights = beta_0 z_0i^2
  (Golub-Welsch)                                                 (quadrature.cpp:68-131, 147-169)
* a_mod = a * exp(r^2) * r^2, every quantity rounded to double at the end
                                                                 (quadrature.cpp:170-177)

The reference runs this in boost cpp_bin_float<60|260> and refuses N > 128
(quadrature.hpp:43).  Here the moment reduction runs in mpmath at
dps = 2.6 N + 40 (ill-conditioned step), and the eigen-step is done as
Newton-polished zeros of the monic recurrence with Christoffel weights
a_i = 1 / sum_k phat_k(r_i)^2 (mathematically identical to beta_0 z_0i^2),
which lifts the cap to N = 512 (B = 256).

File layout (precompute_store.hpp:14-30): "SGLT" | u32 version=1 | u32 B |
u8 kind=1 | f64 LE r[2B], a[2B], a_mod[2B] | u32 CRC-32(payload).
File name radial_rule_B{B}.sglt (precompute_store.cpp:150).

Usage:  python -m paper_1604_05140_b200.tables.gen_radial_rules 16 32 64 128 256
"""
from __future__ import annotations

import os
import struct
import sys
import zlib

import mpmath as mp
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def recurrence_from_moments(N: int):
    """Chebyshev algorithm on the raw moments (quadrature.cpp:30-62)."""
    mom = [mp.mpf(0)] * (2 * N)
    mom[0] = mp.sqrt(mp.pi) / 2
    if 2 * N > 1:
        mom[1] = mp.mpf(1) / 2
    for k in range(2, 2 * N):
        mom[k] = mom[k - 2] * (k - 1) / 2
    alpha = [mp.mpf(0)] * N
    beta = [mp.mpf(0)] * N
    alpha[0] = mom[1] / mom[0]
    beta[0] = mom[0]
    prev = list(mom)
    prev2 = None
    cur = [mp.mpf(0)] * (2 * N)
    for k in range(1, N):
        lmax = 2 * N - k - 1
        for l in range(k, lmax + 1):
            v = prev[l + 1] - alpha[k - 1] * prev[l]
            if k >= 2:
                v -= beta[k - 1] * prev2[l]
            cur[l] = v
        beta[k] = cur[k] / prev[k - 1]
        alpha[k] = cur[k + 1] / cur[k] - prev[k] / prev[k - 1]
        if beta[k] <= 0:
            raise ArithmeticError(f"precision fault: beta_{k} lost positivity (order {N})")
        prev2 = prev
        prev = list(cur)
    return alpha, beta


def rule(N: int, dps: int | None = None):
    """Returns (r, a, a_mod) as lists of python floats (rounded from mp)."""
    if dps is None:
        dps = int(2.6 * N + 40)
    with mp.workdps(dps):
        alpha, beta = recurrence_from_moments(N)
    # Eigen step at moderate precision: the three-term evaluation is stable.
    with mp.workdps(80):
        al = [mp.mpf(x) for x in alpha]
        be = [mp.mpf(x) for x in beta]
        sq = [mp.sqrt(b) for b in be]
        # initial guesses from the double Jacobi matrix
        J = np.diag(np.array([float(x) for x in al]))
        off = np.array([float(x) for x in sq[1:]])
        J += np.diag(off, 1) + np.diag(off, -1)
        guesses = np.sort(np.linalg.eigvalsh(J))

        def orthonormal(x):
            # phat_0 = 1/sqrt(beta_0); sqrt(b_{k+1}) phat_{k+1} = (x-a_k) phat_k - sqrt(b_k) phat_{k-1}
            p_prev = mp.mpf(0)
            dp_prev = mp.mpf(0)
            p = 1 / sq[0]
            dp = mp.mpf(0)
            ssum = p * p
            for k in range(N):
                nxt_scale = sq[k + 1] if k + 1 < N else mp.mpf(1)
                p_next = ((x - al[k]) * p - (sq[k] * p_prev if k >= 1 else 0)) / nxt_scale
                dp_next = (p + (x - al[k]) * dp - (sq[k] * dp_prev if k >= 1 else 0)) / nxt_scale
                p_prev, p = p, p_next
                dp_prev, dp = dp, dp_next
                if k + 1 < N:
                    ssum += p * p
            return p, dp, ssum   # p = scaled pi_N(x), dp its derivative

        rs, as_, amods = [], [], []
        for g in guesses:
            x = mp.mpf(float(g))
            for _ in range(60):
                p, dp, _s = orthonormal(x)
                dx = p / dp
                x -= dx
                if abs(dx) <= abs(x) * mp.mpf(10) ** (-60):
                    break
            _p, _dp, ssum = orthonormal(x)
            w = 1 / ssum
            if x <= 0 or w <= 0:
                raise ArithmeticError("precision fault: node or weight lost positivity")
            rs.append(x)
            as_.append(w)
            amods.append(w * mp.exp(x * x) * x * x)
    r = [float(x) for x in rs]
    a = [float(x) for x in as_]
    am = [float(x) for x in amods]
    for i in range(1, N):
        if not r[i] > r[i - 1]:
            raise ArithmeticError("precision fault: nodes are not strictly increasing")
    return r, a, am


def sglt_bytes(B: int, kind: int, payload: np.ndarray) -> bytes:
    body = np.ascontiguousarray(payload, dtype="<f8").tobytes()
    crc = zlib.crc32(body) & 0xFFFFFFFF
    return b"SGLT" + struct.pack("<IIB", 1, B, kind) + body + struct.pack("<I", crc)


def radial_rule_filename(B: int) -> str:
    return f"radial_rule_B{B}.sglt"


def write_rule(B: int, out_dir: str = HERE) -> str:
    r, a, am = rule(2 * B)
    payload = np.array(r + a + am, dtype=np.float64)
    path = os.path.join(out_dir, radial_rule_filename(B))
    with open(path, "wb") as f:
        f.write(sglt_bytes(B, 1, payload))
    return path


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        print(write_rule(int(arg)), flush=True)
