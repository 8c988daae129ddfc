"""numpy model of the CUDA algorithm (same tables, same intermediate layouts).

Used by the CPU test-suite to validate the device algorithm's math and layouts
(equatorial fold, (|m|, parity) grouping, nu-major S, radial grouping per l)
against the oracle without a GPU.  Tables come from the library's host-only
generator (sglgpu_host_tables), so this also checks the table generator.
"""
from __future__ import annotations

import ctypes

import numpy as np

import paper_1604_05140_b200 as sgl


def host_tables(B, r, a_mod, bcal=None):
    L = sgl.lib()
    vp = ctypes.c_void_p
    L.sglgpu_host_tables.argtypes = [ctypes.c_int] + [vp] * 10
    sizes = np.zeros(3, dtype=np.int64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    a_mod = np.ascontiguousarray(a_mod, dtype=np.float64)
    bptr = None
    if bcal is not None:
        bcal = np.ascontiguousarray(bcal, dtype=np.float64)
        bptr = bcal.ctypes.data
    assert L.sglgpu_host_tables(B, r.ctypes.data, a_mod.ctypes.data, bptr, sizes.ctypes.data,
                                None, None, None, None, None, None) == 0
    leg = np.zeros(sizes[0])
    leg_off = np.zeros(2 * B + 1, dtype=np.int64)
    W = np.zeros(sizes[1])
    W_off = np.zeros(B + 1, dtype=np.int64)
    V = np.zeros(sizes[2])
    V_off = np.zeros(B + 1, dtype=np.int64)
    assert L.sglgpu_host_tables(B, r.ctypes.data, a_mod.ctypes.data, bptr, sizes.ctypes.data,
                                leg.ctypes.data, leg_off.ctypes.data, W.ctypes.data, W_off.ctypes.data,
                                V.ctypes.data, V_off.ctypes.data) == 0
    return dict(leg=leg, leg_off=leg_off, W=W, W_off=W_off, V=V, V_off=V_off)


class DeviceModel:
    def __init__(self, B, r, a_mod, bcal):
        self.B = B
        self.bcal = np.asarray(bcal)
        self.t = host_tables(B, r, a_mod, bcal)

    def leg_rows(self, am, p):
        B = self.B
        rows = max(0, (B - am - p + 1) // 2)
        o = self.t["leg_off"][2 * am + p]
        return self.t["leg"][o:o + rows * B].reshape(rows, B)

    def forward(self, grid):
        B = self.B
        N = 2 * B
        X = grid.reshape(N, N, N)  # [i][j][k]
        F = np.fft.fft(X, axis=2)  # sign -1, unnormalized
        jp = np.arange(B)
        E = self.bcal[jp][None, :, None] * (F[:, jp, :] + F[:, N - 1 - jp, :])
        O = self.bcal[jp][None, :, None] * (F[:, jp, :] - F[:, N - 1 - jp, :])
        S = np.zeros((B * B, N), dtype=complex)  # [nu][i]
        for am in range(B):
            for p in range(2):
                A = self.leg_rows(am, p)
                if A.shape[0] == 0:
                    continue
                src = E if p == 0 else O
                for sgn in ((0, 1) if am > 0 else (0,)):
                    m = -am if sgn else am
                    bin_ = m % N
                    Xm = src[:, :, bin_].T  # [j'][i]
                    out = A @ Xm            # [row][i]
                    scale = -1.0 if (sgn and am % 2) else 1.0
                    for row in range(A.shape[0]):
                        l = am + p + 2 * row
                        S[l * (l + 1) + m] = scale * out[row]
        C = np.zeros(B * (B + 1) * (2 * B + 1) // 6, dtype=complex)
        for l in range(B):
            Wl = self.t["W"][self.t["W_off"][l]:self.t["W_off"][l + 1]].reshape(B - l, N)
            Sl = S[l * l:(l + 1) ** 2]  # [m+l][i]
            out = Wl @ Sl.T             # [n_idx][m+l]
            for q in range(B - l):
                n = l + 1 + q
                o = (n - 1) * n * (2 * n - 1) // 6 + l * l
                C[o:o + 2 * l + 1] = out[q]
        return C

    def inverse(self, coeffs):
        B = self.B
        N = 2 * B
        S = np.zeros((B * B, N), dtype=complex)
        for l in range(B):
            Vl = self.t["V"][self.t["V_off"][l]:self.t["V_off"][l + 1]].reshape(N, B - l)
            T = np.zeros((B - l, 2 * l + 1), dtype=complex)
            for q in range(B - l):
                n = l + 1 + q
                o = (n - 1) * n * (2 * n - 1) // 6 + l * l
                T[q] = coeffs[o:o + 2 * l + 1]
            S[l * l:(l + 1) ** 2] = (Vl @ T).T
        rings = np.zeros((N, N, N), dtype=complex)  # [i][j][bin]
        for am in range(B):
            for sgn in ((0, 1) if am > 0 else (0,)):
                m = -am if sgn else am
                scale = -1.0 if (sgn and am % 2) else 1.0
                Y = []
                for p in range(2):
                    A = self.leg_rows(am, p)
                    acc = np.zeros((B, N), dtype=complex)  # [j'][i]
                    for row in range(A.shape[0]):
                        l = am + p + 2 * row
                        acc += np.outer(A[row], S[l * (l + 1) + m])
                    Y.append(scale * acc)
                jp = np.arange(B)
                rings[:, jp, m % N] = (Y[0] + Y[1]).T
                rings[:, N - 1 - jp, m % N] = (Y[0] - Y[1]).T
        return (np.fft.ifft(rings, axis=2) * N).reshape(-1)
