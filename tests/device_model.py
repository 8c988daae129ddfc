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
        ls = B + (B & 1)  # rows padded to an even length (sgl_tables.hpp legendre_stride)
        return self.t["leg"][o:o + rows * ls].reshape(rows, ls)[:, :B]

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
            Vl = self.t["V"][self.t["V_off"][l]:self.t["V_off"][l + 1]].reshape(B - l, N).T  # stored [n][i]
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


class ModelStages:
    """CPU stand-in for distributed.CudaStages (test infrastructure): the same four
    stage entry points and layouts, computed with the oracle's stage functions
    (sft_seminaive_* and drt_* restatements).  Lets the multi-GPU orchestration
    run over gloo on CPU."""

    def __init__(self, B):
        from oracle_bindings import Oracle

        self.B = B
        self.o = Oracle(B)

    def spherical_forward(self, samples_local, s0, sc, batch):
        import torch

        B = self.B
        x = samples_local.numpy().reshape(batch, sc, 4 * B * B)
        out = np.zeros((B * B, batch, sc), dtype=np.complex128)
        for f in range(batch):
            for i in range(sc):
                out[:, f, i] = self.o.sft_forward(x[f, i])
        return torch.from_numpy(out.reshape(-1))

    def radial_forward(self, blocks, l0, l1, spb, batch, coeffs_out):
        B = self.B
        nb = 2 * B // spb
        nnu = l1 * l1 - l0 * l0
        blk = blocks.numpy().reshape(nb, nnu, batch, spb)
        c = coeffs_out.numpy()
        for l in range(l0, l1):
            for m in range(-l, l + 1):
                nu = l * (l + 1) + m - l0 * l0
                for f in range(batch):
                    s = blk[:, nu, f, :].reshape(-1)
                    t = self.o.drt_forward(l, s)
                    for n in range(l + 1, B + 1):
                        c[f, (n - 1) * n * (2 * n - 1) // 6 + l * (l + 1) + m] = t[n - l - 1]

    def radial_inverse(self, coeffs, l0, l1, spb, batch):
        import torch

        B = self.B
        nb = 2 * B // spb
        nnu = l1 * l1 - l0 * l0
        out = np.zeros((nb, nnu, batch, spb), dtype=np.complex128)
        c = coeffs.numpy()
        for l in range(l0, l1):
            for m in range(-l, l + 1):
                nu = l * (l + 1) + m - l0 * l0
                for f in range(batch):
                    t = np.array([c[f, (n - 1) * n * (2 * n - 1) // 6 + l * (l + 1) + m] for n in range(l + 1, B + 1)])
                    out[:, nu, f, :] = self.o.drt_inverse(l, t).reshape(nb, spb)
        return torch.from_numpy(out.reshape(-1))

    def spherical_inverse(self, shells_local, s0, sc, batch):
        import torch

        B = self.B
        S = shells_local.numpy().reshape(B * B, batch, sc)
        out = np.zeros((batch, sc, 4 * B * B), dtype=np.complex128)
        for f in range(batch):
            for i in range(sc):
                out[f, i] = self.o.sft_inverse(S[:, f, i])
        return torch.from_numpy(out.reshape(-1))
