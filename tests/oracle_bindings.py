"""ctypes bindings for the TEST-ONLY CPU checkers under oracle/.

* ``Oracle``  -- oracle/_build/liboracle.so, the plain-C restatement
  (oracle/sgl_oracle.c) of the reference's fsglft / ifsglft.
* ``Reference`` -- oracle/_ref/libsglref.so, the unmodified reference library
  compiled from /root/reference by oracle/Makefile (only present where the
  reference sources were available at build time).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  The product (paper_1604_05140_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(REPO, "oracle", "_build", "liboracle.so")
REF_SO = os.path.join(REPO, "oracle", "_ref", "libsglref.so")
TABLES = os.path.join(REPO, "paper_1604_05140_b200", "tables")

_vp = ctypes.c_void_p
_P = lambda a: a.ctypes.data_as(_vp)  # noqa: E731


def sample_count(B: int) -> int:
    return 8 * B ** 3


def coefficient_count(B: int) -> int:
    return B * (B + 1) * (2 * B + 1) // 6


def omega_index(n: int, l: int, m: int) -> int:
    return (n - 1) * n * (2 * n - 1) // 6 + l * (l + 1) + m


def psi_index(i: int, j: int, k: int, B: int) -> int:
    return 4 * B * B * i + 2 * B * j + k


def read_radial_rule(B: int, tables: str = TABLES):
    """SGLT kind-1 reader (precompute_store.hpp:14-30)."""
    import struct
    import zlib

    with open(os.path.join(tables, f"radial_rule_B{B}.sglt"), "rb") as f:
        data = f.read()
    assert data[:4] == b"SGLT"
    version, b, kind = struct.unpack("<IIB", data[4:13])
    assert version == 1 and b == B and kind == 1
    body = data[13:-4]
    (crc,) = struct.unpack("<I", data[-4:])
    assert zlib.crc32(body) & 0xFFFFFFFF == crc
    v = np.frombuffer(body, dtype="<f8")
    n = 2 * B
    return v[:n].copy(), v[n:2 * n].copy(), v[2 * n:].copy()


def _ensure_built(path: str, target: str):
    if not os.path.exists(path):
        subprocess.run(["make", "-C", os.path.join(REPO, "oracle"), target], check=True,
                       stdout=subprocess.DEVNULL)


class Oracle:
    """The C restatement.  One plan per bandlimit."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            _ensure_built(ORACLE_SO, "all")
            L = ctypes.CDLL(ORACLE_SO)
            L.orc_plan_create.restype = _vp
            L.orc_plan_create.argtypes = [ctypes.c_int, _vp, _vp]
            L.orc_plan_destroy.argtypes = [_vp]
            for name in ("orc_fsglft", "orc_ifsglft"):
                getattr(L, name).argtypes = [_vp, _vp, _vp, ctypes.c_int]
            for name in ("orc_sft_forward", "orc_sft_inverse"):
                getattr(L, name).argtypes = [_vp, _vp, _vp]
            for name in ("orc_drt_forward", "orc_drt_inverse"):
                getattr(L, name).argtypes = [_vp, ctypes.c_int, _vp, _vp]
            L.orc_sample_basis.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]
            L.orc_sgl_basis.argtypes = [ctypes.c_int] * 3 + [ctypes.c_double] * 3 + [_vp]
            L.orc_sphere_rule.argtypes = [ctypes.c_int, _vp, _vp, _vp, _vp]
            L.orc_plan_sphere.argtypes = [_vp, _vp, _vp, _vp]
            L.orc_random_coefficients.argtypes = [ctypes.c_uint64, ctypes.c_size_t, _vp]
            cls._lib = L
        return cls._lib

    def __init__(self, B: int):
        self.B = B
        self.r, self.a, self.a_mod = read_radial_rule(B)
        L = self.lib()
        self._p = L.orc_plan_create(B, _P(self.r), _P(self.a_mod))
        if not self._p:
            raise ValueError(f"oracle plan creation failed for B={B}")
        n2 = 2 * B
        self.theta = np.zeros(n2)
        self.phi = np.zeros(n2)
        self.b_cal = np.zeros(n2)
        L.orc_plan_sphere(self._p, _P(self.theta), _P(self.phi), _P(self.b_cal))

    def __del__(self):
        if getattr(self, "_p", None):
            self.lib().orc_plan_destroy(self._p)
            self._p = None

    def forward(self, grid: np.ndarray, threads: int = 0) -> np.ndarray:
        g = np.ascontiguousarray(grid, dtype=np.complex128)
        assert g.size == sample_count(self.B)
        out = np.zeros(coefficient_count(self.B), dtype=np.complex128)
        assert self.lib().orc_fsglft(self._p, _P(g), _P(out), threads) == 0
        return out

    def inverse(self, coeffs: np.ndarray, threads: int = 0) -> np.ndarray:
        c = np.ascontiguousarray(coeffs, dtype=np.complex128)
        assert c.size == coefficient_count(self.B)
        out = np.zeros(sample_count(self.B), dtype=np.complex128)
        assert self.lib().orc_ifsglft(self._p, _P(c), _P(out), threads) == 0
        return out

    def sft_forward(self, samples):
        s = np.ascontiguousarray(samples, dtype=np.complex128)
        out = np.zeros(self.B * self.B, dtype=np.complex128)
        self.lib().orc_sft_forward(self._p, _P(s), _P(out))
        return out

    def sft_inverse(self, coeffs):
        c = np.ascontiguousarray(coeffs, dtype=np.complex128)
        out = np.zeros(4 * self.B * self.B, dtype=np.complex128)
        self.lib().orc_sft_inverse(self._p, _P(c), _P(out))
        return out

    def drt_forward(self, l, s):
        s = np.ascontiguousarray(s, dtype=np.complex128)
        out = np.zeros(self.B - l, dtype=np.complex128)
        assert self.lib().orc_drt_forward(self._p, l, _P(s), _P(out)) == 0
        return out

    def drt_inverse(self, l, t):
        t = np.ascontiguousarray(t, dtype=np.complex128)
        out = np.zeros(2 * self.B, dtype=np.complex128)
        assert self.lib().orc_drt_inverse(self._p, l, _P(t), _P(out)) == 0
        return out

    def sample_basis(self, n, l, m):
        out = np.zeros(sample_count(self.B), dtype=np.complex128)
        assert self.lib().orc_sample_basis(self._p, n, l, m, _P(out)) == 0
        return out

    @classmethod
    def sgl_basis(cls, n, l, m, r, theta, phi) -> complex:
        out = np.zeros(2)
        cls.lib().orc_sgl_basis(n, l, m, r, theta, phi, _P(out))
        return complex(out[0], out[1])

    @classmethod
    def random_coefficients(cls, B: int, seed: int) -> np.ndarray:
        """The reference's acceptance-suite draw (acceptance_main.cpp:50-63)."""
        n = coefficient_count(B)
        out = np.zeros(2 * n)
        cls.lib().orc_random_coefficients(seed, n, _P(out))
        return out.view(np.complex128)


class Reference:
    """The reference library itself (oracle/_ref).  Raises if not built."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(REF_SO)
            os.environ.setdefault("SGL_RADIAL_DIR", TABLES)
            L = ctypes.CDLL(REF_SO)
            L.ref_plan_create.restype = _vp
            L.ref_plan_create.argtypes = [ctypes.c_int]
            L.ref_plan_destroy.argtypes = [_vp]
            L.ref_last_error.restype = ctypes.c_char_p
            L.ref_forward.argtypes = [_vp, ctypes.c_int, _vp, _vp, ctypes.c_uint]
            L.ref_inverse.argtypes = [_vp, ctypes.c_int, _vp, _vp, ctypes.c_uint]
            L.ref_roundtrip_batch.argtypes = [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int]
            L.ref_sample_basis.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]
            L.ref_sft_forward.argtypes = [_vp, _vp, _vp]
            L.ref_sft_inverse.argtypes = [_vp, _vp, _vp]
            L.ref_drt_forward.argtypes = [_vp, ctypes.c_int, _vp, _vp]
            L.ref_drt_inverse.argtypes = [_vp, ctypes.c_int, _vp, _vp]
            L.ref_plan_arrays.argtypes = [_vp] * 9
            L.ref_save_tables.argtypes = [_vp, ctypes.c_char_p]
            cls._lib = L
        return cls._lib

    def __init__(self, B: int):
        self.B = B
        L = self.lib()
        self._p = L.ref_plan_create(B)
        if not self._p:
            raise RuntimeError(L.ref_last_error().decode())
        n2 = 2 * B
        self.r, self.a, self.a_mod, self.theta, self.phi, self.b_cal, self.exp_neg_r2 = (
            np.zeros(n2) for _ in range(7))
        self.m_norm = np.zeros(B * B)
        L.ref_plan_arrays(self._p, *(_P(x) for x in (self.r, self.a, self.a_mod, self.theta,
                                                      self.phi, self.b_cal, self.exp_neg_r2,
                                                      self.m_norm)))

    def __del__(self):
        if getattr(self, "_p", None):
            self.lib().ref_plan_destroy(self._p)
            self._p = None

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib().ref_last_error().decode())

    def forward(self, grid, threads: int = 0, variant: int = 0):
        g = np.ascontiguousarray(grid, dtype=np.complex128)
        out = np.zeros(coefficient_count(self.B), dtype=np.complex128)
        self._check(self.lib().ref_forward(self._p, variant, _P(g), _P(out), threads))
        return out

    def inverse(self, coeffs, threads: int = 0, variant: int = 0):
        c = np.ascontiguousarray(coeffs, dtype=np.complex128)
        out = np.zeros(sample_count(self.B), dtype=np.complex128)
        self._check(self.lib().ref_inverse(self._p, variant, _P(c), _P(out), threads))
        return out

    def save_tables(self, directory: str):
        """SGLT kinds 1-3 written by the reference itself (precompute_store.cpp)."""
        self._check(self.lib().ref_save_tables(self._p, directory.encode()))

    def roundtrip_batch(self, coeffs: np.ndarray, pool: int):
        c = np.ascontiguousarray(coeffs, dtype=np.complex128)
        out = np.zeros_like(c)
        self._check(self.lib().ref_roundtrip_batch(self._p, _P(c), _P(out), c.shape[0], pool))
        return out

    def sample_basis(self, n, l, m):
        out = np.zeros(sample_count(self.B), dtype=np.complex128)
        self._check(self.lib().ref_sample_basis(self._p, n, l, m, _P(out)))
        return out

    def sft_forward(self, samples):
        s = np.ascontiguousarray(samples, dtype=np.complex128)
        out = np.zeros(self.B * self.B, dtype=np.complex128)
        self._check(self.lib().ref_sft_forward(self._p, _P(s), _P(out)))
        return out

    def drt_forward(self, l, s):
        s = np.ascontiguousarray(s, dtype=np.complex128)
        out = np.zeros(self.B - l, dtype=np.complex128)
        self._check(self.lib().ref_drt_forward(self._p, l, _P(s), _P(out)))
        return out

    def drt_inverse(self, l, t):
        t = np.ascontiguousarray(t, dtype=np.complex128)
        out = np.zeros(2 * self.B, dtype=np.complex128)
        self._check(self.lib().ref_drt_inverse(self._p, l, _P(t), _P(out)))
        return out


def normwise(a: np.ndarray, ref: np.ndarray) -> float:
    """max|a - ref| / max|ref| -- the parity metric of SURVEY.md section 8(d)."""
    den = np.abs(ref).max()
    return float(np.abs(a - ref).max() / den) if den > 0 else float(np.abs(a).max())


def per_shell(a: np.ndarray, ref: np.ndarray, B: int, shells: int = 0) -> float:
    """max over radial shells of the shell-wise normwise error (grids; `shells`
    shells per function, default all 2B)."""
    sh = shells or 2 * B
    a = a.reshape(-1, sh, 4 * B * B)
    ref = ref.reshape(-1, sh, 4 * B * B)
    d = np.abs(a - ref).max(axis=2)
    s = np.abs(ref).max(axis=2)
    s = np.where(s > 0, s, 1.0)
    return float((d / s).max())
