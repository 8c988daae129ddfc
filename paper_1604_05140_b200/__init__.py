"""B200-native SGL Fourier transform (arXiv 1604.05140) -- Python host mirror.

Mirrors the reference's hot-path API (/root/reference/proj/core/include/sgl/
sgl_transform.hpp:15-89): ``TransformPlan``, ``SampleGrid``, ``SglCoefficients``,
``fsglft``, ``ifsglft``, ``roundtrip_error``, with the same layouts (psi-order
samples, omega-order coefficients, complex128) and the same error messages for
shape errors (sgl_transform.cpp:18-35; ``ValueError`` stands in for
``std::invalid_argument``).  Every transform runs the sm_100a CUDA kernels of
``libsglb200.so`` through its C ABI (include/sglgpu.h).  There is no CPU
fallback: without the library or a CUDA device the calls raise.

Additive API: ``fsglft_batch`` / ``ifsglft_batch`` take numpy arrays (host) or
CUDA torch tensors (device, asynchronous on the current stream).
"""
from __future__ import annotations

import ctypes
import os
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SGL_B200_LIB", os.path.join(_PKG, "libsglb200.so"))
TABLES_DIR = os.environ.get("SGL_TABLES", os.path.join(_PKG, "tables"))

SGLGPU_OK, SGLGPU_EINVAL, SGLGPU_ECUDA, SGLGPU_ENOMEM, SGLGPU_ENODEV = range(5)
MEM_HOST, MEM_DEVICE = 0, 1

_vp = ctypes.c_void_p


class _PlanDesc(ctypes.Structure):
    _fields_ = [("bandlimit", ctypes.c_int), ("r", _vp), ("a_mod", _vp), ("b_cal", _vp),
                ("device", ctypes.c_int)]


_lib = None


def lib():
    """Loads libsglb200.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing; run python -m paper_1604_05140_b200.build")
        L = ctypes.CDLL(LIB_PATH)
        L.sglgpu_last_error.restype = ctypes.c_char_p
        L.sglgpu_plan_create.argtypes = [ctypes.POINTER(_PlanDesc), ctypes.POINTER(_vp)]
        L.sglgpu_plan_destroy.argtypes = [_vp]
        L.sglgpu_plan_bandlimit.argtypes = [_vp]
        L.sglgpu_plan_table_bytes.argtypes = [_vp]
        L.sglgpu_plan_table_bytes.restype = ctypes.c_size_t
        L.sglgpu_last_launch_count.argtypes = [_vp]
        for name in ("sglgpu_forward", "sglgpu_inverse", "sglgpu_forward_real", "sglgpu_inverse_real",
                     "sglgpu_forward_separated", "sglgpu_inverse_separated", "sglgpu_forward_naive",
                     "sglgpu_inverse_naive"):
            getattr(L, name).argtypes = [_vp, _vp, _vp, ctypes.c_size_t, ctypes.c_int, _vp]
        for name in ("sglgpu_spherical_forward", "sglgpu_spherical_inverse"):
            getattr(L, name).argtypes = [_vp, _vp, ctypes.c_size_t, _vp, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_size_t, _vp]
        for name in ("sglgpu_radial_forward", "sglgpu_radial_inverse"):
            getattr(L, name).argtypes = [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_size_t,
                                         _vp]
        L.sglgpu_spherical_forward_to.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_size_t, ctypes.c_int, _vp, _vp, _vp]
        for name in ("sglgpu_radial_inverse_to", "sglgpu_radial_forward_to"):
            getattr(L, name).argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_size_t, ctypes.c_int, _vp, _vp]
        L.sglgpu_device_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(_vp)]
        L.sglgpu_device_free.argtypes = [_vp]
        L.sglgpu_ipc_export.argtypes = [_vp, _vp]
        L.sglgpu_ipc_open.argtypes = [_vp, ctypes.POINTER(_vp)]
        L.sglgpu_ipc_close.argtypes = [_vp]
        L.sglgpu_sample_basis.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp]
        L.sglgpu_profile_begin.argtypes = [_vp]
        L.sglgpu_profile_end.argtypes = [_vp, _vp, _vp]
        _lib = L
    return _lib


def _check(status: int):
    if status == SGLGPU_OK:
        return
    msg = lib().sglgpu_last_error().decode()
    if status == SGLGPU_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


# ----------------------------------------------------------------- layouts (indexing.cpp:38-78)
def sample_count(B: int) -> int:
    if B < 1 or B > 512:
        raise ValueError(f"bandlimit must be in [1, 512], got {B}")
    return 8 * B ** 3


def coefficient_count(B: int) -> int:
    if B < 1 or B > 512:
        raise ValueError(f"bandlimit must be in [1, 512], got {B}")
    return B * (B + 1) * (2 * B + 1) // 6


def psi_index(i: int, j: int, k: int, B: int) -> int:
    """indexing.cpp:50-78 (IndexError stands in for std::out_of_range)."""
    sample_count(B)
    if not (0 <= i < 2 * B and 0 <= j < 2 * B and 0 <= k < 2 * B):
        raise IndexError("psi_index: node indices out of range")
    return 4 * B * B * i + 2 * B * j + k


def nu_index(l: int, m: int) -> int:
    if l < 0 or abs(m) > l:
        raise IndexError("nu_index: require |m| <= l")
    return l * (l + 1) + m


def omega_index(n: int, l: int, m: int) -> int:
    if n < 1 or l < 0 or l >= n or abs(m) > l:
        raise IndexError("omega_index: require |m| <= l < n")
    return (n - 1) * n * (2 * n - 1) // 6 + l * (l + 1) + m


# ----------------------------------------------------------------- rules and store
@dataclass
class SphericalRule:
    order: int
    theta: np.ndarray
    phi: np.ndarray
    b_raw: np.ndarray
    b_cal: np.ndarray


@dataclass
class RadialRule:
    order: int
    r: np.ndarray
    a: np.ndarray
    a_mod: np.ndarray


def sphere_rule(L: int) -> SphericalRule:
    """quadrature.cpp:189-211 (closed form)."""
    if L < 1:
        raise ValueError("sphere_rule: order must be positive")
    j = np.arange(2 * L)
    theta = (2 * j + 1) * np.pi / (4.0 * L)
    phi = j * np.pi / L
    b_raw = np.empty(2 * L)
    for jj in range(2 * L):
        acc = 0.0
        for l in range(L):
            acc += np.sin((2 * jj + 1) * (2 * l + 1) * np.pi / (4.0 * L)) / (2 * l + 1)
        b_raw[jj] = np.sin((2 * jj + 1) * np.pi / (4.0 * L)) * (2.0 / L) * acc
    return SphericalRule(L, theta, phi, b_raw, np.pi / L * b_raw)


def _read_sglt(path: str, kind: int):
    """SGLT reader (precompute_store.hpp:14-30)."""
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 17:
        raise RuntimeError(f"file too short: {path}")
    if data[:4] != b"SGLT":
        raise RuntimeError(f"not a table file: {path}")
    version, B, k = struct.unpack("<IIB", data[4:13])
    if version != 1:
        raise RuntimeError(f"unsupported format version {version} in {path}")
    if k != kind:
        raise RuntimeError(f"unexpected table kind {k} in {path}")
    body = data[13:-4]
    if len(body) % 8:
        raise RuntimeError(f"payload is not a whole number of doubles: {path}")
    if zlib.crc32(body) & 0xFFFFFFFF != struct.unpack("<I", data[-4:])[0]:
        raise RuntimeError(f"payload checksum mismatch: {path}")
    return B, np.frombuffer(body, dtype="<f8").copy()


def load_radial_rule(path: str) -> RadialRule:
    B, v = _read_sglt(path, 1)
    if v.size != 6 * B:
        raise RuntimeError(f"payload length does not match the declared bandlimit: {path}")
    n = 2 * B
    return RadialRule(n, v[:n], v[n:2 * n], v[2 * n:])


def radial_rule_filename(B: int) -> str:
    return f"radial_rule_B{B}.sglt"


# ----------------------------------------------------------------- plan
@dataclass
class SglCoefficients:
    """sgl_transform.hpp:15-19"""
    bandlimit: int
    values: np.ndarray


@dataclass
class SampleGrid:
    """sgl_transform.hpp:21-25"""
    bandlimit: int
    values: np.ndarray


@dataclass
class TransformPlan:
    """sgl_transform.hpp:30-49, plus the device plan handle (tables uploaded once)."""
    bandlimit: int
    radial: RadialRule
    sphere: SphericalRule
    device: int = -1
    _handle: int | None = field(default=None, repr=False)

    @staticmethod
    def compute(B: int, device: int = -1) -> "TransformPlan":
        if B < 1:
            raise ValueError("TransformPlan: bandlimit must be positive")
        path = os.path.join(TABLES_DIR, radial_rule_filename(B))
        if not os.path.exists(path):
            raise RuntimeError(
                f"no tabulated radial rule of order {2 * B} in {TABLES_DIR}; generate it with "
                f"python -m paper_1604_05140_b200.tables.gen_radial_rules {B}")
        return TransformPlan.assemble(B, load_radial_rule(path), sphere_rule(B), device)

    @staticmethod
    def from_tables(directory: str, B: int, device: int = -1) -> "TransformPlan":
        return TransformPlan.assemble(B, load_radial_rule(os.path.join(directory, radial_rule_filename(B))),
                                      sphere_rule(B), device)

    @staticmethod
    def assemble(B: int, radial: RadialRule, sphere: SphericalRule, device: int = -1) -> "TransformPlan":
        if B < 1:
            raise ValueError("TransformPlan: bandlimit must be positive")
        if radial.order != 2 * B:
            raise ValueError("TransformPlan: radial rule order must be 2B")
        if sphere.order != B:
            raise ValueError("TransformPlan: spherical tables must have order B")
        return TransformPlan(B, radial, sphere, device)

    @property
    def handle(self) -> int:
        """The sglgpu_plan* (created on first use)."""
        if self._handle is None:
            r = np.ascontiguousarray(self.radial.r, dtype=np.float64)
            am = np.ascontiguousarray(self.radial.a_mod, dtype=np.float64)
            bc = np.ascontiguousarray(self.sphere.b_cal, dtype=np.float64)
            d = _PlanDesc(self.bandlimit, r.ctypes.data, am.ctypes.data, bc.ctypes.data, self.device)
            h = _vp()
            _check(lib().sglgpu_plan_create(ctypes.byref(d), ctypes.byref(h)))
            self._handle = h.value
        return self._handle

    def table_bytes(self) -> int:
        return int(lib().sglgpu_plan_table_bytes(self.handle))

    def last_launch_count(self) -> int:
        return int(lib().sglgpu_last_launch_count(self.handle))

    def close(self):
        if self._handle is not None and _lib is not None:
            _lib.sglgpu_plan_destroy(self._handle)
        self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------- transforms
def _check_plan_grid(grid: SampleGrid, plan: TransformPlan):
    """sgl_transform.cpp:18-25"""
    if grid.bandlimit != plan.bandlimit:
        raise ValueError("transform: grid and plan bandlimits disagree")
    if np.asarray(grid.values).size != sample_count(plan.bandlimit):
        raise ValueError("transform: sample grid must have length 8B^3")


def _check_plan_coeffs(coeffs: SglCoefficients, plan: TransformPlan):
    """sgl_transform.cpp:27-35"""
    if coeffs.bandlimit != plan.bandlimit:
        raise ValueError("transform: coefficient and plan bandlimits disagree")
    if np.asarray(coeffs.values).size != coefficient_count(plan.bandlimit):
        raise ValueError("transform: coefficient vector must have length B(B+1)(2B+1)/6")


def fsglft(grid: SampleGrid, plan: TransformPlan, threads: int = 1) -> SglCoefficients:
    """Fast SGL transform (sgl_transform.cpp:274-310) on the GPU; `threads` is ignored."""
    _check_plan_grid(grid, plan)
    g = np.ascontiguousarray(grid.values, dtype=np.complex128)
    out = np.zeros(coefficient_count(plan.bandlimit), dtype=np.complex128)
    _check(lib().sglgpu_forward(plan.handle, g.ctypes.data, out.ctypes.data, 1, MEM_HOST, None))
    return SglCoefficients(plan.bandlimit, out)


def ifsglft(coeffs: SglCoefficients, plan: TransformPlan, threads: int = 1) -> SampleGrid:
    """Fast inverse (sgl_transform.cpp:312-348) on the GPU; `threads` is ignored."""
    _check_plan_coeffs(coeffs, plan)
    c = np.ascontiguousarray(coeffs.values, dtype=np.complex128)
    out = np.zeros(sample_count(plan.bandlimit), dtype=np.complex128)
    _check(lib().sglgpu_inverse(plan.handle, c.ctypes.data, out.ctypes.data, 1, MEM_HOST, None))
    return SampleGrid(plan.bandlimit, out)


def dsglft_separated(grid: SampleGrid, plan: TransformPlan, threads: int = 1) -> SglCoefficients:
    """Separated forward transform (sgl_transform.cpp:189-229) as an on-device cross-oracle:
    closed-form basis values and direct quadratures, independent of the fast path. B <= 64."""
    _check_plan_grid(grid, plan)
    g = np.ascontiguousarray(grid.values, dtype=np.complex128)
    out = np.zeros(coefficient_count(plan.bandlimit), dtype=np.complex128)
    _check(lib().sglgpu_forward_separated(plan.handle, g.ctypes.data, out.ctypes.data, 1, MEM_HOST, None))
    return SglCoefficients(plan.bandlimit, out)


def idsglft_separated(coeffs: SglCoefficients, plan: TransformPlan, threads: int = 1) -> SampleGrid:
    """Separated inverse transform (sgl_transform.cpp:231-272) as an on-device cross-oracle. B <= 64."""
    _check_plan_coeffs(coeffs, plan)
    c = np.ascontiguousarray(coeffs.values, dtype=np.complex128)
    out = np.zeros(sample_count(plan.bandlimit), dtype=np.complex128)
    _check(lib().sglgpu_inverse_separated(plan.handle, c.ctypes.data, out.ctypes.data, 1, MEM_HOST, None))
    return SampleGrid(plan.bandlimit, out)


def dsglft_naive(grid: SampleGrid, plan: TransformPlan, threads: int = 1) -> SglCoefficients:
    """Naive O(B^7) forward transform (sgl_transform.cpp:122-153) on the device. B <= 32."""
    _check_plan_grid(grid, plan)
    g = np.ascontiguousarray(grid.values, dtype=np.complex128)
    out = np.zeros(coefficient_count(plan.bandlimit), dtype=np.complex128)
    _check(lib().sglgpu_forward_naive(plan.handle, g.ctypes.data, out.ctypes.data, 1, MEM_HOST, None))
    return SglCoefficients(plan.bandlimit, out)


def idsglft_naive(coeffs: SglCoefficients, plan: TransformPlan, threads: int = 1) -> SampleGrid:
    """Naive O(B^7) inverse transform (sgl_transform.cpp:155-187) on the device. B <= 32."""
    _check_plan_coeffs(coeffs, plan)
    c = np.ascontiguousarray(coeffs.values, dtype=np.complex128)
    out = np.zeros(sample_count(plan.bandlimit), dtype=np.complex128)
    _check(lib().sglgpu_inverse_naive(plan.handle, c.ctypes.data, out.ctypes.data, 1, MEM_HOST, None))
    return SampleGrid(plan.bandlimit, out)


def sample_sgl_basis(n: int, l: int, m: int, plan: TransformPlan) -> SampleGrid:
    """H_nlm sampled on the plan's grid, psi-order (sgl_transform.cpp:368-389), on the device."""
    B = plan.bandlimit
    if n < 1 or n > B or l < 0 or l >= n or abs(m) > l:
        raise ValueError("sample_sgl_basis: invalid (n, l, m) for this plan")
    out = np.zeros(sample_count(B), dtype=np.complex128)
    _check(lib().sglgpu_sample_basis(plan.handle, n, l, m, out.ctypes.data, MEM_HOST, None))
    return SampleGrid(B, out)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _plan_device(plan: TransformPlan) -> int:
    if plan.device >= 0:
        return plan.device
    import torch

    return torch.cuda.current_device()


def _check_torch_out(plan, src, out, batch, n_out, dtype):
    """A caller-supplied `out` must match what the C ABI will write: shape, dtype,
    contiguity and memory kind / device of `src` (a host pointer handed to the
    kernels, or a short buffer, would be memory corruption, not an exception)."""
    if not _is_torch(out):
        raise ValueError("out must be a torch tensor when the input is one")
    if out.dtype != dtype or not out.is_contiguous() or out.numel() != batch * n_out:
        raise ValueError(f"out must be a contiguous {dtype} tensor of {batch} x {n_out} elements")
    if out.device != src.device:
        raise ValueError(f"out is on {out.device}, the input on {src.device}")
    if src.is_cuda and src.device.index != _plan_device(plan):
        raise ValueError(f"input is on {src.device}, the plan on cuda:{_plan_device(plan)}")


def _check_numpy_out(out, batch, n_out, dtype):
    if not isinstance(out, np.ndarray) or out.dtype != dtype or not out.flags.c_contiguous \
            or out.size != batch * n_out or not out.flags.writeable:
        raise ValueError(f"out must be a writeable C-contiguous {np.dtype(dtype).name} array of "
                         f"{batch} x {n_out} elements")


def _batch_call(fn, plan: TransformPlan, src, n_in: int, n_out: int, out=None, stream=None):
    return _batch_call_real(fn, plan, src, n_in, n_out, np.complex128, np.complex128, out, stream)


def fsglft_batch(plan: TransformPlan, samples, out=None, stream=None):
    """Forward transform of a batch [batch, 8B^3] -> [batch, Omega] (numpy: host; torch CUDA: device)."""
    B = plan.bandlimit
    return _batch_call(lib().sglgpu_forward, plan, samples, sample_count(B), coefficient_count(B), out, stream)


def ifsglft_batch(plan: TransformPlan, coeffs, out=None, stream=None):
    """Inverse transform of a batch [batch, Omega] -> [batch, 8B^3]."""
    B = plan.bandlimit
    return _batch_call(lib().sglgpu_inverse, plan, coeffs, coefficient_count(B), sample_count(B), out, stream)


def _batch_call_real(fn, plan, src, n_in, n_out, in_dtype, out_dtype, out=None, stream=None):
    if _is_torch(src):
        import torch

        td = {np.float64: torch.float64, np.complex128: torch.complex128}
        if src.dtype != td[in_dtype] or not src.is_contiguous():
            raise ValueError(f"expected a contiguous {td[in_dtype]} tensor")
        if src.numel() % n_in:
            raise ValueError("input length is not a whole number of functions")
        batch = src.numel() // n_in
        if out is None:
            out = torch.empty((batch, n_out), dtype=td[out_dtype], device=src.device)
        else:
            _check_torch_out(plan, src, out, batch, n_out, td[out_dtype])
        if src.is_cuda:
            st = stream if stream is not None else torch.cuda.current_stream(src.device).cuda_stream
            _check(fn(plan.handle, src.data_ptr(), out.data_ptr(), batch, MEM_DEVICE, st))
        else:
            _check(fn(plan.handle, src.data_ptr(), out.data_ptr(), batch, MEM_HOST, None))
        return out
    a = np.ascontiguousarray(src, dtype=in_dtype)
    if a.size % n_in:
        raise ValueError("input length is not a whole number of functions")
    batch = a.size // n_in
    if out is None:
        out = np.empty((batch, n_out), dtype=out_dtype)
    else:
        _check_numpy_out(out, batch, n_out, out_dtype)
    _check(fn(plan.handle, a.ctypes.data, out.ctypes.data, batch, MEM_HOST, None))
    return out


def fsglft_real_batch(plan: TransformPlan, samples, out=None, stream=None):
    """Real-valued fast path: real samples [batch, 8B^3] (float64) -> complex
    coefficients [batch, Omega] with f_{n,l,-m} = (-1)^m conj(f_nlm)."""
    B = plan.bandlimit
    return _batch_call_real(lib().sglgpu_forward_real, plan, samples, sample_count(B), coefficient_count(B),
                            np.float64, np.complex128, out, stream)


def ifsglft_real_batch(plan: TransformPlan, coeffs, out=None, stream=None):
    """Real-valued fast path: Hermitian coefficients [batch, Omega] -> real samples
    [batch, 8B^3] (float64).  Only the m >= 0 entries are read."""
    B = plan.bandlimit
    return _batch_call_real(lib().sglgpu_inverse_real, plan, coeffs, coefficient_count(B), sample_count(B),
                            np.complex128, np.float64, out, stream)


@dataclass
class RoundtripError:
    max_abs: float = 0.0
    max_rel: float = 0.0
    skipped_zero: int = 0
    nonfinite: int = 0


def roundtrip_error(reference, actual) -> RoundtripError:
    """sgl_transform.cpp:350-366 (plus an explicit non-finite count)."""
    ref = np.asarray(reference)
    act = np.asarray(actual)
    if ref.shape != act.shape:
        raise ValueError("roundtrip_error: vector lengths disagree")
    diff = np.abs(ref - act)
    mag = np.abs(ref)
    nz = mag != 0
    fin = np.isfinite(diff)
    err = RoundtripError()
    err.nonfinite = int((~np.isfinite(act)).sum())
    err.max_abs = float(diff[fin].max()) if fin.any() else 0.0
    rel = diff[nz & fin] / mag[nz & fin]
    err.max_rel = float(rel.max()) if rel.size else 0.0
    err.skipped_zero = int((~nz).sum())
    return err


__all__ = [
    "SphericalRule", "RadialRule", "TransformPlan", "SglCoefficients", "SampleGrid", "fsglft", "ifsglft",
    "dsglft_separated", "idsglft_separated", "dsglft_naive", "idsglft_naive", "sample_sgl_basis", "fsglft_batch", "ifsglft_batch", "fsglft_real_batch",
    "ifsglft_real_batch", "roundtrip_error", "sphere_rule", "load_radial_rule", "sample_count",
    "coefficient_count", "psi_index", "nu_index", "omega_index", "lib",
]
