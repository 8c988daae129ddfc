"""Numerics model of the INT8 tensor-core contraction (csrc/sgl_ozaki.cu, sgl_ozaki.cuh).

The kernels turn each fp64 row (table) / column (data) into 56-bit two's-complement
fixed point with its own power-of-two scale, split it into 7 byte digits (digit 0
signed, 1..6 unsigned; the data biased by 2^55 so that all of its digits are
unsigned, the bias undone by per-row constants), form the digit products level by
level (levels i + j <= 6) exactly in integers, and recombine the 7 level sums into
an fp64 value.  This CPU model does the same integer arithmetic (numpy int64 /
float64 sums of small integers are exact) and pins the design choices the kernels
rely on:

* the byte digits reconstruct the fixed-point value exactly (both the signed and the
  biased-unsigned form), and the bias correction is exact;
* 7 x 7 digits with levels <= 6 reach ~1e-13 normwise on Legendre-table contractions
  (the DMMA tolerance is 1e-12), while 6 x 6 digits do not reliably (measured here
  and in DESIGN.md section 4) -- the reason for 28 products per k step;
* the level recombination used by the epilogue (two exact int64 halves, then the
  magic-number conversion) equals the exact integer sum to one rounding.
"""
import numpy as np
import pytest

rng = np.random.default_rng(7)


def legendre_rows(B, am):
    """Fully normalized Pbar_l^|m|(cos theta_j) for l = am .. B-1 at B polar nodes (long double recurrence)."""
    th = (np.arange(B) + 0.5) * np.pi / (2 * B)
    x = np.cos(th).astype(np.longdouble)
    s = np.sin(th).astype(np.longdouble)
    pmm = np.ones(B, dtype=np.longdouble) * np.sqrt(np.longdouble(0.5))
    for m in range(1, am + 1):
        pmm = -np.sqrt((2 * m + 1) / np.longdouble(2 * m)) * s * pmm
    rows = [pmm]
    if am + 1 < B:
        rows.append(np.sqrt(np.longdouble(2 * am + 3)) * x * pmm)
    for l in range(am + 2, B):
        a = np.sqrt((4 * l * l - 1) / np.longdouble(l * l - am * am))
        b = np.sqrt(((l - 1) ** 2 - am * am) / np.longdouble(4 * (l - 1) ** 2 - 1))
        rows.append(a * (x * rows[-1] - b * rows[-2]))
    return np.array(rows)


def to_fixed(x, axis, nd):
    """trunc(x 2^(8 nd - 1 - e)) with e the frexp exponent of the max along `axis`."""
    bits = 8 * nd - 1
    e = np.frexp(np.max(np.abs(x), axis=axis, keepdims=True))[1]
    return np.trunc(np.ldexp(x, bits - e)).astype(np.int64), e, bits


def digits(X, nd, biased=False):
    """Byte digits, most significant first (digit 0 signed unless biased)."""
    if biased:
        X = X + (np.int64(1) << (8 * nd - 1))
    out = []
    for i in range(nd):
        d = (X >> (8 * (nd - 1 - i))) & 255
        if i == 0 and not biased:
            d = np.where(d >= 128, d - 256, d)
        out.append(d)
    return out


def contract(A, Bm, nd=7, maxlev=6, biased=True):
    """sum_k A[r][k] Bm[k][c] through the digit / level scheme (A: table, Bm: data)."""
    XA, ea, ba = to_fixed(A, 1, nd)
    XB, eb, bb = to_fixed(Bm, 0, nd)
    da = digits(XA, nd)
    db = digits(XB, nd, biased=biased)
    lev = []
    for s in range(maxlev + 1):
        acc = np.zeros((A.shape[0], Bm.shape[1]), dtype=np.int64)
        for i in range(nd):
            j = s - i
            if 0 <= j < nd:
                acc += da[i] @ db[j]
        if biased and s < nd:  # the data's top digit carries +128: subtract 128 * sum_k Y_s[r][k]
            acc -= 128 * da[s].sum(axis=1, keepdims=True)
        lev.append(acc)
    if maxlev == 6:  # the epilogue's recombination: exact int64 halves (levels 0-2, 3-6), one rounding
        hi = lev[0] * 65536 + lev[1] * 256 + lev[2]
        lo = lev[3] * 16777216 + lev[4] * 65536 + lev[5] * 256 + lev[6]
        T = hi.astype(np.float64) * 4294967296.0 + lo.astype(np.float64)
    else:
        T = sum(l.astype(np.float64) * 2.0 ** (8 * (maxlev - s)) for s, l in enumerate(lev))
    # sum_k y x = 2^(8 (2 nd - 2 - maxlev)) T * 2^(ea - ba) * 2^(eb - bb)
    return T * 2.0 ** (8 * (2 * nd - 2 - maxlev)) * np.ldexp(1.0, ea - ba) * np.ldexp(1.0, eb - bb)


def test_digits_reconstruct_exactly():
    x = rng.standard_normal((5, 64)) * np.exp(rng.uniform(-30, 30, (5, 1)))
    X, _, _ = to_fixed(x, 1, 7)
    for biased in (False, True):
        d = digits(X, 7, biased=biased)
        back = sum(di.astype(object) * (1 << (8 * (6 - i))) for i, di in enumerate(d))
        want = X.astype(object) + ((1 << 55) if biased else 0)
        assert np.all(back == want)
        lo = 0 if biased else -128
        assert all(int(di.min()) >= lo and int(di.max()) <= 255 for di in d)
    assert np.all(np.abs(X) < (1 << 55))


def test_level_recombination_is_one_rounding():
    lev = [rng.integers(-(1 << 25), 1 << 25, 1000) for _ in range(7)]
    exact = sum(l.astype(object) * (1 << (8 * (6 - s))) for s, l in enumerate(lev))
    hi = lev[0] * 65536 + lev[1] * 256 + lev[2]
    lo = lev[3] * 16777216 + lev[4] * 65536 + lev[5] * 256 + lev[6]
    assert np.all(np.abs(hi) < (1 << 43)) and np.all(np.abs(lo) < (1 << 51))
    T = hi.astype(np.float64) * 4294967296.0 + lo.astype(np.float64)
    for t, e in zip(T, exact):
        assert abs(float(e) - t) <= abs(float(e)) * 2.0 ** -52


@pytest.mark.parametrize("am,p", [(0, 0), (0, 1), (3, 0), (40, 1), (100, 0)])
def test_seven_digits_reach_fp64_level_on_legendre_contractions(am, p):
    B = 128
    P = legendre_rows(B, am)[p::2]  # rows l = am + p + 2k
    K = P.shape[0]
    S = rng.standard_normal((K, 96)) / (1.0 + am + 2 * np.arange(K))[:, None]  # C4-like decay in l
    A = P.T.astype(np.float64)  # Legendre inverse: rows j', K = degrees
    ref = (P.T @ S.astype(np.longdouble)).astype(np.float64)
    out = contract(A, S, nd=7, maxlev=6, biased=True)
    err = np.max(np.abs(out - ref)) / np.max(np.abs(ref))
    assert err <= 2e-13, err
    # unbiased (signed) data digits give the same integers
    assert np.array_equal(contract(A, S, 7, 6, biased=False), out)


def test_six_digits_are_not_enough():
    B = 128
    P = legendre_rows(B, 0)[0::2]
    K = P.shape[0]
    S = rng.standard_normal((K, 96)) / (1.0 + 2 * np.arange(K))[:, None]
    ref = (P.T @ S.astype(np.longdouble)).astype(np.float64)
    e7 = np.max(np.abs(contract(P.T.astype(np.float64), S, 7, 6) - ref)) / np.max(np.abs(ref))
    e6 = np.max(np.abs(contract(P.T.astype(np.float64), S, 6, 5, biased=False) - ref)) / np.max(np.abs(ref))
    assert e6 > 20 * e7
