// Plan-time tables (see sgl_tables.hpp).  Host code, long double, threaded over
// orders / degrees.  Cost O(B^3) once per plan.
#include "sgl_tables.hpp"

#include <algorithm>
#include <cmath>
#include <thread>

namespace sglhost {

namespace {

constexpr long double kPiL = 3.141592653589793238462643383279502884L;

template <class F>
void parallel_range(int n, F&& f) {
    const int hw = std::max(1u, std::thread::hardware_concurrency());
    const int nt = std::min(hw, std::max(1, n));
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
        th.emplace_back([&, t] {
            for (int i = t; i < n; i += nt) f(i);
        });
    }
    for (auto& x : th) x.join();
}

}  // namespace

std::vector<double> sphere_bcal(int B) {
    const double pi = 3.14159265358979323846;
    std::vector<double> b(2 * B);
    for (int j = 0; j < 2 * B; ++j) {
        double acc = 0.0;
        for (int l = 0; l < B; ++l) acc += std::sin((2 * j + 1) * (2 * l + 1) * pi / (4.0 * B)) / (2 * l + 1);
        const double braw = std::sin((2 * j + 1) * pi / (4.0 * B)) * (2.0 / B) * acc;
        b[j] = pi / B * braw;
    }
    return b;
}

Tables build_tables(int B, const double* r, const double* a_mod, const double* bcal) {
    Tables t;
    t.B = B;
    const int n2 = 2 * B;
    t.twiddle.resize(2 * n2);
    for (int x = 0; x < n2; ++x) {
        const long double ang = -2.0L * kPiL * x / n2;
        t.twiddle[2 * x] = (double)cosl(ang);
        t.twiddle[2 * x + 1] = (double)sinl(ang);
    }
    // Per-pass twiddle tables of the radix-16 Stockham FFT (sgl_kernels.cu,
    // ring_fft_io / FFTShape): for every pass after the first, radix 16 with Ns
    // outputs already combined, entries w[(r - 1) Ns + k] = tw[r k N / (16 Ns)],
    // r = 1..15, k < Ns -- consecutive threads read consecutive entries.
    if ((n2 & (n2 - 1)) == 0 && n2 >= 32) {
        int logn = 0;
        while ((1 << logn) < n2) ++logn;
        const int r0 = logn % 4 == 0 ? 16 : 1 << (logn % 4);
        const bool head = r0 != 16;
        const int npass = (head ? 1 : 0) + (logn - (head ? logn % 4 : 0)) / 4;
        int ns = head ? r0 : 16;
        for (int pass = 1; pass < npass; ++pass, ns *= 16)
            for (int rr = 1; rr < 16; ++rr)
                for (int k = 0; k < ns; ++k) {
                    const long long x = ((long long)rr * k * (n2 / (ns * 16))) % n2;
                    const long double ang = -2.0L * kPiL * x / n2;
                    t.twiddle.push_back((double)cosl(ang));
                    t.twiddle.push_back((double)sinl(ang));
                }
    }
    // N = 512 forward (radices 16, 16 and a final radix 2 fused into the azimuthal
    // kernel's epilogue, sgl_kernels.cu SGL_AZ512_FUSE2): the radix-16 pass with
    // Ns = 16, appended after the (2, 16, 16) tables the inverse uses.
    if (n2 == 512)
        for (int rr = 1; rr < 16; ++rr)
            for (int k = 0; k < 16; ++k) {
                const long long x = ((long long)rr * k * (n2 / (16 * 16))) % n2;
                const long double ang = -2.0L * kPiL * x / n2;
                t.twiddle.push_back((double)cosl(ang));
                t.twiddle.push_back((double)sinl(ang));
            }
    t.bcal.assign(bcal, bcal + n2);

    // ---- normalized Legendre table, rows grouped by (|m|, parity); rows padded
    // to an even length (legendre_stride) so every row starts 16-byte aligned
    // (the GEMM moves table elements in pairs); the pad entry is 0
    const int LS = legendre_stride(B);
    t.legendre_off.assign(2 * B + 1, 0);
    {
        long long off = 0;
        for (int am = 0; am < B; ++am) {
            for (int p = 0; p < 2; ++p) {
                t.legendre_off[2 * am + p] = off;
                const int rows = std::max(0, (B - am - p + 1) / 2);
                off += (long long)rows * LS;
            }
        }
        t.legendre_off[2 * B] = off;
        t.legendre.assign(off, 0.0);
    }
    std::vector<long double> tj(B);
    for (int j = 0; j < B; ++j) tj[j] = cosl((2 * j + 1) * kPiL / (4.0L * B));
    parallel_range(B, [&](int am) {
        // recurrence coefficients for this order
        std::vector<long double> ca(B + 1, 0.0L), cb(B + 1, 0.0L);
        for (int l = am + 2; l < B; ++l) {
            ca[l] = sqrtl((4.0L * l * l - 1.0L) / ((long double)l * l - (long double)am * am));
            cb[l] = sqrtl(((long double)(l - 1) * (l - 1) - (long double)am * am) /
                          (4.0L * (l - 1) * (l - 1) - 1.0L));
        }
        long double fac = sqrtl((2 * am + 1) / (4.0L * kPiL));
        for (int j = 0; j < B; ++j) {
            const long double x = tj[j];
            const long double s = sqrtl((1.0L - x) * (1.0L + x));
            long double pmm = fac;
            for (int k = 1; k <= am; ++k) pmm *= -sqrtl((2.0L * k - 1.0L) / (2.0L * k)) * s;
            long double p0 = 0.0L, p1 = pmm;
            for (int l = am; l < B; ++l) {
                long double v;
                if (l == am) {
                    v = pmm;
                } else if (l == am + 1) {
                    v = sqrtl(2.0L * am + 3.0L) * x * pmm;
                    p0 = pmm;
                    p1 = v;
                } else {
                    v = ca[l] * (x * p1 - cb[l] * p0);
                    p0 = p1;
                    p1 = v;
                }
                const int p = (l - am) & 1;
                const int row = (l - am) >> 1;
                t.legendre[t.legendre_off[2 * am + p] + (long long)row * LS + j] = (double)v;
            }
        }
    });

    // ---- radial tables
    t.radial_fwd_off.assign(B + 1, 0);
    t.radial_inv_off.assign(B + 1, 0);
    for (int l = 0; l < B; ++l) {
        t.radial_fwd_off[l + 1] = t.radial_fwd_off[l] + (long long)(B - l) * n2;
        t.radial_inv_off[l + 1] = t.radial_inv_off[l] + (long long)(B - l) * n2;
    }
    t.radial_fwd.assign(t.radial_fwd_off[B], 0.0);
    t.radial_inv.assign(t.radial_inv_off[B], 0.0);
    parallel_range(B, [&](int l) {
        const int rows = B - l;
        std::vector<long double> c1(rows), c2(rows), c3(rows);
        for (int n = l + 1; n < B; ++n) {
            const int q = n - l - 1;
            const long double denom = sqrtl((n + 0.5L) * (n - l));
            c1[q] = (2.0L * n - l - 0.5L) / denom;
            c2[q] = 1.0L / denom;
            c3[q] = sqrtl((n - 0.5L) / (n + 0.5L) * ((long double)(n - l - 1) / (n - l)));
        }
        const long double lseed = 0.5L * logl(2.0L) - 0.5L * lgammal(l + 1.5L);
        for (int i = 0; i < n2; ++i) {
            const long double ri = r[i];
            const long double r2 = ri * ri;
            // phi = N_nl R_nl e^{-r^2/2}, bounded; seed in log space
            long double cur = expl(lseed + l * logl(ri) - r2 / 2.0L);
            long double prev = 0.0L;
            const long double wf = (long double)a_mod[i] * expl(-r2 / 2.0L);
            const long double gi = expl(r2 / 2.0L);
            for (int q = 0; q < rows; ++q) {
                if (q > 0) {
                    const long double next = (c1[q - 1] - c2[q - 1] * r2) * cur - c3[q - 1] * prev;
                    prev = cur;
                    cur = next;
                }
                t.radial_fwd[t.radial_fwd_off[l] + (long long)q * n2 + i] = (double)(cur * wf);
                t.radial_inv[t.radial_inv_off[l] + (long long)q * n2 + i] = (double)(cur * gi);
            }
        }
    });
    return t;
}

}  // namespace sglhost

// Host-only inspection hook (no CUDA): sizes (when the out pointers are NULL) or
// copies of the plan tables.  Used by the CPU test-suite to check the table
// generator against the oracle's closed forms without a GPU.
extern "C" int sglgpu_host_tables(int B, const double* r, const double* a_mod, const double* bcal,
                                  long long* sizes /* [3]: legendre, radial_fwd, radial_inv */,
                                  double* legendre, long long* legendre_off, double* radial_fwd,
                                  long long* radial_fwd_off, double* radial_inv, long long* radial_inv_off) {
    if (B < 1 || B > 256 || !r || !a_mod || !sizes) return 1;
    const std::vector<double> bc = bcal ? std::vector<double>(bcal, bcal + 2 * B) : sglhost::sphere_bcal(B);
    const sglhost::Tables t = sglhost::build_tables(B, r, a_mod, bc.data());
    sizes[0] = (long long)t.legendre.size();
    sizes[1] = (long long)t.radial_fwd.size();
    sizes[2] = (long long)t.radial_inv.size();
    if (legendre) std::copy(t.legendre.begin(), t.legendre.end(), legendre);
    if (legendre_off) std::copy(t.legendre_off.begin(), t.legendre_off.end(), legendre_off);
    if (radial_fwd) std::copy(t.radial_fwd.begin(), t.radial_fwd.end(), radial_fwd);
    if (radial_fwd_off) std::copy(t.radial_fwd_off.begin(), t.radial_fwd_off.end(), radial_fwd_off);
    if (radial_inv) std::copy(t.radial_inv.begin(), t.radial_inv.end(), radial_inv);
    if (radial_inv_off) std::copy(t.radial_inv_off.begin(), t.radial_inv_off.end(), radial_inv_off);
    return 0;
}
