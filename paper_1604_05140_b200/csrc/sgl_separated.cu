// On-device cross-oracle: the reference's separated transforms
// dsglft_separated / idsglft_separated (sgl_transform.cpp:189-272) on sm_100a.
//
// SURVEY.md section 8(f) rank 4.  Independent of the fast path on purpose: no
// FFT, no equatorial fold, no host-generated tables, no DMMA.  Every basis value
// is computed in the kernel from the reference's closed forms --
//   Y_lm:  sph_harm_norm * assoc_legendre (special_functions.cpp:21-47, 81-108),
//          the unnormalized Condon-Shortley recurrence seeded with P_mm,
//   R_nl:  norm_const * gen_laguerre(n-l-1, l+1/2, r^2) * r^l
//          (special_functions.cpp:64-79, 110-127),
// and the sums are the direct quadratures of sft_naive_forward / _inverse
// (spherical_transform.cpp:122-166) and the naive radial matrix products.
// Like the reference these lose accuracy for large l + |m| (the unnormalized
// Legendre seed); they are meant for B <= 64 (the C ABI rejects larger B).
#include "sgl_kernels.cuh"

#include <cmath>

namespace sglk {
namespace {

__device__ __forceinline__ double lgam(double x) { return lgamma(x); }

// assoc_legendre(l, m, t), m >= 0 (special_functions.cpp:21-47)
__device__ double assoc_legendre(int l, int m, double t) {
    double pmm = 1.0;
    if (m > 0) {
        const double s = sqrt((1.0 - t) * (1.0 + t));
        double fact = 1.0;
        for (int i = 0; i < m; ++i) {
            pmm *= -fact * s;
            fact += 2.0;
        }
    }
    if (l == m) return pmm;
    double pm1 = pmm;
    double p = t * (2 * m + 1) * pmm;
    for (int ll = m + 2; ll <= l; ++ll) {
        const double next = ((2 * ll - 1) * t * p - (ll - 1 + m) * pm1) / (ll - m);
        pm1 = p;
        p = next;
    }
    return p;
}

// sph_harm_norm(l, |m|) * assoc_legendre(l, |m|, cos theta) (special_functions.cpp:81-102)
__device__ double legendre_normed(int l, int am, double ct) {
    const double ratio = exp(lgam((double)(l - am + 1)) - lgam((double)(l + am + 1)));
    return sqrt((2 * l + 1) / (4.0 * 3.14159265358979323846) * ratio) * assoc_legendre(l, am, ct);
}

// norm_const(n, l) * radial_raw(n, l, r) (special_functions.cpp:64-79, 110-127)
__device__ double radial_closed(int n, int l, double r) {
    const double nc = exp(0.5 * (0.69314718055994530942 + lgam((double)(n - l)) - lgam(n + 0.5)));
    const int k = n - l - 1;
    const double alpha = l + 0.5, t = r * r;
    double lag = 1.0;
    if (k > 0) {
        double prev = 1.0, cur = alpha + 1.0 - t;
        for (int j = 1; j < k; ++j) {
            const double next = ((2 * j + alpha + 1.0 - t) * cur - (j + alpha) * prev) / (j + 1);
            prev = cur;
            cur = next;
        }
        lag = cur;
    }
    return nc * lag * pow(r, (double)l);
}

__device__ __forceinline__ void nu_to_lm(int nu, int& l, int& m) {
    l = (int)sqrt((double)nu);
    while (l * l > nu) --l;
    while ((l + 1) * (l + 1) <= nu) ++l;
    m = nu - l * (l + 1);
}

// Forward stage 1 (sft_naive_forward per shell): S[f][i][nu] = sum_{j,k} b_j g[f][i][j][k] conj(Y_lm(theta_j, phi_k))
__global__ void sep_sphere_forward(int B, int batch, const double2* __restrict__ X, double2* __restrict__ S,
                                   const double* __restrict__ bcal) {
    const int N = 2 * B, nnu = B * B;
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)batch * N * nnu) return;
    const int nu = (int)(idx % nnu);
    const long long fi = idx / nnu;  // f * N + i
    int l, m;
    nu_to_lm(nu, l, m);
    const int am = m < 0 ? -m : m;
    const double2* g = X + fi * N * N;
    // conj(Y_lm) = pl e^{-i m phi}, times (-1)^|m| for m < 0 (Y_{l,-a} = (-1)^a conj Y_{l,a})
    double ar = 0.0, ai = 0.0;
    for (int j = 0; j < N; ++j) {
        const double ct = cos((2 * j + 1) * 3.14159265358979323846 / (2.0 * N));
        const double pl = legendre_normed(l, am, ct) * bcal[j];
        double sr = 0.0, si = 0.0;
        for (int k = 0; k < N; ++k) {
            double sn, cs;
            sincospi((double)(m * k) / B, &sn, &cs);  // phi_k = k pi / B
            const double2 v = g[j * N + k];
            sr += v.x * cs + v.y * sn;
            si += v.y * cs - v.x * sn;
        }
        ar += pl * sr;
        ai += pl * si;
    }
    if (m < 0 && (am & 1)) {
        ar = -ar;
        ai = -ai;
    }
    S[fi * nnu + nu] = make_double2(ar, ai);
}

// Forward stage 2: c[f][omega(n,l,m)] = sum_i R_nl(r_i) e^{-r_i^2} a_mod_i S[f][i][nu]
__global__ void sep_radial_forward(int B, int batch, const double2* __restrict__ S, double2* __restrict__ C,
                                   const double* __restrict__ r, const double* __restrict__ a_mod) {
    const int N = 2 * B, nnu = B * B;
    const long long om = (long long)B * (B + 1) * (2 * B + 1) / 6;
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= batch * om) return;
    const int f = (int)(idx / om);
    const long long w = idx - (long long)f * om;
    int n = 1;
    while ((long long)n * (n + 1) * (2 * n + 1) / 6 <= w) ++n;
    const int nu = (int)(w - (long long)(n - 1) * n * (2 * n - 1) / 6);
    int l, m;
    nu_to_lm(nu, l, m);
    double ar = 0.0, ai = 0.0;
    for (int i = 0; i < N; ++i) {
        const double e = radial_closed(n, l, r[i]) * exp(-r[i] * r[i]) * a_mod[i];
        const double2 s = S[((long long)f * N + i) * nnu + nu];
        ar += e * s.x;
        ai += e * s.y;
    }
    C[idx] = make_double2(ar, ai);
}

// Inverse stage 1: S[f][i][nu] = sum_{n > l} c[f][omega(n,l,m)] R_nl(r_i)
__global__ void sep_radial_inverse(int B, int batch, const double2* __restrict__ C, double2* __restrict__ S,
                                   const double* __restrict__ r) {
    const int N = 2 * B, nnu = B * B;
    const long long om = (long long)B * (B + 1) * (2 * B + 1) / 6;
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)batch * N * nnu) return;
    const int nu = (int)(idx % nnu);
    const long long fi = idx / nnu;
    const int f = (int)(fi / N), i = (int)(fi - (long long)f * N);
    int l, m;
    nu_to_lm(nu, l, m);
    double ar = 0.0, ai = 0.0;
    for (int n = l + 1; n <= B; ++n) {
        const double e = radial_closed(n, l, r[i]);
        const double2 c = C[(long long)f * om + (long long)(n - 1) * n * (2 * n - 1) / 6 + nu];
        ar += e * c.x;
        ai += e * c.y;
    }
    S[idx] = make_double2(ar, ai);
}

// Inverse stage 2 (sft_naive_inverse per shell): g[f][i][j][k] = sum_{l,m} S[f][i][nu] Y_lm(theta_j, phi_k)
__global__ void sep_sphere_inverse(int B, int batch, const double2* __restrict__ S, double2* __restrict__ X) {
    const int N = 2 * B, nnu = B * B;
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)batch * N * N * N) return;
    const int k = (int)(idx % N);
    const int j = (int)((idx / N) % N);
    const long long fi = idx / ((long long)N * N);
    const double ct = cos((2 * j + 1) * 3.14159265358979323846 / (2.0 * N));
    const double2* sh = S + fi * nnu;
    double ar = 0.0, ai = 0.0;
    const double st = sqrt((1.0 - ct) * (1.0 + ct));
    double pmm = 1.0;  // unnormalized P_am^am, advanced with am (special_functions.cpp:27-35)
    for (int am = 0; am < B; ++am) {
        if (am > 0) pmm *= -(2.0 * am - 1.0) * st;
        double sn, cs;
        sincospi((double)(am * k) / B, &sn, &cs);
        double p0 = 0.0, p1 = pmm;
        for (int l = am; l < B; ++l) {
            double pu;  // unnormalized P_l^am (special_functions.cpp:36-46)
            if (l == am) {
                pu = pmm;
            } else if (l == am + 1) {
                pu = ct * (2 * am + 1) * pmm;
                p0 = pmm;
                p1 = pu;
            } else {
                pu = ((2 * l - 1) * ct * p1 - (l - 1 + am) * p0) / (l - am);
                p0 = p1;
                p1 = pu;
            }
            const double pl =
                sqrt((2 * l + 1) / (4.0 * 3.14159265358979323846) *
                     exp(lgam((double)(l - am + 1)) - lgam((double)(l + am + 1)))) * pu;
            // Y_{l,am} = pl e^{i am phi};  Y_{l,-am} = (-1)^am conj(Y_{l,am})
            const double2 cp = sh[l * (l + 1) + am];
            ar += pl * (cp.x * cs - cp.y * sn);
            ai += pl * (cp.x * sn + cp.y * cs);
            if (am > 0) {
                const double2 cn = sh[l * (l + 1) - am];
                const double sg = (am & 1) ? -pl : pl;
                ar += sg * (cn.x * cs + cn.y * sn);
                ai += sg * (cn.y * cs - cn.x * sn);
            }
        }
    }
    X[idx] = make_double2(ar, ai);
}

int grid_of(long long n, int threads) { return (int)((n + threads - 1) / threads); }

}  // namespace

int launch_separated_forward(int B, int batch, const double* samples, double* coeffs, double* shells,
                             const double* r, const double* a_mod, const double* bcal, cudaStream_t s) {
    const int N = 2 * B;
    const long long ns = (long long)batch * N * B * B;
    const long long nc = (long long)batch * B * (B + 1) * (2 * B + 1) / 6;
    sep_sphere_forward<<<grid_of(ns, 128), 128, 0, s>>>(B, batch, reinterpret_cast<const double2*>(samples),
                                                         reinterpret_cast<double2*>(shells), bcal);
    sep_radial_forward<<<grid_of(nc, 128), 128, 0, s>>>(B, batch, reinterpret_cast<const double2*>(shells),
                                                        reinterpret_cast<double2*>(coeffs), r, a_mod);
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

int launch_separated_inverse(int B, int batch, const double* coeffs, double* samples, double* shells,
                             const double* r, cudaStream_t s) {
    const int N = 2 * B;
    const long long ns = (long long)batch * N * B * B;
    const long long nx = (long long)batch * N * N * N;
    sep_radial_inverse<<<grid_of(ns, 128), 128, 0, s>>>(B, batch, reinterpret_cast<const double2*>(coeffs),
                                                        reinterpret_cast<double2*>(shells), r);
    sep_sphere_inverse<<<grid_of(nx, 128), 128, 0, s>>>(B, batch, reinterpret_cast<const double2*>(shells),
                                                        reinterpret_cast<double2*>(samples));
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

}  // namespace sglk
