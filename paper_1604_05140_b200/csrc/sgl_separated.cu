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

// ------------------------------------------------------------------ naive rung and basis sampling
// The reference's O(B^7) naive transforms (sgl_transform.cpp:122-187) and
// sample_sgl_basis (:368-389): every basis value H_nlm(r_i, theta_j, phi_k)
// evaluated afresh at every node.  Unlike the separated kernels above these use
// normalized recurrences, so the basis stays finite at every bandlimit:
//   Pbar_lm(t) = M_lm P_lm(t): Pbar_mm in log space, Pbar_{m+1,m} = sqrt(2m+3) t Pbar_mm,
//     Pbar_l = a_l (t Pbar_{l-1} - Pbar_{l-2} / a_{l-1}),  a_l = sqrt((4l^2-1)/(l^2-m^2));
//   N_nl R_nl(r) = sqrt(2) q_k(r^2) r^l, k = n-l-1, alpha = l+1/2, with the
//     normalized Laguerre q_k = sqrt(k!/Gamma(k+alpha+1)) L_k^alpha:
//     q_{k+1} = ((2k+alpha+1-t) q_k - sqrt(k(k+alpha)) q_{k-1}) / sqrt((k+1)(k+alpha+1)),
//     seeded in log space (the e^{-r^2} of the forward folded into the seed).
__device__ double pbar_lm(int l, int am, double t) {
    const double s2 = (1.0 - t) * (1.0 + t);
    double lg = 0.5 * log((2 * am + 1) / (4.0 * 3.14159265358979323846));
    for (int k = 1; k <= am; ++k) lg += 0.5 * log((2.0 * k - 1.0) / (2.0 * k));
    double pmm;
    if (am == 0) pmm = exp(lg);
    else pmm = s2 > 0.0 ? ((am & 1) ? -1.0 : 1.0) * exp(lg + 0.5 * am * log(s2)) : 0.0;
    if (l == am) return pmm;
    double p0 = pmm, p1 = sqrt(2.0 * am + 3.0) * t * pmm;
    for (int ll = am + 2; ll <= l; ++ll) {
        const double a = sqrt((4.0 * ll * ll - 1.0) / ((double)ll * ll - (double)am * am));
        const double b = sqrt(((double)(ll - 1) * (ll - 1) - (double)am * am) / (4.0 * (ll - 1) * (ll - 1) - 1.0));
        const double p = a * (t * p1 - b * p0);
        p0 = p1;
        p1 = p;
    }
    return p1;
}

// N_nl R_nl(r) (decayed: times e^{-r^2})
__device__ double radial_norm(int n, int l, double r, bool decayed) {
    const double alpha = l + 0.5, t = r * r;
    double lg = 0.5 * 0.69314718055994530942 - 0.5 * lgamma(alpha + 1.0);
    if (l > 0) lg += l * log(r);
    if (decayed) lg -= t;
    double q0 = 0.0, q1 = exp(lg);
    for (int k = 0; k < n - l - 1; ++k) {
        const double q = ((2 * k + alpha + 1.0 - t) * q1 - sqrt(k * (k + alpha)) * q0) / sqrt((k + 1) * (k + alpha + 1.0));
        q0 = q1;
        q1 = q;
    }
    return q1;
}

__device__ void omega_to_nlm(long long w, int& n, int& l, int& m) {
    n = 1;
    while ((long long)n * (n + 1) * (2 * n + 1) / 6 <= w) ++n;
    nu_to_lm((int)(w - (long long)(n - 1) * n * (2 * n - 1) / 6), l, m);
}

__device__ __forceinline__ double cos_theta(int j, int N) { return cospi((2 * j + 1) / (2.0 * N)); }

// out[f][omega] = sum_psi a_mod_i b_j e^{-r_i^2} conj(H_nlm(psi)) X[f][psi]; one CTA per (f, omega)
__global__ void naive_forward(int B, const double2* __restrict__ X, double2* __restrict__ C,
                              const double* __restrict__ r, const double* __restrict__ a_mod,
                              const double* __restrict__ bcal) {
    const int N = 2 * B;
    const long long om = (long long)B * (B + 1) * (2 * B + 1) / 6;
    const long long w = blockIdx.x;
    const int f = blockIdx.y;
    int n, l, m;
    omega_to_nlm(w, n, l, m);
    const int am = m < 0 ? -m : m;
    const double sg = (m < 0 && (am & 1)) ? -1.0 : 1.0;  // M_{l,-a} P_{l,-a} = (-1)^a M_la P_la (sgl_transform.cpp:80-85)
    const double2* x = X + (long long)f * N * N * N;
    double ar = 0.0, ai = 0.0;
    for (long long q = threadIdx.x; q < (long long)N * N * N; q += blockDim.x) {
        const int k = (int)(q % N), j = (int)((q / N) % N), i = (int)(q / ((long long)N * N));
        const double basis = radial_norm(n, l, r[i], true) * sg * pbar_lm(l, am, cos_theta(j, N)) * a_mod[i] * bcal[j];
        double sn, cs;
        sincospi((double)(m * k) / B, &sn, &cs);  // conj(e^{i m phi_k}), phi_k = k pi / B
        const double2 v = x[q];
        ar += basis * (v.x * cs + v.y * sn);
        ai += basis * (v.y * cs - v.x * sn);
    }
    __shared__ double red[2][256];
    red[0][threadIdx.x] = ar;
    red[1][threadIdx.x] = ai;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            red[0][threadIdx.x] += red[0][threadIdx.x + h];
            red[1][threadIdx.x] += red[1][threadIdx.x + h];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) C[(long long)f * om + w] = make_double2(red[0][0], red[1][0]);
}

// X[f][psi] = sum_omega c[f][omega] H_nlm(psi); one thread per (f, psi)
__global__ void naive_inverse(int B, int batch, const double2* __restrict__ C, double2* __restrict__ X,
                              const double* __restrict__ r) {
    const int N = 2 * B;
    const long long om = (long long)B * (B + 1) * (2 * B + 1) / 6, ns = (long long)N * N * N;
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= batch * ns) return;
    const int f = (int)(idx / ns);
    const long long q = idx - f * ns;
    const int k = (int)(q % N), j = (int)((q / N) % N), i = (int)(q / ((long long)N * N));
    const double2* c = C + (long long)f * om;
    const double t = cos_theta(j, N);
    double ar = 0.0, ai = 0.0;
    for (int n = 1; n <= B; ++n)
        for (int l = 0; l < n; ++l) {
            const double rad = radial_norm(n, l, r[i], false);
            for (int m = -l; m <= l; ++m) {
                const int am = m < 0 ? -m : m;
                const double sg = (m < 0 && (am & 1)) ? -1.0 : 1.0;
                const double basis = rad * sg * pbar_lm(l, am, t);
                double sn, cs;
                sincospi((double)(m * k) / B, &sn, &cs);
                const double2 v = c[(long long)(n - 1) * n * (2 * n - 1) / 6 + l * (l + 1) + m];
                ar += basis * (v.x * cs - v.y * sn);
                ai += basis * (v.x * sn + v.y * cs);
            }
        }
    X[idx] = make_double2(ar, ai);
}

// X[psi] = H_nlm(r_i, theta_j, phi_k)
__global__ void basis_samples(int B, int n, int l, int m, double2* __restrict__ X, const double* __restrict__ r) {
    const int N = 2 * B;
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q >= (long long)N * N * N) return;
    const int k = (int)(q % N), j = (int)((q / N) % N), i = (int)(q / ((long long)N * N));
    const int am = m < 0 ? -m : m;
    const double sg = (m < 0 && (am & 1)) ? -1.0 : 1.0;
    const double base = radial_norm(n, l, r[i], false) * sg * pbar_lm(l, am, cos_theta(j, N));
    double sn, cs;
    sincospi((double)(m * k) / B, &sn, &cs);
    X[q] = make_double2(base * cs, base * sn);
}

}  // namespace

int launch_naive_forward(int B, int batch, const double* samples, double* coeffs, const double* r,
                         const double* a_mod, const double* bcal, cudaStream_t s) {
    const long long om = (long long)B * (B + 1) * (2 * B + 1) / 6;
    naive_forward<<<dim3((unsigned)om, batch), 256, 0, s>>>(B, reinterpret_cast<const double2*>(samples),
                                                              reinterpret_cast<double2*>(coeffs), r, a_mod, bcal);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_naive_inverse(int B, int batch, const double* coeffs, double* samples, const double* r, cudaStream_t s) {
    const long long nx = (long long)batch * 8 * B * B * B;
    naive_inverse<<<grid_of(nx, 128), 128, 0, s>>>(B, batch, reinterpret_cast<const double2*>(coeffs),
                                                   reinterpret_cast<double2*>(samples), r);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_sample_basis(int B, int n, int l, int m, double* samples, const double* r, cudaStream_t s) {
    basis_samples<<<grid_of(8LL * B * B * B, 128), 128, 0, s>>>(B, n, l, m, reinterpret_cast<double2*>(samples), r);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}


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
