// Small bandlimits (2B <= 32, config C1's B = 16): the whole transform in ONE
// launch per direction.  At these sizes every stage kernel of the general path
// is a single latency-bound wave (C1: six launches of ~4.7 us in a 28 us round
// trip), so the stages are fused per shell: the inverse needs no exchange at all
// -- a CTA owns SPC radial shells of one function and runs the radial
// synthesis (all coefficients in shared memory), the Legendre synthesis and the
// azimuthal DFT for them, writing its rings of the grid; the forward mirrors it
// and ends with the radial sum over shells, reduced across the cluster of CTAs
// that share the function through distributed shared memory (deterministic).
// Same algorithm, tables and conventions as the general path (sgl_kernels.cu:
// the folded even/odd G rows, the b_cal weights, the reference's sign of odd
// negative m, the psi / nu / omega layouts); plain fp64 FMAs (the work is ~1e6
// multiply-adds per function).
#include <algorithm>
#include <atomic>
#include <cooperative_groups.h>

#include "sgl_kernels.cuh"

namespace sglk {
namespace cg = cooperative_groups;

namespace {

__device__ __forceinline__ double2 cadd2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cfma(double2 acc, double s, double2 v) {
    return make_double2(fma(s, v.x, acc.x), fma(s, v.y, acc.y));
}

// forward: shells per CTA, so that the function's CTAs fit one cluster (<= 16)
__host__ __device__ constexpr int small_spc(int N) { return N > 16 ? N / 16 : 1; }

struct SmallParams {
    int B;
    int batch;
    const double2* in;   // coefficients (inverse) or samples (forward)
    double2* out;
    long long in_stride, out_stride;  // complex per function
    const double* leg;     // Legendre table (rows grouped by (|m|, parity), legendre_stride)
    const double* W;       // radial forward table [l][n][i]
    const double* V;       // radial inverse table
    const double* bcal;
    const double2* tw;     // e^{-2 pi i x / N}, x < N
};

// table sizes (doubles): the Legendre table holds B (B + 1) / 2 rows of legendre_stride
__host__ __device__ constexpr int leg_doubles(int B) { return (B + (B & 1)) * B * (B + 1) / 2; }
__host__ __device__ constexpr int rad_rows(int B) { return B * (B + 1) / 2; }  // rows (l, n) of a radial table
__device__ __forceinline__ int rad_row(int B, int l) { return l * B - l * (l - 1) / 2; }

__device__ __forceinline__ int deg_off(int n) { return (n - 1) * n * (2 * n - 1) / 6; }  // coefficients of degrees < n
__device__ __forceinline__ int nu_of(int l, int m) { return l * l + l + m; }
__device__ __forceinline__ int omega_of(int n, int l, int m) { return deg_off(n) + l * l + l + m; }

// Staging through cp.async: every thread issues all of its copies before anyone
// waits, so a CTA pays one L2 latency for its inputs instead of one per loop trip.
__device__ __forceinline__ void cpa(void* dst, const void* src, int bytes16) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    if (bytes16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void stage(void* dst, const void* src, int bytes, int tid, int nt) {
    const bool v16 = ((reinterpret_cast<size_t>(src) | reinterpret_cast<size_t>(dst) | (size_t)bytes) & 15) == 0;
    const int step = v16 ? 16 : 8;
    for (int o = tid * step; o < bytes; o += nt * step)
        cpa(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, v16);
}
// the SPC shells' column of a radial table: rows (l, n), entry [row][sl]
__device__ __forceinline__ void stage_rad(double* dst, const double* tab, int B, int N, int s0, int spc, int tid,
                                          int nt) {
    for (int e = tid; e < rad_rows(B) * spc; e += nt) cpa(dst + e, tab + (size_t)(e / spc) * N + s0 + e % spc, 0);
}
// double2 rows into a padded shared array (row stride ds elements)
__device__ __forceinline__ void stage_rows(double2* dst, int ds, const double2* src, int rows, int cols, int tid,
                                           int nt) {
    const bool v16 = (reinterpret_cast<size_t>(src) & 15) == 0;
    for (int e = tid; e < rows * cols; e += nt) {
        double2* d = dst + (e / cols) * ds + e % cols;
        if (v16) {
            cpa(d, src + e, 1);
        } else {
            cpa(d, src + e, 0);
            cpa(reinterpret_cast<double*>(d) + 1, reinterpret_cast<const double*>(src + e) + 1, 0);
        }
    }
}
// The azimuthal DFTs split the N outputs as k + (N / R) q (radix R = 4, or 2 at N = 2):
// a lane owns one k, accumulates the R partial sums Y_r over the inputs x = r (mod R),
// then X[k + (N / R) q] = sum_r w^(r q) Y_r with w = e^(sgn 2 pi i / R).  One
// twiddle table read and one complex MAC per input per lane, R outputs per lane.
template <int R, bool INV>
__device__ __forceinline__ void radix_out(const double2 (&Y)[R], double2 (&X)[R]) {
    if constexpr (R == 4) {
        const double2 A = cadd2(Y[0], Y[2]), Bv = csub2(Y[0], Y[2]), C = cadd2(Y[1], Y[3]), D = csub2(Y[1], Y[3]);
        const double2 iD = INV ? make_double2(-D.y, D.x) : make_double2(D.y, -D.x);  // (+-i) D
        X[0] = cadd2(A, C);
        X[1] = cadd2(Bv, iD);
        X[2] = csub2(A, C);
        X[3] = csub2(Bv, iD);
    } else {
        X[0] = cadd2(Y[0], Y[1]);
        X[1] = csub2(Y[0], Y[1]);
    }
}
__device__ __forceinline__ void stage_wait() {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
}

}  // namespace

// ---------------------------------------------------------------- inverse
template <int N, int SPC>
__global__ void __launch_bounds__(256) small_inverse_kernel(const __grid_constant__ SmallParams P) {
    constexpr int B = N / 2, LS = B + (B & 1), NU = B * B, R = N >= 4 ? 4 : 2, KQ = N / R, NP = N + 1;
    constexpr int OM = B * (B + 1) * (2 * B + 1) / 6;
    extern __shared__ __align__(16) double2 smx[];
    double2* c = smx;                                            // [OM] the function's coefficients
    auto S = reinterpret_cast<double2(*)[NU]>(c + OM);           // [SPC][NU] radial synthesis, nu order
    auto H = reinterpret_cast<double2(*)[N][NP]>(c + OM + SPC * NU);  // [SPC][ring j][bin] E +- O (rows padded)
    double2* tw = c + OM + SPC * NU + SPC * N * NP;              // [N]
    double* leg = reinterpret_cast<double*>(tw + N);             // staged Legendre table
    double* V = leg + leg_doubles(B);                            // [row][sl] this CTA's radial columns
    const int tid = threadIdx.x, nt = blockDim.x;
    const int s0 = blockIdx.x * SPC;
    // persistent over functions: the tables once per CTA, the next function's
    // coefficients prefetched as soon as the radial stage has consumed these
    stage(tw, P.tw, N * 16, tid, nt);
    stage(leg, P.leg, leg_doubles(B) * 8, tid, nt);
    stage_rad(V, P.V, B, N, s0, SPC, tid, nt);
    if (blockIdx.y < P.batch) stage(c, P.in + (size_t)blockIdx.y * P.in_stride, OM * 16, tid, nt);
    for (int f = blockIdx.y; f < P.batch; f += gridDim.y) {
    stage_wait();
    // radial: S[i][nu(l, m)] = sum_n V_l[n][i] c[n, l, m]
    for (int e = tid; e < SPC * NU; e += nt) {
        const int sl = e / NU, nu = e - sl * NU;
        const int l = (int)sqrtf((float)nu + 0.5f), m = nu - l * l - l;
        const double* v = V + rad_row(B, l) * SPC + sl;
        const double2* cc = c + l * l + l + m;
        double2 acc = make_double2(0.0, 0.0);
        for (int n = l + 1; n <= B; ++n) acc = cfma(acc, v[(n - 1 - l) * SPC], cc[deg_off(n)]);
        S[sl][nu] = acc;
    }
    __syncthreads();
    if (f + gridDim.y < P.batch) stage(c, P.in + (size_t)(f + gridDim.y) * P.in_stride, OM * 16, tid, nt);
    // polar: E / O[bin][j'] = sum_k Pbar_{l_k |m|}(t_j') S[nu(l_k, +-m)], l_k = |m| + p + 2k;
    // ring j' takes E + O, its mirror 2B-1-j' takes E - O; the Nyquist bin is zero
    for (int e = tid; e < SPC * N * B; e += nt) {
        const int jp = e % B, rest = e / B;
        const int bin = rest % N, sl = rest / N;
        double2 ev = make_double2(0.0, 0.0), od = ev;
        if (bin != B) {
            const int am = bin < B ? bin : N - bin;
            const int m = bin < B ? bin : -am;
            const double* re = leg + leg_table_off(B, 2 * am) + jp;
            const double* ro = leg + leg_table_off(B, 2 * am + 1) + jp;
            for (int l = am, k = 0; l < B; l += 2, ++k) ev = cfma(ev, re[k * LS], S[sl][nu_of(l, m)]);
            for (int l = am + 1, k = 0; l < B; l += 2, ++k) od = cfma(od, ro[k * LS], S[sl][nu_of(l, m)]);
            if (m < 0 && (am & 1)) {
                ev = make_double2(-ev.x, -ev.y);
                od = make_double2(-od.x, -od.y);
            }
        }
        H[sl][jp][bin] = cadd2(ev, od);
        H[sl][N - 1 - jp][bin] = csub2(ev, od);
    }
    __syncthreads();
    // azimuthal: x_j[k] = sum_bin H_j[bin] e^{+2 pi i bin k / N}, radix split of the outputs
    for (int e = tid; e < SPC * N * KQ; e += nt) {
        const int k = e % KQ, rest = e / KQ;
        const int j = rest % N, sl = rest / N;
        double2 Y[R];
#pragma unroll
        for (int r = 0; r < R; ++r) Y[r] = make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < N / R; ++t) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int bin = R * t + r;
                const double2 v = H[sl][j][bin], w = tw[(bin * k) & (N - 1)];  // conj(w): e^{+i ...}
                Y[r].x = fma(v.x, w.x, fma(v.y, w.y, Y[r].x));
                Y[r].y = fma(v.y, w.x, fma(-v.x, w.y, Y[r].y));
            }
        }
        double2 X[R];
        radix_out<R, true>(Y, X);
        double2* out = P.out + (size_t)f * P.out_stride + ((size_t)(s0 + sl) * N + j) * N + k;
#pragma unroll
        for (int q = 0; q < R; ++q) out[q * KQ] = X[q];
    }
    __syncthreads();  // H and S are rewritten for the next function
    }
}

// ---------------------------------------------------------------- forward
template <int N>
__global__ void __launch_bounds__(256 * small_spc(N)) small_forward_kernel(const __grid_constant__ SmallParams P) {
    constexpr int B = N / 2, SPC = small_spc(N), LS = B + (B & 1), NU = B * B, R = N >= 4 ? 4 : 2, KQ = N / R;
    constexpr int NP = N + 1, OM = B * (B + 1) * (2 * B + 1) / 6, ROWS = B * (B + 1) / 2;
    constexpr int CS = N / SPC;  // CTAs per function (the cluster)
    extern __shared__ __align__(16) double2 smx[];
    auto X = reinterpret_cast<double2(*)[N][NP]>(smx);                  // [SPC][ring j][k] (rows padded)
    auto F = reinterpret_cast<double2(*)[N][NP]>(smx + SPC * N * NP);   // [SPC][ring j][bin]
    auto S = reinterpret_cast<double2(*)[NU]>(smx + 2 * SPC * N * NP);
    double2* part = smx + 2 * SPC * N * NP + SPC * NU;                  // [OM] radial partial sums
    double2* tw = part + OM;                                            // [N]
    double* legT = reinterpret_cast<double*>(tw + N);                   // [j'][row] Legendre table, transposed
    double* W = legT + B * ROWS;                                        // [row][sl] radial columns
    double* bc = W + ROWS * SPC;
    cg::cluster_group cluster = cg::this_cluster();
    const int tid = threadIdx.x, nt = blockDim.x;
    const int s0 = blockIdx.x * SPC;
    auto rings = [&](int f) {
        stage_rows(&X[0][0][0], NP, P.in + (size_t)f * P.in_stride + (size_t)s0 * N * N, SPC * N, N, tid, nt);
    };
    // persistent over functions (the cluster walks them together): the tables once
    // per CTA, the next function's rings prefetched once the DFTs have read these
    stage(tw, P.tw, N * 16, tid, nt);
    for (int e = tid; e < ROWS * B; e += nt) cpa(legT + (e % B) * ROWS + e / B, P.leg + (e / B) * LS + e % B, 0);
    stage_rad(W, P.W, B, N, s0, SPC, tid, nt);
    stage(bc, P.bcal, B * 8, tid, nt);
    stage_wait();
    // fold the quadrature weights into the table (read again only after the next barrier)
    for (int e = tid; e < ROWS * B; e += nt) legT[e] *= bc[e / ROWS];
    if (blockIdx.y < P.batch) rings(blockIdx.y);
    for (int f = blockIdx.y; f < P.batch; f += gridDim.y) {
    stage_wait();
    // azimuthal: F_j[bin] = sum_k x_j[k] e^{-2 pi i bin k / N}, radix split of the outputs
    for (int e = tid; e < SPC * N * KQ; e += nt) {
        const int b = e % KQ, rest = e / KQ;
        const int j = rest % N, sl = rest / N;
        double2 Y[R];
#pragma unroll
        for (int r = 0; r < R; ++r) Y[r] = make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < N / R; ++t) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int k = R * t + r;
                const double2 a = X[sl][j][k], w = tw[(b * k) & (N - 1)];
                Y[r].x = fma(a.x, w.x, fma(-a.y, w.y, Y[r].x));
                Y[r].y = fma(a.y, w.x, fma(a.x, w.y, Y[r].y));
            }
        }
        double2 Z[R];
        radix_out<R, false>(Y, Z);
#pragma unroll
        for (int q = 0; q < R; ++q) F[sl][j][b + q * KQ] = Z[q];
    }
    __syncthreads();
    if (f + gridDim.y < P.batch) rings(f + gridDim.y);
    // polar: S[nu(l, +-m)] = sum_j' b_cal[j'] Pbar_{l |m|}(t_j') (F_j' +- F_{2B-1-j'})[bin(+-m)]
    for (int e = tid; e < SPC * NU; e += nt) {
        const int sl = e / NU, nu = e - sl * NU;
        const int l = (int)sqrtf((float)nu + 0.5f), m = nu - l * l - l;
        const int am = m < 0 ? -m : m, p = (l - am) & 1;
        const int bin = m >= 0 ? m : N + m;
        const double* col = legT + leg_table_off(B, 2 * am + p) / LS + ((l - am) >> 1);
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll 4
        for (int jp = 0; jp < B; ++jp) {
            const double2 u = F[sl][jp][bin], v = F[sl][N - 1 - jp][bin];
            acc = cfma(acc, col[jp * ROWS], p ? csub2(u, v) : cadd2(u, v));
        }
        if (m < 0 && (am & 1)) acc = make_double2(-acc.x, -acc.y);
        S[sl][nu] = acc;
    }
    __syncthreads();
    // radial partial sums: part[n, l, m] = sum_{i in this CTA} W_l[n][i] S[i][nu(l, m)]
    for (int nu = tid; nu < NU; nu += nt) {
        const int l = (int)sqrtf((float)nu + 0.5f);
        double2 s[SPC];
#pragma unroll
        for (int sl = 0; sl < SPC; ++sl) s[sl] = S[sl][nu];
        const double* w = W + rad_row(B, l) * SPC;
        for (int n = l + 1; n <= B; ++n) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int sl = 0; sl < SPC; ++sl) acc = cfma(acc, w[(n - 1 - l) * SPC + sl], s[sl]);
            part[deg_off(n) + nu] = acc;
        }
    }
    // sum over the cluster's CTAs (the function's shells) in rank order, each CTA one
    // contiguous slice of the coefficients
    cluster.sync();
    const int rank = (int)cluster.block_rank();
    constexpr int CH = (OM + CS - 1) / CS;
    double2* out = P.out + (size_t)f * P.out_stride;
    for (int e = rank * CH + tid; e < min(OM, (rank + 1) * CH); e += nt) {
        double2 v[CS];
#pragma unroll
        for (int q = 0; q < CS; ++q) v[q] = cluster.map_shared_rank(part, q)[e];
        double2 acc = v[0];
#pragma unroll
        for (int q = 1; q < CS; ++q) acc = cadd2(acc, v[q]);
        out[e] = acc;
    }
    cluster.sync();  // partials are rewritten (or the CTA leaves) only after every read
    }
}

template <int N, bool FWD, int SPC>
static int small_launch(const SmallParams& prm, cudaStream_t s) {
    constexpr int B = N / 2, cs = N / SPC, nt = FWD ? 256 * SPC : 256;
    constexpr size_t om = (size_t)B * (B + 1) * (2 * B + 1) / 6, nu = (size_t)B * B;
    constexpr size_t smem = sizeof(double2) * (FWD ? 2 * SPC * N * (N + 1) + SPC * nu + om + N
                                                   : om + SPC * nu + SPC * N * (N + 1) + N) +
                            sizeof(double) * (leg_doubles(B) + rad_rows(B) * SPC + (FWD ? B : 0));
    void (*k)(SmallParams);
    if constexpr (FWD) k = small_forward_kernel<N>;
    else k = small_inverse_kernel<N, SPC>;
    static SmemAttrOnce once, np;  // per instantiation and device: not per launch (host time)
    once.ensure(k, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs, prm.batch);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    if (FWD) {  // the CTAs of a function form one cluster (the radial reduction)
        if (cs > 8) np.ensure_attr(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    // enough function slots for every resident CTA; the CTAs loop over the rest
    static std::atomic<int> occ[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return -1;
    if (!occ[dev].load()) {
        int o = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, nt, smem);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        occ[dev] = std::max(1, o * sms / cs);
    }
    cfg.gridDim.y = std::min(prm.batch, occ[dev].load());
    return cudaLaunchKernelEx(&cfg, k, prm) == cudaSuccess ? 1 : -1;
}

bool small_path_ok(int B) { return B >= 1 && B <= 16 && ((2 * B) & (2 * B - 1)) == 0; }

int launch_small_inverse(int B, int batch, const double* C, long long c_stride, double* X, long long x_stride,
                         const double* leg, const double* V, const double* tw, cudaStream_t s) {
    SmallParams p{B, batch, reinterpret_cast<const double2*>(C), reinterpret_cast<double2*>(X), c_stride, x_stride,
                  leg, nullptr, V, nullptr, reinterpret_cast<const double2*>(tw)};
    switch (2 * B) {
        case 2: return small_launch<2, false, 1>(p, s);
        case 4: return small_launch<4, false, 1>(p, s);
        case 8: return small_launch<8, false, 1>(p, s);
        case 16: return small_launch<16, false, 1>(p, s);
        case 32: return small_launch<32, false, 1>(p, s);
        default: return -2;
    }
}

int launch_small_forward(int B, int batch, const double* X, long long x_stride, double* C, long long c_stride,
                         const double* leg, const double* W, const double* bcal, const double* tw, cudaStream_t s) {
    SmallParams p{B, batch, reinterpret_cast<const double2*>(X), reinterpret_cast<double2*>(C), x_stride, c_stride,
                  leg, W, nullptr, bcal, reinterpret_cast<const double2*>(tw)};
    switch (2 * B) {
        case 2: return small_launch<2, true, small_spc(2)>(p, s);
        case 4: return small_launch<4, true, small_spc(4)>(p, s);
        case 8: return small_launch<8, true, small_spc(8)>(p, s);
        case 16: return small_launch<16, true, small_spc(16)>(p, s);
        case 32: return small_launch<32, true, small_spc(32)>(p, s);
        default: return -2;
    }
}

}  // namespace sglk
