// FP64 contractions of the SGL transform on the B200 INT8 tensor cores
// (tcgen05.mma.cta_group::1.kind::i8, int32 accumulators in TMEM), by exact
// fixed-point slicing -- see sgl_ozaki.cuh for the number format and the error
// bound.  B200 runs kind::i8 at ~3.9 POPS (tools/i8_umma.cu, measured) against
// 37 TFLOP/s of FP64 DMMA: even the 28 int8 GEMMs one fp64 GEMM becomes leave
// the tensor cores ~3x faster than the DMMA path, and the contraction ends up
// bound by its fp64 operand / result traffic instead of the FP64 pipe.
//
// Legendre inverse (reference: the per-order synthesis of ifsglft,
// spherical_transform.cpp:254-306 -- DCT-III of the truncated Legendre rows --
// restated here, as in the DMMA path, as the direct contraction over the folded
// polar nodes): per problem (|m|, parity p)
//     G[j'][n] = sum_k Pbar_{l_k, |m|}(cos theta_j') S[nu(l_k, +-m)][n],   l_k = |m| + p + 2k,
// with the table as the MMA A operand (M = 128 polar nodes j', a host-built
// digit image in shared memory) and the data as B (N = 64 columns of S per tile,
// converted to digits in the CTA).  One CTA runs `tpc` column tiles of one
// (problem, m-tile, sign half) so the table image is loaded once.
#include "sgl_ozaki.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>

#ifndef SGL_OZ_EXP
#define SGL_OZ_EXP 0  // timing-only experiments (wrong results): 1 = no G stores, 2 = no level combination
#endif

namespace sglk {
namespace oz {

// ------------------------------------------------------------------ tcgen05 / mbarrier helpers
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// Shared-memory matrix descriptor, K-major, no swizzle: core matrices of 8 rows x
// 16 bytes; lbo = bytes between the two 16-byte K halves of a 32-deep step,
// sbo = bytes between 8-row groups.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ULL << 46);  // version 1 (sm_100)
}

// Instruction descriptor: D s32, A/B s8 or u8, K-major both, N >> 3, M >> 4.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed, bool b_signed) {
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

// Issued by a whole warp with warp-uniform operands (they stay in uniform
// registers); one elected lane issues.
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// Issued by one thread (measured faster than a warp-wide elect + uniform-register
// broadcast per MMA: tools/i8_umma.cu modes 0 / 1).
__device__ __forceinline__ void mma_i8_1(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_1(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {  // whole warp; one elected lane commits
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(bar)
        : "memory");
}

__device__ __forceinline__ void bar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}

__device__ __forceinline__ void bar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "OZW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra OZW_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

// One bulk copy global -> shared completing on an mbarrier (bytes: multiple of 16).
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(bar),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(dst_smem), "r"(cols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(cols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// 8 consecutive 32-bit TMEM columns of this thread's lane (warp w reads lanes
// 32 (w % 4) ..).
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
// 16 lanes x 8 columns per warp: thread t gets (lane t/4, columns 2(t%4), 2(t%4)+1)
// in v[0..1] and (lane t/4 + 8, the same columns) in v[2..3] -- four consecutive
// threads hold 8 consecutive columns of one row, so the epilogue's global stores
// cover 64-byte runs.
__device__ __forceinline__ void tmem_ld16x256(uint32_t taddr, int (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NLEFT>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NLEFT) : "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// ------------------------------------------------------------------ number format
__device__ __forceinline__ int exp_bits(double x) { return (int)((__double_as_longlong(x) >> 52) & 0x7ff); }

// X = trunc(x * 2^(55 - e)) for a column whose largest biased exponent is cE
// (|x| < 2^e, e = cE - 1022), by integer shifts of the significand.
__device__ __forceinline__ long long to_fixed(double x, int cE) {
    const long long bits = __double_as_longlong(x);
    const int E = (int)((bits >> 52) & 0x7ff);
    const unsigned long long m = ((unsigned long long)bits & 0xFFFFFFFFFFFFFULL) | 0x10000000000000ULL;
    const int sh = cE - E - 2;
    unsigned long long X = sh >= 0 ? (sh < 64 ? m >> sh : 0ULL) : (m << (-sh));
    if (E == 0) X = 0;
    return bits < 0 ? -(long long)X : (long long)X;
}

// v * 2^e
__device__ __forceinline__ double scale2(double v, int e) {
    if (e >= -1022 && e <= 1023) return v * __longlong_as_double((long long)(e + 1023) << 52);
    return ldexp(v, e);
}

// The 16 values of one (column, 16-deep k chunk) as 7 digit planes of 16 bytes
// (plane i = byte 6 - i of the fixed-point two's complement).
__device__ __forceinline__ void pack_digits(const double (&v)[16], int cE, uint32_t (&w)[kDigits][4]) {
#pragma unroll
    for (int qd = 0; qd < 4; ++qd) {
        const long long X0 = to_fixed(v[4 * qd], cE), X1 = to_fixed(v[4 * qd + 1], cE),
                        X2 = to_fixed(v[4 * qd + 2], cE), X3 = to_fixed(v[4 * qd + 3], cE);
        const uint32_t l0 = (uint32_t)X0, l1 = (uint32_t)X1, l2 = (uint32_t)X2, l3 = (uint32_t)X3;
        const uint32_t h0 = (uint32_t)(X0 >> 32), h1 = (uint32_t)(X1 >> 32), h2 = (uint32_t)(X2 >> 32),
                       h3 = (uint32_t)(X3 >> 32);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t s = (uint32_t)(b | ((b + 4) << 4));
            w[6 - b][qd] = __byte_perm(__byte_perm(l0, l1, s), __byte_perm(l2, l3, s), 0x5410);
        }
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const uint32_t s = (uint32_t)(b | ((b + 4) << 4));
            w[2 - b][qd] = __byte_perm(__byte_perm(h0, h1, s), __byte_perm(h2, h3, s), 0x5410);
        }
    }
}

// Seven int32 level accumulators -> sum_s acc_s 2^(8 (6 - s)) as fp64 (one
// rounding).  The sum is split into exact int64 halves (|hi| < 2^43, |lo| < 2^51)
// turned into doubles by the magic-number trick (integer add into the significand
// of 1.5 * 2^84 resp. 1.5 * 2^52, one DADD each) -- FP64-pipe work instead of the
// slow I2F.F64 conversion unit.
__device__ __forceinline__ double combine_levels(int a0, int a1, int a2, int a3, int a4, int a5, int a6) {
    const long long hi = (long long)a0 * 65536 + (long long)a1 * 256 + a2;
    const long long lo = (long long)a3 * 16777216 + (long long)a4 * 65536 + (long long)a5 * 256 + a6;
    const double dh = __longlong_as_double(0x4538000000000000LL + hi) - 29014219670751100192948224.0;  // hi * 2^32
    const double dl = __longlong_as_double(0x4338000000000000LL + lo) - 6755399441055744.0;             // lo
    return dh + dl;
}

// 2^e for a row / column scale exponent (0 below the normal range: such rows /
// columns are negligible against 2^-1022)
__device__ __forceinline__ double pow2(int e) {
    return e < -1022 ? 0.0 : __longlong_as_double((long long)(min(e, 1023) + 1023) << 52);
}

// ------------------------------------------------------------------ Legendre inverse
// CTA of 8 warps.  Per column tile: (1) threads (c, kc) load 16 k-values of
// column c, the column scale is an atomicMax of biased exponents, the digits
// go to shared memory as 7 planes; (2) the TMEM accumulators (7 levels x 32
// columns, 256 columns allocated: two CTAs per SM can hold theirs, so one's
// epilogue overlaps the other's MMAs) are allocated and one thread issues the
// 28 int8 GEMMs per 32-deep k step; (3) the 8 warps drain them with 16x256b
// loads and store G.
template <int KPMAX>
__global__ void __launch_bounds__(256, KPMAX > 64 ? 1 : 2) leginv_i8_kernel(const __grid_constant__ LegInvI8 P) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ int colE[kTileN];
    __shared__ double rowS[kTileM];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) unsigned long long bars[2];  // table image, MMA completion
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const Unit u = P.units[blockIdx.x];
    const Geo& g = P.g;
    const int B = g.B, am = u.pid >> 1, p = u.pid & 1;
    const int K = (B - am - p) > 0 ? (B - am - p + 1) / 2 : 0;
    const int Kp = P.kpad[u.pid];
    const int NB = (int)g.NB;
    uint8_t* sA = sm;
    uint8_t* sB = sm + kDigits * KPMAX * kTileM;
    long long* trace = P.trace ? P.trace + (long long)blockIdx.x * 64 : nullptr;  // phase clocks (experiments)
#define OZ_MARK(i) \
    if (trace && tid == 0 && t < 8) trace[t * 8 + (i)] = clock64();
    const uint32_t aA = su32(sA), aB = su32(sB);
    const uint32_t bar_tab = su32(&bars[0]), bar_mma = su32(&bars[1]);
    if (tid == 0) {
        bar_init(bar_tab, 1);
        bar_init(bar_mma, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int tix = u.pid * P.mtiles + u.mt;
    if (tid == 0 && K > 0) bulk_load(aA, P.img + P.img_off[tix], (uint32_t)(kDigits * Kp * kTileM), bar_tab);
    if (tid < kTileM) rowS[tid] = pow2(P.rexp[tix * kTileM + tid]);

    const int ntiles_half = (NB + kTileN - 1) / kTileN;
    const int ntl = min(P.tpc, ntiles_half - u.nt0);  // tiles of this unit
    const int nkc = Kp / 16;
    const int c = tid & (kTileN - 1), kc0 = tid / kTileN;  // conversion: column, first 16-deep k chunk
    constexpr int CPT = KPMAX / 16 / (256 / kTileN);      // k chunks per thread
    const int rs = g_rowstride(g);
    const bool neg = u.half == 1 && (am & 1);  // the reference's sign of odd negative m
    // epilogue geometry: warp w drains lanes 32 (w % 4) + 16 (w / 4) .. + 15
    const int q = warp & 3, hh = warp >> 2, t0 = lane & 3, t1 = lane >> 2;
    const int ra = q * 32 + hh * 16 + t1, rb = ra + 8;
    const int jpa = u.mt * kTileM + ra, jpb = jpa + 8;
    uint32_t mma_phase = 0;
    for (int t = 0; t < ntl; ++t) {
        const int nloc0 = (u.nt0 + t) * kTileN;  // first column inside the sign half
        const int ncols = min(kTileN, NB - nloc0);
        const int n0 = u.half * NB + nloc0;
        OZ_MARK(0)
        // ---- data tile: fp64 -> per-column scale -> 7 digit planes (B operand)
        if (tid < kTileN) colE[tid] = 0;
        __syncthreads();
        double v[CPT][16];
        {
            int mE = 0;
            const long long cb = c < ncols ? (long long)s_col(g, P.sv, am, n0 + c) : 0;
#pragma unroll
            for (int ci = 0; ci < CPT; ++ci) {
                const int kc = kc0 + ci * (256 / kTileN);
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const int k = kc * 16 + r;
                    double x = 0.0;
                    if (k < K && c < ncols) {
                        const long long l = am + p + 2 * k;
                        x = __ldg(P.S + l * (l + 1) * P.sv.NB + cb);
                    }
                    v[ci][r] = x;
                    mE = max(mE, exp_bits(x));
                }
            }
            if (mE) atomicMax(&colE[c], mE);
        }
        __syncthreads();
        OZ_MARK(1)
#pragma unroll
        for (int ci = 0; ci < CPT; ++ci) {
            const int kc = kc0 + ci * (256 / kTileN);
            if (kc >= nkc) continue;
            uint32_t w[kDigits][4];
            pack_digits(v[ci], colE[c], w);
#pragma unroll
            for (int i = 0; i < kDigits; ++i)
                *reinterpret_cast<uint4*>(sB + i * (Kp * kTileN) + kc * (kTileN * 16) + c * 16) =
                    make_uint4(w[i][0], w[i][1], w[i][2], w[i][3]);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // digits -> tensor-core (async) proxy
        // ---- tensor cores: 28 int8 GEMMs per 32-deep k step into 7 level accumulators
        if (K > 0 && warp == 0) {
            tmem_alloc(su32(&tmem_base), kTmemCols);
            if (t == ntl - 1) tmem_relinquish();
        }
        fence_before();
        __syncthreads();
        fence_after();
        OZ_MARK(2)
        const uint32_t td = tmem_base;
        if (K > 0 && tid == 0) {
            if (t == 0) bar_wait(bar_tab, 0);
            fence_after();
            // descriptors advance by adding (byte offset >> 4) to the start-address field
            const uint64_t da0 = sdesc(aA, kTileM * 16, 128), db0 = sdesc(aB, kTileN * 16, 128);
            const uint32_t pa = (uint32_t)(Kp * kTileM) >> 4, pb = (uint32_t)(Kp * kTileN) >> 4;
            for (int ks = 0; ks < Kp / 32; ++ks) {
#pragma unroll
                for (int i = 0; i < kDigits; ++i) {
#pragma unroll
                    for (int j = 0; i + j <= kMaxLevel; ++j)
                        mma_i8_1(td + (uint32_t)((i + j) * kTileN), da0 + (i * pa + ks * (2 * kTileM)),
                                 db0 + (j * pb + ks * (2 * kTileN)), idesc_i8(kTileM, kTileN, i == 0, j == 0),
                                 (ks | i) ? 1u : 0u);
                }
            }
            mma_commit_1(bar_mma);
        }
        OZ_MARK(3)
        if (K > 0) {
            bar_wait(bar_mma, mma_phase);
            mma_phase ^= 1;
        }
        OZ_MARK(4)
        fence_after();
        // ---- epilogue: levels -> fp64, scaled, stored into the blocked G (four
        // threads per row, 64-byte runs)
        {
            const double sa = rowS[ra], sb = rowS[rb];
            double* outa = P.G + (long long)jpa * rs;
            double* outb = P.G + (long long)jpb * rs;
            const uint32_t tl = td + ((uint32_t)(q * 32 + hh * 16) << 16);
#pragma unroll 1
            for (int ch2 = 0; ch2 < kTileN / 16; ++ch2) {
                int a[2][kLevels][4] = {};
                if (K > 0) {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int s = 0; s < kLevels; ++s)
                            tmem_ld16x256(tl + (uint32_t)(s * kTileN + ch2 * 16 + h * 8), a[h][s]);
                    tmem_wait_ld();
                }
                if (ch2 == 0) {
                    OZ_MARK(7)
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cc = ch2 * 16 + h * 8 + 2 * t0;  // this thread's first column in the tile
                    const int e0 = colE[cc], e1 = colE[cc + 1];
                    const double s0 = e0 ? pow2(e0 - 1084) : 0.0, s1 = e1 ? pow2(e1 - 1084) : 0.0;
                    double o[4];
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const double cs = (w & 1) ? s1 : s0;
                        if (SGL_OZ_EXP & 2)
                            o[w] = (double)(a[h][0][w] + a[h][1][w] + a[h][2][w] + a[h][3][w] + a[h][4][w] + a[h][5][w] + a[h][6][w]);
                        else
                            o[w] = combine_levels(a[h][0][w], a[h][1][w], a[h][2][w], a[h][3][w], a[h][4][w], a[h][5][w],
                                                  a[h][6][w]) *
                                   ((w & 2) ? sb : sa) * (neg ? -cs : cs);
                    }
                    if ((SGL_OZ_EXP & 1) && o[0] != 1.2345e-300) continue;
                    if (cc < ncols) {
                        const int off = g_col(g, p, am, n0 + cc);
                        if (jpa < B) *reinterpret_cast<double2*>(outa + off) = make_double2(o[0], o[1]);
                        if (jpb < B) *reinterpret_cast<double2*>(outb + off) = make_double2(o[2], o[3]);
                    }
                }
            }
        }
        OZ_MARK(5)
        fence_before();
        __syncthreads();
        if (K > 0 && warp == 0) tmem_dealloc(td, kTmemCols);
        OZ_MARK(6)
    }
#undef OZ_MARK
}

size_t leginv_smem(int B) {
    const int kp = B > 128 ? 128 : 64;
    return (size_t)kDigits * kp * (kTileM + kTileN);  // table image + data digits
}

int launch_legendre_inverse_i8(const LegInvI8& prm, int nunits, cudaStream_t s) {
    if (nunits <= 0) return 0;
    const size_t smem = leginv_smem(prm.g.B);
    if (prm.g.B > 128) {
        static SmemAttrOnce attr;
        attr.ensure(leginv_i8_kernel<128>, smem);
        leginv_i8_kernel<128><<<nunits, 256, smem, s>>>(prm);
    } else {
        static SmemAttrOnce attr;
        attr.ensure(leginv_i8_kernel<64>, smem);
        leginv_i8_kernel<64><<<nunits, 256, smem, s>>>(prm);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// ------------------------------------------------------------------ Legendre inverse, warp-specialised
__device__ __forceinline__ void bar_arrive(uint32_t a) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// 16 lanes x 16 columns: v[0..3] as tmem_ld16x256 for columns 0..7, v[4..7] for 8..15
__device__ __forceinline__ void tmem_ld16x256x2(uint32_t taddr, int (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

template <int KPMAX, int NT>
__global__ void __launch_bounds__(512, 1) leginv_ws_kernel(const __grid_constant__ LegInvI8 P) {
    constexpr int NR = kDigits * NT;        // stacked data-digit rows (224 / 448)
    constexpr int SB = KPMAX * NR;          // bytes per data stage
    constexpr int TM = kLevels * NT;        // TMEM columns per buffer
    constexpr int NBUF = 2 * TM <= 512 ? 2 : 1;  // TMEM buffers (64-column tiles: one, drained early)
    constexpr int NPW = 7;                  // producer warps (9 .. 15)
    constexpr int CPT = (NT * (KPMAX / 16) + 32 * NPW - 1) / (32 * NPW);  // (column, 16-deep k chunk) pairs per thread
    constexpr int FST = KPMAX > 64 ? 1 : 3;            // fp64 staging buffers (tiles in flight)
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* sA = sm;
    uint8_t* sB = sm + kDigits * KPMAX * kTileM;
    double* sF = reinterpret_cast<double*>(sB + 2 * SB);
    __shared__ int colE[4][NT];
    // 0 table, 1-2 data full, 3-4 data empty, 5-6 TMEM full, 7-8 TMEM empty
    __shared__ __align__(8) unsigned long long bars[9];
    __shared__ uint32_t tmem_base;
    __shared__ int s_unit;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const Geo& g = P.g;
    const int B = g.B, NB = (int)g.NB;
    const int ntl = (NB + NT - 1) / NT;  // column tiles of a sign half
    const int rs = g_rowstride(g);
    auto bar = [&](int i) { return su32(&bars[i]); };
    if (tid == 0) {
        bar_init(bar(0), 1);
        for (int s = 0; s < 2; ++s) {
            bar_init(bar(1 + s), 1);
            bar_init(bar(3 + s), 1);
            bar_init(bar(5 + s), 1);
            bar_init(bar(7 + s), 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 8) tmem_alloc(su32(&tmem_base), 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t td = tmem_base;
    // persistent: units (problem, m-tile, sign half; heaviest first) from a global
    // counter; T0 = tiles this CTA ran before the unit (barrier phases continue)
    int T0 = 0, nunit = 0;
    for (;;) {
        if (tid == 0) s_unit = atomicAdd(P.counter, 1);
        __syncthreads();
        const int ui = s_unit;
        if (ui >= P.nunits) break;
        const Unit u = P.units[ui];
        const int am = u.pid >> 1, p = u.pid & 1;
        const int K = (B - am - p) > 0 ? (B - am - p + 1) / 2 : 0;
        const int Kp = P.kpad[u.pid];
        const int tix = u.pid * P.mtiles + u.mt;
        const bool neg = u.half == 1 && (am & 1);  // the reference's sign of odd negative m
        if (K == 0) {  // no degrees of this parity: G is zero there
            for (int e = tid; e < kTileM * NB; e += blockDim.x) {
                const int r = e / NB, c = e - r * NB, jp = u.mt * kTileM + r;
                if (jp < B && (c & 1) == 0)
                    *reinterpret_cast<double2*>(P.G + (long long)jp * rs + g_col(g, p, am, u.half * NB + c)) =
                        make_double2(0.0, 0.0);
            }
        } else if (warp >= 9) {
            // ---- producers: S tile -> column scales -> stacked unsigned digit planes.
            // The fp64 tile is staged by cp.async (8-byte copies, one row of 32
            // columns per warp instruction), FST - 1 tiles ahead.
            if (tid == 288) bulk_load(su32(sA), P.img + P.img_off[tix], (uint32_t)(kDigits * Kp * kTileM), bar(0));
            const int pt = tid - 288, wp = pt >> 5;
            const int nkc = Kp / 16;
            auto stage_tile = [&](int t) {  // cp.async of tile t's S rows into staging buffer (T0 + t) % FST
                const int nloc0 = t * NT, ncols = min(NT, NB - nloc0), n0 = u.half * NB + nloc0;
#pragma unroll
                for (int cc = 0; cc < NT / 32; ++cc) {
                    const int c = lane + 32 * cc;
                    if (c < ncols) {
                        const double* src = P.S + s_col(g, P.sv, am, n0 + c);
                        double* dst = sF + ((T0 + t) % FST) * (KPMAX * NT) + c;
                        for (int k = wp; k < K; k += NPW) {
                            const long long l = am + p + 2 * k;
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(su32(dst + k * NT)),
                                         "l"(src + l * (l + 1) * P.sv.NB));
                        }
                    }
                }
                cp_async_commit();
            };
            stage_tile(0);
            if (FST == 3) {
                if (1 < ntl) stage_tile(1);
                else cp_async_commit();
            }
            for (int t = 0; t < ntl; ++t) {
                const int T = T0 + t, s = T & 1;
                const int ncols = min(NT, NB - t * NT);
                if (FST == 3) {
                    if (t + 2 < ntl) stage_tile(t + 2);
                    else cp_async_commit();
                    cp_async_wait_group<2>();
                } else {
                    cp_async_wait_group<0>();
                }
                if (T >= 2) bar_wait(bar(3 + s), ((T >> 1) - 1) & 1);  // the MMAs of tile T - 2 have read stage s
                if (pt < NT) colE[T & 3][pt] = 0;
                named_sync(1, 32 * NPW);
                double v[CPT][16];
                {
                    const double* fs = sF + (T % FST) * (KPMAX * NT);
#pragma unroll
                    for (int ci = 0; ci < CPT; ++ci) {
                        const int pr = pt + 32 * NPW * ci, c = pr % NT, kc = pr / NT;
                        int mE = 0;
#pragma unroll
                        for (int r = 0; r < 16; ++r) {
                            const int k = kc * 16 + r;
                            const double x = (k < K && c < ncols && kc < nkc) ? fs[k * NT + c] : 0.0;
                            v[ci][r] = x;
                            mE = max(mE, exp_bits(x));
                        }
                        if (mE) atomicMax(&colE[T & 3][c], mE);
                    }
                }
                named_sync(1, 32 * NPW);
#pragma unroll
                for (int ci = 0; ci < CPT; ++ci) {
                    const int pr = pt + 32 * NPW * ci, c = pr % NT, kc = pr / NT;
                    if (kc >= nkc) continue;
                    // X = trunc(x 2^(55 - e)) + 2^55 (e = cE - 1022; the scale as the product of
                    // two normal powers of two: exact down to subnormals), F2I.S64, PRMT planes
                    const int cE = colE[T & 3][c];
                    const int e = 1077 - cE, e2 = min(e, 1000);
                    const double s2 = __longlong_as_double((long long)(e2 + 1023) << 52);
                    const double s1 = __longlong_as_double((long long)(max(0, e - e2) + 1023) << 52);
                    auto fx = [&](double x) { return __double2ll_rz(x * s1 * s2) + (1LL << 55); };
                    uint8_t* dst = sB + s * SB + kc * (NR * 16) + c * 16;
#pragma unroll
                    for (int qd = 0; qd < 4; ++qd) {
                        const long long X0 = fx(v[ci][4 * qd]), X1 = fx(v[ci][4 * qd + 1]), X2 = fx(v[ci][4 * qd + 2]),
                                        X3 = fx(v[ci][4 * qd + 3]);
                        const uint32_t l0 = (uint32_t)X0, l1 = (uint32_t)X1, l2 = (uint32_t)X2, l3 = (uint32_t)X3;
                        const uint32_t h0 = (uint32_t)(X0 >> 32), h1 = (uint32_t)(X1 >> 32), h2 = (uint32_t)(X2 >> 32),
                                       h3 = (uint32_t)(X3 >> 32);
#pragma unroll
                        for (int bb = 0; bb < 4; ++bb) {
                            const uint32_t sel = (uint32_t)(bb | ((bb + 4) << 4));
                            reinterpret_cast<uint32_t*>(dst + (6 - bb) * (NT * 16))[qd] =
                                __byte_perm(__byte_perm(l0, l1, sel), __byte_perm(l2, l3, sel), 0x5410);
                        }
#pragma unroll
                        for (int bb = 0; bb < 3; ++bb) {
                            const uint32_t sel = (uint32_t)(bb | ((bb + 4) << 4));
                            reinterpret_cast<uint32_t*>(dst + (2 - bb) * (NT * 16))[qd] =
                                __byte_perm(__byte_perm(h0, h1, sel), __byte_perm(h2, h3, sel), 0x5410);
                        }
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                named_sync(1, 32 * NPW);
                if (pt == 0) bar_arrive(bar(1 + s));
                if (FST == 1 && t + 1 < ntl) stage_tile(t + 1);
            }
        } else if (warp == 8) {
            // ---- MMA issuer: per 32-deep k step, digit i of the table against the
            // stacked data planes 0 .. 6 - i (N = 32 (7 - i)) into levels i .. 6
            if (lane == 0) {
                bar_wait(bar(0), nunit & 1);
                const uint32_t aA = su32(sA), aB = su32(sB);
                const uint32_t pa = (uint32_t)(Kp * kTileM);
                for (int t = 0; t < ntl; ++t) {
                    const int T = T0 + t, s = T & 1, b = T % NBUF;
                    bar_wait(bar(1 + s), (T >> 1) & 1);
                    if (T >= NBUF) bar_wait(bar(7 + b), ((T / NBUF) - 1) & 1);
                    fence_after();
                    for (int ks = 0; ks < Kp / 32; ++ks) {
                        const uint32_t b0 = aB + s * SB + ks * 2 * (NR * 16);
#pragma unroll
                        for (int i = 0; i < kDigits; ++i) {
                            const uint64_t da = sdesc(aA + i * pa + ks * 2 * (kTileM * 16), kTileM * 16, 128);
                            const int rows = (kDigits - i) * NT;
#pragma unroll
                            for (int a0 = 0; a0 < rows; a0 += 256) {
                                const int n = min(256, rows - a0);
                                mma_i8_1(td + (uint32_t)(b * TM + i * NT + a0), da, sdesc(b0 + a0 * 16, NR * 16, 128),
                                         idesc_i8(kTileM, n, i == 0, false), (ks | i) ? 1u : 0u);
                            }
                        }
                    }
                    mma_commit_1(bar(3 + s));
                    mma_commit_1(bar(5 + b));
                }
            }
            __syncwarp();
        } else {
            // ---- epilogue: warp w drains TMEM lanes 32 (w % 4) + 16 (w / 4) .. + 15
            // with 16x256b loads (four threads per row, 64-byte store runs) and
            // releases the buffer after its last load
            const int q = warp & 3, h = warp >> 2, t0 = lane & 3, t1 = lane >> 2;
            // per row (w: +0 / +8): scale 2^e, and the magic constants of the int64 ->
            // fp64 conversions with the bias correction folded in (hi: levels 0-2,
            // lo: levels 3-6; exact in int64)
            double rsc[2];
            long long mhi[2], mlo[2];
#pragma unroll
            for (int w = 0; w < 2; ++w) {
                const int row = q * 32 + h * 16 + t1 + 8 * w;
                rsc[w] = pow2(P.rexp[tix * kTileM + row]);
                const int* cr = P.corr + (size_t)tix * kDigits * kTileM + row;
                mhi[w] = 0x4538000000000000LL - ((long long)cr[0] * 65536 + (long long)cr[kTileM] * 256 + cr[2 * kTileM]);
                mlo[w] = 0x4338000000000000LL - ((long long)cr[3 * kTileM] * 16777216 + (long long)cr[4 * kTileM] * 65536 +
                                                 (long long)cr[5 * kTileM] * 256 + cr[6 * kTileM]);
            }
            const int ja = u.mt * kTileM + q * 32 + h * 16 + t1;
            double* outa = P.G + (long long)ja * rs;
            double* outb = P.G + (long long)(ja + 8) * rs;
            for (int t = 0; t < ntl; ++t) {
                const int T = T0 + t, b = T % NBUF;
                const int nloc0 = t * NT, ncols = min(NT, NB - nloc0), n0 = u.half * NB + nloc0;
                bar_wait(bar(5 + b), (T / NBUF) & 1);
                fence_after();
                const uint32_t ta = td + ((uint32_t)(q * 32 + h * 16) << 16) + (uint32_t)(b * TM);
#pragma unroll
                for (int cp = 0; cp < NT / 16; ++cp) {
                    int a[kLevels][8];
#pragma unroll
                    for (int lv = 0; lv < kLevels; ++lv) tmem_ld16x256x2(ta + (uint32_t)(lv * NT + cp * 16), a[lv]);
                    tmem_wait_ld();
                    if (cp == NT / 16 - 1) {  // this warp's last TMEM load of the buffer
                        fence_before();
                        __syncwarp();
                        if (lane == 0) bar_arrive(bar(7 + b));
                    }
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const int cc = cp * 16 + r * 8 + 2 * t0;
                        double cs[2];
#pragma unroll
                        for (int y = 0; y < 2; ++y) {
                            const int e = colE[T & 3][cc + y];
                            const double sc = e ? pow2(e - 1084) : 0.0;
                            cs[y] = neg ? -sc : sc;
                        }
                        double o[4];
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            const int w = x >> 1, vi = r * 4 + x;  // x: (row w, column x & 1)
                            if (SGL_OZ_EXP & 2) {
                                o[x] = (double)(a[0][vi] + a[3][vi] + a[6][vi]);
                                continue;
                            }
                            const long long hi = (long long)a[0][vi] * 65536 + (long long)a[1][vi] * 256 + a[2][vi] + mhi[w];
                            const long long lo = (long long)a[3][vi] * 16777216 + (long long)a[4][vi] * 65536 +
                                                 (long long)a[5][vi] * 256 + a[6][vi] + mlo[w];
                            const double dh = __longlong_as_double(hi) - 29014219670751100192948224.0;
                            const double dl = __longlong_as_double(lo) - 6755399441055744.0;
                            o[x] = (dh + dl) * rsc[w] * cs[x & 1];
                        }
                        if ((SGL_OZ_EXP & 1) && o[0] != 1.2345e-300) continue;
                        if (cc < ncols) {
                            const int off = g_col(g, p, am, n0 + cc);
                            if (ja < B) *reinterpret_cast<double2*>(outa + off) = make_double2(o[0], o[1]);
                            if (ja + 8 < B) *reinterpret_cast<double2*>(outb + off) = make_double2(o[2], o[3]);
                        }
                    }
                }
            }
        }
        if (K > 0) {
            T0 += ntl;
            ++nunit;
        }
        fence_before();
        __syncthreads();  // every MMA of the unit has completed (the epilogue drained them): the table may be reloaded
        fence_after();
    }
    fence_before();
    __syncthreads();
    if (warp == 8) tmem_dealloc(td, 512);
}

int ws_tile_columns(int B) {
    const char* e = std::getenv("SGL_I8_WSN");
    return (B <= 128 && e && std::atoi(e) == 64) ? 64 : 32;
}

size_t leginv_ws_smem(int B) {
    const int kp = B > 128 ? 128 : 64;
    const int fst = B > 128 ? 1 : 3;  // fp64 staging buffers (FST in the kernel)
    const int nt = ws_tile_columns(B);
    return (size_t)kDigits * kp * kTileM + 2 * (size_t)kp * kDigits * nt + (size_t)fst * kp * nt * 8;
}

int launch_legendre_inverse_ws(const LegInvI8& prm_in, int nunits, cudaStream_t s) {
    if (nunits <= 0) return 0;
    LegInvI8 prm = prm_in;
    prm.nunits = nunits;
    if (cudaMemsetAsync(prm.counter, 0, sizeof(int), s) != cudaSuccess) return -1;
    const size_t smem = leginv_ws_smem(prm.g.B);
    const int grid = std::min(nunits, prm.grid);
    if (prm.g.B > 128) {
        static SmemAttrOnce attr;
        attr.ensure(leginv_ws_kernel<128, 32>, smem);
        leginv_ws_kernel<128, 32><<<grid, 512, smem, s>>>(prm);
    } else if (ws_tile_columns(prm.g.B) == 64) {
        static SmemAttrOnce attr;
        attr.ensure(leginv_ws_kernel<64, 64>, smem);
        leginv_ws_kernel<64, 64><<<grid, 512, smem, s>>>(prm);
    } else {
        static SmemAttrOnce attr;
        attr.ensure(leginv_ws_kernel<64, 32>, smem);
        leginv_ws_kernel<64, 32><<<grid, 512, smem, s>>>(prm);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

std::vector<Unit> leginv_ws_units(int B, long long NB, bool real) {
    const int mtiles = (B + kTileM - 1) / kTileM;
    struct W {
        int K;
        Unit u;
    };
    std::vector<W> ws;
    for (int pid = 0; pid < 2 * B; ++pid) {
        const int am = pid >> 1, p = pid & 1, r = B - am - p;
        const int K = r > 0 ? (r + 1) / 2 : 0;
        const int halves = (am == 0 || real) ? 1 : 2;
        for (int mt = 0; mt < mtiles; ++mt)
            for (int h = 0; h < halves; ++h) ws.push_back({(K + 31) / 32, Unit{pid, mt, h, 0}});
    }
    std::stable_sort(ws.begin(), ws.end(), [](const W& a, const W& b) { return a.K > b.K; });
    std::vector<Unit> us;
    for (const W& w : ws) us.push_back(w.u);
    (void)NB;
    return us;
}

// ------------------------------------------------------------------ host: table images and units
namespace {
// 7 digit bytes of trunc(y * 2^(55 - e)) (digit 0 most significant, signed)
void digits_of(double y, int e, uint8_t (&d)[kDigits]) {
    const double sy = std::ldexp(y, 55 - e);
    const long long X = (long long)std::trunc(sy);
    for (int i = 0; i < kDigits; ++i) d[i] = (uint8_t)((unsigned long long)X >> (8 * (6 - i)));
}
}  // namespace

TableImage build_leginv_image(int B, const std::vector<double>& leg, const std::vector<long long>& leg_off) {
    TableImage im;
    const int LS = B + (B & 1);
    im.mtiles = (B + kTileM - 1) / kTileM;
    const int np = 2 * B;
    im.off.assign((size_t)np * im.mtiles, -1);
    im.kpad.assign(np, 0);
    im.rexp.assign((size_t)np * im.mtiles * kTileM, 0);
    im.corr.assign((size_t)np * im.mtiles * kDigits * kTileM, 0);
    size_t total = 0;
    for (int pid = 0; pid < np; ++pid) {
        const int am = pid >> 1, p = pid & 1, r = B - am - p;
        const int K = r > 0 ? (r + 1) / 2 : 0;
        im.kpad[pid] = (K + 31) / 32 * 32;
        for (int mt = 0; mt < im.mtiles; ++mt) {
            if (K == 0) continue;
            im.off[(size_t)pid * im.mtiles + mt] = (long long)total;
            total += (size_t)kDigits * im.kpad[pid] * kTileM;
        }
    }
    im.bytes.assign(total, 0);
    for (int pid = 0; pid < np; ++pid) {
        const int am = pid >> 1, p = pid & 1, r = B - am - p;
        const int K = r > 0 ? (r + 1) / 2 : 0, Kp = im.kpad[pid];
        if (K == 0) continue;
        for (int mt = 0; mt < im.mtiles; ++mt) {
            uint8_t* base = im.bytes.data() + im.off[(size_t)pid * im.mtiles + mt];
            for (int rr = 0; rr < kTileM; ++rr) {
                const int jp = mt * kTileM + rr;
                if (jp >= B) continue;
                double mx = 0.0;
                for (int k = 0; k < K; ++k) mx = std::max(mx, std::fabs(leg[leg_off[pid] + (long long)k * LS + jp]));
                int e = 0;
                if (mx > 0) std::frexp(mx, &e);
                im.rexp[((size_t)pid * im.mtiles + mt) * kTileM + rr] = e;
                if (mx == 0) continue;
                int* corr = im.corr.data() + ((size_t)pid * im.mtiles + mt) * kDigits * kTileM + rr;
                for (int k = 0; k < K; ++k) {
                    uint8_t d[kDigits];
                    digits_of(leg[leg_off[pid] + (long long)k * LS + jp], e, d);
                    for (int i = 0; i < kDigits; ++i) {
                        base[(size_t)i * Kp * kTileM + (size_t)(k / 16) * (kTileM * 16) + rr * 16 + (k % 16)] = d[i];
                        corr[i * kTileM] += 128 * (i == 0 ? (int)(int8_t)d[i] : (int)d[i]);
                    }
                }
            }
        }
    }
    return im;
}

std::vector<Unit> leginv_units(int B, long long NB, bool real, int tpc) {
    const int mtiles = (B + kTileM - 1) / kTileM;
    const int nth = (int)((NB + kTileN - 1) / kTileN);
    struct W {
        int K;
        Unit u;
    };
    std::vector<W> ws;
    for (int pid = 0; pid < 2 * B; ++pid) {
        const int am = pid >> 1, p = pid & 1, r = B - am - p;
        const int K = r > 0 ? (r + 1) / 2 : 0;
        const int halves = (am == 0 || real) ? 1 : 2;
        for (int mt = 0; mt < mtiles; ++mt)
            for (int h = 0; h < halves; ++h)
                for (int nt = 0; nt < nth; nt += tpc) ws.push_back({K, Unit{pid, mt, h, nt}});
    }
    std::stable_sort(ws.begin(), ws.end(), [](const W& a, const W& b) { return a.K > b.K; });
    std::vector<Unit> us;
    us.reserve(ws.size());
    for (const W& w : ws) us.push_back(w.u);
    return us;
}

}  // namespace oz
}  // namespace sglk
