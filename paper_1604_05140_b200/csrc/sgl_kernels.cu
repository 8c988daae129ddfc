// sm_100a kernels of the SGL transform pair (fsglft / ifsglft of
// /root/reference/proj/core/src/sgl_transform.cpp:274-348), re-designed for B200:
//
//  * az_forward / az_inverse  -- the per-ring azimuthal DFT of length 2B
//    (reference: DftPlan::forward_rows / synthesize_rows, kernels.cpp:478-502,
//    FftCore radix-2, kernels.cpp:85-195) as a shared-memory Stockham FFT with
//    in-register radix-16 butterflies.  The forward epilogue applies b_cal
//    (spherical_transform.cpp:214-220), folds each ring with its equatorial mirror
//    (theta_{2B-1-j} = pi - theta_j) into even/odd parts and scatters to the
//    m-major intermediate G; the inverse prologue undoes the fold and drops the
//    Nyquist bin (spherical_transform.cpp:295-303).
//  * legendre_forward / legendre_inverse -- the polar Legendre contraction,
//    mathematically sum_j Pbar_lm(cos theta_j) b_j G_m[j] (the reference does it
//    seminaively: DCT/DST + truncated rows, spherical_transform.cpp:222-243 and
//    273-294).  Here it is a direct contraction over the folded K = B polar nodes
//    as grouped fp64 DMMA (mma.sync m8n8k4 .f64) GEMMs, one problem per
//    (|m|, parity); +m and -m share the table and are batched along N.
//  * radial_forward / radial_inverse -- the discrete R transform per (l, m)
//    (drt_forward / drt_inverse, radial_transform.cpp:75-133) as one grouped DMMA
//    GEMM per l, shared by all 2l+1 orders m and all functions of the batch.
//
// All arithmetic is fp64.
#include "sgl_kernels.cuh"

#include <cuda.h>  // CUtensorMap (the TMA descriptor type; no driver-library link)
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdlib>
#include <type_traits>
#include <utility>

namespace sglk {

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }

// e^{SIGN * 2 pi i k / 16} times a, k compile-time after unrolling.
template <int SIGN>
__device__ __forceinline__ double2 rot16(double2 a, int k) {
    constexpr double c1 = 0.92387953251128675613;  // cos(pi/8)
    constexpr double s1 = 0.38268343236508977173;  // sin(pi/8)
    constexpr double h = 0.70710678118654752440;   // cos(pi/4)
    k &= 15;
    if (k == 0) return a;
    if (k == 4) return SIGN > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
    if (k == 8) return make_double2(-a.x, -a.y);
    if (k == 12) return SIGN > 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
    double c, s;
    switch (k) {
        case 1: c = c1; s = s1; break;
        case 2: c = h; s = h; break;
        case 3: c = s1; s = c1; break;
        case 5: c = -s1; s = c1; break;
        case 6: c = -h; s = h; break;
        case 7: c = -c1; s = s1; break;
        case 9: c = -c1; s = -s1; break;
        case 10: c = -h; s = -h; break;
        case 11: c = -s1; s = -c1; break;
        case 13: c = s1; s = -c1; break;
        case 14: c = h; s = -h; break;
        default: c = c1; s = -s1; break;  // 15
    }
    if (SIGN < 0) s = -s;
    return cmul(a, make_double2(c, s));
}

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
__host__ __device__ constexpr int brevc(int x, int bits) {
    int r = 0;
    for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
    return r;
}

// In-register DFT of size R <= 16, natural order in and out:
// y_p = sum_q x_q e^{SIGN 2 pi i p q / R}.
template <int R, int SIGN>
__device__ __forceinline__ void dft_reg(double2 (&v)[R]) {
    constexpr int bits = ilog2c(R);
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int j = brevc(i, bits);
        if (i < j) {
            const double2 t = v[i];
            v[i] = v[j];
            v[j] = t;
        }
    }
#pragma unroll
    for (int len = 2; len <= R; len <<= 1) {
#pragma unroll
        for (int i = 0; i < R; i += len) {
#pragma unroll
            for (int j = 0; j < len / 2; ++j) {
                const double2 t = rot16<SIGN>(v[i + j + len / 2], j * (16 / len));
                v[i + j + len / 2] = csub(v[i + j], t);
                v[i + j] = cadd(v[i + j], t);
            }
        }
    }
}

// Padded position of element x inside a ring in shared memory (one pad slot per
// 16 elements keeps the radix-16 scatters bank-conflict free).
__device__ __forceinline__ int phys(int x) { return x + (x >> 4); }

#ifndef SGL_AZ_ELEMS
#define SGL_AZ_ELEMS 1024  // ring elements per shell-pair group and CTA (sets IG = SGL_AZ_ELEMS / N)
#endif
#ifndef SGL_AZ_MINB
#define SGL_AZ_MINB 4
#endif

#ifndef SGL_AZI_ELEMS
#define SGL_AZI_ELEMS SGL_AZ_ELEMS  // inverse kernel tile size
#endif
#ifndef SGL_AZ_BIG512
#define SGL_AZ_BIG512 1
#endif
// Geo::az2x (set by the host for large complex batches at B = 64): azimuthal CTAs of twice
// the elements -- 16-shell G groups, twice as long runs for the Legendre GEMMs.  Measured
// (B = 64 x 64, us): az 667 / 680 -> 673 / 708, legendre 479 / 564 -> 435 / 502: -72 per round
// trip; even at 8 functions, worse for one (and for the real path: not used there).
constexpr int kAz2xElems = 2 * SGL_AZ_ELEMS;

template <int N, int ELEMS = SGL_AZ_ELEMS>
struct FFTShape {
    static constexpr int RMAX = N < 16 ? N : 16;
    static constexpr int T = N / RMAX;              // threads per ring
    static constexpr int STRIDE = N + N / 16 + 1;   // padded ring stride (complex)
    static constexpr int LOGN = ilog2c(N);
    static constexpr int R0 = 1 << (LOGN % 4 == 0 ? (N < 16 ? LOGN : 4) : LOGN % 4);  // first radix
    // N = 512 (B = 256) takes twice the elements per CTA: 4-shell G groups (64-byte
    // runs for the Legendre GEMMs instead of 32) at 256 threads and 2 CTAs/SM
    static constexpr int EL = (N >= 512 && SGL_AZ_BIG512) ? 2 * ELEMS : ELEMS;
    static constexpr int IG = (T * 2 <= 256) ? (EL / 16) / T : 1;  // shell pairs per CTA
    static constexpr int THREADS = 2 * IG * T;
    static constexpr int MINB = SGL_AZ_MINB * 128 / THREADS > 0 ? SGL_AZ_MINB * 128 / THREADS : 1;  // CTAs/SM
    // twiddle table: N plain entries, then 15 Ns entries per pass after the first
    // (sgl_tables.cpp); HEAD: a leading small-radix pass
    static constexpr bool HEAD = (R0 != RMAX || N < 16);
    static constexpr int NPASS = (HEAD ? 1 : 0) + ((N >= 16) ? (LOGN - (HEAD ? ilog2c(R0) : 0)) / 4 : 0);
    static constexpr int tw_count() {
        int n = N, ns = HEAD ? R0 : 16;
        for (int p = 1; p < NPASS; ++p, ns *= 16) n += 15 * ns;
        return n;
    }
    static constexpr int TWN = tw_count();
};

// Synchronizes the threads that share a ring pair (j', 2B-1-j'): one warp when
// the pair fits in a warp, else the CTA (uniform control flow in both kernels).
template <int N>
__device__ __forceinline__ void pair_sync() {
    if constexpr (2 * FFTShape<N>::T <= 32) {
        __syncwarp();
    } else {
        __syncthreads();
    }
}

// One Stockham pass of radix R on a ring of length N held by T threads.
// Ns = product of the radices already applied.  twp: this pass's twiddles,
// twp[(r - 1) Ns + k] = e^{-2 pi i r k / (R Ns)} (consecutive threads read
// consecutive entries; a plain e^{-2 pi i x / N} table read at r k N / (R Ns)
// scatters the reads and cost the forward kernel 10 us).  Unused when Ns = 1.
// Inputs come from ld(x), outputs go to st(x, v): the first pass of the forward
// FFT reads global memory directly into registers and the last pass of the
// inverse writes global memory directly, so only the middle exchanges touch
// shared memory.  When IN_PLACE, all reads complete (pair_sync) before any write.
// PAIRED (first pass only, Ns = 1, PER even): thread t runs the consecutive
// butterflies j = t PER + b, so its inputs come in pairs of consecutive elements
// (x, x + 1) that ld2(x, v0, v1) fetches with vector loads; the output position
// j R + r of a first-pass butterfly depends on j alone, so any butterfly-to-thread
// assignment is valid there.
struct NoPairLoad {};
// NS2 (radix 16 after a radix-2 pass, Ns = 2): the pass's twiddles are 1 (k = 0)
// or e^{-+2 pi i r / 32} (k = 1) -- compile-time constants selected per thread
// instead of 15 table loads (the N = 512 inverse was throttled on its global
// load/store queue: lg_throttle in ncu).
template <int N, int R, int SIGN, bool IN_PLACE, class Ld, class St, class Ld2 = NoPairLoad, bool NS2 = false>
__device__ __forceinline__ void stockham_pass(int Ns, int t, const double2* twp, Ld&& ld, St&& st,
                                              Ld2&& ld2 = NoPairLoad{}) {
    constexpr double kC32[16] = {1.00000000000000000000, 0.98078528040323043058, 0.92387953251128673848, 0.83146961230254523567, 0.70710678118654757274, 0.55557023301960228867, 0.38268343236508983729, 0.19509032201612833135, 0.00000000000000006123, -0.19509032201612819257, -0.38268343236508972627, -0.55557023301960195560, -0.70710678118654746172, -0.83146961230254534669, -0.92387953251128673848, -0.98078528040323043058};
    constexpr double kS32[16] = {0.00000000000000000000, 0.19509032201612824808, 0.38268343236508978178, 0.55557023301960217765, 0.70710678118654746172, 0.83146961230254523567, 0.92387953251128673848, 0.98078528040323043058, 1.00000000000000000000, 0.98078528040323043058, 0.92387953251128673848, 0.83146961230254545772, 0.70710678118654757274, 0.55557023301960217765, 0.38268343236508989280, 0.19509032201612860891};
    constexpr int T = FFTShape<N>::T;
    constexpr int NBF = N / R;          // butterflies in this pass
    constexpr int PER = NBF / T;        // butterflies per thread
    constexpr bool PAIRED = !std::is_same_v<std::decay_t<Ld2>, NoPairLoad> && PER % 2 == 0;
    auto bj = [&](int b) { return PAIRED ? t * PER + b : t + b * T; };
    double2 v[PER][R];
    if constexpr (PAIRED) {
#pragma unroll
        for (int b = 0; b < PER; b += 2) {
#pragma unroll
            for (int r = 0; r < R; ++r) ld2(bj(b) + r * NBF, v[b][r], v[b + 1][r]);
        }
    } else {
#pragma unroll
        for (int b = 0; b < PER; ++b) {
            const int j = bj(b);
#pragma unroll
            for (int r = 0; r < R; ++r) v[b][r] = ld(j + r * NBF);
        }
    }
#pragma unroll
    for (int b = 0; b < PER; ++b) {
        const int j = bj(b);
        const int k = j & (Ns - 1);
        if constexpr (NS2 && R == 16) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const double2 w = make_double2(k ? kC32[r] : 1.0, k ? (SIGN > 0 ? kS32[r] : -kS32[r]) : 0.0);
                v[b][r] = cmul(v[b][r], w);
            }
        } else if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                double2 w = twp[(r - 1) * Ns + k];
                if (SIGN > 0) w.y = -w.y;
                v[b][r] = cmul(v[b][r], w);
            }
        }
        dft_reg<R, SIGN>(v[b]);
    }
    if (IN_PLACE) pair_sync<N>();
#pragma unroll
    for (int b = 0; b < PER; ++b) {
        const int j = bj(b);
        const int k = j & (Ns - 1);
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) st(base + r * Ns, v[b][r]);
    }
}

// Full FFT of one ring: first pass reads ld, last pass writes st, middle
// passes run in place on `ring` (padded).  Ends without a trailing sync.
template <int N, int SIGN, bool FIRST_IN_PLACE, class Ld, class St, class Ld2 = NoPairLoad>
__device__ __forceinline__ void ring_fft_io(double2* ring, int t, const double2* tw, Ld&& ld, St&& st,
                                            Ld2&& ld2 = NoPairLoad{}) {
    using S = FFTShape<N>;
    auto rd = [&](int x) { return ring[phys(x)]; };
    auto wr = [&](int x, double2 v) { ring[phys(x)] = v; };
    constexpr bool head = (S::R0 != S::RMAX || N < 16);        // a leading small-radix pass
    constexpr int P16 = (N >= 16) ? (S::LOGN - (head ? ilog2c(S::R0) : 0)) / 4 : 0;
    constexpr int NPASS = (head ? 1 : 0) + P16;
    if constexpr (NPASS == 1) {
        if constexpr (head) stockham_pass<N, S::R0, SIGN, FIRST_IN_PLACE>(1, t, tw, ld, st, ld2);
        else stockham_pass<N, 16, SIGN, FIRST_IN_PLACE>(1, t, tw, ld, st, ld2);
    } else {
        int Ns = 1;
        if constexpr (head) {
            stockham_pass<N, S::R0, SIGN, FIRST_IN_PLACE>(Ns, t, tw, ld, wr, ld2);
            Ns *= S::R0;
        } else {
            stockham_pass<N, 16, SIGN, FIRST_IN_PLACE>(Ns, t, tw, ld, wr, ld2);
            Ns *= 16;
        }
        pair_sync<N>();
        const double2* twp = tw + N;  // per-pass tables follow the N plain twiddles
#pragma unroll 1
        for (int p = 1; p < NPASS - 1; ++p) {
            stockham_pass<N, 16, SIGN, true>(Ns, t, twp, rd, wr);
            twp += 15 * Ns;
            Ns *= 16;
            pair_sync<N>();
        }
        stockham_pass<N, 16, SIGN, true>(Ns, t, twp, rd, st);
    }
}

// ------------------------------------------------------------------ streaming loads
// Read-only streaming loads of the azimuthal kernels: non-coherent path, no L1
// allocation, 256-byte L2 prefetch hint (measured against ld.global.cs:
// az_forward 96.7 -> 95.1 us, az_inverse 93.3 -> 92.6 us at B = 128; the
// .L2::128B / .L2::256B hints on ld.global.cs alone changed nothing; the real
// path's 8-byte loads keep ld.global.cs: the same path measured 4164 -> 4521 us).
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

// L2 eviction-priority policies (createpolicy): streamed-once data (samples in,
// S out) marked evict_first so that the intermediate G, written by one kernel and
// read by the next, is what the L2 keeps (SGL_L2HINTS experiments).
#ifndef SGL_L2HINTS
#define SGL_L2HINTS 0
#endif
__device__ __forceinline__ unsigned long long policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ld_stream_hint(const double2* p, unsigned long long pol) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
}

// Round-trip L2 reuse (round 2): the grid the inverse writes last is what a
// following forward reads first when the forward's CTAs run in reverse order
// (SGL_AZF_REV), provided the inverse's stores stay in L2: SGL_AZI_STORE 0 =
// st.global.cs (streaming), 1 = plain, 2 = L2 evict_last.  Measured at B = 128
// (exp/l2order.sh, stage times): az_forward 95.8 -> 92.6 us reversed -> 91.0 with
// plain stores -> 90.7 with evict_last (and the Legendre stages ~1 us faster).
// The same trick for G (SGL_AZI_REV or the polar-slab-major tile order of the
// Legendre inverse, SGL_LEGINV_ORDER in sgl_capi.cpp) costs the Legendre inverse
// 3.3 us and gains the azimuthal inverse 1.7: off.  SGL_AZI_LOAD 1 = the G
// loads marked L2 evict_first (no change).
// N = 512 (B = 256): the radix-2 pass of the (2, 16, 16) ring FFT fused into the
// kernels' own shared-memory traffic -- forward as radices (16, 16) with the
// final radix-2 butterfly done by the epilogue on its ring reads, inverse with
// the leading radix-2 butterfly done in the prologue's registers (a thread holds
// bins k and k + 256 of its rows): one shared-memory pass and one CTA barrier
// fewer per direction.
#ifndef SGL_AZ512_FUSE2
#define SGL_AZ512_FUSE2 1
#endif
#ifndef SGL_AZ512_NS2
#define SGL_AZ512_NS2 1
#endif
#ifndef SGL_AZI_EO_PRE
#define SGL_AZI_EO_PRE 1
#endif
#ifndef SGL_AZF_REV
#define SGL_AZF_REV 1
#endif
#ifndef SGL_AZI_REV
#define SGL_AZI_REV 0
#endif
#ifndef SGL_AZI_STORE
#define SGL_AZI_STORE 2
#endif
#ifndef SGL_AZI_LOAD
#define SGL_AZI_LOAD 0
#endif

// ------------------------------------------------------------------ async copy helpers
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NLEFT>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NLEFT)); }
// mbarrier / TMA helpers (shared::cta addresses)
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned a, unsigned bytes) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(a),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_5d(unsigned dst, const void* tmap, unsigned bar, int c0, int c1, int c2,
                                            int c3, int c4) {
#if SGL_L2HINTS
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7], %8;\n" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar), "l"(pol)
        : "memory");
#else
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
        "[%7];\n" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
        : "memory");
#endif
}

// G block of one azimuthal CTA: the CTA's shells are exactly one shell group
// (2^lgib shells, g_layout), so element (p, bin, s0 + sl) of polar node jp sits at
// block + (p * nbins + bin) * 2^lgib + sl -- for the kernels' idx = row * shells + sl
// enumeration simply block[idx] (the general g_index costs ~25 integer
// instructions per element, half of the real inverse kernel's instruction count).
__device__ __forceinline__ long long g_block(const Geo& g, int jp, int s0) {
    return ((((long long)jp * g.ngx + (s0 >> g.lgib)) * 2) * g.nbins) << g.lgib;
}

// ------------------------------------------------------------------ azimuthal forward
// grid.x = ceil(nshell / IG), grid.y = B (j' = polar node in the northern half).
// CTA holds rings (s, j') and (s, 2B-1-j') for IG consecutive flat shells s.
// The first FFT pass loads each ring straight from HBM into registers
// (coalesced: the T threads of a ring read consecutive elements); the result
// lands in shared memory, where the epilogue folds the ring pair into even/odd
// parts, applies b_cal and writes rows of G[p][|m|][j'][sgn][s] (IG shells
// contiguous per row).
// One azimuthal-forward work item: shells [s0, s0 + IG) at polar node pair
// (jp, 2B-1-jp), on `rings` (2 IG padded rings of shared memory).  Called by
// az_forward_kernel (one item per CTA) and by the fused persistent spherical
// forward (sph_fwd_fused_kernel).
template <int N, int ELEMS = SGL_AZ_ELEMS>
__device__ __forceinline__ void az_fwd_item(const Geo& g, const double2* __restrict__ X, size_t fstride,
                                            double2* __restrict__ G, const double* __restrict__ bcal,
                                            const double2* __restrict__ twg, int s0, int jp, double2* rings) {
    using S = FFTShape<N, ELEMS>;
    constexpr int B = N / 2;
    const int tid = threadIdx.x;
    const int nshell = g.batch * g.SC;
    if constexpr (N == 512 && SGL_AZ512_FUSE2) {
        static_assert(N != 512 || (S::T == 32 && S::TWN == 1022), "N = 512 twiddle layout (sgl_tables.cpp)");
        const int q = tid / S::T, tt = tid - q * S::T;
        const int s = s0 + (q >> 1);
        const int j = (q & 1) ? (N - 1 - jp) : jp;
        const double2* src = X;
        const bool ok = s < nshell;
        if (ok) {
            const int f = s / g.SC, i = s - f * g.SC;
            src = X + (size_t)f * fstride + ((size_t)i * N + j) * N;
        }
        double2* ring = rings + q * S::STRIDE;
        auto rd = [&](int x) { return ring[phys(x)]; };
        auto wr = [&](int x, double2 v) { ring[phys(x)] = v; };
        stockham_pass<N, 16, -1, false>(1, tt, twg, [&](int x) { return ok ? ld_stream(src + x) : make_double2(0.0, 0.0); },
                                        wr);
        __syncthreads();
        stockham_pass<N, 16, -1, true>(16, tt, twg + S::TWN, rd, wr);
        __syncthreads();
        // epilogue: final radix-2 butterfly X[k] = y[k] + w^k y[k + 256], X[k + 256] = y[k] - w^k y[k + 256]
        // (linear, so applied to the E/O fold of the ring pair), b_cal, blocked G rows
        const double b = __ldg(bcal + jp);
        double2* const Gblk = G + g_block(g, jp, s0);
#pragma unroll 2
        for (int idx = tid; idx < B * S::IG; idx += S::THREADS) {
            const int sl = idx % S::IG, k = idx / S::IG;
            const int sh = s0 + sl;
            if (sh >= nshell) continue;
            const double2* rj = rings + (2 * sl) * S::STRIDE;
            const double2* rm = rj + S::STRIDE;
            const double2 yj0 = rj[phys(k)], yj1 = rj[phys(k + B)], ym0 = rm[phys(k)], ym1 = rm[phys(k + B)];
            const double2 w = __ldg(twg + k);
            const double2 a0 = cadd(yj0, ym0), a1 = csub(yj0, ym0);
            const double2 b0 = cmul(w, cadd(yj1, ym1)), b1 = cmul(w, csub(yj1, ym1));
            double2* Gb = Gblk + idx;  // (p, bin) row at (p * N + bin) * IG
            Gb[0] = cscale(b, cadd(a0, b0));
            Gb[N * S::IG] = cscale(b, cadd(a1, b1));
            if (k != 0) {  // bin B (Nyquist) is not part of G
                Gb[B * S::IG] = cscale(b, csub(a0, b0));
                Gb[(N + B) * S::IG] = cscale(b, csub(a1, b1));
            }
        }
        return;
    }
    {
        // twiddles come straight from the (L1-resident) per-pass global tables;
        // the ring loads go straight to registers (staging small-N rings through
        // shared memory for longer coalesced runs measured slower: B = 32 7.8 ->
        // 9.3 ms, B = 64 0.81 -> 0.97 ms for the C5 / C2 batches)
        const int q = tid / S::T, tt = tid - q * S::T;
        const int s = s0 + (q >> 1);
        const int j = (q & 1) ? (N - 1 - jp) : jp;
        const double2* src = X;
        const bool ok = s < nshell;
        if (ok) {
            const int f = s / g.SC, i = s - f * g.SC;
            src = X + (size_t)f * fstride + ((size_t)i * N + j) * N;
        }
        double2* ring = rings + q * S::STRIDE;
        const unsigned long long pol = SGL_L2HINTS ? policy_evict_first() : 0ull;
        ring_fft_io<N, -1, false>(
            ring, tt, twg,
            [&](int x) {
                return ok ? (SGL_L2HINTS ? ld_stream_hint(src + x, pol) : ld_stream(src + x)) : make_double2(0.0, 0.0);
            },
            [&](int x, double2 v) { ring[phys(x)] = v; });
    }
    __syncthreads();
    // epilogue: E/O fold, b_cal, scatter rows G[p][|m|][j'][sgn][s]
    // both parities of a (shell, bin) from one pair of ring reads; the shell of
    // idx = tid + it THREADS is a per-thread constant and the CTA's G block is
    // contiguous (g_block): rows p = 0 at block[idx], p = 1 one half block further
    const unsigned long long gpol = SGL_L2HINTS ? policy_evict_last() : 0ull;
    const double b = __ldg(bcal + jp);
    double2* const Gblk = G + g_block(g, jp, s0);
    static_assert(S::THREADS % S::IG == 0 && (N * S::IG) % S::THREADS == 0, "epilogue enumeration");
    const int sl = tid % S::IG;
    if (s0 + sl >= nshell) return;
    const double2* r1 = rings + (2 * sl) * S::STRIDE;
    const double2* r2 = r1 + S::STRIDE;
#pragma unroll 4
    for (int it = 0; it < N * S::IG / S::THREADS; ++it) {
        const int idx = tid + it * S::THREADS;
        const int bin = tid / S::IG + it * (S::THREADS / S::IG);
        if (bin == B) continue;
        const double2 f1 = r1[phys(bin)], f2 = r2[phys(bin)];
        const double2 ve = cscale(b, cadd(f1, f2)), vo = cscale(b, csub(f1, f2));
        if (SGL_L2HINTS) {
            st_hint(Gblk + idx, ve, gpol);
            st_hint(Gblk + idx + N * S::IG, vo, gpol);
        } else {
            Gblk[idx] = ve;
            Gblk[idx + N * S::IG] = vo;
        }
    }
}

template <int N, int ELEMS = SGL_AZ_ELEMS>
__global__ void __launch_bounds__((FFTShape<N, ELEMS>::THREADS), (FFTShape<N, ELEMS>::MINB))
az_forward_kernel(Geo g, const double2* __restrict__ X, size_t fstride, double2* __restrict__ G,
                  const double* __restrict__ bcal, const double2* __restrict__ twg) {
    extern __shared__ double2 smem[];
    const int bx = (SGL_AZF_REV ? gridDim.x - 1 - blockIdx.x : blockIdx.x) + g.gx0;
    const int by = (SGL_AZF_REV ? gridDim.y - 1 - blockIdx.y : blockIdx.y) + g.jp0;
    az_fwd_item<N, ELEMS>(g, X, fstride, G, bcal, twg, bx * FFTShape<N, ELEMS>::IG, by, smem);
}

// ------------------------------------------------------------------ azimuthal inverse
// Prologue: cp.async E (p = 0) rows into the ring-j' buffer and O (p = 1) rows
// into the ring-(2B-1-j') buffer.  The first FFT pass reads E +- O straight
// from both buffers (Nyquist bin B zero); the last pass writes the psi-order
// samples straight to HBM (coalesced).
template <int N, int ELEMS = SGL_AZI_ELEMS>
__global__ void __launch_bounds__((FFTShape<N, ELEMS>::THREADS), (FFTShape<N, ELEMS>::MINB))
az_inverse_kernel(Geo g, const double2* __restrict__ G, double2* __restrict__ X, size_t fstride,
                  const double2* __restrict__ twg) {
    using S = FFTShape<N, ELEMS>;
    constexpr int B = N / 2;
    extern __shared__ double2 smem[];
    // the plain twiddle table staged in shared memory under the prologue barrier
    // (measured: 118 us; the forward kernel's per-pass tables from global 120 us,
    // per-pass tables in shared memory 125 us)
    double2* rings = smem;  // twiddles: per-pass tables from global (93 us; a shared-memory copy 104 us)
    const int tid = threadIdx.x;
    const int jp = (SGL_AZI_REV ? gridDim.y - 1 - blockIdx.y : blockIdx.y) + g.jp0;
    const int s0 = ((SGL_AZI_REV ? gridDim.x - 1 - blockIdx.x : blockIdx.x) + g.gx0) * S::IG;
    const int nshell = g.batch * g.SC;
    // prologue: all of this thread's G loads in flight before the first shared
    // store (a partially unrolled load -> store loop kept only 4 in flight)
    constexpr int PER = 2 * N * S::IG / S::THREADS;
    static_assert(PER * S::THREADS == 2 * N * S::IG, "prologue must divide evenly");
    double2 pv[PER];
    // idx = tid + q THREADS enumerates the CTA's contiguous G block [p][bin][shell]
    // (g_block): the shell is a per-thread constant, the address an immediate offset
    static_assert(S::THREADS % S::IG == 0 && (N & (N - 1)) == 0, "shell of a prologue load is per-thread");
    const bool sok = s0 + tid % S::IG < nshell;
    const double2* Gb = G + g_block(g, jp, s0) + tid;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int bin = (tid / S::IG + q * (S::THREADS / S::IG)) & (N - 1);
#ifdef SGL_G_WRAP
        pv[q] = (bin != B && sok) ? ld_stream(G + (g_block(g, jp, s0) + tid + q * S::THREADS) % (SGL_G_WRAP * 65536LL))
                                  : make_double2(0.0, 0.0);
#else
        pv[q] = (bin != B && sok)
                    ? ((SGL_L2HINTS || SGL_AZI_LOAD) ? ld_stream_hint(Gb + q * S::THREADS, policy_evict_first())
                                                     : ld_stream(Gb + q * S::THREADS))
                    : make_double2(0.0, 0.0);
#endif
    }
    // ring values in the prologue's registers: a thread's loads q and q + PER / 2
    // are E (p = 0) and O (p = 1) of the same (shell, bin), so ring j' = E + O and
    // its mirror 2B-1-j' = E - O are formed here and every FFT pass reads its own
    // ring only (SGL_AZI_EO_PRE, N >= 256: az_inverse 92.3 -> 89.8 us at B = 128,
    // 914 -> 862 us at B = 256; at N <= 128 the two-ring stores conflict in shared
    // memory -- B = 64 x 64: 733 -> 750 us -- so there the first pass still reads
    // both parity buffers)
    constexpr int HP = PER / 2;
    static_assert(HP * S::THREADS == N * S::IG, "parity partner of load q is load q + PER / 2");
    const int fq = tid / S::T, tt = tid - fq * S::T;  // FFT role: ring fq of the CTA, thread tt of the ring
    const int fs = s0 + (fq >> 1);
    const bool ok = fs < nshell;
    double2* dst = X;
    if (ok) {
        const int f = fs / g.SC, i = fs - f * g.SC;
        const int j = (fq & 1) ? (N - 1 - jp) : jp;
        dst = X + (size_t)f * fstride + ((size_t)i * N + j) * N;
    }
    double2* ring = rings + fq * S::STRIDE;
    auto st_out = [&](int x, double2 v) {
        if (!ok) return;
        if (SGL_AZI_STORE == 0) __stcs(dst + x, v);
        else if (SGL_AZI_STORE == 1) dst[x] = v;
        else st_hint(dst + x, v, policy_evict_last());
    };
    if constexpr (N == 512 && SGL_AZ512_FUSE2) {
        // ... and the leading radix-2 butterfly of the (2, 16, 16) FFT: loads q and
        // q + HQ are bins k and k + 256 of the same row
        constexpr int HQ = (B * S::IG) / S::THREADS;
        static_assert(HQ * S::THREADS == B * S::IG && PER == 4 * HQ, "prologue pairing");
#pragma unroll
        for (int q = 0; q < HQ; ++q) {
            const int idx = tid + q * S::THREADS;
            const int sl = idx % S::IG, k = idx / S::IG;  // k < B
            const double2 xj0 = cadd(pv[q], pv[q + HP]), xm0 = csub(pv[q], pv[q + HP]);
            const double2 xj1 = cadd(pv[q + HQ], pv[q + HQ + HP]), xm1 = csub(pv[q + HQ], pv[q + HQ + HP]);
            double2* rj = rings + (2 * sl) * S::STRIDE;
            double2* rm = rj + S::STRIDE;
            // ring pairs sit 32 bytes apart (mod 128): odd shells store the odd
            // element first so that a warp's 16-byte stores cover all banks
            const int odd = sl & 1;
            const double2 sj = cadd(xj0, xj1), dj = csub(xj0, xj1), sm = cadd(xm0, xm1), dm = csub(xm0, xm1);
            rj[phys(2 * k + odd)] = odd ? dj : sj;
            rj[phys(2 * k + 1 - odd)] = odd ? sj : dj;
            rm[phys(2 * k + odd)] = odd ? dm : sm;
            rm[phys(2 * k + 1 - odd)] = odd ? sm : dm;
        }
        __syncthreads();
        auto rd_ring = [&](int x) { return ring[phys(x)]; };
        auto wr_ring = [&](int x, double2 v) { ring[phys(x)] = v; };
        stockham_pass<N, 16, +1, true, decltype(rd_ring)&, decltype(wr_ring)&, NoPairLoad, SGL_AZ512_NS2 != 0>(
            2, tt, twg + N, rd_ring, wr_ring);
        __syncthreads();
        stockham_pass<N, 16, +1, false>(32, tt, twg + N + 15 * 2, rd_ring, st_out);
        return;
    }
    if constexpr (SGL_AZI_EO_PRE && N >= 256) {
#pragma unroll
    for (int q = 0; q < HP; ++q) {
        const int idx = tid + q * S::THREADS;
        const int sl = idx % S::IG, bin = idx / S::IG;
        rings[(2 * sl) * S::STRIDE + phys(bin)] = cadd(pv[q], pv[q + HP]);
        rings[(2 * sl + 1) * S::STRIDE + phys(bin)] = csub(pv[q], pv[q + HP]);
    }
    __syncthreads();
    ring_fft_io<N, +1, true>(ring, tt, twg, [&](int x) { return ring[phys(x)]; }, st_out);
    return;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int idx = tid + q * S::THREADS;
        const int sl = idx % S::IG;
        const int rowi = idx / S::IG;
        const int p = rowi / N, bin = rowi - p * N;
        rings[(2 * sl + p) * S::STRIDE + phys(bin)] = pv[q];
    }
    __syncthreads();
    {
        const bool mirror = fq & 1;
        const double2* e_buf = rings + (fq & ~1) * S::STRIDE;
        const double2* o_buf = e_buf + S::STRIDE;
        ring_fft_io<N, +1, true>(
            ring, tt, twg,
            [&](int x) {
                const double2 e = e_buf[phys(x)], o = o_buf[phys(x)];
                return mirror ? csub(e, o) : cadd(e, o);
            },
            st_out);
    }
}

// 256-bit global accesses (sm_100a: LDG / STG .ENL2.256) and a 4 x 4 transpose of
// doubles across the 4 lanes of a ring (N = 64: T = 4), for the real-valued
// kernels at B = 32 (config C5), whose 8-byte samples otherwise move 32 bytes per
// ring and instruction.
__device__ __forceinline__ void ld_v4_cs(const double* p, double (&v)[4]) {
    asm volatile("ld.global.cs.v4.f64 {%0, %1, %2, %3}, [%4];\n" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void st_v4_cs(double* p, const double (&v)[4]) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
}
// in: lane t of an aligned 4-lane group holds M[t][b] in m[b]; out: m[b] = M[b][t]
__device__ __forceinline__ void transpose4_lanes(double (&m)[4], int t) {
    {
        const bool hi = t & 1;
        double s0 = hi ? m[0] : m[1], s1 = hi ? m[2] : m[3];
        s0 = __shfl_xor_sync(0xffffffffu, s0, 1);
        s1 = __shfl_xor_sync(0xffffffffu, s1, 1);
        if (hi) { m[0] = s0; m[2] = s1; } else { m[1] = s0; m[3] = s1; }
    }
    {
        const bool hi = t & 2;
        double s0 = hi ? m[0] : m[2], s1 = hi ? m[1] : m[3];
        s0 = __shfl_xor_sync(0xffffffffu, s0, 2);
        s1 = __shfl_xor_sync(0xffffffffu, s1, 2);
        if (hi) { m[0] = s0; m[1] = s1; } else { m[2] = s0; m[3] = s1; }
    }
}
#ifndef SGL_AZR_V4
#define SGL_AZR_V4 1
#endif
// Ring of FFT role q (4 threads per ring, N = 64): shared memory serves 16-byte
// accesses a quarter-warp at a time, i.e. two rings' threads together, and rings
// one padded stride apart (69 = 5 mod 8 slots of 16 bytes) overlap in one slot --
// every FFT-pass LDS / STS ran at 2x its ideal wavefronts (ncu, round 2).  Roles
// 2a and 2a + 1 take rings 4 apart instead (20 = 4 mod 8 slots: disjoint halves of
// the 128-byte line); the prologue / epilogue, whose lanes run over consecutive
// rings, are unaffected.
#ifndef SGL_AZR_RINGPERM
#define SGL_AZR_RINGPERM 1
#endif
template <int T>
__device__ __forceinline__ int ring_of_role(int q) {
    if constexpr (T == 4 && SGL_AZR_RINGPERM) {
        const int a = q >> 1;
        return ((a >> 2) << 3) + (a & 3) + 4 * (q & 1);
    } else {
        return q;
    }
}

// ------------------------------------------------------------------ real-valued azimuthal stage
// Real samples: the rings j' and 2B-1-j' of a shell are packed into one complex
// ring z = x1 + i x2 and transformed with ONE complex FFT; with Z = FFT(z),
//   X1[m] = (Z[m] + conj Z[-m]) / 2,   X2[m] = (Z[m] - conj Z[-m]) / (2i),
// and for real data only m >= 0 is needed (G[-m] = conj G[m]).  Half the bytes
// in (8 B per sample) and half the FFTs of the complex path.  CTA: 2*IG shells,
// one packed ring each (same thread count and shared memory as the complex path).
template <int N, bool V4 = false>
__global__ void __launch_bounds__(FFTShape<N>::THREADS, FFTShape<N>::MINB)
az_forward_real_kernel(Geo g, const double* __restrict__ X, size_t fstride, double2* __restrict__ G,
                       const double* __restrict__ bcal, const double2* __restrict__ twg) {
    using S = FFTShape<N>;
    constexpr int B = N / 2;
    constexpr int IGR = 2 * S::IG;
    extern __shared__ double2 smem[];
    double2* rings = smem;  // twiddles: per-pass tables from global (as in az_forward_kernel)
    const int tid = threadIdx.x;
    const int jp = blockIdx.y;
    const int s0 = blockIdx.x * IGR;
    const int nshell = g.batch * g.SC;
    {
        const int tt = tid % S::T;
        const int q = ring_of_role<S::T>(tid / S::T);
        const int s = s0 + q;
        const double* src1 = X;
        const double* src2 = X;
        const bool ok = s < nshell;
        if (ok) {
            const int f = s / g.SC, i = s - f * g.SC;
            src1 = X + f * fstride + ((size_t)i * N + jp) * N;
            src2 = X + f * fstride + ((size_t)i * N + (N - 1 - jp)) * N;
        }
        double2* ring = rings + q * S::STRIDE;
        // first-pass inputs in pairs of consecutive samples: 16-byte loads of both rings
        auto ld2 = [&](int x, double2& z0, double2& z1) {
            if (ok) {
                const double2 a = __ldcs(reinterpret_cast<const double2*>(src1 + x));
                const double2 b = __ldcs(reinterpret_cast<const double2*>(src2 + x));
                z0 = make_double2(a.x, b.x);
                z1 = make_double2(a.y, b.y);
            } else {
                z0 = z1 = make_double2(0.0, 0.0);
            }
        };
        if constexpr (V4) {
            // head pass (radix 4, thread tt runs butterflies 4 tt .. 4 tt + 3) on 32-byte
            // loads: 4 consecutive samples of both rings per radix input
            static_assert(S::T == 4 && S::R0 == 4 && N == 64, "N = 64: radix 4 then radix 16, 4 threads per ring");
            double2 v[4][4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                double a[4] = {0.0, 0.0, 0.0, 0.0}, c[4] = {0.0, 0.0, 0.0, 0.0};
                if (ok) {
                    ld_v4_cs(src1 + 4 * tt + 16 * r, a);
                    ld_v4_cs(src2 + 4 * tt + 16 * r, c);
                }
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) v[bb][r] = make_double2(a[bb], c[bb]);
            }
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                dft_reg<4, -1>(v[bb]);
#pragma unroll
                for (int r = 0; r < 4; ++r) ring[phys((4 * tt + bb) * 4 + r)] = v[bb][r];
            }
            pair_sync<N>();
            stockham_pass<N, 16, -1, true>(4, tt, twg + N, [&](int x) { return ring[phys(x)]; },
                                           [&](int x, double2 w) { ring[phys(x)] = w; });
        } else {
        ring_fft_io<N, -1, false>(
            ring, tt, twg, [&](int x) { return ok ? make_double2(__ldcs(src1 + x), __ldcs(src2 + x)) : make_double2(0.0, 0.0); },
            [&](int x, double2 v) { ring[phys(x)] = v; }, ld2);
        }
    }
    __syncthreads();
    const double b = __ldg(bcal + jp);
    double2* const Gblk = G + g_block(g, jp, s0);
    // one (shell, m) per iteration: both parities from the same Z[m], Z[-m]
#pragma unroll 4
    for (int idx = tid; idx < B * IGR; idx += S::THREADS) {
        const int sl = idx % IGR;
        const int m = idx / IGR;
        const int s = s0 + sl;
        if (s >= nshell) continue;
        const double2 zm = rings[sl * S::STRIDE + phys(m)];
        const double2 zn = rings[sl * S::STRIDE + phys((N - m) & (N - 1))];
        const double2 x1 = make_double2(0.5 * (zm.x + zn.x), 0.5 * (zm.y - zn.y));
        const double2 x2 = make_double2(0.5 * (zm.y + zn.y), -0.5 * (zm.x - zn.x));
        double2* Gb = Gblk + idx;
        Gb[0] = cscale(b, cadd(x1, x2));
        Gb[B * IGR] = cscale(b, csub(x1, x2));
    }
}

#ifndef SGL_AZR_REGSTAGE
#define SGL_AZR_REGSTAGE 1
#endif
#ifndef SGL_AZR_ZPRE
#define SGL_AZR_ZPRE 1
#endif
#ifndef SGL_AZRI_MINB64
#define SGL_AZRI_MINB64 4  // CTAs/SM of the real inverse at N = 64
#endif
template <int N, bool V4 = false>
__global__ void __launch_bounds__(FFTShape<N>::THREADS, (N == 64 ? SGL_AZRI_MINB64 : FFTShape<N>::MINB))
az_inverse_real_kernel(Geo g, const double2* __restrict__ G, double* __restrict__ X, size_t fstride,
                       const double2* __restrict__ twg) {
    using S = FFTShape<N>;
    constexpr int B = N / 2;
    constexpr int IGR = 2 * S::IG;
    constexpr int EOS = S::STRIDE;  // per shell: E[0..B) then O[0..B), in the shell's own ring buffer
    extern __shared__ double2 smem[];
    double2* rings = smem;  // twiddles: per-pass tables from global
    // E/O rows share the ring buffers (the first FFT pass reads all its inputs
    // before its pair-synchronized writes), halving the CTA's shared memory
    double2* eo = rings;
    const int tid = threadIdx.x;
    const int jp = blockIdx.y;
    const int s0 = blockIdx.x * IGR;
    const int nshell = g.batch * g.SC;
#if SGL_AZR_REGSTAGE
    // all of this thread's G loads in flight before the first shared store (as in
    // az_inverse_kernel); the cp.async form ran its shared-memory side at 8x the
    // ideal wavefronts (ncu, round 2)
    constexpr int PER = 2 * B * IGR / S::THREADS;
    static_assert(PER * S::THREADS == 2 * B * IGR, "prologue must divide evenly");
    double2 pv[PER];
    // idx = tid + q THREADS enumerates the CTA's contiguous G block [p][m][shell]
    // (g_block): the shell (idx % IGR) is a per-thread constant, the address an
    // immediate offset from one pointer
    static_assert(S::THREADS % IGR == 0, "shell of a prologue load is per-thread");
    const bool sok = s0 + tid % IGR < nshell;
    const double2* Gb = G + g_block(g, jp, s0) + tid;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
#ifdef SGL_AZR_DBG_NOLD  // timing-only (wrong results): no G loads
        pv[q] = make_double2((double)(tid + q), (double)(q - tid));
#else
        pv[q] = sok ? ld_stream(Gb + q * S::THREADS) : make_double2(0.0, 0.0);
#endif
    }
#if SGL_AZR_ZPRE
    // the thread holds E (q) and O (q + PER / 2) of the same (shell, m): form the
    // packed FFT input here, Z[m] = X1 + i X2 and Z[N - m] = conj X1 + i conj X2
    // (X1 = E + O, X2 = E - O; Z[B] = 0), written in natural order so that the
    // first FFT pass reads the ring like the complex path
    static_assert(PER % 2 == 0, "E and O of one bin in one thread");
#pragma unroll
    double2* const zring = eo + (tid % IGR) * EOS;
    for (int q = 0; q < PER / 2; ++q) {
        const int m = tid / IGR + q * (S::THREADS / IGR);  // row < B: p = 0
        const double2 e = pv[q], o = pv[q + PER / 2];
        const double2 x1 = cadd(e, o), x2 = csub(e, o);
        double2* ring = zring;
        if (m == 0) {
            ring[phys(0)] = make_double2(x1.x, x2.x);
            ring[phys(B)] = make_double2(0.0, 0.0);
        } else {
            ring[phys(m)] = make_double2(x1.x - x2.y, x1.y + x2.x);
            ring[phys(N - m)] = make_double2(x1.x + x2.y, x2.x - x1.y);
        }
    }
#else
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int idx = tid + q * S::THREADS;
        const int sl = idx % IGR;
        const int rowi = idx / IGR;
        eo[sl * EOS + rowi] = pv[q];
    }
#endif
#else
#pragma unroll 4
    for (int idx = tid; idx < 2 * B * IGR; idx += S::THREADS) {
        const int sl = idx % IGR;
        const int rowi = idx / IGR;  // p * B + m
        const int p = rowi / B, m = rowi - p * B;
        const int s = s0 + sl;
        double2* dst = eo + sl * EOS + p * B + m;
        if (s < nshell) {
            cp_async16(dst, G + g_index(g, p, m, jp, s));
        } else {
            *dst = make_double2(0.0, 0.0);
        }
    }
    cp_async_wait_all();
#endif
    __syncthreads();
    {
        const int tt = tid % S::T;
        const int q = ring_of_role<S::T>(tid / S::T);
        const int s = s0 + q;
        const double2* e_buf = eo + q * EOS;
        double* dst1 = X;
        double* dst2 = X;
        const bool ok = s < nshell;
        if (ok) {
            const int f = s / g.SC, i = s - f * g.SC;
            dst1 = X + f * fstride + ((size_t)i * N + jp) * N;
            dst2 = X + f * fstride + ((size_t)i * N + (N - 1 - jp)) * N;
#ifdef SGL_AZR_DBG_CONTIG  // timing-only (wrong results): each CTA writes one contiguous block
            dst1 = X + (((size_t)blockIdx.y * gridDim.x + blockIdx.x) * IGR * 2 + 2 * q) * N;
            dst2 = dst1 + N;
#endif
        }
        double2* ring = rings + q * S::STRIDE;
        auto in = [&](int bin) {
            if (SGL_AZR_REGSTAGE && SGL_AZR_ZPRE) return e_buf[phys(bin)];  // formed in the prologue
            if (bin == B) return make_double2(0.0, 0.0);
            const int m = bin < B ? bin : N - bin;
            const double2 e = e_buf[m], o = e_buf[B + m];
            const double2 x1 = cadd(e, o), x2 = csub(e, o);
            if (bin == 0) return make_double2(x1.x, x2.x);
            if (bin < B) return make_double2(x1.x - x2.y, x1.y + x2.x);  // X1 + i X2
            return make_double2(x1.x + x2.y, x2.x - x1.y);                // conj X1 + i conj X2
        };
        if constexpr (V4) {
            // radices (16, 4) instead of the generic (4, 16): the last pass's thread tt runs
            // the radix-4 butterflies j = 4 tt .. 4 tt + 3, whose outputs j + 16 r are 4
            // consecutive samples per r -- 32-byte stores per ring, no transposition.
            // Pass 1 (radix 16, thread tt = butterfly tt): element y[16 u + 4 v + b] is
            // parked at 16 b + 4 u + ((u + v) & 3), which keeps both its writes (4 threads
            // u) and pass 2's reads (4 threads v) on 4 distinct 16-byte slots of one half
            // of the 128-byte line; the quarter-warp's other ring sits on the other half.
            double2 v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = in(tt + 4 * r);
            dft_reg<16, +1>(v);
            pair_sync<N>();  // every read of the natural-order ring before the in-place writes
#pragma unroll
            for (int r = 0; r < 16; ++r) ring[16 * (r & 3) + 4 * tt + ((tt + (r >> 2)) & 3)] = v[r];
            pair_sync<N>();
            double2 u4[4][4];
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
#pragma unroll
                for (int r = 0; r < 4; ++r) u4[bb][r] = ring[16 * bb + 4 * r + ((r + tt) & 3)];
#pragma unroll
                for (int r = 1; r < 4; ++r) {
                    double2 w = twg[r * (4 * tt + bb)];  // e^{-2 pi i r k / 64}, k = 4 tt + bb
                    w.y = -w.y;
                    u4[bb][r] = cmul(u4[bb][r], w);
                }
                dft_reg<4, +1>(u4[bb]);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double m1[4] = {u4[0][r].x, u4[1][r].x, u4[2][r].x, u4[3][r].x};
                const double m2[4] = {u4[0][r].y, u4[1][r].y, u4[2][r].y, u4[3][r].y};
#ifdef SGL_AZR_DBG_NOST  // timing-only (wrong results): stores only if a value is NaN
                if (ok && m1[0] != m1[0]) {
#else
                if (ok) {
#endif
                    st_v4_cs(dst1 + 16 * r + 4 * tt, m1);
                    st_v4_cs(dst2 + 16 * r + 4 * tt, m2);
                }
            }
        } else {
        ring_fft_io<N, +1, true>(ring, tt, twg, in, [&](int x, double2 v) {
            if (ok) {
                __stcs(dst1 + x, v.x);
                __stcs(dst2 + x, v.y);
            }
        });
        }
    }
}

template <int N>
static int az_fwd_real_launch(const Geo& g, const double* X, size_t fstride, double* G, const double* bcal,
                              const double* tw, cudaStream_t s) {
    using S = FFTShape<N>;
    constexpr int IGR = 2 * S::IG;
    const size_t smem = sizeof(double2) * (IGR * S::STRIDE);
    const int nshell = g.batch * g.SC;
    dim3 grid((nshell + IGR - 1) / IGR, g.B);
    if constexpr (N == 64 && SGL_AZR_V4) {
        // 32-byte sample accesses need 32-byte aligned rings (any cudaMalloc / torch buffer)
        if (reinterpret_cast<uintptr_t>(X) % 32 == 0 && fstride % 4 == 0) {
            static SmemAttrOnce attr4;
            attr4.ensure(az_forward_real_kernel<N, true>, smem);
            az_forward_real_kernel<N, true><<<grid, S::THREADS, smem, s>>>(g, X, fstride, reinterpret_cast<double2*>(G),
                                                                          bcal, reinterpret_cast<const double2*>(tw));
            return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
        }
    }
    static SmemAttrOnce attr;
    attr.ensure(az_forward_real_kernel<N>, smem);
    az_forward_real_kernel<N><<<grid, S::THREADS, smem, s>>>(g, X, fstride, reinterpret_cast<double2*>(G), bcal,
                                                              reinterpret_cast<const double2*>(tw));
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <int N>
static int az_inv_real_launch(const Geo& g, const double* G, double* X, size_t fstride, const double* tw,
                              cudaStream_t s) {
    using S = FFTShape<N>;
    constexpr int IGR = 2 * S::IG;
    const size_t smem = sizeof(double2) * (IGR * S::STRIDE);  // E/O rows live in the ring buffers
    const int nshell = g.batch * g.SC;
    dim3 grid((nshell + IGR - 1) / IGR, g.B);
    if constexpr (N == 64 && SGL_AZR_V4) {
        if (reinterpret_cast<uintptr_t>(X) % 32 == 0 && fstride % 4 == 0) {
            static SmemAttrOnce attr4;
            attr4.ensure(az_inverse_real_kernel<N, true>, smem);
            az_inverse_real_kernel<N, true><<<grid, S::THREADS, smem, s>>>(g, reinterpret_cast<const double2*>(G), X,
                                                                          fstride, reinterpret_cast<const double2*>(tw));
            return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
        }
    }
    static SmemAttrOnce attr;
    attr.ensure(az_inverse_real_kernel<N>, smem);
    az_inverse_real_kernel<N><<<grid, S::THREADS, smem, s>>>(g, reinterpret_cast<const double2*>(G), X, fstride,
                                                              reinterpret_cast<const double2*>(tw));
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// sample_stride: doubles per function (8B^3 for real samples)
int launch_az_forward_real(const Geo& g, const double* samples, size_t sample_stride, double* G,
                           const double* bcal, const double* twiddle, cudaStream_t s) {
    switch (2 * g.B) {
        case 4: return az_fwd_real_launch<4>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 8: return az_fwd_real_launch<8>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 16: return az_fwd_real_launch<16>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 32: return az_fwd_real_launch<32>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 64: return az_fwd_real_launch<64>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 128: return az_fwd_real_launch<128>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 256: return az_fwd_real_launch<256>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 512: return az_fwd_real_launch<512>(g, samples, sample_stride, G, bcal, twiddle, s);
        default: return -2;  // real fast path needs a power-of-two 2B >= 4
    }
}

int launch_az_inverse_real(const Geo& g, const double* G, double* samples, size_t sample_stride,
                           const double* twiddle, cudaStream_t s) {
    switch (2 * g.B) {
        case 4: return az_inv_real_launch<4>(g, G, samples, sample_stride, twiddle, s);
        case 8: return az_inv_real_launch<8>(g, G, samples, sample_stride, twiddle, s);
        case 16: return az_inv_real_launch<16>(g, G, samples, sample_stride, twiddle, s);
        case 32: return az_inv_real_launch<32>(g, G, samples, sample_stride, twiddle, s);
        case 64: return az_inv_real_launch<64>(g, G, samples, sample_stride, twiddle, s);
        case 128: return az_inv_real_launch<128>(g, G, samples, sample_stride, twiddle, s);
        case 256: return az_inv_real_launch<256>(g, G, samples, sample_stride, twiddle, s);
        case 512: return az_inv_real_launch<512>(g, G, samples, sample_stride, twiddle, s);
        default: return -2;
    }
}

// ------------------------------------------------------------------ naive azimuthal (non-pow2 2B)
// Direct DFT per ring for bandlimits whose 2B is not a power of two (the
// reference's naive fallback, kernels.cpp:35-45).  One CTA per (shell, j').
__global__ void az_forward_naive_kernel(Geo g, const double2* __restrict__ X, size_t fstride,
                                        double2* __restrict__ G, const double* __restrict__ bcal,
                                        const double2* __restrict__ twg) {
    extern __shared__ double2 smem[];
    const int B = g.B, N = 2 * B;
    const int jp = blockIdx.y, s = blockIdx.x;
    const int f = s / g.SC, i = s - f * g.SC;
    double2* r1 = smem;
    double2* r2 = smem + N;
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
        r1[e] = X[(size_t)f * fstride + ((size_t)i * N + jp) * N + e];
        r2[e] = X[(size_t)f * fstride + ((size_t)i * N + (N - 1 - jp)) * N + e];
    }
    __syncthreads();
    for (int bin = threadIdx.x; bin < N; bin += blockDim.x) {
        if (bin == B) continue;
        double2 a1 = make_double2(0, 0), a2 = make_double2(0, 0);
        for (int k = 0; k < N; ++k) {
            const double2 w = twg[(int)(((long long)bin * k) % N)];
            a1 = cadd(a1, cmul(r1[k], w));
            a2 = cadd(a2, cmul(r2[k], w));
        }
        for (int p = 0; p < 2; ++p) {
            const double2 v = p ? csub(a1, a2) : cadd(a1, a2);
            G[g_index(g, p, bin, jp, s)] = cscale(bcal[jp], v);
        }
    }
}

__global__ void az_inverse_naive_kernel(Geo g, const double2* __restrict__ G, double2* __restrict__ X,
                                        size_t fstride, const double2* __restrict__ twg) {
    extern __shared__ double2 smem[];
    const int B = g.B, N = 2 * B;
    const int jp = blockIdx.y, s = blockIdx.x;
    const int f = s / g.SC, i = s - f * g.SC;
    double2* r1 = smem;
    double2* r2 = smem + N;
    for (int bin = threadIdx.x; bin < N; bin += blockDim.x) {
        double2 e = make_double2(0, 0), o = make_double2(0, 0);
        if (bin != B) {
            e = G[g_index(g, 0, bin, jp, s)];
            o = G[g_index(g, 1, bin, jp, s)];
        }
        r1[bin] = cadd(e, o);
        r2[bin] = csub(e, o);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double2 a1 = make_double2(0, 0), a2 = make_double2(0, 0);
        for (int bin = 0; bin < N; ++bin) {
            double2 w = twg[(int)(((long long)bin * k) % N)];
            w.y = -w.y;
            a1 = cadd(a1, cmul(r1[bin], w));
            a2 = cadd(a2, cmul(r2[bin], w));
        }
        X[(size_t)f * fstride + ((size_t)i * N + jp) * N + k] = a1;
        X[(size_t)f * fstride + ((size_t)i * N + (N - 1 - jp)) * N + k] = a2;
    }
}

// ------------------------------------------------------------------ grouped DMMA GEMM
// C[row][col] = sum_k A[row][k] * Bm[k][col], addresses separable:
//   A:  A + rowA(row) + colA(k)        Bm: Bm + rowB(k) + colB(col)
//   C:  C + rowC(row) + colC(col), value negated where negC(col)
// cols come in (re, im) pairs that are adjacent in memory for Bm and C.
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

#ifndef SGL_MINB_RADINV
#define SGL_MINB_RADINV 0
#endif
#ifndef SGL_ST_RADINV
#define SGL_ST_RADINV 0
#endif
#ifndef SGL_BK_RADINV
#define SGL_BK_RADINV 0
#endif
#ifndef SGL_MINB_RADFWD
#define SGL_MINB_RADFWD 0
#endif
#ifndef SGL_ST_RADFWD
#define SGL_ST_RADFWD 0
#endif
#ifndef SGL_BK_RADFWD
#define SGL_BK_RADFWD 0
#endif
#ifndef SGL_MINB_LEGINV
#define SGL_MINB_LEGINV 0
#endif
#ifndef SGL_ST_LEGINV
#define SGL_ST_LEGINV 0
#endif
#ifndef SGL_BK_LEGINV
#define SGL_BK_LEGINV 0
#endif
#ifndef SGL_MINB_LEGFWD
#define SGL_MINB_LEGFWD 0
#endif
#ifndef SGL_ST_LEGFWD
#define SGL_ST_LEGFWD 0
#endif
#ifndef SGL_BK_LEGFWD
#define SGL_BK_LEGFWD 0
#endif
#ifndef SGL_ISSUE_LEGFWD
#define SGL_ISSUE_LEGFWD -1
#endif
#ifndef SGL_ISSUE_LEGINV
#define SGL_ISSUE_LEGINV -1
#endif
#ifndef SGL_ISSUE_RADFWD
#define SGL_ISSUE_RADFWD -1
#endif
#ifndef SGL_ISSUE_RADINV
#define SGL_ISSUE_RADINV -1
#endif
// Per-kind pipeline shape: k-chunk (BK), cp.async stages (ST), CTAs per SM
// (__launch_bounds__), where the next chunk's loads are issued (GEMM_ISSUE:
// measured at B = 128 -- after the MMAs: legendre_inverse 110 -> 108.7 us,
// radial_forward 53.1 -> 51.2 us; before them: radial_inverse 45.9 vs 50.6 us).
// Measured at B = 128 (exp/stage_times.py): BK 8 with 3 stages keeps more bytes in flight per CTA than BK 16 with 2 at the same
// shared-memory footprint (4 CTAs / SM): 585 -> 565 us per round trip; LegInv
// and LegFwd (ring sized for wm <= 2) run 4 stages (-1 us, -3.6 us).
#define SGL_KIND_CFG(NAME, DBK, DST, DMINB, DISSUE)          \
    static constexpr int GEMM_ISSUE = SGL_ISSUE_##NAME >= 0 ? SGL_ISSUE_##NAME : DISSUE; \
    static constexpr int GEMM_BK = SGL_BK_##NAME > 0 ? SGL_BK_##NAME : DBK; \
    static constexpr int GEMM_ST = SGL_ST_##NAME > 0 ? SGL_ST_##NAME : DST; \
    static constexpr int GEMM_MINB = SGL_MINB_##NAME > 0 ? SGL_MINB_##NAME : DMINB; \
    static constexpr int GEMM_MAXWM = SGL_MAXWM_##NAME; \
    static constexpr bool GEMM_SEQ = false;

// --- problem kinds
// Legendre forward: prob = 2|m| + p.  rows l = |m|+p+2r, K = B (j'), cols n' = sgn*NB + n.
// Column n of a Legendre problem is (sgn, f, i_local, c) over the G chunk
// (g.SC shells per function); it lands in S at (nu, f, sv.i0 + i_local, c)
// of an S with sv.sc shells per function and sv.NB reals per nu row.
struct LegFwd {
    SGL_KIND_CFG(LEGFWD, 8, 4, 4, 0)
    Geo g;
    const double* A;        // table
    const long long* aoff;  // per prob
    const double* Bm;       // G
    double* C;              // S
    SView sv;
    static constexpr bool A_KCONTIG = true;
    static constexpr bool B_KCONTIG = false;
    static constexpr int B_ROW_TABLE = 0;  // rowB affine in k: pointer increments
    __device__ int am(int pid) const { return pid >> 1; }
    __device__ int M(int pid) const { const int r = g.B - am(pid) - (pid & 1); return r > 0 ? (r + 1) / 2 : 0; }
    __device__ int N(int pid) const { return am(pid) == 0 || g.real ? (int)g.NB : 2 * (int)g.NB; }
    __device__ int K(int) const { return g.B; }
    static constexpr bool B_COL_AFFINE = false;  // blocked G: per-column offsets
    // end (exclusive) of the sign half that column n0 lies in
    __device__ int nlim(int pid, int n0) const { return n0 < g.NB ? (int)g.NB : N(pid); }
    __device__ long long rowA(int pid, int r) const { return leg_table_off(g.B, pid) + r * lstride(); }
    __device__ long long colA(int, int k) const { return k; }
    __device__ int a_sr(int) const { return lstride(); }
    __device__ int a_sk(int) const { return 1; }
    __device__ int lstride() const { return g.B + (g.B & 1); }  // legendre_stride (sgl_tables.hpp)
    __device__ long long rowB(int, int k) const { return k * g_rowstride(g); }
    __device__ long long b_kstep(int) const { return g_rowstride(g); }
    __device__ long long colB(int pid, int n) const { return g_col(g, pid & 1, am(pid), n); }
    __device__ long long rowC(int pid, int r) const {
        const int l = am(pid) + (pid & 1) + 2 * r;
        return l * (l + 1) * (int)sv.NB;
    }
    __device__ long long colC(int pid, int n) const { return s_col(g, sv, am(pid), n); }
    __device__ bool negC(int pid, int n) const { return n >= g.NB && (am(pid) & 1); }
    // tiles start at multiples of bn inside a sign half; no function boundary inside
    // the tile when bn divides the per-function width 2 SC
    __device__ bool c_affine(int, int, int bn) const { return (2 * g.SC) % bn == 0; }
};

// Legendre inverse: prob = 2|m| + p.  rows j' (M = B), K = #l of parity p, cols n'.
struct LegInv {
    SGL_KIND_CFG(LEGINV, 8, 4, 4, 2)
    Geo g;
    const double* A;
    const long long* aoff;
    const double* Bm;  // S
    double* C;         // G
    SView sv;
    static constexpr bool A_KCONTIG = false;
    static constexpr bool B_KCONTIG = false;
    static constexpr int B_ROW_TABLE = 128;  // K <= (B + 1) / 2 rows, B <= 256
    __device__ int am(int pid) const { return pid >> 1; }
    __device__ int M(int) const { return g.B; }
    __device__ int N(int pid) const { return am(pid) == 0 || g.real ? (int)g.NB : 2 * (int)g.NB; }
    __device__ int K(int pid) const { const int r = g.B - am(pid) - (pid & 1); return r > 0 ? (r + 1) / 2 : 0; }
    static constexpr bool B_COL_AFFINE = true;
    __device__ int nlim(int pid, int n0) const { return n0 < g.NB ? (int)g.NB : N(pid); }
    __device__ long long rowA(int pid, int j) const { return leg_table_off(g.B, pid) + j; }
    __device__ long long colA(int, int k) const { return k * lstride(); }
    __device__ int a_sr(int) const { return 1; }
    __device__ int a_sk(int) const { return lstride(); }
    __device__ int lstride() const { return g.B + (g.B & 1); }  // legendre_stride (sgl_tables.hpp)
    __device__ long long rowB(int pid, int k) const {
        const int l = am(pid) + (pid & 1) + 2 * k;
        return l * (l + 1) * (int)sv.NB;
    }
    __device__ long long b_kstep(int) const { return 0; }
    __device__ long long colB(int pid, int n) const { return s_col(g, sv, am(pid), n); }
    __device__ long long rowC(int, int j) const { return j * g_rowstride(g); }
    __device__ long long colC(int pid, int n) const { return g_col(g, pid & 1, am(pid), n); }
    __device__ bool negC(int pid, int n) const { return n >= g.NB && (am(pid) & 1); }
    __device__ bool c_affine(int, int, int) const { return false; }  // blocked G: per-column offsets
    // offsets of columns col0 + 8 fn (fn < 4, all inside col0's sign half): the
    // sign, bin and row part of g_col computed once
    static constexpr bool HAS_COLC4 = true;
    __device__ void colC4(int pid, int col0, int (&o)[4]) const {
        const int NB = (int)g.NB;
        const int sgn = col0 >= NB;
        const int nn = col0 - (sgn ? NB : 0);
        const int a = am(pid), p = pid & 1;
        const int bin = sgn ? 2 * g.B - a : a;
        const int gs = (2 * g.nbins) << g.lgib;          // complex per shell group
        const int inner = ((p * g.nbins + bin) << g.lgib);  // (p, bin) row inside a group
        const int mask = (1 << g.lgib) - 1;
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
            const int sh = (nn >> 1) + 4 * fn;
            o[fn] = 2 * ((sh >> g.lgib) * gs + inner + (sh & mask)) + (nn & 1);
        }
    }
};

__host__ __device__ inline long long degree_offset(long long n) { return (n - 1) * n * (2 * n - 1) / 6; }
__device__ __forceinline__ int degree_offset32(int n) { return (n - 1) * n * (2 * n - 1) / 6; }  // n <= 257

// Shell-block view of the nu-major intermediate S for the radial stage.  On one
// GPU S is a single block S[nu][f][i] (i < 2B).  Under the multi-GPU shell / (l, m)
// split every rank receives one block per source rank, S_r[nu - nu0][f][i_local]
// (i_local < sc_blk), placed blk_stride reals apart; the radial GEMM reads them
// in place, so the exchange needs no re-interleaving pass.
struct ShellBlocks {
    int sc_blk;            // shells per block
    long long blk_stride;  // reals between blocks
    long long nu0;         // first nu held
    __device__ long long row(int i) const {
        if (blk_stride == 0) return 2 * i;  // one block (single GPU)
        const int b = i / sc_blk;
        return b * (int)blk_stride + 2 * (i - b * sc_blk);
    }
};

// Radial forward: prob = l.  rows n = l+1+r (M = B-l), K = 2B (i), cols (mf, c),
// mf = f * (2l+1) + (m + l).  g.SC = sc_blk, g.NB = batch * sc_blk * 2.
struct RadFwd {
    SGL_KIND_CFG(RADFWD, 8, 3, 4, 2)
    Geo g;
    const double* A;        // W
    const long long* aoff;
    const double* Bm;       // S blocks
    double* C;              // coefficients
    long long omega;        // coefficients per function
    ShellBlocks sb;
    static constexpr bool A_KCONTIG = true;
    static constexpr bool B_KCONTIG = true;
    static constexpr int B_ROW_TABLE = 512;  // K = 2B rows (shell blocks: not affine under the split)
    __device__ int M(int l) const { return g.B - l; }
    __device__ int mw(int l) const { return g.real ? l + 1 : 2 * l + 1; }  // orders per (l, f)
    __device__ int N(int l) const { return mw(l) * g.batch * 2; }
    __device__ int K(int) const { return 2 * g.B; }
    static constexpr bool B_COL_AFFINE = false;
    __device__ int nlim(int l, int) const { return N(l); }
    __device__ long long rowA(int l, int r) const { return rad_table_off(g.B, l) + r * 2 * g.B; }
    __device__ long long colA(int, int k) const { return k; }
    __device__ int a_sr(int) const { return 2 * g.B; }
    __device__ int a_sk(int) const { return 1; }
    __device__ long long rowB(int, int k) const { return sb.row(k); }
    __device__ long long b_kstep(int) const { return sb.sc_blk == 2 * g.B ? 2 : 0; }
    __device__ long long colB(int l, int n) const {
        const int mf = n >> 1, w = mw(l);
        const int f = g.batch == 1 ? 0 : mf / w, mm = mf - f * w + (g.real ? l : 0);  // mm = m + l
        return (l * l + mm - (int)sb.nu0) * (int)g.NB + f * 2 * g.SC + (n & 1);
    }
    __device__ long long rowC(int l, int r) const { return 2 * degree_offset32(l + 1 + r); }
    __device__ long long colC(int l, int n) const {
        const int mf = n >> 1, w = mw(l);
        const int f = g.batch == 1 ? 0 : mf / w, mm = mf - f * w + (g.real ? l : 0);
        return f * 2 * (int)omega + 2 * (l * l + mm) + (n & 1);
    }
    __device__ bool negC(int, int) const { return false; }
    __device__ bool c_affine(int, int, int) const { return false; }
    // real-valued path: every m > 0 coefficient also lands at -m as (-1)^m conj
    static constexpr bool MIRROR = true;
    __device__ long long colC_mirror(int l, int n, bool& neg) const {
        if (!g.real) return -1;
        const int mf = n >> 1, w = mw(l);
        const int f = g.batch == 1 ? 0 : mf / w, m = mf - f * w;
        if (m == 0) return -1;
        neg = m & 1;
        return f * 2 * (int)omega + 2 * (l * l + l - m) + (n & 1);
    }
};

// Radial inverse: prob = l.  rows i (M = 2B), K = B-l (n), cols (mf, c).
struct RadInv {
    SGL_KIND_CFG(RADINV, 8, 3, 4, 0)
    Geo g;
    const double* A;        // V
    const long long* aoff;
    const double* Bm;       // coefficients
    double* C;              // S blocks
    long long omega;
    ShellBlocks sb;
    static constexpr bool A_KCONTIG = false;  // V_l stored [n][i]: rows i contiguous
    static constexpr bool B_KCONTIG = false;
    static constexpr int B_ROW_TABLE = 256;  // K = B - l rows
    __device__ int M(int) const { return 2 * g.B; }
    __device__ int mw(int l) const { return g.real ? l + 1 : 2 * l + 1; }
    __device__ int N(int l) const { return mw(l) * g.batch * 2; }
    __device__ int K(int l) const { return g.B - l; }
    static constexpr bool B_COL_AFFINE = false;
    __device__ int nlim(int l, int) const { return N(l); }
    __device__ long long rowA(int l, int i) const { return rad_table_off(g.B, l) + i; }
    __device__ long long colA(int, int k) const { return k * 2 * g.B; }
    __device__ int a_sr(int) const { return 1; }
    __device__ int a_sk(int) const { return 2 * g.B; }
    __device__ long long rowB(int l, int k) const { return 2 * degree_offset32(l + 1 + k); }
    __device__ long long b_kstep(int) const { return 0; }
    __device__ long long colB(int l, int n) const {
        const int mf = n >> 1, w = mw(l);
        const int f = g.batch == 1 ? 0 : mf / w, mm = mf - f * w + (g.real ? l : 0);
        return f * 2 * (int)omega + 2 * (l * l + mm) + (n & 1);
    }
    __device__ long long rowC(int, int i) const { return sb.row(i); }
    __device__ long long colC(int l, int n) const {
        const int mf = n >> 1, w = mw(l);
        const int f = g.batch == 1 ? 0 : mf / w, mm = mf - f * w + (g.real ? l : 0);
        return (l * l + mm - (int)sb.nu0) * (int)g.NB + f * 2 * g.SC + (n & 1);
    }
    __device__ bool negC(int, int) const { return false; }
    __device__ bool c_affine(int, int, int) const { return false; }
};

__device__ __forceinline__ void cp_async16_zfill(void* smem_dst, const void* gmem_src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem_src), "r"(ok ? 16 : 0));
}

// Grouped DMMA GEMM, one tile per CTA (the block scheduler balances the
// ragged tiles; tiles are issued heaviest first).  4 warps of 32 x 32
// (4 x 4 m8n8k4 fragments) arranged WM x (4/WM): the CTA tile is (32 WM) x
// (128 / WM), chosen per tile by the host to fit the problem's M x N
// (narrow-N radial problems use 128 x 32, wide Legendre ones 32 x 128).
// k-chunks of P::GEMM_BK flow through a P::GEMM_ST-deep cp.async pipeline with zero-fill
// predication; shared-memory tiles keep the operand's contiguous dimension
// innermost (padded) so fills and fragment loads are bank-conflict free.
// 8-row fragments past M, 8-col fragments past N and k-steps past K are skipped.
// Multi-GPU variants whose epilogue stores go straight to the peers that own
// the output rows (NVLink peer stores; the fused exchange of distributed.py).
struct LegFwdPeers : LegFwd {
    PeerDest pd;  // rows of degree l go to the owner of l
    __device__ double* out_row(int pid, int r) const {
        const int l = am(pid) + (pid & 1) + 2 * r;
        int q = 0;
        while (q + 1 < pd.n && l >= pd.bound[q + 1]) ++q;
        return pd.base[q] + rowC(pid, r);
    }
};
// Legendre forward whose B tiles (the blocked G, 4-shell groups) arrive by TMA:
// one cp.async.bulk.tensor per chunk, issued by one thread and completing on an
// mbarrier, into a [group][k][8] shared layout that the 8 x 8 x 4 fragment reads
// hit without bank conflicts; the A tiles keep cp.async.  32 x 128 tiles only.
#ifndef SGL_LEGFWD_SPLIT
#define SGL_LEGFWD_SPLIT 0  // measured: no gain (round 2)
#endif
struct LegFwdTma : LegFwd {
    static constexpr bool B_TMA = true;
    static constexpr int GEMM_MAXWM = 1;
    // 5 CTAs / SM (96 registers, no spills; the cp.async-fed LegFwd would spill):
    // 94.9 -> 92.0 us at B = 128 (round 2)
    static constexpr int GEMM_MINB = SGL_MINB_LEGFWD > 0 ? SGL_MINB_LEGFWD : 5;
    alignas(64) CUtensorMap tmap;  // G viewed as [p][bin][group][j'][8 doubles]
};
// The same with each 8-double shell-group block landing as two 4-double halves,
// [group][half][k][4] (4-shell groups only, a 5-D box {4, BK, 2, groups, 1}): a
// half-warp's B fragment (4 k x 4 columns) is then 16 consecutive doubles instead
// of two 32-byte windows of 64-byte rows that fall on the same banks (ncu,
// round 2: the B-operand LDS.64 ran at 2x their ideal wavefronts).
struct LegFwdTmaSplit : LegFwdTma {
    static constexpr bool B_SPLIT = true;
};
// ... and its multi-GPU form (S rows to their owners' receive buffers).
struct LegFwdTmaPeers : LegFwdTma {
    PeerDest pd;
    __device__ double* out_row(int pid, int r) const {
        const int l = am(pid) + (pid & 1) + 2 * r;
        int q = 0;
        while (q + 1 < pd.n && l >= pd.bound[q + 1]) ++q;
        return pd.base[q] + rowC(pid, r);
    }
};
// Legendre forward over one SLICE of at most 32 shells (the fused persistent
// spherical forward): 32 x 128 tiles that straddle the +m / -m halves (NB <= 64
// reals per half), so a tile's B operand is two TMA boxes per k-chunk -- bin m and
// bin 2B - m of the slice's shell groups -- and the G block a slice needs stays
// L2-sized.  The tensor map lives in the kernel's grid-constant parameters
// (tmap_ptr points there); gx_base is the slice's first shell group.
struct LegFwdSlice : LegFwd {
    static constexpr bool B_TMA = true;
    static constexpr bool STRADDLE = true;
    static constexpr int GEMM_MAXWM = 1;
    const CUtensorMap* tmap_ptr;
    int gx_base;
    unsigned box_bytes;  // one half's box: NB x BK doubles
    __device__ int nlim(int pid, int) const { return N(pid); }
};
struct LegInvSeq : LegInv {  // CTAs run TileMap::seq consecutive n-blocks
    static constexpr bool GEMM_SEQ = true;
};
// Radial inverse of ONE complex function whose CTAs run consecutive n-blocks of a
// degree (the coefficient columns 2 (l^2 + l + m) + c are then affine in n): the
// short-K problems of high degree amortize the CTA prologue over the sequence.
struct RadInvSeq : RadInv {
    static constexpr bool GEMM_SEQ = true;
    static constexpr bool B_COL_AFFINE = true;
};
// Radial forward of one rank's degree range under the multi-GPU split whose
// coefficients are stored into every rank's coefficient vector (pd.base[q]; the
// degree ranges are disjoint, so each entry is written by exactly one rank): the
// assembly all-reduce becomes NVLink peer stores overlapped with the GEMM.
struct RadFwdBcast : RadFwd {
    PeerDest pd;
    static constexpr bool BCAST = true;
};
struct RadInvPeers : RadInv {
    PeerDest pd;  // shell block b goes to its owner (base[b])
    __device__ double* out_row(int l, int i) const {
        const int b = i / sb.sc_blk;
        return pd.base[b] + 2LL * (i - b * sb.sc_blk);
    }
};

template <class P, class = void>
struct has_peers : std::false_type {};
template <class P>
struct has_peers<P, std::void_t<decltype(std::declval<const P&>().pd)>> : std::true_type {};

template <class P, class = void>
struct has_out_row : std::false_type {};
template <class P>
struct has_out_row<P, std::void_t<decltype(std::declval<const P&>().out_row(0, 0))>> : std::true_type {};

template <class P, class = void>
struct has_colc4 : std::false_type {};
template <class P>
struct has_colc4<P, std::void_t<decltype(P::HAS_COLC4)>> : std::bool_constant<P::HAS_COLC4> {};

template <class P, class = void>
struct has_btma : std::false_type {};
template <class P>
struct has_btma<P, std::void_t<decltype(P::B_TMA)>> : std::bool_constant<P::B_TMA> {};

template <class P, class = void>
struct has_bsplit : std::false_type {};
template <class P>
struct has_bsplit<P, std::void_t<decltype(P::B_SPLIT)>> : std::bool_constant<P::B_SPLIT> {};

template <class P, class = void>
struct has_straddle : std::false_type {};
template <class P>
struct has_straddle<P, std::void_t<decltype(P::STRADDLE)>> : std::bool_constant<P::STRADDLE> {};

template <class P, class = void>
struct has_bcast : std::false_type {};
template <class P>
struct has_bcast<P, std::void_t<decltype(P::BCAST)>> : std::bool_constant<P::BCAST> {};

template <class P, class = void>
struct has_mirror : std::false_type {};
template <class P>
struct has_mirror<P, std::void_t<decltype(P::MIRROR)>> : std::bool_constant<P::MIRROR> {};

template <class P, int WM>
struct GemmCfg {
    static constexpr int FM = 4;
    static constexpr int BM = 32 * WM, BN = 128 / WM, BK = P::GEMM_BK, ST = P::GEMM_ST;
    static constexpr int LDA = P::A_KCONTIG ? BK + 4 : BM + 4;
    static constexpr int LDB = BN + 4;
    static constexpr int A_STAGE = P::A_KCONTIG ? BM * LDA : BK * LDA;
    // TMA-fed B ([group of 8 columns][k][8], unpadded) starts 128-byte aligned
    static constexpr int B_STAGE = has_btma<P>::value ? BK * BN : BK * LDB;
    static constexpr int STAGE = A_STAGE + B_STAGE;
    static constexpr int AQ = BM * BK / 128;  // A elements per thread
    static constexpr int BQ = BK * BN / 256;  // B (re, im) pairs per thread
};

template <class P>
constexpr size_t gemm_smem_bytes() {
    constexpr int s1 = GemmCfg<P, 1>::STAGE, s2 = P::GEMM_MAXWM >= 2 ? GemmCfg<P, 2>::STAGE : 0,
                  s4 = P::GEMM_MAXWM >= 4 ? GemmCfg<P, 4>::STAGE : 0;
    constexpr int m = s1 > s2 ? (s1 > s4 ? s1 : s4) : (s2 > s4 ? s2 : s4);
    return sizeof(double) * (P::GEMM_ST * m + P::B_ROW_TABLE + P::GEMM_ST);  // + B row table + TMA mbarriers
}

// One k-chunk of MMAs for a warp with FA x NA active 8 x 8 fragments.  mid()
// (the next chunk's cp.async issue) runs once, where the kind's GEMM_ISSUE puts
// it: 0 before the MMAs, 1 after the first k-step, 2 after the chunk.
template <class P, int WM, int FA, int NA, bool FULL, class Mid>
__device__ __forceinline__ void mma_chunk(const double* as, const double* bs, double (&acc)[4][4][2], int ksteps,
                                          int wr, int wc, int lane, Mid&& mid) {
    using C = GemmCfg<P, WM>;
#pragma unroll
    for (int kk = 0; kk < C::BK; kk += 4) {
        if (!FULL && kk >= ksteps) break;
        double af[FA > 0 ? FA : 1], bf[NA > 0 ? NA : 1];
#pragma unroll
        for (int fm = 0; fm < FA; ++fm) {
            const int r = wr + fm * 8 + (lane >> 2), k = kk + (lane & 3);
            af[fm] = P::A_KCONTIG ? as[r * C::LDA + k] : as[k * C::LDA + r];
        }
#pragma unroll
        for (int fn = 0; fn < NA; ++fn)
            bf[fn] = has_bsplit<P>::value
                         ? bs[((wc >> 3) + fn) * (C::BK * 8) + (lane >> 4) * (C::BK * 4) + (kk + (lane & 3)) * 4 +
                              ((lane >> 2) & 3)]
                     : has_btma<P>::value ? bs[((wc >> 3) + fn) * (C::BK * 8) + (kk + (lane & 3)) * 8 + (lane >> 2)]
                                        : bs[(kk + (lane & 3)) * C::LDB + wc + fn * 8 + (lane >> 2)];
#pragma unroll
        for (int fm = 0; fm < FA; ++fm)
#pragma unroll
            for (int fn = 0; fn < NA; ++fn) dmma884(acc[fm][fn], af[fm], bf[fn]);
        if (P::GEMM_ISSUE == 1 && kk == 0) mid();
    }
    if (P::GEMM_ISSUE == 2) mid();
}

template <class P, int WM, bool FULL, class Mid>
__device__ __forceinline__ void dispatch_chunk(int fa, int na, const double* as, const double* bs,
                                               double (&acc)[4][4][2], int ksteps, int wr, int wc, int lane,
                                               Mid&& mid) {
    if (P::GEMM_ISSUE == 0) mid();
    auto mid2 = [&] {
        if (P::GEMM_ISSUE != 0) mid();
    };
    if (fa == 4 && na == 4) {  // the common full-fragment case first
        mma_chunk<P, WM, 4, 4, FULL>(as, bs, acc, ksteps, wr, wc, lane, mid2);
        return;
    }
#define SGL_MMA_CASE(A_, N_) \
    case A_ * 8 + N_: mma_chunk<P, WM, A_, N_, FULL>(as, bs, acc, ksteps, wr, wc, lane, mid2); break;
    switch (fa * 8 + na) {
        SGL_MMA_CASE(4, 4) SGL_MMA_CASE(4, 3) SGL_MMA_CASE(4, 2) SGL_MMA_CASE(4, 1)
        SGL_MMA_CASE(3, 4) SGL_MMA_CASE(3, 3) SGL_MMA_CASE(3, 2) SGL_MMA_CASE(3, 1)
        SGL_MMA_CASE(2, 4) SGL_MMA_CASE(2, 3) SGL_MMA_CASE(2, 2) SGL_MMA_CASE(2, 1)
        SGL_MMA_CASE(1, 4) SGL_MMA_CASE(1, 3) SGL_MMA_CASE(1, 2) SGL_MMA_CASE(1, 1)
        default: mid2(); break;  // a warp with no active fragment only helps with the loads
    }
#undef SGL_MMA_CASE
}

// Epilogue (registers -> global).  The column part of the output address and
// the sign are per column only: computed once per fragment column (and, where
// the problem's columns are affine inside this tile, from one base).
template <class P, int WM>
__device__ __forceinline__ void gemm_epilogue(const P& pr, int pid, int m0, int n0, int M, int N,
                                              const double (&acc)[4][4][2], int wr, int wc, int lane) {
    using C = GemmCfg<P, WM>;
    constexpr int BN = C::BN, FM = C::FM;
    // signs are applied as sign-bit flips (a DMUL would compete with the DMMAs
    // for the FP64 pipe)
    int cofs[4];
    unsigned long long csg[4];
    const bool caff = pr.c_affine(pid, n0, BN);
    const int cbase = caff ? (int)pr.colC(pid, n0) : 0;
    if constexpr (has_colc4<P>::value) pr.colC4(pid, n0 + wc + 2 * (lane & 3), cofs);
#pragma unroll
    for (int fn = 0; fn < 4; ++fn) {
        const int col = n0 + wc + fn * 8 + 2 * (lane & 3);
        const bool ok = col < N;
        if constexpr (!has_colc4<P>::value) cofs[fn] = ok ? (caff ? cbase + (col - n0) : (int)pr.colC(pid, col)) : 0;
        csg[fn] = ok && pr.negC(pid, col) ? 0x8000000000000000ULL : 0ULL;
    }
    auto flip = [](double v, unsigned long long m) { return __longlong_as_double(__double_as_longlong(v) ^ m); };
#pragma unroll
    for (int fm = 0; fm < FM; ++fm) {
        const int row = m0 + wr + fm * 8 + (lane >> 2);
        if (row >= M) continue;
        double* out;
        if constexpr (has_out_row<P>::value) out = pr.out_row(pid, row);
        else out = pr.C + (int)pr.rowC(pid, row);
        if constexpr (has_bcast<P>::value) {  // every destination gets the row (pr.C unused)
            const int ro = (int)pr.rowC(pid, row);
#pragma unroll
            for (int fn = 0; fn < 4; ++fn) {
                const int col = n0 + wc + fn * 8 + 2 * (lane & 3);
                if (col >= N) continue;
                const double2 v = make_double2(flip(acc[fm][fn][0], csg[fn]), flip(acc[fm][fn][1], csg[fn]));
                bool neg = false;
                const long long mo = has_mirror<P>::value ? pr.colC_mirror(pid, col, neg) : -1;
                const unsigned long long ms = neg ? 0x8000000000000000ULL : 0ULL;
                for (int q = 0; q < pr.pd.n; ++q) {
                    double* o = pr.pd.base[q] + ro;
                    *reinterpret_cast<double2*>(o + cofs[fn]) = v;
                    if (mo >= 0)  // (-1)^m conj (real path)
                        *reinterpret_cast<double2*>(o + mo) =
                            make_double2(flip(acc[fm][fn][0], ms), flip(acc[fm][fn][1], ms ^ 0x8000000000000000ULL));
                }
            }
            continue;
        }
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
            const int col = n0 + wc + fn * 8 + 2 * (lane & 3);
            if (col >= N) continue;
            const double2 v = make_double2(flip(acc[fm][fn][0], csg[fn]), flip(acc[fm][fn][1], csg[fn]));
            if (SGL_L2HINTS && has_colc4<P>::value)  // the Legendre inverse writes G: keep it in L2
                st_hint(reinterpret_cast<double2*>(out + cofs[fn]), v, policy_evict_last());
            else
                *reinterpret_cast<double2*>(out + cofs[fn]) = v;
            if constexpr (has_mirror<P>::value) {
                bool neg = false;
                const long long mo = pr.colC_mirror(pid, col, neg);
                const unsigned long long ms = neg ? 0x8000000000000000ULL : 0ULL;
                if (mo >= 0)  // (-1)^m conj
                    *reinterpret_cast<double2*>(out + mo) =
                        make_double2(flip(acc[fm][fn][0], ms), flip(acc[fm][fn][1], ms ^ 0x8000000000000000ULL));
            }
        }
    }
    if constexpr (has_peers<P>::value) {
        // peer (NVLink) stores are made visible system-wide before the kernel retires
        __threadfence_system();
    }
}

#ifndef SGL_A_QUAD
#define SGL_A_QUAD 0  // measured: no gain (round 2)
#endif
#ifndef SGL_GEMM_FASTISSUE
#define SGL_GEMM_FASTISSUE 1
#endif
template <class P, int WM>
__device__ __forceinline__ void gemm_tile(const P& pr, const Tile& t, double* smem) {
    using C = GemmCfg<P, WM>;
    constexpr int BM = C::BM, BN = C::BN, BK = C::BK, ST = C::ST, FM = C::FM;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = (warp % WM) * 32, wc = (warp / WM) * 32;
    const int pid = t.prob, m0 = t.m0, n0 = t.n0;
    const int M = pr.M(pid), N = pr.nlim(pid, n0), K = pr.K(pid);
    const int nch = K > 0 ? (K + BK - 1) / BK : 1;

    // ---- per-tile load plan: every address this thread will fetch is
    // base + k0 * step, so a chunk issue is a handful of 64-bit adds.  A moves in
    // 2-element units along its contiguous dimension (k for A_KCONTIG, rows
    // otherwise): one 16-byte cp.async when the tile's rows are 16-byte aligned,
    // else two 8-byte ones.
    constexpr int AU = C::AQ / 2;
    const int a_sk = pr.a_sk(pid);
    const int a_sr = pr.a_sr(pid);
    const double* a_ptr[AU];
    int a_so[AU], a_k[AU];
    unsigned a_ok = 0, a_ok2 = 0;  // first / second element's row inside M
    {
        // every kind's A is 16-byte aligned in 2-element units: tables start at even
        // offsets with even row strides (the Legendre rows are padded to an even
        // length, sgl_tables.cpp) and the unit's second element is the next k
        // (A_KCONTIG) or the next row
        const long long abase = pr.rowA(pid, m0);
#pragma unroll
        for (int u = 0; u < AU; ++u) {
            const int e = tid + 128 * u;
            int row, k;
            if (P::A_KCONTIG && BK == 8 && SGL_A_QUAD) {
                // eight 16-byte units per quarter-warp (one shared-memory wavefront):
                // 4 rows x 2 units, whose row starts (96-byte stride) fall on
                // distinct 32-byte bank windows -- 2 rows x 4 units would collide
                const int q = e >> 3, w = e & 7;
                row = (q >> 1) * 4 + (w >> 1);
                k = 2 * (2 * (q & 1) + (w & 1));
                a_so[u] = row * C::LDA + k;
            } else if (P::A_KCONTIG) {
                row = e / (BK / 2);
                k = 2 * (e % (BK / 2));
                a_so[u] = row * C::LDA + k;
            } else {
                row = 2 * (e % (BM / 2));
                k = e / (BM / 2);
                a_so[u] = k * C::LDA + row;
            }
            a_k[u] = k;
            const bool ok = m0 + row < M;
            a_ok |= (ok ? 1u : 0u) << u;
            a_ok2 |= ((P::A_KCONTIG ? ok : m0 + row + 1 < M) ? 1u : 0u) << u;
            a_ptr[u] = ok ? pr.A + abase + (row * a_sr + k * a_sk) : pr.A;
        }
    }
    // B rows: affine kinds (B_ROW_TABLE == 0) advance their pointers by a fixed
    // stride per chunk; the others read row k's offset from a per-tile table in
    // shared memory (rowB(pid, k) for k < K, 0 past K), built once here, so a
    // chunk issue is one LDS + one 64-bit add per transfer instead of the row map
    // (quadratic / cubic in k for the Legendre-inverse / radial-inverse rows).
    constexpr bool TAB = P::B_ROW_TABLE > 0;
    const long long b_step = TAB ? 0 : pr.b_kstep(pid);
    int* ktab = reinterpret_cast<int*>(smem + ST * C::STAGE);
    if constexpr (TAB) {
        const int kr = nch * BK;  // <= P::B_ROW_TABLE (K <= the kind's maximum)
        for (int k = tid; k < kr; k += 128) ktab[k] = k < K ? (int)pr.rowB(pid, k) : 0;
        __syncthreads();
    }
    const double* b_ptr[C::BQ];
    int b_k[C::BQ], b_so[C::BQ];
    unsigned b_ok = 0;
    constexpr bool SEQ = P::GEMM_SEQ;
    static_assert(!SEQ || P::B_COL_AFFINE, "n-block sequences shift affine B columns");
    int b_bc[SEQ ? C::BQ : 1];
    {
        const long long bcol0 = P::B_COL_AFFINE ? pr.colB(pid, n0) : 0;
#pragma unroll
        for (int q = 0; q < C::BQ; ++q) {
            const int e = tid + 128 * q;
            int bc;
            if (P::B_KCONTIG) {  // 8 consecutive k per column pair: 128 B global runs
                const int hi = e >> 3;
                b_k[q] = (e & 7) + 8 * (hi / (BN / 2));
                bc = (hi % (BN / 2)) * 2;
            } else {
                bc = (e % (BN / 2)) * 2;
                b_k[q] = e / (BN / 2);
            }
            b_so[q] = b_k[q] * C::LDB + bc;
            if constexpr (SEQ) b_bc[q] = bc;
            const bool ok = n0 + bc < N;
            b_ok |= (ok ? 1u : 0u) << q;
            const long long col = !ok ? 0 : (P::B_COL_AFFINE ? bcol0 + bc : pr.colB(pid, n0 + bc));
            // affine rows: the k = b_k[q] row offset is folded in here
            b_ptr[q] = pr.Bm + col + (TAB ? 0 : (int)pr.rowB(pid, 0) + b_k[q] * (int)b_step);
        }
    }
    // A is affine in k for every kind: per-chunk advance k0 * a_sk.  Byte counts
    // of the 16-byte units for chunks entirely inside K (no k check needed).
    int a_nb[AU];
#pragma unroll
    for (int u = 0; u < AU; ++u) {
        const bool o1 = (a_ok >> u) & 1u, o2 = P::A_KCONTIG ? o1 : ((a_ok2 >> u) & 1u);
        a_nb[u] = o1 ? (o2 ? 16 : 8) : 0;
    }

    // Fast chunk issue (SGL_GEMM_FASTISSUE): when every transfer of this warp is a
    // full 16-byte unit inside M and N -- interior tiles, the vast majority -- a
    // chunk inside K is issued without predicates, selects or zero-fill sizes,
    // straight from precomputed 32-bit shared-memory destinations (the general path
    // spends ~20 instructions per cp.async).  Warp-uniform, so no divergence.
    unsigned a_dst[AU], b_dst[C::BQ];
    bool fast_issue = false;
    if constexpr (SGL_GEMM_FASTISSUE) {
        bool all = true;
#pragma unroll
        for (int u = 0; u < AU; ++u) {
            all = all && a_nb[u] == 16;
            a_dst[u] = static_cast<unsigned>(__cvta_generic_to_shared(smem + a_so[u]));
        }
#pragma unroll
        for (int q = 0; q < C::BQ; ++q)
            b_dst[q] = static_cast<unsigned>(__cvta_generic_to_shared(smem + C::A_STAGE + b_so[q]));
        if constexpr (SEQ) all = all && n0 + t.nseq * BN <= N;
        else all = all && b_ok == (1u << C::BQ) - 1u;
        fast_issue = __all_sync(0xffffffffu, all);
    }

    // SEQ: the CTA runs t.nseq consecutive n-blocks of the problem as one
    // pipelined sequence of chunks v = tile * nch + c (A is the same for all of
    // them; B columns shift by BN per tile), so each tile's epilogue overlaps the
    // next tile's loads and the CTA prologue is paid once per sequence.
    // TMA-fed B: one mbarrier per ring slot (thread 0 arrives with the expected
    // byte count; the TMA's completion flips it)
    unsigned tma_bar0 = 0;
    if constexpr (has_btma<P>::value) {
        tma_bar0 = static_cast<unsigned>(__cvta_generic_to_shared(smem + ST * C::STAGE + P::B_ROW_TABLE));
        if (tid == 0) {
#pragma unroll
            for (int q = 0; q < ST; ++q) mbar_init(tma_bar0 + 8u * q, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
    }
    // issue() is called for v = 0, 1, 2, ... in order: (tile, chunk) of the next
    // issue are counters (no division by nch per chunk)
    int is_tile = 0, is_chunk = 0;
    auto issue = [&](int v) {
        const int tv = SEQ ? is_tile : 0;
        const int c = SEQ ? is_chunk : v;
        if constexpr (SEQ) {
            if (++is_chunk == nch) {
                is_chunk = 0;
                ++is_tile;
            }
        }
        const int cs = tv * BN;  // column shift of tile tv
#ifdef SGL_GEMM_NOLOAD  // experiment: compute-only timing (wrong results)
        if (v > 0) { cp_async_commit(); return; }
#endif
        double* as = smem + (v % ST) * C::STAGE;
        double* bs = as + C::A_STAGE;
        const int k0 = c * BK;
        const bool kfull = k0 + BK <= K;
        const int a_adv = k0 * a_sk;
        if constexpr (SGL_GEMM_FASTISSUE && !has_btma<P>::value) {
            if (fast_issue && kfull) {
                const unsigned so = (unsigned)((v % ST) * C::STAGE * (int)sizeof(double));
#pragma unroll
                for (int u = 0; u < AU; ++u)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(a_dst[u] + so), "l"(a_ptr[u] + a_adv));
                const int b_adv = k0 * (int)b_step;
#pragma unroll
                for (int q = 0; q < C::BQ; ++q) {
                    const double* src = (TAB ? b_ptr[q] + ktab[k0 + b_k[q]] : b_ptr[q] + b_adv) + cs;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(b_dst[q] + so), "l"(src));
                }
                cp_async_commit();
                return;
            }
        }
#pragma unroll
        for (int u = 0; u < AU; ++u) {
#ifdef SGL_TABLE_L2  // experiment (wrong results): every table read from one 64 KB, L2-resident block
            const double* src = pr.A + (((a_ptr[u] - pr.A) + a_adv) & 8190);
#else
            const double* src = a_ptr[u] + a_adv;
#endif
            bool ok1, ok2;  // the unit's two elements
            if (kfull) {
                ok1 = a_nb[u] >= 8;
                ok2 = a_nb[u] == 16;
            } else if (P::A_KCONTIG) {
                const int kv = K - (k0 + a_k[u]);
                ok1 = ((a_ok >> u) & 1u) && kv >= 1;
                ok2 = ((a_ok >> u) & 1u) && kv >= 2;
            } else {
                const bool kok = k0 + a_k[u] < K;
                ok1 = ((a_ok >> u) & 1u) && kok;
                ok2 = ((a_ok2 >> u) & 1u) && kok;
            }
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(as + a_so[u]));
            const int nb = ok1 ? (ok2 ? 16 : 8) : 0;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(ok1 ? src : pr.A), "r"(nb));
        }
        if constexpr (has_straddle<P>::value) {
            // two TMA boxes per chunk: the slice's shells at bin m (columns [0, NB))
            // and, for m != 0, at bin 2B - m (columns [NB, 2 NB))
            if (tid == 0) {
                const int a = pr.am(pid);
                const bool two = N > (int)pr.g.NB;
                const unsigned bar = tma_bar0 + 8u * (unsigned)(v % ST);
                const int row = (pid & 1) * pr.g.nbins;
                mbar_expect_tx(bar, two ? 2 * pr.box_bytes : pr.box_bytes);
                const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(bs));
                tma_load_5d(dst, pr.tmap_ptr, bar, 0, k0, 0, pr.gx_base, row + a);
                if (two) tma_load_5d(dst + pr.box_bytes, pr.tmap_ptr, bar, 0, k0, 0, pr.gx_base, row + 2 * pr.g.B - a);
            }
            cp_async_commit();
            return;
        } else if constexpr (has_btma<P>::value) {
            // one TMA per chunk: box {8 doubles, BK rows j', BN/8 groups} of G
            if (tid == 0) {
                const int NB = (int)pr.g.NB;
                const int sgn = n0 >= NB;
                const int a = pr.am(pid);
                const int bin = sgn ? 2 * pr.g.B - a : a;
                const int gx0 = ((n0 - (sgn ? NB : 0)) >> 1) >> pr.g.lgib;
                const unsigned bar = tma_bar0 + 8u * (unsigned)(v % ST);
                mbar_expect_tx(bar, (unsigned)(BK * BN * sizeof(double)));
                tma_load_5d(static_cast<unsigned>(__cvta_generic_to_shared(bs)), &pr.tmap, bar, 0, k0, 0, gx0,
                            (pid & 1) * pr.g.nbins + bin);
            }
            cp_async_commit();
            return;
        }
        const int b_adv = k0 * (int)b_step;
#pragma unroll
        for (int q = 0; q < C::BQ; ++q) {
            const int k = k0 + b_k[q];
            bool ok;
            if constexpr (SEQ) ok = n0 + cs + b_bc[q] < N && (kfull || k < K);
            else ok = ((b_ok >> q) & 1u) && (kfull || k < K);
            const double* src = (TAB ? b_ptr[q] + ktab[k] : b_ptr[q] + b_adv) + cs;
            cp_async16_zfill(bs + b_so[q], ok ? src : pr.Bm, ok);
        }
        cp_async_commit();
    };

    const int fm_active = max(0, min(FM, (M - m0 - wr + 7) >> 3));
    const int fn_active = max(0, min(4, (N - n0 - wc + 7) >> 3));
    double acc[FM][4][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    if constexpr (SEQ) {
        const int nv = t.nseq * nch;
        int fna = fn_active;
#pragma unroll
        for (int v = 0; v < ST - 1; ++v) {
            if (v < nv) issue(v);
            else cp_async_commit();
        }
        int c = 0, tv = 0;
        for (int v = 0; v < nv; ++v) {
            cp_async_wait_group<ST - 2>();
            __syncthreads();
            auto mid = [&] {
                if (v + ST - 1 < nv) issue(v + ST - 1);
                else cp_async_commit();
            };
            const double* as = smem + (v % ST) * C::STAGE;
            const double* bs = as + C::A_STAGE;
            const int ksteps = min(BK, K - c * BK);
            if (ksteps == BK) {
                dispatch_chunk<P, WM, true>(fm_active, fna, as, bs, acc, BK, wr, wc, lane, mid);
            } else {
                dispatch_chunk<P, WM, false>(fm_active, fna, as, bs, acc, ksteps, wr, wc, lane, mid);
            }
            if (++c == nch) {  // tile tv complete: write it, reset for tile tv + 1
                gemm_epilogue<P, WM>(pr, pid, m0, n0 + tv * BN, M, N, acc, wr, wc, lane);
#pragma unroll
                for (int i = 0; i < FM; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
                c = 0;
                ++tv;
                fna = max(0, min(4, (N - (n0 + tv * BN) - wc + 7) >> 3));
            }
        }
        cp_async_wait_group<0>();
        return;
    }
#pragma unroll
    for (int c = 0; c < ST - 1; ++c) {
        if (c < nch) issue(c);
        else cp_async_commit();
    }
    for (int c = 0; c < nch; ++c) {
        cp_async_wait_group<ST - 2>();
        __syncthreads();
        if constexpr (has_btma<P>::value) mbar_wait(tma_bar0 + 8u * (unsigned)(c % ST), (unsigned)((c / ST) & 1));
        auto mid = [&] {
            if (c + ST - 1 < nch) issue(c + ST - 1);
            else cp_async_commit();
        };
        const double* as = smem + (c % ST) * C::STAGE;
        const double* bs = as + C::A_STAGE;
        const int ksteps = min(BK, K - c * BK);  // k-steps past K carry zeros: skip them
        // warp-uniform dispatch to straight-line MMA code: no per-MMA guards
        // (a guarded mma.sync costs ISETP + WARPSYNC + NOP per DMMA)
        if (ksteps == BK) {
            dispatch_chunk<P, WM, true>(fm_active, fn_active, as, bs, acc, BK, wr, wc, lane, mid);
        } else {
            dispatch_chunk<P, WM, false>(fm_active, fn_active, as, bs, acc, ksteps, wr, wc, lane, mid);
        }
    }
    cp_async_wait_group<0>();
    gemm_epilogue<P, WM>(pr, pid, m0, n0, M, N, acc, wr, wc, lane);
}

// Tile of this CTA from the launch's problem table (kernel parameter space: a
// handful of constant-cache reads instead of a dependent global load at CTA start).
template <int SEQ>
__device__ __forceinline__ Tile decode_tile(const TileMap& tm, long long NB, int b) {
    int lo = 0, hi = tm.nprob - 1;  // last entry with first[q] <= b
    if (tm.first[tm.nprob] == tm.nprob) lo = hi = b;  // one entry per tile
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tm.first[mid] <= b) lo = mid;
        else hi = mid - 1;
    }
    const int info = tm.info[lo], tn = tm.tn[lo], local = b - tm.first[lo];
    const int lwm = (info >> 16) & 3, halves = ((info >> 18) & 1) + 1;
    if constexpr (SEQ) {  // CTAs run groups of `seq` consecutive n-blocks (seq chosen per launch)
        const int seq = ((info >> 26) & 7) + 1;
        const int tg = (tn + seq - 1) / seq;
        const int per_m = halves * tg;
        const int mi = local / per_m, rest = local - mi * per_m;
        const int hl = rest / tg, gi = rest - hl * tg, h = hl + ((info >> 19) & 1);
        const int ni = gi * seq + tm.ni0[lo];
        return Tile{info & 0xffff, (mi + ((info >> 20) & 63)) * (32 << lwm), (int)(h * NB) + ni * (128 >> lwm),
                    1 << lwm, min(seq, tn - gi * seq)};
    }
    const int per_m = halves * tn;
    const int mi = local / per_m, rest = local - mi * per_m;
    const int hl = rest / tn, ni = rest - hl * tn + tm.ni0[lo], h = hl + ((info >> 19) & 1);
    return Tile{info & 0xffff, (mi + (info >> 20)) * (32 << lwm), (int)(h * NB) + ni * (128 >> lwm), 1 << lwm, 1};
}

template <class P>
__global__ void __launch_bounds__(128, P::GEMM_MINB) gemm_dmma_kernel(const __grid_constant__ P pr, const __grid_constant__ TileMap tm) {
    extern __shared__ __align__(128) double gsm[];
    const Tile t = decode_tile<P::GEMM_SEQ>(tm, pr.g.NB, blockIdx.x);
    switch (t.pad) {  // warp layout chosen per tile (the host keeps wm <= P::GEMM_MAXWM)
        case 1: gemm_tile<P, 1>(pr, t, gsm); break;
        case 2: if constexpr (P::GEMM_MAXWM >= 2) gemm_tile<P, 2>(pr, t, gsm); break;
        default: if constexpr (P::GEMM_MAXWM >= 4) gemm_tile<P, 4>(pr, t, gsm); break;
    }
}

// ------------------------------------------------------------------ Legendre inverse, warp-private pipelines
// The Legendre inverse's problems are short in K (<= B/2 degrees of one parity) and
// wide in N, so the general engine's per-chunk CTA barrier and per-chunk A reload
// weigh heavily.  Here a CTA (one 32-row block of a problem, a sequence of 128-column
// n-blocks) loads its whole A panel -- 32 table rows x K -- once, and each warp then
// runs its own 32 x 32 pipeline: it copies its own 32 columns of S chunk by chunk
// (cp.async ring private to the warp), waits on its own copies (wait_group +
// __syncwarp) and never meets the other warps again: no CTA barrier after the panel,
// warps drift freely across chunks and tiles, one A transfer per problem row block.
// Used when every n-block is full (NB % 128 == 0), B % 32 == 0 and 64 <= B <= 256.
#ifndef SGL_LEGINV_WP
#define SGL_LEGINV_WP 1
#endif
#ifndef SGL_LEGINV_WP_SWZ
#define SGL_LEGINV_WP_SWZ 0
#endif
// SWZ: unpadded 32-double rows with an XOR swizzle (element (k, x) of the panel or of a
// ring stage at k * 32 + (x ^ 4 (k & 3)): a DMMA fragment's 4 k x 4 rows / columns still
// cover 16 distinct doubles of a 128-byte line, 16-byte units stay intact) and 3 ring
// stages -- 40 KB per CTA at K <= 64, so 5 CTAs per SM fit instead of 4.
template <int KMAX, bool SWZ>
struct LegInvWp {
    static constexpr int ST = SWZ ? 3 : 4, BK = 8, LDA = SWZ ? 32 : 36, LDB = LDA;
    static constexpr int A_PANEL = KMAX * LDA;        // doubles: [k][row]
    static constexpr int B_STAGE = BK * LDB;          // doubles per warp and stage
    static constexpr int MINB = SWZ ? 5 : (KMAX <= 64 ? 4 : 3);
    static constexpr size_t smem_bytes() { return sizeof(double) * (A_PANEL + 4 * ST * B_STAGE); }
    static __host__ __device__ constexpr int sw(int k) { return SWZ ? 4 * (k & 3) : 0; }
};

template <int KMAX, bool SWZ>
__global__ void __launch_bounds__(128, (LegInvWp<KMAX, SWZ>::MINB))
leginv_wp_kernel(const __grid_constant__ LegInv pr, const __grid_constant__ TileMap tm) {
    using W = LegInvWp<KMAX, SWZ>;
    constexpr int ST = W::ST, BK = W::BK, LDA = W::LDA, LDB = W::LDB;
    extern __shared__ __align__(128) double gsm[];
    double* As = gsm;
    double* Bw = gsm + W::A_PANEL + (threadIdx.x >> 5) * (ST * W::B_STAGE);
    const Tile t = decode_tile<true>(tm, pr.g.NB, blockIdx.x);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int pid = t.prob, m0 = t.m0, n0 = t.n0;
    const int M = pr.M(pid), N = pr.nlim(pid, n0), K = pr.K(pid);
    const int nch = K > 0 ? (K + BK - 1) / BK : 1;
    const int kr = nch * BK;

    // ---- A panel (table rows m0 .. m0 + 31, all K degrees; zero past K) and the row-offset table
    {
        const double* a0 = pr.A + pr.rowA(pid, m0);
        const int a_sk = pr.a_sk(pid);
        for (int e = tid; e < kr * 16; e += 128) {  // 16-byte units: k = e / 16, rows 2 (e % 16), +1
            const int k = e >> 4, r = (e & 15) * 2;
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(As + k * LDA + (r ^ W::sw(k))));
            const bool ok = k < K;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(ok ? a0 + (long long)k * a_sk + r : pr.A),
                         "r"(ok ? 16 : 0));
        }
        cp_async_commit();
    }
    // ---- this warp's B pipeline: chunk v = (tile tv, k-chunk c); lane copies rows r0 + 2 i, unit u.
    // Row k of the chunk is degree l = l0 + 2 k of the nu-major S, at l (l + 1) NB reals
    // (LegInv::rowB); the lane's four rows are l, l + 4, l + 8, l + 12 with l = la, and la
    // advances by 16 per chunk: off(l) and e = (2 l + 1) NB are carried incrementally,
    //   off(l + 16) = off(l) + 16 e + 256 NB,  off(l + 4 i) = off(l) + 4 i e + 16 i^2 NB.
    const int r0 = lane >> 4, u = lane & 15;
    const double* bcol = pr.Bm + pr.colB(pid, n0) + 32 * warp + 2 * u;
    // ring rows r0, r0 + 4 (copies 0, 2) and r0 + 2, r0 + 6 (copies 1, 3) share a swizzle
    const unsigned bdst = static_cast<unsigned>(__cvta_generic_to_shared(Bw + r0 * LDB + ((2 * u) ^ W::sw(r0))));
    const unsigned bdst2 = static_cast<unsigned>(__cvta_generic_to_shared(Bw + (r0 + 2) * LDB + ((2 * u) ^ W::sw(r0 + 2))));
    const int nv = t.nseq * nch;
    const int snb = (int)pr.sv.NB;
    const int la0 = pr.am(pid) + (pid & 1) + 2 * r0;
    const int off_init = la0 * (la0 + 1) * snb, e_init = (2 * la0 + 1) * snb;
    int off = off_init, e = e_init;
    int is_chunk = 0;
    const double* bcs = bcol;  // + 128 per finished tile
    auto issue = [&](int v) {
        const unsigned sto = (unsigned)((v % ST) * W::B_STAGE * (int)sizeof(double));
        const unsigned so = bdst + sto, so2 = bdst2 + sto;
        const int o1 = off + 4 * e + 16 * snb, o2 = off + 8 * e + 64 * snb, o3 = off + 12 * e + 144 * snb;
        const bool tail = is_chunk == nch - 1;
        if (!tail || K == kr) {  // every row of the chunk inside K (uniform)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(so), "l"(bcs + off));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(so2), "l"(bcs + o1));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(so + 4u * LDB * 8u), "l"(bcs + o2));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(so2 + 4u * LDB * 8u), "l"(bcs + o3));
        } else {
            const int kb = is_chunk * BK + r0;
            const int oo[4] = {off, o1, o2, o3};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const bool ok = kb + 2 * i < K;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(((i & 1) ? so2 : so) + (unsigned)((i >> 1) * 4 * LDB * 8)),
                             "l"(ok ? bcs + oo[i] : pr.Bm), "r"(ok ? 16 : 0));
            }
        }
        cp_async_commit();
        if (tail) {  // next chunk starts the next n-block
            is_chunk = 0;
            off = off_init;
            e = e_init;
            bcs += 128;
        } else {
            ++is_chunk;
            off += 16 * e + 256 * snb;
            e += 32 * snb;
        }
    };
    // the first B chunks are in flight while the panel arrives
#pragma unroll
    for (int v = 0; v < ST - 1; ++v) {
        if (v < nv) issue(v);
        else cp_async_commit();
    }
    cp_async_wait_group<ST - 1>();  // this thread's share of the panel (the oldest group)
    __syncthreads();                // panel visible to all warps: the only CTA barrier
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    int c = 0, tv = 0;
    for (int v = 0; v < nv; ++v) {
        cp_async_wait_group<ST - 2>();
        __syncwarp();
        if (v + ST - 1 < nv) issue(v + ST - 1);
        else cp_async_commit();
        const double* as = As + c * BK * LDA;
        const double* bs = Bw + (v % ST) * W::B_STAGE;
        const int ksteps = min(BK, K - c * BK);
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            if (kk >= ksteps) break;
            double af[4], bf[4];
#pragma unroll
            for (int fm = 0; fm < 4; ++fm) af[fm] = as[(kk + (lane & 3)) * LDA + ((fm * 8 + (lane >> 2)) ^ W::sw(lane & 3))];
#pragma unroll
            for (int fn = 0; fn < 4; ++fn) bf[fn] = bs[(kk + (lane & 3)) * LDB + ((fn * 8 + (lane >> 2)) ^ W::sw(lane & 3))];
#pragma unroll
            for (int fm = 0; fm < 4; ++fm)
#pragma unroll
                for (int fn = 0; fn < 4; ++fn) dmma884(acc[fm][fn], af[fm], bf[fn]);
        }
        if (++c == nch) {
            // epilogue of a full interior tile: the column offsets of the blocked G once per
            // tile (colC4), the (-1)^m of the -m half as a uniform sign flip, rows one G
            // row stride apart -- no bounds checks (M, N full by construction)
            {
                const int ncol = n0 + tv * 128 + 32 * warp;
                int cofs[4];
                pr.colC4(pid, ncol + 2 * (lane & 3), cofs);
                if (pr.negC(pid, ncol)) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            // sign-bit flips on the integer pipe (a plain negation, and an XOR with a
                            // constant mask too, compile to DADD: FP64 pipe work next to the DMMAs)
#pragma unroll
                            for (int c2 = 0; c2 < 2; ++c2) {
                                int hi = __double2hiint(acc[i][j][c2]);
                                asm volatile("xor.b32 %0, %0, 0x80000000;" : "+r"(hi));
                                acc[i][j][c2] = __hiloint2double(hi, __double2loint(acc[i][j][c2]));
                            }
                        }
                }
                const int rs = g_rowstride(pr.g);
                double* out = pr.C + (long long)(m0 + (lane >> 2)) * rs;
#pragma unroll
                for (int fm = 0; fm < 4; ++fm) {
#pragma unroll
                    for (int fn = 0; fn < 4; ++fn)
                        *reinterpret_cast<double2*>(out + cofs[fn]) = make_double2(acc[fm][fn][0], acc[fm][fn][1]);
                    out += 8 * rs;
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            c = 0;
            ++tv;
        }
    }
    cp_async_wait_group<0>();
}

bool leginv_wp_ok(const Geo& g) {
    // B = 256 runs the K <= 128 instantiation at 3 CTAs/SM: 1243 -> 1206 us (SGL_LEGINV_WP_BMAX=128: off)
    const char* e = std::getenv("SGL_LEGINV_WP_BMAX");
    const int bmax = e ? std::atoi(e) : 256;
    return g.NB % 128 == 0 && g.B % 32 == 0 && g.B >= 64 && g.B <= bmax;
}

template <int KMAX, bool SWZ>
static int leginv_wp_launch(const LegInv& p, const TileMap* tiles, int ntiles, cudaStream_t s) {
    const size_t smem = LegInvWp<KMAX, SWZ>::smem_bytes();
    static SmemAttrOnce attr;
    attr.ensure(leginv_wp_kernel<KMAX, SWZ>, smem);
    leginv_wp_kernel<KMAX, SWZ><<<ntiles, 128, smem, s>>>(p, *tiles);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// ------------------------------------------------------------------ radial forward, warp-private pipelines
// Batched transforms at small bandlimits (B <= 64: configs C2, C5): a degree's radial
// problem is M = B - l <= 64 rows against K = 2B shells and a very wide N (all orders of
// all functions), and in the general engine its tiles -- half-empty in M, 8 to 16 chunks
// deep -- are dominated by per-tile and per-chunk overhead (radial_forward at 18% of the
// DMMA peak for B = 32 x 4096).  As in leginv_wp_kernel: a CTA takes one 32-row block of
// a degree and a sequence of 128-column n-blocks, loads its A panel (32 rows of W_l, all
// K shells) once, and each warp streams its own 32 columns of S through a private
// cp.async ring with no CTA barrier after the panel.  The (order, function) column pairs
// of a warp are 16 runs of S, each contiguous over the shells (re, im interleaved):
// lane (k, pair) copies 16 bytes of 8 lanes' 128-byte run.  Opt-in (SGL_RADFWD_WP=1):
// measured equal or slower than the general engine (sgl_capi.cpp, tiles_for).
template <int KMAX>
struct RadFwdWp {
    static constexpr int ST = 4, BK = 8, LDA = KMAX + 4, LDB = 36;
    static constexpr int A_PANEL = 32 * LDA;  // doubles: [row][k]
    static constexpr int B_STAGE = BK * LDB;
    static constexpr size_t smem_bytes() { return sizeof(double) * (A_PANEL + 4 * ST * B_STAGE); }
};

template <int FA>
__device__ __forceinline__ void radfwd_wp_chunk(const double* as, const double* bs, double (&acc)[4][4][2], int lane,
                                                int lda, int ldb) {
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4) {
        double af[FA], bf[4];
#pragma unroll
        for (int fm = 0; fm < FA; ++fm) af[fm] = as[(fm * 8 + (lane >> 2)) * lda + kk + (lane & 3)];
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) bf[fn] = bs[(kk + (lane & 3)) * ldb + fn * 8 + (lane >> 2)];
#pragma unroll
        for (int fm = 0; fm < FA; ++fm)
#pragma unroll
            for (int fn = 0; fn < 4; ++fn) dmma884(acc[fm][fn], af[fm], bf[fn]);
    }
}

template <int KMAX>
__global__ void __launch_bounds__(128, (KMAX <= 64 ? 4 : 3))
radfwd_wp_kernel(const __grid_constant__ RadFwd pr, const __grid_constant__ TileMap tm) {
    using W = RadFwdWp<KMAX>;
    constexpr int ST = W::ST, BK = W::BK, LDA = W::LDA, LDB = W::LDB;
    extern __shared__ __align__(128) double gsm[];
    double* As = gsm;
    double* Bw = gsm + W::A_PANEL + (threadIdx.x >> 5) * (ST * W::B_STAGE);
    const Tile t = decode_tile<true>(tm, pr.g.NB, blockIdx.x);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int l = t.prob, m0 = t.m0, n0 = t.n0;
    const int M = pr.M(l), N = pr.N(l), K = pr.K(l);  // K = 2B, a multiple of 8, <= KMAX
    const int nch = K / BK;
    {
        // A panel: rows m0 .. m0 + 31 of W_l (zero past M), K shells each, in 16-byte units
        const double* a0 = pr.A + pr.rowA(l, m0);
        const int ku = K / 2, a_sr = pr.a_sr(l);
        for (int e = tid; e < 32 * ku; e += 128) {
            const int r = e / ku, k2 = 2 * (e - r * ku);
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(As + r * LDA + k2));
            const bool ok = m0 + r < M;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(ok ? a0 + (long long)r * a_sr + k2 : pr.A),
                         "r"(ok ? 16 : 0));
        }
        cp_async_commit();
    }
    // this warp's B pipeline: lane = (shell kq of the chunk, pair group pq); its 4 copies per
    // chunk are column pairs pq + 4 i of the warp's 16 (S is contiguous over shells per pair)
    const int kq = lane & 7, pq = lane >> 3;
    const unsigned bdst = static_cast<unsigned>(__cvta_generic_to_shared(Bw + kq * LDB + 2 * pq));
    const int nv = t.nseq * nch;
    int is_chunk = 0, is_tile = 0;
    const double* bp[4];
    auto issue = [&](int v) {
        if (is_chunk == 0) {  // new n-block: the lane's four column-pair pointers (null past N)
            const int ncol = n0 + is_tile * 128 + 32 * warp + 2 * pq;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int col = ncol + 8 * i;
                bp[i] = col < N ? pr.Bm + pr.colB(l, col) + 2 * kq : nullptr;
            }
        }
        const unsigned so = bdst + (unsigned)((v % ST) * W::B_STAGE * (int)sizeof(double));
        const int adv = is_chunk * (2 * BK);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const bool ok = bp[i] != nullptr;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(so + (unsigned)(8 * i * 8)),
                         "l"(ok ? bp[i] + adv : pr.Bm), "r"(ok ? 16 : 0));
        }
        cp_async_commit();
        if (++is_chunk == nch) {
            is_chunk = 0;
            ++is_tile;
        }
    };
#pragma unroll
    for (int v = 0; v < ST - 1; ++v) {
        if (v < nv) issue(v);
        else cp_async_commit();
    }
    cp_async_wait_group<ST - 1>();
    __syncthreads();  // panel visible: the only CTA barrier
    const int fa = max(0, min(4, (M - m0 + 7) >> 3));
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    int c = 0, tv = 0;
    for (int v = 0; v < nv; ++v) {
        cp_async_wait_group<ST - 2>();
        __syncwarp();
        if (v + ST - 1 < nv) issue(v + ST - 1);
        else cp_async_commit();
        const double* as = As + c * BK;
        const double* bs = Bw + (v % ST) * W::B_STAGE;
        switch (fa) {  // 8-row fragments past M skipped (warp-uniform, straight-line MMAs)
            case 4: radfwd_wp_chunk<4>(as, bs, acc, lane, LDA, LDB); break;
            case 3: radfwd_wp_chunk<3>(as, bs, acc, lane, LDA, LDB); break;
            case 2: radfwd_wp_chunk<2>(as, bs, acc, lane, LDA, LDB); break;
            default: radfwd_wp_chunk<1>(as, bs, acc, lane, LDA, LDB); break;
        }
        if (++c == nch) {
            gemm_epilogue<RadFwd, 1>(pr, l, m0, n0 + tv * 128, M, N, acc, 0, 32 * warp, lane);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            c = 0;
            ++tv;
        }
    }
    cp_async_wait_group<0>();
}

bool radfwd_wp_ok(const Geo& g, const RadialBlocks& rb) {
    return g.B % 4 == 0 && g.B <= 64 && rb.blk_stride == 0 && rb.sc_blk == 2 * g.B;
}

template <int KMAX>
static int radfwd_wp_launch(const RadFwd& p, const TileMap* tiles, int ntiles, cudaStream_t s) {
    const size_t smem = RadFwdWp<KMAX>::smem_bytes();
    static SmemAttrOnce attr;
    attr.ensure(radfwd_wp_kernel<KMAX>, smem);
    radfwd_wp_kernel<KMAX><<<ntiles, 128, smem, s>>>(p, *tiles);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// ------------------------------------------------------------------ Legendre forward, warp-private pipelines
// The forward counterpart of leginv_wp_kernel: a CTA takes one 32-row block of a problem
// (rows = degrees l of one parity) and a sequence of 128-column n-blocks, loads its A
// panel (32 table rows x K = B polar nodes) once, and each warp streams its own 32 columns
// (16 shells) of the blocked G through a private cp.async ring -- no CTA barrier per chunk
// (the general TMA-fed kernel spends 23% of its stall samples at that barrier).  Rows of
// G are one row stride apart (affine), a lane's column offset is fixed per n-block.
// 64 <= B <= 128 (the panel is 32 x (B + 4) doubles), full n-blocks.
// Measured and NOT the default (SGL_LEGFWD_WP=1 turns it on): B = 128 90.7 -> 108.2 us with
// sequences of 4 (97.2 with 2) -- the 34 KB panel leaves 3 CTAs/SM against the TMA-fed
// kernel's 5; B = 64 x 64 479.3 -> 476.6 us (HBM-bound either way).
#ifndef SGL_LEGFWD_WP
#define SGL_LEGFWD_WP 0
#endif
template <int KMAX>
__global__ void __launch_bounds__(128, (KMAX <= 64 ? 4 : 3))
legfwd_wp_kernel(const __grid_constant__ LegFwd pr, const __grid_constant__ TileMap tm) {
    using W = RadFwdWp<KMAX>;  // same shared-memory plan: A panel [row][k], 4 x 4 stages of 8 x 36
    constexpr int ST = W::ST, BK = W::BK, LDA = W::LDA, LDB = W::LDB;
    extern __shared__ __align__(128) double gsm[];
    double* As = gsm;
    double* Bw = gsm + W::A_PANEL + (threadIdx.x >> 5) * (ST * W::B_STAGE);
    const Tile t = decode_tile<true>(tm, pr.g.NB, blockIdx.x);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int pid = t.prob, m0 = t.m0, n0 = t.n0;
    const int M = pr.M(pid), N = pr.nlim(pid, n0), K = pr.K(pid);  // K = B, a multiple of 8, <= KMAX
    const int nch = K / BK;
    {
        const double* a0 = pr.A + pr.rowA(pid, m0);
        const int ku = K / 2, a_sr = pr.a_sr(pid);
        for (int e = tid; e < 32 * ku; e += 128) {
            const int r = e / ku, k2 = 2 * (e - r * ku);
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(As + r * LDA + k2));
            const bool ok = m0 + r < M;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(ok ? a0 + (long long)r * a_sr + k2 : pr.A),
                         "r"(ok ? 16 : 0));
        }
        cp_async_commit();
    }
    // lane = (row r0 + 2 i of the chunk, shell u of the warp's 16): one column offset per n-block
    const int r0 = lane >> 4, u = lane & 15;
    const unsigned bdst = static_cast<unsigned>(__cvta_generic_to_shared(Bw + r0 * LDB + 2 * u));
    const int rs = g_rowstride(pr.g);
    const int nv = t.nseq * nch;
    int is_chunk = 0, is_tile = 0;
    const double* bp = pr.Bm;
    auto issue = [&](int v) {
        if (is_chunk == 0) bp = pr.Bm + pr.colB(pid, n0 + is_tile * 128 + 32 * warp + 2 * u) + (long long)r0 * rs;
        const unsigned so = bdst + (unsigned)((v % ST) * W::B_STAGE * (int)sizeof(double));
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(so + (unsigned)(2 * i * LDB * 8)),
                         "l"(bp + (long long)(2 * i) * rs));
        cp_async_commit();
        bp += (long long)BK * rs;
        if (++is_chunk == nch) {
            is_chunk = 0;
            ++is_tile;
        }
    };
#pragma unroll
    for (int v = 0; v < ST - 1; ++v) {
        if (v < nv) issue(v);
        else cp_async_commit();
    }
    cp_async_wait_group<ST - 1>();
    __syncthreads();  // panel visible: the only CTA barrier
    const int fa = max(0, min(4, (M - m0 + 7) >> 3));
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    int c = 0, tv = 0;
    for (int v = 0; v < nv; ++v) {
        cp_async_wait_group<ST - 2>();
        __syncwarp();
        if (v + ST - 1 < nv) issue(v + ST - 1);
        else cp_async_commit();
        const double* as = As + c * BK;
        const double* bs = Bw + (v % ST) * W::B_STAGE;
        switch (fa) {
            case 4: radfwd_wp_chunk<4>(as, bs, acc, lane, LDA, LDB); break;
            case 3: radfwd_wp_chunk<3>(as, bs, acc, lane, LDA, LDB); break;
            case 2: radfwd_wp_chunk<2>(as, bs, acc, lane, LDA, LDB); break;
            default: radfwd_wp_chunk<1>(as, bs, acc, lane, LDA, LDB); break;
        }
        if (++c == nch) {
            gemm_epilogue<LegFwd, 1>(pr, pid, m0, n0 + tv * 128, M, N, acc, 0, 32 * warp, lane);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            c = 0;
            ++tv;
        }
    }
    cp_async_wait_group<0>();
}

bool legfwd_wp_ok(const Geo& g) {
    const char* e = std::getenv("SGL_LEGFWD_WP");
    return (e ? std::atoi(e) : SGL_LEGFWD_WP) && g.NB % 128 == 0 && g.B % 32 == 0 && g.B >= 64 && g.B <= 128;
}

template <int KMAX>
static int legfwd_wp_launch(const LegFwd& p, const TileMap* tiles, int ntiles, cudaStream_t s) {
    const size_t smem = RadFwdWp<KMAX>::smem_bytes();
    static SmemAttrOnce attr;
    attr.ensure(legfwd_wp_kernel<KMAX>, smem);
    legfwd_wp_kernel<KMAX><<<ntiles, 128, smem, s>>>(p, *tiles);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// ------------------------------------------------------------------ G layout
long long g_layout(Geo& g) {
    const int N = 2 * g.B;
    int gib;
    switch (N) {  // the azimuthal kernels' shells per CTA (FFTShape<N>::IG, x2 for real)
        case 2: gib = FFTShape<2>::IG; break;
        case 4: gib = FFTShape<4>::IG; break;
        case 8: gib = FFTShape<8>::IG; break;
        case 16: gib = FFTShape<16>::IG; break;
        case 32: gib = FFTShape<32>::IG; break;
        case 64: gib = FFTShape<64>::IG; break;
        case 128: gib = g.az2x && !g.real ? FFTShape<128, kAz2xElems>::IG : FFTShape<128>::IG; break;
        case 256: gib = FFTShape<256>::IG; break;
        case 512: gib = FFTShape<512>::IG; break;
        default: gib = 1; break;  // naive DFT kernels: one shell per CTA
    }
    if (g.real) gib *= 2;
    int lg = 0;
    while ((1 << lg) < gib) ++lg;
    g.lgib = lg;
    g.nbins = g.real ? g.B : N;
    const long long nshell = (long long)g.batch * g.SC;
    g.ngx = (nshell + (1LL << lg) - 1) >> lg;
    return (long long)g.B * g.ngx * 2 * g.nbins << lg;
}

// ------------------------------------------------------------------ launchers
template <int N, int ELEMS = SGL_AZ_ELEMS>
static int az_fwd_launch(const Geo& g, const double* X, size_t fstride, double* G, const double* bcal,
                         const double* tw, cudaStream_t s) {
    using S = FFTShape<N, ELEMS>;
    const size_t smem = sizeof(double2) * (2 * S::IG * S::STRIDE);
    static SmemAttrOnce attr;
    attr.ensure(az_forward_kernel<N, ELEMS>, smem);
    const int nshell = g.batch * g.SC;
    dim3 grid(g.gxn ? g.gxn : (nshell + S::IG - 1) / S::IG, g.jpn ? g.jpn : g.B);
    az_forward_kernel<N, ELEMS><<<grid, S::THREADS, smem, s>>>(g, reinterpret_cast<const double2*>(X), fstride / 2,
                                                         reinterpret_cast<double2*>(G), bcal,
                                                         reinterpret_cast<const double2*>(tw));
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <int N, int ELEMS = SGL_AZI_ELEMS>
static int az_inv_launch(const Geo& g, const double* G, double* X, size_t fstride, const double* tw,
                         cudaStream_t s) {
    using S = FFTShape<N, ELEMS>;
    static_assert(ELEMS != SGL_AZI_ELEMS || S::IG == FFTShape<N>::IG,
                  "forward and inverse azimuthal tiles must match the G blocking");
    const size_t smem = sizeof(double2) * (2 * S::IG * S::STRIDE);
    static SmemAttrOnce attr;
    attr.ensure(az_inverse_kernel<N, ELEMS>, smem);
    const int nshell = g.batch * g.SC;
    dim3 grid(g.gxn ? g.gxn : (nshell + S::IG - 1) / S::IG, g.jpn ? g.jpn : g.B);
    az_inverse_kernel<N, ELEMS><<<grid, S::THREADS, smem, s>>>(g, reinterpret_cast<const double2*>(G),
                                                         reinterpret_cast<double2*>(X), fstride / 2,
                                                         reinterpret_cast<const double2*>(tw));
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// sample_stride is in doubles here (2 per complex); kernels take complex strides.
int launch_az_forward(const Geo& g, const double* samples, size_t sample_stride, double* G,
                      const double* bcal, const double* twiddle, cudaStream_t s) {
    switch (2 * g.B) {
        case 2: return az_fwd_launch<2>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 4: return az_fwd_launch<4>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 8: return az_fwd_launch<8>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 16: return az_fwd_launch<16>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 32: return az_fwd_launch<32>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 64: return az_fwd_launch<64>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 128:
            return g.az2x ? az_fwd_launch<128, kAz2xElems>(g, samples, sample_stride, G, bcal, twiddle, s)
                          : az_fwd_launch<128>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 256: return az_fwd_launch<256>(g, samples, sample_stride, G, bcal, twiddle, s);
        case 512: return az_fwd_launch<512>(g, samples, sample_stride, G, bcal, twiddle, s);
        default: break;
    }
    const int N = 2 * g.B;
    dim3 grid(g.batch * g.SC, g.B);
    az_forward_naive_kernel<<<grid, 128, 2 * N * sizeof(double2), s>>>(
        g, reinterpret_cast<const double2*>(samples), sample_stride / 2, reinterpret_cast<double2*>(G), bcal,
        reinterpret_cast<const double2*>(twiddle));
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_az_inverse(const Geo& g, const double* G, double* samples, size_t sample_stride,
                      const double* twiddle, cudaStream_t s) {
    switch (2 * g.B) {
        case 2: return az_inv_launch<2>(g, G, samples, sample_stride, twiddle, s);
        case 4: return az_inv_launch<4>(g, G, samples, sample_stride, twiddle, s);
        case 8: return az_inv_launch<8>(g, G, samples, sample_stride, twiddle, s);
        case 16: return az_inv_launch<16>(g, G, samples, sample_stride, twiddle, s);
        case 32: return az_inv_launch<32>(g, G, samples, sample_stride, twiddle, s);
        case 64: return az_inv_launch<64>(g, G, samples, sample_stride, twiddle, s);
        case 128:
            return g.az2x ? az_inv_launch<128, kAz2xElems>(g, G, samples, sample_stride, twiddle, s)
                          : az_inv_launch<128>(g, G, samples, sample_stride, twiddle, s);
        case 256: return az_inv_launch<256>(g, G, samples, sample_stride, twiddle, s);
        case 512: return az_inv_launch<512>(g, G, samples, sample_stride, twiddle, s);
        default: break;
    }
    const int N = 2 * g.B;
    dim3 grid(g.batch * g.SC, g.B);
    az_inverse_naive_kernel<<<grid, 128, 2 * N * sizeof(double2), s>>>(
        g, reinterpret_cast<const double2*>(G), reinterpret_cast<double2*>(samples), sample_stride / 2,
        reinterpret_cast<const double2*>(twiddle));
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <class P>
static int gemm_launch(const P& p, const TileMap* tiles, int ntiles, cudaStream_t s) {
    if (ntiles <= 0) return 0;
    // SGL_GEMM_SMEM_PAD: extra dynamic shared memory per CTA (occupancy experiments)
    static const size_t pad = [] {
        const char* e = std::getenv("SGL_GEMM_SMEM_PAD");
        return e ? (size_t)std::atol(e) : (size_t)0;
    }();
    const size_t smem = gemm_smem_bytes<P>() + pad;
    static SmemAttrOnce attr;
    attr.ensure(gemm_dmma_kernel<P>, smem);
    gemm_dmma_kernel<P><<<ntiles, 128, smem, s>>>(p, *tiles);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

#ifndef SGL_LEGFWD_TMA
#define SGL_LEGFWD_TMA 1  // measured at B = 128: 98.6 -> 94.4 us; B = 256: 1184 -> 1133 us
#endif
// TMA descriptor of the blocked G as a 5-D tensor [p][bin][group][j'][8 doubles]
// (innermost first: 8 doubles = 4 shells x re/im, j', group, bin, p) whose box
// {8, BK, 16, 1, 1} is one 32 x 128 tile's k-chunk of B.
static bool make_g_tensor_map(const Geo& g, const double* G, int bk, CUtensorMap* out, int box_groups = 0,
                              bool split = false) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    // groups of 2^lgib shells = W = 2^(lgib+1) doubles, split into H blocks of 8
    if (!encode || g.lgib < 2 || g.lgib > 6) return false;
    const cuuint64_t W = 2ULL << g.lgib, H = W / 8, groups = (cuuint64_t)g.ngx;
    const cuuint64_t row = 2ULL * groups * 2 * g.nbins * W / 2;  // doubles per j' row (g_rowstride)
    // dims (innermost first): 8 doubles, j', block of 8 inside a group, group,
    // (p, bin) as one index p * nbins + bin (its stride is W doubles either way)
    // split (4-shell groups): the H = 1 dimension becomes the two 4-double halves
    // of the group, ordered outside j' in shared memory ([group][half][j'][4])
    if (split && H != 1) return false;
    const cuuint64_t dims[5] = {split ? 4ULL : 8ULL, (cuuint64_t)g.B, split ? 2ULL : H, groups, 2ULL * g.nbins};
    const cuuint64_t strides[4] = {row * 8, split ? 32ULL : 64ULL, 2ULL * g.nbins * W * 8, W * 8};
    const cuuint32_t box[5] = {split ? 4u : 8u, (cuuint32_t)bk, split ? 2u : (cuuint32_t)H,
                               (cuuint32_t)(box_groups > 0 ? box_groups : 128 / W), 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(G), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ------------------------------------------------------------------ fused spherical forward
// One persistent launch for the whole spherical forward stage: CTAs pull work
// items from a global ticket counter -- azimuthal items (IG shells x one polar
// node pair, az_fwd_item) and Legendre tiles (LegFwdSlice) -- in the order
//   A_0, A_1 L_0, A_2 L_1, ..., A_{S-1} L_{S-2}, L_{S-1}
// (A_s: the azimuthal items of shell slice s, L_s: its Legendre tiles), so the
// DMMA-bound Legendre tiles of one slice run on the same SMs as, and overlap, the
// HBM-bound FFTs of the next.  A Legendre tile waits (one thread, acquire loads)
// until its slice's azimuthal items are all done; azimuthal items never wait, so
// the ticket order makes the schedule deadlock-free (every item a waiter depends
// on holds a lower ticket and is running or finished).  A slice's G block (at most
// 32 shells: 32 MB at B = 128) is consumed right after it is produced, from L2;
// with `discard` the last tile of a slice drops the slice's G lines from L2
// (discard.global.L2) so they are never written back to HBM.
struct SphFwdFused {
    Geo g;  // the call (batch, SC = 2B, G layout)
    const double2* X;
    size_t fstride;
    double2* G;
    const double* bcal;
    const double2* twg;
    LegFwdSlice leg;  // slice template: C = S base, sv = the full S view
    alignas(64) CUtensorMap tmap;
    int slice_shells, nslices, az_per_slice, leg_per_slice, total, discard;
    int mode;  // experiments (timing only, wrong results): 1 = azimuthal items only, 2 = Legendre tiles only
    int* ticket;
    int* az_done;
    int* leg_done;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int N>
__global__ void __launch_bounds__(128, 4)
sph_fwd_fused_kernel(const __grid_constant__ SphFwdFused prm, const __grid_constant__ TileMap tm) {
    if constexpr (FFTShape<N>::THREADS != 128) {  // fused items share 128-thread CTAs (the launcher declines)
        return;
    } else {
    extern __shared__ __align__(128) double gsm[];
    __shared__ int s_item, s_last;
    const int tid = threadIdx.x;
    const int nA = prm.az_per_slice, nL = prm.leg_per_slice, S = prm.nslices;
    constexpr int IG = FFTShape<N>::IG;
    for (;;) {
        if (tid == 0) s_item = atomicAdd(prm.ticket, 1);
        __syncthreads();
        const int t = s_item;
        __syncthreads();
        if (t >= prm.total) return;
        int slice, idx;
        bool az;
        if (t < nA) {
            az = true;
            slice = 0;
            idx = t;
        } else {
            const int u = t - nA, k = 1 + u / (nA + nL), r = u - (k - 1) * (nA + nL);
            if (k < S && r < nA) {
                az = true;
                slice = k;
                idx = r;
            } else {
                az = false;
                slice = k - 1;
                idx = k < S ? r - nA : r;
            }
        }
        const int s_first = slice * prm.slice_shells;
        if ((prm.mode == 1 && !az) || (prm.mode == 2 && az)) continue;
        if (az) {
            const int gps = prm.slice_shells / IG;  // shell groups per slice
            az_fwd_item<N>(prm.g, prm.X, prm.fstride, prm.G, prm.bcal, prm.twg, s_first + (idx % gps) * IG, idx / gps,
                           reinterpret_cast<double2*>(gsm));
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicAdd(prm.az_done + slice, 1);
            continue;
        }
        if (tid == 0) {
            while (prm.mode == 0 && ld_acquire_gpu(prm.az_done + slice) < nA) __nanosleep(200);
            // the G block was written through the generic proxy by other CTAs; the
            // TMA reads it through the async proxy
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
        }
        __syncthreads();
        LegFwdSlice pr = prm.leg;
        const int f = s_first / prm.g.SC;
        pr.C = prm.leg.C + (size_t)f * 2 * prm.g.SC;  // S[nu][f][i]: this function's block
        pr.sv.i0 = s_first - f * prm.g.SC;
        pr.gx_base = s_first >> prm.g.lgib;
        pr.tmap_ptr = &prm.tmap;
        gemm_tile<LegFwdSlice, 1>(pr, decode_tile<false>(tm, pr.g.NB, idx), gsm);
        __syncthreads();
        if (tid == 0) s_last = prm.discard && atomicAdd(prm.leg_done + slice, 1) + 1 == nL;
        __syncthreads();
        if (s_last) {  // every tile of the slice has read its G block: drop it from L2 unwritten
            const long long row = (long long)prm.g.ngx * 2 * prm.g.nbins * IG;  // complex per j' row
            const long long blk = 2LL * prm.g.nbins * prm.slice_shells;         // the slice's complex per row
            const long long lines = blk * 16 / 128;
            const double2* base = prm.G + (long long)(s_first >> prm.g.lgib) * 2 * prm.g.nbins * IG;
            for (long long q = tid; q < (long long)prm.g.B * lines; q += 128) {
                const long long jp = q / lines, ln = q - jp * lines;
                const char* a = reinterpret_cast<const char*>(base + jp * row) + ln * 128;
                asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(a) : "memory");
            }
        }
    }
    }
}

template <int N>
static int sph_fwd_fused_launch(const SphFwdFused& prm, const TileMap* tiles, int grid, cudaStream_t s) {
    using S = FFTShape<N>;
    if (S::THREADS != 128) return -2;  // fused items share 128-thread CTAs: the caller takes the staged path
    constexpr size_t az_smem = sizeof(double2) * (2 * S::IG * S::STRIDE);
    constexpr size_t gm_smem = gemm_smem_bytes<LegFwdSlice>();
    constexpr size_t smem = az_smem > gm_smem ? az_smem : gm_smem;
    static SmemAttrOnce attr;
    attr.ensure(sph_fwd_fused_kernel<N>, smem);
    if (grid <= 0) {
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sph_fwd_fused_kernel<N>, 128, smem);
        grid = sms * (per > 0 ? per : 1);
    }
    sph_fwd_fused_kernel<N><<<grid, 128, smem, s>>>(prm, *tiles);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_spherical_forward_fused(const Geo& g, const double* X, size_t sample_stride, double* G, const double* bcal,
                                   const double* tw, double* S, const SView& sv, const double* tab,
                                   const long long* tab_off, const TileMap* tiles, int tiles_per_slice,
                                   int slice_shells, int* counters, bool discard, int grid, cudaStream_t s) {
    const int nshell = g.batch * g.SC;
    const int ig = 1 << g.lgib;
    if (g.real || slice_shells <= 0 || slice_shells > 32 || slice_shells % ig || nshell % slice_shells ||
        g.SC % slice_shells)
        return -2;
    SphFwdFused prm{};
    prm.g = g;
    prm.X = reinterpret_cast<const double2*>(X);
    prm.fstride = sample_stride / 2;
    prm.G = reinterpret_cast<double2*>(G);
    prm.bcal = bcal;
    prm.twg = reinterpret_cast<const double2*>(tw);
    Geo gs = g;  // one slice's Legendre geometry (the G row stride keeps the full ngx)
    gs.SC = slice_shells;
    gs.batch = 1;
    gs.NB = 2LL * slice_shells;
    static_cast<LegFwd&>(prm.leg) = LegFwd{gs, tab, tab_off, G, S, sv};
    prm.leg.box_bytes = (unsigned)(gs.NB * LegFwd::GEMM_BK * sizeof(double));
    if (!make_g_tensor_map(g, G, LegFwd::GEMM_BK, &prm.tmap, slice_shells / ig)) return -2;
    prm.slice_shells = slice_shells;
    prm.nslices = nshell / slice_shells;
    prm.az_per_slice = (slice_shells / ig) * g.B;
    prm.leg_per_slice = tiles_per_slice;
    prm.total = prm.nslices * (prm.az_per_slice + tiles_per_slice);
    prm.discard = discard ? 1 : 0;
    if (const char* e = std::getenv("SGL_FUSED_MODE")) prm.mode = std::atoi(e);
    prm.ticket = counters;
    prm.az_done = counters + 1;
    prm.leg_done = counters + 1 + prm.nslices;
    if (cudaMemsetAsync(counters, 0, sizeof(int) * (1 + 2 * prm.nslices), s) != cudaSuccess) return -1;
    switch (2 * g.B) {
        case 32: return sph_fwd_fused_launch<32>(prm, tiles, grid, s);
        case 64: return sph_fwd_fused_launch<64>(prm, tiles, grid, s);
        case 128: return sph_fwd_fused_launch<128>(prm, tiles, grid, s);
        case 256: return sph_fwd_fused_launch<256>(prm, tiles, grid, s);
        default: return -2;
    }
}

int launch_legendre_forward(const Geo& g, const SView& sv, const double* G, double* S, const double* tab,
                            const long long* tab_off, const TileMap* tiles, int ntiles, cudaStream_t s) {
    LegFwd p{g, tab, tab_off, G, S, sv};
    if (ntiles > 0 && tiles->seq > 1)  // the tile builder emits sequences only where legfwd_wp_ok holds
        return g.B <= 64 ? legfwd_wp_launch<64>(p, tiles, ntiles, s) : legfwd_wp_launch<128>(p, tiles, ntiles, s);
    if (SGL_LEGFWD_TMA) {
        LegFwdTma q;
        static_cast<LegFwd&>(q) = p;
        if (SGL_LEGFWD_SPLIT && g.lgib == 2) {
            LegFwdTmaSplit qs;
            static_cast<LegFwd&>(qs) = p;
            if (make_g_tensor_map(g, G, LegFwd::GEMM_BK, &qs.tmap, 0, true)) return gemm_launch<LegFwdTmaSplit>(qs, tiles, ntiles, s);
        }
        if (make_g_tensor_map(g, G, LegFwd::GEMM_BK, &q.tmap)) return gemm_launch<LegFwdTma>(q, tiles, ntiles, s);
    }
    return gemm_launch<LegFwd>(p, tiles, ntiles, s);
}

int launch_legendre_forward_peers(const Geo& g, const SView& sv, const double* G, const PeerDest& pd,
                                  const double* tab, const long long* tab_off, const TileMap* tiles, int ntiles,
                                  cudaStream_t s) {
    if (SGL_LEGFWD_TMA) {
        LegFwdTmaPeers q;
        static_cast<LegFwd&>(q) = LegFwd{g, tab, tab_off, G, nullptr, sv};
        q.pd = pd;
        if (make_g_tensor_map(g, G, LegFwd::GEMM_BK, &q.tmap)) return gemm_launch<LegFwdTmaPeers>(q, tiles, ntiles, s);
    }
    LegFwdPeers p;
    static_cast<LegFwd&>(p) = LegFwd{g, tab, tab_off, G, nullptr, sv};
    p.pd = pd;
    return gemm_launch<LegFwdPeers>(p, tiles, ntiles, s);
}

int launch_legendre_inverse(const Geo& g, const SView& sv, const double* S, double* G, const double* tab,
                            const long long* tab_off, const TileMap* tiles, int ntiles, cudaStream_t s) {
    LegInv p{g, tab, tab_off, S, G, sv};
    {
        // warp-private pipelines: full n-blocks, full 32-row blocks, K <= 64 (B <= 128)
        const char* e = std::getenv("SGL_LEGINV_WP");  // read per call (the tests flip it)
        const int wp = e ? std::atoi(e) : SGL_LEGINV_WP;
        // (B = 32: K <= 16, two chunks per tile -- the panel and its barrier do not pay: 444 -> 488 us
        // for 512 functions; B = 64 x 64: 570 -> 561 us; B = 128: 101.9 -> 97.4 us)
        if (wp && ntiles > 0 && leginv_wp_ok(g))
        {
            const char* z = std::getenv("SGL_LEGINV_WP_SWZ");  // 5-CTA swizzled form (K <= 64)
            const bool swz = z ? std::atoi(z) != 0 : SGL_LEGINV_WP_SWZ != 0;
            if (g.B > 128) return leginv_wp_launch<128, false>(p, tiles, ntiles, s);
            if (g.B <= 64)
                return swz ? leginv_wp_launch<32, true>(p, tiles, ntiles, s) : leginv_wp_launch<32, false>(p, tiles, ntiles, s);
            return swz ? leginv_wp_launch<64, true>(p, tiles, ntiles, s) : leginv_wp_launch<64, false>(p, tiles, ntiles, s);
        }
    }
    if (ntiles > 0 && tiles->seq > 1) {
        LegInvSeq q;
        static_cast<LegInv&>(q) = p;
        return gemm_launch<LegInvSeq>(q, tiles, ntiles, s);
    }
    return gemm_launch<LegInv>(p, tiles, ntiles, s);
}

int launch_radial_forward(const Geo& g, const RadialBlocks& rb, const double* S, double* C,
                          const double* W, const long long* w_off, const TileMap* tiles, int ntiles,
                          cudaStream_t s) {
    RadFwd p{g, W, w_off, S, C, degree_offset(g.B + 1), ShellBlocks{rb.sc_blk, rb.blk_stride, rb.nu0}};
    if (ntiles > 0 && tiles->seq > 1)  // the tile builder asks for sequences only where radfwd_wp_ok holds
        return g.B <= 32 ? radfwd_wp_launch<64>(p, tiles, ntiles, s) : radfwd_wp_launch<128>(p, tiles, ntiles, s);
    return gemm_launch<RadFwd>(p, tiles, ntiles, s);
}

int launch_radial_forward_bcast(const Geo& g, const RadialBlocks& rb, const double* S, const PeerDest& pd,
                                const double* W, const long long* w_off, const TileMap* tiles, int ntiles,
                                cudaStream_t s) {
    RadFwdBcast p;
    static_cast<RadFwd&>(p) = RadFwd{g, W, w_off, S, nullptr, degree_offset(g.B + 1),
                                     ShellBlocks{rb.sc_blk, rb.blk_stride, rb.nu0}};
    p.pd = pd;
    return gemm_launch<RadFwdBcast>(p, tiles, ntiles, s);
}

int launch_radial_inverse(const Geo& g, const RadialBlocks& rb, const double* C, double* S,
                          const double* V, const long long* v_off, const TileMap* tiles, int ntiles,
                          cudaStream_t s) {
    RadInv p{g, V, v_off, C, S, degree_offset(g.B + 1), ShellBlocks{rb.sc_blk, rb.blk_stride, rb.nu0}};
    if (ntiles > 0 && tiles->seq > 1 && g.batch == 1 && !g.real) {
        RadInvSeq q;
        static_cast<RadInv&>(q) = p;
        return gemm_launch<RadInvSeq>(q, tiles, ntiles, s);
    }
    return gemm_launch<RadInv>(p, tiles, ntiles, s);
}

int launch_radial_inverse_peers(const Geo& g, const RadialBlocks& rb, const double* C, const PeerDest& pd,
                                const double* V, const long long* v_off, const TileMap* tiles, int ntiles,
                                cudaStream_t s) {
    RadInvPeers p;
    static_cast<RadInv&>(p) = RadInv{g, V, v_off, C, nullptr, degree_offset(g.B + 1),
                                     ShellBlocks{rb.sc_blk, rb.blk_stride, rb.nu0}};
    p.pd = pd;
    return gemm_launch<RadInvPeers>(p, tiles, ntiles, s);
}

}  // namespace sglk
