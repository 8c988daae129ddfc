// Launch interface of the sm_100a kernels (sgl_kernels.cu).  Host-side callers:
// sgl_capi.cpp.  All pointers are device pointers; every launcher enqueues on
// `stream` and returns the number of kernels it launched (or -1 on a launch error).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include <atomic>
#include <mutex>

namespace sglk {

// Opt-in to more than 48 KB of dynamic shared memory, once per kernel and
// device: the attribute belongs to the current device's context, and plans may
// live on several devices of one process (sglgpu_plan_desc::device) and be used
// from several threads.
struct SmemAttrOnce {
    std::atomic<unsigned long long> done{0};  // bit d: set on device d
    std::mutex mu;
    template <class Kernel>
    void ensure(Kernel k, size_t smem) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
        const unsigned long long bit = 1ULL << dev;
        if (done.load(std::memory_order_acquire) & bit) return;
        std::lock_guard<std::mutex> lock(mu);
        if (done.load(std::memory_order_relaxed) & bit) return;
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess)
            done.fetch_or(bit, std::memory_order_release);
    }
    template <class Kernel>
    void ensure_attr(Kernel k, cudaFuncAttribute a, int v) {  // any other attribute, same once-per-device rule
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
        const unsigned long long bit = 1ULL << dev;
        if (done.load(std::memory_order_acquire) & bit) return;
        std::lock_guard<std::mutex> lock(mu);
        if (done.load(std::memory_order_relaxed) & bit) return;
        if (cudaFuncSetAttribute(k, a, v) == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
    }
};


// Tile descriptor for the grouped DMMA contraction: {problem, m0, n0, warp layout wm}.
struct Tile {
    int prob, m0, n0, pad;
    int nseq;  // consecutive n-blocks this CTA runs (kinds with GEMM_SEQ > 1)
};

// Tiles of one grouped contraction, passed by value in kernel parameter space.
// Entry q is a block of tiles of one problem, listed heaviest tile first; it owns
// tiles [first[q], first[q + 1]), enumerated m-block major (from m-block mi0),
// then sign half (from h0; Legendre problems with m != 0 split N into the +m / -m
// halves of NB columns), then n-block (from n-block ni0).  Launches of at most
// kMaxProblems tiles get one entry per tile (a global heaviest-first order),
// larger ones one entry per problem (sibling tiles, which share an operand,
// run back to back).
#ifndef SGL_MAX_PROBLEMS
#define SGL_MAX_PROBLEMS 1024
#endif
constexpr int kMaxProblems = SGL_MAX_PROBLEMS;
struct TileMap {
    int nprob;
    int seq;  // n-blocks per CTA (1: one tile per CTA)
    int first[kMaxProblems + 1];
    int info[kMaxProblems];  // pid | log2(wm) << 16 | (halves - 1) << 18 | h0 << 19 | mi0 << 20
    int tn[kMaxProblems];    // n-blocks per half
    int ni0[kMaxProblems];
};

// The 4-warp GEMM CTA computes a (32 wm) x (128 / wm) tile, wm in {1, 2, 4}
// chosen per tile (Tile::pad) by the host.
constexpr int tile_rows(int wm) { return 32 * wm; }
constexpr int tile_cols(int wm) { return 128 / wm; }
// Largest wm each kind's kernel is built for (its shared-memory ring is sized for
// the largest stage it can see): the Legendre-forward problems have M <= B/2 + 1
// rows and always took 32 x 128 tiles, the only shape its TMA-fed kernel has.
// The Legendre inverse (B columns affine in n) has a second kernel whose CTAs run
// several consecutive n-blocks of a problem as one pipelined chunk sequence; the
// count is chosen per launch (TileMap::seq) and seq > 1 selects that kernel.
#ifndef SGL_MAXWM_LEGFWD
#define SGL_MAXWM_LEGFWD 1  // 32 x 128 tiles (the only shape the tile chooser picked; the TMA-fed kernel's)
#endif
#ifndef SGL_MAXWM_LEGINV
#define SGL_MAXWM_LEGINV 1  // 32 x 128 only (the chooser's pick at every B): one code path, 104.5 -> 103.1 us at B = 128
#endif
#ifndef SGL_MAXWM_RADFWD
#define SGL_MAXWM_RADFWD 4
#endif
#ifndef SGL_MAXWM_RADINV
#define SGL_MAXWM_RADINV 4
#endif

// Geometry shared by the stages.  "shell" is a flat index s = f * SC + i over
// the functions of the batch and the SC radial shells handled by the call.
struct Geo {
    int B;          // bandlimit
    int SC;         // shells per function in this call (2B for the whole transform)
    int batch;      // functions
    long long NB;   // reals per nu-row of S and per G row half: batch * SC * 2
    int real = 0;   // real-valued fast path: only m >= 0 is computed (f_{n,l,-m} = (-1)^m conj f_nlm)
    // Blocked layout of the azimuthal -> polar intermediate G (see g_index):
    // G[j'][shell group gx][p][bin][s_local], one contiguous block per azimuthal CTA.
    int lgib = 0;        // log2(shells per group) = log2 of the azimuthal kernel's tile
    int nbins = 0;       // bins per (p, shell): 2B (complex path, bin B unused) or B (real path)
    long long ngx = 0;   // shell groups = ceil(batch * SC / 2^lgib)
    // Sub-range of the azimuthal launch (the pipelined spherical stage, sgl_capi.cpp):
    // polar nodes j' in [jp0, jp0 + jpn) and shell groups [gx0, gx0 + gxn); 0 counts = all.
    int jp0 = 0, jpn = 0, gx0 = 0, gxn = 0;
    // complex path, 2B = 128: azimuthal CTAs of twice the elements (16-shell G groups); set by the
    // host for large batches before g_layout()
    int az2x = 0;
};

// Complex index of G(p, bin, j', flat shell s).
__host__ __device__ inline long long g_index(const Geo& g, int p, int bin, int jp, int s) {
    const long long gx = s >> g.lgib;
    const int sl = s & ((1 << g.lgib) - 1);
    return ((((long long)jp * g.ngx + gx) * 2 + p) * g.nbins + bin) * (1LL << g.lgib) + sl;
}

// Shells per azimuthal CTA (the G block size) for bandlimit B; fills the layout
// fields of g.  Returns the number of complex values G needs.
long long g_layout(Geo& g);

// Does the Legendre inverse of this geometry run on the warp-private kernel
// (leginv_wp_kernel)?  The tile builder uses longer n-block sequences for it.
bool leginv_wp_ok(const Geo& g);

// Azimuthal stage (forward): FFT of length 2B per ring (sign -1, kernels.cpp:478),
// b_cal weighting, equatorial fold E/O and scatter to the m-major intermediate
//   G[p][|m|][j'][sgn][f][i]  (complex), p = parity, j' < B, sgn = (m < 0).
int launch_az_forward(const Geo& g, const double* samples, size_t sample_stride,
                      double* G, const double* bcal, const double* twiddle, cudaStream_t s);
// Real-valued variants: samples are 8B^3 reals per function (psi-order); the ring
// pair (j', 2B-1-j') is packed into one complex FFT and only m >= 0 is kept.
int launch_az_forward_real(const Geo& g, const double* samples, size_t sample_stride, double* G,
                           const double* bcal, const double* twiddle, cudaStream_t s);
int launch_az_inverse_real(const Geo& g, const double* G, double* samples, size_t sample_stride,
                           const double* twiddle, cudaStream_t s);
// Azimuthal stage (inverse): unfold E/O, zero Nyquist bin, FFT sign +1 without
// 1/N (kernels.cpp:491), write psi-order rings.
int launch_az_inverse(const Geo& g, const double* G, double* samples, size_t sample_stride,
                      const double* twiddle, cudaStream_t s);

// Window of the nu-major intermediate S[nu][f][i] a Legendre call touches: the
// g.SC shells of the G chunk are shells [i0, i0 + g.SC) of an S with `sc`
// shells per function and NB = batch * sc * 2 reals per nu row.
struct SView {
    long long NB;
    int sc;
    int i0;
};

// --- addressing of the Legendre problems (device)
// Index math inside one call's G, S and coefficient arrays is 32-bit: the host
// keeps every array a GEMM touches below 2^31 doubles (batch_chunk).
__device__ __forceinline__ int s_col(const Geo& g, const SView& sv, int am, int n) {
    const int NB = (int)g.NB;
    const int sgn = n >= NB;
    const int nn = n - (sgn ? NB : 0);
    const int f = g.batch == 1 ? 0 : nn / (2 * g.SC), rem = nn - f * 2 * g.SC;  // no division for one function
    return (sgn ? -am : am) * (int)sv.NB + f * 2 * sv.sc + 2 * sv.i0 + rem;
}

// Real offset of column n of a Legendre problem inside the blocked G (the row
// part, j' * row stride, is separate): n = (sgn, flat shell s, re/im).
__device__ __forceinline__ int g_col(const Geo& g, int p, int am, int n) {
    const int NB = (int)g.NB;
    const int sgn = n >= NB;
    const int nn = n - (sgn ? NB : 0);
    const int s = nn >> 1;
    const int bin = sgn ? 2 * g.B - am : am;
    const int gx = s >> g.lgib;
    const int sl = s & ((1 << g.lgib) - 1);
    return 2 * ((((gx * 2 + p) * g.nbins + bin) << g.lgib) + sl) + (nn & 1);
}
// Table offsets in closed form (no dependent global load at CTA start; the
// host tables' offset arrays, sgl_tables.cpp, hold the same values -- pinned by
// tests/test_tables_and_model.py): Legendre problem 2|m| + p starts after
// sum_{|m'| < |m|} (B - |m'|) rows plus, for p = 1, the (B - |m| + 1) / 2 rows of
// parity 0; radial degree l after sum_{l' < l} (B - l') rows of 2B.
__device__ __forceinline__ int leg_table_off(int B, int pid) {
    const int am = pid >> 1, p = pid & 1;
    return (B + (B & 1)) * (am * B - am * (am - 1) / 2 + p * ((B - am + 1) / 2));
}
__device__ __forceinline__ int rad_table_off(int B, int l) { return 2 * B * (l * B - l * (l - 1) / 2); }
__device__ __forceinline__ int g_rowstride(const Geo& g) { return (2 * (int)g.ngx * 2 * g.nbins) << g.lgib; }

// Polar stage: per (|m|, parity) DMMA contraction against the normalized
// Legendre table.  tab: rows Pbar_{l,|m|}(cos theta_j'), j' < B.
int launch_legendre_forward(const Geo& g, const SView& sv, const double* G, double* S, const double* tab,
                            const long long* tab_off, const TileMap* tiles, int ntiles,
                            cudaStream_t s);
int launch_legendre_inverse(const Geo& g, const SView& sv, const double* S, double* G, const double* tab,
                            const long long* tab_off, const TileMap* tiles, int ntiles,
                            cudaStream_t s);

// The whole spherical forward (azimuthal FFT + Legendre contraction) as ONE
// persistent launch over shell slices of `slice_shells` (<= 32) shells: the
// Legendre tiles of a slice (a straddling tile map from the host, tiles_per_slice
// entries) overlap the FFTs of the next slice and read its G block from L2.
// counters: 1 + 2 * nslices ints of device scratch (zeroed by the launcher).
// grid <= 0: one CTA per resident slot.  Returns -2 if the shape is unsupported.
int launch_spherical_forward_fused(const Geo& g, const double* X, size_t sample_stride, double* G, const double* bcal,
                                   const double* tw, double* S, const SView& sv, const double* tab,
                                   const long long* tab_off, const TileMap* tiles, int tiles_per_slice,
                                   int slice_shells, int* counters, bool discard, int grid, cudaStream_t s);

// Radial stage: per l DMMA contraction against W_l (forward) / V_l (inverse).
// S is read/written as shell blocks (see ShellBlocks in sgl_kernels.cu); for the
// single-GPU transform rb = {2B, 0, 0} and g.SC = 2B.
struct RadialBlocks {
    int sc_blk;
    long long blk_stride;
    long long nu0;
};
// ... and the Legendre forward (legfwd_wp_kernel; the tile builder then emits n-block
// sequences, TileMap::seq > 1, which select it in launch_legendre_forward).
bool legfwd_wp_ok(const Geo& g);
// Does the radial forward of this geometry run on the warp-private kernel
// (radfwd_wp_kernel: batched small bandlimits)?  The tile builder then emits n-block
// sequences of 32 x 128 tiles (TileMap::seq > 1), which select that kernel.
bool radfwd_wp_ok(const Geo& g, const RadialBlocks& rb);
// Peer destinations for the multi-GPU exchange fused into a stage's epilogue
// (NVLink peer stores instead of an all-to-all): output row r goes to base[q]
// for the q with bound[q] <= key(r) < bound[q + 1] (key: l for the Legendre
// forward, the shell for the radial inverse).  n = 0: the plain output pointer.
constexpr int kMaxPeers = 8;
struct PeerDest {
    int n = 0;
    int bound[kMaxPeers + 1] = {};
    double* base[kMaxPeers] = {};
};

// Legendre forward whose S rows go straight to their owners' shell blocks.
int launch_legendre_forward_peers(const Geo& g, const SView& sv, const double* G, const PeerDest& pd,
                                  const double* tab, const long long* tab_off, const TileMap* tiles, int ntiles,
                                  cudaStream_t s);
// Radial forward whose coefficients go to every destination (pd.base[q], pd.n of them).
int launch_radial_forward_bcast(const Geo& g, const RadialBlocks& rb, const double* S, const PeerDest& pd,
                                const double* W, const long long* w_off, const TileMap* tiles, int ntiles,
                                cudaStream_t s);
// Radial inverse whose shell blocks go straight to the shells' owners.
int launch_radial_inverse_peers(const Geo& g, const RadialBlocks& rb, const double* C, const PeerDest& pd,
                                const double* V, const long long* v_off, const TileMap* tiles, int ntiles,
                                cudaStream_t s);

int launch_radial_forward(const Geo& g, const RadialBlocks& rb, const double* S, double* C,
                          const double* W, const long long* w_off, const TileMap* tiles, int ntiles,
                          cudaStream_t s);
int launch_radial_inverse(const Geo& g, const RadialBlocks& rb, const double* C, double* S,
                          const double* V, const long long* v_off, const TileMap* tiles, int ntiles,
                          cudaStream_t s);

// Small bandlimits (sgl_small.cu): the whole transform of 2B <= 32 in one launch
// per direction (per-shell fusion of the three stages; the forward's radial sum
// reduced across a cluster of CTAs).  Strides in complex elements per function.
bool small_path_ok(int B);
int launch_small_inverse(int B, int batch, const double* C, long long c_stride, double* X, long long x_stride,
                         const double* leg, const double* V, const double* tw, cudaStream_t s);
int launch_small_forward(int B, int batch, const double* X, long long x_stride, double* C, long long c_stride,
                         const double* leg, const double* W, const double* bcal, const double* tw, cudaStream_t s);

// On-device cross-oracle (sgl_separated.cu): the reference's separated transforms
// with closed-form basis values, direct quadratures, no tables.  shells: scratch
// of batch * 2B * B^2 complex.  r, a_mod: the radial rule (2B each).
int launch_separated_forward(int B, int batch, const double* samples, double* coeffs, double* shells,
                             const double* r, const double* a_mod, const double* bcal, cudaStream_t s);
int launch_separated_inverse(int B, int batch, const double* coeffs, double* samples, double* shells,
                             const double* r, cudaStream_t s);

// The reference's naive O(B^7) rung (sgl_transform.cpp:122-187) and
// sample_sgl_basis (:368-389) with normalized closed-form basis values.
int launch_naive_forward(int B, int batch, const double* samples, double* coeffs, const double* r,
                         const double* a_mod, const double* bcal, cudaStream_t s);
int launch_naive_inverse(int B, int batch, const double* coeffs, double* samples, const double* r, cudaStream_t s);
int launch_sample_basis(int B, int n, int l, int m, double* samples, const double* r, cudaStream_t s);

}  // namespace sglk
