// FP64 contractions on the B200 INT8 tensor cores (tcgen05.mma kind::i8): the
// fixed-point slicing ("Ozaki") scheme.  Declarations shared by sgl_ozaki.cu
// (kernels + table builders) and sgl_capi.cpp (plan tables, launches).
//
// Numbers.  Every fp64 operand row (table) / column (data) gets its own power-of-
// two scale 2^e (e = the largest frexp exponent along the contraction index K),
// and each value x becomes the 56-bit two's-complement integer
// X = trunc(x * 2^(55 - e)), |X| < 2^55, stored as 7 byte "digits"
// X = sum_i X_i 2^(8 (6 - i)) (X_0 signed, X_1..X_6 unsigned).  A contraction
// sum_k y_k x_k is then sum_{i,j} (sum_k Y_i[k] X_j[k]) 2^(8 (12 - i - j)): each
// (i, j) is one exact int8 x int8 -> int32 tensor-core GEMM, accumulated per
// level s = i + j in TMEM.  Levels s <= 6 (28 GEMMs per 32-deep K step) are kept;
// the dropped tail is below 2^-54 of |y|max |x|max K, and the operand truncation
// (2^-55 relative to each row / column maximum) is what bounds the error: ~1e-15
// to 1e-13 normwise against long-double references (prototype:
// tests/test_ozaki_model.py).  The epilogue folds the 7 int32 levels exactly into
// two int64 halves and one fp64 FMA.
#pragma once

#include <cstdint>
#include <vector>

#include "sgl_kernels.cuh"

namespace sglk {
namespace oz {

constexpr int kDigits = 7;  // bytes per fixed-point operand
constexpr int kMaxLevel = 6;
constexpr int kLevels = kMaxLevel + 1;
constexpr int kTileN = 64;      // data columns per tensor-core tile (7 levels x 64 = 448 TMEM columns)
constexpr int kTmemCols = 512;   // allocated per tile: two CTAs per SM take turns
constexpr int kTileM = 128;     // table rows per tile (UMMA M)

// Host-built table image for one grouped contraction: per (problem, m-tile) a
// contiguous block [digit][K/16][128 rows][16 bytes] -- the tcgen05 K-major
// no-swizzle canonical layout, so a CTA moves it with one bulk copy -- and the
// per-row scale exponents.
struct TableImage {
    std::vector<uint8_t> bytes;
    std::vector<long long> off;  // per (problem * mtiles + mt): byte offset, -1: empty problem
    std::vector<int> kpad;       // per problem: K rounded up to 32
    std::vector<int> rexp;       // per (problem * mtiles + mt) * 128 + row: frexp exponent of the row maximum
    std::vector<int> corr;       // per (problem * mtiles + mt) * 7 * 128 + digit * 128 + row: 128 * sum_k Y_digit[row][k]
    int mtiles = 1;
};

// Legendre inverse (D[j'][n] = sum_l Pbar_l(t_j') S[l][n] per (|m|, parity)):
// rows j' (M = B, 128 per m-tile), K = degrees l of the problem's parity.
TableImage build_leginv_image(int B, const std::vector<double>& legendre, const std::vector<long long>& legendre_off);

struct Unit {  // one CTA: n-tiles [nt0, nt0 + count) of (problem, m-tile, sign half)
    int pid, mt, half, nt0;
};

struct LegInvI8 {
    Geo g;
    SView sv;
    const double* S;
    double* G;
    const uint8_t* img;
    const long long* img_off;
    const int* rexp;
    const int* kpad;
    const Unit* units;
    int tpc;      // n-tiles per unit
    int mtiles;
    long long* trace = nullptr;  // experiments: per-CTA phase clocks [unit][tile < 8][phase < 8]
    const int* corr = nullptr;   // warp-specialised kernel: bias corrections (TableImage::corr)
    int* counter = nullptr;      // ... its unit ticket (zeroed by the launcher)
    int nunits = 0;
    int grid = 148;              // ... persistent CTAs (one per SM)
};

// Warp-specialised form (leginv_ws_kernel): 32-column tiles whose 7 data digit
// planes are stacked along N (224 rows), so ONE int8 MMA per table digit i
// covers all products (i, j <= 6 - i) -- 7 MMAs of N = 224 ... 32 per 32-deep
// k step instead of 28 of N = 32 -- landing in TMEM levels i .. 6 by the column
// offset i * 32; all data digits are unsigned (the top one biased by 128, undone by
// a per-row constant in the epilogue).  Two TMEM buffers (2 x 224 columns), two
// shared-memory stages: producers (8 warps), one MMA warp and 4 epilogue warps
// overlap.  One CTA per (problem, m-tile, sign half).
constexpr int kWsN = 32;
std::vector<Unit> leginv_ws_units(int B, long long NB, bool real);
size_t leginv_ws_smem(int B);
int launch_legendre_inverse_ws(const LegInvI8& prm, int nunits, cudaStream_t s);

// Host: the units of a Legendre-inverse launch (heaviest first) for NB reals per
// nu row of S; returns the unit count.
std::vector<Unit> leginv_units(int B, long long NB, bool real, int tpc);
size_t leginv_smem(int B);
int launch_legendre_inverse_i8(const LegInvI8& prm, int nunits, cudaStream_t s);

}  // namespace oz
}  // namespace sglk
