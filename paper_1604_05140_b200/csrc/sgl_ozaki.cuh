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
};

// Host: the units of a Legendre-inverse launch (heaviest first) for NB reals per
// nu row of S; returns the unit count.
std::vector<Unit> leginv_units(int B, long long NB, bool real, int tpc);
size_t leginv_smem(int B);
int launch_legendre_inverse_i8(const LegInvI8& prm, int nunits, cudaStream_t s);

}  // namespace oz
}  // namespace sglk
