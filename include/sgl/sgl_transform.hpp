// C++ host API of the B200 SGL transform: a source-level drop-in for the
// reference's hot-path interface (/root/reference/proj/core/include/sgl/
// sgl_transform.hpp:15-89), implemented on the C ABI of include/sglgpu.h.
// Same header path (sgl/sgl_transform.hpp), names, data layouts (psi-order
// samples, omega-order coefficients, std::complex<double>) and exceptions with
// the same messages for shape errors (sgl_transform.cpp:18-35).
//
// Every transform runs on the GPU (sm_100a kernels); there is no CPU path:
//   fsglft / ifsglft                   the fast O(B^4) pair (the hot path)
//   dsglft_separated / idsglft_separated, dsglft_naive / idsglft_naive
//                                      the reference's oracle rungs, as
//                                      independent device kernels (closed-form
//                                      basis values, direct sums)
//   sample_sgl_basis                   H_nlm on the grid, a device kernel
// Differences (additive only):
//  * TransformPlan carries a shared handle to the device plan (tables uploaded
//    once, on first use, on the device current at that time).
//  * `threads` is accepted and ignored (the reference caps CPU workers with it;
//    results are bitwise independent of it in both implementations).
//  * Batched and device-pointer entry points.
#pragma once

#include <cstddef>
#include <filesystem>
#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

#include "sgl/indexing.hpp"
#include "sgl/quadrature.hpp"
#include "sgl/spherical_transform.hpp"
#include "sgl/types.hpp"

struct sglgpu_plan;

namespace sgl {

/// sgl_transform.hpp:15-19
struct SglCoefficients {
    int bandlimit = 0;
    cvector values;
};

/// sgl_transform.hpp:21-25
struct SampleGrid {
    int bandlimit = 0;
    cvector values;
};

/// sgl_transform.hpp:30-49
struct TransformPlan {
    int bandlimit = 0;
    RadialRule radial;               // order 2B
    SftPlan sphere;                  // order B
    std::vector<double> exp_neg_r2;  // e^{-r_i^2}
    std::vector<double> cos_theta;   // cos(theta_j)
    std::vector<double> seed_norm;   // sqrt(2/Gamma(l+3/2)), as the reference computes it
    std::vector<double> m_norm;      // M_lm per nu, sign-folded, as the reference computes it
    std::shared_ptr<sglgpu_plan> device;  // additive: the uploaded device plan

    /// Radial rule of order 2B from the packaged SGLT tables (quadrature.hpp);
    /// the Legendre DCT table is not materialized (the GPU builds its own).
    static TransformPlan compute(int B);
    /// Radial rule, spherical rule and Legendre DCT table from SGLT kinds 1, 2
    /// and 3 named as precompute_store.cpp:146-158 names them
    /// (sgl_transform.cpp:98-102).
    static TransformPlan from_tables(const std::filesystem::path& dir, int B);
    /// sgl_transform.cpp:52-88: validates the orders (messages included).
    static TransformPlan assemble(int B, RadialRule radial, SphericalRule sphere, LegendreDctTable table);
    /// Same, without a Legendre DCT table (additive).
    static TransformPlan assemble(int B, RadialRule radial, SphericalRule sphere);

    /// Creates (once) and returns the device plan on the current CUDA device.
    sglgpu_plan* device_plan() const;
};

/// O(B^7) direct sums (sgl_transform.cpp:122-187), on the device.  B <= 32.
SglCoefficients dsglft_naive(const SampleGrid& grid, const TransformPlan& plan, unsigned threads = 1);
SampleGrid idsglft_naive(const SglCoefficients& coeffs, const TransformPlan& plan, unsigned threads = 1);

/// O(B^6) separated transforms (sgl_transform.cpp:189-272), on the device.  B <= 64.
SglCoefficients dsglft_separated(const SampleGrid& grid, const TransformPlan& plan, unsigned threads = 1);
SampleGrid idsglft_separated(const SglCoefficients& coeffs, const TransformPlan& plan, unsigned threads = 1);

/// Fast SGL Fourier transform (sgl_transform.hpp:71-72).
SglCoefficients fsglft(const SampleGrid& grid, const TransformPlan& plan, unsigned threads = 1);
/// Fast inverse (sgl_transform.hpp:74-76).
SampleGrid ifsglft(const SglCoefficients& coeffs, const TransformPlan& plan, unsigned threads = 1);

/// Batched, host or device memory (see sglgpu.h for mem_kind).
void fsglft_batch(const TransformPlan& plan, const cplx* samples, cplx* coeffs, std::size_t batch,
                  bool device_pointers = false, void* stream = nullptr);
void ifsglft_batch(const TransformPlan& plan, const cplx* coeffs, cplx* samples, std::size_t batch,
                   bool device_pointers = false, void* stream = nullptr);

/// sgl_transform.hpp:78-84.  Same semantics as the reference; `nonfinite`
/// (additive) counts entries of `actual` that are NaN/Inf, which the reference's
/// std::max-based maxima silently skip.
struct RoundtripError {
    double max_abs = 0.0;
    double max_rel = 0.0;
    std::size_t skipped_zero = 0;
    std::size_t nonfinite = 0;
};
RoundtripError roundtrip_error(std::span<const cplx> reference, std::span<const cplx> actual);

/// Samples H_nlm on the plan's grid, psi-order (sgl_transform.hpp:87-89,
/// sgl_transform.cpp:368-389); a device kernel with normalized recurrences.
SampleGrid sample_sgl_basis(int n, int l, int m, const TransformPlan& plan);

}  // namespace sgl
