// C++ host API of the B200 SGL transform: a source-level mirror of the
// reference's hot-path interface (/root/reference/proj/core/include/sgl/
// sgl_transform.hpp:15-89, quadrature.hpp:13-32), implemented on the C ABI of
// include/sglgpu.h.  Same names, same data layouts (psi-order samples,
// omega-order coefficients, std::complex<double>), same exceptions with the same
// messages for shape errors (sgl_transform.cpp:18-35).
//
// Differences (additive only):
//  * TransformPlan carries a shared handle to the device plan (tables uploaded
//    once, on first use).  The reference's per-plan CPU tables (SftPlan's DCT
//    plans, LegendreDctTable) are not materialized; the GPU path generates its own
//    normalized tables.
//  * `threads` is accepted and ignored (the reference caps CPU workers with it;
//    results are bitwise independent of it in both implementations).
//  * Batched and device-pointer entry points.
#pragma once

#include <complex>
#include <cstddef>
#include <filesystem>
#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

struct sglgpu_plan;

namespace sgl {

using cplx = std::complex<double>;
using cvector = std::vector<cplx>;
using rvector = std::vector<double>;

/// quadrature.hpp:13-20
struct SphericalRule {
    int order = 0;
    std::vector<double> theta;
    std::vector<double> phi;
    std::vector<double> b_raw;
    std::vector<double> b_cal;
};

/// quadrature.hpp:27-32
struct RadialRule {
    int order = 0;
    std::vector<double> r;
    std::vector<double> a;
    std::vector<double> a_mod;
};

/// quadrature.hpp:36-38
struct QuadratureError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// The spherical part of the plan; the reference's SftPlan also holds CPU DCT /
/// DFT plans and the Legendre DCT table (spherical_transform.hpp:35-49).
struct SftPlan {
    int order = 0;
    SphericalRule rule;
};

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

    /// The radial rule of order 2B is read from the packaged SGLT tables
    /// ($SGL_TABLES, else the library's tables directory), which
    /// paper_1604_05140_b200/tables/gen_radial_rules.py generates with the
    /// reference's extended-precision algorithm (quadrature.cpp:133-227).
    static TransformPlan compute(int B);
    /// Radial rule (and, when present, the spherical rule) from SGLT files
    /// named as precompute_store.cpp:150-158 names them.
    static TransformPlan from_tables(const std::filesystem::path& dir, int B);
    static TransformPlan assemble(int B, RadialRule radial, SphericalRule sphere);

    /// Creates (once) and returns the device plan on the current CUDA device.
    sglgpu_plan* device_plan() const;
};

SphericalRule sphere_rule(int L);
RadialRule load_radial_rule(const std::filesystem::path& path);
SphericalRule load_spherical_rule(const std::filesystem::path& path);

/// Fast SGL Fourier transform (sgl_transform.hpp:71-72).
SglCoefficients fsglft(const SampleGrid& grid, const TransformPlan& plan, unsigned threads = 1);
/// Fast inverse (sgl_transform.hpp:74-76).
SampleGrid ifsglft(const SglCoefficients& coeffs, const TransformPlan& plan, unsigned threads = 1);

/// Separated transforms (sgl_transform.hpp, dsglft_separated / idsglft_separated;
/// sgl_transform.cpp:189-272) run on the device as a cross-oracle of the fast
/// path: closed-form basis values, direct quadratures.  B <= 64.
SglCoefficients dsglft_separated(const SampleGrid& grid, const TransformPlan& plan, unsigned threads = 1);
SampleGrid idsglft_separated(const SglCoefficients& coeffs, const TransformPlan& plan, unsigned threads = 1);

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

/// indexing.hpp:26-40
std::size_t sample_count(int B);
std::size_t coefficient_count(int B);
int psi_index(int i, int j, int k, int B);
int nu_index(int l, int m);
int omega_index(int n, int l, int m);

}  // namespace sgl
