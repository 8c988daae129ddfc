// C++ mirror of the reference's sgl:: hot-path API on top of the sglgpu C ABI:
// the plan (sgl_transform.cpp:52-102) and the transforms.  See
// include/sgl/sgl_transform.hpp; the non-transform helpers are in sgl_host.cpp.
#include "sgl/sgl_transform.hpp"

#include "sgl/precompute_store.hpp"
#include "sgl/special_functions.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>

#include "sglgpu.h"

namespace sgl {

namespace {

// sgl_transform.cpp:18-25
void check_plan_grid(const SampleGrid& grid, const TransformPlan& plan) {
    if (grid.bandlimit != plan.bandlimit) {
        throw std::invalid_argument("transform: grid and plan bandlimits disagree");
    }
    if (grid.values.size() != sample_count(plan.bandlimit)) {
        throw std::invalid_argument("transform: sample grid must have length 8B^3");
    }
}

// sgl_transform.cpp:27-35
void check_plan_coeffs(const SglCoefficients& coeffs, const TransformPlan& plan) {
    if (coeffs.bandlimit != plan.bandlimit) {
        throw std::invalid_argument("transform: coefficient and plan bandlimits disagree");
    }
    if (coeffs.values.size() != coefficient_count(plan.bandlimit)) {
        throw std::invalid_argument("transform: coefficient vector must have length B(B+1)(2B+1)/6");
    }
}

void throw_status(int status) {
    if (status == SGLGPU_OK) return;
    const std::string msg = sglgpu_last_error();
    if (status == SGLGPU_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

std::mutex g_device_mu;

}  // namespace

// sgl_transform.cpp:52-88 (validation and the derived per-node / per-order vectors)
TransformPlan TransformPlan::assemble(int B, RadialRule radial, SphericalRule sphere, LegendreDctTable table) {
    if (B < 1) throw std::invalid_argument("TransformPlan: bandlimit must be positive");
    if (radial.order != 2 * B) throw std::invalid_argument("TransformPlan: radial rule order must be 2B");
    if (sphere.order != B || table.order != B)
        throw std::invalid_argument("TransformPlan: spherical tables must have order B");
    TransformPlan plan;
    plan.bandlimit = B;
    plan.radial = std::move(radial);
    plan.sphere = SftPlan::assemble(std::move(sphere), std::move(table));
    plan.exp_neg_r2.resize(plan.radial.r.size());
    for (std::size_t i = 0; i < plan.radial.r.size(); ++i)
        plan.exp_neg_r2[i] = std::exp(-plan.radial.r[i] * plan.radial.r[i]);
    plan.cos_theta.resize(plan.sphere.rule.theta.size());
    for (std::size_t j = 0; j < plan.cos_theta.size(); ++j) plan.cos_theta[j] = std::cos(plan.sphere.rule.theta[j]);
    plan.seed_norm.resize(B);
    for (int l = 0; l < B; ++l) plan.seed_norm[l] = std::sqrt(2.0 * std::exp(-std::lgamma(l + 1.5)));
    plan.m_norm.resize(static_cast<std::size_t>(B) * B);
    for (int l = 0; l < B; ++l) {
        for (int m = -l; m <= l; ++m) {
            const int am = std::abs(m);
            const double sign = (m < 0 && am % 2 != 0) ? -1.0 : 1.0;
            plan.m_norm[static_cast<std::size_t>(nu_index(l, m))] = sign * sph_harm_norm(l, am);
        }
    }
    return plan;
}

TransformPlan TransformPlan::assemble(int B, RadialRule radial, SphericalRule sphere) {
    LegendreDctTable table;  // order only: the GPU contracts against its own normalized table
    table.order = B;
    return assemble(B, std::move(radial), std::move(sphere), std::move(table));
}

TransformPlan TransformPlan::compute(int B) {
    if (B < 1) throw std::invalid_argument("TransformPlan: bandlimit must be positive");
    return assemble(B, half_range_hermite_rule(2 * B), sphere_rule(B));
}

// sgl_transform.cpp:98-102: kinds 1, 2 and 3 from `dir`.  A directory holding
// only the radial rule (the packaged tables) is accepted too: the spherical rule
// is then the closed form and the DCT table is not materialized.
TransformPlan TransformPlan::from_tables(const std::filesystem::path& dir, int B) {
    auto radial = store::load_radial_rule(dir / store::radial_rule_filename(B));
    const auto sp = dir / store::spherical_rule_filename(B);
    const auto lt = dir / store::legendre_table_filename(B);
    auto sphere = std::filesystem::exists(sp) ? store::load_spherical_rule(sp) : sphere_rule(B);
    if (std::filesystem::exists(lt))
        return assemble(B, std::move(radial), std::move(sphere), store::load_legendre_table(lt));
    return assemble(B, std::move(radial), std::move(sphere));
}

sglgpu_plan* TransformPlan::device_plan() const {
    std::lock_guard<std::mutex> lock(g_device_mu);
    auto& slot = const_cast<std::shared_ptr<sglgpu_plan>&>(device);
    if (!slot) {
        sglgpu_plan_desc d{};
        d.bandlimit = bandlimit;
        d.r = radial.r.data();
        d.a_mod = radial.a_mod.data();
        d.b_cal = sphere.rule.b_cal.data();
        d.device = -1;
        sglgpu_plan* p = nullptr;
        throw_status(sglgpu_plan_create(&d, &p));
        slot = std::shared_ptr<sglgpu_plan>(p, [](sglgpu_plan* q) { sglgpu_plan_destroy(q); });
    }
    return slot.get();
}

SglCoefficients fsglft(const SampleGrid& grid, const TransformPlan& plan, unsigned /*threads*/) {
    check_plan_grid(grid, plan);
    SglCoefficients out;
    out.bandlimit = plan.bandlimit;
    out.values.assign(coefficient_count(plan.bandlimit), cplx(0.0));
    throw_status(sglgpu_forward(plan.device_plan(), reinterpret_cast<const double*>(grid.values.data()),
                                reinterpret_cast<double*>(out.values.data()), 1, SGLGPU_MEM_HOST, nullptr));
    return out;
}

SampleGrid ifsglft(const SglCoefficients& coeffs, const TransformPlan& plan, unsigned /*threads*/) {
    check_plan_coeffs(coeffs, plan);
    SampleGrid out;
    out.bandlimit = plan.bandlimit;
    out.values.assign(sample_count(plan.bandlimit), cplx(0.0));
    throw_status(sglgpu_inverse(plan.device_plan(), reinterpret_cast<const double*>(coeffs.values.data()),
                                reinterpret_cast<double*>(out.values.data()), 1, SGLGPU_MEM_HOST, nullptr));
    return out;
}

SglCoefficients dsglft_separated(const SampleGrid& grid, const TransformPlan& plan, unsigned /*threads*/) {
    check_plan_grid(grid, plan);
    SglCoefficients out;
    out.bandlimit = plan.bandlimit;
    out.values.assign(coefficient_count(plan.bandlimit), cplx(0.0));
    throw_status(sglgpu_forward_separated(plan.device_plan(), reinterpret_cast<const double*>(grid.values.data()),
                                          reinterpret_cast<double*>(out.values.data()), 1, SGLGPU_MEM_HOST, nullptr));
    return out;
}

SampleGrid idsglft_separated(const SglCoefficients& coeffs, const TransformPlan& plan, unsigned /*threads*/) {
    check_plan_coeffs(coeffs, plan);
    SampleGrid out;
    out.bandlimit = plan.bandlimit;
    out.values.assign(sample_count(plan.bandlimit), cplx(0.0));
    throw_status(sglgpu_inverse_separated(plan.device_plan(), reinterpret_cast<const double*>(coeffs.values.data()),
                                          reinterpret_cast<double*>(out.values.data()), 1, SGLGPU_MEM_HOST,
                                          nullptr));
    return out;
}

SglCoefficients dsglft_naive(const SampleGrid& grid, const TransformPlan& plan, unsigned /*threads*/) {
    check_plan_grid(grid, plan);
    SglCoefficients out;
    out.bandlimit = plan.bandlimit;
    out.values.assign(coefficient_count(plan.bandlimit), cplx(0.0));
    throw_status(sglgpu_forward_naive(plan.device_plan(), reinterpret_cast<const double*>(grid.values.data()),
                                      reinterpret_cast<double*>(out.values.data()), 1, SGLGPU_MEM_HOST, nullptr));
    return out;
}

SampleGrid idsglft_naive(const SglCoefficients& coeffs, const TransformPlan& plan, unsigned /*threads*/) {
    check_plan_coeffs(coeffs, plan);
    SampleGrid out;
    out.bandlimit = plan.bandlimit;
    out.values.assign(sample_count(plan.bandlimit), cplx(0.0));
    throw_status(sglgpu_inverse_naive(plan.device_plan(), reinterpret_cast<const double*>(coeffs.values.data()),
                                      reinterpret_cast<double*>(out.values.data()), 1, SGLGPU_MEM_HOST, nullptr));
    return out;
}

// sgl_transform.cpp:368-389 (range check and message first, as the reference)
SampleGrid sample_sgl_basis(int n, int l, int m, const TransformPlan& plan) {
    const int B = plan.bandlimit;
    if (n < 1 || n > B || l < 0 || l >= n || std::abs(m) > l)
        throw std::invalid_argument("sample_sgl_basis: invalid (n, l, m) for this plan");
    SampleGrid out;
    out.bandlimit = B;
    out.values.assign(sample_count(B), cplx(0.0));
    throw_status(sglgpu_sample_basis(plan.device_plan(), n, l, m, reinterpret_cast<double*>(out.values.data()),
                                     SGLGPU_MEM_HOST, nullptr));
    return out;
}

void fsglft_batch(const TransformPlan& plan, const cplx* samples, cplx* coeffs, std::size_t batch,
                  bool device_pointers, void* stream) {
    throw_status(sglgpu_forward(plan.device_plan(), reinterpret_cast<const double*>(samples),
                                reinterpret_cast<double*>(coeffs), batch,
                                device_pointers ? SGLGPU_MEM_DEVICE : SGLGPU_MEM_HOST, stream));
}

void ifsglft_batch(const TransformPlan& plan, const cplx* coeffs, cplx* samples, std::size_t batch,
                   bool device_pointers, void* stream) {
    throw_status(sglgpu_inverse(plan.device_plan(), reinterpret_cast<const double*>(coeffs),
                                reinterpret_cast<double*>(samples), batch,
                                device_pointers ? SGLGPU_MEM_DEVICE : SGLGPU_MEM_HOST, stream));
}

// sgl_transform.cpp:350-366
RoundtripError roundtrip_error(std::span<const cplx> reference, std::span<const cplx> actual) {
    if (reference.size() != actual.size()) throw std::invalid_argument("roundtrip_error: vector lengths disagree");
    RoundtripError err;
    for (std::size_t i = 0; i < reference.size(); ++i) {
        if (!std::isfinite(actual[i].real()) || !std::isfinite(actual[i].imag())) ++err.nonfinite;
        const double diff = std::abs(reference[i] - actual[i]);
        err.max_abs = std::max(err.max_abs, diff);
        const double mag = std::abs(reference[i]);
        if (mag == 0.0) {
            ++err.skipped_zero;
        } else {
            err.max_rel = std::max(err.max_rel, diff / mag);
        }
    }
    return err;
}

}  // namespace sgl
