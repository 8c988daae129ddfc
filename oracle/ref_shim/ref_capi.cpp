// Test infrastructure only: a flat C ABI over the UNMODIFIED reference
// library (compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libsglref.so) so that pytest, the golden-vector script and
// bench.py's reference arm can call the reference's own fsglft / ifsglft
// (sgl_transform.hpp:71-76) and its oracle rungs without a C++ binding layer.
// Never linked into the product.
#include <algorithm>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "sgl/indexing.hpp"
#include "sgl/precompute_store.hpp"
#include "sgl/radial_transform.hpp"
#include "sgl/sgl_transform.hpp"
#include "sgl/spherical_transform.hpp"

using namespace sgl;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

cvector to_cvec(const double* p, std::size_t n) {
    cvector v(n);
    std::memcpy(v.data(), p, n * sizeof(cplx));
    return v;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_plan_create(int B) {
    TransformPlan* out = nullptr;
    guard([&] { out = new TransformPlan(TransformPlan::compute(B)); });
    return out;
}

void ref_plan_destroy(void* p) { delete static_cast<TransformPlan*>(p); }

// The reference's own SGLT writers for the plan-table kinds 1-3
// (precompute_store.cpp:160-194): the radial rule the plan was built with, the
// closed-form spherical rule and LegendreDctTable::build(B).
int ref_save_tables(void* p, const char* dir) {
    return guard([&] {
        const auto* plan = static_cast<TransformPlan*>(p);
        const int B = plan->bandlimit;
        const std::filesystem::path d(dir);
        store::save_radial_rule(plan->radial, d / store::radial_rule_filename(B));
        store::save_spherical_rule(sphere_rule(B), d / store::spherical_rule_filename(B));
        store::save_legendre_table(LegendreDctTable::build(B), d / store::legendre_table_filename(B));
    });
}

int ref_plan_arrays(void* p, double* r, double* a, double* a_mod, double* theta, double* phi,
                    double* b_cal, double* exp_neg_r2, double* m_norm) {
    return guard([&] {
        const auto& plan = *static_cast<TransformPlan*>(p);
        const int n = 2 * plan.bandlimit;
        std::copy_n(plan.radial.r.data(), n, r);
        std::copy_n(plan.radial.a.data(), n, a);
        std::copy_n(plan.radial.a_mod.data(), n, a_mod);
        std::copy_n(plan.sphere.rule.theta.data(), n, theta);
        std::copy_n(plan.sphere.rule.phi.data(), n, phi);
        std::copy_n(plan.sphere.rule.b_cal.data(), n, b_cal);
        std::copy_n(plan.exp_neg_r2.data(), n, exp_neg_r2);
        std::copy_n(plan.m_norm.data(), plan.m_norm.size(), m_norm);
    });
}

// variant: 0 fast (fsglft), 1 separated, 2 naive
int ref_forward(void* p, int variant, const double* grid, double* coeffs, unsigned threads) {
    return guard([&] {
        const auto& plan = *static_cast<TransformPlan*>(p);
        SampleGrid g;
        g.bandlimit = plan.bandlimit;
        g.values = to_cvec(grid, sample_count(plan.bandlimit));
        SglCoefficients c = variant == 0   ? fsglft(g, plan, threads)
                            : variant == 1 ? dsglft_separated(g, plan, threads)
                                           : dsglft_naive(g, plan, threads);
        std::memcpy(coeffs, c.values.data(), c.values.size() * sizeof(cplx));
    });
}

int ref_inverse(void* p, int variant, const double* coeffs, double* grid, unsigned threads) {
    return guard([&] {
        const auto& plan = *static_cast<TransformPlan*>(p);
        SglCoefficients c;
        c.bandlimit = plan.bandlimit;
        c.values = to_cvec(coeffs, coefficient_count(plan.bandlimit));
        SampleGrid g = variant == 0   ? ifsglft(c, plan, threads)
                       : variant == 1 ? idsglft_separated(c, plan, threads)
                                      : idsglft_naive(c, plan, threads);
        std::memcpy(grid, g.values.data(), g.values.size() * sizeof(cplx));
    });
}

// Batched round trip (inverse then forward) with an outer pool of `pool`
// threads and threads=1 per transform -- the protocol SURVEY.md section 6 used.
int ref_roundtrip_batch(void* p, const double* coeffs, double* back, int batch, int pool) {
    return guard([&] {
        const auto& plan = *static_cast<TransformPlan*>(p);
        const std::size_t omega = coefficient_count(plan.bandlimit);
        pool = std::max(1, std::min(pool, batch));
        std::vector<std::thread> workers;
        std::vector<std::string> errs(pool);
        for (int t = 0; t < pool; ++t) {
            workers.emplace_back([&, t] {
                try {
                    for (int b = t; b < batch; b += pool) {
                        SglCoefficients c;
                        c.bandlimit = plan.bandlimit;
                        c.values = to_cvec(coeffs + 2 * omega * b, omega);
                        const auto g = ifsglft(c, plan, 1);
                        const auto f = fsglft(g, plan, 1);
                        std::memcpy(back + 2 * omega * b, f.values.data(), omega * sizeof(cplx));
                    }
                } catch (const std::exception& e) {
                    errs[t] = e.what();
                }
            });
        }
        for (auto& w : workers) w.join();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
    });
}

int ref_sample_basis(void* p, int n, int l, int m, double* grid) {
    return guard([&] {
        const auto g = sample_sgl_basis(n, l, m, *static_cast<TransformPlan*>(p));
        std::memcpy(grid, g.values.data(), g.values.size() * sizeof(cplx));
    });
}

int ref_sft_forward(void* p, const double* samples, double* out) {
    return guard([&] {
        const auto& plan = *static_cast<TransformPlan*>(p);
        const int B = plan.bandlimit;
        const auto in = to_cvec(samples, 4 * static_cast<std::size_t>(B) * B);
        cvector o(static_cast<std::size_t>(B) * B);
        sft_seminaive_forward_into(in, plan.sphere, o);
        std::memcpy(out, o.data(), o.size() * sizeof(cplx));
    });
}

int ref_sft_inverse(void* p, const double* coeffs, double* out) {
    return guard([&] {
        const auto& plan = *static_cast<TransformPlan*>(p);
        const int B = plan.bandlimit;
        const auto in = to_cvec(coeffs, static_cast<std::size_t>(B) * B);
        cvector o(4 * static_cast<std::size_t>(B) * B);
        sft_seminaive_inverse_into(in, plan.sphere, o);
        std::memcpy(out, o.data(), o.size() * sizeof(cplx));
    });
}

int ref_drt_forward(void* p, int l, const double* s, double* out) {
    return guard([&] {
        const auto& plan = *static_cast<TransformPlan*>(p);
        const int B = plan.bandlimit;
        const auto in = to_cvec(s, 2 * static_cast<std::size_t>(B));
        cvector o(static_cast<std::size_t>(B - l));
        drt_forward(l, B, plan.radial, in, o);
        std::memcpy(out, o.data(), o.size() * sizeof(cplx));
    });
}

int ref_drt_inverse(void* p, int l, const double* t, double* out) {
    return guard([&] {
        const auto& plan = *static_cast<TransformPlan*>(p);
        const int B = plan.bandlimit;
        const auto in = to_cvec(t, static_cast<std::size_t>(B - l));
        cvector o(2 * static_cast<std::size_t>(B));
        drt_inverse(l, B, plan.radial, in, o);
        std::memcpy(out, o.data(), o.size() * sizeof(cplx));
    });
}

}  // extern "C"
