// Reference-style tests through the C++ mirror of the reference API
// (include/sgl_b200/sgl_transform.hpp), i.e. the drop-in surface a caller of
// sgl::fsglft / sgl::ifsglft links against.  Cases restate
// /root/reference/proj/tests/test_sgl_transform.cpp (cited per case).  Needs a
// GPU; the CPU oracle is not involved -- expectations are closed-form.
// Prints one "[PASS]/[FAIL] name detail" line per case; exit code = #failures.
#include <cmath>
#include <complex>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>

#include "sgl_b200/sgl_transform.hpp"

using namespace sgl;

static int failures = 0;
static void report(bool ok, const char* name, const std::string& detail) {
    std::printf("[%s] %s %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
    if (!ok) ++failures;
}

static cvector random_complex(std::size_t n, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    cvector v(n);
    for (auto& x : v) x = {dist(rng), dist(rng)};
    return v;
}

int main() {
    // fast roundtrip identity over a range of bandlimits (test_sgl_transform.cpp:193-203)
    {
        double worst = 0.0;
        for (int B : {2, 4, 8, 16, 32}) {
            const auto plan = TransformPlan::compute(B);
            SglCoefficients c{B, random_complex(coefficient_count(B), 500 + B)};
            const auto grid = ifsglft(c, plan, 2);
            const auto back = fsglft(grid, plan, 2);
            const auto err = roundtrip_error(c.values, back.values);
            worst = std::max(worst, err.max_abs);
            if (err.nonfinite || err.skipped_zero) worst = 1.0;
        }
        report(worst < 1e-10, "fast roundtrip B<=32", "max_abs=" + std::to_string(worst));
    }
    // inverse of the unit coefficient omega(1,0,0) is pi^{-3/4} everywhere (:127-146)
    {
        const auto plan = TransformPlan::compute(2);
        SglCoefficients unit{2, cvector(coefficient_count(2), 0.0)};
        unit.values[0] = 1.0;
        const auto g = ifsglft(unit, plan);
        double worst = 0.0;
        for (const auto& v : g.values) worst = std::max(worst, std::abs(v - std::pow(M_PI, -0.75)));
        report(worst < 1e-12, "unit coefficient -> pi^-3/4", std::to_string(worst));
    }
    // zero maps to zero (:216-236)
    {
        const auto plan = TransformPlan::compute(2);
        SampleGrid zg{2, cvector(sample_count(2), 0.0)};
        SglCoefficients zc{2, cvector(coefficient_count(2), 0.0)};
        bool ok = true;
        for (const auto& v : fsglft(zg, plan).values) ok = ok && std::abs(v) == 0.0;
        for (const auto& v : ifsglft(zc, plan).values) ok = ok && std::abs(v) == 0.0;
        report(ok, "zero -> zero", "");
    }
    // linearity (:238-255)
    {
        const auto plan = TransformPlan::compute(4);
        SampleGrid g1{4, random_complex(sample_count(4), 41)}, g2{4, random_complex(sample_count(4), 42)};
        const cplx alpha(1.4, -0.3);
        SampleGrid mix{4, cvector(g1.values.size())};
        for (std::size_t i = 0; i < mix.values.size(); ++i) mix.values[i] = alpha * g1.values[i] + g2.values[i];
        const auto f1 = fsglft(g1, plan), f2 = fsglft(g2, plan), fm = fsglft(mix, plan);
        double worst = 0.0;
        for (std::size_t w = 0; w < fm.values.size(); ++w)
            worst = std::max(worst, std::abs(fm.values[w] - (alpha * f1.values[w] + f2.values[w])));
        report(worst < 1e-11, "linearity", std::to_string(worst));
    }
    // Parseval (:257-279)
    {
        double worst = 0.0;
        for (int B : {2, 4, 8}) {
            const auto plan = TransformPlan::compute(B);
            SglCoefficients c{B, random_complex(coefficient_count(B), 600 + B)};
            const auto grid = ifsglft(c, plan, 2);
            double gn = 0.0, cn = 0.0;
            for (int i = 0; i < 2 * B; ++i) {
                const double wr = plan.radial.a[i] * plan.radial.r[i] * plan.radial.r[i];
                for (int j = 0; j < 2 * B; ++j)
                    for (int k = 0; k < 2 * B; ++k)
                        gn += wr * plan.sphere.rule.b_cal[j] * std::norm(grid.values[psi_index(i, j, k, B)]);
            }
            for (const auto& v : c.values) cn += std::norm(v);
            worst = std::max(worst, std::abs(gn / cn - 1.0));
        }
        report(worst < 1e-9, "Parseval", std::to_string(worst));
    }
    // results independent of `threads` (:348-371) -- bitwise
    {
        const auto plan = TransformPlan::compute(4);
        SampleGrid g{4, random_complex(sample_count(4), 77)};
        const auto c1 = fsglft(g, plan, 1), c4 = fsglft(g, plan, 4);
        bool ok = true;
        for (std::size_t w = 0; w < c1.values.size(); ++w) ok = ok && c1.values[w] == c4.values[w];
        report(ok, "bitwise thread-count independence", "");
    }
    // size and bandlimit mismatches are rejected with the reference's messages (:405-415)
    {
        const auto plan = TransformPlan::compute(2);
        bool ok = false;
        try {
            SampleGrid bad{2, cvector(10)};
            fsglft(bad, plan);
        } catch (const std::invalid_argument& e) {
            ok = std::string(e.what()) == "transform: sample grid must have length 8B^3";
        }
        bool ok2 = false;
        try {
            SglCoefficients wrongB{3, cvector(coefficient_count(3))};
            ifsglft(wrongB, plan);
        } catch (const std::invalid_argument& e) {
            ok2 = std::string(e.what()) == "transform: coefficient and plan bandlimits disagree";
        }
        report(ok && ok2, "shape errors", "");
    }
    // fast == separated (the oracle chain, :148-174; here the separated rung runs on the device)
    {
        const auto plan = TransformPlan::compute(8);
        SampleGrid g{8, random_complex(sample_count(8), 88)};
        const auto f = fsglft(g, plan), s = dsglft_separated(g, plan);
        double num = 0.0, den = 0.0;
        for (std::size_t w = 0; w < f.values.size(); ++w) {
            num = std::max(num, std::abs(f.values[w] - s.values[w]));
            den = std::max(den, std::abs(s.values[w]));
        }
        report(num / den < 1e-12, "fast == separated (device)", std::to_string(num / den));
    }
    // B = 128: valid where the reference's M_lm underflows
    {
        const auto plan = TransformPlan::compute(128);
        SglCoefficients c{128, random_complex(coefficient_count(128), 128)};
        const auto grid = ifsglft(c, plan);
        const auto back = fsglft(grid, plan);
        const auto err = roundtrip_error(c.values, back.values);
        report(err.nonfinite == 0 && err.max_abs < 1e-11, "roundtrip B=128", "max_abs=" + std::to_string(err.max_abs));
    }
    std::printf("%d failure(s)\n", failures);
    return failures;
}
