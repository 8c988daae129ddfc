// Test infrastructure only (oracle/_ref build).  Replaces the one reference
// translation unit that cannot build here, proj/core/src/quadrature.cpp, which
// needs boost::multiprecision from the absent vendor/ tree
// (quadrature.cpp:3, proj/.gitignore:2).  Implements the four functions that
// proj/core/include/sgl/quadrature.hpp:45-58 declares:
//
//  * sphere_rule          closed form, restated from quadrature.cpp:189-211
//  * half_range_hermite_rule(N)
//                         loads the SGLT kind-1 file radial_rule_B{N/2}.sglt
//                         produced by paper_1604_05140_b200/tables/
//                         gen_radial_rules.py (same moment -> Chebyshev ->
//                         Golub-Welsch route in mpmath).  Directory from
//                         $SGL_RADIAL_DIR, else the compiled-in default.
//                         The reference's N <= 128 cap (quadrature.hpp:43,
//                         quadrature.cpp:217-222) is NOT enforced so that the
//                         reference can be run (and shown to fail) at B = 128.
//  * modified_radial_weights, half_range_hermite_moment
//                         one-liners restated from quadrature.cpp:229-242.
#include "sgl/quadrature.hpp"

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numbers>
#include <string>
#include <vector>

#ifndef SGL_RADIAL_DEFAULT_DIR
#define SGL_RADIAL_DEFAULT_DIR "/root/repo/paper_1604_05140_b200/tables"
#endif

namespace sgl {

SphericalRule sphere_rule(int L) {
    if (L < 1) {
        throw std::invalid_argument("sphere_rule: order must be positive");
    }
    const double pi = std::numbers::pi;
    SphericalRule rule;
    rule.order = L;
    const int count = 2 * L;
    rule.theta.resize(count);
    rule.phi.resize(count);
    rule.b_raw.resize(count);
    rule.b_cal.resize(count);
    for (int j = 0; j < count; ++j) {
        rule.theta[j] = (2 * j + 1) * pi / (4.0 * L);
        rule.phi[j] = j * pi / L;
        double acc = 0.0;
        for (int l = 0; l < L; ++l) {
            acc += std::sin((2 * j + 1) * (2 * l + 1) * pi / (4.0 * L)) / (2 * l + 1);
        }
        rule.b_raw[j] = std::sin((2 * j + 1) * pi / (4.0 * L)) * (2.0 / L) * acc;
        rule.b_cal[j] = pi / L * rule.b_raw[j];
    }
    return rule;
}

RadialRule half_range_hermite_rule(int N) {
    if (N < 1) {
        throw std::invalid_argument("half_range_hermite_rule: order must be positive");
    }
    if (N % 2 != 0) {
        throw QuadratureError("shim: only even orders 2B are tabulated");
    }
    const char* env = std::getenv("SGL_RADIAL_DIR");
    const std::string dir = env ? env : SGL_RADIAL_DEFAULT_DIR;
    const std::string path = dir + "/radial_rule_B" + std::to_string(N / 2) + ".sglt";
    std::ifstream in(path, std::ios::binary);
    if (!in) {
        throw QuadratureError("shim: missing radial rule table " + path);
    }
    char magic[4];
    std::uint32_t version = 0, B = 0;
    std::uint8_t kind = 0;
    in.read(magic, 4);
    in.read(reinterpret_cast<char*>(&version), 4);
    in.read(reinterpret_cast<char*>(&B), 4);
    in.read(reinterpret_cast<char*>(&kind), 1);
    if (std::memcmp(magic, "SGLT", 4) != 0 || version != 1 || kind != 1 ||
        B != static_cast<std::uint32_t>(N / 2)) {
        throw QuadratureError("shim: malformed radial rule table " + path);
    }
    std::vector<double> payload(3 * static_cast<std::size_t>(N));
    in.read(reinterpret_cast<char*>(payload.data()),
            static_cast<std::streamsize>(payload.size() * sizeof(double)));
    if (!in) {
        throw QuadratureError("shim: short radial rule table " + path);
    }
    RadialRule rule;
    rule.order = N;
    rule.r.assign(payload.begin(), payload.begin() + N);
    rule.a.assign(payload.begin() + N, payload.begin() + 2 * N);
    rule.a_mod.assign(payload.begin() + 2 * N, payload.end());
    return rule;
}

std::vector<double> modified_radial_weights(const RadialRule& rule) {
    std::vector<double> out(rule.r.size());
    for (std::size_t i = 0; i < rule.r.size(); ++i) {
        out[i] = std::exp(std::log(rule.a[i]) + rule.r[i] * rule.r[i] + 2.0 * std::log(rule.r[i]));
    }
    return out;
}

double half_range_hermite_moment(int k) {
    if (k < 0) {
        throw std::invalid_argument("half_range_hermite_moment: negative power");
    }
    return 0.5 * std::exp(std::lgamma((k + 1) / 2.0));
}

}  // namespace sgl
