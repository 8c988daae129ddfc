// Mirror of /root/reference/proj/core/include/sgl/quadrature.hpp:13-58.
//
// The half-range Hermite rule is not generated at run time here: the library
// reads the order-2B rules that paper_1604_05140_b200/tables/gen_radial_rules.py
// computed with the reference's extended-precision algorithm
// (quadrature.cpp:30-227, mpmath instead of boost::multiprecision) and stored
// as SGLT kind-1 files ($SGL_TABLES, else the tables/ directory next to
// libsglb200.so).  That lifts the reference's order cap of 128 (B <= 64) to 512.
#pragma once

#include <stdexcept>
#include <vector>

namespace sgl {

/// quadrature.hpp:13-20: equiangular rule of order L; b_cal = (pi / L) b_raw.
struct SphericalRule {
    int order = 0;
    std::vector<double> theta;
    std::vector<double> phi;
    std::vector<double> b_raw;
    std::vector<double> b_cal;
};

/// quadrature.hpp:27-32: order-N rule for e^{-r^2} on [0, inf);
/// a_mod = a e^{r^2} r^2.
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

/// Largest tabulated half-range Hermite order (B = 256); the reference's is 128.
inline constexpr int kMaxRadialOrder = 512;

SphericalRule sphere_rule(int L);
/// The tabulated rule of order N (N even); QuadratureError if it is absent.
RadialRule half_range_hermite_rule(int N);
/// a_mod recomputed from (r, a) in log space: exp(log a + r^2 + 2 log r).
std::vector<double> modified_radial_weights(const RadialRule& rule);
/// Gamma((k+1)/2) / 2.
double half_range_hermite_moment(int k);

}  // namespace sgl
