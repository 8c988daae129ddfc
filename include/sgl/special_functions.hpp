// Mirror of /root/reference/proj/core/include/sgl/special_functions.hpp:10-50:
// scalar closed forms of the SGL basis (host; test and diagnostic aids -- no
// transform uses them).  Evaluated with normalized recurrences in long double,
// so they stay finite where the reference's unnormalized seeds under/overflow.
#pragma once

#include <complex>

namespace sgl {

double assoc_legendre(int l, int m, double t);
double assoc_legendre_signed(int l, int m, double t);
double gen_laguerre(int k, double alpha, double t);
double sph_harm_norm(int l, int m);
std::complex<double> sph_harm(int l, int m, double theta, double phi);
double norm_const(int n, int l);
double radial_raw(int n, int l, double r);
double radial_normalized(int n, int l, double r);
double radial_normalized_decayed(int n, int l, double r);
std::complex<double> sgl_basis(int n, int l, int m, double r, double theta, double phi);

namespace detail {
double radial_from_seed(int n, int l, double r, double seed_value);
}  // namespace detail

}  // namespace sgl
