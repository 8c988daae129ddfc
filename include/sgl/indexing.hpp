// Mirror of /root/reference/proj/core/include/sgl/indexing.hpp: the psi / nu /
// omega layouts every transform, file and kernel of this library uses
// (samples psi = 4B^2 i + 2B j + k, coefficients omega = n(n-1)(2n-1)/6 +
// l(l+1) + m).  Same range checks (std::out_of_range) as indexing.cpp:50-118.
#pragma once

#include <array>
#include <cstddef>
#include <utility>

namespace sgl {

struct Layout {
    int bandlimit;

    explicit Layout(int B);

    std::size_t sample_count() const;       // 8 B^3
    std::size_t coefficient_count() const;  // B (B+1) (2B+1) / 6
};

std::size_t sample_count(int B);
std::size_t coefficient_count(int B);

int mu_index(int j, int k, int B);
int psi_index(int i, int j, int k, int B);
int nu_index(int l, int m);
int omega_index(int n, int l, int m);

std::pair<int, int> mu_inverse(int mu, int B);
std::array<int, 3> psi_inverse(int psi, int B);
std::pair<int, int> nu_inverse(int nu);
std::array<int, 3> omega_inverse(int omega);

}  // namespace sgl
