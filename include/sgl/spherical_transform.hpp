// Mirror of the plan types of /root/reference/proj/core/include/sgl/
// spherical_transform.hpp:10-49.  The reference's per-shell CPU stage
// functions (sft_*) have no counterpart: on the GPU the spherical stage is the
// azimuthal FFT kernel plus one grouped DMMA contraction over all shells
// (sglgpu_spherical_forward / _inverse in sglgpu.h).
#pragma once

#include <vector>

#include "sgl/quadrature.hpp"
#include "sgl/types.hpp"

namespace sgl {

/// spherical_transform.hpp:13-16
struct SphericalCoefficients {
    int order = 0;
    cvector values;
};

/// spherical_transform.hpp:27-32: row nu(l, m) = the leading l+1 entries of
/// the orthonormal DCT-II (even |m|) / DST-II (odd |m|) of
/// (M_lm P_lm(cos theta_j))_j, sign-folded for odd negative m.  The GPU path
/// does not consume it (it contracts against its own fully normalized
/// P-bar table, which stays finite where M_lm underflows); TransformPlan
/// carries it for API parity and validates its order.
struct LegendreDctTable {
    int order = 0;
    std::vector<std::vector<double>> rows;

    /// Builds the rows (host, long double, fully normalized recurrence: valid at
    /// every order, unlike the reference's unnormalized seed).
    static LegendreDctTable build(int L);
};

/// spherical_transform.hpp:35-49 without the CPU DCT / DFT plans.
struct SftPlan {
    int order = 0;
    SphericalRule rule;
    LegendreDctTable table;  // rows empty unless supplied (assemble) or built

    static SftPlan build(int L);
    static SftPlan assemble(SphericalRule rule, LegendreDctTable table);
};

}  // namespace sgl
