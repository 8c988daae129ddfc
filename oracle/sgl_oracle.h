/* TEST INFRASTRUCTURE -- NOT THE PRODUCT.
 *
 * CPU restatement ("oracle") of the reference's fast SGL transform pair
 * sgl::fsglft / sgl::ifsglft (/root/reference/proj/core/src/sgl_transform.cpp:274-348)
 * in plain C.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker or the timed CPU
 * baseline.  The CUDA product never links or calls it.
 *
 * Same algorithm, layouts and stage order as the reference (seminaive spherical
 * transform with FFT + DCT/DST + truncated Legendre rows, then the discrete R
 * transform by three-term recurrence / Clenshaw).  Numerics changes only (see
 * sgl_oracle.c header): normalized Legendre seeding and log-space radial seeds
 * in long double, which keep the restatement valid at B = 128, 256 where the
 * reference underflows.
 *
 * Parity pin: tests/test_oracle.py checks this restatement against the
 * reference itself (oracle/_ref, compiled from /root/reference) and against the
 * committed golden vectors in tests/golden/ (made by tests/golden/make_golden.py).
 *
 * All complex arrays are interleaved fp64 (re, im), i.e. std::complex<double>.
 */
#ifndef SGL_ORACLE_H
#define SGL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_plan orc_plan;

/* r, a_mod: the order-2B half-range Hermite rule (quadrature.hpp:27-32). */
orc_plan* orc_plan_create(int B, const double* r, const double* a_mod);
void orc_plan_destroy(orc_plan* p);
int orc_plan_bandlimit(const orc_plan* p);

/* fsglft: psi-order grid (8B^3 complex) -> omega-order coefficients. */
int orc_fsglft(const orc_plan* p, const double* grid, double* coeffs, int threads);
/* ifsglft: omega-order coefficients -> psi-order grid. */
int orc_ifsglft(const orc_plan* p, const double* coeffs, double* grid, int threads);

/* Stage functions (the reference's public stage oracles). */
int orc_sft_forward(const orc_plan* p, const double* samples, double* out);  /* 4B^2 -> B^2 */
int orc_sft_inverse(const orc_plan* p, const double* coeffs, double* out);   /* B^2 -> 4B^2 */
int orc_drt_forward(const orc_plan* p, int l, const double* s, double* out); /* 2B -> B-l */
int orc_drt_inverse(const orc_plan* p, int l, const double* t, double* out); /* B-l -> 2B */

/* Sampled basis function H_nlm on the grid (sgl_transform.cpp:368-389). */
int orc_sample_basis(const orc_plan* p, int n, int l, int m, double* grid);

/* Closed-form basis value via the associated Laguerre route
 * (special_functions.cpp:110-181), for the explicit-matrix KAT. */
void orc_sgl_basis(int n, int l, int m, double r, double theta, double phi, double* out2);

/* Sphere rule of order L (quadrature.cpp:189-211). */
void orc_sphere_rule(int L, double* theta, double* phi, double* b_raw, double* b_cal);

/* Plan tables used by the transforms (for tests). */
void orc_plan_sphere(const orc_plan* p, double* theta, double* phi, double* b_cal);

/* mt19937_64 + the reference's portable top-53-bit map to [-1, 1)
 * (acceptance_main.cpp:50-63, commands.cpp:73-88): n complex values. */
void orc_random_coefficients(uint64_t seed, size_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif
