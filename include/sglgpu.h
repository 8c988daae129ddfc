/* sglgpu -- C ABI of the B200 (sm_100a) SGL Fourier transform library.
 *
 * This is the drop-in boundary for the reference's hot path, the fast SGL
 * transform pair of /root/reference/proj/core:
 *
 *   SglCoefficients fsglft(const SampleGrid&, const TransformPlan&, unsigned threads)
 *   SampleGrid      ifsglft(const SglCoefficients&, const TransformPlan&, unsigned threads)
 *       (include/sgl/sgl_transform.hpp:71-76, bodies src/sgl_transform.cpp:274-348)
 *
 * The reference has no FFI; its interface is that C++ API.  The C++ mirror of it
 * lives in include/sgl/sgl_transform.hpp (the reference's own header path) and is implemented on top of the
 * entry points below, which is also what a ctypes / cgo / JNI binding would bind
 * (see INTEGRATION.md).  Plain pointers and sizes only.
 *
 * Data layouts are the reference's (indexing.hpp:8-40):
 *   samples       psi-order,   psi = 4B^2 i + 2B j + k,  8B^3 complex per function
 *   coefficients  omega-order, omega = n(n-1)(2n-1)/6 + l(l+1) + m,
 *                 B(B+1)(2B+1)/6 complex per function
 * A complex value is two doubles (re, im), i.e. std::complex<double> /
 * cuDoubleComplex.  A batch is `batch` functions stored back to back.
 *
 * Errors: every entry returns SGLGPU_OK (0) or a nonzero status; the message of
 * the most recent failure on the calling thread is sglgpu_last_error().
 * Shape errors are SGLGPU_EINVAL (the C++ wrapper maps them to
 * std::invalid_argument, as the reference throws at sgl_transform.cpp:18-35).
 */
#ifndef SGLGPU_H
#define SGLGPU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SGLGPU_OK = 0,
    SGLGPU_EINVAL = 1,  /* bad argument / shape (reference: std::invalid_argument) */
    SGLGPU_ECUDA = 2,   /* CUDA runtime error (reference: n/a; C++ wrapper: std::runtime_error) */
    SGLGPU_ENOMEM = 3,  /* device allocation failed */
    SGLGPU_ENODEV = 4   /* no usable CUDA device */
};

enum {
    SGLGPU_MEM_HOST = 0,   /* pointers are host memory; the call copies in and out and
                              returns after the result is in host memory */
    SGLGPU_MEM_DEVICE = 1  /* pointers are device memory on the plan's device; the call is
                              asynchronous on `stream` */
};

typedef struct sglgpu_plan sglgpu_plan;

/* Everything TransformPlan::assemble consumes that is not generated in closed
 * form (sgl_transform.cpp:52-88): the order-2B half-range Hermite rule
 * (RadialRule r, a_mod; quadrature.hpp:27-32) and the calibrated polar weights
 * (SphericalRule b_cal; quadrature.hpp:13-20).  The library derives cos(theta_j),
 * the normalized Legendre table and the radial tables from these, in long
 * double on the host, once per plan, and uploads them. */
typedef struct {
    int bandlimit;        /* B, 1 <= B <= 256 */
    const double* r;      /* 2B radial nodes, increasing */
    const double* a_mod;  /* 2B modified radial weights a * e^{r^2} * r^2 */
    const double* b_cal;  /* 2B polar weights; NULL = closed form of quadrature.cpp:189-211 */
    int device;           /* CUDA device ordinal; -1 = current device */
} sglgpu_plan_desc;

/* Creates a plan: generates and uploads the tables.  Cost O(B^3) host time. */
int sglgpu_plan_create(const sglgpu_plan_desc* desc, sglgpu_plan** out);
int sglgpu_plan_destroy(sglgpu_plan* plan);
int sglgpu_plan_bandlimit(const sglgpu_plan* plan);
/* Bytes of device memory held by the plan's tables. */
size_t sglgpu_plan_table_bytes(const sglgpu_plan* plan);

/* Forward transform (fsglft) of `batch` functions: samples -> coefficients. */
int sglgpu_forward(sglgpu_plan* plan, const double* samples, double* coeffs, size_t batch,
                   int mem_kind, void* stream);

/* Inverse transform (ifsglft) of `batch` functions: coefficients -> samples. */
int sglgpu_inverse(sglgpu_plan* plan, const double* coeffs, double* samples, size_t batch,
                   int mem_kind, void* stream);

/* Real-valued fast path (BASELINE config C5).
 * forward_real: `samples` are 8B^3 REAL doubles per function (psi-order); returns
 *   the full omega-order complex coefficients, identical (to rounding) to
 *   sglgpu_forward of the same samples promoted to complex, which for real data
 *   satisfy f_{n,l,-m} = (-1)^m conj(f_nlm).
 * inverse_real: reads only the m >= 0 coefficients, assumes that symmetry, and
 *   returns the 8B^3 real samples (the real part of sglgpu_inverse).
 * Ring pairs are packed into one complex FFT and only m >= 0 is propagated
 * through the polar and radial stages: about half the bytes and flops of the
 * complex path.  Requires 2B a power of two >= 4. */
int sglgpu_forward_real(sglgpu_plan* plan, const double* samples, double* coeffs, size_t batch,
                        int mem_kind, void* stream);
int sglgpu_inverse_real(sglgpu_plan* plan, const double* coeffs, double* samples, size_t batch,
                        int mem_kind, void* stream);

/* On-device cross-oracle: the reference's separated transforms
 * dsglft_separated / idsglft_separated (sgl_transform.cpp:189-272) with
 * closed-form basis values (assoc_legendre x sph_harm_norm, norm_const x
 * gen_laguerre x r^l; special_functions.cpp) and direct quadratures -- no FFT,
 * no fold, no tables, no DMMA -- to check the fast path on the device.  Same
 * layouts and batching as sglgpu_forward / sglgpu_inverse; B <= 64 (beyond that
 * the reference's unnormalized Legendre seed is not valid), else SGLGPU_EINVAL. */
int sglgpu_forward_separated(sglgpu_plan* plan, const double* samples, double* coeffs, size_t batch,
                             int mem_kind, void* stream);
int sglgpu_inverse_separated(sglgpu_plan* plan, const double* coeffs, double* samples, size_t batch,
                             int mem_kind, void* stream);

/* The reference's naive O(B^7) transforms dsglft_naive / idsglft_naive
 * (sgl_transform.cpp:122-187) on the device: every basis value evaluated afresh
 * at every node from normalized closed forms, direct sums.  The last rung of the
 * reference's oracle chain; B <= 32, else SGLGPU_EINVAL. */
int sglgpu_forward_naive(sglgpu_plan* plan, const double* samples, double* coeffs, size_t batch,
                         int mem_kind, void* stream);
int sglgpu_inverse_naive(sglgpu_plan* plan, const double* coeffs, double* samples, size_t batch,
                         int mem_kind, void* stream);
/* sample_sgl_basis (sgl_transform.cpp:368-389): H_nlm on the plan's grid,
 * psi-order, 8B^3 complex; SGLGPU_EINVAL unless |m| <= l < n <= B. */
int sglgpu_sample_basis(sglgpu_plan* plan, int n, int l, int m, double* samples, int mem_kind, void* stream);

/* Stage entry points (device memory only, asynchronous on `stream`), used by the
 * multi-GPU shell / (l, m) decomposition.  `shells` is the nu-major intermediate
 * S[nu][f][i] (nu = l(l+1)+m, f < batch, i < shell_count), i.e. the transpose of
 * the reference's shells[i][nu] buffer (sgl_transform.cpp:281, 319).
 *   spherical_forward: samples of shells [shell_begin, shell_begin+shell_count)
 *                      (psi-order slice, per function 4B^2*shell_count complex,
 *                      function stride `sample_stride` complex) -> shells (all nu)
 *   radial_forward:    degrees l in [l_begin, l_end) -> coefficients (omega-order,
 *                      function stride Omega; only those l's entries are written).
 *                      The 2B shells arrive as 2B/shells_per_block blocks
 *                      S_b[nu - l_begin^2][f][i_local] placed back to back (block b
 *                      holds shells [b*spb, (b+1)*spb)) -- exactly what an
 *                      all-to-all of per-rank spherical outputs delivers.
 *   radial_inverse:    the mirror image (writes the same block layout)
 *   spherical_inverse: shells (all nu, local shells) -> samples of those shells. */
int sglgpu_spherical_forward(sglgpu_plan* plan, const double* samples, size_t sample_stride,
                             double* shells, int shell_begin, int shell_count, size_t batch,
                             void* stream);
int sglgpu_radial_forward(sglgpu_plan* plan, const double* shells, double* coeffs, int l_begin,
                          int l_end, int shells_per_block, size_t batch, void* stream);
int sglgpu_radial_inverse(sglgpu_plan* plan, const double* coeffs, double* shells, int l_begin,
                          int l_end, int shells_per_block, size_t batch, void* stream);
int sglgpu_spherical_inverse(sglgpu_plan* plan, const double* shells, double* samples,
                             size_t sample_stride, int shell_begin, int shell_count,
                             size_t batch, void* stream);

/* Multi-GPU exchange fused into the stage epilogues (NVLink peer stores instead
 * of the all-to-all between the stages).  Device memory only.
 *
 * spherical_forward_to: like sglgpu_spherical_forward, but the Legendre
 *   epilogue stores the S rows of degree l in [l_bounds[q], l_bounds[q+1]) at
 *   dst[q] + (nu - l_bounds[q]^2) * NB (NB = 2 * batch * shell_count reals per
 *   nu row): dst[q] is this rank's shell block inside rank q's receive buffer,
 *   i.e. exactly what sglgpu_radial_forward reads there (shells_per_block =
 *   shell_count).  ndst <= 8.
 * radial_inverse_to: like sglgpu_radial_inverse, but shell block b
 *   ([b * spb, (b+1) * spb)) is stored in rank b's full-nu S buffer dst[b]
 *   ([nu][f][i_local], NB = 2 * batch * spb), which sglgpu_spherical_inverse
 *   then reads; ndst = 2B / spb <= 8.
 * radial_forward_to: like sglgpu_radial_forward (shell blocks of spb shells,
 *   degrees [l_begin, l_end)), but every coefficient is stored into each of the
 *   ndst <= 8 omega-order coefficient vectors dst[q] (batch * Omega complex each):
 *   with disjoint degree ranges per rank this assembles the full vector on every
 *   rank (replaces the all-reduce; fsglft's output).
 * The caller orders the peers' kernels (e.g. an NCCL barrier on the stream)
 * before the receive buffers are read. */
int sglgpu_radial_forward_to(sglgpu_plan* plan, const double* shells, int l_begin, int l_end, int shells_per_block,
                             size_t batch, int ndst, double* const* dst, void* stream);
int sglgpu_spherical_forward_to(sglgpu_plan* plan, const double* samples, size_t sample_stride, int shell_begin,
                                int shell_count, size_t batch, int ndst, double* const* dst, const int* l_bounds,
                                void* stream);
int sglgpu_radial_inverse_to(sglgpu_plan* plan, const double* coeffs, int l_begin, int l_end, int shells_per_block,
                             size_t batch, int ndst, double* const* dst, void* stream);
/* Peer-mappable device buffers (cudaMalloc + CUDA IPC, 64-byte handles). */
int sglgpu_device_alloc(size_t bytes, void** ptr);
int sglgpu_device_free(void* ptr);
int sglgpu_ipc_export(void* ptr, void* handle64);
int sglgpu_ipc_open(const void* handle64, void** ptr);
int sglgpu_ipc_close(void* ptr);

/* Number of kernels the most recent forward/inverse call on this plan launched
 * (for the bench's gpu_launches count). */
int sglgpu_last_launch_count(const sglgpu_plan* plan);

/* Live per-stage timing for benchmarks: between begin and end every stage launch
 * of sglgpu_forward / sglgpu_inverse is bracketed by CUDA events on the call's
 * stream; end synchronizes and returns, per stage, the summed milliseconds and
 * the number of launches.  Stages: 0 az_forward, 1 legendre_forward,
 * 2 radial_forward, 3 radial_inverse, 4 legendre_inverse, 5 az_inverse,
 * 6 spherical_forward (the fused persistent az + Legendre launch),
 * 7 spherical_inverse (fused).  Arrays have SGLGPU_NUM_STAGES entries. */
#define SGLGPU_NUM_STAGES 8
int sglgpu_profile_begin(sglgpu_plan* plan);
int sglgpu_profile_end(sglgpu_plan* plan, double* stage_ms, int* stage_launches);

const char* sglgpu_last_error(void);

/* Host-only (no CUDA) copy of the plan tables the kernels stream, for tests:
 * with all output pointers NULL only sizes[0..2] (doubles in the Legendre,
 * forward-radial and inverse-radial tables) are filled.  Offsets arrays have
 * 2B+1 (Legendre, per (|m|, parity)) and B+1 (radial, per l) entries. */
int sglgpu_host_tables(int B, const double* r, const double* a_mod, const double* bcal,
                       long long* sizes, double* legendre, long long* legendre_off,
                       double* radial_fwd, long long* radial_fwd_off, double* radial_inv,
                       long long* radial_inv_off);

#ifdef __cplusplus
}
#endif
#endif /* SGLGPU_H */
