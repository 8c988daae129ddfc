/* TEST INFRASTRUCTURE -- NOT THE PRODUCT.  See sgl_oracle.h.
 *
 * Plain-C restatement of the reference's O(B^4) SGL transform pair.  Every
 * function names the reference file:line it follows (paths relative to
 * /root/reference/proj/core/).  Differences from the reference are numerics
 * only, and are listed here:
 *
 *  (N1) Legendre rows.  The reference forms M_lm * P_lm(cos theta_j) with an
 *       unnormalized P_lm seeded by (2m-1)!! (special_functions.cpp:21-47) and
 *       M_lm = sqrt(... exp(lgamma ratio)) (special_functions.cpp:81-88); M_lm
 *       leaves the fp64 range for l+m >~ 172 and P_mm overflows for m >~ 151.
 *       Here Pbar_lm = M_lm P_lm is generated directly by the fully normalized
 *       recurrence in long double (range 1e+-4932), then rounded to double and
 *       pushed through the same DCT-II/DST-II + truncation as
 *       spherical_transform.cpp:31-86.
 *  (N2) Radial seeds.  The reference forms seed_norm * r^l * exp(-r^2) with a
 *       double seed sqrt(2/Gamma(l+3/2)) that underflows for l >= 170
 *       (radial_transform.cpp:44, 65-71, 88).  Here the seeds are evaluated in
 *       log space in long double and the decay is split: the forward recurrence
 *       runs on N_nl R_nl e^{-r^2/2} and the node weight carries
 *       a_mod e^{-r^2/2}; the inverse multiplies the Clenshaw sum by
 *       seed * r^l, as radial_transform.cpp:131 does.
 *
 * Parallelism: OpenMP over radial shells and over (m, l) pairs, exactly the
 * two loops of sgl_transform.cpp:282-308 / 321-346.  Per-slice writes only.
 */
#include "sgl_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double re, im;
} cpx;

static inline cpx cmul(cpx a, cpx b) { return (cpx){a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
static inline cpx cadd(cpx a, cpx b) { return (cpx){a.re + b.re, a.im + b.im}; }
static inline cpx csub(cpx a, cpx b) { return (cpx){a.re - b.re, a.im - b.im}; }
static inline cpx cscale(double s, cpx a) { return (cpx){s * a.re, s * a.im}; }
static inline cpx cconj(cpx a) { return (cpx){a.re, -a.im}; }

static const double kPi = 3.14159265358979323846;
static const long double kPiL = 3.141592653589793238462643383279502884L;

/* ---------------------------------------------------------------- indexing
 * indexing.cpp:50-78: mu = 2Bj+k, psi = 4B^2 i + 2Bj + k, nu = l(l+1)+m,
 * omega = n(n-1)(2n-1)/6 + nu. */
static inline size_t nu_index(int l, int m) { return (size_t)(l * (l + 1) + m); }
static inline size_t omega_index(int n, int l, int m) {
    return (size_t)((long long)(n - 1) * n * (2 * n - 1) / 6) + nu_index(l, m);
}
static inline size_t coefficient_count(int B) { return (size_t)B * (B + 1) * (2 * B + 1) / 6; }

/* ---------------------------------------------------------------- FFT core
 * kernels.cpp:85-195: radix-2 DIT, bit reversal, twiddle e^{-2 pi i j / n},
 * sign -1 analysis, +1 synthesis (conjugated twiddles, no 1/n).  Naive DFT for
 * non-power-of-two lengths (kernels.cpp:35-45, 446-502). */
typedef struct {
    int n, pow2;
    int* bitrev;
    cpx* tw;
} fft_plan;

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

static void fft_init(fft_plan* f, int n) {
    f->n = n;
    f->pow2 = is_pow2(n);
    f->bitrev = NULL;
    f->tw = NULL;
    if (!f->pow2) return;
    f->bitrev = (int*)calloc((size_t)n, sizeof(int));
    for (int i = 1, j = 0; i < n; ++i) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        f->bitrev[i] = j;
    }
    f->tw = (cpx*)calloc((size_t)(n / 2 + 1), sizeof(cpx));
    for (int j = 0; j < n / 2; ++j) {
        const double ang = -2.0 * kPi * j / (double)n;
        f->tw[j] = (cpx){cos(ang), sin(ang)};
    }
}

static void fft_free(fft_plan* f) {
    free(f->bitrev);
    free(f->tw);
}

/* in place; scratch of length n needed only for the naive path */
static void fft_exec(const fft_plan* f, cpx* a, int sign, cpx* scratch) {
    const int n = f->n;
    if (!f->pow2) {
        const double base = sign * 2.0 * kPi / (double)n;
        for (int b = 0; b < n; ++b) {
            cpx acc = {0, 0};
            for (int k = 0; k < n; ++k) {
                const double ang = base * (double)((size_t)b * (size_t)k);
                acc = cadd(acc, cmul(a[k], (cpx){cos(ang), sin(ang)}));
            }
            scratch[b] = acc;
        }
        memcpy(a, scratch, sizeof(cpx) * (size_t)n);
        return;
    }
    for (int i = 1; i < n; ++i) {
        const int j = f->bitrev[i];
        if (i < j) {
            cpx t = a[i];
            a[i] = a[j];
            a[j] = t;
        }
    }
    for (int len = 2; len <= n; len <<= 1) {
        const int half = len / 2, step = n / len;
        for (int i = 0; i < n; i += len) {
            for (int j = 0; j < half; ++j) {
                const cpx tw = f->tw[j * step];
                const double wr = tw.re, wi = sign < 0 ? tw.im : -tw.im;
                cpx* lo = &a[i + j];
                cpx* hi = &a[i + j + half];
                const double xr = hi->re, xi = hi->im;
                const double vr = xr * wr - xi * wi, vi = xr * wi + xi * wr;
                const double ur = lo->re, ui = lo->im;
                *lo = (cpx){ur + vr, ui + vi};
                *hi = (cpx){ur - vr, ui - vi};
            }
        }
    }
}

/* ---------------------------------------------------------------- DCT/DST
 * kernels.cpp:47-50 (row_scale), 201-221 (plan), 317-350 (complex dct2/dct3
 * via FFT), 352-428 (forward/inverse incl. DST by flip + reversal),
 * 52-79 (naive fallback for non-power-of-two). */
typedef struct {
    int n, sine, fast;
    fft_plan fft;
    cpx* phase;     /* e^{-i pi k / 2n} */
    double* scale;  /* orthonormal row scales */
} dct_plan;

static double row_scale(int n, int k, int sine) {
    const int unit_row = sine ? n - 1 : 0;
    return sqrt((k == unit_row ? 1.0 : 2.0) / (double)n);
}

static void dct_init(dct_plan* d, int n, int sine) {
    d->n = n;
    d->sine = sine;
    d->fast = is_pow2(n);
    d->phase = NULL;
    if (d->fast) {
        fft_init(&d->fft, n);
        d->phase = (cpx*)calloc((size_t)n, sizeof(cpx));
        for (int k = 0; k < n; ++k) {
            const double ang = -kPi * k / (2.0 * (double)n);
            d->phase[k] = (cpx){cos(ang), sin(ang)};
        }
    } else {
        d->fft.bitrev = NULL;
        d->fft.tw = NULL;
    }
    d->scale = (double*)calloc((size_t)n, sizeof(double));
    for (int k = 0; k < n; ++k) d->scale[k] = row_scale(n, k, sine);
}

static void dct_free(dct_plan* d) {
    if (d->fast) fft_free(&d->fft);
    free(d->phase);
    free(d->scale);
}

/* scratch: 3n complex */
static void dct2_unscaled_c(const dct_plan* d, const cpx* in, cpx* out, cpx* buf, cpx* scr) {
    const int n = d->n;
    for (int i = 0; i < n / 2; ++i) {
        buf[i] = in[2 * i];
        buf[n - 1 - i] = in[2 * i + 1];
    }
    if (n % 2 == 1) buf[n / 2] = in[n - 1];
    fft_exec(&d->fft, buf, -1, scr);
    out[0] = buf[0];
    for (int k = 1; k < n; ++k)
        out[k] = cscale(0.5, cadd(cmul(d->phase[k], buf[k]), cmul(cconj(d->phase[k]), buf[n - k])));
}

static void dct3_unscaled_c(const dct_plan* d, const cpx* in, cpx* out, cpx* buf, cpx* scr) {
    const int n = d->n;
    buf[0] = in[0];
    for (int k = 1; k < n; ++k) {
        const cpx v = {in[k].re + in[n - k].im, in[k].im - in[n - k].re}; /* in[k] - i in[n-k] */
        buf[k] = cmul(cconj(d->phase[k]), v);
    }
    fft_exec(&d->fft, buf, +1, scr);
    const double inv_n = 1.0 / (double)n;
    for (int i = 0; i < n / 2; ++i) {
        out[2 * i] = cscale(inv_n, buf[i]);
        out[2 * i + 1] = cscale(inv_n, buf[n - 1 - i]);
    }
    if (n % 2 == 1) out[n - 1] = cscale(inv_n, buf[n / 2]);
}

static double trig(int sine, double arg) { return sine ? sin(arg) : cos(arg); }

/* complex forward (kernels.cpp:352-388); scratch 4n */
static void dct_forward_c(const dct_plan* d, const cpx* in, cpx* out, cpx* scratch) {
    const int n = d->n;
    if (!d->fast) {
        for (int k = 0; k < n; ++k) {
            const double freq = d->sine ? (double)(k + 1) : (double)k;
            double ar = 0, ai = 0;
            for (int j = 0; j < n; ++j) {
                const double t = trig(d->sine, freq * (2.0 * j + 1.0) * kPi / (2.0 * (double)n));
                ar += in[j].re * t;
                ai += in[j].im * t;
            }
            out[k] = (cpx){d->scale[k] * ar, d->scale[k] * ai};
        }
        return;
    }
    cpx* buf = scratch;
    cpx* scr = scratch + n;
    cpx* flipped = scratch + 2 * n;
    cpx* tmp = scratch + 3 * n;
    if (!d->sine) {
        dct2_unscaled_c(d, in, out, buf, scr);
        for (int k = 0; k < n; ++k) out[k] = cscale(d->scale[k], out[k]);
    } else {
        for (int j = 0; j < n; ++j) flipped[j] = (j % 2 == 0) ? in[j] : cscale(-1.0, in[j]);
        dct2_unscaled_c(d, flipped, tmp, buf, scr);
        for (int k = 0; k < n; ++k) out[k] = cscale(d->scale[k], tmp[n - 1 - k]);
    }
}

/* complex inverse (kernels.cpp:390-428); scratch 4n */
static void dct_inverse_c(const dct_plan* d, const cpx* in, cpx* out, cpx* scratch) {
    const int n = d->n;
    if (!d->fast) {
        for (int j = 0; j < n; ++j) {
            double ar = 0, ai = 0;
            for (int k = 0; k < n; ++k) {
                const double freq = d->sine ? (double)(k + 1) : (double)k;
                const double t = d->scale[k] * trig(d->sine, freq * (2.0 * j + 1.0) * kPi / (2.0 * (double)n));
                ar += in[k].re * t;
                ai += in[k].im * t;
            }
            out[j] = (cpx){ar, ai};
        }
        return;
    }
    cpx* buf = scratch;
    cpx* scr = scratch + n;
    cpx* unscaled = scratch + 2 * n;
    cpx* tmp = scratch + 3 * n;
    if (!d->sine) {
        for (int k = 0; k < n; ++k) unscaled[k] = cscale(d->scale[k] * (double)n / 2.0, in[k]);
        unscaled[0] = cscale(2.0, unscaled[0]);
        dct3_unscaled_c(d, unscaled, out, buf, scr);
    } else {
        for (int k = 0; k < n; ++k) unscaled[n - 1 - k] = cscale(d->scale[k] * (double)n / 2.0, in[k]);
        unscaled[0] = cscale(2.0, unscaled[0]);
        dct3_unscaled_c(d, unscaled, tmp, buf, scr);
        for (int j = 0; j < n; ++j) out[j] = (j % 2 == 0) ? tmp[j] : cscale(-1.0, tmp[j]);
    }
}

/* real forward, used only to build the Legendre rows (kernels.cpp:284-313) */
static void dct_forward_real(const dct_plan* d, const double* in, double* out, cpx* scratch) {
    const int n = d->n;
    cpx* cin = scratch + 4 * n;
    cpx* cout = scratch + 5 * n;
    for (int j = 0; j < n; ++j) cin[j] = (cpx){in[j], 0.0};
    dct_forward_c(d, cin, cout, scratch);
    for (int k = 0; k < n; ++k) out[k] = cout[k].re;
}

/* ---------------------------------------------------------------- sphere rule
 * quadrature.cpp:189-211 */
void orc_sphere_rule(int L, double* theta, double* phi, double* b_raw, double* b_cal) {
    const int count = 2 * L;
    for (int j = 0; j < count; ++j) {
        theta[j] = (2 * j + 1) * kPi / (4.0 * L);
        phi[j] = j * kPi / L;
        double acc = 0.0;
        for (int l = 0; l < L; ++l) acc += sin((2 * j + 1) * (2 * l + 1) * kPi / (4.0 * L)) / (2 * l + 1);
        const double braw = sin((2 * j + 1) * kPi / (4.0 * L)) * (2.0 / L) * acc;
        if (b_raw) b_raw[j] = braw;
        b_cal[j] = kPi / L * braw;
    }
}

/* ---------------------------------------------------------------- plan */
struct orc_plan {
    int B, n2;
    double *r, *a_mod;
    double *theta, *phi, *b_cal, *cos_theta;
    /* Legendre DCT rows (spherical_transform.cpp:31-86), row nu has l+1 entries */
    size_t* row_off;
    double* rows;
    fft_plan azimuth;
    dct_plan cosine, sine_;
    /* radial recurrence (radial_transform.cpp:29-46), per l: B-l-1 entries */
    size_t* rec_off;
    double *c1, *c2, *c3;
    double* seed_fwd;  /* [l][i] seed * r^l * e^{-r^2/2}  (N2) */
    double* seed_inv;  /* [l][i] seed * r^l                 */
    double* wfwd;      /* [i]    a_mod * e^{-r^2/2}         */
};

/* Fully normalized Pbar_lm(t) = M_lm P_lm(t) (Condon-Shortley phase included)
 * for l = m..L-1, long double (N1).  out[l - m]. */
static void pbar_column(int m, int L, long double t, long double* out) {
    const long double s = sqrtl((1.0L - t) * (1.0L + t));
    long double pmm = sqrtl((2 * m + 1) / (4.0L * kPiL));
    for (int k = 1; k <= m; ++k) pmm *= -sqrtl((2.0L * k - 1.0L) / (2.0L * k)) * s;
    out[0] = pmm;
    if (m + 1 >= L) return;
    long double p1 = sqrtl(2.0L * m + 3.0L) * t * pmm;
    out[1] = p1;
    long double p0 = pmm;
    for (int l = m + 2; l < L; ++l) {
        const long double a = sqrtl((4.0L * l * l - 1.0L) / ((long double)l * l - (long double)m * m));
        const long double b =
            sqrtl(((long double)(l - 1) * (l - 1) - (long double)m * m) / (4.0L * (l - 1) * (l - 1) - 1.0L));
        const long double p2 = a * (t * p1 - b * p0);
        out[l - m] = p2;
        p0 = p1;
        p1 = p2;
    }
}

orc_plan* orc_plan_create(int B, const double* r, const double* a_mod) {
    if (B < 1 || B > 512) return NULL;
    orc_plan* p = (orc_plan*)calloc(1, sizeof(orc_plan));
    const int n2 = 2 * B;
    p->B = B;
    p->n2 = n2;
    p->r = (double*)malloc(sizeof(double) * n2);
    p->a_mod = (double*)malloc(sizeof(double) * n2);
    memcpy(p->r, r, sizeof(double) * n2);
    memcpy(p->a_mod, a_mod, sizeof(double) * n2);
    p->theta = (double*)malloc(sizeof(double) * n2);
    p->phi = (double*)malloc(sizeof(double) * n2);
    p->b_cal = (double*)malloc(sizeof(double) * n2);
    p->cos_theta = (double*)malloc(sizeof(double) * n2);
    orc_sphere_rule(B, p->theta, p->phi, NULL, p->b_cal);
    for (int j = 0; j < n2; ++j) p->cos_theta[j] = cos(p->theta[j]);
    fft_init(&p->azimuth, n2);
    dct_init(&p->cosine, n2, 0);
    dct_init(&p->sine_, n2, 1);

    /* Legendre rows: per m ascend l, scale by the sign fold for odd negative m,
     * DCT (even |m|) / DST (odd |m|), truncate at l+1 (spherical_transform.cpp:51-84). */
    const size_t nrows = (size_t)B * B;
    p->row_off = (size_t*)malloc(sizeof(size_t) * (nrows + 1));
    p->row_off[0] = 0;
    for (int l = 0; l < B; ++l)
        for (int m = -l; m <= l; ++m) p->row_off[nu_index(l, m) + 1] = (size_t)(l + 1);
    for (size_t v = 0; v < nrows; ++v) p->row_off[v + 1] += p->row_off[v];
    p->rows = (double*)malloc(sizeof(double) * p->row_off[nrows]);
#pragma omp parallel
    {
        long double* col = (long double*)malloc(sizeof(long double) * (size_t)B);
        double* vec = (double*)malloc(sizeof(double) * (size_t)n2 * (size_t)B);
        double* tr = (double*)malloc(sizeof(double) * (size_t)n2);
        cpx* scratch = (cpx*)malloc(sizeof(cpx) * 6 * (size_t)n2);
#pragma omp for schedule(dynamic)
        for (int am = 0; am < B; ++am) {
            for (int j = 0; j < n2; ++j) {
                pbar_column(am, B, (long double)cosl((2 * j + 1) * kPiL / (4.0L * B)), col);
                for (int l = am; l < B; ++l) vec[(size_t)(l - am) * n2 + j] = (double)col[l - am];
            }
            const dct_plan* t = (am % 2 == 0) ? &p->cosine : &p->sine_;
            for (int l = am; l < B; ++l) {
                dct_forward_real(t, vec + (size_t)(l - am) * n2, tr, scratch);
                for (int sgn = 0; sgn < 2; ++sgn) {
                    if (sgn == 1 && am == 0) break;
                    const int m = sgn ? -am : am;
                    const double sign = (m < 0 && am % 2 != 0) ? -1.0 : 1.0;
                    double* row = p->rows + p->row_off[nu_index(l, m)];
                    for (int q = 0; q <= l; ++q) row[q] = sign * tr[q];
                }
            }
        }
        free(col);
        free(vec);
        free(tr);
        free(scratch);
    }

    /* radial recurrence coefficients (radial_transform.cpp:29-46) */
    p->rec_off = (size_t*)malloc(sizeof(size_t) * (size_t)(B + 1));
    p->rec_off[0] = 0;
    for (int l = 0; l < B; ++l) p->rec_off[l + 1] = p->rec_off[l] + (size_t)(B - l - 1);
    const size_t nrec = p->rec_off[B] > 0 ? p->rec_off[B] : 1;
    p->c1 = (double*)malloc(sizeof(double) * nrec);
    p->c2 = (double*)malloc(sizeof(double) * nrec);
    p->c3 = (double*)malloc(sizeof(double) * nrec);
    for (int l = 0; l < B; ++l) {
        size_t o = p->rec_off[l];
        for (int n = l + 1; n < B; ++n, ++o) {
            const double denom = sqrt((n + 0.5) * (n - l));
            p->c1[o] = (2 * n - l - 0.5) / denom;
            p->c2[o] = 1.0 / denom;
            p->c3[o] = sqrt((n - 0.5) / (n + 0.5) * ((double)(n - l - 1) / (n - l)));
        }
    }
    /* seeds (N2): sqrt(2/Gamma(l+3/2)) r^l [e^{-r^2/2}] in log space, long double */
    p->seed_fwd = (double*)malloc(sizeof(double) * (size_t)B * n2);
    p->seed_inv = (double*)malloc(sizeof(double) * (size_t)B * n2);
    p->wfwd = (double*)malloc(sizeof(double) * (size_t)n2);
    for (int i = 0; i < n2; ++i) {
        const long double ri = r[i];
        p->wfwd[i] = (double)((long double)a_mod[i] * expl(-ri * ri / 2.0L));
        for (int l = 0; l < B; ++l) {
            const long double lg = 0.5L * logl(2.0L) - 0.5L * lgammal(l + 1.5L) + (long double)l * logl(ri);
            p->seed_inv[(size_t)l * n2 + i] = (double)expl(lg);
            p->seed_fwd[(size_t)l * n2 + i] = (double)expl(lg - ri * ri / 2.0L);
        }
    }
    return p;
}

void orc_plan_destroy(orc_plan* p) {
    if (!p) return;
    free(p->r);
    free(p->a_mod);
    free(p->theta);
    free(p->phi);
    free(p->b_cal);
    free(p->cos_theta);
    free(p->row_off);
    free(p->rows);
    fft_free(&p->azimuth);
    dct_free(&p->cosine);
    dct_free(&p->sine_);
    free(p->rec_off);
    free(p->c1);
    free(p->c2);
    free(p->c3);
    free(p->seed_fwd);
    free(p->seed_inv);
    free(p->wfwd);
    free(p);
}

int orc_plan_bandlimit(const orc_plan* p) { return p->B; }

void orc_plan_sphere(const orc_plan* p, double* theta, double* phi, double* b_cal) {
    memcpy(theta, p->theta, sizeof(double) * p->n2);
    memcpy(phi, p->phi, sizeof(double) * p->n2);
    memcpy(b_cal, p->b_cal, sizeof(double) * p->n2);
}

/* ---------------------------------------------------------------- spherical stage */
/* workspace: rings 4B^2, t 2B, u 2B, scratch 4*2B complex */
static size_t sft_workspace(int B) { return (size_t)4 * B * B + 8 * (size_t)B + 8 * (size_t)B + 2 * (size_t)B; }

/* sft_seminaive_forward_into, spherical_transform.cpp:194-244 */
static void sft_forward(const orc_plan* p, const cpx* samples, cpx* out, cpx* ws) {
    const int B = p->B, n2 = p->n2;
    cpx* rings = ws;
    cpx* t = rings + (size_t)n2 * n2;
    cpx* u = t + n2;
    cpx* scratch = u + n2;
    memcpy(rings, samples, sizeof(cpx) * (size_t)n2 * n2);
    for (int j = 0; j < n2; ++j) fft_exec(&p->azimuth, rings + (size_t)j * n2, -1, scratch);
    for (int m = -(B - 1); m < B; ++m) {
        const int am = abs(m);
        const int bin = m >= 0 ? m : n2 + m;
        for (int j = 0; j < n2; ++j) t[j] = cscale(p->b_cal[j], rings[(size_t)j * n2 + bin]);
        dct_forward_c((am % 2 == 0) ? &p->cosine : &p->sine_, t, u, scratch);
        for (int l = am; l < B; ++l) {
            const double* row = p->rows + p->row_off[nu_index(l, m)];
            cpx acc = {0, 0};
            for (int q = 0; q <= l; ++q) acc = cadd(acc, cscale(row[q], u[q]));
            out[nu_index(l, m)] = acc;
        }
    }
}

/* sft_seminaive_inverse_into, spherical_transform.cpp:254-306 */
static void sft_inverse(const orc_plan* p, const cpx* coeffs, cpx* out, cpx* ws) {
    const int B = p->B, n2 = p->n2;
    cpx* rings = ws;
    cpx* w = rings + (size_t)n2 * n2;
    cpx* vals = w + n2;
    cpx* scratch = vals + n2;
    memset(rings, 0, sizeof(cpx) * (size_t)n2 * n2);
    for (int m = -(B - 1); m < B; ++m) {
        const int am = abs(m);
        memset(w, 0, sizeof(cpx) * n2);
        for (int l = am; l < B; ++l) {
            const double* row = p->rows + p->row_off[nu_index(l, m)];
            const cpx c = coeffs[nu_index(l, m)];
            for (int q = 0; q <= l; ++q) w[q] = cadd(w[q], cscale(row[q], c));
        }
        dct_inverse_c((am % 2 == 0) ? &p->cosine : &p->sine_, w, vals, scratch);
        const int bin = m >= 0 ? m : n2 + m;
        for (int j = 0; j < n2; ++j) rings[(size_t)j * n2 + bin] = vals[j];
    }
    memcpy(out, rings, sizeof(cpx) * (size_t)n2 * n2);
    for (int j = 0; j < n2; ++j) fft_exec(&p->azimuth, out + (size_t)j * n2, +1, scratch);
}

/* ---------------------------------------------------------------- radial stage */
/* drt_forward, radial_transform.cpp:75-97 (with N2) */
static void drt_forward(const orc_plan* p, int l, const cpx* s, cpx* out) {
    const int B = p->B, n2 = p->n2;
    const double* c1 = p->c1 + p->rec_off[l];
    const double* c2 = p->c2 + p->rec_off[l];
    const double* c3 = p->c3 + p->rec_off[l];
    for (int q = 0; q < B - l; ++q) out[q] = (cpx){0, 0};
    for (int i = 0; i < n2; ++i) {
        const double r = p->r[i];
        const double r2 = r * r;
        const cpx data = cscale(p->wfwd[i], s[i]);
        double prev = 0.0;
        double cur = p->seed_fwd[(size_t)l * n2 + i];
        out[0] = cadd(out[0], cscale(cur, data));
        for (int idx = 0; idx < B - l - 1; ++idx) {
            const double next = (c1[idx] - c2[idx] * r2) * cur - c3[idx] * prev;
            prev = cur;
            cur = next;
            out[idx + 1] = cadd(out[idx + 1], cscale(cur, data));
        }
    }
}

/* drt_inverse, radial_transform.cpp:99-133 */
static void drt_inverse(const orc_plan* p, int l, const cpx* t, cpx* out) {
    const int B = p->B, n2 = p->n2;
    const double* c1 = p->c1 + p->rec_off[l];
    const double* c2 = p->c2 + p->rec_off[l];
    const double* c3 = p->c3 + p->rec_off[l];
    const int top = B - l - 1;
    for (int i = 0; i < n2; ++i) {
        const double r = p->r[i];
        const double r2 = r * r;
        cpx y1 = {0, 0}, y2 = {0, 0};
        if (top >= 1) {
            y1 = t[top];
            for (int k = top - 1; k >= 1; --k) {
                const double ak = c1[k] - c2[k] * r2;
                cpx y = cadd(t[k], cscale(ak, y1));
                if (k + 1 < top) y = csub(y, cscale(c3[k + 1], y2));
                y2 = y1;
                y1 = y;
            }
        }
        cpx result = t[0];
        if (top >= 1) {
            result = cadd(result, cscale(c1[0] - c2[0] * r2, y1));
            if (top >= 2) result = csub(result, cscale(c3[1], y2));
        }
        out[i] = cscale(p->seed_inv[(size_t)l * n2 + i], result);
    }
}

/* ---------------------------------------------------------------- composed transforms */
static int nthreads(int threads) { return threads > 0 ? threads : omp_get_max_threads(); }

/* fsglft, sgl_transform.cpp:274-310 */
int orc_fsglft(const orc_plan* p, const double* grid_, double* coeffs_, int threads) {
    const int B = p->B, n2 = p->n2;
    const cpx* grid = (const cpx*)grid_;
    cpx* coeffs = (cpx*)coeffs_;
    const size_t nu_count = (size_t)B * B;
    cpx* shells = (cpx*)malloc(sizeof(cpx) * (size_t)n2 * nu_count);
    if (!shells) return 2;
#pragma omp parallel num_threads(nthreads(threads))
    {
        cpx* ws = (cpx*)malloc(sizeof(cpx) * sft_workspace(B));
#pragma omp for schedule(static)
        for (int i = 0; i < n2; ++i) sft_forward(p, grid + (size_t)i * n2 * n2, shells + (size_t)i * nu_count, ws);
        free(ws);
    }
    /* (m, l) pairs in order_pairs order (sgl_transform.cpp:39-48), m outer */
#pragma omp parallel num_threads(nthreads(threads))
    {
        cpx* s = (cpx*)malloc(sizeof(cpx) * (size_t)n2);
        cpx* t = (cpx*)malloc(sizeof(cpx) * (size_t)B);
#pragma omp for schedule(dynamic, 8)
        for (int pr = 0; pr < B * B; ++pr) {
            /* decode pair index -> (m, l) */
            int m = 1 - B, rem = pr;
            while (rem >= B - abs(m)) {
                rem -= B - abs(m);
                ++m;
            }
            const int l = abs(m) + rem;
            const size_t nu = nu_index(l, m);
            for (int i = 0; i < n2; ++i) s[i] = shells[(size_t)i * nu_count + nu];
            drt_forward(p, l, s, t);
            for (int n = l + 1; n <= B; ++n) coeffs[omega_index(n, l, m)] = t[n - l - 1];
        }
        free(s);
        free(t);
    }
    free(shells);
    return 0;
}

/* ifsglft, sgl_transform.cpp:312-348 */
int orc_ifsglft(const orc_plan* p, const double* coeffs_, double* grid_, int threads) {
    const int B = p->B, n2 = p->n2;
    const cpx* coeffs = (const cpx*)coeffs_;
    cpx* grid = (cpx*)grid_;
    const size_t nu_count = (size_t)B * B;
    cpx* shells = (cpx*)calloc((size_t)n2 * nu_count, sizeof(cpx));
    if (!shells) return 2;
#pragma omp parallel num_threads(nthreads(threads))
    {
        cpx* s = (cpx*)malloc(sizeof(cpx) * (size_t)n2);
        cpx* t = (cpx*)malloc(sizeof(cpx) * (size_t)B);
#pragma omp for schedule(dynamic, 8)
        for (int pr = 0; pr < B * B; ++pr) {
            int m = 1 - B, rem = pr;
            while (rem >= B - abs(m)) {
                rem -= B - abs(m);
                ++m;
            }
            const int l = abs(m) + rem;
            const size_t nu = nu_index(l, m);
            for (int n = l + 1; n <= B; ++n) t[n - l - 1] = coeffs[omega_index(n, l, m)];
            drt_inverse(p, l, t, s);
            for (int i = 0; i < n2; ++i) shells[(size_t)i * nu_count + nu] = s[i];
        }
        free(s);
        free(t);
    }
#pragma omp parallel num_threads(nthreads(threads))
    {
        cpx* ws = (cpx*)malloc(sizeof(cpx) * sft_workspace(B));
#pragma omp for schedule(static)
        for (int i = 0; i < n2; ++i) sft_inverse(p, shells + (size_t)i * nu_count, grid + (size_t)i * n2 * n2, ws);
        free(ws);
    }
    free(shells);
    return 0;
}

int orc_sft_forward(const orc_plan* p, const double* samples, double* out) {
    cpx* ws = (cpx*)malloc(sizeof(cpx) * sft_workspace(p->B));
    sft_forward(p, (const cpx*)samples, (cpx*)out, ws);
    free(ws);
    return 0;
}

int orc_sft_inverse(const orc_plan* p, const double* coeffs, double* out) {
    cpx* ws = (cpx*)malloc(sizeof(cpx) * sft_workspace(p->B));
    sft_inverse(p, (const cpx*)coeffs, (cpx*)out, ws);
    free(ws);
    return 0;
}

int orc_drt_forward(const orc_plan* p, int l, const double* s, double* out) {
    if (l < 0 || l >= p->B) return 1;
    drt_forward(p, l, (const cpx*)s, (cpx*)out);
    return 0;
}

int orc_drt_inverse(const orc_plan* p, int l, const double* t, double* out) {
    if (l < 0 || l >= p->B) return 1;
    drt_inverse(p, l, (const cpx*)t, (cpx*)out);
    return 0;
}

/* ---------------------------------------------------------------- basis sampling */
/* N_nl R_nl(r) by the Lemma recurrence from the seed (special_functions.cpp:131-144),
 * long double, seed in log space (N2). */
static long double radial_ld(int n, int l, long double r) {
    if (n <= l) return 0.0L;
    const long double r2 = r * r;
    long double cur = expl(0.5L * logl(2.0L) - 0.5L * lgammal(l + 1.5L) + l * logl(r));
    long double prev = 0.0L;
    for (int nn = l + 1; nn < n; ++nn) {
        const long double a = (2 * nn - l - 0.5L - r2) / sqrtl((nn + 0.5L) * (nn - l));
        const long double b = sqrtl((nn - 0.5L) / (nn + 0.5L) * ((long double)(nn - l - 1) / (nn - l)));
        const long double next = a * cur - b * prev;
        prev = cur;
        cur = next;
    }
    return cur;
}

/* sample_sgl_basis, sgl_transform.cpp:368-389 */
int orc_sample_basis(const orc_plan* p, int n, int l, int m, double* grid_) {
    const int B = p->B, n2 = p->n2;
    if (n < 1 || n > B || l < 0 || l >= n || abs(m) > l) return 1;
    cpx* grid = (cpx*)grid_;
    const int am = abs(m);
    const double sign = (m < 0 && am % 2 != 0) ? -1.0 : 1.0;
    long double* col = (long double*)malloc(sizeof(long double) * (size_t)B);
    for (int i = 0; i < n2; ++i) {
        const long double radial = radial_ld(n, l, p->r[i]);
        for (int j = 0; j < n2; ++j) {
            pbar_column(am, l + 1, (long double)p->cos_theta[j], col);
            const double base = (double)(radial * col[l - am]) * sign;
            for (int k = 0; k < n2; ++k) {
                const double ang = m * p->phi[k];
                grid[(size_t)i * n2 * n2 + (size_t)j * n2 + k] = (cpx){base * cos(ang), base * sin(ang)};
            }
        }
    }
    free(col);
    return 0;
}

/* Closed-form basis value (special_functions.cpp:62-79 gen_laguerre, 110-127
 * norm_const / radial_raw, 90-108 sph_harm), long double. */
void orc_sgl_basis(int n, int l, int m, double r_, double theta, double phi, double* out2) {
    const long double r = r_;
    const long double t = r * r;
    const long double alpha = l + 0.5L;
    const int k = n - l - 1;
    long double lag = 1.0L;
    if (k > 0) {
        long double prev = 1.0L, cur = alpha + 1.0L - t;
        for (int j = 1; j < k; ++j) {
            const long double next = ((2 * j + alpha + 1.0L - t) * cur - (j + alpha) * prev) / (j + 1);
            prev = cur;
            cur = next;
        }
        lag = cur;
    }
    const long double nc = expl(0.5L * (logl(2.0L) + lgammal((long double)(n - l)) - lgammal(n + 0.5L)));
    const long double radial = nc * lag * powl(r, l);
    const int am = abs(m);
    long double* col = (long double*)malloc(sizeof(long double) * (size_t)(l + 1));
    pbar_column(am, l + 1, cosl((long double)theta), col);
    const long double base = radial * col[l - am];
    free(col);
    long double yr = base * cosl(am * (long double)phi), yi = base * sinl(am * (long double)phi);
    if (m < 0) {
        yi = -yi; /* conj */
        if (am % 2 != 0) {
            yr = -yr;
            yi = -yi;
        }
    }
    out2[0] = (double)yr;
    out2[1] = (double)yi;
}

/* ---------------------------------------------------------------- mt19937_64 */
void orc_random_coefficients(uint64_t seed, size_t n, double* out) {
    enum { NN = 312, MM = 156 };
    uint64_t mt[NN];
    mt[0] = seed;
    for (int i = 1; i < NN; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    int mti = NN;
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, MATRIX_A = 0xB5026F5AA96619E9ULL;
    for (size_t c = 0; c < 2 * n; ++c) {
        if (mti >= NN) {
            for (int i = 0; i < NN; ++i) {
                const uint64_t x = (mt[i] & UM) | (mt[(i + 1) % NN] & LM);
                mt[i] = mt[(i + MM) % NN] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
            }
            mti = 0;
        }
        uint64_t x = mt[mti++];
        x ^= (x >> 29) & 0x5555555555555555ULL;
        x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
        x ^= (x << 37) & 0xFFF7EEE000000000ULL;
        x ^= x >> 43;
        out[c] = 2.0 * ((double)(x >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
    }
}
