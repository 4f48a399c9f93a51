/*
 * oec_oracle.c -- the CPU ORACLE for hdiff and vadv.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  The product path (paper_2005_13014_b200/) never links, loads or calls it,
 * and shares no code, header, table or helper with it.
 *
 * What it computes: the plain definition of each stencil program (§4.3-4.4): every
 * stencil operator is evaluated "as in a loop nest" over its domain, each
 * stencil.access reads its input at point + constant offset, and -- in the UNFUSED
 * variant -- every intermediate is materialised over the range shape inference gives it
 * (P:480-482), i.e. the paper's "original" optimisation level.  The FUSED variant is the
 * inlined per-point expression (stencil inlining): it clones producer expression trees
 * and never reassociates, so both variants must agree bitwise (tests pin that).
 *
 * Arithmetic: IEEE fp64 (the f32 instance: binary32), round-to-nearest-even, NO contraction (built with -O2 -fno-fast-math
 * -ffp-contract=off).  Sums are evaluated exactly in the parenthesised order
 * written below (readings R3, R10).  Out-of-range reads are detected and make the
 * call return ORACLE_ERR_RANGE ("out-of-range access traps").
 *
 * Definitions (PAPER.md does not define hdiff/vadv; readings R1-R11 in DESIGN.md, after
 * SURVEY.md §8(c) c3/c4 [EXT: COSMO / GridTools benchmark definitions]):
 *
 *   hdiff, per level k (P:119 cites COSMO; north_star "Laplacian, flux limiter and update"):
 *     lap(i,j) = ((in(i-1,j)+in(i+1,j)) + (in(i,j-1)+in(i,j+1))) - 4*in(i,j)
 *     flx(i,j) = f*(in(i+1,j)-in(i,j)) > 0 ? 0 : f,   f = lap(i+1,j)-lap(i,j)
 *     fly(i,j) = g*(in(i,j+1)-in(i,j)) > 0 ? 0 : g,   g = lap(i,j+1)-lap(i,j)
 *     out(i,j) = in(i,j) - coeff(i,j)*((flx(i,j)-flx(i-1,j)) + (fly(i,j)-fly(i,j-1)))
 *
 *   vadv, per column (i,j): tridiagonal a_k x_{k-1} + b_k x_k + c_k x_{k+1} = d_k solved by the
 *   Thomas algorithm ("Some use the Thomas algorithm to perform implicit integration in the
 *   vertical direction"), coefficients of the GridTools vertical_advection_dycore
 *   benchmark [EXT], BET_M = BET_P = 0.5.
 *
 * Parity pins (tests/test_oracle_pins.py): constant / linear / quadratic fields, the unit spike,
 * the quartic limiter closed form, hand-built limiter patches (tests/golden/), the limiter-off
 * 13-point biharmonic, Thomas vs dense LU, wcon == 0 and constant u_stage special cases, fused ==
 * unfused, reversed loop order, an independent numpy implementation (oracle/numpy_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_RANGE 2
#define ORACLE_ERR_ARG 1

/* Precision ("single-precision (f32) and double-precision (f64)"): compiled twice, once
 * with real = double (entry points oracle_*) and once with -DORACLE_F32, real = float (entry
 * points oracle_*_f32).  Every constant is rounded to `real` (R()), so an f32 expression is
 * evaluated entirely in IEEE binary32 (FLT_EVAL_METHOD 0 on x86-64), as written. */
#ifdef ORACLE_F32
typedef float real;
#define SFX(name) name##_f32
#else
typedef double real;
#define SFX(name) name
#endif
#define R(x) ((real)(x))

/* A dense host field over its allocated range [lb, ub), index order [k][j][i] (i fastest).
 * A k-invariant (2D) field has lb[2] = 0, ub[2] = 1 and ignores k. */
typedef struct {
    real *d;
    int64_t lb[3];
    int64_t ub[3];
    int32_t k_invariant;
} ofield;

static int g_range_error; /* set when any access falls outside a field's allocation */

static real *at(const ofield *f, int64_t i, int64_t j, int64_t k) {
    if (f->k_invariant) k = 0;
    if (i < f->lb[0] || i >= f->ub[0] || j < f->lb[1] || j >= f->ub[1] || k < f->lb[2] || k >= f->ub[2]) {
        g_range_error = 1;
        static real trap = NAN;
        return &trap;
    }
    int64_t ni = f->ub[0] - f->lb[0], nj = f->ub[1] - f->lb[1];
    return f->d + ((k - f->lb[2]) * nj + (j - f->lb[1])) * ni + (i - f->lb[0]);
}
#define A(f, i, j, k) (*at((f), (i), (j), (k)))

static ofield temp_field(const int64_t lb[3], const int64_t ub[3]) {
    ofield t;
    int64_t n = 1;
    for (int d = 0; d < 3; ++d) {
        t.lb[d] = lb[d];
        t.ub[d] = ub[d];
        n *= (ub[d] - lb[d]) > 0 ? (ub[d] - lb[d]) : 0;
    }
    t.k_invariant = 0;
    t.d = (real *)malloc((size_t)(n > 0 ? n : 1) * sizeof(real));
    for (int64_t q = 0; q < n; ++q) t.d[q] = NAN;
    return t;
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

#ifndef ORACLE_F32
int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
#endif

/* ------------------------------------------------------------------------------------------ */
/* hdiff                                                                                      */
/* ------------------------------------------------------------------------------------------ */

/* The flux limiter (reading R4): strict '>' -- a product of exactly 0 keeps the flux; a NaN
 * product compares false and keeps the flux. */
static real limit(real f, real din) { return (f * din > R(0.0)) ? R(0.0) : f; }

static real lap_at(const ofield *in, int64_t i, int64_t j, int64_t k) {
    return ((A(in, i - 1, j, k) + A(in, i + 1, j, k)) + (A(in, i, j - 1, k) + A(in, i, j + 1, k))) -
           R(4.0) * A(in, i, j, k);
}

/* limiter_on = 0 is the debug "limiter off" variant used only by the biharmonic pin. */
static int hdiff_unfused(const ofield *in, const ofield *coeff, ofield *out, const int64_t lo[3],
                         const int64_t hi[3], int limiter_on) {
    /* shape inference: lap on the bounding box of its consumers' extents,
     * flx on [lo0-1,hi0) x [lo1,hi1), fly on [lo0,hi0) x [lo1-1,hi1). */
    int64_t llo[3] = {lo[0] - 1, lo[1] - 1, lo[2]}, lhi[3] = {hi[0] + 1, hi[1] + 1, hi[2]};
    int64_t xlo[3] = {lo[0] - 1, lo[1], lo[2]}, xhi[3] = {hi[0], hi[1], hi[2]};
    int64_t ylo[3] = {lo[0], lo[1] - 1, lo[2]}, yhi[3] = {hi[0], hi[1], hi[2]};
    ofield lap = temp_field(llo, lhi), flx = temp_field(xlo, xhi), fly = temp_field(ylo, yhi);
#pragma omp parallel for schedule(static)
    for (int64_t k = lo[2]; k < hi[2]; ++k) {
        for (int64_t j = llo[1]; j < lhi[1]; ++j)
            for (int64_t i = llo[0]; i < lhi[0]; ++i) A(&lap, i, j, k) = lap_at(in, i, j, k);
        for (int64_t j = xlo[1]; j < xhi[1]; ++j)
            for (int64_t i = xlo[0]; i < xhi[0]; ++i) {
                real f = A(&lap, i + 1, j, k) - A(&lap, i, j, k);
                A(&flx, i, j, k) = limiter_on ? limit(f, A(in, i + 1, j, k) - A(in, i, j, k)) : f;
            }
        for (int64_t j = ylo[1]; j < yhi[1]; ++j)
            for (int64_t i = ylo[0]; i < yhi[0]; ++i) {
                real g = A(&lap, i, j + 1, k) - A(&lap, i, j, k);
                A(&fly, i, j, k) = limiter_on ? limit(g, A(in, i, j + 1, k) - A(in, i, j, k)) : g;
            }
        for (int64_t j = lo[1]; j < hi[1]; ++j)
            for (int64_t i = lo[0]; i < hi[0]; ++i)
                A(out, i, j, k) = A(in, i, j, k) - A(coeff, i, j, k) * ((A(&flx, i, j, k) - A(&flx, i - 1, j, k)) +
                                                                        (A(&fly, i, j, k) - A(&fly, i, j - 1, k)));
    }
    free(lap.d);
    free(flx.d);
    free(fly.d);
    return 0;
}

/* Fused: the inlined per-point expression, producer trees cloned at every offset. */
static real flx_at(const ofield *in, int64_t i, int64_t j, int64_t k) {
    real f = lap_at(in, i + 1, j, k) - lap_at(in, i, j, k);
    return limit(f, A(in, i + 1, j, k) - A(in, i, j, k));
}
static real fly_at(const ofield *in, int64_t i, int64_t j, int64_t k) {
    real g = lap_at(in, i, j + 1, k) - lap_at(in, i, j, k);
    return limit(g, A(in, i, j + 1, k) - A(in, i, j, k));
}

static int hdiff_fused(const ofield *in, const ofield *coeff, ofield *out, const int64_t lo[3], const int64_t hi[3],
                       int reverse) {
#pragma omp parallel for schedule(static)
    for (int64_t kk = lo[2]; kk < hi[2]; ++kk) {
        int64_t k = reverse ? (hi[2] - 1 - (kk - lo[2])) : kk;
        for (int64_t jj = lo[1]; jj < hi[1]; ++jj) {
            int64_t j = reverse ? (hi[1] - 1 - (jj - lo[1])) : jj;
            for (int64_t ii = lo[0]; ii < hi[0]; ++ii) {
                int64_t i = reverse ? (hi[0] - 1 - (ii - lo[0])) : ii;
                A(out, i, j, k) = A(in, i, j, k) - A(coeff, i, j, k) * ((flx_at(in, i, j, k) - flx_at(in, i - 1, j, k)) +
                                                                        (fly_at(in, i, j, k) - fly_at(in, i, j - 1, k)));
            }
        }
    }
    return 0;
}

/* variant: 0 = unfused ("original"), 1 = fused (inlined), 2 = fused with reversed loop order,
 * 3 = unfused with the limiter switched off (debug variant for the biharmonic pin only). */
int SFX(oracle_hdiff)(const ofield *in, const ofield *coeff, ofield *out, const int64_t lo[3], const int64_t hi[3],
                 int variant, int nthreads) {
    if (!in || !coeff || !out || !lo || !hi) return ORACLE_ERR_ARG;
    set_threads(nthreads);
    g_range_error = 0;
    switch (variant) {
    case 0: hdiff_unfused(in, coeff, out, lo, hi, 1); break;
    case 1: hdiff_fused(in, coeff, out, lo, hi, 0); break;
    case 2: hdiff_fused(in, coeff, out, lo, hi, 1); break;
    case 3: hdiff_unfused(in, coeff, out, lo, hi, 0); break;
    default: return ORACLE_ERR_ARG;
    }
    return g_range_error ? ORACLE_ERR_RANGE : ORACLE_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* vadv                                                                                       */
/* ------------------------------------------------------------------------------------------ */

#define BET_M R(0.5)
#define BET_P R(0.5)

/* Tridiagonal coefficients (a, b, c, d) of level k of column (i,j); k0 = top, kN = bottom
 * level of the domain (reading R8: the k = k0 / k = kN branches are the boundary rows). */
static void vadv_coeffs(const ofield *u_stage, const ofield *wcon, const ofield *u_pos, const ofield *utens,
                        const ofield *utens_stage_in, real dtr, int64_t i, int64_t j, int64_t k, int64_t k0,
                        int64_t kN, real *a, real *b, real *c, real *d) {
    real corr;
    if (k == k0) {
        real gcv = R(0.25) * (A(wcon, i + 1, j, k + 1) + A(wcon, i, j, k + 1));
        real cs = gcv * BET_M;
        *a = R(0.0);
        *c = gcv * BET_P;
        *b = dtr - *c;
        corr = -cs * (A(u_stage, i, j, k + 1) - A(u_stage, i, j, k));
    } else if (k == kN) {
        real gav = R(-0.25) * (A(wcon, i + 1, j, k) + A(wcon, i, j, k));
        real as = gav * BET_M;
        *a = gav * BET_P;
        *c = R(0.0);
        *b = dtr - *a;
        corr = -as * (A(u_stage, i, j, k - 1) - A(u_stage, i, j, k));
    } else {
        real gav = R(-0.25) * (A(wcon, i + 1, j, k) + A(wcon, i, j, k));
        real gcv = R(0.25) * (A(wcon, i + 1, j, k + 1) + A(wcon, i, j, k + 1));
        real as = gav * BET_M;
        real cs = gcv * BET_M;
        *a = gav * BET_P;
        *c = gcv * BET_P;
        *b = (dtr - *a) - *c;
        corr = (-as * (A(u_stage, i, j, k - 1) - A(u_stage, i, j, k))) - cs * (A(u_stage, i, j, k + 1) - A(u_stage, i, j, k));
    }
    *d = ((dtr * A(u_pos, i, j, k) + A(utens, i, j, k)) + A(utens_stage_in, i, j, k)) + corr;
}

/* Unfused: the coefficient stencil materialises a,b,c,d over the domain; the forward sweep
 * materialises c', d'; the backward sweep materialises x; the output stencil writes
 * utens_stage_out = dtr*(x - u_pos). */
static int vadv_unfused(const ofield *u_stage, const ofield *wcon, const ofield *u_pos, const ofield *utens,
                        const ofield *utens_stage_in, ofield *out, real dtr, const int64_t lo[3], const int64_t hi[3]) {
    ofield fa = temp_field(lo, hi), fb = temp_field(lo, hi), fc = temp_field(lo, hi), fd = temp_field(lo, hi);
    ofield cp = temp_field(lo, hi), dp = temp_field(lo, hi), x = temp_field(lo, hi);
    int64_t k0 = lo[2], kN = hi[2] - 1;
#pragma omp parallel for schedule(static)
    for (int64_t j = lo[1]; j < hi[1]; ++j) {
        for (int64_t k = k0; k <= kN; ++k)
            for (int64_t i = lo[0]; i < hi[0]; ++i)
                vadv_coeffs(u_stage, wcon, u_pos, utens, utens_stage_in, dtr, i, j, k, k0, kN, &A(&fa, i, j, k),
                            &A(&fb, i, j, k), &A(&fc, i, j, k), &A(&fd, i, j, k));
        /* forward sweep (Thomas elimination): reciprocal, then multiply (reading R10) */
        for (int64_t i = lo[0]; i < hi[0]; ++i) {
            real r = R(1.0) / A(&fb, i, j, k0);
            A(&cp, i, j, k0) = A(&fc, i, j, k0) * r;
            A(&dp, i, j, k0) = A(&fd, i, j, k0) * r;
        }
        for (int64_t k = k0 + 1; k <= kN; ++k)
            for (int64_t i = lo[0]; i < hi[0]; ++i) {
                real r = R(1.0) / (A(&fb, i, j, k) - A(&cp, i, j, k - 1) * A(&fa, i, j, k));
                A(&cp, i, j, k) = A(&fc, i, j, k) * r;
                A(&dp, i, j, k) = (A(&fd, i, j, k) - A(&dp, i, j, k - 1) * A(&fa, i, j, k)) * r;
            }
        /* backward sweep */
        for (int64_t i = lo[0]; i < hi[0]; ++i) A(&x, i, j, kN) = A(&dp, i, j, kN);
        for (int64_t k = kN - 1; k >= k0; --k)
            for (int64_t i = lo[0]; i < hi[0]; ++i)
                A(&x, i, j, k) = A(&dp, i, j, k) - A(&cp, i, j, k) * A(&x, i, j, k + 1);
        /* output stencil */
        for (int64_t k = k0; k <= kN; ++k)
            for (int64_t i = lo[0]; i < hi[0]; ++i) A(out, i, j, k) = dtr * (A(&x, i, j, k) - A(u_pos, i, j, k));
    }
    free(fa.d); free(fb.d); free(fc.d); free(fd.d); free(cp.d); free(dp.d); free(x.d);
    return 0;
}

/* Fused: one pass per column, c' and d' in a per-column scratch (never a global temporary). */
static int vadv_fused(const ofield *u_stage, const ofield *wcon, const ofield *u_pos, const ofield *utens,
                      const ofield *utens_stage_in, ofield *out, real dtr, const int64_t lo[3], const int64_t hi[3],
                      int reverse) {
    int64_t k0 = lo[2], kN = hi[2] - 1, K = hi[2] - lo[2];
#pragma omp parallel
    {
        real *cp = (real *)malloc((size_t)K * sizeof(real));
        real *dp = (real *)malloc((size_t)K * sizeof(real));
#pragma omp for schedule(static)
        for (int64_t jj = lo[1]; jj < hi[1]; ++jj) {
            int64_t j = reverse ? (hi[1] - 1 - (jj - lo[1])) : jj;
            for (int64_t ii = lo[0]; ii < hi[0]; ++ii) {
                int64_t i = reverse ? (hi[0] - 1 - (ii - lo[0])) : ii;
                for (int64_t k = k0; k <= kN; ++k) {
                    real a, b, c, d;
                    vadv_coeffs(u_stage, wcon, u_pos, utens, utens_stage_in, dtr, i, j, k, k0, kN, &a, &b, &c, &d);
                    if (k == k0) {
                        real r = R(1.0) / b;
                        cp[0] = c * r;
                        dp[0] = d * r;
                    } else {
                        real r = R(1.0) / (b - cp[k - k0 - 1] * a);
                        cp[k - k0] = c * r;
                        dp[k - k0] = (d - dp[k - k0 - 1] * a) * r;
                    }
                }
                real x = dp[K - 1];
                A(out, i, j, kN) = dtr * (x - A(u_pos, i, j, kN));
                for (int64_t k = kN - 1; k >= k0; --k) {
                    x = dp[k - k0] - cp[k - k0] * x;
                    A(out, i, j, k) = dtr * (x - A(u_pos, i, j, k));
                }
            }
        }
        free(cp);
        free(dp);
    }
    return 0;
}

/* variant: 0 = unfused, 1 = fused, 2 = fused with reversed column order. K >= 2 required. */
int SFX(oracle_vadv)(const ofield *u_stage, const ofield *wcon, const ofield *u_pos, const ofield *utens,
                const ofield *utens_stage_in, ofield *out, double dtr_stage, const int64_t lo[3], const int64_t hi[3],
                int variant, int nthreads) {
    if (!u_stage || !wcon || !u_pos || !utens || !utens_stage_in || !out || !lo || !hi) return ORACLE_ERR_ARG;
    if (hi[2] - lo[2] < 2) return ORACLE_ERR_ARG;
    set_threads(nthreads);
    g_range_error = 0;
    switch (variant) {
    case 0: vadv_unfused(u_stage, wcon, u_pos, utens, utens_stage_in, out, R(dtr_stage), lo, hi); break;
    case 1: vadv_fused(u_stage, wcon, u_pos, utens, utens_stage_in, out, R(dtr_stage), lo, hi, 0); break;
    case 2: vadv_fused(u_stage, wcon, u_pos, utens, utens_stage_in, out, R(dtr_stage), lo, hi, 1); break;
    default: return ORACLE_ERR_ARG;
    }
    return g_range_error ? ORACLE_ERR_RANGE : ORACLE_OK;
}

/* Exposed for the dense-solve pin: the (a, b, c, d) rows of one column, k = lo2 .. hi2-1. */
int SFX(oracle_vadv_system)(const ofield *u_stage, const ofield *wcon, const ofield *u_pos, const ofield *utens,
                       const ofield *utens_stage_in, double dtr_stage, int64_t i, int64_t j, int64_t k_lo,
                       int64_t k_hi, real *a, real *b, real *c, real *d) {
    if (k_hi - k_lo < 2) return ORACLE_ERR_ARG;
    g_range_error = 0;
    for (int64_t k = k_lo; k < k_hi; ++k)
        vadv_coeffs(u_stage, wcon, u_pos, utens, utens_stage_in, R(dtr_stage), i, j, k, k_lo, k_hi - 1, &a[k - k_lo],
                    &b[k - k_lo], &c[k - k_lo], &d[k - k_lo]);
    return g_range_error ? ORACLE_ERR_RANGE : ORACLE_OK;
}
