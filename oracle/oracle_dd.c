/*
 * oracle_dd.c — plain CPU oracle for the EXTENDED-PRECISION refinement of SURVEY.md §8(f) NEXT-4,
 * the paper's "Extension to Quadruple Precision": QDGESV factors A with the
 * double precision LU (DGETRF), solves with DGETRS, and refines with the residual r = b - A x
 * computed in quadruple precision (QGEMV) and the update x += z carried in quadruple precision.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.c's header).
 *
 * Readings: Q-0 "quadruple precision" is carried as double-double (a value is the
 * unevaluated sum hi + lo of two binary64 numbers, |lo| <= ulp(hi)/2: 106 significand bits
 * against binary128's 113), the standard substitute on hardware without binary128; the error-free
 * transformations below (Knuth's TwoSum, the FMA-based TwoProd) are exact.  Q-1 stop test: B:5's
 * criterion with the double-double unit roundoff: ||r||_2 < ||x||_2 ||A||_F 2^-104 sqrt(n), r and x
 * rounded to binary64 for the norms.  Q-2 no convergence within 30 corrections: iters = -31 and X is
 * the last iterate (there is no higher-precision solver to fall back to; the paper's QGESV is the
 * comparison program, not a fallback).  Q-3 A and b are binary64 and are used exactly.
 *
 * Arithmetic: -ffp-contract=off (no implicit contraction); fma() only where written.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_ITERMAX 30

int oracle_dgetf2(int64_t n, double *A, int64_t lda, int32_t *ipiv);                     /* oracle.c */
void oracle_dgetrs(int64_t n, int64_t nrhs, const double *LU, int64_t lda, const int32_t *ipiv, double *B);
double oracle_fro_norm(int64_t n, const double *A, int64_t lda);

typedef struct { double hi, lo; } dd_t;

/* TwoSum (Knuth): s + e == a + b exactly */
static dd_t two_sum(double a, double b)
{
    double s = a + b;
    double bb = s - a;
    double e = (a - (s - bb)) + (b - bb);
    dd_t r = {s, e};
    return r;
}

/* FastTwoSum, |a| >= |b| */
static dd_t quick_two_sum(double a, double b)
{
    double s = a + b;
    double e = b - (s - a);
    dd_t r = {s, e};
    return r;
}

/* TwoProd: p + e == a * b exactly (FMA) */
static dd_t two_prod(double a, double b)
{
    double p = a * b;
    double e = fma(a, b, -p);
    dd_t r = {p, e};
    return r;
}

/* double-double + double-double (the accurate variant: two TwoSums) */
static dd_t dd_add(dd_t a, dd_t b)
{
    dd_t s = two_sum(a.hi, b.hi);
    dd_t t = two_sum(a.lo, b.lo);
    s.lo = s.lo + t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo = s.lo + t.lo;
    return quick_two_sum(s.hi, s.lo);
}

/* double-double * double */
static dd_t dd_mul_d(dd_t a, double b)
{
    dd_t p = two_prod(a.hi, b);
    p.lo = p.lo + a.lo * b;
    return quick_two_sum(p.hi, p.lo);
}

/* exported for the pins: the primitives on one pair */
void oracle_dd_two_sum(double a, double b, double *s, double *e) { dd_t r = two_sum(a, b); *s = r.hi; *e = r.lo; }
void oracle_dd_two_prod(double a, double b, double *p, double *e) { dd_t r = two_prod(a, b); *p = r.hi; *e = r.lo; }
void oracle_dd_add(double ah, double al, double bh, double bl, double *sh, double *sl)
{
    dd_t a = {ah, al}, b = {bh, bl};
    dd_t r = dd_add(a, b);
    *sh = r.hi; *sl = r.lo;
}

/* ------------------------------------------------------------------------ */
/* QGEMV step: r = b - A x with x = xh + xl, in double-double;  */
/* r_i = b_i; for j = 0..n-1: r_i = r_i - a_ij (xh_j + xl_j)   (fixed j).   */
/* ------------------------------------------------------------------------ */
void oracle_dd_residual(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B,
                        const double *Xh, const double *Xl, double *Rh, double *Rl)
{
    for (int64_t c = 0; c < nrhs; ++c) {
#pragma omp parallel for schedule(static) if (n >= 256)
        for (int64_t i = 0; i < n; ++i) {
            dd_t r = {B[i + c * n], 0.0};
            for (int64_t j = 0; j < n; ++j) {
                dd_t xj = {Xh[j + c * n], Xl[j + c * n]};
                dd_t p = dd_mul_d(xj, A[i + j * lda]);
                p.hi = -p.hi; p.lo = -p.lo;
                r = dd_add(r, p);
            }
            Rh[i + c * n] = r.hi;
            Rl[i + c * n] = r.lo;
        }
    }
}

static double nrm2(int64_t n, const double *v)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) { double sq = v[i] * v[i]; s = s + sq; }
    return sqrt(s);
}

/* ------------------------------------------------------------------------ */
/* QDGESV: binary64 GEPP, x0 = DGETRS(b); loop: double-double    */
/* residual, stop test Q-1, z = DGETRS(fl64(r)), x = x + z in double-double. */
/* iters >= 0 corrections; -31 no convergence (Q-2).  info: 0, -i argument, */
/* +k exact zero pivot in the binary64 LU (X unspecified).                  */
/* ------------------------------------------------------------------------ */
int oracle_qdgesv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *Xh, double *Xl,
                     int *iters, int *info, int itermax, double *hist, int *nhist)
{
    *info = 0; *iters = 0;
    if (nhist) *nhist = 0;
    if (n < 0) { *info = -1; return 0; }
    if (nrhs < 0) { *info = -2; return 0; }
    if (lda < (n > 1 ? n : 1)) { *info = -4; return 0; }
    if (n == 0 || nrhs == 0) return 0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i)
            if (!isfinite(A[i + j * lda])) { *info = -3; return 0; }
    for (int64_t t = 0; t < n * nrhs; ++t)
        if (!isfinite(B[t])) { *info = -5; return 0; }
    const double cte = oracle_fro_norm(n, A, lda) * ldexp(1.0, -104) * sqrt((double)n);   /* Q-1 */
    double *LU = (double *)malloc((size_t)n * n * sizeof(double));
    int32_t *ipiv = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    double *Z = (double *)malloc((size_t)n * nrhs * sizeof(double));
    double *Rh = (double *)malloc((size_t)n * nrhs * sizeof(double));
    double *Rl = (double *)malloc((size_t)n * nrhs * sizeof(double));
    for (int64_t j = 0; j < n; ++j) memcpy(LU + j * n, A + j * lda, (size_t)n * sizeof(double));
    int z = oracle_dgetf2(n, LU, n, ipiv);
    if (z) { *info = z; goto done; }
    memcpy(Z, B, (size_t)n * nrhs * sizeof(double));
    oracle_dgetrs(n, nrhs, LU, n, ipiv, Z);                                  /* x0 (binary64) */
    for (int64_t t = 0; t < n * nrhs; ++t) { Xh[t] = Z[t]; Xl[t] = 0.0; }
    *iters = -31;
    for (int it = 0; it <= itermax; ++it) {
        oracle_dd_residual(n, nrhs, A, lda, B, Xh, Xl, Rh, Rl);
        int conv = 1, bad = 0;
        double worst = 0.0;
        for (int64_t c = 0; c < nrhs; ++c) {
            double rn = nrm2(n, Rh + c * n), xn = nrm2(n, Xh + c * n);
            if (!isfinite(rn) || !isfinite(xn)) { bad = 1; break; }
            double ratio = rn == 0.0 ? 0.0 : rn / (xn * cte);
            if (ratio > worst) worst = ratio;
            if (!(rn < xn * cte || rn == 0.0)) conv = 0;
        }
        if (bad) break;
        if (hist) hist[it] = worst;
        if (nhist) *nhist = it + 1;
        if (conv) { *iters = it; break; }
        if (it == itermax) break;
        memcpy(Z, Rh, (size_t)n * nrhs * sizeof(double));                     /* fl64(r) */
        oracle_dgetrs(n, nrhs, LU, n, ipiv, Z);
        for (int64_t t = 0; t < n * nrhs; ++t) {
            dd_t x = {Xh[t], Xl[t]}, zz = {Z[t], 0.0};
            x = dd_add(x, zz);
            Xh[t] = x.hi; Xl[t] = x.lo;
        }
    }
done:
    free(LU); free(ipiv); free(Z); free(Rh); free(Rl);
    return 0;
}
