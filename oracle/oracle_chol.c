/*
 * oracle_chol.c — plain CPU oracle for the SYMMETRIC POSITIVE DEFINITE variant of the
 * mixed-precision iterative-refinement solve.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.c's header): only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg use it; it shares nothing with the CUDA path.
 *
 * The passage: PAPER.md P:369-371 — "For the symmetric case the SGETRF, SGETRS and DGEMM
 * subroutines were replaced by the SPOTRF, SPOTRS and DSYMM subroutines, respectively",
 * i.e. Algorithm 1 with step 1 a binary32 Cholesky factorisation A = L L^T,
 * steps 2-3 / 5-6 the two binary32 triangular solves with L and L^T, step 4 the binary64
 * residual with the symmetric A, step 7 the binary64 update; B:5's stop test, 30-correction
 * cap and binary64 fallback carry over unchanged.
 *
 * Storage convention (LAPACK UPLO = 'L'): A is n x n column-major, only its LOWER triangle
 * (i >= j) is read; the strict upper triangle is never touched.  L is returned in the lower
 * triangle.  Arithmetic: -ffp-contract=off, separate multiply and subtract, IEEE division
 * and square root, fixed loop orders (textbook right-looking column Cholesky).
 *
 * Readings: C-1 the binary32 Cholesky breaks down when a pivot a_jj (after the
 * updates) is not > 0 (or is NaN) — the fallback code is iters = -3, as a zero pivot in
 * the LU case; C-2 the binary64 Cholesky's breakdown at column k is info = k + 1 (LAPACK
 * DPOTRF: "the leading minor of order k is not positive definite"); C-3 ||A||_F is the
 * Frobenius norm of the full symmetric matrix (each strictly-lower entry counted twice).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_ITERMAX 30

/* a_sym(i, j) from the lower triangle */
static double asym(const double *A, int64_t lda, int64_t i, int64_t j)
{
    return i >= j ? A[i + j * lda] : A[j + i * lda];
}

/* ------------------------------------------------------------------------ */
/* Step 1, SPD case ("SPOTRF"): A = L L^T, binary32, in place in  */
/* the lower triangle.  Column j: l_jj = sqrt(a_jj); l_ij = a_ij / l_jj;    */
/* then a_ik -= l_ij l_kj for j < k <= i (lower part of the trailing block).*/
/* Returns 0, or k + 1 when the pivot at column k is not > 0 (reading C-1). */
/* ------------------------------------------------------------------------ */
int oracle_spotf2(int64_t n, float *A, int64_t lda)
{
    for (int64_t j = 0; j < n; ++j) {
        float *aj = A + j * lda;
        const float d = aj[j];
        if (!(d > 0.0f)) return (int)(j + 1);
        const float ljj = sqrtf(d);
        aj[j] = ljj;
        for (int64_t i = j + 1; i < n; ++i) aj[i] = aj[i] / ljj;
#pragma omp parallel for schedule(static) if ((n - j) * (n - j) > 131072)
        for (int64_t k = j + 1; k < n; ++k) {
            float *ak = A + k * lda;
            const float lkj = aj[k];
            for (int64_t i = k; i < n; ++i) {
                float prod = aj[i] * lkj;
                ak[i] = ak[i] - prod;
            }
        }
    }
    return 0;
}

int oracle_dpotf2(int64_t n, double *A, int64_t lda)
{
    for (int64_t j = 0; j < n; ++j) {
        double *aj = A + j * lda;
        const double d = aj[j];
        if (!(d > 0.0)) return (int)(j + 1);
        const double ljj = sqrt(d);
        aj[j] = ljj;
        for (int64_t i = j + 1; i < n; ++i) aj[i] = aj[i] / ljj;
#pragma omp parallel for schedule(static) if ((n - j) * (n - j) > 131072)
        for (int64_t k = j + 1; k < n; ++k) {
            double *ak = A + k * lda;
            const double lkj = aj[k];
            for (int64_t i = k; i < n; ++i) {
                double prod = aj[i] * lkj;
                ak[i] = ak[i] - prod;
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Steps 2-3 / 5-6, SPD case ("SPOTRS"): L y = b (forward, column sweep,    */
/* divide by l_jj), then L^T x = y (backward; column j of L^T is row j of   */
/* L).  binary32; B is n x nrhs, ld n, overwritten by X.                    */
/* ------------------------------------------------------------------------ */
void oracle_spotrs(int64_t n, int64_t nrhs, const float *L, int64_t ldl, float *B)
{
#pragma omp parallel for schedule(static) if (nrhs > 1)
    for (int64_t c = 0; c < nrhs; ++c) {
        float *b = B + c * n;
        for (int64_t j = 0; j < n; ++j) {
            const float *l = L + j * ldl;
            b[j] = b[j] / l[j];
            const float yj = b[j];
            for (int64_t i = j + 1; i < n; ++i) {
                float prod = l[i] * yj;
                b[i] = b[i] - prod;
            }
        }
        for (int64_t j = n - 1; j >= 0; --j) {
            b[j] = b[j] / L[j + j * ldl];
            const float xj = b[j];
            for (int64_t i = 0; i < j; ++i) {
                float prod = L[j + i * ldl] * xj;               /* L^T(i, j) = L(j, i) */
                b[i] = b[i] - prod;
            }
        }
    }
}

void oracle_dpotrs(int64_t n, int64_t nrhs, const double *L, int64_t ldl, double *B)
{
#pragma omp parallel for schedule(static) if (nrhs > 1)
    for (int64_t c = 0; c < nrhs; ++c) {
        double *b = B + c * n;
        for (int64_t j = 0; j < n; ++j) {
            const double *l = L + j * ldl;
            b[j] = b[j] / l[j];
            const double yj = b[j];
            for (int64_t i = j + 1; i < n; ++i) {
                double prod = l[i] * yj;
                b[i] = b[i] - prod;
            }
        }
        for (int64_t j = n - 1; j >= 0; --j) {
            b[j] = b[j] / L[j + j * ldl];
            const double xj = b[j];
            for (int64_t i = 0; i < j; ++i) {
                double prod = L[j + i * ldl] * xj;
                b[i] = b[i] - prod;
            }
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Step 4, SPD case ("DSYMM"): r = b - A x in binary64 with the  */
/* symmetric A given by its lower triangle.  r_i = b_i; for j = 0..n-1:     */
/* r_i = r_i - a_sym(i, j) x_j (fixed j order).                             */
/* ------------------------------------------------------------------------ */
void oracle_symv_residual(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                          const double *B, const double *X, double *R)
{
    for (int64_t c = 0; c < nrhs; ++c) {
        const double *b = B + c * n, *x = X + c * n;
        double *r = R + c * n;
#pragma omp parallel for schedule(static) if (n >= 512)
        for (int64_t i = 0; i < n; ++i) {
            double ri = b[i];
            for (int64_t j = 0; j < n; ++j) {
                double prod = asym(A, lda, i, j) * x[j];
                ri = ri - prod;
            }
            r[i] = ri;
        }
    }
}

/* ||A||_F of the full symmetric matrix from its lower triangle (reading C-3). */
double oracle_sym_fro_norm(int64_t n, const double *A, int64_t lda)
{
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) {
            double a = asym(A, lda, i, j);
            double sq = a * a;
            s = s + sq;
        }
    return sqrt(s);
}

static double nrm2(int64_t n, const double *v)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) { double sq = v[i] * v[i]; s = s + sq; }
    return sqrt(s);
}

static int lower_nonfinite(int64_t n, const double *A, int64_t lda)
{
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = j; i < n; ++i)
            if (!isfinite(A[i + j * lda])) return 1;
    return 0;
}

static int any_nonfinite(int64_t cnt, const double *v)
{
    for (int64_t t = 0; t < cnt; ++t)
        if (!isfinite(v[t])) return 1;
    return 0;
}

static int args_bad(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, const double *X,
                    int *info)
{
    int64_t mx = n > 1 ? n : 1;
    if (n < 0) { *info = -1; return 1; }
    if (nrhs < 0) { *info = -2; return 1; }
    if (n > 0 && A == NULL) { *info = -3; return 1; }
    if (lda < mx) { *info = -4; return 1; }
    if (n > 0 && nrhs > 0 && B == NULL) { *info = -5; return 1; }
    if (n > 0 && nrhs > 0 && X == NULL) { *info = -6; return 1; }
    return 0;
}

/* The binary64 SPD solver (fallback and mp_dposv semantics): Cholesky + the two solves,
   no refinement.  Returns info: 0, or k + 1 at a breakdown in column k (reading C-2). */
static int dposv_body(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X)
{
    double *W = (double *)malloc((size_t)n * n * sizeof(double));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = j; i < n; ++i) W[i + j * n] = A[i + j * lda];
    int z = oracle_dpotf2(n, W, n);
    if (z == 0) {
        memcpy(X, B, (size_t)n * nrhs * sizeof(double));
        oracle_dpotrs(n, nrhs, W, n, X);
    }
    free(W);
    return z;
}

int oracle_dposv(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int *info)
{
    *info = 0;
    if (args_bad(n, nrhs, A, lda, B, X, info)) return 0;
    if (n == 0 || nrhs == 0) return 0;
    if (lower_nonfinite(n, A, lda)) { *info = -3; return 0; }
    if (any_nonfinite(n * nrhs, B)) { *info = -5; return 0; }
    *info = dposv_body(n, nrhs, A, lda, B, X);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1 in its SPD form (P:112-127 with P:369-371), B:5's stop test, */
/* cap and fallback.  iters: >= 0 corrections; -2 demotion overflow; -3 the */
/* binary32 Cholesky broke down (C-1); -31 no convergence.  iters < 0: X is */
/* the binary64 Cholesky solution; info = k + 1 if that one breaks down.    */
/* ------------------------------------------------------------------------ */
int oracle_dsposv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X,
                     int *iters, int *info, int itermax, double *hist, int *nhist, double *anrm_out)
{
    *info = 0; *iters = 0;
    if (nhist) *nhist = 0;
    if (args_bad(n, nrhs, A, lda, B, X, info)) return 0;
    if (n == 0 || nrhs == 0) return 0;
    if (lower_nonfinite(n, A, lda)) { *info = -3; return 0; }
    if (any_nonfinite(n * nrhs, B)) { *info = -5; return 0; }

    const double anrm = oracle_sym_fro_norm(n, A, lda);
    if (anrm_out) *anrm_out = anrm;
    const double cte = anrm * ldexp(1.0, -53) * sqrt((double)n);

    float *Ls = (float *)calloc((size_t)n * n, sizeof(float));
    float *Ws = (float *)malloc((size_t)n * nrhs * sizeof(float));
    double *R = (double *)malloc((size_t)n * nrhs * sizeof(double));
    int code = 0;
    for (int64_t j = 0; j < n && !code; ++j)
        for (int64_t i = j; i < n; ++i) {
            float v = (float)A[i + j * lda];
            if (isinf(v)) { code = -2; break; }
            Ls[i + j * n] = v;
        }
    if (!code && oracle_spotf2(n, Ls, n) != 0) code = -3;                 /* step 1 */
    if (!code) {
        for (int64_t t = 0; t < n * nrhs; ++t) Ws[t] = (float)B[t];
        oracle_spotrs(n, nrhs, Ls, n, Ws);                                 /* steps 2-3 */
        for (int64_t t = 0; t < n * nrhs; ++t) X[t] = (double)Ws[t];
        code = -31;
        for (int it = 0; it <= itermax; ++it) {
            oracle_symv_residual(n, nrhs, A, lda, B, X, R);                /* step 4 */
            int conv = 1, bad = 0;
            double worst = 0.0;
            for (int64_t c = 0; c < nrhs; ++c) {
                double rn = nrm2(n, R + c * n), xn = nrm2(n, X + c * n);
                if (!isfinite(rn) || !isfinite(xn)) { bad = 1; break; }
                double ratio = (rn == 0.0) ? 0.0 : rn / (xn * cte);
                if (ratio > worst || isnan(ratio)) worst = ratio;
                if (!(rn < xn * cte || rn == 0.0)) conv = 0;
            }
            if (hist && !bad) hist[it] = worst;
            if (nhist && !bad) *nhist = it + 1;
            if (bad) break;
            if (conv) { *iters = it; code = 0; break; }
            if (it == itermax) break;
            for (int64_t t = 0; t < n * nrhs; ++t) Ws[t] = (float)R[t];
            oracle_spotrs(n, nrhs, Ls, n, Ws);                             /* steps 5-6 */
            for (int64_t t = 0; t < n * nrhs; ++t) X[t] = X[t] + (double)Ws[t];   /* step 7 */
        }
    }
    free(Ls); free(Ws); free(R);
    if (code) {
        *iters = code;
        *info = dposv_body(n, nrhs, A, lda, B, X);
    }
    return 0;
}
