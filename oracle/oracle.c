/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for the mixed-precision
 * iterative-refinement solve of arXiv 0808.2794 (Algorithm 1).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path (the CUDA library
 * under paper_0808_2794_b200/) may link, import or call this file; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg use it.  It shares no code, header, table or helper with the
 * GPU path.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n; B:5 = BASELINE.json
 * north_star; S:n = SPEC.md line n (interfaces/examples only); A-k = a reading
 * listed in DESIGN.md "Readings of the paper" (= SURVEY.md §8(c) A-k).
 *
 * Conventions (mirroring include/mp_solve.h, but declared independently here):
 *   A is n x n, column-major, leading dimension lda >= max(1,n); entry (i,j)
 *   at A[i + j*lda].  B, X are n x nrhs column-major with leading dimension n.
 *   Pivots ipiv[k] are 0-based row indices (LAPACK-style sequential list:
 *   at step k rows k and ipiv[k] were interchanged).
 *
 * Arithmetic: compiled with -ffp-contract=off -fno-fast-math (no FMA
 * contraction, IEEE binary32 / binary64 round-to-nearest-even).  Every loop
 * runs in a fixed order; OpenMP only splits independent columns (rank-1
 * update, triangular solves per right-hand side) or independent rows
 * (residual), so results do not depend on the thread count.
 *
 * Pins (tests/test_oracle_*.py): exact rational elimination on small integer
 * systems (P1), constructed exact-LU family (P2, bitwise), SPEC worked
 * examples (P3), closed forms (P4), invariants (P5), LAPACK special cases
 * (P6), forward-error bound for prescribed-kappa inputs (P8), long-double
 * certificate (P9).  Every function below is pinned by at least one of them.
 */
#include <math.h>
#include <float.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_ITERMAX 30 /* P:625-627 "maximum number of iterations allowed was set to 30"; B:5 */

/* ------------------------------------------------------------------------ */
/* Step 1 of Alg. 1: LU <- PA by Gaussian elimination with  */
/* partial row pivoting, textbook right-looking (kji) order, binary32.       */
/* Pivot: largest |a_ik| on/below the diagonal, smallest row index on ties   */
/* (S:137).  Exact zero pivot -> return k+1 and stop.                */
/* ------------------------------------------------------------------------ */
int oracle_sgetf2(int64_t n, float *A, int64_t lda, int32_t *ipiv)
{
    for (int64_t k = 0; k < n; ++k) {
        float *ak = A + k * lda;
        int64_t p = k;
        float amax = fabsf(ak[k]);
        for (int64_t i = k + 1; i < n; ++i) {
            float v = fabsf(ak[i]);
            if (v > amax) { amax = v; p = i; }   /* strict '>' : first max wins */
        }
        ipiv[k] = (int32_t)p;
        if (ak[p] == 0.0f) return (int)(k + 1);
        if (p != k) {                            /* interchange rows k and p over all n columns */
            for (int64_t j = 0; j < n; ++j) {
                float t = A[k + j * lda];
                A[k + j * lda] = A[p + j * lda];
                A[p + j * lda] = t;
            }
        }
        const float piv = ak[k];
        for (int64_t i = k + 1; i < n; ++i) ak[i] = ak[i] / piv;   /* multipliers l_ik (A-7: divide) */
#pragma omp parallel for schedule(static) if ((n - k) * (n - k) > 65536)
        for (int64_t j = k + 1; j < n; ++j) {                      /* rank-1 update of the trailing matrix */
            float *aj = A + j * lda;
            const float ukj = aj[k];
            for (int64_t i = k + 1; i < n; ++i) {
                float prod = ak[i] * ukj;                           /* separate multiply ...   */
                aj[i] = aj[i] - prod;                               /* ... and subtract (A-8)  */
            }
        }
    }
    return 0;
}

/* Same elimination in binary64: the full double-precision solver used as the  */
/* fallback "standard double precision solver" and for mp_dgesv.  */
int oracle_dgetf2(int64_t n, double *A, int64_t lda, int32_t *ipiv)
{
    for (int64_t k = 0; k < n; ++k) {
        double *ak = A + k * lda;
        int64_t p = k;
        double amax = fabs(ak[k]);
        for (int64_t i = k + 1; i < n; ++i) {
            double v = fabs(ak[i]);
            if (v > amax) { amax = v; p = i; }
        }
        ipiv[k] = (int32_t)p;
        if (ak[p] == 0.0) return (int)(k + 1);
        if (p != k) {
            for (int64_t j = 0; j < n; ++j) {
                double t = A[k + j * lda];
                A[k + j * lda] = A[p + j * lda];
                A[p + j * lda] = t;
            }
        }
        const double piv = ak[k];
        for (int64_t i = k + 1; i < n; ++i) ak[i] = ak[i] / piv;
#pragma omp parallel for schedule(static) if ((n - k) * (n - k) > 65536)
        for (int64_t j = k + 1; j < n; ++j) {
            double *aj = A + j * lda;
            const double ukj = aj[k];
            for (int64_t i = k + 1; i < n; ++i) {
                double prod = ak[i] * ukj;
                aj[i] = aj[i] - prod;
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Steps 2-3 / 5-6: apply P (the ipiv list   */
/* in order), solve L y = P b (unit lower, forward substitution), then       */
/* U x = y (backward substitution), all in binary32.  B is n x nrhs, ld n.   */
/* ------------------------------------------------------------------------ */
void oracle_sgetrs(int64_t n, int64_t nrhs, const float *LU, int64_t lda,
                   const int32_t *ipiv, float *B)
{
#pragma omp parallel for schedule(static) if (nrhs > 1)
    for (int64_t c = 0; c < nrhs; ++c) {
        float *b = B + c * n;
        for (int64_t k = 0; k < n; ++k) {                 /* b <- P b */
            int64_t p = ipiv[k];
            if (p != k) { float t = b[k]; b[k] = b[p]; b[p] = t; }
        }
        for (int64_t j = 0; j < n; ++j) {                 /* L y = P b, column sweep */
            const float yj = b[j];
            const float *l = LU + j * lda;
            for (int64_t i = j + 1; i < n; ++i) {
                float prod = l[i] * yj;
                b[i] = b[i] - prod;
            }
        }
        for (int64_t j = n - 1; j >= 0; --j) {            /* U x = y, column sweep */
            const float *u = LU + j * lda;
            b[j] = b[j] / u[j];
            const float xj = b[j];
            for (int64_t i = 0; i < j; ++i) {
                float prod = u[i] * xj;
                b[i] = b[i] - prod;
            }
        }
    }
}

void oracle_dgetrs(int64_t n, int64_t nrhs, const double *LU, int64_t lda,
                   const int32_t *ipiv, double *B)
{
#pragma omp parallel for schedule(static) if (nrhs > 1)
    for (int64_t c = 0; c < nrhs; ++c) {
        double *b = B + c * n;
        for (int64_t k = 0; k < n; ++k) {
            int64_t p = ipiv[k];
            if (p != k) { double t = b[k]; b[k] = b[p]; b[p] = t; }
        }
        for (int64_t j = 0; j < n; ++j) {
            const double yj = b[j];
            const double *l = LU + j * lda;
            for (int64_t i = j + 1; i < n; ++i) {
                double prod = l[i] * yj;
                b[i] = b[i] - prod;
            }
        }
        for (int64_t j = n - 1; j >= 0; --j) {
            const double *u = LU + j * lda;
            b[j] = b[j] / u[j];
            const double xj = b[j];
            for (int64_t i = 0; i < j; ++i) {
                double prod = u[i] * xj;
                b[i] = b[i] - prod;
            }
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Step 4: r = b - A x in binary64 with the ORIGINAL A.   */
/* r_i = b_i; for j = 0..n-1: r_i = r_i - a_ij x_j   (fixed j order).        */
/* ------------------------------------------------------------------------ */
void oracle_residual(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                     const double *B, const double *X, double *R)
{
    const int64_t RB = 256;                               /* independent row blocks */
    const int64_t nblk = (n + RB - 1) / RB;
    for (int64_t c = 0; c < nrhs; ++c) {
        const double *b = B + c * n, *x = X + c * n;
        double *r = R + c * n;
#pragma omp parallel for schedule(static) if (n >= 512)
        for (int64_t ib = 0; ib < nblk; ++ib) {
            int64_t i0 = ib * RB, i1 = i0 + RB < n ? i0 + RB : n;
            for (int64_t i = i0; i < i1; ++i) r[i] = b[i];
            for (int64_t j = 0; j < n; ++j) {
                const double xj = x[j];
                const double *a = A + j * lda;
                for (int64_t i = i0; i < i1; ++i) {
                    double prod = a[i] * xj;
                    r[i] = r[i] - prod;
                }
            }
        }
    }
}

/* ||A||_F, computed once from the original binary64 A (B:5 Frobenius; A-2). */
double oracle_fro_norm(int64_t n, const double *A, int64_t lda)
{
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) {
            double a = A[i + j * lda];
            double sq = a * a;
            s = s + sq;
        }
    return sqrt(s);
}

/* plain 2-norm of one column vector */
static double vec_nrm2(int64_t n, const double *v)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) { double sq = v[i] * v[i]; s = s + sq; }
    return sqrt(s);
}

static int has_nonfinite(int64_t rows, int64_t cols, const double *M, int64_t ld)
{
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i)
            if (!isfinite(M[i + j * ld])) return 1;
    return 0;
}

static int overlaps(const void *a, size_t abytes, const void *b, size_t bbytes)
{
    const char *pa = (const char *)a, *pb = (const char *)b;
    return pa < pb + bbytes && pb < pa + abytes;
}

/* ------------------------------------------------------------------------ */
/* Full binary64 solver: GEPP + substitution, no refinement (A-11).          */
/* Returns info: 0 ok, k+1 when U(k,k) is an exact zero.                     */
/* ------------------------------------------------------------------------ */
static int dgesv_body(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                      const double *B, double *X)
{
    double *W = (double *)malloc((size_t)n * n * sizeof(double));
    int32_t *ipiv = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    for (int64_t j = 0; j < n; ++j) memcpy(W + j * n, A + j * lda, (size_t)n * sizeof(double));
    int z = oracle_dgetf2(n, W, n, ipiv);
    if (z == 0) {
        memcpy(X, B, (size_t)n * nrhs * sizeof(double));
        oracle_dgetrs(n, nrhs, W, n, ipiv, X);
    }
    free(W); free(ipiv);
    return z;
}

static int check_args(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                      const double *B, const double *X, int *info)
{
    int64_t mx = n > 1 ? n : 1;
    if (n < 0) { *info = -1; return 1; }
    if (nrhs < 0) { *info = -2; return 1; }
    if (n > 0 && A == NULL) { *info = -3; return 1; }
    if (lda < mx) { *info = -4; return 1; }
    if (n > 0 && nrhs > 0 && B == NULL) { *info = -5; return 1; }
    if (n > 0 && nrhs > 0 && X == NULL) { *info = -6; return 1; }
    if (n > 0 && nrhs > 0) {
        size_t xb = (size_t)n * nrhs * sizeof(double);
        size_t ab = (size_t)((n - 1) * lda + n) * sizeof(double);
        if (overlaps(X, xb, A, ab) || overlaps(X, xb, B, xb)) { *info = -6; return 1; }
    }
    return 0;
}

/* oracle_dgesv: the "standard double precision solver". */
int oracle_dgesv(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                 const double *B, double *X, int *info)
{
    *info = 0;
    if (check_args(n, nrhs, A, lda, B, X, info)) return 0;
    if (n == 0 || nrhs == 0) return 0;
    if (has_nonfinite(n, n, A, lda)) { *info = -3; return 0; }
    if (has_nonfinite(n, nrhs, B, n)) { *info = -5; return 0; }
    *info = dgesv_body(n, nrhs, A, lda, B, X);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1, mixed binary32 / binary64, with B:5's stop test  */
/*   converged  <=>  for every column c:  rn_c < xn_c * ||A||_F * 2^-53 * sqrt(n)  */
/*                   or rn_c == 0        (A-1, A-2, A-3, A-5)                */
/* and the 30-correction cap / binary64 fallback.     */
/*                                                                           */
/* iters >= 0 : number of corrections applied (A-4)                          */
/* iters = -2 : a finite entry of A overflowed on demotion            */
/* iters = -3 : exact zero pivot in the binary32 LU                  */
/* iters = -31: no convergence within 30 corrections or non-finite norms     */
/* When iters < 0 the binary64 solver produced X (A-11).                     */
/*                                                                           */
/* hist (optional, length itermax+1): ratio max_c rn_c / (xn_c*cte) per     */
/* residual check; *nhist receives the number of entries written.            */
/* itermax: pass 30 (B:5); exposed only so tests can probe the cap.          */
/* ------------------------------------------------------------------------ */
int oracle_dsgesv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                     const double *B, double *X, int *iters, int *info,
                     int itermax, double *hist, int *nhist, double *anrm_out)
{
    *info = 0; *iters = 0;
    if (nhist) *nhist = 0;
    if (check_args(n, nrhs, A, lda, B, X, info)) return 0;
    if (n == 0 || nrhs == 0) return 0;
    if (has_nonfinite(n, n, A, lda)) { *info = -3; return 0; }      /* A-6 */
    if (has_nonfinite(n, nrhs, B, n)) { *info = -5; return 0; }

    const double anrm = oracle_fro_norm(n, A, lda);
    if (anrm_out) *anrm_out = anrm;
    const double cte = anrm * ldexp(1.0, -53) * sqrt((double)n);   /* eps_64 = 2^-53 (A-1) */

    /* demotion "converted to single precision", RN-even */
    float *As = (float *)malloc((size_t)n * n * sizeof(float));
    int32_t *ipiv = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    float *Ws = (float *)malloc((size_t)n * nrhs * sizeof(float));
    double *R = (double *)malloc((size_t)n * nrhs * sizeof(double));
    int code = 0;
    for (int64_t j = 0; j < n && !code; ++j)
        for (int64_t i = 0; i < n; ++i) {
            float v = (float)A[i + j * lda];
            if (isinf(v)) { code = -2; break; }
            As[i + j * n] = v;
        }
    if (!code && oracle_sgetf2(n, As, n, ipiv) != 0) code = -3;      /* step 1 */

    if (!code) {
        /* steps 2-3: x0 = (double) LUsolve_32((float) b)   (A-14) */
        for (int64_t t = 0; t < n * nrhs; ++t) Ws[t] = (float)B[t];
        oracle_sgetrs(n, nrhs, As, n, ipiv, Ws);
        for (int64_t t = 0; t < n * nrhs; ++t) X[t] = (double)Ws[t];
        code = -31;
        for (int it = 0; it <= itermax; ++it) {
            oracle_residual(n, nrhs, A, lda, B, X, R);             /* step 4 (eps_d) */
            int conv = 1, bad = 0;
            double worst = 0.0;
            for (int64_t c = 0; c < nrhs; ++c) {
                double rn = vec_nrm2(n, R + c * n), xn = vec_nrm2(n, X + c * n);
                if (!isfinite(rn) || !isfinite(xn)) { bad = 1; break; }
                double ratio = (rn == 0.0) ? 0.0 : rn / (xn * cte);
                if (ratio > worst || isnan(ratio)) worst = ratio;
                if (!(rn < xn * cte || rn == 0.0)) conv = 0;
            }
            if (hist && !bad) hist[it] = worst;
            if (nhist && !bad) *nhist = it + 1;
            if (bad) break;                                      /* -> fallback -31 */
            if (conv) { *iters = it; code = 0; break; }          /* check convergence */
            if (it == itermax) break;                            /* 30 corrections used */
            for (int64_t t = 0; t < n * nrhs; ++t) Ws[t] = (float)R[t];   /* A-10: no scaling */
            oracle_sgetrs(n, nrhs, As, n, ipiv, Ws);             /* steps 5-6 (eps_s) */
            for (int64_t t = 0; t < n * nrhs; ++t) X[t] = X[t] + (double)Ws[t];  /* step 7 (eps_d) */
        }
    }
    free(As); free(ipiv); free(Ws); free(R);
    if (code) {                                                  /* fall back */
        *iters = code;
        *info = dgesv_body(n, nrhs, A, lda, B, X);
    }
    return 0;
}

int oracle_dsgesv(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                  const double *B, double *X, int *iters, int *info)
{
    return oracle_dsgesv_ex(n, nrhs, A, lda, B, X, iters, info, OR_ITERMAX, NULL, NULL, NULL);
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
