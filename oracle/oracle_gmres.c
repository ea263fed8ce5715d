/*
 * oracle_gmres.c — plain CPU oracle for SURVEY.md §8(f) NEXT-3: PAPER.md Algorithm 2,
 * "Mixed precision, inner-outer FGMRES(m_out)-GMRES_SP(m_in)".
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.c's header).
 *
 * Algorithm 2 as printed:
 *   for i = 0, 1, ...
 *     r = b - A x_i; beta = h_{1,0} = ||r||_2                              (eps_d)
 *     check convergence and exit if done
 *     for k = 1 .. m_out
 *       v_k = r / h_{k,k-1}                                                 (eps_d)
 *       one cycle of GMRES_SP(m_in) to approximately solve A z_k = v_k, z_k = 0 initially (eps_s)
 *       r = A z_k; for j = 1..k: h_{j,k} = r^T v_j; r = r - h_{j,k} v_j     (eps_d)
 *       h_{k+1,k} = ||r||_2                                                 (eps_d)
 *     y_k = argmin ||beta e_1 - H_k y||_2;  x_{i+1} = x_i + Z_k y_k         (eps_d)
 *
 * Readings: G-1 the convergence check is B:5's backward test ||r||_2 < ||x||_2 ||A||_F
 * 2^-53 sqrt(n) (or r == 0), at the top of every outer cycle as printed (the paper's own code checks at
 * every inner iteration); G-2 at most 30 outer cycles, then iters = -31 with the last iterate
 * (no fallback: the paper's iterative solvers have none); G-3 GMRES_SP is the textbook GMRES with
 * modified Gram-Schmidt Arnoldi, started from z = 0, run for m_in steps (fewer on a happy breakdown,
 * h_{j+1,j} == 0), its least-squares problem solved with Givens rotations, all in binary32 with the
 * binary32 copy of A ("single precision arithmetic matrix-vector product"); G-4 an outer
 * cycle stops early at a happy breakdown (h_{k+1,k} == 0) and uses the k columns it has; G-5 the outer
 * least-squares problem is solved with Givens rotations in binary64.
 * Arithmetic: -ffp-contract=off, fixed loop orders.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_ITERMAX 30

double oracle_fro_norm(int64_t n, const double *A, int64_t lda);   /* oracle.c */

/* y = A x, binary64, A column-major; y_i = sum_j a_ij x_j in increasing j */
static void gemv_d(int64_t n, const double *A, int64_t lda, const double *x, double *y)
{
#pragma omp parallel for schedule(static) if (n >= 512)
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) { double p = A[i + j * lda] * x[j]; s = s + p; }
        y[i] = s;
    }
}

/* y = A32 x, binary32 (A32 column-major) */
static void gemv_s(int64_t n, const float *A, int64_t lda, const float *x, float *y)
{
#pragma omp parallel for schedule(static) if (n >= 512)
    for (int64_t i = 0; i < n; ++i) {
        float s = 0.0f;
        for (int64_t j = 0; j < n; ++j) { float p = A[i + j * lda] * x[j]; s = s + p; }
        y[i] = s;
    }
}

static double dot_d(int64_t n, const double *a, const double *b)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) { double p = a[i] * b[i]; s = s + p; }
    return s;
}

static float dot_s(int64_t n, const float *a, const float *b)
{
    float s = 0.0f;
    for (int64_t i = 0; i < n; ++i) { float p = a[i] * b[i]; s = s + p; }
    return s;
}

/* Givens rotation (c, s) with c a + s b = r, -s a + c b = 0 (textbook, no scaling) */
static void givens_d(double a, double b, double *c, double *s)
{
    if (b == 0.0) { *c = 1.0; *s = 0.0; return; }
    double r = sqrt(a * a + b * b);
    *c = a / r; *s = b / r;
}

static void givens_s(float a, float b, float *c, float *s)
{
    if (b == 0.0f) { *c = 1.0f; *s = 0.0f; return; }
    float r = sqrtf(a * a + b * b);
    *c = a / r; *s = b / r;
}

/* ------------------------------------------------------------------------ */
/* One cycle of GMRES_SP(m_in) for A32 z = v (reading G-3).  z (binary32)   */
/* out.  Returns the number of Arnoldi steps taken.                         */
/* ------------------------------------------------------------------------ */
int oracle_gmres_sp_cycle(int64_t n, const float *A32, int64_t lda, const float *v, int m, float *z)
{
    float *V = (float *)calloc((size_t)n * (m + 1), sizeof(float));
    float *H = (float *)calloc((size_t)(m + 1) * m, sizeof(float));     /* H[i + j (m+1)] */
    float *cs = (float *)calloc((size_t)m, sizeof(float)), *sn = (float *)calloc((size_t)m, sizeof(float));
    float *g = (float *)calloc((size_t)m + 1, sizeof(float)), *y = (float *)calloc((size_t)m, sizeof(float));
    float beta = sqrtf(dot_s(n, v, v));
    for (int64_t i = 0; i < n; ++i) z[i] = 0.0f;
    int steps = 0;
    if (beta == 0.0f) goto done;
    for (int64_t i = 0; i < n; ++i) V[i] = v[i] / beta;
    g[0] = beta;
    for (int j = 0; j < m; ++j) {
        float *w = V + (int64_t)(j + 1) * n;
        gemv_s(n, A32, lda, V + (int64_t)j * n, w);
        for (int i = 0; i <= j; ++i) {                                      /* modified Gram-Schmidt */
            const float h = dot_s(n, w, V + (int64_t)i * n);
            H[i + j * (m + 1)] = h;
            for (int64_t t = 0; t < n; ++t) { float p = h * V[t + (int64_t)i * n]; w[t] = w[t] - p; }
        }
        const float hn = sqrtf(dot_s(n, w, w));
        H[j + 1 + j * (m + 1)] = hn;
        steps = j + 1;
        for (int i = 0; i < j; ++i) {                                       /* previous rotations */
            const float a = H[i + j * (m + 1)], b = H[i + 1 + j * (m + 1)];
            H[i + j * (m + 1)] = cs[i] * a + sn[i] * b;
            H[i + 1 + j * (m + 1)] = -sn[i] * a + cs[i] * b;
        }
        givens_s(H[j + j * (m + 1)], H[j + 1 + j * (m + 1)], &cs[j], &sn[j]);
        H[j + j * (m + 1)] = cs[j] * H[j + j * (m + 1)] + sn[j] * H[j + 1 + j * (m + 1)];
        H[j + 1 + j * (m + 1)] = 0.0f;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        if (hn == 0.0f) break;                                              /* happy breakdown */
        for (int64_t t = 0; t < n; ++t) w[t] = w[t] / hn;
    }
    for (int i = steps - 1; i >= 0; --i) {                                  /* R y = g */
        float s = g[i];
        for (int l = i + 1; l < steps; ++l) { float p = H[i + l * (m + 1)] * y[l]; s = s - p; }
        y[i] = s / H[i + i * (m + 1)];
    }
    for (int i = 0; i < steps; ++i)
        for (int64_t t = 0; t < n; ++t) { float p = y[i] * V[t + (int64_t)i * n]; z[t] = z[t] + p; }
done:
    free(V); free(H); free(cs); free(sn); free(g); free(y);
    return steps;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 2.  x in/out (initial guess, binary64).  iters = outer cycles  */
/* performed before convergence (0: x passed); -31 no convergence (G-2).    */
/* hist[i] = ||r_i|| / (||x_i|| ||A||_F 2^-53 sqrt(n)) at each check.       */
/* ------------------------------------------------------------------------ */
int oracle_fgmres_ex(int64_t n, const double *A, int64_t lda, const double *b, double *x, int m_out, int m_in,
                     int *iters, int *info, int itermax, double *hist, int *nhist)
{
    *info = 0; *iters = 0;
    if (nhist) *nhist = 0;
    if (n < 0) { *info = -1; return 0; }
    if (lda < (n > 1 ? n : 1)) { *info = -3; return 0; }
    if (m_out < 1 || m_in < 1) { *info = -6; return 0; }
    if (n == 0) return 0;
    const double cte = oracle_fro_norm(n, A, lda) * ldexp(1.0, -53) * sqrt((double)n);
    float *A32 = (float *)malloc((size_t)n * n * sizeof(float));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) A32[i + j * n] = (float)A[i + j * lda];
    double *V = (double *)calloc((size_t)n * (m_out + 1), sizeof(double));
    double *Z = (double *)calloc((size_t)n * m_out, sizeof(double));
    double *H = (double *)calloc((size_t)(m_out + 1) * m_out, sizeof(double));
    double *cs = (double *)calloc((size_t)m_out, sizeof(double)), *sn = (double *)calloc((size_t)m_out, sizeof(double));
    double *g = (double *)calloc((size_t)m_out + 1, sizeof(double)), *y = (double *)calloc((size_t)m_out, sizeof(double));
    double *r = (double *)malloc((size_t)n * sizeof(double));
    float *vs = (float *)malloc((size_t)n * sizeof(float)), *zs = (float *)malloc((size_t)n * sizeof(float));
    *iters = -31;
    for (int it = 0; it <= itermax; ++it) {
        gemv_d(n, A, lda, x, r);
        for (int64_t t = 0; t < n; ++t) r[t] = b[t] - r[t];                  /* r = b - A x_i */
        const double beta = sqrt(dot_d(n, r, r)), xn = sqrt(dot_d(n, x, x));
        if (!isfinite(beta) || !isfinite(xn)) break;
        if (hist) hist[it] = beta == 0.0 ? 0.0 : beta / (xn * cte);
        if (nhist) *nhist = it + 1;
        if (beta < xn * cte || beta == 0.0) { *iters = it; break; }         /* G-1 */
        if (it == itermax) break;
        memset(g, 0, (size_t)(m_out + 1) * sizeof(double));
        g[0] = beta;
        double hprev = beta;
        int kk = 0;
        for (int k = 0; k < m_out; ++k) {
            double *vk = V + (int64_t)k * n;
            for (int64_t t = 0; t < n; ++t) vk[t] = r[t] / hprev;            /* v_k = r / h_{k,k-1} */
            for (int64_t t = 0; t < n; ++t) vs[t] = (float)vk[t];
            oracle_gmres_sp_cycle(n, A32, n, vs, m_in, zs);                  /* z_k ~ A^-1 v_k (eps_s) */
            double *zk = Z + (int64_t)k * n;
            for (int64_t t = 0; t < n; ++t) zk[t] = (double)zs[t];
            gemv_d(n, A, lda, zk, r);                                        /* r = A z_k */
            for (int j = 0; j <= k; ++j) {                                   /* MGS, eps_d */
                const double h = dot_d(n, r, V + (int64_t)j * n);
                H[j + k * (m_out + 1)] = h;
                for (int64_t t = 0; t < n; ++t) { double p = h * V[t + (int64_t)j * n]; r[t] = r[t] - p; }
            }
            const double hn = sqrt(dot_d(n, r, r));
            H[k + 1 + k * (m_out + 1)] = hn;
            kk = k + 1;
            for (int i = 0; i < k; ++i) {
                const double a = H[i + k * (m_out + 1)], bb = H[i + 1 + k * (m_out + 1)];
                H[i + k * (m_out + 1)] = cs[i] * a + sn[i] * bb;
                H[i + 1 + k * (m_out + 1)] = -sn[i] * a + cs[i] * bb;
            }
            givens_d(H[k + k * (m_out + 1)], H[k + 1 + k * (m_out + 1)], &cs[k], &sn[k]);
            H[k + k * (m_out + 1)] = cs[k] * H[k + k * (m_out + 1)] + sn[k] * H[k + 1 + k * (m_out + 1)];
            H[k + 1 + k * (m_out + 1)] = 0.0;
            g[k + 1] = -sn[k] * g[k];
            g[k] = cs[k] * g[k];
            if (hn == 0.0) break;                                            /* G-4 */
            hprev = hn;
        }
        for (int i = kk - 1; i >= 0; --i) {
            double s = g[i];
            for (int l = i + 1; l < kk; ++l) { double p = H[i + l * (m_out + 1)] * y[l]; s = s - p; }
            y[i] = s / H[i + i * (m_out + 1)];
        }
        for (int i = 0; i < kk; ++i)
            for (int64_t t = 0; t < n; ++t) { double p = y[i] * Z[t + (int64_t)i * n]; x[t] = x[t] + p; }
    }
    free(A32); free(V); free(Z); free(H); free(cs); free(sn); free(g); free(y); free(r); free(vs); free(zs);
    return 0;
}
