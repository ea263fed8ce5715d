/*
 * oracle_lp.c — plain CPU oracle for SURVEY.md §8(f) NEXT-2: the lower-precision tensor-core
 * factorisation and its refinement.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.c's header).
 *
 * The paper's premise is that the O(n^3) work runs in the fastest arithmetic
 * the hardware has and refinement restores binary64 accuracy, as long as kappa(A) * eps_s < 1
 * (P:600-605).  On B200 the fastest FP32-input arithmetic is the TF32 tensor-core product: operands
 * rounded to 10 stored significand bits (u_f = 2^-11), binary32 accumulation.
 *
 * Readings (T-1..T-4):
 *  T-1 "TF32 factorisation": a blocked right-looking GEPP with panel width nb.  The panel (unblocked
 *      kji elimination, oracle_sgetf2's arithmetic) and the triangular solve for U12 run in binary32;
 *      every trailing update A22 -= L21 U12 takes the operands rounded to TF32 (round to nearest, ties
 *      away from zero: cvt.rna.tf32.f32) and accumulates the exact products in binary32 in
 *      increasing k.  The stored factors keep their binary32 values; only the update operands are
 *      rounded.
 *  T-2 refinement with these factors is Algorithm 1 unchanged (oracle_dsgesv_ex's loop).
 *  T-3 GMRES-IR: x0 = LUsolve(fl32(b)); restarted FGMRES(m) in binary64 on A x = b starting from
 *      x0, every direction preconditioned by the binary32 LU solve z_k = LUsolve(fl32(v_k)), modified
 *      Gram-Schmidt and Givens rotations in binary64 (Algorithm 2's outer solver with the factors as
 *      the inner solver).  B:5's test at the top of every restart; a cycle ends early when its
 *      Givens residual estimate |g_{k+1}| < ||x||_2 ||A||_F 2^-53 sqrt(n) / 2 (||x|| at the cycle
 *      start) or at an exact breakdown.
 *  T-4 iters = LU-solve applications after x0 (the analog of Algorithm 1's corrections); at most
 *      itermax (30); a column that fails -> iters = -31 and the binary64 fallback.
 *
 * Arithmetic: -ffp-contract=off; fixed loop orders.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int oracle_sgetf2(int64_t n, float *A, int64_t lda, int32_t *ipiv);                       /* oracle.c */
void oracle_sgetrs(int64_t n, int64_t nrhs, const float *LU, int64_t lda, const int32_t *ipiv, float *B);
int oracle_dgesv(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int *info);
double oracle_fro_norm(int64_t n, const double *A, int64_t lda);

/* round to TF32: nearest, ties away from zero, 13 low significand bits cleared (T-1) */
float oracle_rna_tf32(float x)
{
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return x;     /* inf / nan */
    u = (u + 0x1000u) & ~0x1fffu;                         /* add half an ulp of the magnitude, truncate */
    float r;
    memcpy(&r, &u, 4);
    return r;
}

void oracle_rna_tf32_array(int64_t n, const float *x, float *y)
{
    for (int64_t i = 0; i < n; ++i) y[i] = oracle_rna_tf32(x[i]);
}

/* ------------------------------------------------------------------------ */
/* T-1: blocked GEPP, TF32 trailing updates.  Returns 0 or k+1 (zero pivot). */
/* ------------------------------------------------------------------------ */
int oracle_sgetrf_tf32(int64_t n, float *A, int64_t lda, int64_t nb, int32_t *ipiv)
{
    if (nb < 1) nb = 1;
    for (int64_t k0 = 0; k0 < n; k0 += nb) {
        const int64_t w = (n - k0 < nb) ? n - k0 : nb, k1 = k0 + w;
        /* panel: columns [k0, k1), rows [k0, n), unblocked, interchanges over all n columns */
        for (int64_t k = k0; k < k1; ++k) {
            float *ak = A + k * lda;
            int64_t p = k;
            float amax = fabsf(ak[k]);
            for (int64_t i = k + 1; i < n; ++i) {
                float v = fabsf(ak[i]);
                if (v > amax) { amax = v; p = i; }
            }
            ipiv[k] = (int32_t)p;
            if (ak[p] == 0.0f) return (int)(k + 1);
            if (p != k)
                for (int64_t j = 0; j < n; ++j) {
                    float t = A[k + j * lda];
                    A[k + j * lda] = A[p + j * lda];
                    A[p + j * lda] = t;
                }
            const float piv = ak[k];
            for (int64_t i = k + 1; i < n; ++i) ak[i] = ak[i] / piv;
            for (int64_t j = k + 1; j < k1; ++j) {                 /* within the panel only */
                float *aj = A + j * lda;
                const float ukj = aj[k];
                for (int64_t i = k + 1; i < n; ++i) { float prod = ak[i] * ukj; aj[i] = aj[i] - prod; }
            }
        }
        if (k1 >= n) break;
        /* U12 = L11^-1 A12 (unit lower, binary32) */
        for (int64_t j = k1; j < n; ++j) {
            float *aj = A + j * lda;
            for (int64_t k = k0; k < k1; ++k) {
                const float ukj = aj[k];
                for (int64_t i = k + 1; i < k1; ++i) { float prod = A[i + k * lda] * ukj; aj[i] = aj[i] - prod; }
            }
        }
        /* A22 -= tf32(L21) tf32(U12), exact products, binary32 accumulation in increasing k */
#pragma omp parallel for schedule(static) if ((n - k1) * (n - k1) > 65536)
        for (int64_t j = k1; j < n; ++j) {
            float *aj = A + j * lda;
            for (int64_t i = k1; i < n; ++i) {
                float s = aj[i];
                for (int64_t k = k0; k < k1; ++k) {
                    float prod = oracle_rna_tf32(A[i + k * lda]) * oracle_rna_tf32(aj[k]);
                    s = s - prod;
                }
                aj[i] = s;
            }
        }
    }
    return 0;
}

/* ---------------------------------------------------------------- GMRES-IR (T-3) */
static void gemv(int64_t n, const double *A, int64_t lda, const double *x, double *y)
{
#pragma omp parallel for schedule(static) if (n >= 512)
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) { double p = A[i + j * lda] * x[j]; s = s + p; }
        y[i] = s;
    }
}

static double dot(int64_t n, const double *a, const double *b)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) { double p = a[i] * b[i]; s = s + p; }
    return s;
}

/* z = (double) LUsolve_32((float) v) */
static void precond(int64_t n, const float *LU, const int32_t *ipiv, const double *v, double *z, float *ws)
{
    for (int64_t t = 0; t < n; ++t) ws[t] = (float)v[t];
    oracle_sgetrs(n, 1, LU, n, ipiv, ws);
    for (int64_t t = 0; t < n; ++t) z[t] = (double)ws[t];
}

/* One column: x in/out (x0 in).  Returns LU applications used, -1 on failure (cap / non-finite). */
static int gmres_ir_column(int64_t n, const double *A, int64_t lda, const double *b, double *x, const float *LU,
                           const int32_t *ipiv, int m, int itermax, double cte, double *hist, int *nhist)
{
    double *V = (double *)calloc((size_t)n * (m + 1), sizeof(double));
    double *Z = (double *)calloc((size_t)n * m, sizeof(double));
    double *H = (double *)calloc((size_t)(m + 1) * m, sizeof(double));
    double *cs = (double *)calloc((size_t)m, sizeof(double)), *sn = (double *)calloc((size_t)m, sizeof(double));
    double *g = (double *)calloc((size_t)m + 1, sizeof(double)), *y = (double *)calloc((size_t)m, sizeof(double));
    double *r = (double *)malloc((size_t)n * sizeof(double));
    float *ws = (float *)malloc((size_t)n * sizeof(float));
    int apps = 0, result = -1;
    for (;;) {
        gemv(n, A, lda, x, r);
        for (int64_t t = 0; t < n; ++t) r[t] = b[t] - r[t];                   /* r = b - A x (eps_d) */
        const double beta = sqrt(dot(n, r, r)), xn = sqrt(dot(n, x, x));
        if (!isfinite(beta) || !isfinite(xn)) break;
        if (hist && *nhist < 64) hist[(*nhist)++] = beta == 0.0 ? 0.0 : beta / (xn * cte);
        if (beta < xn * cte || beta == 0.0) { result = apps; break; }        /* B:5 */
        if (apps >= itermax) break;
        memset(g, 0, (size_t)(m + 1) * sizeof(double));
        g[0] = beta;
        double hprev = beta;
        int kk = 0;
        for (int k = 0; k < m; ++k) {
            double *vk = V + (int64_t)k * n, *zk = Z + (int64_t)k * n;
            for (int64_t t = 0; t < n; ++t) vk[t] = r[t] / hprev;
            precond(n, LU, ipiv, vk, zk, ws);                                   /* z_k = M^-1 v_k */
            ++apps;
            gemv(n, A, lda, zk, r);                                             /* r = A z_k */
            for (int j = 0; j <= k; ++j) {                                      /* MGS (eps_d) */
                const double h = dot(n, r, V + (int64_t)j * n);
                H[j + k * (m + 1)] = h;
                for (int64_t t = 0; t < n; ++t) { double p = h * V[t + (int64_t)j * n]; r[t] = r[t] - p; }
            }
            const double hn = sqrt(dot(n, r, r));
            H[k + 1 + k * (m + 1)] = hn;
            kk = k + 1;
            for (int i = 0; i < k; ++i) {
                const double a = H[i + k * (m + 1)], bb = H[i + 1 + k * (m + 1)];
                H[i + k * (m + 1)] = cs[i] * a + sn[i] * bb;
                H[i + 1 + k * (m + 1)] = -sn[i] * a + cs[i] * bb;
            }
            {
                const double a = H[k + k * (m + 1)], bb = H[k + 1 + k * (m + 1)];
                double c = 1.0, s = 0.0;
                if (bb != 0.0) { const double rr = sqrt(a * a + bb * bb); c = a / rr; s = bb / rr; }
                cs[k] = c; sn[k] = s;
                H[k + k * (m + 1)] = c * a + s * bb;
                H[k + 1 + k * (m + 1)] = 0.0;
                g[k + 1] = -s * g[k];
                g[k] = c * g[k];
            }
            if (hn == 0.0) break;                                               /* exact breakdown */
            if (fabs(g[k + 1]) < 0.5 * xn * cte) break;                         /* T-3 early end */
            if (apps >= itermax) break;
            hprev = hn;
        }
        for (int i = kk - 1; i >= 0; --i) {
            double s = g[i];
            for (int l = i + 1; l < kk; ++l) { double p = H[i + l * (m + 1)] * y[l]; s = s - p; }
            const double d = H[i + i * (m + 1)];
            y[i] = d == 0.0 ? 0.0 : s / d;
        }
        for (int i = 0; i < kk; ++i)
            for (int64_t t = 0; t < n; ++t) { double p = y[i] * Z[t + (int64_t)i * n]; x[t] = x[t] + p; }
    }
    free(V); free(Z); free(H); free(cs); free(sn); free(g); free(y); free(r); free(ws);
    return result;
}

/* ------------------------------------------------------------------------ */
/* The NEXT-2 solve: factor fl32(A) (tf32 != 0: T-1 with panel nb; else      */
/* oracle_sgetf2), x0, then GMRES-IR(m) (T-3) per column.  iters: max LU     */
/* applications over the columns, or -31 (then X = the binary64 solution),   */
/* -3 zero pivot in the binary32 LU (X = binary64 solution).  info as        */
/* oracle_dsgesv_ex.  hist: column 0's per-restart ratios.                   */
/* ------------------------------------------------------------------------ */
int oracle_gmres_ir_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int tf32,
                       int64_t nb, int m, int itermax, int *iters, int *info, double *hist, int *nhist)
{
    *info = 0; *iters = 0;
    if (nhist) *nhist = 0;
    if (n < 0) { *info = -1; return 0; }
    if (nrhs < 0) { *info = -2; return 0; }
    if (lda < (n > 1 ? n : 1)) { *info = -4; return 0; }
    if (m < 1 || m > 31) { *info = -9; return 0; }
    if (n == 0 || nrhs == 0) return 0;
    const double cte = oracle_fro_norm(n, A, lda) * ldexp(1.0, -53) * sqrt((double)n);
    float *LU = (float *)malloc((size_t)n * n * sizeof(float));
    int32_t *ipiv = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    float *ws = (float *)malloc((size_t)n * sizeof(float));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) LU[i + j * n] = (float)A[i + j * lda];
    int code = tf32 ? oracle_sgetrf_tf32(n, LU, n, nb, ipiv) : oracle_sgetf2(n, LU, n, ipiv);
    code = code ? -3 : 0;
    int worst = 0;
    int nh = 0;
    for (int64_t c = 0; c < nrhs && !code; ++c) {
        double *x = X + c * n;
        for (int64_t t = 0; t < n; ++t) ws[t] = (float)B[t + c * n];
        oracle_sgetrs(n, 1, LU, n, ipiv, ws);                                    /* x0 */
        for (int64_t t = 0; t < n; ++t) x[t] = (double)ws[t];
        const int a = gmres_ir_column(n, A, lda, B + c * n, x, LU, ipiv, m, itermax, cte, c == 0 ? hist : NULL,
                                      &nh);
        if (a < 0) code = -31;
        else if (a > worst) worst = a;
    }
    if (nhist) *nhist = nh;
    *iters = code ? code : worst;
    if (code) oracle_dgesv(n, nrhs, A, lda, B, X, info);
    free(LU); free(ipiv); free(ws);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* T-2: Algorithm 1 unchanged, with the T-1 factors (panel nb).  */
/* Codes as oracle_dsgesv_ex: iters >= 0 corrections, -3 zero pivot, -31 no  */
/* convergence (X then from the binary64 solver).                */
/* ------------------------------------------------------------------------ */
int oracle_dsgesv_tf32_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X,
                          int64_t nb, int *iters, int *info, int itermax, double *hist, int *nhist)
{
    *info = 0; *iters = 0;
    if (nhist) *nhist = 0;
    if (n < 0) { *info = -1; return 0; }
    if (nrhs < 0) { *info = -2; return 0; }
    if (lda < (n > 1 ? n : 1)) { *info = -4; return 0; }
    if (n == 0 || nrhs == 0) return 0;
    const double cte = oracle_fro_norm(n, A, lda) * ldexp(1.0, -53) * sqrt((double)n);
    float *LU = (float *)malloc((size_t)n * n * sizeof(float));
    int32_t *ipiv = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    float *Ws = (float *)malloc((size_t)n * nrhs * sizeof(float));
    double *R = (double *)malloc((size_t)n * nrhs * sizeof(double));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) LU[i + j * n] = (float)A[i + j * lda];
    int code = oracle_sgetrf_tf32(n, LU, n, nb, ipiv) ? -3 : 0;                /* step 1 (T-1) */
    if (!code) {
        for (int64_t t = 0; t < n * nrhs; ++t) Ws[t] = (float)B[t];
        oracle_sgetrs(n, nrhs, LU, n, ipiv, Ws);                                 /* steps 2-3 */
        for (int64_t t = 0; t < n * nrhs; ++t) X[t] = (double)Ws[t];
        code = -31;
        for (int it = 0; it <= itermax; ++it) {
            for (int64_t c = 0; c < nrhs; ++c) {                                 /* step 4 (eps_d) */
                gemv(n, A, lda, X + c * n, R + c * n);
                for (int64_t t = 0; t < n; ++t) R[t + c * n] = B[t + c * n] - R[t + c * n];
            }
            int conv = 1, bad = 0;
            double worst = 0.0;
            for (int64_t c = 0; c < nrhs; ++c) {
                const double rn = sqrt(dot(n, R + c * n, R + c * n)), xn = sqrt(dot(n, X + c * n, X + c * n));
                if (!isfinite(rn) || !isfinite(xn)) { bad = 1; break; }
                const double ratio = rn == 0.0 ? 0.0 : rn / (xn * cte);
                if (ratio > worst) worst = ratio;
                if (!(rn < xn * cte || rn == 0.0)) conv = 0;
            }
            if (bad) break;
            if (hist) hist[it] = worst;
            if (nhist) *nhist = it + 1;
            if (conv) { *iters = it; code = 0; break; }
            if (it == itermax) break;
            for (int64_t t = 0; t < n * nrhs; ++t) Ws[t] = (float)R[t];
            oracle_sgetrs(n, nrhs, LU, n, ipiv, Ws);                             /* steps 5-6 */
            for (int64_t t = 0; t < n * nrhs; ++t) X[t] = X[t] + (double)Ws[t];  /* step 7 */
        }
    }
    free(LU); free(ipiv); free(Ws); free(R);
    if (code) {
        *iters = code;
        oracle_dgesv(n, nrhs, A, lda, B, X, info);
    }
    return 0;
}
