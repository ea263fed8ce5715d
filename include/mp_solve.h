/*
 * mp_solve.h — C-ABI of libmpsolve.so, the B200 (sm_100a) mixed-precision
 * iterative-refinement dense solver of arXiv 0808.2794.
 *
 * Operation (Algorithm 1; BASELINE.json north_star B:5):
 *   1  LU <- PA             binary32 blocked right-looking GEPP of fl32(A)
 *   2-3 L y = P b; U x0 = y  binary32 substitution
 *   loop k = 1, 2, ...
 *   4  r_k <- b - A x_{k-1} binary64, with the ORIGINAL A
 *   5-6 L y = P r_k; U z_k = y  binary32
 *   7  x_k <- x_{k-1} + z_k binary64
 *   check convergence: for every rhs column c
 *        ||r_c||_2 < ||x_c||_2 * ||A||_F * 2^-53 * sqrt(n)   or  ||r_c||_2 == 0
 *   (B:5 replaces the paper's spectral norm, by ||A||_F; readings
 *   A-1..A-5 in DESIGN.md), at most 30 corrections, then the full
 *   binary64 solver on a fresh copy of A.
 *
 * Layout: column-major.  A is n x n with leading dimension lda >= max(1,n),
 * entry (i,j) at A[i + j*lda].  B and X are n x nrhs with leading dimension n.
 *
 * Pointers: every matrix/vector argument may be a CUDA device pointer (the
 * device current on the calling thread) or a host pointer (pinned or
 * pageable); the library detects which with cudaPointerGetAttributes and, for
 * host buffers, stages the copies itself (H2D of A and B, D2H of X) on the
 * library stream.  A host call is the "end-to-end" path.
 *
 * Ownership: the caller owns A, B, X.  A and B are read-only (never
 * overwritten, unlike LAPACK DSGESV).  X is written.  The library allocates
 * its workspace stream-ordered (cudaMallocAsync): a binary32 n x n working
 * copy (the "+50 % memory" of P:145-146) plus O(n * nrhs) vectors; a binary64
 * n x n copy only when the fallback runs.  Workspace is released before the
 * call returns.
 *
 * Synchronisation: every solve call is synchronous with respect to the host
 * (the convergence test reads one small status record per iteration).  Calls
 * are not re-entrant for the same device from several threads.
 *
 * Return value: MP_OK (0), or a runtime failure code (MP_ERR_*): a CUDA error,
 * an allocation failure, or an internal error; mp_last_error() describes it.
 * Numerical outcomes go to *info / *iters, never to the return value.
 *
 * *info: 0 success; -i: the i-th argument is illegal (1 n < 0, 2 nrhs < 0,
 *   3 A NULL / A has a NaN or Inf entry, 4 lda < max(1,n), 5 B NULL / B has a
 *   NaN or Inf entry, 6 X NULL or X overlaps A or B); +i: U(i,i) (1-based) is
 *   exactly zero in the binary64 factorisation, X is unspecified.
 * *iters: >= 0 number of refinement corrections applied (0: x0 passed the
 *   test); -2 a finite entry of A overflowed binary32 on demotion; -3 exact
 *   zero pivot in the binary32 LU; -31 no convergence within itermax (30)
 *   corrections, or a non-finite residual/solution norm.  iters < 0 means
 *   the binary64 solver produced X.
 * Quick return: n == 0 or nrhs == 0 -> info = 0, iters = 0, nothing touched.
 */
#ifndef MP_SOLVE_H
#define MP_SOLVE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MP_OK            0
#define MP_ERR_CUDA      1
#define MP_ERR_NOMEM     2
#define MP_ERR_INTERNAL  3
#define MP_ERR_NCCL      4
#define MP_ERR_UNSUPPORTED 5

#define MP_ITERMAX_DEFAULT 30

/* Trailing-update (Schur complement A22 -= L21 U12) variant of the binary32
 * factorisation.  Both compute in binary32 precision; B:5 keeps a variant only
 * if refinement still reaches the binary64 backward criterion. */
#define MP_VARIANT_FFMA    0   /* FP32 FFMA SGEMM (CUDA cores) */
#define MP_VARIANT_3XTF32  1   /* tcgen05 tensor cores, 3xTF32 split (hi*hi + hi*lo + lo*hi) */
/* SURVEY 8(f) NEXT-2, the lower-precision tensor-core factorisation: every tensor-core Schur update
 * takes operands rounded to TF32 (cvt.rna, 10 stored significand bits: u_f = 2^-11) with binary32
 * accumulation, one MMA per product (3x fewer than 3xTF32).  The factors are then accurate to
 * ~2^-11 kappa, so Algorithm 1 converges only for kappa * 2^-11 well below 1; for
 * harder systems select the GMRES-IR refinement (opts.flags bit 8). */
#define MP_VARIANT_TF32    2

typedef struct mp_opts {
    int32_t nb;        /* panel width; 0 = default (64 for n<=1024, 128 for n<=4096, else 256) */
    int32_t itermax;   /* refinement cap; 0 = MP_ITERMAX_DEFAULT */
    int32_t variant;   /* MP_VARIANT_* (default MP_VARIANT_3XTF32) */
    int32_t flags;     /* bit 0: force the binary64 fallback path after the binary32 factorisation (testing);
                          bit 1: per-kernel-class CUDA-event timing into mp_report.k_* (measurement);
                          bit 2: with bit 1, keep the events of successive calls and resolve them only in
                                 mp_profile_collect() (keeps event queries out of timed loops);
                          bit 3: with bit 1, record only the trailing update and the residual classes
                                 (a handful of events per solve: cheap enough for a timed region);
                          bit 4: disable the look-ahead (panel k+1 factored on a 16-SM green context
                                 while the trailing update of step k runs on the other SMs);
                          bit 5: binary32 triangular solves by plain substitution inside the 64-row
                                 diagonal blocks instead of the default inverted diagonal blocks
                                 (reading A-19); exact inputs then stay exact (pin P2);
                          bit 6: host A: one copy before the factorisation instead of streaming it in
                                 by column blocks under the factorisation (mp_dsgesv, n >= 4096);
                          bit 7: mp_fgmres: run each binary32 GMRES_SP cycle as a sequence of small
                                 kernels instead of the one cooperative launch (testing);
                          bit 8: mp_dsgesv: refine by GMRES-IR instead of Algorithm 1's loop (SURVEY
                                 8(f) NEXT-2): restarted FGMRES(20) in binary64 on A x = b from x0
                                 (each right-hand side on its own), every Krylov direction preconditioned by the
                                 binary32 LU factors (one forward/backward sweep pair); B:5's test at
                                 every restart, each cycle ends early once its Givens residual
                                 estimate meets the test; *iters = LU-solve applications */
} mp_opts;

#define MP_HIST_MAX 64

typedef struct mp_report {
    int32_t iters, info;        /* same values as the *iters / *info outputs */
    int32_t nhist;              /* number of residual checks recorded in hist[] */
    int32_t nb, variant;        /* panel width / variant actually used */
    int32_t solve_inv;          /* 1: binary32 solves used inverted 64x64 diagonal blocks (reading A-19),
                                   0: substitution (flags bit 5, or a block with kappa_inf > 1e5) */
    double  anrm;               /* ||A||_F (binary64, computed once on device) */
    double  hist[MP_HIST_MAX];  /* per residual check: max_c ||r_c|| / (||x_c|| * ||A||_F * 2^-53 * sqrt(n)) */
    double  t_total_ms;         /* device time of the whole call (CUDA events) */
    double  t_demote_ms;        /* K1: demote + ||A||_F */
    double  t_factor_ms;        /* binary32 (or binary64 for mp_dgesv) factorisation */
    double  t_refine_ms;        /* x0 + refinement loop */
    double  t_fallback_ms;      /* binary64 fallback, if it ran */
    double  t_copy_ms;          /* host<->device staging (host-pointer calls only) */
    int64_t workspace_bytes;    /* peak bytes allocated by the library for this call */
    int64_t kernel_launches;    /* number of library kernels launched by this call */
    /* per kernel class (filled when opts.flags bit 1 is set), index = MP_KC_*:
       summed device time of the launches (CUDA events on the launching stream),
       number of launches, and their summed ALGORITHMIC work (flops for
       MP_KC_GEMM / MP_KC_TRSM, bytes for the bandwidth-bound classes). */
    double  k_ms[8];
    double  k_work[8];
    int64_t k_launches[8];
} mp_report;

#define MP_KC_DEMOTE   0   /* K1 demote + ||A||_F          work = bytes (12 n^2)          */
#define MP_KC_PANEL    1   /* K2 panel factorisation       work = flops of the leaf       */
#define MP_KC_LASWP    2   /* K3 row interchanges          work = bytes moved             */
#define MP_KC_TRSM     3   /* K4 U12 <- L11^-1 A12         work = flops (w^2 N)           */
#define MP_KC_GEMM     4   /* K5 in-panel Schur updates    work = flops (2 M N K)         */
#define MP_KC_SOLVE    5   /* K6/K7/K9 triangular solves   work = bytes of the factors    */
#define MP_KC_RESIDUAL 6   /* K8/K10 residual + test       work = bytes (8 n^2 + vectors)  */
#define MP_KC_TRAIL    7   /* K5 on the trailing matrix A22 (3xTF32 tcgen05 or FFMA), work = flops (2 M N K) */

/* Fill *o with the defaults above. */
void mp_default_opts(mp_opts *o);

/* Mixed-precision solve A X = B (Algorithm 1 + B:5 stop test + fallback). */
int mp_dsgesv(int64_t n, int64_t nrhs, const double *A, int64_t lda,
              const double *B, double *X, int *iters, int *info);

/* Same, with options (NULL = defaults) and an optional report (NULL = none). */
int mp_dsgesv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                 const double *B, double *X, int *iters, int *info,
                 const mp_opts *opts, mp_report *rep);

/* Binary64 reference solver built the same way (DGETRF + DGETRS semantics,
 * no refinement): the denominator of the speedup (B:5). */
int mp_dgesv(int64_t n, int64_t nrhs, const double *A, int64_t lda,
             const double *B, double *X, int *info);

int mp_dgesv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                const double *B, double *X, int *info,
                const mp_opts *opts, mp_report *rep);

/* Step 1 alone, for factor-level parity: demote A (RN-even),
 * factor PA = LU in binary32 with the same kernels as mp_dsgesv, and return
 * the packed factors LU (n x n column-major, leading dimension n, unit lower
 * L below the diagonal, U on/above) and ipiv (0-based LAPACK-style sequential
 * pivot list: at step k rows k and ipiv[k] were interchanged).  *info: as
 * above for argument errors (-1 n, -3 A, -4 lda, -5 LU NULL, -6 ipiv NULL);
 * +k when the first exact zero pivot is at column k (1-based); -2 when a
 * finite entry of A overflowed binary32. */
int mp_sgetrf(int64_t n, const double *A, int64_t lda, float *LU, int32_t *ipiv,
              int *info, const mp_opts *opts);

/* Same in binary64 (the fallback / mp_dgesv factorisation). */
int mp_dgetrf(int64_t n, const double *A, int64_t lda, double *LU, int32_t *ipiv,
              int *info, const mp_opts *opts);

/* ------------------------------------------------------------------------------------------
 * SPD variant.  PAPER.md P:369-371: "For the symmetric case the SGETRF,
 * SGETRS and DGEMM subroutines were replaced by the SPOTRF, SPOTRS and DSYMM subroutines":
 * Algorithm 1 with step 1 a binary32 Cholesky A = L L^T, steps 2-3 / 5-6 the two binary32
 * triangular solves with L and L^T, step 4 r = b - A x in binary64 with the symmetric A; the
 * stop test, the 30-correction cap and the binary64 fallback are those of mp_dsgesv.
 *
 * A: n x n symmetric positive definite, column-major, leading dimension lda; ONLY its LOWER
 * triangle (i >= j) is read (LAPACK UPLO = 'L'); the strict upper triangle is never touched and
 * may hold anything.  B, X, pointers, ownership, synchronisation, return value: as mp_dsgesv.
 * ||A||_F in the stop test is the norm of the full symmetric matrix (reading C-3).
 *
 * *info: 0; -i argument errors as mp_dsgesv (-3 also: a NaN/Inf in the lower triangle);
 *   +k: the binary64 Cholesky broke down at column k (the leading minor of order k is not
 *   positive definite, reading C-2); X is unspecified.
 * *iters: >= 0 corrections; -2 demotion overflow; -3 the binary32 Cholesky broke down (a pivot
 *   not > 0, reading C-1); -31 no convergence within 30 corrections.  iters < 0: X came from
 *   the binary64 Cholesky solver.
 * opts.variant selects the trailing (SYRK) update: MP_VARIANT_3XTF32 (default, lower tiles only)
 * or MP_VARIANT_FFMA; opts.nb <= 256 (binary32) / 128 (binary64). */
int mp_dsposv(int64_t n, int64_t nrhs, const double *A, int64_t lda,
              const double *B, double *X, int *iters, int *info);
int mp_dsposv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                 const double *B, double *X, int *iters, int *info,
                 const mp_opts *opts, mp_report *rep);

/* The binary64 SPD solver (Cholesky + the two solves, no refinement): the T3 "reference time"
 * of the symmetric column and mp_dsposv's fallback.  info as above. */
int mp_dposv(int64_t n, int64_t nrhs, const double *A, int64_t lda,
             const double *B, double *X, int *info);
int mp_dposv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda,
                const double *B, double *X, int *info, const mp_opts *opts, mp_report *rep);

/* Step 1 of the SPD variant alone: the Cholesky factor of fl32(A) (mp_spotrf) or A (mp_dpotrf)
 * from A's lower triangle.  L: n x n column-major output, leading dimension n (device or host):
 * L in the lower triangle, its strict upper triangle holds L^T.  info: argument errors as
 * mp_sgetrf (-5: L NULL); +k breakdown at column k (1-based); -2 demotion overflow. */
int mp_spotrf(int64_t n, const double *A, int64_t lda, float *L, int *info, const mp_opts *opts);
int mp_dpotrf(int64_t n, const double *A, int64_t lda, double *L, int *info, const mp_opts *opts);

/* ------------------------------------------------------------------------------------------
 * Extended-precision refinement: "Extension to Quadruple
 * Precision" — QDGESV factors A in binary64 (DGETRF), solves with DGETRS, and carries the residual
 * r = b - A x (QGEMV) and the update x += z in quadruple precision, here double-double (reading
 * Q-0: X = Xhi + Xlo, |Xlo| <= ulp(Xhi)/2, 106 significand bits).  Stop test (Q-1):
 *     ||fl64(r_c)||_2 < ||Xhi_c||_2 * ||A||_F * 2^-104 * sqrt(n)  or  r_c == 0, for every column;
 * at most 30 corrections; no fallback (Q-2): iters = -31 returns the last iterate.
 * A (n x n, lda), B (n x nrhs, ld n): binary64, used exactly.  Xhi, Xlo: n x nrhs outputs, ld n,
 * device or host (as mp_dsgesv), must not overlap A, B or each other (info -6 / -7).
 * *info: 0; -i argument errors (-3 A NaN/Inf, -5 B NaN/Inf, -7 Xlo NULL/overlapping);
 *   +k exact zero pivot at column k in the binary64 LU (X unspecified).
 * *iters: >= 0 corrections applied; -31 no convergence (rows of X = the last iterate). */
int mp_qdgesv(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B,
              double *Xhi, double *Xlo, int *iters, int *info);
int mp_qdgesv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B,
                 double *Xhi, double *Xlo, int *iters, int *info, const mp_opts *opts, mp_report *rep);

/* ---------------------------------------------------------------- NEXT-3: Algorithm 2
 * Mixed precision inner-outer FGMRES(m_out)-GMRES_SP(m_in) (Algorithm 2,
 * P:240-279).  Outer: flexible GMRES in binary64 with the caller's A (products r = A z_k, modified
 * Gram-Schmidt, Givens least squares, x += Z y); preconditioner: one cycle of GMRES_SP(m_in) in
 * binary32 with fl32(A), started from z = 0.  x0 = 0.  One right-hand side.
 * Readings (G-1..G-6): the stop test is B:5's ||b - A x||_2 < ||x||_2 ||A||_F 2^-53 sqrt(n)
 * (or r == 0), checked at the top of every outer cycle (G-1); at most opts.itermax (default 30)
 * outer cycles, then *iters = -31 and x is the last iterate (G-2, no fallback); an exact breakdown
 * ends the basis (G-4); the binary32 Arnoldi orthogonalises by classical Gram-Schmidt applied twice
 * (G-6; the oracle follows the printed MGS).
 * A: n x n binary64, column-major, lda >= max(1, n); b: n; x: n output.  Device or host pointers (host
 * buffers are staged).  1 <= m_out, m_in <= 31.
 * *info: 0; -1 n < 0; -2 A NULL or NaN/Inf; -3 lda; -4 b NULL or NaN/Inf; -5 x NULL; -6 m_out / m_in.
 * *iters: outer cycles applied before convergence (>= 0); -31 no convergence.
 * Workspace: 4 n^2 + O(n (m_out + m_in)) bytes (the binary32 copy of A dominates). */
int mp_fgmres(int64_t n, const double *A, int64_t lda, const double *b, double *x, int m_out, int m_in,
              int *iters, int *info);
int mp_fgmres_ex(int64_t n, const double *A, int64_t lda, const double *b, double *x, int m_out, int m_in,
                 int *iters, int *info, const mp_opts *opts, mp_report *rep);

/* Resolve the per-launch events recorded by calls made with opts.flags = 2|4 since the
 * last collection: fills rep->k_ms / k_work / k_launches (summed over those calls, all
 * other fields untouched) and clears the records.  Synchronises the device. */
int mp_profile_collect(mp_report *rep);

/* Use this CUDA stream (a cudaStream_t, NULL = the legacy default stream) for
 * all subsequent library work on the calling thread. */
int mp_set_stream(void *stream);

/* Human-readable description of the last runtime failure on this thread. */
const char *mp_last_error(void);

/* Library version / build string (arch, variant support). */
const char *mp_version(void);

/* Execution resources of the factorisation on the current device: *lookahead = 1 when the
 * look-ahead partition is active, *sms_update = SMs of the trailing-update green context,
 * *sms_panel = SMs kept free for the panel stream (0 / device SM count when inactive).
 * Returns MP_OK or MP_ERR_CUDA. */
int mp_exec_info(int *lookahead, int *sms_panel, int *sms_update);

/* ---------------------------------------------------------------- multi-GPU: 1D block-cyclic
 * SURVEY 8(e), B:5 ("the matrix is distributed 1D block-cyclic by column blocks; each factored
 * panel and its pivot vector are broadcast ... the distributed residual GEMV is followed by an
 * allreduce of r").  One process per GPU.  Global column block j (nb columns) lives on rank
 * j mod P at local block slot j / P; A_local holds this rank's columns in increasing global
 * order (column-major, lda_local >= max(1, local columns)); B and X are replicated on every
 * rank (n x nrhs, ld n).  All matrix / vector pointers are DEVICE pointers.  Calls are
 * collective: every rank calls with the same n, nrhs, nb and returns the same iters / info
 * (conventions as mp_dsgesv / mp_dgesv; info -5 / -7 for non-finite A / B).  Argument errors
 * return info = -i for the i-th argument.  Collective failures return MP_ERR_NCCL. */
typedef struct mp_comm mp_comm;

/* NCCL unique id for mp_comm_init (create on one rank, share it with the others). */
int mp_get_unique_id(char id[128]);
/* NCCL communicator of rank `rank` of `nranks` (one process per GPU, current device). */
int mp_comm_init(int nranks, int rank, const char id[128], mp_comm **comm);
/* `nranks` emulated ranks of ONE process on the current GPU (testing the P > 1 algorithm on
 * a single GPU): comms[r] is used by the host thread playing rank r; collectives meet at a
 * host barrier and move data with device copies (no kernel ever waits for another rank). */
int mp_comm_init_loopback(int nranks, mp_comm **comms);
int mp_comm_destroy(mp_comm *comm);
/* Number of columns of A owned by `rank` (the width of its A_local). */
int64_t mp_1dbc_local_cols(int64_t n, int64_t nb, int nranks, int rank);

int mp_dsgesv_1dbc(mp_comm *comm, int64_t n, int64_t nrhs, int64_t nb, const double *A_local,
                   int64_t lda_local, const double *B, double *X, int *iters, int *info);
int mp_dsgesv_1dbc_ex(mp_comm *comm, int64_t n, int64_t nrhs, int64_t nb, const double *A_local,
                      int64_t lda_local, const double *B, double *X, int *iters, int *info,
                      const mp_opts *opts, mp_report *rep);
/* Distributed binary64 solver built the same way (the speedup denominator at P > 1). */
int mp_dgesv_1dbc(mp_comm *comm, int64_t n, int64_t nrhs, int64_t nb, const double *A_local,
                  int64_t lda_local, const double *B, double *X, int *info);

#ifdef __cplusplus
}
#endif

#endif /* MP_SOLVE_H */
