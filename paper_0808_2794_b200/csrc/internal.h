// internal.h — shared declarations of the sm_100a kernels (K1..K11) and the
// host driver of libmpsolve.so.  Not part of the public ABI (include/mp_solve.h).
//
// Working-copy layout: the binary32 (or, for
// the binary64 path, binary64) working copy W is ROW-major, n rows x ldw
// columns, ldw = round_up(n, 64): W[i*ldw + j] = fl(A(i,j)).  Row interchanges
// are then contiguous 1 KB+ row segments, panel rows are contiguous,
// and the Schur update C -= L21*U12 reads both operands with unit stride.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace mp {

constexpr int kMaxSMs = 256;

// ---------------------------------------------------------------- errors
struct CudaError {
    cudaError_t err;
    const char *what;
    int line;
};

#define MP_CUDA(call)                                                         \
    do {                                                                      \
        cudaError_t e_ = (call);                                              \
        if (e_ != cudaSuccess) throw ::mp::CudaError{e_, #call, __LINE__};    \
    } while (0)

#define MP_LAUNCH_CHECK() MP_CUDA(cudaGetLastError())

// ---------------------------------------------------------------- small helpers
__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Status record written by the device, read by the host once per iteration.
struct DevStatus {
    int32_t flags;        // bit0 A non-finite, bit1 demotion overflow, bit2 B non-finite,
                          // bit3 zero pivot seen, bit4 norms non-finite
    int32_t zero_col;     // 1-based column of the first exact zero pivot (0 = none)
    int32_t converged;    // residual check verdict
    int32_t pad;
    double anrm2;         // sum of squares of A (binary64)
    double ratio;         // max_c ||r_c|| / (||x_c|| cte)
    double rn[16];
    double xn[16];
};

enum : int32_t {
    ST_A_NONFINITE = 1,
    ST_OVERFLOW = 2,
    ST_B_NONFINITE = 4,
    ST_ZERO_PIVOT = 8,
    ST_NORM_NONFINITE = 16,
};

// Raise a kernel's dynamic shared-memory limit / allow non-portable cluster sizes,
// once per (kernel, device): the attribute calls cost microseconds and must stay off
// the per-launch path (thousands of launches per factorisation).
void func_smem_once(const void *fn, size_t bytes);
void func_cluster16_once(const void *fn);

// Per-launch counters (how many library kernels ran), read by the report.
extern thread_local int64_t g_launches;

// ---------------------------------------------------------------- programmatic dependent launch
// The factorisation's panel path is a chain of short dependent kernels (leaf -> laswp -> TRSM
// -> GEMM -> leaf ...).  Kernels on it are launched with programmatic stream serialisation:
// the next kernel's CTAs are scheduled while the current one runs and block in pdl_wait()
// (griddepcontrol.wait: returns once every prerequisite grid has COMPLETED and its memory
// is visible), so the launch latency of each link is hidden.  Every kernel launched this
// way calls pdl_wait() before its first global-memory access (read or write) and then
// pdl_trigger() (its own dependents may be scheduled).  Both are no-ops for a kernel
// launched without the attribute.  MP_NO_PDL=1 disables the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();

// Launch kern<<<grid, block, smem, s>>>(args...) with the PDL attribute (when enabled) and
// up to one extra attribute (cluster dimension / cooperative), through cudaLaunchKernelEx.
template <typename... KArgs, typename... Args>
void launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
               const cudaLaunchAttribute *extra, Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    unsigned na = 0;
    if (extra) at[na++] = *extra;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    MP_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
    ++g_launches;
}

// Optional per-kernel-class timing (mp_opts.flags bit 1): CUDA events recorded
// on the launching stream around every launch of a class, summed after the
// call.  Classes follow DESIGN.md's kernel list.
enum KClass : int { KC_DEMOTE = 0, KC_PANEL, KC_LASWP, KC_TRSM, KC_GEMM, KC_SOLVE, KC_RESIDUAL, KC_TRAIL, KC_COUNT };
void prof_begin(int cls, cudaStream_t s);
void prof_end(int cls, double work, cudaStream_t s);   // work: algorithmic flops (or bytes) of the launch

// ---------------------------------------------------------------- K1 demote (k_demote.cu)
// W[i*ldw + j] = (T)A[i + j*lda] for i,j < n; zero for j in [n, ldw).
// For T=float also: sum of squares (binary64) into st->anrm2 (deterministic
// two-level reduction), ST_A_NONFINITE / ST_OVERFLOW flags.
template <typename T>
void launch_demote_transpose(const double *A, int64_t lda, int64_t n, T *W, int64_t ldw,
                             double *partials, unsigned *counter, DevStatus *st, cudaStream_t s);

// Rectangular form: rows n, columns ncols of A (column-major, lda) into W (row-major, ldw).
template <typename T>
void launch_demote_rect(const double *A, int64_t lda, int64_t n, int64_t ncols, T *W, int64_t ldw,
                        double *partials, unsigned *counter, DevStatus *st, cudaStream_t s);

// Streamed e2e path (k_h2d.cu): device view of a pinned host pointer (nullptr if not device-accessible);
// copy ncols columns (host ld lda_h) into dA (ld n) with nctas CTAs of SM loads over PCIe and
// L2 evict-first stores.  Returns false (nothing launched) when n / alignment do not allow it.
const double *h2d_device_view(const double *hA);
bool launch_h2d_cols(const double *hA_dev, int64_t lda_h, double *dA, int64_t n, int64_t ncols, int nctas,
                     cudaStream_t s);

// W[i][c] = S[perm[i]][c] (i < n, c < ncols; S row-major with ld lds; 16-byte aligned rows)
void launch_gather_rows(const float *S, int64_t lds, int64_t ncols, const int32_t *perm, int64_t n, float *W,
                        int64_t ldw, cudaStream_t s);

// LU[i + j*n] = W[i*ldw + j]: packed factors back to the column-major ABI layout.
template <typename T>
void launch_transpose_out(const T *W, int64_t ldw, int64_t n, T *LU, cudaStream_t s);

// B non-finite check + y[pinv[i]] = (T)B[i + c*n] (demote + permute the rhs, K6).
template <typename T>
void launch_permute_demote_rhs(const double *B, int64_t n, int64_t nrhs, const int32_t *pinv,
                               T *Y, DevStatus *st, cudaStream_t s);

// ---------------------------------------------------------------- K2 panel (k_panel.cu)
struct PanelScratch {
    int32_t *orig;        // [n] panel-level origin of the row at each position
    int32_t *pairs;       // leaf-level (position, origin) pairs [2*nbmax][2]
    int32_t *npairs;      // 1
    int32_t *ppairs;      // panel-level pairs [2*nbmax][2]
    int32_t *nppairs;     // 1
    int32_t *ticket;      // 1, zero: fused TRSM+GEMM write-back ticket (launch_trsm_gemm_fused)
};
// Widest leaf one thread-block cluster can hold for m = n - c0 rows (0: too tall).
template <typename T>
int panel_leaf_width(int64_t m);
// whether the triangular-solve helper grid covers n (checked up front by the drivers)
template <typename T>
bool solve_fits(int64_t n);
// Factor the leaf rows [c0, n) x columns [c0, c0+w) of W in place (GEPP, binary T).
// Writes ipiv[c0 .. c0+w) (0-based global rows), updates ps.orig for the rows,
// and emits the leaf's (position <- position-at-leaf-start) pairs.
template <typename T>
// first_np != nullptr: the panel's first leaf (orig[] taken as the identity, *first_np zeroed)
// ll_k / lpos (lpos != nullptr): left-looking leaf of the binary32 panel starting at ll_k (k_panel.cu)
void launch_panel_leaf(T *W, int64_t ldw, int64_t n, int64_t c0, int w, int32_t *ipiv, PanelScratch &ps,
                       DevStatus *st, cudaStream_t s, int32_t *first_np = nullptr, int64_t ll_k = 0,
                       int32_t *lpos = nullptr, int64_t ll_kend = 0);
void launch_emit_pairs(const int32_t *orig, int64_t k, int64_t n, int32_t *pairs, int32_t *npairs, cudaStream_t s);

// ---------------------------------------------------------------- K3 laswp (k_laswp.cu)
// Apply a (position <- origin row) pair list to columns [c_lo, c_hi) minus
// [x_lo, x_hi); optionally also perm[pos] <- perm[orig] (perm != nullptr).
// Optional extra work of a laswp launch: the panel-level pair emission of emit_pairs_kernel
// (rows [k, n) whose origin orig[i] != i -> (i, orig[i]) appended at *npairs).
struct EmitJob {
    const int32_t *orig = nullptr;
    int64_t k = 0, n = 0;
    int32_t *pairs = nullptr, *npairs = nullptr;
};
template <typename T>
void launch_laswp_pairs(T *W, int64_t ldw, const int32_t *pairs, const int32_t *npairs, int max_pairs,
                        int64_t c_lo, int64_t c_hi, int64_t x_lo, int64_t x_hi, int32_t *perm,
                        cudaStream_t s, const EmitJob &ej = EmitJob{});
void launch_init_perm(int32_t *perm, int64_t n, cudaStream_t s);
void launch_invert_perm(const int32_t *perm, int32_t *pinv, int64_t n, cudaStream_t s);

// ---------------------------------------------------------------- K4 trsm (k_trsm.cu)
// U12 <- L11^{-1} A12: rows [r0, r0+w), columns [c_lo, c_hi), L11 = unit lower of W[r0.., r0..].
// sh/sl (binary32, optional): also write U12's 3xTF32 hi/lo split, K-major with row stride kp (the
// B operand layout of launch_gemm_ops_3xtf32; then call it with reuse_b).
template <typename T>
void launch_trsm_lower_unit(T *W, int64_t ldw, int64_t r0, int w, int64_t c_lo, int64_t c_hi,
                            cudaStream_t s, float *sh = nullptr, float *sl = nullptr, int kp = 0);
// Same with separate operands: X[w x ncols] <- L^{-1} X, L = unit lower w x w (row-major, ldl).
template <typename T>
void launch_trsm_ops(const T *L, int64_t ldl, T *X, int64_t ldx, int w, int64_t ncols, cudaStream_t s,
                     float *sh = nullptr, float *sl = nullptr, int kp = 0);

// ---------------------------------------------------------------- K5 Schur update (k_gemm.cu)
// C[M x N] -= A[M x K] * B[K x N], all row-major views into W with stride ldw:
//   A at W[r0*ldw + k0], B at W[k0*ldw + c0], C at W[r0*ldw + c0].
template <typename T>
void launch_gemm_update(T *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N,
                        int64_t K, cudaStream_t s);

// Same update with separate row-major operands: C[M x N] -= A[M x K] * B[K x N] (lda, ldb, ldc).
// binary64 trailing update on the FP64 tensor pipe (DMMA, k_gemm_f64.cu); false = shape or
// alignment not supported (the caller uses the DFMA tile kernel)
void launch_dgemm_dfma(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc,
                       int64_t M, int64_t N, int64_t K, cudaStream_t s);
bool launch_dgemm_dmma(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc,
                       int64_t M, int64_t N, int64_t K, cudaStream_t s, bool lower = false);
// binary32 FFMA update with TMA-staged tiles (k_sgemm_tma.cu): C[M x N] -= A[M x K] B[K x N], row-major;
// false = TMA alignment not met (16-byte bases, leading dimensions multiple of 4), nothing launched
bool launch_sgemm_tma(const float *A, int64_t lda, const float *B, int64_t ldb, float *C, int64_t ldc, int64_t M,
                      int64_t N, int64_t K, cudaStream_t s);
template <typename T>
void launch_gemm_ops(const T *A, int64_t lda, const T *B, int64_t ldb, T *C, int64_t ldc, int64_t M, int64_t N,
                     int64_t K, cudaStream_t s);

// 3xTF32 tcgen05 variant (k_gemm_tf32.cu): same operation, binary32 W; scratch holds the
// hi/lo splits of L21 and U12^T (tf32_scratch_floats(n, nb) floats).
size_t tf32_scratch_floats(int64_t n, int nbmax);
// K4 fused into K5 for the small in-panel levels (K in {32, 64}, N <= 64): A12 -> U12 in place
// and C -= L21 U12; false = no fused variant for this shape (launch K4 + K5).  ticket: one
// zero-initialised int per stream (re-armed by the kernel).
template <typename T>
bool launch_trsm_gemm_fused(T *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N, int64_t K,
                            int32_t *ticket, cudaStream_t s);
// cluster size of the tensor-core update for the calling thread's launches (0: the default policy)
void set_gemm_tf32_cluster(int cs);
void launch_gemm_update_3xtf32(float *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N,
                               int64_t K, float *scratch, int num_sms, cudaStream_t s, bool reuse_a = false, int terms = 3, bool reuse_b = false,
                               float *bscratch = nullptr);
// split of the A operand only (see launch_gemm_ops_3xtf32's reuse_a)
void launch_split_a_3xtf32(const float *A, int64_t lda, int64_t M, int64_t K, float *scratch, cudaStream_t s);
void launch_gemm_ops_3xtf32(const float *A, int64_t lda, const float *B, int64_t ldb, float *C, int64_t ldc, int64_t M,
                            int64_t N, int64_t K, float *scratch, int num_sms, cudaStream_t s, bool reuse_a = false, int terms = 3, bool reuse_b = false,
                            float *bscratch = nullptr);

// ---------------------------------------------------------------- K7/K9 triangular solves (k_solve.cu)
struct SolveScratch {
    unsigned *flags;      // [4][nblk] y / F ready flags (forward, backward), epoch-tagged, zeroed once
    void *F;              // [min(nrhs,16)][n] far partial sums (element type of the solve)
    unsigned epoch;       // last epoch used (incremented per sweep)
    // binary32 solves: [2][tag_cols][n] 64-bit words {value bits, sweep tag} for the y (chain ->
    // helpers) and F (helpers -> chain) exchanges, zeroed once; nullptr = flag exchange
    uint64_t *tags = nullptr;
    int tag_cols = 0;
};
size_t solve_tag_words(int64_t n, int64_t nrhs);
// Forward (unit L) then backward (U) substitution on Y (n x nrhs, T, column-major
// with ld n) with the packed LU in W; then X (double, ld n) = (mode 0) or += (mode 1) Y.
// inv (binary32 solves only; nullptr = substitution): the inverted diagonal blocks and the
// M blocks of launch_solve_inverses (reading A-19); the dependent chain is then one GEMV per block.
template <typename T>
void launch_lu_solve(const T *W, int64_t ldw, int64_t n, int64_t nrhs, T *Y, double *X, int accumulate,
                     SolveScratch &ss, cudaStream_t s, const float *inv = nullptr);
size_t solve_flag_words(int64_t n);
// K7 for 2..16+ right-hand sides (k_solve_mr.cu): right-looking blocked sweeps with fixed row
// ownership and the inverted diagonal blocks (inv required); flags: the 4 nblk words of
// SolveScratch, epoch: its counter.  launch_lu_solve takes this path when mr_solve_supported().
bool mr_solve_supported(int64_t n, int64_t nrhs);
// tags / tag_cols: SolveScratch's tagged words (nullptr: flag hand-off)
void launch_lu_solve_mr(const float *W, int64_t ldw, int64_t n, int64_t nrhs, float *Y, double *X, int accumulate,
                        unsigned *flags, unsigned &epoch, const float *inv, cudaStream_t s, uint64_t *tags = nullptr,
                        int tag_cols = 0);
size_t solve_inv_floats(int64_t n);      // [D_L | M_L | D_U | M_U], each ceil(n/64) 64x64 blocks
void launch_solve_inverses(const float *W, int64_t ldw, int64_t n, float *inv, cudaStream_t s);
// max over the diagonal blocks of kappa_inf (L and U) computed by launch_solve_inverses (synchronises s)
double solve_inverses_cond(const float *inv, int64_t n, cudaStream_t s);
// inverted diagonal blocks are used only when every block has kappa_inf below this (reading A-19)
constexpr double kInvCondMax = 1e5;
int solve_block_rows();

// ---------------------------------------------------------------- K8/K10 residual (k_residual.cu)
// R = B - A X (binary64, original A, column-major), then Y[pinv[i]] = (T)R[i],
// per-column norms and the B:5 convergence verdict into *st.
struct ResidualScratch {
    double *partial;      // [splits][n][nrhs]
    double *blocksums;    // [nblocks][2*nrhs]
    unsigned *counter;    // last-block ticket
};
int64_t residual_splits(int64_t n, int64_t nrhs, int num_sms);
size_t residual_partial_elems(int64_t n, int64_t nrhs, int num_sms);
template <typename T>
void launch_residual(const double *A, int64_t lda, int64_t n, int64_t nrhs, const double *B, const double *X,
                     double *R, const int32_t *pinv, T *Y, double cte, ResidualScratch &rs, DevStatus *st,
                     int num_sms, cudaStream_t s);

// ---------------------------------------------------------------- multi-GPU (comm.cu)
struct CommError {
    const char *what;
};
// Collectives of the 1D block-cyclic path, enqueued on (or synchronised with) stream s.
struct Comm {
    int rank = 0, size = 1;
    bool shared_device = false;   // loopback: every rank on this process's GPU (no shared streams)
    virtual ~Comm() {}
    virtual void bcast(void *buf, size_t bytes, int root, cudaStream_t s) = 0;
    virtual void allreduce_sum(double *buf, size_t count, cudaStream_t s) = 0;
    virtual void allreduce_max(int32_t *buf, size_t count, cudaStream_t s) = 0;
    virtual void allgather(const void *send, void *recv, size_t bytes_per_rank, cudaStream_t s) = 0;
};
bool nccl_available();
void nccl_unique_id(char id[128]);
Comm *make_nccl_comm(int nranks, int rank, const char id[128]);
void make_loopback_comms(int nranks, Comm **out);

// AX = A X for a rows x cols block of A (column-major, lda) and X (cols x nrhs, ld ldx);
// AX is rows x nrhs with ld rows (binary64; split-K partials reduced in a fixed order).
void launch_residual_products(const double *A, int64_t lda, int64_t rows, int64_t cols, int64_t nrhs,
                              const double *X, int64_t ldx, double *AX, ResidualScratch &rs, int num_sms,
                              cudaStream_t s);
// R = B - AX, norms and the B:5 verdict into *st, Y[pinv[i]] = (T) R[i] (as launch_residual).
template <typename T>
void launch_residual_finalize(const double *AX, int64_t n, int64_t nrhs, const double *B, const double *X, double *R,
                              const int32_t *pinv, T *Y, double cte, ResidualScratch &rs, DevStatus *st,
                              cudaStream_t s);

}  // namespace mp

namespace mp {
// ---------------------------------------------------------------- SPD variant (k_chol.cu, NEXT-1)
// Lower triangle of the column-major A -> full symmetric row-major W (fl32 RN for T = float),
// ||A||_F^2 of the symmetric matrix into st->anrm2, flags.  partials: demote_sym_partials() doubles.
template <typename T>
void launch_demote_sym(const double *A, int64_t lda, int64_t n, T *W, int64_t ldw, double *partials,
                       unsigned *counter, DevStatus *st, int num_sms, cudaStream_t s);
size_t demote_sym_partials(int num_sms);
template <typename T>
int chol_block_max();                     // widest diagonal block of potrf / trsm_chol (256 / 128)
template <typename T>
void launch_potrf_diag(T *W, int64_t ldw, int64_t k, int w, DevStatus *st, cudaStream_t s);
template <typename T>
void launch_trsm_chol(T *W, int64_t ldw, int64_t k, int w, int64_t n, cudaStream_t s);
template <typename T>
void launch_chol_to_lu(T *W, int64_t ldw, int64_t n, T *dscratch, cudaStream_t s);
size_t symv_partial_elems(int64_t n);
// AX = A_sym X from the lower triangle of the column-major A (n x nrhs, ld n)
void launch_symv_products(const double *A, int64_t lda, int64_t n, int64_t nrhs, const double *X, double *AX,
                          double *partials, cudaStream_t s);
// C[M x M] lower tiles -= L21 L21^T, L21 = A[M x K] row-major (3xTF32 tcgen05)
void launch_syrk_lower_3xtf32(const float *A, int64_t lda, float *C, int64_t ldc, int64_t M, int64_t K, float *scratch,
                              int num_sms, cudaStream_t s, int terms = 3);
}  // namespace mp

namespace mp {
// ---------------------------------------------------------------- NEXT-4 double-double refinement (k_dd.cu)
size_t dd_scratch_doubles(int64_t n, int num_sms);
void launch_dd_residual(const double *A, int64_t lda, int64_t n, int64_t nrhs, const double *B, const double *Xh,
                        const double *Xl, double *Rh, double *Rl, const int32_t *pinv, double *Y, double cte,
                        double *scratch, unsigned *counter, DevStatus *st, int num_sms, cudaStream_t s);
void launch_dd_update(double *Xh, double *Xl, const double *Z, int64_t count, cudaStream_t s);
}  // namespace mp

namespace mp {
// ---------------------------------------------------------------- NEXT-3 Algorithm 2 (k_gmres.cu)
void launch_gemv_rows_f32(const float *W, int64_t ldw, int64_t n, const float *x, float *y, cudaStream_t s);
size_t gmres_partial_elems(int64_t n);
// G7: one whole binary32 GMRES_SP(m) cycle (z = 0 start, right-hand side v) as one cooperative launch of
// `sms` CTAs; z written in binary64.  V: ldv x m, raw: 2 x ldv, part: sp_cycle_part_elems(sms), bar: 1.
bool sp_cycle_supported(int64_t n, int sms);
size_t sp_cycle_part_elems(int sms);
void launch_gmres_sp_cycle(const float *W, int64_t ldw, int64_t n, const float *v, float *V, int64_t ldv, float *raw,
                           double *z, int m, float *part, unsigned *bar, int sms, cudaStream_t s);
void launch_convert_f32_f64(const float *a, double *b, int64_t n, cudaStream_t s);
template <typename T>
void launch_multidot(const T *V, int64_t ldv, int k, const T *w, int64_t n, T *partial, T *out, bool accumulate,
                     cudaStream_t s);
template <typename T>
void launch_combine(T *w, const T *V, int64_t ldv, int k, const T *coef, T alpha, T beta, int64_t n, cudaStream_t s);
template <typename T, typename TS>
void launch_scale_copy(const T *w, const T *scale, bool invert, T *out, TS *outs, int64_t n, cudaStream_t s);
template <typename T>
void launch_givens_step(const T *hcol, const T *hnorm2, int j, int m, T *R, T *cs, T *sn, T *g, T *hout,
                        cudaStream_t s);
template <typename T>
void launch_backsolve(const T *R, int m, int steps, const T *g, T *y, const T *hn, cudaStream_t s);
template <typename T>
void launch_cycle_start(const T *norm2, T *g, int m, T *beta, cudaStream_t s);
}  // namespace mp
