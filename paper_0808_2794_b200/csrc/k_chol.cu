// k_chol.cu — the SPD variant of the hot path ("For the
// symmetric case the SGETRF, SGETRS and DGEMM subroutines were replaced by the SPOTRF, SPOTRS and
// DSYMM subroutines").  Kernels:
//
//  * C1 demote_sym_kernel    A (column-major, LOWER triangle only, LAPACK UPLO = 'L') -> the
//                            row-major working copy W holding the full symmetric matrix, fl32 RN;
//                            ||A||_F of the symmetric matrix (reading C-3), non-finite / overflow
//                            flags.  HBM-bound: reads 4 n^2 B (the lower triangle), writes 4 n^2 B.
//  * C2 potrf_diag_kernel    Cholesky of one diagonal block (w <= 256 binary32 / 128 binary64)
//                            in shared memory (packed lower triangle), right-looking column
//                            order as the oracle ("SPOTRF"); writes L11 and L11^T.
//  * C3 trsm_chol_kernel     L21 = A21 L11^-T, one CTA per 64 rows, column sweep; writes L21 into
//                            the lower block and L21^T into the upper block (the B operand the
//                            row-major Schur-update kernels read).
//  * (SYRK) the trailing update A22 -= L21 L21^T runs on the K5 kernels restricted to the tiles
//    that touch the lower triangle (k_gemm_tf32.cu / k_gemm_f64.cu).
//  * C4 chol_to_lu_kernel    L L^T -> the unit-lower / upper packed form the triangular-solve
//                            kernels (K7) take: Lhat = L D^-1, Uhat = D L^T, D = diag(L)
//                            (reading C-4: one rounding per entry; exact for power-of-two l_jj).
//  * C5 symv_partial_kernel  r = b - A x with the symmetric A read from its lower triangle only
//                            ("DSYMM"): each lower tile contributes A_IJ x_J to r_I and
//                            A_IJ^T x_I to r_J; fixed-order reduction (deterministic).  HBM-bound:
//                            4 n^2 B per residual, half of the nonsymmetric K8.
#include <algorithm>

#include "internal.h"

namespace mp {

namespace {

// ---------------------------------------------------------------- C1 demote (lower -> symmetric W)
constexpr int DT = 64;          // tile
constexpr int DTHREADS = 256;

template <typename T>
__global__ void __launch_bounds__(DTHREADS)
demote_sym_kernel(const double *__restrict__ A, int64_t lda, int64_t n, T *__restrict__ W, int64_t ldw,
                  double *__restrict__ partials, unsigned *counter, DevStatus *st)
{
    constexpr bool LOW = sizeof(T) == 4;
    __shared__ T tile[DT][DT + 1];                 // [jj][ii] = A(i0 + ii, j0 + jj)
    __shared__ double red[DTHREADS / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nt = ceil_div(n, DT);
    const int64_t ntiles = nt * (nt + 1) / 2;      // lower tiles (I >= J), row-major over I
    double ss = 0.0;
    int flags = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // t -> (I, J), I >= J: I = floor((sqrt(8t + 1) - 1) / 2)
        int64_t I = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
        while (I * (I + 1) / 2 > t) --I;
        while ((I + 1) * (I + 2) / 2 <= t) ++I;
        const int64_t J = t - I * (I + 1) / 2;
        const int64_t i0 = I * DT, j0 = J * DT;
        const bool diag = I == J;
#pragma unroll
        for (int p = 0; p < DT / 8; ++p) {
            const int jj = warp + 8 * p, ii = lane * 2;
            const int64_t j = j0 + jj, i = i0 + ii;
            double a[2] = {0.0, 0.0};
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const bool ok = j < n && i + e < n && (!diag || ii + e >= jj);
                if (ok) {
                    a[e] = __ldcs(A + j * lda + i + e);
                    if (!isfinite(a[e])) flags |= ST_A_NONFINITE;
                    const double w2 = (i + e == j) ? 1.0 : 2.0;     // reading C-3: off-diagonal twice
                    ss = fma(w2 * a[e], a[e], ss);
                }
                T v;
                if (LOW) {
                    const float f = __double2float_rn(a[e]);
                    if (ok && isfinite(a[e]) && isinf(f)) flags |= ST_OVERFLOW;
                    v = (T)f;
                } else {
                    v = (T)a[e];
                }
                tile[jj][ii + e] = v;
            }
        }
        __syncthreads();
        // lower part: W[i][j] = tile[jj][ii] (row-major rows i, coalesced along j)
#pragma unroll
        for (int p = 0; p < DT / 8; ++p) {
            const int ii = warp + 8 * p;
            const int64_t i = i0 + ii;
            if (i < n) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int jj = lane * 2 + e;
                    const int64_t j = j0 + jj;
                    if (j < n && (!diag || ii >= jj)) W[i * ldw + j] = tile[jj][ii];
                }
            }
        }
        // upper part (the mirror): W[j][i] = tile[jj][ii] (rows j, coalesced along i)
#pragma unroll
        for (int p = 0; p < DT / 8; ++p) {
            const int jj = warp + 8 * p;
            const int64_t j = j0 + jj;
            if (j < n) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int ii = lane * 2 + e;
                    const int64_t i = i0 + ii;
                    if (i < n && (!diag || ii > jj)) W[j * ldw + i] = tile[jj][ii];
                }
            }
        }
        __syncthreads();
    }
    // deterministic reduction of the sum of squares: warp -> block -> last block over blocks
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0) {
        red[warp] = ss;
        if (flags) atomicOr(&st->flags, flags);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < DTHREADS / 32; ++w) b += red[w];
        partials[blockIdx.x] = b;
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        double b = 0.0;
        for (int64_t k = threadIdx.x; k < gridDim.x; k += DTHREADS) b += __ldcg(partials + k);
        for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
        if (lane == 0) red[warp] = b;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int w = 0; w < DTHREADS / 32; ++w) tot += red[w];
            st->anrm2 = tot;
            *counter = 0u;
        }
    }
}

// ---------------------------------------------------------------- C2 diagonal-block Cholesky
// The w x w diagonal block lives in shared memory as a packed lower triangle (row r contiguous:
// element (r, k) at r (r + 1) / 2 + k).  Left-looking by 32-column chunks c, three barriers each:
//   (1) columns of chunk c, rows [32c, w): a_rj -= sum_{k < 32c} l_rk l_jk   (dot products)
//   (2) one warp factors the 32 x 32 diagonal sub-block: lane i holds row i in registers; per
//       column j every lane forms l_jj = sqrt(a_jj) itself (IEEE), divides (IEEE), and applies
//       the column to its row with the other lanes' l_kj obtained by shuffles
//   (3) rows below the sub-block (within the block): thread-per-row forward substitution with
//       the 32 x 32 factor: l_rj = (a_rj - sum_{i < j} l_ri l_ji) / l_jj.
// The operations per entry are the oracle's (square root, division, products and differences;
// FMA-contracted: reading A-8), only grouped by chunk, so the exact family stays bitwise.
__host__ __device__ constexpr int pk(int i, int j) { return i * (i + 1) / 2 + j; }   // packed lower, j <= i

constexpr int PTHREADS = 512;
constexpr int CW = 32;           // chunk width

template <typename T>
__device__ __forceinline__ T sqrt_rn(T x) { return sqrt(x); }

template <typename T>
__global__ void __launch_bounds__(PTHREADS)
potrf_diag_kernel(T *__restrict__ W, int64_t ldw, int64_t k, int w, DevStatus *st)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *P = reinterpret_cast<T *>(smem_raw);                       // packed lower, w (w + 1) / 2
    T *LT = P + pk(w, 0);                                         // [w][CW] chunk rows, transposed
    // no early trigger: the dependent TRSM's CTAs (~100 KB of shared memory each) would sit
    // resident for the whole factorisation of this block, on SMs the look-ahead's concurrent
    // SYRK launches need (measured: C3-size SPD 48.4 vs 42.2 ms with the trigger at the start)
    pdl_wait();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = PTHREADS / 32;
    T *Wd = W + k * ldw + k;
    for (int i = warp; i < w; i += NW)
        for (int j = lane; j <= i; j += 32) P[pk(i, j)] = Wd[(int64_t)i * ldw + j];
    __syncthreads();
    for (int c0 = 0; c0 < w; c0 += CW) {
        const int cw = min(CW, w - c0);
        // (1) left-looking update of the chunk's columns, rows [c0, w): the chunk's L rows are first
        //     copied transposed (LT[kk][j], lanes read consecutive j: no bank conflicts); a thread
        //     owns 4 rows of one column (4 independent chains, the row operands broadcast)
        if (c0 > 0) {
            for (int idx = tid; idx < c0 * CW; idx += PTHREADS) {
                const int kk = idx / CW, j = idx % CW;
                LT[idx] = j < cw ? P[pk(c0 + j, kk)] : T(0);
            }
            __syncthreads();
            const int rows = w - c0, ngr = (rows + 3) / 4;
            for (int o = tid; o < ngr * CW; o += PTHREADS) {
                const int j = o % CW, rb = c0 + 4 * (o / CW);
                if (j >= cw) continue;
                const int jr = c0 + j;
                T acc[4];
                const T *lr[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int r = min(rb + q, w - 1);
                    lr[q] = P + pk(r, 0);
                    acc[q] = (rb + q < w && jr <= rb + q) ? P[pk(rb + q, jr)] : T(0);
                }
#pragma unroll 4
                for (int kk = 0; kk < c0; ++kk) {
                    const T l = LT[kk * CW + j];
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[q] = fma(-lr[q][kk], l, acc[q]);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (rb + q < w && jr <= rb + q) P[pk(rb + q, jr)] = acc[q];
            }
            __syncthreads();
        }
        // (2) the cw x cw diagonal sub-block, one warp
        if (warp == 0) {
            T row[CW];
#pragma unroll
            for (int j = 0; j < CW; ++j) row[j] = (lane < cw && j <= lane) ? P[pk(c0 + lane, c0 + j)] : T(0);
#pragma unroll
            for (int j = 0; j < CW; ++j) {
                if (j < cw) {
                    const T d = __shfl_sync(0xffffffffu, row[j], j);
                    const bool ok = d > T(0);
                    const T l = ok ? sqrt_rn(d) : T(1);
                    if (lane == 0 && !ok) {
                        atomicOr(&st->flags, (int)ST_ZERO_PIVOT);
                        atomicMin(&st->zero_col, (int)(k + c0 + j + 1));
                    }
                    if (lane == j) row[j] = l;
                    else if (lane > j) row[j] = row[j] / l;               // IEEE division
                    const T lij = row[j];
#pragma unroll
                    for (int kk = j + 1; kk < CW; ++kk) {
                        const T lkj = __shfl_sync(0xffffffffu, row[j], kk);
                        if (lane >= kk && kk < cw) row[kk] = fma(-lij, lkj, row[kk]);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < CW; ++j)
                if (lane < cw && j <= lane) P[pk(c0 + lane, c0 + j)] = row[j];
        }
        __syncthreads();
        // (3) rows below the sub-block: forward substitution with the cw x cw factor
        for (int r = c0 + cw + tid; r < w; r += PTHREADS) {
            // substitution in place in the row's packed storage (no unrolled register array:
            // the kernel stays small enough for the instruction cache)
            T *xr = P + pk(r, c0);
#pragma unroll 1
            for (int j = 0; j < cw; ++j) {
                const T *lj = P + pk(c0 + j, c0);
                T a = xr[j], b = T(0);                 // two interleaved partial sums (even / odd i)
                int i = 0;
#pragma unroll 2
                for (; i + 1 < j; i += 2) {
                    a = fma(-xr[i], lj[i], a);
                    b = fma(-xr[i + 1], lj[i + 1], b);
                }
                if (i < j) a = fma(-xr[i], lj[i], a);
                xr[j] = (a + b) / lj[j];                   // IEEE division
            }
        }
        __syncthreads();
    }
    pdl_trigger();
    // L11 into the lower block, L11^T into the upper block
    for (int i = warp; i < w; i += NW)
        for (int j = lane; j <= i; j += 32) {
            const T v = P[pk(i, j)];
            Wd[(int64_t)i * ldw + j] = v;
            Wd[(int64_t)j * ldw + i] = v;
        }
}

// ---------------------------------------------------------------- C3 L21 = A21 L11^-T
// One CTA per 64 rows of L21, the rows in shared memory.  Left-looking by 32-column chunks:
//   (1) X[:, chunk] -= X[:, 0:32c] L11[chunk, 0:32c]^T   (dot products; L11's chunk rows staged)
//   (2) thread-per-row substitution with the 32 x 32 diagonal factor of the chunk.
constexpr int TRB = 64;          // rows per CTA
constexpr int TTHREADS = 256;

template <typename T>
__global__ void __launch_bounds__(TTHREADS)
trsm_chol_kernel(T *__restrict__ W, int64_t ldw, int64_t k, int w, int64_t n)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ldx = w + 1;
    T *X = reinterpret_cast<T *>(smem_raw);                       // [TRB][w + 1]
    T *LcT = X + round_up((int64_t)TRB * ldx, 4);                 // [w][CW]: L11 rows of the chunk, transposed
    pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x;
    const int64_t r0 = k + w + (int64_t)blockIdx.x * TRB;
    const int nr = (int)std::min<int64_t>(TRB, n - r0);
    const T *Wd = W + k * ldw + k;
    for (int idx = tid; idx < TRB * w; idx += TTHREADS) {
        const int r = idx / w, c = idx - r * w;
        X[r * ldx + c] = r < nr ? W[(r0 + r) * ldw + k + c] : T(0);
    }
    for (int c0 = 0; c0 < w; c0 += CW) {
        const int cw = min(CW, w - c0);
        for (int idx = tid; idx < (c0 + cw) * CW; idx += TTHREADS) {           // the chunk's rows of L11,
            const int kk = idx / CW, j = idx % CW;                              // transposed: LcT[kk][j]
            LcT[idx] = j < cw ? Wd[(int64_t)(c0 + j) * ldw + kk] : T(0);
        }
        __syncthreads();
        if (c0 > 0) {
            // thread -> 2 rows x 4 chunk columns (8 independent chains; 16-byte loads of LcT)
            const int r = 2 * (tid >> 3), jg = (tid & 7) * 4;
            T acc[2][4];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[a][q] = X[(r + a) * ldx + c0 + jg + q];
#pragma unroll 4
            for (int kk = 0; kk < c0; ++kk) {
                const T x0 = X[r * ldx + kk], x1 = X[(r + 1) * ldx + kk];
                T l[4];
                if constexpr (sizeof(T) == 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(LcT + kk * CW + jg);
                    l[0] = v.x; l[1] = v.y; l[2] = v.z; l[3] = v.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) l[q] = LcT[kk * CW + jg + q];
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[0][q] = fma(-x0, l[q], acc[0][q]);
                    acc[1][q] = fma(-x1, l[q], acc[1][q]);
                }
            }
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (jg + q < cw) X[(r + a) * ldx + c0 + jg + q] = acc[a][q];
            __syncthreads();
        }
        if (tid < TRB) {
            T *xr = X + tid * ldx + c0;
#pragma unroll 1
            for (int j = 0; j < cw; ++j) {
                const T *lj = LcT + c0 * CW + j;           // lj[i * CW] = L11(c0 + j, c0 + i)
                T a = xr[j], b = T(0);
                int i = 0;
#pragma unroll 2
                for (; i + 1 < j; i += 2) {
                    a = fma(-xr[i], lj[i * CW], a);
                    b = fma(-xr[i + 1], lj[(i + 1) * CW], b);
                }
                if (i < j) a = fma(-xr[i], lj[i * CW], a);
                xr[j] = (a + b) / lj[j * CW];              // IEEE division
            }
        }
        __syncthreads();
    }
    for (int idx = tid; idx < nr * w; idx += TTHREADS) {              // lower block: rows, coalesced along c
        const int r = idx / w, c = idx - r * w;
        W[(r0 + r) * ldw + k + c] = X[r * ldx + c];
    }
    for (int idx = tid; idx < nr * w; idx += TTHREADS) {              // upper block: L21^T, coalesced along r
        const int c = idx / nr, r = idx - c * nr;
        W[(k + c) * ldw + r0 + r] = X[r * ldx + c];
    }
}

// ---------------------------------------------------------------- C4 L L^T -> unit-lower / upper form
template <typename T>
__global__ void copy_diag_kernel(const T *__restrict__ W, int64_t ldw, int64_t n, T *__restrict__ d)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = W[i * ldw + i];
}

template <typename T>
__global__ void chol_to_lu_kernel(T *__restrict__ W, int64_t ldw, int64_t n, const T *__restrict__ d)
{
    const int64_t i = blockIdx.y;
    for (int64_t i_ = i; i_ < n; i_ += gridDim.y) {
        T *row = W + i_ * ldw;
        const T di = d[i_];
        for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
            row[j] = (j < i_) ? row[j] / d[j] : row[j] * di;          // Lhat = L D^-1, Uhat = D L^T
    }
}

// ---------------------------------------------------------------- C5 symmetric residual products
constexpr int SRT = 256;                    // threads, 2 rows each
constexpr int SROWS = 2 * SRT;              // rows per chunk
constexpr int SCOLS = 256;                  // columns per strip
constexpr int SG = 16;                      // columns per group

// partialD[s][i]: sum over the strip s of a(i, j) x_j, j <= i (rows of chunk c)
// partialT[c][j]: sum over the chunk c of a(i, j) x_i, i > j (columns of strip s)
__global__ void __launch_bounds__(SRT)
symv_partial_kernel(const double *__restrict__ A, int64_t lda, int64_t n, const double *__restrict__ x,
                    double *__restrict__ partialD, double *__restrict__ partialT)
{
    __shared__ double xs[SCOLS];
    __shared__ double red[SRT / 32][SG];
    const int c = blockIdx.x, s = blockIdx.y;
    const int64_t i0c = (int64_t)c * SROWS, j0s = (int64_t)s * SCOLS;
    if (i0c + SROWS - 1 < j0s) return;                       // chunk entirely above the strip's diagonal
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int t = tid; t < SCOLS; t += SRT) xs[t] = j0s + t < n ? x[j0s + t] : 0.0;
    const int64_t i = i0c + 2 * tid;
    const double xi0 = i < n ? x[i] : 0.0, xi1 = i + 1 < n ? x[i + 1] : 0.0;
    __syncthreads();
    const bool vec = (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && i + 1 < n;
    double acc0 = 0.0, acc1 = 0.0;
    for (int g = 0; g < SCOLS; g += SG) {
        const int64_t jg = j0s + g;
        double a0[SG], a1[SG];
#pragma unroll
        for (int u = 0; u < SG; ++u) {
            const int64_t j = jg + u;
            a0[u] = 0.0; a1[u] = 0.0;
            if (j < n && i + 1 >= j) {                       // some of the two rows is on/below the diagonal
                const double *col = A + j * lda + i;
                if (vec && i >= j) {
                    const double2 v = __ldcs(reinterpret_cast<const double2 *>(col));
                    a0[u] = v.x; a1[u] = v.y;
                } else {
                    if (i < n && i >= j) a0[u] = __ldcs(col);
                    if (i + 1 < n) a1[u] = __ldcs(col + 1);
                }
            }
        }
        double v[SG];
#pragma unroll
        for (int u = 0; u < SG; ++u) {
            const int64_t j = jg + u;
            const double xj = xs[g + u];
            acc0 = fma(a0[u], xj, acc0);                     // a0/a1 are zero off the lower triangle
            acc1 = fma(a1[u], xj, acc1);
            // transposed contribution (strictly lower only)
            const double t0 = (i > j) ? a0[u] * xi0 : 0.0;
            v[u] = (i + 1 > j) ? fma(a1[u], xi1, t0) : t0;
        }
        // warp transpose-reduce: lane l (l & 15) ends with the warp's sum for column g + (l & 15)
#pragma unroll
        for (int sh = SG / 2; sh >= 1; sh >>= 1) {
            const bool up = (lane & sh) != 0;
#pragma unroll
            for (int q = 0; q < sh; ++q) {
                const double send = up ? v[q] : v[q + sh];
                const double keep = up ? v[q + sh] : v[q];
                v[q] = keep + __shfl_xor_sync(0xffffffffu, send, sh);
            }
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 16);
        if (lane < SG) red[warp][lane] = v[0];
        __syncthreads();
        if (tid < SG) {
            double tsum = 0.0;
#pragma unroll
            for (int w = 0; w < SRT / 32; ++w) tsum += red[w][tid];
            if (jg + tid < n) partialT[(int64_t)c * n + jg + tid] = tsum;
        }
        __syncthreads();
    }
    if (i < n) partialD[(int64_t)s * n + i] = acc0;
    if (i + 1 < n) partialD[(int64_t)s * n + i + 1] = acc1;
}

__global__ void symv_reduce_kernel(int64_t n, const double *__restrict__ partialD, const double *__restrict__ partialT,
                                   double *__restrict__ ax)
{
    const int64_t nsj = ceil_div(n, SCOLS), nci = ceil_div(n, SROWS);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ci = i / SROWS, si = i / SCOLS;
        double v = 0.0;
        for (int64_t s = 0; s < nsj; ++s)                           // strips whose CTA ran for row chunk ci
            if (ci * SROWS + SROWS - 1 >= s * SCOLS) v += partialD[s * n + i];
        for (int64_t c = 0; c < nci; ++c)                           // chunks whose CTA ran for strip si
            if (c * SROWS + SROWS - 1 >= si * SCOLS) v += partialT[c * n + i];
        ax[i] = v;
    }
}

}  // namespace

// ---------------------------------------------------------------- host launchers
template <typename T>
void launch_demote_sym(const double *A, int64_t lda, int64_t n, T *W, int64_t ldw, double *partials,
                       unsigned *counter, DevStatus *st, int num_sms, cudaStream_t s)
{
    if (n <= 0) return;
    if (ldw > n) MP_CUDA(cudaMemset2DAsync(W + n, ldw * sizeof(T), 0, (ldw - n) * sizeof(T), n, s));
    const int64_t nt = ceil_div(n, DT);
    const int grid = (int)std::min<int64_t>(nt * (nt + 1) / 2, (int64_t)num_sms * 8);
    demote_sym_kernel<T><<<grid, DTHREADS, 0, s>>>(A, lda, n, W, ldw, partials, counter, st);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

size_t demote_sym_partials(int num_sms) { return (size_t)num_sms * 8; }

template <typename T>
int chol_block_max() { return sizeof(T) == 4 ? 256 : 128; }

template <typename T>
void launch_potrf_diag(T *W, int64_t ldw, int64_t k, int w, DevStatus *st, cudaStream_t s)
{
    const int wm = chol_block_max<T>();
    const size_t smem = ((size_t)pk(w, 0) + (size_t)w * CW) * sizeof(T);
    func_smem_once((const void *)potrf_diag_kernel<T>, ((size_t)pk(wm, 0) + (size_t)wm * CW) * sizeof(T));
    launch_ex(potrf_diag_kernel<T>, dim3(1), dim3(PTHREADS), smem, s, nullptr, W, ldw, k, w, st);
}

template <typename T>
void launch_trsm_chol(T *W, int64_t ldw, int64_t k, int w, int64_t n, cudaStream_t s)
{
    const int64_t m = n - k - w;
    if (m <= 0) return;
    const int wm = chol_block_max<T>();
    auto bytes = [](int ww) { return (round_up((int64_t)TRB * (ww + 1), 4) + (size_t)ww * CW) * sizeof(T); };
    func_smem_once((const void *)trsm_chol_kernel<T>, bytes(wm));
    const size_t smem = bytes(w);
    launch_ex(trsm_chol_kernel<T>, dim3((unsigned)ceil_div(m, TRB)), dim3(TTHREADS), smem, s, nullptr, W, ldw, k, w, n);
}

template <typename T>
void launch_chol_to_lu(T *W, int64_t ldw, int64_t n, T *dscratch, cudaStream_t s)
{
    if (n <= 0) return;
    copy_diag_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, s>>>(W, ldw, n, dscratch);
    MP_LAUNCH_CHECK();
    dim3 g((unsigned)std::min<int64_t>(ceil_div(n, 256), 8), (unsigned)std::min<int64_t>(n, 8192));
    chol_to_lu_kernel<T><<<g, 256, 0, s>>>(W, ldw, n, dscratch);
    MP_LAUNCH_CHECK();
    g_launches += 2;
}

size_t symv_partial_elems(int64_t n)
{
    return (size_t)(ceil_div(n, SCOLS) + ceil_div(n, SROWS)) * (size_t)n;
}

void launch_symv_products(const double *A, int64_t lda, int64_t n, int64_t nrhs, const double *X, double *AX,
                          double *partials, cudaStream_t s)
{
    if (n <= 0) return;
    double *pD = partials, *pT = partials + (size_t)ceil_div(n, SCOLS) * n;
    dim3 g((unsigned)ceil_div(n, SROWS), (unsigned)ceil_div(n, SCOLS));
    for (int64_t c = 0; c < nrhs; ++c) {
        symv_partial_kernel<<<g, SRT, 0, s>>>(A, lda, n, X + c * n, pD, pT);
        MP_LAUNCH_CHECK();
        symv_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, s>>>(n, pD, pT, AX + c * n);
        MP_LAUNCH_CHECK();
        g_launches += 2;
    }
}

template void launch_demote_sym<float>(const double *, int64_t, int64_t, float *, int64_t, double *, unsigned *,
                                       DevStatus *, int, cudaStream_t);
template void launch_demote_sym<double>(const double *, int64_t, int64_t, double *, int64_t, double *, unsigned *,
                                        DevStatus *, int, cudaStream_t);
template int chol_block_max<float>();
template int chol_block_max<double>();
template void launch_potrf_diag<float>(float *, int64_t, int64_t, int, DevStatus *, cudaStream_t);
template void launch_potrf_diag<double>(double *, int64_t, int64_t, int, DevStatus *, cudaStream_t);
template void launch_trsm_chol<float>(float *, int64_t, int64_t, int, int64_t, cudaStream_t);
template void launch_trsm_chol<double>(double *, int64_t, int64_t, int, int64_t, cudaStream_t);
template void launch_chol_to_lu<float>(float *, int64_t, int64_t, float *, cudaStream_t);
template void launch_chol_to_lu<double>(double *, int64_t, int64_t, double *, cudaStream_t);

}  // namespace mp
