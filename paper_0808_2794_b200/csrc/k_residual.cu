// k_residual.cu — K8 + K10: binary64 residual with the original A, the
// demoted/permuted correction right-hand side, and the convergence test.
//
// PAPER.md Alg. 1 step 4: r_k <- b - A x_{k-1} in double precision,
// "using the original double precision coefficients".  Step 5's
// right-hand side P r_k is demoted to binary32 here (reading A-10: RN, no
// scaling) and scattered through pinv, so the solve kernels read it directly.
// "check convergence" with B:5's test (readings A-1..A-5):
//   converged  <=>  for all c:  ||r_c||_2 < ||x_c||_2 * cte  or  ||r_c||_2 == 0,
//   cte = ||A||_F * 2^-53 * sqrt(n); any non-finite norm -> ST_NORM_NONFINITE.
//
// HBM-bound: A (8 n^2 bytes, column-major, the caller's layout) is streamed
// once per iteration with coalesced 128-bit loads; the column range is split
// over `splits` CTAs per row tile (split-K) and the partial sums are reduced
// in a fixed order by the finalize kernel (deterministic).
#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace mp {

namespace {

constexpr int RT = 256;              // threads per CTA (2 rows each)
constexpr int ROWS = 2 * RT;         // rows per row tile
constexpr int MAXR = 16;
constexpr int JU = 8;                // column unroll (loads in flight per thread)

template <bool VEC, int R>
__global__ void __launch_bounds__(RT)
residual_partial_kernel(const double *__restrict__ A, int64_t lda, int64_t n, int64_t ncols, int nrhs,
                        const double *__restrict__ X, int64_t ldx, double *__restrict__ partial,
                        int64_t cols_per_split, int c_off, int nrhs_total)
{
    extern __shared__ __align__(16) double xs[];        // [cols_per_split][R]
    const int s = blockIdx.y;
    const int64_t j0 = (int64_t)s * cols_per_split;
    const int64_t j1 = (ncols < j0 + cols_per_split) ? ncols : j0 + cols_per_split;
    const int64_t i = (int64_t)blockIdx.x * ROWS + 2 * threadIdx.x;
    for (int64_t idx = threadIdx.x; idx < (j1 - j0) * nrhs; idx += RT) {
        const int64_t jj = idx / nrhs;
        const int c = (int)(idx - jj * nrhs);
        xs[jj * R + c] = X[c * ldx + j0 + jj];
    }
    __syncthreads();
    double acc0[R], acc1[R];
#pragma unroll
    for (int c = 0; c < R; ++c) { acc0[c] = 0.0; acc1[c] = 0.0; }
    const bool r0 = i < n, r1 = i + 1 < n;
    int64_t j = j0;
    if (VEC && r1) {
        for (; j + JU <= j1; j += JU) {
            double2 a[JU];
#pragma unroll
            for (int u = 0; u < JU; ++u) a[u] = __ldcs(reinterpret_cast<const double2 *>(A + (j + u) * lda + i));
#pragma unroll
            for (int u = 0; u < JU; ++u) {
                const double *xj = xs + (j + u - j0) * R;
#pragma unroll
                for (int c = 0; c < R; ++c)
                    if (c < nrhs) {
                        acc0[c] = fma(a[u].x, xj[c], acc0[c]);
                        acc1[c] = fma(a[u].y, xj[c], acc1[c]);
                    }
            }
        }
    }
    for (; j < j1; ++j) {
        const double *col = A + j * lda;
        const double a0 = r0 ? __ldcs(col + i) : 0.0, a1 = r1 ? __ldcs(col + i + 1) : 0.0;
        const double *xj = xs + (j - j0) * R;
#pragma unroll
        for (int c = 0; c < R; ++c)
            if (c < nrhs) {
                acc0[c] = fma(a0, xj[c], acc0[c]);
                acc1[c] = fma(a1, xj[c], acc1[c]);
            }
    }
    double *ps = partial + ((int64_t)s * nrhs_total + c_off) * n;
#pragma unroll
    for (int c = 0; c < R; ++c)
        if (c < nrhs) {
            if (r0) ps[c * n + i] = acc0[c];
            if (r1) ps[c * n + i + 1] = acc1[c];
        }
}

// The same partial products with ONE row per thread (ROWS threads per CTA) for 9..16 right-hand
// sides: the two-row kernel's 2 x 16 binary64 accumulators kept occupancy at 2 CTAs (16 warps) per SM
// and left it latency-bound (ncu: long-scoreboard stalls, 0.3 of HBM); this one runs 32 warps.
template <int R>
__global__ void __launch_bounds__(ROWS)
residual_partial_r1_kernel(const double *__restrict__ A, int64_t lda, int64_t n, int64_t ncols, int nrhs,
                           const double *__restrict__ X, int64_t ldx, double *__restrict__ partial,
                           int64_t cols_per_split, int c_off, int nrhs_total)
{
    extern __shared__ __align__(16) double xs[];        // [cols_per_split][R]
    const int s = blockIdx.y;
    const int64_t j0 = (int64_t)s * cols_per_split;
    const int64_t j1 = (ncols < j0 + cols_per_split) ? ncols : j0 + cols_per_split;
    const int64_t i = (int64_t)blockIdx.x * ROWS + threadIdx.x;
    for (int64_t idx = threadIdx.x; idx < (j1 - j0) * R; idx += ROWS) {
        const int64_t jj = idx / R;
        const int c = (int)(idx - jj * R);
        xs[idx] = c < nrhs ? X[c * ldx + j0 + jj] : 0.0;
    }
    __syncthreads();
    double acc[R];
#pragma unroll
    for (int c = 0; c < R; ++c) acc[c] = 0.0;
    if (i < n) {
        int64_t j = j0;
        for (; j + JU <= j1; j += JU) {
            double a[JU];
#pragma unroll
            for (int u = 0; u < JU; ++u) a[u] = __ldcs(A + (j + u) * lda + i);
#pragma unroll
            for (int u = 0; u < JU; ++u) {
                const double *xj = xs + (j + u - j0) * R;
#pragma unroll
                for (int c = 0; c < R; ++c) acc[c] = fma(a[u], xj[c], acc[c]);
            }
        }
        for (; j < j1; ++j) {
            const double a0 = __ldcs(A + j * lda + i);
            const double *xj = xs + (j - j0) * R;
#pragma unroll
            for (int c = 0; c < R; ++c) acc[c] = fma(a0, xj[c], acc[c]);
        }
        double *ps = partial + ((int64_t)s * nrhs_total + c_off) * n;
#pragma unroll
        for (int c = 0; c < R; ++c)
            if (c < nrhs) ps[c * n + i] = acc[c];
    }
}

template <typename T>
__global__ void __launch_bounds__(RT)
residual_finalize_kernel(int64_t n, int nrhs, int splits, const double *__restrict__ B, const double *__restrict__ X,
                         const double *__restrict__ partial, double *__restrict__ R, const int32_t *__restrict__ pinv,
                         T *__restrict__ Y, double cte, double *blocksums, unsigned *counter, DevStatus *st)
{
    __shared__ double red[RT / 32][2 * MAXR];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x;
    const int32_t pi = i < n ? pinv[i] : 0;
    for (int cb = 0; cb < nrhs; cb += MAXR) {
        const int nc = (nrhs - cb < MAXR) ? (nrhs - cb) : MAXR;
        for (int cc = 0; cc < nc; ++cc) {
            const int c = cb + cc;
            double rr = 0.0, xx = 0.0;
            if (i < n) {
                double sum = 0.0;
                for (int s = 0; s < splits; ++s) sum += partial[((int64_t)s * nrhs + c) * n + i];
                const double r = B[c * n + i] - sum;
                R[c * n + i] = r;
                Y[c * n + pi] = (T)r;                  // y = fl32(P r)   (A-10)
                const double x = X[c * n + i];
                rr = r * r;
                xx = x * x;
            }
            for (int o = 16; o; o >>= 1) {
                rr += __shfl_xor_sync(0xffffffffu, rr, o);
                xx += __shfl_xor_sync(0xffffffffu, xx, o);
            }
            if (lane == 0) { red[warp][2 * cc] = rr; red[warp][2 * cc + 1] = xx; }
        }
        __syncthreads();
        if (threadIdx.x < 2 * nc) {
            double v = 0.0;
            for (int w = 0; w < RT / 32; ++w) v += red[w][threadIdx.x];
            blocksums[(int64_t)blockIdx.x * 2 * nrhs + 2 * cb + threadIdx.x] = v;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    __shared__ int s_conv, s_bad;
    __shared__ double s_worst;
    if (threadIdx.x == 0) { s_conv = 1; s_bad = 0; s_worst = 0.0; }
    __syncthreads();
    for (int c = threadIdx.x; c < nrhs; c += RT) {     // fixed-order sums over blocks, one column per thread
        double r2 = 0.0, x2 = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) {
            r2 += __ldcg(blocksums + (int64_t)b * 2 * nrhs + 2 * c);
            x2 += __ldcg(blocksums + (int64_t)b * 2 * nrhs + 2 * c + 1);
        }
        const double rn = sqrt(r2), xn = sqrt(x2);
        if (c < MAXR) { st->rn[c] = rn; st->xn[c] = xn; }
        if (!isfinite(rn) || !isfinite(xn)) { atomicOr(&s_bad, 1); continue; }
        const double ratio = rn == 0.0 ? 0.0 : rn / (xn * cte);
        atomicMax(reinterpret_cast<unsigned long long *>(&s_worst), (unsigned long long)__double_as_longlong(ratio));
        if (!(rn < xn * cte || rn == 0.0)) atomicAnd(&s_conv, 0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int conv = s_conv;
        if (s_bad) { atomicOr(&st->flags, (int)ST_NORM_NONFINITE); conv = 0; }
        st->converged = conv;
        st->ratio = s_worst;                          // non-negative doubles order like their bit patterns
        *counter = 0u;
    }
}

}  // namespace

// right-hand sides per partial-kernel instantiation (1, 2, 4, 8, 16): the smallest that holds nc
static int rbucket(int64_t nc) { return nc <= 1 ? 1 : nc <= 2 ? 2 : nc <= 4 ? 4 : nc <= 8 ? 8 : MAXR; }

int64_t residual_splits(int64_t n, int64_t nrhs, int num_sms)
{
    const int64_t tiles = ceil_div(n, ROWS);
    int64_t s = ceil_div((int64_t)num_sms * 8, tiles);
    // the x slice of a split lives in shared memory: at most 64 KB per CTA
    const int64_t r = rbucket(std::min<int64_t>(nrhs, MAXR));
    s = std::max<int64_t>(s, ceil_div(n * r * (int64_t)sizeof(double), 64 * 1024));
    s = std::max<int64_t>(1, std::min<int64_t>(s, ceil_div(n, 64)));
    return s;
}

size_t residual_partial_elems(int64_t n, int64_t nrhs, int num_sms)
{
    return (size_t)residual_splits(n, nrhs, num_sms) * (size_t)nrhs * (size_t)n;
}

// split-K partial products of a rows x cols block: partial[s][c][i]
static int64_t launch_partials(const double *A, int64_t lda, int64_t rows, int64_t cols, int64_t nrhs,
                               const double *X, int64_t ldx, ResidualScratch &rs, int num_sms, cudaStream_t s)
{
    const int nr = (int)nrhs;
    const int64_t splits = residual_splits(std::max(rows, cols), nrhs, num_sms);
    const int64_t cps = ceil_div(cols, splits);
    const int64_t real_splits = ceil_div(cols, cps);
    dim3 g1((unsigned)ceil_div(rows, ROWS), (unsigned)real_splits);
    const bool vec = (lda % 2 == 0) && (((uintptr_t)A & 15) == 0);
    for (int c0 = 0; c0 < nr; c0 += MAXR) {
        const int nc = std::min(MAXR, nr - c0);
        const int rb = rbucket(nc);
        const size_t smem = (size_t)cps * rb * sizeof(double);
        using KF = void (*)(const double *, int64_t, int64_t, int64_t, int, const double *, int64_t, double *, int64_t,
                            int, int);
        const KF kv[5] = {residual_partial_kernel<true, 1>, residual_partial_kernel<true, 2>,
                          residual_partial_kernel<true, 4>, residual_partial_kernel<true, 8>,
                          residual_partial_kernel<true, MAXR>};
        const KF ks[5] = {residual_partial_kernel<false, 1>, residual_partial_kernel<false, 2>,
                          residual_partial_kernel<false, 4>, residual_partial_kernel<false, 8>,
                          residual_partial_kernel<false, MAXR>};
        const int bi = rb == 1 ? 0 : rb == 2 ? 1 : rb == 4 ? 2 : rb == 8 ? 3 : 4;
        auto kern = vec ? kv[bi] : ks[bi];
        static const bool r1_off = std::getenv("MP_RESIDUAL_R1_OFF") != nullptr;
        if (rb == MAXR && !r1_off) {                 // 9..16 right-hand sides: one row per thread
            auto k1 = residual_partial_r1_kernel<MAXR>;
            if (smem > 48 * 1024) func_smem_once((const void *)k1, smem);
            k1<<<g1, ROWS, smem, s>>>(A, lda, rows, cols, nc, X + c0 * ldx, ldx, rs.partial, cps, c0, nr);
            continue;
        }
        if (smem > 48 * 1024) func_smem_once((const void *)kern, smem);
        kern<<<g1, RT, smem, s>>>(A, lda, rows, cols, nc, X + c0 * ldx, ldx, rs.partial, cps, c0, nr);
    }
    MP_LAUNCH_CHECK();
    g_launches += ceil_div(nr, MAXR);
    return real_splits;
}

__global__ void reduce_splits_kernel(const double *__restrict__ partial, int64_t count, int splits, double *__restrict__ out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int s = 0; s < splits; ++s) v += partial[(int64_t)s * count + i];
        out[i] = v;
    }
}

void launch_residual_products(const double *A, int64_t lda, int64_t rows, int64_t cols, int64_t nrhs,
                              const double *X, int64_t ldx, double *AX, ResidualScratch &rs, int num_sms,
                              cudaStream_t s)
{
    if (cols <= 0) {
        MP_CUDA(cudaMemsetAsync(AX, 0, (size_t)rows * nrhs * sizeof(double), s));
        return;
    }
    const int64_t splits = launch_partials(A, lda, rows, cols, nrhs, X, ldx, rs, num_sms, s);
    const int64_t count = rows * nrhs;
    reduce_splits_kernel<<<(int)std::min<int64_t>(ceil_div(count, 256), 1024), 256, 0, s>>>(rs.partial, count,
                                                                                              (int)splits, AX);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template <typename T>
void launch_residual_finalize(const double *AX, int64_t n, int64_t nrhs, const double *B, const double *X, double *R,
                              const int32_t *pinv, T *Y, double cte, ResidualScratch &rs, DevStatus *st,
                              cudaStream_t s)
{
    const int g2 = (int)ceil_div(n, RT);
    residual_finalize_kernel<T><<<g2, RT, 0, s>>>(n, (int)nrhs, 1, B, X, AX, R, pinv, Y, cte, rs.blocksums,
                                                  rs.counter, st);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template <typename T>
void launch_residual(const double *A, int64_t lda, int64_t n, int64_t nrhs, const double *B, const double *X,
                     double *R, const int32_t *pinv, T *Y, double cte, ResidualScratch &rs, DevStatus *st,
                     int num_sms, cudaStream_t s)
{
    const int64_t splits = launch_partials(A, lda, n, n, nrhs, X, n, rs, num_sms, s);
    const int g2 = (int)ceil_div(n, RT);
    residual_finalize_kernel<T><<<g2, RT, 0, s>>>(n, (int)nrhs, (int)splits, B, X, rs.partial, R, pinv, Y, cte,
                                                  rs.blocksums, rs.counter, st);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template void launch_residual_finalize<float>(const double *, int64_t, int64_t, const double *, const double *,
                                              double *, const int32_t *, float *, double, ResidualScratch &,
                                              DevStatus *, cudaStream_t);
template void launch_residual_finalize<double>(const double *, int64_t, int64_t, const double *, const double *,
                                               double *, const int32_t *, double *, double, ResidualScratch &,
                                               DevStatus *, cudaStream_t);
template void launch_residual<float>(const double *, int64_t, int64_t, int64_t, const double *, const double *,
                                     double *, const int32_t *, float *, double, ResidualScratch &, DevStatus *, int,
                                     cudaStream_t);

}  // namespace mp
