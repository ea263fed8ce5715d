// k_demote.cu — K1: demotion of A to binary32 + ||A||_F, and K6: demotion /
// permutation of the right-hand side.
//
// "The coefficient matrix A is converted to single
// precision for the LU factorization"; B:5: the stop test uses ||A||_F of the
// original binary64 A (reading A-2).  Rounding is RN-even (cvt.rn.f32.f64,
// no .ftz: reading A-9).  The kernel also transposes column-major A into the
// row-major working copy W, so its cost is
// one coalesced read of A (8 n^2 B) and one coalesced write of W (4 n^2 B):
// HBM-bound, algorithmic bytes 12 n^2 per launch.
#include <algorithm>

#include "internal.h"

namespace mp {

namespace {

constexpr int TILE = 64;
constexpr int THREADS = 256;

__device__ __forceinline__ float to_low(double a) { return __double2float_rn(a); }

template <typename T, bool VEC>
__global__ void __launch_bounds__(THREADS)
demote_transpose_kernel(const double *__restrict__ A, int64_t lda, int64_t n, int64_t ncols, T *__restrict__ W,
                        int64_t ldw, double *__restrict__ partials, unsigned *counter, DevStatus *st)
{
    constexpr bool LOW = sizeof(T) == 4;
    __shared__ T tile[TILE][TILE + 1];            // [col][row]
    __shared__ double red[THREADS / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t tiles_i = ceil_div(n, TILE), tiles_j = ldw / TILE;
    const int64_t ntiles = tiles_i * tiles_j;
    double ss = 0.0;
    int flags = 0;

    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t i0 = (t % tiles_i) * TILE, j0 = (t / tiles_i) * TILE;
        // ---- load 64 columns x 64 rows of A (column-major, coalesced along i)
#pragma unroll
        for (int p = 0; p < TILE / 8; ++p) {
            const int jj = warp + 8 * p;
            const int64_t j = j0 + jj;
            const int ii = lane * 2;
            const int64_t i = i0 + ii;
            double a0 = 0.0, a1 = 0.0;
            if (j < ncols) {
                const double *col = A + j * lda;
                if (VEC && i + 1 < n) {
                    double2 v = __ldcs(reinterpret_cast<const double2 *>(col + i));
                    a0 = v.x; a1 = v.y;
                } else {
                    if (i < n) a0 = __ldcs(col + i);
                    if (i + 1 < n) a1 = __ldcs(col + i + 1);
                }
            }
            if (LOW) {
                const float f0 = to_low(a0), f1 = to_low(a1);
                // A-6: non-finite A is an argument error; finite |a| > FLT_MAX overflows (iters = -2)
                if (!isfinite(a0) || !isfinite(a1)) flags |= ST_A_NONFINITE;
                else if (isinf(f0) || isinf(f1)) flags |= ST_OVERFLOW;
                ss = fma(a0, a0, ss);
                ss = fma(a1, a1, ss);
                tile[jj][ii] = (T)f0;
                tile[jj][ii + 1] = (T)f1;
            } else {
                if (!isfinite(a0) || !isfinite(a1)) flags |= ST_A_NONFINITE;
                tile[jj][ii] = (T)a0;
                tile[jj][ii + 1] = (T)a1;
            }
        }
        __syncthreads();
        // ---- store 64 rows x 64 columns of W (row-major, coalesced along j)
#pragma unroll
        for (int p = 0; p < TILE / 8; ++p) {
            const int ii = warp + 8 * p;
            const int64_t i = i0 + ii;
            if (i < n) {
                const int jj = lane * 2;
                T *row = W + i * ldw + j0 + jj;
                if (LOW) {
                    float2 v = make_float2((float)tile[jj][ii], (float)tile[jj + 1][ii]);
                    *reinterpret_cast<float2 *>(row) = v;
                } else {
                    row[0] = tile[jj][ii];
                    row[1] = tile[jj + 1][ii];
                }
            }
        }
        __syncthreads();
    }

    if (!LOW) {
        flags = __reduce_or_sync(0xffffffffu, flags);
        if (lane == 0 && flags && st) atomicOr(&st->flags, flags);
        return;
    }
    // ---- deterministic reduction of sum(a^2): warp -> block -> last block over blocks
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0) {
        red[warp] = ss;
        if (flags) atomicOr(&st->flags, flags);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < THREADS / 32; ++w) b += red[w];
        partials[blockIdx.x] = b;
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        double b = 0.0;
        for (int64_t k = threadIdx.x; k < gridDim.x; k += THREADS) b += __ldcg(partials + k);
        for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
        if (lane == 0) red[warp] = b;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int w = 0; w < THREADS / 32; ++w) tot += red[w];
            st->anrm2 = tot;
            *counter = 0u;
        }
    }
}

template <typename T>
__global__ void permute_demote_rhs_kernel(const double *__restrict__ B, int64_t n, int64_t nrhs,
                                          const int32_t *__restrict__ pinv, T *__restrict__ Y,
                                          DevStatus *st)
{
    int flags = 0;
    const int64_t tot = n * nrhs;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / n, i = t - c * n;
        const double b = B[t];
        if (!isfinite(b)) flags |= ST_B_NONFINITE;
        Y[c * n + pinv[i]] = (T)b;   // y = P b (P applied as the scatter through pinv); RN demotion
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if ((threadIdx.x & 31) == 0 && flags) atomicOr(&st->flags, flags);
}

template <typename T>
__global__ void transpose_out_kernel(const T *__restrict__ W, int64_t ldw, int64_t n, T *__restrict__ LU)
{
    __shared__ T tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + r, j = j0 + threadIdx.x;
        if (i < n && j < n) tile[r][threadIdx.x] = W[i * ldw + j];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t j = j0 + r, i = i0 + threadIdx.x;
        if (i < n && j < n) LU[j * n + i] = tile[threadIdx.x][r];
    }
}

}  // namespace

template <typename T>
void launch_transpose_out(const T *W, int64_t ldw, int64_t n, T *LU, cudaStream_t s)
{
    dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32));
    transpose_out_kernel<T><<<grid, dim3(32, 8), 0, s>>>(W, ldw, n, LU);
    MP_LAUNCH_CHECK();
    ++g_launches;
}
template void launch_transpose_out<float>(const float *, int64_t, int64_t, float *, cudaStream_t);
template void launch_transpose_out<double>(const double *, int64_t, int64_t, double *, cudaStream_t);

template <typename T>
void launch_demote_rect(const double *A, int64_t lda, int64_t n, int64_t ncols, T *W, int64_t ldw, double *partials,
                             unsigned *counter, DevStatus *st, cudaStream_t s)
{
    const int64_t ntiles = ceil_div(n, TILE) * (ldw / TILE);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sms * 8);
    const bool vec = (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    if (vec)
        demote_transpose_kernel<T, true><<<grid, THREADS, 0, s>>>(A, lda, n, ncols, W, ldw, partials, counter, st);
    else
        demote_transpose_kernel<T, false><<<grid, THREADS, 0, s>>>(A, lda, n, ncols, W, ldw, partials, counter, st);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template <typename T>
void launch_demote_transpose(const double *A, int64_t lda, int64_t n, T *W, int64_t ldw, double *partials,
                             unsigned *counter, DevStatus *st, cudaStream_t s)
{
    launch_demote_rect<T>(A, lda, n, n, W, ldw, partials, counter, st, s);
}

template <typename T>
void launch_permute_demote_rhs(const double *B, int64_t n, int64_t nrhs, const int32_t *pinv, T *Y,
                               DevStatus *st, cudaStream_t s)
{
    const int64_t tot = n * nrhs;
    const int grid = (int)std::min<int64_t>(ceil_div(tot, 256), 4096);
    permute_demote_rhs_kernel<T><<<grid, 256, 0, s>>>(B, n, nrhs, pinv, Y, st);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

// W[i][c0 + c] = S[perm[i]][c] for i < n, c < ncols (S row-major, lds): a demoted column block, received in
// the original row order, brought to the current row order of the factorisation (streamed e2e path).
__global__ void gather_rows_kernel(const float *__restrict__ S, int64_t lds, int64_t ncols, const int32_t *__restrict__ perm,
                                   int64_t n, float *__restrict__ W, int64_t ldw)
{
    const int64_t q4 = ncols / 4;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const float4 *src = reinterpret_cast<const float4 *>(S + (int64_t)perm[i] * lds);
        float4 *dst = reinterpret_cast<float4 *>(W + i * ldw);
        for (int64_t c = threadIdx.x; c < q4; c += blockDim.x) dst[c] = src[c];
    }
}

void launch_gather_rows(const float *S, int64_t lds, int64_t ncols, const int32_t *perm, int64_t n, float *W,
                        int64_t ldw, cudaStream_t s)
{
    if (n <= 0 || ncols <= 0) return;
    if ((ncols % 4) || (lds % 4) || (ldw % 4) || (reinterpret_cast<uintptr_t>(W) & 15) || (reinterpret_cast<uintptr_t>(S) & 15))
        throw CudaError{cudaErrorInvalidValue, "gather_rows: 16-byte aligned rows required", __LINE__};
    gather_rows_kernel<<<(unsigned)std::min<int64_t>(n, 8192), 256, 0, s>>>(S, lds, ncols, perm, n, W, ldw);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template void launch_demote_rect<float>(const double *, int64_t, int64_t, int64_t, float *, int64_t, double *,
                                        unsigned *, DevStatus *, cudaStream_t);
template void launch_demote_rect<double>(const double *, int64_t, int64_t, int64_t, double *, int64_t, double *,
                                         unsigned *, DevStatus *, cudaStream_t);
template void launch_demote_transpose<float>(const double *, int64_t, int64_t, float *, int64_t, double *,
                                             unsigned *, DevStatus *, cudaStream_t);
template void launch_demote_transpose<double>(const double *, int64_t, int64_t, double *, int64_t, double *,
                                              unsigned *, DevStatus *, cudaStream_t);
template void launch_permute_demote_rhs<float>(const double *, int64_t, int64_t, const int32_t *, float *,
                                               DevStatus *, cudaStream_t);
template void launch_permute_demote_rhs<double>(const double *, int64_t, int64_t, const int32_t *, double *,
                                                DevStatus *, cudaStream_t);

}  // namespace mp
