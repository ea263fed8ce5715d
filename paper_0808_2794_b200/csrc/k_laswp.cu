// k_laswp.cu — K3: row interchanges (LAPACK xLASWP semantics).
//
// A leaf panel factorisation produces its interchanges as a list of
// (position <- origin row) pairs (at most 2w rows move for w sequential
// swaps).  Applying that list to the columns outside the panel is a gather:
// every CTA owns a 32-column strip, reads all origin rows of its strip into
// shared memory, then writes them to their positions — the result equals the
// sequential swaps of ipiv.  In the row-major working copy each pair moves a
// contiguous 128 B segment per strip: coalesced, HBM/L2-bound, 2 x 4 B x
// (#pairs) x (#columns) algorithmic bytes.
#include <algorithm>

#include "internal.h"

namespace mp {

namespace {

constexpr int LT = 256;
constexpr int STRIP = 32;

template <typename T>
__global__ void __launch_bounds__(LT)
laswp_pairs_kernel(T *__restrict__ W, int64_t ldw, const int32_t *__restrict__ pairs,
                   const int32_t *__restrict__ npairs, int64_t c_lo, int64_t c_hi, int64_t x_lo,
                   int64_t x_hi, int32_t *__restrict__ perm, int nstrips)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int np = *npairs;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if ((int)blockIdx.x == nstrips) {          // extra CTA: compose the running permutation
        int32_t *tmp = reinterpret_cast<int32_t *>(smem_raw);
        for (int i = threadIdx.x; i < np; i += LT) tmp[i] = perm[pairs[2 * i + 1]];
        __syncthreads();
        for (int i = threadIdx.x; i < np; i += LT) perm[pairs[2 * i]] = tmp[i];
        return;
    }
    T *buf = reinterpret_cast<T *>(smem_raw);  // [np][STRIP]
    const int64_t s0 = c_lo + (int64_t)blockIdx.x * STRIP;
    if (s0 >= x_lo && s0 + STRIP <= x_hi) return;   // strip entirely inside the excluded panel
    const int64_t col = s0 + lane;
    const bool valid = col < c_hi && !(col >= x_lo && col < x_hi);
    for (int i = warp; i < np; i += LT / 32) {
        const int64_t src = pairs[2 * i + 1];
        buf[i * STRIP + lane] = valid ? W[src * ldw + col] : T(0);
    }
    __syncthreads();
    for (int i = warp; i < np; i += LT / 32) {
        const int64_t dst = pairs[2 * i];
        if (valid) W[dst * ldw + col] = buf[i * STRIP + lane];
    }
}

__global__ void init_perm_kernel(int32_t *perm, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        perm[i] = (int32_t)i;
}

__global__ void invert_perm_kernel(const int32_t *perm, int32_t *pinv, int64_t n)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        pinv[perm[t]] = (int32_t)t;
}

}  // namespace

template <typename T>
void launch_laswp_pairs(T *W, int64_t ldw, const int32_t *pairs, const int32_t *npairs, int max_pairs,
                        int64_t c_lo, int64_t c_hi, int64_t x_lo, int64_t x_hi, int32_t *perm, cudaStream_t s)
{
    const int nstrips = c_hi > c_lo ? (int)ceil_div(c_hi - c_lo, STRIP) : 0;
    const int grid = nstrips + (perm ? 1 : 0);
    if (grid == 0) return;
    const size_t smem = std::max<size_t>((size_t)max_pairs * STRIP * sizeof(T), (size_t)max_pairs * 4);
    auto kern = laswp_pairs_kernel<T>;
    if (smem > 48 * 1024) func_smem_once((const void *)kern, smem);
    kern<<<grid, LT, smem, s>>>(W, ldw, pairs, npairs, c_lo, c_hi, x_lo, x_hi, perm, nstrips);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

void launch_init_perm(int32_t *perm, int64_t n, cudaStream_t s)
{
    init_perm_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, s>>>(perm, n);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

void launch_invert_perm(const int32_t *perm, int32_t *pinv, int64_t n, cudaStream_t s)
{
    invert_perm_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, s>>>(perm, pinv, n);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template void launch_laswp_pairs<float>(float *, int64_t, const int32_t *, const int32_t *, int, int64_t, int64_t,
                                        int64_t, int64_t, int32_t *, cudaStream_t);
template void launch_laswp_pairs<double>(double *, int64_t, const int32_t *, const int32_t *, int, int64_t,
                                         int64_t, int64_t, int64_t, int32_t *, cudaStream_t);

}  // namespace mp
