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
#include <cstdlib>

#include "internal.h"

namespace mp {

namespace {

constexpr int LT = 256;

// SW columns per CTA (32: one lane per column; 8: a warp instruction covers 4 rows x 8 columns
// = 32-byte row segments, 4x the CTAs for narrow column ranges such as one panel's columns)
template <typename T, int SW>
__global__ void __launch_bounds__(LT)
laswp_pairs_kernel(T *__restrict__ W, int64_t ldw, const int32_t *__restrict__ pairs,
                   const int32_t *__restrict__ npairs, int max_pairs, int64_t c_lo, int64_t c_hi, int64_t x_lo,
                   int64_t x_hi, int32_t *__restrict__ perm, int nstrips, EmitJob ej)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    pdl_trigger();
    const int np = *npairs;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nfirst = nstrips + (perm ? 1 : 0);
    if ((int)blockIdx.x >= nfirst) {           // extra CTAs: the panel-level pair emission (emit_pairs)
        const int64_t stride = (int64_t)(gridDim.x - nfirst) * LT;
        for (int64_t i = ej.k + (int64_t)(blockIdx.x - nfirst) * LT + threadIdx.x; i < ej.n; i += stride) {
            const int32_t o = ej.orig[i];
            if (o != (int32_t)i) {
                const int slot = atomicAdd(ej.npairs, 1);
                ej.pairs[2 * slot] = (int32_t)i;
                ej.pairs[2 * slot + 1] = o;
            }
        }
        return;
    }
    if ((int)blockIdx.x == nstrips) {          // extra CTA: compose the running permutation
        int32_t *tmp = reinterpret_cast<int32_t *>(smem_raw);
        for (int i = threadIdx.x; i < np; i += LT) tmp[i] = perm[pairs[2 * i + 1]];
        __syncthreads();
        for (int i = threadIdx.x; i < np; i += LT) perm[pairs[2 * i]] = tmp[i];
        return;
    }
    T *buf = reinterpret_cast<T *>(smem_raw);  // [np][SW]
    const int64_t s0 = c_lo + (int64_t)blockIdx.x * SW;
    if (s0 >= x_lo && s0 + SW <= x_hi) return;   // strip entirely inside the excluded panel
    constexpr int RPW = 32 / SW;                 // rows per warp instruction
    const int cl = lane % SW, rs = lane / SW;
    const int64_t col = s0 + cl;
    const bool valid = col < c_hi && !(col >= x_lo && col < x_hi);
    // U row groups per warp per round: all pair indices, then all row loads, in flight together.
    // The pair entries below max_pairs (the list's capacity) are read without waiting for the count
    // (one dependent round trip fewer; entries at or beyond the count are masked afterwards).
    constexpr int U = 8, NW = LT / 32, STEP = NW * RPW;
    for (int i0 = warp * RPW + rs; i0 < max_pairs; i0 += STEP * U) {
        int32_t src[U];
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + STEP * u;
            src[u] = i < max_pairs ? pairs[2 * i + 1] : 0;
        }
        if (i0 >= np) break;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + STEP * u;
            v[u] = (i < np && valid) ? W[(int64_t)src[u] * ldw + col] : T(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + STEP * u;
            if (i < np) buf[i * SW + cl] = v[u];
        }
    }
    __syncthreads();
    for (int i0 = warp * RPW + rs; i0 < np; i0 += STEP * U) {
        int32_t dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + STEP * u;
            dst[u] = i < np ? pairs[2 * i] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + STEP * u;
            if (i < np && valid) W[(int64_t)dst[u] * ldw + col] = buf[i * SW + cl];
        }
    }
}

__global__ void init_perm_kernel(int32_t *perm, int64_t n)
{
    pdl_wait();
    pdl_trigger();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        perm[i] = (int32_t)i;
}

__global__ void invert_perm_kernel(const int32_t *perm, int32_t *pinv, int64_t n)
{
    pdl_wait();
    pdl_trigger();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        pinv[perm[t]] = (int32_t)t;
}

}  // namespace

template <typename T>
void launch_laswp_pairs(T *W, int64_t ldw, const int32_t *pairs, const int32_t *npairs, int max_pairs,
                        int64_t c_lo, int64_t c_hi, int64_t x_lo, int64_t x_hi, int32_t *perm, cudaStream_t s, const EmitJob &ej)
{
    // narrow column ranges (one panel's columns): 8-column strips, 4x the CTAs
    static const bool allnarrow = [] { const char *e = std::getenv("MP_LASWP_WIDE"); return !(e && e[0] == '1'); }();
    const bool narrow = allnarrow || c_hi - c_lo <= 1024;
    const int sw = narrow ? 8 : 32;
    const int nstrips = c_hi > c_lo ? (int)ceil_div(c_hi - c_lo, sw) : 0;
    const int nemit = ej.orig ? (int)std::min<int64_t>(ceil_div(ej.n - ej.k, LT), 64) : 0;
    const int grid = nstrips + (perm ? 1 : 0) + nemit;
    if (grid == 0) return;
    const size_t smem = std::max<size_t>((size_t)max_pairs * sw * sizeof(T), (size_t)max_pairs * 4);
    auto kern = narrow ? laswp_pairs_kernel<T, 8> : laswp_pairs_kernel<T, 32>;
    if (smem > 48 * 1024) func_smem_once((const void *)kern, smem);
    launch_ex(kern, dim3(grid), dim3(LT), smem, s, nullptr, W, ldw, pairs, npairs, max_pairs, c_lo, c_hi, x_lo, x_hi,
              perm, nstrips, ej);
}

void launch_init_perm(int32_t *perm, int64_t n, cudaStream_t s)
{
    launch_ex(init_perm_kernel, dim3((unsigned)std::min<int64_t>(ceil_div(n, 256), 1024)), dim3(256), 0, s, nullptr,
              perm, n);
}

void launch_invert_perm(const int32_t *perm, int32_t *pinv, int64_t n, cudaStream_t s)
{
    launch_ex(invert_perm_kernel, dim3((unsigned)std::min<int64_t>(ceil_div(n, 256), 1024)), dim3(256), 0, s, nullptr,
              perm, pinv, n);
}

template void launch_laswp_pairs<float>(float *, int64_t, const int32_t *, const int32_t *, int, int64_t, int64_t,
                                        int64_t, int64_t, int32_t *, cudaStream_t, const EmitJob &);
template void launch_laswp_pairs<double>(double *, int64_t, const int32_t *, const int32_t *, int, int64_t,
                                         int64_t, int64_t, int64_t, int32_t *, cudaStream_t, const EmitJob &);

}  // namespace mp
