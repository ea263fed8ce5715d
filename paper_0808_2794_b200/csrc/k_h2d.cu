// k_h2d.cu — host-to-device copy of A's column blocks by SM loads over PCIe (the streamed e2e path).
//
// The end-to-end call takes A in host memory (8 n^2 bytes): it crosses PCIe while the
// factorisation runs.  A copy-engine DMA writes every byte through L2 with normal priority, and
// at ~57 GB/s over the ~38 ms of the copy that evicts the panel chain's working set (the leaf,
// interchange and in-panel kernels, latency-bound and L2-resident, ran 2-4x slower while the DMA
// was active; profiles/r02_e2e_timeline_*.txt).  Here a few CTAs read the pinned host block
// through its device mapping (16-byte loads, several in flight per thread) and store it with an
// L2 evict-first policy, so A's bytes leave L2 first and the panel's lines stay.
// HBM traffic: 8 bytes written per element (the same as the DMA); PCIe-bound.
#include "internal.h"

namespace mp {

namespace {

constexpr int H2D_THREADS = 512;
constexpr int H2D_UNROLL = 8;

__device__ __forceinline__ uint64_t evict_first_policy()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// columns [0, ncols) of a column-major block (host ld lda_h) into dA (ld n); n even, 16-byte aligned
__global__ void __launch_bounds__(H2D_THREADS)
h2d_cols_kernel(const double *__restrict__ hA, int64_t lda_h, double *__restrict__ dA, int64_t n, int64_t ncols)
{
    const uint64_t pol = evict_first_policy();
    const int64_t per_col = n / 2;                             // 16-byte units per column
    const int64_t total = per_col * ncols;
    const int64_t stride = (int64_t)gridDim.x * H2D_THREADS;
    for (int64_t u0 = (int64_t)blockIdx.x * H2D_THREADS + threadIdx.x; u0 < total; u0 += stride * H2D_UNROLL) {
        double2 v[H2D_UNROLL];
#pragma unroll
        for (int q = 0; q < H2D_UNROLL; ++q) {
            const int64_t u = u0 + q * stride;
            if (u < total) {
                const int64_t j = u / per_col, i = (u - j * per_col) * 2;
                const double *src = hA + j * lda_h + i;
                asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                             : "=d"(v[q].x), "=d"(v[q].y)
                             : "l"(src));
            }
        }
#pragma unroll
        for (int q = 0; q < H2D_UNROLL; ++q) {
            const int64_t u = u0 + q * stride;
            if (u < total) {
                const int64_t j = u / per_col, i = (u - j * per_col) * 2;
                double *dst = dA + j * n + i;
                asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(dst),
                             "d"(v[q].x), "d"(v[q].y), "l"(pol)
                             : "memory");
            }
        }
    }
}

}  // namespace

// Device-accessible address of a host pointer (pinned / registered memory), else nullptr.
const double *h2d_device_view(const double *hA)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, hA) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    if (at.type != cudaMemoryTypeHost || at.devicePointer == nullptr) return nullptr;
    return static_cast<const double *>(at.devicePointer);
}

bool launch_h2d_cols(const double *hA_dev, int64_t lda_h, double *dA, int64_t n, int64_t ncols, int nctas,
                     cudaStream_t s)
{
    if ((n & 1) || (lda_h & 1) || (reinterpret_cast<uintptr_t>(hA_dev) & 15) ||
        (reinterpret_cast<uintptr_t>(dA) & 15))
        return false;
    if (ncols <= 0) return true;
    launch_ex(h2d_cols_kernel, dim3(nctas), dim3(H2D_THREADS), 0, s, nullptr, hA_dev, lda_h, dA, n, ncols);
    return true;
}

}  // namespace mp
