// Micro-benchmark: cycles of one diag_solve (k_solve.cu) call by one warp, tile resident in smem.
#include <cstdio>
#include "../paper_0808_2794_b200/csrc/internal.h"
namespace mp {
thread_local int64_t g_launches = 0;
void func_smem_once(const void *fn, size_t bytes) { cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes); }
void func_cluster16_once(const void *fn) { cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); }
bool pdl_enabled() { return false; }
}
#include "../paper_0808_2794_b200/csrc/k_solve.cu"
using namespace mp;
template <typename T, bool LOWER>
__global__ void kdiag(const T *g, T *out, long long *cyc, int iters, int mode, unsigned *gflag, const float *big)
{
    __shared__ __align__(1024) T dg[BS * BS];
    __shared__ __align__(128) float tbuf[2][2048];
    __shared__ T rinv[BS];
    __shared__ __align__(8) uint64_t bar;
    __shared__ volatile int done;
    if (blockIdx.x > 0) {                                  // other SMs: stream HBM until CTA 0 is done
        float acc = 0.f;
        const float4 *bp = reinterpret_cast<const float4 *>(big);
        for (long long k = 0; ld_relaxed_u32(gflag + 1) == 0; ++k) {
            const size_t base = ((size_t)(k * gridDim.x + blockIdx.x) * blockDim.x * 8) % ((size_t)4096 * 4096 / 4 - 8 * 1024);
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(bp + base + u * blockDim.x + threadIdx.x);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].w;
        }
        if (acc == 1.2345f) out[1] = acc;
        return;
    }
    for (int i = threadIdx.x; i < BS * BS; i += blockDim.x) dg[i] = g[i];
    if (threadIdx.x == 0) { mbar_init(&bar, 1); done = 0; }
    __syncthreads();
    if (threadIdx.x >= 32) {
        if (mode == 5) {                                   // 4 warps: tile-GEMV-like LDS.128 traffic
            float acc = 0.f;
            const float4 *tp = reinterpret_cast<const float4 *>(tbuf[0]);
            for (long long k = 0; !done; ++k) {
#pragma unroll 8
                for (int q = 0; q < 64; ++q) {
                    const float4 v = tp[((threadIdx.x & 127) + 32 * q) & 511];
                    acc += v.x * v.y + v.z * v.w;
                }
            }
            if (acc == 1234.5f) out[0] = acc;
            return;
        }
        if (threadIdx.x == 32) {
            if (mode == 1) mbar_wait(&bar, 0);
            if (mode == 2) while (ld_relaxed_u32(gflag) == 0 && !done) {}
            if (mode == 3) while (!done) {}
            if (mode == 4) {                                   // bulk copies global -> smem, 16 KB each
                __shared__ __align__(8) uint64_t tb;
                mbar_init(&tb, 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                uint32_t ph = 0;
                for (long long k = 0; !done; ++k) {
                    mbar_expect_tx(&tb, 2 * 8192);
                    for (int q = 0; q < 2; ++q)
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                     :: "r"(smem_u32(tbuf[q])), "l"(big + ((k * 4 + q) % 4096) * 4096), "r"(8192), "r"(smem_u32(&tb)) : "memory");
                    mbar_wait(&tb, ph); ph ^= 1;
                }
            }
        }
        return;
    }
    const int lane = threadIdx.x;
    T v0 = T(lane) * T(0.01), v1 = T(lane) * T(0.02);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        diag_solve<T, LOWER>(dg, rinv, lane, BS, v0, v1);
        v0 = v0 * T(1e-3) + T(1); v1 = v1 * T(1e-3) + T(1);
    }
    long long t1 = clock64();
    out[lane] = v0 + v1;
    if (lane == 0) { done = 1; mbar_arrive(&bar); }
    if (lane == 0) { *cyc = (t1 - t0) / iters; st_release_u32(gflag + 1, 1u); }
}
template <typename T, bool LOWER>
void run(const char *name)
{
    T h[BS * BS];
    for (int i = 0; i < BS * BS; ++i) h[i] = T(1) + T(i % 7) * T(0.01);
    T *g, *o; long long *c;
    cudaMalloc(&g, sizeof(h)); cudaMalloc(&o, 64 * sizeof(T)); cudaMalloc(&c, 8);
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
    unsigned *fl; cudaMalloc(&fl, 8); cudaMemset(fl, 0, 8);
    float *big; cudaMalloc(&big, (size_t)4096 * 4096 * 4);
    for (int mode = 0; mode < 6; ++mode) {
        cudaMemset(fl, 0, 8);
        kdiag<T, LOWER><<<1, mode == 5 ? 160 : 64>>>(g, o, c, 1000, mode, fl, big);
        long long cy0; cudaMemcpy(&cy0, c, 8, cudaMemcpyDeviceToHost);
        if (mode == 0) {
            cudaMemset(fl, 0, 8);
            kdiag<T, LOWER><<<148, 64>>>(g, o, c, 1000, mode, fl, big);
            long long cy1; cudaMemcpy(&cy1, c, 8, cudaMemcpyDeviceToHost);
            printf("%s mode 0 with 147 streaming CTAs: %lld cycles (%s)\n", name, cy1, cudaGetErrorString(cudaGetLastError()));
        }
        long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("%s mode %d: %lld cycles / diag_solve (%s)\n", name, mode, cy, cudaGetErrorString(cudaGetLastError()));
    }
}
int main()
{
    run<float, true>("float lower");
    run<float, false>("float upper");


}
