// Micro-benchmark: cycles of one diag_solve (k_solve.cu) call by one warp, tile resident in smem.
#include <cstdio>
#include "../paper_0808_2794_b200/csrc/internal.h"
namespace mp {
thread_local int64_t g_launches = 0;
void func_smem_once(const void *fn, size_t bytes) { cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes); }
void func_cluster16_once(const void *fn) { cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); }
}
#include "../paper_0808_2794_b200/csrc/k_solve.cu"
using namespace mp;
template <typename T, bool LOWER>
__global__ void kdiag(const T *g, T *out, long long *cyc, int iters, int mode, unsigned *gflag)
{
    __shared__ __align__(1024) T dg[BS * BS];
    __shared__ T rinv[BS];
    __shared__ __align__(8) uint64_t bar;
    __shared__ volatile int done;
    for (int i = threadIdx.x; i < BS * BS; i += blockDim.x) dg[i] = g[i];
    if (threadIdx.x == 0) { mbar_init(&bar, 1); done = 0; }
    __syncthreads();
    if (threadIdx.x >= 32) {
        if (threadIdx.x == 32) {
            if (mode == 1) mbar_wait(&bar, 0);
            if (mode == 2) while (ld_relaxed_u32(gflag) == 0 && !done) {}
            if (mode == 3) while (!done) {}
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
    if (lane == 0) *cyc = (t1 - t0) / iters;
}
template <typename T, bool LOWER>
void run(const char *name)
{
    T h[BS * BS];
    for (int i = 0; i < BS * BS; ++i) h[i] = T(1) + T(i % 7) * T(0.01);
    T *g, *o; long long *c;
    cudaMalloc(&g, sizeof(h)); cudaMalloc(&o, 64 * sizeof(T)); cudaMalloc(&c, 8);
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
    unsigned *fl; cudaMalloc(&fl, 4); cudaMemset(fl, 0, 4);
    for (int mode = 0; mode < 4; ++mode) {
        kdiag<T, LOWER><<<1, 64>>>(g, o, c, 1000, mode, fl);
        long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("%s mode %d: %lld cycles / diag_solve (%s)\n", name, mode, cy, cudaGetErrorString(cudaGetLastError()));
    }
}
int main()
{
    run<float, true>("float lower");
    run<float, false>("float upper");
    run<double, true>("double lower");
    run<double, false>("double upper");
}
