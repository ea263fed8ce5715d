// probe: can a 16-CTA cluster kernel on a 16-SM green context run concurrently with a
// persistent kernel on the remaining SMs?  Prints SM ids and overlap.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("ERR %s: %s (line %d)\n", #x, s, __LINE__); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("RT ERR %s: %s (line %d)\n", #x, cudaGetErrorString(r), __LINE__); return 1; } } while (0)

__device__ unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ unsigned smid() { unsigned s; asm volatile("mov.u32 %0, %smid;" : "=r"(s)); return s; }

__global__ void spin_kernel(unsigned long long ns, unsigned *sm, unsigned long long *t) {
  unsigned long long t0 = gtime();
  while (gtime() - t0 < ns) {}
  if (threadIdx.x == 0) { sm[blockIdx.x] = smid(); t[2*blockIdx.x] = t0; t[2*blockIdx.x+1] = gtime(); }
}
__global__ void cluster_kernel(unsigned long long ns, unsigned *sm, unsigned long long *t) {
  cg::cluster_group cl = cg::this_cluster();
  unsigned long long t0 = gtime();
  for (int i = 0; i < 1000; ++i) cl.sync();
  unsigned long long t1 = gtime();
  while (gtime() - t0 < ns) {}
  if (threadIdx.x == 0) { sm[blockIdx.x] = smid(); t[2*blockIdx.x] = t0; t[2*blockIdx.x+1] = gtime(); t[64 + blockIdx.x] = (t1 - t0); }
}

int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  RK(cudaSetDevice(0)); RK(cudaFree(0));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", all.sm.smCount);
  for (unsigned flags : {0u, 2u}) {
    CUdevResource grp[1], rest; unsigned ng = 1;
    CUresult r = cuDevSmResourceSplitByCount(grp, &ng, &all, &rest, flags, 16);
    printf("split flags=%u -> r=%d ng=%u grp=%u rest=%u\n", flags, (int)r, ng, grp[0].sm.smCount, rest.sm.smCount);
  }
  CUdevResource grp[1], rest; unsigned ng = 1;
  CK(cuDevSmResourceSplitByCount(grp, &ng, &all, &rest, 2, 16));
  CUdevResourceDesc d1, d2; CK(cuDevResourceGenerateDesc(&d1, grp, 1)); CK(cuDevResourceGenerateDesc(&d2, &rest, 1));
  CUgreenCtx g1, g2; CK(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM)); CK(cuGreenCtxCreate(&g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s1, s2; CK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0)); CK(cuGreenCtxStreamCreate(&s2, g2, CU_STREAM_NON_BLOCKING, 0));
  unsigned *sm; unsigned long long *t; RK(cudaMalloc(&sm, 4096 * 4)); RK(cudaMalloc(&t, 8192 * 8));
  RK(cudaFuncSetAttribute(cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int ncl = 0;
  for (int csz : {16, 8}) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(csz); cfg.blockDim = dim3(512); cfg.stream = (cudaStream_t)s1;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, cluster_kernel, &cfg);
    printf("occupancy (current ctx) cluster %d: %d (%s)\n", csz, ncl, cudaGetErrorString(e));
  }
  // persistent spin on rest, then cluster kernel on grp
  int nrest = rest.sm.smCount;
  spin_kernel<<<nrest, 256, 0, (cudaStream_t)s2>>>(2000000ull, sm, t);
  RK(cudaGetLastError());
  {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(16); cfg.blockDim = dim3(512); cfg.stream = (cudaStream_t)s1;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, cluster_kernel, 1000000ull, sm + 2048, t + 4096);
    printf("cluster launch: %s\n", cudaGetErrorString(e));
  }
  RK(cudaDeviceSynchronize());
  std::vector<unsigned> hs(4096); std::vector<unsigned long long> ht(8192);
  RK(cudaMemcpy(hs.data(), sm, 4096 * 4, cudaMemcpyDeviceToHost)); RK(cudaMemcpy(ht.data(), t, 8192 * 8, cudaMemcpyDeviceToHost));
  unsigned long long smin = ~0ull, smax = 0, cmin = ~0ull, cmax = 0;
  for (int i = 0; i < nrest; ++i) { smin = std::min(smin, ht[2*i]); smax = std::max(smax, ht[2*i+1]); }
  printf("cluster SMs:"); for (int i = 0; i < 16; ++i) { printf(" %u", hs[2048+i]); cmin = std::min(cmin, ht[4096+2*i]); cmax = std::max(cmax, ht[4096+2*i+1]); } printf("\n");
  printf("rest SMs sample:"); for (int i = 0; i < 16; ++i) printf(" %u", hs[i]); printf("\n");
  printf("spin [%llu, %llu] us, cluster [%llu, %llu] us (relative to spin start)\n", 0ull, (smax - smin)/1000, (cmin - smin)/1000, (cmax - smin)/1000);
  printf("cluster.sync x1000: %.3f us per sync\n", ht[4096+64] / 1000.0 / 1000.0);
  return 0;
}
