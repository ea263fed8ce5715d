// Probe: events between a primary-context stream and two green-context streams, a kernel
// with 100 KB of dynamic shared memory (attribute set through the runtime) on a green
// stream, memory from cudaMallocAsync used on green streams, and true concurrency.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("ERR %s: %s (line %d)\n", #x, s, __LINE__); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("RT ERR %s: %s (line %d)\n", #x, cudaGetErrorString(r), __LINE__); return 1; } } while (0)
__device__ unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ unsigned smid() { unsigned s; asm volatile("mov.u32 %0, %smid;" : "=r"(s)); return s; }
__global__ void big_smem_kernel(float *out, unsigned long long ns, unsigned *sms, unsigned long long *tt) {
  extern __shared__ float sm[];
  unsigned long long t0 = gtime();
  sm[threadIdx.x] = threadIdx.x; __syncthreads();
  while (gtime() - t0 < ns) {}
  if (threadIdx.x == 0) { out[blockIdx.x] = sm[5] + 1.f; sms[blockIdx.x] = smid(); tt[2*blockIdx.x] = t0; tt[2*blockIdx.x+1] = gtime(); }
}
__global__ void add_kernel(float *x, int n, float v) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) x[i] += v; }
int main() {
  CK(cuInit(0)); CUdevice dev; CK(cuDeviceGet(&dev, 0)); RK(cudaSetDevice(0)); RK(cudaFree(0));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  CUdevResource grp[1], rest; unsigned ng = 1;
  CK(cuDevSmResourceSplitByCount(grp, &ng, &all, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, 16));
  CUdevResourceDesc d1, d2; CK(cuDevResourceGenerateDesc(&d1, grp, 1)); CK(cuDevResourceGenerateDesc(&d2, &rest, 1));
  CUgreenCtx gP, gU; CK(cuGreenCtxCreate(&gP, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM)); CK(cuGreenCtxCreate(&gU, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sP, sU; CK(cuGreenCtxStreamCreate(&sP, gP, CU_STREAM_NON_BLOCKING, 0)); CK(cuGreenCtxStreamCreate(&sU, gU, CU_STREAM_NON_BLOCKING, 0));
  printf("partitions: P=%u SMs, U=%u SMs\n", grp[0].sm.smCount, rest.sm.smCount);
  cudaStream_t s0; RK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  float *x; RK(cudaMallocAsync((void**)&x, 1024 * 4, s0)); RK(cudaMemsetAsync(x, 0, 1024 * 4, s0));
  cudaEvent_t e0, eP, eU; RK(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming)); RK(cudaEventCreateWithFlags(&eP, cudaEventDisableTiming)); RK(cudaEventCreateWithFlags(&eU, cudaEventDisableTiming));
  RK(cudaEventRecord(e0, s0));
  RK(cudaStreamWaitEvent((cudaStream_t)sP, e0, 0)); RK(cudaStreamWaitEvent((cudaStream_t)sU, e0, 0));
  add_kernel<<<4, 256, 0, (cudaStream_t)sP>>>(x, 1024, 1.f); RK(cudaGetLastError());
  RK(cudaEventRecord(eP, (cudaStream_t)sP));
  RK(cudaStreamWaitEvent((cudaStream_t)sU, eP, 0));
  add_kernel<<<4, 256, 0, (cudaStream_t)sU>>>(x, 1024, 10.f); RK(cudaGetLastError());
  RK(cudaEventRecord(eU, (cudaStream_t)sU));
  RK(cudaStreamWaitEvent(s0, eU, 0));
  add_kernel<<<4, 256, 0, s0>>>(x, 1024, 100.f);
  float h[4]; RK(cudaMemcpyAsync(h, x, 16, cudaMemcpyDeviceToHost, s0)); RK(cudaStreamSynchronize(s0));
  printf("event chain primary->P->U->primary: x = %.0f (expect 111)\n", h[0]);
  // big smem kernels on both partitions concurrently
  RK(cudaFuncSetAttribute(big_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  float *o; unsigned *sms; unsigned long long *tt;
  RK(cudaMalloc(&o, 4096 * 4)); RK(cudaMalloc(&sms, 4096 * 4)); RK(cudaMalloc(&tt, 8192 * 8));
  big_smem_kernel<<<rest.sm.smCount, 256, 100 * 1024, (cudaStream_t)sU>>>(o, 3000000ull, sms, tt); RK(cudaGetLastError());
  big_smem_kernel<<<16, 256, 100 * 1024, (cudaStream_t)sP>>>(o + 2048, 1000000ull, sms + 2048, tt + 4096); RK(cudaGetLastError());
  RK(cudaDeviceSynchronize());
  unsigned hs[4096]; unsigned long long ht[8192];
  RK(cudaMemcpy(hs, sms, sizeof(hs), cudaMemcpyDeviceToHost)); RK(cudaMemcpy(ht, tt, sizeof(ht), cudaMemcpyDeviceToHost));
  unsigned long long u0 = ~0ull, u1 = 0, p0 = ~0ull, p1 = 0;
  for (unsigned i = 0; i < rest.sm.smCount; ++i) { if (ht[2*i] < u0) u0 = ht[2*i]; if (ht[2*i+1] > u1) u1 = ht[2*i+1]; }
  for (int i = 0; i < 16; ++i) { if (ht[4096+2*i] < p0) p0 = ht[4096+2*i]; if (ht[4096+2*i+1] > p1) p1 = ht[4096+2*i+1]; }
  printf("U kernel [0, %llu] us, P kernel [%lld, %lld] us (overlap if P starts before U ends)\n", (u1-u0)/1000, (long long)(p0-u0)/1000, (long long)(p1-u0)/1000);
  int overlapSM = 0; for (int i = 0; i < 16; ++i) for (unsigned j = 0; j < rest.sm.smCount; ++j) if (hs[2048+i] == hs[j]) overlapSM++;
  printf("P kernel SMs shared with U kernel: %d\n", overlapSM);
  // occupancy query on a green stream's context
  int nb = 0; RK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, big_smem_kernel, 256, 100 * 1024));
  printf("occupancy (primary): %d blocks/SM\n", nb);
  return 0;
}
