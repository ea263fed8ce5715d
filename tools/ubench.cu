// Latency microbenchmarks of the primitives on the leaf's per-column chain (clock64 deltas).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ long long out[64];
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __cluster_dims__(1, 1, 1) lat_kernel(int iters, unsigned seed) {
  __shared__ unsigned buf[1024];
  __shared__ __align__(8) unsigned long long bar[2];
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned v = seed + tid;
  long long t0, t1;
  // 1. redux.sync max chain
  __syncthreads(); t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __reduce_max_sync(0xffffffffu, v ^ i) + lane;
  t1 = clock64(); if (tid == 0) out[0] = (t1 - t0) / iters;
  // 2. shfl chain
  __syncthreads(); t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + i;
  t1 = clock64(); if (tid == 0) out[1] = (t1 - t0) / iters;
  // 3. LDS dependent chain
  for (int i = tid; i < 1024; i += blockDim.x) buf[i] = (i * 7 + 1) & 1023;
  __syncthreads(); unsigned idx = v & 1023; t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = buf[idx];
  t1 = clock64(); if (tid == 0) out[2] = (t1 - t0) / iters; v += idx;
  // 4. __syncthreads round (all warps)
  __syncthreads(); t0 = clock64();
  for (int i = 0; i < iters; ++i) { __syncthreads(); }
  t1 = clock64(); if (tid == 0) out[3] = (t1 - t0) / iters;
  // 5. STS -> bar -> LDS by another warp (ping)
  __syncthreads(); t0 = clock64();
  for (int i = 0; i < iters; ++i) { if (tid == 32) buf[i & 1023] = v + i; __syncthreads(); v += buf[i & 1023]; }
  t1 = clock64(); if (tid == 0) out[4] = (t1 - t0) / iters;
  // 6. MUFU.RCP + IEEE rcp chain
  float f = 1.0f + v * 1e-9f; __syncthreads(); t0 = clock64();
  for (int i = 0; i < iters; ++i) f = __frcp_rn(f) + 1.0f;
  t1 = clock64(); if (tid == 0) out[5] = (t1 - t0) / iters;
  // 7. FFMA dependent chain
  __syncthreads(); t0 = clock64();
  for (int i = 0; i < iters; ++i) f = fmaf(f, 0.999f, 0.001f);
  t1 = clock64(); if (tid == 0) out[6] = (t1 - t0) / iters;
  // 8. IEEE division chain
  __syncthreads(); t0 = clock64();
  for (int i = 0; i < iters; ++i) f = __fdiv_rn(1.5f, f) + 0.5f;
  t1 = clock64(); if (tid == 0) out[7] = (t1 - t0) / iters;
  // 9. local st.async + mbarrier round trip (one thread)
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[0]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (tid == 0) {
    unsigned rb, ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rb) : "r"(smem_u32(&bar[0])));
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ra) : "r"(smem_u32(&buf[0])));
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" :: "r"(smem_u32(&bar[0])) : "memory");
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %1, %1, %1}, [%2];" :: "r"(ra), "r"(v), "r"(rb) : "memory");
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(smem_u32(&bar[0])), "r"(i & 1) : "memory");
    }
    t1 = clock64(); out[8] = (t1 - t0) / iters;
    // 10. same with acquire.cta
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" :: "r"(smem_u32(&bar[0])) : "memory");
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %1, %1, %1}, [%2];" :: "r"(ra), "r"(v), "r"(rb) : "memory");
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(smem_u32(&bar[0])), "r"((i + iters) & 1) : "memory");
    }
    t1 = clock64(); out[9] = (t1 - t0) / iters;
  }
  // 11. named barrier arrive/sync pair between warp 0 and others
  __syncthreads(); t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (tid < 32) asm volatile("bar.sync 1, %0;" :: "r"((int)blockDim.x) : "memory");
    else asm volatile("bar.arrive 1, %0;" :: "r"((int)blockDim.x) : "memory");
    asm volatile("bar.sync 2, %0;" :: "r"((int)blockDim.x) : "memory");
  }
  t1 = clock64(); if (tid == 0) out[10] = (t1 - t0) / iters;
  if (v == 12345 && f == 0.f) out[63] = v;
}

// DSMEM ping-pong between CTA 0 and CTA 1 of a cluster of 2 via st.async + mbarrier
__global__ void __cluster_dims__(2, 1, 1) pingpong_kernel(int iters) {
  __shared__ __align__(16) unsigned buf[4];
  __shared__ __align__(8) unsigned long long bar;
  cg::cluster_group cl = cg::this_cluster();
  const int r = cl.block_rank();
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  cl.sync();
  if (threadIdx.x == 0) {
    unsigned rb, ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(&bar)), "r"(1 - r));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&buf[0])), "r"(1 - r));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" :: "r"(smem_u32(&bar)) : "memory");
      if (r == 0 || i > 0) {}
      if (r == 0) {
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %1, %1, %1}, [%2];" :: "r"(ra), "r"(i), "r"(rb) : "memory");
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(smem_u32(&bar)), "r"(i & 1) : "memory");
      } else {
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(smem_u32(&bar)), "r"(i & 1) : "memory");
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %1, %1, %1}, [%2];" :: "r"(ra), "r"(i), "r"(rb) : "memory");
      }
    }
    long long t1 = clock64();
    if (r == 0) out[11] = (t1 - t0) / iters;   // one round trip = two one-way hops
  }
  cl.sync();
}

int main() {
  const char *names[] = {"redux.max chain", "shfl chain", "LDS dep chain", "__syncthreads x128thr", "STS-bar-LDS", "frcp_rn chain", "FFMA chain", "fdiv_rn chain", "st.async+mbar local (acq.cluster)", "st.async+mbar local (acq.cta)", "bar.arrive/sync pair", "DSMEM st.async ping-pong RTT"};
  for (int nt : {128, 512}) {
    lat_kernel<<<1, nt>>>(1000, 1);
    pingpong_kernel<<<2, 32>>>(1000);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[64]; cudaMemcpyFromSymbol(h, out, sizeof(h));
    printf("threads=%d (%s)\n", nt, cudaGetErrorString(e));
    for (int i = 0; i < 12; ++i) printf("  %-36s %lld cycles\n", names[i], h[i]);
  }
  return 0;
}
