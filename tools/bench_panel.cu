// Standalone timing of the K2 leaf kernel: m x 32 leaf, per-column phase trace (clock64).
// nvcc -DMP_PANEL_TRACE ... tools/bench_panel.cu  (includes the library source directly)
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_0808_2794_b200/csrc/internal.h"
namespace mp {
thread_local int64_t g_launches = 0;
void func_smem_once(const void *fn, size_t bytes) { cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes); }
void func_cluster16_once(const void *fn) { cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); }
bool pdl_enabled() { return false; }
}
#include "../paper_0808_2794_b200/csrc/k_panel.cu"
using namespace mp;
int main(int argc, char **argv) {
  for (int m : {512, 1024, 2048, 4096, 6144, 8192, 12288, 16384}) {
    const int n = m, ldw = ((n + 63) / 64) * 64, w = panel_leaf_width<float>(m);
    std::vector<float> h((size_t)n * ldw);  // (pairs buffer below: 2w pairs)
    std::mt19937 rng(1); std::normal_distribution<float> nd;
    for (auto &v : h) v = nd(rng);
    float *W; int32_t *ipiv, *orig, *pairs, *np; DevStatus *st;
    cudaMalloc(&W, h.size() * 4); cudaMalloc(&ipiv, n * 4); cudaMalloc(&orig, n * 4); cudaMalloc(&pairs, 4 * 128 * 4);
    cudaMalloc(&np, 4); cudaMalloc(&st, sizeof(DevStatus)); cudaMemset(st, 0, sizeof(DevStatus));
    std::vector<int> o(n); for (int i = 0; i < n; ++i) o[i] = i; cudaMemcpy(orig, o.data(), n * 4, cudaMemcpyHostToDevice);
    PanelScratch ps{orig, pairs, np, nullptr, nullptr, nullptr};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemcpy(W, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
      cudaEventRecord(e0);
      launch_panel_leaf<float>(W, ldw, n, 0, w, ipiv, ps, st, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float t; cudaEventElapsedTime(&t, e0, e1); if (t < best) best = t;
    }
    cudaError_t e = cudaGetLastError();
    long long tr[64][8] = {};
#ifdef MP_PANEL_TRACE
    cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr));
#endif
    printf("m=%d leaf w=%d: %.1f us (%s)  per-column cycles [argmax, push, wait, reduce, update]:\n", m, w, best * 1e3, cudaGetErrorString(e));
    double acc[5] = {0};
    for (int c = 1; c < 31; ++c) {
      acc[0] += tr[c][1] - tr[c][0]; acc[1] += tr[c][2] - tr[c][1]; acc[2] += tr[c][3] - tr[c][2]; acc[3] += tr[c][4] - tr[c][3]; acc[4] += tr[c + 1][0] - tr[c][4];
    }
    printf("   avg %.0f %.0f %.0f %.0f %.0f  total/col %.0f\n", acc[0] / 30, acc[1] / 30, acc[2] / 30, acc[3] / 30, acc[4] / 30, (acc[0] + acc[1] + acc[2] + acc[3] + acc[4]) / 30);
    cudaFree(W); cudaFree(ipiv); cudaFree(orig); cudaFree(pairs); cudaFree(np); cudaFree(st);
  }
  return 0;
}
