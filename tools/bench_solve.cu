// Standalone timing of one forward+backward sweep pair (k_solve.cu) with a per-block trace.
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include <cstdlib>
#include "../paper_0808_2794_b200/csrc/internal.h"
namespace mp {
thread_local int64_t g_launches = 0;
void func_smem_once(const void *fn, size_t bytes) { cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes); }
void func_cluster16_once(const void *fn) { cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); }
bool pdl_enabled() { return false; }

}
#include "../paper_0808_2794_b200/csrc/k_solve.cu"
using namespace mp;
int main(int argc, char **argv) {
  for (int n : {1024, 4096, 16384}) {
    const int64_t ldw = ((n + 63) / 64) * 64;
    std::vector<float> h((size_t)n * ldw, 0.f);
    std::mt19937 rng(1); std::uniform_real_distribution<float> ud(-1.f, 1.f);
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) h[(size_t)i * ldw + j] = (i == j) ? 2.f + ud(rng) * 0.5f : ud(rng) / n;
    std::vector<float> y(n); for (auto &v : y) v = ud(rng);
    float *W, *Y, *F; double *X; unsigned *fl;
    cudaMalloc(&W, h.size() * 4); cudaMalloc(&Y, n * 4); cudaMalloc(&F, n * 4); cudaMalloc(&X, n * 8);
    cudaMalloc(&fl, solve_flag_words(n) * 4); cudaMemset(fl, 0, solve_flag_words(n) * 4);
    cudaMemcpy(W, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    SolveScratch ss{fl, F, 0u};
    if (!getenv("NOTAGS")) {
      cudaMalloc(&ss.tags, solve_tag_words(n, 1) * 8); cudaMemset(ss.tags, 0, solve_tag_words(n, 1) * 8); ss.tag_cols = 1;
    }
    float *inv = nullptr;
    if (getenv("INV")) { cudaMalloc(&inv, solve_inv_floats(n) * 4); launch_solve_inverses(W, ldw, n, inv, 0); }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemcpy(Y, y.data(), n * 4, cudaMemcpyHostToDevice);
      cudaEventRecord(e0);
      launch_lu_solve<float>(W, ldw, n, 1, Y, X, 0, ss, 0, inv);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float t; cudaEventElapsedTime(&t, e0, e1); best = std::min(best, t);
    }
    printf("n=%d: forward+backward %.1f us (%s)\n", n, best * 1e3, cudaGetErrorString(cudaGetLastError()));
#ifdef MP_SOLVE_TRACE
    static unsigned long long tr[4096][12];
    cudaMemcpyFromSymbol(tr, g_strace, sizeof(tr));
    const int nblk = (n + 63) / 64;
    double acc[5] = {0};
    for (int t = 1; t < nblk; ++t) for (int k = 0; k < 3; ++k) acc[k] += (double)(tr[t][k + 1] - tr[t][k]);
    printf("  backward sweep, per block cycles: near %.0f, solve %.0f, end-bar %.0f; block-to-block %.0f\n",
           acc[0] / (nblk - 1), acc[1] / (nblk - 1), acc[2] / (nblk - 1),
           (double)(tr[nblk - 1][0] - tr[1][0]) / (nblk - 2));
    double sp = 0, prep_start_rel = 0; int cnt = 0;
    for (int t = 6; t < nblk; ++t) { sp += (double)(tr[t][5] - tr[t][4]); prep_start_rel += (double)((long long)tr[t][4] - (long long)tr[t - 1][1]); ++cnt; }
    double w6 = 0, w7 = 0, w8 = 0; int c6 = 0;
    for (int t = 6; t < nblk; ++t) { w6 += (double)(tr[t][6] - tr[t][1]); w7 += (double)(tr[t][7] - tr[t][6]); w8 += (double)(tr[t][2] - tr[t][7]); ++c6; }
    printf("  solve phase: diag-tile wait %.0f, diag_solve %.0f, stores %.0f\n", w6 / c6, w7 / c6, w8 / c6);
    if (inv) {
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, b9 = 0, b10 = 0, b11 = 0, b2 = 0; int c = 0;
      for (int t = 6; t < nblk - 1; ++t) {
        a0 += (double)(tr[t][2] - tr[t][0]);                  // chain GEMV + stores
        a5 += (double)(tr[t][1] - tr[t][0]);                  // chain: M tile wait
        a6 += (double)(tr[t][8] - tr[t][1]);                  // chain: GEMV
        b9 += (double)(tr[t][9] - tr[t][8]); b10 += (double)(tr[t][10] - tr[t][9]); b11 += (double)(tr[t][11] - tr[t][10]); b2 += (double)(tr[t][2] - tr[t][11]);
        a1 += (double)(tr[t][6] - tr[t][0]);                  // L: make_w(t+1) done
        a2 += (double)((long long)tr[t + 1][4] - (long long)tr[t][0]);   // prep(t+1) start
        a3 += (double)(tr[t + 1][5] - tr[t + 1][4]);           // prep(t+1) fflag spin
        a4 += (double)(tr[t][7] - tr[t][0]);                  // prep(t+1) done
        ++c;
      }
      printf("  INV: M-tile wait %.0f, GEMV %.0f, p0 %.0f, p1 %.0f, p2-3 %.0f, rest %.0f\n", a5 / c, a6 / c, b9 / c, b10 / c, b11 / c, b2 / c);
      printf("  INV: from block start: chain done %.0f, L done %.0f, prep start %.0f (spin %.0f), prep done %.0f\n",
             a0 / c, a1 / c, a2 / c, a3 / c, a4 / c);
    }
    printf("  prep: fflag spin %.0f cycles/block; prep start - previous block phase-A end %.0f\n", sp / cnt, prep_start_rel / cnt);
#endif
    cudaFree(W); if (inv) cudaFree(inv); cudaFree(Y); cudaFree(F); cudaFree(X); cudaFree(fl);
  }
  return 0;
}
