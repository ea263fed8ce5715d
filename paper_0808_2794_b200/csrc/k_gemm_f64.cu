// k_gemm_f64.cu — the binary64 trailing (Schur complement) update C <- C - A B of the FP64 path
// (mp_dgesv, the binary64 fallback, B:5's speedup denominator) on the FP64 tensor pipe.
//
// PAPER.md T3 compares the mixed solve against "a full double precision solve (reference time)"
// (P:393-394); B:5 asks for that denominator built the same way as the mixed path.  Its O(n^3)
// step is DGETRF's trailing update (P:365-368 in binary64), so it gets the same care as K5:
//
//  * sm_100a runs binary64 matrix products as DMMA (mma.sync m8n8k4 f64: 256 FMAs per warp
//    instruction, tools/ubench_fp64.cu measures it against the DFMA pipe);
//  * CTA tile 128 x 128, k-slices of 16 staged by cp.async (16-byte, L2-only .cg) through a
//    3-stage ring; 8 warps in a 2 x 4 grid, warp tile 64 x 32 = 8 x 4 mma tiles, the 64
//    accumulators of a lane live in registers for the whole K loop;
//  * shared tiles are padded (A rows 16 + 4 doubles, B rows 128 + 4 doubles) so the fragment
//    loads (A: lane -> row lane/4, k lane%4; B: k lane%4, column lane/4) hit distinct banks;
//  * epilogue: each lane owns two adjacent columns of 8 rows per mma tile: C is read and
//    written once with 16-byte accesses.
// Operands are the row-major views into the binary64 working copy (as K5a): A = L21 (K
// contiguous), B = U12 (N contiguous), C = A22.  Algorithmic work 2 M N K flops.
#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace mp {

namespace {

constexpr int BM = 128, BK = 16, STAGES = 3;
constexpr int APAD = BK + 4;
constexpr int A_ELEMS = BM * APAD;
template <int BN> struct TileCfg {
    static constexpr int NT = 2 * BN;                   // warps: 2 along M x BN/32 along N
    static constexpr int BPAD = BN + 4;
    static constexpr int B_ELEMS = BK * BPAD;
    static constexpr size_t SMEM = (size_t)STAGES * (A_ELEMS + B_ELEMS) * sizeof(double);
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 16 : 0;                       // src-size 0: zero-fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// A: M x K (lda), B: K x N (ldb), C: M x N (ldc), all row-major; every row start and ld is a
// multiple of 2 doubles (16 bytes), checked by the host.
template <int BN, int MINB>
__global__ void __launch_bounds__(TileCfg<BN>::NT, MINB)
dgemm_dmma_kernel(const double *__restrict__ A, int64_t lda, const double *__restrict__ B, int64_t ldb,
                  double *__restrict__ C, int64_t ldc, int M, int N, int K, int lower)
{
    constexpr int NT = TileCfg<BN>::NT, BPAD = TileCfg<BN>::BPAD, B_ELEMS = TileCfg<BN>::B_ELEMS;
    constexpr int WN = BN / 32;                          // warps along N
    extern __shared__ __align__(16) double smem[];
    double *As = smem;                                   // [STAGES][BM][APAD]
    double *Bs = smem + STAGES * A_ELEMS;                // [STAGES][BK][BPAD]
    pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    if (lower && m0 + BM - 1 < n0) return;               // SPD SYRK: tile entirely above the diagonal
    const int wm = (warp / WN) * 64, wn = (warp % WN) * 32;
    const int nk = (K + BK - 1) / BK;
    // pull this tile of C into L2 now, so the epilogue's read-modify-write does not wait on HBM
    // while the SM's tensor pipe idles (one 128-byte line per row segment)
    for (int i = tid; i < BM * (BN / 16); i += NT) {
        const int r = m0 + i / (BN / 16), c = n0 + (i % (BN / 16)) * 16;
        if (r < M && c < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(C + (int64_t)r * ldc + c));
    }

    // loader: A slice 128 x 16 doubles = 1024 chunks of 2; B slice 16 x BN = 8 BN chunks
    auto load = [&](int kt, int st) {
        const int k0 = kt * BK;
        double *as = As + st * A_ELEMS, *bs = Bs + st * B_ELEMS;
#pragma unroll
        for (int i = 0; i < 1024 / NT; ++i) {
            const int c = tid + NT * i;
            const int r = c >> 3, kc = (c & 7) * 2;      // A: row r, k pair kc
            const int gr = m0 + r, gk = k0 + kc;
            const bool ok = gr < M && gk < K;            // K even (host check): a pair is all-in or all-out
            cp_async16(as + r * APAD + kc, ok ? A + (int64_t)gr * lda + gk : A, ok);
        }
#pragma unroll
        for (int i = 0; i < 8 * BN / NT; ++i) {
            const int c = tid + NT * i;
            const int kr = c / (BN / 2), nc = (c % (BN / 2)) * 2;   // B: k row kr, column pair nc
            const int gk2 = k0 + kr, gn = n0 + nc;
            const bool ok2 = gk2 < K && gn < N;          // N even (host check)
            cp_async16(bs + kr * BPAD + nc, ok2 ? B + (int64_t)gk2 * ldb + gn : B, ok2);
        }
    };

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load(s, s);
        cp_async_commit();
    }
    const int ar = lane >> 2, ak = lane & 3;             // A fragment: row, k
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();                                 // slice kt visible; slice kt-1's stage free
        if (kt + STAGES - 1 < nk) load(kt + STAGES - 1, (kt + STAGES - 1) % STAGES);
        cp_async_commit();
        const double *as = As + (kt % STAGES) * A_ELEMS + (wm + ar) * APAD + ak;
        const double *bs = Bs + (kt % STAGES) * B_ELEMS + ak * BPAD + wn + ar;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[8], b[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = as[i * 8 * APAD + kk];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = bs[kk * BPAD + j * 8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
        }
    }
    cp_async_wait<0>();

    // epilogue: lane holds C[row = lane/4][col = 2 (lane%4) + {0,1}] of every 8 x 8 tile
    const int cr = lane >> 2, cc = (lane & 3) * 2;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + wm + i * 8 + cr;
        if (row >= M) continue;
        double *crow = C + (int64_t)row * ldc;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = n0 + wn + j * 8 + cc;
            if (col < N) {                               // N even: the pair is all-in
                double2 v = *reinterpret_cast<double2 *>(crow + col);
                v.x -= acc[i][j][0];
                v.y -= acc[i][j][1];
                *reinterpret_cast<double2 *>(crow + col) = v;
            }
        }
    }
}

}  // namespace

bool launch_dgemm_dmma(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc,
                       int64_t M, int64_t N, int64_t K, cudaStream_t s, bool lower)
{
    auto al = [](const void *p, int64_t ld) { return ((uintptr_t)p % 16 == 0) && (ld % 2 == 0); };
    if (M <= 0 || N <= 0 || K <= 0) return true;
    if (!al(A, lda) || !al(B, ldb) || !al(C, ldc) || (N & 1) || (K & 1) || M > INT32_MAX / 2 || N > INT32_MAX / 2)
        return false;
    // 128 x 64 tiles, 4 warps, 2 CTAs per SM (one CTA's epilogue overlaps the other's MMAs) by
    // default; MP_DMMA_BN=128: 128 x 128 tiles, 8 warps, 1 CTA per SM
    static const int bn = [] { const char *e = std::getenv("MP_DMMA_BN"); return e ? std::atoi(e) : 64; }();
    if (bn == 128) {
        auto kern = dgemm_dmma_kernel<128, 1>;
        func_smem_once((const void *)kern, TileCfg<128>::SMEM);
        launch_ex(kern, dim3((unsigned)ceil_div(N, 128), (unsigned)ceil_div(M, BM)), dim3(TileCfg<128>::NT),
                  TileCfg<128>::SMEM, s, nullptr, A, lda, B, ldb, C, ldc, (int)M, (int)N, (int)K, (int)lower);
    } else {
        auto kern = dgemm_dmma_kernel<64, 2>;
        func_smem_once((const void *)kern, TileCfg<64>::SMEM);
        launch_ex(kern, dim3((unsigned)ceil_div(N, 64), (unsigned)ceil_div(M, BM)), dim3(TileCfg<64>::NT),
                  TileCfg<64>::SMEM, s, nullptr, A, lda, B, ldb, C, ldc, (int)M, (int)N, (int)K, (int)lower);
    }
    return true;
}

}  // namespace mp
