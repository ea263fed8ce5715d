// k_gemm.cu — K5a: trailing (Schur complement) update  A22 <- A22 - L21 * U12.
//
// "the only operation with computational complexity of
// O(n^3) is handled in single precision"; SGETRF's trailing update
// (P:366).  This is the FFMA variant (binary32 CUDA-core FMAs; the binary64
// instantiation is the DGEMM of the mp_dgesv path and of the fallback).
//
// All three operands are row-major views into the working copy W (stride
// ldw): L21 rows are K-contiguous, U12 rows are N-contiguous, so both tiles
// are read with 128-bit unit-stride loads.  Classic register-blocked SGEMM:
// BM x BN block tile, BK-deep k-slices double-buffered in shared memory
// (register-staged prefetch of slice t+1 while slice t is consumed), TM x TN
// micro-tile per thread split in two halves to keep LDS.128 conflict-free.
// Algorithmic work 2*M*N*K flops; C is read and written once (8 M N bytes).
#include <algorithm>

#include <cstdlib>

#include "internal.h"

namespace mp {

namespace {

template <typename T, int N> struct Vec;
template <> struct Vec<float, 4> { using type = float4; };
template <> struct Vec<float, 2> { using type = float2; };
template <> struct Vec<double, 2> { using type = double2; };
template <> struct Vec<double, 4> { using type = double4; };

template <typename T, int BM, int BN, int BK, int TM, int TN>
struct Cfg {
    static constexpr int NT = (BM / TM) * (BN / TN);
    static constexpr int A_PER = BM * BK / NT;       // elements of the A slice per thread (along k)
    static constexpr int B_PER = BK * BN / NT;       // elements of the B slice per thread (along n)
    static constexpr int A_TPR = BK / A_PER;         // threads per A row
    static constexpr int B_TPR = BN / B_PER;         // threads per B row
    static_assert(BK % A_PER == 0 && BN % B_PER == 0, "tile split");
};

template <typename T, int BM, int BN, int BK, int TM, int TN, bool VEC>
__global__ void __launch_bounds__(Cfg<T, BM, BN, BK, TM, TN>::NT, 2)
gemm_update_kernel(const T *__restrict__ A, int64_t lda, const T *__restrict__ B, int64_t ldb, T *__restrict__ C,
                   int64_t ldc, int64_t M, int64_t N, int64_t K)
{
    using Cf = Cfg<T, BM, BN, BK, TM, TN>;
    constexpr int NT = Cf::NT;
    __shared__ __align__(16) T As[2][BK][BM];
    __shared__ __align__(16) T Bs[2][BK][BN];
    pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x;
    const int64_t bm0 = (int64_t)blockIdx.y * BM, bn0 = (int64_t)blockIdx.x * BN;
    const T *Ag = A + bm0 * lda;                      // L21 block rows
    const T *Bg = B + bn0;                            // U12 block columns
    T *Cg = C + bm0 * ldc + bn0;

    // loader coordinates
    const int a_row = tid / Cf::A_TPR, a_k = (tid % Cf::A_TPR) * Cf::A_PER;
    const int b_k = tid / Cf::B_TPR, b_n = (tid % Cf::B_TPR) * Cf::B_PER;
    T ra[Cf::A_PER], rb[Cf::B_PER];

    auto load_slice = [&](int64_t kk) {
        const bool arow_ok = bm0 + a_row < M;
        if (VEC && arow_ok && kk + a_k + Cf::A_PER <= K) {
            using V = typename Vec<T, Cf::A_PER>::type;
            V v = *reinterpret_cast<const V *>(Ag + a_row * lda + kk + a_k);
            const T *pv = reinterpret_cast<const T *>(&v);
#pragma unroll
            for (int e = 0; e < Cf::A_PER; ++e) ra[e] = pv[e];
        } else {
#pragma unroll
            for (int e = 0; e < Cf::A_PER; ++e)
                ra[e] = (arow_ok && kk + a_k + e < K) ? Ag[a_row * lda + kk + a_k + e] : T(0);
        }
        const bool bk_ok = kk + b_k < K;
        if (VEC && bk_ok && bn0 + b_n + Cf::B_PER <= N) {
            using V = typename Vec<T, Cf::B_PER>::type;
            V v = *reinterpret_cast<const V *>(Bg + (kk + b_k) * ldb + b_n);
            const T *pv = reinterpret_cast<const T *>(&v);
#pragma unroll
            for (int e = 0; e < Cf::B_PER; ++e) rb[e] = pv[e];
        } else {
#pragma unroll
            for (int e = 0; e < Cf::B_PER; ++e)
                rb[e] = (bk_ok && bn0 + b_n + e < N) ? Bg[(kk + b_k) * ldb + b_n + e] : T(0);
        }
    };
    auto store_slice = [&](int buf) {
#pragma unroll
        for (int e = 0; e < Cf::A_PER; ++e) As[buf][a_k + e][a_row] = ra[e];
#pragma unroll
        for (int e = 0; e < Cf::B_PER; ++e) Bs[buf][b_k][b_n + e] = rb[e];
    };

    constexpr int TX = BN / TN;                       // threads along n
    const int ty = tid / TX, tx = tid % TX;
    constexpr int HM = TM / 2, HN = TN / 2;
    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

    const int nslices = (int)ceil_div(K, BK);
    load_slice(0);
    store_slice(0);
    __syncthreads();
    for (int t = 0; t < nslices; ++t) {
        const int buf = t & 1;
        if (t + 1 < nslices) load_slice((int64_t)(t + 1) * BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            T a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < HM; ++i) {
                a[i] = As[buf][kk][ty * HM + i];
                a[HM + i] = As[buf][kk][BM / 2 + ty * HM + i];
            }
#pragma unroll
            for (int j = 0; j < HN; ++j) {
                b[j] = Bs[buf][kk][tx * HN + j];
                b[HN + j] = Bs[buf][kk][BN / 2 + tx * HN + j];
            }
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        if (t + 1 < nslices) {
            store_slice(buf ^ 1);
            __syncthreads();
        }
    }

    // epilogue: C <- C - acc
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int row = (i < HM) ? ty * HM + i : BM / 2 + ty * HM + (i - HM);
        if (bm0 + row >= M) continue;
        T *crow = Cg + (int64_t)row * ldc;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int col = (h == 0) ? tx * HN : BN / 2 + tx * HN;
            if (VEC && bn0 + col + HN <= N) {
                using V = typename Vec<T, HN>::type;
                V v = *reinterpret_cast<V *>(crow + col);
                T *pv = reinterpret_cast<T *>(&v);
#pragma unroll
                for (int j = 0; j < HN; ++j) pv[j] -= acc[i][h * HN + j];
                *reinterpret_cast<V *>(crow + col) = v;
            } else {
#pragma unroll
                for (int j = 0; j < HN; ++j)
                    if (bn0 + col + j < N) crow[col + j] -= acc[i][h * HN + j];
            }
        }
    }
}

template <typename T, int BM, int BN, int BK, int TM, int TN>
void launch_tiles(const T *A, int64_t lda, const T *B, int64_t ldb, T *C, int64_t ldc, int64_t M, int64_t N,
                  int64_t K, cudaStream_t s)
{
    using Cf = Cfg<T, BM, BN, BK, TM, TN>;
    dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM));
    auto al = [](const void *p, int64_t ld) { return ((uintptr_t)p % 32 == 0) && (ld % 8 == 0); };
    const bool vec = al(A, lda) && al(B, ldb) && al(C, ldc);
    if (vec)
        launch_ex(gemm_update_kernel<T, BM, BN, BK, TM, TN, true>, grid, dim3(Cf::NT), 0, s, nullptr, A, lda, B, ldb, C,
                  ldc, M, N, K);
    else
        launch_ex(gemm_update_kernel<T, BM, BN, BK, TM, TN, false>, grid, dim3(Cf::NT), 0, s, nullptr, A, lda, B, ldb,
                  C, ldc, M, N, K);
}

// ---------------------------------------------------------------- tall-skinny variant
// In-panel Schur updates of the recursive panel (N, K <= 128, M up to n): one CTA per
// BM-row slab; the whole K x N block B = U12 and the CTA's BM x K slab of L21 are staged
// in shared memory once (B is shared by every CTA and L2-resident), then a register-
// blocked FMA loop over K.  Latency-oriented: a single load phase, no k-slice pipeline.
//
// KT > 0 (K == KT): B is A12 before the TRSM and the kernel applies L11^-1 itself (K4 fused
// into K5 for the small in-panel levels): every CTA solves the KT x N unit-lower system in
// shared memory (one column per thread, the column in registers, substitution in the same
// order as K4 -> identical U12 bits), uses it, and the LAST CTA to have read A12 (ticket
// counter, so no CTA ever waits) writes U12 back over it and re-arms the counter.
template <typename T, int BM, int NMAX, int KT>
__global__ void __launch_bounds__(256)
tsgemm_kernel(const T *__restrict__ A, int64_t lda, T *__restrict__ B, int64_t ldb, T *__restrict__ C,
              int64_t ldc, int M, int N, int K, const T *__restrict__ L11, int32_t *__restrict__ ticket)
{
    constexpr int TX = 16, TY = 16;                     // threads along N, along rows
    constexpr int TN = NMAX / TX, TM = BM / TY;
    constexpr int APAD = BM + 4, BPAD = NMAX + 4;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    pdl_trigger();
    T *As = reinterpret_cast<T *>(smem_raw);            // [K][APAD]  As[k][i] = L21(i, k)
    T *Bs = As + (size_t)128 * APAD;                    // [K][BPAD]  Bs[k][j] = U12(k, j)
    const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
    const int64_t bm0 = (int64_t)blockIdx.x * BM;
    // stage B (coalesced along N) and the A slab (coalesced along K, stored transposed)
    // (8 independent global loads in flight per thread before the shared-memory stores)
    for (int b0 = tid; b0 < K * NMAX; b0 += 8 * 256) {
        T v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = b0 + u * 256, k = idx / NMAX, j = idx - k * NMAX;
            v[u] = (idx < K * NMAX && j < N) ? B[(int64_t)k * ldb + j] : T(0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = b0 + u * 256, k = idx / NMAX, j = idx - k * NMAX;
            if (idx < K * NMAX) Bs[k * BPAD + j] = v[u];
        }
    }
    for (int b0 = tid; b0 < BM * K; b0 += 8 * 256) {
        T v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = b0 + u * 256, i = idx / K, k = idx - i * K;
            v[u] = (idx < BM * K && bm0 + i < M) ? A[(bm0 + i) * lda + k] : T(0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = b0 + u * 256, i = idx / K, k = idx - i * K;
            if (idx < BM * K) As[k * APAD + i] = v[u];
        }
    }
    __syncthreads();
    if constexpr (KT > 0) {
        // ---- U12 = L11^-1 A12 (unit lower, forward substitution per column)
        T *Ls = Bs + (size_t)128 * BPAD;                    // [KT][KT] L11
        for (int idx = tid; idx < KT * KT; idx += 256) {
            const int i = idx / KT, k = idx - i * KT;
            Ls[idx] = i > k ? L11[(int64_t)i * lda + k] : T(0);
        }
        __syncthreads();
        if (tid < N) {
            T x[KT];
#pragma unroll
            for (int i = 0; i < KT; ++i) x[i] = Bs[i * BPAD + tid];
#pragma unroll
            for (int k = 0; k < KT; ++k)
#pragma unroll
                for (int i = k + 1; i < KT; ++i) x[i] = fma(-Ls[i * KT + k], x[k], x[i]);
#pragma unroll
            for (int i = 0; i < KT; ++i) Bs[i * BPAD + tid] = x[i];
        }
        __shared__ int s_last;
        if (tid == 0) s_last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;   // this CTA's A12 reads are done
        __syncthreads();
        if (s_last) {
            for (int idx = tid; idx < KT * N; idx += 256) {
                const int k = idx / N, j = idx - k * N;
                B[(int64_t)k * ldb + j] = Bs[k * BPAD + j];
            }
            if (tid == 0) *ticket = 0;
        }
    }
    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
        T a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = As[k * APAD + ty * TM + i];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = Bs[k * BPAD + tx * TN + j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int64_t row = bm0 + ty * TM + i;
        if (row >= M) continue;
        T *crow = C + row * ldc;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int col = tx * TN + j;
            if (col < N) crow[col] -= acc[i][j];
        }
    }
}

template <typename T, int BM, int NMAX, int KT = 0>
void launch_ts(const T *A, int64_t lda, const T *B, int64_t ldb, T *C, int64_t ldc, int64_t M, int64_t N, int64_t K,
               cudaStream_t s, const T *L11 = nullptr, int32_t *ticket = nullptr)
{
    const size_t smem = ((size_t)128 * (BM + 4) + (size_t)128 * (NMAX + 4) + (size_t)KT * KT) * sizeof(T);
    auto kern = tsgemm_kernel<T, BM, NMAX, KT>;
    func_smem_once((const void *)kern, smem);
    launch_ex(kern, dim3((unsigned)ceil_div(M, BM)), dim3(256), smem, s, nullptr, A, lda, const_cast<T *>(B), ldb, C,
              ldc, (int)M, (int)N, (int)K, L11, ticket);
}

// Persistent, software-pipelined form of the fused in-panel update (K = KT in {32, 64},
// N <= NMAX <= 64): the U12 solve happens ONCE per CTA, then each CTA walks its BM-row blocks
// with the next block's L21 slab and C tile loaded (into registers) while the current one is
// multiplied — the slab is latency-bound, so overlapping the round trips is the whole gain.
template <typename T, int BM, int NMAX, int KT>
__global__ void __launch_bounds__(256)
tsgemm_fused_persist_kernel(const T *__restrict__ A, int64_t lda, T *__restrict__ B, int64_t ldb,
                            T *__restrict__ C, int64_t ldc, int M, int N, const T *__restrict__ L11,
                            int32_t *__restrict__ ticket)
{
    constexpr int TX = 16, TY = 16, TN = NMAX / TX, TM = BM / TY;
    constexpr int APAD = BM + 4, BPAD = NMAX + 4;
    constexpr int AV = BM * KT / 256;                     // slab elements per thread
    static_assert(BM * KT % 256 == 0, "slab split");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    pdl_trigger();
    T *Bs = reinterpret_cast<T *>(smem_raw);              // [KT][BPAD]  U12 (after the solve)
    T *As = Bs + (size_t)KT * BPAD;                       // [2][KT][APAD] L21 slab, transposed
    T *Ls = As + (size_t)2 * KT * APAD;                   // [KT][KT] L11
    const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
    const int nblk = (M + BM - 1) / BM;
    auto load_slab = [&](int rb, T (&v)[AV]) {
#pragma unroll
        for (int u = 0; u < AV; ++u) {
            const int idx = tid + 256 * u, i = idx / KT, k = idx - i * KT;
            const int64_t row = (int64_t)rb * BM + i;
            v[u] = (rb < nblk && row < M) ? A[row * lda + k] : T(0);
        }
    };
    auto store_slab = [&](T *dst, const T (&v)[AV]) {
#pragma unroll
        for (int u = 0; u < AV; ++u) {
            const int idx = tid + 256 * u, i = idx / KT, k = idx - i * KT;
            dst[k * APAD + i] = v[u];
        }
    };
    auto load_c = [&](int rb, T (&cv)[TM][TN]) {
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int64_t row = (int64_t)rb * BM + ty * TM + i;
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int col = tx * TN + j;
                cv[i][j] = (rb < nblk && row < M && col < N) ? C[row * ldc + col] : T(0);
            }
        }
    };
    int rb = blockIdx.x;
    T av[AV], cv[TM][TN];
    load_slab(rb, av);
    load_c(rb, cv);
    // ---- B = A12, L11 (every CTA; cp.async: every element in flight at once), then
    // U12 = L11^-1 A12 in place (the order of K4; only the strictly lower part of L11 is read)
    {
        const uint32_t bsb = (uint32_t)__cvta_generic_to_shared(Bs), lsb = (uint32_t)__cvta_generic_to_shared(Ls);
        for (int idx = tid; idx < KT * NMAX; idx += 256) {
            const int k = idx / NMAX, j = idx - k * NMAX;
            const bool ok = j < N;
            asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(bsb + (uint32_t)(k * BPAD + j) * (uint32_t)sizeof(T)),
                         "l"(B + (int64_t)k * ldb + (ok ? j : 0)), "n"((int)sizeof(T)), "r"(ok ? (int)sizeof(T) : 0) : "memory");
        }
        for (int idx = tid; idx < KT * KT; idx += 256) {
            const int i = idx / KT, k = idx - i * KT;
            asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(lsb + (uint32_t)idx * (uint32_t)sizeof(T)),
                         "l"(L11 + (int64_t)i * lda + k), "n"((int)sizeof(T)) : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    store_slab(As, av);
    __syncthreads();
    if (tid < N) {
        T x[KT];
#pragma unroll
        for (int i = 0; i < KT; ++i) x[i] = Bs[i * BPAD + tid];
#pragma unroll
        for (int k = 0; k < KT; ++k)
#pragma unroll
            for (int i = k + 1; i < KT; ++i) x[i] = fma(-Ls[i * KT + k], x[k], x[i]);
#pragma unroll
        for (int i = 0; i < KT; ++i) Bs[i * BPAD + tid] = x[i];
    }
    __shared__ int s_last;
    if (tid == 0) s_last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;   // this CTA's A12 reads are done
    __syncthreads();
    if (s_last) {
        for (int idx = tid; idx < KT * N; idx += 256) {
            const int k = idx / N, j = idx - k * N;
            B[(int64_t)k * ldb + j] = Bs[k * BPAD + j];
        }
        if (tid == 0) *ticket = 0;
    }
    // ---- the row blocks of this CTA, next block's loads in flight during the current multiply
    for (int it = 0; rb < nblk; ++it, rb += gridDim.x) {
        const int rbn = rb + gridDim.x;
        T avn[AV], cvn[TM][TN];
        load_slab(rbn, avn);
        load_c(rbn, cvn);
        const T *Ab = As + (size_t)(it & 1) * KT * APAD;
        T acc[TM][TN];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
#pragma unroll 8
        for (int k = 0; k < KT; ++k) {
            T a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = Ab[k * APAD + ty * TM + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) b[j] = Bs[k * BPAD + tx * TN + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int64_t row = (int64_t)rb * BM + ty * TM + i;
            if (row >= M) continue;
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int col = tx * TN + j;
                if (col < N) C[row * ldc + col] = cv[i][j] - acc[i][j];
            }
        }
        store_slab(As + (size_t)((it + 1) & 1) * KT * APAD, avn);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) cv[i][j] = cvn[i][j];
        __syncthreads();
    }
}

template <typename T, int BM, int NMAX, int KT>
void launch_fused_persist(const T *A, int64_t lda, T *B, int64_t ldb, T *C, int64_t ldc, int64_t M, int64_t N,
                          const T *L11, int32_t *ticket, int grid_max, cudaStream_t s)
{
    const size_t smem = ((size_t)KT * (NMAX + 4) + (size_t)2 * KT * (BM + 4) + (size_t)KT * KT) * sizeof(T);
    auto kern = tsgemm_fused_persist_kernel<T, BM, NMAX, KT>;
    func_smem_once((const void *)kern, smem);
    const int grid = (int)std::min<int64_t>(ceil_div(M, BM), grid_max);
    launch_ex(kern, dim3(grid), dim3(256), smem, s, nullptr, A, lda, B, ldb, C, ldc, (int)M, (int)N, L11, ticket);
}

}  // namespace

// In-panel Schur update with the TRSM fused (K = w1 in {32, 64}, N <= 64): W rows [k0, k0+K)
// of columns [c0, c0+N) hold A12 on entry and U12 on exit; rows [r0, r0+M) are updated.
// Returns false (nothing launched) when the shape has no fused variant.
template <typename T>
bool launch_trsm_gemm_fused(T *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N, int64_t K,
                            int32_t *ticket, cudaStream_t s)
{
    if (M <= 0 || N <= 0 || N > 64 || !(K == 32 || K == 64)) return false;
    const T *A = W + r0 * ldw + k0, *L11 = W + k0 * ldw + k0;
    T *B = W + k0 * ldw + c0, *C = W + r0 * ldw + c0;
    static const int persist = [] { const char *e = std::getenv("MP_FUSED_GRID"); return e ? std::atoi(e) : 96; }();
    if constexpr (sizeof(T) == 4) {
        if (persist > 0) {                                   // persistent pipelined form (default)
            if (K == 32) {
                if (N <= 32) launch_fused_persist<T, 64, 32, 32>(A, ldw, B, ldw, C, ldw, M, N, L11, ticket, persist, s);
                else launch_fused_persist<T, 64, 64, 32>(A, ldw, B, ldw, C, ldw, M, N, L11, ticket, persist, s);
            } else {
                if (N <= 32) launch_fused_persist<T, 64, 32, 64>(A, ldw, B, ldw, C, ldw, M, N, L11, ticket, persist, s);
                else launch_fused_persist<T, 64, 64, 64>(A, ldw, B, ldw, C, ldw, M, N, L11, ticket, persist, s);
            }
            return true;
        }
    }
    constexpr int BMF = sizeof(T) == 4 ? 64 : 32;
    if (K == 32) {
        if (N <= 32) launch_ts<T, BMF, 32, 32>(A, ldw, B, ldw, C, ldw, M, N, K, s, L11, ticket);
        else launch_ts<T, BMF, 64, 32>(A, ldw, B, ldw, C, ldw, M, N, K, s, L11, ticket);
    } else {
        if (N <= 32) launch_ts<T, BMF, 32, 64>(A, ldw, B, ldw, C, ldw, M, N, K, s, L11, ticket);
        else launch_ts<T, BMF, 64, 64>(A, ldw, B, ldw, C, ldw, M, N, K, s, L11, ticket);
    }
    return true;
}
template bool launch_trsm_gemm_fused<float>(float *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                                            int32_t *, cudaStream_t);
template bool launch_trsm_gemm_fused<double>(double *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                                             int32_t *, cudaStream_t);

template <>
void launch_gemm_ops<float>(const float *A, int64_t lda, const float *B, int64_t ldb, float *C, int64_t ldc,
                            int64_t M, int64_t N, int64_t K, cudaStream_t s)
{
    if (M <= 0 || N <= 0 || K <= 0) return;
    if (K <= 128 && N <= 32) return launch_ts<float, 64, 32>(A, lda, B, ldb, C, ldc, M, N, K, s);
    if (K <= 128 && N <= 64) return launch_ts<float, 64, 64>(A, lda, B, ldb, C, ldc, M, N, K, s);
    if (K <= 128 && N <= 128) return launch_ts<float, 64, 128>(A, lda, B, ldb, C, ldc, M, N, K, s);
    static const bool no_tma = std::getenv("MP_NO_SGEMM_TMA") != nullptr;   // A/B: the register-staged tile kernel
    if (!no_tma && launch_sgemm_tma(A, lda, B, ldb, C, ldc, M, N, K, s)) return;
    launch_tiles<float, 128, 128, 8, 8, 8>(A, lda, B, ldb, C, ldc, M, N, K, s);
}

template <>
void launch_gemm_ops<double>(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc,
                             int64_t M, int64_t N, int64_t K, cudaStream_t s)
{
    if (M <= 0 || N <= 0 || K <= 0) return;
    if (K <= 128 && N <= 32) return launch_ts<double, 32, 32>(A, lda, B, ldb, C, ldc, M, N, K, s);
    if (K <= 128 && N <= 64) return launch_ts<double, 32, 64>(A, lda, B, ldb, C, ldc, M, N, K, s);
    static const bool no_dmma = std::getenv("MP_NO_DMMA") != nullptr;   // A/B: the DFMA tile kernel
    if (!no_dmma && launch_dgemm_dmma(A, lda, B, ldb, C, ldc, M, N, K, s)) return;
    launch_tiles<double, 128, 64, 8, 8, 4>(A, lda, B, ldb, C, ldc, M, N, K, s);
}

// the binary64 DFMA tile kernel alone (kernel tests / A-B against DMMA)
void launch_dgemm_dfma(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc,
                       int64_t M, int64_t N, int64_t K, cudaStream_t s)
{
    if (M <= 0 || N <= 0 || K <= 0) return;
    launch_tiles<double, 128, 64, 8, 8, 4>(A, lda, B, ldb, C, ldc, M, N, K, s);
}

template <typename T>
void launch_gemm_update(T *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N, int64_t K,
                        cudaStream_t s)
{
    launch_gemm_ops<T>(W + r0 * ldw + k0, ldw, W + k0 * ldw + c0, ldw, W + r0 * ldw + c0, ldw, M, N, K, s);
}

template void launch_gemm_update<float>(float *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                                        cudaStream_t);
template void launch_gemm_update<double>(double *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                                         cudaStream_t);

}  // namespace mp
