// k_sgemm_tma.cu — K5a: the FFMA trailing update C <- C - A B (binary32 CUDA-core FMAs), with the
// operand tiles staged by TMA through an mbarrier ring (north_star's "FP32 FFMA SGEMM with
// TMA-staged tiles", SGETRF's trailing update in single precision).
//
// Operands are row-major views into the working copy: A = L21 (M x K, K contiguous), B = U12
// (K x N, N contiguous), C = A22 (M x N).  One CTA computes a 128 x 128 tile of C:
//   * thread 0: per 32-deep K chunk one TMA box of A (128 rows x 32 k, SWIZZLE_128B) and one of
//     B (32 k x 128 n, unswizzled 512-byte rows) into a 3-stage ring, two chunks ahead, mbarrier
//     expect_tx; out-of-range rows / columns / k are zero-filled by the TMA unit;
//   * all 8 warps (256 threads): thread (tr = tid / 16, tc = tid % 16) owns rows tr + 16 r (r < 8)
//     and columns 4 tc + 64 h + e (h < 2, e < 4): per k 8 LDS.32 of A (a quarter warp shares tr:
//     broadcast) and 2 LDS.128 of B (16 lanes read 256 contiguous bytes), then 64 FFMAs; each warp
//     chunk ends with a CTA barrier (the slot is then free for thread 0's next TMA);
//   * epilogue: C -= acc with 16-byte accesses, a half warp covering 256 contiguous bytes of a row.
// 2 CTAs per SM (96 KB ring each): one CTA's prologue / epilogue overlaps the other's FMAs.  Per element the products are summed in k order from zero and
// subtracted from C once, as in the register-staged tile kernel it replaces (k_gemm.cu).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "internal.h"

namespace mp {

namespace {

constexpr int SBM = 128, SBN = 128, SBK = 32, SST = 3;
constexpr int SNT = 256;                                    // 8 warps; thread 0 also issues the TMA
constexpr uint32_t SA_BYTES = SBM * SBK * 4, SB_BYTES = SBK * SBN * 4;
constexpr uint32_t SSTAGE = SA_BYTES + SB_BYTES;            // 32 KB

__device__ __forceinline__ uint32_t s_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sm_bar_init(uint64_t *b, uint32_t c)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(c));
}
__device__ __forceinline__ bool sm_bar_try(uint64_t *b, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(s_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void sm_bar_wait(uint64_t *b, uint32_t parity)
{
    while (!sm_bar_try(b, parity)) { }
}
__device__ __forceinline__ void sm_tma2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            s_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(s_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(SNT, 2)
sgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 float *__restrict__ C, int64_t ldc, int M, int N, int K)
{
    extern __shared__ __align__(1024) unsigned char sg_raw[];
    // 1 KB alignment (SWIZZLE_128B) by an offset on the shared array: the loads below stay LDS
    unsigned char *ring = sg_raw + ((1024u - (s_u32(sg_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t full[SST];
    const int tid = threadIdx.x;
    const int bm0 = blockIdx.y * SBM, bn0 = blockIdx.x * SBN;
    const int nk = (K + SBK - 1) / SBK;
    auto issue = [&](int kc) {            // thread 0: chunk kc into its ring slot
        const int s = kc % SST;
        unsigned char *st = ring + (size_t)s * SSTAGE;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&full[s])), "r"(SSTAGE)
                     : "memory");
        sm_tma2d(st, &tmA, &full[s], kc * SBK, bm0);
        sm_tma2d(st + SA_BYTES, &tmB, &full[s], bn0, kc * SBK);
    };
    if (tid == 0) {
        for (int s = 0; s < SST; ++s) sm_bar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();                 // (no early trigger: a dependent parked beside the GEMM only holds resources)
    if (tid == 0)
        for (int kc = 0; kc < SST - 1 && kc < nk; ++kc) issue(kc);
    const int tr = tid >> 4, tc = tid & 15;
    float acc[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
    for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % SST;
        // the slot of chunk kc + SST - 1 was consumed in iteration kc - 1 (every thread passed its
        // closing barrier), so thread 0 refills it now, SST - 1 chunks ahead of the consumers
        if (tid == 0 && kc + SST - 1 < nk) issue(kc + SST - 1);
        sm_bar_wait(&full[s], (uint32_t)((kc / SST) & 1));
        const unsigned char *As = ring + (size_t)s * SSTAGE;   // [128 rows][128 B], 16-byte chunk q of row i at q ^ (i & 7)
        const float *Bs = reinterpret_cast<const float *>(As + SA_BYTES);   // [32 k][128 n]
#pragma unroll
        for (int k = 0; k < SBK; ++k) {
            // A(i, k) for the thread's 8 rows (a quarter warp shares tr: broadcast), B(k, 8 columns)
            float av[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int i = tr + 16 * r;
                av[r] = *reinterpret_cast<const float *>(As + i * 128 + (((k >> 2) ^ (i & 7)) << 4) + ((k & 3) << 2));
            }
            const float4 b0 = *reinterpret_cast<const float4 *>(Bs + k * SBN + tc * 4);
            const float4 b1 = *reinterpret_cast<const float4 *>(Bs + k * SBN + 64 + tc * 4);
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
        }
        __syncthreads();
    }
    // ---- epilogue: C -= acc
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int i = bm0 + tr + 16 * r;
        if (i >= M) continue;
        float *crow = C + (int64_t)i * ldc + bn0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = h * 64 + tc * 4;
            if (bn0 + j + 3 < N) {
                float4 v = *reinterpret_cast<float4 *>(crow + j);
                v.x -= acc[r][4 * h]; v.y -= acc[r][4 * h + 1]; v.z -= acc[r][4 * h + 2]; v.w -= acc[r][4 * h + 3];
                *reinterpret_cast<float4 *>(crow + j) = v;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (bn0 + j + e < N) crow[j + e] -= acc[r][4 * h + e];
            }
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 s_encode = nullptr;

bool encode2d(CUtensorMap *map, const float *base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_in,
              uint32_t box_out, CUtensorMapSwizzle sw)
{
    if (!s_encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return false;
        }
        s_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t gdim[2] = {inner, outer};
    cuuint64_t gstride[1] = {ld * sizeof(float)};
    cuuint32_t box[2] = {box_in, box_out};
    cuuint32_t estr[2] = {1, 1};
    return s_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// C[M x N] -= A[M x K] B[K x N] (row-major, binary32 FFMA).  false: the TMA constraints (16-byte
// aligned bases, leading dimensions multiple of 4) do not hold and nothing was launched.
bool launch_sgemm_tma(const float *A, int64_t lda, const float *B, int64_t ldb, float *C, int64_t ldc, int64_t M,
                      int64_t N, int64_t K, cudaStream_t s)
{
    if (M <= 0 || N <= 0 || K <= 0) return true;
    if ((uintptr_t)A % 16 || (uintptr_t)B % 16 || lda % 4 || ldb % 4 || M > (1 << 30) || N > (1 << 30)) return false;
    CUtensorMap mA, mB;
    if (!encode2d(&mA, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, SBK, SBM, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
    if (!encode2d(&mB, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, SBN, SBK, CU_TENSOR_MAP_SWIZZLE_NONE)) return false;
    const size_t smem = (size_t)SST * SSTAGE + 1024;
    func_smem_once((const void *)sgemm_tma_kernel, smem);
    dim3 grid((unsigned)ceil_div(N, (int64_t)SBN), (unsigned)ceil_div(M, (int64_t)SBM));
    launch_ex(sgemm_tma_kernel, grid, dim3(SNT), smem, s, nullptr, mA, mB, C, ldc, (int)M, (int)N, (int)K);
    return true;
}

}  // namespace mp
