// k_solve.cu — K7 + K9: the binary32 triangular solves with the packed LU and
// the binary64 update of the solution.
//
// PAPER.md Alg. 1 steps 2-3 / 5-6: "solve L y = P r_k",
// "solve U z_k = y" in single precision; step 7: x_k <- x_{k-1} + z_k
// in double (fused into the backward solve's write-back).  The permutation P
// was already applied when y was demoted (K6 / the residual epilogue).
//
// One kernel per triangle.  The n rows are cut into BS-row block rows; CTAs
// take block rows in dependency order from an atomic ticket and chain on
// per-block ready flags (no grid barrier, no per-block launches).  CTA I
// streams the off-diagonal tiles L(I, J) (or U(I, J)) as soon as block J is
// published — the GEMV part, HBM-bound, 4 n^2 bytes per forward+backward pair
// — then one warp per right-hand side runs the BS-step substitution of the
// diagonal block (latency-bound), publishes its block and sets its flag.
#include <algorithm>

#include "internal.h"

namespace mp {

namespace {

constexpr int BS = 128;           // block-row height
constexpr int ST = 256;           // threads per CTA
constexpr int MAXR = 16;          // right-hand sides per launch
constexpr int LDD = BS + 1;       // smem stride of the transposed diagonal block

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T> struct V4;
template <> struct V4<float> { using type = float4; };
template <> struct V4<double> { using type = double4; };

// LOWER = true : unit-lower forward substitution, block rows in increasing order.
// LOWER = false: upper backward substitution (non-unit diagonal), decreasing order;
//                X[rows] = (double) z  (accumulate = 0)  or  X += (double) z  (accumulate = 1).
template <typename T, bool LOWER>
__global__ void __launch_bounds__(ST, 1)
tri_solve_kernel(const T *__restrict__ W, int64_t ldw, int64_t n, int nrhs, T *Y, int64_t ldy, double *X,
                 int accumulate, unsigned *flags, unsigned *ticket)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *Ld = reinterpret_cast<T *>(smem_raw);             // [BS][LDD]   Ld[j][i] = Tri(i, j) of the diagonal block
    T *ys = Ld + BS * LDD;                               // [BS][MAXR]  published block J / final block I
    __shared__ int s_blk;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nblk = (int)ceil_div(n, BS);
    if (tid == 0) {
        const unsigned t = atomicAdd(ticket, 1u);
        s_blk = LOWER ? (int)t : nblk - 1 - (int)t;
    }
    __syncthreads();
    const int I = s_blk;
    const int64_t i0 = (int64_t)I * BS;
    const int nr = (int)((n - i0 < (int64_t)BS) ? (n - i0) : (int64_t)BS);

    // stage the diagonal block transposed (Ld[j][i] = Tri(i0+i, i0+j)) and this block's
    // right-hand side first: neither depends on other blocks, so this overlaps the waits.
    // Warp-per-row, lanes along j: coalesced 128 B reads, conflict-free transposed stores.
    for (int i = warp; i < BS; i += ST / 32) {
#pragma unroll
        for (int k = 0; k < BS / 32; ++k) {
            const int j = lane + 32 * k;
            Ld[j * LDD + i] = (i < nr && j < nr) ? W[(i0 + i) * ldw + i0 + j] : T(0);
        }
    }
    T rhs[MAXR];
    {
        const int rr = tid >> 1;
#pragma unroll
        for (int c = 0; c < MAXR; ++c) rhs[c] = (c < nrhs && rr < nr && (tid & 1) == 0) ? Y[c * ldy + i0 + rr] : T(0);
    }

    // ---- off-diagonal GEMV part: 2 threads per row, each half of every tile
    const int r = tid >> 1, half = tid & 1;
    T psum[MAXR];
#pragma unroll
    for (int c = 0; c < MAXR; ++c) psum[c] = T(0);
    // visit the off-diagonal blocks in the order they become ready: increasing J for
    // the forward sweep, DECREASING J for the backward sweep (block nblk-1 is published first)
    const int ntiles = LOWER ? I : nblk - 1 - I;
    for (int t = 0; t < ntiles; ++t) {
        const int J = LOWER ? t : nblk - 1 - t;
        const int64_t j0 = (int64_t)J * BS;
        const int nc = (int)((n - j0 < (int64_t)BS) ? (n - j0) : (int64_t)BS);
        if (tid == 0) {
            // relaxed polling (an acquire load per poll would invalidate L1 every time),
            // then one acquire fence once the flag is seen
            while (ld_relaxed_u32(flags + J) == 0u) { }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
        for (int idx = tid; idx < nc * nrhs; idx += ST) {
            const int j = idx % nc, c = idx / nc;
            ys[j * MAXR + c] = __ldcg(Y + c * ldy + j0 + j);
        }
        __syncthreads();
        if (r < nr) {
            const T *lrow = W + (i0 + r) * ldw + j0;
            const int jlo = half * (BS / 2);
            const int jhi = (nc < jlo + BS / 2) ? nc : jlo + BS / 2;
            if (nc == BS) {
                using V = typename V4<T>::type;
#pragma unroll 4
                for (int j = jlo; j < jhi; j += 4) {
                    const V lv = *reinterpret_cast<const V *>(lrow + j);
                    const T *yj = ys + j * MAXR;
#pragma unroll
                    for (int c = 0; c < MAXR; ++c) {
                        if (c < nrhs) {
                            psum[c] = fma(lv.x, yj[c], psum[c]);
                            psum[c] = fma(lv.y, yj[MAXR + c], psum[c]);
                            psum[c] = fma(lv.z, yj[2 * MAXR + c], psum[c]);
                            psum[c] = fma(lv.w, yj[3 * MAXR + c], psum[c]);
                        }
                    }
                }
            } else {
                for (int j = jlo; j < jhi; ++j) {
                    const T lv = lrow[j];
#pragma unroll
                    for (int c = 0; c < MAXR; ++c)
                        if (c < nrhs) psum[c] = fma(lv, ys[j * MAXR + c], psum[c]);
                }
            }
        }
        __syncthreads();
    }
    // combine the two halves; rhs block I minus the off-diagonal sums -> ys[r][c]
#pragma unroll
    for (int c = 0; c < MAXR; ++c) psum[c] += __shfl_xor_sync(0xffffffffu, psum[c], 1);
    if (half == 0 && r < nr) {
#pragma unroll
        for (int c = 0; c < MAXR; ++c)
            if (c < nrhs) ys[r * MAXR + c] = rhs[c] - psum[c];
    }
    __syncthreads();

    // ---- substitution on the diagonal block, in 32-row sub-blocks (forward: top-down,
    //      backward: bottom-up).  The 32 x 32 triangle: lane i keeps row i of the triangle in
    //      registers and its rhs b_i; a fully unrolled chain x_j = shfl(b, j), b_i -= t_ij x_j
    //      (one warp per right-hand side).  The rows of the block not yet solved then get the
    //      sub-block's contribution from all 256 threads.
#pragma unroll 1
    for (int sbi = 0; sbi < BS / 32; ++sbi) {
        const int sb = LOWER ? sbi : BS / 32 - 1 - sbi;
        const int s0 = sb * 32;
        if (s0 >= nr) continue;
        const int i = s0 + lane;                           // this lane's row
        for (int c = warp; c < nrhs; c += ST / 32) {
            T trow[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) trow[j] = Ld[(s0 + j) * LDD + i];
            T b = i < nr ? ys[i * MAXR + c] : T(0);
            if (LOWER) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const T xj = __shfl_sync(0xffffffffu, b, j);
                    if (lane > j && s0 + j < nr) b = fma(-trow[j], xj, b);
                }
            } else {
#pragma unroll
                for (int j = 31; j >= 0; --j) {
                    if (s0 + j < nr) {
                        if (lane == j) b = b / trow[j];        // U(j, j): non-unit diagonal
                        const T xj = __shfl_sync(0xffffffffu, b, j);
                        if (lane < j) b = fma(-trow[j], xj, b);
                    }
                }
            }
            if (i < nr) ys[i * MAXR + c] = b;
        }
        __syncthreads();
        // contribution of the 32 solved rows to the block rows still to be solved
        const int rlo = LOWER ? s0 + 32 : 0, rhi = LOWER ? nr : s0;
        const int nrem = rhi > rlo ? rhi - rlo : 0;
        for (int idx = tid; idx < nrem * nrhs; idx += ST) {
            const int r = rlo + idx % nrem, c = idx / nrem;
            T acc = ys[r * MAXR + c];
#pragma unroll 8
            for (int j = 0; j < 32; ++j)
                if (s0 + j < nr) acc = fma(-Ld[(s0 + j) * LDD + r], ys[(s0 + j) * MAXR + c], acc);
            ys[r * MAXR + c] = acc;
        }
        __syncthreads();
    }
    // publish the solved block (and, backward, x += z in binary64: step 7)
    for (int idx = tid; idx < nr * nrhs; idx += ST) {
        const int r = idx % nr, c = idx / nr;
        const T v = ys[r * MAXR + c];
        Y[c * ldy + i0 + r] = v;
        if (!LOWER) {
            double *xp = X + c * ldy + i0 + r;
            *xp = accumulate ? *xp + (double)v : (double)v;
        }
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        st_release_u32(flags + I, 1u);
    }
}

template <typename T>
size_t tri_smem() { return (size_t)BS * LDD * sizeof(T) + (size_t)BS * MAXR * sizeof(T); }

}  // namespace

int solve_block_rows() { return BS; }

template <typename T>
void launch_lu_solve(const T *W, int64_t ldw, int64_t n, int64_t nrhs, T *Y, double *X, int accumulate,
                     SolveScratch &ss, cudaStream_t s)
{
    const int nblk = (int)ceil_div(n, BS);
    const size_t smem = tri_smem<T>();
    auto kl = tri_solve_kernel<T, true>;
    auto ku = tri_solve_kernel<T, false>;
    func_smem_once((const void *)kl, smem);
    func_smem_once((const void *)ku, smem);
    for (int64_t c0 = 0; c0 < nrhs; c0 += MAXR) {
        const int nc = (int)std::min<int64_t>(MAXR, nrhs - c0);
        MP_CUDA(cudaMemsetAsync(ss.flags, 0, sizeof(unsigned) * (2 * (size_t)nblk), s));
        MP_CUDA(cudaMemsetAsync(ss.tickets, 0, sizeof(unsigned) * 2, s));
        kl<<<nblk, ST, smem, s>>>(W, ldw, n, nc, Y + c0 * n, n, X + c0 * n, accumulate, ss.flags, ss.tickets);
        MP_LAUNCH_CHECK();
        ku<<<nblk, ST, smem, s>>>(W, ldw, n, nc, Y + c0 * n, n, X + c0 * n, accumulate, ss.flags + nblk,
                                  ss.tickets + 1);
        MP_LAUNCH_CHECK();
        g_launches += 2;
    }
}

template void launch_lu_solve<float>(const float *, int64_t, int64_t, int64_t, float *, double *, int,
                                     SolveScratch &, cudaStream_t);
template void launch_lu_solve<double>(const double *, int64_t, int64_t, int64_t, double *, double *, int,
                                      SolveScratch &, cudaStream_t);

}  // namespace mp
