// k_trsm.cu — K4: U12 <- L11^{-1} A12 (left, lower, unit diagonal).
//
// Blocked right-looking LU (SGETRF's blocked form): after a
// panel of width w is factored, its unit-lower block L11 is applied to the w
// rows of the columns to its right by forward SUBSTITUTION (no explicit
// inverse, so exact inputs stay exact — pin P2).
//
// Each lane owns one column (32 columns per warp); a row block of 32 rows is
// held in registers; L11 sub-blocks are staged in shared memory, transposed
// so that 4 consecutive rows are one broadcast LDS.128.  FMA-bound,
// w^2/2 FMAs per column.
#include <algorithm>

#include "internal.h"

namespace mp {

namespace {

constexpr int TW = 4;             // warps per CTA
constexpr int TT = TW * 32;
constexpr int RB = 32;            // rows per register block
constexpr int LS = RB + 4;        // smem row stride of the transposed L block (16B aligned)

template <typename T>
__global__ void __launch_bounds__(TT)
trsm_lower_unit_kernel(T *__restrict__ W, int64_t ldw, int64_t r0, int w, int64_t c_lo, int64_t c_hi)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *Ls = reinterpret_cast<T *>(smem_raw);   // [w][LS]: Ls[j][i] = L(rb+i, j)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t col = c_lo + (int64_t)blockIdx.x * TT + warp * 32 + lane;
    const bool valid = col < c_hi;
    T acc[RB];

    for (int rb = 0; rb < w; rb += RB) {
        const int nr = (w - rb < RB) ? (w - rb) : RB;
        const int ncols = rb + nr;             // L columns 0 .. rb+nr-1 are needed
        __syncthreads();
        for (int idx = threadIdx.x; idx < RB * ncols; idx += TT) {
            const int i = idx / ncols, j = idx - i * ncols;
            T v = T(0);
            if (i < nr && j < rb + i) v = W[(r0 + rb + i) * ldw + r0 + j];   // strictly lower part only
            Ls[j * LS + i] = v;
        }
        __syncthreads();
        if (valid) {
#pragma unroll
            for (int i = 0; i < RB; ++i) acc[i] = i < nr ? W[(r0 + rb + i) * ldw + col] : T(0);
            // contributions of the already-solved rows 0 .. rb-1
            // (x_j of the already-solved rows: 8 independent loads in flight per step)
            for (int j = 0; j < rb; j += 8) {
                T xv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) xv[u] = W[(r0 + j + u) * ldw + col];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const T *lj = Ls + (j + u) * LS;
#pragma unroll
                    for (int i = 0; i < RB; ++i) acc[i] -= lj[i] * xv[u];
                }
            }
            // the 32 x 32 diagonal block
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                const T xj = acc[j];
                const T *lj = Ls + (rb + j) * LS;
#pragma unroll
                for (int i = j + 1; i < RB; ++i) acc[i] -= lj[i] * xj;
            }
#pragma unroll
            for (int i = 0; i < RB; ++i)
                if (i < nr) W[(r0 + rb + i) * ldw + col] = acc[i];
        }
    }
}

}  // namespace

template <typename T>
void launch_trsm_lower_unit(T *W, int64_t ldw, int64_t r0, int w, int64_t c_lo, int64_t c_hi, cudaStream_t s)
{
    if (c_hi <= c_lo || w <= 0) return;
    const int grid = (int)ceil_div(c_hi - c_lo, TT);
    const size_t smem = (size_t)round_up(w, RB) * LS * sizeof(T);
    auto kern = trsm_lower_unit_kernel<T>;
    if (smem > 48 * 1024) func_smem_once((const void *)kern, smem);
    kern<<<grid, TT, smem, s>>>(W, ldw, r0, w, c_lo, c_hi);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template void launch_trsm_lower_unit<float>(float *, int64_t, int64_t, int, int64_t, int64_t, cudaStream_t);
template void launch_trsm_lower_unit<double>(double *, int64_t, int64_t, int, int64_t, int64_t, cudaStream_t);

}  // namespace mp
