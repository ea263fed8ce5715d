// k_trsm.cu — K4: U12 <- L11^{-1} A12 (left, lower, unit diagonal).
//
// Blocked right-looking LU (SGETRF's blocked form): after a
// panel of width w is factored, its unit-lower block L11 is applied to the w
// rows of the columns to its right by forward SUBSTITUTION (no explicit
// inverse, so exact inputs stay exact — pin P2).
//
// One CTA per 32-column strip; warp b owns row block b (32 rows x 32 columns
// in registers, lane = column).  Warp b applies X_b -= L(b, k) X_k for every
// earlier row block k as soon as warp k has published X_k in shared memory
// (only k = b-1 is on the dependent chain), then solves its 32 x 32 unit-lower
// diagonal block column-oriented (x_i final -> x_m -= l_mi x_i, m > i), and
// publishes X_b.  L blocks are staged transposed in shared memory so every
// inner step is one broadcast LDS.128 + 4 FMAs.  FMA-bound: w^2 N flops.
#include <algorithm>

#include "internal.h"

namespace mp {

namespace {

constexpr int CWS = 32;           // columns per CTA (one per lane)
constexpr int RB = 32;            // rows per warp block
constexpr int MAXB = 8;           // w <= MAXB * RB = 256
constexpr int LP = RB + 4;        // padded stride of a transposed L block (16-byte aligned rows)

template <typename T>
__device__ __forceinline__ void load_lt(const T *W, int64_t ldw, int64_t r, int64_t c, int nrows, int ncols,
                                        T *lt, int lane)
{
    // lt[kk * LP + i] = L(r + i, c + kk): lane kk reads column kk of rows i (coalesced row
    // segments); all 32 loads are issued before the first store (one memory round trip)
#pragma unroll
    for (int h = 0; h < RB; h += 16) {
        T v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
            v[i] = (h + i < nrows && lane < ncols) ? __ldg(W + (r + h + i) * ldw + c + lane) : T(0);
#pragma unroll
        for (int i = 0; i < 16; ++i) lt[lane * LP + h + i] = v[i];
    }
}

template <int BYTES>
__device__ __forceinline__ void cp_async(uint32_t dst, const void *src, bool ok)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(dst), "l"(src), "n"(BYTES), "r"(ok ? BYTES : 0)
                 : "memory");
}

// L: top-left of the unit-lower w x w block (row-major, ldl); X: top-left of the w x ncols target.
// The lower-triangular blocks of L are staged ONCE per CTA, transposed, with cp.async (every
// element in flight at once, no register staging), so the warp chain below never waits on
// global memory: Lt[tri(b, k)][kk][i] = L(32b + i, 32k + kk), tri(b, k) = b(b+1)/2 + k.
template <typename T>
__global__ void __launch_bounds__(MAXB * 32, 1)
trsm_lower_unit_kernel(const T *L, int64_t ldl, T *__restrict__ X, int64_t ldx, int w, int64_t ncols)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    pdl_trigger();
    const int nb = (w + RB - 1) / RB;
    const int lane = threadIdx.x & 31, b = threadIdx.x >> 5;
    T *Xs = reinterpret_cast<T *>(smem_raw);                  // [nb][RB][CWS] published row blocks
    T *Lt = Xs + (size_t)nb * RB * CWS;                       // [nb(nb+1)/2][RB][LP] transposed L blocks
    const int ntri = nb * (nb + 1) / 2;
    volatile int *flag = reinterpret_cast<volatile int *>(Lt + (size_t)ntri * RB * LP);   // [nb]
    if (threadIdx.x < MAXB) flag[threadIdx.x] = 0;
    // ---- stage: thread -> (row i, column kk) of a block, consecutive threads along kk (coalesced)
    for (int bb = 0; bb < nb; ++bb)
        for (int kb = 0; kb <= bb; ++kb) {
            const int t = bb * (bb + 1) / 2 + kb;
            const uint32_t base = (uint32_t)__cvta_generic_to_shared(Lt + (size_t)t * RB * LP);
            for (int e = threadIdx.x; e < RB * RB; e += blockDim.x) {
                const int i = e >> 5, kk = e & 31;
                const int gr = bb * RB + i, gc = kb * RB + kk;
                const bool ok = gr < w && gc < w && (kb < bb || kk < i);
                cp_async<(int)sizeof(T)>(base + (uint32_t)(kk * LP + i) * sizeof(T),
                                         L + (int64_t)(ok ? gr : 0) * ldl + (ok ? gc : 0), ok);
            }
        }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (b >= nb) return;
    const int64_t col = (int64_t)blockIdx.x * CWS + lane;
    const bool cvalid = col < ncols;
    const int rows = (w - b * RB < RB) ? (w - b * RB) : RB;   // rows of this block
    const int64_t rb0 = (int64_t)b * RB;                       // block row offset inside L / X

    T x[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) x[i] = (cvalid && i < rows) ? X[(rb0 + i) * ldx + col] : T(0);

    // contributions of the earlier row blocks, in the order they are published
    for (int k = 0; k < b; ++k) {
        const T *lt = Lt + (size_t)(b * (b + 1) / 2 + k) * RB * LP;   // L(b, k)
        while (flag[k] == 0) { }
        __threadfence_block();
        __syncwarp();
        const T *xk = Xs + (size_t)k * RB * CWS;
#pragma unroll 4
        for (int kk = 0; kk < RB; ++kk) {
            const T xv = xk[kk * CWS + lane];
            const T *lc = lt + kk * LP;
#pragma unroll
            for (int i = 0; i < RB; i += 4) {
                x[i] = fma(-lc[i], xv, x[i]);
                x[i + 1] = fma(-lc[i + 1], xv, x[i + 1]);
                x[i + 2] = fma(-lc[i + 2], xv, x[i + 2]);
                x[i + 3] = fma(-lc[i + 3], xv, x[i + 3]);
            }
        }
        __syncwarp();
    }
    // the 32 x 32 unit-lower diagonal block (strictly lower part staged; zeros elsewhere)
    {
        const T *lt = Lt + (size_t)(b * (b + 1) / 2 + b) * RB * LP;
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const T *lc = lt + i * LP;
#pragma unroll
            for (int m = i + 1; m < RB; ++m) x[m] = fma(-lc[m], x[i], x[m]);
        }
    }
    // publish X_b (shared, for later blocks) and store U12 rows
    T *xb = Xs + (size_t)b * RB * CWS;
#pragma unroll
    for (int i = 0; i < RB; ++i) xb[i * CWS + lane] = x[i];
    __threadfence_block();
    __syncwarp();
    if (lane == 0) flag[b] = 1;
#pragma unroll
    for (int i = 0; i < RB; ++i)
        if (cvalid && i < rows) X[(rb0 + i) * ldx + col] = x[i];
}

}  // namespace

template <typename T>
size_t trsm_smem(int w)
{
    const int nb = (w + RB - 1) / RB;
    return ((size_t)nb * RB * CWS + (size_t)(nb * (nb + 1) / 2) * RB * LP) * sizeof(T) + MAXB * sizeof(int) + 16;
}

template <typename T>
void launch_trsm_ops(const T *L, int64_t ldl, T *X, int64_t ldx, int w, int64_t ncols, cudaStream_t s)
{
    if (ncols <= 0 || w <= 0) return;
    if (w > MAXB * RB) throw CudaError{cudaErrorInvalidValue, "trsm block wider than 256", __LINE__};
    constexpr int WMAX = sizeof(T) == 4 ? 256 : 128;          // staged triangle must fit shared memory
    if (w > WMAX) {                                            // [L11 0; L21 L22]: X1, X2 -= L21 X1, X2
        const int w1 = WMAX;
        launch_trsm_ops<T>(L, ldl, X, ldx, w1, ncols, s);
        launch_gemm_ops<T>(L + (int64_t)w1 * ldl, ldl, X, ldx, X + (int64_t)w1 * ldx, ldx, w - w1, ncols, w1, s);
        launch_trsm_ops<T>(L + (int64_t)w1 * ldl + w1, ldl, X + (int64_t)w1 * ldx, ldx, w - w1, ncols, s);
        return;
    }
    const int nb = (w + RB - 1) / RB;
    const int grid = (int)ceil_div(ncols, CWS);
    auto kern = trsm_lower_unit_kernel<T>;
    func_smem_once((const void *)kern, trsm_smem<T>(WMAX));   // the largest request, set once
    launch_ex(kern, dim3(grid), dim3(nb * 32), trsm_smem<T>(w), s, nullptr, L, ldl, X, ldx, w, ncols);
}

template <typename T>
void launch_trsm_lower_unit(T *W, int64_t ldw, int64_t r0, int w, int64_t c_lo, int64_t c_hi, cudaStream_t s)
{
    launch_trsm_ops<T>(W + r0 * ldw + r0, ldw, W + r0 * ldw + c_lo, ldw, w, c_hi - c_lo, s);
}

template void launch_trsm_ops<float>(const float *, int64_t, float *, int64_t, int, int64_t, cudaStream_t);
template void launch_trsm_ops<double>(const double *, int64_t, double *, int64_t, int, int64_t, cudaStream_t);
template void launch_trsm_lower_unit<float>(float *, int64_t, int64_t, int, int64_t, int64_t, cudaStream_t);
template void launch_trsm_lower_unit<double>(double *, int64_t, int64_t, int, int64_t, int64_t, cudaStream_t);

}  // namespace mp
