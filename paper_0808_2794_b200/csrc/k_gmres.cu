// k_gmres.cu — SURVEY §8(f) NEXT-3: PAPER.md Algorithm 2, inner-outer
// FGMRES(m_out)-GMRES_SP(m_in): the outer FGMRES in binary64 with the original A, every
// "preconditioner" application one cycle of GMRES in binary32 with the binary32 copy of A (P:231-235:
// "we use single precision arithmetic matrix-vector product as a fast approximation of the double
// precision operator in the inner iterative solver").
//
// The hot operations are matrix-vector products with a dense operator (HBM-bound: 4 n^2 bytes for the
// binary32 one, 8 n^2 for the binary64 one, the latter with the residual kernel K8) and the Krylov basis
// work (Gram-Schmidt, norms, combinations: O(n m) bytes).  Kernels here:
//  * G1 gemv_rows_f32        y = W x, W the row-major binary32 working copy (a warp per row, 16-byte loads)
//  * G2 multidot / reduce    h_i = V_i . w for i < k at once (fixed-order two-level reduction)
//  * G3 combine              w = alpha w + sum_i beta h_i V_i  (w -= V h, z = V y, x += Z y)
//  * G4 givens_step          one Hessenberg column: previous rotations, the new one, g; 1/h_{j+1,j}
//  * G5 backsolve            y = R^-1 g (the least-squares solution)
//  * G6 scale_copy           V_{j+1} = w / h_{j+1,j} (and the binary64 -> binary32 demotion of v_k)
// Deterministic: every reduction has a fixed order.
#include <algorithm>

#include "internal.h"

namespace mp {

namespace {

constexpr int GT = 256;

__global__ void __launch_bounds__(GT) gemv_rows_f32_kernel(const float *__restrict__ W, int64_t ldw, int64_t n,
                                                           const float *__restrict__ x, float *__restrict__ y)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n4 = n / 4;
    for (int64_t i = (int64_t)blockIdx.x * (GT / 32) + warp; i < n; i += (int64_t)gridDim.x * (GT / 32)) {
        const float *row = W + i * ldw;
        float s = 0.f;
        for (int64_t c = lane; c < n4; c += 32) {
            const float4 a = __ldcs(reinterpret_cast<const float4 *>(row) + c);
            const float4 v = __ldg(reinterpret_cast<const float4 *>(x) + c);
            s = fmaf(a.x, v.x, s); s = fmaf(a.y, v.y, s); s = fmaf(a.z, v.z, s); s = fmaf(a.w, v.w, s);
        }
        for (int64_t c = 4 * n4 + lane; c < n; c += 32) s = fmaf(row[c], x[c], s);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) y[i] = s;
    }
}

// partial[b * k + i] = sum over the rows of block b of V[r + i ldv] w[r]   (k <= 32)
template <typename T>
__global__ void __launch_bounds__(GT) multidot_kernel(const T *__restrict__ V, int64_t ldv, int k,
                                                      const T *__restrict__ w, int64_t n, int64_t rows_per_block,
                                                      T *__restrict__ partial)
{
    __shared__ T red[GT / 32][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_block, r1 = min(n, r0 + rows_per_block);
    T acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = T(0);
    for (int64_t r = r0 + threadIdx.x; r < r1; r += GT) {
        const T wr = w[r];
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (i < k) acc[i] = fma(V[r + i * ldv], wr, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        if (i < k) {
            T v = acc[i];
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) red[warp][i] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x < k) {
        T v = T(0);
        for (int wp = 0; wp < GT / 32; ++wp) v += red[wp][threadIdx.x];
        partial[(int64_t)blockIdx.x * k + threadIdx.x] = v;
    }
}

// out[i] (+)= sum_b partial[b k + i], fixed order; accumulate: add to out (the second CGS pass)
template <typename T>
__global__ void reduce_partials_kernel(const T *__restrict__ partial, int nblocks, int k, T *__restrict__ out,
                                       int accumulate)
{
    const int i = threadIdx.x;
    if (i >= k) return;
    T v = T(0);
    for (int b = 0; b < nblocks; ++b) v += partial[(int64_t)b * k + i];
    out[i] = accumulate ? out[i] + v : v;
}

// w[r] = alpha w[r] + beta sum_{i<k} coef[i] V[r + i ldv]; coef on the device
template <typename T>
__global__ void combine_kernel(T *__restrict__ w, const T *__restrict__ V, int64_t ldv, int k,
                               const T *__restrict__ coef, T alpha, T beta, int64_t n)
{
    __shared__ T c[32];
    if (threadIdx.x < k) c[threadIdx.x] = coef[threadIdx.x];
    __syncthreads();
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        T s = alpha == T(0) ? T(0) : alpha * w[r];
        for (int i = 0; i < k; ++i) s = fma(beta * c[i], V[r + i * ldv], s);
        w[r] = s;
    }
}

// V_{j+1}[r] = w[r] * scale[0] (T) ; optionally its binary32 demotion into vs (the inner right-hand side)
template <typename T, typename TS>
__global__ void scale_copy_kernel(const T *__restrict__ w, const T *__restrict__ scale, int invert, T *__restrict__ out,
                                  TS *__restrict__ outs, int64_t n)
{
    const T s0 = scale[0];
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        // v = w / h (IEEE division, as the oracle); h == 0 (an exact breakdown): a zero vector, which the
        // back-substitution then leaves out (reading G-4)
        const T v = invert ? (s0 == T(0) ? T(0) : w[r] / s0) : w[r] * s0;
        if (out) out[r] = v;
        if (outs) outs[r] = (TS)v;
    }
}

// One Hessenberg column j: hcol[0..j] (the Gram-Schmidt coefficients) and hnorm2 = ||w||^2 in, the
// previous rotations applied, the new rotation, g updated; R column j stored (ld m + 1); hout[0] = h_{j+1,j}.
// Textbook Givens as the oracle (no scaling).  One thread.
template <typename T>
__global__ void givens_step_kernel(const T *__restrict__ hcol, const T *__restrict__ hnorm2, int j, int m,
                                   T *__restrict__ R, T *__restrict__ cs, T *__restrict__ sn, T *__restrict__ g,
                                   T *__restrict__ hout)
{
    if (threadIdx.x != 0) return;
    const T hn = sqrt(hnorm2[0]);
    T *col = R + (int64_t)j * (m + 1);
    for (int i = 0; i <= j; ++i) col[i] = hcol[i];
    col[j + 1] = hn;
    for (int i = 0; i < j; ++i) {
        const T a = col[i], b = col[i + 1];
        col[i] = cs[i] * a + sn[i] * b;
        col[i + 1] = -sn[i] * a + cs[i] * b;
    }
    const T a = col[j], b = col[j + 1];
    T c = T(1), s = T(0);
    if (b != T(0)) {
        const T r = sqrt(a * a + b * b);
        c = a / r;
        s = b / r;
    }
    cs[j] = c;
    sn[j] = s;
    col[j] = c * a + s * b;
    col[j + 1] = T(0);
    g[j + 1] = -s * g[j];
    g[j] = c * g[j];
    hout[0] = hn;
}

// hn[i] = h_{i+1,i} of column i: a zero (exact breakdown) ends the basis after column i (reading G-4);
// y[i] = 0 beyond it
template <typename T>
__global__ void backsolve_kernel(const T *__restrict__ R, int m, int steps, const T *__restrict__ g, T *__restrict__ y,
                                 const T *__restrict__ hn)
{
    if (threadIdx.x != 0) return;
    if (hn)
        for (int i = 0; i < steps; ++i)
            if (hn[i] == T(0)) { steps = i + 1; break; }
    for (int i = steps; i < m; ++i) y[i] = T(0);
    for (int i = steps - 1; i >= 0; --i) {
        T s = g[i];
        for (int l = i + 1; l < steps; ++l) s = s - R[i + (int64_t)l * (m + 1)] * y[l];
        const T d = R[i + (int64_t)i * (m + 1)];
        y[i] = d == T(0) ? T(0) : s / d;        // a zero start vector (beta = 0): y = 0, not 0/0
    }
}

// beta = ||v||, g = (beta, 0, ...): the start of a cycle.  One warp.
template <typename T>
__global__ void cycle_start_kernel(const T *__restrict__ norm2, T *__restrict__ g, int m, T *__restrict__ beta)
{
    const T b = sqrt(norm2[0]);
    for (int i = threadIdx.x; i <= m; i += blockDim.x) g[i] = i == 0 ? b : T(0);
    if (threadIdx.x == 0) beta[0] = b;
}

__global__ void convert_f32_f64_kernel(const float *__restrict__ a, double *__restrict__ b, int64_t n)
{
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        b[r] = (double)a[r];
}

int grid_for(int64_t n) { return (int)std::min<int64_t>(ceil_div(n, GT), 1184); }
int dot_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 2048), 592)); }

}  // namespace

// ---------------------------------------------------------------- host launchers
void launch_gemv_rows_f32(const float *W, int64_t ldw, int64_t n, const float *x, float *y, cudaStream_t s)
{
    if ((ldw % 4) || (reinterpret_cast<uintptr_t>(W) & 15) || (reinterpret_cast<uintptr_t>(x) & 15))
        throw CudaError{cudaErrorInvalidValue, "gemv_rows_f32: 16-byte aligned rows required", __LINE__};
    gemv_rows_f32_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, GT / 32), 148 * 16), GT, 0, s>>>(W, ldw, n, x, y);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

size_t gmres_partial_elems(int64_t n) { return (size_t)dot_blocks(n) * 32; }

void launch_convert_f32_f64(const float *a, double *b, int64_t n, cudaStream_t s)
{
    convert_f32_f64_kernel<<<grid_for(n), GT, 0, s>>>(a, b, n);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template <typename T>
void launch_multidot(const T *V, int64_t ldv, int k, const T *w, int64_t n, T *partial, T *out, bool accumulate,
                     cudaStream_t s)
{
    const int nb = dot_blocks(n);
    const int64_t rpb = ceil_div(n, (int64_t)nb);
    multidot_kernel<T><<<nb, GT, 0, s>>>(V, ldv, k, w, n, rpb, partial);
    MP_LAUNCH_CHECK();
    reduce_partials_kernel<T><<<1, 32, 0, s>>>(partial, nb, k, out, accumulate ? 1 : 0);
    MP_LAUNCH_CHECK();
    g_launches += 2;
}

template <typename T>
void launch_combine(T *w, const T *V, int64_t ldv, int k, const T *coef, T alpha, T beta, int64_t n, cudaStream_t s)
{
    combine_kernel<T><<<grid_for(n), GT, 0, s>>>(w, V, ldv, k, coef, alpha, beta, n);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template <typename T, typename TS>
void launch_scale_copy(const T *w, const T *scale, bool invert, T *out, TS *outs, int64_t n, cudaStream_t s)
{
    scale_copy_kernel<T, TS><<<grid_for(n), GT, 0, s>>>(w, scale, invert ? 1 : 0, out, outs, n);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template <typename T>
void launch_givens_step(const T *hcol, const T *hnorm2, int j, int m, T *R, T *cs, T *sn, T *g, T *hout,
                        cudaStream_t s)
{
    givens_step_kernel<T><<<1, 32, 0, s>>>(hcol, hnorm2, j, m, R, cs, sn, g, hout);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template <typename T>
void launch_backsolve(const T *R, int m, int steps, const T *g, T *y, const T *hn, cudaStream_t s)
{
    backsolve_kernel<T><<<1, 32, 0, s>>>(R, m, steps, g, y, hn);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template <typename T>
void launch_cycle_start(const T *norm2, T *g, int m, T *beta, cudaStream_t s)
{
    cycle_start_kernel<T><<<1, 32, 0, s>>>(norm2, g, m, beta);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

#define INST(T)                                                                                                   \
    template void launch_multidot<T>(const T *, int64_t, int, const T *, int64_t, T *, T *, bool, cudaStream_t);  \
    template void launch_combine<T>(T *, const T *, int64_t, int, const T *, T, T, int64_t, cudaStream_t);        \
    template void launch_givens_step<T>(const T *, const T *, int, int, T *, T *, T *, T *, T *, cudaStream_t);   \
    template void launch_backsolve<T>(const T *, int, int, const T *, T *, const T *, cudaStream_t);              \
    template void launch_cycle_start<T>(const T *, T *, int, T *, cudaStream_t);
INST(float)
INST(double)
#undef INST
template void launch_scale_copy<float, float>(const float *, const float *, bool, float *, float *, int64_t,
                                              cudaStream_t);
template void launch_scale_copy<double, float>(const double *, const double *, bool, double *, float *, int64_t,
                                               cudaStream_t);
template void launch_scale_copy<double, double>(const double *, const double *, bool, double *, double *, int64_t,
                                                cudaStream_t);

}  // namespace mp
