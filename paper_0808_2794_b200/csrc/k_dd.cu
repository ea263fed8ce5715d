// k_dd.cu — the extended-precision refinement of SURVEY §8(f) NEXT-4
// ("Extension to Quadruple Precision": QDGESV = DGETRF + DGETRS + a quadruple-precision residual
// QGEMV and update), with quadruple precision carried as double-double (reading Q-0).
//
//  * Q1 dd_residual_partial_kernel  split-K partial sums of A (xh + xl) in double-double; A is read
//                                   once per residual with coalesced 16-byte loads (8 n^2 B).  Per
//                                   entry: TwoProd(xh, a) (FMA) + a xl, and one double-double add,
//                                   ~20 binary64 flops per 8 bytes: still below the FP64 ridge
//                                   (37.1 TF/s / 6.5 TB/s = 5.7 flop/B), so HBM-bound.  The paper
//                                   notes QGEMV dominated its QDGESV (T7).
//  * Q2 dd_residual_finalize_kernel  fixed-order double-double sum of the partials, r = b - A x in
//                                   double-double, y = fl64(P r) for the binary64 solve, the norms
//                                   and the stop test (reading Q-1) on the device.
//  * Q3 dd_update_kernel            x = x + z in double-double (step 7 carried in extended precision).
// The binary64 factorisation and solves are the mp_dgesv kernels.
#include <algorithm>

#include "internal.h"

namespace mp {

namespace {

struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b)
{
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b)
{
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b)
{
    const double p = __dmul_rn(a, b);
    return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b)
{
    dd s = two_sum(a.hi, b.hi);
    const dd t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}
// a * (xh + xl) as a double-double
__device__ __forceinline__ dd dd_mul_d(double xh, double xl, double a)
{
    dd p = two_prod(xh, a);
    p.lo = __dadd_rn(p.lo, __dmul_rn(xl, a));
    return quick_two_sum(p.hi, p.lo);
}

constexpr int RT = 256;          // threads, 2 rows each
constexpr int ROWS = 2 * RT;
constexpr int JU = 8;

__global__ void __launch_bounds__(RT)
dd_residual_partial_kernel(const double *__restrict__ A, int64_t lda, int64_t n, const double *__restrict__ xh,
                           const double *__restrict__ xl, double *__restrict__ ph, double *__restrict__ pl,
                           int64_t cols_per_split)
{
    extern __shared__ __align__(16) double xs[];     // [cols_per_split][2]
    const int s = blockIdx.y;
    const int64_t j0 = (int64_t)s * cols_per_split, j1 = std::min<int64_t>(n, j0 + cols_per_split);
    for (int64_t t = threadIdx.x; t < j1 - j0; t += RT) {
        xs[2 * t] = xh[j0 + t];
        xs[2 * t + 1] = xl[j0 + t];
    }
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * ROWS + 2 * threadIdx.x;
    const bool r0 = i < n, r1 = i + 1 < n;
    const bool vec = r1 && (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    dd s0{0.0, 0.0}, s1{0.0, 0.0};
    int64_t j = j0;
    if (vec) {
        for (; j + JU <= j1; j += JU) {
            double2 a[JU];
#pragma unroll
            for (int u = 0; u < JU; ++u) a[u] = __ldcs(reinterpret_cast<const double2 *>(A + (j + u) * lda + i));
#pragma unroll
            for (int u = 0; u < JU; ++u) {
                const double h = xs[2 * (j + u - j0)], l = xs[2 * (j + u - j0) + 1];
                s0 = dd_add(s0, dd_mul_d(h, l, a[u].x));
                s1 = dd_add(s1, dd_mul_d(h, l, a[u].y));
            }
        }
    }
    for (; j < j1; ++j) {
        const double *col = A + j * lda;
        const double a0 = r0 ? __ldcs(col + i) : 0.0, a1 = r1 ? __ldcs(col + i + 1) : 0.0;
        const double h = xs[2 * (j - j0)], l = xs[2 * (j - j0) + 1];
        s0 = dd_add(s0, dd_mul_d(h, l, a0));
        s1 = dd_add(s1, dd_mul_d(h, l, a1));
    }
    if (r0) { ph[s * n + i] = s0.hi; pl[s * n + i] = s0.lo; }
    if (r1) { ph[s * n + i + 1] = s1.hi; pl[s * n + i + 1] = s1.lo; }
}

constexpr int FT = 256;

__global__ void __launch_bounds__(FT)
dd_residual_finalize_kernel(int64_t n, int splits, const double *__restrict__ ph, const double *__restrict__ pl,
                            const double *__restrict__ b, const double *__restrict__ xh, double *__restrict__ rh,
                            double *__restrict__ rl, const int32_t *__restrict__ pinv, double *__restrict__ y,
                            double *blocksums, unsigned *counter, double cte, DevStatus *st, int col, int ncols)
{
    __shared__ double red[FT / 32][2];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * FT + threadIdx.x;
    double rr = 0.0, xx = 0.0;
    if (i < n) {
        dd sum{0.0, 0.0};
        for (int s = 0; s < splits; ++s) sum = dd_add(sum, dd{ph[(int64_t)s * n + i], pl[(int64_t)s * n + i]});
        const dd r = dd_add(dd{b[i], 0.0}, dd{-sum.hi, -sum.lo});
        rh[i] = r.hi;
        rl[i] = r.lo;
        y[pinv[i]] = r.hi;                       // fl64(P r): the normalised head is the rounded value
        rr = r.hi * r.hi;
        xx = xh[i] * xh[i];
    }
    for (int o = 16; o; o >>= 1) {
        rr += __shfl_xor_sync(0xffffffffu, rr, o);
        xx += __shfl_xor_sync(0xffffffffu, xx, o);
    }
    if (lane == 0) { red[warp][0] = rr; red[warp][1] = xx; }
    __syncthreads();
    if (threadIdx.x < 2) {
        double v = 0.0;
        for (int w = 0; w < FT / 32; ++w) v += red[w][threadIdx.x];
        blocksums[2 * blockIdx.x + threadIdx.x] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    double r2 = 0.0, x2 = 0.0;
    for (unsigned k = 0; k < gridDim.x; ++k) {
        r2 += __ldcg(blocksums + 2 * k);
        x2 += __ldcg(blocksums + 2 * k + 1);
    }
    const double rn = sqrt(r2), xn = sqrt(x2);
    if (col < 16) { st->rn[col] = rn; st->xn[col] = xn; }
    *counter = 0u;
    // the verdict over all columns: column 0 initialises, later columns AND in / max in (reading Q-1)
    const bool bad = !isfinite(rn) || !isfinite(xn);
    const double ratio = rn == 0.0 ? 0.0 : rn / (xn * cte);
    const int conv = !bad && (rn < xn * cte || rn == 0.0);
    if (col == 0) {
        st->converged = conv;
        st->ratio = bad ? 0.0 : ratio;
    } else {
        st->converged = st->converged && conv;
        if (!bad && ratio > st->ratio) st->ratio = ratio;
    }
    if (bad) atomicOr(&st->flags, (int)ST_NORM_NONFINITE);
    (void)ncols;
}

__global__ void dd_update_kernel(double *__restrict__ xh, double *__restrict__ xl, const double *__restrict__ z,
                                 int64_t count)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        const dd x = dd_add(dd{xh[t], xl[t]}, dd{z[t], 0.0});
        xh[t] = x.hi;
        xl[t] = x.lo;
    }
}

int64_t dd_splits(int64_t n, int num_sms)
{
    const int64_t tiles = ceil_div(n, ROWS);
    int64_t s = ceil_div((int64_t)num_sms * 8, tiles);
    s = std::max<int64_t>(s, ceil_div(n * 2 * (int64_t)sizeof(double), 64 * 1024));   // x slice <= 64 KB
    return std::max<int64_t>(1, std::min<int64_t>(s, ceil_div(n, 64)));
}

}  // namespace

size_t dd_scratch_doubles(int64_t n, int num_sms)
{
    return (size_t)2 * dd_splits(n, num_sms) * n + (size_t)2 * ceil_div(n, FT) + 64;
}

// r = b - A x (double-double) for every right-hand side; y = fl64(P r); the verdict into st.
void launch_dd_residual(const double *A, int64_t lda, int64_t n, int64_t nrhs, const double *B, const double *Xh,
                        const double *Xl, double *Rh, double *Rl, const int32_t *pinv, double *Y, double cte,
                        double *scratch, unsigned *counter, DevStatus *st, int num_sms, cudaStream_t s)
{
    const int64_t splits = dd_splits(n, num_sms);
    const int64_t cps = ceil_div(n, splits);
    const int64_t real = ceil_div(n, cps);
    double *ph = scratch, *pl = scratch + (size_t)real * n, *bs = pl + (size_t)real * n;
    const size_t smem = (size_t)cps * 2 * sizeof(double);
    if (smem > 48 * 1024) func_smem_once((const void *)dd_residual_partial_kernel, smem);
    for (int64_t c = 0; c < nrhs; ++c) {
        dd_residual_partial_kernel<<<dim3((unsigned)ceil_div(n, ROWS), (unsigned)real), RT, smem, s>>>(
            A, lda, n, Xh + c * n, Xl + c * n, ph, pl, cps);
        MP_LAUNCH_CHECK();
        dd_residual_finalize_kernel<<<(unsigned)ceil_div(n, FT), FT, 0, s>>>(
            n, (int)real, ph, pl, B + c * n, Xh + c * n, Rh + c * n, Rl + c * n, pinv, Y + c * n, bs, counter, cte,
            st, (int)c, (int)nrhs);
        MP_LAUNCH_CHECK();
        g_launches += 2;
    }
}

void launch_dd_update(double *Xh, double *Xl, const double *Z, int64_t count, cudaStream_t s)
{
    dd_update_kernel<<<(unsigned)std::min<int64_t>(ceil_div(count, 256), 4096), 256, 0, s>>>(Xh, Xl, Z, count);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

}  // namespace mp
