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
//  * G7 gmres_sp_cycle_kernel  the whole binary32 GMRES_SP(m_in) cycle as ONE persistent cooperative kernel
//                            (one CTA of 1024 threads per SM, 1 + 3 m_in grid barriers): each CTA owns a
//                            contiguous block of rows; per Arnoldi step it stages x = V_j in shared memory,
//                            streams its rows of W (the HBM-bound part), and runs both classical
//                            Gram-Schmidt passes, the norm and the Givens rotation on its rows, exchanging
//                            only 32-float partial sums per CTA through global memory (every CTA reduces them
//                            itself in the same fixed order, so all CTAs hold the same Hessenberg column).
//                            The least-squares state lives in shared memory; z = V y is written in binary64
//                            (the outer solver's Z_k).  Replaces ~12 launches per Arnoldi step of G1-G6.
// Deterministic: every reduction has a fixed order.
#include <algorithm>
#include <cstdlib>

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


// ---------------------------------------------------------------- G7: the cooperative GMRES_SP cycle
constexpr int CT = 1024;             // threads per CTA
constexpr int CW = CT / 32;
#ifndef MP_G7_SEG4
#define MP_G7_SEG4 1024
#endif
#ifndef MP_G7_GU
#define MP_G7_GU 4
#endif
#ifndef MP_G7_LD
#define MP_G7_LD 2
#endif
__device__ __forceinline__ float4 ld_stream(const float4 *p)
{
#if MP_G7_LD == 0
    return __ldcs(p);
#elif MP_G7_LD == 1
    return __ldg(p);
#else
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
#endif
}
constexpr int SEG4 = MP_G7_SEG4;     // float4 per gemv work unit (4096 columns of one row)
constexpr int GU = MP_G7_GU;         // loads in flight per lane

struct SpCycle {
    const float *W;                  // row-major binary32 copy of A, ldw (multiple of 4), zero padded
    int64_t ldw, n;
    const float *v;                  // the right-hand side v_k (binary32)
    float *V;                        // normalised basis columns 0..m-1 (ld ldv)
    int64_t ldv;
    float *raw;                      // 2 x ldv: unnormalised w_{j+1} (ping-pong)
    double *z;                       // output z = V y (binary64)
    float *part;                     // 3 x gridDim.x x 32 partial sums
    unsigned *bar;                   // grid barrier counter (zeroed before the launch)
    int m, nseg;
    int64_t rpb;                     // rows per CTA
};

__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned &target)
{
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
        __threadfence();
    }
    __syncthreads();
}

// part[blockIdx.x * 32 + l] = sum over this CTA's rows of f(l, r), l < k (fixed order: rows by thread, then a
// butterfly per warp, then warps in order)
template <typename F>
__device__ __forceinline__ void cta_partials(int k, int64_t cnt, float *red, float *part, F f)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int l = 0; l < k; ++l) {
        float a = 0.f;
        for (int64_t r = threadIdx.x; r < cnt; r += CT) a += f(l, r);
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) red[warp * 32 + l] = a;
    }
    __syncthreads();
    if (threadIdx.x < k) {
        float a = 0.f;
        for (int w = 0; w < CW; ++w) a += red[w * 32 + threadIdx.x];
        part[(int64_t)blockIdx.x * 32 + threadIdx.x] = a;
    }
}

// out[l] = sum over CTAs of part[b * 32 + l], l < k: every CTA computes the same value (warp l, fixed order)
__device__ __forceinline__ void grid_reduce(int k, const float *part, float *out)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp < k) {
        float a = 0.f;
        for (unsigned b = lane; b < gridDim.x; b += 32) a += __ldcg(part + (int64_t)b * 32 + warp);
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) out[warp] = a;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(CT, 1) gmres_sp_cycle_kernel(const SpCycle a)
{
    extern __shared__ __align__(16) float sm[];
    const int64_t n = a.n, n4 = ceil_div(n, (int64_t)4);
    float *xs = sm;                                       // [4 n4]  x = V_j
    float *seg = xs + 4 * n4;                             // [rpb][nseg] gemv unit sums
    float *wv = seg + a.rpb * a.nseg;                     // [rpb]   w on this CTA's rows
    float *red = wv + a.rpb;                              // [CW][32]
    float *R = red + CW * 32;                             // [(m+1) m]
    float *cs = R + 33 * 32, *sn = cs + 32, *g = sn + 32, *y = g + 33, *h1 = y + 32, *h2 = h1 + 32, *hv = h2 + 32;
    float *sc = hv + 32;                                  // [0] inverse of the current norm, [1] scratch
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = a.m;
    const int64_t row0 = (int64_t)blockIdx.x * a.rpb;
    const int64_t cnt = row0 < n ? min(a.rpb, n - row0) : 0;
    unsigned target = 0;
    float *P[3] = {a.part, a.part + (int64_t)gridDim.x * 32, a.part + (int64_t)gridDim.x * 64};
    // ---- beta = ||v||, V_0 = v / beta, g = beta e_1
    cta_partials(1, cnt, red, P[2], [&](int, int64_t r) { const float t = a.v[row0 + r]; return t * t; });
    grid_sync(a.bar, target);
    grid_reduce(1, P[2], h1);
    if (threadIdx.x == 0) {
        const float beta = sqrtf(h1[0]);
        for (int i = 0; i <= m; ++i) g[i] = i == 0 ? beta : 0.f;
        sc[0] = beta == 0.f ? 0.f : 1.f / beta;
    }
    __syncthreads();
    const float *xsrc = a.v;
    for (int j = 0; j < m; ++j) {
        // ---- phase a: x = V_j (staged), w = W x on this CTA's rows, pass-1 dots V_l . w
        const float inv = sc[0];
        for (int64_t t = threadIdx.x; t < n4; t += CT) {
            float4 q;
            if (4 * t + 3 < n) {
                q = __ldcg(reinterpret_cast<const float4 *>(xsrc) + t);
            } else {
                q.x = 4 * t < n ? __ldcg(xsrc + 4 * t) : 0.f;
                q.y = 4 * t + 1 < n ? __ldcg(xsrc + 4 * t + 1) : 0.f;
                q.z = 4 * t + 2 < n ? __ldcg(xsrc + 4 * t + 2) : 0.f;
                q.w = 0.f;
            }
            q.x *= inv; q.y *= inv; q.z *= inv; q.w *= inv;
            reinterpret_cast<float4 *>(xs)[t] = q;
        }
        __syncthreads();
        float *Vj = a.V + (int64_t)j * a.ldv;
        for (int64_t r = threadIdx.x; r < cnt; r += CT) Vj[row0 + r] = xs[row0 + r];
        const float4 *x4 = reinterpret_cast<const float4 *>(xs);
        const int64_t units = cnt * a.nseg;
        for (int64_t u = warp; u < units; u += CW) {
            const int64_t r = u / a.nseg, sg = u - r * a.nseg;
            const float4 *w4 = reinterpret_cast<const float4 *>(a.W + (row0 + r) * a.ldw);
            const int64_t c0 = sg * SEG4, c1 = min(n4, c0 + SEG4);
            float s0 = 0.f, s1 = 0.f;
            int64_t c = c0 + lane;
            for (; c + 32 * (GU - 1) < c1; c += 32 * GU) {        // GU independent 16-byte loads in flight
                float4 p[GU];
#pragma unroll
                for (int k = 0; k < GU; ++k) p[k] = ld_stream(w4 + c + 32 * k);
#pragma unroll
                for (int k = 0; k < GU; ++k) {
                    const float4 q = x4[c + 32 * k];
                    float &t = (k & 1) ? s1 : s0;
                    t = fmaf(p[k].x, q.x, t); t = fmaf(p[k].y, q.y, t); t = fmaf(p[k].z, q.z, t); t = fmaf(p[k].w, q.w, t);
                }
            }
            for (; c < c1; c += 32) {
                const float4 p0 = ld_stream(w4 + c), q0 = x4[c];
                s0 = fmaf(p0.x, q0.x, s0); s0 = fmaf(p0.y, q0.y, s0); s0 = fmaf(p0.z, q0.z, s0); s0 = fmaf(p0.w, q0.w, s0);
            }
            float sum = s0 + s1;
            for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (lane == 0) seg[r * a.nseg + sg] = sum;
        }
        __syncthreads();
        for (int64_t r = threadIdx.x; r < cnt; r += CT) {
            float w = 0.f;
            for (int q = 0; q < a.nseg; ++q) w += seg[r * a.nseg + q];
            wv[r] = w;
        }
        __syncthreads();
        cta_partials(j + 1, cnt, red, P[0], [&](int l, int64_t r) {
            const float vl = l == j ? xs[row0 + r] : a.V[(int64_t)l * a.ldv + row0 + r];
            return vl * wv[r];
        });
        grid_sync(a.bar, target);
        // ---- phase b: h1 = V^T w; w -= V h1; pass-2 dots
        grid_reduce(j + 1, P[0], h1);
        for (int64_t r = threadIdx.x; r < cnt; r += CT) {
            float w = wv[r];
            for (int l = 0; l <= j; ++l) w = fmaf(-h1[l], a.V[(int64_t)l * a.ldv + row0 + r], w);
            wv[r] = w;
        }
        __syncthreads();
        cta_partials(j + 1, cnt, red, P[1],
                     [&](int l, int64_t r) { return a.V[(int64_t)l * a.ldv + row0 + r] * wv[r]; });
        grid_sync(a.bar, target);
        // ---- phase c: h2; w -= V h2; ||w||^2; w published for the next step's x
        grid_reduce(j + 1, P[1], h2);
        float *rawn = a.raw + (int64_t)(j & 1) * a.ldv;
        for (int64_t r = threadIdx.x; r < cnt; r += CT) {
            float w = wv[r];
            for (int l = 0; l <= j; ++l) w = fmaf(-h2[l], a.V[(int64_t)l * a.ldv + row0 + r], w);
            wv[r] = w;
            rawn[row0 + r] = w;
        }
        __syncthreads();
        cta_partials(1, cnt, red, P[2], [&](int, int64_t r) { return wv[r] * wv[r]; });
        grid_sync(a.bar, target);
        // ---- phase d: h_{j+1,j}; the Givens rotation (every CTA, identical)
        grid_reduce(1, P[2], sc + 1);
        if (threadIdx.x == 0) {
            const float hn = sqrtf(sc[1]);
            float *col = R + j * (m + 1);
            for (int i = 0; i <= j; ++i) col[i] = h1[i] + h2[i];
            col[j + 1] = hn;
            for (int i = 0; i < j; ++i) {
                const float p = col[i], q = col[i + 1];
                col[i] = cs[i] * p + sn[i] * q;
                col[i + 1] = -sn[i] * p + cs[i] * q;
            }
            const float p = col[j], q = col[j + 1];
            float c = 1.f, s = 0.f;
            if (q != 0.f) {
                const float rr = sqrtf(p * p + q * q);
                c = p / rr;
                s = q / rr;
            }
            cs[j] = c;
            sn[j] = s;
            col[j] = c * p + s * q;
            col[j + 1] = 0.f;
            g[j + 1] = -s * g[j];
            g[j] = c * g[j];
            hv[j] = hn;
            sc[0] = hn == 0.f ? 0.f : 1.f / hn;
        }
        __syncthreads();
        xsrc = rawn;
    }
    // ---- y = R^-1 g (up to the first exact breakdown), z = V y in binary64
    if (threadIdx.x == 0) {
        int steps = m;
        for (int i = 0; i < m; ++i)
            if (hv[i] == 0.f) { steps = i + 1; break; }
        for (int i = steps; i < m; ++i) y[i] = 0.f;
        for (int i = steps - 1; i >= 0; --i) {
            float t = g[i];
            for (int l = i + 1; l < steps; ++l) t = t - R[i + l * (m + 1)] * y[l];
            const float d = R[i + i * (m + 1)];
            y[i] = d == 0.f ? 0.f : t / d;
        }
    }
    __syncthreads();
    for (int64_t r = threadIdx.x; r < cnt; r += CT) {
        float t = 0.f;
        for (int l = 0; l < m; ++l) t = fmaf(y[l], a.V[(int64_t)l * a.ldv + row0 + r], t);
        a.z[row0 + r] = (double)t;
    }
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


// ---------------------------------------------------------------- G7 host side
size_t sp_cycle_smem(int64_t n, int sms, int64_t *rpb_out, int *nseg_out)
{
    const int64_t n4 = ceil_div(n, (int64_t)4);
    const int64_t rpb = ceil_div(n, (int64_t)sms);
    const int nseg = (int)ceil_div(n4, (int64_t)SEG4);
    if (rpb_out) *rpb_out = rpb;
    if (nseg_out) *nseg_out = nseg;
    return sizeof(float) * (size_t)(4 * n4 + rpb * nseg + rpb + CW * 32 + 33 * 32 + 32 * 8 + 8);
}

size_t sp_cycle_part_elems(int sms) { return (size_t)3 * sms * 32; }

bool sp_cycle_supported(int64_t n, int sms)
{
    static const bool off = std::getenv("MP_GMRES_NO_COOP") != nullptr;
    if (off || n < 1) return false;
    int dev = 0, coop = 0, maxsm = 0;
    MP_CUDA(cudaGetDevice(&dev));
    MP_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    MP_CUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    return coop && sp_cycle_smem(n, sms, nullptr, nullptr) <= (size_t)maxsm;
}

void launch_gmres_sp_cycle(const float *W, int64_t ldw, int64_t n, const float *v, float *V, int64_t ldv, float *raw,
                           double *z, int m, float *part, unsigned *bar, int sms, cudaStream_t s)
{
    if ((ldw % 4) || (reinterpret_cast<uintptr_t>(W) & 15) || (ldv % 4) || (reinterpret_cast<uintptr_t>(v) & 15) ||
        (reinterpret_cast<uintptr_t>(raw) & 15))
        throw CudaError{cudaErrorInvalidValue, "gmres_sp_cycle: 16-byte aligned rows required", __LINE__};
    SpCycle a{W, ldw, n, v, V, ldv, raw, z, part, bar, m, 0, 0};
    const size_t smem = sp_cycle_smem(n, sms, &a.rpb, &a.nseg);
    func_smem_once((const void *)gmres_sp_cycle_kernel, smem);
    MP_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), s));
    void *args[] = {&a};
    MP_CUDA(cudaLaunchCooperativeKernel((const void *)gmres_sp_cycle_kernel, dim3(sms), dim3(CT), args, smem, s));
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
