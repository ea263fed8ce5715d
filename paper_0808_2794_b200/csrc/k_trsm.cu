// k_trsm.cu — K4: U12 <- L11^{-1} A12 (left, lower, unit diagonal).
//
// Blocked right-looking LU (SGETRF's blocked form): after a
// panel of width w is factored, its unit-lower block L11 is applied to the w
// rows of the columns to its right by forward SUBSTITUTION (no explicit
// inverse, so exact inputs stay exact — pin P2).
//
// One CTA per 32-column strip (see the kernel): the strip and the triangle of L11 are staged in
// shared memory once; per 32-row block, 8 warps subtract the previous block's contribution (older
// ones were subtracted during the previous diagonal solve) and a ninth warp solves the 32 x 32
// unit-lower diagonal block.  FMA work w^2 N; the chain is nb = w/32 links of (one 32x32x32
// contribution over 8 warps + one 32-step substitution).
#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace mp {

namespace {

constexpr int CWS = 32;           // columns per CTA (one per lane)
constexpr int RB = 32;            // rows per warp block
constexpr int MAXB = 8;           // w <= MAXB * RB = 256
constexpr int LP = RB + 4;        // padded stride of a transposed L block (16-byte aligned rows)
constexpr int TW = 9;             // warps per CTA: 8 updaters + 1 diagonal-block solver

__device__ __forceinline__ void named_bar_sync(int id, int count)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int BYTES>
__device__ __forceinline__ void cp_async(uint32_t dst, const void *src, bool ok)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(dst), "l"(src), "n"(BYTES), "r"(ok ? BYTES : 0)
                 : "memory");
}

// L: top-left of the unit-lower w x w block (row-major, ldl); X: top-left of the w x ncols target.
// One CTA per 32-column strip (lane = column), 9 warps.  The strip of X and the lower-triangular
// 32 x 32 blocks of L are staged ONCE with 16-byte cp.async (row-major, rows padded to LP:
// Ls[tri(b, k)][i][kk] = L(32b + i, 32k + kk), tri(b, k) = b(b+1)/2 + k).  Block b of the chain:
// warps 0-7 (4 rows each) subtract the contribution of block b-1 (the only one on the chain:
// older blocks were subtracted while the solver worked on block b-1), then warp 8 solves the
// 32 x 32 unit-lower diagonal block row by row (x_m -= sum_{i<m} l_mi x_i, four partial sums).
__device__ __forceinline__ float rna_tf32(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// sh/sl (binary32 only, optional): also write U12 split for the 3xTF32 update, transposed K-major
// (sh[j * kp + k] = rna_tf32(U12(k, j)), sl = rna_tf32(U12 - sh)) — split_cols_T_kernel's output
// CW = 16 (narrow column ranges: twice the CTAs): lanes l and l + 16 share column l & 15 and
// split each warp's 4 update rows (2 each); the solver's upper half-warp recomputes, writes nothing
template <typename T, int CW>
__global__ void __launch_bounds__(TW * 32, 1)
trsm_lower_unit_kernel(const T *L, int64_t ldl, T *__restrict__ X, int64_t ldx, int w, int64_t ncols,
                       float *__restrict__ sh, float *__restrict__ sl, int kp)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    pdl_trigger();
    constexpr int EPC = 16 / (int)sizeof(T);                  // elements per 16-byte chunk
    const int nb = (w + RB - 1) / RB;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    T *Xs = reinterpret_cast<T *>(smem_raw);                  // [nb * RB][CW] the strip
    T *Ls = Xs + (size_t)nb * RB * CW;                        // [nb(nb+1)/2][RB][LP]
    const int64_t c0 = (int64_t)blockIdx.x * CW;
    constexpr int NR = 4 * CW / 32;                           // update rows per thread
    const int cl = lane % CW, hr = lane / CW;                 // column, row half
    const bool vec = ((reinterpret_cast<uintptr_t>(L) | reinterpret_cast<uintptr_t>(X)) & 15) == 0 &&
                     (ldl % EPC) == 0 && (ldx % EPC) == 0;
    // ---- stage the strip and the triangle (16-byte chunks when aligned, else elements)
    {
        const uint32_t xb = (uint32_t)__cvta_generic_to_shared(Xs);
        constexpr int CPR = CW / EPC;                         // chunks per strip row
        for (int e = tid; e < nb * RB * CPR; e += blockDim.x) {
            const int r = e / CPR, cc = (e - r * CPR) * EPC;
            if (vec && r < w && c0 + cc + EPC <= ncols) {
                cp_async<16>(xb + (uint32_t)(r * CW + cc) * sizeof(T), X + (int64_t)r * ldx + c0 + cc, true);
            } else {
#pragma unroll
                for (int q = 0; q < EPC; ++q) {
                    const bool ok = r < w && c0 + cc + q < ncols;
                    cp_async<(int)sizeof(T)>(xb + (uint32_t)(r * CW + cc + q) * sizeof(T),
                                             X + (int64_t)(ok ? r : 0) * ldx + (ok ? c0 + cc + q : 0), ok);
                }
            }
        }
        const uint32_t lb = (uint32_t)__cvta_generic_to_shared(Ls);
        constexpr int CPL = RB / EPC;                         // chunks per L block row
        for (int bb = 0; bb < nb; ++bb)
            for (int kb = 0; kb <= bb; ++kb) {
                const int t = bb * (bb + 1) / 2 + kb;
                for (int e = tid; e < RB * CPL; e += blockDim.x) {
                    const int i = e / CPL, kk = (e - i * CPL) * EPC;
                    const int gr = bb * RB + i, gc = kb * RB + kk;
                    const uint32_t d = lb + (uint32_t)((t * RB + i) * LP + kk) * sizeof(T);
                    // diagonal blocks need only their strictly lower part; stage all of a chunk
                    // that touches it and zero the rest in the solver's reads (m > i only)
                    if (vec && gr < w && gc + EPC <= w) {
                        cp_async<16>(d, L + (int64_t)gr * ldl + gc, true);
                    } else {
#pragma unroll
                        for (int q = 0; q < EPC; ++q) {
                            const bool ok = gr < w && gc + q < w;
                            cp_async<(int)sizeof(T)>(d + q * sizeof(T), L + (int64_t)(ok ? gr : 0) * ldl + (ok ? gc + q : 0),
                                                     ok);
                        }
                    }
                }
            }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    constexpr int NU = TW - 1;                                // updater warps
    const int r4 = 4 * warp + NR * hr;                        // updater: rows r4 .. r4+NR-1 of each block
    T acc[NR];                                                // updater: pending sum for the next block
#pragma unroll
    for (int i = 0; i < NR; ++i) acc[i] = T(0);
    auto contrib = [&](int bt, int k) {                       // acc += L(bt, k) X_k for this thread's rows
        const T *lr = Ls + (size_t)(bt * (bt + 1) / 2 + k) * RB * LP + (size_t)r4 * LP;
        const T *xk = Xs + (size_t)k * RB * CW + cl;
#pragma unroll 2
        for (int kk = 0; kk < RB; kk += 4) {
            T xv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) xv[j] = xk[(kk + j) * CW];
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                const T *l = lr + i * LP + kk;
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i] = fma(l[j], xv[j], acc[i]);
            }
        }
    };
    for (int b = 0; b < nb; ++b) {
        if (warp < NU) {
            if (b > 0) {
                contrib(b, b - 1);                            // the chain's contribution
                T *xr = Xs + (size_t)(b * RB + r4) * CW + cl;
#pragma unroll
                for (int i = 0; i < NR; ++i) { xr[i * CW] -= acc[i]; acc[i] = T(0); }
            }
            named_bar_sync(1, TW * 32);                       // rows of block b ready for the solver
            if (b + 1 < nb)
                for (int k = 0; k < b; ++k) contrib(b + 1, k); // block b+1, everything but X_b
            named_bar_sync(2, TW * 32);                       // X_b published
        } else {
            named_bar_sync(1, TW * 32);
            const T *ld = Ls + (size_t)(b * (b + 1) / 2 + b) * RB * LP;
            T *xb = Xs + (size_t)b * RB * CW + cl;
            T x[RB];
#pragma unroll
            for (int i = 0; i < RB; ++i) x[i] = xb[i * CW];
#pragma unroll
            for (int m = 1; m < RB; ++m) {
                const T *lm = ld + m * LP;
                T p[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
                for (int i = 0; i < m; ++i) p[i & 3] = fma(lm[i], x[i], p[i & 3]);
                x[m] -= (p[0] + p[1]) + (p[2] + p[3]);
            }
            if (hr == 0) {
#pragma unroll
                for (int i = 0; i < RB; ++i) xb[i * CW] = x[i];
            }
            named_bar_sync(2, TW * 32);
        }
    }
    // ---- U12 back to global memory (coalesced rows)
    for (int e = tid; e < nb * RB * CW; e += blockDim.x) {
        const int r = e / CW, cc = e % CW;
        if (r < w && c0 + cc < ncols) X[(int64_t)r * ldx + c0 + cc] = Xs[e];
    }
    if constexpr (sizeof(T) == 4) {
        if (sh) {
            // the hi/lo split: warp-strided 32-row blocks, lane = column (conflict-free shared reads);
            // each lane then writes 32 consecutive k of its column (16-byte stores)
            const int nwarp = blockDim.x >> 5;
            const bool cok = lane < CW && c0 + lane < ncols;
            for (int rb = warp; rb * 32 < kp; rb += nwarp) {
                const int r0 = rb * 32;
                float h[32], l[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const float x = r0 + i < w ? (float)Xs[(size_t)(r0 + i) * CW + cl] : 0.f;
                    h[i] = rna_tf32(x);
                    l[i] = rna_tf32(x - h[i]);
                }
                if (!cok) continue;
                float *ph = sh + (c0 + lane) * (int64_t)kp + r0, *pl = sl + (c0 + lane) * (int64_t)kp + r0;
                if (r0 + 32 <= kp && (kp & 3) == 0) {
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        *reinterpret_cast<float4 *>(ph + i) = make_float4(h[i], h[i + 1], h[i + 2], h[i + 3]);
                        *reinterpret_cast<float4 *>(pl + i) = make_float4(l[i], l[i + 1], l[i + 2], l[i + 3]);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (r0 + i < kp) { ph[i] = h[i]; pl[i] = l[i]; }
                }
            }
        }
    }
}

}  // namespace

template <typename T>
size_t trsm_smem(int w, int cw = CWS)
{
    const int nb = (w + RB - 1) / RB;
    return ((size_t)nb * RB * cw + (size_t)(nb * (nb + 1) / 2) * RB * LP) * sizeof(T) + 16;
}

template <typename T>
void launch_trsm_ops(const T *L, int64_t ldl, T *X, int64_t ldx, int w, int64_t ncols, cudaStream_t s, float *sh,
                     float *sl, int kp)
{
    if (ncols <= 0 || w <= 0) return;
    constexpr int WMAX = sizeof(T) == 4 ? 256 : 128;          // staged triangle must fit shared memory
    if (w > WMAX) {                                            // [L11 0; L21 L22]: X1, X2 -= L21 X1, X2
        const int w1 = WMAX;
        launch_trsm_ops<T>(L, ldl, X, ldx, w1, ncols, s);
        launch_gemm_ops<T>(L + (int64_t)w1 * ldl, ldl, X, ldx, X + (int64_t)w1 * ldx, ldx, w - w1, ncols, w1, s);
        launch_trsm_ops<T>(L + (int64_t)w1 * ldl + w1, ldl, X + (int64_t)w1 * ldx, ldx, w - w1, ncols, s);
        return;
    }
    // narrow ranges (a panel's columns): 16-column strips while twice the CTAs still fit one wave
    static const int sms = [] { int d = 0, v = 0; cudaGetDevice(&d); cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d); return v; }();
    static const int cwn = [] { const char *e = std::getenv("MP_TRSM_CW"); return e ? std::atoi(e) : 16; }();
    int cw = CWS;
    if (cwn == 8 && ceil_div(ncols, 8) <= std::min(96, sms)) cw = 8;
    else if (cwn <= 16 && ceil_div(ncols, 16) <= std::min(96, sms)) cw = 16;
    const int grid = (int)ceil_div(ncols, cw);
    auto kern = cw == 8 ? trsm_lower_unit_kernel<T, 8> : cw == 16 ? trsm_lower_unit_kernel<T, 16> : trsm_lower_unit_kernel<T, CWS>;
    func_smem_once((const void *)kern, trsm_smem<T>(WMAX, cw));   // the largest request, set once per kernel
    if (w > (sizeof(T) == 4 ? 256 : 128)) sh = sl = nullptr;
    launch_ex(kern, dim3(grid), dim3(TW * 32), trsm_smem<T>(w, cw), s, nullptr, L, ldl, X, ldx, w, ncols, sh, sl, kp);
}

template <typename T>
void launch_trsm_lower_unit(T *W, int64_t ldw, int64_t r0, int w, int64_t c_lo, int64_t c_hi, cudaStream_t s,
                            float *sh, float *sl, int kp)
{
    launch_trsm_ops<T>(W + r0 * ldw + r0, ldw, W + r0 * ldw + c_lo, ldw, w, c_hi - c_lo, s, sh, sl, kp);
}

template void launch_trsm_ops<float>(const float *, int64_t, float *, int64_t, int, int64_t, cudaStream_t, float *,
                                     float *, int);
template void launch_trsm_ops<double>(const double *, int64_t, double *, int64_t, int, int64_t, cudaStream_t, float *,
                                      float *, int);
template void launch_trsm_lower_unit<float>(float *, int64_t, int64_t, int, int64_t, int64_t, cudaStream_t, float *,
                                            float *, int);
template void launch_trsm_lower_unit<double>(double *, int64_t, int64_t, int, int64_t, int64_t, cudaStream_t, float *,
                                             float *, int);

}  // namespace mp
