// k_solve.cu — K7 + K9: the triangular solves with the packed LU factors and
// the binary64 update of the solution.
//
// PAPER.md Alg. 1 steps 2-3 / 5-6: "solve L y = P r_k",
// "solve U z_k = y" in the factorisation precision; step 7:
// x_k <- x_{k-1} + z_k in double (fused into the backward sweep's write-back).
// The permutation P was already applied when y was demoted (K6 / the residual
// epilogue).
//
// One sweep = one cooperative kernel.  The n rows are cut into BS = 64-row
// blocks, visited in dependency order (top-down for L, bottom-up for U).
//
//   * The CHAIN CTA (block 0) runs the whole dependent substitution on ONE SM,
//     so the serial chain never pays a cross-SM hand-off: for every block it
//     forms r_I = b_I - F_I - sum_{d=1..DN} T(I, I-d) y_{I-d} (the DN "near"
//     tiles from shared memory), then warp c solves the 64 x 64 diagonal block
//     for right-hand side c: lanes own two rows each; rows are finished in
//     8-row chunks whose 8 x 8 triangle every lane solves redundantly (no
//     shuffle chain), followed by 8 FMAs per owned row.
//   * The HELPER CTAs accumulate the "far" part F_I = sum_{J older than I-DN}
//     T(I, J) y_J as soon as the y_J are published (flags with an epoch), and
//     publish F_I with a flag; they run DN blocks ahead of the chain.
//   * Every tile is streamed HBM -> shared memory by a producer warp with TMA
//     (2D tensor map over the row-major working copy, out-of-range rows and
//     columns zero-filled), through an mbarrier ring, ahead of its use.
//
// Unit lower L (forward) uses no division.  The upper sweep computes
// x_i = b_i / u_ii as q = b*r, r = 1/u_ii correctly rounded, with one residual
// correction q += (b - u q) r: the IEEE quotient except in rare double-rounding
// cases, <= 1 ulp (reading A-7, extended to the substitution; exact whenever
// u_ii is a power of two, as in the exact-LU pin P2).
// HBM traffic: 2 n^2 sizeof(T) per sweep (each factor read once), plus O(n).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace mp {

namespace {

constexpr int BS = 64;                 // block rows
constexpr int NCW = 8;                 // compute warps per CTA
constexpr int WPUB = NCW;              // chain CTA: publisher warp (fence + y flag)
constexpr int WPREP = NCW + 1;         // chain CTA: prepares the next block (rhs, F, diagonal copy)
constexpr int WPROD = NCW + 2;         // TMA producer warp
constexpr int NTH = (NCW + 3) * 32;
constexpr int MAXR = 16;               // right-hand sides per launch

template <typename T> struct SCfg;
template <> struct SCfg<float> {
#ifndef MP_SOLVE_DN
#define MP_SOLVE_DN 3                 // swept 1..5: 2 was best (0.77 vs 0.83 ms per pair at n = 16384) while the publisher's
                                      // fence sat on every block; without it 3 is (0.612 -> 0.567 ms with YB = 4)
#endif
#ifndef MP_SOLVE_CHB
#define MP_SOLVE_CHB 2
#endif
    static constexpr int DN = MP_SOLVE_DN;        // near tiles handled by the chain CTA
    static constexpr int CHB = MP_SOLVE_CHB;      // chain ring: blocks in flight
#ifndef MP_HS
#define MP_HS 8
#endif
#ifndef MP_YB
#define MP_YB 4                       // y blocks per helper batch (8: 0.585 vs 0.567 ms per pair at DN = 3)
#endif
    static constexpr int HS = MP_HS;              // helper ring stages
    static constexpr int YB = MP_YB;              // y blocks fetched per helper batch
    static constexpr int MAXOWN = 12;             // far blocks owned by one helper CTA
};
template <> struct SCfg<double> {
    static constexpr int DN = 2;
    static constexpr int CHB = 1;
    static constexpr int HS = 3;
    static constexpr int YB = 4;
    static constexpr int MAXOWN = 8;
};

template <typename T>
constexpr size_t tile_bytes() { return (size_t)BS * BS * sizeof(T); }

// near tiles handled by the chain CTA (per right-hand-side count: the per-block buffers are
// sized by R; DN = 5 for a single binary32 right-hand side fits but measured slower, 9.6 vs 9.4 ms)
template <typename T, int R>
constexpr int sweep_dn() { return SCfg<T>::DN; }

// Tiles land in shared memory through TMA with SWIZZLE_128B: a 64 x 64 tile is NBOX boxes
// of 64 rows x 128 bytes; inside a box the 16-byte chunk c of row r is stored at chunk
// c ^ (r & 7).  Rows read by consecutive lanes then fall in different banks.
template <typename T> struct Sw {
    static constexpr int EPB = 128 / (int)sizeof(T);     // elements per 128-byte box row
    static constexpr int NBOX = BS / EPB;
    static constexpr int EPC = 16 / (int)sizeof(T);      // elements per 16-byte chunk
    __device__ __forceinline__ static int off(int r, int c)
    {
        const int h = c / EPB, cc = c - h * EPB;
        const int ch = cc / EPC, w = cc - ch * EPC;
        return h * (BS * EPB) + r * EPB + ((ch ^ (r & 7)) * EPC) + w;
    }
};

template <typename T, int R>
constexpr size_t chain_smem()
{
    using C = SCfg<T>;
    constexpr int DN = sweep_dn<T, R>();
    return (size_t)C::CHB * (1 + DN) * tile_bytes<T>() + (size_t)(DN + 1) * R * BS * sizeof(T) +
           4 * (size_t)R * BS * sizeof(T) + (size_t)NCW * BS * sizeof(T) + (size_t)R * BS * sizeof(T) +
           2 * (size_t)R * BS * sizeof(double);
}
template <typename T, int R>
constexpr size_t helper_smem()
{
    return (size_t)SCfg<T>::HS * tile_bytes<T>() + (size_t)SCfg<T>::YB * R * BS * sizeof(T) +
           (size_t)SCfg<T>::MAXOWN * R * BS * sizeof(T);
}
template <typename T, int R>
constexpr size_t sweep_smem()
{
    return (chain_smem<T, R>() > helper_smem<T, R>() ? chain_smem<T, R>() : helper_smem<T, R>()) + 1024;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// the same wait for warps OFF the critical chain: polling backs off with nanosleep (callable
// from a single lane; full-warp callers reconverge with __syncwarp() themselves)
__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_idle(uint64_t *bar, uint32_t parity)
{
#ifndef MP_IDLE_NS
#define MP_IDLE_NS 0                  // swept 0/20/100 ns: plain polling is ~1 % faster
#endif
    while (!mbar_try(bar, parity))
        if (MP_IDLE_NS > 0) __nanosleep(MP_IDLE_NS);
}
// Spin-wait on an mbarrier phase.  The loop is C++ (not a branch inside inline asm), so the
// compiler places the reconvergence point after it: lanes that leave the loop in different
// iterations would otherwise run the following code diverged (every instruction issued
// once per lane group, shuffles on the divergent slow path) until the next warp barrier.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    while (!mbar_try(bar, parity)) { }
    __syncwarp();
}
// tile (row block I, column block J) -> smem, NBOX swizzled boxes (out of range: zero-filled)
template <typename T>
__device__ __forceinline__ void tma_tile(T *dst, const CUtensorMap *map, uint64_t *bar, int J, int I)
{
#pragma unroll
    for (int hb = 0; hb < Sw<T>::NBOX; ++hb)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(dst + hb * BS * Sw<T>::EPB)),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(J * BS + hb * Sw<T>::EPB), "r"(I * BS), "r"(smem_u32(bar))
            : "memory");
}
// named barriers: 1 = compute warps (helpers) / compute + prep + publisher (chain); 2 = solvers -> publisher
__device__ __forceinline__ void nbar_sync(int id, int count) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int count) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory"); }
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
// tagged exchange word {value bits (low), sweep tag (high)}: one 64-bit access is single-copy
// atomic, so a consumer that sees the tag sees the value; no flag, no fence
__device__ __forceinline__ unsigned long long ld_tag(const uint64_t *p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_tag(uint64_t *p, float v, unsigned tag)
{
    const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ void spin_until(const unsigned *flag, unsigned epoch)
{
    while (ld_relaxed_u32(flag) != epoch) { }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

#ifdef MP_SOLVE_TRACE
__device__ unsigned long long g_strace[4096][12];
// the volatile shared load forces a deferred-blocking bar.sync to complete before the clock read
#define STRACE(t, k) do { if (tid == 0 && (t) < 4096) { const int d_ = *(volatile int *)&s_nready; \
    g_strace[(t)][(k)] = (unsigned long long)clock64() + (unsigned long long)(d_ & 0); } } while (0)
// the clock read waits (branch dependency) for value v to exist
#define STRACEV(t, k, v) do { if (tid == 0 && (t) < 4096) { s_tv = (v); const float d_ = *(volatile float *)&s_tv; \
    if (d_ != 1.2345e-30f) g_strace[(t)][(k)] = (unsigned long long)clock64(); } } while (0)
#else
#define STRACE(t, k) do { } while (0)
#define STRACEV(t, k, v) do { } while (0)
#endif

template <typename T>
struct SweepArgs {
    T *Y;                  // [nrhs][n] right-hand sides in, solutions out
    double *X;             // [nrhs][n] binary64 solution (upper sweep only)
    T *F;                  // [nrhs][n] far partial sums
    unsigned *yflag, *fflag;
    uint64_t *tY, *tF;     // binary32 only: tagged y / F words [nrhs][n], nullptr = flags
    int64_t n;
    int nrhs, nblk, accumulate;
    unsigned epoch;
    unsigned tag;          // this sweep's tag in tY / tF
};

__device__ __forceinline__ float rcp_rn(float v) { return __frcp_rn(v); }
__device__ __forceinline__ double rcp_rn(double v) { return __drcp_rn(v); }

// logical block t -> row block index
template <bool LOWER>
__device__ __forceinline__ int blk_of(int t, int nblk) { return LOWER ? t : nblk - 1 - t; }

// acc[p][c] += tile row (r0 + p*rstep) . y(c) over this thread's 8 columns tq*4 + 32m (m = 0, 1)
template <typename T, int R, int NP>
__device__ __forceinline__ void tile_gemv(const T *__restrict__ tl, const T *__restrict__ yv, int r0, int rstep, int tq,
                                          int nrhs, T (&acc)[NP][R])
{
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        const int j = tq * 4 + 32 * m;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int row = r0 + p * rstep;
            T l[4];
            if constexpr (sizeof(T) == 4) {
                const float4 v = *reinterpret_cast<const float4 *>(tl + Sw<T>::off(row, j));
                l[0] = v.x; l[1] = v.y; l[2] = v.z; l[3] = v.w;
            } else {
                const double2 v0 = *reinterpret_cast<const double2 *>(tl + Sw<T>::off(row, j));
                const double2 v1 = *reinterpret_cast<const double2 *>(tl + Sw<T>::off(row, j + 2));
                l[0] = v0.x; l[1] = v0.y; l[2] = v1.x; l[3] = v1.y;
            }
#pragma unroll
            for (int c = 0; c < R; ++c)
                if (c < nrhs) {
                    const T *yp = yv + c * BS + j;
                    acc[p][c] = fma(l[0], yp[0], fma(l[1], yp[1], fma(l[2], yp[2], fma(l[3], yp[3], acc[p][c]))));
                }
        }
    }
}

// reduce over the 8 threads of a row (lanes 8g .. 8g+7) and subtract from dst[c*BS + row]
template <typename T, int R, int NP>
__device__ __forceinline__ void reduce_sub(T (&acc)[NP][R], int r0, int rstep, int tq, int nrhs, T *dst)
{
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int c = 0; c < R; ++c)
            if (c < nrhs) {
                T v = acc[p][c];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                if (tq == 0) dst[c * BS + r0 + p * rstep] -= v;
            }
}

// rsb = Y - F for block t (one warp), several right-hand sides: rounds of 4 rows per lane (issuing
// every round's loads at once measured slower for R = 16: register pressure)
template <typename T, bool LOWER, int DN>
__device__ __forceinline__ void prep_rhs_rounds(const SweepArgs<T> &a, int t, int lane, T *rsb)
{
    const int I = blk_of<LOWER>(t, a.nblk);
    const int64_t i0 = (int64_t)I * BS, n = a.n;
    const int nr = (int)((n - i0 < (int64_t)BS) ? (n - i0) : (int64_t)BS);
    const bool far = t >= DN + 1;
#ifdef MP_SOLVE_TRACE
    if (lane == 0 && t < 4096) g_strace[t][4] = (unsigned long long)clock64();
#endif
    if constexpr (sizeof(T) == 4) {
        if (far && a.tF != nullptr) {
            // poll the tagged F words of the block directly: one round trip, no flag
            for (int i0b = 0; i0b < a.nrhs * BS; i0b += 128) {
                T yv[4], fv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int idx = i0b + lane + 32 * u, c = idx / BS, r = idx - c * BS;
                    yv[u] = (idx < a.nrhs * BS && r < nr) ? a.Y[(int64_t)c * n + i0 + r] : T(0);
                }
                for (;;) {
                    bool ok = true;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int idx = i0b + lane + 32 * u, c = idx / BS, r = idx - c * BS;
                        fv[u] = T(0);
                        if (idx < a.nrhs * BS && r < nr) {
                            const unsigned long long w = ld_tag(a.tF + (int64_t)c * n + i0 + r);
                            fv[u] = __uint_as_float((unsigned)w);
                            ok &= (unsigned)(w >> 32) == a.tag;
                        }
                    }
                    if (__all_sync(0xffffffffu, ok)) break;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int idx = i0b + lane + 32 * u;
                    if (idx < a.nrhs * BS) rsb[idx] = yv[u] - fv[u];
                }
            }
#ifdef MP_SOLVE_TRACE
            if (lane == 0 && t < 4096) g_strace[t][5] = (unsigned long long)clock64();
#endif
            return;
        }
    }
    if (far && lane == 0) spin_until(a.fflag + I, a.epoch);
    __syncwarp();
#ifdef MP_SOLVE_TRACE
    if (lane == 0 && t < 4096) g_strace[t][5] = (unsigned long long)clock64();
#endif
    // 4 rows per lane per round, all 8 loads in flight together
    for (int i0b = 0; i0b < a.nrhs * BS; i0b += 128) {
        T yv[4], fv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int idx = i0b + lane + 32 * u, c = idx / BS, r = idx - c * BS;
            const bool ok = idx < a.nrhs * BS && r < nr;
            yv[u] = ok ? a.Y[(int64_t)c * n + i0 + r] : T(0);
            fv[u] = (ok && far) ? __ldcg(a.F + (int64_t)c * n + i0 + r) : T(0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int idx = i0b + lane + 32 * u;
            if (idx < a.nrhs * BS) rsb[idx] = yv[u] - fv[u];
        }
    }
}

// rsb = Y - F for block t (one warp).  One right-hand side: every load of the block is issued before
// any is consumed (NU = BS / 32 per lane), one memory round trip per block; the tagged F words are
// re-polled together until all carry the sweep's tag.
template <typename T, bool LOWER, int DN, int R>
__device__ __forceinline__ void prep_rhs(const SweepArgs<T> &a, int t, int lane, T *rsb)
{
    if constexpr (R > 1) {
        prep_rhs_rounds<T, LOWER, DN>(a, t, lane, rsb);
        return;
    }
    constexpr int NU = R * BS / 32;
    const int I = blk_of<LOWER>(t, a.nblk);
    const int64_t i0 = (int64_t)I * BS, n = a.n;
    const int nr = (int)((n - i0 < (int64_t)BS) ? (n - i0) : (int64_t)BS);
    const bool far = t >= DN + 1;
    const int tot = a.nrhs * BS;
#ifdef MP_SOLVE_TRACE
    if (lane == 0 && t < 4096) g_strace[t][4] = (unsigned long long)clock64();
#endif
    T yv[NU], fv[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        const int idx = lane + 32 * u, c = idx / BS, r = idx - c * BS;
        yv[u] = (idx < tot && r < nr) ? a.Y[(int64_t)c * n + i0 + r] : T(0);
        fv[u] = T(0);
    }
    bool tagged = false;
    if constexpr (sizeof(T) == 4) tagged = a.tF != nullptr;
    if (far && tagged) {
        if constexpr (sizeof(T) == 4) {
            for (;;) {
                bool ok = true;
#pragma unroll
                for (int u = 0; u < NU; ++u) {
                    const int idx = lane + 32 * u, c = idx / BS, r = idx - c * BS;
                    if (idx < tot && r < nr) {
                        const unsigned long long w = ld_tag(a.tF + (int64_t)c * n + i0 + r);
                        fv[u] = __uint_as_float((unsigned)w);
                        ok &= (unsigned)(w >> 32) == a.tag;
                    }
                }
                if (__all_sync(0xffffffffu, ok)) break;
            }
        }
    } else if (far) {
        if (lane == 0) spin_until(a.fflag + I, a.epoch);
        __syncwarp();
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            const int idx = lane + 32 * u, c = idx / BS, r = idx - c * BS;
            if (idx < tot && r < nr) fv[u] = __ldcg(a.F + (int64_t)c * n + i0 + r);
        }
    }
#ifdef MP_SOLVE_TRACE
    if (lane == 0 && t < 4096) g_strace[t][5] = (unsigned long long)clock64();
#endif
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        const int idx = lane + 32 * u;
        if (idx < tot) rsb[idx] = yv[u] - fv[u];
    }
}

// 8 consecutive elements (r, c0 .. c0+7) of a swizzled tile, c0 % 8 == 0: 16-byte loads
template <typename T>
__device__ __forceinline__ void ld8(const T *__restrict__ tl, int r, int c0, T (&o)[8])
{
    constexpr int EPC = Sw<T>::EPC;
#pragma unroll
    for (int q = 0; q < 8 / EPC; ++q) {
        const T *p = tl + Sw<T>::off(r, c0 + q * EPC);
        if constexpr (sizeof(T) == 4) {
            const float4 v = *reinterpret_cast<const float4 *>(p);
            o[4 * q] = v.x; o[4 * q + 1] = v.y; o[4 * q + 2] = v.z; o[4 * q + 3] = v.w;
        } else {
            const double2 v = *reinterpret_cast<const double2 *>(p);
            o[2 * q] = v.x; o[2 * q + 1] = v.y;
        }
    }
}

// diagonal block solve for one right-hand side (one warp): lanes own rows lane and lane+32;
// rows are finished in 8-row chunks whose 8 x 8 triangle every lane solves redundantly.
// rinv: per-warp shared scratch of BS reciprocals (upper sweep).
template <typename T, bool LOWER>
__device__ __forceinline__ void diag_solve(const T *__restrict__ dg, T *__restrict__ rinv, int lane, int nr, T &v0, T &v1)
{
    T ri0 = T(1), ri1 = T(1), u0 = T(1), u1 = T(1);
    if (!LOWER) {
        u0 = dg[Sw<T>::off(lane, lane)];
        u1 = dg[Sw<T>::off(lane + 32, lane + 32)];
        ri0 = (lane < nr && u0 != T(0)) ? rcp_rn(u0) : T(0);
        ri1 = (lane + 32 < nr && u1 != T(0)) ? rcp_rn(u1) : T(0);
        rinv[lane] = ri0;
        rinv[lane + 32] = ri1;
        __syncwarp();
    }
    constexpr int AHEAD = sizeof(T) == 4 ? 1 : 0;            // operand prefetch distance (chunks)
    T Lc[AHEAD + 1][8][8], Lr[AHEAD + 1][2][8], Ri[AHEAD + 1][8];
#pragma unroll
    for (int kk = 0; kk < BS / 8; ++kk) {
#pragma unroll
        for (int kl = (kk == 0 ? 0 : kk + AHEAD); kl <= kk + AHEAD && kl < BS / 8; ++kl) {
            const int k = LOWER ? kl : BS / 8 - 1 - kl;
            const int r0 = 8 * k, cb = AHEAD ? (kl & 1) : 0;
#pragma unroll
            for (int m = 0; m < 8; ++m) ld8<T>(dg, r0 + m, r0, Lc[cb][m]);
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) ld8<T>(dg, lane + 32 * rr, r0, Lr[cb][rr]);
            if (!LOWER)
#pragma unroll
                for (int i = 0; i < 8; ++i) Ri[cb][i] = rinv[r0 + i];
        }
        const int k = LOWER ? kk : BS / 8 - 1 - kk;
        const int r0 = 8 * k, cb = AHEAD ? (kk & 1) : 0;
        T bb[8], xx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) bb[i] = __shfl_sync(0xffffffffu, k < 4 ? v0 : v1, (r0 + i) & 31);
        if (LOWER) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                xx[i] = (r0 + i < nr) ? bb[i] : T(0);
#pragma unroll
                for (int m = i + 1; m < 8; ++m) bb[m] = fma(-Lc[cb][m][i], xx[i], bb[m]);
            }
        } else {
#pragma unroll
            for (int i = 7; i >= 0; --i) {
                const T u = Lc[cb][i][i], ri = Ri[cb][i];
                T q = bb[i] * ri;
                q = fma(fma(-u, q, bb[i]), ri, q);
                xx[i] = (r0 + i < nr) ? q : T(0);
#pragma unroll
                for (int m = 0; m < i; ++m) bb[m] = fma(-Lc[cb][m][i], xx[i], bb[m]);
            }
        }
        // own rows: the same operations in the same order as the redundant chunk solve, so
        // in-chunk rows reproduce xx bit for bit (no dynamic register indexing)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int row = lane + 32 * rr;
            T sv = rr ? v1 : v0;
            if (LOWER) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (r0 + i < row) sv = fma(-Lr[cb][rr][i], xx[i], sv);
                if (row >= r0 && row < r0 + 8 && row >= nr) sv = T(0);
            } else {
#pragma unroll
                for (int i = 7; i >= 0; --i)
                    if (r0 + i > row) sv = fma(-Lr[cb][rr][i], xx[i], sv);
                if (row >= r0 && row < r0 + 8) {
                    const T u = rr ? u1 : u0, ri = rr ? ri1 : ri0;
                    T q = sv * ri;
                    q = fma(fma(-u, q, sv), ri, q);
                    sv = row < nr ? q : T(0);
                }
            }
            if (rr) v1 = sv; else v0 = sv;
        }
    }
}

template <typename T, bool LOWER, int R, bool INV>
__global__ void __launch_bounds__(NTH, 1) tri_sweep_kernel(const __grid_constant__ CUtensorMap tmW,
                                                           const __grid_constant__ CUtensorMap tmD,
                                                           const __grid_constant__ CUtensorMap tmM, SweepArgs<T> a)
{
    using C = SCfg<T>;
    constexpr int DN = sweep_dn<T, R>();
    constexpr int TILE = BS * BS;
    constexpr uint32_t TB = (uint32_t)tile_bytes<T>();
    extern __shared__ unsigned char smem_raw[];
    // 1 KB alignment by pointer arithmetic on the shared array (keeps the shared state space: LDS)
    T *sm = reinterpret_cast<T *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    __shared__ __align__(8) uint64_t full[16], empty[16];
    __shared__ int s_nready;
    __shared__ unsigned s_ymask[3];
#ifdef MP_SOLVE_TRACE
    __shared__ float s_tv;
#endif

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nblk = a.nblk, nrhs = a.nrhs;
    const int64_t n = a.n;

    bool tagged_y = false;                                    // y exchanged through tagged words
    if constexpr (sizeof(T) == 4) tagged_y = a.tY != nullptr;
    if (blockIdx.x == 0) {
        // =================================================================== chain CTA
        constexpr int NST = C::CHB * (1 + DN);
        constexpr int NCH = (NCW + 2) * 32;                   // compute + publisher + prep threads
        T *tiles = sm;                                        // [NST][TILE] (1 KB aligned)
        T *ys = tiles + (size_t)NST * TILE;                   // [DN+1][R][BS] last solved blocks
        T *rs = ys + (size_t)(DN + 1) * R * BS;            // [2][R][BS]  right-hand sides
        T *nacc = rs + 2 * (size_t)R * BS;                 // [2][R][BS]  near tiles d >= 2, precomputed
        T *rinvs = nacc + 2 * (size_t)R * BS;              // [NCW][BS] reciprocals of the U diagonal
        T *sbuf = rinvs + (size_t)NCW * BS;                   // [R][BS] (INV) s of the next block
        double *xs = reinterpret_cast<double *>(sbuf + (size_t)R * BS);   // [2][R][BS] (INV) x of the next block
        if (tid == 0) {
            // INV: a stage is released by the 4 chain warps right after their GEMV (count 4)
            for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], INV ? 4 : 1); }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        for (int i = tid; i < (DN + 1) * R * BS + 5 * R * BS + NCW * BS; i += NTH) ys[i] = T(0);
        __syncthreads();
        if (warp == WPROD) {
            // ---------------- producer: diagonal + DN near tiles of every block, in order
            if (lane == 0) {
                for (int t = 0; t < nblk; ++t) {
                    const int I = blk_of<LOWER>(t, nblk);
                    const int b = t % C::CHB;
                    const uint32_t ph = (uint32_t)((t / C::CHB) & 1);
                    for (int k = 0; k <= DN; ++k) {
                        const int s = b * (1 + DN) + k;
                        mbar_wait_idle(&empty[s], ph ^ 1u);
                        mbar_expect_tx(&full[s], TB);
                        // k = 0: diagonal tile; k = d: column block of the logically earlier
                        // block t - d (t - d < 0: out of range, zero-filled by the TMA unit)
                        // (INV: k = 0 the inverse of the diagonal block, k = 1 M = Dinv T(I, J_1))
                        const CUtensorMap *map = &tmW;
                        int J = LOWER ? I - k : I + k;
                        if (INV && k <= 1) { map = k == 0 ? &tmD : &tmM; J = 0; }
                        tma_tile<T>(tiles + (size_t)s * TILE, map, &full[s], J, I);
                    }
                }
            }
            return;
        }
        if (warp == WPREP) prep_rhs<T, LOWER, DN, R>(a, 0, lane, rs);
        nbar_sync(1, NCH);
        if constexpr (INV) {
            // ---------------- inverted-diagonal-block chain (reading A-19):
            //   y_t = w_t - M_t y_{t-1},   M_t = D_t^-1 T(t, t-1)                  (group P, warps 0-3)
            //   w_{t+1} = D_{t+1}^-1 (rs_{t+1} - sum_{d=2..DN} T(t+1, t+1-d) y_{t+1-d}) (group L, warps 4-7)
            // so the dependent chain per block is ONE 64 x 64 GEMV; w_{t+1} only needs y up to
            // y_{t-1} and is formed while block t runs.
            T *wbuf = nacc;                                   // [2][R][BS]
            const int lt = tid & 127, gr = lt >> 3, gq = lt & 7;   // rows gr + 16p, cols gq*4 + 32m
            auto make_w = [&](int tt, bool prep_sync) {
                const int b1 = tt % C::CHB;
                const uint32_t ph1 = (uint32_t)((tt / C::CHB) & 1);
                T acc[4][R];
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int c = 0; c < R; ++c) acc[p][c] = T(0);
                for (int d = 2; d <= DN; ++d) {
                    const int s = b1 * (1 + DN) + d;
                    mbar_wait_idle(&full[s], ph1);
                    __syncwarp();
                    tile_gemv<T, R, 4>(tiles + (size_t)s * TILE, ys + (size_t)((tt - d + 2 * (DN + 1)) % (DN + 1)) * R * BS,
                                       gr, 16, gq, nrhs, acc);
                }
                if (prep_sync) nbar_sync(3, 160);             // rs_tt prepared by the prep warp
                const T *r1 = rs + (size_t)(tt & 1) * R * BS;
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int c = 0; c < R; ++c)
                        if (c < nrhs) {
                            T v = acc[p][c];
                            v += __shfl_xor_sync(0xffffffffu, v, 1);
                            v += __shfl_xor_sync(0xffffffffu, v, 2);
                            v += __shfl_xor_sync(0xffffffffu, v, 4);
                            if (gq == 0) sbuf[c * BS + gr + 16 * p] = r1[c * BS + gr + 16 * p] - v;
                            acc[p][c] = T(0);
                        }
                nbar_sync(4, 128);
                const int s0 = b1 * (1 + DN);
                mbar_wait_idle(&full[s0], ph1);
                __syncwarp();
                tile_gemv<T, R, 4>(tiles + (size_t)s0 * TILE, sbuf, gr, 16, gq, nrhs, acc);
                T *wb = wbuf + (size_t)(tt & 1) * R * BS;
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int c = 0; c < R; ++c)
                        if (c < nrhs) {
                            T v = acc[p][c];
                            v += __shfl_xor_sync(0xffffffffu, v, 1);
                            v += __shfl_xor_sync(0xffffffffu, v, 2);
                            v += __shfl_xor_sync(0xffffffffu, v, 4);
                            if (gq == 0) wb[c * BS + gr + 16 * p] = v;
                        }
            };
            // backward sweep with accumulation: the prep warp also fetches x of the block it prepares,
            // so the chain's x += z never waits on global memory
            // (loads issued before the F wait, stored after it: their latency hides under the spin)
            constexpr int XR = 2 * R;                          // R * BS / 32 values per lane
            auto prep_x_load = [&](int tt, double (&v)[XR]) {
                const int64_t j0 = (int64_t)blk_of<LOWER>(tt, nblk) * BS;
#pragma unroll
                for (int u = 0; u < XR; ++u) {
                    const int idx = lane + 32 * u, c = idx / BS, r = idx - c * BS;
                    v[u] = (!LOWER && a.accumulate && c < nrhs && j0 + r < n) ? a.X[(int64_t)c * n + j0 + r] : 0.0;
                }
            };
            auto prep_x_store = [&](int tt, const double (&v)[XR]) {
                double *xb = xs + (size_t)(tt & 1) * R * BS;
#pragma unroll
                for (int u = 0; u < XR; ++u) xb[lane + 32 * u] = v[u];
            };
            if (warp == WPREP) {
                double v[XR];
                prep_x_load(0, v);
                prep_x_store(0, v);
            }
            if (warp >= 4 && warp < NCW) make_w(0, false);
            nbar_sync(1, NCH);
            for (int t = 0; t < nblk; ++t) {
                const int I = blk_of<LOWER>(t, nblk);
                const int64_t i0 = (int64_t)I * BS;
                const int nr = (int)std::min<int64_t>(BS, n - i0);
                const int b = t % C::CHB;
                const uint32_t ph = (uint32_t)((t / C::CHB) & 1);
                const int slot = t % (DN + 1);
                STRACE(t, 0);
                if (warp < 4) {
                    const double *xb = xs + (size_t)(t & 1) * R * BS;   // x of this block (prep warp)
                    T acc[4][R];
#pragma unroll
                    for (int p = 0; p < 4; ++p)
#pragma unroll
                        for (int c = 0; c < R; ++c) acc[p][c] = T(0);
                    const int s1 = b * (1 + DN) + 1;
                    mbar_wait(&full[s1], ph);
#ifdef MP_SOLVE_TRACE
                    if (tid == 0 && t < 4096) g_strace[t][1] = (unsigned long long)clock64();
#endif
                    tile_gemv<T, R, 4>(tiles + (size_t)s1 * TILE, ys + (size_t)((t + DN) % (DN + 1)) * R * BS, gr, 16,
                                       gq, nrhs, acc);
                    STRACEV(t, 8, (float)acc[0][0]);
                    // every tile of stage b is consumed (L read D_t, T(t, t-d) during block t-1)
                    __syncwarp();
                    if (lane == 0)
                        for (int k = 0; k <= DN; ++k) mbar_arrive(&empty[b * (1 + DN) + k]);
                    // the 8-lane reductions of all rows first (independent shuffles in flight)
#pragma unroll
                    for (int p = 0; p < 4; ++p)
#pragma unroll
                        for (int c = 0; c < R; ++c)
                            if (c < nrhs) acc[p][c] += __shfl_xor_sync(0xffffffffu, acc[p][c], 1);
#pragma unroll
                    for (int p = 0; p < 4; ++p)
#pragma unroll
                        for (int c = 0; c < R; ++c)
                            if (c < nrhs) acc[p][c] += __shfl_xor_sync(0xffffffffu, acc[p][c], 2);
#pragma unroll
                    for (int p = 0; p < 4; ++p)
#pragma unroll
                        for (int c = 0; c < R; ++c)
                            if (c < nrhs) acc[p][c] += __shfl_xor_sync(0xffffffffu, acc[p][c], 4);
                    STRACEV(t, 9, (float)acc[3][0]);
                    const T *wb = wbuf + (size_t)(t & 1) * R * BS;
                    T *yo = ys + (size_t)slot * R * BS;
                    if (gq == 0) {
#pragma unroll
                        for (int p = 0; p < 4; ++p)
#pragma unroll
                            for (int c = 0; c < R; ++c)
                                if (c < nrhs) {
                                    const int row = gr + 16 * p;
                                    const T y = wb[c * BS + row] - acc[p][c];
                                    yo[c * BS + row] = y;
                                    if (row < nr) {
                                        const int64_t gi = (int64_t)c * n + i0 + row;
                                        a.Y[gi] = y;
                                        if constexpr (sizeof(T) == 4)
                                            if (a.tY != nullptr) st_tag(a.tY + gi, y, a.tag);
                                        if (!LOWER) {
                                            const double xv = a.accumulate ? xb[c * BS + row] : 0.0;
                                            a.X[gi] = xv + (double)y;
                                        }
                                    }
                                }
                    }
                    STRACE(t, 2);
                    nbar_arrive(2, 160);                      // hand the stores to the publisher
                } else if (warp < NCW) {
                    if (t + 1 < nblk) make_w(t + 1, true);
#ifdef MP_SOLVE_TRACE
                    if (tid == 128 && t < 4096) g_strace[t][6] = (unsigned long long)clock64();
#endif
                } else if (warp == WPUB) {
                    nbar_sync(2, 160);
                    // the flag exchange only: with tagged words the helpers read y itself, and the
                    // fence (waiting for the y / x stores to reach L2) would sit on every block's step
                    if (lane == 0 && !tagged_y) {
                        __threadfence();
                        st_release_u32(a.yflag + I, a.epoch);
                    }
                } else if (warp == WPREP) {
                    if (t + 1 < nblk) {
                        double xv[XR];
                        prep_x_load(t + 1, xv);
                        prep_rhs<T, LOWER, DN, R>(a, t + 1, lane, rs + (size_t)((t + 1) & 1) * R * BS);
                        prep_x_store(t + 1, xv);
                        __syncwarp();
#ifdef MP_SOLVE_TRACE
                        if (lane == 0 && t < 4096) g_strace[t][7] = (unsigned long long)clock64();
#endif
                        nbar_arrive(3, 160);
                    }
                }
                nbar_sync(1, NCH);                             // y_t, w_{t+1} ready
                STRACE(t, 3);
            }
            return;
        }
        const int nsolv = nrhs < NCW ? nrhs : NCW;
        // idle warps precompute the next block's near tiles d >= 2 (needs a second ring slot)
        const bool split = nsolv <= NCW / 2 && C::CHB > 1;
        const int tr = tid >> 3, tq = tid & 7;                // rows tr, tr+32; cols tq*4 + 32m
        for (int t = 0; t < nblk; ++t) {
            const int I = blk_of<LOWER>(t, nblk);
            const int64_t i0 = (int64_t)I * BS;
            const int nr = (int)std::min<int64_t>(BS, n - i0);
            const int b = t % C::CHB;
            const uint32_t ph = (uint32_t)((t / C::CHB) & 1);
            const int slot = t % (DN + 1);
            T *rsb = rs + (size_t)(t & 1) * R * BS;
            const T *dg = tiles + (size_t)(b * (1 + DN)) * TILE;
            STRACE(t, 0);
            // ---- phase A: near tile d = 1 (all DN when not split): rs -= T(I, J_d) y_{t-d} (+ nacc)
            if (warp < NCW) {
                T acc[2][R];
#pragma unroll
                for (int p = 0; p < 2; ++p)
#pragma unroll
                    for (int c = 0; c < R; ++c) acc[p][c] = T(0);
                const int dmax = split ? 1 : DN;
                for (int d = 1; d <= dmax; ++d) {
                    const int s = b * (1 + DN) + d;
                    mbar_wait(&full[s], ph);
                    tile_gemv<T, R, 2>(tiles + (size_t)s * TILE, ys + (size_t)((t - d + 2 * (DN + 1)) % (DN + 1)) * R * BS,
                                       tr, 32, tq, nrhs, acc);
                }
                if (split && tq == 0) {
                    const T *nb = nacc + (size_t)(t & 1) * R * BS;
#pragma unroll
                    for (int p = 0; p < 2; ++p)
#pragma unroll
                        for (int c = 0; c < R; ++c)
                            if (c < nrhs) acc[p][c] += nb[c * BS + tr + 32 * p];
                }
                reduce_sub<T, R, 2>(acc, tr, 32, tq, nrhs, rsb);
            }
            nbar_sync(1, NCH);
            STRACE(t, 1);
            // ---- phase B
            if (warp < nsolv) {
                mbar_wait(&full[b * (1 + DN)], ph);
#ifdef MP_SOLVE_TRACE
                if (tid == 0 && t < 4096) g_strace[t][6] = (unsigned long long)clock64();
#endif
                for (int c = warp; c < nrhs; c += NCW) {
                    double xo0 = 0.0, xo1 = 0.0;              // x of the owned rows, fetched early
                    if (!LOWER && a.accumulate) {
                        if (lane < nr) xo0 = a.X[(int64_t)c * n + i0 + lane];
                        if (lane + 32 < nr) xo1 = a.X[(int64_t)c * n + i0 + lane + 32];
                    }
                    T v0 = rsb[c * BS + lane], v1 = rsb[c * BS + lane + 32];
                    diag_solve<T, LOWER>(dg, rinvs + warp * BS, lane, nr, v0, v1);
#ifdef MP_SOLVE_TRACE
                    if (tid == 0 && t < 4096) g_strace[t][7] = (unsigned long long)clock64() + (unsigned long long)(__float_as_int((float)v0) & 0);
#endif
                    // y (or z) to shared (near tiles of later blocks) and global; x (+)= z
                    ys[(size_t)slot * R * BS + c * BS + lane] = v0;
                    ys[(size_t)slot * R * BS + c * BS + lane + 32] = v1;
                    if (lane < nr) {
                        a.Y[(int64_t)c * n + i0 + lane] = v0;
                        if constexpr (sizeof(T) == 4)
                            if (a.tY != nullptr) st_tag(a.tY + (int64_t)c * n + i0 + lane, v0, a.tag);
                        if (!LOWER) a.X[(int64_t)c * n + i0 + lane] = xo0 + (double)v0;
                    }
                    if (lane + 32 < nr) {
                        a.Y[(int64_t)c * n + i0 + lane + 32] = v1;
                        if constexpr (sizeof(T) == 4)
                            if (a.tY != nullptr) st_tag(a.tY + (int64_t)c * n + i0 + lane + 32, v1, a.tag);
                        if (!LOWER) a.X[(int64_t)c * n + i0 + lane + 32] = xo1 + (double)v1;
                    }
                }
                STRACE(t, 2);
                nbar_arrive(2, (nsolv + 1) * 32);             // hand the stores to the publisher
            } else if (warp == WPUB) {
                // publish y_I for the helpers: the barrier orders the solvers' stores before the
                // release (cumulativity), so the solvers never wait on the fence
                nbar_sync(2, (nsolv + 1) * 32);
                if (lane == 0 && !tagged_y) {
                    __threadfence();
                    st_release_u32(a.yflag + I, a.epoch);
                }
            } else if (warp == WPREP) {
                if (t + 1 < nblk) prep_rhs<T, LOWER, DN, R>(a, t + 1, lane, rs + (size_t)((t + 1) & 1) * R * BS);
            } else if (split && warp >= NCW / 2 && warp < NCW && t + 1 < nblk) {
                // next block's near tiles d = 2..DN (their y blocks are all solved)
                const int lt = tid - (NCW / 2) * 32;          // 0..127: rows (lt>>3) + 16p, cols (lt&7)*4 + 32m
                const int b1 = (t + 1) % C::CHB;
                const uint32_t ph1 = (uint32_t)(((t + 1) / C::CHB) & 1);
                T acc[4][R];
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int c = 0; c < R; ++c) acc[p][c] = T(0);
                for (int d = 2; d <= DN; ++d) {
                    const int s = b1 * (1 + DN) + d;
                    mbar_wait_idle(&full[s], ph1);
                    __syncwarp();
                    tile_gemv<T, R, 4>(tiles + (size_t)s * TILE,
                                       ys + (size_t)((t + 1 - d + 2 * (DN + 1)) % (DN + 1)) * R * BS, lt >> 3, 16,
                                       lt & 7, nrhs, acc);
                }
                T *nb = nacc + (size_t)((t + 1) & 1) * R * BS;
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int c = 0; c < R; ++c)
                        if (c < nrhs) {
                            T v = acc[p][c];
                            v += __shfl_xor_sync(0xffffffffu, v, 1);
                            v += __shfl_xor_sync(0xffffffffu, v, 2);
                            v += __shfl_xor_sync(0xffffffffu, v, 4);
                            if ((lt & 7) == 0) nb[c * BS + (lt >> 3) + 16 * p] = v;
                        }
            }
            nbar_sync(1, NCH);                                 // ys[slot], rs/nacc[t+1] ready
            STRACE(t, 3);
            if (tid == 0)                                      // every tile of block t consumed
                for (int k = 0; k <= DN; ++k) mbar_arrive(&empty[b * (1 + DN) + k]);
        }
        return;
    }

    // =================================================================== helper CTAs
    const int h = (int)blockIdx.x - 1, H = (int)gridDim.x - 1;
    constexpr int HS = C::HS, YB = C::YB, MAXOWN = C::MAXOWN;
    constexpr int NHC = NCW * 32;
    T *tiles = sm;                                            // [HS][TILE]
    T *yb = tiles + (size_t)HS * TILE;                        // [YB][R][BS]
    T *accs = yb + (size_t)YB * R * BS;                    // [MAXOWN][R][BS]
    int town[MAXOWN];
    int nown = 0;
    for (int t = DN + 1 + h; t < nblk && nown < MAXOWN; t += H) town[nown++] = t;
    if (nown == 0) return;
    const int tmax = town[nown - 1] - DN - 1;                 // last y block this CTA consumes
    if (tid == 0) {
        for (int s = 0; s < HS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < MAXOWN * R * BS; i += NTH) accs[i] = T(0);
    if (tid < 3) s_ymask[tid] = ~0u;
    __syncthreads();
    if (warp == WPROD) {
        // ---------------- producer: tiles (I_o, J_tp) in consumption order
        if (lane == 0) {
            int seq = 0;
            for (int tp = 0; tp <= tmax; ++tp) {
                const int J = blk_of<LOWER>(tp, nblk);
                for (int o = 0; o < nown; ++o) {
                    if (town[o] < tp + DN + 1) continue;
                    const int s = seq % HS;
                    mbar_wait_idle(&empty[s], (uint32_t)(((seq / HS) & 1) ^ 1));
                    mbar_expect_tx(&full[s], TB);
                    tma_tile<T>(tiles + (size_t)s * TILE, &tmW, &full[s], J, blk_of<LOWER>(town[o], nblk));
                    ++seq;
                }
            }
        }
        return;
    }
    if (warp >= NCW) return;
    const int tr = tid >> 3, tq = tid & 7;
    int seq = 0;
    int tp = 0;
    unsigned round = 0;
    const bool tagged = sizeof(T) == 4 && a.tY != nullptr;
    auto helper_block = [&](int k) {
        const T *yv = yb + (size_t)k * R * BS;
        for (int o = 0; o < nown; ++o) {
            if (town[o] < tp + DN + 1) continue;
            const int s = seq % HS;
            mbar_wait(&full[s], (uint32_t)((seq / HS) & 1));
            T acc[2][R];
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int c = 0; c < R; ++c) acc[p][c] = T(0);
            tile_gemv<T, R, 2>(tiles + (size_t)s * TILE, yv, tr, 32, tq, nrhs, acc);
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int c = 0; c < R; ++c)
                    if (c < nrhs) {
                        T v = acc[p][c];
                        v += __shfl_xor_sync(0xffffffffu, v, 1);
                        v += __shfl_xor_sync(0xffffffffu, v, 2);
                        v += __shfl_xor_sync(0xffffffffu, v, 4);
                        if (tq == 0) accs[((size_t)o * R + c) * BS + tr + 32 * p] += v;
                    }
            nbar_sync(1, NHC);
            if (tid == 0) mbar_arrive(&empty[s]);
            ++seq;
            if (town[o] == tp + DN + 1) {                 // F of block o complete: publish
                const int64_t i0 = (int64_t)blk_of<LOWER>(town[o], nblk) * BS;
                if constexpr (sizeof(T) == 4) {
                    if (tagged) {
                        for (int idx = tid; idx < nrhs * BS; idx += NHC) {
                            const int c = idx / BS, r = idx - c * BS;
                            if (i0 + r < n) st_tag(a.tF + (int64_t)c * n + i0 + r, accs[((size_t)o * R + c) * BS + r], a.tag);
                        }
                        continue;
                    }
                }
                for (int idx = tid; idx < nrhs * BS; idx += NHC) {
                    const int c = idx / BS, r = idx - c * BS;
                    if (i0 + r < n) a.F[(int64_t)c * n + i0 + r] = accs[((size_t)o * R + c) * BS + r];
                }
                // the barrier orders every thread's F stores before thread 0's fence + release
                // (cumulativity): one fence per publish instead of one per thread
                nbar_sync(1, NHC);
                if (tid == 0) {
                    __threadfence();
                    st_release_u32(a.fflag + blk_of<LOWER>(town[o], nblk), a.epoch);
                }
            }
        }
    };
    while (tp <= tmax) {
        if (tagged) {
            // read up to YB y blocks straight from their tagged words; the AND over all
            // threads of the per-block validity masks gives the published prefix
            const int nbmax = min(YB, tmax - tp + 1);
            int nb = 0;
            while (nb == 0) {
                unsigned mine = (1u << nbmax) - 1u;
                for (int idx = tid; idx < nbmax * nrhs * BS; idx += NHC) {
                    const int k = idx / (nrhs * BS), rem = idx - k * nrhs * BS;
                    const int c = rem / BS, r = rem - c * BS;
                    const int64_t j = (int64_t)blk_of<LOWER>(tp + k, nblk) * BS + r;
                    T v = T(0);
                    if (j < n) {
                        const unsigned long long w = ld_tag(a.tY + (int64_t)c * n + j);
                        v = __uint_as_float((unsigned)w);
                        if ((unsigned)(w >> 32) != a.tag) mine &= ~(1u << k);
                    }
                    yb[(size_t)k * R * BS + c * BS + r] = v;
                }
                mine = __reduce_and_sync(0xffffffffu, mine);
                unsigned *mk = s_ymask + round % 3;
                if (lane == 0) atomicAnd(mk, mine);
                nbar_sync(1, NHC);
                const unsigned m = *mk;
                if (tid == 0) s_ymask[(round + 2) % 3] = ~0u;   // read last in round - 1
                ++round;
                nb = __ffs(~m) - 1;
                if (nb > nbmax) nb = nbmax;
            }
            for (int k = 0; k < nb; ++k, ++tp) helper_block(k);
            continue;
        }
        // how many consecutive y blocks are published (at least one: wait for it)
        if (tid == 0) {
            spin_until(a.yflag + blk_of<LOWER>(tp, nblk), a.epoch);
            int k = 1;
            while (k < YB && tp + k <= tmax && ld_relaxed_u32(a.yflag + blk_of<LOWER>(tp + k, nblk)) == a.epoch) ++k;
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            s_nready = k;
        }
        nbar_sync(1, NHC);
        const int nb = s_nready;
        for (int idx = tid; idx < nb * nrhs * BS; idx += NHC) {
            const int k = idx / (nrhs * BS), rem = idx - k * nrhs * BS;
            const int c = rem / BS, r = rem - c * BS;
            const int64_t j = (int64_t)blk_of<LOWER>(tp + k, nblk) * BS + r;
            yb[(size_t)k * R * BS + c * BS + r] = j < n ? __ldcg(a.Y + (int64_t)c * n + j) : T(0);
        }
        nbar_sync(1, NHC);
        for (int k = 0; k < nb; ++k, ++tp) helper_block(k);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode_tm = nullptr;

// 2D map over a row-major array of `rows` rows x `cols` columns (row stride ld elements)
template <typename T>
void encode_map(CUtensorMap *map, const T *W, int64_t ld, int64_t cols, int64_t rows)
{
    if (!g_encode_tm) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        MP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) throw CudaError{cudaErrorNotSupported, "cuTensorMapEncodeTiled", __LINE__};
        g_encode_tm = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)ld * sizeof(T)};
    cuuint32_t box[2] = {(cuuint32_t)Sw<T>::EPB, (cuuint32_t)BS};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode_tm(map, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                             const_cast<T *>(W), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError{cudaErrorInvalidValue, "cuTensorMapEncodeTiled (solve) failed", __LINE__};
}

template <typename T, bool LOWER>
void launch_sweep(const CUtensorMap &tm, const CUtensorMap &tD, const CUtensorMap &tM, bool inv, SweepArgs<T> &a,
                  int grid, cudaStream_t s)
{
    // right-hand sides per launch: 1, up to 4, up to 8, up to MAXR (the per-block chain work scales with R)
    const int rk = a.nrhs == 1 ? 0 : a.nrhs <= 4 ? 1 : a.nrhs <= 8 ? 2 : 3;
    using KFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, SweepArgs<T>);
    const KFn sub[4] = {tri_sweep_kernel<T, LOWER, 1, false>, tri_sweep_kernel<T, LOWER, 4, false>,
                        tri_sweep_kernel<T, LOWER, 8, false>, tri_sweep_kernel<T, LOWER, MAXR, false>};
    KFn kern = sub[rk];
    if constexpr (sizeof(T) == 4) {
        const KFn ik[4] = {tri_sweep_kernel<T, LOWER, 1, true>, tri_sweep_kernel<T, LOWER, 4, true>,
                           tri_sweep_kernel<T, LOWER, 8, true>, tri_sweep_kernel<T, LOWER, MAXR, true>};
        if (inv) kern = ik[rk];
    }
    const size_t sm[4] = {sweep_smem<T, 1>(), sweep_smem<T, 4>(), sweep_smem<T, 8>(), sweep_smem<T, MAXR>()};
    const size_t smem = sm[rk];
    func_smem_once((const void *)kern, smem);
    void *args[] = {(void *)&tm, (void *)&tD, (void *)&tM, (void *)&a};
    MP_CUDA(cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(NTH), args, smem, s));
}

// Inverted diagonal blocks for the INV sweeps (reading A-19), once per factorisation.
// Block I (rows i0 .. i0+nr-1): D_I = inverse of the diagonal block of L (unit lower) or U
// (upper), formed in binary64 from the binary32 factors by column substitution, and
// M_I = D_I T(I, J) with J = I - 1 (L) / I + 1 (U) the block the sweep visits just before I;
// both rounded once to binary32.  Rows / columns >= nr and a missing J give zeros, so the
// sweep's padded rows stay zero.  A zero u_ii (only with a recorded zero pivot, which
// sends the driver to the fallback before any solve) gives a zero row.
template <bool LOWER>
__device__ __forceinline__ void diag_inv_block(const float *__restrict__ W, int64_t ldw, int64_t n,
                                               float *__restrict__ Dinv, float *__restrict__ Mo,
                                               unsigned long long *__restrict__ cond_max)
{
    constexpr int LD = BS + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *Ls = reinterpret_cast<double *>(smem_raw);       // [BS][LD] diagonal block (unit / identity padded)
    double *Xs = Ls + BS * LD;                               // [BS][LD] its inverse
    double *Os = Xs + BS * LD;                               // [BS][LD] T(I, J)
    const int I = blockIdx.x, nblk = gridDim.x, tid = threadIdx.x;
    const int64_t i0 = (int64_t)I * BS;
    const int nr = (int)((n - i0 < (int64_t)BS) ? (n - i0) : (int64_t)BS);
    const int J = LOWER ? I - 1 : I + 1;
    for (int idx = tid; idx < BS * BS; idx += blockDim.x) {
        const int r = idx / BS, c = idx - r * BS;
        double d = (r == c) ? 1.0 : 0.0;
        if (r < nr && c < nr && (LOWER ? r > c : r <= c)) d = (double)W[(i0 + r) * ldw + i0 + c];
        Ls[r * LD + c] = d;
        double o = 0.0;
        if (J >= 0 && J < nblk && r < nr) {
            const int64_t jc = (int64_t)J * BS + c;
            if (jc < n) o = (double)W[(i0 + r) * ldw + jc];
        }
        Os[r * LD + c] = o;
    }
    __syncthreads();
    if (tid < BS) {                                          // column j of the inverse
        const int j = tid;
        if (LOWER) {
            for (int i = 0; i < BS; ++i) {
                double acc = (i == j) ? 1.0 : 0.0;
                for (int k = j; k < i; ++k) acc = fma(-Ls[i * LD + k], Xs[k * LD + j], acc);
                Xs[i * LD + j] = acc;
            }
        } else {
            for (int i = BS - 1; i >= 0; --i) {
                double acc = (i == j) ? 1.0 : 0.0;
                for (int k = i + 1; k <= j; ++k) acc = fma(-Ls[i * LD + k], Xs[k * LD + j], acc);
                const double u = Ls[i * LD + i];
                Xs[i * LD + j] = (i > j || u == 0.0) ? 0.0 : acc / u;
            }
        }
    }
    __syncthreads();
    // kappa_inf(T_II) = ||T_II||_inf ||T_II^-1||_inf, max over blocks (the driver keeps
    // substitution when it is large: the inverse's rounding error grows with it)
    __shared__ double rs_t[BS], rs_x[BS];
    if (tid < BS) {
        double a = 0.0, x = 0.0;
        if (tid < nr)
            for (int c = 0; c < nr; ++c) { a += fabs(Ls[tid * LD + c]); x += fabs(Xs[tid * LD + c]); }
        rs_t[tid] = a;
        rs_x[tid] = x;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0, x = 0.0;
        for (int r = 0; r < BS; ++r) { a = fmax(a, rs_t[r]); x = fmax(x, rs_x[r]); }
        double kap = a * x;
        if (!(kap <= 1e300)) kap = 1e300;                    // non-finite -> huge
        atomicMax(cond_max, (unsigned long long)__double_as_longlong(kap));   // non-negative: bit order = value order
    }
    for (int idx = tid; idx < BS * BS; idx += blockDim.x) {
        const int r = idx / BS, c = idx - r * BS;
        double m = 0.0;
        for (int k = 0; k < BS; ++k) m = fma(Xs[r * LD + k], Os[k * LD + c], m);
        Dinv[(i0 + r) * BS + c] = (r < nr && c < nr) ? (float)Xs[r * LD + c] : 0.f;
        Mo[(i0 + r) * BS + c] = r < nr ? (float)m : 0.f;
    }
}

// blockIdx.y = 0: L blocks, 1: U blocks (one launch: the two sets are independent)
__global__ void __launch_bounds__(256) diag_inv_kernel(const float *__restrict__ W, int64_t ldw, int64_t n,
                                                       float *__restrict__ inv, size_t blk,
                                                       unsigned long long *__restrict__ cond_max)
{
    if (blockIdx.y == 0) diag_inv_block<true>(W, ldw, n, inv, inv + blk, cond_max);
    else diag_inv_block<false>(W, ldw, n, inv + 2 * blk, inv + 3 * blk, cond_max);
}

}  // namespace

int solve_block_rows() { return BS; }

size_t solve_flag_words(int64_t n) { return 4 * (size_t)ceil_div(n, BS); }
size_t solve_tag_words(int64_t n, int64_t nrhs) { return 2 * (size_t)std::min<int64_t>(std::max<int64_t>(nrhs, 1), MAXR) * n; }

size_t solve_inv_floats(int64_t n) { return (size_t)4 * (size_t)ceil_div(n, BS) * BS * BS + 2; }

void launch_solve_inverses(const float *W, int64_t ldw, int64_t n, float *inv, cudaStream_t s)
{
    if (n <= 0) return;
    unsigned long long *cond = reinterpret_cast<unsigned long long *>(inv + (size_t)4 * ceil_div(n, BS) * BS * BS);
    MP_CUDA(cudaMemsetAsync(cond, 0, sizeof(unsigned long long), s));
    const int nblk = (int)ceil_div(n, BS);
    const size_t blk = (size_t)nblk * BS * BS;
    const size_t smem = (size_t)3 * BS * (BS + 1) * sizeof(double);
    func_smem_once((const void *)diag_inv_kernel, smem);
    launch_ex(diag_inv_kernel, dim3(nblk, 2), dim3(256), smem, s, nullptr, W, ldw, n, inv, blk, cond);
}

double solve_inverses_cond(const float *inv, int64_t n, cudaStream_t s)
{
    if (n <= 0) return 0.0;
    const unsigned long long *cond =
        reinterpret_cast<const unsigned long long *>(inv + (size_t)4 * ceil_div(n, BS) * BS * BS);
    unsigned long long v = 0;
    MP_CUDA(cudaMemcpyAsync(&v, cond, sizeof(v), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    double d;
    std::memcpy(&d, &v, sizeof(d));
    return d;
}

template <typename T>
void launch_lu_solve(const T *W, int64_t ldw, int64_t n, int64_t nrhs, T *Y, double *X, int accumulate,
                     SolveScratch &ss, cudaStream_t s, const float *inv)
{
    if constexpr (sizeof(T) == 4) {
        if (inv != nullptr && nrhs >= 2 && mr_solve_supported(n, nrhs)) {
            launch_lu_solve_mr(reinterpret_cast<const float *>(W), ldw, n, nrhs, reinterpret_cast<float *>(Y), X,
                               accumulate, ss.flags, ss.epoch, inv, s, ss.tags, ss.tag_cols);
            return;
        }
    }
    const int nblk = (int)ceil_div(n, BS);
    CUtensorMap tm, tDL, tML, tDU, tMU;
    encode_map<T>(&tm, W, ldw, ldw, n);
    const bool use_inv = sizeof(T) == 4 && inv != nullptr;
    if (use_inv) {
        const size_t blk = (size_t)nblk * BS * BS;
        const T *b = reinterpret_cast<const T *>(inv);
        encode_map<T>(&tDL, b, BS, BS, (int64_t)nblk * BS);
        encode_map<T>(&tML, b + blk, BS, BS, (int64_t)nblk * BS);
        encode_map<T>(&tDU, b + 2 * blk, BS, BS, (int64_t)nblk * BS);
        encode_map<T>(&tMU, b + 3 * blk, BS, BS, (int64_t)nblk * BS);
    } else {
        tDL = tML = tDU = tMU = tm;
    }
    int dev = 0, sms = 0;
    MP_CUDA(cudaGetDevice(&dev));
    MP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int dnmin = std::min(sweep_dn<T, 1>(), sweep_dn<T, MAXR>());
    static const bool tags_off = std::getenv("MP_SOLVE_FLAGS") != nullptr;   // A/B: flag exchange
    static const int hmax = [] { const char *e = std::getenv("MP_SOLVE_HELPERS"); return e ? std::atoi(e) : 0; }();
    const int hcap = hmax > 0 ? std::min(hmax, sms - 1) : sms - 1;
    const int helpers = std::max(1, std::min(hcap, nblk - dnmin - 1));
    if (ceil_div(std::max(0, nblk - dnmin - 1), helpers) > SCfg<T>::MAXOWN)
        throw CudaError{cudaErrorInvalidValue, "matrix too large for the triangular-solve helper grid", __LINE__};
    for (int64_t c0 = 0; c0 < nrhs; c0 += MAXR) {
        const int nc = (int)std::min<int64_t>(MAXR, nrhs - c0);
        SweepArgs<T> a;
        a.Y = Y + c0 * n;
        a.X = X + c0 * n;
        a.F = static_cast<T *>(ss.F);
        a.n = n;
        a.nrhs = nc;
        a.nblk = nblk;
        a.accumulate = accumulate;
        a.yflag = ss.flags;
        a.fflag = ss.flags + nblk;
        a.epoch = ++ss.epoch;
        const bool tagged = sizeof(T) == 4 && ss.tags != nullptr && nc <= ss.tag_cols && !tags_off;
        a.tY = tagged ? ss.tags : nullptr;
        a.tF = tagged ? ss.tags + (size_t)ss.tag_cols * n : nullptr;
        a.tag = 2u * a.epoch;
        launch_sweep<T, true>(tm, tDL, tML, use_inv, a, 1 + helpers, s);
        a.yflag = ss.flags + 2 * nblk;
        a.fflag = ss.flags + 3 * nblk;
        a.tag = 2u * a.epoch + 1u;
        launch_sweep<T, false>(tm, tDU, tMU, use_inv, a, 1 + helpers, s);
        g_launches += 2;
    }
}

template <typename T>
bool solve_fits(int64_t n)
{
    // the same helper-grid arithmetic as launch_lu_solve, checked before any launch
    const int nblk = (int)ceil_div(n, BS);
    int dev = 0, sms = 0;
    MP_CUDA(cudaGetDevice(&dev));
    MP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int dnmin = std::min(sweep_dn<T, 1>(), sweep_dn<T, MAXR>());
    static const int hmax = [] { const char *e = std::getenv("MP_SOLVE_HELPERS"); return e ? std::atoi(e) : 0; }();
    const int hcap = hmax > 0 ? std::min(hmax, sms - 1) : sms - 1;
    const int helpers = std::max(1, std::min(hcap, nblk - dnmin - 1));
    return ceil_div(std::max(0, nblk - dnmin - 1), helpers) <= SCfg<T>::MAXOWN;
}

template bool solve_fits<float>(int64_t);
template bool solve_fits<double>(int64_t);
template void launch_lu_solve<float>(const float *, int64_t, int64_t, int64_t, float *, double *, int,
                                     SolveScratch &, cudaStream_t, const float *);
template void launch_lu_solve<double>(const double *, int64_t, int64_t, int64_t, double *, double *, int,
                                      SolveScratch &, cudaStream_t, const float *);

}  // namespace mp
