// k_solve_mr.cu — K7 for several right-hand sides (2 <= nrhs <= 16 per launch): the triangular
// sweeps of Alg. 1 steps 2-3 / 5-6 with the inverted diagonal blocks of
// reading A-19, and step 7's binary64 update fused into the backward sweep.
//
// With one right-hand side the sweep is a latency chain (k_solve.cu: one chain CTA + helpers).  With
// 16 the work per 64-row block is 16x larger and that design ran ~10x off the HBM floor (ncu: 11x
// more instructions than FMAs, mostly polling).  This kernel is a right-looking blocked sweep with
// FIXED ROW OWNERSHIP: block I (64 rows) belongs to CTA I mod G for the whole sweep and lives in that
// CTA's shared memory, so every update of a block is made by one CTA in step order and no block ever
// changes hands.  Step t (block I = the t-th in dependency order):
//   * every CTA waits for Y_I's flag, stages Y_I and updates its own later blocks R_J -= T(J, I) Y_I;
//   * the owner of the NEXT block J = I +- 1 instead forms Y_J = P_J - M_J Y_I and publishes it (the
//     rows of Y, then an epoch-tagged flag) before anything else, where M_J = D_J T(J, I) comes with
//     the inverses (reading A-19) and P_J = D_J R'_J was computed while waiting (R'_J: every update
//     but step I's).  The dependent chain per step is one flag hand-off and ONE 64 x 64 x R product
//     on one SM.
// Tiles T(J, I) stream HBM -> shared memory with cp.async through a 6-slot ring, prefetched five work
// items ahead (they never depend on the chain); D / M tiles are loaded one solve ahead.
// HBM traffic per sweep: n^2/2 * 4 bytes of the factor (each tile once) + the D blocks + O(n R).
#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace mp {

namespace {

constexpr int MB = 64;            // block rows (= the A-19 inverse blocks)
constexpr int MNT = 256;          // threads: 64 rows x 4 right-hand-side groups
constexpr int TLD = MB + 4;       // padded shared row (conflict-free 16-byte row reads)
#ifndef MP_MR_SLOTS
#define MP_MR_SLOTS 6
#endif
constexpr int NSLOT = MP_MR_SLOTS;   // tile ring: NSLOT - 1 items in flight ahead of the one in use

struct MrArgs {
    const float *W;
    int64_t ldw, n;
    int nblk;
    const float *D;               // inverted diagonal blocks D_I, row-major 64 x 64 each
    const float *M;               // M_I = D_I T(I, I -+ 1) (reading A-19), same layout
    float *Y;                     // n x nrhs (ld n): rhs in, y / z out
    double *X;                    // backward: X (+)= z (ld n)
    int nrhs, accumulate;
    unsigned *flag;               // [nblk]
    unsigned epoch;
    // tagged exchange (nullptr: flags): Y of each solved block also written as 64-bit words {value
    // bits, tag} [nrhs][n]; a consumer that sees the tag sees the value (single-copy atomic 64-bit
    // access), so the hand-off needs no fence and no flag
    uint64_t *tY;
    unsigned tag;
};

__device__ __forceinline__ void cp16(float *dst, const float *src, bool ok)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const int sz = ok ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
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
__device__ __forceinline__ void st_release(unsigned *p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 64 x 64 tile at W rows [r0, r0+64), columns [c0, c0+64) -> padded shared tile (zero outside n)
__device__ __forceinline__ void load_tile(float *dst, const float *W, int64_t ldw, int64_t n, int64_t r0, int64_t c0)
{
    for (int e = threadIdx.x; e < MB * (MB / 4); e += MNT) {
        const int r = e >> 4, c4 = (e & 15) * 4;
        const bool ok = r0 + r < n && c0 + c4 < n;
        cp16(dst + r * TLD + c4, ok ? W + (r0 + r) * ldw + c0 + c4 : W, ok);
    }
}

// acc[i] += sum_k A[r][k] Ys[k][q*RQ + i] (A: padded 64 x 64 tile in shared, Ys: [64][R])
template <int R>
__device__ __forceinline__ void tile_times(const float *A, const float *Ys, int r, int q, float (&acc)[R / 4])
{
    constexpr int RQ = R / 4;
#pragma unroll 4
    for (int k = 0; k < MB; k += 4) {
        const float4 a = *reinterpret_cast<const float4 *>(A + r * TLD + k);
        const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float *yk = Ys + (k + u) * R + q * RQ;
#pragma unroll
            for (int i = 0; i < RQ; ++i) acc[i] = fmaf(av[u], yk[i], acc[i]);
        }
    }
}

template <bool LOWER, int R>
__global__ void __launch_bounds__(MNT, 1) mr_sweep_kernel(const MrArgs a)
{
    constexpr int RQ = R / 4;
    extern __shared__ __align__(16) float sm[];
    const int G = gridDim.x, g = blockIdx.x, nblk = a.nblk;
    const int nown = (nblk - g + G - 1) / G;                 // blocks g, g + G, ...
    const int64_t n = a.n;
    float *Rs = sm;                                          // [nown][64][R]
    // Y of the current / next step: Yb(0), Yb(1) — computed from `sm` (never through an array of
    // pointers: the compiler then keeps shared-memory instructions instead of generic ones)
    float *const Ybase = Rs + (size_t)nown * MB * R;         // [2][64][R]
    auto Yb = [&](int b) { return Ybase + b * (MB * R); };
    float *Pb = Ybase + 2 * MB * R;                          // [64][R]  D R' of the next block to solve
    float *ring = Pb + MB * R;                               // [NSLOT][64][TLD]
    float *Ds = ring + NSLOT * MB * TLD;                     // [64][TLD]
    float *Ms = Ds + MB * TLD;                               // [64][TLD]
    const int r = threadIdx.x & 63, q = threadIdx.x >> 6;
    // the k-th owned block in step order, its position
    auto owned = [&](int k) { return LOWER ? g + k * G : g + (nown - 1 - k) * G; };
    auto posof = [&](int I) { return LOWER ? I : nblk - 1 - I; };
    auto blk = [&](int t) { return LOWER ? t : nblk - 1 - t; };
    // first owned ordinal whose position is > t (positions increase with the ordinal)
    auto first_after = [&](int t) {
        int lo = 0, hi = nown;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (posof(owned(mid)) > t) hi = mid; else lo = mid + 1;
        }
        return lo;
    };
    // ---- owned right-hand sides into shared memory
    for (int k = 0; k < nown; ++k) {
        const int64_t i0 = (int64_t)owned(k) * MB;
        for (int e = threadIdx.x; e < MB * R; e += MNT) {
            const int c = e / MB, rr = e - c * MB;
            Rs[((size_t)k * MB + rr) * R + c] = (c < a.nrhs && i0 + rr < n) ? a.Y[(int64_t)c * n + i0 + rr] : 0.f;
        }
    }
    // ---- tile work items: (step t, owned ordinal k) with position(owned(k)) > t + 1, in step order
    // (the block at t + 1 takes step t's contribution through M instead: Y = D R' - M Y_t)
    struct Item { int t, k; };
    auto next_item = [&](Item it) -> Item {
        if (it.k + 1 < nown) return {it.t, it.k + 1};
        for (int t = it.t + 1; t < nblk; ++t) {
            const int k = first_after(t + 1);
            if (k < nown) return {t, k};
        }
        return {nblk, 0};
    };
    auto first_item = [&]() -> Item {
        for (int t = 0; t < nblk; ++t) {
            const int k = first_after(t + 1);
            if (k < nown) return {t, k};
        }
        return {nblk, 0};
    };
    auto issue = [&](Item it, int slot) {
        if (it.t < nblk) {
            const int I = blk(it.t), J = owned(it.k);
            load_tile(ring + slot * MB * TLD, a.W, a.ldw, n, (int64_t)J * MB, (int64_t)I * MB);
        }
        cp_commit();
    };
    // D and M of an owned block: plain loads, issued right after the previous solve (off the chain)
    auto load_dm = [&](int k) {
        const int64_t d0 = (int64_t)owned(k) * MB;
        for (int e = threadIdx.x; e < MB * (MB / 4); e += MNT) {
            const int rr = e >> 4, c4 = (e & 15) * 4;
            *reinterpret_cast<float4 *>(Ds + rr * TLD + c4) =
                __ldg(reinterpret_cast<const float4 *>(a.D + (d0 + rr) * MB + c4));
            *reinterpret_cast<float4 *>(Ms + rr * TLD + c4) =
                __ldg(reinterpret_cast<const float4 *>(a.M + (d0 + rr) * MB + c4));
        }
    };
    // P = D_k R'_k (R'_k: every update except the one of the step just before the block's own)
    auto make_p = [&](int k) {
        __syncthreads();
        float acc[RQ];
#pragma unroll
        for (int i = 0; i < RQ; ++i) acc[i] = 0.f;
        tile_times<R>(Ds, Rs + (size_t)k * MB * R, r, q, acc);
#pragma unroll
        for (int i = 0; i < RQ; ++i) Pb[r * R + q * RQ + i] = acc[i];
        __syncthreads();
    };
    // the block's rows of Y (and X) from Yo, then its flag
    auto publish = [&](int k, const float *Yo) {
        const int64_t i0 = (int64_t)owned(k) * MB;
#pragma unroll
        for (int i = 0; i < RQ; ++i) {
            const int c = q * RQ + i;
            if (c < a.nrhs && i0 + r < n) {
                const float v = Yo[r * R + c];
                a.Y[(int64_t)c * n + i0 + r] = v;
                if (a.tY != nullptr) st_tag(a.tY + (int64_t)c * n + i0 + r, v, a.tag);
                if (!LOWER) {
                    double *xp = a.X + (int64_t)c * n + i0 + r;
                    *xp = a.accumulate ? *xp + (double)v : (double)v;
                }
            }
        }
        if (a.tY != nullptr) return;                          // (tagged: the words are the hand-off)
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            st_release(a.flag + owned(k), a.epoch);
        }
    };
    int dk = 0;                                              // ordinal of the next owned block to solve
    if (nown > 0) load_dm(0);
    // the first NSLOT - 1 tiles (item i lives in ring slot i mod NSLOT)
    Item pf = first_item();
    int slot = 0;
    issue(pf, 0);
    for (int j = 1; j < NSLOT - 1; ++j) {
        pf = next_item(pf);
        issue(pf, j);
    }
    int yb = 0;                                              // Yb(yb) holds Y of the current step
    bool have = false;                                       // Yb(yb) already holds Y_blk(t) (solved here)
    if (nown > 0 && posof(owned(0)) == 0) {                  // the first block: Y = D R
        make_p(0);
#pragma unroll
        for (int i = 0; i < RQ; ++i) Yb(0)[r * R + q * RQ + i] = Pb[r * R + q * RQ + i];
        publish(0, Yb(0));
        dk = 1;
        have = true;
        if (dk < nown) load_dm(dk);
    }
    if (dk < nown && posof(owned(dk)) == 1) make_p(dk);     // its R' is the right-hand side itself
    for (int t = 0; t < nblk; ++t) {
        const int I = blk(t);
        const int k0 = first_after(t);
        if (k0 >= nown) break;                               // every owned block is solved
        if (!have) {
            const int64_t i0 = (int64_t)I * MB;
            if (a.tY != nullptr) {
                // poll the block's tagged words directly: one round trip brings the values with their tags
                constexpr int PE = MB * R / MNT;
                float v[PE];
                for (;;) {
                    bool ok = true;
#pragma unroll
                    for (int u = 0; u < PE; ++u) {
                        const int e = threadIdx.x + MNT * u, c = e / MB, rr = e - c * MB;
                        v[u] = 0.f;
                        if (c < a.nrhs && i0 + rr < n) {
                            const unsigned long long w = ld_tag(a.tY + (int64_t)c * n + i0 + rr);
                            v[u] = __uint_as_float((unsigned)w);
                            ok &= (unsigned)(w >> 32) == a.tag;
                        }
                    }
                    if (__syncthreads_and(ok)) break;
                }
#pragma unroll
                for (int u = 0; u < PE; ++u) {
                    const int e = threadIdx.x + MNT * u, c = e / MB, rr = e - c * MB;
                    Yb(yb)[rr * R + c] = v[u];
                }
            } else {
                if (threadIdx.x == 0) {
                    while (ld_relaxed(a.flag + I) != a.epoch) { }   // poll without invalidating L1 each time
                    (void)ld_acquire(a.flag + I);                      // then one acquire (orders the Y reads)
                }
                __syncthreads();
                for (int e = threadIdx.x; e < MB * R; e += MNT) {
                    const int c = e / MB, rr = e - c * MB;
                    Yb(yb)[rr * R + c] = (c < a.nrhs && i0 + rr < n) ? __ldcg(a.Y + (int64_t)c * n + i0 + rr) : 0.f;
                }
            }
        }
        __syncthreads();
        have = false;
        int kt = k0;
        if (posof(owned(k0)) == t + 1) {                     // the chain: Y_next = P - M Y_t, published now
            float acc[RQ];
#pragma unroll
            for (int i = 0; i < RQ; ++i) acc[i] = 0.f;
            tile_times<R>(Ms, Yb(yb), r, q, acc);
            float *Yn = Yb(yb ^ 1);
#pragma unroll
            for (int i = 0; i < RQ; ++i) Yn[r * R + q * RQ + i] = Pb[r * R + q * RQ + i] - acc[i];
            publish(k0, Yn);
            have = true;
            dk = k0 + 1;
            kt = k0 + 1;
            __syncthreads();                                 // Ms / Ds reads done
            if (dk < nown) load_dm(dk);
        }
        for (int k = kt; k < nown; ++k) {
            // item (t, k): tile T(owned(k), I) in ring slot `slot`; the item NSLOT - 1 ahead goes into
            // the slot consumed last (free since the barrier that ended it)
            pf = next_item(pf);
            issue(pf, slot == 0 ? NSLOT - 1 : slot - 1);
            cp_wait<NSLOT - 1>();                            // this item's group is complete
            __syncthreads();
            float acc[RQ];
#pragma unroll
            for (int i = 0; i < RQ; ++i) acc[i] = 0.f;
            tile_times<R>(ring + slot * MB * TLD, Yb(yb), r, q, acc);
            float *Rk = Rs + ((size_t)k * MB + r) * R + q * RQ;
#pragma unroll
            for (int i = 0; i < RQ; ++i) Rk[i] -= acc[i];
            __syncthreads();                                 // slot consumed
            slot = slot + 1 == NSLOT ? 0 : slot + 1;
            // the chain block of step t + 1 (this CTA's next solve): its R' is complete now — form
            // P before the step's other tiles (it is the one thing the next hand-off waits for here)
            if (k == dk && posof(owned(dk)) == t + 2) make_p(dk);
        }
        if (have) yb ^= 1;
    }
    cp_wait<0>();
}

template <bool LOWER, int R>
void launch_mr(const MrArgs &a, int grid, cudaStream_t s)
{
    const int nown = (a.nblk + grid - 1) / grid;
    const size_t smem = sizeof(float) * ((size_t)nown * MB * R + 3 * MB * R + (size_t)(NSLOT + 2) * MB * TLD);
    auto kern = mr_sweep_kernel<LOWER, R>;
    func_smem_once((const void *)kern, smem);
    void *args[] = {(void *)&a};
    MP_CUDA(cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(MNT), args, smem, s));
}

}  // namespace

bool mr_solve_supported(int64_t n, int64_t nrhs)
{
    static const bool off = std::getenv("MP_SOLVE_MR_OFF") != nullptr;
    if (off || nrhs < 2) return false;
    int dev = 0, sms = 0, maxsm = 0;
    MP_CUDA(cudaGetDevice(&dev));
    MP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MP_CUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const int64_t nblk = ceil_div(n, (int64_t)MB);
    const int grid = (int)std::min<int64_t>(sms, nblk);
    const int64_t nown = ceil_div(nblk, (int64_t)grid);
    const size_t smem = sizeof(float) * ((size_t)nown * MB * 16 + 3 * MB * 16 + (size_t)(NSLOT + 2) * MB * TLD);
    return smem <= (size_t)maxsm;
}

// Forward (unit lower, D_L) then backward (upper, D_U) sweeps for up to 16 right-hand sides.
void launch_lu_solve_mr(const float *W, int64_t ldw, int64_t n, int64_t nrhs, float *Y, double *X, int accumulate,
                        unsigned *flags, unsigned &epoch, const float *inv, cudaStream_t s, uint64_t *tags, int tag_cols)
{
    static const bool tags_off = std::getenv("MP_SOLVE_FLAGS") != nullptr;   // A/B: flag exchange
    const int nblk = (int)ceil_div(n, (int64_t)MB);
    const size_t blk = (size_t)nblk * MB * MB;
    int dev = 0, sms = 0;
    MP_CUDA(cudaGetDevice(&dev));
    MP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = std::min(sms, nblk);
    for (int64_t c0 = 0; c0 < nrhs; c0 += 16) {
        const int nc = (int)std::min<int64_t>(16, nrhs - c0);
        MrArgs a{W, ldw, n, nblk, inv, inv + blk, Y + c0 * n, X + c0 * n, nc, accumulate, flags, ++epoch, nullptr, 0u};
        if (tags != nullptr && nc <= tag_cols && !tags_off) {
            a.tY = tags;
            a.tag = 2u * a.epoch;
        }
        auto go = [&](auto lower) {
            constexpr bool L = decltype(lower)::value;
            if (nc <= 4) launch_mr<L, 4>(a, grid, s);
            else if (nc <= 8) launch_mr<L, 8>(a, grid, s);
            else launch_mr<L, 16>(a, grid, s);
        };
        go(std::true_type{});
        a.D = inv + 2 * blk;
        a.M = inv + 3 * blk;
        a.flag = flags + 2 * nblk;
        a.epoch = ++epoch;
        if (a.tY != nullptr) a.tag = 2u * a.epoch + 1u;
        go(std::false_type{});
        g_launches += 2;
    }
}

}  // namespace mp
