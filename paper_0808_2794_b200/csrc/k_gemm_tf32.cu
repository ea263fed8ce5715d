// k_gemm_tf32.cu — K5b: the trailing (Schur complement) update A22 <- A22 - L21 U12
// on the 5th-generation tensor cores, 3xTF32 (B:5's second variant).
//
// the O(n^3) step is the one that runs in single precision.
// Every operand x is split x = hi + lo with hi = rna_tf32(x), lo = rna_tf32(x - hi);
// the product L21 U12 is formed as Lhi Uhi + Lhi Ulo + Llo Uhi with FP32 accumulation
// in TMEM (the lo*lo term, ~2^-22 relative, is dropped), which keeps the update at
// binary32-level accuracy so refinement still reaches the binary64 criterion.
//
// Orientation: D^T = U12^T L21^T.  The MMA's M dimension (TMEM lanes) runs over the
// COLUMNS j of the row-major trailing matrix and its N dimension over the ROWS i, so in
// the epilogue each thread owns one column and a warp reads / writes 128 contiguous
// bytes per row: the read-modify-write of C is fully coalesced.
//
// Kernel structure (persistent, one CTA per SM, 384 threads):
//   warp 0     TMA producer: per 32-deep K chunk, 4 boxes (Uhi, Ulo 128x32; Lhi, Llo 256x32)
//              SWIZZLE_128B into a 2-stage shared-memory ring, mbarrier expect_tx
//   warp 1     MMA issuer (one thread): 4 k-steps x 3 tcgen05.mma.cta_group::1.kind::tf32
//              (M=128, N=256, K=8) per chunk, tcgen05.commit -> ring slot free / accumulator full
//   warp 2     TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warps 4..11 epilogue: tcgen05.ld 32x32b.x32 -> C -= D (coalesced RMW), accumulator free
// Two accumulators let the epilogue of tile t overlap the MMAs of tile t+1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "internal.h"

#ifndef MP_TF32_TERMS
#define MP_TF32_TERMS 3
#endif

namespace mp {

namespace {

constexpr int TM_COLS = 128;      // C columns per tile (MMA M, TMEM lanes)
constexpr int TM_ROWS = 256;      // C rows per tile (MMA N)
#ifndef MP_TF32_KC
#define MP_TF32_KC 32
#endif
// K chunk per ring stage: KC tf32 = KC*4-byte rows, one swizzle atom (SWIZZLE_64B for KC = 16,
// SWIZZLE_128B for KC = 32); the ring holds 192 KB either way (4 x 48 KB or 2 x 96 KB).
constexpr int KC = MP_TF32_KC;
constexpr int STAGES = KC == 16 ? 4 : 2;
constexpr uint32_t SW_BYTES = KC * 4;                 // swizzle atom row bytes
constexpr uint64_t SW_MODE = KC == 16 ? 4u : 2u;      // UMMA descriptor layout: 4 = SWIZZLE_64B, 2 = SWIZZLE_128B
constexpr int A_BYTES = TM_COLS * KC * 4;     // 16 KB
constexpr int B_BYTES = TM_ROWS * KC * 4;     // 32 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;   // 96 KB
constexpr int GT = 384;            // 4 role warps + 8 epilogue warps

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// The same box written into the shared memory of every CTA in `mask` (same CTA-relative offset),
// completing the bytes on each destination CTA's mbarrier at the same offset.
__device__ __forceinline__ void tma_load_2d_mc(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, uint16_t mask)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major operand, swizzled rows of SW_BYTES, 8-row groups
// 8 * SW_BYTES apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);          // start address
    d |= (uint64_t)1u << 16;                          // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)((8u * SW_BYTES) >> 4) << 32;      // stride byte offset: 8 rows x SW_BYTES
    d |= (uint64_t)1u << 46;                          // descriptor version (sm_100)
    d |= SW_MODE << 61;                               // layout: swizzle mode
    return d;
}

// Instruction descriptor: kind::tf32, D fp32, A/B tf32 K-major, M = 128, N = 256.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TM_ROWS >> 3) << 17) |
                            ((uint32_t)(TM_COLS >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// the same arrive on the mbarrier at this offset in every CTA of `mask`
__device__ __forceinline__ void umma_commit_mc(uint64_t *bar, uint16_t mask)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "h"(mask)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32])
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16])
{
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// CS > 1: clusters of CS CTAs take CS neighbouring tiles of one tile row (same L21 rows): each
// CTA loads its own U box and 1/CS of the L boxes, multicast into every CTA of the cluster, so a
// CTA pulls (128 + 256 / CS) instead of 384 operand rows per K chunk through L2 (the kernel runs
// at the L2 slices' throughput cap with CS = 1).  A ring slot is refilled
// only when every CTA of the cluster has consumed it: the MMA issuers commit to the slot's
// "empty" mbarrier of all CS CTAs (count CS).
template <bool LOWER, int CS>
__global__ void __launch_bounds__(GT, 1)
gemm_3xtf32_kernel(const __grid_constant__ CUtensorMap tmUh, const __grid_constant__ CUtensorMap tmUl,
                   const __grid_constant__ CUtensorMap tmLh, const __grid_constant__ CUtensorMap tmLl,
                   float *__restrict__ C, int64_t ldc, int M, int N, int K, int terms)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte aligned ring (SWIZZLE_128B atoms)
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_n = (N + TM_COLS - 1) / TM_COLS, tiles_m = (M + TM_ROWS - 1) / TM_ROWS;
    // tile groups: CS neighbouring tiles of a tile row, one per CTA of the cluster (a CTA whose
    // tile lies beyond the last column still loads its share of L and runs the protocol; its U
    // boxes are out of range (zero-filled) and its epilogue stores nothing)
    const int tiles_ng = (tiles_n + CS - 1) / CS;
    const int ntiles = tiles_ng * tiles_m;
    const int nk = (K + KC - 1) / KC;
    const int crank = CS > 1 ? (int)cluster_ctarank() : 0;
    const int first = (int)blockIdx.x / CS, step = (int)gridDim.x / CS;
    constexpr uint16_t kMask = (uint16_t)((1u << CS) - 1u);
    // LOWER (the SPD path's SYRK, C square with its diagonal at i == j): tiles entirely above
    // the diagonal (every row index below every column index) are skipped by all three roles;
    // a group is skipped when its first (leftmost) tile is — the others lie further right
    auto skip_tile = [&](int tm, int tn) {
        if constexpr (!LOWER) return false;
        return tm * TM_ROWS + TM_ROWS - 1 < tn * TM_COLS;
    };
    auto skip = [&](int t) { return skip_tile(t / tiles_ng, (t % tiles_ng) * CS); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], CS); }
        for (int a = 0; a < 2; ++a) { mbar_init(&acc_full[a], 1); mbar_init(&acc_empty[a], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CS > 1) cluster_sync_all();       // every CTA's mbarriers exist before any remote signal
    tc_fence_after();
    const uint32_t tmem_base = tmem_base_sh;
    // PDL: barrier init and the TMEM allocation above overlap the previous kernel; no early
    // trigger (a dependent parked on the update partition for the whole GEMM would only
    // hold resources)
    pdl_wait();

    if (warp == 0) {
        // ================= TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            // this CTA's share of the L boxes: rows [lr0, lr0 + TM_ROWS / CS) of the tile row, at
            // byte offset lb0 of the B operand (8-row swizzle atoms: the shares stack contiguously)
            constexpr int LROWS = TM_ROWS / CS, LBYTES = B_BYTES / CS;
            const int lr0 = crank * LROWS, lb0 = crank * LBYTES;
            auto load_l = [&](unsigned char *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
                if constexpr (CS > 1) tma_load_2d_mc(dst + lb0, map, bar, c0, c1 + lr0, kMask);
                else tma_load_2d(dst, map, bar, c0, c1);
            };
            for (int t = first; t < ntiles; t += step) {
                if (skip(t)) continue;
                const int tn = (t % tiles_ng) * CS + crank, tm = t / tiles_ng;
                for (int kc = 0; kc < nk; ++kc) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);          // (CS > 1: consumed by every CTA of the cluster)
                    unsigned char *st = smem + stage * STAGE_BYTES;
                    if (terms == 1) {                                 // 1xTF32 (NEXT-2): the hi boxes only
                        mbar_expect_tx(&full_bar[stage], A_BYTES + B_BYTES);
                        tma_load_2d(st, &tmUh, &full_bar[stage], kc * KC, tn * TM_COLS);
                        load_l(st + 2 * A_BYTES, &tmLh, &full_bar[stage], kc * KC, tm * TM_ROWS);
                    } else {
                        mbar_expect_tx(&full_bar[stage], STAGE_BYTES);
                        tma_load_2d(st, &tmUh, &full_bar[stage], kc * KC, tn * TM_COLS);
                        tma_load_2d(st + A_BYTES, &tmUl, &full_bar[stage], kc * KC, tn * TM_COLS);
                        load_l(st + 2 * A_BYTES, &tmLh, &full_bar[stage], kc * KC, tm * TM_ROWS);
                        load_l(st + 2 * A_BYTES + B_BYTES, &tmLl, &full_bar[stage], kc * KC, tm * TM_ROWS);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t acc_phase[2] = {0, 0};
            int a = 0;
            for (int t = first; t < ntiles; t += step) {
                if (skip(t)) continue;
                mbar_wait(&acc_empty[a], acc_phase[a] ^ 1);           // epilogue drained this accumulator
                tc_fence_after();
                const uint32_t tacc = tmem_base + (uint32_t)(a * TM_ROWS);
                for (int kc = 0; kc < nk; ++kc) {
                    mbar_wait(&full_bar[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
                    const uint32_t sAh = sa, sAl = sa + A_BYTES, sBh = sa + 2 * A_BYTES, sBl = sa + 2 * A_BYTES + B_BYTES;
#pragma unroll
                    for (int ks = 0; ks < KC / 8; ++ks) {
                        const uint32_t off = ks * 32;                  // 8 tf32 = 32 B along the swizzled row
                        const uint64_t dAh = umma_desc_sw128(sAh + off), dAl = umma_desc_sw128(sAl + off);
                        const uint64_t dBh = umma_desc_sw128(sBh + off), dBl = umma_desc_sw128(sBl + off);
                        if (terms == 1) {                                 // 1xTF32: hi*hi only
                            umma_tf32(tacc, dAh, dBh, (kc | ks) ? 1u : 0u);
                            continue;
                        }
                        if (MP_TF32_TERMS == 4 || terms == 4) {
                            umma_tf32(tacc, dAl, dBl, (kc | ks) ? 1u : 0u);  // lo*lo (4xTF32)
                            umma_tf32(tacc, dAl, dBh, 1u);
                        } else {
                            umma_tf32(tacc, dAl, dBh, (kc | ks) ? 1u : 0u);  // small terms first
                        }
                        umma_tf32(tacc, dAh, dBl, 1u);
                        umma_tf32(tacc, dAh, dBh, 1u);
                    }
                    // ring slot free when these MMAs finish (in every CTA of the cluster: they all
                    // multicast into it)
                    if constexpr (CS > 1) umma_commit_mc(&empty_bar[stage], kMask);
                    else umma_commit(&empty_bar[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                umma_commit(&acc_full[a]);                             // accumulator ready for the epilogue
                acc_phase[a] ^= 1;
                a ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ================= epilogue: C[i][j] -= D^T[j][i]
        // 8 warps: TMEM lane quarter q = warp % 4 (columns j), row half h (TMEM columns).
        // C rows are loaded one 32-row group ahead (the first group before the accumulator
        // is ready), so each SM keeps ~64 KB of C loads in flight.
        const int q = warp & 3, h = (warp - 4) >> 2;
        uint32_t acc_phase[2] = {0, 0};
        int a = 0;
        for (int t = first; t < ntiles; t += step) {
            if (skip(t)) continue;
            const int tn = (t % tiles_ng) * CS + crank, tm = t / tiles_ng;
            const int j = tn * TM_COLS + q * 32 + lane;
            const int i0 = tm * TM_ROWS + h * (TM_ROWS / 2);
            // (a tile of the group that lies above the diagonal, or beyond the last column, stores nothing)
            const bool jv = j < N && !(CS > 1 && skip_tile(tm, tn));
            constexpr int GR = 16, NG = TM_ROWS / 2 / GR, PD = 2;   // 16-row groups, 2 groups ahead
            float cb[PD + 1][GR];
            const int nrow_ok = jv ? M : 0;                        // rows i < nrow_ok exist
            auto load_group = [&](float (&dst)[GR], int ib) {
                const float *cp = C + (int64_t)ib * ldc + j;
#pragma unroll
                for (int rr = 0; rr < GR; ++rr) dst[rr] = (ib + rr < nrow_ok) ? __ldcs(cp + (int64_t)rr * ldc) : 0.f;
            };
#pragma unroll
            for (int g = 0; g < PD; ++g) load_group(cb[g], i0 + GR * g);
            mbar_wait(&acc_full[a], acc_phase[a]);
            __syncwarp();                                          // lanes leave the wait loop together
            acc_phase[a] ^= 1;
            tc_fence_after();
            const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * TM_ROWS + h * (TM_ROWS / 2));
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                if (g + PD < NG) load_group(cb[(g + PD) % (PD + 1)], i0 + GR * (g + PD));
                float v[GR];
                tmem_ld16(tacc + (uint32_t)(GR * g), v);
                const int ib = i0 + GR * g;
                float *cp = C + (int64_t)ib * ldc + j;
#pragma unroll
                for (int rr = 0; rr < GR; ++rr)
                    if (ib + rr < nrow_ok) __stcs(cp + (int64_t)rr * ldc, cb[g % (PD + 1)][rr] - v[rr]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[a]);
            a ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CS > 1) cluster_sync_all();       // no CTA leaves while a peer may still signal its mbarriers
    tc_fence_after();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

// ---- CTA-pair variant (tcgen05 cta_group::2).  Two CTAs of one TPC take two neighbouring tiles of
// a tile row as ONE 256 (columns, MMA M) x 256 (rows, MMA N) instruction tile: each CTA stages its
// own 128 U rows and HALF of the L rows (128), the tensor core reads the other half from the peer's
// shared memory, and each CTA's TMEM receives its own 128 x 256 accumulator.  A CTA therefore pulls
// 256 instead of 384 operand rows per K chunk over the crossbar (64 KB per stage, 3 stages) — the
// single-CTA kernel runs at the L2 slices' throughput cap, and TMA multicast
// (CS above) does not lower the bytes delivered per SM.  Only the leader (rank 0) issues MMAs and
// commits; its "full" mbarrier collects both CTAs' TMA bytes, its "accumulator empty" mbarrier
// both CTAs' epilogue warps; commits are multicast to both CTAs' "slot empty" / "accumulator full".
constexpr int P_STAGE_BYTES = 2 * A_BYTES + B_BYTES;       // Uhi, Ulo (128 rows) + Lhi, Llo halves (128 rows)
constexpr int P_STAGES = 3;
constexpr uint32_t kIdescPair = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TM_ROWS >> 3) << 17) |
                                ((uint32_t)((2 * TM_COLS) >> 4) << 24);

__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map, uint32_t leader_bar, int c0, int c1)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
        : "memory");
}
__device__ __forceinline__ void umma_tf32_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdescPair), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "h"((uint16_t)3)
                 : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t raddr)
{
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr) : "memory");
}

template <bool LOWER>
__global__ void __launch_bounds__(GT, 1)
gemm_3xtf32_pair_kernel(const __grid_constant__ CUtensorMap tmUh, const __grid_constant__ CUtensorMap tmUl,
                        const __grid_constant__ CUtensorMap tmLh, const __grid_constant__ CUtensorMap tmLl,
                        float *__restrict__ C, int64_t ldc, int M, int N, int K, int terms)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full_bar[P_STAGES], empty_bar[P_STAGES], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_n = (N + TM_COLS - 1) / TM_COLS, tiles_m = (M + TM_ROWS - 1) / TM_ROWS;
    const int tiles_ng = (tiles_n + 1) / 2;
    const int ntiles = tiles_ng * tiles_m;
    const int nk = (K + KC - 1) / KC;
    const int crank = (int)cluster_ctarank();
    const bool leader = crank == 0;
    const int first = (int)blockIdx.x / 2, step = (int)gridDim.x / 2;
    auto skip_tile = [&](int tm, int tn) {
        if constexpr (!LOWER) return false;
        return tm * TM_ROWS + TM_ROWS - 1 < tn * TM_COLS;
    };
    // Tile order: column bands of bw tile pairs, swept row by row, so that a band's U boxes
    // (bw x 256 columns x K x 8 B, kept to ~32 MB: half of L2 is what one die's SMs see) stay in L2
    // while the trailing matrix streams through once.  (Row-major order over all tile columns
    // re-reads U from HBM on every tile row once 2 N K 4 B exceeds that: ncu at M = N = 48128,
    // K = 512 showed 38.4 GB of DRAM reads against 9.7 GB algorithmic.)
    // (LOWER keeps row-major order, bw = all tile pairs of a row: with a fixed tile column per cluster
    // the clusters left of the diagonal would do all the rows and those on the right almost none —
    // SPD n = 16384 37.3 -> 40.1 ms with bands)
    const int bw = LOWER ? max(1, tiles_ng) : max(1, min(step, (32 << 20) / (2 * TM_COLS * 8 * max(K, 1))));
    const int nfull = tiles_ng / bw, rem = tiles_ng - nfull * bw, per_band = bw * tiles_m;
    auto tile_of = [&](int t, int &tm, int &g) {
        if (t < nfull * per_band) {
            const int band = t / per_band, r = t - band * per_band;
            tm = r / bw;
            g = band * bw + (r - tm * bw);
        } else {
            const int r = t - nfull * per_band;
            tm = r / rem;
            g = nfull * bw + (r - tm * rem);
        }
    };
    auto skip = [&](int t) { int tm, g; tile_of(t, tm, g); return skip_tile(tm, g * 2); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < P_STAGES; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&acc_full[a], 1); mbar_init(&acc_empty[a], 16); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = tmem_base_sh;
    pdl_wait();

    if (warp == 0) {
        // ================= TMA producer (both CTAs): bytes complete on the LEADER's full barrier
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const int lr0 = crank * (TM_ROWS / 2);
            for (int t = first; t < ntiles; t += step) {
                if (skip(t)) continue;
                int tm, g;
                tile_of(t, tm, g);
                const int tn = g * 2 + crank;
                for (int kc = 0; kc < nk; ++kc) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    unsigned char *st = smem + stage * P_STAGE_BYTES;
                    const uint32_t lbar = mapa_u32(smem_u32(&full_bar[stage]), 0);
                    if (terms == 1) {
                        if (leader) mbar_expect_tx(&full_bar[stage], 2 * (A_BYTES + B_BYTES / 2));
                        tma_load_2d_pair(st, &tmUh, lbar, kc * KC, tn * TM_COLS);
                        tma_load_2d_pair(st + 2 * A_BYTES, &tmLh, lbar, kc * KC, tm * TM_ROWS + lr0);
                    } else {
                        if (leader) mbar_expect_tx(&full_bar[stage], 2 * P_STAGE_BYTES);
                        tma_load_2d_pair(st, &tmUh, lbar, kc * KC, tn * TM_COLS);
                        tma_load_2d_pair(st + A_BYTES, &tmUl, lbar, kc * KC, tn * TM_COLS);
                        tma_load_2d_pair(st + 2 * A_BYTES, &tmLh, lbar, kc * KC, tm * TM_ROWS + lr0);
                        tma_load_2d_pair(st + 2 * A_BYTES + B_BYTES / 2, &tmLl, lbar, kc * KC, tm * TM_ROWS + lr0);
                    }
                    if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (leader CTA only)
        if (lane == 0 && leader) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t acc_phase[2] = {0, 0};
            int a = 0;
            for (int t = first; t < ntiles; t += step) {
                if (skip(t)) continue;
                mbar_wait(&acc_empty[a], acc_phase[a] ^ 1);           // both CTAs' epilogues drained it
                tc_fence_after();
                const uint32_t tacc = tmem_base + (uint32_t)(a * TM_ROWS);
                for (int kc = 0; kc < nk; ++kc) {
                    mbar_wait(&full_bar[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * P_STAGE_BYTES);
                    const uint32_t sAh = sa, sAl = sa + A_BYTES, sBh = sa + 2 * A_BYTES, sBl = sa + 2 * A_BYTES + B_BYTES / 2;
#pragma unroll
                    for (int ks = 0; ks < KC / 8; ++ks) {
                        const uint32_t off = ks * 32;
                        const uint64_t dAh = umma_desc_sw128(sAh + off), dAl = umma_desc_sw128(sAl + off);
                        const uint64_t dBh = umma_desc_sw128(sBh + off), dBl = umma_desc_sw128(sBl + off);
                        if (terms == 1) {
                            umma_tf32_pair(tacc, dAh, dBh, (kc | ks) ? 1u : 0u);
                            continue;
                        }
                        if (MP_TF32_TERMS == 4 || terms == 4) {
                            umma_tf32_pair(tacc, dAl, dBl, (kc | ks) ? 1u : 0u);
                            umma_tf32_pair(tacc, dAl, dBh, 1u);
                        } else {
                            umma_tf32_pair(tacc, dAl, dBh, (kc | ks) ? 1u : 0u);
                        }
                        umma_tf32_pair(tacc, dAh, dBl, 1u);
                        umma_tf32_pair(tacc, dAh, dBh, 1u);
                    }
                    umma_commit_pair(&empty_bar[stage]);               // slot free in both CTAs
                    if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
                }
                umma_commit_pair(&acc_full[a]);                        // accumulator ready in both CTAs
                acc_phase[a] ^= 1;
                a ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ================= epilogue (both CTAs, their own TMEM): C[i][j] -= D^T[j][i]
        const int q = warp & 3, h = (warp - 4) >> 2;
        uint32_t acc_phase[2] = {0, 0};
        int a = 0;
        const uint32_t lempty[2] = {mapa_u32(smem_u32(&acc_empty[0]), 0), mapa_u32(smem_u32(&acc_empty[1]), 0)};
        for (int t = first; t < ntiles; t += step) {
            if (skip(t)) continue;
            int tm, g;
            tile_of(t, tm, g);
            const int tn = g * 2 + crank;
            const int j = tn * TM_COLS + q * 32 + lane;
            const int i0 = tm * TM_ROWS + h * (TM_ROWS / 2);
            const bool jv = j < N && !skip_tile(tm, tn);
            constexpr int GR = 16, NG = TM_ROWS / 2 / GR, PD = 2;
            float cb[PD + 1][GR];
            const int nrow_ok = jv ? M : 0;
            auto load_group = [&](float (&dst)[GR], int ib) {
                const float *cp = C + (int64_t)ib * ldc + j;
#pragma unroll
                for (int rr = 0; rr < GR; ++rr) dst[rr] = (ib + rr < nrow_ok) ? __ldcs(cp + (int64_t)rr * ldc) : 0.f;
            };
#pragma unroll
            for (int g = 0; g < PD; ++g) load_group(cb[g], i0 + GR * g);
            mbar_wait(&acc_full[a], acc_phase[a]);
            __syncwarp();
            acc_phase[a] ^= 1;
            tc_fence_after();
            const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * TM_ROWS + h * (TM_ROWS / 2));
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                if (g + PD < NG) load_group(cb[(g + PD) % (PD + 1)], i0 + GR * (g + PD));
                float v[GR];
                tmem_ld16(tacc + (uint32_t)(GR * g), v);
                const int ib = i0 + GR * g;
                float *cp = C + (int64_t)ib * ldc + j;
#pragma unroll
                for (int rr = 0; rr < GR; ++rr)
                    if (ib + rr < nrow_ok) __stcs(cp + (int64_t)rr * ldc, cb[g % (PD + 1)][rr] - v[rr]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(lempty[a]);
            a ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

// ---- split: Lh/Ll[i][k] = split(L21(i, k)),  Uh/Ul[j][k] = split(U12(k, j)) (transposed)
__device__ __forceinline__ float rna_tf32(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__global__ void split_rows_kernel(const float *__restrict__ A, int64_t lda, int M, int K,
                                  float *__restrict__ hi, float *__restrict__ lo, int kp)
{
    pdl_wait();
    pdl_trigger();
    const int64_t tot = (int64_t)M * kp;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / kp;
        const int k = (int)(t - i * kp);
        const float x = k < K ? A[i * lda + k] : 0.f;
        const float h = rna_tf32(x);
        hi[t] = h;
        lo[t] = rna_tf32(x - h);
    }
}

__global__ void split_cols_T_kernel(const float *__restrict__ B, int64_t ldb, int N, int K,
                                    float *__restrict__ hi, float *__restrict__ lo, int kp)
{
    __shared__ float tile[32][33];
    pdl_wait();
    pdl_trigger();
    const int jb = blockIdx.x * 32, kb = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {               // read U12(kb + r, jb + tx): coalesced
        const int k = kb + r, j = jb + threadIdx.x;
        tile[r][threadIdx.x] = (k < K && j < N) ? B[(int64_t)k * ldb + j] : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {               // write [j][k]: coalesced along k
        const int j = jb + r, k = kb + threadIdx.x;
        if (j < N && k < kp) {
            const float x = tile[threadIdx.x][r];
            const float h = rna_tf32(x);
            hi[(int64_t)j * kp + k] = h;
            lo[(int64_t)j * kp + k] = rna_tf32(x - h);
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

void encode_kmajor(CUtensorMap *map, const float *base, int rows, int kdim, int kp, int box_rows)
{
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        MP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) throw CudaError{cudaErrorNotSupported, "cuTensorMapEncodeTiled", __LINE__};
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t gdim[2] = {(cuuint64_t)kdim, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)kp * sizeof(float)};
    cuuint32_t box[2] = {(cuuint32_t)KC, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), gdim, gstride, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, KC == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError{cudaErrorInvalidValue, "cuTensorMapEncodeTiled failed", __LINE__};
}


// Cluster mode of the tensor-core update: MP_GEMM_CLUSTER = 8 (default) the CTA-pair kernel
// (cta_group::2), 2 / 4 the multicast clusters of the single-CTA kernel (measured: C4's update
// 555 ms single CTAs, 542 ms multicast 2, 585 ms multicast 4, 518 ms CTA pairs), 1 single CTAs —
// for launches of at least MP_GEMM_CLUSTER_WAVES (default 2) waves of tiles; smaller launches (the
// in-panel levels, the look-ahead's next-panel columns) keep single CTAs.  set_gemm_tf32_cluster()
// overrides it for the calling thread (kernel tests).
thread_local int g_cluster_force = 0;

int pick_cluster(int64_t ntiles, int num_sms)
{
    if (g_cluster_force > 0) return g_cluster_force >= 8 ? 8 : (g_cluster_force >= 4 ? 4 : (g_cluster_force >= 2 ? 2 : 1));
    static const int env_cs = [] { const char *e = std::getenv("MP_GEMM_CLUSTER"); return e ? std::atoi(e) : 8; }();
    static const int waves = [] { const char *e = std::getenv("MP_GEMM_CLUSTER_WAVES"); return e ? std::atoi(e) : 2; }();
    if (env_cs <= 1 || ntiles < (int64_t)waves * num_sms) return 1;
    return env_cs >= 8 ? 8 : (env_cs >= 4 ? 4 : 2);       // 8: the CTA-pair kernel (cta_group::2)
}

// Clusters of this kernel that can be resident at once on the SMs stream s can use (its green
// context's partition), cached per (kernel, SM budget): a persistent grid larger than that would
// run its surplus clusters after the others have finished all their tiles.
template <bool LOWER, int CS>
int resident_clusters(int num_sms, size_t smem, cudaStream_t s)
{
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;
    int dev = 0;
    MP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, num_sms});
    if (it != cache.end()) return it->second;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(num_sms / CS * CS));
    cfg.blockDim = dim3(GT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, (const void *)gemm_3xtf32_kernel<LOWER, CS>, &cfg) != cudaSuccess || ncl <= 0) {
        cudaGetLastError();
        ncl = num_sms / CS;
    }
    ncl = std::min(ncl, num_sms / CS);
    if (std::getenv("MP_GEMM_CLUSTER_DEBUG"))
        std::fprintf(stderr, "[mp] gemm_3xtf32 cluster %d: %d resident clusters on a %d-SM budget\n", CS, ncl, num_sms);
    cache[{dev, num_sms}] = ncl;
    return ncl;
}

template <bool LOWER, int CS>
void launch_tc_cs(const float *Uh, const float *Ul, const float *Lh, const float *Ll, float *C, int64_t ldc, int64_t M,
                  int64_t N, int64_t K, int kp, int num_sms, cudaStream_t s, int terms)
{
    CUtensorMap mUh, mUl, mLh, mLl;
    encode_kmajor(&mUh, Uh, (int)N, (int)K, kp, TM_COLS);
    encode_kmajor(&mUl, Ul, (int)N, (int)K, kp, TM_COLS);
    encode_kmajor(&mLh, Lh, (int)M, (int)K, kp, TM_ROWS / CS);
    encode_kmajor(&mLl, Ll, (int)M, (int)K, kp, TM_ROWS / CS);
    const int64_t ngroups = ceil_div(ceil_div(N, (int64_t)TM_COLS), (int64_t)CS) * ceil_div(M, (int64_t)TM_ROWS);
    const size_t smem = (size_t)STAGES * STAGE_BYTES + 1024;
    func_smem_once((const void *)gemm_3xtf32_kernel<LOWER, CS>, smem);
    if constexpr (CS == 1) {
        const int grid = (int)std::min<int64_t>(ngroups, num_sms);
        launch_ex(gemm_3xtf32_kernel<LOWER, 1>, dim3(grid), dim3(GT), smem, s, nullptr, mUh, mUl, mLh, mLl, C, ldc,
                  (int)M, (int)N, (int)K, terms);
    } else {
        const int ncl = (int)std::min<int64_t>(ngroups, resident_clusters<LOWER, CS>(num_sms, smem, s));
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = CS; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
        launch_ex(gemm_3xtf32_kernel<LOWER, CS>, dim3(ncl * CS), dim3(GT), smem, s, &at, mUh, mUl, mLh, mLl, C, ldc,
                  (int)M, (int)N, (int)K, terms);
    }
}

// the CTA-pair kernel (cta_group::2): L boxes of 128 rows, clusters of 2
template <bool LOWER>
void launch_tc_pair(const float *Uh, const float *Ul, const float *Lh, const float *Ll, float *C, int64_t ldc, int64_t M,
                    int64_t N, int64_t K, int kp, int num_sms, cudaStream_t s, int terms)
{
    CUtensorMap mUh, mUl, mLh, mLl;
    encode_kmajor(&mUh, Uh, (int)N, (int)K, kp, TM_COLS);
    encode_kmajor(&mUl, Ul, (int)N, (int)K, kp, TM_COLS);
    encode_kmajor(&mLh, Lh, (int)M, (int)K, kp, TM_ROWS / 2);
    encode_kmajor(&mLl, Ll, (int)M, (int)K, kp, TM_ROWS / 2);
    const int64_t ngroups = ceil_div(ceil_div(N, (int64_t)TM_COLS), (int64_t)2) * ceil_div(M, (int64_t)TM_ROWS);
    const size_t smem = (size_t)P_STAGES * P_STAGE_BYTES + 1024;
    func_smem_once((const void *)gemm_3xtf32_pair_kernel<LOWER>, smem);
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;
    int dev = 0, ncl = 0;
    MP_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find({dev, num_sms});
        if (it == cache.end()) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(num_sms / 2 * 2));
            cfg.blockDim = dim3(GT);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute a1[1];
            a1[0].id = cudaLaunchAttributeClusterDimension;
            a1[0].val.clusterDim.x = 2; a1[0].val.clusterDim.y = 1; a1[0].val.clusterDim.z = 1;
            cfg.attrs = a1;
            cfg.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&ncl, (const void *)gemm_3xtf32_pair_kernel<LOWER>, &cfg) != cudaSuccess || ncl <= 0) {
                cudaGetLastError();
                ncl = num_sms / 2;
            }
            ncl = std::min(ncl, num_sms / 2);
            it = cache.emplace(std::make_pair(dev, num_sms), ncl).first;
        }
        ncl = it->second;
    }
    ncl = (int)std::min<int64_t>(ngroups, ncl);
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 2; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    launch_ex(gemm_3xtf32_pair_kernel<LOWER>, dim3(ncl * 2), dim3(GT), smem, s, &at, mUh, mUl, mLh, mLl, C, ldc, (int)M,
              (int)N, (int)K, terms);
}

template <bool LOWER>
void launch_tc(const float *Uh, const float *Ul, const float *Lh, const float *Ll, float *C, int64_t ldc, int64_t M,
               int64_t N, int64_t K, int kp, int num_sms, cudaStream_t s, int terms)
{
    const int64_t ntiles = ceil_div(N, (int64_t)TM_COLS) * ceil_div(M, (int64_t)TM_ROWS);
    const int cs = num_sms >= 4 ? pick_cluster(ntiles, num_sms) : 1;
    if (cs == 8) launch_tc_pair<LOWER>(Uh, Ul, Lh, Ll, C, ldc, M, N, K, kp, num_sms, s, terms);
    else if (cs == 4) launch_tc_cs<LOWER, 4>(Uh, Ul, Lh, Ll, C, ldc, M, N, K, kp, num_sms, s, terms);
    else if (cs == 2) launch_tc_cs<LOWER, 2>(Uh, Ul, Lh, Ll, C, ldc, M, N, K, kp, num_sms, s, terms);
    else launch_tc_cs<LOWER, 1>(Uh, Ul, Lh, Ll, C, ldc, M, N, K, kp, num_sms, s, terms);
}

}  // namespace

void set_gemm_tf32_cluster(int cs) { g_cluster_force = cs; }

size_t tf32_scratch_floats(int64_t n, int nbmax)
{
    const int64_t kp = round_up(nbmax, 4);
    return (size_t)4 * (size_t)n * (size_t)kp + 4096;
}

void launch_gemm_ops_3xtf32(const float *A, int64_t lda, const float *B, int64_t ldb, float *C, int64_t ldc, int64_t M,
                            int64_t N, int64_t K, float *scratch, int num_sms, cudaStream_t s, bool reuse_a, int terms, bool reuse_b,
                            float *bscratch)
{
    if (M <= 0 || N <= 0 || K <= 0) return;
    const int kp = (int)round_up(K, 4);
    float *Lh = scratch, *Ll = Lh + (size_t)M * kp;
    // bscratch: the B operand's split lives in its own buffer (the look-ahead's next-panel update on
    // the panel stream shares the A split with the update stream but not the B split)
    float *Uh = bscratch ? bscratch : Ll + (size_t)M * kp, *Ul = Uh + (size_t)N * kp;
    {
        const int64_t tot = M * kp;
        if (!reuse_a)                       // reuse_a: Lh/Ll already hold this A (same M, K, scratch)
            launch_ex(split_rows_kernel, dim3((unsigned)std::min<int64_t>(ceil_div(tot, 256), 4096)), dim3(256), 0, s,
                      nullptr, A, lda, (int)M, (int)K, Lh, Ll, kp);
        dim3 g((unsigned)ceil_div(N, 32), (unsigned)ceil_div(kp, 32));
        if (!reuse_b)                       // reuse_b: Uh/Ul written by the TRSM that produced B
            launch_ex(split_cols_T_kernel, g, dim3(32, 8), 0, s, nullptr, B, ldb, (int)N, (int)K, Uh, Ul, kp);
    }
    launch_tc<false>(Uh, Ul, Lh, Ll, C, ldc, M, N, K, kp, num_sms, s, terms);
}

// SPD path: C[M x M] (lower tiles) -= L21 L21^T with L21 = A[M x K] (row-major, lda).  The B operand of
// the 3xTF32 kernel is K-major U^T = L21 itself, so one hi/lo split of L21 serves as both operands.
void launch_syrk_lower_3xtf32(const float *A, int64_t lda, float *C, int64_t ldc, int64_t M, int64_t K, float *scratch,
                              int num_sms, cudaStream_t s, int terms)
{
    if (M <= 0 || K <= 0) return;
    const int kp = (int)round_up(K, 4);
    float *Lh = scratch, *Ll = Lh + (size_t)M * kp;
    const int64_t tot = M * kp;
    launch_ex(split_rows_kernel, dim3((unsigned)std::min<int64_t>(ceil_div(tot, 256), 4096)), dim3(256), 0, s, nullptr,
              A, lda, (int)M, (int)K, Lh, Ll, kp);
    launch_tc<true>(Lh, Ll, Lh, Ll, C, ldc, M, M, K, kp, num_sms, s, terms);
}

// The hi/lo split of the A operand alone (M x K rows at A, lda) into scratch, in the layout
// launch_gemm_ops_3xtf32 expects (so a later call with reuse_a = true and the same M, K uses it).
void launch_split_a_3xtf32(const float *A, int64_t lda, int64_t M, int64_t K, float *scratch, cudaStream_t s)
{
    if (M <= 0 || K <= 0) return;
    const int kp = (int)round_up(K, 4);
    const int64_t tot = M * kp;
    launch_ex(split_rows_kernel, dim3((unsigned)std::min<int64_t>(ceil_div(tot, 256), 4096)), dim3(256), 0, s, nullptr,
              A, lda, (int)M, (int)K, scratch, scratch + (size_t)M * kp, kp);
}

void launch_gemm_update_3xtf32(float *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N,
                               int64_t K, float *scratch, int num_sms, cudaStream_t s, bool reuse_a, int terms,
                               bool reuse_b, float *bscratch)
{
    launch_gemm_ops_3xtf32(W + r0 * ldw + k0, ldw, W + k0 * ldw + c0, ldw, W + r0 * ldw + c0, ldw, M, N, K, scratch,
                           num_sms, s, reuse_a, terms, reuse_b, bscratch);
}

}  // namespace mp
