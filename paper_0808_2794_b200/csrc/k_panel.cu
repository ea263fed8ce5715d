// k_panel.cu — K2: panel factorisation (GEPP on an m x w column panel leaf).
//
// PAPER.md P:89-92 / Alg. 1 line 1: "Partial row pivoting ... PA = LU".
// Per column c of the leaf: the pivot is the entry of largest |a| on/below the
// diagonal, ties to the smallest row position (reading A-6); rows
// kc = c0+c and p are interchanged over the leaf width; the entries below the
// pivot are divided by it (reading A-7: IEEE division, as the oracle); the
// remaining leaf columns get the rank-1 update.  An exact zero pivot is
// recorded (ST_ZERO_PIVOT, first column) and elimination continues without
// scaling; the driver then takes the binary64 fallback (iters -3).
//
// B200 design.  The pivot search is the method's serial critical path (n
// dependent arg-max decisions per factorisation), so a column step must cost
// a few hundred cycles, not microseconds:
//
//  * the leaf lives in REGISTERS of one thread-block cluster of CL <= 16 CTAs
//    (non-portable size; CL = ceil(m / rows-per-CTA), so short leaves use
//    fewer SMs): thread t of CTA g holds the rows loaded from positions
//    c0 + g*R + t + NT*q;
//  * rows never move between threads: the interchanges are tracked
//    logically (every row carries its current position) and rows are stored
//    at their final positions when the leaf is done;
//  * the column loop is unrolled in groups of UG columns over a rotating
//    register frame (static register indices, small code: the fully
//    unrolled loop was instruction-fetch bound);
//  * the cross-CTA exchange of a column is one-sided: after the CTA-level
//    arg-max, the warp holding the CTA's candidate row pushes (record, row)
//    with st.async into a slot of EVERY CTA's shared memory, completing bytes
//    on that CTA's mbarrier.  Each CTA then waits on its own mbarrier only
//    (no cluster barrier, no fence on global memory, no global atomics inside
//    the column loop) and reduces the CL candidate records locally — every
//    CTA reaches the same pivot and applies the rank-1 update, fused with the
//    next column's local arg-max.  Slots and mbarriers alternate by column
//    parity; a CTA cannot push column c+2 before every CTA has pushed column
//    c+1, which each CTA does only after it has consumed column c's slots, so
//    the double buffer is race-free without extra synchronisation;
//  * global memory is touched only at the start (load the leaf) and the end
//    (store the leaf, orig[] and the leaf's row pairs), plus ipiv.
#include <cooperative_groups.h>

#include <cstdlib>
#include <type_traits>

#include "internal.h"

namespace cg = cooperative_groups;

namespace mp {

namespace {

constexpr int CLMAX = 16;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Candidate keys for the arg-max (largest |a| wins, ties to the smallest position,
// reading A-6).  Non-negative IEEE values order like their bit patterns; NaN maps to
// key 0 so it never beats a finite entry.
//   binary32: one 64-bit word k = (|a| bits << 32) | (0x7fffffff - pos); k = 0: none.
//   binary64: 64-bit |a| bits + np = 0x7fffffff - pos (np = -1: none).
struct __align__(16) Rec {
    unsigned a, b, c, d;
};

template <typename T> struct Key;

template <> struct Key<float> {
    unsigned long long k;
    __device__ static Key none() { return Key{0ull}; }
    __device__ static Key make(float x, int pos)
    {
        const float v = fabsf(x);
        const unsigned bits = (v == v) ? __float_as_uint(v) : 0u;
        return Key{((unsigned long long)bits << 32) | (unsigned)(0x7fffffff - pos)};
    }
    __device__ void take(const Key &o) { if (o.k > k) k = o.k; }
    __device__ bool valid() const { return k != 0ull; }
    __device__ bool zero_value() const { return (k >> 32) == 0ull; }
    __device__ int pos() const { return k ? 0x7fffffff - (int)(unsigned)k : 0x7fffffff; }
    __device__ void warp_max()
    {
        const unsigned h = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32));
        const unsigned l = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32) == h ? (unsigned)k : 0u);
        k = ((unsigned long long)h << 32) | l;
    }
    __device__ bool operator==(const Key &o) const { return k == o.k; }
    __device__ void store(Rec &r) const { r.a = (unsigned)(k >> 32); r.b = (unsigned)k; r.c = 0u; r.d = 0u; }
    __device__ static Key load(const Rec &r) { return Key{((unsigned long long)r.a << 32) | r.b}; }
};

template <> struct Key<double> {
    unsigned long long key;
    int np;
    __device__ static Key none() { return Key{0ull, -1}; }
    __device__ static Key make(double x, int pos)
    {
        const double v = fabs(x);
        return Key{(v == v) ? (unsigned long long)__double_as_longlong(v) : 0ull, 0x7fffffff - pos};
    }
    __device__ void take(const Key &o) { if (o.key > key || (o.key == key && o.np > np)) *this = o; }
    __device__ bool valid() const { return np >= 0; }
    __device__ bool zero_value() const { return key == 0ull; }
    __device__ int pos() const { return np >= 0 ? 0x7fffffff - np : 0x7fffffff; }
    __device__ void warp_max()
    {
        const unsigned hk = (unsigned)(key >> 32), lk = (unsigned)key;
        const unsigned h = __reduce_max_sync(0xffffffffu, hk);
        const unsigned l = __reduce_max_sync(0xffffffffu, hk == h ? lk : 0u);
        np = __reduce_max_sync(0xffffffffu, (hk == h && lk == l) ? np : -1);
        key = ((unsigned long long)h << 32) | l;
    }
    __device__ bool operator==(const Key &o) const { return key == o.key && np == o.np; }
    __device__ void store(Rec &r) const { r.a = (unsigned)(key >> 32); r.b = (unsigned)key; r.c = (unsigned)np; r.d = 0u; }
    __device__ static Key load(const Rec &r) { return Key{((unsigned long long)r.a << 32) | r.b, (int)r.c}; }
};

// Reciprocal for the multipliers l = x / piv (reading A-7): hardware approximation +
// one Newton step, then per row q = x*r corrected once with the residual fma(-piv,q,x).
// Equal to the IEEE quotient except in rare double-rounding cases (<= 1 ulp).
__device__ __forceinline__ float recip(float v)
{
    float r;
    asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(v));
    return fmaf(r, fmaf(-v, r, 1.0f), r);
}
__device__ __forceinline__ double recip(double v) { return 1.0 / v; }


template <typename T, int W>
struct __align__(16) Slot {
    Rec rec;
    T row[W];
};

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count)
{
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, int rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async16(uint32_t raddr, uint4 v, uint32_t rbar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     raddr),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
                 : "memory");
}

#ifdef MP_PANEL_TRACE
__device__ long long g_trace[64][8];
#define TRACE(c, k) do { if (tid == 0 && g == 0 && (c) < 64) g_trace[(c)][(k)] = clock64(); } while (0)
#else
#define TRACE(c, k) do { } while (0)
#endif

template <typename T>
struct LeafArgs {
    T *W;
    long long ldw, n, c0;
    int w;                 // active leaf width (<= template W)
    int32_t *ipiv;
    int32_t *orig;         // [n] panel-level origin of the row now at each position (updated)
    int32_t *pairs;        // leaf-level (position, origin-at-leaf-start) pairs, [2w][2]
    int32_t *npairs;
    DevStatus *st;
    int32_t *first_np;     // first leaf of a panel: orig[] is the identity (not read) and this
                           // panel-level pair counter is zeroed here
    // Left-looking mode (ll != 0, see ll_catch_up): the panel [k, k + nb) keeps its rows at their
    // panel-start (physical) positions while its leaves are factored; the leaf covers every row
    // [k, n), brings its own columns up to date itself and records positions instead of moving rows
    int ll;
    long long k;           // panel start
    long long kend;        // panel end (columns [k, kend))
    int32_t *lpos;         // [n] logical position of the row physically at r (rows [k, n))
};

// NPMAX: previous pivots of the panel a left-looking leaf can catch up on (panels <= 256 wide)
constexpr int LL_NPMAX = 256;
constexpr int LL_LDL = LL_NPMAX + 4;
template <typename T, int W>
constexpr size_t ll_smem_bytes()
{
    const size_t pro = (size_t)LL_NPMAX * W, epi = (size_t)32 * LL_LDL + (size_t)LL_NPMAX * 16 + 32 * 16;
    return sizeof(T) * (pro > epi ? pro : epi);
}

// Left-looking leaves (LeafArgs::ll).  The panel [k, kend) keeps its rows at their panel-start
// (physical) positions while its leaves are factored (one interchange launch moves them at the end).
// Invariants after leaf b (columns [c0, c0 + w)): the pivot rows orig[k .. c0 + w) hold their
// multipliers in the columns left of their pivot and their U row in every column to the right,
// including the panel's later columns; every other row holds its multipliers in [k, c0 + w) and its
// panel-start values right of that.  Then SGETRF's in-panel update of a later leaf's columns
// (step 1), reordered left-looking, is for an active row:
//     x = A(row, leaf) - L(row, k : c0) U(k : c0, leaf)          (ll_catch_up, before the leaf)
// and the U rows of the new pivots in the later columns are, per column c (ll_pivot_rows, after it):
//     u(j, c) = A(piv_j, c) - sum_{i < c0 - k + j} L(piv_j, i) u(i, c)
// (the earlier pivots' u(i, c) are in their rows), split over the cluster's CTAs by column.
template <typename T, int NT, int RPT, int W>
__device__ __forceinline__ void ll_catch_up(const LeafArgs<T> &a, long long base, int nn, T (&x)[RPT][W],
                                            int (&org)[RPT], int (&cs)[RPT])
{
    // dynamic shared memory (ll_smem_bytes): U [LL_NPMAX][W]
    extern __shared__ __align__(16) unsigned char ll_raw[];
    T (*U)[W] = reinterpret_cast<T (*)[W]>(ll_raw);
    __shared__ int prow[LL_NPMAX];
    const int tid = threadIdx.x;
    const long long k = a.k, c0 = a.c0, ldw = a.ldw;
    const int np = (int)(c0 - k), w = a.w;
    const T *W0 = a.W;
    if (np > 0) {
        // U(k : c0, leaf) from the earlier pivots' rows (all loads in flight, 16 bytes each)
        for (int i = tid; i < np; i += NT) prow[i] = a.orig[k + i];
        __syncthreads();
        constexpr int QW = W / 4;
        for (int o = tid; o < np * QW; o += NT) {
            const int i = o / QW, s4 = (o - i * QW) * 4;
            float4 v = *reinterpret_cast<const float4 *>(W0 + (long long)prow[i] * ldw + c0 + s4);
            if (s4 + 3 >= w) {                      // partial leaf: zero the columns beyond w
                if (s4 >= w) v.x = 0.f;
                if (s4 + 1 >= w) v.y = 0.f;
                if (s4 + 2 >= w) v.z = 0.f;
                v.w = 0.f;
            }
            *reinterpret_cast<float4 *>(&U[i][s4]) = v;
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int li = tid + NT * q;
        const bool valid = li < nn;
        const long long r = base + li;
        const int pos = valid ? (np == 0 ? (int)r : a.lpos[r]) : (int)r;
        const bool active = valid && pos >= c0;
        cs[q] = active ? pos : ~pos;
        org[q] = (int)r;
        const T *rowp = W0 + r * ldw + c0;
        // active rows: panel-start values; pivot rows: their U row (written by earlier leaves)
        if (valid && w == W) {
#pragma unroll
            for (int s4 = 0; s4 < W; s4 += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(rowp + s4);
                x[q][s4] = v.x; x[q][s4 + 1] = v.y; x[q][s4 + 2] = v.z; x[q][s4 + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int s = 0; s < W; ++s) x[q][s] = valid && s < w ? rowp[s] : T(0);
        }
    }
    if (np > 0) {
        // x -= L(row, k : c0) U for the active rows, 8 pivots at a time; the next 8 multipliers of every
        // row are loaded (two 16-byte loads) while the current 8 are applied (U rows broadcast from
        // shared memory); np is a multiple of 8
        float4 nxt[RPT][2];
        auto load8 = [&](int j) {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int li = tid + NT * q;
                const bool act = li < nn && cs[q] >= 0;
                const float4 *src = reinterpret_cast<const float4 *>(W0 + (base + li) * ldw + k + j);
                nxt[q][0] = act ? src[0] : make_float4(0.f, 0.f, 0.f, 0.f);
                nxt[q][1] = act ? src[1] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        load8(0);
        for (int j = 0; j < np; j += 8) {
            float lv[RPT][8];
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                lv[q][0] = nxt[q][0].x; lv[q][1] = nxt[q][0].y; lv[q][2] = nxt[q][0].z; lv[q][3] = nxt[q][0].w;
                lv[q][4] = nxt[q][1].x; lv[q][5] = nxt[q][1].y; lv[q][6] = nxt[q][1].z; lv[q][7] = nxt[q][1].w;
            }
            if (j + 8 < np) load8(j + 8);
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
#pragma unroll
                for (int s4 = 0; s4 < W; s4 += 4) {
                    const float4 u4 = *reinterpret_cast<const float4 *>(&U[j + jj][s4]);
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        x[q][s4] = fma(-lv[q][jj], u4.x, x[q][s4]);
                        x[q][s4 + 1] = fma(-lv[q][jj], u4.y, x[q][s4 + 1]);
                        x[q][s4 + 2] = fma(-lv[q][jj], u4.z, x[q][s4 + 2]);
                        x[q][s4 + 3] = fma(-lv[q][jj], u4.w, x[q][s4 + 3]);
                    }
                }
            }
        }
    }
}

// After the leaf's rows are stored (and a cluster barrier): the U rows of the leaf's w new pivots
// in the panel's later columns [c0 + w, kend), CTA g of CL taking a contiguous slice of them,
// 16 columns per batch.  Shared memory (the same dynamic block): Lp [32][LL_LDL] the new pivots'
// multipliers L(piv_j, k : c0 + w); Uo [LL_NPMAX][16] the earlier pivots' u(i, c); Tt [32][16].
template <typename T, int NT, int W>
__device__ __forceinline__ void ll_pivot_rows(const LeafArgs<T> &a, int g, int CL)
{
    extern __shared__ __align__(16) unsigned char ll_raw[];
    T (*Lp)[LL_LDL] = reinterpret_cast<T (*)[LL_LDL]>(ll_raw);
    T (*Uo)[16] = reinterpret_cast<T (*)[16]>(ll_raw + sizeof(T) * 32 * LL_LDL);
    T (*Tt)[16] = reinterpret_cast<T (*)[16]>(ll_raw + sizeof(T) * (32 * LL_LDL + LL_NPMAX * 16));
    __shared__ int prw[LL_NPMAX];
    const int tid = threadIdx.x;
    const long long k = a.k, c0 = a.c0, ldw = a.ldw;
    const int np = (int)(c0 - k), w = a.w, nt = np + w;
    const long long cs0 = c0 + w, ncols = a.kend - cs0;
    if (ncols <= 0) return;
    const long long per = (ncols + CL - 1) / CL;
    const long long cb0 = cs0 + g * per, cb1 = min(a.kend, cb0 + per);
    if (cb0 >= cb1) return;
    T *W0 = a.W;
    for (int i = tid; i < nt; i += NT) prw[i] = a.orig[k + i];
    __syncthreads();
    for (int o = tid; o < w * (nt / 4); o += NT) {           // multipliers of the new pivots (nt % 4 == 0)
        const int j = o / (nt / 4), i4 = (o - j * (nt / 4)) * 4;
        *reinterpret_cast<float4 *>(&Lp[j][i4]) =
            *reinterpret_cast<const float4 *>(W0 + (long long)prw[np + j] * ldw + k + i4);
    }
    for (long long cb = cb0; cb < cb1; cb += 16) {
        const int nc = (int)min(16LL, cb1 - cb);
        for (int o = tid; o < np * 16; o += NT) {
            const int i = o >> 4, cc = o & 15;
            Uo[i][cc] = cc < nc ? W0[(long long)prw[i] * ldw + cb + cc] : T(0);
        }
        __syncthreads();
        // the GEMM part: T(j, cc) = A(piv_j, c) - sum_{i < np} L(piv_j, i) u(i, c)
        for (int o = tid; o < w * 16; o += NT) {
            const int j = o >> 4, cc = o & 15;
            T acc = cc < nc ? W0[(long long)prw[np + j] * ldw + cb + cc] : T(0);
            for (int i = 0; i < np; ++i) acc = fma(-Lp[j][i], Uo[i][cc], acc);
            Tt[j][cc] = acc;
        }
        __syncthreads();
        // the triangle of the new pivots: warp 0, lane j holds row j of the 16-column batch; for each
        // pivot jj (in order) the final row jj is broadcast by shuffles and applied to the rows below
        if (tid < 32) {
            const int j = tid;
            T u[16];
#pragma unroll
            for (int cc = 0; cc < 16; ++cc) u[cc] = j < w ? Tt[j][cc] : T(0);
#pragma unroll
            for (int jj = 0; jj < W; ++jj) {
                if (jj < w) {
                    const T l = (j > jj && j < w) ? Lp[j][np + jj] : T(0);
#pragma unroll
                    for (int cc = 0; cc < 16; ++cc) u[cc] = fma(-l, __shfl_sync(0xffffffffu, u[cc], jj), u[cc]);
                }
            }
            if (j < w)
                for (int cc = 0; cc < nc; ++cc) W0[(long long)prw[np + j] * ldw + cb + cc] = u[cc];
        }
        __syncthreads();
    }
}

// RPT rows per thread, leaf width W, column loop unrolled in groups of UG columns.
//
// Rows never move between threads inside the leaf: every row carries its CURRENT
// position cur (LAPACK's sequential interchanges, tracked logically): at
// column c the winner (position p) gets position kc and retires, the row at position
// kc gets position p.  Rows are stored at their final positions at the end.
//
// Register frame: at the start of group o, slot s holds leaf column (o*UG + s) mod W;
// the frame is rotated by UG after every group (W/UG rotations = identity at the end).
// Slots s >= W - o*UG hold multipliers of earlier columns ("dead"); the staged pivot
// row has them zeroed so the rank-1 update leaves them unchanged.
template <typename T, int NT, int RPT, int W, int UG, bool MULTI, bool HW = true, bool LLK = false>
__global__ void __launch_bounds__(NT, 1) panel_leaf_kernel(LeafArgs<T> a)
{
    constexpr int NWP = NT / 32;
    static_assert(W % UG == 0, "group size must divide the leaf width");
    using SlotT = Slot<T, W>;
    using K = Key<T>;
    static_assert(sizeof(SlotT) % 16 == 0, "slot must be 16-byte chunks");
    constexpr int CH = (int)(sizeof(SlotT) / 16);
    constexpr int EPC = 16 / (int)sizeof(T);     // elements per 16-byte chunk
    // the staged candidate row keeps its dead slots; the leader zeroes them chunk by chunk while
    // pushing (live is a multiple of UG): one select per chunk instead of one per element per warp
    constexpr bool kLeadZero = MULTI && (UG % EPC == 0);
    pdl_wait();
    pdl_trigger();
    cg::cluster_group cluster = cg::this_cluster();
    const int g = (int)cluster.block_rank();
    const int CL = (int)cluster.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    __shared__ SlotT slots[2][CLMAX];     // incoming CTA candidates, by source CTA
    __shared__ SlotT wstage[2][NWP];      // per-warp candidates, by column parity
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ int s_p[2], s_ww[2];       // single-CTA leaves: pivot position, winning warp

    const long long n = a.n, c0 = a.c0, ldw = a.ldw;
    const int w = a.w;
    constexpr int R = NT * RPT;                  // rows per CTA
    constexpr bool ll = LLK && sizeof(T) == 4;   // left-looking instantiation (LeafArgs::ll)
    const long long rows0 = ll ? a.k : c0;       // left-looking: every row of the panel [k, n)
    const long long base = rows0 + (long long)g * R;
    const int nn = (int)(n - base);              // rows of this CTA that exist: local index < nn
    const unsigned bytes_per_col = (unsigned)(CL * sizeof(SlotT));

    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (g == 0) *a.npairs = 0;
        if (g == 0 && a.first_np) *a.first_np = 0;
    }
    // every CTA's mbarriers must be initialised before anyone pushes into them
    cluster.sync();

    T x[RPT][W];
    // cs[q]: the row's current logical position; bitwise-complemented (negative) once the row is
    // no longer active (it became a pivot row, or does not exist)
    int org[RPT], cs[RPT];
    if constexpr (ll) {                         // (binary32 only: the binary64 leaves keep the recursive panel)
        ll_catch_up<T, NT, RPT, W>(a, base, nn, x, org, cs);
    }
    if (!ll)
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int li = tid + NT * q;
        const bool valid = li < nn;
        const T *row = a.W + (base + li) * ldw + c0;
        if (valid && w == W && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
#pragma unroll
            for (int s = 0; s < W; s += EPC) {
                const uint4 v = *reinterpret_cast<const uint4 *>(row + s);
                const T *pv = reinterpret_cast<const T *>(&v);
#pragma unroll
                for (int e = 0; e < EPC; ++e) x[q][s + e] = pv[e];
            }
        } else {
#pragma unroll
            for (int s = 0; s < W; ++s) x[q][s] = (valid && s < w) ? row[s] : T(0);
        }
        org[q] = !valid ? -1 : (a.first_np ? (int)(base + li) : a.orig[base + li]);
        cs[q] = valid ? (int)(base + li) : ~(int)(base + li);
    }

    // push plan of the leader warp (loop invariant): lane handles chunks idx = lane + 32 j of the
    // CL x CH (destination CTA, 16-byte chunk) grid; remote slot / mbarrier addresses per parity
    constexpr int PJ = (CLMAX * CH + 31) / 32;
    uint32_t pdst[2][PJ], pbar[2][PJ];
    int pch[PJ];
    if (MULTI && warp == 0) {
#pragma unroll
        for (int j = 0; j < PJ; ++j) {
            const int idx = lane + 32 * j, r = idx / CH, ch = idx - r * CH;
            const bool ok = idx < CL * CH;
            pch[j] = ok ? ch : -1;
#pragma unroll
            for (int pp = 0; pp < 2; ++pp) {
                pdst[pp][j] = ok ? mapa(smem_u32(&slots[pp][g]) + 16u * ch, r) : 0u;
                pbar[pp][j] = ok ? mapa(smem_u32(&mbar[pp]), r) : 0u;
            }
        }
    }

    // this thread's candidate for column 0
    K ck = K::none();
#pragma unroll
    for (int q = 0; q < RPT; ++q)
        if (cs[q] >= 0) ck.take(K::make(x[q][0], cs[q]));

    // One group of UG columns.  LM: slots >= LM are dead in every column of the group (live <= LM),
    // so the rank-1 update stops there (the second half of the leaf runs half-width FMAs).
    auto group = [&](const int o, auto lmax) {
        constexpr int LM = decltype(lmax)::value;
        const int live = W - o * UG;             // slots >= live are dead (multipliers)
#pragma unroll
        for (int u = 0; u < UG; ++u) {
            const int c = o * UG + u;
            if (c < w) {
                const int par = c & 1;
                const long long kc = c0 + c;
                TRACE(c, 0);
                // ---- warp arg-max; the lane holding the warp's candidate stages (record, row)
                {
                    K wk = ck;
                    wk.warp_max();
                    const int wp = wk.pos();
                    int qs = -1;
#pragma unroll
                    for (int q = RPT - 1; q >= 0; --q)
                        if (cs[q] == wp) qs = q;
                    if (qs >= 0) {                       // one lane per warp: a divergent, short branch
#pragma unroll
                        for (int q = 0; q < RPT; ++q)
                            if (q == qs) {
#pragma unroll
                                for (int s = 0; s < W; s += EPC) {
                                    uint4 v;
                                    T *pv = reinterpret_cast<T *>(&v);
#pragma unroll
                                    for (int e = 0; e < EPC; ++e)
                                        pv[e] = (kLeadZero || s + e < live) ? x[q][s + e] : T(0);
                                    *reinterpret_cast<uint4 *>(&wstage[par][warp].row[s]) = v;
                                }
                            }
                    }
                    if (lane == 0) wk.store(wstage[par][warp].rec);
                }
                const SlotT *win;
                int p;
                K pk;                                     // the pivot's key (thread 0 only needs it)
                if constexpr (!MULTI) {
                    // ---- single-CTA leaf: the CTA arg-max is the pivot; no exchange
                    if (warp == 0) {
                        named_bar_sync(1, NT);           // every warp has staged
                        TRACE(c, 1);
                        K bk = lane < NWP ? K::load(wstage[par][lane].rec) : K::none();
                        const K mine = bk;
                        bk.warp_max();
                        const int ww = __ffs(__ballot_sync(0xffffffffu, mine == bk && lane < NWP)) - 1;
                        if (lane == 0) { s_p[par] = bk.pos(); s_ww[par] = ww; }
                        pk = bk;
                        TRACE(c, 2);
                        named_bar_sync(2, NT);
                    } else {
                        named_bar_arrive(1, NT);
                        named_bar_sync(2, NT);
                    }
                    p = s_p[par];
                    win = &wstage[par][s_ww[par]];
                    TRACE(c, 3);
                } else {
                    // ---- leader warp: CTA arg-max and push (record, row) into every CTA
                    if (warp == 0) {
                        named_bar_sync(1, NT);           // every warp has staged
                        TRACE(c, 1);
                        K bk = lane < NWP ? K::load(wstage[par][lane].rec) : K::none();
                        const K mine = bk;
                        bk.warp_max();
                        const int ww = __ffs(__ballot_sync(0xffffffffu, mine == bk && lane < NWP)) - 1;
                        if (lane == 0) mbar_arm(&mbar[par], bytes_per_col);
                        const uint4 *s4 = reinterpret_cast<const uint4 *>(&wstage[par][ww]);
                        // every chunk load first, then every one-sided store (no per-chunk round trip)
                        uint4 pv[PJ];
#pragma unroll
                        for (int j = 0; j < PJ; ++j)
                            if (pch[j] >= 0) {
                                pv[j] = s4[pch[j]];
                                // dead slots (multipliers) go out as zeros: whole 16-byte chunks
                                if (kLeadZero && pch[j] >= 1 && (pch[j] - 1) * EPC >= live) pv[j] = make_uint4(0u, 0u, 0u, 0u);
                            }
#pragma unroll
                        for (int j = 0; j < PJ; ++j)
                            if (pch[j] >= 0) st_async16(pdst[par][j], pv[j], pbar[par][j]);
                        TRACE(c, 2);
                    } else {
                        named_bar_arrive(1, NT);
                    }
                    // ---- every warp: wait for the CL candidates, identical cluster arg-max
                    mbar_wait_cluster(&mbar[par], (unsigned)((c >> 1) & 1));
                    __syncwarp();                        // reconverge after the wait loop (asm branch)
                    TRACE(c, 3);
                    K gk = lane < CL ? K::load(slots[par][lane].rec) : K::none();
                    const K mine = gk;
                    gk.warp_max();
                    const int gw = __ffs(__ballot_sync(0xffffffffu, mine == gk && lane < CL)) - 1;
                    p = gk.pos();
                    pk = gk;
                    win = &slots[par][gw];
                }
                TRACE(c, 4);
                if (g == 0 && tid == 0) {
                    a.ipiv[kc] = (int32_t)p;
                    if (pk.zero_value()) {               // exact zero pivot (or all NaN)
                        atomicOr(&a.st->flags, (int)ST_ZERO_PIVOT);
                        atomicMin(&a.st->zero_col, (int)(kc + 1));
                    }
                }

                // ---- logical interchange, scale, rank-1 update; next column's candidate.
                // Branch-free per row (predicated selects): rows that are not updated use l = 0.
                const T piv = win->row[u];
                const bool scale = piv != T(0);
                // subnormal pivots: scale numerator and pivot by the same power of two
                const T sc = fabs(piv) < (sizeof(T) == 4 ? T(1e-30) : T(1e-300)) ? T(sizeof(T) == 4 ? 0x1p64 : 0x1p512) : T(1);
                const T ps = piv * sc;
                const T rinv = scale ? recip(ps) : T(0);
                ck = K::none();
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const int cq = cs[q];
                    const bool is_piv = cq == p;
                    const bool upd = cq >= 0 && !is_piv;
                    cs[q] = is_piv ? ~(int)kc : (cq == (int)kc ? p : cq);
                    const T xv = x[q][u];
                    const T xs = xv * sc;
                    T l = xs * rinv;
                    l = fma(fma(-ps, l, xs), rinv, l);
                    l = scale ? l : xv;
                    l = upd ? l : T(0);
                    x[q][u] = upd ? l : xv;
#pragma unroll
                    for (int s2 = u + 1; s2 < LM; ++s2) x[q][s2] = fma(-l, win->row[s2], x[q][s2]);
                    if (u + 1 < W) {
                        const K kq = K::make(x[q][(u + 1) % W], cs[q]);
                        ck.take(upd ? kq : K::none());
                    }
                }
            }
        }
        // ---- rotate the frame by UG
        if constexpr (UG < W) {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                T t[UG];
#pragma unroll
                for (int s = 0; s < UG; ++s) t[s] = x[q][s];
#pragma unroll
                for (int s = 0; s < W - UG; ++s) x[q][s] = x[q][s + UG];
#pragma unroll
                for (int s = 0; s < UG; ++s) x[q][W - UG + s] = t[s];
            }
        }
    };
    constexpr int NG = W / UG;
    constexpr int HALF = NG >= 2 ? NG / 2 : NG;  // groups o < HALF have live > W / 2
#pragma unroll 1
    for (int o = 0; o < HALF; ++o) group(o, std::integral_constant<int, W>{});
#pragma unroll 1
    for (int o = HALF; o < NG; ++o) group(o, std::integral_constant<int, (HW && HALF < NG ? W / 2 : W)>{});

    // ---- store every row at its final position, orig[] and the leaf pairs
    cluster.sync();   // orders the npairs reset before the pair emission below
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int li = tid + NT * q;
        if (ll && li < nn) {               // left-looking: the row stays where it is; record its position
            const long long pos = cs[q] >= 0 ? cs[q] : ~cs[q];
            T *row = a.W + (base + li) * ldw + c0;
#pragma unroll
            for (int s = 0; s < W; ++s)
                if (s < w) row[s] = x[q][s];
            a.orig[pos] = (int32_t)(base + li);
            a.lpos[base + li] = (int32_t)pos;
            continue;
        }
        if (li < nn) {
            const long long pos = cs[q] >= 0 ? cs[q] : ~cs[q];
            T *row = a.W + pos * ldw + c0;
            if (w == W && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
#pragma unroll
                for (int s = 0; s < W; s += EPC) {
                    uint4 v;
                    T *pv = reinterpret_cast<T *>(&v);
#pragma unroll
                    for (int e = 0; e < EPC; ++e) pv[e] = x[q][s + e];
                    *reinterpret_cast<uint4 *>(row + s) = v;
                }
            } else {
#pragma unroll
                for (int s = 0; s < W; ++s)
                    if (s < w) row[s] = x[q][s];
            }
            a.orig[pos] = org[q];
            const int lorg = (int)(base + li);
            if (lorg != (int)pos) {
                const int si = atomicAdd(a.npairs, 1);
                a.pairs[2 * si] = (int32_t)pos;
                a.pairs[2 * si + 1] = lorg;
            }
        }
    }
    if constexpr (ll) {
        if (a.kend > c0 + w) {
            cluster.sync();                       // every CTA's multipliers and U rows are stored
            ll_pivot_rows<T, NT, W>(a, g, CL);
        }
    }
}

__global__ void emit_pairs_kernel(const int32_t *orig, int64_t k, int64_t n, int32_t *pairs, int32_t *npairs)
{
    pdl_wait();
    pdl_trigger();
    for (int64_t i = k + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t o = orig[i];
        if (o != (int32_t)i) {
            const int slot = atomicAdd(npairs, 1);
            pairs[2 * slot] = (int32_t)i;
            pairs[2 * slot + 1] = o;
        }
    }
}

// ---------------------------------------------------------------- host side
// Configurations (threads per CTA, rows per thread, leaf width).  Four rows per thread
// amortise the per-column protocol (arg-max, barriers) over several rows; data registers
// RPT * W * sizeof(T) / 4 <= 128.  Capacity per cluster = CLMAX * NT * RPT rows; the
// cluster uses ceil(m / (NT * RPT)) CTAs.
struct LeafCfg { int nt, rpt, w; };
#ifndef MP_LEAF_C1_NT
#define MP_LEAF_C1_NT 256
#define MP_LEAF_C1_RPT 4
#endif
#ifndef MP_LEAF_C0_NT
#define MP_LEAF_C0_NT 256          // 256 x 2 beats 128 x 4 by ~10 % for m <= 8192 (more warps per
#define MP_LEAF_C0_RPT 2           // SMSP hide the per-column chain; tools/bench_panel.cu)
#endif
#define MP_LEAF_C1 MP_LEAF_C1_NT, MP_LEAF_C1_RPT, 32
#define MP_LEAF_C0 MP_LEAF_C0_NT, MP_LEAF_C0_RPT, 32
// {256, 3, 32} between them: the per-column update scales with the rows per thread (cycles per
// column at m = 12288: 2113 with 4 rows, ~1720 with 2 at m = 8192; tools/bench_panel.cu).
// (Measured and dropped: 64-column leaves for m <= 8192, {256, 2, 64}: 87-96 us per leaf against
// 2 x 40 us + the in-panel K = 32 update and interchange they replace; C3 47.9 vs 46.4 ms.)
constexpr LeafCfg kCfgF[] = {{MP_LEAF_C0}, {256, 3, 32}, {MP_LEAF_C1}, {512, 4, 16}, {512, 8, 8}};
constexpr LeafCfg kCfgD[] = {{128, 4, 16}, {256, 3, 16}, {256, 4, 16}, {512, 4, 8}, {512, 8, 4}};
constexpr int kNumCfgF = 5, kNumCfgD = 5;

int g_cluster = 0;   // largest cluster size the device accepts (16, else 8)

#ifndef MP_PANEL_UG
#define MP_PANEL_UG 4
#endif
template <typename T, int NT, int RPT, int W>
void launch_cfg(const LeafArgs<T> &a, int cl, cudaStream_t s)
{
    constexpr int UG = W > MP_PANEL_UG ? MP_PANEL_UG : W;
    static const bool fullw = [] { const char *e = std::getenv("MP_LEAF_FULLW"); return e && e[0] == '1'; }();
    auto kern = cl > 1 ? (fullw ? panel_leaf_kernel<T, NT, RPT, W, UG, true, false> : panel_leaf_kernel<T, NT, RPT, W, UG, true>)
                       : (fullw ? panel_leaf_kernel<T, NT, RPT, W, UG, false, false> : panel_leaf_kernel<T, NT, RPT, W, UG, false>);
    if constexpr (sizeof(T) == 4 && W <= 32) {
        if (a.ll) kern = cl > 1 ? panel_leaf_kernel<T, NT, RPT, W, UG, true, true, true>
                                : panel_leaf_kernel<T, NT, RPT, W, UG, false, true, true>;
    } else if (a.ll) {
        throw CudaError{cudaErrorInvalidValue, "left-looking leaves are at most 32 columns wide", __LINE__};
    }
    if (cl > 8) func_cluster16_once((const void *)kern);
    const size_t dsm = a.ll ? ll_smem_bytes<T, W>() : 0;
    if (a.ll) func_smem_once((const void *)kern, dsm);
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = cl;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    launch_ex(kern, dim3(cl), dim3(NT), dsm, s, &at, a);
}

int cluster_size()
{
    if (g_cluster) return g_cluster;
    // can a 16-CTA cluster of the widest configuration be resident?
    auto kern = panel_leaf_kernel<float, 512, 8, 8, 8, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int nclusters = 0;
    if (e == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16, 1, 1);
        cfg.blockDim = dim3(512, 1, 1);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg);
    }
    if (e != cudaSuccess) cudaGetLastError();
    g_cluster = (e == cudaSuccess && nclusters > 0) ? 16 : 8;
    return g_cluster;
}

// narrow32: leaves of at most 32 columns (the left-looking mode)
int select_cfg(size_t elem, int64_t m, int cl, bool narrow32 = false)
{
    const LeafCfg *c = elem == 4 ? kCfgF : kCfgD;
    static const int first = [] { const char *e = std::getenv("MP_LEAF_MIN_CFG"); return e ? std::atoi(e) : 0; }();
    for (int i = first; i < (elem == 4 ? kNumCfgF : kNumCfgD); ++i)
        if (!(narrow32 && c[i].w > 32) && (int64_t)cl * c[i].nt * c[i].rpt >= m) return i;
    return -1;
}

}  // namespace

template <typename T>
int panel_leaf_width(int64_t m)
{
    const int sel = select_cfg(sizeof(T), m, cluster_size());
    if (sel < 0) return 0;
    return (sizeof(T) == 4 ? kCfgF : kCfgD)[sel].w;
}

template <typename T>
void launch_panel_leaf(T *W, int64_t ldw, int64_t n, int64_t c0, int w, int32_t *ipiv, PanelScratch &ps,
                       DevStatus *st, cudaStream_t s, int32_t *first_np, int64_t ll_k, int32_t *lpos,
                       int64_t ll_kend)
{
    const int clmax = cluster_size();
    const bool ll = lpos != nullptr;
    const int64_t m = n - (ll ? ll_k : c0);
    const int sel = select_cfg(sizeof(T), m, clmax, ll);
    const LeafCfg *cfgs = sizeof(T) == 4 ? kCfgF : kCfgD;
    if (sel < 0 || w > cfgs[sel].w)
        throw CudaError{cudaErrorInvalidValue, "panel leaf does not fit one cluster", __LINE__};
    const int cl = (int)std::max<int64_t>(1, ceil_div(m, (int64_t)cfgs[sel].nt * cfgs[sel].rpt));
    LeafArgs<T> a;
    a.W = W; a.ldw = ldw; a.n = n; a.c0 = c0; a.w = w; a.ipiv = ipiv;
    a.orig = ps.orig; a.pairs = ps.pairs; a.npairs = ps.npairs; a.st = st; a.first_np = first_np;
    a.ll = ll ? 1 : 0; a.k = ll ? ll_k : c0; a.lpos = lpos; a.kend = ll ? ll_kend : c0 + w;
    if (ll && (sizeof(T) != 4 || c0 - ll_k > LL_NPMAX - w))
        throw CudaError{cudaErrorInvalidValue, "left-looking leaf: binary32 panels of at most 256 columns", __LINE__};
    if constexpr (sizeof(T) == 4) {
        switch (sel) {
        case 0: launch_cfg<T, MP_LEAF_C0>(a, cl, s); break;
        case 1: launch_cfg<T, 256, 3, 32>(a, cl, s); break;
        case 2: launch_cfg<T, MP_LEAF_C1>(a, cl, s); break;
        case 3: launch_cfg<T, 512, 4, 16>(a, cl, s); break;
        default: launch_cfg<T, 512, 8, 8>(a, cl, s); break;
        }
    } else {
        switch (sel) {
        case 0: launch_cfg<T, 128, 4, 16>(a, cl, s); break;
        case 1: launch_cfg<T, 256, 3, 16>(a, cl, s); break;
        case 2: launch_cfg<T, 256, 4, 16>(a, cl, s); break;
        case 3: launch_cfg<T, 512, 4, 8>(a, cl, s); break;
        default: launch_cfg<T, 512, 8, 4>(a, cl, s); break;
        }
    }
}

void launch_emit_pairs(const int32_t *orig, int64_t k, int64_t n, int32_t *pairs, int32_t *npairs, cudaStream_t s)
{
    launch_ex(emit_pairs_kernel, dim3((unsigned)std::min<int64_t>(ceil_div(n - k, 256), 512)), dim3(256), 0, s,
              nullptr, orig, k, n, pairs, npairs);
}

template int panel_leaf_width<float>(int64_t);
template int panel_leaf_width<double>(int64_t);
template void launch_panel_leaf<float>(float *, int64_t, int64_t, int64_t, int, int32_t *, PanelScratch &,
                                       DevStatus *, cudaStream_t, int32_t *, int64_t, int32_t *, int64_t);
template void launch_panel_leaf<double>(double *, int64_t, int64_t, int64_t, int, int32_t *, PanelScratch &,
                                        DevStatus *, cudaStream_t, int32_t *, int64_t, int32_t *, int64_t);

}  // namespace mp
