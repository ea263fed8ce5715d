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
// B200 design — one THREAD-BLOCK CLUSTER of CL = 16 CTAs (non-portable size;
// 8 if the device refuses 16) owns the whole leaf, held in REGISTERS: thread t
// of CTA g keeps RPT rows x W columns (rows g*R + t + NT*q).  Per column there
// is exactly ONE cluster barrier (barrier.cluster, ~0.2 us) instead of a
// grid-wide barrier: before it every CTA writes its (|a|, position) candidate
// into every CTA's shared-memory slot (DSMEM stores) and leaves its candidate
// row (and row kc, if owned) in its own shared memory; after it every CTA
// reduces the CL slots identically, pulls the winning row (one warp, 128 B of
// DSMEM loads), installs the interchange in registers and applies the rank-1
// update, fusing the arg-max of the next column into it.  Double-buffered
// slots (by column parity) make the next column's writes safe without a second
// barrier.  Latency-bound: n cluster barriers per factorisation.  The rest of
// the GPU stays free for the trailing update (look-ahead).
#include <cooperative_groups.h>

#include "internal.h"

namespace cg = cooperative_groups;

namespace mp {

namespace {

constexpr int CLMAX = 16;

// Order-preserving key of |a| for the arg-max (non-negative IEEE values order like their
// bit patterns; NaN is mapped to 0 so it never wins against a finite entry).
__device__ __forceinline__ void abs_key(float v, unsigned &hi, unsigned &lo)
{
    const float a = fabsf(v);
    hi = (a == a) ? __float_as_uint(a) : 0u;
    lo = 0u;
}
__device__ __forceinline__ void abs_key(double v, unsigned &hi, unsigned &lo)
{
    const double a = fabs(v);
    const unsigned long long b = (a == a) ? (unsigned long long)__double_as_longlong(a) : 0ull;
    hi = (unsigned)(b >> 32);
    lo = (unsigned)b;
}

// Warp arg-max of (key, position): largest key, ties to the smallest position.
// Three redux.sync instructions instead of a shuffle tree.  Inactive lanes pass pos = INT_MAX.
__device__ __forceinline__ void warp_argmax(unsigned &hi, unsigned &lo, int &pos)
{
    const unsigned full = 0xffffffffu;
    const unsigned h = __reduce_max_sync(full, hi);
    const unsigned l = __reduce_max_sync(full, hi == h ? lo : 0u);
    const unsigned pm = __reduce_min_sync(full, (hi == h && lo == l) ? (unsigned)pos : 0x7fffffffu);
    hi = h;
    lo = l;
    pos = (int)pm;
}

struct __align__(16) Cand {
    unsigned hi, lo;
    int pos, pad;
    int org, lorg, pad1, pad2;
};

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
};

template <typename T, int NT, int RPT, int W>
__global__ void __launch_bounds__(NT, 1) panel_cluster_kernel(LeafArgs<T> a)
{
    // Register frame: every active row keeps its W leaf values ROTATED by the number of
    // columns eliminated so far: slot s holds column (c + s) for s < W - c and the
    // multiplier l of column (s - (W - c)) for s >= W - c.  All active rows share the
    // frame, so a column step is a constant-size body (update slots 1..W-1 with the
    // pivot row, consumed slots masked to zero, then rotate by one) and the column loop
    // stays rolled: small code, no instruction-cache misses, no dynamic indexing.
    //
    // Per column: one __syncthreads (warp candidates -> CTA candidate) and ONE cluster
    // barrier.  Before the barrier the winning warp of every CTA pushes its candidate
    // record and candidate row into every CTA's shared memory, and the warp owning row
    // kc pushes row kc: afterwards everything is local.  All shared buffers touched
    // across the barrier are double-buffered by column parity.
    constexpr int NWP = NT / 32;
    cg::cluster_group cluster = cg::this_cluster();
    const int g = (int)cluster.block_rank();
    const int CL = (int)cluster.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned full = 0xffffffffu;

    __shared__ __align__(16) T cand_rows[2][CLMAX][W];   // pushed by every CTA
    __shared__ __align__(16) T diag_rows[2][W];          // pushed by the owner of row kc
    __shared__ Cand slot[2][CLMAX];                       // pushed by every CTA
    __shared__ int diag_org[2], diag_lorg[2];
    __shared__ unsigned whi[2][NWP], wlo[2][NWP];
    __shared__ int wpos[2][NWP];

    const long long n = a.n, c0 = a.c0, ldw = a.ldw;
    const int w = a.w;
    constexpr int R = NT * RPT;                  // rows per CTA
    const long long base = c0 + (long long)g * R;
    const int nn = (int)(n - base);              // rows of this CTA that exist: local index < nn

    T x[RPT][W];
    int org[RPT], lorg[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int li = tid + NT * q;
        const bool valid = li < nn;
        const T *row = a.W + (base + li) * ldw + c0;
#pragma unroll
        for (int s = 0; s < W; ++s) x[q][s] = (valid && s < w) ? row[s] : T(0);
        org[q] = valid ? a.orig[base + li] : -1;
        lorg[q] = (int)(base + li);
    }

#pragma unroll 1
    for (int c = 0; c < w; ++c) {
        const int par = c & 1;
        const long long kc = c0 + c;
        const int kl = (int)(kc - base);          // local index of row kc (may be out of range)
        // ---- this thread's candidate for column c (slot 0 of the frame), then warp / CTA arg-max
        unsigned hi = 0u, lo = 0u;
        int pos = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int li = tid + NT * q;
            if (li < nn && li >= kl) {
                unsigned h, l;
                abs_key(x[q][0], h, l);
                if (pos == 0x7fffffff || h > hi || (h == hi && l > lo)) { hi = h; lo = l; pos = (int)(base + li); }
            }
        }
        warp_argmax(hi, lo, pos);
        if (lane == 0) { whi[par][warp] = hi; wlo[par][warp] = lo; wpos[par][warp] = pos; }
        __syncthreads();
        {
            unsigned h = lane < NWP ? whi[par][lane] : 0u;
            unsigned l = lane < NWP ? wlo[par][lane] : 0u;
            int ps = lane < NWP ? wpos[par][lane] : 0x7fffffff;
            warp_argmax(h, l, ps);
            hi = h; lo = l; pos = ps;             // CTA candidate, known to every warp
        }
        // ---- the warp holding the CTA candidate pushes record + row into every CTA
        if (pos != 0x7fffffff) {
            const int li = (int)(pos - base);
            if ((li % NT) / 32 == warp) {
                const int src = li % 32, qq = li / NT;
                T v = T(0);
                int o = 0, lo_ = 0;
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
#pragma unroll
                    for (int s = 0; s < W; ++s) {
                        const T t = __shfl_sync(full, x[q][s], src);
                        if (q == qq && s == (lane % W)) v = t;
                    }
                    const int to = __shfl_sync(full, org[q], src);
                    const int tl = __shfl_sync(full, lorg[q], src);
                    if (q == qq) { o = to; lo_ = tl; }
                }
                // lanes 0..W-1 push element lane to CTAs r = 0.. (32/W lanes per element cover CTAs)
                for (int r = lane / W; r < CL; r += 32 / W)
                    *cluster.map_shared_rank(&cand_rows[par][g][lane % W], r) = v;
                if (lane < CL) {
                    Cand rec;
                    rec.hi = hi; rec.lo = lo; rec.pos = pos; rec.pad = 0;
                    rec.org = o; rec.lorg = lo_; rec.pad1 = rec.pad2 = 0;
                    *cluster.map_shared_rank(&slot[par][g], lane) = rec;
                }
            }
        } else if (warp == 0 && lane < CL) {
            Cand rec = {0u, 0u, 0x7fffffff, 0, -1, -1, 0, 0};
            *cluster.map_shared_rank(&slot[par][g], lane) = rec;
        }
        // ---- the warp holding row kc pushes it (the owner of p needs it after the barrier)
        if (kl >= 0 && kl < R && kl < nn && (kl % NT) / 32 == warp) {
            const int src = kl % 32, qq = kl / NT;
            T v = T(0);
            int o = 0, lo_ = 0;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
#pragma unroll
                for (int s = 0; s < W; ++s) {
                    const T t = __shfl_sync(full, x[q][s], src);
                    if (q == qq && s == (lane % W)) v = t;
                }
                const int to = __shfl_sync(full, org[q], src);
                const int tl = __shfl_sync(full, lorg[q], src);
                if (q == qq) { o = to; lo_ = tl; }
            }
            for (int r = lane / W; r < CL; r += 32 / W)
                *cluster.map_shared_rank(&diag_rows[par][lane % W], r) = v;
            if (lane < CL) {
                *cluster.map_shared_rank(&diag_org[par], lane) = o;
                *cluster.map_shared_rank(&diag_lorg[par], lane) = lo_;
            }
        }
        cluster.sync();                                   // the one cluster barrier of this column

        // ---- every warp: identical arg-max over the CL slots (all local now)
        unsigned ph = lane < CL ? slot[par][lane].hi : 0u;
        unsigned pl = lane < CL ? slot[par][lane].lo : 0u;
        int p = lane < CL ? slot[par][lane].pos : 0x7fffffff;
        const int myp = p;
        warp_argmax(ph, pl, p);
        const int gw = __ffs(__ballot_sync(full, myp == p && lane < CL)) - 1;
        const T *prow = &cand_rows[par][gw][0];
        const T *drow = &diag_rows[par][0];
        const bool zero_piv = (ph == 0u && pl == 0u);
        // row kc is final: its owner CTA writes it out (un-rotating through shared memory)
        if (kl >= 0 && kl < R) {
            if (tid < w) a.W[kc * ldw + c0 + tid] = prow[(tid - c + W) % W];
            if (tid == 0) {
                a.orig[kc] = slot[par][gw].org;
                const int plorg = slot[par][gw].lorg;
                if (plorg != (int)kc) {
                    const int si = atomicAdd(a.npairs, 1);
                    a.pairs[2 * si] = (int32_t)kc;
                    a.pairs[2 * si + 1] = plorg;
                }
            }
        }
        if (g == 0 && tid == 0) {
            a.ipiv[kc] = (int32_t)p;
            if (zero_piv) {                               // exact zero pivot
                atomicOr(&a.st->flags, (int)ST_ZERO_PIVOT);
                atomicMin(&a.st->zero_col, (int)(kc + 1));
            }
        }

        // ---- install the interchange, scale, rank-1 update, rotate
        const T piv = prow[0];
        const bool scale = piv != T(0);
        T pu[W];
#pragma unroll
        for (int s = 1; s < W; ++s) pu[s] = (s < W - c) ? prow[s] : T(0);
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int li = tid + NT * q;
            if (p != (int)kc && base + li == p) {
#pragma unroll
                for (int s = 0; s < W; ++s) x[q][s] = drow[s];
                org[q] = diag_org[par];
                lorg[q] = diag_lorg[par];
            }
            if (li > kl && li < nn) {
                const T l = scale ? x[q][0] / piv : x[q][0];
#pragma unroll
                for (int s = 1; s < W; ++s) x[q][s] = fma(-l, pu[s], x[q][s]);
#pragma unroll
                for (int s = 0; s < W - 1; ++s) x[q][s] = x[q][s + 1];
                x[q][W - 1] = l;
            }
        }
    }

    // ---- write back the rows below the leaf's diagonal block (rotated by w: column j
    //      lives in slot j + W - w); rows c0 .. c0+w-1 were written when they became final
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int li = tid + NT * q;
        const long long pos = base + li;
        if (pos >= c0 + w && li < nn) {
            T *row = a.W + pos * ldw + c0;
#pragma unroll
            for (int s = 0; s < W; ++s) {
                const int j = s - (W - w);
                if (j >= 0) row[j] = x[q][s];
            }
            a.orig[pos] = org[q];
            if (lorg[q] != (int)pos) {
                const int si = atomicAdd(a.npairs, 1);
                a.pairs[2 * si] = (int32_t)pos;
                a.pairs[2 * si + 1] = lorg[q];
            }
        }
    }
    cluster.sync();   // no CTA may exit while others can still write into its shared memory
}

__global__ void orig_init_kernel(int32_t *orig, int64_t k, int64_t n)
{
    for (int64_t i = k + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        orig[i] = (int32_t)i;
}

__global__ void emit_pairs_kernel(const int32_t *orig, int64_t k, int64_t n, int32_t *pairs, int32_t *npairs)
{
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
struct LeafCfg { int nt, rpt, w; };

// capacity per cluster = CL * nt * rpt rows; data registers rpt * w * sizeof(T) / 4 <= 64
constexpr LeafCfg kCfgF[] = {{256, 1, 32}, {512, 2, 32}, {512, 4, 16}, {512, 8, 8}};
constexpr LeafCfg kCfgD[] = {{256, 1, 32}, {512, 2, 16}, {512, 4, 8}, {512, 8, 4}};

int g_cluster = 0;   // cluster size chosen at first use (16, else 8)

template <typename T, int NT, int RPT, int W>
void launch_cfg(const LeafArgs<T> &a, int cl, cudaStream_t s)
{
    auto kern = panel_cluster_kernel<T, NT, RPT, W>;
    if (cl > 8) func_cluster16_once((const void *)kern);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl, 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MP_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
}

int cluster_size()
{
    if (g_cluster) return g_cluster;
    // can a 16-CTA cluster of the widest configuration be resident?
    auto kern = panel_cluster_kernel<float, 512, 2, 32>;
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

int select_cfg(size_t elem, int64_t m, int cl)
{
    const LeafCfg *c = elem == 4 ? kCfgF : kCfgD;
    for (int i = 0; i < 4; ++i)
        if ((int64_t)cl * c[i].nt * c[i].rpt >= m) return i;
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
                       DevStatus *st, cudaStream_t s)
{
    const int cl = cluster_size();
    const int sel = select_cfg(sizeof(T), n - c0, cl);
    if (sel < 0 || w > (sizeof(T) == 4 ? kCfgF : kCfgD)[sel].w)
        throw CudaError{cudaErrorInvalidValue, "panel leaf does not fit one cluster", __LINE__};
    LeafArgs<T> a;
    a.W = W; a.ldw = ldw; a.n = n; a.c0 = c0; a.w = w; a.ipiv = ipiv;
    a.orig = ps.orig; a.pairs = ps.pairs; a.npairs = ps.npairs; a.st = st;
    MP_CUDA(cudaMemsetAsync(ps.npairs, 0, sizeof(int32_t), s));
    if constexpr (sizeof(T) == 4) {
        switch (sel) {
        case 0: launch_cfg<T, 256, 1, 32>(a, cl, s); break;
        case 1: launch_cfg<T, 512, 2, 32>(a, cl, s); break;
        case 2: launch_cfg<T, 512, 4, 16>(a, cl, s); break;
        default: launch_cfg<T, 512, 8, 8>(a, cl, s); break;
        }
    } else {
        switch (sel) {
        case 0: launch_cfg<T, 256, 1, 32>(a, cl, s); break;
        case 1: launch_cfg<T, 512, 2, 16>(a, cl, s); break;
        case 2: launch_cfg<T, 512, 4, 8>(a, cl, s); break;
        default: launch_cfg<T, 512, 8, 4>(a, cl, s); break;
        }
    }
    ++g_launches;
}

void launch_orig_init(int32_t *orig, int64_t k, int64_t n, cudaStream_t s)
{
    orig_init_kernel<<<(int)std::min<int64_t>(ceil_div(n - k, 256), 512), 256, 0, s>>>(orig, k, n);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

void launch_emit_pairs(const int32_t *orig, int64_t k, int64_t n, int32_t *pairs, int32_t *npairs, cudaStream_t s)
{
    MP_CUDA(cudaMemsetAsync(npairs, 0, sizeof(int32_t), s));
    emit_pairs_kernel<<<(int)std::min<int64_t>(ceil_div(n - k, 256), 512), 256, 0, s>>>(orig, k, n, pairs, npairs);
    MP_LAUNCH_CHECK();
    ++g_launches;
}

template int panel_leaf_width<float>(int64_t);
template int panel_leaf_width<double>(int64_t);
template void launch_panel_leaf<float>(float *, int64_t, int64_t, int64_t, int, int32_t *, PanelScratch &,
                                       DevStatus *, cudaStream_t);
template void launch_panel_leaf<double>(double *, int64_t, int64_t, int64_t, int, int32_t *, PanelScratch &,
                                        DevStatus *, cudaStream_t);

}  // namespace mp
