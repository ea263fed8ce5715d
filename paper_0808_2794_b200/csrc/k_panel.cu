// k_panel.cu — K2: panel factorisation (GEPP on an m x w column panel).
//
// PAPER.md P:89-92 / Alg. 1 line 1: "Partial row pivoting ... PA = LU".
// Per column c of the panel: the pivot is the entry of largest |a| on/below
// the diagonal, ties to the smallest row position (reading A-6); rows
// kc = c0+c and p are interchanged over the whole panel width; the entries
// below the pivot are divided by it (reading A-7: IEEE division, as the
// oracle); the remaining panel columns get the rank-1 update.  An exact zero
// pivot is recorded (status ST_ZERO_PIVOT, first column) and elimination
// continues without scaling (the driver then takes the binary64 fallback,
// P:603-605 / iters = -3).
//
// B200 design: the panel rows are distributed over G <= #SM co-resident CTAs
// (cooperative launch), each holding its R x w slab in SHARED MEMORY for the
// whole leaf (227 KB per SM; 148 SMs hold a 16384 x 256 binary32 panel).  One
// grid barrier per column: before it every CTA publishes its local pivot
// candidate *with the candidate row* (and the owner of row kc publishes row
// kc); after it every CTA redundantly reduces the <= 148 candidates, installs
// the swap locally and applies the rank-1 update, fusing the arg-max search of
// the next column into that update.  Latency-bound: ~1 barrier per column.
#include <algorithm>
#include <cooperative_groups.h>

#include "internal.h"


namespace mp {

namespace {

constexpr int PT = 256;          // threads per CTA
constexpr int NW = PT / 32;

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire_u32(bar) < target) { }
        __threadfence();
    }
    __syncthreads();
}

template <typename T>
__device__ __forceinline__ double absd(T v) { return (double)fabs(v); }

// better candidate: larger |a|, ties -> smaller position; NaN never wins
__device__ __forceinline__ bool better(double v, long long pos, double bv, long long bpos)
{
    return v > bv || (v == bv && pos >= 0 && (bpos < 0 || pos < bpos));
}

template <typename T>
struct LeafArgs {
    T *W;
    long long ldw, n, c0;
    int w, R, G;
    int32_t *ipiv;
    T *cand_rows;        // [2][G][w]
    T *diag_rows;        // [2][w]
    double *cand_val;    // [2][G]
    int32_t *cand_pos;   // [2][G]
    int32_t *cand_orig;  // [2][G]
    int32_t *diag_orig;  // [2]
    unsigned *bar;
    int32_t *pairs;      // [2w][2]
    int32_t *npairs;
    DevStatus *st;
};

template <typename T>
__global__ void __launch_bounds__(PT, 1) panel_leaf_kernel(LeafArgs<T> a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int w = a.w, R = a.R, G = a.G;
    T *slab = reinterpret_cast<T *>(smem_raw);                 // [R][w]
    T *prow = slab + (size_t)R * w;                              // [w]
    int32_t *orig = reinterpret_cast<int32_t *>(prow + w);       // [R]
    __shared__ double red_v[NW];
    __shared__ long long red_p[NW];
    __shared__ int red_r[NW];
    __shared__ double s_cval;
    __shared__ long long s_cpos;
    __shared__ int s_crow;
    __shared__ long long s_p;
    __shared__ int s_pg;
    __shared__ T s_piv;

    const int g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m = a.n - a.c0;
    const long long pos0 = a.c0 + (long long)g * R;                  // first position owned
    const long long rem = m - (long long)g * R;
    const int nloc = rem <= 0 ? 0 : (rem < R ? (int)rem : R);
    T *W = a.W;
    const long long ldw = a.ldw, c0 = a.c0;

    // ---- load slab (rows pos0.., columns c0..c0+w) and origins
    for (int idx = tid; idx < nloc * w; idx += PT) {
        const int r = idx / w, cc = idx - r * w;
        slab[idx] = W[(pos0 + r) * ldw + c0 + cc];
    }
    for (int r = tid; r < nloc; r += PT) orig[r] = (int32_t)(pos0 + r);
    __syncthreads();

    // ---- candidate for column 0
    {
        double bv = -1.0; long long bp = -1; int br = -1;
        for (int r = tid; r < nloc; r += PT) {
            const double v = absd(slab[r * w + 0]);
            if (better(v, pos0 + r, bv, bp)) { bv = v; bp = pos0 + r; br = r; }
        }
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const long long op = __shfl_xor_sync(0xffffffffu, bp, o);
            const int orr = __shfl_xor_sync(0xffffffffu, br, o);
            if (better(ov, op, bv, bp)) { bv = ov; bp = op; br = orr; }
        }
        if (lane == 0) { red_v[warp] = bv; red_p[warp] = bp; red_r[warp] = br; }
        __syncthreads();
        if (tid == 0) {
            double v = -1.0; long long p = -1; int rr = -1;
            for (int k = 0; k < NW; ++k)
                if (better(red_v[k], red_p[k], v, p)) { v = red_v[k]; p = red_p[k]; rr = red_r[k]; }
            s_cval = v; s_cpos = p; s_crow = rr;
        }
        __syncthreads();
    }

    for (int c = 0; c < w; ++c) {
        const int par = c & 1;
        const long long kc = c0 + c;
        T *crow_g = a.cand_rows + ((size_t)par * G + g) * w;
        T *drow_g = a.diag_rows + (size_t)par * w;
        // ---- publish candidate (+ row) and, if owned, row kc
        const int crow = s_crow;
        if (tid == 0) {
            a.cand_val[par * G + g] = s_cval;
            a.cand_pos[par * G + g] = (int32_t)s_cpos;
            a.cand_orig[par * G + g] = crow >= 0 ? orig[crow] : -1;
        }
        if (crow >= 0)
            for (int cc = tid; cc < w; cc += PT) crow_g[cc] = slab[crow * w + cc];
        const long long kl = kc - pos0;                            // local index of row kc
        const bool own_k = kl >= 0 && kl < nloc;
        if (own_k) {
            for (int cc = tid; cc < w; cc += PT) drow_g[cc] = slab[kl * w + cc];
            if (tid == 0) a.diag_orig[par] = orig[kl];
        }
        grid_barrier(a.bar, (unsigned)(c + 1) * (unsigned)G);

        // ---- reduce the G candidates (every CTA, identical result)
        {
            double bv = -1.0; long long bp = -1; int bg = -1;
            for (int t = tid; t < G; t += PT) {
                const double v = __ldcg(a.cand_val + par * G + t);
                const long long p = __ldcg(a.cand_pos + par * G + t);
                if (p >= 0 && better(v, p, bv, bp)) { bv = v; bp = p; bg = t; }
            }
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const long long op = __shfl_xor_sync(0xffffffffu, bp, o);
                const int og = __shfl_xor_sync(0xffffffffu, bg, o);
                if (better(ov, op, bv, bp)) { bv = ov; bp = op; bg = og; }
            }
            if (lane == 0) { red_v[warp] = bv; red_p[warp] = bp; red_r[warp] = bg; }
            __syncthreads();
            if (tid == 0) {
                double v = -1.0; long long p = -1; int pg = -1;
                for (int k = 0; k < NW; ++k)
                    if (better(red_v[k], red_p[k], v, p)) { v = red_v[k]; p = red_p[k]; pg = red_r[k]; }
                if (p < 0) { p = kc; pg = -1; }                  // all-NaN column: no interchange
                s_p = p; s_pg = pg;
                if (g == 0) {
                    a.ipiv[kc] = (int32_t)p;
                    if (v == 0.0) {                              // exact zero pivot
                        atomicOr(&a.st->flags, (int)ST_ZERO_PIVOT);
                        atomicMin(&a.st->zero_col, (int)(kc + 1));
                    }
                }
            }
            __syncthreads();
        }
        const long long p = s_p;
        const int pg = s_pg;
        // ---- fetch the pivot row; install the interchange locally
        if (pg >= 0) {
            const T *src = a.cand_rows + ((size_t)par * G + pg) * w;
            for (int cc = tid; cc < w; cc += PT) prow[cc] = __ldcg(src + cc);
        } else if (own_k) {
            for (int cc = tid; cc < w; cc += PT) prow[cc] = slab[kl * w + cc];
        } else {
            for (int cc = tid; cc < w; cc += PT) prow[cc] = __ldcg(drow_g + cc);
        }
        __syncthreads();
        if (p != kc) {
            if (own_k) {
                for (int cc = tid; cc < w; cc += PT) slab[kl * w + cc] = prow[cc];
                if (tid == 0) orig[kl] = __ldcg(a.cand_orig + par * G + pg);
            }
            const long long pl = p - pos0;
            if (pl >= 0 && pl < nloc) {
                for (int cc = tid; cc < w; cc += PT) slab[pl * w + cc] = __ldcg(drow_g + cc);
                if (tid == 0) orig[pl] = __ldcg(a.diag_orig + par);
            }
        }
        if (tid == 0) s_piv = prow[c];
        __syncthreads();

        // ---- scale + rank-1 update of local rows below kc; arg-max of column c+1
        const T piv = s_piv;
        const bool scale = piv != (T)0;
        const int r_begin = (kc + 1 - pos0 > 0) ? (int)(kc + 1 - pos0) : 0;
        double bv = -1.0; long long bp = -1; int br = -1;
        for (int r = r_begin + warp; r < nloc; r += NW) {
            T *row = slab + (size_t)r * w;
            const T v = row[c];
            const T l = scale ? v / piv : v;
            for (int cc = c + 1 + lane; cc < w; cc += 32) {
                const T nv = row[cc] - l * prow[cc];
                row[cc] = nv;
                if (cc == c + 1) {
                    const double av = absd(nv);
                    if (better(av, pos0 + r, bv, bp)) { bv = av; bp = pos0 + r; br = r; }
                }
            }
            __syncwarp();
            if (lane == 0) row[c] = l;
        }
        if (c + 1 < w) {
            // lane 0 of every warp holds its warp's candidate for column c+1
            if (lane == 0) { red_v[warp] = bv; red_p[warp] = bp; red_r[warp] = br; }
            __syncthreads();
            if (tid == 0) {
                double v = -1.0; long long pp = -1; int rr = -1;
                for (int k = 0; k < NW; ++k)
                    if (better(red_v[k], red_p[k], v, pp)) { v = red_v[k]; pp = red_p[k]; rr = red_r[k]; }
                s_cval = v; s_cpos = pp; s_crow = rr;
            }
        }
        __syncthreads();
    }

    // ---- write back the slab; emit (position, origin) pairs of moved rows
    for (int idx = tid; idx < nloc * w; idx += PT) {
        const int r = idx / w, cc = idx - r * w;
        W[(pos0 + r) * ldw + c0 + cc] = slab[idx];
    }
    for (int r = tid; r < nloc; r += PT) {
        if (orig[r] != (int32_t)(pos0 + r)) {
            const int slot = atomicAdd(a.npairs, 1);
            a.pairs[2 * slot] = (int32_t)(pos0 + r);
            a.pairs[2 * slot + 1] = orig[r];
        }
    }
}

constexpr size_t kSmemCap = 227 * 1024 - 2048;   // leave room for static smem

template <typename T>
size_t leaf_smem(int R, int w) { return (size_t)R * w * sizeof(T) + (size_t)w * sizeof(T) + (size_t)R * 4 + 16; }

template <typename T>
int choose_R(int64_t m, int w, int num_sms)
{
    long long R = std::max<long long>(32, ceil_div(m, num_sms));
    R = round_up(R, 8);
    if (R > m) R = std::max<long long>(1, m);
    return (int)R;
}

}  // namespace

size_t panel_scratch_bytes(int wmax, size_t elem)
{
    size_t b = 0;
    b += 2 * (size_t)kMaxSMs * wmax * elem;          // cand_rows
    b += 2 * (size_t)wmax * elem;                    // diag_rows
    b += 2 * (size_t)kMaxSMs * sizeof(double);       // cand_val
    b += 2 * (size_t)kMaxSMs * 4 * 2;                // cand_pos, cand_orig
    b += 2 * 4 + 4 + 4 * 2 * 2 * (size_t)wmax + 64; // diag_orig, barrier, pairs, npairs
    return b + 256;
}

void panel_scratch_carve(PanelScratch &ps, void *base, int wmax, size_t elem)
{
    unsigned char *p = static_cast<unsigned char *>(base);
    auto take = [&](size_t bytes) { void *r = p; p += round_up((int64_t)bytes, 16); return r; };
    ps.cand_rows = take(2 * (size_t)kMaxSMs * wmax * elem);
    ps.diag_rows = take(2 * (size_t)wmax * elem);
    ps.cand_val = static_cast<double *>(take(2 * (size_t)kMaxSMs * sizeof(double)));
    ps.cand_pos = static_cast<int32_t *>(take(2 * (size_t)kMaxSMs * 4));
    ps.cand_orig = static_cast<int32_t *>(take(2 * (size_t)kMaxSMs * 4));
    ps.diag_orig = static_cast<int32_t *>(take(2 * 4));
    ps.barrier = static_cast<unsigned *>(take(4));
    ps.npairs = static_cast<int32_t *>(take(4));
    ps.pairs = static_cast<int32_t *>(take(4 * 2 * 2 * (size_t)wmax));
}

template <typename T>
int panel_leaf_fits(int64_t m, int w, int num_sms)
{
    const int R = choose_R<T>(m, w, num_sms);
    return leaf_smem<T>(R, w) <= kSmemCap && ceil_div(m, R) <= num_sms;
}

template <typename T>
void launch_panel_leaf(T *W, int64_t ldw, int64_t n, int64_t c0, int w, int32_t *ipiv, PanelScratch &ps,
                       DevStatus *st, int num_sms, cudaStream_t s)
{
    const int64_t m = n - c0;
    const int R = choose_R<T>(m, w, num_sms);
    const int G = (int)ceil_div(m, R);
    const size_t smem = leaf_smem<T>(R, w);
    LeafArgs<T> a;
    a.W = W; a.ldw = ldw; a.n = n; a.c0 = c0; a.w = w; a.R = R; a.G = G; a.ipiv = ipiv;
    a.cand_rows = static_cast<T *>(ps.cand_rows);
    a.diag_rows = static_cast<T *>(ps.diag_rows);
    a.cand_val = ps.cand_val; a.cand_pos = ps.cand_pos; a.cand_orig = ps.cand_orig;
    a.diag_orig = ps.diag_orig; a.bar = ps.barrier; a.pairs = ps.pairs; a.npairs = ps.npairs; a.st = st;
    MP_CUDA(cudaMemsetAsync(ps.barrier, 0, 4, s));
    MP_CUDA(cudaMemsetAsync(ps.npairs, 0, 4, s));
    auto kern = panel_leaf_kernel<T>;
    MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    void *args[] = {&a};
    MP_CUDA(cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(PT), args, smem, s));
    ++g_launches;
}

template int panel_leaf_fits<float>(int64_t, int, int);
template int panel_leaf_fits<double>(int64_t, int, int);
template void launch_panel_leaf<float>(float *, int64_t, int64_t, int64_t, int, int32_t *, PanelScratch &,
                                       DevStatus *, int, cudaStream_t);
template void launch_panel_leaf<double>(double *, int64_t, int64_t, int64_t, int, int32_t *, PanelScratch &,
                                        DevStatus *, int, cudaStream_t);

}  // namespace mp
