// driver.cu — host orchestration of the hot path and the C-ABI entry points of
// include/mp_solve.h.
//
// mp_dsgesv  = PAPER.md Algorithm 1 with BASELINE.json B:5's stop
//              test, 30-correction cap and binary64 fallback
//              (P:603-605):
//   K1 demote+||A||_F -> binary32 blocked GEPP (K2 panel / K3 laswp / K4 trsm /
//   K5 Schur update) -> x0 (K6 + K7) -> loop { K8+K10 residual & test ->
//   host reads one status record -> K7+K9 correction }.
// mp_dgesv   = the same blocked GEPP and solves instantiated in binary64, no
//              refinement (the "standard double precision solver").
//
// Every step runs in the kernels of this library; the host only sequences
// launches and reads the per-iteration status.  There is no CPU fallback: a
// missing GPU or a CUDA error is returned as MP_ERR_CUDA.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "../../include/mp_solve.h"
#include "../../include/mp_kernels.h"
#include "internal.h"

namespace mp {

thread_local int64_t g_launches = 0;
bool pdl_enabled()
{
    static const bool on = [] {
        const char *e = std::getenv("MP_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

namespace {
std::mutex g_attr_mu;
std::map<std::pair<const void *, int>, size_t> g_attr_smem;
std::set<std::pair<const void *, int>> g_attr_cl16;
}  // namespace

void func_smem_once(const void *fn, size_t bytes)
{
    int dev = 0;
    MP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t &cur = g_attr_smem[{fn, dev}];
    if (bytes > cur) {
        MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        cur = bytes;
    }
}

void func_cluster16_once(const void *fn)
{
    int dev = 0;
    MP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (g_attr_cl16.insert({fn, dev}).second)
        MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}
static thread_local std::string g_err;
static thread_local cudaStream_t g_stream = nullptr;

struct NoMem {};

// ------------------------------------------------------------------ per-class timing
namespace {
struct ProfRec { int cls, a, b; double work; cudaStream_t s; };
struct ProfState {
    bool on = false;
    unsigned mask = ~0u;         // classes recorded (flags bit 3: trailing update + residual only)
    std::vector<cudaEvent_t> ev;
    size_t used = 0;
    int open[KC_COUNT] = {0};
    std::vector<ProfRec> recs;
    int take() {
        if (used == ev.size()) {
            cudaEvent_t e;
            MP_CUDA(cudaEventCreate(&e));
            ev.push_back(e);
        }
        return (int)used++;
    }
    bool deferred = false;       // keep records across calls until mp_profile_collect()
    void reset(bool enable, bool defer) {
        on = enable;
        if (!(deferred && defer)) { used = 0; recs.clear(); }
        deferred = defer;
    }
};
thread_local ProfState g_prof;
}  // namespace

void prof_begin(int cls, cudaStream_t s)
{
    if (!g_prof.on || !((g_prof.mask >> cls) & 1u)) return;
    const int i = g_prof.take();
    MP_CUDA(cudaEventRecord(g_prof.ev[i], s));
    g_prof.open[cls] = i;
}

void prof_end(int cls, double work, cudaStream_t s)
{
    if (!g_prof.on || !((g_prof.mask >> cls) & 1u)) return;
    const int i = g_prof.take();
    MP_CUDA(cudaEventRecord(g_prof.ev[i], s));
    g_prof.recs.push_back({cls, g_prof.open[cls], i, work, s});
}

static void prof_collect(mp_report *rep)
{
    if (!rep || g_prof.recs.empty()) return;
    if (const char *path = std::getenv("MP_TIMELINE")) {        // debug: per-launch device timeline
        if (FILE *f = std::fopen(path, "a")) {
            static const char *names[] = {"demote", "panel", "laswp", "trsm", "gemm", "solve", "residual", "trail"};
            std::fprintf(f, "# call\n");
            std::vector<cudaStream_t> sids;
            for (const ProfRec &r : g_prof.recs) {
                int sid = 0;
                while (sid < (int)sids.size() && sids[sid] != r.s) ++sid;
                if (sid == (int)sids.size()) sids.push_back(r.s);
                float t0 = 0.f, t1 = 0.f;
                cudaEventElapsedTime(&t0, g_prof.ev[g_prof.recs[0].a], g_prof.ev[r.a]);
                cudaEventElapsedTime(&t1, g_prof.ev[g_prof.recs[0].a], g_prof.ev[r.b]);
                std::fprintf(f, "%s %.4f %.4f %d\n", names[r.cls], t0, t1, sid);
            }
            std::fclose(f);
        }
        cudaGetLastError();
    }
    for (const ProfRec &r : g_prof.recs) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, g_prof.ev[r.a], g_prof.ev[r.b]) != cudaSuccess) { cudaGetLastError(); t = 0.f; }
        rep->k_ms[r.cls] += t;
        rep->k_work[r.cls] += r.work;
        rep->k_launches[r.cls] += 1;
    }
}

namespace {

// ------------------------------------------------------------------ memory
cudaMemPool_t library_pool();

struct Pool {
    cudaStream_t s;
    std::vector<void *> ptrs;
    int64_t bytes = 0;
    explicit Pool(cudaStream_t st) : s(st) {}
    const int exc_at_ctor = std::uncaught_exceptions();
    ~Pool()
    {
        // unwinding from an error: work queued earlier on the look-ahead panel / update streams
        // may still use these buffers; wait for the device before handing them back
        if (std::uncaught_exceptions() > exc_at_ctor) cudaDeviceSynchronize();
        release();
    }
    void release() {
        for (void *p : ptrs) cudaFreeAsync(p, s);
        ptrs.clear();
    }
    template <typename T>
    T *get(size_t count) {
        if (count == 0) count = 1;
        void *p = nullptr;
        const size_t b = round_up((int64_t)(count * sizeof(T)), 256);
        cudaError_t e = cudaMallocFromPoolAsync(&p, b, library_pool(), s);
        if (e == cudaErrorMemoryAllocation) { cudaGetLastError(); throw NoMem{}; }
        MP_CUDA(e);
        ptrs.push_back(p);
        bytes += (int64_t)b;
        return static_cast<T *>(p);
    }
};

// The library's own stream-ordered memory pool (one per device), kept warm between calls
// (release threshold = max) without touching the device's default pool, which other
// cudaMallocAsync users in the host process own.
cudaMemPool_t library_pool()
{
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    int dev = 0;
    MP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = pools.find(dev);
    if (it != pools.end()) return it->second;
    cudaMemPoolProps props;
    std::memset(&props, 0, sizeof(props));
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    MP_CUDA(cudaMemPoolCreate(&pool, &props));
    uint64_t thr = UINT64_MAX;
    MP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    pools.emplace(dev, pool);
    return pool;
}

// Size limits of the leaf cluster (one panel column fits one thread-block cluster) and of the
// triangular-solve helper grid, for both precisions (the binary64 fallback may run): checked
// before any allocation or launch, so an unsupported n fails without queued work.
void check_size_limits(int64_t n)
{
    if (n <= 0) return;
    if (panel_leaf_width<float>(n) <= 0 || panel_leaf_width<double>(n) <= 0)
        throw std::runtime_error("n exceeds the rows one panel cluster holds on this device");
    if (!solve_fits<float>(n) || !solve_fits<double>(n))
        throw std::runtime_error("n exceeds the triangular-solve helper grid");
}

bool is_device_ptr(const void *p)
{
    if (!p) return false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

bool overlaps(const void *a, size_t ab, const void *b, size_t bb)
{
    const char *pa = static_cast<const char *>(a), *pb = static_cast<const char *>(b);
    return pa < pb + bb && pb < pa + ab;
}

int num_sms()
{
    int dev = 0, sms = 0;
    MP_CUDA(cudaGetDevice(&dev));
    MP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return std::min(sms, kMaxSMs);
}

int default_nb(int64_t n) { return n <= 1024 ? 64 : (n <= 4096 ? 128 : 256); }

struct Timer {
    cudaEvent_t *e;
    int k = 0;
    cudaStream_t s;
    explicit Timer(cudaStream_t st) : s(st) {
        static thread_local cudaEvent_t pool[12];
        static thread_local bool made = false;
        if (!made) {
            for (auto &x : pool) MP_CUDA(cudaEventCreate(&x));
            made = true;
        }
        e = pool;
    }
    int mark() { MP_CUDA(cudaEventRecord(e[k], s)); return k++; }
    double ms(int a, int b) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, e[a], e[b]) != cudaSuccess) { cudaGetLastError(); return 0.0; }
        return (double)t;
    }
};

// ------------------------------------------------------------------ look-ahead execution resources
// the factorisation of panel k+1 overlaps the trailing update of step k.
// The panel work (leaf clusters, in-panel updates, the next panel's columns) runs on a
// stream of a 16-SM green context (one 16-CTA leaf cluster fits), the trailing update on
// a stream of a green context holding the remaining SMs, so the two never compete for SMs.
// Created once per device through driver entry points; if the device or driver refuses,
// the factorisation runs sequentially on the caller's stream.
struct ExecRes {
    bool ok = false;
    cudaStream_t sP = nullptr, sU = nullptr;
    int smsP = 0, smsU = 0;
    // a second stream on the update partition (the streamed e2e path's concurrent catch-up)
    cudaStream_t sC = nullptr;
    // a second, larger update partition for the early steps (the trailing update is then the
    // critical path); sU2 == nullptr: not available
    cudaStream_t sU2 = nullptr;
    int smsU2 = 0;
    double big_frac = 0.0;      // steps with n - k > big_frac * n use sU2
    // and a smaller one for the late steps (the panel is then the critical path)
    cudaStream_t sU3 = nullptr;
    int smsU3 = 0;
    double small_frac = 0.0;    // steps with n - k < small_frac * n use sU3
    // and the largest one for very large trailing matrices (C4 sizes: the update, not the panel,
    // is then the critical path at every step; the panel keeps one 16-SM cluster)
    cudaStream_t sU4 = nullptr;
    int smsU4 = 0;
    int64_t huge_rows = 0;      // steps with n - k > huge_rows use sU4
};

ExecRes make_exec_res(int dev)
{
    ExecRes r;
    if (const char *e = std::getenv("MP_NO_LOOKAHEAD"))
        if (e[0] == '1') return r;
    auto entry = [](const char *name) -> void * {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        return fn;
    };
    auto getRes = reinterpret_cast<PFN_cuDeviceGetDevResource_v12040>(entry("cuDeviceGetDevResource"));
    auto split = reinterpret_cast<PFN_cuDevSmResourceSplitByCount_v12040>(entry("cuDevSmResourceSplitByCount"));
    auto genDesc = reinterpret_cast<PFN_cuDevResourceGenerateDesc_v12040>(entry("cuDevResourceGenerateDesc"));
    auto mkCtx = reinterpret_cast<PFN_cuGreenCtxCreate_v12040>(entry("cuGreenCtxCreate"));
    auto mkStream = reinterpret_cast<PFN_cuGreenCtxStreamCreate_v12050>(entry("cuGreenCtxStreamCreate"));
    if (!getRes || !split || !genDesc || !mkCtx || !mkStream) return r;
    CUdevResource all, grp[1], rest;
    unsigned ng = 1;
    if (getRes((CUdevice)dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return r;
    unsigned psms = 40;                       // SMs kept free of the trailing update (MP_PANEL_SMS)
    if (const char *e = std::getenv("MP_PANEL_SMS")) psms = (unsigned)std::max(16, std::atoi(e));
    if (split(grp, &ng, &all, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, psms) != CUDA_SUCCESS || ng != 1)
        return r;
    if (grp[0].sm.smCount < 16 || rest.sm.smCount < 32) return r;
    CUdevResourceDesc dP, dU;
    CUgreenCtx gP, gU;
    CUstream sP, sU;
    if (genDesc(&dP, grp, 1) != CUDA_SUCCESS || genDesc(&dU, &rest, 1) != CUDA_SUCCESS) return r;
    if (mkCtx(&gP, dP, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return r;
    if (mkCtx(&gU, dU, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return r;
    if (mkStream(&sU, gU, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return r;
    {
        CUstream sC;
        if (mkStream(&sC, gU, CU_STREAM_NON_BLOCKING, 0) == CUDA_SUCCESS) r.sC = (cudaStream_t)sC;
        cudaGetLastError();
    }
    {
        unsigned psms2 = 32;                  // SMs kept free during the early steps (MP_PANEL_SMS_EARLY)
        if (const char *e = std::getenv("MP_PANEL_SMS_EARLY")) psms2 = (unsigned)std::max(16, std::atoi(e));
        double frac = 0.75;                   // MP_EARLY_FRAC: trailing size above which they are "early"
        if (const char *e = std::getenv("MP_EARLY_FRAC")) frac = std::atof(e);
        CUdevResource grp2[1], rest2;
        unsigned ng2 = 1;
        CUdevResourceDesc dU2;
        CUgreenCtx gU2;
        CUstream sU2;
        if (psms2 < psms && frac < 1.0 &&
            split(grp2, &ng2, &all, &rest2, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, psms2) == CUDA_SUCCESS &&
            ng2 == 1 && grp2[0].sm.smCount >= 16 && genDesc(&dU2, &rest2, 1) == CUDA_SUCCESS &&
            mkCtx(&gU2, dU2, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM) == CUDA_SUCCESS &&
            mkStream(&sU2, gU2, CU_STREAM_NON_BLOCKING, 0) == CUDA_SUCCESS) {
            r.sU2 = (cudaStream_t)sU2;
            r.smsU2 = (int)rest2.sm.smCount;
            r.big_frac = frac;
        }
        cudaGetLastError();
    }
    {
        unsigned psms3 = 48;                  // SMs kept free during the late steps (MP_PANEL_SMS_LATE)
        if (const char *e = std::getenv("MP_PANEL_SMS_LATE")) psms3 = (unsigned)std::max(16, std::atoi(e));
        double frac = 0.0;                    // MP_LATE_FRAC: trailing size below which they are "late"
        if (const char *e = std::getenv("MP_LATE_FRAC")) frac = std::atof(e);
        CUdevResource grp3[1], rest3;
        unsigned ng3 = 1;
        CUdevResourceDesc dU3;
        CUgreenCtx gU3;
        CUstream sU3;
        if (psms3 > psms && frac > 0.0 &&
            split(grp3, &ng3, &all, &rest3, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, psms3) == CUDA_SUCCESS &&
            ng3 == 1 && rest3.sm.smCount >= 32 && genDesc(&dU3, &rest3, 1) == CUDA_SUCCESS &&
            mkCtx(&gU3, dU3, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM) == CUDA_SUCCESS &&
            mkStream(&sU3, gU3, CU_STREAM_NON_BLOCKING, 0) == CUDA_SUCCESS) {
            r.sU3 = (cudaStream_t)sU3;
            r.smsU3 = (int)rest3.sm.smCount;
            r.small_frac = frac;
        }
        cudaGetLastError();
    }
    {
        unsigned psms4 = 16;                  // SMs kept free for trailing matrices > MP_HUGE_ROWS rows (MP_PANEL_SMS_HUGE)
        if (const char *e = std::getenv("MP_PANEL_SMS_HUGE")) psms4 = (unsigned)std::max(16, std::atoi(e));
        int64_t rows = 16384;                 // (C3, n = 16384, never qualifies; C4 at n = 49152: 819 -> 768 ms)
        if (const char *e = std::getenv("MP_HUGE_ROWS")) rows = std::atoll(e);
        CUdevResource grp4[1], rest4;
        unsigned ng4 = 1;
        CUdevResourceDesc dU4;
        CUgreenCtx gU4;
        CUstream sU4;
        if (psms4 < psms && rows > 0 &&
            split(grp4, &ng4, &all, &rest4, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, psms4) == CUDA_SUCCESS &&
            ng4 == 1 && grp4[0].sm.smCount >= 16 && genDesc(&dU4, &rest4, 1) == CUDA_SUCCESS &&
            mkCtx(&gU4, dU4, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM) == CUDA_SUCCESS &&
            mkStream(&sU4, gU4, CU_STREAM_NON_BLOCKING, 0) == CUDA_SUCCESS) {
            r.sU4 = (cudaStream_t)sU4;
            r.smsU4 = (int)rest4.sm.smCount;
            r.huge_rows = rows;
        }
        cudaGetLastError();
    }
    // The panel stream is an ordinary (full-device, highest-priority) stream: its kernels run on
    // the SMs the update partition leaves free (a cluster-capable 16-SM group) while the
    // trailing update runs, and on the whole GPU otherwise.
    if (std::getenv("MP_PANEL_GREEN")) {
        if (mkStream(&sP, gP, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return r;
    } else {
        int lo = 0, hi = 0;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return r;
        cudaStream_t ps;
        if (cudaStreamCreateWithPriority(&ps, cudaStreamNonBlocking, hi) != cudaSuccess) return r;
        sP = (CUstream)ps;
    }
    r.ok = true;
    r.sP = (cudaStream_t)sP;
    r.sU = (cudaStream_t)sU;
    r.smsP = (int)grp[0].sm.smCount;
    r.smsU = (int)rest.sm.smCount;
    return r;
}

ExecRes &exec_res()
{
    static std::mutex mu;
    static std::map<int, ExecRes> per_dev;
    int dev = 0;
    MP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = per_dev.find(dev);
    if (it == per_dev.end()) it = per_dev.emplace(dev, make_exec_res(dev)).first;
    return it->second;
}

// small reusable event pool (disable-timing events for cross-stream ordering)
cudaEvent_t la_event(int i)
{
    static thread_local std::vector<cudaEvent_t> evs;
    while ((int)evs.size() <= i) {
        cudaEvent_t e;
        MP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs.push_back(e);
    }
    return evs[i];
}

// one non-blocking host-to-device copy stream per device (the streamed e2e path)
cudaStream_t copy_stream()
{
    static std::mutex mu;
    static std::map<int, cudaStream_t> per_dev;
    int dev = 0;
    MP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = per_dev.find(dev);
    if (it != per_dev.end()) return it->second;
    cudaStream_t cs;
    MP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    per_dev.emplace(dev, cs);
    return cs;
}

// ------------------------------------------------------------------ blocked GEPP
// Right-looking blocked LU (SGETRF's structure): for every panel of nb
// columns — recursive panel factorisation (cluster leaves K2 + in-panel K3/K4/K5),
// the panel's interchanges applied once to every other column (K3), U12 (K4),
// Schur update of the trailing matrix (K5).

// tensor-core trailing-update variants: 3xTF32 (binary32-accurate, the default) and 1xTF32 (SURVEY 8(f)
// NEXT-2: operands rounded to TF32, ~2^-11; refinement then needs kappa * 2^-11 < 1 or GMRES-IR)
inline bool tc_variant(int v) { return v == MP_VARIANT_3XTF32 || v == MP_VARIANT_TF32; }

template <typename T>
struct Factor {
    T *W;
    int64_t n, ldw;
    int32_t *ipiv, *perm;
    PanelScratch ps;
    int32_t *ppairs[2], *nppairs[2];   // panel-level pairs, double-buffered for the look-ahead
    // streamed path: every panel's pairs kept (slot k / nb), and the interchanges of the steps applied
    // to the columns [swap_lo, nc) only (the left factors get them later)
    int32_t *pairs_all = nullptr, *npairs_all = nullptr;
    int64_t swap_lo = 0;
    DevStatus *st;
    int nb;
    // wider panels while the trailing matrix is large (update-bound steps: the update's intensity on
    // the trailing matrix's HBM traffic doubles): steps with n - k > big_rows
    // take nb_big columns; 0 = every panel nb wide
    int nb_big = 0;
    int64_t big_rows = 0;
    int width_at(int64_t k) const { return (nb_big > nb && n - k > big_rows) ? nb_big : nb; }
    int variant = MP_VARIANT_FFMA;
    bool fuse_trsm = true;                 // MP_NO_FUSED_TRSM=1: separate K4 + K5 in the panel
    bool tc_inpanel = true;                // MP_NO_TC_INPANEL=1: FFMA tall-skinny GEMM for every in-panel level
    int psms = 148;                        // SMs the panel stream can count on
    int32_t *cur_np = nullptr;             // panel-level pair counter of the panel being factored
    EmitJob emit_job;                      // its pair emission, folded into the last leaf's laswp
    bool emitted = false;
    double terms4_frac = 0.0;              // MP_TF32_TERMS4_FRAC: steps with n - k below this * n use 4 MMAs
    float *tf32[2] = {nullptr, nullptr};
    float *tfU[2] = {nullptr, nullptr};    // look-ahead: update-stream scratch per step parity (the panel
                                           // stream writes step k+1's L21 split while step k still runs)   // 3xTF32 split scratch: [0] trailing stream, [1] panel stream
    int sms = 148;
    cudaStream_t s;

    void leaf(cudaStream_t q, int64_t c0, int w, int64_t klo, int64_t khi) {
        const double m = (double)(n - c0);
        prof_begin(KC_PANEL, q);
        launch_panel_leaf<T>(W, ldw, n, c0, w, ipiv, ps, st, q, c0 == klo ? cur_np : nullptr);
        prof_end(KC_PANEL, m * w * w - (double)w * w * w / 3.0, q);
        if (khi - klo > w) {   // the leaf's interchanges, on the rest of its panel
            prof_begin(KC_LASWP, q);
            // the panel's last leaf: the same launch emits the panel-level pairs
            const bool last = c0 + w == khi;
            launch_laswp_pairs<T>(W, ldw, ps.pairs, ps.npairs, 2 * w, klo, khi, c0, c0 + w, nullptr, q,
                                  last ? emit_job : EmitJob{});
            if (last) emitted = true;
            prof_end(KC_LASWP, 2.0 * 2 * w * (double)(khi - klo - w) * sizeof(T), q);
        }
    }
    void trsm(cudaStream_t q, int64_t r0, int w, int64_t c_lo, int64_t c_hi, float *sh = nullptr, float *sl = nullptr,
              int kp = 0) {
        prof_begin(KC_TRSM, q);
        launch_trsm_lower_unit<T>(W, ldw, r0, w, c_lo, c_hi, q, sh, sl, kp);
        prof_end(KC_TRSM, (double)w * w * (double)(c_hi - c_lo), q);
    }
    // Schur update C -= L U.  big: the trailing update or the next panel's columns
    // (tensor-core variant when selected); scratch / nsm: the launching stream's.
    void gemm(cudaStream_t q, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N, int64_t K, bool big,
              int cls, float *scratch, int nsm, bool reuse_a = false, int terms = 3, bool reuse_b = false,
              float *bscratch = nullptr) {
        prof_begin(cls, q);
        if constexpr (sizeof(T) == 4) {
            if (big && tc_variant(variant) && M >= 256 && N >= 128)
                launch_gemm_update_3xtf32(W, ldw, r0, c0, k0, M, N, K, scratch, nsm, q, reuse_a,
                                          variant == MP_VARIANT_TF32 ? 1 : terms, reuse_b, bscratch);
            else
                launch_gemm_update<T>(W, ldw, r0, c0, k0, M, N, K, q);
        } else {
            launch_gemm_update<T>(W, ldw, r0, c0, k0, M, N, K, q);
        }
        prof_end(cls, 2.0 * M * N * K, q);
    }
    // recursive panel: columns [c0, c0+w) of the panel [klo, khi), rows [c0, n)
    void panel(cudaStream_t q, int64_t c0, int w, int64_t klo, int64_t khi) {
        const int wl = panel_leaf_width<T>(n - c0);
        if (wl <= 0) throw std::runtime_error("matrix too tall for one panel cluster");
        if (w <= wl) { leaf(q, c0, w, klo, khi); return; }
        int w1 = (int)round_up(w / 2, 8);
        if (w1 > wl && w1 % wl) w1 = (int)round_up(w1, wl);
        // leaves narrower than 8 columns (binary64 leaves of m > 32768 rows are 4 wide): split on
        // the leaf width instead, so the recursion always shrinks
        if (w1 >= w) w1 = (int)round_up(w / 2, wl);
        if (w1 >= w) w1 = w - wl;
        panel(q, c0, w1, klo, khi);
        prof_begin(KC_GEMM, q);
        const bool fused = fuse_trsm &&
                           launch_trsm_gemm_fused<T>(W, ldw, c0 + w1, c0 + w1, c0, n - c0 - w1, w - w1, w1, ps.ticket, q);
        prof_end(KC_GEMM, fused ? 2.0 * (n - c0 - w1) * (w - w1) * w1 + (double)w1 * w1 * (w - w1) : 0.0, q);
        if (!fused) {
            // the widest in-panel level (K >= 128) on the tensor cores too, on the SMs the update leaves;
            // its TRSM writes U12's hi/lo split when the GEMM takes the 3xTF32 path
            const bool tc = tc_inpanel && w1 >= 128;
            const int64_t M = n - c0 - w1;
            const int kp = (int)round_up(w1, 4);
            const bool bsplit = sizeof(T) == 4 && tc && tc_variant(variant) && tf32[1] && M >= 256 &&
                                w - w1 >= 128 && w1 <= 256;
            float *bh = bsplit ? tf32[1] + 2 * (size_t)M * kp : nullptr;
            trsm(q, c0, w1, c0 + w1, c0 + w, bh, bsplit ? bh + (size_t)(w - w1) * kp : nullptr, kp);
            gemm(q, c0 + w1, c0 + w1, c0, M, w - w1, w1, tc, KC_GEMM, tc ? tf32[1] : nullptr, psms, false, 3, bsplit);
        }
        panel(q, c0 + w1, w - w1, klo, khi);
    }
    // panel [k, k+w) on stream q, its panel-level pairs into buffer b
    // Left-looking panel (binary32, w <= 256, MP_PANEL_LL=1 enables; off by default): the leaves run back to back,
    // each bringing its own columns up to date (k_panel.cu ll_catch_up) on rows that stay at their
    // panel-start positions; one interchange launch at the end moves the panel's rows to their
    // final positions.  Replaces the recursive panel's in-panel interchanges, TRSMs and updates.
    int32_t *lpos = nullptr;
    bool ll_panel = false;
    // step range and column limit (the streamed e2e path factors column blocks as they arrive):
    // panels k in [kb, ke), interchanges / U12 / Schur updates on columns [0, nc); rows always [0, n)
    int64_t kb = 0, ke = -1, nc = -1;
    void factor_panel(cudaStream_t q, int64_t k, int w, int b) {
        if (pairs_all) {
            ppairs[b] = pairs_all + (k / nb) * 4 * (int64_t)nb;
            nppairs[b] = npairs_all + k / nb;
        }
        cur_np = nppairs[b];                 // the first leaf zeroes it and starts orig[] as the identity
        emit_job = EmitJob{ps.orig, k, n, ppairs[b], nppairs[b]};
        emitted = false;
        if (ll_panel && lpos && sizeof(T) == 4 && w <= 256) {
            const int wl = std::min(32, panel_leaf_width<T>(n - k));   // (left-looking leaves: <= 32 wide)
            if (wl <= 0) throw std::runtime_error("matrix too tall for one panel cluster");
            for (int64_t c0 = k; c0 < k + w; c0 += wl) {
                const int ww = (int)std::min<int64_t>(wl, k + w - c0);
                prof_begin(KC_PANEL, q);
                launch_panel_leaf<T>(W, ldw, n, c0, ww, ipiv, ps, st, q, c0 == k ? cur_np : nullptr, k, lpos, k + w);
                prof_end(KC_PANEL, (double)(n - c0) * ww * ww + 2.0 * (double)(n - k) * (c0 - k) * ww, q);
            }
            launch_emit_pairs(ps.orig, k, n, ppairs[b], nppairs[b], q);
            prof_begin(KC_LASWP, q);
            launch_laswp_pairs<T>(W, ldw, ppairs[b], nppairs[b], 2 * w, k, k + w, 0, 0, nullptr, q);
            prof_end(KC_LASWP, 2.0 * 2 * w * (double)w * sizeof(T), q);
            return;
        }
        panel(q, k, w, k, k + w);
        if (!emitted) launch_emit_pairs(ps.orig, k, n, ppairs[b], nppairs[b], q);
    }
    void run_sequential() {
        psms = sms;
        if (kb == 0) launch_init_perm(perm, n, s);
        for (int64_t k = kb; k < ke;) {
            const int w = (int)std::min<int64_t>(width_at(k), ke - k);
            factor_panel(s, k, w, 0);
            // the panel's interchanges on every other column (left factors + trailing matrix)
            prof_begin(KC_LASWP, s);
            launch_laswp_pairs<T>(W, ldw, ppairs[0], nppairs[0], 2 * w, swap_lo, nc, k, k + w, perm, s);
            prof_end(KC_LASWP, 2.0 * 2 * w * (double)(nc - w) * sizeof(T), s);
            if (k + w < nc) {
                trsm(s, k, w, k + w, nc);                                                  // U12 <- L11^-1 A12
                gemm(s, k + w, k + w, k, n - k - w, nc - k - w, w, true, KC_TRAIL, tf32[0], sms);   // A22 -= L21 U12
            }
            k += w;
        }
    }
    // Bring the column block [c_lo, c_hi) (its rows already permuted by perm) up to date with the
    // panels [0, c_lo): U12 and the Schur update of every earlier step, in order (the right-looking
    // updates it missed while it was in flight; the later interchanges commute).
    float *tfC = nullptr;                  // the catch-up's own 3xTF32 scratch (it may run beside the look-ahead)
    void catch_up_panel(int64_t k, int64_t c_lo, int64_t c_hi, cudaStream_t q, int nsm) {
        const int w = (int)std::min<int64_t>(nb, c_lo - k);
        trsm(q, k, w, c_lo, c_hi);
        gemm(q, k + w, c_lo, k, n - k - w, c_hi - c_lo, w, true, KC_TRAIL, tfC ? tfC : tf32[0], nsm);
    }
    void catch_up(int64_t c_lo, int64_t c_hi, cudaStream_t q, int nsm) {
        for (int64_t k = 0; k < c_lo; k += nb) catch_up_panel(k, c_lo, c_hi, q, nsm);
    }
    // Streamed look-ahead: the column blocks of A join ONE look-ahead loop while it runs.
    // Block j joins at step join_at (on the update stream, after that step's interchanges: demote,
    // rows gathered into the current order, so from then on every panel's interchanges reach it), is
    // caught up panel by panel (U12 and Schur update of each earlier panel, in order, a share per step
    // so the work hides behind the panel chain like the ordinary trailing update), and receives the
    // ordinary per-step updates once caught up (nc_upd).  It must be caught up before the step whose
    // next-panel update reaches its first panel (need_at = c_lo - 2 nb).  Per entry: the same
    // operations in the same order as the one-shot factorisation (the interchanges commute, §9b).
    struct StreamBlock {
        int64_t c_lo, c_hi;
        cudaEvent_t ev;
        int64_t join_at, need_at;
        int64_t cu = 0;                    // caught up on the panels [0, cu)
        bool joined = false, regular = false;
    };
    struct Streamer {
        std::vector<StreamBlock> blk;
        const double *dA = nullptr;        // device A (column-major, ld n), filled block by block
        float *S = nullptr;                // binary32 staging of one block (row-major, ld lds)
        double *dpart = nullptr, *anrm_parts = nullptr;
        unsigned *dcnt = nullptr;
        int64_t nc_swap = 0, nc_upd = 0;   // columns reached by the interchanges / by the per-step update
        size_t next_join = 1;
        int ahead = 3;                     // look-ahead steps the host may enqueue beyond the device
    };
    Streamer *str = nullptr;
    void stream_join(StreamBlock &B, size_t j, cudaStream_t q) {
        const int64_t wcols = B.c_hi - B.c_lo, lds = round_up(wcols, 64);
        MP_CUDA(cudaStreamWaitEvent(q, B.ev, 0));
        if constexpr (sizeof(T) == 4) {          // (the streamed path is the binary32 factorisation's)
            prof_begin(KC_DEMOTE, q);
            launch_demote_rect<float>(str->dA + B.c_lo * n, n, n, wcols, str->S, lds, str->dpart, str->dcnt, st, q);
            MP_CUDA(cudaMemcpyAsync(str->anrm_parts + j, &st->anrm2, sizeof(double), cudaMemcpyDeviceToDevice, q));
            launch_gather_rows(str->S, lds, round_up(wcols, 4), perm, n, W + B.c_lo, ldw, q);
            prof_end(KC_DEMOTE, 12.0 * n * wcols, q);
        }
        B.joined = true;
        str->nc_swap = B.c_hi;
    }
    // step k's share of the streamed work (update stream q, after the step's interchanges)
    void stream_step(int64_t k, cudaStream_t q, int nsm) {
        Streamer &z = *str;
        // a block joins once its copy has landed (host-side query: the host runs at most a few steps
        // ahead of the device, see run_lookahead), at the latest at need_at (the update stream then
        // waits for the copy)
        while (z.next_join < z.blk.size() &&
               (z.blk[z.next_join].need_at <= k ||
                (z.blk[z.next_join].join_at <= k && cudaEventQuery(z.blk[z.next_join].ev) == cudaSuccess))) {
            stream_join(z.blk[z.next_join], z.next_join, q);
            ++z.next_join;
        }
        for (size_t j = 1; j < z.blk.size(); ++j) {
            StreamBlock &B = z.blk[j];
            if (B.regular) continue;
            if (!B.joined) break;
            // spread the remaining catch-up panels evenly over the steps left before need_at
            const int64_t left = (k - B.cu + nb - 1) / nb;
            const int64_t steps = std::max<int64_t>(1, (B.need_at - k) / nb + 1);
            int64_t todo = k >= B.need_at ? left : (left + steps - 1) / steps;
            while (B.cu < k && todo-- > 0) {
                catch_up_panel(B.cu, B.c_lo, B.c_hi, q, nsm);
                B.cu += nb;
            }
            if (B.cu < k) break;           // later blocks wait (updates stay contiguous)
            B.regular = true;              // caught up on [0, k): step k's own update is the ordinary one
            z.nc_upd = B.c_hi;
        }
    }
    // Look-ahead (depth 1).  Step k:
    //   update stream : [wait: panel k] panel-k interchanges on every other column; U12 and Schur
    //                   update of the NEXT panel's columns [kn, kn+wn) (all update-stream SMs,
    //                   tensor cores), event; then U12 and Schur update of the rest [kn+wn, n)
    //   panel stream  : [wait: next panel's columns updated] factor panel kn
    // so the factorisation of panel kn overlaps the trailing update of the rest; concurrent
    // work touches disjoint column sets; pair lists alternate between two buffers.
    void run_lookahead(const ExecRes &ex) {
        cudaStream_t sP = ex.sP, cur = ex.sU;
        psms = std::max(8, sms - ex.smsU);
        cudaEvent_t e0 = la_event(0), eP[2] = {la_event(1), la_event(2)}, eN = la_event(3);
        cudaEvent_t eEndP = la_event(4), eEndU = la_event(5), eSw = la_event(6), eS[2] = {la_event(7), la_event(8)};
        cudaEvent_t eR[2] = {la_event(9), la_event(10)};
        static const bool next_on_panel_env = [] { const char *e = std::getenv("MP_LA_NEXT_ON_PANEL"); return !e || e[0] != '0'; }();
        const bool next_on_panel = next_on_panel_env && sizeof(T) == 4;
        // L21 of panel j (rows [j + w, n) x its columns) split hi/lo on the panel stream right after
        // the panel, into the update scratch of that step's parity: the update stream's interchanges
        // and TRSM of the next panel's columns run meanwhile (the split is off its critical path)
        const bool presplit = sizeof(T) == 4 && tc_variant(variant) && tfU[1] != nullptr;
        auto split_l21 = [&](int64_t kp0, int wp, int bb, cudaStream_t q) -> bool {
            const int64_t M = n - kp0 - wp;
            if (!presplit || M < 256) return false;
            if constexpr (sizeof(T) == 4)
                launch_split_a_3xtf32(W + (kp0 + wp) * ldw + kp0, ldw, M, wp, tfU[bb], q);
            MP_CUDA(cudaEventRecord(eS[bb], q));
            return true;
        };
        bool split_ok[2] = {false, false};
        // steps that bring the next panel's columns up to date on the panel stream (see below); their
        // L21 split runs on the (then idle) update stream at the start of the step instead (pending)
        auto on_panel_step = [&](int64_t kk) {
            if (!next_on_panel || str || kk >= ke) return false;
            const int64_t kn_ = kk + std::min<int64_t>(width_at(kk), ke - kk);
            const bool huge_ = ex.sU4 && n - kn_ > ex.huge_rows;
            const bool early_ = !huge_ && ex.sU2 && (double)(n - kn_) > ex.big_frac * (double)n;
            return !huge_ && !early_ && kn_ < ke;
        };
        bool pending[2] = {false, false};
        MP_CUDA(cudaEventRecord(e0, s));
        MP_CUDA(cudaStreamWaitEvent(sP, e0, 0));
        MP_CUDA(cudaStreamWaitEvent(cur, e0, 0));
        if (kb == 0) launch_init_perm(perm, n, cur);
        factor_panel(sP, kb, (int)std::min<int64_t>(width_at(kb), ke - kb), 0);
        MP_CUDA(cudaEventRecord(eP[0], sP));
        if (on_panel_step(kb)) pending[0] = true;
        else split_ok[0] = split_l21(kb, (int)std::min<int64_t>(width_at(kb), ke - kb), 0, sP);
        int idx = 0;
        for (int64_t k = kb, knext = kb; k < ke; k = knext, ++idx) {
            if (str && idx >= str->ahead) {   // streamed: the host enqueues at most `ahead` steps ahead
                const cudaError_t e = cudaEventSynchronize(la_event(70 + (idx - str->ahead) % 8));
                if (e != cudaSuccess) MP_CUDA(e);
            }
            const int w = (int)std::min<int64_t>(width_at(k), ke - k);
            const int64_t kn = k + w;
            knext = kn;
            const int wn = kn < ke ? (int)std::min<int64_t>(width_at(kn), ke - kn) : 0;
            const int b = idx & 1;
            // early steps (large trailing matrix): the larger update partition
            const bool huge = ex.sU4 && n - kn > ex.huge_rows;
            const bool early = !huge && ex.sU2 && (double)(n - kn) > ex.big_frac * (double)n;
            const bool late = !huge && !early && ex.sU3 && (double)(n - kn) < ex.small_frac * (double)n;
            cudaStream_t sU = huge ? ex.sU4 : early ? ex.sU2 : (late ? ex.sU3 : ex.sU);
            const int smsu = huge ? ex.smsU4 : early ? ex.smsU2 : (late ? ex.smsU3 : ex.smsU);
            if (sU != cur) {                                   // keep the update work in order
                MP_CUDA(cudaEventRecord(eSw, cur));
                MP_CUDA(cudaStreamWaitEvent(sU, eSw, 0));
                cur = sU;
            }
            MP_CUDA(cudaStreamWaitEvent(sU, eP[b], 0));
            // (default; MP_LA_NEXT_ON_PANEL=0 disables) steps whose update is hidden (neither the early nor the huge phase):
            // the next panel's columns are brought up to date on the PANEL stream itself (no hop to the
            // update stream and back on the critical path); it waits for the previous step's trailing
            // update (eR), shares the L21 split with the update stream and keeps U12's split of those
            // columns in the panel stream's own scratch
            const bool on_panel = on_panel_step(k);
            if (on_panel) {
                if (pending[b]) { split_ok[b] = split_l21(k, w, b, sU); pending[b] = false; }
                if (idx > 0) MP_CUDA(cudaStreamWaitEvent(sP, eR[b ^ 1], 0));
                prof_begin(KC_LASWP, sP);
                launch_laswp_pairs<T>(W, ldw, ppairs[b], nppairs[b], 2 * w, kn, kn + wn, 0, 0, nullptr, sP);
                prof_end(KC_LASWP, 2.0 * 2 * w * (double)wn * sizeof(T), sP);
                const int kp = (int)round_up(w, 4);
                // A split: the shared one in tfU[b] when it exists; B split: always the panel stream's
                // own (second half of tf32[1]; the update stream writes its U12 split into tfU[b])
                float *bs = split_ok[b] && tf32[1] ? tf32[1] + 2 * (size_t)n * kp : nullptr;
                const bool bsplit = bs && wn >= 128 && w <= 256;
                trsm(sP, k, w, kn, kn + wn, bsplit ? bs : nullptr, bsplit ? bs + (size_t)wn * kp : nullptr, kp);
                const int terms = (double)(n - kn) < terms4_frac * (double)n ? 4 : 3;
                if (split_ok[b]) MP_CUDA(cudaStreamWaitEvent(sP, eS[b], 0));
                gemm(sP, kn, kn, k, n - kn, wn, w, true, KC_TRAIL, bs ? tfU[b] : tf32[1], sms, bs != nullptr, terms, bsplit, bs);
                psms = std::max(8, sms - smsu);
                factor_panel(sP, kn, wn, b ^ 1);
                MP_CUDA(cudaEventRecord(eP[b ^ 1], sP));
                if (on_panel_step(kn)) { pending[b ^ 1] = true; split_ok[b ^ 1] = false; }
                else split_ok[b ^ 1] = split_l21(kn, wn, b ^ 1, sP);
                if (split_ok[b]) MP_CUDA(cudaStreamWaitEvent(sU, eS[b], 0));
            } else
            if (kn < ke) {
                // the next panel's columns first (on the panel's critical path) ...
                prof_begin(KC_LASWP, sU);
                launch_laswp_pairs<T>(W, ldw, ppairs[b], nppairs[b], 2 * w, kn, kn + wn, 0, 0, nullptr, sU);
                prof_end(KC_LASWP, 2.0 * 2 * w * (double)wn * sizeof(T), sU);
                // the TRSM also writes U12's hi/lo split when the update takes the 3xTF32 path
                const int kp = (int)round_up(w, 4);
                const bool bsplit = split_ok[b] && wn >= 128 && w <= 256;   // (the TRSM writes it for w <= 256)
                float *bh = bsplit ? tfU[b] + 2 * (size_t)(n - kn) * kp : nullptr;
                trsm(sU, k, w, kn, kn + wn, bh, bsplit ? bh + (size_t)wn * kp : nullptr, kp);
                if (split_ok[b]) MP_CUDA(cudaStreamWaitEvent(sU, eS[b], 0));
                // late steps (trailing matrix < terms4_frac n, off the critical path): a fourth MMA
                const int terms = (double)(n - kn) < terms4_frac * (double)n ? 4 : 3;
                gemm(sU, kn, kn, k, n - kn, wn, w, true, KC_TRAIL, split_ok[b] ? tfU[b] : tf32[0], smsu, split_ok[b],
                     terms, bsplit);
                MP_CUDA(cudaEventRecord(eN, sU));
                MP_CUDA(cudaStreamWaitEvent(sP, eN, 0));
                psms = std::max(8, sms - smsu);
                factor_panel(sP, kn, wn, b ^ 1);
                MP_CUDA(cudaEventRecord(eP[b ^ 1], sP));
                if (on_panel_step(kn)) { pending[b ^ 1] = true; split_ok[b ^ 1] = false; }
                else split_ok[b ^ 1] = split_l21(kn, wn, b ^ 1, sP);
            }
            // ... then every other column (left factors, rest of the trailing matrix), off it
            // (streamed: the columns that have joined so far; their catch-up share of this step)
            const int64_t ncs = str ? str->nc_swap : nc;
            prof_begin(KC_LASWP, sU);
            launch_laswp_pairs<T>(W, ldw, ppairs[b], nppairs[b], 2 * w, swap_lo, ncs, k, kn + wn, perm, sU);
            prof_end(KC_LASWP, 2.0 * 2 * w * (double)(ncs - w - wn) * sizeof(T), sU);
            if (str) stream_step(k, sU, smsu);
            const int64_t ncu = str ? str->nc_upd : nc;
            if (kn < ncu && kn + wn < ncu) {
                const int kp = (int)round_up(w, 4);
                const int64_t nr = ncu - kn - wn;
                const bool bsplit = split_ok[b] && nr >= 128 && w <= 256;
                float *bh = bsplit ? tfU[b] + 2 * (size_t)(n - kn) * kp : nullptr;
                trsm(sU, k, w, kn + wn, ncu, bh, bsplit ? bh + (size_t)nr * kp : nullptr, kp);
                // same L21 as the next panel's update just before: its hi/lo split is reused
                const bool reuse = split_ok[b] || (!on_panel && kn < n && n - kn >= 256 && wn >= 128);
                const int terms = (double)(n - kn) < terms4_frac * (double)n ? 4 : 3;
                gemm(sU, kn, kn + wn, k, n - kn, nr, w, true, KC_TRAIL, split_ok[b] ? tfU[b] : tf32[0], smsu,
                     reuse, terms, bsplit);
            }
            if (str) MP_CUDA(cudaEventRecord(la_event(70 + idx % 8), sU));
            if (next_on_panel) MP_CUDA(cudaEventRecord(eR[b], sU));
        }
        MP_CUDA(cudaEventRecord(eEndP, sP));
        MP_CUDA(cudaEventRecord(eEndU, cur));
        MP_CUDA(cudaStreamWaitEvent(s, eEndP, 0));
        MP_CUDA(cudaStreamWaitEvent(s, eEndU, 0));
    }
    void run(bool lookahead) {
        if (ke < 0) ke = n;
        if (nc < 0) nc = n;
        if (lookahead && ke - kb > 2 * (int64_t)nb) {
            const ExecRes &ex = exec_res();
            if (ex.ok) { run_lookahead(ex); return; }
        }
        run_sequential();
    }
};

template <typename T>
void make_factor(Factor<T> &f, T *W, int64_t n, int64_t ldw, int nb, int32_t *ipiv, int32_t *perm, DevStatus *st,
                 Pool &pool, cudaStream_t s, int variant, bool auto_nb = false)
{
    f.W = W; f.n = n; f.ldw = ldw; f.ipiv = ipiv; f.perm = perm; f.st = st; f.nb = nb; f.s = s;
    f.sms = num_sms();
    f.variant = variant;
    // the library's own panel width (opts.nb = 0) on the tensor-core path: nb_big-wide panels while
    // more than big_rows rows remain (MP_NB_BIG, MP_NB_BIG_ROWS; 0 disables)
    if (auto_nb && sizeof(T) == 4 && tc_variant(variant)) {
        static const int env_big = [] { const char *e = std::getenv("MP_NB_BIG"); return e ? std::atoi(e) : 512; }();
        static const long long env_rows = [] { const char *e = std::getenv("MP_NB_BIG_ROWS"); return e ? std::atoll(e) : 16384LL; }();
        if (env_big > nb && env_big % nb == 0 && env_rows > 0 && n > env_rows) { f.nb_big = env_big; f.big_rows = env_rows; }
    }
    const int nbmax = std::max(nb, f.nb_big);
    if (sizeof(T) == 4 && tc_variant(variant)) {
        f.tf32[0] = pool.get<float>(tf32_scratch_floats(n, nbmax));
        f.tf32[1] = pool.get<float>(tf32_scratch_floats(n, nbmax));
        f.tfU[0] = f.tf32[0];
        f.tfU[1] = pool.get<float>(tf32_scratch_floats(n, nbmax));
    }
    f.ps.orig = pool.get<int32_t>(n);
    // left-looking leaves (MP_PANEL_LL=1, experimental: bitwise-correct but slower than the recursive
    // panel on B200)
    static const bool ll_env = [] { const char *e = std::getenv("MP_PANEL_LL"); return e && e[0] == '1'; }();
    if (sizeof(T) == 4 && ll_env && nbmax <= 256 && nb % 8 == 0) {   // (16-byte loads of the multipliers)
        f.lpos = pool.get<int32_t>(n);
        f.ll_panel = true;
    }
    f.ps.pairs = pool.get<int32_t>(4 * (size_t)nbmax);
    f.ps.npairs = pool.get<int32_t>(1);
    f.ps.ticket = pool.get<int32_t>(1);
    MP_CUDA(cudaMemsetAsync(f.ps.ticket, 0, sizeof(int32_t), s));
    if (const char *e = std::getenv("MP_NO_FUSED_TRSM")) f.fuse_trsm = e[0] != '1';
    if (const char *e = std::getenv("MP_NO_TC_INPANEL")) f.tc_inpanel = e[0] != '1';
    if (const char *e = std::getenv("MP_TF32_TERMS4_FRAC")) f.terms4_frac = std::atof(e);
    for (int b = 0; b < 2; ++b) {
        f.ppairs[b] = pool.get<int32_t>(4 * (size_t)nbmax);
        f.nppairs[b] = pool.get<int32_t>(1);
    }
    f.ps.ppairs = f.ppairs[0];
    f.ps.nppairs = f.nppairs[0];
}

template <typename T>
void run_factor(T *W, int64_t n, int64_t ldw, int nb, int32_t *ipiv, int32_t *perm, DevStatus *st, Pool &pool,
                cudaStream_t s, int variant = MP_VARIANT_FFMA, bool lookahead = true, bool auto_nb = false)
{
    Factor<T> f;
    make_factor<T>(f, W, n, ldw, nb, ipiv, perm, st, pool, s, variant, auto_nb);
    f.run(lookahead);
}

// e2e path with a host A: the 8 n^2 bytes of A cross PCIe in q column blocks on a copy
// stream while the factorisation runs.  Block j (columns [c_lo, c_hi), multiples of nb) is demoted
// when it lands (its ||A||_F^2 share saved to anrm_parts[j]), its rows put in the current row order
// (perm) and brought up to date with the panels [0, c_lo) (catch_up), then its own panels are
// factored with every update restricted to the columns that have arrived.  Same operations per
// entry as the one-shot factorisation, reordered (the exact-LU family stays bitwise).
// Column-block plan of the streamed path, in panels: with the look-ahead (one loop, blocks joining
// it), blocks of ~nbk/8 panels (at least 3), the last ones halving down to one panel, so that little
// work is left once the last bytes land; without it (blocks factored one after the other) nblocks
// equal blocks.  MP_STREAM_PLAN="w0,w1,..." (panels) overrides the look-ahead plan.
std::vector<int64_t> stream_plan(int64_t nbk, bool joined, int nblocks)
{
    std::vector<int64_t> p;
    if (!joined && !std::getenv("MP_STREAM_PLAN")) {
        const int64_t per = ceil_div(nbk, (int64_t)nblocks);
        for (int64_t r = nbk; r > 0; r -= per) p.push_back(std::min(per, r));
        return p;
    }
    if (const char *e = std::getenv("MP_STREAM_PLAN")) {
        int64_t r = nbk;
        for (const char *c = e; *c && r > 0;) {
            const int64_t v = std::max<int64_t>(1, std::atoll(c));
            p.push_back(std::min(v, r));
            r -= p.back();
            while (*c && *c != ',') ++c;
            if (*c == ',') ++c;
        }
        if (r > 0) p.push_back(r);
        if (p[0] < 2 && p.size() > 1) { p[0] += p[1]; p.erase(p.begin() + 1); }
        return p;
    }
    const int64_t B = std::max<int64_t>(3, ceil_div(nbk, (int64_t)8));
    int64_t r = nbk;
    while (r > B) { p.push_back(B); r -= B; }
    while (r > 1) { const int64_t h = ceil_div(r, (int64_t)2); p.push_back(h); r -= h; }
    if (r > 0) p.push_back(r);
    if (p[0] < 2 && p.size() > 1) { p[0] += p[1]; p.erase(p.begin() + 1); }
    return p;
}

// returns the number of column blocks (anrm_parts[0 .. blocks) hold their ||A||_F^2 shares)
int run_factor_streamed(const double *hA, int64_t lda_h, double *dA, int64_t n, float *W, int64_t ldw, int nb,
                        int32_t *ipiv, int32_t *perm, DevStatus *st, Pool &pool, cudaStream_t s, int variant,
                        bool lookahead, int nblocks, double *anrm_parts, cudaStream_t cs)
{
    Factor<float> f;
    make_factor<float>(f, W, n, ldw, nb, ipiv, perm, st, pool, s, variant);
    if (tc_variant(variant)) f.tfC = pool.get<float>(tf32_scratch_floats(n, nb));
    const int64_t nbk = ceil_div(n, (int64_t)nb);
    // MP_STREAM_JOINED=1: one look-ahead loop the blocks join (measured slower at C3: 66.6-70 vs 64.2 ms,
    // DESIGN §9b); default: the blocks factored one after another, each caught up at full width
    static const bool joined_env = [] { const char *e = std::getenv("MP_STREAM_JOINED"); return e && e[0] == '1'; }();
    const bool joined = lookahead && joined_env && nbk > 4 && exec_res().ok;
    std::vector<int64_t> plan = stream_plan(nbk, joined, nblocks);
    if (plan.size() > 40) throw std::runtime_error("streamed path: more than 40 column blocks");
    int64_t per = 0;
    for (int64_t b : plan) per = std::max(per, b * nb);
    float *S = pool.get<float>((size_t)n * round_up(per, 64));
    double *dpart = pool.get<double>((size_t)num_sms() * 8);
    unsigned *dcnt = pool.get<unsigned>(1);
    MP_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned), s));
    std::vector<cudaEvent_t> ev;
    std::vector<std::pair<int64_t, int64_t>> cols;
    {   // dA was allocated stream-ordered on s: the copy stream starts after that point of s
        cudaEvent_t e0 = la_event(19);
        MP_CUDA(cudaEventRecord(e0, s));
        MP_CUDA(cudaStreamWaitEvent(cs, e0, 0));
    }
    // copy-engine DMA (one linear transfer per block when A's columns are contiguous); MP_H2D_SM=1: SM
    // loads of the pinned block with evict-first stores (k_h2d.cu; measured slower: 75 vs 64.2 ms)
    static const bool dma_env = [] { const char *e = std::getenv("MP_H2D_SM"); return !(e && e[0] == '1'); }();
    static const int h2d_ctas = [] { const char *e = std::getenv("MP_H2D_CTAS"); return e ? std::max(1, std::atoi(e)) : 8; }();
    const double *hA_dev = dma_env ? nullptr : h2d_device_view(hA);
    for (int64_t c_lo = 0, j = 0; c_lo < n; ++j) {
        const int64_t c_hi = std::min(n, c_lo + plan[j] * nb);
        cudaEvent_t e = la_event(20 + (int)j);
        if (hA_dev && launch_h2d_cols(hA_dev + c_lo * lda_h, lda_h, dA + c_lo * n, n, c_hi - c_lo, h2d_ctas, cs)) {
        } else if (lda_h == n) {           // contiguous columns: one linear copy-engine transfer
            MP_CUDA(cudaMemcpyAsync(dA + c_lo * n, hA + c_lo * lda_h, (size_t)(c_hi - c_lo) * n * sizeof(double),
                                    cudaMemcpyHostToDevice, cs));
        } else
            MP_CUDA(cudaMemcpy2DAsync(dA + c_lo * n, n * sizeof(double), hA + c_lo * lda_h, lda_h * sizeof(double),
                                      n * sizeof(double), c_hi - c_lo, cudaMemcpyHostToDevice, cs));
        MP_CUDA(cudaEventRecord(e, cs));
        ev.push_back(e);
        cols.emplace_back(c_lo, c_hi);
        c_lo = c_hi;
    }
    // diagnostic (MP_STREAM_PRECOPY=1): every block lands before the factorisation starts (the same
    // schedule with no copy in flight: per-launch timelines are distorted by a concurrent copy)
    static const bool precopy = [] { const char *e = std::getenv("MP_STREAM_PRECOPY"); return e && e[0] == '1'; }();
    if (precopy)
        for (cudaEvent_t e : ev) MP_CUDA(cudaStreamWaitEvent(s, e, 0));
    if (joined) {
        // block 0 demoted straight into W (rows in their original order); the others join the loop
        const int64_t c_hi0 = cols[0].second;
        MP_CUDA(cudaStreamWaitEvent(s, ev[0], 0));
        prof_begin(KC_DEMOTE, s);
        launch_demote_rect<float>(dA, n, n, c_hi0, W, ldw, dpart, dcnt, st, s);
        prof_end(KC_DEMOTE, 12.0 * n * c_hi0, s);
        MP_CUDA(cudaMemcpyAsync(anrm_parts, &st->anrm2, sizeof(double), cudaMemcpyDeviceToDevice, s));
        static const int64_t dist = [] { const char *e = std::getenv("MP_STREAM_JOIN"); return e ? std::atoll(e) : 64; }();
        static const int ahead = [] { const char *e = std::getenv("MP_STREAM_AHEAD"); return e ? std::max(1, std::atoi(e)) : 3; }();
        Factor<float>::Streamer z;
        z.dA = dA; z.S = S; z.dpart = dpart; z.anrm_parts = anrm_parts; z.dcnt = dcnt;
        z.nc_swap = z.nc_upd = c_hi0;
        z.ahead = ahead;
        for (size_t j = 0; j < cols.size(); ++j) {
            Factor<float>::StreamBlock B;
            B.c_lo = cols[j].first; B.c_hi = cols[j].second; B.ev = ev[j];
            B.need_at = B.c_lo - 2 * nb;
            B.join_at = std::max<int64_t>(0, std::min(B.need_at, B.c_lo - dist * nb));
            B.joined = B.regular = j == 0;
            z.blk.push_back(B);
        }
        f.str = &z;
        f.kb = 0; f.ke = n; f.nc = n;
        f.run(true);
        f.str = nullptr;
        for (const auto &B : z.blk)
            if (!B.regular) throw std::runtime_error("streamed path: a column block was never caught up");
        return (int)cols.size();
    }
    const int sms = num_sms();
    // Overlapped blocks (default with the look-ahead): while block j is factored, block j+1 is demoted,
    // put in the row order of block j's start and caught up with the panels before block j, on a second
    // stream of the update partition.  Block j's interchanges are therefore kept off the columns left of
    // it (its L columns stay as the concurrent catch-up reads them, swap_lo) and applied afterwards to
    // those columns and to block j+1 at once; block j+1 then gets the catch-up of block j's panels
    // only.  Per entry the same operations in the same order (the interchanges commute, §9b).
    static const bool no_overlap = [] { const char *e = std::getenv("MP_STREAM_NO_OVERLAP"); return e && e[0] == '1'; }();
    const ExecRes *exr = lookahead && !no_overlap && cols.size() > 1 ? &exec_res() : nullptr;
    if (exr && exr->ok && exr->sC) {
        cudaStream_t sC = exr->sC;
        f.pairs_all = pool.get<int32_t>((size_t)nbk * 4 * nb);
        f.npairs_all = pool.get<int32_t>((size_t)nbk);
        int32_t *perm_snap = pool.get<int32_t>(n);
        std::vector<cudaEvent_t> eC(cols.size(), nullptr);
        for (size_t j = 0; j < cols.size(); ++j) {
            const int64_t c_lo = cols[j].first, c_hi = cols[j].second;
            if (j == 0) {
                MP_CUDA(cudaStreamWaitEvent(s, ev[0], 0));
                prof_begin(KC_DEMOTE, s);
                launch_demote_rect<float>(dA, n, n, c_hi, W, ldw, dpart, dcnt, st, s);
                prof_end(KC_DEMOTE, 12.0 * n * c_hi, s);
                MP_CUDA(cudaMemcpyAsync(anrm_parts, &st->anrm2, sizeof(double), cudaMemcpyDeviceToDevice, s));
            } else {
                const int64_t p_lo = cols[j - 1].first, p_hi = cols[j - 1].second;
                MP_CUDA(cudaStreamWaitEvent(s, eC[j], 0));
                // block j-1's interchanges on the columns that have not seen them: the left factors and block j
                for (int64_t k = p_lo; k < p_hi; k += nb) {
                    const int w = (int)std::min<int64_t>(nb, p_hi - k);
                    prof_begin(KC_LASWP, s);
                    launch_laswp_pairs<float>(W, ldw, f.pairs_all + (k / nb) * 4 * (int64_t)nb, f.npairs_all + k / nb,
                                              2 * w, 0, c_hi, p_lo, p_hi, nullptr, s);
                    prof_end(KC_LASWP, 2.0 * 2 * w * (double)(c_hi - (p_hi - p_lo)) * sizeof(float), s);
                }
                for (int64_t k = p_lo; k < c_lo; k += nb) f.catch_up_panel(k, c_lo, c_hi, s, sms);
            }
            if (j + 1 < cols.size()) {
                // block j+1 on the catch-up stream, in the row order of block j's start
                const int64_t q_lo = cols[j + 1].first, q_hi = cols[j + 1].second, wq = q_hi - q_lo;
                if (j == 0) launch_init_perm(perm_snap, n, s);
                else MP_CUDA(cudaMemcpyAsync(perm_snap, perm, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
                cudaEvent_t eSnap = la_event(80 + (int)(j % 2));
                MP_CUDA(cudaEventRecord(eSnap, s));
                MP_CUDA(cudaStreamWaitEvent(sC, eSnap, 0));
                MP_CUDA(cudaStreamWaitEvent(sC, ev[j + 1], 0));
                const int64_t lds = round_up(wq, 64);
                prof_begin(KC_DEMOTE, sC);
                launch_demote_rect<float>(dA + q_lo * n, n, n, wq, S, lds, dpart, dcnt, st, sC);
                MP_CUDA(cudaMemcpyAsync(anrm_parts + j + 1, &st->anrm2, sizeof(double), cudaMemcpyDeviceToDevice, sC));
                launch_gather_rows(S, lds, round_up(wq, 4), perm_snap, n, W + q_lo, ldw, sC);
                prof_end(KC_DEMOTE, 12.0 * n * wq, sC);
                for (int64_t k = 0; k < c_lo; k += nb) f.catch_up_panel(k, q_lo, q_hi, sC, exr->smsU);
                eC[j + 1] = la_event(82 + (int)j);
                MP_CUDA(cudaEventRecord(eC[j + 1], sC));
            }
            f.swap_lo = c_lo; f.kb = c_lo; f.ke = c_hi; f.nc = c_hi;
            f.run(true);
        }
        // the last block's interchanges on the left factors
        const int64_t p_lo = cols.back().first, p_hi = cols.back().second;
        for (int64_t k = p_lo; k < p_hi && p_lo > 0; k += nb) {
            const int w = (int)std::min<int64_t>(nb, p_hi - k);
            launch_laswp_pairs<float>(W, ldw, f.pairs_all + (k / nb) * 4 * (int64_t)nb, f.npairs_all + k / nb, 2 * w, 0,
                                      p_lo, 0, 0, nullptr, s);
        }
        f.swap_lo = 0;
        return (int)cols.size();
    }
    for (int64_t j = 0; j < (int64_t)cols.size(); ++j) {
        const int64_t c_lo = cols[j].first, c_hi = cols[j].second, wcols = c_hi - c_lo;
        MP_CUDA(cudaStreamWaitEvent(s, ev[j], 0));
        prof_begin(KC_DEMOTE, s);
        if (c_lo == 0) {
            launch_demote_rect<float>(dA, n, n, wcols, W, ldw, dpart, dcnt, st, s);
        } else {
            const int64_t lds = round_up(wcols, 64);
            launch_demote_rect<float>(dA + c_lo * n, n, n, wcols, S, lds, dpart, dcnt, st, s);
            launch_gather_rows(S, lds, round_up(wcols, 4), perm, n, W + c_lo, ldw, s);
        }
        prof_end(KC_DEMOTE, 12.0 * n * wcols, s);
        MP_CUDA(cudaMemcpyAsync(anrm_parts + j, &st->anrm2, sizeof(double), cudaMemcpyDeviceToDevice, s));
        if (c_lo > 0) f.catch_up(c_lo, c_hi, s, sms);
        f.kb = c_lo; f.ke = c_hi; f.nc = c_hi;
        f.run(lookahead);
    }
    return (int)cols.size();
}

struct Args {
    int64_t n, nrhs, lda;
    const double *A, *B;
    double *X;
};

// Staged device views of the caller's buffers (host pointers are copied in/out).
struct Views {
    const double *A, *B;
    double *X;
    int64_t lda;
    bool x_host;
};

Views stage_in(const Args &a, Pool &pool, cudaStream_t s, bool need_b, bool defer_a = false)
{
    Views v{a.A, a.B, a.X, a.lda, false};
    if (!is_device_ptr(a.A)) {
        double *d = pool.get<double>((size_t)a.n * a.n);
        if (!defer_a)                        // defer_a: the caller streams A in itself (run_factor_streamed)
            MP_CUDA(cudaMemcpy2DAsync(d, a.n * sizeof(double), a.A, a.lda * sizeof(double), a.n * sizeof(double),
                                      a.n, cudaMemcpyHostToDevice, s));
        v.A = d;
        v.lda = a.n;
    }
    if (need_b && !is_device_ptr(a.B)) {
        double *d = pool.get<double>((size_t)a.n * a.nrhs);
        MP_CUDA(cudaMemcpyAsync(d, a.B, (size_t)a.n * a.nrhs * sizeof(double), cudaMemcpyHostToDevice, s));
        v.B = d;
    }
    if (a.X && !is_device_ptr(a.X)) {
        v.X = pool.get<double>((size_t)a.n * std::max<int64_t>(a.nrhs, 1));
        v.x_host = true;
    }
    return v;
}

int check_args(const Args &a, int *info)
{
    const int64_t mx = std::max<int64_t>(1, a.n);
    if (a.n < 0) return *info = -1, 1;
    if (a.nrhs < 0) return *info = -2, 1;
    if (a.n > 0 && !a.A) return *info = -3, 1;
    if (a.lda < mx) return *info = -4, 1;
    if (a.n > 0 && a.nrhs > 0 && !a.B) return *info = -5, 1;
    if (a.n > 0 && a.nrhs > 0 && !a.X) return *info = -6, 1;
    if (a.n > 0 && a.nrhs > 0) {
        const size_t xb = (size_t)a.n * a.nrhs * sizeof(double);
        const size_t ab = (size_t)((a.n - 1) * a.lda + a.n) * sizeof(double);
        if (overlaps(a.X, xb, a.A, ab) || overlaps(a.X, xb, a.B, xb)) return *info = -6, 1;
    }
    return 0;
}

struct StatusIO {
    DevStatus *d;
    DevStatus *h;   // pinned, allocated once per thread (cudaFreeHost would synchronise the device)
    cudaStream_t s;
    StatusIO(Pool &pool, cudaStream_t st) : s(st) {
        static thread_local DevStatus *pinned = nullptr;
        if (!pinned) MP_CUDA(cudaMallocHost(&pinned, sizeof(DevStatus)));
        h = pinned;
        d = pool.get<DevStatus>(1);
        std::memset(h, 0, sizeof(DevStatus));
        h->zero_col = INT_MAX;
        MP_CUDA(cudaMemcpyAsync(d, h, sizeof(DevStatus), cudaMemcpyHostToDevice, s));
    }
    void reset() {
        MP_CUDA(cudaStreamSynchronize(s));
        std::memset(h, 0, sizeof(DevStatus));
        h->zero_col = INT_MAX;
        MP_CUDA(cudaMemcpyAsync(d, h, sizeof(DevStatus), cudaMemcpyHostToDevice, s));
    }
    const DevStatus &read() {
        MP_CUDA(cudaMemcpyAsync(h, d, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
        return *h;
    }
};

// binary64 GEPP + substitution on a fresh working copy (reading A-11).
// Returns info (0, or the 1-based column of the first exact zero pivot).
int fp64_solve(const Views &v, int64_t n, int64_t nrhs, int nb, Pool &pool, StatusIO &sio, cudaStream_t s)
{
    const int64_t ldw = round_up(n, 64);
    double *W = pool.get<double>((size_t)n * ldw);
    int32_t *ipiv = pool.get<int32_t>(n), *perm = pool.get<int32_t>(n), *pinv = pool.get<int32_t>(n);
    double *Y = pool.get<double>((size_t)n * nrhs);
    SolveScratch ss{pool.get<unsigned>(solve_flag_words(n)), pool.get<double>((size_t)n * std::min<int64_t>(nrhs, 16)), 0u};
    MP_CUDA(cudaMemsetAsync(ss.flags, 0, solve_flag_words(n) * sizeof(unsigned), s));
    sio.reset();                                   // fresh status: the binary32 attempt may have flagged a zero pivot
    launch_demote_transpose<double>(v.A, v.lda, n, W, ldw, nullptr, nullptr, sio.d, s);
    run_factor<double>(W, n, ldw, nb, ipiv, perm, sio.d, pool, s);
    const DevStatus &st = sio.read();
    if (st.flags & ST_A_NONFINITE) return -3;
    if (st.flags & ST_ZERO_PIVOT) return st.zero_col;
    launch_invert_perm(perm, pinv, n, s);
    launch_permute_demote_rhs<double>(v.B, n, nrhs, pinv, Y, sio.d, s);
    launch_lu_solve<double>(W, ldw, n, nrhs, Y, v.X, 0, ss, s);
    return 0;
}

void finish_copy_out(const Args &a, const Views &v, cudaStream_t s)
{
    if (v.x_host)
        MP_CUDA(cudaMemcpyAsync(a.X, v.X, (size_t)a.n * a.nrhs * sizeof(double), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
}

// GMRES-IR refinement (opts.flags bit 8; readings T-3/T-4): per right-hand side,
// restarted FGMRES(kGirM) in binary64 on A x = b from the x0 already in X, every Krylov direction
// preconditioned by the binary32 LU (z_k = LUsolve(fl32(P v_k)), the K6 + K7 kernels), the A products by
// K8, modified Gram-Schmidt / Givens / y / x += Z y by the k_gmres kernels.  B:5's test at every restart;
// a cycle ends early once |g_{k+1}| < ||x|| cte / 2.  Returns the LU applications (max over columns),
// or -31 when a column reaches `itermax` applications unconverged or its norms are not finite.
constexpr int kGirM = 20;
int gmres_ir_refine(const Views &v, int64_t n, int64_t nrhs, const float *W, int64_t ldw, const int32_t *pinv,
                    float *Y, const float *inv, SolveScratch &ss, ResidualScratch &rs, StatusIO &sio, double cte,
                    int itermax, double *hist, int &nhist, Pool &pool, cudaStream_t s, int sms)
{
    const int m = kGirM;
    const int64_t ldv = round_up(n, 32);
    double *V = pool.get<double>((size_t)ldv * (m + 1)), *Z = pool.get<double>((size_t)ldv * m);
    double *r = pool.get<double>(n), *ax = pool.get<double>(n);
    double *Rm = pool.get<double>((size_t)(m + 1) * m), *cs = pool.get<double>(32), *sn = pool.get<double>(32);
    double *g = pool.get<double>(33), *y = pool.get<double>(32), *hcol = pool.get<double>(32);
    double *hn = pool.get<double>(32), *sc = pool.get<double>(8), *ones = pool.get<double>(32);
    double *pd = pool.get<double>(gmres_partial_elems(n));
    {
        std::vector<double> h1(32, 1.0);
        MP_CUDA(cudaMemcpyAsync(ones, h1.data(), 32 * sizeof(double), cudaMemcpyHostToDevice, s));
        MP_CUDA(cudaStreamSynchronize(s));
    }
    int worst = 0;
    for (int64_t c = 0; c < nrhs; ++c) {
        double *x = v.X + c * n;
        const double *b = v.B + c * n;
        int apps = 0;
        bool done = false;
        for (;;) {
            // r = b - A x (eps_d), beta, ||x||, the check
            prof_begin(KC_RESIDUAL, s);
            launch_residual_products(v.A, v.lda, n, n, 1, x, n, ax, rs, sms, s);
            MP_CUDA(cudaMemcpyAsync(r, b, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
            launch_combine<double>(r, ax, n, 1, ones, 1.0, -1.0, n, s);
            prof_end(KC_RESIDUAL, 8.0 * n * n, s);
            launch_multidot<double>(r, n, 1, r, n, pd, sc + 0, false, s);
            launch_multidot<double>(x, n, 1, x, n, pd, sc + 1, false, s);
            double hsc[2];
            MP_CUDA(cudaMemcpyAsync(hsc, sc, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
            MP_CUDA(cudaStreamSynchronize(s));
            const double beta = std::sqrt(hsc[0]), xn = std::sqrt(hsc[1]);
            if (!std::isfinite(beta) || !std::isfinite(xn)) break;
            if (c == 0 && nhist < MP_HIST_MAX) hist[nhist++] = beta == 0.0 ? 0.0 : beta / (xn * cte);
            if (beta < xn * cte || beta == 0.0) { done = true; break; }
            if (apps >= itermax) break;
            launch_cycle_start<double>(sc + 0, g, m, sc + 2, s);
            int kk = 0;
            for (int k = 0; k < m; ++k) {
                double *vk = V + (size_t)k * ldv, *zk = Z + (size_t)k * ldv;
                launch_scale_copy<double, double>(r, k == 0 ? sc + 2 : hn + (k - 1), true, vk, nullptr, n, s);
                // z_k = LUsolve(fl32(P v_k)) (eps_s)
                prof_begin(KC_SOLVE, s);
                launch_permute_demote_rhs<float>(vk, n, 1, pinv, Y, sio.d, s);
                launch_lu_solve<float>(W, ldw, n, 1, Y, zk, 0, ss, s, inv);
                prof_end(KC_SOLVE, 4.0 * n * n, s);
                ++apps;
                prof_begin(KC_RESIDUAL, s);
                launch_residual_products(v.A, v.lda, n, n, 1, zk, n, r, rs, sms, s);
                prof_end(KC_RESIDUAL, 8.0 * n * n, s);
                for (int j = 0; j <= k; ++j) {                                   // MGS (eps_d)
                    launch_multidot<double>(V + (size_t)j * ldv, ldv, 1, r, n, pd, hcol + j, false, s);
                    launch_combine<double>(r, V + (size_t)j * ldv, ldv, 1, hcol + j, 1.0, -1.0, n, s);
                }
                launch_multidot<double>(r, n, 1, r, n, pd, sc + 3, false, s);
                launch_givens_step<double>(hcol, sc + 3, k, m, Rm, cs, sn, g, hn + k, s);
                kk = k + 1;
                double est[2];
                MP_CUDA(cudaMemcpyAsync(est, g + k + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
                MP_CUDA(cudaMemcpyAsync(est + 1, hn + k, sizeof(double), cudaMemcpyDeviceToHost, s));
                MP_CUDA(cudaStreamSynchronize(s));
                if (est[1] == 0.0 || !(std::fabs(est[0]) >= 0.5 * xn * cte) || apps >= itermax) break;
            }
            launch_backsolve<double>(Rm, m, kk, g, y, hn, s);
            launch_combine<double>(x, Z, ldv, kk, y, 1.0, 1.0, n, s);
        }
        if (!done) return -31;
        worst = std::max(worst, apps);
    }
    return worst;
}

int dsgesv_impl(const Args &a, int *iters, int *info, const mp_opts *opts, mp_report *rep)
{
    *info = 0; *iters = 0;
    if (rep) { std::memset(rep, 0, sizeof(*rep)); }
    if (check_args(a, info)) { if (rep) rep->info = *info; return MP_OK; }
    if (a.n == 0 || a.nrhs == 0) return MP_OK;

    mp_opts o;
    mp_default_opts(&o);
    if (opts) o = *opts;
    const int nb = o.nb > 0 ? o.nb : default_nb(a.n);
    const int itermax = o.itermax > 0 ? std::min(o.itermax, MP_HIST_MAX - 1) : MP_ITERMAX_DEFAULT;
    if (o.variant != MP_VARIANT_FFMA && !tc_variant(o.variant)) throw std::runtime_error("unknown variant");
    const int64_t n = a.n, nrhs = a.nrhs;
    check_size_limits(n);
    cudaStream_t s = g_stream;
    g_launches = 0;
    g_prof.reset((o.flags & 2) != 0, (o.flags & 4) != 0);
    g_prof.mask = (o.flags & 8) ? ((1u << KC_TRAIL) | (1u << KC_RESIDUAL)) : ~0u;
    Timer tm(s);
    const int t0 = tm.mark();

    Pool pool(s);
    // host A (the end-to-end path): stream it in by column blocks, overlapped with the factorisation
    // (flags bit 6 or MP_NO_STREAM_H2D=1: one copy, then the factorisation)
    static const bool no_stream = std::getenv("MP_NO_STREAM_H2D") != nullptr;
    const bool stream_a = !is_device_ptr(a.A) && n >= 4096 && nb % 4 == 0 && !(o.flags & 64) && !no_stream &&
                          !(o.flags & 1);
    Views v = stage_in(a, pool, s, true, stream_a);
    const int t_staged = tm.mark();
    StatusIO sio(pool, s);
    const int sms = num_sms();
    const int64_t ldw = round_up(n, 64);
    float *W = pool.get<float>((size_t)n * ldw);                   // the +50 % of P:145-146
    int32_t *ipiv = pool.get<int32_t>(n), *perm = pool.get<int32_t>(n), *pinv = pool.get<int32_t>(n);
    float *Y = pool.get<float>((size_t)n * nrhs);
    double *R = pool.get<double>((size_t)n * nrhs);
    ResidualScratch rs;
    rs.partial = pool.get<double>(residual_partial_elems(n, nrhs, sms));
    rs.blocksums = pool.get<double>((size_t)ceil_div(n, 256) * 2 * nrhs);
    rs.counter = pool.get<unsigned>(1);
    SolveScratch ss{pool.get<unsigned>(solve_flag_words(n)), pool.get<float>((size_t)n * std::min<int64_t>(nrhs, 16)), 0u};
    MP_CUDA(cudaMemsetAsync(ss.flags, 0, solve_flag_words(n) * sizeof(unsigned), s));
    ss.tags = pool.get<uint64_t>(solve_tag_words(n, nrhs));
    ss.tag_cols = (int)std::min<int64_t>(nrhs, 16);
    MP_CUDA(cudaMemsetAsync(ss.tags, 0, solve_tag_words(n, nrhs) * sizeof(uint64_t), s));
    double *dpart = pool.get<double>((size_t)sms * 8);
    unsigned *dcnt = pool.get<unsigned>(1);
    MP_CUDA(cudaMemsetAsync(rs.counter, 0, sizeof(unsigned), s));
    MP_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned), s));

    // ---- K1: demote + ||A||_F; B finiteness (identity scatter into Y, discarded)
    double anrm2_streamed = -1.0;
    if (stream_a) {
        // demote + step 1 as the column blocks of A land (the status is checked right after)
        int32_t *ident = pool.get<int32_t>(n);
        launch_init_perm(ident, n, s);
        launch_permute_demote_rhs<float>(v.B, n, nrhs, ident, Y, sio.d, s);
        static const int kBlocks = [] { const char *e = std::getenv("MP_STREAM_BLOCKS"); return e ? std::max(1, std::min(16, std::atoi(e))) : 7; }();
        double *parts = pool.get<double>(40);
        const int nparts = run_factor_streamed(a.A, a.lda, const_cast<double *>(v.A), n, W, ldw, nb, ipiv, perm,
                                               sio.d, pool, s, o.variant, (o.flags & 16) == 0, kBlocks, parts,
                                               copy_stream());
        double hp[40] = {0};
        MP_CUDA(cudaMemcpyAsync(hp, parts, sizeof(hp), cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
        anrm2_streamed = 0.0;
        for (int j = 0; j < nparts; ++j) anrm2_streamed += hp[j];
    } else {
        prof_begin(KC_DEMOTE, s);
        launch_demote_transpose<float>(v.A, v.lda, n, W, ldw, dpart, dcnt, sio.d, s);
        prof_end(KC_DEMOTE, 12.0 * n * n, s);
        launch_init_perm(perm, n, s);
        launch_permute_demote_rhs<float>(v.B, n, nrhs, perm, Y, sio.d, s);
    }
    const int t_dem = tm.mark();
    DevStatus st0 = sio.read();
    if (st0.flags & ST_A_NONFINITE) { *info = -3; if (rep) rep->info = -3; return MP_OK; }
    if (st0.flags & ST_B_NONFINITE) { *info = -5; if (rep) rep->info = -5; return MP_OK; }
    const double anrm = std::sqrt(stream_a ? anrm2_streamed : st0.anrm2);
    const double cte = anrm * std::ldexp(1.0, -53) * std::sqrt((double)n);   // A-1, A-2
    int code = 0;
    int t_fac = t_dem, t_ref = t_dem;
    int nhist = 0;
    double hist[MP_HIST_MAX] = {0};
    bool used_inv = false;

    if (st0.flags & ST_OVERFLOW) code = -2;
    if (!code && stream_a) {
        if (st0.flags & ST_ZERO_PIVOT) code = -3;                   // (step 1 already ran)
    } else if (!code) {
        // ---- step 1: binary32 blocked GEPP
        run_factor<float>(W, n, ldw, nb, ipiv, perm, sio.d, pool, s, o.variant, (o.flags & 16) == 0, o.nb <= 0);
        t_fac = tm.mark();
        const DevStatus &st1 = sio.read();
        if (st1.flags & ST_ZERO_PIVOT) code = -3;
    }
    if (!code && (o.flags & 1)) code = -31;
    if (!code) {
        // ---- steps 2-3: x0 = LUsolve(fl32(P b))
        launch_invert_perm(perm, pinv, n, s);
        launch_permute_demote_rhs<float>(v.B, n, nrhs, pinv, Y, sio.d, s);
        // inverted diagonal blocks for the solves (reading A-19; flags bit 5: substitution)
        float *inv = nullptr;
        if (!(o.flags & 32)) {
            inv = pool.get<float>(solve_inv_floats(n));
            prof_begin(KC_SOLVE, s);
            launch_solve_inverses(W, ldw, n, inv, s);
            prof_end(KC_SOLVE, 0.0, s);
            if (!(solve_inverses_cond(inv, n, s) <= kInvCondMax)) inv = nullptr;   // ill-conditioned block
        }
        used_inv = inv != nullptr;
        prof_begin(KC_SOLVE, s);
        launch_lu_solve<float>(W, ldw, n, nrhs, Y, v.X, 0, ss, s, inv);
        prof_end(KC_SOLVE, 4.0 * n * n, s);
        code = -31;
        if (o.flags & 256) {                                      // GMRES-IR (NEXT-2)
            const int apps = gmres_ir_refine(v, n, nrhs, W, ldw, pinv, Y, inv, ss, rs, sio, cte, itermax, hist, nhist,
                                             pool, s, sms);
            if (apps >= 0) { *iters = apps; code = 0; }
        }
        for (int it = 0; it <= itermax && !(o.flags & 256); ++it) {
            // ---- step 4 + check: r = b - A x (binary64), norms, verdict; y = fl32(P r)
            prof_begin(KC_RESIDUAL, s);
            launch_residual<float>(v.A, v.lda, n, nrhs, v.B, v.X, R, pinv, Y, cte, rs, sio.d, sms, s);
            prof_end(KC_RESIDUAL, 8.0 * n * n + 8.0 * 4 * n * nrhs, s);
            const DevStatus &st = sio.read();
            if (st.flags & ST_NORM_NONFINITE) break;
            hist[nhist++] = st.ratio;
            if (st.converged) { *iters = it; code = 0; break; }
            if (it == itermax) break;
            // ---- steps 5-7: z = LUsolve(y) (binary32), x += z (binary64)
            prof_begin(KC_SOLVE, s);
            launch_lu_solve<float>(W, ldw, n, nrhs, Y, v.X, 1, ss, s, inv);
            prof_end(KC_SOLVE, 4.0 * n * n, s);
        }
        t_ref = tm.mark();
    }
    int t_fb = tm.mark();
    if (code) {
        *iters = code;
        *info = fp64_solve(v, n, nrhs, nb, pool, sio, s);
        t_fb = tm.mark();
    }
    finish_copy_out(a, v, s);
    const int t_end = tm.mark();
    MP_CUDA(cudaStreamSynchronize(s));
    if (rep) {
        rep->iters = *iters; rep->info = *info; rep->nhist = nhist; rep->nb = nb; rep->variant = o.variant;
        rep->solve_inv = used_inv ? 1 : 0;
        rep->anrm = anrm;
        for (int i = 0; i < nhist; ++i) rep->hist[i] = hist[i];
        rep->t_total_ms = tm.ms(t0, t_end);
        rep->t_copy_ms = tm.ms(t0, t_staged);
        rep->t_demote_ms = tm.ms(t_staged, t_dem);
        rep->t_factor_ms = (t_fac != t_dem) ? tm.ms(t_dem, t_fac) : 0.0;
        rep->t_refine_ms = (t_ref != t_dem) ? tm.ms(t_fac, t_ref) : 0.0;
        rep->t_fallback_ms = code ? tm.ms(t_ref, t_fb) : 0.0;
        rep->workspace_bytes = pool.bytes;
        rep->kernel_launches = g_launches;
        if (!g_prof.deferred) prof_collect(rep);
    }
    if (!g_prof.deferred) g_prof.reset(false, false);
    else g_prof.on = false;
    return MP_OK;
}

int dgesv_impl(const Args &a, int *info, const mp_opts *opts, mp_report *rep)
{
    *info = 0;
    if (rep) std::memset(rep, 0, sizeof(*rep));
    if (check_args(a, info)) { if (rep) rep->info = *info; return MP_OK; }
    if (a.n == 0 || a.nrhs == 0) return MP_OK;
    mp_opts o;
    mp_default_opts(&o);
    if (opts) o = *opts;
    const int nb = o.nb > 0 ? o.nb : default_nb(a.n);
    check_size_limits(a.n);
    cudaStream_t s = g_stream;
    g_launches = 0;
    g_prof.reset((o.flags & 2) != 0, (o.flags & 4) != 0);
    g_prof.mask = (o.flags & 8) ? ((1u << KC_TRAIL) | (1u << KC_RESIDUAL)) : ~0u;
    Timer tm(s);
    const int t0 = tm.mark();
    Pool pool(s);
    Views v = stage_in(a, pool, s, true);
    const int t1 = tm.mark();
    StatusIO sio(pool, s);
    {   // B finiteness (identity scatter into a scratch vector)
        int32_t *idp = pool.get<int32_t>(a.n);
        double *Yd = pool.get<double>((size_t)a.n * a.nrhs);
        launch_init_perm(idp, a.n, s);
        launch_permute_demote_rhs<double>(v.B, a.n, a.nrhs, idp, Yd, sio.d, s);
    }
    *info = fp64_solve(v, a.n, a.nrhs, nb, pool, sio, s);
    const DevStatus &st = sio.read();
    if (*info != -3 && (st.flags & ST_B_NONFINITE)) *info = -5;
    finish_copy_out(a, v, s);
    const int t2 = tm.mark();
    MP_CUDA(cudaStreamSynchronize(s));
    if (rep) {
        rep->info = *info; rep->nb = nb;
        rep->t_total_ms = tm.ms(t0, t2);
        rep->t_copy_ms = tm.ms(t0, t1);
        rep->t_factor_ms = tm.ms(t1, t2);
        rep->workspace_bytes = pool.bytes;
        rep->kernel_launches = g_launches;
        if (!g_prof.deferred) prof_collect(rep);
    }
    if (!g_prof.deferred) g_prof.reset(false, false);
    else g_prof.on = false;
    return MP_OK;
}

template <typename T>
int getrf_impl(int64_t n, const double *A, int64_t lda, T *LU, int32_t *ipiv_out, int *info, const mp_opts *opts)
{
    *info = 0;
    if (n < 0) return *info = -1, MP_OK;
    if (n > 0 && !A) return *info = -3, MP_OK;
    if (lda < std::max<int64_t>(1, n)) return *info = -4, MP_OK;
    if (n > 0 && !LU) return *info = -5, MP_OK;
    if (n > 0 && !ipiv_out) return *info = -6, MP_OK;
    if (n == 0) return MP_OK;
    mp_opts o;
    mp_default_opts(&o);
    if (opts) o = *opts;
    const int nb = o.nb > 0 ? o.nb : default_nb(n);
    check_size_limits(n);
    cudaStream_t s = g_stream;
    g_launches = 0;
    Pool pool(s);
    Args a{n, 0, lda, A, nullptr, nullptr};
    Views v = stage_in(a, pool, s, false);
    StatusIO sio(pool, s);
    const int64_t ldw = round_up(n, 64);
    T *W = pool.get<T>((size_t)n * ldw);
    int32_t *ipiv = pool.get<int32_t>(n), *perm = pool.get<int32_t>(n);
    const int sms = num_sms();
    double *dpart = pool.get<double>((size_t)sms * 8);
    unsigned *dcnt = pool.get<unsigned>(1);
    MP_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned), s));
    launch_demote_transpose<T>(v.A, v.lda, n, W, ldw, dpart, dcnt, sio.d, s);
    const DevStatus st0 = sio.read();
    if (st0.flags & ST_A_NONFINITE) return *info = -3, MP_OK;
    if (st0.flags & ST_OVERFLOW) return *info = -2, MP_OK;
    run_factor<T>(W, n, ldw, nb, ipiv, perm, sio.d, pool, s, sizeof(T) == 4 ? o.variant : MP_VARIANT_FFMA);
    const DevStatus &st = sio.read();
    if (st.flags & ST_ZERO_PIVOT) *info = st.zero_col;
    // packed factors back to column-major (leading dimension n)
    const bool lu_dev = is_device_ptr(LU), ip_dev = is_device_ptr(ipiv_out);
    T *dLU = lu_dev ? LU : pool.get<T>((size_t)n * n);
    launch_transpose_out<T>(W, ldw, n, dLU, s);
    if (!lu_dev) MP_CUDA(cudaMemcpyAsync(LU, dLU, (size_t)n * n * sizeof(T), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaMemcpyAsync(ipiv_out, ipiv, (size_t)n * sizeof(int32_t),
                            ip_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    return MP_OK;
}

// ------------------------------------------------------------------ SPD variant
// Algorithm 1 with SPOTRF / SPOTRS / DSYMM.  Step 1 is a blocked right-looking
// Cholesky of the binary32 working copy: per panel the diagonal block (C2), the panel below it
// (C3, which also writes L21^T into the upper block), and the trailing update A22 -= L21 L21^T on
// the tiles that touch the lower triangle (3xTF32 tcgen05 / DMMA; the FFMA variant updates the
// whole square: the upper part is overwritten by later panels).  The factors are then put in the
// unit-lower / upper form of the LU path (C4, reading C-4), so the triangular-solve kernels,
// the refinement loop and the fallback logic are the nonsymmetric path's, with P = I.
int chol_nb(size_t elem, int64_t n, int requested)
{
    const int mx = elem == 4 ? chol_block_max<float>() : chol_block_max<double>();
    const int nb = requested > 0 ? requested : (n <= 1024 ? 64 : (n <= 4096 ? 128 : 256));
    return std::max(1, std::min(nb, mx));
}

// Schur update of the SPD factorisation, C = W[r0.., c0..] (M x N) -= L21 L21^T restricted to the
// rows / columns given, with L21 = W[r0.., k..k+w) and L21^T read from the upper block W[k.., c0..)
// (written there by the TRSM).  lower: C square on the diagonal, only the tiles touching its
// lower triangle (the SYRK); else a plain block (the look-ahead's next block column).
template <typename T>
void chol_update(T *W, int64_t ldw, int64_t k, int w, int64_t r0, int64_t c0, int64_t M, int64_t N, bool lower,
                 float *scratch, int nsm, cudaStream_t q, int variant)
{
    if (M <= 0 || N <= 0) return;
    prof_begin(KC_TRAIL, q);
    T *A21 = W + r0 * ldw + k, *C = W + r0 * ldw + c0;
    if constexpr (sizeof(T) == 4) {
        const int terms = variant == MP_VARIANT_TF32 ? 1 : 3;
        if (scratch && lower && M >= 256)
            launch_syrk_lower_3xtf32(A21, ldw, C, ldw, M, w, scratch, nsm, q, terms);
        else if (scratch && !lower && M >= 256 && N >= 128)
            launch_gemm_update_3xtf32(W, ldw, r0, c0, k, M, N, w, scratch, nsm, q, false, terms);
        else
            launch_gemm_update<T>(W, ldw, r0, c0, k, M, N, w, q);
    } else {
        if (!launch_dgemm_dmma(A21, ldw, W + k * ldw + c0, ldw, C, ldw, M, N, w, q, lower))
            launch_gemm_update<T>(W, ldw, r0, c0, k, M, N, w, q);
    }
    prof_end(KC_TRAIL, lower ? (double)M * (M + 1) * w : 2.0 * M * N * w, q);   // SYRK: lower triangle incl. diagonal
}

template <typename T>
void chol_panel(T *W, int64_t ldw, int64_t n, int64_t k, int w, DevStatus *st, cudaStream_t q)
{
    prof_begin(KC_PANEL, q);
    launch_potrf_diag<T>(W, ldw, k, w, st, q);
    prof_end(KC_PANEL, (double)w * w * w / 3.0, q);
    const int64_t m = n - k - w;
    if (m <= 0) return;
    prof_begin(KC_TRSM, q);
    launch_trsm_chol<T>(W, ldw, k, w, n, q);
    prof_end(KC_TRSM, (double)w * w * m, q);
}

// Right-looking blocked Cholesky (SPOTRF's structure).  With look-ahead (depth 1, the LU
// path's streams, §7): step k's SYRK is split into the next block column [kn, kn + wn) (a plain
// block update, first, on the update partition) and the rest (lower tiles of [kn + wn, n)^2); the
// diagonal block and TRSM of panel kn run on the panel stream as soon as their block column is
// up to date, beside the rest of step k's SYRK.  Concurrent work touches disjoint blocks: the
// panel stream writes block column kn (lower) and block row kn (L21^T, upper), the SYRK only rows
// and columns >= kn + wn.  Every entry receives the same operations in the same order.
template <typename T>
void run_chol(T *W, int64_t n, int64_t ldw, int nb, DevStatus *st, Pool &pool, cudaStream_t s, int variant,
              bool lookahead = true)
{
    float *scratch = nullptr;
    if (sizeof(T) == 4 && tc_variant(variant) && n > nb)
        scratch = pool.get<float>(tf32_scratch_floats(n, nb));
    const int sms = num_sms();
    const ExecRes *ex = nullptr;
    if (lookahead && n > 2 * (int64_t)nb) {
        const ExecRes &e = exec_res();
        if (e.ok) ex = &e;
    }
    if (!ex) {
        for (int64_t k = 0; k < n; k += nb) {
            const int w = (int)std::min<int64_t>(nb, n - k);
            chol_panel<T>(W, ldw, n, k, w, st, s);
            const int64_t m = n - k - w;
            if (m <= 0) break;
            chol_update<T>(W, ldw, k, w, k + w, k + w, m, m, true, scratch, sms, s, variant);
        }
        return;
    }
    cudaStream_t sP = ex->sP, sU = ex->sU;
    const int nsm = ex->smsU;
    cudaEvent_t e0 = la_event(0), eP = la_event(1), eN = la_event(3), eEndP = la_event(4), eEndU = la_event(5);
    MP_CUDA(cudaEventRecord(e0, s));
    MP_CUDA(cudaStreamWaitEvent(sP, e0, 0));
    MP_CUDA(cudaStreamWaitEvent(sU, e0, 0));
    chol_panel<T>(W, ldw, n, 0, (int)std::min<int64_t>(nb, n), st, sP);
    MP_CUDA(cudaEventRecord(eP, sP));
    for (int64_t k = 0; k < n; k += nb) {
        const int w = (int)std::min<int64_t>(nb, n - k);
        const int64_t kn = k + w;
        if (kn >= n) break;
        const int wn = (int)std::min<int64_t>(nb, n - kn);
        const int64_t m = n - kn;
        MP_CUDA(cudaStreamWaitEvent(sU, eP, 0));
        chol_update<T>(W, ldw, k, w, kn, kn, m, wn, false, scratch, nsm, sU, variant);     // next block column
        MP_CUDA(cudaEventRecord(eN, sU));
        MP_CUDA(cudaStreamWaitEvent(sP, eN, 0));
        chol_panel<T>(W, ldw, n, kn, wn, st, sP);                                         // panel kn
        MP_CUDA(cudaEventRecord(eP, sP));
        chol_update<T>(W, ldw, k, w, kn + wn, kn + wn, m - wn, m - wn, true, scratch, nsm, sU, variant);  // the rest
    }
    MP_CUDA(cudaEventRecord(eEndP, sP));
    MP_CUDA(cudaEventRecord(eEndU, sU));
    MP_CUDA(cudaStreamWaitEvent(s, eEndP, 0));
    MP_CUDA(cudaStreamWaitEvent(s, eEndU, 0));
}

// binary64 SPD solve on a fresh working copy (the fallback, and mp_dposv).  Returns info:
// 0, or k + 1 when the binary64 Cholesky breaks down at column k (reading C-2).
int fp64_chol_solve(const Views &v, int64_t n, int64_t nrhs, int nb, Pool &pool, StatusIO &sio, cudaStream_t s)
{
    const int64_t ldw = round_up(n, 64);
    double *W = pool.get<double>((size_t)n * ldw);
    int32_t *ident = pool.get<int32_t>(n);
    double *Y = pool.get<double>((size_t)n * nrhs), *d = pool.get<double>(n);
    SolveScratch ss{pool.get<unsigned>(solve_flag_words(n)), pool.get<double>((size_t)n * std::min<int64_t>(nrhs, 16)), 0u};
    MP_CUDA(cudaMemsetAsync(ss.flags, 0, solve_flag_words(n) * sizeof(unsigned), s));
    const int sms = num_sms();
    double *dpart = pool.get<double>(demote_sym_partials(sms));
    unsigned *dcnt = pool.get<unsigned>(1);
    MP_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned), s));
    sio.reset();
    launch_demote_sym<double>(v.A, v.lda, n, W, ldw, dpart, dcnt, sio.d, sms, s);
    run_chol<double>(W, n, ldw, chol_nb(8, n, nb), sio.d, pool, s, MP_VARIANT_FFMA);
    const DevStatus &st = sio.read();
    if (st.flags & ST_A_NONFINITE) return -3;
    if (st.flags & ST_ZERO_PIVOT) return st.zero_col;
    launch_chol_to_lu<double>(W, ldw, n, d, s);
    launch_init_perm(ident, n, s);
    launch_permute_demote_rhs<double>(v.B, n, nrhs, ident, Y, sio.d, s);
    launch_lu_solve<double>(W, ldw, n, nrhs, Y, v.X, 0, ss, s);
    return 0;
}

int dsposv_impl(const Args &a, int *iters, int *info, const mp_opts *opts, mp_report *rep)
{
    *info = 0; *iters = 0;
    if (rep) std::memset(rep, 0, sizeof(*rep));
    if (check_args(a, info)) { if (rep) rep->info = *info; return MP_OK; }
    if (a.n == 0 || a.nrhs == 0) return MP_OK;
    mp_opts o;
    mp_default_opts(&o);
    if (opts) o = *opts;
    const int64_t n = a.n, nrhs = a.nrhs;
    const int nb = chol_nb(4, n, o.nb);
    const int itermax = o.itermax > 0 ? std::min(o.itermax, MP_HIST_MAX - 1) : MP_ITERMAX_DEFAULT;
    if (o.variant != MP_VARIANT_FFMA && !tc_variant(o.variant)) throw std::runtime_error("unknown variant");
    check_size_limits(n);
    cudaStream_t s = g_stream;
    g_launches = 0;
    g_prof.reset((o.flags & 2) != 0, (o.flags & 4) != 0);
    g_prof.mask = (o.flags & 8) ? ((1u << KC_TRAIL) | (1u << KC_RESIDUAL)) : ~0u;
    Timer tm(s);
    const int t0 = tm.mark();
    Pool pool(s);
    Views v = stage_in(a, pool, s, true);
    const int t_staged = tm.mark();
    StatusIO sio(pool, s);
    const int sms = num_sms();
    const int64_t ldw = round_up(n, 64);
    float *W = pool.get<float>((size_t)n * ldw);
    int32_t *ident = pool.get<int32_t>(n);
    float *Y = pool.get<float>((size_t)n * nrhs), *dsc = pool.get<float>(n);
    double *R = pool.get<double>((size_t)n * nrhs), *AX = pool.get<double>((size_t)n * nrhs);
    double *spart = pool.get<double>(symv_partial_elems(n));
    ResidualScratch rs;
    rs.partial = nullptr;
    rs.blocksums = pool.get<double>((size_t)ceil_div(n, 256) * 2 * nrhs);
    rs.counter = pool.get<unsigned>(1);
    SolveScratch ss{pool.get<unsigned>(solve_flag_words(n)), pool.get<float>((size_t)n * std::min<int64_t>(nrhs, 16)), 0u};
    MP_CUDA(cudaMemsetAsync(ss.flags, 0, solve_flag_words(n) * sizeof(unsigned), s));
    ss.tags = pool.get<uint64_t>(solve_tag_words(n, nrhs));
    ss.tag_cols = (int)std::min<int64_t>(nrhs, 16);
    MP_CUDA(cudaMemsetAsync(ss.tags, 0, solve_tag_words(n, nrhs) * sizeof(uint64_t), s));
    double *dpart = pool.get<double>(demote_sym_partials(sms));
    unsigned *dcnt = pool.get<unsigned>(1);
    MP_CUDA(cudaMemsetAsync(rs.counter, 0, sizeof(unsigned), s));
    MP_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned), s));

    // ---- C1: lower triangle -> symmetric binary32 working copy + ||A||_F; B finiteness
    prof_begin(KC_DEMOTE, s);
    launch_demote_sym<float>(v.A, v.lda, n, W, ldw, dpart, dcnt, sio.d, sms, s);
    prof_end(KC_DEMOTE, 8.0 * n * n, s);
    launch_init_perm(ident, n, s);
    launch_permute_demote_rhs<float>(v.B, n, nrhs, ident, Y, sio.d, s);
    const int t_dem = tm.mark();
    DevStatus st0 = sio.read();
    if (st0.flags & ST_A_NONFINITE) { *info = -3; if (rep) rep->info = -3; return MP_OK; }
    if (st0.flags & ST_B_NONFINITE) { *info = -5; if (rep) rep->info = -5; return MP_OK; }
    const double anrm = std::sqrt(st0.anrm2);
    const double cte = anrm * std::ldexp(1.0, -53) * std::sqrt((double)n);
    int code = (st0.flags & ST_OVERFLOW) ? -2 : 0;
    int t_fac = t_dem, t_ref = t_dem, nhist = 0;
    double hist[MP_HIST_MAX] = {0};
    bool used_inv = false;
    if (!code) {
        run_chol<float>(W, n, ldw, nb, sio.d, pool, s, o.variant, !(o.flags & 16));   // step 1 (SPOTRF)
        t_fac = tm.mark();
        const DevStatus &st1 = sio.read();
        if (st1.flags & ST_ZERO_PIVOT) code = -3;                              // reading C-1
    }
    if (!code && (o.flags & 1)) code = -31;
    if (!code) {
        launch_chol_to_lu<float>(W, ldw, n, dsc, s);                            // reading C-4
        float *inv = nullptr;
        if (!(o.flags & 32)) {
            inv = pool.get<float>(solve_inv_floats(n));
            launch_solve_inverses(W, ldw, n, inv, s);
            if (!(solve_inverses_cond(inv, n, s) <= kInvCondMax)) inv = nullptr;
        }
        used_inv = inv != nullptr;
        prof_begin(KC_SOLVE, s);
        launch_lu_solve<float>(W, ldw, n, nrhs, Y, v.X, 0, ss, s, inv);        // steps 2-3 (SPOTRS)
        prof_end(KC_SOLVE, 4.0 * n * n, s);
        code = -31;
        for (int it = 0; it <= itermax; ++it) {
            prof_begin(KC_RESIDUAL, s);                                         // step 4 (DSYMM)
            launch_symv_products(v.A, v.lda, n, nrhs, v.X, AX, spart, s);
            launch_residual_finalize<float>(AX, n, nrhs, v.B, v.X, R, ident, Y, cte, rs, sio.d, s);
            prof_end(KC_RESIDUAL, 4.0 * n * n * nrhs + 8.0 * 4 * n * nrhs, s);
            const DevStatus &st = sio.read();
            if (st.flags & ST_NORM_NONFINITE) break;
            hist[nhist++] = st.ratio;
            if (st.converged) { *iters = it; code = 0; break; }
            if (it == itermax) break;
            prof_begin(KC_SOLVE, s);
            launch_lu_solve<float>(W, ldw, n, nrhs, Y, v.X, 1, ss, s, inv);    // steps 5-7
            prof_end(KC_SOLVE, 4.0 * n * n, s);
        }
        t_ref = tm.mark();
    }
    int t_fb = tm.mark();
    if (code) {
        *iters = code;
        *info = fp64_chol_solve(v, n, nrhs, o.nb, pool, sio, s);
        t_fb = tm.mark();
    }
    finish_copy_out(a, v, s);
    const int t_end = tm.mark();
    MP_CUDA(cudaStreamSynchronize(s));
    if (rep) {
        rep->iters = *iters; rep->info = *info; rep->nhist = nhist; rep->nb = nb; rep->variant = o.variant;
        rep->solve_inv = used_inv ? 1 : 0;
        rep->anrm = anrm;
        for (int i = 0; i < nhist; ++i) rep->hist[i] = hist[i];
        rep->t_total_ms = tm.ms(t0, t_end);
        rep->t_copy_ms = tm.ms(t0, t_staged);
        rep->t_demote_ms = tm.ms(t_staged, t_dem);
        rep->t_factor_ms = (t_fac != t_dem) ? tm.ms(t_dem, t_fac) : 0.0;
        rep->t_refine_ms = (t_ref != t_dem) ? tm.ms(t_fac, t_ref) : 0.0;
        rep->t_fallback_ms = code ? tm.ms(t_ref, t_fb) : 0.0;
        rep->workspace_bytes = pool.bytes;
        rep->kernel_launches = g_launches;
        if (!g_prof.deferred) prof_collect(rep);
    }
    if (!g_prof.deferred) g_prof.reset(false, false);
    else g_prof.on = false;
    return MP_OK;
}

int dposv_impl(const Args &a, int *info, const mp_opts *opts, mp_report *rep)
{
    *info = 0;
    if (rep) std::memset(rep, 0, sizeof(*rep));
    if (check_args(a, info)) { if (rep) rep->info = *info; return MP_OK; }
    if (a.n == 0 || a.nrhs == 0) return MP_OK;
    mp_opts o;
    mp_default_opts(&o);
    if (opts) o = *opts;
    check_size_limits(a.n);
    cudaStream_t s = g_stream;
    g_launches = 0;
    g_prof.reset((o.flags & 2) != 0, (o.flags & 4) != 0);
    g_prof.mask = (o.flags & 8) ? ((1u << KC_TRAIL) | (1u << KC_RESIDUAL)) : ~0u;
    Timer tm(s);
    const int t0 = tm.mark();
    Pool pool(s);
    Views v = stage_in(a, pool, s, true);
    const int t1 = tm.mark();
    StatusIO sio(pool, s);
    *info = fp64_chol_solve(v, a.n, a.nrhs, o.nb, pool, sio, s);
    const DevStatus &st = sio.read();
    if (*info != -3 && (st.flags & ST_B_NONFINITE)) *info = -5;
    finish_copy_out(a, v, s);
    const int t2 = tm.mark();
    MP_CUDA(cudaStreamSynchronize(s));
    if (rep) {
        rep->info = *info; rep->nb = chol_nb(8, a.n, o.nb);
        rep->t_total_ms = tm.ms(t0, t2);
        rep->t_copy_ms = tm.ms(t0, t1);
        rep->t_factor_ms = tm.ms(t1, t2);
        rep->workspace_bytes = pool.bytes;
        rep->kernel_launches = g_launches;
        if (!g_prof.deferred) prof_collect(rep);
    }
    if (!g_prof.deferred) g_prof.reset(false, false);
    else g_prof.on = false;
    return MP_OK;
}

// Cholesky factor alone (SPOTRF / DPOTRF of the lower triangle): L in the lower triangle of the
// column-major output (leading dimension n); its strict upper triangle holds L^T.
template <typename T>
int potrf_impl(int64_t n, const double *A, int64_t lda, T *L, int *info, const mp_opts *opts)
{
    *info = 0;
    if (n < 0) return *info = -1, MP_OK;
    if (n > 0 && !A) return *info = -3, MP_OK;
    if (lda < std::max<int64_t>(1, n)) return *info = -4, MP_OK;
    if (n > 0 && !L) return *info = -5, MP_OK;
    if (n == 0) return MP_OK;
    mp_opts o;
    mp_default_opts(&o);
    if (opts) o = *opts;
    check_size_limits(n);
    cudaStream_t s = g_stream;
    g_launches = 0;
    Pool pool(s);
    Args a{n, 0, lda, A, nullptr, nullptr};
    Views v = stage_in(a, pool, s, false);
    StatusIO sio(pool, s);
    const int64_t ldw = round_up(n, 64);
    T *W = pool.get<T>((size_t)n * ldw);
    const int sms = num_sms();
    double *dpart = pool.get<double>(demote_sym_partials(sms));
    unsigned *dcnt = pool.get<unsigned>(1);
    MP_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned), s));
    launch_demote_sym<T>(v.A, v.lda, n, W, ldw, dpart, dcnt, sio.d, sms, s);
    const DevStatus st0 = sio.read();
    if (st0.flags & ST_A_NONFINITE) return *info = -3, MP_OK;
    if (st0.flags & ST_OVERFLOW) return *info = -2, MP_OK;
    run_chol<T>(W, n, ldw, chol_nb(sizeof(T), n, o.nb), sio.d, pool, s,
                sizeof(T) == 4 ? o.variant : MP_VARIANT_FFMA);
    const DevStatus &st = sio.read();
    if (st.flags & ST_ZERO_PIVOT) *info = st.zero_col;
    const bool l_dev = is_device_ptr(L);
    T *dL = l_dev ? L : pool.get<T>((size_t)n * n);
    launch_transpose_out<T>(W, ldw, n, dL, s);
    if (!l_dev) MP_CUDA(cudaMemcpyAsync(L, dL, (size_t)n * n * sizeof(T), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    return MP_OK;
}

// ------------------------------------------------------------------ NEXT-4: extended-precision refinement
// PAPER.md P:638-697 ("Extension to Quadruple Precision", QDGESV): the binary64 LU (DGETRF) and
// solves (DGETRS) of mp_dgesv, the residual r = b - A x and the update x += z in double-double
// (reading Q-0), B:5's stop test with the double-double unit roundoff 2^-104 (Q-1), at most 30
// corrections and no fallback (Q-2).  X = Xhi + Xlo.
int qdgesv_impl(const Args &a, double *Xlo, int *iters, int *info, const mp_opts *opts, mp_report *rep)
{
    *info = 0; *iters = 0;
    if (rep) std::memset(rep, 0, sizeof(*rep));
    if (check_args(a, info)) { if (rep) rep->info = *info; return MP_OK; }
    if (a.n > 0 && a.nrhs > 0) {
        const size_t xb = (size_t)a.n * a.nrhs * sizeof(double);
        const size_t ab = (size_t)((a.n - 1) * a.lda + a.n) * sizeof(double);
        if (!Xlo || overlaps(Xlo, xb, a.A, ab) || overlaps(Xlo, xb, a.B, xb) || overlaps(Xlo, xb, a.X, xb)) {
            *info = -7;
            if (rep) rep->info = -7;
            return MP_OK;
        }
    }
    if (a.n == 0 || a.nrhs == 0) return MP_OK;
    mp_opts o;
    mp_default_opts(&o);
    if (opts) o = *opts;
    const int64_t n = a.n, nrhs = a.nrhs;
    const int nb = o.nb > 0 ? o.nb : default_nb(n);
    const int itermax = o.itermax > 0 ? std::min(o.itermax, MP_HIST_MAX - 1) : MP_ITERMAX_DEFAULT;
    check_size_limits(n);
    cudaStream_t s = g_stream;
    g_launches = 0;
    g_prof.reset((o.flags & 2) != 0, (o.flags & 4) != 0);
    g_prof.mask = (o.flags & 8) ? ((1u << KC_TRAIL) | (1u << KC_RESIDUAL)) : ~0u;
    Timer tm(s);
    const int t0 = tm.mark();
    Pool pool(s);
    Views v = stage_in(a, pool, s, true);
    const bool lo_host = !is_device_ptr(Xlo);
    double *XL = lo_host ? pool.get<double>((size_t)n * nrhs) : Xlo;
    const int t_staged = tm.mark();
    StatusIO sio(pool, s);
    const int sms = num_sms();
    const int64_t ldw = round_up(n, 64);
    double *W = pool.get<double>((size_t)n * ldw);
    int32_t *ipiv = pool.get<int32_t>(n), *perm = pool.get<int32_t>(n), *pinv = pool.get<int32_t>(n);
    double *Y = pool.get<double>((size_t)n * nrhs), *Z = pool.get<double>((size_t)n * nrhs);
    double *Rh = pool.get<double>((size_t)n * nrhs), *Rl = pool.get<double>((size_t)n * nrhs);
    double *dds = pool.get<double>(dd_scratch_doubles(n, sms));
    unsigned *cnt = pool.get<unsigned>(1);
    MP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned), s));
    SolveScratch ss{pool.get<unsigned>(solve_flag_words(n)), pool.get<double>((size_t)n * std::min<int64_t>(nrhs, 16)), 0u};
    MP_CUDA(cudaMemsetAsync(ss.flags, 0, solve_flag_words(n) * sizeof(unsigned), s));
    double *dpart = pool.get<double>((size_t)sms * 8);
    unsigned *dcnt = pool.get<unsigned>(1);
    MP_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned), s));
    {   // B finiteness
        launch_init_perm(perm, n, s);
        launch_permute_demote_rhs<double>(v.B, n, nrhs, perm, Y, sio.d, s);
    }
    // ||A||_F in binary64 (the demote kernel's sum of squares runs for the binary32 copy only:
    // take it from a throw-away binary32 demotion into W's storage, then overwrite W)
    launch_demote_transpose<float>(v.A, v.lda, n, reinterpret_cast<float *>(W), ldw, dpart, dcnt, sio.d, s);
    DevStatus st0 = sio.read();
    if (st0.flags & ST_A_NONFINITE) { *info = -3; if (rep) rep->info = -3; return MP_OK; }
    if (st0.flags & ST_B_NONFINITE) { *info = -5; if (rep) rep->info = -5; return MP_OK; }
    const double anrm = std::sqrt(st0.anrm2);
    const double cte = anrm * std::ldexp(1.0, -104) * std::sqrt((double)n);     // reading Q-1
    sio.reset();
    launch_demote_transpose<double>(v.A, v.lda, n, W, ldw, nullptr, nullptr, sio.d, s);
    const int t_dem = tm.mark();
    run_factor<double>(W, n, ldw, nb, ipiv, perm, sio.d, pool, s);                 // DGETRF
    const int t_fac = tm.mark();
    const DevStatus &st1 = sio.read();
    int nhist = 0;
    double hist[MP_HIST_MAX] = {0};
    if (st1.flags & ST_ZERO_PIVOT) {
        *info = st1.zero_col;
    } else {
        launch_invert_perm(perm, pinv, n, s);
        launch_permute_demote_rhs<double>(v.B, n, nrhs, pinv, Y, sio.d, s);
        prof_begin(KC_SOLVE, s);
        launch_lu_solve<double>(W, ldw, n, nrhs, Y, v.X, 0, ss, s);                // x0 = DGETRS(b)
        prof_end(KC_SOLVE, 8.0 * n * n, s);
        MP_CUDA(cudaMemsetAsync(XL, 0, (size_t)n * nrhs * sizeof(double), s));
        *iters = -31;
        for (int it = 0; it <= itermax; ++it) {
            prof_begin(KC_RESIDUAL, s);                                             // QGEMV (double-double)
            launch_dd_residual(v.A, v.lda, n, nrhs, v.B, v.X, XL, Rh, Rl, pinv, Y, cte, dds, cnt, sio.d, sms, s);
            prof_end(KC_RESIDUAL, 8.0 * n * n * nrhs, s);
            const DevStatus &st = sio.read();
            if (st.flags & ST_NORM_NONFINITE) break;
            hist[nhist++] = st.ratio;
            if (st.converged) { *iters = it; break; }
            if (it == itermax) break;
            prof_begin(KC_SOLVE, s);
            launch_lu_solve<double>(W, ldw, n, nrhs, Y, Z, 0, ss, s);               // DGETRS(fl64(P r))
            launch_dd_update(v.X, XL, Z, n * nrhs, s);                              // x += z (double-double)
            prof_end(KC_SOLVE, 8.0 * n * n, s);
        }
    }
    const int t_ref = tm.mark();
    if (lo_host) MP_CUDA(cudaMemcpyAsync(Xlo, XL, (size_t)n * nrhs * sizeof(double), cudaMemcpyDeviceToHost, s));
    finish_copy_out(a, v, s);
    const int t_end = tm.mark();
    MP_CUDA(cudaStreamSynchronize(s));
    if (rep) {
        rep->iters = *iters; rep->info = *info; rep->nhist = nhist; rep->nb = nb; rep->variant = -1;
        rep->anrm = anrm;
        for (int i = 0; i < nhist; ++i) rep->hist[i] = hist[i];
        rep->t_total_ms = tm.ms(t0, t_end);
        rep->t_copy_ms = tm.ms(t0, t_staged);
        rep->t_demote_ms = tm.ms(t_staged, t_dem);
        rep->t_factor_ms = tm.ms(t_dem, t_fac);
        rep->t_refine_ms = tm.ms(t_fac, t_ref);
        rep->workspace_bytes = pool.bytes;
        rep->kernel_launches = g_launches;
        if (!g_prof.deferred) prof_collect(rep);
    }
    if (!g_prof.deferred) g_prof.reset(false, false);
    else g_prof.on = false;
    return MP_OK;
}

// ------------------------------------------------------------------ NEXT-3: Algorithm 2 (FGMRES-GMRES_SP)
// PAPER.md P:240-279.  Outer FGMRES(m_out) in binary64 with the caller's A (its products through the
// residual kernel K8, modified Gram-Schmidt as printed), one GMRES_SP(m_in) cycle per outer step in
// binary32 with the row-major binary32 copy W (products: gemv_rows_f32; Arnoldi by classical
// Gram-Schmidt applied twice, reading G-6), Givens least squares on the device, B:5's test at the top of
// every outer cycle (G-1), at most itermax cycles (G-2).  x0 = 0.  One right-hand side.
int fgmres_impl(int64_t n, const double *A, int64_t lda, const double *b, double *x, int m_out, int m_in, int *iters,
                int *info, const mp_opts *opts, mp_report *rep)
{
    *info = 0; *iters = 0;
    if (rep) std::memset(rep, 0, sizeof(*rep));
    if (n < 0) return *info = -1, MP_OK;
    if (n > 0 && !A) return *info = -2, MP_OK;
    if (lda < std::max<int64_t>(1, n)) return *info = -3, MP_OK;
    if (n > 0 && !b) return *info = -4, MP_OK;
    if (n > 0 && !x) return *info = -5, MP_OK;
    if (m_out < 1 || m_in < 1 || m_out > 31 || m_in > 31) return *info = -6, MP_OK;
    if (n == 0) return MP_OK;
    mp_opts o;
    mp_default_opts(&o);
    if (opts) o = *opts;
    const int itermax = o.itermax > 0 ? std::min(o.itermax, MP_HIST_MAX - 1) : MP_ITERMAX_DEFAULT;
    cudaStream_t s = g_stream;
    g_launches = 0;
    g_prof.reset((o.flags & 2) != 0, (o.flags & 4) != 0);
    g_prof.mask = ~0u;
    Timer tm(s);
    const int t0 = tm.mark();
    Pool pool(s);
    Args a{n, 1, lda, A, b, x};
    Views v = stage_in(a, pool, s, true);
    StatusIO sio(pool, s);
    const int sms = num_sms();
    const int64_t ldw = round_up(n, 64);
    float *W = pool.get<float>((size_t)n * ldw);
    double *dpart = pool.get<double>((size_t)sms * 8);
    unsigned *dcnt = pool.get<unsigned>(1);
    MP_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned), s));
    int32_t *ident = pool.get<int32_t>(n);
    float *ychk = pool.get<float>(n);
    launch_demote_transpose<float>(v.A, v.lda, n, W, ldw, dpart, dcnt, sio.d, s);      // binary32 copy + ||A||_F
    launch_init_perm(ident, n, s);
    launch_permute_demote_rhs<float>(v.B, n, 1, ident, ychk, sio.d, s);
    const DevStatus st0 = sio.read();
    if (st0.flags & ST_A_NONFINITE) { *info = -2; if (rep) rep->info = -2; return MP_OK; }
    if (st0.flags & ST_B_NONFINITE) { *info = -4; if (rep) rep->info = -4; return MP_OK; }
    const double anrm = std::sqrt(st0.anrm2);
    const double cte = anrm * std::ldexp(1.0, -53) * std::sqrt((double)n);
    // binary64 outer workspace
    const int64_t ldv = round_up(n, 32);                     // 16-byte aligned columns for the vector kernels
    double *V = pool.get<double>((size_t)ldv * (m_out + 1)), *Z = pool.get<double>((size_t)ldv * m_out);
    double *r = pool.get<double>(n), *ax = pool.get<double>(n);
    double *R = pool.get<double>((size_t)(m_out + 1) * m_out), *cs = pool.get<double>(32), *sn = pool.get<double>(32);
    double *g = pool.get<double>(33), *y = pool.get<double>(32), *hcol = pool.get<double>(32), *hn = pool.get<double>(32);
    double *sc = pool.get<double>(8), *ones = pool.get<double>(32), *pd = pool.get<double>(gmres_partial_elems(n));
    // binary32 inner workspace
    float *Vs = pool.get<float>((size_t)ldv * (m_in + 1)), *vs = pool.get<float>(n), *zs = pool.get<float>(n);
    float *Rs = pool.get<float>((size_t)(m_in + 1) * m_in), *css = pool.get<float>(32), *sns = pool.get<float>(32);
    float *gs = pool.get<float>(33), *ys = pool.get<float>(32), *hs = pool.get<float>(32), *hs2 = pool.get<float>(32);
    float *hns = pool.get<float>(32), *scs = pool.get<float>(8), *oness = pool.get<float>(32);
    float *ps = pool.get<float>(gmres_partial_elems(n));
    const bool coop = !(o.flags & 128) && sp_cycle_supported(n, sms);   // G7: one launch per inner cycle
    float *cpart = coop ? pool.get<float>(sp_cycle_part_elems(sms)) : nullptr;
    float *craw = coop ? pool.get<float>((size_t)2 * ldv) : nullptr;
    unsigned *cbar = coop ? pool.get<unsigned>(1) : nullptr;
    ResidualScratch rs;
    rs.partial = pool.get<double>(residual_partial_elems(n, 1, sms));
    rs.blocksums = nullptr;
    rs.counter = nullptr;
    {
        std::vector<double> h1(32, 1.0);
        std::vector<float> h1s(32, 1.0f);
        MP_CUDA(cudaMemcpyAsync(ones, h1.data(), 32 * sizeof(double), cudaMemcpyHostToDevice, s));
        MP_CUDA(cudaMemcpyAsync(oness, h1s.data(), 32 * sizeof(float), cudaMemcpyHostToDevice, s));
        MP_CUDA(cudaMemsetAsync(v.X, 0, (size_t)n * sizeof(double), s));                        // x0 = 0
        MP_CUDA(cudaStreamSynchronize(s));                                                    // h1 / h1s lifetime
    }
    int nhist = 0;
    double hist[MP_HIST_MAX] = {0};
    *iters = -31;
    const int t_setup = tm.mark();
    for (int it = 0; it <= itermax; ++it) {
        // ---- r = b - A x_i (eps_d), beta = ||r||, ||x||; the check
        prof_begin(KC_RESIDUAL, s);
        launch_residual_products(v.A, v.lda, n, n, 1, v.X, n, ax, rs, sms, s);
        MP_CUDA(cudaMemcpyAsync(r, v.B, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        launch_combine<double>(r, ax, n, 1, ones, 1.0, -1.0, n, s);
        prof_end(KC_RESIDUAL, 8.0 * n * n, s);
        launch_multidot<double>(r, n, 1, r, n, pd, sc + 0, false, s);
        launch_multidot<double>(v.X, n, 1, v.X, n, pd, sc + 1, false, s);
        double hsc[2];
        MP_CUDA(cudaMemcpyAsync(hsc, sc, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
        const double beta = std::sqrt(hsc[0]), xn = std::sqrt(hsc[1]);
        if (!std::isfinite(beta) || !std::isfinite(xn)) break;
        hist[nhist++] = beta == 0.0 ? 0.0 : beta / (xn * cte);
        if (beta < xn * cte || beta == 0.0) { *iters = it; break; }                          // G-1
        if (it == itermax) break;
        // ---- one FGMRES(m_out) cycle
        launch_cycle_start<double>(sc + 0, g, m_out, sc + 2, s);                            // g = beta e_1
        for (int k = 0; k < m_out; ++k) {
            double *vk = V + (size_t)k * ldv, *zk = Z + (size_t)k * ldv;
            // v_k = r / h_{k,k-1} (eps_d), and its binary32 demotion for the inner solver
            launch_scale_copy<double, float>(r, k == 0 ? sc + 2 : hn + (k - 1), true, vk, vs, n, s);
            // ---- one GMRES_SP(m_in) cycle: A z = v_k, z = 0 initially (eps_s)
            prof_begin(KC_SOLVE, s);
            if (coop) {
                launch_gmres_sp_cycle(W, ldw, n, vs, Vs, ldv, craw, zk, m_in, cpart, cbar, sms, s);
                prof_end(KC_SOLVE, 4.0 * n * n * m_in, s);
            } else {
                launch_multidot<float>(vs, n, 1, vs, n, ps, scs + 0, false, s);
                launch_cycle_start<float>(scs + 0, gs, m_in, scs + 1, s);
                launch_scale_copy<float, float>(vs, scs + 1, true, Vs, nullptr, n, s);
                for (int j = 0; j < m_in; ++j) {
                    float *wj = Vs + (size_t)(j + 1) * ldv;
                    launch_gemv_rows_f32(W, ldw, n, Vs + (size_t)j * ldv, wj, s);
                    launch_multidot<float>(Vs, ldv, j + 1, wj, n, ps, hs, false, s);              // CGS, pass 1
                    launch_combine<float>(wj, Vs, ldv, j + 1, hs, 1.f, -1.f, n, s);
                    launch_multidot<float>(Vs, ldv, j + 1, wj, n, ps, hs2, false, s);             // pass 2 (G-6)
                    launch_combine<float>(wj, Vs, ldv, j + 1, hs2, 1.f, -1.f, n, s);
                    launch_combine<float>(hs, hs2, 32, 1, oness, 1.f, 1.f, j + 1, s);          // h += pass-2 h
                    launch_multidot<float>(wj, n, 1, wj, n, ps, scs + 2, false, s);
                    launch_givens_step<float>(hs, scs + 2, j, m_in, Rs, css, sns, gs, hns + j, s);
                    launch_scale_copy<float, float>(wj, hns + j, true, wj, nullptr, n, s);
                }
                launch_backsolve<float>(Rs, m_in, m_in, gs, ys, hns, s);
                launch_combine<float>(zs, Vs, ldv, m_in, ys, 0.f, 1.f, n, s);                     // z = V y
                prof_end(KC_SOLVE, 4.0 * n * n * m_in, s);
                launch_convert_f32_f64(zs, zk, n, s);
            }
            // ---- r = A z_k (eps_d); modified Gram-Schmidt against v_1..v_k (eps_d); h_{k+1,k}
            prof_begin(KC_RESIDUAL, s);
            launch_residual_products(v.A, v.lda, n, n, 1, zk, n, r, rs, sms, s);
            prof_end(KC_RESIDUAL, 8.0 * n * n, s);
            for (int j = 0; j <= k; ++j) {
                launch_multidot<double>(V + (size_t)j * ldv, ldv, 1, r, n, pd, hcol + j, false, s);
                launch_combine<double>(r, V + (size_t)j * ldv, ldv, 1, hcol + j, 1.0, -1.0, n, s);
            }
            launch_multidot<double>(r, n, 1, r, n, pd, sc + 3, false, s);
            launch_givens_step<double>(hcol, sc + 3, k, m_out, R, cs, sn, g, hn + k, s);
        }
        // ---- y = argmin ||beta e_1 - H y||, x += Z y (eps_d)
        launch_backsolve<double>(R, m_out, m_out, g, y, hn, s);
        launch_combine<double>(v.X, Z, ldv, m_out, y, 1.0, 1.0, n, s);
    }
    const int t_ref = tm.mark();
    finish_copy_out(a, v, s);
    const int t_end = tm.mark();
    MP_CUDA(cudaStreamSynchronize(s));
    if (rep) {
        rep->iters = *iters; rep->info = *info; rep->nhist = nhist; rep->variant = -2;
        rep->anrm = anrm;
        for (int i = 0; i < nhist; ++i) rep->hist[i] = hist[i];
        rep->t_total_ms = tm.ms(t0, t_end);
        rep->t_demote_ms = tm.ms(t0, t_setup);
        rep->t_refine_ms = tm.ms(t_setup, t_ref);
        rep->workspace_bytes = pool.bytes;
        rep->kernel_launches = g_launches;
        if (!g_prof.deferred) prof_collect(rep);
    }
    if (!g_prof.deferred) g_prof.reset(false, false);
    else g_prof.on = false;
    return MP_OK;
}

// ------------------------------------------------------------------ 1D block-cyclic multi-GPU path
// SURVEY 8(e) / B:5: global column block j (nb columns) lives on rank j mod P at local slot
// j / P; A (binary64, caller's) and the working copy use the same distribution; B, X, r, z,
// ipiv and perm are replicated.  Per panel step: the owner factors the panel (the single-GPU
// recursive panel code, addressed through a column-shifted base pointer), broadcasts it with
// its pivot list (NCCL), every rank applies the interchanges, U12 and the Schur update to its
// own columns.  The factors are all-gathered once for the (replicated) triangular solves;
// each residual is a local GEMV followed by an all-reduce of A_loc x_loc; rank 0's demoted
// residual and verdict are broadcast so every rank refines identically.
struct Dist {
    int64_t n = 0, nb = 0, nblk = 0, nloc = 0;
    int P = 1, r = 0;
    int owner(int64_t j) const { return (int)(j % P); }
    int64_t cols_of(int q) const
    {
        int64_t c = 0;
        for (int64_t j = q; j < nblk; j += P) c += std::min<int64_t>(nb, n - j * nb);
        return c;
    }
    // first local column whose global block is after block j
    int64_t local_after(int64_t j) const
    {
        const int64_t s = (j - r) >= 0 ? (j - r) / P + 1 : 0;
        return std::min<int64_t>(s * nb, nloc);
    }
};

__device__ __forceinline__ int64_t gcol_of(int64_t lc, int64_t nb, int P, int q)
{
    return ((lc / nb) * P + q) * nb + lc % nb;
}

// Xloc[c * nloc + lc] = X[c * n + gcol(lc)]
__global__ void gather_cols_kernel(const double *__restrict__ X, int64_t n, int64_t nrhs, double *__restrict__ Xloc,
                                   int64_t nloc, int64_t nb, int P, int q)
{
    const int64_t tot = nloc * nrhs;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / nloc, lc = t - c * nloc;
        Xloc[t] = X[c * n + gcol_of(lc, nb, P, q)];
    }
}

// send[i * nmax + lc] = Wl[i * ldw + lc] (lc < nloc), 0 up to nmax
template <typename T>
__global__ void pack_local_kernel(const T *__restrict__ Wl, int64_t ldw, int64_t n, int64_t nloc, int64_t nmax,
                                  T *__restrict__ send)
{
    const int64_t tot = n * nmax;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / nmax, lc = t - i * nmax;
        send[t] = lc < nloc ? Wl[i * ldw + lc] : T(0);
    }
}

// Wf[i * ldf + gcol(q, lc)] = recv[q][i * nmax + lc] for every rank q and lc < its columns
template <typename T>
__global__ void unpack_gather_kernel(const T *__restrict__ recv, int64_t n, int64_t nmax, int64_t nb, int P,
                                     T *__restrict__ Wf, int64_t ldf)
{
    const int64_t per = n * nmax, tot = per * P;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(t / per);
        const int64_t rem = t - (int64_t)q * per, i = rem / nmax, lc = rem - i * nmax;
        const int64_t g = gcol_of(lc, nb, P, q);
        if (g < n) Wf[i * ldf + g] = recv[t];
    }
}

// status flags over all ranks: every bit (and the first zero-pivot column) is reduced separately
__global__ void flags_to_bits_kernel(const DevStatus *st, int32_t *bits)
{
    const int i = threadIdx.x;
    if (i < 8) bits[i] = i < 5 ? ((st->flags >> i) & 1) : (i == 7 ? -st->zero_col : 0);
}
__global__ void bits_to_flags_kernel(DevStatus *st, const int32_t *bits)
{
    if (threadIdx.x == 0) {
        int f = 0;
        for (int i = 0; i < 5; ++i) f |= bits[i] << i;
        st->flags = f;
        st->zero_col = -bits[7];
    }
}
void sync_status(Comm &cm, DevStatus *st, int32_t *bits, cudaStream_t s)
{
    if (cm.size <= 1) return;
    flags_to_bits_kernel<<<1, 32, 0, s>>>(st, bits);
    MP_LAUNCH_CHECK();
    cm.allreduce_max(bits, 8, s);
    bits_to_flags_kernel<<<1, 32, 0, s>>>(st, bits);
    MP_LAUNCH_CHECK();
}

// binary-T factorisation of the distributed working copy Wl (n rows x ldw, local columns
// [0, nloc), panel receive area [nloc, nloc + nb)); ipiv/perm replicated
template <typename T>
void dist_factor(Comm &cm, const Dist &d, T *Wl, int64_t ldw, int32_t *ipiv, int32_t *perm, DevStatus *st,
                 Pool &pool, cudaStream_t s, int variant)
{
    const int64_t n = d.n, nb = d.nb;
    Factor<T> f;
    f.n = n; f.ldw = ldw; f.ipiv = ipiv; f.perm = perm; f.st = st; f.nb = (int)nb; f.s = s;
    f.sms = num_sms();
    f.variant = variant;
    f.ps.orig = pool.get<int32_t>(n);
    // left-looking leaves (MP_PANEL_LL=1, experimental: bitwise-correct but slower than the recursive
    // panel on B200)
    static const bool ll_env = [] { const char *e = std::getenv("MP_PANEL_LL"); return e && e[0] == '1'; }();
    if (sizeof(T) == 4 && ll_env && nb <= 256 && nb % 8 == 0) {   // (16-byte loads of the multipliers)
        f.lpos = pool.get<int32_t>(n);
        f.ll_panel = true;
    }
    f.ps.pairs = pool.get<int32_t>(4 * (size_t)nb);
    f.ps.npairs = pool.get<int32_t>(1);
    f.ps.ticket = pool.get<int32_t>(1);
    MP_CUDA(cudaMemsetAsync(f.ps.ticket, 0, sizeof(int32_t), s));
    if (const char *e = std::getenv("MP_NO_FUSED_TRSM")) f.fuse_trsm = e[0] != '1';
    if (const char *e = std::getenv("MP_NO_TC_INPANEL")) f.tc_inpanel = e[0] != '1';
    if (const char *e = std::getenv("MP_TF32_TERMS4_FRAC")) f.terms4_frac = std::atof(e);
    f.ppairs[0] = pool.get<int32_t>(4 * (size_t)nb);
    f.nppairs[0] = pool.get<int32_t>(1);
    f.ps.ppairs = f.ppairs[0];
    f.ps.nppairs = f.nppairs[0];
    float *tf = nullptr, *tfp = nullptr;
    if (sizeof(T) == 4 && tc_variant(variant)) {
        tf = pool.get<float>(tf32_scratch_floats(n, (int)nb));
        tfp = pool.get<float>(tf32_scratch_floats(n, (int)nb));
    }
    f.tf32[0] = tf;                                              // update stream
    f.tf32[1] = tfp;                                             // panel stream (in-panel K = 128 level)
    f.ppairs[1] = pool.get<int32_t>(4 * (size_t)nb);
    f.nppairs[1] = pool.get<int32_t>(1);
    // broadcast buffers (double-buffered for the look-ahead):
    // [npairs][pairs 4nb][ipiv nb] then the panel rows (n - k) x nb
    const size_t hdr = (1 + 4 * (size_t)nb + (size_t)nb) * sizeof(int32_t);
    const size_t hdr_al = round_up((int64_t)hdr, 256);
    char *bufs[2] = {pool.get<char>(hdr_al + (size_t)n * nb * sizeof(T)), pool.get<char>(hdr_al + (size_t)n * nb * sizeof(T))};
    // look-ahead (depth 1): the panel stream sP factors panel k+1 on its owner and carries every
    // broadcast; the update stream s applies panel k to the local columns, the next panel's
    // columns first.  MP_NO_LOOKAHEAD=1: everything on s, in order.
    // With the single-GPU execution resources: the update on the 100-SM green context, the panel
    // (and the broadcasts) on the high-priority panel stream; the caller's stream joins both.
    const bool la = !(std::getenv("MP_NO_LOOKAHEAD") && std::getenv("MP_NO_LOOKAHEAD")[0] == '1');
    // (loopback ranks share one GPU and must not share these per-device streams)
    const ExecRes &ex = cm.shared_device ? ExecRes{} : exec_res();
    const cudaStream_t s_caller = s;
    cudaStream_t sP = s;
    bool own_sP = false;
    int sms_upd = f.sms;
    if (la && ex.ok) {
        sP = ex.sP;
        s = ex.sU;
        sms_upd = ex.smsU;
        f.psms = std::max(8, f.sms - ex.smsU);
    } else if (la) {
        int lo = 0, hi = 0;
        MP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        MP_CUDA(cudaStreamCreateWithPriority(&sP, cudaStreamNonBlocking, hi));
        own_sP = true;
    }
    cudaEvent_t eB[2], eU[2], eN, e0;
    for (int i = 0; i < 2; ++i) {
        MP_CUDA(cudaEventCreateWithFlags(&eB[i], cudaEventDisableTiming));
        MP_CUDA(cudaEventCreateWithFlags(&eU[i], cudaEventDisableTiming));
        MP_CUDA(cudaEventRecord(eU[i], s));                     // both buffers free at the start
    }
    MP_CUDA(cudaEventCreateWithFlags(&eN, cudaEventDisableTiming));
    MP_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    if (s != s_caller) {                                         // the set-up above ran on the caller's stream
        MP_CUDA(cudaEventRecord(e0, s_caller));
        MP_CUDA(cudaStreamWaitEvent(s, e0, 0));
        for (int i = 0; i < 2; ++i) MP_CUDA(cudaEventRecord(eU[i], s));
    }
    launch_init_perm(perm, n, s);
    MP_CUDA(cudaEventRecord(e0, s));
    MP_CUDA(cudaStreamWaitEvent(sP, e0, 0));                     // workspace set-up done
    const int64_t nblk = d.nblk;
    auto lcol = [&](int64_t j) { return (j / d.P) * nb; };        // owner's local column of block j
    // panel j on its owner (stream sP, after the owner's update of its columns)
    auto factor_on_owner = [&](int64_t j) {
        const int64_t k = j * nb;
        const int w = (int)std::min<int64_t>(nb, n - k);
        f.W = Wl + (lcol(j) - k);                                // global column c <-> local lcol + (c - k)
        f.factor_panel(sP, k, w, (int)(j & 1));
    };
    // C(local cols [c_lo, c_hi)) -= L21 U12 with U12 = L11^-1 A12, panel k (Lp: its column 0)
    auto update_cols = [&](const T *Lp, int64_t k, int w, int64_t c_lo, int64_t c_hi) {
        const int64_t ncol = c_hi - c_lo;
        if (ncol <= 0 || k + w >= n) return;
        prof_begin(KC_TRSM, s);
        launch_trsm_ops<T>(Lp + k * ldw, ldw, Wl + k * ldw + c_lo, ldw, w, ncol, s);
        prof_end(KC_TRSM, (double)w * w * (double)ncol, s);
        const int64_t M = n - k - w;
        prof_begin(KC_TRAIL, s);
        if constexpr (sizeof(T) == 4) {
            if (tf && M >= 256 && ncol >= 128)
                launch_gemm_ops_3xtf32(Lp + (k + w) * ldw, ldw, Wl + k * ldw + c_lo, ldw, Wl + (k + w) * ldw + c_lo, ldw,
                                       M, ncol, w, tf, sms_upd, s);
            else
                launch_gemm_ops<T>(Lp + (k + w) * ldw, ldw, Wl + k * ldw + c_lo, ldw, Wl + (k + w) * ldw + c_lo, ldw, M,
                                   ncol, w, s);
        } else {
            launch_gemm_ops<T>(Lp + (k + w) * ldw, ldw, Wl + k * ldw + c_lo, ldw, Wl + (k + w) * ldw + c_lo, ldw, M, ncol,
                               w, s);
        }
        prof_end(KC_TRAIL, 2.0 * M * ncol * w, s);
    };
    if (d.r == d.owner(0)) factor_on_owner(0);
    for (int64_t j = 0; j < nblk; ++j) {
        const int64_t k = j * nb;
        const int w = (int)std::min<int64_t>(nb, n - k);
        const int o = d.owner(j), bi = (int)(j & 1);
        char *buf = bufs[bi];
        int32_t *b_np = reinterpret_cast<int32_t *>(buf), *b_pairs = b_np + 1, *b_ipiv = b_pairs + 4 * nb;
        T *b_panel = reinterpret_cast<T *>(buf + hdr_al);
        // ---- pack (owner) and broadcast panel j, on sP (the buffer is free once s unpacked j - 2)
        MP_CUDA(cudaStreamWaitEvent(sP, eU[bi], 0));
        if (d.r == o) {
            MP_CUDA(cudaMemcpyAsync(b_np, f.nppairs[bi], sizeof(int32_t), cudaMemcpyDeviceToDevice, sP));
            MP_CUDA(cudaMemcpyAsync(b_pairs, f.ppairs[bi], 4 * nb * sizeof(int32_t), cudaMemcpyDeviceToDevice, sP));
            MP_CUDA(cudaMemcpyAsync(b_ipiv, ipiv + k, w * sizeof(int32_t), cudaMemcpyDeviceToDevice, sP));
            MP_CUDA(cudaMemcpy2DAsync(b_panel, nb * sizeof(T), Wl + k * ldw + lcol(j), ldw * sizeof(T), w * sizeof(T),
                                      n - k, cudaMemcpyDeviceToDevice, sP));
        }
        if (d.P > 1) cm.bcast(buf, hdr_al + (size_t)(n - k) * nb * sizeof(T), o, sP);
        MP_CUDA(cudaEventRecord(eB[bi], sP));
        // ---- update stream: unpack (non-owners), interchanges, next panel's columns, the rest
        MP_CUDA(cudaStreamWaitEvent(s, eB[bi], 0));
        if (d.r != o) {
            MP_CUDA(cudaMemcpyAsync(f.nppairs[bi], b_np, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
            MP_CUDA(cudaMemcpyAsync(f.ppairs[bi], b_pairs, 4 * nb * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
            MP_CUDA(cudaMemcpyAsync(ipiv + k, b_ipiv, w * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
            MP_CUDA(cudaMemcpy2DAsync(Wl + k * ldw + d.nloc, ldw * sizeof(T), b_panel, nb * sizeof(T), w * sizeof(T),
                                      n - k, cudaMemcpyDeviceToDevice, s));
        }
        MP_CUDA(cudaEventRecord(eU[bi], s));
        // the panel's interchanges on this rank's other columns (+ the replicated permutation)
        const int64_t xlo = d.r == o ? lcol(j) : 0, xhi = d.r == o ? lcol(j) + w : 0;
        prof_begin(KC_LASWP, s);
        launch_laswp_pairs<T>(Wl, ldw, f.ppairs[bi], f.nppairs[bi], 2 * w, 0, d.nloc, xlo, xhi, perm, s);
        prof_end(KC_LASWP, 2.0 * 2 * w * (double)d.nloc * sizeof(T), s);
        const T *Lp = d.r == o ? Wl + lcol(j) : Wl + d.nloc;    // column 0 of the panel
        const int64_t lt0 = d.local_after(j);
        int64_t rest0 = lt0;
        if (j + 1 < nblk && d.r == d.owner(j + 1)) {
            // this rank factors the next panel: its columns first, then the panel on sP
            const int wn = (int)std::min<int64_t>(nb, n - k - nb);
            update_cols(Lp, k, w, lt0, lt0 + wn);
            rest0 = lt0 + wn;
            MP_CUDA(cudaEventRecord(eN, s));
            MP_CUDA(cudaStreamWaitEvent(sP, eN, 0));
            factor_on_owner(j + 1);
        }
        update_cols(Lp, k, w, rest0, d.nloc);
    }
    // join: the caller's stream waits for the panel and update streams' last work
    MP_CUDA(cudaEventRecord(e0, sP));
    MP_CUDA(cudaStreamWaitEvent(s_caller, e0, 0));
    MP_CUDA(cudaEventRecord(eN, s));
    MP_CUDA(cudaStreamWaitEvent(s_caller, eN, 0));
    MP_CUDA(cudaStreamSynchronize(s_caller));
    if (own_sP) MP_CUDA(cudaStreamDestroy(sP));
    for (int i = 0; i < 2; ++i) { MP_CUDA(cudaEventDestroy(eB[i])); MP_CUDA(cudaEventDestroy(eU[i])); }
    MP_CUDA(cudaEventDestroy(eN));
    MP_CUDA(cudaEventDestroy(e0));
}

// all-gather the distributed factors into the full row-major working copy Wf (n x ldf)
template <typename T>
void dist_gather(Comm &cm, const Dist &d, const T *Wl, int64_t ldw, T *Wf, int64_t ldf, Pool &pool, cudaStream_t s)
{
    const int64_t nmax = ceil_div(d.nblk, d.P) * d.nb;
    T *send = pool.get<T>((size_t)d.n * nmax);
    T *recv = pool.get<T>((size_t)d.n * nmax * d.P);
    const int64_t tot = d.n * nmax;
    pack_local_kernel<T><<<(int)std::min<int64_t>(ceil_div(tot, 256), 8192), 256, 0, s>>>(Wl, ldw, d.n, d.nloc, nmax,
                                                                                          send);
    MP_LAUNCH_CHECK();
    cm.allgather(send, recv, (size_t)tot * sizeof(T), s);
    unpack_gather_kernel<T><<<(int)std::min<int64_t>(ceil_div(tot * d.P, 256), 8192), 256, 0, s>>>(
        recv, d.n, nmax, d.nb, d.P, Wf, ldf);
    MP_LAUNCH_CHECK();
    g_launches += 2;
}

// binary64 solve on the distribution (fallback and mp_dgesv_1dbc): returns info
int dist_fp64_solve(Comm &cm, const Dist &d, const double *A, int64_t lda, const double *B, double *X, int64_t nrhs,
                    Pool &pool, StatusIO &sio, cudaStream_t s)
{
    const int64_t n = d.n;
    const int64_t ldw = round_up(d.nloc + d.nb, 64), ldf = round_up(n, 64);
    double *Wl = pool.get<double>((size_t)n * ldw);
    int32_t *ipiv = pool.get<int32_t>(n), *perm = pool.get<int32_t>(n), *pinv = pool.get<int32_t>(n);
    sio.reset();
    launch_demote_rect<double>(A, lda, n, d.nloc, Wl, ldw, nullptr, nullptr, sio.d, s);
    dist_factor<double>(cm, d, Wl, ldw, ipiv, perm, sio.d, pool, s, MP_VARIANT_FFMA);
    // status (a zero pivot is seen by the panel's owner only) -> every rank
    sync_status(cm, sio.d, pool.get<int32_t>(8), s);
    const DevStatus &st = sio.read();
    if (st.flags & ST_A_NONFINITE) return -3;
    if (st.flags & ST_ZERO_PIVOT) return st.zero_col;
    double *Wf = pool.get<double>((size_t)n * ldf);
    MP_CUDA(cudaMemsetAsync(Wf, 0, (size_t)n * ldf * sizeof(double), s));
    dist_gather<double>(cm, d, Wl, ldw, Wf, ldf, pool, s);
    double *Y = pool.get<double>((size_t)n * nrhs);
    SolveScratch ss{pool.get<unsigned>(solve_flag_words(n)), pool.get<double>((size_t)n * std::min<int64_t>(nrhs, 16)), 0u};
    MP_CUDA(cudaMemsetAsync(ss.flags, 0, solve_flag_words(n) * sizeof(unsigned), s));
    launch_invert_perm(perm, pinv, n, s);
    launch_permute_demote_rhs<double>(B, n, nrhs, pinv, Y, sio.d, s);
    launch_lu_solve<double>(Wf, ldf, n, nrhs, Y, X, 0, ss, s);
    return 0;
}

int dsgesv_1dbc_impl(Comm &cm, int64_t n, int64_t nrhs, int64_t nb, const double *A, int64_t lda, const double *B,
                     double *X, int *iters, int *info, const mp_opts *opts, mp_report *rep, bool fp64_only)
{
    *info = 0; *iters = 0;
    if (rep) std::memset(rep, 0, sizeof(*rep));
    Dist d;
    d.n = n; d.nb = nb > 0 ? nb : 256; d.P = cm.size; d.r = cm.rank;
    d.nblk = n > 0 ? ceil_div(n, d.nb) : 0;
    d.nloc = n > 0 ? d.cols_of(d.r) : 0;
    const int64_t mx = std::max<int64_t>(1, d.nloc);
    if (n < 0) return *info = -2, MP_OK;
    if (nrhs < 0) return *info = -3, MP_OK;
    if (nb < 0) return *info = -4, MP_OK;
    if (n > 0 && d.nloc > 0 && !A) return *info = -5, MP_OK;
    if (lda < mx) return *info = -6, MP_OK;
    if (n > 0 && nrhs > 0 && (!B || !X)) return *info = -7, MP_OK;
    if ((d.nloc > 0 && !is_device_ptr(A)) || (n > 0 && nrhs > 0 && (!is_device_ptr(B) || !is_device_ptr(X))))
        throw std::runtime_error("mp_*_1dbc: A_local, B and X must be device pointers");
    if (n == 0 || nrhs == 0) return MP_OK;
    mp_opts o;
    mp_default_opts(&o);
    if (opts) o = *opts;
    const int itermax = o.itermax > 0 ? std::min(o.itermax, MP_HIST_MAX - 1) : MP_ITERMAX_DEFAULT;
    check_size_limits(n);
    cudaStream_t s = g_stream;
    g_launches = 0;
    g_prof.reset((o.flags & 2) != 0, (o.flags & 4) != 0);
    g_prof.mask = (o.flags & 8) ? ((1u << KC_TRAIL) | (1u << KC_RESIDUAL)) : ~0u;
    Timer tm(s);
    const int t0 = tm.mark();
    Pool pool(s);
    StatusIO sio(pool, s);
    if (fp64_only) {
        *info = dist_fp64_solve(cm, d, A, lda, B, X, nrhs, pool, sio, s);
        MP_CUDA(cudaStreamSynchronize(s));
        if (rep) { rep->info = *info; rep->nb = (int)d.nb; rep->t_total_ms = tm.ms(t0, tm.mark()); }
        return MP_OK;
    }
    const int sms = num_sms();
    const int64_t ldw = round_up(d.nloc + d.nb, 64), ldf = round_up(n, 64);
    float *Wl = pool.get<float>((size_t)n * ldw);
    int32_t *ipiv = pool.get<int32_t>(n), *perm = pool.get<int32_t>(n), *pinv = pool.get<int32_t>(n);
    float *Y = pool.get<float>((size_t)n * nrhs);
    double *R = pool.get<double>((size_t)n * nrhs), *AX = pool.get<double>((size_t)n * nrhs);
    double *Xloc = pool.get<double>((size_t)std::max<int64_t>(1, d.nloc) * nrhs);
    ResidualScratch rs;
    rs.partial = pool.get<double>(residual_partial_elems(n, nrhs, sms));
    rs.blocksums = pool.get<double>((size_t)ceil_div(n, 256) * 2 * nrhs);
    rs.counter = pool.get<unsigned>(1);
    SolveScratch ss{pool.get<unsigned>(solve_flag_words(n)), pool.get<float>((size_t)n * std::min<int64_t>(nrhs, 16)), 0u};
    MP_CUDA(cudaMemsetAsync(ss.flags, 0, solve_flag_words(n) * sizeof(unsigned), s));
    ss.tags = pool.get<uint64_t>(solve_tag_words(n, nrhs));
    ss.tag_cols = (int)std::min<int64_t>(nrhs, 16);
    MP_CUDA(cudaMemsetAsync(ss.tags, 0, solve_tag_words(n, nrhs) * sizeof(uint64_t), s));
    double *dpart = pool.get<double>((size_t)sms * 8);
    unsigned *dcnt = pool.get<unsigned>(1);
    MP_CUDA(cudaMemsetAsync(rs.counter, 0, sizeof(unsigned), s));
    MP_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned), s));

    // ---- K1 on the local columns; ||A||_F^2 and the argument / overflow flags over all ranks
    prof_begin(KC_DEMOTE, s);
    launch_demote_rect<float>(A, lda, n, d.nloc, Wl, ldw, dpart, dcnt, sio.d, s);
    prof_end(KC_DEMOTE, 12.0 * n * d.nloc, s);
    launch_init_perm(perm, n, s);
    launch_permute_demote_rhs<float>(B, n, nrhs, perm, Y, sio.d, s);
    int32_t *bits = pool.get<int32_t>(8);
    if (d.P > 1) {
        cm.allreduce_sum(&sio.d->anrm2, 1, s);
        sync_status(cm, sio.d, bits, s);
    }
    DevStatus st0 = sio.read();
    if (st0.flags & ST_A_NONFINITE) { *info = -5; if (rep) rep->info = -5; return MP_OK; }
    if (st0.flags & ST_B_NONFINITE) { *info = -7; if (rep) rep->info = -7; return MP_OK; }
    const double anrm = std::sqrt(st0.anrm2);
    const double cte = anrm * std::ldexp(1.0, -53) * std::sqrt((double)n);
    int code = (st0.flags & ST_OVERFLOW) ? -2 : 0;
    const int t_dem = tm.mark();
    int t_fac = t_dem, t_ref = t_dem;
    int nhist = 0;
    double hist[MP_HIST_MAX] = {0};
    bool used_inv = false;
    float *Wf = nullptr;
    if (!code) {
        dist_factor<float>(cm, d, Wl, ldw, ipiv, perm, sio.d, pool, s, o.variant);
        sync_status(cm, sio.d, bits, s);
        t_fac = tm.mark();
        const DevStatus &st1 = sio.read();
        if (st1.flags & ST_ZERO_PIVOT) code = -3;
    }
    if (!code) {
        Wf = pool.get<float>((size_t)n * ldf);
        MP_CUDA(cudaMemsetAsync(Wf, 0, (size_t)n * ldf * sizeof(float), s));
        dist_gather<float>(cm, d, Wl, ldw, Wf, ldf, pool, s);
        launch_invert_perm(perm, pinv, n, s);
        launch_permute_demote_rhs<float>(B, n, nrhs, pinv, Y, sio.d, s);
        float *inv = nullptr;
        if (!(o.flags & 32)) {
            inv = pool.get<float>(solve_inv_floats(n));
            launch_solve_inverses(Wf, ldf, n, inv, s);
            if (!(solve_inverses_cond(inv, n, s) <= kInvCondMax)) inv = nullptr;
        }
        used_inv = inv != nullptr;
        // With nrhs >= P the triangular solves are split by right-hand-side column: rank r solves
        // (and updates x for) columns [r cpr, (r + 1) cpr) only, then the solution columns are
        // all-gathered, so the refinement's O(n^2 nrhs) solve work scales with P (C4: nrhs = 16).
        // MP_DIST_REPLICATED_SOLVES=1: every rank solves every column (the round-1 scheme).
        static const bool replicated = std::getenv("MP_DIST_REPLICATED_SOLVES") != nullptr;
        const bool split = d.P > 1 && nrhs >= d.P && !replicated;
        const int64_t cpr = split ? ceil_div(nrhs, (int64_t)d.P) : nrhs;
        const int64_t c_lo = split ? std::min<int64_t>(nrhs, (int64_t)d.r * cpr) : 0;
        const int64_t nc = split ? std::max<int64_t>(0, std::min<int64_t>(nrhs, c_lo + cpr) - c_lo) : nrhs;
        double *Zg = split ? pool.get<double>((size_t)n * cpr * d.P) : nullptr;
        auto solve = [&](int accumulate) {
            prof_begin(KC_SOLVE, s);
            if (nc > 0) launch_lu_solve<float>(Wf, ldf, n, nc, Y + c_lo * n, X + c_lo * n, accumulate, ss, s, inv);
            prof_end(KC_SOLVE, 4.0 * n * n, s);
            if (split) {
                if (nc > 0)
                    MP_CUDA(cudaMemcpyAsync(Zg + (size_t)d.r * cpr * n, X + c_lo * n, (size_t)n * nc * sizeof(double),
                                            cudaMemcpyDeviceToDevice, s));
                cm.allgather(Zg + (size_t)d.r * cpr * n, Zg, (size_t)n * cpr * sizeof(double), s);
                MP_CUDA(cudaMemcpyAsync(X, Zg, (size_t)n * nrhs * sizeof(double), cudaMemcpyDeviceToDevice, s));
            }
        };
        solve(0);
        code = -31;
        const int gblk = (int)std::min<int64_t>(ceil_div(d.nloc * nrhs, 256), 4096);
        for (int it = 0; it <= itermax; ++it) {
            prof_begin(KC_RESIDUAL, s);
            if (d.nloc > 0) {
                gather_cols_kernel<<<std::max(1, gblk), 256, 0, s>>>(X, n, nrhs, Xloc, d.nloc, d.nb, d.P, d.r);
                MP_LAUNCH_CHECK();
            }
            launch_residual_products(A, lda, n, d.nloc, nrhs, Xloc, std::max<int64_t>(1, d.nloc), AX, rs, sms, s);
            if (d.P > 1) cm.allreduce_sum(AX, (size_t)n * nrhs, s);
            launch_residual_finalize<float>(AX, n, nrhs, B, X, R, pinv, Y, cte, rs, sio.d, s);
            // rank 0's demoted residual and verdict drive every rank (identical refinement)
            if (d.P > 1) {
                cm.bcast(Y, (size_t)n * nrhs * sizeof(float), 0, s);
                cm.bcast(sio.d, sizeof(DevStatus), 0, s);
            }
            prof_end(KC_RESIDUAL, 8.0 * n * d.nloc + 8.0 * 4 * n * nrhs, s);
            const DevStatus &st = sio.read();
            if (st.flags & ST_NORM_NONFINITE) break;
            hist[nhist++] = st.ratio;
            if (st.converged) { *iters = it; code = 0; break; }
            if (it == itermax) break;
            solve(1);
        }
        t_ref = tm.mark();
    }
    int t_fb = tm.mark();
    if (code) {
        *iters = code;
        *info = dist_fp64_solve(cm, d, A, lda, B, X, nrhs, pool, sio, s);
        t_fb = tm.mark();
    }
    MP_CUDA(cudaStreamSynchronize(s));
    const int t_end = tm.mark();
    MP_CUDA(cudaStreamSynchronize(s));
    if (rep) {
        rep->iters = *iters; rep->info = *info; rep->nhist = nhist; rep->nb = (int)d.nb; rep->variant = o.variant;
        rep->solve_inv = used_inv ? 1 : 0;
        rep->anrm = anrm;
        for (int i = 0; i < nhist; ++i) rep->hist[i] = hist[i];
        rep->t_total_ms = tm.ms(t0, t_end);
        rep->t_demote_ms = tm.ms(t0, t_dem);
        rep->t_factor_ms = (t_fac != t_dem) ? tm.ms(t_dem, t_fac) : 0.0;
        rep->t_refine_ms = (t_ref != t_dem) ? tm.ms(t_fac, t_ref) : 0.0;
        rep->t_fallback_ms = code ? tm.ms(t_ref, t_fb) : 0.0;
        rep->workspace_bytes = pool.bytes;
        rep->kernel_launches = g_launches;
        if (!g_prof.deferred) prof_collect(rep);
    }
    if (!g_prof.deferred) g_prof.reset(false, false);
    else g_prof.on = false;
    return MP_OK;
}

template <typename F>
int guarded(F &&f)
{
    try {
        return f();
    } catch (const CudaError &e) {
        char buf[512];
        std::snprintf(buf, sizeof(buf), "CUDA error %d (%s) at driver/kernels line %d: %s", (int)e.err,
                      cudaGetErrorString(e.err), e.line, e.what);
        g_err = buf;
        return e.err == cudaErrorMemoryAllocation ? MP_ERR_NOMEM : MP_ERR_CUDA;
    } catch (const NoMem &) {
        g_err = "device workspace allocation failed";
        return MP_ERR_NOMEM;
    } catch (const CommError &e) {
        g_err = e.what;
        return MP_ERR_NCCL;
    } catch (const std::exception &e) {
        g_err = e.what();
        return MP_ERR_UNSUPPORTED;
    } catch (...) {
        g_err = "unknown internal error";
        return MP_ERR_INTERNAL;
    }
}

}  // namespace
}  // namespace mp

using namespace mp;

extern "C" {

void mp_default_opts(mp_opts *o)
{
    if (!o) return;
    o->nb = 0;
    o->itermax = MP_ITERMAX_DEFAULT;
    o->variant = MP_VARIANT_3XTF32;
    o->flags = 0;
}

int mp_dsgesv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int *iters,
                 int *info, const mp_opts *opts, mp_report *rep)
{
    if (!iters || !info) { g_err = "iters/info must not be NULL"; return MP_ERR_INTERNAL; }
    return guarded([&] { return dsgesv_impl(Args{n, nrhs, lda, A, B, X}, iters, info, opts, rep); });
}

int mp_dsgesv(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int *iters,
              int *info)
{
    return mp_dsgesv_ex(n, nrhs, A, lda, B, X, iters, info, nullptr, nullptr);
}

int mp_dgesv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int *info,
                const mp_opts *opts, mp_report *rep)
{
    if (!info) { g_err = "info must not be NULL"; return MP_ERR_INTERNAL; }
    return guarded([&] { return dgesv_impl(Args{n, nrhs, lda, A, B, X}, info, opts, rep); });
}

int mp_dgesv(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int *info)
{
    return mp_dgesv_ex(n, nrhs, A, lda, B, X, info, nullptr, nullptr);
}

int mp_sgetrf(int64_t n, const double *A, int64_t lda, float *LU, int32_t *ipiv, int *info, const mp_opts *opts)
{
    if (!info) { g_err = "info must not be NULL"; return MP_ERR_INTERNAL; }
    return guarded([&] { return getrf_impl<float>(n, A, lda, LU, ipiv, info, opts); });
}

int mp_dgetrf(int64_t n, const double *A, int64_t lda, double *LU, int32_t *ipiv, int *info, const mp_opts *opts)
{
    if (!info) { g_err = "info must not be NULL"; return MP_ERR_INTERNAL; }
    return guarded([&] { return getrf_impl<double>(n, A, lda, LU, ipiv, info, opts); });
}

int mp_dsposv(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int *iters, int *info)
{
    return guarded([&] { return dsposv_impl(Args{n, nrhs, lda, A, B, X}, iters, info, nullptr, nullptr); });
}

int mp_dsposv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int *iters,
                 int *info, const mp_opts *opts, mp_report *rep)
{
    return guarded([&] { return dsposv_impl(Args{n, nrhs, lda, A, B, X}, iters, info, opts, rep); });
}

int mp_dposv(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int *info)
{
    return guarded([&] { return dposv_impl(Args{n, nrhs, lda, A, B, X}, info, nullptr, nullptr); });
}

int mp_dposv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *X, int *info,
                const mp_opts *opts, mp_report *rep)
{
    return guarded([&] { return dposv_impl(Args{n, nrhs, lda, A, B, X}, info, opts, rep); });
}

int mp_spotrf(int64_t n, const double *A, int64_t lda, float *L, int *info, const mp_opts *opts)
{
    return guarded([&] { return potrf_impl<float>(n, A, lda, L, info, opts); });
}

int mp_dpotrf(int64_t n, const double *A, int64_t lda, double *L, int *info, const mp_opts *opts)
{
    return guarded([&] { return potrf_impl<double>(n, A, lda, L, info, opts); });
}

int mp_qdgesv(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *Xhi, double *Xlo,
              int *iters, int *info)
{
    if (!iters || !info) { g_err = "iters/info must not be NULL"; return MP_ERR_INTERNAL; }
    return guarded([&] { return qdgesv_impl(Args{n, nrhs, lda, A, B, Xhi}, Xlo, iters, info, nullptr, nullptr); });
}

int mp_qdgesv_ex(int64_t n, int64_t nrhs, const double *A, int64_t lda, const double *B, double *Xhi, double *Xlo,
                 int *iters, int *info, const mp_opts *opts, mp_report *rep)
{
    if (!iters || !info) { g_err = "iters/info must not be NULL"; return MP_ERR_INTERNAL; }
    return guarded([&] { return qdgesv_impl(Args{n, nrhs, lda, A, B, Xhi}, Xlo, iters, info, opts, rep); });
}

int mp_fgmres(int64_t n, const double *A, int64_t lda, const double *b, double *x, int m_out, int m_in, int *iters,
              int *info)
{
    if (!iters || !info) { g_err = "iters/info must not be NULL"; return MP_ERR_INTERNAL; }
    return guarded([&] { return fgmres_impl(n, A, lda, b, x, m_out, m_in, iters, info, nullptr, nullptr); });
}

int mp_fgmres_ex(int64_t n, const double *A, int64_t lda, const double *b, double *x, int m_out, int m_in,
                 int *iters, int *info, const mp_opts *opts, mp_report *rep)
{
    if (!iters || !info) { g_err = "iters/info must not be NULL"; return MP_ERR_INTERNAL; }
    return guarded([&] { return fgmres_impl(n, A, lda, b, x, m_out, m_in, iters, info, opts, rep); });
}

int mp_kernel_schur_update(float *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N,
                           int64_t K, int variant)
{
    const int cluster = (variant >> 8) & 0xf;      // bits 8-11: cluster size of the tcgen05 kernel (0: default policy)
    variant &= 0xff;
    return guarded([&] {
        cudaStream_t s = g_stream;
        if (tc_variant(variant)) {
            struct Force { explicit Force(int c) { set_gemm_tf32_cluster(c); } ~Force() { set_gemm_tf32_cluster(0); } } force(cluster);
            float *scratch = nullptr;
            const size_t bytes = ((size_t)2 * M * round_up(K, 4) + (size_t)2 * N * round_up(K, 4) + 4096) * 4;
            MP_CUDA(cudaMallocFromPoolAsync((void **)&scratch, bytes, library_pool(), s));
            launch_gemm_update_3xtf32(W, ldw, r0, c0, k0, M, N, K, scratch, num_sms(), s, false,
                                      variant == MP_VARIANT_TF32 ? 1 : 3);
            MP_CUDA(cudaFreeAsync(scratch, s));
        } else {
            launch_gemm_update<float>(W, ldw, r0, c0, k0, M, N, K, s);
        }
        MP_CUDA(cudaStreamSynchronize(s));
        return MP_OK;
    });
}

int mp_kernel_schur_update_f64(double *W, int64_t ldw, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N,
                               int64_t K, int pipe)
{
    return guarded([&] {
        cudaStream_t s = g_stream;
        const double *A = W + r0 * ldw + k0, *B = W + k0 * ldw + c0;
        double *C = W + r0 * ldw + c0;
        if (pipe == MP_F64_DMMA) {
            if (!launch_dgemm_dmma(A, ldw, B, ldw, C, ldw, M, N, K, s))
                throw std::runtime_error("DMMA update: N, K and the row starts must be even");
        } else if (pipe == MP_F64_DFMA) {
            launch_dgemm_dfma(A, ldw, B, ldw, C, ldw, M, N, K, s);
        } else {
            launch_gemm_update<double>(W, ldw, r0, c0, k0, M, N, K, s);
        }
        MP_CUDA(cudaStreamSynchronize(s));
        return MP_OK;
    });
}

int mp_profile_collect(mp_report *rep)
{
    return guarded([&] {
        if (!rep) return MP_OK;
        for (int i = 0; i < 8; ++i) { rep->k_ms[i] = 0; rep->k_work[i] = 0; rep->k_launches[i] = 0; }
        prof_collect(rep);
        g_prof.deferred = false;
        g_prof.reset(false, false);
        return MP_OK;
    });
}

int mp_set_stream(void *stream)
{
    g_stream = static_cast<cudaStream_t>(stream);
    return MP_OK;
}

const char *mp_last_error(void) { return g_err.c_str(); }

const char *mp_version(void)
{
    return "libmpsolve 0.3 (sm_100a; variants: ffma, 3xtf32-tcgen05; blocked right-looking GEPP with look-ahead on "
           "green contexts, cluster panel, row-major working copy)";
}

struct mp_comm {
    Comm *c;
};

int mp_get_unique_id(char id[128])
{
    if (!id) { g_err = "id must not be NULL"; return MP_ERR_INTERNAL; }
    return guarded([&] { nccl_unique_id(id); return MP_OK; });
}

int mp_comm_init(int nranks, int rank, const char id[128], mp_comm **comm)
{
    if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) { g_err = "bad mp_comm_init arguments"; return MP_ERR_INTERNAL; }
    return guarded([&] {
        *comm = new mp_comm{make_nccl_comm(nranks, rank, id)};
        return MP_OK;
    });
}

int mp_comm_init_loopback(int nranks, mp_comm **comms)
{
    if (!comms || nranks < 1) { g_err = "bad mp_comm_init_loopback arguments"; return MP_ERR_INTERNAL; }
    return guarded([&] {
        std::vector<Comm *> cs(nranks);
        make_loopback_comms(nranks, cs.data());
        for (int r = 0; r < nranks; ++r) comms[r] = new mp_comm{cs[r]};
        return MP_OK;
    });
}

int mp_comm_destroy(mp_comm *comm)
{
    if (!comm) return MP_OK;
    return guarded([&] {
        delete comm->c;
        delete comm;
        return MP_OK;
    });
}

int64_t mp_1dbc_local_cols(int64_t n, int64_t nb, int nranks, int rank)
{
    if (n <= 0 || nranks < 1 || rank < 0 || rank >= nranks) return 0;
    Dist d;
    d.n = n; d.nb = nb > 0 ? nb : 256; d.P = nranks; d.r = rank; d.nblk = ceil_div(n, d.nb);
    return d.cols_of(rank);
}

int mp_dsgesv_1dbc_ex(mp_comm *comm, int64_t n, int64_t nrhs, int64_t nb, const double *A_local, int64_t lda_local,
                      const double *B, double *X, int *iters, int *info, const mp_opts *opts, mp_report *rep)
{
    if (!comm || !iters || !info) { g_err = "comm/iters/info must not be NULL"; return MP_ERR_INTERNAL; }
    return guarded([&] {
        return dsgesv_1dbc_impl(*comm->c, n, nrhs, nb, A_local, lda_local, B, X, iters, info, opts, rep, false);
    });
}

int mp_dsgesv_1dbc(mp_comm *comm, int64_t n, int64_t nrhs, int64_t nb, const double *A_local, int64_t lda_local,
                   const double *B, double *X, int *iters, int *info)
{
    return mp_dsgesv_1dbc_ex(comm, n, nrhs, nb, A_local, lda_local, B, X, iters, info, nullptr, nullptr);
}

int mp_dgesv_1dbc(mp_comm *comm, int64_t n, int64_t nrhs, int64_t nb, const double *A_local, int64_t lda_local,
                  const double *B, double *X, int *info)
{
    if (!comm || !info) { g_err = "comm/info must not be NULL"; return MP_ERR_INTERNAL; }
    int iters = 0;
    return guarded([&] {
        return dsgesv_1dbc_impl(*comm->c, n, nrhs, nb, A_local, lda_local, B, X, &iters, info, nullptr, nullptr, true);
    });
}

int mp_exec_info(int *lookahead, int *sms_panel, int *sms_update)
{
    return guarded([&] {
        const ExecRes &ex = exec_res();
        const int all = num_sms();
        if (lookahead) *lookahead = ex.ok ? 1 : 0;
        if (sms_panel) *sms_panel = ex.ok ? all - ex.smsU : 0;
        if (sms_update) *sms_update = ex.ok ? ex.smsU : all;
        return MP_OK;
    });
}

}  // extern "C"
