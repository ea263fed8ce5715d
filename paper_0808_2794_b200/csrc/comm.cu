// comm.cu — collectives of the 1D block-cyclic multi-GPU path.
//
// Two implementations of the small Comm interface (internal.h):
//   * NcclComm: one process per GPU; NCCL (the process's libnccl.so.2, loaded with
//     dlopen so the library has no link-time NCCL dependency — under PyTorch it is the
//     NCCL torch already loaded) over NVLink / NVSwitch.  Collectives are enqueued on the
//     caller's stream (stream-ordered, asynchronous).
//   * LoopbackComm: P ranks emulated as P host threads of ONE process on ONE GPU, each
//     with its own stream; a collective synchronises the calling thread's stream, meets
//     the other threads at a host barrier and moves data with device copies.  No kernel
//     ever waits on another rank's kernel, so ranks sharing a GPU cannot deadlock it; this
//     is how the P > 1 algorithm is tested on a single-GPU box.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "internal.h"

namespace mp {

namespace {

// ---------------------------------------------------------------- NCCL through dlopen
struct NcclApi {
    bool ok = false;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*errStr)(ncclResult_t) = nullptr;
};

NcclApi &nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *env = std::getenv("MP_NCCL_LIB");
        void *h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
        api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
        api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
        api.errStr = reinterpret_cast<decltype(api.errStr)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.broadcast && api.allReduce &&
                 api.allGather && api.errStr;
    });
    return api;
}

void nccl_check(ncclResult_t r, const char *what)
{
    if (r != ncclSuccess) {
        static thread_local std::string msg;
        msg = std::string(what) + ": " + (nccl().errStr ? nccl().errStr(r) : "NCCL error");
        throw CommError{msg.c_str()};
    }
}

struct NcclComm final : Comm {
    ncclComm_t c = nullptr;
    ~NcclComm() override
    {
        if (c) nccl().commDestroy(c);
    }
    void bcast(void *buf, size_t bytes, int root, cudaStream_t s) override
    {
        nccl_check(nccl().broadcast(buf, buf, bytes, ncclInt8, root, c, s), "ncclBroadcast");
    }
    void allreduce_sum(double *buf, size_t count, cudaStream_t s) override
    {
        nccl_check(nccl().allReduce(buf, buf, count, ncclFloat64, ncclSum, c, s), "ncclAllReduce");
    }
    void allreduce_max(int32_t *buf, size_t count, cudaStream_t s) override
    {
        nccl_check(nccl().allReduce(buf, buf, count, ncclInt32, ncclMax, c, s), "ncclAllReduce");
    }
    void allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) override
    {
        nccl_check(nccl().allGather(send, recv, bytes, ncclInt8, c, s), "ncclAllGather");
    }
};

// ---------------------------------------------------------------- loopback emulation
struct LoopbackShared {
    int size;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long generation = 0;
    std::vector<const void *> send;   // per-rank source pointers of the current collective
    std::vector<void *> recv;
    explicit LoopbackShared(int p) : size(p), send(p, nullptr), recv(p, nullptr) {}
    void barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        const long long gen = generation;
        if (++arrived == size) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

__global__ void sum_into_kernel(double *dst, const double *src, size_t count)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
        dst[i] += src[i];
}
__global__ void max_into_kernel(int32_t *dst, const int32_t *src, size_t count)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = dst[i] > src[i] ? dst[i] : src[i];
}

struct LoopbackComm final : Comm {
    std::shared_ptr<LoopbackShared> sh;
    void bcast(void *buf, size_t bytes, int root, cudaStream_t s) override
    {
        MP_CUDA(cudaStreamSynchronize(s));
        sh->recv[rank] = buf;
        sh->barrier();
        if (rank != root) MP_CUDA(cudaMemcpyAsync(buf, sh->recv[root], bytes, cudaMemcpyDeviceToDevice, s));
        MP_CUDA(cudaStreamSynchronize(s));
        sh->barrier();
    }
    template <typename T, typename K>
    void allreduce(T *buf, size_t count, cudaStream_t s, K kern)
    {
        MP_CUDA(cudaStreamSynchronize(s));
        T *tmp = nullptr;
        MP_CUDA(cudaMalloc(&tmp, count * sizeof(T) + 1));
        MP_CUDA(cudaMemcpyAsync(tmp, buf, count * sizeof(T), cudaMemcpyDeviceToDevice, s));   // own snapshot
        MP_CUDA(cudaStreamSynchronize(s));
        sh->send[rank] = tmp;
        sh->barrier();
        // every rank reduces all snapshots in rank order (identical results on every rank)
        MP_CUDA(cudaMemcpyAsync(buf, sh->send[0], count * sizeof(T), cudaMemcpyDeviceToDevice, s));
        for (int r = 1; r < size; ++r) {
            kern<<<256, 256, 0, s>>>(buf, static_cast<const T *>(sh->send[r]), count);
            MP_LAUNCH_CHECK();
        }
        MP_CUDA(cudaStreamSynchronize(s));
        sh->barrier();
        MP_CUDA(cudaFree(tmp));
    }
    void allreduce_sum(double *buf, size_t count, cudaStream_t s) override { allreduce(buf, count, s, sum_into_kernel); }
    void allreduce_max(int32_t *buf, size_t count, cudaStream_t s) override
    {
        allreduce(buf, count, s, max_into_kernel);
    }
    void allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) override
    {
        MP_CUDA(cudaStreamSynchronize(s));
        sh->send[rank] = send;
        sh->barrier();
        for (int r = 0; r < size; ++r) {
            char *dst = static_cast<char *>(recv) + (size_t)r * bytes;
            if (dst != sh->send[r])                  // in place (NCCL's convention): own chunk already there
                MP_CUDA(cudaMemcpyAsync(dst, sh->send[r], bytes, cudaMemcpyDeviceToDevice, s));
        }
        MP_CUDA(cudaStreamSynchronize(s));
        sh->barrier();
    }
};

}  // namespace

bool nccl_available() { return nccl().ok; }

void nccl_unique_id(char id[128])
{
    if (!nccl().ok) throw CommError{"libnccl.so.2 not found (set MP_NCCL_LIB)"};
    ncclUniqueId u;
    nccl_check(nccl().getUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, 128);
}

Comm *make_nccl_comm(int nranks, int rank, const char id[128])
{
    if (!nccl().ok) throw CommError{"libnccl.so.2 not found (set MP_NCCL_LIB)"};
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    auto c = std::make_unique<NcclComm>();
    c->rank = rank;
    c->size = nranks;
    nccl_check(nccl().commInitRank(&c->c, nranks, u, rank), "ncclCommInitRank");
    return c.release();
}

void make_loopback_comms(int nranks, Comm **out)
{
    auto sh = std::make_shared<LoopbackShared>(nranks);
    for (int r = 0; r < nranks; ++r) {
        auto *c = new LoopbackComm();
        c->rank = r;
        c->size = nranks;
        c->sh = sh;
        c->shared_device = true;
        out[r] = c;
    }
}

}  // namespace mp
