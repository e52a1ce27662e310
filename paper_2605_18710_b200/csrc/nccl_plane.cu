// nccl_plane.cu — the multi-GPU data plane inside the library: a NCCL communicator built from a
// unique id the caller distributes (mosaic_gpu_nccl_id / mosaic_gpu_set_shard_nccl), and one
// ncclAllGather of the launch's RankRecords per batched launch on the engine's stream.  NCCL is
// resolved at run time (dlopen of libnccl.so.2 — inside a PyTorch process that is the NCCL
// torch already loaded), so the library has no link-time NCCL dependency and a C/C++ caller of
// the ABI gets multi-GPU search without any callback.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "engine.hpp"

namespace mg {

namespace {
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.h = h;
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!api.h || !api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.comm_destroy)
        throw std::runtime_error("NCCL (libnccl.so.2) not available");
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        NcclApi& a = nccl();
        throw std::runtime_error(std::string("NCCL: ") + (a.error_string ? a.error_string(r) : "error") +
                                 " at " + what);
    }
}
}  // namespace

size_t nccl_id_bytes() { return sizeof(ncclUniqueId); }

void nccl_unique_id(void* out) {
    ncclUniqueId id;
    nck(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof id);
}

void Engine::set_shard_nccl(int rank, int world, const void* id) {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank / world");
    if (cudaSetDevice(device_) != cudaSuccess) throw std::runtime_error("cudaSetDevice");
    free_nccl();
    unlink_peers();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclComm_t comm = nullptr;
    nck(nccl().comm_init_rank(&comm, world, uid, rank), "ncclCommInitRank");
    nccl_comm_ = comm;
    rank_ = rank;
    world_ = world;
    ag_ = nullptr;
    ag_user_ = nullptr;
}

void Engine::free_nccl() {
    if (nccl_comm_) nccl().comm_destroy(static_cast<ncclComm_t>(nccl_comm_));
    nccl_comm_ = nullptr;
    cudaFree(d_rec_);
    d_rec_ = nullptr;
    rec_cap_ = 0;
}

// all-gather of `bytes` per rank through the library's communicator: host records in, every
// rank's records out (rank r's at recv + r * bytes), on the engine stream
void Engine::nccl_allgather(const void* send, void* recv, size_t bytes) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
    const size_t need = bytes * (size_t)(world_ + 1);
    if (rec_cap_ < need) {
        cudaFree(d_rec_);
        d_rec_ = nullptr;
        if (cudaMalloc(&d_rec_, need) != cudaSuccess) throw std::runtime_error("cudaMalloc records");
        rec_cap_ = need;
    }
    char* d = static_cast<char*>(d_rec_);
    if (cudaMemcpyAsync(d, send, bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
        throw std::runtime_error("record upload");
    nck(nccl().all_gather(d, d + bytes, bytes, ncclChar, static_cast<ncclComm_t>(nccl_comm_), s),
        "ncclAllGather");
    if (cudaMemcpyAsync(recv, d + bytes, bytes * world_, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        throw std::runtime_error("record read-back");
    if (cudaStreamSynchronize(s) != cudaSuccess) throw std::runtime_error("all-gather sync");
}

}  // namespace mg
