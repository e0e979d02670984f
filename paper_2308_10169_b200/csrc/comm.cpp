// comm.cpp -- NCCL for the sharded large swarm (BASELINE config 4).
//
// libnccl is opened at run time: if the process already loaded one (e.g.
// torch's), that instance is reused (RTLD_NOLOAD), otherwise the system
// libnccl.so.2.  The only collective is one all-gather of each rank's
// population-best candidate per iteration (runner.hpp:88-91 over shards).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "host_runtime.hpp"

namespace sepso {

namespace {
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool load() {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        get_unique_id = reinterpret_cast<decltype(get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        comm_init_rank = reinterpret_cast<decltype(comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        all_gather = reinterpret_cast<decltype(all_gather)>(dlsym(h, "ncclAllGather"));
        comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        error_string = reinterpret_cast<decltype(error_string)>(dlsym(h, "ncclGetErrorString"));
        return get_unique_id && comm_init_rank && all_gather && comm_destroy;
    }
};
Nccl& nccl() {
    static Nccl n;
    return n;
}
int nccl_fail(ncclResult_t r, const char* where) {
    const char* msg = nccl().error_string ? nccl().error_string(r) : "unknown";
    return fail(SF_CUDA_ERROR, std::string(where) + ": " + msg);
}
} // namespace

int comm_unique_id(unsigned char id[128]) {
    if (!nccl().load()) return fail(SF_UNSUPPORTED, "libnccl.so.2 not available");
    ncclUniqueId u;
    const ncclResult_t r = nccl().get_unique_id(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id, u.internal, 128);
    return SF_OK;
}

int comm_init(void** comm, const unsigned char id[128], int nranks, int rank) {
    if (!nccl().load()) return fail(SF_UNSUPPORTED, "libnccl.so.2 not available");
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    ncclComm_t c = nullptr;
    const ncclResult_t r = nccl().comm_init_rank(&c, nranks, u, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *comm = c;
    return SF_OK;
}

int comm_allgather(void* comm, const void* send, void* recv, size_t bytes, cudaStream_t st) {
    const ncclResult_t r =
        nccl().all_gather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(comm), st);
    return r == ncclSuccess ? 0 : 1;
}

int exchange_allgather(sf_ctx* ctx, const void* send, void* recv, size_t bytes) {
    if (ctx->nranks <= 1) {
        std::memcpy(recv, send, bytes);
        return SF_OK;
    }
    if (ctx->xfn) {
        const int r = ctx->xfn(ctx->xuser, send, recv, bytes);
        return r == 0 ? SF_OK : fail(SF_RUNTIME_ERROR, "host all-gather callback failed");
    }
    if (!ctx->comm) return fail(SF_INVALID_ARGUMENT, "sharded run without an exchange");
    unsigned char* d = nullptr;
    cudaError_t e = cudaMalloc(&d, bytes * size_t(ctx->nranks + 1));
    if (e != cudaSuccess) return cuda_fail(e, "exchange staging");
    e = cudaMemcpyAsync(d, send, bytes, cudaMemcpyHostToDevice, ctx->stream);
    int st = e == cudaSuccess ? comm_allgather(ctx->comm, d, d + bytes, bytes, ctx->stream) : 1;
    if (st == 0) e = cudaMemcpyAsync(recv, d + bytes, bytes * size_t(ctx->nranks), cudaMemcpyDeviceToHost, ctx->stream);
    if (st == 0 && e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d);
    if (st) return fail(SF_CUDA_ERROR, "ncclAllGather failed");
    return e == cudaSuccess ? SF_OK : cuda_fail(e, "exchange");
}

void comm_destroy(void* comm) {
    if (comm && nccl().comm_destroy) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

} // namespace sepso
