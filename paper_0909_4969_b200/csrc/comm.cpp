// NCCL inside the library for the time-slab sharded sweep: the
// per-mode all-reduce of the partial Y_(n) runs on the library's own stream,
// between its kernels, so the sharded sweep keeps the overlapped stage 1 and
// is captured into the same CUDA graph as the unsharded one (NCCL
// collectives are graph-capturable).
//
// NCCL is bound at run time (dlopen "libnccl.so.2"): inside a process that
// already loaded torch's NCCL the same library (by soname) is reused, so the
// library and torch.distributed never mix two NCCL versions; a plain C++
// caller gets the system NCCL.  The communicator is created from a unique id
// the caller distributes (mach_comm_unique_id on rank 0, any out-of-band
// broadcast, mach_ctx_comm_init on every rank).
#include <dlfcn.h>
#include <nccl.h>

#include <string>

#include "common.cuh"

namespace machb {

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string err;
};

const NcclApi& api() {
    static NcclApi a = [] {
        NcclApi x;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            x.err = e ? e : "libnccl.so.2 not found";
            return x;
        }
        x.get_unique_id = reinterpret_cast<decltype(x.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        x.comm_init_rank = reinterpret_cast<decltype(x.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        x.all_reduce = reinterpret_cast<decltype(x.all_reduce)>(dlsym(h, "ncclAllReduce"));
        x.comm_destroy = reinterpret_cast<decltype(x.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        x.error_string = reinterpret_cast<decltype(x.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!x.get_unique_id || !x.comm_init_rank || !x.all_reduce || !x.comm_destroy) x.err = "incomplete NCCL library";
        return x;
    }();
    if (!a.err.empty()) throw Error(MACH_ERR_NCCL, "NCCL unavailable: " + a.err);
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const NcclApi& a = api();
        throw Error(MACH_ERR_NCCL, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error"));
    }
}

}  // namespace

void comm_unique_id(unsigned char* out) {
    ncclUniqueId id;
    check(api().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == MACH_COMM_ID_BYTES, "NCCL unique id size");
    std::memcpy(out, &id, sizeof(id));
}

void comm_init(Ctx* ctx, int world, int rank, const unsigned char* id_bytes) {
    if (world < 1 || rank < 0 || rank >= world) throw_arg("rank must satisfy 0 <= rank < world");
    if (ctx->comm) comm_destroy(ctx);
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    ncclComm_t c = nullptr;
    check(api().comm_init_rank(&c, world, id, rank), "ncclCommInitRank");
    ctx->comm = c;
    ctx->comm_world = world;
    ctx->comm_rank = rank;
}

void comm_destroy(Ctx* ctx) {
    if (!ctx->comm) return;
    api().comm_destroy(static_cast<ncclComm_t>(ctx->comm));
    ctx->comm = nullptr;
    ctx->comm_world = 1;
    ctx->comm_rank = 0;
}

// in-place sum over the communicator, on the library stream (capturable)
void comm_allreduce_sum(Ctx* ctx, void* buf, std::size_t count, bool f64) {
    if (!ctx->comm) throw Error(MACH_ERR_NCCL, "no communicator on this context (mach_ctx_comm_init)");
    check(api().all_reduce(buf, buf, count, f64 ? ncclDouble : ncclFloat, ncclSum, static_cast<ncclComm_t>(ctx->comm),
                           ctx->stream),
          "ncclAllReduce");
}

}  // namespace machb
