// comm.cu — population sharding across GPUs: the NCCL
// communicator the C ABI owns, and the sharded generation built on it.
//
// The reference spreads one generation's evaluations over CPU threads with
// parallel_for (evolution.hpp:237-241, parallel.hpp:17-51) and is bitwise
// thread-count invariant (test_evolution.cpp:196-215).  Here each GPU holds
// the replicated GA state (genomes, fitness, RNG: a few GB at P = 65536 of
// 180 GB) and evaluates a strided shard of the children; the ONE exchange per
// generation is a sum all-reduce of the exchange buffer
// [fitness P | spring updates P | material histogram cells x 5] on the
// context stream (evo.cu fills it with zeros outside the rank's shard, so the
// sum is exact and rank-count invariant).  Breeding is replicated, so no
// genome ever crosses NVLink.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): the library carries
// no link-time NCCL dependency, shares the process's NCCL when PyTorch has
// already loaded one, and only vx_comm_* calls need it to exist.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "vx_internal.cuh"

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // an NCCL already in the process (e.g. PyTorch's) wins; else $VX_NCCL_LIBRARY, else the system one.
        // (Loading the system copy first would make a later PyTorch import bind to it.)
        void* h = nullptr;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
            if (h) break;
        }
        if (!h && std::getenv("VX_NCCL_LIBRARY")) h = dlopen(std::getenv("VX_NCCL_LIBRARY"), RTLD_NOW);
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            if (h) break;
            h = dlopen(name, RTLD_NOW);
        }
        if (!h) {
            api.why = std::string("NCCL not loadable: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            return fn != nullptr;
        };
        api.ok = sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
                 sym(api.CommInitAll, "ncclCommInitAll") && sym(api.CommDestroy, "ncclCommDestroy") &&
                 sym(api.AllReduce, "ncclAllReduce") && sym(api.GroupStart, "ncclGroupStart") &&
                 sym(api.GroupEnd, "ncclGroupEnd") && sym(api.GetErrorString, "ncclGetErrorString");
        if (!api.ok) api.why = "NCCL library lacks a required symbol";
    });
    return api;
}

vx_status nccl_status(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return VX_OK;
    vx::set_error(std::string(what) + ": " + nccl().GetErrorString(r));
    return VX_ENCCL;
}

#define VX_NCCL(call)                                           \
    do {                                                        \
        ncclResult_t _r = (call);                               \
        if (_r != ncclSuccess) return nccl_status(_r, #call);   \
    } while (0)

vx_status need_nccl() {
    if (nccl().ok) return VX_OK;
    vx::set_error(nccl().why);
    return VX_ENCCL;
}

}  // namespace

struct vx_comm {
    vx_ctx* ctx = nullptr;
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    ~vx_comm() {
        if (comm && nccl().ok) nccl().CommDestroy(comm);
    }
};

extern "C" {

vx_status vx_comm_available(void) { return need_nccl(); }

vx_status vx_comm_unique_id(uint8_t id[VX_COMM_ID_BYTES]) {
    if (!id) return VX_EINVAL;
    static_assert(sizeof(ncclUniqueId) == VX_COMM_ID_BYTES, "ncclUniqueId size");
    VX_TRY(need_nccl());
    ncclUniqueId u;
    VX_NCCL(nccl().GetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
    return VX_OK;
}

vx_status vx_comm_create(vx_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[VX_COMM_ID_BYTES],
                         vx_comm** out) {
    if (!ctx || !id || !out || world < 1 || rank < 0 || rank >= world) return VX_EINVAL;
    VX_TRY(need_nccl());
    VX_CUDA(cudaSetDevice(ctx->device));
    auto c = std::make_unique<vx_comm>();
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    VX_NCCL(nccl().CommInitRank(&c->comm, world, u, rank));
    c->ctx = ctx;
    c->rank = rank;
    c->world = world;
    *out = c.release();
    return VX_OK;
}

vx_status vx_comm_create_all(int32_t n, vx_ctx* const* ctxs, vx_comm** comms) {
    if (n < 1 || !ctxs || !comms) return VX_EINVAL;
    VX_TRY(need_nccl());
    std::vector<int> devs(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        if (!ctxs[i]) return VX_EINVAL;
        devs[static_cast<size_t>(i)] = ctxs[i]->device;
    }
    std::vector<ncclComm_t> raw(static_cast<size_t>(n));
    VX_NCCL(nccl().CommInitAll(raw.data(), n, devs.data()));
    for (int i = 0; i < n; ++i) {
        comms[i] = new vx_comm;
        comms[i]->ctx = ctxs[i];
        comms[i]->comm = raw[static_cast<size_t>(i)];
        comms[i]->rank = i;
        comms[i]->world = n;
    }
    return VX_OK;
}

vx_status vx_comm_destroy(vx_comm* c) {
    delete c;
    return VX_OK;
}

vx_status vx_comm_rank(const vx_comm* c, int32_t* rank, int32_t* world) {
    if (!c) return VX_EINVAL;
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    return VX_OK;
}

vx_status vx_comm_allreduce_sum_dev(vx_comm* c, double* d_buf, int64_t n) {
    if (!c || (!d_buf && n > 0) || n < 0) return VX_EINVAL;
    if (n == 0) return VX_OK;
    VX_NCCL(nccl().AllReduce(d_buf, d_buf, static_cast<size_t>(n), ncclFloat64, ncclSum, c->comm, c->ctx->stream));
    return VX_OK;
}

}  // extern "C"

namespace vx {

// the exchange step of a sharded generation (evo.cu): sum all-reduce of the
// exchange buffer on the communicator's stream (= the evo's context stream)
vx_status comm_exchange(vx_comm* c, double* d_buf, int64_t n) { return vx_comm_allreduce_sum_dev(c, d_buf, n); }

// several communicators of one vx_comm_create_all, driven by one host thread
vx_status comm_exchange_group(int n, vx_comm* const* cs, double* const* bufs, const int64_t* counts) {
    VX_TRY(need_nccl());
    VX_NCCL(nccl().GroupStart());
    for (int i = 0; i < n; ++i) {
        const ncclResult_t r = nccl().AllReduce(bufs[i], bufs[i], static_cast<size_t>(counts[i]), ncclFloat64, ncclSum,
                                                cs[i]->comm, cs[i]->ctx->stream);
        if (r != ncclSuccess) {
            nccl().GroupEnd();
            return nccl_status(r, "ncclAllReduce");
        }
    }
    VX_NCCL(nccl().GroupEnd());
    return VX_OK;
}

int comm_rank(const vx_comm* c) { return c->rank; }
int comm_world(const vx_comm* c) { return c->world; }
vx_ctx* comm_ctx(const vx_comm* c) { return c->ctx; }

}  // namespace vx
