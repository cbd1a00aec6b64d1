// comm.cpp -- the per-iteration exchange of the column-sharded greedy over NCCL.
//
// The paper's parallel code uses MPI_Allreduce for the pivot
// information, MPI_Send of the pivot column to the orthogonalisation core and MPI_Bcast
// of the new basis vector.  Here one ncclAllGather of a fixed-size slot per rank
// (16-byte maxloc record + the rank's candidate column) replaces all three: every rank
// then selects the winner with the same total order and runs IMGS itself, so there is no
// data-dependent root, no host round trip, and the call is CUDA-graph capturable
// (DESIGN.md "Multi-GPU").
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

namespace rbg {
namespace {

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
    const char *err = nullptr;
};

NcclApi &api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!a.h) {
            a.err = "libnccl.so.2 not found (import torch first or set LD_LIBRARY_PATH)";
            return;
        }
        a.getUniqueId = (decltype(a.getUniqueId))dlsym(a.h, "ncclGetUniqueId");
        a.commInitRank = (decltype(a.commInitRank))dlsym(a.h, "ncclCommInitRank");
        a.allGather = (decltype(a.allGather))dlsym(a.h, "ncclAllGather");
        a.commDestroy = (decltype(a.commDestroy))dlsym(a.h, "ncclCommDestroy");
        a.getErrorString = (decltype(a.getErrorString))dlsym(a.h, "ncclGetErrorString");
        if (!a.getUniqueId || !a.commInitRank || !a.allGather || !a.commDestroy)
            a.err = "libnccl.so.2 lacks a required symbol";
    });
    return a;
}

const char *errstr(ncclResult_t r) {
    NcclApi &a = api();
    return a.getErrorString ? a.getErrorString(r) : "nccl error";
}

}  // namespace

bool nccl_available(const char **why) {
    NcclApi &a = api();
    if (a.err) {
        if (why) *why = a.err;
        return false;
    }
    return true;
}

int nccl_get_unique_id(uint8_t out[128], const char **msg) {
    if (!nccl_available(msg)) return 1;
    ncclUniqueId id;
    ncclResult_t r = api().getUniqueId(&id);
    if (r != ncclSuccess) {
        *msg = errstr(r);
        return 1;
    }
    static_assert(sizeof(id.internal) == 128, "ncclUniqueId size");
    for (int i = 0; i < 128; i++) out[i] = (uint8_t)id.internal[i];
    return 0;
}

int nccl_init(void **comm, int world, int rank, const uint8_t idb[128], const char **msg) {
    if (!nccl_available(msg)) return 1;
    ncclUniqueId id;
    for (int i = 0; i < 128; i++) id.internal[i] = (char)idb[i];
    ncclComm_t c = nullptr;
    ncclResult_t r = api().commInitRank(&c, world, id, rank);
    if (r != ncclSuccess) {
        *msg = errstr(r);
        return 1;
    }
    *comm = c;
    return 0;
}

int nccl_allgather_bytes(const void *send, void *recv, size_t bytes, void *comm, cudaStream_t s,
                         const char **msg) {
    ncclResult_t r = api().allGather(send, recv, bytes, ncclUint8, (ncclComm_t)comm, s);
    if (r != ncclSuccess) {
        *msg = errstr(r);
        return 1;
    }
    return 0;
}

void nccl_destroy(void *comm) {
    if (comm && api().commDestroy) api().commDestroy((ncclComm_t)comm);
}

}  // namespace rbg
