// comm.h -- NCCL loaded at run time (dlopen of libnccl.so.2), so the library has no link
// dependency on a particular NCCL build; it uses the one the process (torch) already has.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace rbg {

bool nccl_available(const char **why);
int nccl_get_unique_id(uint8_t out[128], const char **msg);
int nccl_init(void **comm, int world, int rank, const uint8_t id[128], const char **msg);
int nccl_allgather_bytes(const void *send, void *recv, size_t bytes, void *comm, cudaStream_t s,
                         const char **msg);
void nccl_destroy(void *comm);

}  // namespace rbg
