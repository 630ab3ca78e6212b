// nccl_dl.h -- NCCL loaded at run time with dlopen (the library stays loadable where NCCL is
// absent; multi-GPU calls then fail loudly with CIQ_ERR_NCCL).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace ciq {
bool nccl_load();
const char* nccl_error();
bool nccl_unique_id(void* out128);
// Opaque communicator handle.
void* nccl_comm_init(int world, int rank, const void* id128);
void nccl_comm_destroy(void* comm);
// In-place all-gather of `count` elements per rank (float32 = 7, float64 = 8 in ncclDataType_t).
bool nccl_allgather(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t s);
bool nccl_allreduce_sum(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t s);
}  // namespace ciq
