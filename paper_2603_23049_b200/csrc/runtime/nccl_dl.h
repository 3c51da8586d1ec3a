// Run-time binding of the few NCCL entry points the output all-gather needs (dlopen of
// libnccl.so.2; the process's already-loaded copy — e.g. torch's — is reused when present).
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

namespace pcr {

struct NcclApi {
  // Mirrors of nccl.h types (ABI-stable since NCCL 2.0): ncclResult_t = int,
  // ncclUniqueId = 128 bytes, ncclComm_t = opaque pointer, ncclInt8 = 0.
  using Comm = void*;
  struct UniqueId { char internal[128]; };
  int (*get_unique_id)(UniqueId*) = nullptr;
  int (*comm_init_rank)(Comm*, int, UniqueId, int) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, Comm, cudaStream_t) = nullptr;
  int (*comm_destroy)(Comm) = nullptr;
  const char* (*get_error_string)(int) = nullptr;
};

// nullptr if NCCL cannot be loaded.
const NcclApi* nccl_api();

}  // namespace pcr
