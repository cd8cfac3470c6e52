// Run-time bound NCCL entry points (nccl.cu) and the context's communicator.
#pragma once

#include <nccl.h>

#include "common.cuh"

namespace pactgpu {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

// null when libnccl.so.2 cannot be loaded
const NcclApi* nccl_api();
Status nccl_status(int r, const char* what);

struct NcclComm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
};
// the communicator attached to ctx (comm null: none)
NcclComm ctx_nccl(pact_ctx* ctx);

}  // namespace pactgpu
