// NCCL for the multi-GPU frame in the library itself, so
// a C / C++ caller needs no Python: the context owns the communicator
// (pact_ctx_attach_nccl) and pact_trainer_step_nccl runs a partitioned
// trainer's phases with their collectives (trainer.cu).  NCCL is loaded at run
// time (libnccl.so.2; the one torch already loaded, if any, by soname), so the
// library has no link-time dependency on it.  The declarations come from
// nccl.h; nothing of NCCL is called directly.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "common.cuh"
#include "nccl_api.cuh"

namespace pactgpu {

namespace {
NcclApi g_api;
bool g_api_ok = false;
std::once_flag g_api_once;

template <class F>
bool sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  return f != nullptr;
}

struct NcclSlot {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  ~NcclSlot() {
    if (comm && g_api_ok) g_api.comm_destroy(comm);
  }
};
}  // namespace

const NcclApi* nccl_api() {
  std::call_once(g_api_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_api_ok = sym(h, "ncclGetUniqueId", g_api.get_unique_id) &&
               sym(h, "ncclCommInitRank", g_api.comm_init_rank) &&
               sym(h, "ncclCommDestroy", g_api.comm_destroy) &&
               sym(h, "ncclAllReduce", g_api.all_reduce) &&
               sym(h, "ncclAllGather", g_api.all_gather) &&
               sym(h, "ncclReduceScatter", g_api.reduce_scatter) &&
               sym(h, "ncclGetErrorString", g_api.error_string);
  });
  return g_api_ok ? &g_api : nullptr;
}

Status nccl_status(int r, const char* what) {
  if (r == ncclSuccess) return {};
  const NcclApi* api = nccl_api();
  set_error("%s: %s", what, api ? api->error_string(static_cast<ncclResult_t>(r)) : "NCCL unavailable");
  return {PACT_E_CUDA};
}

NcclComm ctx_nccl(pact_ctx* ctx) {
  if (!ctx || !ctx->ext[kExtNccl]) return {};
  auto* s = static_cast<NcclSlot*>(ctx->ext[kExtNccl]);
  return {s->comm, s->rank, s->world};
}

}  // namespace pactgpu

using namespace pactgpu;

extern "C" int pact_nccl_unique_id(unsigned char* id) {
  if (!id) return validation("pact_nccl_unique_id: null argument").code;
  const NcclApi* api = nccl_api();
  if (!api) return internal_error("pact_nccl_unique_id: libnccl.so.2 could not be loaded").code;
  ncclUniqueId u;
  PACT_TRY(nccl_status(api->get_unique_id(&u), "ncclGetUniqueId"));
  static_assert(sizeof(u.internal) == PACT_NCCL_ID_BYTES, "NCCL unique id size");
  std::memcpy(id, u.internal, PACT_NCCL_ID_BYTES);
  return PACT_OK;
}

extern "C" int pact_ctx_attach_nccl(pact_ctx* ctx, const unsigned char* id, int32_t rank,
                                    int32_t world) {
  if (!ctx || !id) return validation("pact_ctx_attach_nccl: null argument").code;
  if (world < 1 || rank < 0 || rank >= world)
    return validation("pact_ctx_attach_nccl: need 0 <= rank < world").code;
  const NcclApi* api = nccl_api();
  if (!api) return internal_error("pact_ctx_attach_nccl: libnccl.so.2 could not be loaded").code;
  PACT_CUDA(cudaSetDevice(ctx->device));
  auto* slot = ctx_ext<NcclSlot>(ctx, kExtNccl);
  if (slot->comm) {
    api->comm_destroy(slot->comm);
    slot->comm = nullptr;
  }
  ncclUniqueId u;
  std::memcpy(u.internal, id, PACT_NCCL_ID_BYTES);
  PACT_TRY(nccl_status(api->comm_init_rank(&slot->comm, world, u, rank), "ncclCommInitRank"));
  slot->rank = rank;
  slot->world = world;
  return PACT_OK;
}
