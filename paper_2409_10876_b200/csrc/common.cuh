// Shared plumbing for the sm_100a kernels behind include/pact_cuda.h:
// the context object, thread-local error reporting, and launch helpers.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "pact_cuda.h"

namespace pactgpu {

constexpr int kNumSMs = 148;  // B200; the context re-reads the real count

void set_error(const char* fmt, ...);

// Error-carrying status used inside the library; converted to the ABI code at
// the boundary.  `code` is one of PACT_E_*.
struct Status {
  int code = PACT_OK;
  bool ok() const { return code == PACT_OK; }
};

inline Status validation(const char* msg) {
  set_error("%s", msg);
  return {PACT_E_VALIDATION};
}

// A broken library invariant (reported as a CUDA-class failure).
inline Status internal_error(const char* msg) {
  set_error("internal: %s", msg);
  return {PACT_E_CUDA};
}

inline Status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return {};
  set_error("%s: %s", what, cudaGetErrorString(e));
  return {PACT_E_CUDA};
}

}  // namespace pactgpu

// Per-context device scratch: grows monotonically, freed with the context.
struct pact_scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
};

struct pact_ctx {
  int device = 0;
  int num_sms = pactgpu::kNumSMs;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::atomic<int64_t> launches{0};
  // Named scratch slots so independent entry points do not alias.
  pact_scratch scratch[16];
  // Per-context caches of the standalone entry points (api.cu).
  void* api = nullptr;
  void (*api_free)(void*) = nullptr;
  // Ray-plan cache of the standalone ray entry points (raymarch.cu).
  void* rays = nullptr;
  void (*rays_free)(void*) = nullptr;
  // Further per-context caches, one slot per owner (pactgpu::ExtSlot).
  void* ext[4] = {nullptr, nullptr, nullptr, nullptr};
  void (*ext_free[4])(void*) = {nullptr, nullptr, nullptr, nullptr};
};

namespace pactgpu {

enum ScratchSlot {
  kScratchDasPartial = 0,
  kScratchDasGeom = 1,
  kScratchGeneric0 = 2,
  kScratchGeneric1 = 3,
  kScratchGeneric2 = 4,
  kScratchGeneric3 = 5,
  kScratchTables = 6,
  kScratchNyq = 7,
  kScratchRayBorder = 8,
};

Status scratch_get(pact_ctx* ctx, int slot, size_t bytes, void** out);

// Per-context cache slots (pact_ctx::ext): created on first use by their
// owner, destroyed with the context.  Keeping them per context keeps them
// per device and per stream (a cache shared across contexts could be
// rewritten while another context's stream still reads it).
enum ExtSlot {
  kExtFourier = 0,   // fourier.cu: the table of pact_transfer_stack / pact_loss_grad
  kExtComposed = 1,  // composed.cu: fp64 bin tables of the composed-path entry points
  kExtNccl = 2,      // nccl.cu: the NCCL communicator of the multi-GPU frame
};

template <class T>
T* ctx_ext(pact_ctx* ctx, int slot) {
  if (!ctx->ext[slot]) {
    ctx->ext[slot] = new T();
    ctx->ext_free[slot] = [](void* p) { delete static_cast<T*>(p); };
  }
  return static_cast<T*>(ctx->ext[slot]);
}

// Stream-ordered device memory from the device's default pool, whose release
// threshold is raised on first use: buffers freed by one trainer / entry point
// are reused by the next without cudaMalloc / cudaFree (which synchronise the
// device and, for GB-sized arenas, can stall for many milliseconds).
// True for host memory (pinned or pageable): the engine entry points stage
// such inputs / outputs themselves.  NULL and device / managed pointers: false.
bool is_host_pointer(const void* p);
Status pool_alloc(void** ptr, size_t bytes, cudaStream_t stream);
void pool_free(void* ptr, cudaStream_t stream);

// Opt a kernel in to `bytes` of dynamic shared memory on the CURRENT device.
// The attribute is per device context, so the bookkeeping is per (device,
// kernel); thread-safe (ctx.cu).
Status smem_optin_raw(const void* func, size_t bytes);
template <class F>
Status smem_optin(F* func, size_t bytes) {
  return smem_optin_raw(reinterpret_cast<const void*>(func), bytes);
}

// After every launch: count it and surface launch-configuration errors.
inline Status after_launch(pact_ctx* ctx, const char* name) {
  ctx->launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError(), name);
}

inline int div_up(int a, int b) { return (a + b - 1) / b; }

}  // namespace pactgpu

#define PACT_TRY(expr)                                   \
  do {                                                   \
    ::pactgpu::Status _st = (expr);                      \
    if (!_st.ok()) return _st.code;                      \
  } while (0)

#define PACT_TRY_S(expr)                                 \
  do {                                                   \
    ::pactgpu::Status _st = (expr);                      \
    if (!_st.ok()) return _st;                           \
  } while (0)

#define PACT_CUDA(expr) PACT_TRY(::pactgpu::cuda_status((expr), #expr))
#define PACT_CUDA_S(expr) PACT_TRY_S(::pactgpu::cuda_status((expr), #expr))
