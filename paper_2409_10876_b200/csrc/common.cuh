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

// Stream-ordered device memory from the device's default pool, whose release
// threshold is raised on first use: buffers freed by one trainer / entry point
// are reused by the next without cudaMalloc / cudaFree (which synchronise the
// device and, for GB-sized arenas, can stall for many milliseconds).
Status pool_alloc(void** ptr, size_t bytes, cudaStream_t stream);
void pool_free(void* ptr, cudaStream_t stream);

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
