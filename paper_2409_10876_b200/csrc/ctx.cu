// Context, error and memory entry points of include/pact_cuda.h.
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace pactgpu {

static thread_local char g_error[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_error, sizeof(g_error), fmt, ap);
  va_end(ap);
}

Status pool_alloc(void** ptr, size_t bytes, cudaStream_t stream) {
  static std::once_flag once[64];
  int dev = 0;
  PACT_CUDA_S(cudaGetDevice(&dev));
  std::call_once(once[dev & 63], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
  PACT_CUDA_S(cudaMallocAsync(ptr, bytes ? bytes : 1, stream));
  return {};
}

void pool_free(void* ptr, cudaStream_t stream) {
  if (ptr) cudaFreeAsync(ptr, stream);
}

bool is_host_pointer(const void* p) {
  if (!p) return false;
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, p) != cudaSuccess) {
    cudaGetLastError();  // (not a CUDA pointer on old drivers: treat as pageable host)
    return true;
  }
  return pa.type == cudaMemoryTypeHost || pa.type == cudaMemoryTypeUnregistered;
}

Status smem_optin_raw(const void* func, size_t bytes) {
  // (no small-size shortcut: a kernel with static shared memory needs the
  // opt-in even when its dynamic part is <= 48 KB)
  int dev = 0;
  PACT_CUDA_S(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, func}];
  if (have >= bytes) return {};
  PACT_CUDA_S(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(bytes)));
  have = bytes;
  return {};
}

Status scratch_get(pact_ctx* ctx, int slot, size_t bytes, void** out) {
  pact_scratch& s = ctx->scratch[slot];
  if (s.bytes < bytes) {
    // stream-ordered: queued work on ctx->stream still sees the old buffer
    pool_free(s.ptr, ctx->stream);
    s.ptr = nullptr;
    s.bytes = 0;
    size_t want = bytes < 256 ? 256 : bytes;
    PACT_TRY_S(pool_alloc(&s.ptr, want, ctx->stream));
    s.bytes = want;
  }
  *out = s.ptr;
  return {};
}

}  // namespace pactgpu

using namespace pactgpu;

extern "C" {

int pact_abi_version(void) { return PACT_ABI_VERSION; }

const char* pact_last_error(void) { return g_error; }
const char* pact_ctx_last_error(const pact_ctx*) { return g_error; }

int pact_ctx_create(int device, pact_ctx** out) {
  if (!out) return validation("pact_ctx_create: out is null").code;
  *out = nullptr;
  int n = 0;
  PACT_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return validation("pact_ctx_create: no such device").code;
  PACT_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  PACT_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_error("pact_ctx_create: device %d is sm_%d%d; this build targets sm_100a only", device,
              prop.major, prop.minor);
    return PACT_E_UNSUPPORTED;
  }
  auto* ctx = new pact_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return cuda_status(e, "cudaStreamCreateWithFlags").code;
  }
  ctx->stream = ctx->own_stream;
  *out = ctx;
  return PACT_OK;
}

int pact_ctx_destroy(pact_ctx* ctx) {
  if (!ctx) return PACT_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->api && ctx->api_free) ctx->api_free(ctx->api);
  if (ctx->rays && ctx->rays_free) ctx->rays_free(ctx->rays);
  for (int i = 0; i < 4; ++i)
    if (ctx->ext[i] && ctx->ext_free[i]) ctx->ext_free[i](ctx->ext[i]);
  for (auto& s : ctx->scratch) pool_free(s.ptr, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return PACT_OK;
}

void* pact_ctx_stream(pact_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int pact_ctx_set_stream(pact_ctx* ctx, void* stream) {
  if (!ctx) return validation("pact_ctx_set_stream: null context").code;
  ctx->stream = (cudaStream_t)stream;
  return PACT_OK;
}

int pact_ctx_use_own_stream(pact_ctx* ctx) {
  if (!ctx) return validation("pact_ctx_use_own_stream: null context").code;
  ctx->stream = ctx->own_stream;
  return PACT_OK;
}

int pact_ctx_synchronize(pact_ctx* ctx) {
  if (!ctx) return validation("pact_ctx_synchronize: null context").code;
  PACT_CUDA(cudaStreamSynchronize(ctx->stream));
  return PACT_OK;
}

int64_t pact_ctx_launch_count(pact_ctx* ctx) { return ctx ? ctx->launches.load() : -1; }

int pact_device_alloc(pact_ctx* ctx, size_t bytes, void** out) {
  if (!ctx || !out) return validation("pact_device_alloc: null argument").code;
  PACT_CUDA(cudaSetDevice(ctx->device));
  PACT_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  return PACT_OK;
}

int pact_device_free(pact_ctx* ctx, void* ptr) {
  if (!ctx) return validation("pact_device_free: null context").code;
  if (ptr) PACT_CUDA(cudaFree(ptr));
  return PACT_OK;
}

int pact_host_alloc_pinned(size_t bytes, void** out) {
  if (!out) return validation("pact_host_alloc_pinned: null argument").code;
  PACT_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
  return PACT_OK;
}

int pact_host_free_pinned(void* ptr) {
  if (ptr) PACT_CUDA(cudaFreeHost(ptr));
  return PACT_OK;
}

int pact_upload(pact_ctx* ctx, void* dst_device, const void* src_host, size_t bytes) {
  if (!ctx) return validation("pact_upload: null context").code;
  if (bytes == 0) return PACT_OK;
  PACT_CUDA(cudaMemcpyAsync(dst_device, src_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return PACT_OK;
}

int pact_download(pact_ctx* ctx, void* dst_host, const void* src_device, size_t bytes) {
  if (!ctx) return validation("pact_download: null context").code;
  if (bytes == 0) return PACT_OK;
  PACT_CUDA(cudaMemcpyAsync(dst_host, src_device, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  PACT_CUDA(cudaStreamSynchronize(ctx->stream));
  return PACT_OK;
}

int pact_memset(pact_ctx* ctx, void* dst_device, int value, size_t bytes) {
  if (!ctx) return validation("pact_memset: null context").code;
  if (bytes == 0) return PACT_OK;
  PACT_CUDA(cudaMemsetAsync(dst_device, value, bytes, ctx->stream));
  return PACT_OK;
}

int pact_make_delays(double lo, double hi, int32_t count, double* out) {
  // beamform.hpp:113-120
  if (count < 1) return validation("delays: count must be >= 1").code;
  if (count > 1 && !(hi > lo)) return validation("delays: need hi > lo for count > 1").code;
  if (!out) return validation("pact_make_delays: out is null").code;
  for (int j = 0; j < count; ++j) out[j] = count == 1 ? lo : lo + (hi - lo) * j / (count - 1);
  return PACT_OK;
}

}  // extern "C"
