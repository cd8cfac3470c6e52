// Small per-step kernels of the training loop: anisotropic TV and its
// subgradient, loss/flag reduction, gradient finiteness check and Adam.
//
//   tv_loss     optimize.hpp:120-153
//   adam_step   optimize.hpp:87-110
//   finiteness  optimize.hpp:414-417, 444-451, 462-465 (NumericalError)
#include <cmath>

#include "common.cuh"
#include "train_ops.cuh"

namespace pactgpu {
namespace {

__device__ __forceinline__ float sgnf(float x) { return x > 0.f ? 1.f : (x < 0.f ? -1.f : 0.f); }

// Gather-form TV over masked pixels (row-major masked order):
//   value += |v[p+1]-v[p]| + |v[p+W]-v[p]|   for pairs with both pixels in the mask
//   grad[i] = lambda (sgn(v[p]-v[p-1]) + sgn(v[p]-v[p-W]) - sgn(v[p+1]-v[p]) - sgn(v[p+W]-v[p]))
// over the valid pairs.  The raster may hold v or v - v0 (differences agree).
__global__ void tv_kernel(const float* __restrict__ v, const unsigned char* __restrict__ inmask,
                          const int* __restrict__ idx, int n, int W, int H, float lambda,
                          float* __restrict__ grad, double* __restrict__ partial) {
  __shared__ double s_red[32];
  double val = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int p = idx[i];
    int iy = p / W, ix = p - iy * W;
    float c = v[p];
    float g = 0.f;
    if (ix + 1 < W && inmask[p + 1]) {
      float d = v[p + 1] - c;
      val += fabsf(d);
      g -= sgnf(d);
    }
    if (iy + 1 < H && inmask[p + W]) {
      float d = v[p + W] - c;
      val += fabsf(d);
      g -= sgnf(d);
    }
    if (ix > 0 && inmask[p - 1]) g += sgnf(c - v[p - 1]);
    if (iy > 0 && inmask[p - W]) g += sgnf(c - v[p - W]);
    grad[i] = lambda * g;
  }
  for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = val;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? s_red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
  }
}

// report[0] = data = sum_patch loss; report[1] = tv = lambda * sum partial;
// report[2] = total.  Raises flag bits for non-finite terms.  One block of
// 256: strided partial sums, then a fixed-order fold (deterministic).
__global__ void __launch_bounds__(256) step_report_kernel(const double* __restrict__ loss_patch,
                                                         int n_patches,
                                                         const double* __restrict__ tv_partial,
                                                         int n_tv, double lambda,
                                                         double* __restrict__ report,
                                                         unsigned* __restrict__ flags) {
  __shared__ double s_d[8], s_t[8];
  double d = 0.0, t = 0.0;
  for (int i = threadIdx.x; i < n_patches; i += blockDim.x) d += loss_patch[i];
  for (int i = threadIdx.x; i < n_tv; i += blockDim.x) t += tv_partial[i];
  for (int o = 16; o > 0; o >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, o);
    t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_d[threadIdx.x >> 5] = d;
    s_t[threadIdx.x >> 5] = t;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double data = 0.0, tv = 0.0;
  for (int w = 0; w < 8; ++w) {
    data += s_d[w];
    tv += s_t[w];
  }
  tv *= lambda;
  report[0] = data;
  report[1] = tv;
  report[2] = data + tv;
  unsigned f = 0;
  if (!isfinite(data)) f |= kFlagLoss;
  if (!isfinite(tv)) f |= kFlagTv;
  if (f) atomicOr(flags, f);
}

__global__ void check_finite_f32(const float* __restrict__ x, const int* __restrict__ idx, int n,
                                 unsigned bit, unsigned* __restrict__ flags) {
  bool bad = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float v = idx ? x[idx[i]] : x[i];
    bad |= !isfinite(v);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, bit);
}

__global__ void check_finite_f64(const double* __restrict__ x, int n, unsigned bit,
                                 unsigned* __restrict__ flags) {
  bool bad = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, bit);
}

// Adam with the step counter on the device so the whole step can be a CUDA
// graph.  Skipped entirely once any flag is raised (the reference throws
// before updating).  t is incremented by the first thread of block 0 after
// every block has read it (adam_tick runs first, in its own launch).
__global__ void adam_tick_kernel(const unsigned* __restrict__ flags, long long* __restrict__ t) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && *flags == 0) *t += 1;
}

__global__ void adam_kernel(int n, double* __restrict__ theta, const double* __restrict__ grad,
                            double* __restrict__ m, double* __restrict__ v,
                            const long long* __restrict__ t, double lr, double b1, double b2,
                            double eps, const unsigned* __restrict__ flags,
                            float* __restrict__ theta32) {
  if (*flags != 0) return;
  const double tt = static_cast<double>(*t);
  const double bc1 = 1.0 - pow(b1, tt), bc2 = 1.0 - pow(b2, tt);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double g = grad[i];
    double mi = b1 * m[i] + (1.0 - b1) * g;
    double vi = b2 * v[i] + (1.0 - b2) * g * g;
    m[i] = mi;
    v[i] = vi;
    double th = theta[i] - lr * (mi / bc1) / (sqrt(vi / bc2) + eps);
    theta[i] = th;
    if (theta32) theta32[i] = static_cast<float>(th);
  }
}

}  // namespace

Status launch_tv(pact_ctx* ctx, const float* v, const unsigned char* inmask, const int* idx, int n,
                 int W, int H, double lambda, float* grad, double* partial, int n_blocks) {
  if (n == 0) {
    PACT_CUDA_S(cudaMemsetAsync(partial, 0, sizeof(double) * n_blocks, ctx->stream));
    return {};
  }
  tv_kernel<<<n_blocks, 256, 0, ctx->stream>>>(v, inmask, idx, n, W, H, static_cast<float>(lambda),
                                               grad, partial);
  return after_launch(ctx, "tv_kernel");
}

Status launch_step_report(pact_ctx* ctx, const double* loss_patch, int n_patches,
                          const double* tv_partial, int n_tv, double lambda, double* report,
                          unsigned* flags) {
  step_report_kernel<<<1, 256, 0, ctx->stream>>>(loss_patch, n_patches, tv_partial, n_tv, lambda,
                                                report, flags);
  return after_launch(ctx, "step_report_kernel");
}

Status launch_check_finite_f32(pact_ctx* ctx, const float* x, const int* idx, int n, unsigned bit,
                               unsigned* flags) {
  if (n == 0) return {};
  int blocks = std::min(div_up(n, 256), ctx->num_sms * 4);
  check_finite_f32<<<blocks, 256, 0, ctx->stream>>>(x, idx, n, bit, flags);
  return after_launch(ctx, "check_finite_f32");
}

Status launch_check_finite_f64(pact_ctx* ctx, const double* x, int n, unsigned bit,
                               unsigned* flags) {
  if (n == 0) return {};
  int blocks = std::min(div_up(n, 256), ctx->num_sms * 4);
  check_finite_f64<<<blocks, 256, 0, ctx->stream>>>(x, n, bit, flags);
  return after_launch(ctx, "check_finite_f64");
}

Status launch_adam(pact_ctx* ctx, int n, double* theta, const double* grad, double* m, double* v,
                   long long* t, double lr, double b1, double b2, double eps,
                   const unsigned* flags, float* theta32, bool tick) {
  if (tick) {
    adam_tick_kernel<<<1, 32, 0, ctx->stream>>>(flags, t);
    PACT_TRY_S(after_launch(ctx, "adam_tick_kernel"));
  }
  int blocks = std::min(div_up(n, 256), ctx->num_sms * 4);
  adam_kernel<<<blocks, 256, 0, ctx->stream>>>(n, theta, grad, m, v, t, lr, b1, b2, eps, flags,
                                               theta32);
  return after_launch(ctx, "adam_kernel");
}

}  // namespace pactgpu
