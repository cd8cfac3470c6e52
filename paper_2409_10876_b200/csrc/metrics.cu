// Image-quality metrics of the evaluation harness:
//   psnr            evaluate.hpp:39-51
//   ssim            evaluate.hpp:53-96 (11x11 Gaussian window, sigma 1.5,
//                   K1 = 0.01, K2 = 0.03, averaged where the window fits)
//   sos_rmse_masked evaluate.hpp:99-114
// Inputs are device fp64 rasters [H][W] (the reference's RasterGrid values);
// every sum is fp64, reduced per block and then over blocks in a fixed order
// (deterministic).  Each entry point is synchronous and returns the value on
// the host, like the reference functions.
#include <cmath>

#include "common.cuh"
#include "siren.cuh"  // masked_pixels

namespace pactgpu {
namespace {

constexpr int RB = 256;

// Fixed-order block sum of two fp64 values; thread 0 writes them.
__device__ __forceinline__ void block_sum2(double a, double b, double* out2) {
  __shared__ double s[2][RB / 32];
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = a;
    s[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int w = 0; w < RB / 32; ++w) {
      x += s[0][w];
      y += s[1][w];
    }
    out2[0] = x;
    out2[1] = y;
  }
}

__global__ void __launch_bounds__(RB) sq_diff_kernel(const double* __restrict__ a,
                                                     const double* __restrict__ b, size_t n,
                                                     double* __restrict__ part) {
  double acc = 0.0;
  for (size_t i = blockIdx.x * static_cast<size_t>(RB) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * RB) {
    const double d = a[i] - b[i];
    acc += d * d;
  }
  block_sum2(acc, 0.0, part + 2 * blockIdx.x);
}

struct SsimArgs {
  const double* x;  // test
  const double* y;  // truth
  int W, H;
  double c1, c2;
  double k[11];  // normalised 1-D Gaussian
};

// One thread per pixel whose 11x11 window fits entirely.
__global__ void __launch_bounds__(RB) ssim_kernel(SsimArgs a, double* __restrict__ part) {
  const int hw = 5, vw = a.W - 2 * hw, vh = a.H - 2 * hw;
  const int i = blockIdx.x * RB + threadIdx.x;
  double val = 0.0, cnt = 0.0;
  if (i < vw * vh) {
    const int iy = hw + i / vw, ix = hw + i % vw;
    double mx = 0, my = 0, mxx = 0, myy = 0, mxy = 0;
    for (int dy = -hw; dy <= hw; ++dy) {
      const double* rx = a.x + static_cast<size_t>(iy + dy) * a.W + ix;
      const double* ry = a.y + static_cast<size_t>(iy + dy) * a.W + ix;
#pragma unroll
      for (int dx = -hw; dx <= hw; ++dx) {
        const double w = a.k[dy + hw] * a.k[dx + hw];
        const double p = rx[dx], q = ry[dx];
        mx += w * p;
        my += w * q;
        mxx += w * p * p;
        myy += w * q * q;
        mxy += w * p * q;
      }
    }
    const double vx = mxx - mx * mx, vy = myy - my * my, cxy = mxy - mx * my;
    val = ((2 * mx * my + a.c1) * (2 * cxy + a.c2)) /
          ((mx * mx + my * my + a.c1) * (vx + vy + a.c2));
    cnt = 1.0;
  }
  block_sum2(val, cnt, part + 2 * blockIdx.x);
}

// Squared SOS error over the masked pixels (the list of masked_pixels, which
// applies CircularMask::contains to GridSpec::world with std::hypot on the
// host exactly like the reference, core.hpp:71, 179).
__global__ void __launch_bounds__(RB) masked_sq_kernel(const double* __restrict__ a,
                                                       const double* __restrict__ b,
                                                       const int* __restrict__ idx, int n,
                                                       double* __restrict__ part) {
  const int i = blockIdx.x * RB + threadIdx.x;
  double acc = 0.0;
  if (i < n) {
    const double d = a[idx[i]] - b[idx[i]];
    acc = d * d;
  }
  block_sum2(acc, 0.0, part + 2 * blockIdx.x);
}

// Fixed-order sum over the block partials (one block), result to out2[0..1].
__global__ void __launch_bounds__(RB) fold_kernel(const double* __restrict__ part, int n,
                                                  double* __restrict__ out2) {
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < n; i += RB) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  block_sum2(a, b, out2);
}

// Runs `launch(part)` over `blocks` blocks, folds, returns the two sums.
template <class F>
Status reduce2(pact_ctx* ctx, int blocks, F launch, double* host2) {
  void* buf = nullptr;
  PACT_TRY_S(scratch_get(ctx, kScratchGeneric2, sizeof(double) * 2 * (blocks + 1), &buf));
  double* part = static_cast<double*>(buf);
  launch(part);
  PACT_TRY_S(after_launch(ctx, "metric kernel"));
  fold_kernel<<<1, RB, 0, ctx->stream>>>(part, blocks, part + 2 * blocks);
  PACT_TRY_S(after_launch(ctx, "fold_kernel"));
  PACT_CUDA_S(cudaMemcpyAsync(host2, part + 2 * blocks, sizeof(double) * 2, cudaMemcpyDeviceToHost,
                              ctx->stream));
  PACT_CUDA_S(cudaStreamSynchronize(ctx->stream));
  return {};
}

}  // namespace
}  // namespace pactgpu

using namespace pactgpu;

extern "C" int pact_psnr(pact_ctx* ctx, const double* test, const double* truth, int32_t width,
                         int32_t height, double data_range, double* out) {
  if (!ctx || !test || !truth || !out) return validation("pact_psnr: null argument").code;
  if (!(data_range > 0.0)) return validation("psnr: data_range must be > 0").code;
  const size_t n = static_cast<size_t>(width) * height;
  if (n == 0) return validation("psnr: empty image").code;
  const int blocks = static_cast<int>(std::min<size_t>((n + RB - 1) / RB, 4 * ctx->num_sms));
  double s[2];
  PACT_TRY(reduce2(ctx, blocks, [&](double* part) {
    sq_diff_kernel<<<blocks, RB, 0, ctx->stream>>>(test, truth, n, part);
  }, s));
  const double mse = s[0] / static_cast<double>(n);
  *out = mse == 0.0 ? INFINITY : 10.0 * std::log10(data_range * data_range / mse);
  return PACT_OK;
}

extern "C" int pact_ssim(pact_ctx* ctx, const double* test, const double* truth, int32_t width,
                         int32_t height, double data_range, double* out) {
  if (!ctx || !test || !truth || !out) return validation("pact_ssim: null argument").code;
  if (!(data_range > 0.0)) return validation("ssim: data_range must be > 0").code;
  if (width < 11 || height < 11) return validation("ssim: images must be at least 11x11").code;
  SsimArgs a{};
  a.x = test;
  a.y = truth;
  a.W = width;
  a.H = height;
  a.c1 = (0.01 * data_range) * (0.01 * data_range);
  a.c2 = (0.03 * data_range) * (0.03 * data_range);
  double ksum = 0.0;
  for (int i = 0; i < 11; ++i) {
    const double d = i - 5.0;
    a.k[i] = std::exp(-0.5 * d * d / (1.5 * 1.5));
    ksum += a.k[i];
  }
  for (double& k : a.k) k /= ksum;
  const int valid = (width - 10) * (height - 10);
  const int blocks = div_up(valid, RB);
  double s[2];
  PACT_TRY(reduce2(ctx, blocks, [&](double* part) {
    ssim_kernel<<<blocks, RB, 0, ctx->stream>>>(a, part);
  }, s));
  *out = s[0] / s[1];
  return PACT_OK;
}

extern "C" int pact_sos_rmse_masked(pact_ctx* ctx, const double* test, const double* truth,
                                    const pact_grid* grid, const pact_mask* mask, double* out) {
  if (!ctx || !test || !truth || !grid || !mask || !out)
    return validation("pact_sos_rmse_masked: null argument").code;
  const MaskedPixels mp = masked_pixels(*grid, *mask);
  if (mp.n == 0) return validation("sos_rmse: mask covers no pixels").code;
  void* didx = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric3, sizeof(int) * mp.n, &didx));
  PACT_CUDA(cudaMemcpyAsync(didx, mp.idx.data(), sizeof(int) * mp.n, cudaMemcpyHostToDevice,
                            ctx->stream));
  const int blocks = div_up(mp.n, RB);
  double s[2];
  PACT_TRY(reduce2(ctx, blocks, [&](double* part) {
    masked_sq_kernel<<<blocks, RB, 0, ctx->stream>>>(test, truth, static_cast<const int*>(didx),
                                                     mp.n, part);
  }, s));
  s[1] = mp.n;
  *out = std::sqrt(s[0] / s[1]);
  return PACT_OK;
}
