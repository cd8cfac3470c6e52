// Part 2 (ray half) of the hot path: per-patch wavefront error profiles
// w(theta) by a straight-ray march through the SOS raster, and the adjoint
// scatter of dL/dw back onto the raster.
//
//   wavefront_profile    aberration.hpp:134-186
//   wavefront_grad_trace aberration.hpp:333-361
//
// B200 design: one thread per ray (patch, angle); a warp is 32 consecutive
// angles of one patch so its rays have near-equal lengths.  Ray setup is fp64
// (identical step counts to the reference); positions are fp64 per step and
// the bilinear stencil runs in fp32 on the *deviation* raster dv = v - v0,
// which keeps full relative precision of the integrand
// 1 - v0/v = dv / (v0 + dv).  The SOS raster (<= 16 MB) is L2-resident and
// read through the read-only path.
//
// The backward pass coalesces consecutive steps that share a stencil cell in
// registers (a step is 0.05 mm, a pixel 0.05-0.2 mm, and steps beyond the grid
// clamp onto one border cell for long runs) and flushes with fp64 atomics,
// skipping zero-weight corners; fp64 accumulation makes the result
// reproducible to fp32 output precision regardless of atomic order.
#include "common.cuh"
#include "geom.cuh"

namespace pactgpu {

namespace {

__device__ __forceinline__ float sample_dev(const float* __restrict__ dv, const Stencil& s) {
  return s.w00 * __ldg(dv + s.i00) + s.w01 * __ldg(dv + s.i01) + s.w10 * __ldg(dv + s.i10) +
         s.w11 * __ldg(dv + s.i11);
}

__global__ void __launch_bounds__(256) wavefront_kernel(RayArgs a, float* __restrict__ w) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n_rays) return;
  int patch = r / a.n_angles, ang = r - patch * a.n_angles;
  double2 c = a.centers[patch];
  Ray ray = make_ray(c.x, c.y, ang, a.n_angles, a.ring_r, a.mcx, a.mcy, a.mr, a.step);
  // Pixel coordinates along the ray: f(s) = f0 + s * df  (GridSpec::pixel, core.hpp:75)
  const double fx0 = (c.x - a.ox) * a.inv_pitch, fy0 = (c.y - a.oy) * a.inv_pitch;
  const double dfx = ray.ux * a.inv_pitch, dfy = ray.uy * a.inv_pitch;
  const float v0 = static_cast<float>(a.v0);
  float acc = 0.f;
#pragma unroll 4
  for (int i = 0; i < ray.n; ++i) {
    double s = ray.t0 + (i + 0.5) * ray.dl;
    Stencil st = stencil_at(static_cast<float>(fx0 + s * dfx), static_cast<float>(fy0 + s * dfy),
                            a.W, a.H);
    float d = sample_dev(a.dv, st);
    acc += d / (v0 + d);  // (1 - v0/v), v = v0 + d
  }
  w[r] = static_cast<float>(ray.dl) * acc;
}

__device__ __forceinline__ void flush_cell(double* __restrict__ g, int W, int H, int ix, int iy,
                                           const double acc[4]) {
  int ix1 = min(ix + 1, W - 1), iy1 = min(iy + 1, H - 1);
  if (acc[0] != 0.0) atomicAdd(g + iy * W + ix, acc[0]);
  if (acc[1] != 0.0) atomicAdd(g + iy * W + ix1, acc[1]);
  if (acc[2] != 0.0) atomicAdd(g + iy1 * W + ix, acc[2]);
  if (acc[3] != 0.0) atomicAdd(g + iy1 * W + ix1, acc[3]);
}

__global__ void __launch_bounds__(256) ray_backward_kernel(RayArgs a, const float* __restrict__ dw,
                                                           double* __restrict__ grad) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n_rays) return;
  const float gr = dw[r];
  if (gr == 0.f) return;  // aberration.hpp:340
  int patch = r / a.n_angles, ang = r - patch * a.n_angles;
  double2 c = a.centers[patch];
  Ray ray = make_ray(c.x, c.y, ang, a.n_angles, a.ring_r, a.mcx, a.mcy, a.mr, a.step);
  if (ray.n == 0) return;
  const double fx0 = (c.x - a.ox) * a.inv_pitch, fy0 = (c.y - a.oy) * a.inv_pitch;
  const double dfx = ray.ux * a.inv_pitch, dfy = ray.uy * a.inv_pitch;
  const float v0 = static_cast<float>(a.v0);
  // f = g * dl * v0 / v^2 per step (aberration.hpp:354-355)
  const float gscale = static_cast<float>(static_cast<double>(gr) * ray.dl * a.v0);
  const int W = a.W, H = a.H;
  int cx = -1, cy = -1;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i = 0; i < ray.n; ++i) {
    double s = ray.t0 + (i + 0.5) * ray.dl;
    float fx = fminf(fmaxf(static_cast<float>(fx0 + s * dfx), 0.f), static_cast<float>(W - 1));
    float fy = fminf(fmaxf(static_cast<float>(fy0 + s * dfy), 0.f), static_cast<float>(H - 1));
    int ix = min(static_cast<int>(fx), max(W - 2, 0));
    int iy = min(static_cast<int>(fy), max(H - 2, 0));
    float ax = fx - ix, ay = fy - iy;
    int ix1 = min(ix + 1, W - 1), iy1 = min(iy + 1, H - 1);
    float w00 = (1.f - ax) * (1.f - ay), w01 = ax * (1.f - ay), w10 = (1.f - ax) * ay,
          w11 = ax * ay;
    float d = w00 * __ldg(a.dv + iy * W + ix) + w01 * __ldg(a.dv + iy * W + ix1) +
              w10 * __ldg(a.dv + iy1 * W + ix) + w11 * __ldg(a.dv + iy1 * W + ix1);
    float v = v0 + d;
    float f = gscale / (v * v);
    if (ix != cx || iy != cy) {
      if (cx >= 0) flush_cell(grad, W, H, cx, cy, acc);
      cx = ix;
      cy = iy;
      acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
    }
    acc[0] += f * w00;
    acc[1] += f * w01;
    acc[2] += f * w10;
    acc[3] += f * w11;
  }
  flush_cell(grad, W, H, cx, cy, acc);
}

}  // namespace

Status ray_args(const pact_ring& ring, const pact_grid& grid, double v0, const pact_mask& mask,
                int n_angles, double step, RayArgs& a) {
  if (ring.n_transducers < 3) return validation("ring: need at least 3 transducers");
  if (!(ring.radius > 0.0)) return validation("ring: radius must be > 0");
  if (n_angles < 4) return validation("wavefront_profile: need at least 4 angles");
  if (!(step > 0.0)) return validation("wavefront_profile: step must be > 0");
  if (grid.width < 1 || grid.height < 1) return validation("grid: width and height must be >= 1");
  if (!(grid.pitch > 0.0)) return validation("grid: pitch must be > 0");
  a.W = grid.width;
  a.H = grid.height;
  a.ox = grid.origin_x;
  a.oy = grid.origin_y;
  a.inv_pitch = 1.0 / grid.pitch;
  a.v0 = v0;
  a.ring_r = ring.radius;
  a.mcx = mask.center_x;
  a.mcy = mask.center_y;
  a.mr = mask.radius;
  a.step = step;
  a.n_angles = n_angles;
  return {};
}

Status validate_centers(const pact_ring& ring, int n, const double* centers) {
  for (int i = 0; i < n; ++i)
    if (std::hypot(centers[2 * i], centers[2 * i + 1]) >= ring.radius)
      return validation("wavefront_profile: patch center outside the transducer ring");
  return {};
}

Status launch_wavefront(pact_ctx* ctx, const RayArgs& a, float* w) {
  int blocks = div_up(a.n_rays, 256);
  wavefront_kernel<<<blocks, 256, 0, ctx->stream>>>(a, w);
  return after_launch(ctx, "wavefront_kernel");
}

Status launch_ray_backward(pact_ctx* ctx, const RayArgs& a, const float* dw, double* grad) {
  int blocks = div_up(a.n_rays, 256);
  ray_backward_kernel<<<blocks, 256, 0, ctx->stream>>>(a, dw, grad);
  return after_launch(ctx, "ray_backward_kernel");
}

}  // namespace pactgpu

using namespace pactgpu;

extern "C" int pact_wavefront(pact_ctx* ctx, const pact_ring* ring, const pact_grid* grid,
                              const float* sos_dev, double v0, const pact_mask* mask,
                              int32_t n_centers, const double* centers, int32_t n_angles,
                              double step, float* w) {
  if (!ctx || !ring || !grid || !mask || !centers || !sos_dev || !w)
    return validation("pact_wavefront: null argument").code;
  RayArgs a{};
  PACT_TRY(ray_args(*ring, *grid, v0, *mask, n_angles, step, a));
  PACT_TRY(validate_centers(*ring, n_centers, centers));
  if (n_centers <= 0) return PACT_OK;
  void* dc = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric3, sizeof(double2) * n_centers, &dc));
  PACT_CUDA(cudaMemcpyAsync(dc, centers, sizeof(double2) * n_centers, cudaMemcpyHostToDevice,
                            ctx->stream));
  a.dv = sos_dev;
  a.centers = static_cast<const double2*>(dc);
  a.n_rays = n_centers * n_angles;
  PACT_TRY(launch_wavefront(ctx, a, w));
  return PACT_OK;
}

extern "C" int pact_ray_backward(pact_ctx* ctx, const pact_ring* ring, const pact_grid* grid,
                                 const float* sos_dev, double v0, const pact_mask* mask,
                                 int32_t n_centers, const double* centers, int32_t n_angles,
                                 double step, const float* dw, double* grad_v) {
  if (!ctx || !ring || !grid || !mask || !centers || !sos_dev || !dw || !grad_v)
    return validation("pact_ray_backward: null argument").code;
  RayArgs a{};
  PACT_TRY(ray_args(*ring, *grid, v0, *mask, n_angles, step, a));
  if (n_centers <= 0) return PACT_OK;
  void* dc = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric3, sizeof(double2) * n_centers, &dc));
  PACT_CUDA(cudaMemcpyAsync(dc, centers, sizeof(double2) * n_centers, cudaMemcpyHostToDevice,
                            ctx->stream));
  a.dv = sos_dev;
  a.centers = static_cast<const double2*>(dc);
  a.n_rays = n_centers * n_angles;
  PACT_TRY(launch_ray_backward(ctx, a, dw, grad_v));
  return PACT_OK;
}
