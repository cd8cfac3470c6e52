// Declarations of the launch helpers shared between the C-ABI entry points and
// the training engine.
#pragma once

#include "common.cuh"
#include "fourier.cuh"

#include <memory>

namespace pactgpu {

// NumericalError stages, in the order joint_reconstruct checks them.
constexpr unsigned kFlagSos = 1u;    // optimize.hpp:414-417
constexpr unsigned kFlagLoss = 2u;   // optimize.hpp:444-446
constexpr unsigned kFlagTv = 4u;     // optimize.hpp:449-451
constexpr unsigned kFlagGrad = 8u;   // optimize.hpp:462-465

struct RayArgs;

Status ray_args(const pact_ring& ring, const pact_grid& grid, double v0, const pact_mask& mask,
                int n_angles, double step, RayArgs& a);
Status validate_centers(const pact_ring& ring, int n, const double* centers);
// Work plan of the texture-path ray kernels for a fixed geometry (raymarch.cu).
// The immutable part (records, schedule) is built once per geometry and
// shared through `cache_ctx`; each owner (trainer, standalone call) holds its
// own forward partials, allocated on ctx's stream.  ray_plan_get fills the
// plan fields of `a` (centers: host copy of a.centers); synchronous on a miss.
struct RayPlanData;
struct RayPlan {
  std::shared_ptr<RayPlanData> data;
  float* partial = nullptr;
};
Status ray_plan_get(pact_ctx* cache_ctx, pact_ctx* ctx, RayArgs& a, const double* centers,
                    int n_centers, RayPlan& out);
void ray_plan_release(RayPlan& p, cudaStream_t s);
// The standalone entry points' plan (one per context, rebuilt on a new geometry).
Status ray_plan_cached(pact_ctx* ctx, RayArgs& a, const double* centers, int n_centers);
Status launch_wavefront(pact_ctx* ctx, const RayArgs& a, float* w);
Status launch_ray_backward(pact_ctx* ctx, const RayArgs& a, const float* dw, double* grad);

Status launch_transfer_stack(pact_ctx* ctx, const FourierTab& t, const float* w, int n_patches,
                             float2* H);
Status launch_loss_grad(pact_ctx* ctx, const FourierTab& t, const float2* Y, const float* w,
                        int n_patches, double eps, double scale, bool implicit, double* loss,
                        float* dw);
Status launch_wiener(pact_ctx* ctx, const FourierTab& t, const float2* Y, const float* w,
                     int n_patches, double eps, float2* X);

// Spectra of the patches [p_lo, p_hi) (p_hi < 0: all), Y indexed from p_lo.
// stack holds the grid rows [row0, row0 + stack_rows) (stack_rows < 0: H - row0)
Status launch_patch_fft(pact_ctx* ctx, const pact_layout& lay, const float* stack, int K,
                        float2* Y, int p_lo = 0, int p_hi = -1, int row0 = 0, int stack_rows = -1);
Status launch_patch_ifft_real(pact_ctx* ctx, int P, int n_patches, const float2* X, float* out);
Status launch_merge(pact_ctx* ctx, const pact_layout& lay, const float* patches, const float* win,
                    float* img);
// Merge accumulators (sum w x, sum w) of the patches [p_lo, p_hi) only.
Status launch_merge_partial(pact_ctx* ctx, const pact_layout& lay, const float* patches,
                            const float* win, int p_lo, int p_hi, float* num, float* den);

Status launch_tv(pact_ctx* ctx, const float* v, const unsigned char* inmask, const int* idx, int n,
                 int W, int H, double lambda, float* grad, double* partial, int n_blocks);
Status launch_step_report(pact_ctx* ctx, const double* loss_patch, int n_patches,
                          const double* tv_partial, int n_tv, double lambda, double* report,
                          unsigned* flags);
Status launch_check_finite_f32(pact_ctx* ctx, const float* x, const int* idx, int n, unsigned bit,
                               unsigned* flags);
Status launch_check_finite_f64(pact_ctx* ctx, const double* x, int n, unsigned bit,
                               unsigned* flags);
Status launch_adam(pact_ctx* ctx, int n, double* theta, const double* grad, double* m, double* v,
                   long long* t, double lr, double b1, double b2, double eps,
                   const unsigned* flags, float* theta32, bool tick);

// das_stack of the rows [row0, row0 + rows) of `grid` (rows < 0: to the
// bottom) into out [K][rows][W]; values are those of the full-grid stack.
Status das_stack_device(pact_ctx* ctx, const pact_ring& ring, const pact_signal_meta& meta,
                        const float* signals, const pact_grid& grid, double v0,
                        const double* delays, int K, float* out, int row0 = 0, int rows = -1);

// make_patch_layout (core.hpp:252-281) on the host; centres in fp64.
Status make_layout(const pact_grid& grid, double patch_mm, double overlap, pact_layout& out);
void layout_centers(const pact_layout& lay, double* centers /* [2 n] */);

}  // namespace pactgpu
