// dual_sos_das (beamform.hpp:124-150): DAS with a two-speed time of flight —
// the straight path from pixel r to transducer n travels at body_sos over its
// analytic chord through the body disc (segment_circle_intersection,
// core.hpp:184-204) and at v0 elsewhere:
//   y(r) = sum_n S_n(1e-3 ((|r - r_n| - c) / v0 + c / body_sos)),  c = chord length.
//
// One thread per pixel; the transducer positions (fp64) are staged in shared
// memory and the signal matrix (<= 32 MB fp32) is read through L2.  The
// geometry and the sample index are fp64 like the reference, so the time of
// flight carries no fp32 rounding (a 1e-7 relative error in t is already
// 1e-3 samples at T = 8192); the sum is fp64.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "geom.cuh"

namespace pactgpu {
namespace {

struct DualArgs {
  const float* sig;
  int n_tx, n_samples;
  int width, height;
  double ox, oy, pitch;
  double t0, dt, v0;
  double bx, by, br, body_sos;
};

// SignalSet::sample (core.hpp:296-304) on fp32 data.
__device__ __forceinline__ double sample_at(const float* __restrict__ row, int T, double s) {
  if (s < 0.0 || s > T - 1) return 0.0;
  const int i = static_cast<int>(s);
  if (i >= T - 1) return row[T - 1];
  const double f = s - i;
  return (1.0 - f) * row[i] + f * row[i + 1];
}

__global__ void __launch_bounds__(256) dual_das_kernel(DualArgs a, const double2* __restrict__ pos,
                                                       float* __restrict__ out) {
  extern __shared__ double2 s_pos[];
  for (int n = threadIdx.x; n < a.n_tx; n += blockDim.x) s_pos[n] = pos[n];
  __syncthreads();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.width * a.height) return;
  const int iy = p / a.width, ix = p - iy * a.width;
  const double rx = a.ox + ix * a.pitch, ry = a.oy + iy * a.pitch;  // GridSpec::world
  const double inv_v0 = 1.0 / a.v0, inv_vb = 1.0 / a.body_sos;
  double acc = 0.0;
  for (int n = 0; n < a.n_tx; ++n) {
    const double2 q = s_pos[n];
    const double dist = hypot(rx - q.x, ry - q.y);
    double s0, s1;
    seg_circle(rx, ry, q.x, q.y, a.bx, a.by, a.br, s0, s1);
    const double inside = fmax(0.0, s1 - s0);
    const double t = 1e-3 * ((dist - inside) * inv_v0 + inside * inv_vb);
    acc += sample_at(a.sig + static_cast<size_t>(n) * a.n_samples, a.n_samples, (t - a.t0) / a.dt);
  }
  out[p] = static_cast<float>(acc);
}

}  // namespace
}  // namespace pactgpu

using namespace pactgpu;

extern "C" int pact_dual_sos_das(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                                 const float* signals, const pact_grid* grid, double v0,
                                 const pact_body* body, float* out) {
  if (!ctx || !ring || !meta || !grid || !body || !signals || !out)
    return validation("pact_dual_sos_das: null argument").code;
  // Validation order of dual_sos_das (beamform.hpp:126-131).
  if (ring->n_transducers < 3) return validation("ring: need at least 3 transducers").code;
  if (!(ring->radius > 0.0)) return validation("ring: radius must be > 0").code;
  if (meta->n_samples < 2) return validation("signals: need at least 2 samples").code;
  if (!(meta->dt > 0.0)) return validation("signals: dt must be > 0").code;
  if (grid->width < 1 || grid->height < 1)
    return validation("grid: width and height must be >= 1").code;
  if (!(grid->pitch > 0.0)) return validation("grid: pitch must be > 0").code;
  if (!(body->radius > 0.0)) return validation("body model: radius must be > 0").code;
  if (!(body->body_sos >= 1300.0 && body->body_sos <= 1800.0))
    return validation("body model: SOS outside [1300, 1800] m/s").code;
  if (!(v0 > 0.0)) return validation("dual_sos_das: v0 must be > 0").code;
  if (std::hypot(body->center_x, body->center_y) + body->radius >= ring->radius)
    return validation("dual_sos_das: body disc extends outside the transducer ring").code;

  const int N = ring->n_transducers;
  std::vector<double2> pos(N);  // RingGeometry::transducer_position (core.hpp:162-165)
  for (int n = 0; n < N; ++n) {
    const double ang = 2.0 * M_PI * n / N + ring->angle_offset;
    pos[n] = make_double2(ring->radius * std::cos(ang), ring->radius * std::sin(ang));
  }
  void* dpos = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchDasGeom, sizeof(double2) * N, &dpos));
  PACT_CUDA(cudaMemcpyAsync(dpos, pos.data(), sizeof(double2) * N, cudaMemcpyHostToDevice,
                            ctx->stream));
  DualArgs a{signals, N, meta->n_samples, grid->width, grid->height, grid->origin_x,
             grid->origin_y, grid->pitch, meta->t0, meta->dt, v0, body->center_x,
             body->center_y, body->radius, body->body_sos};
  const size_t smem = sizeof(double2) * N;
  if (smem > 48 * 1024)
    PACT_CUDA(cudaFuncSetAttribute(dual_das_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  const int npx = grid->width * grid->height;
  dual_das_kernel<<<div_up(npx, 256), 256, smem, ctx->stream>>>(
      a, static_cast<const double2*>(dpos), out);
  PACT_TRY(after_launch(ctx, "dual_das_kernel"));
  return PACT_OK;
}
