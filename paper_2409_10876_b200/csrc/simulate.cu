// Input-side step before DAS: the reference's straight-ray
// signal simulator, simulate_signals (phantom.hpp:282-362) with
// time_of_flight (aberration.hpp:79-100).
//
// Every pressure-bearing pixel emits S(t) = (2 a / sigma)(1 - u^2) e^{-u^2/2},
// u = (t - tau)/sigma, on each channel, tau being the straight-ray time of
// flight through the SOS raster (uniform background: |r - r_n| / v0).
// One thread per (source, transducer); a warp is 32 transducers of one source
// (neighbouring rays -> L1 locality, distinct output rows -> no atomic
// conflicts inside a warp).  tau's |r - r_n|/v0 part is fp64; the in-mask
// correction integral accumulates fp64 over fp32 bilinear samples of the
// deviation raster.  Samples accumulate in an fp64 buffer (order-independent
// to fp32 output precision), converted to fp32 at the end.
#include <cmath>
#include <string>
#include <vector>

#include "geom.cuh"
#include "train_ops.cuh"

namespace pactgpu {
namespace {

struct SimArgs {
  const double2* src;  // source positions (mm)
  const double* amp;   // amplitudes
  int n_src;
  int n_tx;
  double ring_r, ring_off;
  int T;
  double dt, t0, sigma;
  double v0;
  bool uniform;
  bool spreading;  // amplitude / sqrt(distance) (SimulateOptions::spreading)
  const float* dv;  // SOS deviation raster v - v0
  int W, H;
  double ox, oy, inv_pitch;
  double mcx, mcy, mr;
  double step;
  double* acc;  // [n_tx][T] fp64
};

__global__ void simulate_kernel(SimArgs a) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;  // transducer
  const int s = blockIdx.y;                              // source
  if (n >= a.n_tx || s >= a.n_src) return;
  // RingGeometry::transducer_position (core.hpp:162-165)
  const double ang = 2.0 * M_PI * n / a.n_tx + a.ring_off;
  const double rx = a.ring_r * cos(ang), ry = a.ring_r * sin(ang);
  const double2 p = a.src[s];
  const double dx = rx - p.x, dy = ry - p.y;
  const double dist = hypot(dx, dy);
  double tau;
  if (a.uniform) {
    tau = 1e-3 * dist / a.v0;
  } else {
    // time_of_flight(src = p, dst = r_n), aberration.hpp:79-100
    double corr = 0.0;
    if (dist > 0.0) {
      double t0, t1;
      seg_circle(p.x, p.y, rx, ry, a.mcx, a.mcy, a.mr, t0, t1);
      if (t0 < t1) {
        const double ux = dx * (1.0 / dist), uy = dy * (1.0 / dist);
        int ns = static_cast<int>(ceil((t1 - t0) / a.step));
        ns = ns < 1 ? 1 : ns;
        const double dl = (t1 - t0) / ns;
        const double fx0 = (p.x - a.ox) * a.inv_pitch, fy0 = (p.y - a.oy) * a.inv_pitch;
        const double dfx = ux * a.inv_pitch, dfy = uy * a.inv_pitch;
        const float v0f = static_cast<float>(a.v0);
        double sum = 0.0;
        for (int i = 0; i < ns; ++i) {
          double sp = t0 + (i + 0.5) * dl;
          Stencil st = stencil_at(static_cast<float>(fx0 + sp * dfx),
                                  static_cast<float>(fy0 + sp * dfy), a.W, a.H);
          float d = st.w00 * __ldg(a.dv + st.i00) + st.w01 * __ldg(a.dv + st.i01) +
                    st.w10 * __ldg(a.dv + st.i10) + st.w11 * __ldg(a.dv + st.i11);
          // 1/v - 1/v0 = -d / (v0 (v0 + d))
          sum += static_cast<double>(-d / (v0f * (v0f + d)));
        }
        corr = dl * sum;
      }
    }
    tau = 1e-3 * (dist / a.v0 + corr);
  }
  // pulse, phantom.hpp:347-360
  const double support = 6.0 * a.sigma;
  double amp = a.amp[s];
  if (a.spreading) amp /= sqrt(fmax(dist, 1e-6));
  const double scale = 2.0 * amp / a.sigma;
  int i0 = static_cast<int>(ceil((tau - support - a.t0) / a.dt));
  int i1 = static_cast<int>(floor((tau + support - a.t0) / a.dt));
  i0 = i0 < 0 ? 0 : i0;
  i1 = i1 > a.T - 1 ? a.T - 1 : i1;
  double* row = a.acc + static_cast<size_t>(n) * a.T;
  for (int i = i0; i <= i1; ++i) {
    double u = (a.t0 + i * a.dt - tau) / a.sigma;
    atomicAdd(row + i, scale * (1.0 - u * u) * exp(-0.5 * u * u));
  }
}

__global__ void to_f32_kernel(const double* __restrict__ in, size_t n, float* __restrict__ out) {
  size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = static_cast<float>(in[i]);
}

}  // namespace
}  // namespace pactgpu

using namespace pactgpu;

namespace pactgpu {

// The host scan of simulate_signals (phantom.hpp:284-334): validation in the
// reference's order, the pressure-bearing sources, the SOS range and the
// conservative arrival window [tau_min, tau_max].
struct SimScan {
  std::vector<double2> src;
  std::vector<double> amp;
  bool uniform = false;
  double tau_min = 0.0, tau_max = 0.0;
};

Status sim_scan(const pact_grid& grid, const double* pressure, const double* sos,
                double background_sos, const pact_ring& ring, double pulse_sigma, double dt,
                SimScan& o) {
  if (ring.n_transducers < 3) return validation("ring: need at least 3 transducers");
  if (!(ring.radius > 0.0)) return validation("ring: radius must be > 0");
  if (!(pulse_sigma > 0.0)) return validation("simulate: pulse_sigma must be > 0");
  if (!(dt > 0.0)) return validation("simulate: dt must be > 0");
  const int W = grid.width, H = grid.height;
  double max_r = 0.0;
  for (int iy = 0; iy < H; ++iy)
    for (int ix = 0; ix < W; ++ix) {
      const double a = pressure[static_cast<size_t>(iy) * W + ix];
      if (a == 0.0) continue;
      const double px = grid.origin_x + ix * grid.pitch, py = grid.origin_y + iy * grid.pitch;
      const double r = std::hypot(px, py);
      if (r >= ring.radius)
        return validation("simulate: pressure-bearing pixel outside the transducer ring");
      max_r = std::max(max_r, r);
      o.src.push_back(make_double2(px, py));
      o.amp.push_back(a);
    }
  const size_t npx = static_cast<size_t>(W) * H;
  double vmin = npx ? sos[0] : background_sos, vmax = vmin;
  for (size_t i = 0; i < npx; ++i) {
    vmin = std::min(vmin, sos[i]);
    vmax = std::max(vmax, sos[i]);
  }
  if (!(vmin > 0.0)) return validation("simulate: non-positive SOS value");
  o.uniform = (vmin == vmax && vmin == background_sos);
  o.tau_min = 1e-3 * (ring.radius - max_r) / vmax - 8.0 * pulse_sigma;
  o.tau_max = 1e-3 * (ring.radius + max_r) / vmin + 8.0 * pulse_sigma;
  return {};
}

Status sim_check_window(const SimScan& sc, double t0, int n_samples, double dt) {
  if (!sc.src.empty() && (t0 > sc.tau_min || t0 + (n_samples - 1) * dt < sc.tau_max)) {
    std::string m = "simulate: time window too short, need [" + std::to_string(sc.tau_min) +
                    ", " + std::to_string(sc.tau_max) + "] s";
    set_error("%s", m.c_str());
    return {PACT_E_VALIDATION};
  }
  return {};
}

}  // namespace pactgpu

extern "C" int pact_simulate_window(const pact_grid* grid, const double* pressure,
                                    const double* sos, double background_sos,
                                    const pact_ring* ring, double pulse_sigma, double dt,
                                    double t0, int32_t n_samples, pact_signal_meta* out) {
  using namespace pactgpu;
  if (!grid || !pressure || !sos || !ring || !out)
    return validation("pact_simulate_window: null argument").code;
  SimScan sc;
  PACT_TRY(sim_scan(*grid, pressure, sos, background_sos, *ring, pulse_sigma, dt, sc));
  pact_signal_meta m{};
  m.dt = dt;
  m.background_sos = background_sos;
  // phantom.hpp:320-331: NaN t0 / n_samples 0 -> the auto window
  m.t0 = std::isnan(t0) ? std::floor(sc.tau_min / dt) * dt : t0;
  m.n_samples = n_samples > 0 ? n_samples
                              : static_cast<int>(std::ceil((sc.tau_max - m.t0) / dt)) + 1;
  PACT_TRY(sim_check_window(sc, m.t0, m.n_samples, dt));
  *out = m;
  return PACT_OK;
}

extern "C" int pact_simulate_signals(pact_ctx* ctx, const pact_grid* grid, const double* pressure,
                                     const double* sos, const pact_mask* mask,
                                     double background_sos, const pact_ring* ring,
                                     double pulse_sigma, const pact_signal_meta* meta,
                                     double ray_step, float* out) {
  return pact_simulate_signals_ex(ctx, grid, pressure, sos, mask, background_sos, ring,
                                  pulse_sigma, meta, ray_step, 0, out);
}

extern "C" int pact_simulate_signals_ex(pact_ctx* ctx, const pact_grid* grid,
                                        const double* pressure, const double* sos,
                                        const pact_mask* mask, double background_sos,
                                        const pact_ring* ring, double pulse_sigma,
                                        const pact_signal_meta* meta, double ray_step,
                                        int32_t spreading, float* out) {
  using namespace pactgpu;
  if (!ctx || !grid || !pressure || !sos || !mask || !ring || !meta || !out)
    return validation("pact_simulate_signals: null argument").code;
  if (meta->n_samples < 1) {
    // the reference's checks before the window come first
    SimScan sc;
    PACT_TRY(sim_scan(*grid, pressure, sos, background_sos, *ring, pulse_sigma, meta->dt, sc));
    return validation("simulate: n_samples must be >= 1").code;
  }
  SimScan sc;
  PACT_TRY(sim_scan(*grid, pressure, sos, background_sos, *ring, pulse_sigma, meta->dt, sc));
  PACT_TRY(sim_check_window(sc, meta->t0, meta->n_samples, meta->dt));
  const int W = grid->width, H = grid->height;
  const size_t npx = static_cast<size_t>(W) * H;
  const std::vector<double2>& src = sc.src;
  const std::vector<double>& amp = sc.amp;
  const bool uniform = sc.uniform;
  const int N = ring->n_transducers, T = meta->n_samples;
  std::vector<float> dvh(npx);
  for (size_t i = 0; i < npx; ++i) dvh[i] = static_cast<float>(sos[i] - background_sos);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t ns = std::max<size_t>(src.size(), 1);
  size_t o_acc = 0, o_src = al(sizeof(double) * N * T), o_amp = al(o_src + sizeof(double2) * ns),
         o_dv = al(o_amp + sizeof(double) * ns), total = al(o_dv + sizeof(float) * npx);
  void* base = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric1, total, &base));
  char* b = static_cast<char*>(base);
  SimArgs a{};
  a.acc = reinterpret_cast<double*>(b + o_acc);
  a.src = reinterpret_cast<double2*>(b + o_src);
  a.amp = reinterpret_cast<double*>(b + o_amp);
  a.dv = reinterpret_cast<float*>(b + o_dv);
  PACT_CUDA(cudaMemsetAsync(a.acc, 0, sizeof(double) * N * T, ctx->stream));
  if (!src.empty()) {
    PACT_CUDA(cudaMemcpyAsync(const_cast<double2*>(a.src), src.data(), sizeof(double2) * src.size(),
                              cudaMemcpyHostToDevice, ctx->stream));
    PACT_CUDA(cudaMemcpyAsync(const_cast<double*>(a.amp), amp.data(), sizeof(double) * amp.size(),
                              cudaMemcpyHostToDevice, ctx->stream));
  }
  PACT_CUDA(cudaMemcpyAsync(const_cast<float*>(a.dv), dvh.data(), sizeof(float) * npx,
                            cudaMemcpyHostToDevice, ctx->stream));
  a.n_src = static_cast<int>(src.size());
  a.n_tx = N;
  a.ring_r = ring->radius;
  a.ring_off = ring->angle_offset;
  a.T = T;
  a.dt = meta->dt;
  a.t0 = meta->t0;
  a.sigma = pulse_sigma;
  a.v0 = background_sos;
  a.uniform = uniform;
  a.spreading = spreading != 0;
  a.W = W;
  a.H = H;
  a.ox = grid->origin_x;
  a.oy = grid->origin_y;
  a.inv_pitch = 1.0 / grid->pitch;
  a.mcx = mask->center_x;
  a.mcy = mask->center_y;
  a.mr = mask->radius;
  a.step = ray_step;
  if (a.n_src > 0) {
    // grid.y is limited to 65535: launch in source batches
    for (int s0 = 0; s0 < a.n_src; s0 += 65535) {
      SimArgs b2 = a;
      b2.src = a.src + s0;
      b2.amp = a.amp + s0;
      b2.n_src = std::min(65535, a.n_src - s0);
      dim3 g(div_up(N, 128), b2.n_src);
      simulate_kernel<<<g, 128, 0, ctx->stream>>>(b2);
      PACT_TRY(after_launch(ctx, "simulate_kernel"));
    }
  }
  size_t n = static_cast<size_t>(N) * T;
  to_f32_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, ctx->stream>>>(a.acc, n, out);
  PACT_TRY(after_launch(ctx, "to_f32_kernel"));
  PACT_CUDA(cudaStreamSynchronize(ctx->stream));  // host staging vectors are released
  return PACT_OK;
}
