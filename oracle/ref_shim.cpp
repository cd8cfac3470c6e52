// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference library (header-only C++20,
// /root/reference/proj/include/pact/*.hpp), compiled in place by
// oracle/Makefile into oracle/_ref/libpact_ref.so.  It exists so that
//   * the CPU restatement in oracle/pact_oracle.c can be pinned against the
//     reference itself (tests/golden/ fixtures are generated through it), and
//   * bench.py --impl reference can time the reference's own CPU path.
// Every function forwards to the reference entry point named in its comment;
// the only code here is argument marshalling (flat fp64 arrays <-> pact types).
#include <chrono>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "pact/aberration.hpp"
#include "pact/beamform.hpp"
#include "pact/core.hpp"
#include "pact/evaluate.hpp"
#include "pact/io.hpp"
#include "pact/deconv.hpp"
#include "pact/nfield.hpp"
#include "pact/optimize.hpp"
#include "pact/phantom.hpp"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const pact::ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const pact::NumericalError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

pact::GridSpec grid_of(int w, int h, double pitch, double ox, double oy) {
  pact::GridSpec g;
  g.width = w;
  g.height = h;
  g.pitch = pitch;
  g.origin = {ox, oy};
  return g;
}

pact::RasterGrid raster_of(const pact::GridSpec& g, const double* v) {
  pact::RasterGrid r = pact::RasterGrid::zeros(g);
  std::memcpy(r.values.data(), v, sizeof(double) * r.values.size());
  return r;
}

pact::SignalSet signals_of(int n, double radius, double offset, int T, double dt, double t0,
                           double v0, const double* data) {
  pact::SignalSet s;
  s.geom = {n, radius, offset};
  s.n_samples = T;
  s.dt = dt;
  s.t0 = t0;
  s.background_sos = v0;
  s.data.assign(data, data + static_cast<size_t>(n) * T);
  return s;
}

pact::SirenParams siren_of(int hidden, int layers, double omega0, double out_scale, double v0,
                           const double* theta) {
  pact::SirenParams p;
  p.hidden = hidden;
  p.n_hidden_layers = layers;
  p.omega0 = omega0;
  p.out_scale = out_scale;
  p.v0 = v0;
  p.theta.assign(theta, theta + p.param_count());
  return p;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// das_stack, beamform.hpp:77-110
int ref_das_stack(int n_tx, double radius, double offset, int T, double dt, double t0,
                  const double* sig, int W, int H, double pitch, double ox, double oy, double v0,
                  int K, const double* delays, int workers, double* out) {
  return guarded([&] {
    auto s = signals_of(n_tx, radius, offset, T, dt, t0, v0, sig);
    auto st = pact::das_stack(s, grid_of(W, H, pitch, ox, oy), v0,
                              std::vector<double>(delays, delays + K), workers);
    size_t plane = static_cast<size_t>(W) * H;
    for (int j = 0; j < K; ++j)
      std::memcpy(out + j * plane, st.images[j].values.data(), sizeof(double) * plane);
  });
}

// das, beamform.hpp:56-75
int ref_das(int n_tx, double radius, double offset, int T, double dt, double t0,
            const double* sig, int W, int H, double pitch, double ox, double oy, double v0,
            double d, int workers, double* out) {
  return guarded([&] {
    auto s = signals_of(n_tx, radius, offset, T, dt, t0, v0, sig);
    auto img = pact::das(s, grid_of(W, H, pitch, ox, oy), v0, d, workers);
    std::memcpy(out, img.values.data(), sizeof(double) * img.values.size());
  });
}

// dual_sos_das, beamform.hpp:124-150
int ref_dual_sos_das(int n_tx, double radius, double offset, int T, double dt, double t0,
                     const double* sig, int W, int H, double pitch, double ox, double oy,
                     double v0, double bcx, double bcy, double br, double bsos, double* out) {
  return guarded([&] {
    auto s = signals_of(n_tx, radius, offset, T, dt, t0, v0, sig);
    pact::BodyModel body;
    body.center = {bcx, bcy};
    body.radius = br;
    body.body_sos = bsos;
    auto img = pact::dual_sos_das(s, grid_of(W, H, pitch, ox, oy), v0, body, 0);
    std::memcpy(out, img.values.data(), sizeof(double) * img.values.size());
  });
}

// psnr / ssim / sos_rmse_masked, evaluate.hpp:39-114
static pact::RasterGrid raster_of(const double* v, int W, int H, double pitch, double ox,
                                  double oy) {
  pact::RasterGrid r = pact::RasterGrid::zeros(grid_of(W, H, pitch, ox, oy));
  std::memcpy(r.values.data(), v, sizeof(double) * r.values.size());
  return r;
}
int ref_psnr(const double* test, const double* truth, int W, int H, double data_range,
             double* out) {
  return guarded([&] {
    *out = pact::psnr(raster_of(test, W, H, 0.1, 0, 0), raster_of(truth, W, H, 0.1, 0, 0),
                      data_range);
  });
}
int ref_ssim(const double* test, const double* truth, int W, int H, double data_range,
             double* out) {
  return guarded([&] {
    *out = pact::ssim(raster_of(test, W, H, 0.1, 0, 0), raster_of(truth, W, H, 0.1, 0, 0),
                      data_range);
  });
}
int ref_sos_rmse_masked(const double* test, const double* truth, int W, int H, double pitch,
                        double ox, double oy, double mcx, double mcy, double mr, double* out) {
  return guarded([&] {
    pact::CircularMask m;
    m.center = {mcx, mcy};
    m.radius = mr;
    *out = pact::sos_rmse_masked(raster_of(test, W, H, pitch, ox, oy),
                                 raster_of(truth, W, H, pitch, ox, oy), m);
  });
}

// init_siren, nfield.hpp:83-107
int ref_init_siren(uint64_t seed, int hidden, int layers, double omega0, double out_scale,
                   double v0, double* theta) {
  return guarded([&] {
    auto p = pact::init_siren(seed, hidden, layers, omega0, out_scale, v0);
    std::memcpy(theta, p.theta.data(), sizeof(double) * p.theta.size());
  });
}

long ref_siren_param_count(int hidden, int layers) {
  return static_cast<long>(pact::siren_param_count(2, hidden, layers));
}

// render_sos, nfield.hpp:145-162 ; returns the masked-pixel count
int ref_render_sos(int hidden, int layers, double omega0, double out_scale, double v0,
                   const double* theta, int W, int H, double pitch, double ox, double oy,
                   double mcx, double mcy, double mr, double* raster, int* n_masked) {
  return guarded([&] {
    auto p = siren_of(hidden, layers, omega0, out_scale, v0, theta);
    auto f = pact::render_sos(p, grid_of(W, H, pitch, ox, oy), {{mcx, mcy}, mr});
    std::memcpy(raster, f.raster.values.data(), sizeof(double) * f.raster.values.size());
    if (n_masked) *n_masked = static_cast<int>(f.masked_indices.size());
  });
}

// backprop_sos, nfield.hpp:166-233 ; grad_v is per masked pixel (row-major order)
int ref_backprop_sos(int hidden, int layers, double omega0, double out_scale, double v0,
                     const double* theta, int W, int H, double pitch, double ox, double oy,
                     double mcx, double mcy, double mr, const double* grad_v, double* grad) {
  return guarded([&] {
    auto p = siren_of(hidden, layers, omega0, out_scale, v0, theta);
    auto f = pact::render_sos(p, grid_of(W, H, pitch, ox, oy), {{mcx, mcy}, mr});
    std::vector<double> g(grad_v, grad_v + f.masked_indices.size());
    auto out = pact::backprop_sos(p, f, g);
    std::memcpy(grad, out.data(), sizeof(double) * out.size());
  });
}

// wavefront_profile, aberration.hpp:134-186 (for n_centers centres)
int ref_wavefront_profile(int n_centers, const double* centers, int n_tx, double radius,
                          double offset, int W, int H, double pitch, double ox, double oy,
                          const double* sos, double v0, double mcx, double mcy, double mr,
                          int n_angles, double step, double* w) {
  return guarded([&] {
    auto g = grid_of(W, H, pitch, ox, oy);
    auto r = raster_of(g, sos);
    for (int i = 0; i < n_centers; ++i) {
      auto prof = pact::wavefront_profile({centers[2 * i], centers[2 * i + 1]},
                                          {n_tx, radius, offset}, r, v0, {{mcx, mcy}, mr},
                                          n_angles, step, false);
      std::memcpy(w + static_cast<size_t>(i) * n_angles, prof.w.data(),
                  sizeof(double) * n_angles);
    }
  });
}

// transfer_stack, aberration.hpp:236-265 ; H is interleaved complex [K][P][P]
int ref_transfer_stack(int n_angles, const double* w, int K, const double* delays, int P,
                       double pitch, double* H) {
  return guarded([&] {
    pact::WavefrontProfile prof;
    prof.n_angles = n_angles;
    prof.w.assign(w, w + n_angles);
    auto ts = pact::transfer_stack(prof, std::vector<double>(delays, delays + K), P, pitch);
    for (int j = 0; j < K; ++j)
      std::memcpy(H + 2 * static_cast<size_t>(j) * P * P, ts.spectra[j].data(),
                  sizeof(double) * 2 * P * P);
  });
}

// make_patch_layout, core.hpp:252-281 ; returns P, stride, nx, ny, offsets, centres
int ref_patch_layout(int W, int H, double pitch, double ox, double oy, double patch_mm,
                     double overlap, int* info, int* offsets, double* centers) {
  return guarded([&] {
    auto lay = pact::make_patch_layout(grid_of(W, H, pitch, ox, oy), patch_mm, overlap);
    info[0] = lay.patch_pixels;
    info[1] = lay.stride_pixels;
    info[2] = lay.nx;
    info[3] = lay.ny;
    if (offsets)
      for (int i = 0; i < lay.n_patches(); ++i) {
        offsets[2 * i] = lay.offsets[i].first;
        offsets[2 * i + 1] = lay.offsets[i].second;
      }
    if (centers)
      for (int i = 0; i < lay.n_patches(); ++i) {
        centers[2 * i] = lay.centers[i].x;
        centers[2 * i + 1] = lay.centers[i].y;
      }
  });
}

static pact::DasStack stack_of(int K, const double* delays, double v0, const pact::GridSpec& g,
                               const double* stack) {
  pact::DasStack st;
  st.delays.assign(delays, delays + K);
  st.v0 = v0;
  size_t plane = static_cast<size_t>(g.width) * g.height;
  for (int j = 0; j < K; ++j) st.images.push_back(raster_of(g, stack + j * plane));
  return st;
}

// extract_patch_spectra, deconv.hpp:64-74 ; Y interleaved complex [patch][K][P][P]
int ref_patch_spectra(int K, const double* delays, double v0, int W, int H, double pitch,
                      double ox, double oy, const double* stack, double patch_mm,
                      double overlap, int workers, double* Y) {
  return guarded([&] {
    auto g = grid_of(W, H, pitch, ox, oy);
    auto st = stack_of(K, delays, v0, g, stack);
    auto lay = pact::make_patch_layout(g, patch_mm, overlap);
    auto ps = pact::extract_patch_spectra(st, lay, workers);
    size_t P2 = static_cast<size_t>(lay.patch_pixels) * lay.patch_pixels;
    for (size_t i = 0; i < ps.size(); ++i)
      for (int j = 0; j < K; ++j)
        std::memcpy(Y + 2 * (i * K + j) * P2, ps[i].Y[j].data(), sizeof(double) * 2 * P2);
  });
}

// deconvolve_image, deconv.hpp:176-198
int ref_deconvolve_image(int K, const double* delays, double v0, int W, int H, double pitch,
                         double ox, double oy, const double* stack, const double* sos,
                         int n_tx, double radius, double offset, double mcx, double mcy,
                         double mr, double patch_mm, double overlap, double eps, int n_angles,
                         double ray_step, double merge_fwhm, int workers, double* image) {
  return guarded([&] {
    auto g = grid_of(W, H, pitch, ox, oy);
    auto st = stack_of(K, delays, v0, g, stack);
    auto lay = pact::make_patch_layout(g, patch_mm, overlap);
    pact::DeconvolveOptions opt;
    opt.eps = eps;
    opt.n_angles = n_angles;
    opt.ray_step = ray_step;
    opt.merge_fwhm = merge_fwhm;
    opt.workers = workers;
    auto img = pact::deconvolve_image(st, raster_of(g, sos), {n_tx, radius, offset},
                                      {{mcx, mcy}, mr}, lay, opt);
    std::memcpy(image, img.values.data(), sizeof(double) * img.values.size());
  });
}

// detail::fused_patch_loss_grad, optimize.hpp:234-325, with the training-path
// complex<float> spectra cache (optimize.hpp:382-392).  Yf: float pairs [K][P][P].
int ref_fused_patch_loss_grad(int K, const float* Yf, const double* w, int P, double pitch,
                              int n_angles, const double* delays, double eps, double scale,
                              int implicit, double* loss, double* dw) {
  return guarded([&] {
    size_t P2 = static_cast<size_t>(P) * P;
    std::vector<std::vector<std::complex<float>>> ys(K, std::vector<std::complex<float>>(P2));
    for (int j = 0; j < K; ++j)
      for (size_t b = 0; b < P2; ++b)
        ys[j][b] = {Yf[2 * (j * P2 + b)], Yf[2 * (j * P2 + b) + 1]};
    auto table = pact::PatchBinTable::make(P, pitch, n_angles);
    auto phases =
        pact::detail::make_delay_phases(table, std::vector<double>(delays, delays + K));
    pact::detail::FusedScratch scratch;
    std::vector<double> dwv;
    *loss = pact::detail::fused_patch_loss_grad(ys, std::vector<double>(w, w + n_angles), table,
                                                phases, eps, scale, implicit != 0, scratch,
                                                dwv);
    std::memcpy(dw, dwv.data(), sizeof(double) * n_angles);
  });
}

// wavefront_grad_trace, aberration.hpp:333-361 (accumulates into grad_v, W*H)
int ref_wavefront_grad_trace(double cx, double cy, int n_tx, double radius, double offset,
                             int W, int H, double pitch, double ox, double oy, const double* sos,
                             double v0, double mcx, double mcy, double mr, int n_angles,
                             double step, const double* dw, double* grad_v) {
  return guarded([&] {
    auto g = grid_of(W, H, pitch, ox, oy);
    auto r = raster_of(g, sos);
    std::vector<double> gv(grad_v, grad_v + static_cast<size_t>(W) * H);
    pact::wavefront_grad_trace({cx, cy}, {n_tx, radius, offset}, r, v0, {{mcx, mcy}, mr},
                               n_angles, step, std::vector<double>(dw, dw + n_angles), gv);
    std::memcpy(grad_v, gv.data(), sizeof(double) * gv.size());
  });
}

// tv_loss, optimize.hpp:120-153 on the field render_sos would produce for
// the given raster (masked pixels = mask.contains(world(ix, iy))).
int ref_tv_loss(int W, int H, double pitch, double ox, double oy, const double* raster,
                double mcx, double mcy, double mr, double lambda, double* value,
                double* grad_masked) {
  return guarded([&] {
    auto g = grid_of(W, H, pitch, ox, oy);
    pact::SosField f;
    f.mask = {{mcx, mcy}, mr};
    f.raster = raster_of(g, raster);
    for (int iy = 0; iy < H; ++iy)
      for (int ix = 0; ix < W; ++ix) {
        pact::Vec2 p = g.world(ix, iy);
        if (!f.mask.contains(p)) continue;
        f.masked_indices.push_back(iy * W + ix);
        f.coords.push_back({(p.x - mcx) / mr, (p.y - mcy) / mr});
      }
    auto tv = pact::tv_loss(f, lambda);
    *value = tv.value;
    std::memcpy(grad_masked, tv.grad.data(), sizeof(double) * tv.grad.size());
  });
}

// adam_step, optimize.hpp:87-110 ; state = (m, v, t)
int ref_adam_step(int n, double* params, const double* grads, double* m, double* v, long* t,
                  double lr, double b1, double b2, double eps) {
  return guarded([&] {
    std::vector<double> p(params, params + n), g(grads, grads + n);
    pact::AdamState st;
    if (*t > 0) {
      st.m.assign(m, m + n);
      st.v.assign(v, v + n);
    }
    st.t = *t;
    pact::adam_step(p, g, st, lr, b1, b2, eps);
    std::memcpy(params, p.data(), sizeof(double) * n);
    std::memcpy(m, st.m.data(), sizeof(double) * n);
    std::memcpy(v, st.v.data(), sizeof(double) * n);
    *t = st.t;
  });
}

struct RefTrainCfg {
  int epochs, steps_per_epoch;
  double lr, beta1, beta2, adam_eps, lambda_tv;
  int n_delays;
  const double* delays;
  double eps_deconv;
  int n_angles;
  double ray_step;
  uint64_t seed;
  int hidden, sine_layers;
  double omega0, out_scale, patch_mm, overlap, merge_fwhm;
  int implicit_xhat_grad, workers;
};

// joint_reconstruct, optimize.hpp:367-494.  reports: [epochs][4] = data, tv,
// total, wall_time.  image/sos: W*H.  theta: final parameters.
int ref_joint_reconstruct(int n_tx, double radius, double offset, int T, double dt, double t0,
                          double v0, const double* sig, int W, int H, double pitch, double ox,
                          double oy, double mcx, double mcy, double mr, const RefTrainCfg* c,
                          double* reports, double* image, double* sos, double* theta) {
  return guarded([&] {
    auto s = signals_of(n_tx, radius, offset, T, dt, t0, v0, sig);
    pact::TrainConfig cfg;
    cfg.epochs = c->epochs;
    cfg.steps_per_epoch = c->steps_per_epoch;
    cfg.learning_rate = c->lr;
    cfg.beta1 = c->beta1;
    cfg.beta2 = c->beta2;
    cfg.adam_eps = c->adam_eps;
    cfg.lambda_tv = c->lambda_tv;
    cfg.delays.assign(c->delays, c->delays + c->n_delays);
    cfg.eps_deconv = c->eps_deconv;
    cfg.n_angles = c->n_angles;
    cfg.ray_step = c->ray_step;
    cfg.seed = c->seed;
    cfg.hidden = c->hidden;
    cfg.sine_layers = c->sine_layers;
    cfg.omega0 = c->omega0;
    cfg.out_scale = c->out_scale;
    cfg.patch_mm = c->patch_mm;
    cfg.overlap = c->overlap;
    cfg.merge_fwhm = c->merge_fwhm;
    cfg.implicit_xhat_grad = c->implicit_xhat_grad != 0;
    cfg.workers = c->workers;
    auto jr = pact::joint_reconstruct(s, grid_of(W, H, pitch, ox, oy), {{mcx, mcy}, mr}, cfg);
    for (size_t e = 0; e < jr.reports.size(); ++e) {
      reports[4 * e + 0] = jr.reports[e].data_term;
      reports[4 * e + 1] = jr.reports[e].tv_term;
      reports[4 * e + 2] = jr.reports[e].total;
      reports[4 * e + 3] = jr.reports[e].wall_time;
    }
    if (image) std::memcpy(image, jr.image.values.data(), sizeof(double) * W * H);
    if (sos) std::memcpy(sos, jr.sos.values.data(), sizeof(double) * W * H);
    if (theta) std::memcpy(theta, jr.params.theta.data(), sizeof(double) * jr.params.theta.size());
  });
}

// simulate_signals, phantom.hpp:282-362, on a phantom given as rasters.
// t0 / n_samples fixed by the caller (SimulateOptions.t0 / n_samples).
int ref_simulate_signals(int W, int H, double pitch, double ox, double oy,
                         const double* pressure, const double* sos, double mcx, double mcy,
                         double mr, double background_sos, int n_tx, double radius,
                         double offset, double pulse_sigma, double dt, double t0, int T,
                         double ray_step, int workers, double* out) {
  return guarded([&] {
    auto g = grid_of(W, H, pitch, ox, oy);
    pact::Phantom ph;
    ph.pressure = raster_of(g, pressure);
    ph.sos = raster_of(g, sos);
    ph.mask = {{mcx, mcy}, mr};
    ph.background_sos = background_sos;
    pact::SimulateOptions opt;
    opt.pulse_sigma = pulse_sigma;
    opt.dt = dt;
    opt.t0 = t0;
    opt.n_samples = T;
    opt.ray_step = ray_step;
    opt.workers = workers;
    auto s = pact::simulate_signals(ph, {n_tx, radius, offset}, opt);
    std::memcpy(out, s.data.data(), sizeof(double) * s.data.size());
  });
}

// testsupport::make_small_instance (tests/test_support.hpp:43-75): the
// reference's shared 64x64 fixture.  Call with sig == nullptr to get T.
int ref_small_instance_signals(double* sig, int* T, double* t0) {
  return guarded([&] {
    pact::GridSpec grid = pact::GridSpec::centered(64, 64, 0.1);
    pact::CircularMask mask{{0.0, 0.0}, 2.6};
    pact::RingGeometry ring{64, 50.0, 0.0};
    pact::PhantomSpec spec = pact::builtin_phantom_spec("empty", 1500.0);
    spec.mask = mask;
    spec.discs.push_back({{0.4, -0.3}, 1.2, 1560.0, 0.0});
    spec.points.push_back({{0.0, 0.0}, 1.0});
    spec.points.push_back({{1.0, 0.8}, 0.8});
    spec.points.push_back({{-1.2, 0.4}, 0.9});
    pact::Phantom ph = pact::generate_phantom(grid, spec, 0);
    pact::SignalSet s = pact::simulate_signals(ph, ring);
    *T = s.n_samples;
    *t0 = s.t0;
    if (sig) std::memcpy(sig, s.data.data(), sizeof(double) * s.data.size());
  });
}

static pact::TrainConfig train_config_of(const RefTrainCfg* c) {
  pact::TrainConfig cfg;
  cfg.epochs = c->epochs;
  cfg.steps_per_epoch = c->steps_per_epoch;
  cfg.learning_rate = c->lr;
  cfg.beta1 = c->beta1;
  cfg.beta2 = c->beta2;
  cfg.adam_eps = c->adam_eps;
  cfg.lambda_tv = c->lambda_tv;
  cfg.delays.assign(c->delays, c->delays + c->n_delays);
  cfg.eps_deconv = c->eps_deconv;
  cfg.n_angles = c->n_angles;
  cfg.ray_step = c->ray_step;
  cfg.seed = c->seed;
  cfg.hidden = c->hidden;
  cfg.sine_layers = c->sine_layers;
  cfg.omega0 = c->omega0;
  cfg.out_scale = c->out_scale;
  cfg.patch_mm = c->patch_mm;
  cfg.overlap = c->overlap;
  cfg.merge_fwhm = c->merge_fwhm;
  cfg.implicit_xhat_grad = c->implicit_xhat_grad != 0;
  cfg.workers = c->workers;
  return cfg;
}

// One NF-APACT iteration at parameters `theta` without the Adam update: the
// body of joint_reconstruct's step loop (optimize.hpp:413-461) composed from
// the reference entry points, plus deconvolve_image under theta's SOS
// (optimize.hpp:478-486).  Any output pointer may be null.  patch_lo/hi
// restrict the per-patch work to a sample (bench CPU baseline); pass 0/-1 for all.
int ref_nf_step(int n_tx, double radius, double offset, int T, double dt, double t0, double v0,
                const double* sig, int W, int H, double pitch, double ox, double oy, double mcx,
                double mcy, double mr, const RefTrainCfg* c, const double* theta, int patch_lo,
                int patch_hi, double* data_term, double* tv_term, double* loss_patch,
                double* w_out, double* dw_out, double* sos_out, double* grad_v_masked,
                double* grad_theta, double* image, double* seconds) {
  return guarded([&] {
    auto s = signals_of(n_tx, radius, offset, T, dt, t0, v0, sig);
    pact::TrainConfig cfg = train_config_of(c);
    auto grid = grid_of(W, H, pitch, ox, oy);
    pact::CircularMask mask{{mcx, mcy}, mr};
    auto layout = pact::make_patch_layout(grid, cfg.patch_mm, cfg.overlap);
    const int P = layout.patch_pixels, N = layout.n_patches();
    const size_t M = cfg.delays.size();
    const double loss_scale = 1.0 / (static_cast<double>(N) * M * P * P);
    auto stack = pact::das_stack(s, grid, v0, cfg.delays, cfg.workers);
    std::vector<std::vector<std::vector<std::complex<float>>>> ycache(N);
    pact::parallel_for(N, cfg.workers, [&](int i) {
      pact::PatchSpectra ps = pact::extract_patch_spectra_one(stack, layout, i);
      ycache[i].resize(M);
      for (size_t j = 0; j < M; ++j) {
        ycache[i][j].resize(ps.Y[j].size());
        for (size_t b = 0; b < ps.Y[j].size(); ++b)
          ycache[i][j][b] = std::complex<float>(ps.Y[j][b]);
      }
    });
    auto params = siren_of(cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale, v0, theta);
    const auto table = pact::PatchBinTable::make(P, grid.pitch, cfg.n_angles);
    const auto phases = pact::detail::make_delay_phases(table, cfg.delays);
    int lo = patch_lo, hi = patch_hi < 0 ? N : std::min(N, patch_hi);
    auto t_start = std::chrono::steady_clock::now();
    auto field = pact::render_sos(params, grid, mask);
    std::vector<double> gv(field.raster.values.size(), 0.0);
    std::vector<double> lp(N, 0.0);
    const int nw = pact::resolve_workers(cfg.workers);
    const int span = hi - lo;
    const int n_chunks = std::max(1, std::min(span, nw * 4));
    const int chunk_len = (span + n_chunks - 1) / n_chunks;
    std::vector<std::vector<double>> chunk_gv(n_chunks);
    pact::parallel_for(n_chunks, cfg.workers, [&](int ck) {
      int a = lo + ck * chunk_len, b = std::min(hi, a + chunk_len);
      if (a >= b) return;
      auto& g = chunk_gv[ck];
      g.assign(gv.size(), 0.0);
      pact::detail::FusedScratch scratch;
      std::vector<double> dw;
      for (int i = a; i < b; ++i) {
        auto prof = pact::wavefront_profile(layout.centers[i], s.geom, field.raster, v0, mask,
                                            cfg.n_angles, cfg.ray_step, false);
        lp[i] = pact::detail::fused_patch_loss_grad(ycache[i], prof.w, table, phases,
                                                    cfg.eps_deconv, loss_scale,
                                                    cfg.implicit_xhat_grad, scratch, dw);
        if (w_out) std::memcpy(w_out + static_cast<size_t>(i) * cfg.n_angles, prof.w.data(),
                               sizeof(double) * cfg.n_angles);
        if (dw_out) std::memcpy(dw_out + static_cast<size_t>(i) * cfg.n_angles, dw.data(),
                                sizeof(double) * cfg.n_angles);
        pact::wavefront_grad_trace(layout.centers[i], s.geom, field.raster, v0, mask,
                                   cfg.n_angles, cfg.ray_step, dw, g);
      }
    });
    for (const auto& g : chunk_gv)
      if (!g.empty())
        for (size_t k = 0; k < gv.size(); ++k) gv[k] += g[k];
    double data = 0.0;
    for (int i = 0; i < N; ++i) data += lp[i];
    auto tv = pact::tv_loss(field, cfg.lambda_tv);
    std::vector<double> gm(field.masked_indices.size());
    for (size_t i = 0; i < gm.size(); ++i) gm[i] = gv[field.masked_indices[i]] + tv.grad[i];
    auto grads = pact::backprop_sos(params, field, gm);
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    if (data_term) *data_term = data;
    if (tv_term) *tv_term = tv.value;
    if (loss_patch) std::memcpy(loss_patch, lp.data(), sizeof(double) * N);
    if (sos_out) std::memcpy(sos_out, field.raster.values.data(), sizeof(double) * W * H);
    if (grad_v_masked) std::memcpy(grad_v_masked, gm.data(), sizeof(double) * gm.size());
    if (grad_theta) std::memcpy(grad_theta, grads.data(), sizeof(double) * grads.size());
    if (image) {
      pact::DeconvolveOptions dopt;
      dopt.eps = cfg.eps_deconv;
      dopt.n_angles = cfg.n_angles;
      dopt.ray_step = cfg.ray_step;
      dopt.merge_fwhm = cfg.merge_fwhm;
      dopt.workers = cfg.workers;
      auto img = pact::deconvolve_image(stack, field.raster, s.geom, mask, layout, dopt);
      std::memcpy(image, img.values.data(), sizeof(double) * W * H);
    }
  });
}

// ---- composed (non-fused) path: one patch per call ------------------------
namespace {
pact::TransferStack tstack_of(int K, int P, double pitch, const double* delays, const double* H) {
  pact::TransferStack ts;
  ts.patch_pixels = P;
  ts.pitch = pitch;
  ts.delays.assign(delays, delays + K);
  const size_t P2 = static_cast<size_t>(P) * P;
  const auto* h = reinterpret_cast<const std::complex<double>*>(H);
  for (int j = 0; j < K; ++j) ts.spectra.emplace_back(h + j * P2, h + (j + 1) * P2);
  return ts;
}
pact::PatchSpectra spectra_of(int K, int P, const double* Y) {
  pact::PatchSpectra ps;
  const size_t P2 = static_cast<size_t>(P) * P;
  const auto* y = reinterpret_cast<const std::complex<double>*>(Y);
  for (int j = 0; j < K; ++j) ps.Y.emplace_back(y + j * P2, y + (j + 1) * P2);
  return ps;
}
}  // namespace

// multichannel_deconvolve, deconv.hpp:78-96 (Y, H, X complex128)
int ref_multichannel_deconvolve(int K, int P, const double* Y, const double* H, double eps,
                                double* X) {
  return guarded([&] {
    std::vector<double> d(K, 0.0);
    auto x = pact::multichannel_deconvolve(spectra_of(K, P, Y), tstack_of(K, P, 1.0, d.data(), H), eps);
    std::memcpy(X, x.data(), sizeof(double) * 2 * x.size());
  });
}

// deconv_jacobian_H, deconv.hpp:100-115 -> out[4] = (dre.re, dre.im, dim.re, dim.im)
int ref_deconv_jacobian_H(int K, int P, const double* Y, const double* H, double eps, int j,
                          int bin, double* out) {
  return guarded([&] {
    std::vector<double> d(K, 0.0);
    auto [a, b] = pact::deconv_jacobian_H(spectra_of(K, P, Y), tstack_of(K, P, 1.0, d.data(), H),
                                          eps, j, bin);
    out[0] = a.real();
    out[1] = a.imag();
    out[2] = b.real();
    out[3] = b.imag();
  });
}

// patch_data_loss, optimize.hpp:164-211 (complex<double> Y)
int ref_patch_data_loss(int K, int P, double pitch, const double* Y, const double* H, double eps,
                        double scale, int implicit, double* loss, double* grad_h) {
  return guarded([&] {
    std::vector<double> d(K, 0.0);
    auto r = pact::patch_data_loss(spectra_of(K, P, Y).Y, tstack_of(K, P, pitch, d.data(), H), eps,
                                   scale, implicit != 0);
    *loss = r.value;
    const size_t P2 = static_cast<size_t>(P) * P;
    for (int j = 0; j < K; ++j) std::memcpy(grad_h + 2 * j * P2, r.grad_h[j].data(), sizeof(double) * 2 * P2);
  });
}

// data_loss, optimize.hpp:336-353 over n patches
int ref_data_loss(int n, int K, int P, double pitch, const double* Y, const double* H, double eps,
                  int implicit, double* value, double* grad_h) {
  return guarded([&] {
    std::vector<double> d(K, 0.0);
    const size_t stride = 2 * static_cast<size_t>(K) * P * P;
    std::vector<pact::PatchSpectra> ys;
    std::vector<pact::TransferStack> hs;
    for (int i = 0; i < n; ++i) {
      ys.push_back(spectra_of(K, P, Y + i * stride));
      hs.push_back(tstack_of(K, P, pitch, d.data(), H + i * stride));
    }
    auto r = pact::data_loss(ys, hs, eps, implicit != 0);
    *value = r.value;
    const size_t P2 = static_cast<size_t>(P) * P;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < K; ++j)
        std::memcpy(grad_h + i * stride + 2 * j * P2, r.grad_h[i][j].data(), sizeof(double) * 2 * P2);
  });
}

// transfer_grad_to_wavefront, aberration.hpp:270-313
int ref_transfer_grad_to_wavefront(int A, const double* w, int K, const double* delays, int P,
                                   double pitch, const double* grad_h, double* dw) {
  return guarded([&] {
    pact::WavefrontProfile prof;
    prof.center = {0.0, 0.0};
    prof.n_angles = A;
    prof.w.assign(w, w + A);
    std::vector<std::vector<std::complex<double>>> g;
    const size_t P2 = static_cast<size_t>(P) * P;
    const auto* gh = reinterpret_cast<const std::complex<double>*>(grad_h);
    for (int j = 0; j < K; ++j) g.emplace_back(gh + j * P2, gh + (j + 1) * P2);
    auto out = pact::transfer_grad_to_wavefront(prof, std::vector<double>(delays, delays + K), P,
                                                pitch, g);
    std::memcpy(dw, out.data(), sizeof(double) * A);
  });
}

// wavefront_profile(with_jacobian = true), aberration.hpp:134-186, one centre:
// w[A], row lengths counts[A], and (when pixel != null) the rows concatenated.
// With dw != null also accumulate_wavefront_grad (aberration.hpp:316-326) into grad_v.
int ref_wavefront_jacobian(double cx, double cy, int n_tx, double radius, double offset, int W,
                           int H, double pitch, double ox, double oy, const double* sos,
                           double v0, double mcx, double mcy, double mr, int A, double step,
                           double* w, long* counts, int* pixel, float* dwdv, long cap,
                           const double* dw, double* grad_v) {
  return guarded([&] {
    auto g = grid_of(W, H, pitch, ox, oy);
    auto prof = pact::wavefront_profile({cx, cy}, {n_tx, radius, offset}, raster_of(g, sos), v0,
                                        {{mcx, mcy}, mr}, A, step, true);
    long pos = 0;
    for (int a = 0; a < A; ++a) {
      if (w) w[a] = prof.w[a];
      if (counts) counts[a] = static_cast<long>(prof.jacobian[a].size());
      for (const auto& e : prof.jacobian[a]) {
        if (pixel && pos < cap) {
          pixel[pos] = e.pixel;
          dwdv[pos] = e.dw_dv;
        }
        ++pos;
      }
    }
    if (dw && grad_v) {
      std::vector<double> gv(grad_v, grad_v + static_cast<size_t>(W) * H);
      pact::accumulate_wavefront_grad(prof, std::vector<double>(dw, dw + A), gv);
      std::memcpy(grad_v, gv.data(), sizeof(double) * gv.size());
    }
  });
}

// merge_patches + MergeWindow::make, deconv.hpp:118-164, on make_patch_layout's layout
int ref_merge_patches(int W, int H, double pitch, double ox, double oy, double patch_mm,
                      double overlap, const double* patches, double fwhm, double* image) {
  return guarded([&] {
    auto lay = pact::make_patch_layout(grid_of(W, H, pitch, ox, oy), patch_mm, overlap);
    const size_t P2 = static_cast<size_t>(lay.patch_pixels) * lay.patch_pixels;
    std::vector<std::vector<double>> ps;
    for (int i = 0; i < lay.n_patches(); ++i) ps.emplace_back(patches + i * P2, patches + (i + 1) * P2);
    auto img = pact::merge_patches(ps, lay, pact::MergeWindow::make(fwhm, lay.patch_pixels, pitch));
    std::memcpy(image, img.values.data(), sizeof(double) * img.values.size());
  });
}

// ---- CPU-baseline session (bench.py cpu_baseline leg) ---------------------
// joint_reconstruct's one-time setup (optimize.hpp:374-405: layout, das_stack,
// the complex<float> spectra cache, bin table, delay phases) done once, then
// its step body (optimize.hpp:413-467, Adam included) run on demand with
// per-phase wall-clock timings, so one full iteration can be timed without
// re-running the setup, and the per-patch work can be re-timed at another
// worker count.  Every computation is a reference entry point.
struct RefNfSession {
  pact::SignalSet s;
  pact::GridSpec grid;
  pact::CircularMask mask;
  pact::TrainConfig cfg;
  pact::PatchLayout layout;
  std::vector<std::vector<std::vector<std::complex<float>>>> ycache;
  pact::PatchBinTable table;
  std::vector<std::vector<std::complex<double>>> phases;
  pact::SirenParams params;
  pact::AdamState adam;
  pact::SosField field;  // the last rendered field
  double loss_scale = 0.0;
};

void* ref_nf_session_open(int n_tx, double radius, double offset, int T, double dt, double t0,
                          double v0, const double* sig, int W, int H, double pitch, double ox,
                          double oy, double mcx, double mcy, double mr, const RefTrainCfg* c,
                          double* setup_seconds) {
  RefNfSession* out = nullptr;
  int rc = guarded([&] {
    auto t_start = std::chrono::steady_clock::now();
    auto* h = new RefNfSession;
    h->s = signals_of(n_tx, radius, offset, T, dt, t0, v0, sig);
    h->cfg = train_config_of(c);
    h->grid = grid_of(W, H, pitch, ox, oy);
    h->mask = {{mcx, mcy}, mr};
    h->layout = pact::make_patch_layout(h->grid, h->cfg.patch_mm, h->cfg.overlap);
    const int P = h->layout.patch_pixels, N = h->layout.n_patches();
    const size_t M = h->cfg.delays.size();
    h->loss_scale = 1.0 / (static_cast<double>(N) * M * P * P);
    auto stack = pact::das_stack(h->s, h->grid, v0, h->cfg.delays, h->cfg.workers);
    h->ycache.resize(N);
    pact::parallel_for(N, h->cfg.workers, [&](int i) {
      pact::PatchSpectra ps = pact::extract_patch_spectra_one(stack, h->layout, i);
      h->ycache[i].resize(M);
      for (size_t j = 0; j < M; ++j) {
        h->ycache[i][j].resize(ps.Y[j].size());
        for (size_t b = 0; b < ps.Y[j].size(); ++b)
          h->ycache[i][j][b] = std::complex<float>(ps.Y[j][b]);
      }
    });
    h->params = pact::init_siren(h->cfg.seed, h->cfg.hidden, h->cfg.sine_layers, h->cfg.omega0,
                                 h->cfg.out_scale, v0);
    h->table = pact::PatchBinTable::make(P, h->grid.pitch, h->cfg.n_angles);
    h->phases = pact::detail::make_delay_phases(h->table, h->cfg.delays);
    if (setup_seconds)
      *setup_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    out = h;
  });
  return rc == 0 ? out : nullptr;
}

// One step of optimize.hpp:413-467 with `workers` threads over patches
// [patch_lo, patch_hi) (0/-1 = all).  with_siren = 0 skips render/TV/backprop/
// Adam (times only the per-patch loop on the session's last rendered field).
// t[0..5] = render, per-patch loop, TV, backprop, Adam, total (seconds).
int ref_nf_session_step(void* hp, int workers, int patch_lo, int patch_hi, int with_siren,
                        double* t, double* data_term) {
  return guarded([&] {
    auto* h = static_cast<RefNfSession*>(hp);
    using clk = std::chrono::steady_clock;
    auto sec = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double>(b - a).count();
    };
    pact::SosField& field = h->field;
    const double v0 = h->s.background_sos;
    const int N = h->layout.n_patches();
    const int lo = patch_lo, hi = patch_hi < 0 ? N : std::min(N, patch_hi);
    auto t0 = clk::now();
    if (with_siren || field.raster.values.empty()) field = pact::render_sos(h->params, h->grid, h->mask);
    auto t1 = clk::now();
    const int nw = pact::resolve_workers(workers);
    const int span = hi - lo;
    const int n_chunks = std::max(1, std::min(span, nw * 4));
    const int chunk_len = (span + n_chunks - 1) / n_chunks;
    std::vector<double> patch_loss(N, 0.0);
    std::vector<std::vector<double>> chunk_gv(n_chunks);
    pact::parallel_for(n_chunks, workers, [&](int ck) {
      int a = lo + ck * chunk_len, b = std::min(hi, a + chunk_len);
      if (a >= b) return;
      auto& gv = chunk_gv[ck];
      gv.assign(field.raster.values.size(), 0.0);
      pact::detail::FusedScratch scratch;
      std::vector<double> dw;
      for (int i = a; i < b; ++i) {
        auto prof = pact::wavefront_profile(h->layout.centers[i], h->s.geom, field.raster, v0,
                                            h->mask, h->cfg.n_angles, h->cfg.ray_step, false);
        patch_loss[i] = pact::detail::fused_patch_loss_grad(
            h->ycache[i], prof.w, h->table, h->phases, h->cfg.eps_deconv, h->loss_scale,
            h->cfg.implicit_xhat_grad, scratch, dw);
        pact::wavefront_grad_trace(h->layout.centers[i], h->s.geom, field.raster, v0, h->mask,
                                   h->cfg.n_angles, h->cfg.ray_step, dw, gv);
      }
    });
    double data = 0.0;
    for (int i = 0; i < N; ++i) data += patch_loss[i];
    auto t2 = clk::now();
    auto t3 = t2, t4 = t2, t5 = t2;
    if (with_siren) {
      auto tv = pact::tv_loss(field, h->cfg.lambda_tv);
      t3 = clk::now();
      std::vector<double> gm(field.masked_indices.size(), 0.0);
      for (const auto& gv : chunk_gv) {
        if (gv.empty()) continue;
        for (size_t i = 0; i < gm.size(); ++i) gm[i] += gv[field.masked_indices[i]];
      }
      for (size_t i = 0; i < gm.size(); ++i) gm[i] += tv.grad[i];
      auto grads = pact::backprop_sos(h->params, field, gm);
      t4 = clk::now();
      pact::adam_step(h->params.theta, grads, h->adam, h->cfg.learning_rate, h->cfg.beta1,
                      h->cfg.beta2, h->cfg.adam_eps);
      t5 = clk::now();
    }
    if (t) {
      t[0] = sec(t0, t1);
      t[1] = sec(t1, t2);
      t[2] = sec(t2, t3);
      t[3] = sec(t3, t4);
      t[4] = sec(t4, t5);
      t[5] = sec(t0, t5);
    }
    if (data_term) *data_term = data;
  });
}

void ref_nf_session_close(void* h) { delete static_cast<RefNfSession*>(h); }

// Wall-clock of `reps` calls of das_stack (the CPU baseline of bench.py).
double ref_time_das_stack(int reps, int n_tx, double radius, double offset, int T, double dt,
                          double t0, const double* sig, int W, int H, double pitch, double ox,
                          double oy, double v0, int K, const double* delays, int workers) {
  auto s = signals_of(n_tx, radius, offset, T, dt, t0, v0, sig);
  auto g = grid_of(W, H, pitch, ox, oy);
  std::vector<double> d(delays, delays + K);
  auto t_start = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    auto st = pact::das_stack(s, g, v0, d, workers);
    (void)st;
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
}

// ---- §8(f)-3: file formats, phantoms, PSFs (the pactrec tool path) --------

// pact::builtin_phantom_spec + generate_phantom (phantom.hpp:145-266) with the
// spec mask replaced as pactrec does (pactrec.cpp:196-199).
int ref_generate_phantom(const char* name, int W, int H, double pitch, double bg, double mcx,
                         double mcy, double mr, uint64_t seed, double* pressure, double* sos) {
  return guarded([&] {
    pact::PhantomSpec spec = pact::builtin_phantom_spec(name, bg);
    spec.mask = {{mcx, mcy}, mr};
    auto ph = pact::generate_phantom(pact::GridSpec::centered(W, H, pitch), spec, seed);
    std::memcpy(pressure, ph.pressure.values.data(), sizeof(double) * ph.pressure.values.size());
    std::memcpy(sos, ph.sos.values.data(), sizeof(double) * ph.sos.values.size());
  });
}

// io::read_pgrid (io.hpp:93-112); values may be NULL (header query) or hold cap doubles.
int ref_read_pgrid(const char* path, int* W, int* H, double* geo /* pitch, ox, oy */,
                   double* values, size_t cap) {
  return guarded([&] {
    auto g = pact::io::read_pgrid(path);
    *W = g.width;
    *H = g.height;
    geo[0] = g.pitch;
    geo[1] = g.origin.x;
    geo[2] = g.origin.y;
    if (values) std::memcpy(values, g.values.data(), sizeof(double) * std::min(cap, g.values.size()));
  });
}

int ref_write_pgrid(const char* path, int W, int H, double pitch, double ox, double oy,
                    const double* values) {
  return guarded([&] { pact::io::write_pgrid(path, raster_of(grid_of(W, H, pitch, ox, oy), values)); });
}

// io::read_sigset (io.hpp:129-150): meta = {dt, t0, radius, angle_offset, background_sos}.
int ref_read_sigset(const char* path, int* n_tx, int* T, double* meta, double* data, size_t cap) {
  return guarded([&] {
    auto s = pact::io::read_sigset(path);
    *n_tx = s.geom.n_transducers;
    *T = s.n_samples;
    meta[0] = s.dt;
    meta[1] = s.t0;
    meta[2] = s.geom.radius;
    meta[3] = s.geom.angle_offset;
    meta[4] = s.background_sos;
    if (data) std::memcpy(data, s.data.data(), sizeof(double) * std::min(cap, s.data.size()));
  });
}

int ref_write_sigset(const char* path, int n_tx, int T, const double* meta, const double* data) {
  return guarded([&] {
    pact::SignalSet s;
    s.geom = {n_tx, meta[2], meta[3]};
    s.n_samples = T;
    s.dt = meta[0];
    s.t0 = meta[1];
    s.background_sos = meta[4];
    s.data.assign(data, data + static_cast<size_t>(n_tx) * T);
    pact::io::write_sigset(path, s);
  });
}

// load_sirn / write_sirn (nfield.hpp:235-289): shape = {in_dim, hidden, n_hidden_layers},
// scal = {omega0, out_scale, v0}; theta may be NULL (header query).
int ref_load_sirn(const char* path, int* shape, double* scal, double* theta, size_t cap) {
  return guarded([&] {
    auto p = pact::load_sirn(path);
    shape[0] = p.in_dim;
    shape[1] = p.hidden;
    shape[2] = p.n_hidden_layers;
    scal[0] = p.omega0;
    scal[1] = p.out_scale;
    scal[2] = p.v0;
    if (theta) std::memcpy(theta, p.theta.data(), sizeof(double) * std::min(cap, p.theta.size()));
  });
}

int ref_write_sirn(const char* path, int hidden, int layers, double omega0, double out_scale,
                   double v0, const double* theta) {
  return guarded([&] {
    auto p = siren_of(hidden, layers, omega0, out_scale, v0, theta);
    pact::write_sirn(path, p);
  });
}

// psf_from_transfer (aberration.hpp:407-445): spectrum as interleaved re, im.
int ref_psf_from_transfer(int P, double pitch, const double* spectrum, double* psf) {
  return guarded([&] {
    std::vector<std::complex<double>> sp(static_cast<size_t>(P) * P);
    for (size_t i = 0; i < sp.size(); ++i) sp[i] = {spectrum[2 * i], spectrum[2 * i + 1]};
    auto r = pact::psf_from_transfer(sp, P, pitch);
    std::memcpy(psf, r.values.data(), sizeof(double) * r.values.size());
  });
}

// simulate_signals (phantom.hpp:282-362) with the automatic window and
// SimulateOptions::spreading, as `pactrec simulate` calls it.  meta = {t0, T}
// out; out may be NULL (window query) or hold cap doubles.
int ref_simulate_auto(int W, int H, double pitch, double ox, double oy, const double* pressure,
                      const double* sos, double mcx, double mcy, double mr, double background_sos,
                      int n_tx, double radius, double offset, double pulse_sigma, double dt,
                      int spreading, double ray_step, double* meta, double* out, size_t cap) {
  return guarded([&] {
    auto g = grid_of(W, H, pitch, ox, oy);
    pact::Phantom ph;
    ph.pressure = raster_of(g, pressure);
    ph.sos = raster_of(g, sos);
    ph.mask = {{mcx, mcy}, mr};
    ph.background_sos = background_sos;
    pact::SimulateOptions opt;
    opt.pulse_sigma = pulse_sigma;
    opt.dt = dt;
    opt.spreading = spreading != 0;
    opt.ray_step = ray_step;
    auto s = pact::simulate_signals(ph, {n_tx, radius, offset}, opt);
    meta[0] = s.t0;
    meta[1] = s.n_samples;
    if (out) std::memcpy(out, s.data.data(), sizeof(double) * std::min(cap, s.data.size()));
  });
}

double ref_water_sos(double t) { return pact::water_sos(t); }

}  // extern "C"
