// Drop-in host API — the self-supervised training loop (reference:
// proj/include/pact/optimize.hpp:40-494): TV, Adam and joint_reconstruct.
#ifndef PACT_B200_OPTIMIZE_HPP
#define PACT_B200_OPTIMIZE_HPP

#include <vector>

#include "pact/deconv.hpp"
#include "pact/nfield.hpp"

namespace pact {

struct LossReport {
  int epoch = 0;
  double data_term = 0.0, tv_term = 0.0, total = 0.0;
  double wall_time = 0.0;  // seconds spent in this epoch
};

struct TrainConfig {
  int epochs = 10;
  int steps_per_epoch = 30;
  double learning_rate = 1e-3, beta1 = 0.9, beta2 = 0.999, adam_eps = 1e-8;
  double lambda_tv = 3e9;
  std::vector<double> delays = make_delays(-0.8, 0.8, 32);
  double eps_deconv = 1e-3;
  int n_angles = 512;
  double ray_step = 0.05;
  uint64_t seed = 0;
  int hidden = 64, sine_layers = 2;
  double omega0 = 30.0, out_scale = 100.0;
  double patch_mm = 3.2, overlap = 0.75, merge_fwhm = 1.5;
  bool implicit_xhat_grad = true;
  int workers = 0;

  pact_train_config c() const {
    pact_train_config t{};
    t.epochs = epochs;
    t.steps_per_epoch = steps_per_epoch;
    t.learning_rate = learning_rate;
    t.beta1 = beta1;
    t.beta2 = beta2;
    t.adam_eps = adam_eps;
    t.lambda_tv = lambda_tv;
    t.n_delays = static_cast<int32_t>(delays.size());
    t.delays = delays.data();
    t.eps_deconv = eps_deconv;
    t.n_angles = n_angles;
    t.ray_step = ray_step;
    t.seed = seed;
    t.hidden = hidden;
    t.sine_layers = sine_layers;
    t.omega0 = omega0;
    t.out_scale = out_scale;
    t.patch_mm = patch_mm;
    t.overlap = overlap;
    t.merge_fwhm = merge_fwhm;
    t.implicit_xhat_grad = implicit_xhat_grad ? 1 : 0;
    t.workers = workers;
    t.use_cuda_graph = 1;
    return t;
  }
};

struct PatchLossResult {
  double value = 0.0;
  std::vector<std::vector<cplx>> grad_h;  // dL/dRe H + j dL/dIm H, per delay per bin
};

/// patch_data_loss (optimize.hpp:155-211): |k|-weighted residual loss of one
/// patch and its gradient w.r.t. H (explicit + optional implicit term through
/// X-hat), fp64 on the GPU.  YScalar is float (the training cache) or double.
template <typename YScalar>
PatchLossResult patch_data_loss(const std::vector<std::vector<std::complex<YScalar>>>& Y,
                                const TransferStack& H, double eps, double scale,
                                bool implicit_grad) {
  const size_t M = Y.size();
  if (M != H.spectra.size()) throw ValidationError("data_loss: Y/H channel mismatch");
  if (M == 0) throw ValidationError("data_loss: no channels");
  const int P = H.patch_pixels;
  const size_t P2 = static_cast<size_t>(P) * P;
  std::vector<cplx> y;
  y.reserve(M * P2);
  for (const auto& c : Y) {
    if (c.size() != P2) throw ValidationError("data_loss: Y/H channel mismatch");
    for (const auto& v : c) y.push_back(cplx(v));
  }
  cuda::Buffer<double> dY(2 * M * P2), dH(2 * M * P2), dG(2 * M * P2), loss(1);
  cuda::check(pact_upload(cuda::context(), dY.ptr, y.data(), sizeof(cplx) * y.size()));
  detail::upload_c128(dH, H.spectra);
  cuda::check(pact_patch_data_loss(cuda::context(), 1, static_cast<int>(M), P, H.pitch, dY.ptr,
                                   dH.ptr, eps, scale, implicit_grad ? 1 : 0, loss.ptr, dG.ptr));
  PatchLossResult res;
  loss.download(&res.value);
  std::vector<cplx> g(M * P2);
  dG.download(reinterpret_cast<double*>(g.data()));
  for (size_t j = 0; j < M; ++j) res.grad_h.emplace_back(g.begin() + j * P2, g.begin() + (j + 1) * P2);
  return res;
}

struct DataLossResult {
  double value = 0.0;
  std::vector<std::vector<std::vector<cplx>>> grad_h;  // per patch, per delay, per bin
};

/// data_loss (optimize.hpp:329-353): all patches, normalised by N * M * P^2.
inline DataLossResult data_loss(const std::vector<PatchSpectra>& ys,
                                const std::vector<TransferStack>& hs, double eps,
                                bool implicit_grad = true) {
  if (ys.size() != hs.size()) throw ValidationError("data_loss: patch count mismatch");
  if (ys.empty()) throw ValidationError("data_loss: no patches");
  const size_t N = ys.size(), M = ys[0].Y.size();
  const int P = hs[0].patch_pixels;
  const size_t P2 = static_cast<size_t>(P) * P, per = 2 * M * P2;
  for (size_t i = 0; i < N; ++i)
    if (ys[i].Y.size() != M || hs[i].spectra.size() != M)
      throw ValidationError("data_loss: Y/H channel mismatch");
  if (M == 0) throw ValidationError("data_loss: no channels");
  cuda::Buffer<double> dY(per * N), dH(per * N), dG(per * N);
  for (size_t i = 0; i < N; ++i) {
    detail::upload_c128(dY, ys[i].Y, i * per);
    detail::upload_c128(dH, hs[i].spectra, i * per);
  }
  DataLossResult out;
  cuda::check(pact_data_loss(cuda::context(), static_cast<int>(N), static_cast<int>(M), P,
                             hs[0].pitch, dY.ptr, dH.ptr, eps, implicit_grad ? 1 : 0, &out.value,
                             nullptr, dG.ptr));
  std::vector<cplx> g(N * M * P2);
  dG.download(reinterpret_cast<double*>(g.data()));
  out.grad_h.resize(N);
  for (size_t i = 0; i < N; ++i)
    for (size_t j = 0; j < M; ++j)
      out.grad_h[i].emplace_back(g.begin() + (i * M + j) * P2, g.begin() + (i * M + j + 1) * P2);
  return out;
}

struct AdamState {
  std::vector<double> m, v;
  long t = 0;
};

/// adam_step (optimize.hpp:87-110) on the GPU (fp64).
inline void adam_step(std::vector<double>& params, const std::vector<double>& grads,
                      AdamState& state, double lr, double beta1, double beta2, double eps) {
  if (grads.size() != params.size())
    throw ValidationError("adam_step: gradient size does not match parameters");
  if (state.m.empty()) {
    state.m.assign(params.size(), 0.0);
    state.v.assign(params.size(), 0.0);
  }
  if (state.m.size() != params.size())
    throw ValidationError("adam_step: state size does not match parameters");
  const size_t n = params.size();
  cuda::Buffer<double> p(n), g(n), m(n), v(n);
  p.upload(params.data());
  g.upload(grads.data());
  m.upload(state.m.data());
  v.upload(state.v.data());
  cuda::check(pact_adam_step(cuda::context(), static_cast<int64_t>(n), p.ptr, g.ptr, m.ptr, v.ptr,
                             state.t + 1, lr, beta1, beta2, eps));
  state.t += 1;
  p.download(params.data());
  m.download(state.m.data());
  v.download(state.v.data());
}

struct TvLossResult {
  double value = 0.0;
  std::vector<double> grad;  // per masked pixel, field order
};

/// tv_loss (optimize.hpp:120-153).
inline TvLossResult tv_loss(const SosField& field, double lambda) {
  GridSpec grid = field.raster.spec();
  pact_grid g = grid.c();
  pact_mask m = field.mask.c();
  // deviation from the first value keeps fp32 resolution (differences agree)
  double ref = field.raster.values.empty() ? 0.0 : field.raster.values[0];
  cuda::Buffer<float> r(field.raster.values.size());
  cuda::upload_f32(r, field.raster.values, ref);
  cuda::Buffer<float> gr(field.masked_indices.size());
  TvLossResult out;
  cuda::check(pact_tv_loss(cuda::context(), &g, &m, r.ptr, lambda, &out.value, gr.ptr));
  out.grad = cuda::download_f64(gr);
  return out;
}

struct JointResult {
  RasterGrid image;
  RasterGrid sos;
  std::vector<LossReport> reports;
  SirenParams params;
};

/// joint_reconstruct (optimize.hpp:367-494) on one B200: one-time DAS stack
/// and spectra, then every iteration as a CUDA graph, then the final
/// deconvolution.  Reports match the reference per epoch.
inline JointResult joint_reconstruct(const SignalSet& signals, const GridSpec& grid,
                                     const CircularMask& mask, const TrainConfig& cfg) {
  signals.validate();
  pact_ring r = signals.geom.c();
  pact_signal_meta meta = signals.meta();
  pact_grid g = grid.c();
  pact_mask m = mask.c();
  pact_train_config tc = cfg.c();
  cuda::Buffer<float> sig(signals.data.size());
  cuda::upload_f32(sig, signals.data);
  pact_trainer* tr = nullptr;
  cuda::check(pact_trainer_create(cuda::context(), &r, &meta, sig.ptr, &g, &m, &tc, &tr));
  struct Guard {
    pact_trainer* t;
    ~Guard() { pact_trainer_destroy(t); }
  } guard{tr};
  JointResult out;
  for (int e = 1; e <= cfg.epochs; ++e) {
    double rep[4];
    cuda::check(pact_trainer_run_epoch(tr, e, rep));
    out.reports.push_back({e, rep[0], rep[1], rep[2], rep[3]});
  }
  const size_t npx = static_cast<size_t>(grid.width) * grid.height;
  cuda::Buffer<float> img(npx), sos(npx);
  cuda::check(pact_trainer_finish(tr, img.ptr, sos.ptr));
  out.image = RasterGrid::zeros(grid);
  out.image.values = cuda::download_f64(img);
  out.sos = RasterGrid::zeros(grid);
  out.sos.values = cuda::download_f64(sos);
  out.params = init_siren(cfg.seed, cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale,
                          signals.background_sos);
  cuda::check(pact_trainer_get_theta(tr, out.params.theta.data()));
  return out;
}

}  // namespace pact

#endif
