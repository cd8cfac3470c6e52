// The drop-in C++ API (paper_2409_10876_b200/include/pact/*.hpp, same names as
// the reference's proj/include/pact) exercised the way the reference's own
// Catch2 suites exercise it (proj/tests/test_*.cpp), on the GPU, with the CPU
// oracle (oracle/pact_oracle.c) as the checker where a comparison is needed.
// Built and run by tests/test_cpp_dropin.py.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "pact/beamform.hpp"
#include "pact/evaluate.hpp"
#include "pact/core.hpp"
#include "pact/deconv.hpp"
#include "pact/nfield.hpp"
#include "pact/optimize.hpp"
#include "pact/phantom.hpp"
#include "pact_oracle.h"

using namespace pact;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
    }                                                                            \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1));
}

static const RingGeometry kRing{128, 50.0, 0.0};

// One point source at `pos` simulated by the oracle (simulate_signals, phantom.hpp:282-362).
static SignalSet point_signals(Vec2 pos) {
  GridSpec g = GridSpec::centered(255, 255, 0.1);
  std::vector<double> pr(255 * 255, 0.0), sos(255 * 255, 1500.0);
  Vec2 q = g.pixel(pos);
  pr[std::lround(q.y) * 255 + std::lround(q.x)] = 1.0;
  SignalSet s;
  s.geom = kRing;
  s.n_samples = 1400;
  s.dt = 25e-9;
  s.t0 = 32e-6;
  s.background_sos = 1500.0;
  s.data.resize(128 * 1400);
  orc_simulate_signals(255, 255, 0.1, g.origin.x, g.origin.y, pr.data(), sos.data(), 0, 0, 10.0,
                       1500.0, 128, 50.0, 0.0, 100e-9, 25e-9, 32e-6, 1400, 0.05, 1,
                       s.data.data());
  for (double& v : s.data) v = static_cast<float>(v);
  return s;
}

static std::pair<int, int> argmax_abs(const RasterGrid& img) {
  int bx = 0, by = 0;
  double best = -1;
  for (int y = 0; y < img.height; ++y)
    for (int x = 0; x < img.width; ++x)
      if (std::abs(img.at(x, y)) > best) {
        best = std::abs(img.at(x, y));
        bx = x;
        by = y;
      }
  return {bx, by};
}

static void test_beamform() {
  // test_beamform.cpp:55-70
  SignalSet s = point_signals({0.0, 0.0});
  GridSpec grid = GridSpec::centered(65, 65, 0.1);
  auto [bx, by] = argmax_abs(das(s, grid, 1500.0, 0.0));
  CHECK(bx == 32 && by == 32);
  RasterGrid ring = das(s, grid, 1500.0, 0.5);
  auto [rx, ry] = argmax_abs(ring);
  double r = ring.world(rx, ry).norm();
  CHECK(r > 0.35 && r < 0.65);
  // test_beamform.cpp:99-111: stack element == das at that delay (bitwise)
  GridSpec small = GridSpec::centered(33, 33, 0.1);
  std::vector<double> d = {-0.4, 0.0, 0.3};
  DasStack st = das_stack(s, small, 1500.0, d);
  CHECK(st.n_delays() == 3);
  for (int j = 0; j < 3; ++j) CHECK(st.images[j].values == das(s, small, 1500.0, d[j]).values);
  CHECK(throws<ValidationError>([&] { das_stack(s, small, 1500.0, {0.1, 0.1}); }));
  CHECK(throws<ValidationError>([&] { das_stack(s, small, -1.0, {0.0}); }));
  // parity with the oracle on random signals (north_star tolerance 1e-4)
  std::mt19937_64 rng(9);
  std::normal_distribution<double> nd;
  for (double& v : s.data) v = static_cast<float>(nd(rng));
  std::vector<double> want(3 * 33 * 33);
  orc_das_stack(128, 50.0, 0.0, 1400, 25e-9, 32e-6, s.data.data(), 33, 33, 0.1, small.origin.x,
                small.origin.y, 1500.0, 3, d.data(), 1, want.data());
  st = das_stack(s, small, 1500.0, d);
  std::vector<double> got;
  for (auto& im : st.images) got.insert(got.end(), im.values.begin(), im.values.end());
  CHECK(rel_l2(got, want) <= 1e-4);
  // dual_sos_das (beamform.hpp:124-150): parity with the oracle, the body_sos = v0
  // degenerate case (test_beamform.cpp:133-141) and the validation messages
  BodyModel body{{1.0, -0.5}, 6.0, 1580.0};
  std::vector<double> dwant(33 * 33);
  orc_dual_sos_das(128, 50.0, 0.0, 1400, 25e-9, 32e-6, s.data.data(), 33, 33, 0.1, small.origin.x,
                   small.origin.y, 1500.0, body.center.x, body.center.y, body.radius,
                   body.body_sos, dwant.data());
  CHECK(rel_l2(dual_sos_das(s, small, 1500.0, body).values, dwant) <= 1e-4);
  RasterGrid same = dual_sos_das(s, small, 1500.0, BodyModel{{0.0, 0.0}, 8.0, 1500.0});
  CHECK(rel_l2(same.values, das(s, small, 1500.0, 0.0).values) <= 1e-6);
  CHECK(throws<ValidationError>([&] { dual_sos_das(s, small, 1500.0, BodyModel{{0, 0}, 0.0, 1500.0}); }));
  CHECK(throws<ValidationError>([&] { dual_sos_das(s, small, 1500.0, BodyModel{{45, 0}, 8.0, 1500.0}); }));
}

static void test_evaluate() {
  // test_evaluate.cpp:38-112 through the GPU metrics
  GridSpec g = GridSpec::centered(32, 32, 0.1);
  RasterGrid truth = RasterGrid::zeros(g);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> u(0, 1);
  for (double& v : truth.values) v = u(rng);
  CHECK(std::isinf(psnr(truth, truth, 1.0)));
  RasterGrid off = truth;
  for (double& v : off.values) v += 0.1;
  CHECK(std::abs(psnr(off, truth, 1.0) - 20.0) < 1e-9);
  CHECK(std::abs(ssim(truth, truth, 1.0) - 1.0) < 1e-12);
  CHECK(throws<ValidationError>([&] { psnr(truth, truth, 0.0); }));
  CHECK(throws<ValidationError>([&] { ssim(RasterGrid::zeros(GridSpec::centered(8, 8, 0.1)),
                                           RasterGrid::zeros(GridSpec::centered(8, 8, 0.1)), 1.0); }));
  GridSpec g33 = GridSpec::centered(33, 33, 0.1);
  CHECK(std::abs(sos_rmse_masked(RasterGrid::constant(g33, 1510.0), RasterGrid::constant(g33, 1500.0),
                                 CircularMask{{0, 0}, 1.0}) - 10.0) < 1e-12);
}

static void test_nfield() {
  // test_nfield.cpp:26-32
  CHECK(init_siren(0).param_count() == 4417);
  CHECK(init_siren(0, 16, 2).param_count() == 337);
  CHECK(siren_param_count(2, 64, 2) == 4417);
  SirenParams p = init_siren(2, 8, 2, 30.0, 60.0, 1500.0);
  std::vector<double> want(p.theta.size());
  orc_init_siren(2, 8, 2, 30.0, 60.0, 1500.0, want.data());
  CHECK(p.theta == want);  // bit-identical initialisation
  GridSpec grid = GridSpec::centered(64, 64, 0.1);
  CircularMask mask{{0.0, 0.0}, 2.6};
  SosField f = render_sos(p, grid, mask);
  std::vector<double> ref(64 * 64);
  orc_render_sos(8, 2, 30.0, 60.0, 1500.0, p.theta.data(), 64, 64, 0.1, grid.origin.x,
                 grid.origin.y, 0, 0, 2.6, ref.data(), nullptr);
  CHECK(rel_l2(f.raster.values, ref) <= 1e-6);
  std::vector<double> g(f.masked_indices.size());
  for (size_t i = 0; i < g.size(); ++i) g[i] = std::sin(0.01 * i);
  std::vector<double> grad = backprop_sos(p, f, g), gref(p.theta.size());
  orc_backprop_sos(8, 2, 30.0, 60.0, 1500.0, p.theta.data(), 64, 64, 0.1, grid.origin.x,
                   grid.origin.y, 0, 0, 2.6, g.data(), gref.data());
  CHECK(rel_l2(grad, gref) <= 1e-3);
}

static void test_aberration() {
  // transfer function identities (test_aberration.cpp:165-191), fp32 margins
  const int P = 32;
  WavefrontProfile zero;
  zero.n_angles = 64;
  zero.w.assign(64, 0.0);
  TransferStack t0 = transfer_stack(zero, {0.0}, P, 0.1);
  double e = 0;
  for (auto& h : t0.spectra[0]) e = std::max(e, std::abs(h - cplx(1.0)));
  CHECK(e < 1e-6);
  TransferStack t1 = transfer_stack(zero, {0.35}, P, 0.1);
  e = 0;
  for (int by = 0; by < P; ++by)
    for (int bx = 0; bx < P; ++bx) {
      double s = 2 * M_PI / (P * 0.1);
      double k = std::hypot(s * (bx <= P / 2 ? bx : bx - P), s * (by <= P / 2 ? by : by - P));
      e = std::max(e, std::abs(t1.spectra[0][by * P + bx] - cplx(std::cos(k * 0.35))));
    }
  CHECK(e < 1e-5);
  WavefrontProfile flat = zero;
  flat.w.assign(64, 0.21);
  TransferStack t2 = transfer_stack(flat, {0.21}, P, 0.1);
  e = 0;
  for (auto& h : t2.spectra[0]) e = std::max(e, std::abs(h - cplx(1.0)));
  CHECK(e < 1e-5);
  // conjugate symmetry, |H| <= 1, DC = 1 (193-214)
  std::mt19937_64 rng(3);
  std::uniform_real_distribution<double> u(-0.5, 0.5);
  WavefrontProfile p = zero;
  for (double& w : p.w) w = u(rng);
  TransferStack ts = transfer_stack(p, {-0.3, 0.0, 0.4}, P, 0.1);
  for (const auto& h : ts.spectra) {
    double asym = 0, mx = 0;
    for (int by = 0; by < P; ++by)
      for (int bx = 0; bx < P; ++bx) {
        size_t i = by * P + bx, j = ((P - by) % P) * P + (P - bx) % P;
        asym = std::max(asym, std::abs(h[i] - std::conj(h[j])));
        mx = std::max(mx, std::abs(h[i]));
      }
    CHECK(asym < 1e-6);
    CHECK(mx <= 1.0 + 1e-6);
    CHECK(std::abs(h[0] - cplx(1.0)) < 1e-7);
  }
  // wavefront at the centre of a 5 mm disc is (1 - v0/v1) r (92-98)
  GridSpec g = GridSpec::centered(509, 509, 0.05);
  RasterGrid sos = RasterGrid::constant(g, 1500.0);
  for (int y = 0; y < g.height; ++y)
    for (int x = 0; x < g.width; ++x) {
      int in = 0;
      for (int sy = 0; sy < 8; ++sy)
        for (int sx = 0; sx < 8; ++sx) {
          Vec2 q = g.world(x - 0.5 + (sx + 0.5) / 8, y - 0.5 + (sy + 0.5) / 8);
          in += q.norm() <= 5.0;
        }
      sos.at(x, y) = 1500.0 + 50.0 * in / 64.0;
    }
  RingGeometry ring{512, 50.0, 0.0};
  WavefrontProfile w = wavefront_profile({0, 0}, ring, sos, 1500.0, {{0, 0}, 10.0}, 512, 0.05, false);
  double want = (1.0 - 1500.0 / 1550.0) * 5.0;
  double worst = 0;
  for (double v : w.w) worst = std::max(worst, std::abs(v - want) / want);
  CHECK(worst < 1e-3);
  CHECK(throws<ValidationError>(
      [&] { wavefront_profile({60.0, 0.0}, ring, sos, 1500.0, {{0, 0}, 10.0}, 64, 0.05, false); }));
  CHECK(throws<ValidationError>(
      [&] { wavefront_profile({1.0, 2.0}, ring, sos, 1500.0, {{0, 0}, 10.0}, 3, 0.05, false); }));
}

static void test_optimize() {
  // Adam (test_optimize.cpp:27-66)
  std::vector<double> params{1.0, -2.0, 0.5};
  AdamState st;
  adam_step(params, {0.0, 0.0, 0.0}, st, 1e-3, 0.9, 0.999, 1e-8);
  CHECK(st.t == 1 && params == (std::vector<double>{1.0, -2.0, 0.5}));
  params = {0.0, 0.0};
  st = AdamState{};
  adam_step(params, {3.7, -0.002}, st, 1e-3, 0.9, 0.999, 1e-8);
  CHECK(std::abs(params[0] + 1e-3) < 1e-7 && std::abs(params[1] - 1e-3) < 1e-5);
  params = {0.0};
  st = AdamState{};
  double prev = 0, step = 0;
  for (int t = 0; t < 200; ++t) {
    adam_step(params, {0.42}, st, 1e-3, 0.9, 0.999, 1e-8);
    step = prev - params[0];
    prev = params[0];
  }
  CHECK(std::abs(step - 1e-3) < 1e-6);
  st = AdamState{};
  CHECK(throws<NumericalError>([&] { adam_step(params, {NAN}, st, 1e-3, 0.9, 0.999, 1e-8); }));
  // TV: constant field is zero; a step edge gives lambda h L (97-104)
  GridSpec g = GridSpec::centered(12, 12, 0.1);
  SosField f;
  f.mask = {{0, 0}, 10.0};
  f.raster = RasterGrid::constant(g, 1500.0);
  for (int i = 0; i < 144; ++i) {
    f.masked_indices.push_back(i);
    f.coords.push_back({0, 0});
  }
  TvLossResult tv = tv_loss(f, 2.0);
  CHECK(tv.value == 0.0);
  for (int y = 0; y < 12; ++y)
    for (int x = 0; x < 12; ++x) f.raster.at(x, y) = g.world(x, y).x > 0 ? 7.5 : 0.0;
  tv = tv_loss(f, 0.3);
  CHECK(std::abs(tv.value - 0.3 * 7.5 * 12) < 1e-5);
}

static void test_joint_reconstruct() {
  // a small joint reconstruction against the oracle's (optimize.hpp:367-494)
  SignalSet s = point_signals({0.3, -0.2});
  GridSpec grid = GridSpec::centered(64, 64, 0.1);
  CircularMask mask{{0.0, 0.0}, 2.6};
  TrainConfig cfg;
  cfg.epochs = 2;
  cfg.steps_per_epoch = 2;
  cfg.delays = make_delays(-0.4, 0.4, 4);
  cfg.n_angles = 32;
  cfg.ray_step = 0.1;
  cfg.patch_mm = 3.2;
  cfg.overlap = 0.0;
  cfg.hidden = 8;
  cfg.out_scale = 60.0;
  cfg.lambda_tv = 1e-4;
  JointResult jr = joint_reconstruct(s, grid, mask, cfg);
  OrcTrainCfg oc{cfg.epochs, cfg.steps_per_epoch, cfg.learning_rate, cfg.beta1, cfg.beta2,
                 cfg.adam_eps, cfg.lambda_tv, static_cast<int>(cfg.delays.size()),
                 cfg.delays.data(), cfg.eps_deconv, cfg.n_angles, cfg.ray_step, cfg.seed,
                 cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale, cfg.patch_mm,
                 cfg.overlap, cfg.merge_fwhm, 1, 1};
  std::vector<double> reps(4 * cfg.epochs), img(64 * 64), sos(64 * 64), th(jr.params.theta.size());
  orc_joint_reconstruct(128, 50.0, 0.0, s.n_samples, s.dt, s.t0, 1500.0, s.data.data(), 64, 64,
                        0.1, grid.origin.x, grid.origin.y, 0, 0, 2.6, &oc, reps.data(),
                        img.data(), sos.data(), th.data());
  CHECK(jr.reports.size() == 2u);
  for (int e = 0; e < cfg.epochs; ++e) {
    CHECK(std::abs(jr.reports[e].data_term - reps[4 * e]) <= 1e-3 * std::abs(reps[4 * e]));
    CHECK(std::abs(jr.reports[e].total - (jr.reports[e].data_term + jr.reports[e].tv_term)) <=
          1e-9 * std::abs(jr.reports[e].total));
  }
  CHECK(rel_l2(jr.image.values, img) <= 1e-3);
  CHECK(rel_l2(jr.params.theta, th) <= 1e-3);
}

// ---- the composed path (deconv.hpp:78-164, optimize.hpp:155-353,
// aberration.hpp:134-326) and the reference's contracts for it -------------

// forward 2-D DFT of a real P x P patch (test-side helper for the spectra)
static std::vector<cplx> dft2(const std::vector<double>& x, int P) {
  std::vector<cplx> out(P * P);
  for (int ky = 0; ky < P; ++ky)
    for (int kx = 0; kx < P; ++kx) {
      cplx acc = 0.0;
      for (int y = 0; y < P; ++y)
        for (int xx = 0; xx < P; ++xx)
          acc += x[y * P + xx] * std::polar(1.0, -2.0 * M_PI * (double(kx) * xx + double(ky) * y) / P);
      out[ky * P + kx] = acc;
    }
  return out;
}

static WavefrontProfile random_profile(std::mt19937_64& rng, int A, double lo, double hi) {
  std::uniform_real_distribution<double> u(lo, hi);
  WavefrontProfile p;
  p.center = {0, 0};
  p.n_angles = A;
  p.w.resize(A);
  for (double& w : p.w) w = u(rng);
  return p;
}

static void test_deconv_composed() {
  // deconvolution Jacobian w.r.t. H vs finite differences (test_deconv.cpp:149-181)
  const int P = 8, M = 3;
  std::mt19937_64 rng(9);
  std::uniform_real_distribution<double> u(-1, 1);
  TransferStack hs = transfer_stack(random_profile(rng, 16, -0.2, 0.2), make_delays(-0.3, 0.3, M),
                                    P, 0.1);
  PatchSpectra ys;
  for (int j = 0; j < M; ++j) {
    std::vector<double> x(P * P);
    for (double& v : x) v = u(rng);
    ys.Y.push_back(dft2(x, P));
  }
  const double eps = 1e-3;
  std::uniform_int_distribution<size_t> pick_bin(0, P * P - 1);
  std::uniform_int_distribution<int> pick_ch(0, M - 1);
  double worst = 0.0;
  for (int trial = 0; trial < 20; ++trial) {
    size_t bin = pick_bin(rng);
    int j = pick_ch(rng);
    auto [dre, dim] = deconv_jacobian_H(ys, hs, eps, j, bin);
    const double h = 1e-6;
    TransferStack hp = hs, hm = hs;
    hp.spectra[j][bin] += h;
    hm.spectra[j][bin] -= h;
    cplx fd_re = (multichannel_deconvolve(ys, hp, eps)[bin] - multichannel_deconvolve(ys, hm, eps)[bin]) / (2 * h);
    hp = hs;
    hm = hs;
    hp.spectra[j][bin] += cplx(0, h);
    hm.spectra[j][bin] -= cplx(0, h);
    cplx fd_im = (multichannel_deconvolve(ys, hp, eps)[bin] - multichannel_deconvolve(ys, hm, eps)[bin]) / (2 * h);
    double scale = std::max(1.0, std::abs(dre) + std::abs(dim));
    worst = std::max({worst, std::abs(fd_re - dre) / scale, std::abs(fd_im - dim) / scale});
  }
  std::printf("  deconv Jacobian vs FD: max err %.2e (bar 1e-4)\n", worst);
  CHECK(worst < 1e-4);
  // identity channel passes through, exact noiseless recovery (test_deconv.cpp:114-147)
  TransferStack one = hs;
  for (auto& c : one.spectra) std::fill(c.begin(), c.end(), cplx(1.0));
  std::vector<cplx> x = multichannel_deconvolve(ys, one, 0.0), want(P * P, 0.0);
  for (int j = 0; j < M; ++j)
    for (int b = 0; b < P * P; ++b) want[b] += ys.Y[j][b] / double(M);
  double e = 0, xm = 0;
  for (int b = 0; b < P * P; ++b) {
    e = std::max(e, std::abs(x[b] - want[b]));
    xm = std::max(xm, std::abs(want[b]));
  }
  CHECK(e < 1e-12 * xm);
  PatchSpectra yc = ys;
  for (int j = 0; j < M; ++j)
    for (int b = 0; b < P * P; ++b) yc.Y[j][b] = hs.spectra[j][b] * ys.Y[0][b];
  std::vector<cplx> rec = multichannel_deconvolve(yc, hs, 0.0);
  e = xm = 0;
  for (int b = 0; b < P * P; ++b) {
    if (std::norm(hs.spectra[0][b]) + std::norm(hs.spectra[1][b]) + std::norm(hs.spectra[2][b]) < 1e-6)
      continue;
    e = std::max(e, std::abs(rec[b] - ys.Y[0][b]));
    xm = std::max(xm, std::abs(ys.Y[0][b]));
  }
  CHECK(e < 1e-6 * xm);
  CHECK(throws<ValidationError>([&] { multichannel_deconvolve(ys, TransferStack{}, 1e-3); }));
  // merge partition of unity (test_deconv.cpp:259-277)
  GridSpec g = GridSpec::centered(64, 64, 0.1);
  PatchLayout lay = make_patch_layout(g, 3.2, 0.5);
  const int Pm = lay.patch_pixels;
  std::vector<std::vector<double>> ones(lay.n_patches(), std::vector<double>(Pm * Pm, 1.0));
  RasterGrid m = merge_patches(ones, lay, MergeWindow::make(1.5, Pm, g.pitch));
  double dev = 0;
  for (double v : m.values) dev = std::max(dev, std::abs(v - 1.0));
  CHECK(dev < 2e-6);
  CHECK(throws<ValidationError>([&] { merge_patches({}, lay, MergeWindow::make(1.5, Pm, g.pitch)); }));
  CHECK(throws<ValidationError>([&] { MergeWindow::make(0.0, Pm, g.pitch); }));
}

static void test_data_loss_composed() {
  // vanishes on exactly consistent channels; DC carries no weight (test_optimize.cpp:124-155)
  {
    const int P = 16, M = 3;
    std::mt19937_64 rng(17);
    std::uniform_real_distribution<double> u(-1, 1);
    TransferStack hs = transfer_stack(random_profile(rng, 32, 0.1, 0.2), make_delays(-0.3, 0.3, M), P, 0.1);
    std::vector<double> xr(P * P);
    for (double& v : xr) v = u(rng);
    std::vector<cplx> x = dft2(xr, P);
    PatchSpectra ys;
    ys.Y.resize(M);
    for (int j = 0; j < M; ++j) {
      ys.Y[j].resize(x.size());
      for (size_t b = 0; b < x.size(); ++b) ys.Y[j][b] = hs.spectra[j][b] * x[b];
    }
    double yscale = 0.0;
    for (const auto& v : ys.Y[0]) yscale = std::max(yscale, std::norm(v));
    CHECK(data_loss({ys}, {hs}, 0.0).value < 1e-18 * yscale);
    PatchSpectra ydc = ys;
    ydc.Y[0][0] += cplx(1e6, 0.0);
    CHECK(data_loss({ydc}, {hs}, 0.0).value < 1e-18 * yscale);
  }
  // dL/dH vs finite differences (test_optimize.cpp:157-203)
  const int P = 8, M = 3;
  std::mt19937_64 rng(19);
  std::uniform_real_distribution<double> u(-1, 1);
  TransferStack hs = transfer_stack(random_profile(rng, 16, -0.2, 0.2), make_delays(-0.25, 0.25, M), P, 0.1);
  std::vector<PatchSpectra> ys(1);
  for (int j = 0; j < M; ++j) {
    std::vector<double> x(P * P);
    for (double& v : x) v = u(rng);
    ys[0].Y.push_back(dft2(x, P));
  }
  DataLossResult dl = data_loss(ys, {hs}, 1e-3, true);
  std::uniform_int_distribution<size_t> pick_bin(0, P * P - 1);
  std::uniform_int_distribution<int> pick_ch(0, M - 1);
  double worst = 0.0;
  for (int trial = 0; trial < 12; ++trial) {
    size_t bin = pick_bin(rng);
    int j = pick_ch(rng);
    const double h = 1e-6;
    auto value_with = [&](cplx delta) {
      std::vector<TransferStack> hp{hs};
      hp[0].spectra[j][bin] += delta;
      return data_loss(ys, hp, 1e-3, true).value;
    };
    double fd_re = (value_with(cplx(h, 0)) - value_with(cplx(-h, 0))) / (2 * h);
    double fd_im = (value_with(cplx(0, h)) - value_with(cplx(0, -h))) / (2 * h);
    cplx g = dl.grad_h[0][j][bin];
    double scale = std::max({1.0, std::abs(fd_re), std::abs(fd_im)});
    worst = std::max({worst, std::abs(g.real() - fd_re) / scale, std::abs(g.imag() - fd_im) / scale});
  }
  std::printf("  data loss dL/dH vs FD: max err %.2e (bar 1e-4)\n", worst);
  CHECK(worst < 1e-4);
  // patch_data_loss with the training cache's complex<float> Y equals the complex<double> one
  std::vector<std::vector<std::complex<float>>> yf;
  for (const auto& c : ys[0].Y) {
    yf.emplace_back();
    for (const auto& v : c) yf.back().push_back(std::complex<float>(v));
  }
  const double sc = 1.0 / (M * P * P);
  PatchLossResult a = patch_data_loss(yf, hs, 1e-3, sc, true);
  CHECK(std::abs(a.value - dl.value) <= 1e-6 * std::abs(dl.value));
  CHECK(throws<ValidationError>([&] { data_loss({}, {}, 1e-3); }));
  CHECK(throws<ValidationError>([&] { data_loss(ys, {hs, hs}, 1e-3); }));
}

// testsupport::make_small_instance (test_support.hpp:43-75) through the drop-in
struct SmallInstance {
  GridSpec grid = GridSpec::centered(64, 64, 0.1);
  CircularMask mask{{0.0, 0.0}, 2.6};
  RingGeometry ring{64, 50.0, 0.0};
  TrainConfig cfg;
  SignalSet signals;
  DasStack stack;
  PatchLayout layout;
  std::vector<PatchSpectra> spectra;
};

static SmallInstance make_small_instance() {
  SmallInstance si;
  si.cfg.delays = make_delays(-0.4, 0.4, 4);
  si.cfg.n_angles = 32;
  si.cfg.ray_step = 0.1;
  si.cfg.patch_mm = 3.2;
  si.cfg.overlap = 0.0;
  si.cfg.hidden = 8;
  si.cfg.sine_layers = 2;
  si.cfg.out_scale = 60.0;
  si.cfg.lambda_tv = 1e-4;
  si.cfg.workers = 1;
  PhantomSpec spec = builtin_phantom_spec("empty", 1500.0);
  spec.mask = si.mask;
  spec.discs.push_back({{0.4, -0.3}, 1.2, 1560.0, 0.0});
  spec.points.push_back({{0.0, 0.0}, 1.0});
  spec.points.push_back({{1.0, 0.8}, 0.8});
  spec.points.push_back({{-1.2, 0.4}, 0.9});
  Phantom ph = generate_phantom(si.grid, spec, 0);
  si.signals = simulate_signals(ph, si.ring);
  si.stack = das_stack(si.signals, si.grid, 1500.0, si.cfg.delays, 1);
  si.layout = make_patch_layout(si.grid, si.cfg.patch_mm, si.cfg.overlap);
  si.spectra = extract_patch_spectra(si.stack, si.layout, 1);
  return si;
}

// testsupport::full_chain_loss / full_chain_grad (test_support.hpp:79-118)
static double full_chain_loss(const SmallInstance& si, const SirenParams& params) {
  SosField field = render_sos(params, si.grid, si.mask);
  std::vector<TransferStack> hs;
  for (int i = 0; i < si.layout.n_patches(); ++i) {
    WavefrontProfile prof = wavefront_profile(si.layout.centers[i], si.ring, field.raster,
                                              si.stack.v0, si.mask, si.cfg.n_angles,
                                              si.cfg.ray_step, false);
    hs.push_back(transfer_stack(prof, si.cfg.delays, si.layout.patch_pixels, si.grid.pitch));
  }
  DataLossResult dl = data_loss(si.spectra, hs, si.cfg.eps_deconv, si.cfg.implicit_xhat_grad);
  return dl.value + tv_loss(field, si.cfg.lambda_tv).value;
}

static std::vector<double> full_chain_grad(const SmallInstance& si, const SirenParams& params,
                                           std::vector<double>* grad_v_out = nullptr) {
  SosField field = render_sos(params, si.grid, si.mask);
  std::vector<double> gv(field.raster.values.size(), 0.0);
  const int P = si.layout.patch_pixels;
  const double scale = 1.0 / (double(si.layout.n_patches()) * si.cfg.delays.size() * P * P);
  for (int i = 0; i < si.layout.n_patches(); ++i) {
    WavefrontProfile prof = wavefront_profile(si.layout.centers[i], si.ring, field.raster,
                                              si.stack.v0, si.mask, si.cfg.n_angles,
                                              si.cfg.ray_step, true);
    TransferStack hs = transfer_stack(prof, si.cfg.delays, P, si.grid.pitch);
    PatchLossResult pl = patch_data_loss(si.spectra[i].Y, hs, si.cfg.eps_deconv, scale,
                                         si.cfg.implicit_xhat_grad);
    std::vector<double> dw = transfer_grad_to_wavefront(prof, si.cfg.delays, P, si.grid.pitch, pl.grad_h);
    accumulate_wavefront_grad(prof, dw, gv);
  }
  TvLossResult tv = tv_loss(field, si.cfg.lambda_tv);
  std::vector<double> gm(field.masked_indices.size());
  for (size_t i = 0; i < gm.size(); ++i) gm[i] = gv[field.masked_indices[i]] + tv.grad[i];
  if (grad_v_out) *grad_v_out = gv;
  return backprop_sos(params, field, gm);
}

static void test_full_chain() {
  SmallInstance si = make_small_instance();
  // the Jacobian rows reproduce the wavefront values and the fused adjoint
  // (test_optimize.cpp:306-351: fused == composed), per patch
  SirenParams params = init_siren(2, si.cfg.hidden, si.cfg.sine_layers, si.cfg.omega0,
                                  si.cfg.out_scale, 1500.0);
  SosField field = render_sos(params, si.grid, si.mask);
  double worst_w = 0, worst_gv = 0;
  for (int i = 0; i < si.layout.n_patches(); ++i) {
    WavefrontProfile pj = wavefront_profile(si.layout.centers[i], si.ring, field.raster, 1500.0,
                                            si.mask, si.cfg.n_angles, si.cfg.ray_step, true);
    WavefrontProfile pf = wavefront_profile(si.layout.centers[i], si.ring, field.raster, 1500.0,
                                            si.mask, si.cfg.n_angles, si.cfg.ray_step, false);
    worst_w = std::max(worst_w, rel_l2(pf.w, pj.w));
    std::vector<double> dw(si.cfg.n_angles);
    for (int a = 0; a < si.cfg.n_angles; ++a) dw[a] = std::sin(0.3 * a + i);
    std::vector<double> gj(field.raster.values.size(), 0.0), gf(gj.size(), 0.0);
    accumulate_wavefront_grad(pj, dw, gj);
    wavefront_grad_trace(si.layout.centers[i], si.ring, field.raster, 1500.0, si.mask,
                         si.cfg.n_angles, si.cfg.ray_step, dw, gf);
    std::vector<double> a, b;
    for (int idx : field.masked_indices) {
      a.push_back(gf[idx]);
      b.push_back(gj[idx]);
    }
    worst_gv = std::max(worst_gv, rel_l2(a, b));
  }
  std::printf("  Jacobian path vs fused: w %.2e, J^T dw on masked pixels %.2e\n", worst_w, worst_gv);
  CHECK(worst_w < 1e-5);
  CHECK(worst_gv < 1e-5);
  CHECK(throws<ValidationError>([&] {
    std::vector<double> g(4096, 0.0);
    accumulate_wavefront_grad(WavefrontProfile{}, {}, g);
  }));
  // full-chain gradient vs finite differences (test_optimize.cpp:205-229).
  // The device path evaluates the SIREN, the rays and H in fp32, so the FD
  // step is 1e-3 (the reference's 1e-5 would be below the fp32 loss noise).
  SirenParams p0 = init_siren(0, si.cfg.hidden, si.cfg.sine_layers, si.cfg.omega0, si.cfg.out_scale, 1500.0);
  std::vector<double> grad = full_chain_grad(si, p0);
  std::mt19937_64 rng(23);
  std::uniform_int_distribution<size_t> pick(0, p0.param_count() - 1);
  const double eps = 1e-3;
  double max_rel = 0.0;
  for (int t = 0; t < 20; ++t) {
    size_t i = pick(rng);
    SirenParams pp = p0, pm = p0;
    pp.theta[i] += eps;
    pm.theta[i] -= eps;
    double fd = (full_chain_loss(si, pp) - full_chain_loss(si, pm)) / (2 * eps);
    double scale = std::max(std::abs(fd), std::abs(grad[i]));
    if (scale < 1e-12) continue;
    max_rel = std::max(max_rel, std::abs(grad[i] - fd) / scale);
  }
  std::printf("  full-chain grad vs FD (eps 1e-3, 20 params): max rel %.2e\n", max_rel);
  CHECK(max_rel < 1e-2);
}

int main() {
  struct Case {
    const char* name;
    std::function<void()> fn;
  } cases[] = {{"beamform", test_beamform},
               {"evaluate", test_evaluate},
               {"nfield", test_nfield},
               {"aberration", test_aberration},
               {"optimize", test_optimize},
               {"joint_reconstruct", test_joint_reconstruct},
               {"deconv_composed", test_deconv_composed},
               {"data_loss_composed", test_data_loss_composed},
               {"full_chain", test_full_chain}};
  for (auto& c : cases) {
    int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  EXCEPTION %s\n", e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "ok" : "FAIL", c.name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
