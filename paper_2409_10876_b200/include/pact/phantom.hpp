// Drop-in host API (namespace pact) — numerical phantoms and the signal
// simulator (the reference's proj/include/pact/phantom.hpp).
//
//   PhantomSpec / builtin_phantom_spec   phantom.hpp:36-181
//   generate_phantom                     phantom.hpp:186-266 (host, bit-identical:
//                                        same seed stream, same coverage sums)
//   SimulateOptions / simulate_signals   phantom.hpp:268-362 (on the B200:
//                                        pact_simulate_window + pact_simulate_signals_ex)
//
// Phantom rasterisation is the input-fixture generator, not the hot path; it
// stays on the host like the reference, with each region's rows split over
// threads (every pixel's coverage is an independent fixed-order sum, so the
// result does not depend on the split).
#ifndef PACT_B200_PHANTOM_HPP
#define PACT_B200_PHANTOM_HPP

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "pact/core.hpp"

namespace pact {

struct DiscSpec {
  Vec2 center;
  double radius = 0.0;    // mm
  double sos = 0.0;       // m/s (the background value for pressure-only discs)
  double pressure = 0.0;  // fill amplitude
};

struct VesselSpec {
  Vec2 a, b;
  double radius = 0.0;  // capsule half-width, mm
  double pressure = 0.0;
};

struct RingSpec {
  Vec2 center;
  double radius = 0.0;
  double width = 0.0;  // full annulus width, mm
  double pressure = 0.0;
};

struct PointSpec {
  Vec2 pos;
  double amplitude = 0.0;
};

struct PhantomSpec {
  double background_sos = 1499.4;  // m/s
  CircularMask mask{{0.0, 0.0}, 10.0};
  std::vector<DiscSpec> discs;
  std::vector<VesselSpec> vessels;
  std::vector<RingSpec> rings;
  std::vector<PointSpec> points;
  double jitter_mm = 0.0;  // seed-driven perturbation of vessels and points
  bool antialias = true;
};

struct Phantom {
  RasterGrid pressure;
  RasterGrid sos;
  CircularMask mask;
  double background_sos = 0.0;
};

namespace phantom_detail {

constexpr double kSosLo = 1300.0, kSosHi = 1800.0;

inline double segment_distance(Vec2 p, Vec2 a, Vec2 b) {
  const Vec2 d = b - a;
  const double len2 = d.dot(d);
  if (len2 == 0.0) return (p - a).norm();
  const double t = std::clamp((p - a).dot(d) / len2, 0.0, 1.0);
  return (p - (a + d * t)).norm();
}

/// Fraction of the tent-weighted 2x2-pixel footprint around `c` inside the
/// region, on an S x S subsample lattice (the bilinear prefilter of
/// phantom.hpp:62-78; the sums run in the same order).
template <typename Inside>
double coverage(Vec2 c, double pitch, const Inside& inside, int S) {
  double hit = 0.0, total = 0.0;
  for (int sy = 0; sy < S; ++sy) {
    const double dy = 2.0 * (sy + 0.5) / S - 1.0;
    for (int sx = 0; sx < S; ++sx) {
      const double dx = 2.0 * (sx + 0.5) / S - 1.0;
      const double w = (1.0 - std::abs(dx)) * (1.0 - std::abs(dy));
      hit += w * (inside(Vec2{c.x + dx * pitch, c.y + dy * pitch}) ? 1.0 : 0.0);
      total += w;
    }
  }
  return hit / total;
}

enum class Compose { kBlend, kMax };  // SOS: coverage blend; pressure: max composite

/// Paints one region over its bounding box [lo, hi] (+1 px margin),
/// phantom.hpp:80-102.  Rows are split over host threads.
template <typename Inside>
void paint(RasterGrid& r, Vec2 lo, Vec2 hi, const Inside& inside, double value, Compose mode,
           bool antialias, const CircularMask* clip) {
  const GridSpec gs = r.spec();
  const Vec2 plo = gs.pixel(lo), phi = gs.pixel(hi);
  const int x0 = std::max(0, static_cast<int>(std::floor(plo.x)) - 1);
  const int y0 = std::max(0, static_cast<int>(std::floor(plo.y)) - 1);
  const int x1 = std::min(gs.width - 1, static_cast<int>(std::ceil(phi.x)) + 1);
  const int y1 = std::min(gs.height - 1, static_cast<int>(std::ceil(phi.y)) + 1);
  if (y1 < y0 || x1 < x0) return;
  const int S = antialias ? 32 : 1;
  auto rows = [&](int ya, int yb) {
    for (int iy = ya; iy < yb; ++iy)
      for (int ix = x0; ix <= x1; ++ix) {
        const Vec2 c = gs.world(ix, iy);
        if (clip && !clip->contains(c)) continue;
        const double cov = coverage(c, gs.pitch, inside, S);
        if (cov <= 0.0) continue;
        double& px = r.at(ix, iy);
        px = mode == Compose::kBlend ? (1.0 - cov) * px + cov * value : std::max(px, value * cov);
      }
  };
  const int n_rows = y1 - y0 + 1;
  const int n_thr = std::max(1, std::min<int>(n_rows / 8, std::thread::hardware_concurrency()));
  if (n_thr <= 1) {
    rows(y0, y1 + 1);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < n_thr; ++t)
    pool.emplace_back(rows, y0 + n_rows * t / n_thr, y0 + n_rows * (t + 1) / n_thr);
  for (auto& th : pool) th.join();
}

}  // namespace phantom_detail

/// builtin_phantom_spec (phantom.hpp:145-181): "default" / "liver" (liver-like
/// slice), "twobody" (one body disc in water), "empty".
inline PhantomSpec builtin_phantom_spec(const std::string& name, double background_sos = 1499.4) {
  PhantomSpec s;
  s.background_sos = background_sos;
  s.mask = {{0.0, 0.0}, 10.0};
  if (name == "empty") return s;
  if (name == "twobody") {
    s.discs = {{{0.0, 0.0}, 9.0, 1561.0, 0.05}};
    s.rings = {{{0.0, 0.0}, 9.0, 0.25, 0.8}};
    s.points = {{{0.0, 0.0}, 1.5}, {{4.5, 1.0}, 1.5}, {{-3.0, -4.0}, 1.5}};
    return s;
  }
  if (name == "default" || name == "liver") {
    s.jitter_mm = 0.35;
    s.discs = {{{0.0, 0.0}, 9.0, 1545.0, 0.02},          // body
               {{-2.0, 1.5}, 4.8, 1590.0, 0.05},         // organ
               {{4.5, 3.5}, 1.8, background_sos, 0.0},  // water hole
               {{3.0, -4.0}, 1.2, 1650.0, 0.3},          // stiff inclusions
               {{-5.5, -2.5}, 1.5, 1620.0, 0.25}};
    s.rings = {{{0.0, 0.0}, 9.0, 0.25, 0.8}, {{-2.0, 1.5}, 4.8, 0.2, 0.5}, {{4.5, 3.5}, 1.8, 0.2, 0.4}};
    s.vessels = {{{-6.0, -5.0}, {-1.5, -1.0}, 0.25, 1.0},
                 {{-1.5, -1.0}, {2.5, -2.5}, 0.22, 0.9},
                 {{-1.5, -1.0}, {0.5, 2.8}, 0.2, 0.9},
                 {{1.0, 4.5}, {5.0, 1.2}, 0.2, 0.8}};
    s.points = {{{0.0, 0.0}, 1.5}, {{4.8, 0.8}, 1.5}, {{-5.2, 1.0}, 1.5}, {{0.5, -5.6}, 1.5},
                {{2.5, 4.2}, 1.5}};
    return s;
  }
  throw ValidationError("unknown builtin phantom spec: " + name);
}

/// generate_phantom (phantom.hpp:186-266).  Deterministic for a seed: the
/// seed drives only the vessel and point jitter (mt19937_64, one uniform draw
/// per coordinate in spec order: vessels a then b, then points).
inline Phantom generate_phantom(const GridSpec& grid, const PhantomSpec& spec, uint64_t seed) {
  using namespace phantom_detail;
  grid.validate();
  const CircularMask& m = spec.mask;
  if (!(spec.background_sos >= kSosLo && spec.background_sos <= kSosHi))
    throw ValidationError("phantom: background SOS outside [1300, 1800] m/s");
  for (const DiscSpec& d : spec.discs) {
    if (!(d.sos >= kSosLo && d.sos <= kSosHi))
      throw ValidationError("phantom: disc SOS outside [1300, 1800] m/s");
    if ((d.center - m.center).norm() + d.radius > m.radius)
      throw ValidationError("phantom: disc region extends outside the mask");
  }
  for (const RingSpec& r : spec.rings)
    if ((r.center - m.center).norm() + r.radius + 0.5 * r.width > m.radius)
      throw ValidationError("phantom: ring region extends outside the mask");

  std::mt19937_64 rng(seed);
  auto jitter = [&](Vec2 p) {
    if (spec.jitter_mm <= 0.0) return p;
    std::uniform_real_distribution<double> u(-spec.jitter_mm, spec.jitter_mm);
    const double jx = u(rng);
    const double jy = u(rng);
    return Vec2{p.x + jx, p.y + jy};
  };
  std::vector<VesselSpec> vessels = spec.vessels;
  for (VesselSpec& v : vessels) {
    v.a = jitter(v.a);
    v.b = jitter(v.b);
    const bool axis_out = segment_distance(m.center, v.a, v.b) + v.radius > m.radius;
    const bool end_out = (v.a - m.center).norm() + v.radius > m.radius ||
                         (v.b - m.center).norm() + v.radius > m.radius;
    if (axis_out && end_out) throw ValidationError("phantom: vessel extends outside the mask");
  }
  std::vector<PointSpec> points = spec.points;
  for (PointSpec& p : points) {
    p.pos = jitter(p.pos);
    if (!m.contains(p.pos)) throw ValidationError("phantom: point target outside the mask");
  }

  Phantom ph;
  ph.mask = m;
  ph.background_sos = spec.background_sos;
  ph.sos = RasterGrid::constant(grid, spec.background_sos);
  ph.pressure = RasterGrid::zeros(grid);
  const bool aa = spec.antialias;
  for (const DiscSpec& d : spec.discs) {
    auto in = [&](Vec2 p) { return (p - d.center).norm() <= d.radius; };
    const Vec2 lo{d.center.x - d.radius, d.center.y - d.radius};
    const Vec2 hi{d.center.x + d.radius, d.center.y + d.radius};
    paint(ph.sos, lo, hi, in, d.sos, Compose::kBlend, aa, &m);
    if (d.pressure > 0.0) paint(ph.pressure, lo, hi, in, d.pressure, Compose::kMax, aa, nullptr);
  }
  for (const RingSpec& r : spec.rings) {
    const double rout = r.radius + 0.5 * r.width;
    auto in = [&](Vec2 p) { return std::abs((p - r.center).norm() - r.radius) <= 0.5 * r.width; };
    paint(ph.pressure, {r.center.x - rout, r.center.y - rout}, {r.center.x + rout, r.center.y + rout},
          in, r.pressure, Compose::kMax, aa, nullptr);
  }
  for (const VesselSpec& v : vessels) {
    auto in = [&](Vec2 p) { return segment_distance(p, v.a, v.b) <= v.radius; };
    const Vec2 lo{std::min(v.a.x, v.b.x) - v.radius, std::min(v.a.y, v.b.y) - v.radius};
    const Vec2 hi{std::max(v.a.x, v.b.x) + v.radius, std::max(v.a.y, v.b.y) + v.radius};
    paint(ph.pressure, lo, hi, in, v.pressure, Compose::kMax, aa, nullptr);
  }
  for (const PointSpec& p : points) {
    const Vec2 q = grid.pixel(p.pos);
    const int ix = static_cast<int>(std::lround(q.x)), iy = static_cast<int>(std::lround(q.y));
    if (ix >= 0 && ix < grid.width && iy >= 0 && iy < grid.height) ph.pressure.at(ix, iy) += p.amplitude;
  }
  return ph;
}

struct SimulateOptions {
  double pulse_sigma = 100e-9;  // s
  double dt = 25e-9;            // s (40 MHz)
  bool spreading = false;       // 1/sqrt(distance) amplitude falloff
  double t0 = std::numeric_limits<double>::quiet_NaN();  // NaN -> automatic window
  int n_samples = 0;                                     // 0 -> automatic window
  double ray_step = 0.05;  // mm, straight-ray TOF quadrature step
  int workers = 0;         // accepted, ignored (one B200)
};

/// simulate_signals (phantom.hpp:282-362) on the B200: the window and
/// validation on the host (pact_simulate_window), the per-(transducer, source)
/// TOF and pulse synthesis on the device.  Samples come back through fp32.
inline SignalSet simulate_signals(const Phantom& ph, const RingGeometry& geom,
                                  const SimulateOptions& opt = {}) {
  geom.validate();
  if (!ph.pressure.spec().same_geometry(ph.sos.spec()))
    throw ValidationError("pressure and SOS rasters have different grids");
  const pact_grid g = ph.pressure.spec().c();
  const pact_ring r = geom.c();
  pact_signal_meta meta{};
  cuda::check(pact_simulate_window(&g, ph.pressure.values.data(), ph.sos.values.data(),
                                   ph.background_sos, &r, opt.pulse_sigma, opt.dt, opt.t0,
                                   opt.n_samples, &meta));
  SignalSet s;
  s.geom = geom;
  s.n_samples = meta.n_samples;
  s.dt = meta.dt;
  s.t0 = meta.t0;
  s.background_sos = ph.background_sos;
  const size_t n = static_cast<size_t>(geom.n_transducers) * meta.n_samples;
  cuda::Buffer<float> out(n);
  const pact_mask mk = ph.mask.c();
  cuda::check(pact_simulate_signals_ex(cuda::context(), &g, ph.pressure.values.data(),
                                       ph.sos.values.data(), &mk, ph.background_sos, &r,
                                       opt.pulse_sigma, &meta, opt.ray_step, opt.spreading ? 1 : 0,
                                       out.ptr));
  std::vector<float> h(n);
  out.download(h.data());
  s.data.assign(h.begin(), h.end());
  return s;
}

}  // namespace pact

#endif  // PACT_B200_PHANTOM_HPP
