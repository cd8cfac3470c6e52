// Drop-in host API (namespace pact) over the B200 C-ABI — core types.
//
// Same type names, fields and semantics as the reference's
// proj/include/pact/core.hpp (GridSpec 58-89, RasterGrid 93-149,
// RingGeometry 152-173, CircularMask 175-180, PatchLayout 222-281,
// SignalSet 284-313) so code written against the reference compiles
// unchanged for the hot-path entry points.  Rasters stay fp64 row-major on the
// host; the entry points in beamform.hpp / nfield.hpp / aberration.hpp /
// deconv.hpp / optimize.hpp convert to fp32 device buffers and call
// include/pact_cuda.h.  There is no CPU fallback: without a B200 every
// compute entry point throws.
#ifndef PACT_B200_CORE_HPP
#define PACT_B200_CORE_HPP

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pact_cuda.h"

namespace pact {

/// Bad arguments (the reference's ValidationError; CLI exit code 2).
struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

/// Non-finite results (the reference's NumericalError; CLI exit code 3).
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Vec2 {
  double x = 0.0, y = 0.0;
  Vec2 operator+(Vec2 o) const { return {x + o.x, y + o.y}; }
  Vec2 operator-(Vec2 o) const { return {x - o.x, y - o.y}; }
  Vec2 operator*(double s) const { return {x * s, y * s}; }
  double dot(Vec2 o) const { return x * o.x + y * o.y; }
  double norm() const { return std::hypot(x, y); }
};

struct GridSpec {
  int width = 0, height = 0;
  double pitch = 0.0;  // mm
  Vec2 origin;         // world position of pixel (0, 0)

  void validate() const {
    if (width < 1 || height < 1) throw ValidationError("grid: width and height must be >= 1");
    if (!(pitch > 0.0)) throw ValidationError("grid: pitch must be > 0");
  }
  Vec2 world(double ix, double iy) const { return {origin.x + ix * pitch, origin.y + iy * pitch}; }
  Vec2 pixel(Vec2 p) const { return {(p.x - origin.x) / pitch, (p.y - origin.y) / pitch}; }
  bool same_geometry(const GridSpec& o) const {
    return width == o.width && height == o.height && pitch == o.pitch && origin.x == o.origin.x &&
           origin.y == o.origin.y;
  }
  static GridSpec centered(int w, int h, double pitch) {
    GridSpec g{w, h, pitch, {-0.5 * (w - 1) * pitch, -0.5 * (h - 1) * pitch}};
    g.validate();
    return g;
  }
  pact_grid c() const { return {width, height, pitch, origin.x, origin.y}; }
};

struct RasterGrid {
  int width = 0, height = 0;
  double pitch = 0.0;
  Vec2 origin;
  std::vector<double> values;  // row-major [iy * width + ix]

  static RasterGrid zeros(const GridSpec& g) { return constant(g, 0.0); }
  static RasterGrid constant(const GridSpec& g, double v) {
    g.validate();
    RasterGrid r{g.width, g.height, g.pitch, g.origin, {}};
    r.values.assign(static_cast<size_t>(g.width) * g.height, v);
    return r;
  }
  GridSpec spec() const { return {width, height, pitch, origin}; }
  double& at(int ix, int iy) { return values[static_cast<size_t>(iy) * width + ix]; }
  double at(int ix, int iy) const { return values[static_cast<size_t>(iy) * width + ix]; }
  Vec2 world(double ix, double iy) const { return spec().world(ix, iy); }
  bool in_bounds(int ix, int iy) const { return ix >= 0 && ix < width && iy >= 0 && iy < height; }
  double max_abs() const {
    double m = 0.0;
    for (double v : values) m = std::max(m, std::abs(v));
    return m;
  }
};

struct RingGeometry {
  int n_transducers = 0;
  double radius = 0.0;        // mm
  double angle_offset = 0.0;  // rad

  void validate() const {
    if (n_transducers < 3) throw ValidationError("ring: need at least 3 transducers");
    if (!(radius > 0.0)) throw ValidationError("ring: radius must be > 0");
  }
  Vec2 transducer_position(int n) const {
    double a = 2.0 * M_PI * n / n_transducers + angle_offset;
    return {radius * std::cos(a), radius * std::sin(a)};
  }
  pact_ring c() const { return {n_transducers, radius, angle_offset}; }
};

inline std::vector<Vec2> transducer_positions(const RingGeometry& g) {
  g.validate();
  std::vector<Vec2> p;
  for (int n = 0; n < g.n_transducers; ++n) p.push_back(g.transducer_position(n));
  return p;
}

struct CircularMask {
  Vec2 center;
  double radius = 0.0;
  bool contains(Vec2 p) const { return (p - center).norm() <= radius; }
  pact_mask c() const { return {center.x, center.y, radius}; }
};

/// water_sos (core.hpp:208-218): fifth-order polynomial in temperature (deg C).
inline double water_sos(double temperature_celsius) {
  const double t = temperature_celsius;
  if (!(t >= 0.0 && t <= 95.0))
    throw ValidationError("water_sos: temperature " + std::to_string(t) +
                          " outside valid range [0, 95] C");
  static constexpr double c[6] = {1.402385e3, 5.038813, -5.799136e-2, 3.287156e-4, -1.398845e-6,
                                  2.787860e-9};
  return c[0] + t * (c[1] + t * (c[2] + t * (c[3] + t * (c[4] + t * c[5]))));
}

struct PatchLayout {
  GridSpec grid;
  double patch_mm = 0.0, overlap = 0.0;
  int patch_pixels = 0, stride_pixels = 0, nx = 0, ny = 0;
  std::vector<std::pair<int, int>> offsets;
  std::vector<Vec2> centers;
  int n_patches() const { return static_cast<int>(offsets.size()); }
  pact_layout c() const {
    pact_layout l{grid.c(), patch_pixels, stride_pixels, nx, ny,
                  grid.width <= patch_pixels ? 0 : grid.width - patch_pixels,
                  grid.height <= patch_pixels ? 0 : grid.height - patch_pixels};
    return l;
  }
};

struct SignalSet {
  RingGeometry geom;
  int n_samples = 0;
  double dt = 0.0, t0 = 0.0, background_sos = 0.0;
  std::vector<double> data;  // [channel * n_samples + sample]

  double& at(int ch, int s) { return data[static_cast<size_t>(ch) * n_samples + s]; }
  double at(int ch, int s) const { return data[static_cast<size_t>(ch) * n_samples + s]; }
  void validate() const {
    geom.validate();
    if (n_samples < 2) throw ValidationError("signals: need at least 2 samples");
    if (!(dt > 0.0)) throw ValidationError("signals: dt must be > 0");
    if (data.size() != static_cast<size_t>(geom.n_transducers) * n_samples)
      throw ValidationError("signals: data size does not match N_t x n_samples");
  }
  pact_signal_meta meta() const { return {n_samples, dt, t0, background_sos}; }
};

namespace cuda {

/// Throws the reference exception type for a C-ABI status.
inline void check(int rc) {
  if (rc == PACT_OK) return;
  std::string msg = pact_last_error();
  if (rc == PACT_E_VALIDATION) throw ValidationError(msg);
  if (rc == PACT_E_NUMERICAL) throw NumericalError(msg);
  throw std::runtime_error("pact_cuda: " + msg);
}

/// Per-thread context on device 0 (PACT_DEVICE selects another).
inline pact_ctx* context() {
  struct Holder {
    pact_ctx* ctx = nullptr;
    ~Holder() {
      if (ctx) pact_ctx_destroy(ctx);
    }
  };
  static thread_local Holder h;
  if (!h.ctx) {
    const char* d = std::getenv("PACT_DEVICE");
    check(pact_ctx_create(d ? std::atoi(d) : 0, &h.ctx));
  }
  return h.ctx;
}

/// RAII device buffer of T.
template <typename T>
struct Buffer {
  T* ptr = nullptr;
  size_t n = 0;
  explicit Buffer(size_t count) : n(count) {
    void* p = nullptr;
    check(pact_device_alloc(context(), sizeof(T) * (count ? count : 1), &p));
    ptr = static_cast<T*>(p);
  }
  Buffer(const Buffer&) = delete;
  Buffer& operator=(const Buffer&) = delete;
  ~Buffer() {
    if (ptr) pact_device_free(context(), ptr);
  }
  void upload(const T* host) { check(pact_upload(context(), ptr, host, sizeof(T) * n)); }
  void download(T* host) const { check(pact_download(context(), host, ptr, sizeof(T) * n)); }
};

/// fp64 host values -> fp32 device buffer.
inline void upload_f32(Buffer<float>& b, const std::vector<double>& v, double shift = 0.0) {
  std::vector<float> f(v.size());
  for (size_t i = 0; i < v.size(); ++i) f[i] = static_cast<float>(v[i] - shift);
  b.upload(f.data());
}

inline std::vector<double> download_f64(const Buffer<float>& b, double shift = 0.0) {
  std::vector<float> f(b.n);
  b.download(f.data());
  std::vector<double> d(f.size());
  for (size_t i = 0; i < f.size(); ++i) d[i] = static_cast<double>(f[i]) + shift;
  return d;
}

}  // namespace cuda

/// make_patch_layout (core.hpp:252-281) through the C-ABI.
inline PatchLayout make_patch_layout(const GridSpec& grid, double patch_mm, double overlap) {
  pact_grid g = grid.c();
  pact_layout l{};
  cuda::check(pact_make_patch_layout(&g, patch_mm, overlap, &l));
  PatchLayout lay;
  lay.grid = grid;
  lay.patch_mm = patch_mm;
  lay.overlap = overlap;
  lay.patch_pixels = l.patch_pixels;
  lay.stride_pixels = l.stride_pixels;
  lay.nx = l.nx;
  lay.ny = l.ny;
  int n = l.nx * l.ny;
  std::vector<int32_t> off(2 * n);
  std::vector<double> cen(2 * n);
  cuda::check(pact_layout_patches(&l, off.data(), cen.data()));
  for (int i = 0; i < n; ++i) {
    lay.offsets.emplace_back(off[2 * i], off[2 * i + 1]);
    lay.centers.push_back({cen[2 * i], cen[2 * i + 1]});
  }
  return lay;
}

}  // namespace pact

#endif
