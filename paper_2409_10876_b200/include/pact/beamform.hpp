// Drop-in host API — part 1, the multi-delay DAS stack
// (reference: proj/include/pact/beamform.hpp:35-120).
#ifndef PACT_B200_BEAMFORM_HPP
#define PACT_B200_BEAMFORM_HPP

#include <vector>

#include "pact/core.hpp"

namespace pact {

struct DasStack {
  std::vector<double> delays;  // mm, strictly increasing
  std::vector<RasterGrid> images;
  double v0 = 0.0;
  int n_delays() const { return static_cast<int>(delays.size()); }
};

/// make_delays (beamform.hpp:113-120).
inline std::vector<double> make_delays(double lo, double hi, int count) {
  std::vector<double> d(count > 0 ? count : 1);
  cuda::check(pact_make_delays(lo, hi, count, d.data()));
  d.resize(count);
  return d;
}

/// das_stack (beamform.hpp:77-110) on the GPU; `workers` is accepted and ignored.
inline DasStack das_stack(const SignalSet& signals, const GridSpec& grid, double v0,
                          const std::vector<double>& delays, int workers = 0) {
  (void)workers;
  if (delays.empty()) throw ValidationError("das_stack: need at least one delay");
  for (size_t j = 1; j < delays.size(); ++j)
    if (!(delays[j] > delays[j - 1]))
      throw ValidationError("das_stack: delays must be strictly increasing");
  signals.validate();
  grid.validate();
  if (!(v0 > 0.0)) throw ValidationError("das_stack: v0 must be > 0");
  cuda::Buffer<float> sig(signals.data.size());
  cuda::upload_f32(sig, signals.data);
  const size_t plane = static_cast<size_t>(grid.width) * grid.height;
  cuda::Buffer<float> out(plane * delays.size());
  pact_ring r = signals.geom.c();
  pact_signal_meta m = signals.meta();
  pact_grid g = grid.c();
  cuda::check(pact_das_stack(cuda::context(), &r, &m, sig.ptr, &g, v0, delays.data(),
                             static_cast<int32_t>(delays.size()), out.ptr));
  std::vector<double> all = cuda::download_f64(out);
  DasStack st;
  st.delays = delays;
  st.v0 = v0;
  for (size_t j = 0; j < delays.size(); ++j) {
    RasterGrid img = RasterGrid::zeros(grid);
    std::copy(all.begin() + j * plane, all.begin() + (j + 1) * plane, img.values.begin());
    st.images.push_back(std::move(img));
  }
  return st;
}

/// das (beamform.hpp:56-75): the single-delay stack.
inline RasterGrid das(const SignalSet& signals, const GridSpec& grid, double v0, double d,
                      int workers = 0) {
  return das_stack(signals, grid, v0, {d}, workers).images[0];
}

/// BodyModel (beamform.hpp:44-54).
struct BodyModel {
  Vec2 center;
  double radius = 0.0;    // mm
  double body_sos = 0.0;  // m/s

  void validate() const {
    if (!(radius > 0.0)) throw ValidationError("body model: radius must be > 0");
    if (!(body_sos >= 1300.0 && body_sos <= 1800.0))
      throw ValidationError("body model: SOS outside [1300, 1800] m/s");
  }
};

/// dual_sos_das (beamform.hpp:124-150) on the GPU; `workers` is accepted and ignored.
inline RasterGrid dual_sos_das(const SignalSet& signals, const GridSpec& grid, double v0,
                               const BodyModel& body, int workers = 0) {
  (void)workers;
  signals.validate();
  grid.validate();
  body.validate();
  if (!(v0 > 0.0)) throw ValidationError("dual_sos_das: v0 must be > 0");
  if (body.center.norm() + body.radius >= signals.geom.radius)
    throw ValidationError("dual_sos_das: body disc extends outside the transducer ring");
  cuda::Buffer<float> sig(signals.data.size());
  cuda::upload_f32(sig, signals.data);
  cuda::Buffer<float> out(static_cast<size_t>(grid.width) * grid.height);
  pact_ring r = signals.geom.c();
  pact_signal_meta m = signals.meta();
  pact_grid g = grid.c();
  pact_body b{body.center.x, body.center.y, body.radius, body.body_sos};
  cuda::check(pact_dual_sos_das(cuda::context(), &r, &m, sig.ptr, &g, v0, &b, out.ptr));
  RasterGrid img = RasterGrid::zeros(grid);
  img.values = cuda::download_f64(out);
  return img;
}

}  // namespace pact

#endif
