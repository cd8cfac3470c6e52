// Drop-in host API — part 2, wavefront profiles and transfer stacks, and the
// adjoint ray trace (reference: proj/include/pact/aberration.hpp:105-361).
//
// Deviation from the reference (documented in INTEGRATION.md): the sparse
// per-angle Jacobian rows (`with_jacobian = true`) are not materialised — the
// GPU training path uses wavefront_grad_trace instead, exactly as the
// reference's own training loop does (optimize.hpp:437-438).
#ifndef PACT_B200_ABERRATION_HPP
#define PACT_B200_ABERRATION_HPP

#include <algorithm>
#include <cmath>
#include <complex>
#include <string>
#include <vector>

#include "pact/core.hpp"

namespace pact {

using cplx = std::complex<double>;

struct WavefrontProfile {
  Vec2 center;
  int n_angles = 0;
  std::vector<double> w;  // mm, w[a] for direction 2 pi a / n_angles

  double angle(int a) const { return 2.0 * M_PI * a / n_angles; }
  double interpolate(double theta) const {
    const double tau = 2.0 * M_PI;
    double pos = std::fmod(theta, tau);
    if (pos < 0) pos += tau;
    pos = pos / tau * n_angles;
    int a0 = static_cast<int>(pos) % n_angles;
    double f = pos - std::floor(pos);
    return (1.0 - f) * w[a0] + f * w[(a0 + 1) % n_angles];
  }
};

namespace detail {
/// The SOS raster as the fp32 deviation v - v0 the ray kernels consume.
inline void upload_sos_dev(cuda::Buffer<float>& b, const RasterGrid& sos, double v0) {
  cuda::upload_f32(b, sos.values, v0);
}
}  // namespace detail

/// wavefront_profile (aberration.hpp:134-186).
inline WavefrontProfile wavefront_profile(Vec2 center, const RingGeometry& geom,
                                          const RasterGrid& sos, double v0,
                                          const CircularMask& mask, int n_angles, double step_mm,
                                          bool with_jacobian) {
  geom.validate();
  if (with_jacobian)
    throw ValidationError("wavefront_profile: Jacobian rows are not produced by the GPU path "
                          "(use wavefront_grad_trace)");
  pact_ring r = geom.c();
  pact_grid g = sos.spec().c();
  pact_mask m = mask.c();
  cuda::Buffer<float> dev(sos.values.size());
  detail::upload_sos_dev(dev, sos, v0);
  cuda::Buffer<float> w(n_angles > 0 ? n_angles : 1);
  double c[2] = {center.x, center.y};
  cuda::check(pact_wavefront(cuda::context(), &r, &g, dev.ptr, v0, &m, 1, c, n_angles, step_mm,
                             w.ptr));
  WavefrontProfile p;
  p.center = center;
  p.n_angles = n_angles;
  p.w = cuda::download_f64(w);
  return p;
}

struct TransferStack {
  int patch_pixels = 0;
  double pitch = 0.0;
  std::vector<double> delays;
  std::vector<std::vector<cplx>> spectra;  // per delay, P*P row-major
};

/// transfer_stack (aberration.hpp:236-265).
inline TransferStack transfer_stack(const WavefrontProfile& profile,
                                    const std::vector<double>& delays, int patch_pixels,
                                    double pitch) {
  const int P = patch_pixels;
  const int K = static_cast<int>(delays.size());
  cuda::Buffer<float> w(profile.w.size());
  cuda::upload_f32(w, profile.w);
  const size_t P2 = static_cast<size_t>(P > 0 ? P : 1) * (P > 0 ? P : 1);
  cuda::Buffer<float> H(2 * P2 * (K > 0 ? K : 1));
  cuda::check(pact_transfer_stack(cuda::context(), 1, w.ptr, profile.n_angles, delays.data(), K,
                                  P, pitch, H.ptr));
  std::vector<double> h = cuda::download_f64(H);
  TransferStack ts;
  ts.patch_pixels = P;
  ts.pitch = pitch;
  ts.delays = delays;
  for (int j = 0; j < K; ++j) {
    std::vector<cplx> s(P2);
    for (size_t b = 0; b < P2; ++b) s[b] = {h[2 * (j * P2 + b)], h[2 * (j * P2 + b) + 1]};
    ts.spectra.push_back(std::move(s));
  }
  return ts;
}

/// wavefront_grad_trace (aberration.hpp:333-361): grad_v += dL/dw -> dL/dv.
inline void wavefront_grad_trace(Vec2 center, const RingGeometry& geom, const RasterGrid& sos,
                                 double v0, const CircularMask& mask, int n_angles, double step_mm,
                                 const std::vector<double>& dw, std::vector<double>& grad_v) {
  pact_ring r = geom.c();
  pact_grid g = sos.spec().c();
  pact_mask m = mask.c();
  cuda::Buffer<float> dev(sos.values.size());
  detail::upload_sos_dev(dev, sos, v0);
  cuda::Buffer<float> d(dw.size());
  cuda::upload_f32(d, dw);
  cuda::Buffer<double> gv(grad_v.size());
  gv.upload(grad_v.data());
  double c[2] = {center.x, center.y};
  cuda::check(pact_ray_backward(cuda::context(), &r, &g, dev.ptr, v0, &m, 1, c, n_angles, step_mm,
                                d.ptr, gv.ptr));
  gv.download(grad_v.data());
}

/// psf_from_transfer (aberration.hpp:407-445): the real, centred PSF of one
/// conjugate-symmetric P x P transfer spectrum (zero lag at pixel (P/2, P/2),
/// origin chosen so that pixel sits at world (0, 0)).  Host-side (the
/// `psf dump` tool path): the symmetry check, a separable inverse DFT with an
/// exact twiddle table (scaled 1 / P^2), the imaginary-residue check and the
/// centring shift, with the reference's thresholds and messages.
inline RasterGrid psf_from_transfer(const std::vector<cplx>& spectrum, int patch_pixels,
                                    double pitch = 1.0) {
  const int P = patch_pixels;
  if (P < 1 || spectrum.size() != static_cast<size_t>(P) * P)
    throw ValidationError("psf_from_transfer: spectrum size mismatch");
  double max_mag = 0.0, asym = 0.0;
  for (const cplx& v : spectrum) max_mag = std::max(max_mag, std::abs(v));
  for (int by = 0; by < P; ++by)
    for (int bx = 0; bx < P; ++bx) {
      const cplx a = spectrum[static_cast<size_t>(by) * P + bx];
      const cplx b = spectrum[static_cast<size_t>((P - by) % P) * P + (P - bx) % P];
      asym = std::max(asym, std::abs(a - std::conj(b)));
    }
  if (asym > 1e-9 * std::max(1.0, max_mag))
    throw ValidationError("psf_from_transfer: spectrum not conjugate-symmetric, max asymmetry " +
                          std::to_string(asym));
  std::vector<cplx> tw(P);  // e^{+2 pi i k / P}
  for (int k = 0; k < P; ++k) {
    const double a = 2.0 * M_PI * k / P;
    tw[k] = {std::cos(a), std::sin(a)};
  }
  // rows, then columns (the reference's inverse_2d order), then 1 / P^2
  std::vector<cplx> rows(static_cast<size_t>(P) * P), out(static_cast<size_t>(P) * P);
  for (int y = 0; y < P; ++y)
    for (int x = 0; x < P; ++x) {
      cplx acc = 0.0;
      for (int k = 0; k < P; ++k)
        acc += spectrum[static_cast<size_t>(y) * P + k] * tw[(static_cast<size_t>(k) * x) % P];
      rows[static_cast<size_t>(y) * P + x] = acc;
    }
  const double inv = 1.0 / (static_cast<double>(P) * P);
  double max_real = 0.0, max_imag = 0.0;
  for (int y = 0; y < P; ++y)
    for (int x = 0; x < P; ++x) {
      cplx acc = 0.0;
      for (int k = 0; k < P; ++k)
        acc += rows[static_cast<size_t>(k) * P + x] * tw[(static_cast<size_t>(k) * y) % P];
      acc *= inv;
      out[static_cast<size_t>(y) * P + x] = acc;
      max_real = std::max(max_real, std::abs(acc.real()));
      max_imag = std::max(max_imag, std::abs(acc.imag()));
    }
  if (max_real > 0.0 && max_imag > 1e-9 * max_real)
    throw NumericalError("psf_from_transfer: imaginary residue " + std::to_string(max_imag) +
                         " exceeds 1e-9 of max " + std::to_string(max_real));
  GridSpec gs{P, P, pitch, {-(P / 2) * pitch, -(P / 2) * pitch}};
  RasterGrid psf = RasterGrid::zeros(gs);
  for (int y = 0; y < P; ++y)
    for (int x = 0; x < P; ++x)
      psf.at((x + P / 2) % P, (y + P / 2) % P) = out[static_cast<size_t>(y) * P + x].real();
  return psf;
}

}  // namespace pact

#endif
