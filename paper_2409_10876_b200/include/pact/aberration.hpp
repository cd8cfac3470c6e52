// Drop-in host API — part 2, wavefront profiles and transfer stacks, and the
// adjoints: the fused ray trace (the training path) and the composed
// transfer_grad_to_wavefront / Jacobian rows / accumulate_wavefront_grad
// (reference: proj/include/pact/aberration.hpp:105-361).
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

  struct JacobianEntry {
    int32_t pixel;
    float dw_dv;  // mm per (m/s)
  };
  std::vector<std::vector<JacobianEntry>> jacobian;  // per angle; empty if not requested

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

/// wavefront_profile (aberration.hpp:134-186).  with_jacobian = true runs the
/// fp64 composed-path kernel (pact_wavefront_jacobian) and returns the sparse
/// rows w.r.t. the in-mask SOS pixels; otherwise the fp32 training-path march.
inline WavefrontProfile wavefront_profile(Vec2 center, const RingGeometry& geom,
                                          const RasterGrid& sos, double v0,
                                          const CircularMask& mask, int n_angles, double step_mm,
                                          bool with_jacobian) {
  geom.validate();
  pact_ring r = geom.c();
  pact_grid g = sos.spec().c();
  pact_mask m = mask.c();
  cuda::Buffer<float> dev(sos.values.size());
  detail::upload_sos_dev(dev, sos, v0);
  double c[2] = {center.x, center.y};
  WavefrontProfile p;
  p.center = center;
  p.n_angles = n_angles;
  if (with_jacobian) {
    const int A = n_angles > 0 ? n_angles : 1;
    cuda::Buffer<int64_t> rs(A + 1);
    int64_t nnz = 0;
    cuda::check(pact_wavefront_jacobian(cuda::context(), &r, &g, dev.ptr, v0, &m, 1, c, n_angles,
                                        step_mm, nullptr, rs.ptr, nullptr, nullptr, 0, &nnz));
    cuda::Buffer<double> w(A);
    cuda::Buffer<int32_t> pix(nnz > 0 ? nnz : 1);
    cuda::Buffer<float> val(nnz > 0 ? nnz : 1);
    cuda::check(pact_wavefront_jacobian(cuda::context(), &r, &g, dev.ptr, v0, &m, 1, c, n_angles,
                                        step_mm, w.ptr, rs.ptr, pix.ptr, val.ptr, pix.n, &nnz));
    p.w.resize(A);
    w.download(p.w.data());
    std::vector<int64_t> start(A + 1);
    rs.download(start.data());
    std::vector<int32_t> px(pix.n);
    std::vector<float> vv(val.n);
    pix.download(px.data());
    val.download(vv.data());
    p.jacobian.resize(A);
    for (int a = 0; a < A; ++a)
      for (int64_t e = start[a]; e < start[a + 1]; ++e) p.jacobian[a].push_back({px[e], vv[e]});
    return p;
  }
  cuda::Buffer<float> w(n_angles > 0 ? n_angles : 1);
  cuda::check(pact_wavefront(cuda::context(), &r, &g, dev.ptr, v0, &m, 1, c, n_angles, step_mm,
                             w.ptr));
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

/// transfer_grad_to_wavefront (aberration.hpp:270-313): dL/dH (per delay, per
/// bin; dL/dRe H + i dL/dIm H) -> dL/dw per profile angle, fp64 on the GPU.
inline std::vector<double> transfer_grad_to_wavefront(
    const WavefrontProfile& profile, const std::vector<double>& delays, int patch_pixels,
    double pitch, const std::vector<std::vector<cplx>>& grad_h) {
  const int P = patch_pixels, A = profile.n_angles, K = static_cast<int>(delays.size());
  const size_t P2 = static_cast<size_t>(P > 0 ? P : 1) * (P > 0 ? P : 1);
  if (static_cast<int>(grad_h.size()) != K)
    throw ValidationError("transfer_grad_to_wavefront: gradient / delay count mismatch");
  cuda::Buffer<double> w(A > 0 ? A : 1), dw(A > 0 ? A : 1), g(2 * P2 * (K > 0 ? K : 1));
  w.upload(profile.w.data());
  std::vector<cplx> flat;
  flat.reserve(P2 * K);
  for (const auto& gj : grad_h) {
    if (gj.size() != P2) throw ValidationError("transfer_grad_to_wavefront: spectrum size mismatch");
    flat.insert(flat.end(), gj.begin(), gj.end());
  }
  g.upload(reinterpret_cast<const double*>(flat.data()));
  cuda::check(pact_transfer_grad_to_wavefront(cuda::context(), 1, w.ptr, A, delays.data(), K, P,
                                              pitch, g.ptr, dw.ptr));
  std::vector<double> out(A);
  dw.download(out.data());
  return out;
}

/// accumulate_wavefront_grad (aberration.hpp:316-326): grad_v += J^T dL/dw over
/// the profile's Jacobian rows (on the GPU; fp64 accumulation).
inline void accumulate_wavefront_grad(const WavefrontProfile& profile,
                                      const std::vector<double>& dw,
                                      std::vector<double>& grad_v) {
  if (profile.jacobian.empty())
    throw ValidationError("accumulate_wavefront_grad: profile has no jacobian");
  const int A = profile.n_angles;
  std::vector<int64_t> start(A + 1, 0);
  for (int a = 0; a < A; ++a) start[a + 1] = start[a] + profile.jacobian[a].size();
  const int64_t nnz = start[A];
  std::vector<int32_t> px(nnz > 0 ? nnz : 1);
  std::vector<float> vv(nnz > 0 ? nnz : 1);
  for (int a = 0; a < A; ++a)
    for (size_t e = 0; e < profile.jacobian[a].size(); ++e) {
      px[start[a] + e] = profile.jacobian[a][e].pixel;
      vv[start[a] + e] = profile.jacobian[a][e].dw_dv;
    }
  cuda::Buffer<int64_t> rs(A + 1);
  cuda::Buffer<int32_t> pix(px.size());
  cuda::Buffer<float> val(vv.size());
  cuda::Buffer<double> d(A > 0 ? A : 1), gv(grad_v.size());
  rs.upload(start.data());
  pix.upload(px.data());
  val.upload(vv.data());
  d.upload(dw.data());
  gv.upload(grad_v.data());
  cuda::check(pact_accumulate_wavefront_grad(cuda::context(), A, rs.ptr, pix.ptr, val.ptr, d.ptr,
                                             gv.ptr));
  gv.download(grad_v.data());
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
/// origin chosen so that pixel sits at world (0, 0)).  On the GPU in fp64
/// (pact_psf_from_transfer): the symmetry check, the inverse 2-D DFT (rows,
/// then columns, scaled 1 / P^2), the imaginary-residue check and the
/// centring shift, with the reference's thresholds and messages.
inline RasterGrid psf_from_transfer(const std::vector<cplx>& spectrum, int patch_pixels,
                                    double pitch = 1.0) {
  const int P = patch_pixels;
  if (P < 1 || spectrum.size() != static_cast<size_t>(P) * P)
    throw ValidationError("psf_from_transfer: spectrum size mismatch");
  const size_t P2 = static_cast<size_t>(P) * P;
  cuda::Buffer<double> s(2 * P2), out(P2);
  cuda::check(pact_upload(cuda::context(), s.ptr, spectrum.data(), sizeof(cplx) * P2));
  cuda::check(pact_psf_from_transfer(cuda::context(), 1, P, s.ptr, out.ptr));
  GridSpec gs{P, P, pitch, {-(P / 2) * pitch, -(P / 2) * pitch}};
  RasterGrid psf = RasterGrid::zeros(gs);
  out.download(psf.values.data());
  return psf;
}

}  // namespace pact

#endif
