// Drop-in host API — part 3, patch spectra and the multichannel Wiener
// deconvolution pipeline (reference: proj/include/pact/deconv.hpp:39-198).
#ifndef PACT_B200_DECONV_HPP
#define PACT_B200_DECONV_HPP

#include <cmath>
#include <complex>
#include <utility>
#include <vector>

#include "pact/aberration.hpp"
#include "pact/beamform.hpp"

namespace pact {

struct PatchSpectra {
  int patch_index = 0;
  std::pair<int, int> offset;
  std::vector<std::vector<cplx>> Y;  // per delay, P*P row-major
};

namespace detail {
inline void upload_stack(cuda::Buffer<float>& b, const DasStack& stack) {
  std::vector<float> f;
  for (const auto& img : stack.images)
    for (double v : img.values) f.push_back(static_cast<float>(v));
  b.upload(f.data());
}
}  // namespace detail

/// extract_patch_spectra (deconv.hpp:64-74): fp32 batched FFT on the GPU.
inline std::vector<PatchSpectra> extract_patch_spectra(const DasStack& stack,
                                                       const PatchLayout& layout,
                                                       int workers = 0) {
  (void)workers;
  if (stack.images.empty()) throw ValidationError("extract_patch_spectra: empty stack");
  if (!stack.images[0].spec().same_geometry(layout.grid))
    throw ValidationError("extract_patch_spectra: layout grid does not match stack grid");
  const int K = stack.n_delays(), P = layout.patch_pixels, n = layout.n_patches();
  const size_t P2 = static_cast<size_t>(P) * P;
  cuda::Buffer<float> st(stack.images[0].values.size() * K);
  detail::upload_stack(st, stack);
  cuda::Buffer<float> Y(2 * P2 * K * n);
  pact_layout l = layout.c();
  cuda::check(pact_patch_spectra(cuda::context(), &l, st.ptr, K, Y.ptr));
  std::vector<double> y = cuda::download_f64(Y);
  std::vector<PatchSpectra> out(n);
  for (int i = 0; i < n; ++i) {
    out[i].patch_index = i;
    out[i].offset = layout.offsets[i];
    for (int j = 0; j < K; ++j) {
      std::vector<cplx> c(P2);
      size_t base = (static_cast<size_t>(i) * K + j) * P2;
      for (size_t b = 0; b < P2; ++b) c[b] = {y[2 * (base + b)], y[2 * (base + b) + 1]};
      out[i].Y.push_back(std::move(c));
    }
  }
  return out;
}

namespace detail {
/// PatchSpectra / TransferStack channels -> one complex128 device block [K][P2].
inline void upload_c128(cuda::Buffer<double>& b, const std::vector<std::vector<cplx>>& chans,
                        size_t offset_values = 0) {
  std::vector<cplx> flat;
  for (const auto& c : chans) flat.insert(flat.end(), c.begin(), c.end());
  if (flat.size() * 2 + offset_values > b.n)
    throw ValidationError("spectra: channel sizes differ");
  cuda::check(pact_upload(cuda::context(), b.ptr + offset_values, flat.data(),
                          sizeof(cplx) * flat.size()));
}
}  // namespace detail

/// multichannel_deconvolve (deconv.hpp:78-96), fp64 on the GPU:
///   X(k) = sum_j conj(H_j) Y_j / (sum_j |H_j|^2 + eps * M).
inline std::vector<cplx> multichannel_deconvolve(const PatchSpectra& ys, const TransferStack& hs,
                                                 double eps) {
  if (ys.Y.size() != hs.spectra.size())
    throw ValidationError("deconvolve: Y and H channel counts differ");
  if (ys.Y.empty()) throw ValidationError("deconvolve: no channels");
  const size_t P2 = ys.Y[0].size();
  const int P = static_cast<int>(std::lround(std::sqrt(static_cast<double>(P2))));
  const int K = static_cast<int>(ys.Y.size());
  cuda::Buffer<double> Y(2 * P2 * K), H(2 * P2 * K), X(2 * P2);
  detail::upload_c128(Y, ys.Y);
  detail::upload_c128(H, hs.spectra);
  cuda::check(pact_multichannel_deconvolve(cuda::context(), 1, K, P, Y.ptr, H.ptr, eps, X.ptr));
  std::vector<cplx> x(P2);
  X.download(reinterpret_cast<double*>(x.data()));
  return x;
}

/// deconv_jacobian_H (deconv.hpp:100-115): dX(bin)/d(Re H_j(bin)), dX(bin)/d(Im H_j(bin)).
inline std::pair<cplx, cplx> deconv_jacobian_H(const PatchSpectra& ys, const TransferStack& hs,
                                               double eps, size_t j, size_t bin) {
  const size_t P2 = ys.Y.at(0).size();
  const int P = static_cast<int>(std::lround(std::sqrt(static_cast<double>(P2))));
  const int K = static_cast<int>(ys.Y.size());
  cuda::Buffer<double> Y(2 * P2 * K), H(2 * P2 * K), out(4);
  detail::upload_c128(Y, ys.Y);
  detail::upload_c128(H, hs.spectra);
  int32_t q[3] = {0, static_cast<int32_t>(j), static_cast<int32_t>(bin)};
  cuda::Buffer<int32_t> dq(3);
  dq.upload(q);
  cuda::check(pact_deconv_jacobian_H(cuda::context(), K, P, Y.ptr, H.ptr, eps, 1, dq.ptr, out.ptr));
  double o[4];
  out.download(o);
  return {cplx(o[0], o[1]), cplx(o[2], o[3])};
}

/// Gaussian merging window, peak 1 at the patch center (deconv.hpp:118-139).
struct MergeWindow {
  double fwhm_mm = 0.0;
  int patch_pixels = 0;
  std::vector<double> weights;  // P*P, > 0

  static MergeWindow make(double fwhm_mm, int patch_pixels, double pitch) {
    if (!(fwhm_mm > 0.0)) throw ValidationError("merge window: FWHM must be > 0");
    MergeWindow w;
    w.fwhm_mm = fwhm_mm;
    w.patch_pixels = patch_pixels;
    w.weights.resize(static_cast<size_t>(patch_pixels) * patch_pixels);
    cuda::check(pact_merge_window(fwhm_mm, patch_pixels, pitch, w.weights.data()));
    return w;
  }
};

/// merge_patches (deconv.hpp:142-164): weight-normalised overlap-add on the GPU.
inline RasterGrid merge_patches(const std::vector<std::vector<double>>& patches,
                                const PatchLayout& layout, const MergeWindow& window) {
  if (patches.size() != static_cast<size_t>(layout.n_patches()))
    throw ValidationError("merge_patches: patch count does not match layout");
  const int P = layout.patch_pixels;
  if (window.patch_pixels != P)
    throw ValidationError("merge_patches: window size does not match layout");
  const size_t P2 = static_cast<size_t>(P) * P;
  std::vector<float> f;
  f.reserve(P2 * patches.size());
  for (const auto& p : patches) {
    if (p.size() != P2) throw ValidationError("merge_patches: patch size does not match layout");
    for (double v : p) f.push_back(static_cast<float>(v));
  }
  cuda::Buffer<float> dp(f.size()),
      img(static_cast<size_t>(layout.grid.width) * layout.grid.height);
  dp.upload(f.data());
  pact_layout l = layout.c();
  cuda::check(pact_merge_patches(cuda::context(), &l, dp.ptr, window.weights.data(),
                                 window.fwhm_mm, img.ptr));
  RasterGrid out = RasterGrid::zeros(layout.grid);
  out.values = cuda::download_f64(img);
  return out;
}

struct DeconvolveOptions {
  double eps = 1e-3;
  int n_angles = 512;
  double ray_step = 0.05;  // mm
  double merge_fwhm = 1.5;  // mm
  int workers = 0;
};

/// deconvolve_image (deconv.hpp:176-198): spectra -> wavefronts -> H ->
/// pseudo-inverse -> inverse FFT -> Gaussian merge, all on the GPU.
inline RasterGrid deconvolve_image(const DasStack& stack, const RasterGrid& sos,
                                   const RingGeometry& geom, const CircularMask& mask,
                                   const PatchLayout& layout, const DeconvolveOptions& opt = {}) {
  if (stack.images.empty()) throw ValidationError("deconvolve_image: empty stack");
  if (!stack.images[0].spec().same_geometry(layout.grid))
    throw ValidationError("deconvolve_image: layout grid does not match stack grid");
  const int K = stack.n_delays();
  cuda::Buffer<float> st(stack.images[0].values.size() * K);
  detail::upload_stack(st, stack);
  cuda::Buffer<float> dev(sos.values.size());
  detail::upload_sos_dev(dev, sos, stack.v0);
  cuda::Buffer<float> img(sos.values.size());
  pact_ring r = geom.c();
  pact_mask m = mask.c();
  pact_layout l = layout.c();
  pact_deconv_options o{opt.eps, opt.n_angles, opt.ray_step, opt.merge_fwhm};
  cuda::check(pact_deconvolve_image(cuda::context(), st.ptr, K, stack.delays.data(), stack.v0,
                                    dev.ptr, &r, &m, &l, &o, img.ptr));
  RasterGrid out = RasterGrid::zeros(layout.grid);
  out.values = cuda::download_f64(img);
  return out;
}

}  // namespace pact

#endif
