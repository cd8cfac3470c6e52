// Drop-in host API — part 3, patch spectra and the multichannel Wiener
// deconvolution pipeline (reference: proj/include/pact/deconv.hpp:39-198).
#ifndef PACT_B200_DECONV_HPP
#define PACT_B200_DECONV_HPP

#include <complex>
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
