// Standalone C-ABI entry points of include/pact_cuda.h (layout, SIREN,
// spectra, deconvolution, TV, Adam).  Each one mirrors one reference function
// (same validation order and messages) over device buffers; they share the
// kernels of the training engine (trainer.cu).
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "geom.cuh"
#include "siren.cuh"
#include "train_ops.cuh"

namespace pactgpu {

Status make_layout(const pact_grid& grid, double patch_mm, double overlap, pact_layout& out) {
  // make_patch_layout, core.hpp:252-281
  if (grid.width < 1 || grid.height < 1) return validation("grid: width and height must be >= 1");
  if (!(grid.pitch > 0.0)) return validation("grid: pitch must be > 0");
  if (!(overlap >= 0.0 && overlap < 1.0))
    return validation("patch layout: overlap must be in [0, 1)");
  int P = static_cast<int>(std::lround(patch_mm / grid.pitch));
  if (P < 1) return validation("patch layout: patch smaller than one pixel");
  if (P > grid.width || P > grid.height) {
    std::string m = "patch layout: patch of " + std::to_string(P) + " px exceeds grid extent";
    set_error("%s", m.c_str());
    return {PACT_E_VALIDATION};
  }
  int stride = std::max(1, static_cast<int>(std::lround(P * (1.0 - overlap))));
  auto count = [&](int extent) {  // detail::patch_offsets_1d, core.hpp:232-241
    if (extent <= P) return 1;
    int last = extent - P, n = 0;
    for (int o = 0; o < last; o += stride) ++n;
    return n + 1;
  };
  out.grid = grid;
  out.patch_pixels = P;
  out.stride_pixels = stride;
  out.nx = count(grid.width);
  out.ny = count(grid.height);
  out.last_x = grid.width <= P ? 0 : grid.width - P;
  out.last_y = grid.height <= P ? 0 : grid.height - P;
  return {};
}

void layout_centers(const pact_layout& lay, double* centers) {
  const double half = 0.5 * (lay.patch_pixels - 1);
  for (int py = 0; py < lay.ny; ++py)
    for (int px = 0; px < lay.nx; ++px) {
      int ox = px == lay.nx - 1 ? lay.last_x : px * lay.stride_pixels;
      int oy = py == lay.ny - 1 ? lay.last_y : py * lay.stride_pixels;
      int i = py * lay.nx + px;
      centers[2 * i] = lay.grid.origin_x + (ox + half) * lay.grid.pitch;
      centers[2 * i + 1] = lay.grid.origin_y + (oy + half) * lay.grid.pitch;
    }
}

namespace {

bool same_grid(const pact_grid& a, const pact_grid& b) {
  return a.width == b.width && a.height == b.height && a.pitch == b.pitch &&
         a.origin_x == b.origin_x && a.origin_y == b.origin_y;
}

SirenShape shape_of(const pact_siren& s) {
  SirenShape sh;
  sh.in_dim = s.in_dim;
  sh.hidden = s.hidden;
  sh.layers = s.n_hidden_layers;
  sh.omega0 = s.omega0;
  sh.out_scale = s.out_scale;
  sh.v0 = s.v0;
  return sh;
}

// Cached per-(grid, mask) state of the standalone entry points.
struct ApiCache {
  pact_grid grid{};
  pact_mask mask{};
  bool valid = false;
  MaskedPixels mp;
  SirenWork sw;
  int sw_hidden = -1, sw_layers = -1;
  unsigned char* inmask = nullptr;
  FourierTable ftab;
  ~ApiCache() {
    siren_work_free(sw);
    if (inmask) cudaFree(inmask);
    fourier_table_free(ftab);
  }
};

void api_free(void* p) { delete static_cast<ApiCache*>(p); }

ApiCache* cache(pact_ctx* ctx) {
  if (!ctx->api) {
    ctx->api = new ApiCache();
    ctx->api_free = api_free;
  }
  return static_cast<ApiCache*>(ctx->api);
}

Status masked_state(pact_ctx* ctx, const pact_grid& g, const pact_mask& m, ApiCache*& c) {
  c = cache(ctx);
  if (c->valid && same_grid(c->grid, g) && c->mask.center_x == m.center_x &&
      c->mask.center_y == m.center_y && c->mask.radius == m.radius)
    return {};
  PACT_CUDA_S(cudaStreamSynchronize(ctx->stream));
  siren_work_free(c->sw);
  c->sw_hidden = c->sw_layers = -1;
  if (c->inmask) cudaFree(c->inmask);
  c->inmask = nullptr;
  c->mp = masked_pixels(g, m);
  std::vector<unsigned char> flag(static_cast<size_t>(g.width) * g.height, 0);
  for (int i : c->mp.idx) flag[i] = 1;
  PACT_CUDA_S(cudaMalloc(&c->inmask, flag.size()));
  PACT_CUDA_S(cudaMemcpy(c->inmask, flag.data(), flag.size(), cudaMemcpyHostToDevice));
  c->grid = g;
  c->mask = m;
  c->valid = true;
  return {};
}

Status siren_state(pact_ctx* ctx, const pact_siren& s, const pact_grid& g, const pact_mask& m,
                   ApiCache*& c) {
  if (s.in_dim != 2) return validation("siren: only 2-D coordinates are supported");
  if (s.hidden < 1) return validation("init_siren: hidden must be >= 1");
  if (s.n_hidden_layers < 1) return validation("init_siren: need at least one sine layer");
  if (g.width < 1 || g.height < 1) return validation("grid: width and height must be >= 1");
  if (!(g.pitch > 0.0)) return validation("grid: pitch must be > 0");
  if (!(m.radius > 0.0)) return validation("render_sos: mask radius must be > 0");
  PACT_TRY_S(masked_state(ctx, g, m, c));
  if (c->sw_hidden != s.hidden || c->sw_layers != s.n_hidden_layers) {
    PACT_TRY_S(siren_work_alloc(c->sw, c->mp, shape_of(s), ctx->stream));
    c->sw_hidden = s.hidden;
    c->sw_layers = s.n_hidden_layers;
  }
  return {};
}

__global__ void add_const_kernel(const float* __restrict__ dv, size_t n, float v0,
                                 float* __restrict__ out) {
  size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = v0 + dv[i];
}

}  // namespace

// MergeWindow::make, deconv.hpp:124-138 (host fp64 -> fp32)
Status merge_window(double fwhm, int P, double pitch, std::vector<float>& w) {
  if (!(fwhm > 0.0)) return validation("merge window: FWHM must be > 0");
  double sigma_px = fwhm / (2.0 * std::sqrt(2.0 * std::log(2.0))) / pitch;
  double c = 0.5 * (P - 1);
  w.resize(static_cast<size_t>(P) * P);
  for (int y = 0; y < P; ++y)
    for (int x = 0; x < P; ++x) {
      double r2 = (x - c) * (x - c) + (y - c) * (y - c);
      w[static_cast<size_t>(y) * P + x] = static_cast<float>(std::exp(-0.5 * r2 / (sigma_px * sigma_px)));
    }
  return {};
}

Status launch_sos_from_dev(pact_ctx* ctx, const float* dv, size_t n, double v0, float* out) {
  add_const_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, ctx->stream>>>(
      dv, n, static_cast<float>(v0), out);
  return after_launch(ctx, "add_const_kernel");
}

}  // namespace pactgpu

using namespace pactgpu;

extern "C" {

int pact_make_patch_layout(const pact_grid* grid, double patch_mm, double overlap,
                           pact_layout* out) {
  if (!grid || !out) return validation("pact_make_patch_layout: null argument").code;
  return make_layout(*grid, patch_mm, overlap, *out).code;
}

int32_t pact_layout_n_patches(const pact_layout* layout) {
  return layout ? layout->nx * layout->ny : 0;
}

int pact_layout_patches(const pact_layout* lay, int32_t* offsets, double* centers) {
  if (!lay) return validation("pact_layout_patches: null layout").code;
  for (int py = 0; py < lay->ny; ++py)
    for (int px = 0; px < lay->nx; ++px) {
      int i = py * lay->nx + px;
      if (offsets) {
        offsets[2 * i] = px == lay->nx - 1 ? lay->last_x : px * lay->stride_pixels;
        offsets[2 * i + 1] = py == lay->ny - 1 ? lay->last_y : py * lay->stride_pixels;
      }
    }
  if (centers) layout_centers(*lay, centers);
  return PACT_OK;
}

int64_t pact_siren_param_count(const pact_siren* s) {
  if (!s) return -1;
  // siren_param_count, nfield.hpp:73-78
  int64_t n = static_cast<int64_t>(s->hidden) * s->in_dim + s->hidden;
  for (int l = 1; l < s->n_hidden_layers; ++l)
    n += static_cast<int64_t>(s->hidden) * s->hidden + s->hidden;
  n += s->hidden + 1;
  return n;
}

int pact_init_siren(uint64_t seed, const pact_siren* s, double* theta) {
  // init_siren, nfield.hpp:83-107 — same engine and distribution as the reference
  if (!s || !theta) return validation("pact_init_siren: null argument").code;
  if (s->hidden < 1) return validation("init_siren: hidden must be >= 1").code;
  if (s->n_hidden_layers < 1) return validation("init_siren: need at least one sine layer").code;
  if (!(s->omega0 > 0.0)) return validation("init_siren: omega0 must be > 0").code;
  SirenShape sh = shape_of(*s);
  std::mt19937_64 rng(seed);
  size_t off = 0;
  for (int l = 0; l <= sh.layers; ++l) {
    int rows = sh.rows(l), cols = sh.cols(l);
    double bound = (l == 0) ? 1.0 / sh.in_dim : std::sqrt(6.0 / cols) / sh.omega0;
    std::uniform_real_distribution<double> u(-bound, bound);
    size_t n = static_cast<size_t>(rows) * cols + rows;
    for (size_t i = 0; i < n; ++i) theta[off + i] = u(rng);
    off += n;
  }
  return PACT_OK;
}

int32_t pact_masked_count(const pact_grid* grid, const pact_mask* mask) {
  if (!grid || !mask) return -1;
  return masked_pixels(*grid, *mask).n;
}

int pact_masked_pixels(const pact_grid* grid, const pact_mask* mask, int32_t* idx, float* coords) {
  if (!grid || !mask) return validation("pact_masked_pixels: null argument").code;
  MaskedPixels mp = masked_pixels(*grid, *mask);
  if (idx) std::memcpy(idx, mp.idx.data(), sizeof(int) * mp.n);
  if (coords) std::memcpy(coords, mp.coords.data(), sizeof(float) * 2 * mp.n);
  return PACT_OK;
}

int pact_render_sos(pact_ctx* ctx, const pact_siren* s, const float* theta, const pact_grid* grid,
                    const pact_mask* mask, float* raster, float* sos_dev) {
  if (!ctx || !s || !theta || !grid || !mask)
    return validation("pact_render_sos: null argument").code;
  ApiCache* c = nullptr;
  PACT_TRY(siren_state(ctx, *s, *grid, *mask, c));
  const size_t n = static_cast<size_t>(grid->width) * grid->height;
  void* tmp = nullptr;
  float* dv = sos_dev;
  if (!dv) {
    PACT_TRY(scratch_get(ctx, kScratchGeneric0, sizeof(float) * n, &tmp));
    dv = static_cast<float*>(tmp);
  }
  PACT_CUDA(cudaMemsetAsync(dv, 0, sizeof(float) * n, ctx->stream));
  PACT_TRY(siren_forward(ctx, shape_of(*s), theta, c->sw, dv));
  if (raster) PACT_TRY(launch_sos_from_dev(ctx, dv, n, s->v0, raster));
  return PACT_OK;
}

int pact_siren_backward(pact_ctx* ctx, const pact_siren* s, const float* theta,
                        const pact_grid* grid, const pact_mask* mask, const float* grad_masked,
                        double* grad_theta) {
  if (!ctx || !s || !theta || !grid || !mask || !grad_masked || !grad_theta)
    return validation("pact_siren_backward: null argument").code;
  ApiCache* c = nullptr;
  PACT_TRY(siren_state(ctx, *s, *grid, *mask, c));
  const size_t n = static_cast<size_t>(grid->width) * grid->height;
  void* tmp = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric0, sizeof(float) * n, &tmp));
  SirenShape sh = shape_of(*s);
  PACT_TRY(siren_forward(ctx, sh, theta, c->sw, static_cast<float*>(tmp)));
  PACT_TRY(siren_backward(ctx, sh, theta, c->sw, nullptr, grad_masked, grad_theta));
  return PACT_OK;
}

int pact_patch_spectra(pact_ctx* ctx, const pact_layout* lay, const float* stack, int32_t K,
                       float* Y) {
  if (!ctx || !lay || !stack || !Y) return validation("pact_patch_spectra: null argument").code;
  if (K < 1) return validation("extract_patch_spectra: empty stack").code;
  PACT_TRY(launch_patch_fft(ctx, *lay, stack, K, reinterpret_cast<float2*>(Y)));
  return PACT_OK;
}

int pact_deconvolve_image(pact_ctx* ctx, const float* stack, int32_t K, const double* delays,
                          double v0, const float* sos_dev, const pact_ring* ring,
                          const pact_mask* mask, const pact_layout* lay,
                          const pact_deconv_options* opt, float* image) {
  if (!ctx || !stack || !sos_dev || !ring || !mask || !lay || !opt || !image ||
      (!delays && K > 0))
    return validation("pact_deconvolve_image: null argument").code;
  if (K < 1) return validation("deconvolve_image: empty stack").code;
  const int n = lay->nx * lay->ny, P = lay->patch_pixels, P2 = P * P;
  std::vector<double> centers(2 * n);
  layout_centers(*lay, centers.data());
  RayArgs ra{};
  PACT_TRY(ray_args(*ring, lay->grid, v0, *mask, opt->n_angles, opt->ray_step, ra));
  PACT_TRY(validate_centers(*ring, n, centers.data()));
  std::vector<float> win;
  PACT_TRY(merge_window(opt->merge_fwhm, P, lay->grid.pitch, win));
  ApiCache* c = cache(ctx);
  PACT_TRY(fourier_table(ctx, c->ftab, P, lay->grid.pitch, opt->n_angles, delays, K));
  // scratch: Y [n][K][P2] c64 | w [n][A] | X [n][P2] c64 | patches [n][P2] | centres | window
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t oY = 0, ow = al(oY + sizeof(float2) * static_cast<size_t>(n) * K * P2),
         oX = al(ow + sizeof(float) * static_cast<size_t>(n) * opt->n_angles),
         oP = al(oX + sizeof(float2) * static_cast<size_t>(n) * P2),
         oC = al(oP + sizeof(float) * static_cast<size_t>(n) * P2),
         oW = al(oC + sizeof(double2) * n), total = al(oW + sizeof(float) * P2);
  void* base = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric1, total, &base));
  char* b = static_cast<char*>(base);
  float2* Y = reinterpret_cast<float2*>(b + oY);
  float* w = reinterpret_cast<float*>(b + ow);
  float2* X = reinterpret_cast<float2*>(b + oX);
  float* patches = reinterpret_cast<float*>(b + oP);
  double2* dc = reinterpret_cast<double2*>(b + oC);
  float* dwin = reinterpret_cast<float*>(b + oW);
  PACT_CUDA(cudaMemcpyAsync(dc, centers.data(), sizeof(double2) * n, cudaMemcpyHostToDevice,
                            ctx->stream));
  PACT_CUDA(cudaMemcpyAsync(dwin, win.data(), sizeof(float) * P2, cudaMemcpyHostToDevice,
                            ctx->stream));
  PACT_TRY(launch_patch_fft(ctx, *lay, stack, K, Y));
  ra.dv = sos_dev;
  ra.centers = dc;
  ra.n_rays = n * opt->n_angles;
  make_raster_texture(sos_dev, lay->grid.width, lay->grid.height, &ra.tex);
  Status wst = ray_plan_cached(ctx, ra, centers.data(), n);
  if (wst.ok()) wst = launch_wavefront(ctx, ra, w);
  if (ra.tex) {
    cudaStreamSynchronize(ctx->stream);
    cudaDestroyTextureObject(ra.tex);
  }
  PACT_TRY(wst);
  PACT_TRY(launch_wiener(ctx, c->ftab.tab, Y, w, n, opt->eps, X));
  PACT_TRY(launch_patch_ifft_real(ctx, P, n, X, patches));
  PACT_TRY(launch_merge(ctx, *lay, patches, dwin, image));
  PACT_CUDA(cudaStreamSynchronize(ctx->stream));  // host vectors above are released
  return PACT_OK;
}

int pact_merge_window(double fwhm_mm, int32_t P, double pitch, double* weights) {
  if (!weights) return validation("pact_merge_window: null argument").code;
  if (!(fwhm_mm > 0.0)) return validation("merge window: FWHM must be > 0").code;
  // MergeWindow::make, deconv.hpp:124-138
  const double sigma_px = fwhm_mm / (2.0 * std::sqrt(2.0 * std::log(2.0))) / pitch;
  const double c = 0.5 * (P - 1);
  for (int y = 0; y < P; ++y)
    for (int x = 0; x < P; ++x) {
      const double r2 = (x - c) * (x - c) + (y - c) * (y - c);
      weights[static_cast<size_t>(y) * P + x] = std::exp(-0.5 * r2 / (sigma_px * sigma_px));
    }
  return PACT_OK;
}

int pact_merge_patches(pact_ctx* ctx, const pact_layout* lay, const float* patches,
                       const double* window, double fwhm, float* image) {
  if (!ctx || !lay || !patches || !image) return validation("pact_merge_patches: null argument").code;
  const int P = lay->patch_pixels, P2 = P * P;
  if (P < 1 || lay->nx < 1 || lay->ny < 1) return validation("merge_patches: empty layout").code;
  std::vector<float> win;
  if (window) {
    win.assign(window, window + P2);
  } else {
    PACT_TRY(merge_window(fwhm, P, lay->grid.pitch, win));  // MergeWindow::make, deconv.hpp:124-138
  }
  void* dwin = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric3, sizeof(float) * P2, &dwin));
  PACT_CUDA(cudaMemcpyAsync(dwin, win.data(), sizeof(float) * P2, cudaMemcpyHostToDevice,
                            ctx->stream));
  PACT_TRY(launch_merge(ctx, *lay, patches, static_cast<const float*>(dwin), image));
  PACT_CUDA(cudaStreamSynchronize(ctx->stream));  // `win` is released
  return PACT_OK;
}

int pact_tv_loss(pact_ctx* ctx, const pact_grid* grid, const pact_mask* mask, const float* raster,
                 double lambda, double* value, float* grad_masked) {
  if (!ctx || !grid || !mask || !raster || !value || !grad_masked)
    return validation("pact_tv_loss: null argument").code;
  ApiCache* c = nullptr;
  PACT_TRY(masked_state(ctx, *grid, *mask, c));
  int* didx = nullptr;
  const int n = c->mp.n;
  const int nb = std::max(1, std::min(div_up(std::max(n, 1), 256), ctx->num_sms * 4));
  void* tmp = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric2, sizeof(double) * nb + sizeof(int) * std::max(n, 1),
                       &tmp));
  double* partial = static_cast<double*>(tmp);
  didx = reinterpret_cast<int*>(partial + nb);
  if (n > 0)
    PACT_CUDA(cudaMemcpyAsync(didx, c->mp.idx.data(), sizeof(int) * n, cudaMemcpyHostToDevice,
                              ctx->stream));
  PACT_TRY(launch_tv(ctx, raster, c->inmask, didx, n, grid->width, grid->height, lambda,
                     grad_masked, partial, nb));
  std::vector<double> hp(nb);
  PACT_CUDA(cudaMemcpyAsync(hp.data(), partial, sizeof(double) * nb, cudaMemcpyDeviceToHost,
                            ctx->stream));
  PACT_CUDA(cudaStreamSynchronize(ctx->stream));
  double v = 0.0;
  for (double p : hp) v += p;
  *value = v * lambda;
  return PACT_OK;
}

int pact_adam_step(pact_ctx* ctx, int64_t n, double* theta, const double* grad, double* m,
                   double* v, int64_t t, double lr, double beta1, double beta2, double eps) {
  if (!ctx || !theta || !grad || !m || !v) return validation("pact_adam_step: null argument").code;
  if (t < 1) return validation("adam_step: step count must be >= 1").code;
  void* tmp = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchTables, 64, &tmp));
  unsigned* flags = static_cast<unsigned*>(tmp);
  long long* tdev = reinterpret_cast<long long*>(static_cast<char*>(tmp) + 16);
  long long th = t;
  PACT_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned), ctx->stream));
  PACT_CUDA(cudaMemcpyAsync(tdev, &th, sizeof(th), cudaMemcpyHostToDevice, ctx->stream));
  PACT_TRY(launch_check_finite_f64(ctx, grad, static_cast<int>(n), kFlagGrad, flags));
  unsigned hf = 0;
  PACT_CUDA(cudaMemcpyAsync(&hf, flags, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
  PACT_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hf) {
    set_error("adam_step: non-finite gradient");
    return PACT_E_NUMERICAL;
  }
  PACT_TRY(launch_adam(ctx, static_cast<int>(n), theta, grad, m, v, tdev, lr, beta1, beta2, eps,
                       flags, nullptr, false));
  PACT_CUDA(cudaStreamSynchronize(ctx->stream));
  return PACT_OK;
}

}  // extern "C"
