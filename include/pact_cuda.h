/*
 * pact_cuda.h — C-ABI of the B200 (sm_100a) implementation of the NF-APACT
 * hot path.  This is the drop-in boundary: the reference library `pact`
 * (/root/reference/proj/include/pact/ headers) is header-only C++; its hot entry
 * points are re-exported here as plain `extern "C"` functions over POD structs,
 * raw pointers and sizes.  The C++ host API in
 * paper_2409_10876_b200/include/pact/ (same names/types as the reference)
 * is a thin layer over these calls, and so is the Python ctypes binding.
 *
 * Conventions
 *  - Every compute entry point works on DEVICE pointers (cudaMalloc'd, or
 *    torch CUDA tensors) and is asynchronous on the context's stream.  Host
 *    staging is done with pact_upload/pact_download (pinned or pageable).
 *  - Return value: PACT_OK (0), PACT_E_VALIDATION (2, the reference's
 *    ValidationError, CLI exit 2), PACT_E_NUMERICAL (3, NumericalError,
 *    CLI exit 3), PACT_E_CUDA (4, a CUDA runtime error), PACT_E_UNSUPPORTED (5).
 *    The message is available from pact_last_error() (thread-local).
 *  - Arithmetic on device is fp32 (fp64 where the reference's index math needs
 *    it); geometry scalars cross the boundary as double like the reference.
 *  - The reference's `workers` argument has no meaning here; it is accepted
 *    by the C++ layer and ignored.
 */
#ifndef PACT_CUDA_H
#define PACT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PACT_OK 0
#define PACT_E_VALIDATION 2
#define PACT_E_NUMERICAL 3
#define PACT_E_CUDA 4
#define PACT_E_UNSUPPORTED 5

#define PACT_ABI_VERSION 1

/* ---- geometry PODs (field meaning identical to the reference types) ---- */

/* RingGeometry, core.hpp:152-173: transducer n at angle 2*pi*n/N + angle_offset. */
typedef struct pact_ring {
  int32_t n_transducers;
  double radius;       /* mm */
  double angle_offset; /* rad */
} pact_ring;

/* GridSpec, core.hpp:58-89: pixel (0,0) centre at origin; row-major rasters. */
typedef struct pact_grid {
  int32_t width;
  int32_t height;
  double pitch;    /* mm */
  double origin_x; /* mm */
  double origin_y; /* mm */
} pact_grid;

/* SignalSet metadata, core.hpp:284-313 (the data is a separate N x T array). */
typedef struct pact_signal_meta {
  int32_t n_samples;
  double dt;             /* s */
  double t0;             /* s */
  double background_sos; /* m/s */
} pact_signal_meta;

/* CircularMask, core.hpp:175-180. */
typedef struct pact_mask {
  double center_x;
  double center_y;
  double radius; /* mm */
} pact_mask;

/* PatchLayout, core.hpp:222-281 (offsets are regenerated from nx/ny/stride). */
typedef struct pact_layout {
  pact_grid grid;
  int32_t patch_pixels;
  int32_t stride_pixels;
  int32_t nx;
  int32_t ny;
  int32_t last_x; /* clamped last offset along x (= width - P, or 0) */
  int32_t last_y;
} pact_layout;

/* ---- context, errors, memory ---- */

typedef struct pact_ctx pact_ctx;

int pact_abi_version(void);
const char* pact_last_error(void);
/* The same message through a context handle (SURVEY 8(b)'s
 * pact_last_error(pact_ctx*)): the text of the calling thread's last failed
 * call; messages are thread-local, so contexts used from different threads
 * never see each other's errors.  `ctx` may be NULL. */
const char* pact_ctx_last_error(const pact_ctx* ctx);

/* Creates a context on `device` with its own non-blocking stream. */
int pact_ctx_create(int device, pact_ctx** out);
int pact_ctx_destroy(pact_ctx* ctx);
/* Returns the cudaStream_t the context launches on (as void*). */
void* pact_ctx_stream(pact_ctx* ctx);
/* Makes the context launch on a caller-owned stream.  NULL is the legacy
 * default stream (e.g. torch's default stream); pact_ctx_use_own_stream
 * switches back to the context's private non-blocking stream. */
int pact_ctx_set_stream(pact_ctx* ctx, void* stream);
int pact_ctx_use_own_stream(pact_ctx* ctx);
int pact_ctx_synchronize(pact_ctx* ctx);
/* Number of kernels this library launched on the context so far. */
int64_t pact_ctx_launch_count(pact_ctx* ctx);

int pact_device_alloc(pact_ctx* ctx, size_t bytes, void** out);
int pact_device_free(pact_ctx* ctx, void* ptr);
int pact_host_alloc_pinned(size_t bytes, void** out);
int pact_host_free_pinned(void* ptr);
int pact_upload(pact_ctx* ctx, void* dst_device, const void* src_host, size_t bytes);
int pact_download(pact_ctx* ctx, void* dst_host, const void* src_device, size_t bytes);
int pact_memset(pact_ctx* ctx, void* dst_device, int value, size_t bytes);

/* ---- part 1: delay-and-sum stack ---- */

/* make_delays, beamform.hpp:113-120: `count` evenly spaced delays in [lo, hi]. */
int pact_make_delays(double lo, double hi, int32_t count, double* out);

/* das_stack, beamform.hpp:77-110 (and das, beamform.hpp:56-75, as K = 1).
 *   signals : device fp32 [n_transducers][n_samples] (SignalSet::data layout)
 *   delays  : HOST double[K], strictly increasing (mm)
 *   out     : device fp32 [K][grid.height][grid.width]
 * y_j(r) = sum_n S_n((|r - r_n| - d_j)/v0) with SignalSet::sample semantics
 * (linear interpolation, zero outside [0, n_samples-1], core.hpp:296-304). */
int pact_das_stack(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                   const float* signals, const pact_grid* grid, double v0,
                   const double* delays, int32_t n_delays, float* out);

/* BodyModel, beamform.hpp:44-54: the body disc of the two-speed DAS. */
typedef struct pact_body {
  double center_x; /* mm */
  double center_y; /* mm */
  double radius;   /* mm */
  double body_sos; /* m/s, validated to [1300, 1800] */
} pact_body;

/* dual_sos_das, beamform.hpp:124-150: DAS (K = 1, no delay) whose time of
 * flight runs at body_sos along the analytic chord through the body disc
 * (segment_circle_intersection, core.hpp:184-204) and at v0 elsewhere.
 *   signals : device fp32 [n_transducers][n_samples]
 *   out     : device fp32 [grid.height][grid.width]
 * Same validation order and messages as the reference. */
int pact_dual_sos_das(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                      const float* signals, const pact_grid* grid, double v0,
                      const pact_body* body, float* out);

/* ---- evaluation metrics (evaluate.hpp:39-114), SURVEY §8(f)-4 ----
 * test, truth: device fp64 [height][width] rasters of the same geometry (the
 * shape check of the reference is the caller's: RasterGrid carries it).
 * Synchronous; the value is written to *out (host).  fp64 sums, fixed order. */
/* psnr, evaluate.hpp:39-51: +inf for identical images. */
int pact_psnr(pact_ctx* ctx, const double* test, const double* truth, int32_t width,
              int32_t height, double data_range, double* out);
/* ssim, evaluate.hpp:53-96: 11x11 Gaussian window (sigma 1.5), K1 0.01, K2 0.03,
 * mean over the pixels whose window fits. */
int pact_ssim(pact_ctx* ctx, const double* test, const double* truth, int32_t width,
              int32_t height, double data_range, double* out);
/* sos_rmse_masked, evaluate.hpp:99-114: RMSE over pixels whose centres are in the mask. */
int pact_sos_rmse_masked(pact_ctx* ctx, const double* test, const double* truth,
                         const pact_grid* grid, const pact_mask* mask, double* out);

/* simulate_signals, phantom.hpp:282-362 (+ time_of_flight, aberration.hpp:79-100):
 * the input-side step before DAS.  pressure, sos: HOST fp64 [H][W] rasters of
 * the Phantom on `grid`; mask = Phantom::mask (TOF integration disc);
 * meta->t0 / n_samples fix the window (SimulateOptions t0 / n_samples);
 * out: device fp32 [n_transducers][n_samples]. */
int pact_simulate_signals(pact_ctx* ctx, const pact_grid* grid, const double* pressure,
                          const double* sos, const pact_mask* mask, double background_sos,
                          const pact_ring* ring, double pulse_sigma,
                          const pact_signal_meta* meta, double ray_step, float* out);
/* simulate_signals with SimulateOptions::spreading (amplitude / sqrt(distance),
 * phantom.hpp:351): spreading != 0 enables it; pact_simulate_signals is the
 * spreading = 0 case. */
int pact_simulate_signals_ex(pact_ctx* ctx, const pact_grid* grid, const double* pressure,
                             const double* sos, const pact_mask* mask, double background_sos,
                             const pact_ring* ring, double pulse_sigma,
                             const pact_signal_meta* meta, double ray_step, int32_t spreading,
                             float* out);
/* The acquisition window of simulate_signals (phantom.hpp:284-334), host only:
 * the same validation and messages, t0 = NaN / n_samples = 0 select the
 * automatic window (floor(tau_min/dt) dt, ceil((tau_max - t0)/dt) + 1); fails
 * with the reference's "time window too short" when an explicit window misses
 * the arrivals.  out: {n_samples, dt, t0, background_sos}. */
int pact_simulate_window(const pact_grid* grid, const double* pressure, const double* sos,
                         double background_sos, const pact_ring* ring, double pulse_sigma,
                         double dt, double t0, int32_t n_samples, pact_signal_meta* out);

/* ---- patch layout (host) ---- */

/* make_patch_layout, core.hpp:252-281 (same validation and messages). */
int pact_make_patch_layout(const pact_grid* grid, double patch_mm, double overlap,
                           pact_layout* out);
int32_t pact_layout_n_patches(const pact_layout* layout);
/* PatchLayout::offsets / centers (row-major patch order): offsets[2i] = ox,
 * offsets[2i+1] = oy (pixels); centers[2i], centers[2i+1] world mm.  Either may be NULL. */
int pact_layout_patches(const pact_layout* layout, int32_t* offsets, double* centers);

/* ---- part 2: SOS field, wavefronts, transfer stacks ---- */

/* SirenParams scalars, nfield.hpp:37-71; theta layout is the reference's
 * (per layer: W row-major [rows][cols], then b). */
typedef struct pact_siren {
  int32_t in_dim; /* must be 2 */
  int32_t hidden;
  int32_t n_hidden_layers;
  double omega0;
  double out_scale; /* m/s per unit output */
  double v0;        /* background SOS, m/s */
} pact_siren;

/* siren_param_count, nfield.hpp:73-78. */
int64_t pact_siren_param_count(const pact_siren* siren);
/* init_siren, nfield.hpp:83-107 (host; mt19937_64 + uniform_real_distribution,
 * bit-identical to the reference).  theta: HOST double[param_count]. */
int pact_init_siren(uint64_t seed, const pact_siren* siren, double* theta);
/* Masked pixels of render_sos (nfield.hpp:152-160): row-major flat indices and
 * normalised coordinates (HOST arrays; either may be NULL). */
int32_t pact_masked_count(const pact_grid* grid, const pact_mask* mask);
int pact_masked_pixels(const pact_grid* grid, const pact_mask* mask, int32_t* idx,
                       float* coords);

/* render_sos, nfield.hpp:145-162.  theta: device fp32.  raster: device fp32
 * [H][W], v0 outside the mask.  sos_dev (optional): device fp32 [H][W] holding
 * v - v0 (the full-precision form the ray kernels consume). */
int pact_render_sos(pact_ctx* ctx, const pact_siren* siren, const float* theta,
                    const pact_grid* grid, const pact_mask* mask, float* raster, float* sos_dev);

/* backprop_sos, nfield.hpp:166-233: gradient of sum_m g_m v(m).
 *   grad_masked : device fp32 [n_masked] (render_sos masked order)
 *   grad_theta  : device fp64 [param_count] (overwritten) */
int pact_siren_backward(pact_ctx* ctx, const pact_siren* siren, const float* theta,
                        const pact_grid* grid, const pact_mask* mask, const float* grad_masked,
                        double* grad_theta);

/* wavefront_profile, aberration.hpp:134-186, for n_centers patch centres.
 *   sos_dev : device fp32 [H][W] = v - v0 on `grid`
 *   centers : HOST double[2 n_centers] (mm)
 *   w       : device fp32 [n_centers][n_angles] (mm) */
int pact_wavefront(pact_ctx* ctx, const pact_ring* ring, const pact_grid* grid,
                   const float* sos_dev, double v0, const pact_mask* mask, int32_t n_centers,
                   const double* centers, int32_t n_angles, double step, float* w);

/* transfer_stack, aberration.hpp:236-265, batched over patches.
 *   w      : device fp32 [n_patches][n_angles]
 *   delays : HOST double[K]
 *   H      : device complex64 [n_patches][K][P][P] (interleaved re, im) */
int pact_transfer_stack(pact_ctx* ctx, int32_t n_patches, const float* w, int32_t n_angles,
                        const double* delays, int32_t K, int32_t P, double pitch, float* H);

/* ---- part 3: spectra, deconvolution, loss and gradients ---- */

/* extract_patch_spectra, deconv.hpp:64-74.
 *   stack : device fp32 [K][H][W];  Y : device complex64 [n_patches][K][P][P] */
int pact_patch_spectra(pact_ctx* ctx, const pact_layout* layout, const float* stack, int32_t K,
                       float* Y);

/* DeconvolveOptions, deconv.hpp:166-172 (workers has no meaning here). */
typedef struct pact_deconv_options {
  double eps;
  int32_t n_angles;
  double ray_step;
  double merge_fwhm;
} pact_deconv_options;

/* deconvolve_image, deconv.hpp:176-198.  stack device fp32 [K][H][W];
 * sos_dev device fp32 [H][W] = v - v0 with v0 = the stack's v0; image device fp32 [H][W]. */
int pact_deconvolve_image(pact_ctx* ctx, const float* stack, int32_t K, const double* delays,
                          double v0, const float* sos_dev, const pact_ring* ring,
                          const pact_mask* mask, const pact_layout* layout,
                          const pact_deconv_options* options, float* image);

/* detail::fused_patch_loss_grad, optimize.hpp:234-325, batched over patches:
 *   Y      : device complex64 [n_patches][K][P][P] (the training-path fp32 cache)
 *   w      : device fp32 [n_patches][n_angles]
 *   loss   : device fp64 [n_patches]   (sum_j sum_k |k| scale |Y_j - H_j X|^2)
 *   dw     : device fp32 [n_patches][n_angles]  (dL/dw) */
int pact_loss_grad(pact_ctx* ctx, int32_t n_patches, const float* Y, const float* w,
                   int32_t n_angles, const double* delays, int32_t K, int32_t P, double pitch,
                   double eps, double scale, int32_t implicit, double* loss_per_patch, float* dw);

/* MergeWindow::make, deconv.hpp:124-138 (host): Gaussian window, peak 1 at
 * the patch centre.  weights : HOST double[P * P]. */
int pact_merge_window(double fwhm_mm, int32_t P, double pitch, double* weights);

/* merge_patches, deconv.hpp:142-164: weight-normalised overlap-add of the
 * layout's patch images with the window `window` (HOST double[P * P], e.g.
 * from pact_merge_window; NULL = MergeWindow::make(fwhm_mm)).
 *   patches : device fp32 [n_patches][P][P] (layout order);  image : device fp32 [H][W] */
int pact_merge_patches(pact_ctx* ctx, const pact_layout* layout, const float* patches,
                       const double* window, double fwhm_mm, float* image);

/* ---- part 3, the composed (non-fused) path: fp64, complex128 operands ----
 * The reference's differentiable-by-parts API (used by its gradient tests and
 * by callers that want dL/dH).  Spectra are device complex128
 * [n_patches][K][P][P] (interleaved re, im), the reference's complex<double>.
 */

/* multichannel_deconvolve, deconv.hpp:78-96, batched:
 *   X[p][b] = sum_j conj(H_j) Y_j / (sum_j |H_j|^2 + eps K), 0 where the
 *   denominator is 0.  X : device complex128 [n_patches][P][P]. */
int pact_multichannel_deconvolve(pact_ctx* ctx, int32_t n_patches, int32_t K, int32_t P,
                                 const double* Y, const double* H, double eps, double* X);

/* deconv_jacobian_H, deconv.hpp:100-115: dX(bin)/d(Re H_j(bin)) and
 * dX(bin)/d(Im H_j(bin)) for each query (patch, j, bin) of the device int32
 * array `queries` [n_queries][3]; out : device complex128 [n_queries][2]. */
int pact_deconv_jacobian_H(pact_ctx* ctx, int32_t K, int32_t P, const double* Y, const double* H,
                           double eps, int32_t n_queries, const int32_t* queries, double* out);

/* patch_data_loss, optimize.hpp:164-211, batched with the caller's `scale`:
 *   loss_per_patch : device fp64 [n_patches]
 *   grad_h         : device complex128 [n_patches][K][P][P] (dL/dRe H + i dL/dIm H,
 *                    explicit term plus, with `implicit`, the term through X-hat) */
int pact_patch_data_loss(pact_ctx* ctx, int32_t n_patches, int32_t K, int32_t P, double pitch,
                         const double* Y, const double* H, double eps, double scale,
                         int32_t implicit, double* loss_per_patch, double* grad_h);

/* data_loss, optimize.hpp:336-353: patch_data_loss of every patch with
 * scale = 1 / (n_patches K P^2), summed in patch order.  value : HOST fp64
 * (synchronous); loss_per_patch : device fp64 [n_patches] or NULL. */
int pact_data_loss(pact_ctx* ctx, int32_t n_patches, int32_t K, int32_t P, double pitch,
                   const double* Y, const double* H, double eps, int32_t implicit, double* value,
                   double* loss_per_patch, double* grad_h);

/* transfer_grad_to_wavefront, aberration.hpp:270-313, batched:
 *   w      : device fp64 [n_patches][n_angles] (the profiles H was made from)
 *   delays : HOST double[K]
 *   grad_h : device complex128 [n_patches][K][P][P] (Nyquist-symmetrised inside,
 *            like the reference; the input is not modified)
 *   dw     : device fp64 [n_patches][n_angles] (overwritten) */
int pact_transfer_grad_to_wavefront(pact_ctx* ctx, int32_t n_patches, const double* w,
                                    int32_t n_angles, const double* delays, int32_t K, int32_t P,
                                    double pitch, const double* grad_h, double* dw);

/* wavefront_profile(..., with_jacobian = true), aberration.hpp:134-186: the
 * profiles (fp64) and their sparse Jacobian rows w.r.t. the in-mask SOS pixels,
 * in CSR form with one row per (patch, angle):
 *   row_start : device int64 [n_centers * n_angles + 1]
 *   pixel     : device int32 [n_entries]  (flat row-major grid index)
 *   dw_dv     : device fp32  [n_entries]  (mm per m/s; the reference stores float)
 *   w         : device fp64 [n_centers][n_angles] or NULL
 * Call once with pixel = dw_dv = NULL to size: fills row_start and the HOST
 * *n_entries (synchronous); call again with buffers of >= *n_entries entries
 * (`capacity`) to fill them.  Rows list entries by step, then stencil corner
 * (the reference's order). */
int pact_wavefront_jacobian(pact_ctx* ctx, const pact_ring* ring, const pact_grid* grid,
                            const float* sos_dev, double v0, const pact_mask* mask,
                            int32_t n_centers, const double* centers, int32_t n_angles,
                            double step, double* w, int64_t* row_start, int32_t* pixel,
                            float* dw_dv, int64_t capacity, int64_t* n_entries);

/* accumulate_wavefront_grad, aberration.hpp:316-326: grad_v (device fp64
 * [H][W]) += J^T dw over the CSR rows of pact_wavefront_jacobian;
 * dw : device fp64 [n_rows]. */
int pact_accumulate_wavefront_grad(pact_ctx* ctx, int64_t n_rows, const int64_t* row_start,
                                   const int32_t* pixel, const float* dw_dv, const double* dw,
                                   double* grad_v);

/* psf_from_transfer, aberration.hpp:407-445, batched (fp64): the real,
 * centred spatial PSF of each conjugate-symmetric P x P transfer spectrum
 * (zero lag at pixel (P/2, P/2)), with the reference's symmetry check
 * (ValidationError) and imaginary-residue check (NumericalError), applied to
 * the spectra in order; the message carries the reference's text.
 *   spectra : device complex128 [n][P][P];  psf : device fp64 [n][P][P] */
int pact_psf_from_transfer(pact_ctx* ctx, int32_t n_spectra, int32_t P, const double* spectra,
                           double* psf);

/* wavefront_grad_trace, aberration.hpp:333-361, batched: grad_v (device fp64
 * [H][W]) += sum over rays of dL/dw * dl * v0 / v^2 * bilinear weight. */
int pact_ray_backward(pact_ctx* ctx, const pact_ring* ring, const pact_grid* grid,
                      const float* sos_dev, double v0, const pact_mask* mask, int32_t n_centers,
                      const double* centers, int32_t n_angles, double step, const float* dw,
                      double* grad_v);

/* tv_loss, optimize.hpp:120-153 on the masked pixels of (grid, mask).
 *   raster      : device fp32 [H][W] (v, or v - v0: differences agree)
 *   value       : HOST double (synchronous)
 *   grad_masked : device fp32 [n_masked] */
int pact_tv_loss(pact_ctx* ctx, const pact_grid* grid, const pact_mask* mask, const float* raster,
                 double lambda, double* value, float* grad_masked);

/* adam_step, optimize.hpp:87-110, on device fp64 buffers; `t` is the step
 * count AFTER this update (AdamState::t).  Non-finite gradients ->
 * PACT_E_NUMERICAL and no update (synchronous check). */
int pact_adam_step(pact_ctx* ctx, int64_t n, double* theta, const double* grad, double* m,
                   double* v, int64_t t, double lr, double beta1, double beta2, double eps);

/* ---- the NF-APACT iteration engine: joint_reconstruct, optimize.hpp:367-494 ---- */

/* TrainConfig, optimize.hpp:48-78 (workers is accepted and ignored). */
typedef struct pact_train_config {
  int32_t epochs;
  int32_t steps_per_epoch;
  double learning_rate;
  double beta1;
  double beta2;
  double adam_eps;
  double lambda_tv;
  int32_t n_delays;
  const double* delays; /* HOST */
  double eps_deconv;
  int32_t n_angles;
  double ray_step;
  uint64_t seed;
  int32_t hidden;
  int32_t sine_layers;
  double omega0;
  double out_scale;
  double patch_mm;
  double overlap;
  double merge_fwhm;
  int32_t implicit_xhat_grad;
  int32_t workers;
  int32_t use_cuda_graph; /* capture one step as a CUDA graph (1 = yes) */
} pact_train_config;

typedef struct pact_trainer pact_trainer;

/* Fills `cfg` with the reference defaults (TrainConfig, optimize.hpp:48-69);
 * cfg->delays points to a static make_delays(-0.8, 0.8, 32) array. */
int pact_train_config_default(pact_train_config* cfg);

/* One-time part of joint_reconstruct (optimize.hpp:369-405): layout, DAS
 * stack, fp32 patch spectra, SIREN init, tables.  signals: device fp32 [N][T]. */
int pact_trainer_create(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                        const float* signals, const pact_grid* grid, const pact_mask* mask,
                        const pact_train_config* cfg, pact_trainer** out);
/* Enqueue n_steps full iterations (render -> wavefront -> fused loss ->
 * ray backward -> TV -> SIREN backward -> Adam); asynchronous. */
int pact_trainer_step(pact_trainer* tr, int32_t n_steps);

/* ---- one frame over several GPUs ----
 * Rank `rank` of `world` owns the patch rows [ny*rank/world, ny*(rank+1)/world)
 * (spectra, wavefronts, loss, ray adjoint) and the masked pixels
 * [n*rank/world, n*(rank+1)/world) of the row-major list (SIREN forward and
 * backward, TV); its DAS stack covers only those patches' grid rows.  Every
 * rank keeps the full dv and dL/dv rasters and a replica of theta and Adam.
 * The iteration then runs as phases with the caller's collectives in between
 * (buffers: pact_trainer_buffer):
 *   phase 0  render own pixels into a cleared dv     -> all-reduce dv (2, f32, SUM)
 *            (or all-gather, when the pixel shares are equal raster slabs)
 *   phase 1  wavefront, loss, ray adjoint, TV, report -> all-reduce dL/dv (5, f64, SUM),
 *            report (8, f64[3], SUM), flags (9, u32, MAX)
 *            (phase 1 = phase 6 (wavefront, loss, ray adjoint) then phase 7
 *            (TV, report): the dL/dv collective — a reduce-scatter to the
 *            pixel slabs — can run while phase 7 does)
 *   phase 2  SIREN backward                          -> all-reduce gradient (6, f64, SUM)
 *   phase 3  finiteness check + Adam (identical on every rank)
 * and the final image as
 *   phase 4  render                                  -> all-reduce dv (SUM)
 *   phase 5  deconvolve own patches into merge accumulators num (10), den (11)
 *            (f32 rasters)                            -> all-reduce (SUM); image = num/den
 * world == 1 is the whole frame (phases 0-3 in order == pact_trainer_step). */
typedef struct pact_partition {
  int32_t rank;
  int32_t world;
} pact_partition;
int pact_trainer_create_partitioned(pact_ctx* ctx, const pact_ring* ring,
                                    const pact_signal_meta* meta, const float* signals,
                                    const pact_grid* grid, const pact_mask* mask,
                                    const pact_train_config* cfg, const pact_partition* part,
                                    pact_trainer** out);
int pact_trainer_phase(pact_trainer* tr, int32_t phase);
/* info[9] = {patch lo, patch hi, pixel lo, pixel hi, total patches, rank, world,
 *            first stack row, stack rows}: the DAS stack holds only the grid
 * rows [row0, row0 + rows) the local patches cover (the row-tile split). */
int pact_trainer_local(pact_trainer* tr, int32_t* info);
/* Last step's LossReport terms {data, tv, total} (host) and the NumericalError
 * check of joint_reconstruct; synchronises.  `epoch` is used in the message. */
int pact_trainer_report(pact_trainer* tr, int32_t epoch, double* report3);

/* ---- the multi-GPU frame over NCCL, without a host framework ----
 * (the context owns the NCCL communicator; §8(e): the phase
 * orchestration above.)  libnccl.so.2 is loaded at run time.
 * Rank 0 makes a unique id and hands it to every rank out of band; each rank
 * attaches it to the context that created its partitioned trainer. */
#define PACT_NCCL_ID_BYTES 128
int pact_nccl_unique_id(unsigned char* id /* [PACT_NCCL_ID_BYTES] */);
int pact_ctx_attach_nccl(pact_ctx* ctx, const unsigned char* id, int32_t rank, int32_t world);
/* n_steps iterations of a partitioned trainer (rank and world must match the
 * communicator of the trainer's context): the phases 0, 6, 7, 2, 3 with the
 * all-gather of dv (equal raster slabs; else all-reduce), the reduce-scatter
 * of dL/dv (else all-reduce) overlapping phase 7, the all-reduces of the
 * report, flags and gradient -- on the engine stream and a communication
 * stream ordered by events; asynchronous.  world == 1 is pact_trainer_step
 * by phases. */
int pact_trainer_step_nccl(pact_trainer* tr, int32_t n_steps);
/* The final image and SOS (optimize.hpp:478-486) of the whole frame on every
 * rank: phases 4 (+ dv exchange) and 5 (+ all-reduce of the merge
 * accumulators), image = num / den; device fp32 [H][W] each, on the caller's
 * context stream. */
int pact_trainer_finish_nccl(pact_trainer* tr, float* image, float* sos);
/* One reported epoch (steps_per_epoch steps): report4 = {data, tv, total, wall_s}. */
int pact_trainer_run_epoch(pact_trainer* tr, int32_t epoch, double* report4);
/* Final render + deconvolution (optimize.hpp:478-486): device fp32 [H][W]
 * image and SOS (either may be NULL). */
int pact_trainer_finish(pact_trainer* tr, float* image, float* sos);
/* Current parameters (HOST fp64) / overwrite them (resets nothing else). */
int pact_trainer_get_theta(pact_trainer* tr, double* theta);
int pact_trainer_set_theta(pact_trainer* tr, const double* theta);
/* Device pointers of the engine's state for inspection:
 * what: 0 stack fp32 [K][H][W], 1 spectra c64 [n][K][P][P], 2 sos_dev fp32 [H][W],
 * 3 wavefronts fp32 [n][A], 4 dw fp32 [n][A], 5 grad_v fp64 [H][W],
 * 6 grad_theta fp64 [P], 7 theta fp64 [P], 8 report fp64 [3] (data, tv, total),
 * 9 NumericalError flags u32, 10/11 merge accumulators fp32 [H][W] (world > 1),
 * 12 theta fp32 working copy [P].  Spectra, wavefronts and dw cover the local
 * patches of a partitioned trainer. */
void* pact_trainer_buffer(pact_trainer* tr, int32_t what);
int pact_trainer_destroy(pact_trainer* tr);
/* Kernels the engine launched so far (graph replays counted per kernel). */
int64_t pact_trainer_launch_count(pact_trainer* tr);
/* The engine's private cudaStream_t (as void*), for event timing. */
void* pact_trainer_stream(pact_trainer* tr);
/* One iteration run eagerly with CUDA events between its stages; stage_ms[7]:
 * SIREN forward, wavefront, fused loss, ray backward, TV+report, SIREN
 * backward, Adam (device ms).  Synchronises. */
int pact_trainer_profile_step(pact_trainer* tr, float* stage_ms);

/* joint_reconstruct, optimize.hpp:367-494, end to end.  reports: HOST
 * double[epochs][4] {data, tv, total, wall_s}; image, sos: device fp32
 * [H][W] (may be NULL); theta: HOST fp64 (may be NULL). */
int pact_joint_reconstruct(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                           const float* signals, const pact_grid* grid, const pact_mask* mask,
                           const pact_train_config* cfg, double* reports, float* image,
                           float* sos, double* theta);

/* joint_reconstruct of n_frames independent frames of one geometry (cfg4),
 * run concurrently on one GPU (one engine stream per frame; a frame's first
 * epoch is enqueued when it is created and each next epoch as soon as its
 * report is read, so no frame waits for another).  Results are identical to
 * n_frames separate pact_joint_reconstruct calls.
 *   signals[f]: fp32 [N][T], device or HOST memory;  cfgs[f]: per-frame TrainConfig (equal epochs)
 *   reports: HOST double[n_frames][epochs][4] (wall_s = the batch's epoch time)
 *   images[f], sos[f]: fp32 [H][W], device or HOST memory (arrays may be NULL)
 * Host signals / outputs (here, in pact_joint_reconstruct and in
 * pact_trainer_create / pact_trainer_finish) are staged by the engine on the
 * frame's own stream: pinned host memory keeps the copies asynchronous and
 * lets them overlap the other frames' compute; host outputs are complete
 * once the context stream is synchronised.
 *   thetas: HOST fp64 [n_frames][P] (may be NULL) */
int pact_joint_reconstruct_batch(pact_ctx* ctx, int32_t n_frames, const pact_ring* ring,
                                 const pact_signal_meta* meta, const float* const* signals,
                                 const pact_grid* grid, const pact_mask* mask,
                                 const pact_train_config* cfgs, double* reports,
                                 float* const* images, float* const* sos, double* thetas);

#ifdef __cplusplus
}
#endif

#endif /* PACT_CUDA_H */
