/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 hot path.
 *
 * A plain-C restatement of the reference algorithms (fp64 throughout, like
 * the reference), each function citing the reference file:line it follows.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only as the checker.  It is pinned against the reference
 * itself: tests/golden/ holds fixtures produced by oracle/_ref (the
 * reference headers compiled in place), see tests/golden/make_golden.py and
 * tests/test_oracle_golden.py.
 *
 * Signatures mirror oracle/ref_shim.cpp (prefix orc_ instead of ref_).
 * Complex arrays are interleaved (re, im) doubles; return 0 on success,
 * 2 on a validation failure (the reference's ValidationError), 3 numerical.
 */
#ifndef PACT_ORACLE_H
#define PACT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct OrcTrainCfg { /* = RefTrainCfg (TrainConfig, optimize.hpp:48-69) */
  int epochs, steps_per_epoch;
  double lr, beta1, beta2, adam_eps, lambda_tv;
  int n_delays;
  const double* delays;
  double eps_deconv;
  int n_angles;
  double ray_step;
  uint64_t seed;
  int hidden, sine_layers;
  double omega0, out_scale, patch_mm, overlap, merge_fwhm;
  int implicit_xhat_grad, workers;
} OrcTrainCfg;

int orc_das_stack(int n_tx, double radius, double offset, int T, double dt, double t0,
                  const double* sig, int W, int H, double pitch, double ox, double oy,
                  double v0, int K, const double* delays, int workers, double* out);
int orc_dual_sos_das(int n_tx, double radius, double offset, int T, double dt, double t0,
                     const double* sig, int W, int H, double pitch, double ox, double oy,
                     double v0, double bcx, double bcy, double br, double bsos, double* out);
int orc_psnr(const double* test, const double* truth, int W, int H, double data_range,
             double* out);
int orc_ssim(const double* test, const double* truth, int W, int H, double data_range,
             double* out);
int orc_sos_rmse_masked(const double* test, const double* truth, int W, int H, double pitch,
                        double ox, double oy, double mcx, double mcy, double mr, double* out);
int orc_init_siren(uint64_t seed, int hidden, int layers, double omega0, double out_scale,
                   double v0, double* theta);
int orc_render_sos(int hidden, int layers, double omega0, double out_scale, double v0,
                   const double* theta, int W, int H, double pitch, double ox, double oy,
                   double mcx, double mcy, double mr, double* raster, int* n_masked);
int orc_backprop_sos(int hidden, int layers, double omega0, double out_scale, double v0,
                     const double* theta, int W, int H, double pitch, double ox, double oy,
                     double mcx, double mcy, double mr, const double* grad_v, double* grad);
int orc_wavefront_profile(int n_centers, const double* centers, int n_tx, double radius,
                          double offset, int W, int H, double pitch, double ox, double oy,
                          const double* sos, double v0, double mcx, double mcy, double mr,
                          int n_angles, double step, double* w);
int orc_transfer_stack(int n_angles, const double* w, int K, const double* delays, int P,
                       double pitch, double* Hc);
int orc_patch_layout(int W, int H, double pitch, double ox, double oy, double patch_mm,
                     double overlap, int* info, int* offsets, double* centers);
int orc_patch_spectra(int K, const double* delays, double v0, int W, int H, double pitch,
                      double ox, double oy, const double* stack, double patch_mm, double overlap,
                      int workers, double* Y);
int orc_deconvolve_image(int K, const double* delays, double v0, int W, int H, double pitch,
                         double ox, double oy, const double* stack, const double* sos, int n_tx,
                         double radius, double offset, double mcx, double mcy, double mr,
                         double patch_mm, double overlap, double eps, int n_angles,
                         double ray_step, double merge_fwhm, int workers, double* image);
int orc_fused_patch_loss_grad(int K, const float* Yf, const double* w, int P, double pitch,
                              int n_angles, const double* delays, double eps, double scale,
                              int implicit, double* loss, double* dw);
int orc_wavefront_grad_trace(double cx, double cy, int n_tx, double radius, double offset, int W,
                             int H, double pitch, double ox, double oy, const double* sos,
                             double v0, double mcx, double mcy, double mr, int n_angles,
                             double step, const double* dw, double* grad_v);
int orc_tv_loss(int W, int H, double pitch, double ox, double oy, const double* raster,
                double mcx, double mcy, double mr, double lambda, double* value,
                double* grad_masked);
int orc_adam_step(int n, double* params, const double* grads, double* m, double* v, long* t,
                  double lr, double b1, double b2, double eps);
int orc_nf_step(int n_tx, double radius, double offset, int T, double dt, double t0, double v0,
                const double* sig, int W, int H, double pitch, double ox, double oy, double mcx,
                double mcy, double mr, const OrcTrainCfg* c, const double* theta, int patch_lo,
                int patch_hi, double* data_term, double* tv_term, double* loss_patch,
                double* w_out, double* dw_out, double* sos_out, double* grad_v_masked,
                double* grad_theta, double* image, double* seconds);
int orc_joint_reconstruct(int n_tx, double radius, double offset, int T, double dt, double t0,
                          double v0, const double* sig, int W, int H, double pitch, double ox,
                          double oy, double mcx, double mcy, double mr, const OrcTrainCfg* c,
                          double* reports, double* image, double* sos, double* theta);
int orc_simulate_signals(int W, int H, double pitch, double ox, double oy, const double* pressure,
                         const double* sos, double mcx, double mcy, double mr,
                         double background_sos, int n_tx, double radius, double offset,
                         double pulse_sigma, double dt, double t0, int T, double ray_step,
                         int workers, double* out);

#ifdef __cplusplus
}
#endif

#endif
