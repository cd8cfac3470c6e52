// SIREN coordinate network on the device (nfield.hpp).  Activations are kept
// per masked pixel, row-major [n_masked][hidden] fp32.
#pragma once

#include <vector>

#include "common.cuh"

namespace pactgpu {

// The argument of the MUFU sine / cosine.  __sinf(x) is MUFU.SIN(x / 2pi):
// the unit takes the fractional part of the turns exactly, so the error of an
// unreduced argument is the rounding of that one product, |x| 2^-24 -- the
// size of the rounding of x = w0 a itself.  Measured at cfg3 (one iteration vs
// the reference, tests/test_bench_configs_gpu.py): w 1.0e-6 -> 1.8e-6, SOS
// 1.3e-6 -> 1.9e-6, grad theta 6.9e-6 unchanged, for four instructions fewer
// per activation (forward 0.139 -> 0.120 ms, backward 0.299 -> 0.287 ms).
// PACT_SINE_REDUCE=1 (compile time) restores the two-constant Cody-Waite
// reduction into [-pi, pi] (k = round(x / 2pi) from the 1.5 * 2^23 shifter on
// the FMA pipe; FRND would issue on the MUFU's own quarter-rate unit).  Every
// SIREN kernel (forward and backward) uses this one definition, so
// a_l -> sin(w0 a_l) is the same function everywhere.
#ifndef PACT_SINE_REDUCE
#define PACT_SINE_REDUCE 0
#endif
#ifdef __CUDACC__
__device__ __forceinline__ float sine_reduce(float x) {
  if (!PACT_SINE_REDUCE) return x;
  const float k = __fadd_rn(__fmaf_rn(x, 0.159154943091895336f, 12582912.f), -12582912.f);
  return fmaf(-k, -1.74845553146951720e-07f, fmaf(-k, 6.28318548202514648f, x));
}
#endif

struct SirenShape {
  int in_dim = 2;
  int hidden = 64;
  int layers = 2;  // n_hidden_layers (sine layers)
  double omega0 = 30.0;
  double out_scale = 100.0;
  double v0 = 1500.0;

  // SirenParams::layer_shape / layer_offset / param_count, nfield.hpp:45-63
  int rows(int l) const { return l == layers ? 1 : hidden; }
  int cols(int l) const { return l == 0 ? in_dim : hidden; }
  size_t offset(int l) const {
    size_t o = 0;
    for (int k = 0; k < l; ++k) o += static_cast<size_t>(rows(k)) * cols(k) + rows(k);
    return o;
  }
  size_t count() const { return offset(layers + 1); }
};

// Masked pixels of (grid, mask) in row-major order with their normalised
// coordinates (render_sos, nfield.hpp:152-160), computed in fp64 on the host.
struct MaskedPixels {
  int n = 0;
  std::vector<int> idx;
  std::vector<float> coords;  // [n][2]
};
MaskedPixels masked_pixels(const pact_grid& g, const pact_mask& m);

// Device workspace for one SIREN evaluation over n masked pixels.
struct SirenWork {
  int n = 0, hidden = 0, layers = 0;
  int* idx = nullptr;        // [n]
  float2* coords = nullptr;  // [n]
  float* acts = nullptr;     // [layers][n][hidden] pre-activations a_l
  float* dA = nullptr;       // [n][hidden]  backward ping
  float* dB = nullptr;       // [n][hidden]  backward pong
  float* partial = nullptr;  // split-M weight-gradient partials
  size_t partial_floats = 0;
  float* wplanes = nullptr;  // tcgen05 weight planes of the fused forward (siren_chain.cu)
  size_t wplanes_floats = 0;
  float* wide_planes = nullptr;  // width-256 layers: W and W^T planes per hidden layer (siren_wide.cu)
  size_t wide_planes_floats = 0;
  cudaStream_t stream = nullptr;  // pool stream of the buffers
};

Status siren_work_alloc(SirenWork& w, const MaskedPixels& mp, const SirenShape& s,
                        cudaStream_t stream);
void siren_work_free(SirenWork& w);

// Forward over the masked pixels: a_l for every sine layer, and
// dv[idx[m]] = out_scale * MLP(c_m) written into the deviation raster.
Status siren_forward(pact_ctx* ctx, const SirenShape& s, const float* theta, SirenWork& w,
                     float* dv_raster);

// Reverse mode of sum_m g_m v(m), g_m = gv_raster[idx[m]] (fp64 raster, may
// be null) + g_masked[m] (may be null); grad (fp64, reference layout) is
// overwritten.  Requires siren_forward on the same theta first.
Status siren_backward(pact_ctx* ctx, const SirenShape& s, const float* theta, SirenWork& w,
                      const double* gv_raster, const float* g_masked, double* grad);

// tcgen05 3xTF32 hidden layers (siren_tc.cu), hidden == 128.  The
// SIMT tiles remain for other widths and when PACT_SIREN_SIMT=1.
bool siren_tc_supported(int hidden);
bool siren_use_tc(int hidden);
bool siren_fused_bwd(const SirenShape& s);
// Output layer fused into the last forward layer's epilogue (w == null: not fused):
// dv[idx[m]] = scale * (b[0] + sum_k w[k] sin(w0 a_{L-1}[m][k])).
struct SirenHead {
  const float* w = nullptr;
  const float* b = nullptr;
  const int* idx = nullptr;
  float* dv = nullptr;
  float scale = 0.f;
};
// The whole forward (first layer, tcgen05 hidden layers, head) in one kernel
// for hidden width 128 (siren_chain.cu).
// store_a0 = false: a_0 is not written (the fused backward recomputes it).
Status tc_forward_chain(pact_ctx* ctx, const SirenShape& s, const float* theta, SirenWork& w,
                        float* dv, bool store_a0);
Status tc_forward_layer(pact_ctx* ctx, int H, const float* Ain, const float* W, const float* b,
                        int n, float w0, float* Aout, const SirenHead& head);
Status tc_dgrad_layer(pact_ctx* ctx, int H, const float* dAl, const float* W, const float* Aprev,
                      int n, float w0, float* dAprev);
int tc_wgrad_rows(pact_ctx* ctx, int n);  // pixels per weight-gradient partial
Status tc_wgrad_layer(pact_ctx* ctx, int H, const float* dAl, const float* Aprev, int n, int rows,
                      float w0, float* partial, int n_chunks);

// Fused backward of one tcgen05 layer (siren_bwd.cu, hidden 128): data and
// weight gradients from one pass; TOP forms dA_l from a_l and g (output
// layer), BOTTOM accumulates the layer-0 partials instead of storing dA_0.
struct TcBwdLayer {
  const float* X = nullptr;      // dA_l [n][128]; TOP: a_l
  const float* Aprev = nullptr;  // a_{l-1} [n][128]
  const float* W = nullptr;      // W_l [128][128]
  const double* gv = nullptr;    // TOP
  const float* gmask = nullptr;  // TOP
  const int* idx = nullptr;      // TOP
  const float* wL = nullptr;     // TOP
  float* gpx = nullptr;          // TOP: scratch for g s per masked pixel [n]
  const float2* coords = nullptr;  // BOTTOM
  const float* W0 = nullptr;       // BOTTOM: layer 0 (a_0 is recomputed, not read)
  const float* b0 = nullptr;
  float out_scale = 0.f, w0 = 0.f;
  int n = 0;
  float* Y = nullptr;         // dA_{l-1} (not BOTTOM)
  float* part_w = nullptr;    // [grid][128 * 128 + 128]
  float* part_top = nullptr;  // TOP: [grid][129]
  float* part_0 = nullptr;    // BOTTOM: [grid][384]
};
// Hidden width 256 (cfg5) on tcgen05 (siren_wide.cu): per-layer streamed
// GEMMs with both operands in shared memory.
bool siren_wide_supported(int hidden);
bool siren_use_wide(int hidden);
size_t tc_wide_plane_floats();  // floats of one matrix's hi/lo planes
Status tc_wide_planes(pact_ctx* ctx, const float* W, bool transposed, float* planes);
Status tc_wide_forward_layer(pact_ctx* ctx, const float* Ain, const float* planes, const float* b,
                             int n, float w0, float* Aout);
Status tc_wide_dgrad_layer(pact_ctx* ctx, const float* dAl, const float* planes_t,
                           const float* Aprev, int n, float w0, float* dAprev);
int tc_wide_wgrad_rows(pact_ctx* ctx, int n);
Status tc_wide_wgrad_layer(pact_ctx* ctx, const float* dAl, const float* Aprev, int n, int rows,
                           float w0, float* partial, int n_chunks);
int tc_bwd_grid(pact_ctx* ctx, int n);  // CTAs (= partial rows) of tc_bwd_layer
Status tc_bwd_layer(pact_ctx* ctx, bool top, bool bottom, const TcBwdLayer& layer);
// The same layer on split-fp16 kind::f16 MMAs (siren_bwd16.cu; the default,
// PACT_SIREN_BWD_F16=0 selects tc_bwd_layer).  mx_in: bits of max|dA_l| (TOP:
// written here, max|g s|); mx_out: bits of max|dA_{l-1}| (atomicMax).  Both
// zeroed by the caller before the top layer.
bool tc_bwd_f16();
Status tc_bwd16_layer(pact_ctx* ctx, bool top, bool bottom, const TcBwdLayer& layer, unsigned* mx_in,
                      unsigned* mx_out);

}  // namespace pactgpu
