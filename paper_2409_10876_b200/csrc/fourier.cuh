// Frequency-grid tables shared by the transfer-stack, fused loss/gradient and
// Wiener-deconvolution kernels (one set per patch layout, like the
// reference's PatchBinTable, aberration.hpp:365-402, and delay phase table,
// optimize.hpp:223-232).
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"

namespace pactgpu {

struct FourierTab {
  int P = 0, P2 = 0, A = 0, K = 0;
  const float* kmag = nullptr;    // [P2] |k| rad/mm
  const int4* idx = nullptr;      // [P2] (a0, a1, b0, b1) interpolation indices
  const float2* frac = nullptr;   // [P2] (f1, f2)
  const int* mirror = nullptr;    // [P2] conjugate partner for Nyquist bins, -1 otherwise
  const float2* dp = nullptr;     // [K][P2] exp(-i |k| d_j)
  const float2* rho = nullptr;    // [P2] exp(-i |k| (d_1 - d_0)) for evenly spaced delays, else null:
                                  // dp_j = dp_0 rho^j is then walked in registers
  // dL/dw pullback (optimize.hpp:318-321) as a sort: the 2 P2 (bin, branch)
  // pairs ordered by their lower interpolation angle a0 (then bin, branch);
  // pair (b, r) sits at slot[b].x (r = 1, angle(k)) / slot[b].y (r = 2,
  // angle(k) + pi), and angle a owns slots [sstart[a], sstart[a + 1]).  The
  // loss kernels store ((1 - f) G, f G) of every pair at its slot, so dL/dw[a]
  // is the .x sum over a's slots plus the .y sum over a - 1's slots:
  // contiguous reads, fixed order.
  const int2* slot = nullptr;     // [P2]
  const int* sstart = nullptr;    // [A + 1]
  // most slots any group of kFinishAngles angles reads (their .x slots and the
  // .y slots of the angle before the group): the finish kernel's smem stage
  int fin_span = 0;
};
constexpr int kFinishAngles = 128;

// Host-built table (fp64 reference formulas, stored fp32) + its device copy.
struct FourierTable {
  int P = 0, A = 0, K = 0;
  double pitch = 0.0;
  std::vector<double> delays;
  void* dev = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;  // pool stream of `dev`
  std::shared_ptr<const void> host;  // host image being uploaded (kept alive)
  FourierTab tab;
};

// Builds (or reuses, if parameters match) the table on the device.
Status fourier_table(pact_ctx* ctx, FourierTable& t, int P, double pitch, int n_angles,
                     const double* delays, int K);
void fourier_table_free(FourierTable& t);

}  // namespace pactgpu
