/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 * See pact_oracle.h.  fp64 throughout; OpenMP only parallelises independent
 * outputs (results do not depend on the thread count).
 */
#include "pact_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* SignalSet::sample, core.hpp:296-304: linear interpolation, 0 outside the
 * window, the last sample exactly at s = T-1. */
static double sig_sample(const double* row, int T, double t0, double dt, double t) {
  double s = (t - t0) / dt;
  if (s < 0.0 || s > T - 1) return 0.0;
  int i = (int)s;
  if (i >= T - 1) return row[T - 1];
  double f = s - i;
  return (1.0 - f) * row[i] + f * row[i + 1];
}

/* RingGeometry::transducer_position, core.hpp:162-165 */
static void ring_pos(int n_tx, double radius, double offset, int n, double* x, double* y) {
  double a = 2.0 * M_PI * n / n_tx + offset;
  *x = radius * cos(a);
  *y = radius * sin(a);
}

/* das_stack, beamform.hpp:77-110 (validation beamform.hpp:79-85). */
int orc_das_stack(int n_tx, double radius, double offset, int T, double dt, double t0,
                  const double* sig, int W, int H, double pitch, double ox, double oy,
                  double v0, int K, const double* delays, int workers, double* out) {
  (void)workers;
  if (K < 1) return 2;
  for (int j = 1; j < K; ++j)
    if (!(delays[j] > delays[j - 1])) return 2;
  if (n_tx < 3 || !(radius > 0.0) || T < 2 || !(dt > 0.0)) return 2;
  if (W < 1 || H < 1 || !(pitch > 0.0) || !(v0 > 0.0)) return 2;
  double* px = (double*)malloc(sizeof(double) * 2 * n_tx);
  for (int n = 0; n < n_tx; ++n) ring_pos(n_tx, radius, offset, n, &px[2 * n], &px[2 * n + 1]);
  const size_t plane = (size_t)W * H;
#pragma omp parallel for schedule(dynamic)
  for (int iy = 0; iy < H; ++iy) {
    double* acc = (double*)malloc(sizeof(double) * K);
    for (int ix = 0; ix < W; ++ix) {
      for (int j = 0; j < K; ++j) acc[j] = 0.0;
      double rx = ox + ix * pitch, ry = oy + iy * pitch; /* GridSpec::world, core.hpp:71 */
      for (int n = 0; n < n_tx; ++n) {
        double dist = hypot(rx - px[2 * n], ry - px[2 * n + 1]);
        const double* row = sig + (size_t)n * T;
        for (int j = 0; j < K; ++j)
          acc[j] += sig_sample(row, T, t0, dt, 1e-3 * (dist - delays[j]) / v0);
      }
      for (int j = 0; j < K; ++j) out[j * plane + (size_t)iy * W + ix] = acc[j];
    }
    free(acc);
  }
  free(px);
  return 0;
}
