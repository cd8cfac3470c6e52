/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 * See pact_oracle.h.  fp64 throughout, single-threaded (results do not
 * depend on a worker count).  Each function names the reference routine
 * (file:line under /root/reference/proj/include/pact/) whose arithmetic it
 * restates; branch structure and accumulation order follow the reference so
 * the golden fixtures agree to rounding.
 */
#include "pact_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

typedef double complex cx;

static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }
static double dclamp(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }
static cx polar(double rho, double th) { return CMPLX(rho * cos(th), rho * sin(th)); }
static double cnorm(cx z) { return creal(z) * creal(z) + cimag(z) * cimag(z); }
static cx cmul(cx a, cx b) {  /* plain product, as std::complex without NaN recovery */
  return CMPLX(creal(a) * creal(b) - cimag(a) * cimag(b), creal(a) * cimag(b) + cimag(a) * creal(b));
}

/* ------------------------------------------------------------------ geometry */

/* RingGeometry::transducer_position, core.hpp:162-165 */
static void ring_pos(int n_tx, double radius, double offset, int n, double* x, double* y) {
  double a = 2.0 * M_PI * n / n_tx + offset;
  *x = radius * cos(a);
  *y = radius * sin(a);
}

/* segment_circle_intersection, core.hpp:184-204: [t0, t1] along a->b, empty -> t0 > t1 */
static void seg_circle(double ax, double ay, double bx, double by, double cx_, double cy_,
                       double r, double* t0, double* t1) {
  double dx = bx - ax, dy = by - ay;
  double len = hypot(dx, dy);
  if (len == 0.0) {
    int inside = hypot(ax - cx_, ay - cy_) <= r;
    *t0 = inside ? 0.0 : 1.0;
    *t1 = 0.0;
    return;
  }
  double ux = dx * (1.0 / len), uy = dy * (1.0 / len);
  double mx = ax - cx_, my = ay - cy_;
  double bq = mx * ux + my * uy;
  double cq = (mx * mx + my * my) - r * r;
  double disc = bq * bq - cq;
  if (disc < 0.0) {
    *t0 = 1.0;
    *t1 = 0.0;
    return;
  }
  double s = sqrt(disc);
  double a = fmax(-bq - s, 0.0), b = fmin(-bq + s, len);
  if (a > b) {
    *t0 = 1.0;
    *t1 = 0.0;
    return;
  }
  *t0 = a;
  *t1 = b;
}

/* detail::bilinear_stencil, aberration.hpp:41-72 */
typedef struct {
  int idx[4];
  double w[4];
  double value;
} Stencil;

static Stencil stencil_at(const double* v, int W, int H, double pitch, double ox, double oy,
                          double px, double py) {
  Stencil s;
  double fx = dclamp((px - ox) / pitch, 0.0, (double)(W - 1));
  double fy = dclamp((py - oy) / pitch, 0.0, (double)(H - 1));
  int ix = imin((int)fx, imax(W - 2, 0)), iy = imin((int)fy, imax(H - 2, 0));
  double ax = fx - ix, ay = fy - iy;
  int ix1 = imin(ix + 1, W - 1), iy1 = imin(iy + 1, H - 1);
  s.idx[0] = iy * W + ix;
  s.idx[1] = iy * W + ix1;
  s.idx[2] = iy1 * W + ix;
  s.idx[3] = iy1 * W + ix1;
  s.w[0] = (1 - ax) * (1 - ay);
  s.w[1] = ax * (1 - ay);
  s.w[2] = (1 - ax) * ay;
  s.w[3] = ax * ay;
  s.value = s.w[0] * v[s.idx[0]] + s.w[1] * v[s.idx[1]] + s.w[2] * v[s.idx[2]] +
            s.w[3] * v[s.idx[3]];
  return s;
}

/* -------------------------------------------------------------------- part 1 */

/* SignalSet::sample, core.hpp:296-304 */
static double sig_sample(const double* row, int T, double t0, double dt, double t) {
  double s = (t - t0) / dt;
  if (s < 0.0 || s > T - 1) return 0.0;
  int i = (int)s;
  if (i >= T - 1) return row[T - 1];
  double f = s - i;
  return (1.0 - f) * row[i] + f * row[i + 1];
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
  double* acc = (double*)malloc(sizeof(double) * K);
  for (int iy = 0; iy < H; ++iy)
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
  free(px);
  return 0;
}

/* dual_sos_das, beamform.hpp:124-150 (validation beamform.hpp:126-131): the
 * time of flight runs at body_sos along the chord through the body disc. */
int orc_dual_sos_das(int n_tx, double radius, double offset, int T, double dt, double t0,
                     const double* sig, int W, int H, double pitch, double ox, double oy,
                     double v0, double bcx, double bcy, double br, double bsos, double* out) {
  if (n_tx < 3 || !(radius > 0.0) || T < 2 || !(dt > 0.0)) return 2;
  if (W < 1 || H < 1 || !(pitch > 0.0)) return 2;
  if (!(br > 0.0) || !(bsos >= 1300.0 && bsos <= 1800.0)) return 2;
  if (!(v0 > 0.0)) return 2;
  if (hypot(bcx, bcy) + br >= radius) return 2;
  double* px = (double*)malloc(sizeof(double) * 2 * n_tx);
  for (int n = 0; n < n_tx; ++n) ring_pos(n_tx, radius, offset, n, &px[2 * n], &px[2 * n + 1]);
  for (int iy = 0; iy < H; ++iy)
    for (int ix = 0; ix < W; ++ix) {
      double rx = ox + ix * pitch, ry = oy + iy * pitch, acc = 0.0;
      for (int n = 0; n < n_tx; ++n) {
        double dist = hypot(rx - px[2 * n], ry - px[2 * n + 1]);
        double s0, s1;
        seg_circle(rx, ry, px[2 * n], px[2 * n + 1], bcx, bcy, br, &s0, &s1);
        double inside = s1 - s0 > 0.0 ? s1 - s0 : 0.0;
        double t = 1e-3 * ((dist - inside) / v0 + inside / bsos);
        acc += sig_sample(sig + (size_t)n * T, T, t0, dt, t);
      }
      out[(size_t)iy * W + ix] = acc;
    }
  free(px);
  return 0;
}

/* ------------------------------------------------------------------ metrics */

/* psnr, evaluate.hpp:39-51 */
int orc_psnr(const double* test, const double* truth, int W, int H, double data_range,
             double* out) {
  if (!(data_range > 0.0)) return 2;
  double mse = 0.0;
  const size_t n = (size_t)W * H;
  for (size_t i = 0; i < n; ++i) {
    double d = test[i] - truth[i];
    mse += d * d;
  }
  mse /= (double)n;
  *out = mse == 0.0 ? INFINITY : 10.0 * log10(data_range * data_range / mse);
  return 0;
}

/* ssim, evaluate.hpp:53-96 */
int orc_ssim(const double* test, const double* truth, int W, int H, double data_range,
             double* out) {
  if (!(data_range > 0.0)) return 2;
  if (W < 11 || H < 11) return 2;
  double kern[11], ksum = 0.0;
  for (int i = 0; i < 11; ++i) {
    double d = i - 5.0;
    kern[i] = exp(-0.5 * d * d / (1.5 * 1.5));
    ksum += kern[i];
  }
  for (int i = 0; i < 11; ++i) kern[i] /= ksum;
  const double c1 = (0.01 * data_range) * (0.01 * data_range);
  const double c2 = (0.03 * data_range) * (0.03 * data_range);
  double acc = 0.0;
  long count = 0;
  for (int iy = 5; iy < H - 5; ++iy)
    for (int ix = 5; ix < W - 5; ++ix) {
      double mx = 0, my = 0, mxx = 0, myy = 0, mxy = 0;
      for (int dy = -5; dy <= 5; ++dy)
        for (int dx = -5; dx <= 5; ++dx) {
          double w = kern[dy + 5] * kern[dx + 5];
          double a = test[(size_t)(iy + dy) * W + ix + dx];
          double b = truth[(size_t)(iy + dy) * W + ix + dx];
          mx += w * a;
          my += w * b;
          mxx += w * a * a;
          myy += w * b * b;
          mxy += w * a * b;
        }
      double vx = mxx - mx * mx, vy = myy - my * my, cxy = mxy - mx * my;
      acc += ((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2));
      ++count;
    }
  *out = acc / count;
  return 0;
}

/* sos_rmse_masked, evaluate.hpp:99-114 */
int orc_sos_rmse_masked(const double* test, const double* truth, int W, int H, double pitch,
                        double ox, double oy, double mcx, double mcy, double mr, double* out) {
  double acc = 0.0;
  long n = 0;
  for (int iy = 0; iy < H; ++iy)
    for (int ix = 0; ix < W; ++ix) {
      double px = ox + ix * pitch, py = oy + iy * pitch;
      if (!(hypot(px - mcx, py - mcy) <= mr)) continue;
      double d = test[(size_t)iy * W + ix] - truth[(size_t)iy * W + ix];
      acc += d * d;
      ++n;
    }
  if (n == 0) return 2;
  *out = sqrt(acc / n);
  return 0;
}

/* --------------------------------------------------------------------- SIREN */

/* std::mt19937_64 (the engine init_siren seeds, nfield.hpp:94) */
typedef struct {
  uint64_t s[312];
  int i;
} Mt64;

static void mt_seed(Mt64* m, uint64_t seed) {
  m->s[0] = seed;
  for (int i = 1; i < 312; ++i)
    m->s[i] = 6364136223846793005ULL * (m->s[i - 1] ^ (m->s[i - 1] >> 62)) + (uint64_t)i;
  m->i = 312;
}

static uint64_t mt_next(Mt64* m) {
  const uint64_t up = 0xFFFFFFFF80000000ULL, lo = 0x7FFFFFFFULL, a = 0xB5026F5AA96619E9ULL;
  if (m->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      uint64_t y = (m->s[k] & up) | (m->s[(k + 1) % 312] & lo);
      m->s[k] = m->s[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    m->i = 0;
  }
  uint64_t x = m->s[m->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* uniform_real_distribution<double>(lo, hi) over mt19937_64 (libstdc++
 * generate_canonical<double, 53> with one 64-bit draw). */
static double mt_uniform(Mt64* m, double lo, double hi) {
  double u = (double)mt_next(m) / 18446744073709551616.0;
  if (u >= 1.0) u = nextafter(1.0, 0.0);
  return (hi - lo) * u + lo;
}

/* SirenParams::layer_shape / layer_offset, nfield.hpp:45-63 */
static int s_rows(int l, int H, int L) { return l == L ? 1 : H; }
static int s_cols(int l, int H) { return l == 0 ? 2 : H; }
static size_t s_off(int l, int H, int L) {
  size_t o = 0;
  for (int k = 0; k < l; ++k) o += (size_t)s_rows(k, H, L) * s_cols(k, H) + s_rows(k, H, L);
  return o;
}

/* init_siren, nfield.hpp:83-107 */
int orc_init_siren(uint64_t seed, int hidden, int layers, double omega0, double out_scale,
                   double v0, double* theta) {
  (void)out_scale;
  (void)v0;
  if (hidden < 1 || layers < 1 || !(omega0 > 0.0)) return 2;
  Mt64 m;
  mt_seed(&m, seed);
  size_t off = 0;
  for (int l = 0; l <= layers; ++l) {
    int rows = s_rows(l, hidden, layers), cols = s_cols(l, hidden);
    double bound = (l == 0) ? 1.0 / 2.0 : sqrt(6.0 / cols) / omega0;
    size_t n = (size_t)rows * cols + rows;
    for (size_t i = 0; i < n; ++i) theta[off + i] = mt_uniform(&m, -bound, bound);
    off += n;
  }
  return 0;
}

/* siren_eval_raw, nfield.hpp:110-128; a, z: [L][H] scratch (pre/post sine) */
static double siren_raw(const double* th, int H, int L, double w0, double cxv, double cyv,
                        double* a, double* z) {
  for (int l = 0; l < L; ++l) {
    const double* W = th + s_off(l, H, L);
    int cols = s_cols(l, H);
    const double* b = W + (size_t)H * cols;
    for (int r = 0; r < H; ++r) {
      double acc = b[r];
      if (l == 0) {
        acc += W[2 * r] * cxv;
        acc += W[2 * r + 1] * cyv;
      } else {
        const double* zin = z + (size_t)(l - 1) * H;
        for (int c = 0; c < H; ++c) acc += W[(size_t)r * H + c] * zin[c];
      }
      a[(size_t)l * H + r] = acc;
      z[(size_t)l * H + r] = sin(w0 * acc);
    }
  }
  const double* W = th + s_off(L, H, L);
  double out = W[H];
  const double* zl = z + (size_t)(L - 1) * H;
  for (int c = 0; c < H; ++c) out += W[c] * zl[c];
  return out;
}

/* render_sos, nfield.hpp:145-162 */
int orc_render_sos(int hidden, int layers, double omega0, double out_scale, double v0,
                   const double* theta, int W, int H, double pitch, double ox, double oy,
                   double mcx, double mcy, double mr, double* raster, int* n_masked) {
  if (W < 1 || H < 1 || !(pitch > 0.0) || !(mr > 0.0)) return 2;
  double* a = (double*)malloc(sizeof(double) * hidden * layers);
  double* z = (double*)malloc(sizeof(double) * hidden * layers);
  int n = 0;
  for (int iy = 0; iy < H; ++iy)
    for (int ix = 0; ix < W; ++ix) {
      double px = ox + ix * pitch, py = oy + iy * pitch;
      size_t k = (size_t)iy * W + ix;
      raster[k] = v0;
      if (!(hypot(px - mcx, py - mcy) <= mr)) continue; /* CircularMask::contains */
      ++n;
      raster[k] = v0 + out_scale * siren_raw(theta, hidden, layers, omega0, (px - mcx) / mr,
                                             (py - mcy) / mr, a, z);
    }
  if (n_masked) *n_masked = n;
  free(a);
  free(z);
  return 0;
}

/* backprop_sos, nfield.hpp:166-233 (grad_v per masked pixel, row-major order) */
int orc_backprop_sos(int hidden, int layers, double omega0, double out_scale, double v0,
                     const double* theta, int W, int H, double pitch, double ox, double oy,
                     double mcx, double mcy, double mr, const double* grad_v, double* grad) {
  (void)v0;
  const int Hd = hidden, L = layers;
  size_t np = s_off(L + 1, Hd, L);
  memset(grad, 0, sizeof(double) * np);
  double* a = (double*)malloc(sizeof(double) * Hd * L);
  double* z = (double*)malloc(sizeof(double) * Hd * L);
  double* delta = (double*)malloc(sizeof(double) * Hd);
  double* dprev = (double*)malloc(sizeof(double) * Hd);
  int m = 0;
  for (int iy = 0; iy < H; ++iy)
    for (int ix = 0; ix < W; ++ix) {
      double px = ox + ix * pitch, py = oy + iy * pitch;
      if (!(hypot(px - mcx, py - mcy) <= mr)) continue;
      double g = grad_v[m++] * out_scale;
      if (g == 0.0) continue;
      double in[2] = {(px - mcx) / mr, (py - mcy) / mr};
      siren_raw(theta, Hd, L, omega0, in[0], in[1], a, z);
      {
        const double* WL = theta + s_off(L, Hd, L);
        double* gW = grad + s_off(L, Hd, L);
        for (int c = 0; c < Hd; ++c) gW[c] += g * z[(size_t)(L - 1) * Hd + c];
        gW[Hd] += g;
        for (int c = 0; c < Hd; ++c) delta[c] = g * WL[c];
      }
      for (int l = L - 1; l >= 0; --l) {
        int cols = s_cols(l, Hd);
        const double* Wl = theta + s_off(l, Hd, L);
        double* gW = grad + s_off(l, Hd, L);
        double* gb = gW + (size_t)Hd * cols;
        if (l > 0)
          for (int c = 0; c < Hd; ++c) dprev[c] = 0.0;
        for (int r = 0; r < Hd; ++r) {
          double da = delta[r] * omega0 * cos(omega0 * a[(size_t)l * Hd + r]);
          gb[r] += da;
          for (int c = 0; c < cols; ++c) {
            double zin = l == 0 ? in[c] : z[(size_t)(l - 1) * Hd + c];
            gW[(size_t)r * cols + c] += da * zin;
            if (l > 0) dprev[c] += da * Wl[(size_t)r * cols + c];
          }
        }
        if (l > 0) {
          double* t = delta;
          delta = dprev;
          dprev = t;
        }
      }
    }
  free(a);
  free(z);
  free(delta);
  free(dprev);
  return 0;
}

/* ----------------------------------------------------------------------- FFT */

/* fft.hpp:43-82: radix-2 Cooley-Tukey for powers of two, direct DFT otherwise */
static void fft_radix2(cx* a, int n, int sign) {
  for (int i = 1, j = 0; i < n; ++i) {
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      cx t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
  }
  for (int len = 2; len <= n; len <<= 1) {
    double ang = sign * 2.0 * M_PI / len;
    cx wl = CMPLX(cos(ang), sin(ang));
    for (int i = 0; i < n; i += len) {
      cx w = 1.0;
      for (int k = 0; k < len / 2; ++k) {
        cx u = a[i + k];
        cx v = cmul(a[i + k + len / 2], w);
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
        w = cmul(w, wl);
      }
    }
  }
}

static void fft_direct(cx* a, int n, int sign) {
  cx* out = (cx*)malloc(sizeof(cx) * n);
  for (int k = 0; k < n; ++k) {
    cx acc = 0.0;
    for (int m = 0; m < n; ++m) {
      double ang = sign * 2.0 * M_PI * k * m / n;
      acc += cmul(a[m], CMPLX(cos(ang), sin(ang)));
    }
    out[k] = acc;
  }
  memcpy(a, out, sizeof(cx) * n);
  free(out);
}

static void fft_1d(cx* a, int n, int sign) {
  if (n <= 1) return;
  if ((n & (n - 1)) == 0)
    fft_radix2(a, n, sign);
  else
    fft_direct(a, n, sign);
}

/* forward_2d / inverse_2d, fft.hpp:96-115: rows then columns; inverse /N per 1-D pass */
static void fft_2d(cx* a, int w, int h, int sign) {
  for (int y = 0; y < h; ++y) {
    fft_1d(a + (size_t)y * w, w, sign);
    if (sign > 0)
      for (int x = 0; x < w; ++x) a[(size_t)y * w + x] /= w;
  }
  cx* col = (cx*)malloc(sizeof(cx) * h);
  for (int x = 0; x < w; ++x) {
    for (int y = 0; y < h; ++y) col[y] = a[(size_t)y * w + x];
    fft_1d(col, h, sign);
    if (sign > 0)
      for (int y = 0; y < h; ++y) col[y] /= h;
    for (int y = 0; y < h; ++y) a[(size_t)y * w + x] = col[y];
  }
  free(col);
}

/* ---------------------------------------------------------- patch layout */

typedef struct {
  int P, stride, nx, ny, n;
  int* ox;
  int* oy;
  double* cx;
  double* cy;
} Layout;

static int offsets_1d(int extent, int P, int stride, int* out) { /* core.hpp:232-241 */
  if (extent <= P) {
    if (out) out[0] = 0;
    return 1;
  }
  int last = extent - P, n = 0;
  for (int o = 0; o < last; o += stride) {
    if (out) out[n] = o;
    ++n;
  }
  if (out) out[n] = last;
  return n + 1;
}

/* make_patch_layout, core.hpp:252-281 */
static int make_layout(int W, int H, double pitch, double ox, double oy, double patch_mm,
                       double overlap, Layout* L) {
  if (W < 1 || H < 1 || !(pitch > 0.0)) return 2;
  if (!(overlap >= 0.0 && overlap < 1.0)) return 2;
  int P = (int)lround(patch_mm / pitch);
  if (P < 1 || P > W || P > H) return 2;
  int stride = imax(1, (int)lround(P * (1.0 - overlap)));
  int nx = offsets_1d(W, P, stride, NULL), ny = offsets_1d(H, P, stride, NULL);
  int* xs = (int*)malloc(sizeof(int) * nx);
  int* ys = (int*)malloc(sizeof(int) * ny);
  offsets_1d(W, P, stride, xs);
  offsets_1d(H, P, stride, ys);
  L->P = P;
  L->stride = stride;
  L->nx = nx;
  L->ny = ny;
  L->n = nx * ny;
  L->ox = (int*)malloc(sizeof(int) * L->n);
  L->oy = (int*)malloc(sizeof(int) * L->n);
  L->cx = (double*)malloc(sizeof(double) * L->n);
  L->cy = (double*)malloc(sizeof(double) * L->n);
  double half = 0.5 * (P - 1);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      int k = j * nx + i;
      L->ox[k] = xs[i];
      L->oy[k] = ys[j];
      L->cx[k] = ox + (xs[i] + half) * pitch;
      L->cy[k] = oy + (ys[j] + half) * pitch;
    }
  free(xs);
  free(ys);
  return 0;
}

static void free_layout(Layout* L) {
  free(L->ox);
  free(L->oy);
  free(L->cx);
  free(L->cy);
}

int orc_patch_layout(int W, int H, double pitch, double ox, double oy, double patch_mm,
                     double overlap, int* info, int* offsets, double* centers) {
  Layout L;
  int rc = make_layout(W, H, pitch, ox, oy, patch_mm, overlap, &L);
  if (rc) return rc;
  info[0] = L.P;
  info[1] = L.stride;
  info[2] = L.nx;
  info[3] = L.ny;
  for (int k = 0; k < L.n; ++k) {
    if (offsets) {
      offsets[2 * k] = L.ox[k];
      offsets[2 * k + 1] = L.oy[k];
    }
    if (centers) {
      centers[2 * k] = L.cx[k];
      centers[2 * k + 1] = L.cy[k];
    }
  }
  free_layout(&L);
  return 0;
}

/* extract_patch_spectra_one, deconv.hpp:45-62 (Y: [K][P][P] for one patch) */
static void patch_spectra_one(const double* stack, int K, int W, int H, const Layout* L, int i,
                              cx* Y) {
  const int P = L->P;
  for (int j = 0; j < K; ++j) {
    cx* b = Y + (size_t)j * P * P;
    const double* img = stack + (size_t)j * W * H;
    for (int y = 0; y < P; ++y)
      for (int x = 0; x < P; ++x) b[(size_t)y * P + x] = img[(size_t)(L->oy[i] + y) * W + L->ox[i] + x];
    fft_2d(b, P, P, -1);
  }
}

int orc_patch_spectra(int K, const double* delays, double v0, int W, int H, double pitch,
                      double ox, double oy, const double* stack, double patch_mm, double overlap,
                      int workers, double* Y) {
  (void)delays;
  (void)v0;
  (void)workers;
  if (K < 1) return 2;
  Layout L;
  int rc = make_layout(W, H, pitch, ox, oy, patch_mm, overlap, &L);
  if (rc) return rc;
  size_t per = (size_t)K * L.P * L.P;
  for (int i = 0; i < L.n; ++i) patch_spectra_one(stack, K, W, H, &L, i, (cx*)Y + i * per);
  free_layout(&L);
  return 0;
}

/* ------------------------------------------------------------ wavefronts */

/* wavefront_profile, aberration.hpp:134-186 (one centre) */
static int wavefront_one(double cx_, double cy_, double radius, const double* sos, int W, int H,
                         double pitch, double ox, double oy, double v0, double mcx, double mcy,
                         double mr, int A, double step, double* w) {
  if (A < 4 || !(step > 0.0)) return 2;
  if (hypot(cx_, cy_) >= radius) return 2;
  for (int a = 0; a < A; ++a) {
    double th = 2.0 * M_PI * a / A;
    double ux = cos(th), uy = sin(th);
    double b = cx_ * ux + cy_ * uy;
    double c = (cx_ * cx_ + cy_ * cy_) - radius * radius;
    double t_ring = -b + sqrt(b * b - c);
    double t0, t1;
    seg_circle(cx_, cy_, cx_ + ux * t_ring, cy_ + uy * t_ring, mcx, mcy, mr, &t0, &t1);
    w[a] = 0.0;
    if (t0 >= t1) continue;
    int n = imax(1, (int)ceil((t1 - t0) / step));
    double dl = (t1 - t0) / n, acc = 0.0;
    for (int i = 0; i < n; ++i) {
      double s = t0 + (i + 0.5) * dl;
      Stencil st = stencil_at(sos, W, H, pitch, ox, oy, cx_ + ux * s, cy_ + uy * s);
      acc += dl * (1.0 - v0 / st.value);
    }
    w[a] = acc;
  }
  return 0;
}

int orc_wavefront_profile(int n_centers, const double* centers, int n_tx, double radius,
                          double offset, int W, int H, double pitch, double ox, double oy,
                          const double* sos, double v0, double mcx, double mcy, double mr,
                          int n_angles, double step, double* w) {
  (void)offset;
  if (n_tx < 3 || !(radius > 0.0)) return 2;
  for (int i = 0; i < n_centers; ++i) {
    int rc = wavefront_one(centers[2 * i], centers[2 * i + 1], radius, sos, W, H, pitch, ox, oy, v0,
                           mcx, mcy, mr, n_angles, step, w + (size_t)i * n_angles);
    if (rc) return rc;
  }
  return 0;
}

/* wavefront_grad_trace, aberration.hpp:333-361 */
int orc_wavefront_grad_trace(double cx_, double cy_, int n_tx, double radius, double offset, int W,
                             int H, double pitch, double ox, double oy, const double* sos,
                             double v0, double mcx, double mcy, double mr, int n_angles,
                             double step, const double* dw, double* grad_v) {
  (void)n_tx;
  (void)offset;
  for (int a = 0; a < n_angles; ++a) {
    double g = dw[a];
    if (g == 0.0) continue;
    double th = 2.0 * M_PI * a / n_angles;
    double ux = cos(th), uy = sin(th);
    double b = cx_ * ux + cy_ * uy;
    double c = (cx_ * cx_ + cy_ * cy_) - radius * radius;
    double t_ring = -b + sqrt(b * b - c);
    double t0, t1;
    seg_circle(cx_, cy_, cx_ + ux * t_ring, cy_ + uy * t_ring, mcx, mcy, mr, &t0, &t1);
    if (t0 >= t1) continue;
    int n = imax(1, (int)ceil((t1 - t0) / step));
    double dl = (t1 - t0) / n;
    for (int i = 0; i < n; ++i) {
      double s = t0 + (i + 0.5) * dl;
      Stencil st = stencil_at(sos, W, H, pitch, ox, oy, cx_ + ux * s, cy_ + uy * s);
      double f = g * dl * v0 / (st.value * st.value);
      for (int k = 0; k < 4; ++k) grad_v[st.idx[k]] += f * st.w[k];
    }
  }
  return 0;
}

/* --------------------------------------------------------- transfer stacks */

/* WavefrontProfile::interpolate index/fraction, aberration.hpp:119-128 */
static void interp_idx(double theta, int A, int* i0, int* i1, double* f) {
  double tau = 2.0 * M_PI;
  double pos = fmod(theta, tau);
  if (pos < 0) pos += tau;
  pos = pos / tau * A;
  *i0 = (int)pos % A;
  *f = pos - floor(pos);
  *i1 = (*i0 + 1) % A;
}

/* detail::bin_geometry, aberration.hpp:225-230 (freq_index, fft.hpp:35) */
static void bin_geom(int bx, int by, int P, double pitch, double* kmag, double* ang) {
  double scale = 2.0 * M_PI / (P * pitch);
  double kx = scale * (bx <= P / 2 ? bx : bx - P);
  double ky = scale * (by <= P / 2 ? by : by - P);
  *kmag = hypot(kx, ky);
  *ang = atan2(ky, kx);
}

/* detail::conj_symmetrize_nyquist, aberration.hpp:203-218 */
static void sym_nyquist(cx* h, int P) {
  if (P % 2 != 0) return;
  int half = P / 2;
  for (int pass = 0; pass < 2; ++pass)
    for (int t = 0; t < P; ++t) {
      int bx = pass == 0 ? half : t, by = pass == 0 ? t : half;
      size_t i = (size_t)by * P + bx;
      size_t j = (size_t)((P - by) % P) * P + (P - bx) % P;
      if (j < i) continue;
      cx s = 0.5 * (h[i] + conj(h[j]));
      h[i] = s;
      h[j] = conj(s);
    }
}

/* transfer_stack, aberration.hpp:236-265 */
int orc_transfer_stack(int A, const double* w, int K, const double* delays, int P, double pitch,
                       double* Hc) {
  if (P < 1 || !(pitch > 0.0)) return 2;
  cx* H = (cx*)Hc;
  const size_t P2 = (size_t)P * P;
  for (int by = 0; by < P; ++by)
    for (int bx = 0; bx < P; ++bx) {
      size_t b = (size_t)by * P + bx;
      double k, ang;
      bin_geom(bx, by, P, pitch, &k, &ang);
      if (k == 0.0) {
        for (int j = 0; j < K; ++j) H[j * P2 + b] = 1.0;
        continue;
      }
      int a0, a1, b0, b1;
      double f1, f2;
      interp_idx(ang, A, &a0, &a1, &f1);
      interp_idx(ang + M_PI, A, &b0, &b1, &f2);
      double w1 = (1.0 - f1) * w[a0] + f1 * w[a1];
      double w2 = (1.0 - f2) * w[b0] + f2 * w[b1];
      for (int j = 0; j < K; ++j)
        H[j * P2 + b] = polar(0.5, -k * (delays[j] - w1)) + polar(0.5, +k * (delays[j] - w2));
    }
  for (int j = 0; j < K; ++j) sym_nyquist(H + j * P2, P);
  return 0;
}

/* ------------------------------------------------------------ fused loss */

typedef struct {
  int P, A;
  double* kmag;
  int* idx; /* [4 P2] a0 a1 b0 b1 */
  double* f;    /* [2 P2] f1 f2 */
} BinTable;

/* PatchBinTable::make, aberration.hpp:373-401 */
static void bin_table(int P, double pitch, int A, BinTable* t) {
  size_t P2 = (size_t)P * P;
  t->P = P;
  t->A = A;
  t->kmag = (double*)malloc(sizeof(double) * P2);
  t->idx = (int*)malloc(sizeof(int) * 4 * P2);
  t->f = (double*)malloc(sizeof(double) * 2 * P2);
  for (int by = 0; by < P; ++by)
    for (int bx = 0; bx < P; ++bx) {
      size_t b = (size_t)by * P + bx;
      double ang;
      bin_geom(bx, by, P, pitch, &t->kmag[b], &ang);
      interp_idx(ang, A, &t->idx[4 * b], &t->idx[4 * b + 1], &t->f[2 * b]);
      interp_idx(ang + M_PI, A, &t->idx[4 * b + 2], &t->idx[4 * b + 3], &t->f[2 * b + 1]);
    }
}

static void free_bins(BinTable* t) {
  free(t->kmag);
  free(t->idx);
  free(t->f);
}

/* detail::fused_patch_loss_grad, optimize.hpp:234-325 (phases: make_delay_phases, 223-232) */
static double fused_loss(const float* Yf, const double* w, const BinTable* t, const cx* dph,
                         int K, double eps, double scale, int implicit, double* dw) {
  const int P = t->P, A = t->A;
  const size_t P2 = (size_t)P * P;
  cx* h = (cx*)malloc(sizeof(cx) * K * P2);
  cx* gh = (cx*)calloc(K * P2, sizeof(cx));
  cx* e1 = (cx*)malloc(sizeof(cx) * P2);
  cx* e2 = (cx*)malloc(sizeof(cx) * P2);
  for (int a = 0; a < A; ++a) dw[a] = 0.0;
  for (size_t b = 0; b < P2; ++b) {
    const int* ix = t->idx + 4 * b;
    double w1 = (1 - t->f[2 * b]) * w[ix[0]] + t->f[2 * b] * w[ix[1]];
    double w2 = (1 - t->f[2 * b + 1]) * w[ix[2]] + t->f[2 * b + 1] * w[ix[3]];
    e1[b] = polar(1.0, t->kmag[b] * w1);
    e2[b] = polar(1.0, -t->kmag[b] * w2);
  }
  for (int j = 0; j < K; ++j) {
    for (size_t b = 0; b < P2; ++b)
      h[j * P2 + b] = 0.5 * (cmul(dph[j * P2 + b], e1[b]) + cmul(conj(dph[j * P2 + b]), e2[b]));
    sym_nyquist(h + j * P2, P);
  }
  double value = 0.0;
  for (size_t b = 0; b < P2; ++b) {
    double wk = t->kmag[b] * scale;
    if (wk == 0.0) continue;
    cx num = 0.0;
    double den = eps * (double)K;
    for (int j = 0; j < K; ++j) {
      cx hj = h[j * P2 + b];
      cx yj = CMPLX((double)Yf[2 * (j * P2 + b)], (double)Yf[2 * (j * P2 + b) + 1]);
      num += cmul(conj(hj), yj);
      den += cnorm(hj);
    }
    cx x = den > 0.0 ? num / den : 0.0;
    cx G = 0.0;
    for (int j = 0; j < K; ++j) {
      cx hj = h[j * P2 + b];
      cx yj = CMPLX((double)Yf[2 * (j * P2 + b)], (double)Yf[2 * (j * P2 + b) + 1]);
      cx rj = yj - cmul(hj, x);
      value += wk * cnorm(rj);
      cx z = cmul(conj(rj), x);
      gh[j * P2 + b] += CMPLX(-2.0 * wk * creal(z), 2.0 * wk * cimag(z));
      G += cmul(conj(rj), hj);
    }
    if (implicit && den > 0.0) {
      double gx = creal(G) * creal(x) - cimag(G) * cimag(x);
      for (int j = 0; j < K; ++j) {
        cx hj = h[j * P2 + b];
        cx yj = CMPLX((double)Yf[2 * (j * P2 + b)], (double)Yf[2 * (j * P2 + b) + 1]);
        cx gy = cmul(G, yj);
        gh[j * P2 + b] += CMPLX(-2.0 * wk * creal(gy) / den + 4.0 * wk * gx * creal(hj) / den,
                                -2.0 * wk * cimag(gy) / den + 4.0 * wk * gx * cimag(hj) / den);
      }
    }
  }
  for (int j = 0; j < K; ++j) {
    sym_nyquist(gh + j * P2, P); /* self-adjoint pullback */
    for (size_t b = 0; b < P2; ++b) {
      cx gb = gh[j * P2 + b];
      if (creal(gb) == 0.0 && cimag(gb) == 0.0) continue;
      const int* ix = t->idx + 4 * b;
      cx t1 = 0.5 * cmul(dph[j * P2 + b], e1[b]);
      cx t2 = 0.5 * cmul(conj(dph[j * P2 + b]), e2[b]);
      double g1 = t->kmag[b] * (creal(gb) * -cimag(t1) + cimag(gb) * creal(t1));
      double g2 = t->kmag[b] * (creal(gb) * cimag(t2) + cimag(gb) * -creal(t2));
      dw[ix[0]] += (1 - t->f[2 * b]) * g1;
      dw[ix[1]] += t->f[2 * b] * g1;
      dw[ix[2]] += (1 - t->f[2 * b + 1]) * g2;
      dw[ix[3]] += t->f[2 * b + 1] * g2;
    }
  }
  free(h);
  free(gh);
  free(e1);
  free(e2);
  return value;
}

static cx* delay_phases(const BinTable* t, const double* delays, int K) {
  size_t P2 = (size_t)t->P * t->P;
  cx* d = (cx*)malloc(sizeof(cx) * K * P2);
  for (int j = 0; j < K; ++j)
    for (size_t b = 0; b < P2; ++b) d[j * P2 + b] = polar(1.0, -t->kmag[b] * delays[j]);
  return d;
}

int orc_fused_patch_loss_grad(int K, const float* Yf, const double* w, int P, double pitch,
                              int n_angles, const double* delays, double eps, double scale,
                              int implicit, double* loss, double* dw) {
  BinTable t;
  bin_table(P, pitch, n_angles, &t);
  cx* dph = delay_phases(&t, delays, K);
  *loss = fused_loss(Yf, w, &t, dph, K, eps, scale, implicit, dw);
  free(dph);
  free_bins(&t);
  return 0;
}

/* --------------------------------------------------------------------- TV */

/* tv_loss, optimize.hpp:120-153 over the masked pixels of render_sos */
static double tv_eval(const double* v, const unsigned char* inm, const int* flat2m, int W, int H,
                      double lambda, double* grad, int n) {
  double value = 0.0;
  for (int i = 0; i < n; ++i) grad[i] = 0.0;
  int i = 0;
  for (int p = 0; p < W * H; ++p) {
    if (!inm[p]) continue;
    int ix = p % W, iy = p / W;
    if (ix + 1 < W && inm[p + 1]) {
      double d = v[p + 1] - v[p];
      double sg = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
      value += fabs(d);
      grad[flat2m[p + 1]] += lambda * sg;
      grad[i] -= lambda * sg;
    }
    if (iy + 1 < H && inm[p + W]) {
      double d = v[p + W] - v[p];
      double sg = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
      value += fabs(d);
      grad[flat2m[p + W]] += lambda * sg;
      grad[i] -= lambda * sg;
    }
    ++i;
  }
  return value * lambda;
}

static int mask_map(int W, int H, double pitch, double ox, double oy, double mcx, double mcy,
                    double mr, unsigned char* inm, int* flat2m, int* idx) {
  int n = 0;
  for (int iy = 0; iy < H; ++iy)
    for (int ix = 0; ix < W; ++ix) {
      int p = iy * W + ix;
      inm[p] = hypot(ox + ix * pitch - mcx, oy + iy * pitch - mcy) <= mr;
      flat2m[p] = inm[p] ? n : -1;
      if (inm[p]) {
        if (idx) idx[n] = p;
        ++n;
      }
    }
  return n;
}

int orc_tv_loss(int W, int H, double pitch, double ox, double oy, const double* raster,
                double mcx, double mcy, double mr, double lambda, double* value,
                double* grad_masked) {
  unsigned char* inm = (unsigned char*)malloc((size_t)W * H);
  int* f2m = (int*)malloc(sizeof(int) * W * H);
  int n = mask_map(W, H, pitch, ox, oy, mcx, mcy, mr, inm, f2m, NULL);
  *value = tv_eval(raster, inm, f2m, W, H, lambda, grad_masked, n);
  free(inm);
  free(f2m);
  return 0;
}

/* ------------------------------------------------------------------- Adam */

/* adam_step, optimize.hpp:87-110 (m, v start at zero when t == 0) */
int orc_adam_step(int n, double* p, const double* g, double* m, double* v, long* t, double lr,
                  double b1, double b2, double eps) {
  if (*t == 0)
    for (int i = 0; i < n; ++i) m[i] = v[i] = 0.0;
  for (int i = 0; i < n; ++i)
    if (!isfinite(g[i])) return 3;
  *t += 1;
  double bc1 = 1.0 - pow(b1, (double)*t), bc2 = 1.0 - pow(b2, (double)*t);
  for (int i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    p[i] -= lr * (m[i] / bc1) / (sqrt(v[i] / bc2) + eps);
  }
  return 0;
}

/* ------------------------------------------------------------ deconvolution */

/* MergeWindow::make, deconv.hpp:124-138 */
static double* merge_window(double fwhm, int P, double pitch) {
  double sig = fwhm / (2.0 * sqrt(2.0 * log(2.0))) / pitch;
  double c = 0.5 * (P - 1);
  double* w = (double*)malloc(sizeof(double) * P * P);
  for (int y = 0; y < P; ++y)
    for (int x = 0; x < P; ++x) {
      double r2 = (x - c) * (x - c) + (y - c) * (y - c);
      w[y * P + x] = exp(-0.5 * r2 / (sig * sig));
    }
  return w;
}

/* multichannel_deconvolve (deconv.hpp:78-96) + inverse_2d + merge_patches
 * (deconv.hpp:142-164), the per-patch pipeline of deconvolve_image (176-198). */
static void deconvolve(const double* stack, int K, const double* delays, double v0, int W, int H,
                       double pitch, double ox, double oy, const double* sos, double radius,
                       double mcx, double mcy, double mr, const Layout* L, double eps, int A,
                       double ray_step, double fwhm, double* image) {
  const int P = L->P;
  const size_t P2 = (size_t)P * P;
  double* img = (double*)calloc((size_t)W * H, sizeof(double));
  double* wsum = (double*)calloc((size_t)W * H, sizeof(double));
  double* win = merge_window(fwhm, P, pitch);
  cx* Y = (cx*)malloc(sizeof(cx) * K * P2);
  double* Hc = (double*)malloc(sizeof(double) * 2 * K * P2);
  double* wv = (double*)malloc(sizeof(double) * A);
  cx* x = (cx*)malloc(sizeof(cx) * P2);
  for (int i = 0; i < L->n; ++i) {
    patch_spectra_one(stack, K, W, H, L, i, Y);
    wavefront_one(L->cx[i], L->cy[i], radius, sos, W, H, pitch, ox, oy, v0, mcx, mcy, mr, A,
                  ray_step, wv);
    orc_transfer_stack(A, wv, K, delays, P, pitch, Hc);
    const cx* Hs = (const cx*)Hc;
    for (size_t b = 0; b < P2; ++b) {
      cx num = 0.0;
      double den = eps * (double)K;
      for (int j = 0; j < K; ++j) {
        num += cmul(conj(Hs[j * P2 + b]), Y[j * P2 + b]);
        den += cnorm(Hs[j * P2 + b]);
      }
      x[b] = den > 0.0 ? num / den : 0.0;
    }
    fft_2d(x, P, P, +1);
    for (int y = 0; y < P; ++y)
      for (int xx = 0; xx < P; ++xx) {
        size_t q = (size_t)(L->oy[i] + y) * W + L->ox[i] + xx;
        double wgt = win[y * P + xx];
        img[q] += wgt * creal(x[(size_t)y * P + xx]);
        wsum[q] += wgt;
      }
  }
  for (size_t q = 0; q < (size_t)W * H; ++q) image[q] = wsum[q] > 0.0 ? img[q] / wsum[q] : img[q];
  free(img);
  free(wsum);
  free(win);
  free(Y);
  free(Hc);
  free(wv);
  free(x);
}

int orc_deconvolve_image(int K, const double* delays, double v0, int W, int H, double pitch,
                         double ox, double oy, const double* stack, const double* sos, int n_tx,
                         double radius, double offset, double mcx, double mcy, double mr,
                         double patch_mm, double overlap, double eps, int n_angles,
                         double ray_step, double merge_fwhm, int workers, double* image) {
  (void)n_tx;
  (void)offset;
  (void)workers;
  if (K < 1 || !(merge_fwhm > 0.0)) return 2;
  Layout L;
  int rc = make_layout(W, H, pitch, ox, oy, patch_mm, overlap, &L);
  if (rc) return rc;
  deconvolve(stack, K, delays, v0, W, H, pitch, ox, oy, sos, radius, mcx, mcy, mr, &L, eps,
             n_angles, ray_step, merge_fwhm, image);
  free_layout(&L);
  return 0;
}

/* ---------------------------------------------------------- training loop */

typedef struct {
  int W, H, K, A, np, nm, n_tx;
  double pitch, ox, oy, radius, v0, mcx, mcy, mr, scale;
  Layout L;
  BinTable bins;
  cx* dph;
  float* ycache; /* [n][K][P2] complex<float> (optimize.hpp:382-392) */
  double* stack;
  unsigned char* inm;
  int* f2m;
} Engine;

static int engine_init(Engine* e, int n_tx, double radius, double offset, int T, double dt,
                       double t0, double v0, const double* sig, int W, int H, double pitch,
                       double ox, double oy, double mcx, double mcy, double mr,
                       const OrcTrainCfg* c) {
  int K = c->n_delays;
  e->W = W;
  e->H = H;
  e->K = K;
  e->A = c->n_angles;
  e->n_tx = n_tx;
  e->pitch = pitch;
  e->ox = ox;
  e->oy = oy;
  e->radius = radius;
  e->v0 = v0;
  e->mcx = mcx;
  e->mcy = mcy;
  e->mr = mr;
  int rc = make_layout(W, H, pitch, ox, oy, c->patch_mm, c->overlap, &e->L);
  if (rc) return rc;
  const int P = e->L.P;
  const size_t P2 = (size_t)P * P;
  e->scale = 1.0 / ((double)e->L.n * K * P * P);
  e->stack = (double*)malloc(sizeof(double) * K * W * H);
  rc = orc_das_stack(n_tx, radius, offset, T, dt, t0, sig, W, H, pitch, ox, oy, v0, K, c->delays, 0,
                     e->stack);
  if (rc) return rc;
  e->ycache = (float*)malloc(sizeof(float) * 2 * e->L.n * K * P2);
  cx* Y = (cx*)malloc(sizeof(cx) * K * P2);
  for (int i = 0; i < e->L.n; ++i) {
    patch_spectra_one(e->stack, K, W, H, &e->L, i, Y);
    for (size_t q = 0; q < K * P2; ++q) {
      e->ycache[2 * (i * K * P2 + q)] = (float)creal(Y[q]);
      e->ycache[2 * (i * K * P2 + q) + 1] = (float)cimag(Y[q]);
    }
  }
  free(Y);
  bin_table(P, pitch, e->A, &e->bins);
  e->dph = delay_phases(&e->bins, c->delays, K);
  e->np = (int)s_off(c->sine_layers + 1, c->hidden, c->sine_layers);
  e->inm = (unsigned char*)malloc((size_t)W * H);
  e->f2m = (int*)malloc(sizeof(int) * W * H);
  e->nm = mask_map(W, H, pitch, ox, oy, mcx, mcy, mr, e->inm, e->f2m, NULL);
  return 0;
}

static void engine_free(Engine* e) {
  free_layout(&e->L);
  free_bins(&e->bins);
  free(e->dph);
  free(e->ycache);
  free(e->stack);
  free(e->inm);
  free(e->f2m);
}

/* One step body (optimize.hpp:413-461): loss terms, dL/dv at masked pixels, dL/dtheta. */
static int engine_grad(const Engine* e, const OrcTrainCfg* c, const double* theta, int lo, int hi,
                       double* data, double* tv, double* lp, double* w_out, double* dw_out,
                       double* sos, double* gmask, double* grad) {
  const size_t P2 = (size_t)e->L.P * e->L.P;
  const int W = e->W, H = e->H, A = e->A;
  orc_render_sos(c->hidden, c->sine_layers, c->omega0, c->out_scale, e->v0, theta, W, H, e->pitch,
                 e->ox, e->oy, e->mcx, e->mcy, e->mr, sos, NULL);
  for (int q = 0; q < W * H; ++q)
    if (!isfinite(sos[q])) return 3;
  double* gv = (double*)calloc((size_t)W * H, sizeof(double));
  double* wv = (double*)malloc(sizeof(double) * A);
  double* dw = (double*)malloc(sizeof(double) * A);
  double d = 0.0;
  for (int i = 0; i < e->L.n; ++i) {
    double l = 0.0;
    if (i >= lo && i < hi) {
      wavefront_one(e->L.cx[i], e->L.cy[i], e->radius, sos, W, H, e->pitch, e->ox, e->oy, e->v0,
                    e->mcx, e->mcy, e->mr, A, c->ray_step, wv);
      l = fused_loss(e->ycache + 2 * (size_t)i * e->K * P2, wv, &e->bins, e->dph, e->K,
                     c->eps_deconv, e->scale, c->implicit_xhat_grad, dw);
      orc_wavefront_grad_trace(e->L.cx[i], e->L.cy[i], e->n_tx, e->radius, 0.0, W, H, e->pitch,
                               e->ox, e->oy, sos, e->v0, e->mcx, e->mcy, e->mr, A, c->ray_step,
                               dw, gv);
      if (w_out) memcpy(w_out + (size_t)i * A, wv, sizeof(double) * A);
      if (dw_out) memcpy(dw_out + (size_t)i * A, dw, sizeof(double) * A);
    }
    if (lp) lp[i] = l;
    d += l;
  }
  double* tvg = (double*)malloc(sizeof(double) * (e->nm > 0 ? e->nm : 1));
  double t = tv_eval(sos, e->inm, e->f2m, W, H, c->lambda_tv, tvg, e->nm);
  int m = 0;
  for (int p = 0; p < W * H; ++p)
    if (e->inm[p]) {
      gmask[m] = gv[p] + tvg[m];
      ++m;
    }
  orc_backprop_sos(c->hidden, c->sine_layers, c->omega0, c->out_scale, e->v0, theta, W, H,
                   e->pitch, e->ox, e->oy, e->mcx, e->mcy, e->mr, gmask, grad);
  *data = d;
  *tv = t;
  free(gv);
  free(wv);
  free(dw);
  free(tvg);
  if (!isfinite(d) || !isfinite(t)) return 3;
  for (int i = 0; i < e->np; ++i)
    if (!isfinite(grad[i])) return 3;
  return 0;
}

int orc_nf_step(int n_tx, double radius, double offset, int T, double dt, double t0, double v0,
                const double* sig, int W, int H, double pitch, double ox, double oy, double mcx,
                double mcy, double mr, const OrcTrainCfg* c, const double* theta, int patch_lo,
                int patch_hi, double* data_term, double* tv_term, double* loss_patch,
                double* w_out, double* dw_out, double* sos_out, double* grad_v_masked,
                double* grad_theta, double* image, double* seconds) {
  Engine e;
  int rc = engine_init(&e, n_tx, radius, offset, T, dt, t0, v0, sig, W, H, pitch, ox, oy, mcx, mcy,
                       mr, c);
  if (rc) return rc;
  double* sos = (double*)malloc(sizeof(double) * W * H);
  double* gm = (double*)malloc(sizeof(double) * (e.nm > 0 ? e.nm : 1));
  double* grad = (double*)malloc(sizeof(double) * e.np);
  double d = 0.0, t = 0.0;
  int hi = patch_hi < 0 ? e.L.n : imin(patch_hi, e.L.n);
  clock_t c0 = clock();
  rc = engine_grad(&e, c, theta, patch_lo, hi, &d, &t, loss_patch, w_out, dw_out, sos, gm, grad);
  if (seconds) *seconds = (double)(clock() - c0) / CLOCKS_PER_SEC;
  if (data_term) *data_term = d;
  if (tv_term) *tv_term = t;
  if (sos_out) memcpy(sos_out, sos, sizeof(double) * W * H);
  if (grad_v_masked) memcpy(grad_v_masked, gm, sizeof(double) * e.nm);
  if (grad_theta) memcpy(grad_theta, grad, sizeof(double) * e.np);
  if (image)
    deconvolve(e.stack, e.K, c->delays, v0, W, H, pitch, ox, oy, sos, radius, mcx, mcy, mr, &e.L,
               c->eps_deconv, c->n_angles, c->ray_step, c->merge_fwhm, image);
  free(sos);
  free(gm);
  free(grad);
  engine_free(&e);
  return rc;
}

/* joint_reconstruct, optimize.hpp:367-494 */
int orc_joint_reconstruct(int n_tx, double radius, double offset, int T, double dt, double t0,
                          double v0, const double* sig, int W, int H, double pitch, double ox,
                          double oy, double mcx, double mcy, double mr, const OrcTrainCfg* c,
                          double* reports, double* image, double* sos_out, double* theta_out) {
  if (c->epochs < 1 || c->steps_per_epoch < 1 || !(c->lr > 0.0) || !(c->lambda_tv >= 0.0) ||
      c->n_delays < 1 || !(v0 > 0.0))
    return 2;
  Engine e;
  int rc = engine_init(&e, n_tx, radius, offset, T, dt, t0, v0, sig, W, H, pitch, ox, oy, mcx, mcy,
                       mr, c);
  if (rc) return rc;
  double* theta = (double*)malloc(sizeof(double) * e.np);
  orc_init_siren(c->seed, c->hidden, c->sine_layers, c->omega0, c->out_scale, v0, theta);
  double* m = (double*)calloc(e.np, sizeof(double));
  double* v = (double*)calloc(e.np, sizeof(double));
  double* grad = (double*)malloc(sizeof(double) * e.np);
  double* sos = (double*)malloc(sizeof(double) * W * H);
  double* gm = (double*)malloc(sizeof(double) * (e.nm > 0 ? e.nm : 1));
  long t = 0;
  for (int ep = 1; ep <= c->epochs && !rc; ++ep) {
    double d = 0.0, tv = 0.0;
    clock_t c0 = clock();
    for (int s = 0; s < c->steps_per_epoch && !rc; ++s) {
      rc = engine_grad(&e, c, theta, 0, e.L.n, &d, &tv, NULL, NULL, NULL, sos, gm, grad);
      if (!rc) rc = orc_adam_step(e.np, theta, grad, m, v, &t, c->lr, c->beta1, c->beta2,
                                  c->adam_eps);
    }
    if (reports) {
      reports[4 * (ep - 1)] = d;
      reports[4 * (ep - 1) + 1] = tv;
      reports[4 * (ep - 1) + 2] = d + tv;
      reports[4 * (ep - 1) + 3] = (double)(clock() - c0) / CLOCKS_PER_SEC;
    }
  }
  if (!rc) {
    orc_render_sos(c->hidden, c->sine_layers, c->omega0, c->out_scale, v0, theta, W, H, pitch, ox,
                   oy, mcx, mcy, mr, sos, NULL);
    if (image)
      deconvolve(e.stack, e.K, c->delays, v0, W, H, pitch, ox, oy, sos, radius, mcx, mcy, mr, &e.L,
                 c->eps_deconv, c->n_angles, c->ray_step, c->merge_fwhm, image);
    if (sos_out) memcpy(sos_out, sos, sizeof(double) * W * H);
    if (theta_out) memcpy(theta_out, theta, sizeof(double) * e.np);
  }
  free(theta);
  free(m);
  free(v);
  free(grad);
  free(sos);
  free(gm);
  engine_free(&e);
  return rc;
}

/* ------------------------------------------------------------ simulator */

/* RasterGrid::sample_bilinear, core.hpp:129-144 */
static double sample_bilinear(const double* v, int W, int H, double pitch, double ox, double oy,
                              double px, double py) {
  double fx = dclamp((px - ox) / pitch, 0.0, (double)(W - 1));
  double fy = dclamp((py - oy) / pitch, 0.0, (double)(H - 1));
  int ix = imin((int)fx, W - 2 >= 0 ? W - 2 : 0), iy = imin((int)fy, H - 2 >= 0 ? H - 2 : 0);
  if (W == 1) ix = 0;
  if (H == 1) iy = 0;
  double ax = fx - ix, ay = fy - iy;
  int ix1 = imin(ix + 1, W - 1), iy1 = imin(iy + 1, H - 1);
  return (1 - ax) * (1 - ay) * v[iy * W + ix] + ax * (1 - ay) * v[iy * W + ix1] +
         (1 - ax) * ay * v[iy1 * W + ix] + ax * ay * v[iy1 * W + ix1];
}

/* simulate_signals, phantom.hpp:282-362, with time_of_flight (aberration.hpp:79-100) */
int orc_simulate_signals(int W, int H, double pitch, double ox, double oy, const double* pressure,
                         const double* sos, double mcx, double mcy, double mr,
                         double background_sos, int n_tx, double radius, double offset,
                         double pulse_sigma, double dt, double t0, int T, double ray_step,
                         int workers, double* out) {
  (void)workers;
  if (n_tx < 3 || !(radius > 0.0) || !(pulse_sigma > 0.0) || !(dt > 0.0)) return 2;
  int ns = 0;
  double max_r = 0.0;
  for (int q = 0; q < W * H; ++q)
    if (pressure[q] != 0.0) {
      double px = ox + (q % W) * pitch, py = oy + (q / W) * pitch;
      double r = hypot(px, py);
      if (r >= radius) return 2;
      max_r = fmax(max_r, r);
      ++ns;
    }
  double vmin = (W * H > 0) ? sos[0] : background_sos, vmax = vmin;
  for (int q = 0; q < W * H; ++q) {
    vmin = fmin(vmin, sos[q]);
    vmax = fmax(vmax, sos[q]);
  }
  if (!(vmin > 0.0)) return 2;
  int uniform = (vmin == vmax && vmin == background_sos);
  double tau_min = 1e-3 * (radius - max_r) / vmax - 8.0 * pulse_sigma;
  double tau_max = 1e-3 * (radius + max_r) / vmin + 8.0 * pulse_sigma;
  if (ns > 0 && (t0 > tau_min || t0 + (T - 1) * dt < tau_max)) return 2;
  memset(out, 0, sizeof(double) * n_tx * T);
  const double sigma = pulse_sigma, support = 6.0 * sigma;
  for (int n = 0; n < n_tx; ++n) {
    double rx, ry;
    ring_pos(n_tx, radius, offset, n, &rx, &ry);
    double* row = out + (size_t)n * T;
    for (int q = 0; q < W * H; ++q) {
      double amp = pressure[q];
      if (amp == 0.0) continue;
      double px = ox + (q % W) * pitch, py = oy + (q / W) * pitch;
      double dist = hypot(rx - px, ry - py);
      double tau;
      if (uniform) {
        tau = 1e-3 * dist / background_sos;
      } else {
        double corr = 0.0;
        if (dist > 0.0) {
          double a, b;
          seg_circle(px, py, rx, ry, mcx, mcy, mr, &a, &b);
          if (a < b) {
            double ux = (rx - px) * (1.0 / dist), uy = (ry - py) * (1.0 / dist);
            int k = imax(1, (int)ceil((b - a) / ray_step));
            double dl = (b - a) / k, inv0 = 1.0 / background_sos;
            for (int i = 0; i < k; ++i) {
              double s = a + (i + 0.5) * dl;
              double v = sample_bilinear(sos, W, H, pitch, ox, oy, px + ux * s, py + uy * s);
              corr += dl * (1.0 / v - inv0);
            }
          }
        }
        tau = 1e-3 * (dist / background_sos + corr);
      }
      double scale = 2.0 * amp / sigma;
      int i0 = imax(0, (int)ceil((tau - support - t0) / dt));
      int i1 = imin(T - 1, (int)floor((tau + support - t0) / dt));
      for (int i = i0; i <= i1; ++i) {
        double u = (t0 + i * dt - tau) / sigma;
        row[i] += scale * (1.0 - u * u) * exp(-0.5 * u * u);
      }
    }
  }
  return 0;
}
