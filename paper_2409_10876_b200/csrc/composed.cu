// The composed (non-fused) loss path of the reference and its adjoints, as
// batched fp64 device kernels:
//
//   multichannel_deconvolve     deconv.hpp:78-96
//   deconv_jacobian_H           deconv.hpp:100-115
//   patch_data_loss, data_loss  optimize.hpp:155-211, 329-353
//   transfer_grad_to_wavefront  aberration.hpp:270-313
//   wavefront_profile(with_jacobian = true)  aberration.hpp:134-186
//   accumulate_wavefront_grad   aberration.hpp:316-326
//
// The reference's training loop does not use these (it runs the fused
// detail::fused_patch_loss_grad + wavefront_grad_trace, built in fourier.cu /
// raymarch.cu in fp32); they are its composed, differentiable-by-parts API,
// used by its gradient tests (test_support.hpp:79-118) and by callers that want
// dL/dH.  Their operands are the reference's complex<double> spectra, so the
// arithmetic here is fp64 (B200 runs fp64 at full vector rate), which keeps the
// reference's finite-difference contracts (1e-4 with 1e-6 steps) meaningful.
//
// Layouts: spectra are complex128 [patch][K][P][P] (interleaved re, im);
// wavefront profiles fp64 [patch][A].  All sums are in a fixed order (no
// atomics) except accumulate_wavefront_grad's scatter, which is fp64 atomics
// like any J^T product over shared pixels.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "geom.cuh"

namespace pactgpu {
namespace {

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zmulc(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double znorm(double2 a) { return a.x * a.x + a.y * a.y; }

// Per-bin geometry of a P x P patch spectrum in fp64 (detail::bin_geometry,
// aberration.hpp:225-230; interpolation indices of transfer_grad_to_wavefront,
// aberration.hpp:279-286) and the angle -> (bin, weight) gather table of the
// dL/dw pullback.
struct BinTab64 {
  int P = 0, P2 = 0, A = 0;
  const double* kmag = nullptr;   // [P2]
  const int4* idx = nullptr;      // [P2] (a0, a1, b0, b1)
  const double2* frac = nullptr;  // [P2] (f1, f2)
  const int* mirror = nullptr;    // [P2] Nyquist partner (even P) or -1
  const int* csr_start = nullptr; // [A + 1]
  const int* csr_key = nullptr;   // [4 P2] (bin << 2) | {0: 1-f1, 1: f1, 2: 1-f2, 3: f2}
};

struct ComposedCache {
  int P = 0, A = -1;
  double pitch = 0.0;
  void* dev = nullptr;
  cudaStream_t stream = nullptr;
  std::vector<char> host;  // kept alive until the upload has run
  BinTab64 tab;
  ~ComposedCache() { pool_free(dev, stream); }
};

Status bin_table(pact_ctx* ctx, int P, double pitch, int A, BinTab64& out) {
  ComposedCache* c = ctx_ext<ComposedCache>(ctx, kExtComposed);
  if (c->dev && c->P == P && c->pitch == pitch && c->A == A) {
    out = c->tab;
    return {};
  }
  const int P2 = P * P;
  const double tau = 2.0 * M_PI;
  const double scale = 2.0 * M_PI / (P * pitch);
  std::vector<double> kmag(P2);
  std::vector<int4> idx(P2);
  std::vector<double2> frac(P2);
  std::vector<int> mirror(P2, -1);
  auto interp = [&](double theta, int& i0, int& i1, double& f) {
    double pos = std::fmod(theta, tau);
    if (pos < 0) pos += tau;
    pos = pos / tau * A;
    i0 = static_cast<int>(pos) % A;
    f = pos - std::floor(pos);
    i1 = (i0 + 1) % A;
  };
  for (int by = 0; by < P; ++by)
    for (int bx = 0; bx < P; ++bx) {
      const int b = by * P + bx;
      const double kx = scale * freq_index(bx, P), ky = scale * freq_index(by, P);
      kmag[b] = std::hypot(kx, ky);
      if (P % 2 == 0 && (bx == P / 2 || by == P / 2)) mirror[b] = ((P - by) % P) * P + (P - bx) % P;
      int a0 = 0, a1 = 0, b0 = 0, b1 = 0;
      double f1 = 0.0, f2 = 0.0;
      if (A > 0) {
        const double ang = std::atan2(ky, kx);
        interp(ang, a0, a1, f1);
        interp(ang + M_PI, b0, b1, f2);
      }
      idx[b] = make_int4(a0, a1, b0, b1);
      frac[b] = make_double2(f1, f2);
    }
  std::vector<int> start(std::max(A, 0) + 1, 0), key;
  if (A > 0) {
    for (int b = 0; b < P2; ++b)
      if (kmag[b] != 0.0) {
        start[idx[b].x + 1]++;
        start[idx[b].y + 1]++;
        start[idx[b].z + 1]++;
        start[idx[b].w + 1]++;
      }
    for (int a = 0; a < A; ++a) start[a + 1] += start[a];
    key.resize(start[A]);
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (int b = 0; b < P2; ++b) {  // ascending bins per angle: the reference's order
      if (kmag[b] == 0.0) continue;
      key[fill[idx[b].x]++] = (b << 2) | 0;
      key[fill[idx[b].y]++] = (b << 2) | 1;
      key[fill[idx[b].z]++] = (b << 2) | 2;
      key[fill[idx[b].w]++] = (b << 2) | 3;
    }
  }
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t o_k = 0, o_i = al(o_k + 8 * P2), o_f = al(o_i + 16 * P2), o_m = al(o_f + 16 * P2),
               o_s = al(o_m + 4 * P2), o_e = al(o_s + 4 * start.size()),
               total = al(o_e + 4 * std::max<size_t>(key.size(), 1));
  if (c->dev) {
    pool_free(c->dev, c->stream);
    c->dev = nullptr;
  }
  PACT_CUDA_S(cudaStreamSynchronize(ctx->stream));  // the previous host image may be in flight
  c->host.assign(total, 0);
  std::memcpy(c->host.data() + o_k, kmag.data(), 8 * P2);
  std::memcpy(c->host.data() + o_i, idx.data(), 16 * P2);
  std::memcpy(c->host.data() + o_f, frac.data(), 16 * P2);
  std::memcpy(c->host.data() + o_m, mirror.data(), 4 * P2);
  std::memcpy(c->host.data() + o_s, start.data(), 4 * start.size());
  if (!key.empty()) std::memcpy(c->host.data() + o_e, key.data(), 4 * key.size());
  PACT_TRY_S(pool_alloc(&c->dev, total, ctx->stream));
  c->stream = ctx->stream;
  PACT_CUDA_S(cudaMemcpyAsync(c->dev, c->host.data(), total, cudaMemcpyHostToDevice, ctx->stream));
  char* d = static_cast<char*>(c->dev);
  c->P = P;
  c->A = A;
  c->pitch = pitch;
  c->tab.P = P;
  c->tab.P2 = P2;
  c->tab.A = A;
  c->tab.kmag = reinterpret_cast<const double*>(d + o_k);
  c->tab.idx = reinterpret_cast<const int4*>(d + o_i);
  c->tab.frac = reinterpret_cast<const double2*>(d + o_f);
  c->tab.mirror = reinterpret_cast<const int*>(d + o_m);
  c->tab.csr_start = reinterpret_cast<const int*>(d + o_s);
  c->tab.csr_key = reinterpret_cast<const int*>(d + o_e);
  out = c->tab;
  return {};
}

// ---- multichannel_deconvolve (deconv.hpp:78-96) ----------------------------
__global__ void deconvolve64_kernel(const double2* __restrict__ Y, const double2* __restrict__ H,
                                    int K, int P2, double eps_m, double2* __restrict__ X) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= P2) return;
  const size_t base = static_cast<size_t>(blockIdx.y) * K * P2 + b;
  double2 num = make_double2(0.0, 0.0);
  double den = eps_m;
  for (int j = 0; j < K; ++j) {
    const double2 h = H[base + static_cast<size_t>(j) * P2], y = Y[base + static_cast<size_t>(j) * P2];
    const double2 c = zmulc(h, y);
    num.x += c.x;
    num.y += c.y;
    den += znorm(h);
  }
  X[static_cast<size_t>(blockIdx.y) * P2 + b] =
      den > 0.0 ? make_double2(num.x / den, num.y / den) : make_double2(0.0, 0.0);
}

// ---- deconv_jacobian_H (deconv.hpp:100-115), one thread per query ----------
__global__ void deconv_jacobian64_kernel(const double2* __restrict__ Y,
                                         const double2* __restrict__ H, int K, int P2,
                                         double eps_m, const int* __restrict__ q, int n_q,
                                         double2* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_q) return;
  const int patch = q[3 * t], j = q[3 * t + 1], bin = q[3 * t + 2];
  const size_t base = static_cast<size_t>(patch) * K * P2 + bin;
  double2 num = make_double2(0.0, 0.0);
  double den = eps_m;
  for (int m = 0; m < K; ++m) {
    const double2 h = H[base + static_cast<size_t>(m) * P2], y = Y[base + static_cast<size_t>(m) * P2];
    const double2 c = zmulc(h, y);
    num.x += c.x;
    num.y += c.y;
    den += znorm(h);
  }
  const double2 h = H[base + static_cast<size_t>(j) * P2], y = Y[base + static_cast<size_t>(j) * P2];
  const double2 x = make_double2(num.x / den, num.y / den);
  // X = num / den; d num = conj(dH) y; d den = 2 Re(conj(h) dH)
  out[2 * t] = make_double2((y.x - x.x * 2.0 * h.x) / den, (y.y - x.y * 2.0 * h.x) / den);
  out[2 * t + 1] = make_double2((y.y - x.x * 2.0 * h.y) / den, (-y.x - x.y * 2.0 * h.y) / den);
}

// ---- patch_data_loss (optimize.hpp:164-211), one thread per bin ------------
constexpr int kLB = 128;

__global__ void __launch_bounds__(kLB) patch_loss64_kernel(BinTab64 t, const double2* __restrict__ Y,
                                                           const double2* __restrict__ H, int K,
                                                           double eps_m, double scale, int implicit,
                                                           double2* __restrict__ grad_h,
                                                           double* __restrict__ part, int n_parts) {
  __shared__ double s_red[kLB / 32];
  const int P2 = t.P2, b = blockIdx.x * kLB + threadIdx.x;
  const size_t base = static_cast<size_t>(blockIdx.y) * K * P2 + b;
  double value = 0.0;
  if (b < P2) {
    const double wk = t.kmag[b] * scale;
    if (wk == 0.0) {
      for (int j = 0; j < K; ++j) grad_h[base + static_cast<size_t>(j) * P2] = make_double2(0.0, 0.0);
    } else {
      double2 num = make_double2(0.0, 0.0);
      double den = eps_m;
      for (int j = 0; j < K; ++j) {
        const double2 h = H[base + static_cast<size_t>(j) * P2];
        const double2 c = zmulc(h, Y[base + static_cast<size_t>(j) * P2]);
        num.x += c.x;
        num.y += c.y;
        den += znorm(h);
      }
      const double2 x = den > 0.0 ? make_double2(num.x / den, num.y / den) : make_double2(0.0, 0.0);
      double2 G = make_double2(0.0, 0.0);  // sum_j conj(R_j) H_j
      for (int j = 0; j < K; ++j) {
        const double2 h = H[base + static_cast<size_t>(j) * P2], y = Y[base + static_cast<size_t>(j) * P2];
        const double2 hx = zmul(h, x);
        const double2 r = make_double2(y.x - hx.x, y.y - hx.y);
        value += wk * znorm(r);
        const double2 z = zmulc(r, x);
        double2 g = make_double2(-2.0 * wk * z.x, 2.0 * wk * z.y);
        const double2 c = zmulc(r, h);
        G.x += c.x;
        G.y += c.y;
        grad_h[base + static_cast<size_t>(j) * P2] = g;
      }
      if (implicit && den > 0.0) {
        const double gx = G.x * x.x - G.y * x.y;  // Re(G X)
        for (int j = 0; j < K; ++j) {
          const size_t e = base + static_cast<size_t>(j) * P2;
          const double2 h = H[e], gy = zmul(G, Y[e]);
          double2 g = grad_h[e];
          g.x += -2.0 * wk * gy.x / den + 4.0 * wk * gx * h.x / den;
          g.y += -2.0 * wk * gy.y / den + 4.0 * wk * gx * h.y / den;
          grad_h[e] = g;
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) value += __shfl_xor_sync(0xffffffffu, value, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = value;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < kLB / 32; ++w) v += s_red[w];
    part[blockIdx.y * n_parts + blockIdx.x] = v;
  }
}

// per-patch loss = its chunk partials in order; *total = sum over patches in order
__global__ void loss_sum64_kernel(const double* __restrict__ part, int n_parts, int n_patches,
                                  double* __restrict__ per_patch, double* __restrict__ total) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double all = 0.0;
  for (int p = 0; p < n_patches; ++p) {
    double v = 0.0;
    for (int c = 0; c < n_parts; ++c) v += part[p * n_parts + c];
    if (per_patch) per_patch[p] = v;
    all += v;
  }
  if (total) *total = all;
}

// ---- transfer_grad_to_wavefront (aberration.hpp:270-313) -------------------
// Stage 1, one thread per (patch, bin): Nyquist-symmetrised dL/dH (the map is
// self-adjoint, aberration.hpp:287-288) pulled back to (dL/dw1, dL/dw2) of the
// bin, summed over delays.
__global__ void __launch_bounds__(kLB) tgw64_bins_kernel(BinTab64 t, const double* __restrict__ w_all,
                                                         const double* __restrict__ delays, int K,
                                                         const double2* __restrict__ grad_h,
                                                         double2* __restrict__ G) {
  const int P2 = t.P2, b = blockIdx.x * kLB + threadIdx.x, patch = blockIdx.y;
  if (b >= P2) return;
  const double k = t.kmag[b];
  double g1 = 0.0, g2 = 0.0;
  if (k != 0.0) {
    const double* w = w_all + static_cast<size_t>(patch) * t.A;
    const int4 ix = t.idx[b];
    const double2 fr = t.frac[b];
    const double w1 = (1 - fr.x) * w[ix.x] + fr.x * w[ix.y];
    const double w2 = (1 - fr.y) * w[ix.z] + fr.y * w[ix.w];
    const int m = t.mirror[b];
    const double2* g = grad_h + static_cast<size_t>(patch) * K * P2;
    for (int j = 0; j < K; ++j) {
      double2 gb = g[static_cast<size_t>(j) * P2 + b];
      if (m >= 0) {  // conj_symmetrize_nyquist: (g_b + conj g_m) / 2
        const double2 gm = g[static_cast<size_t>(j) * P2 + m];
        gb = make_double2(0.5 * (gb.x + gm.x), 0.5 * (gb.y - gm.y));
      }
      if (gb.x == 0.0 && gb.y == 0.0) continue;
      double s1, c1, s2, c2;
      sincos(-k * (delays[j] - w1), &s1, &c1);
      sincos(+k * (delays[j] - w2), &s2, &c2);
      const double2 e1 = make_double2(0.5 * c1, 0.5 * s1), e2 = make_double2(0.5 * c2, 0.5 * s2);
      g1 += k * (gb.x * -e1.y + gb.y * e1.x);
      g2 += k * (gb.x * e2.y + gb.y * -e2.x);
    }
  }
  G[static_cast<size_t>(patch) * P2 + b] = make_double2(g1, g2);
}

// Stage 2, one thread per (patch, angle): gather through the CSR table.
__global__ void tgw64_angles_kernel(BinTab64 t, const double2* __restrict__ G, int n_patches,
                                    double* __restrict__ dw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_patches * t.A) return;
  const int patch = i / t.A, a = i - patch * t.A;
  const double2* g = G + static_cast<size_t>(patch) * t.P2;
  double acc = 0.0;
  for (int e = t.csr_start[a]; e < t.csr_start[a + 1]; ++e) {
    const int key = t.csr_key[e], b = key >> 2, which = key & 3;
    const double2 fr = t.frac[b];
    const double wt = which == 0 ? 1.0 - fr.x : which == 1 ? fr.x : which == 2 ? 1.0 - fr.y : fr.y;
    acc += wt * (which < 2 ? g[b].x : g[b].y);
  }
  dw[i] = acc;
}

// ---- wavefront_profile(with_jacobian = true) (aberration.hpp:134-186) ------
// One thread per (patch, angle), the reference's quadrature in fp64: the
// clamped bilinear stencil of every midpoint (detail::bilinear_stencil,
// aberration.hpp:49-72) and, per in-mask corner pixel, dw/dv = dl v0 / v^2
// * weight.  COUNT: only the row lengths; otherwise rows are written at
// row_start (ascending step, then corner: the reference's push_back order).
struct JacArgs {
  const float* dv;  // v - v0 [H][W]
  int W, H;
  double ox, oy, pitch, v0, ring_r, mcx, mcy, mr, step;
  int n_angles, n_rays;
  const double2* centers;
};

template <bool COUNT>
__global__ void jacobian64_kernel(JacArgs g, double* __restrict__ w_out, int64_t* __restrict__ row_len,
                                  const int64_t* __restrict__ row_start, int* __restrict__ pixel,
                                  float* __restrict__ dwdv) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= g.n_rays) return;
  const int patch = r / g.n_angles, a = r - patch * g.n_angles;
  const double2 c = g.centers[patch];
  const Ray ray = make_ray(c.x, c.y, a, g.n_angles, g.ring_r, g.mcx, g.mcy, g.mr, g.step);
  int64_t cnt = 0, pos = COUNT ? 0 : row_start[r];
  double acc = 0.0;
  for (int i = 0; i < ray.n; ++i) {
    const double s = ray.t0 + (i + 0.5) * ray.dl;
    const double px = c.x + ray.ux * s, py = c.y + ray.uy * s;
    double fx = (px - g.ox) / g.pitch, fy = (py - g.oy) / g.pitch;
    fx = fmin(fmax(fx, 0.0), static_cast<double>(g.W - 1));
    fy = fmin(fmax(fy, 0.0), static_cast<double>(g.H - 1));
    const int ix = min(static_cast<int>(fx), max(g.W - 2, 0));
    const int iy = min(static_cast<int>(fy), max(g.H - 2, 0));
    const double ax = fx - ix, ay = fy - iy;
    const int ix1 = min(ix + 1, g.W - 1), iy1 = min(iy + 1, g.H - 1);
    const int idx[4] = {iy * g.W + ix, iy * g.W + ix1, iy1 * g.W + ix, iy1 * g.W + ix1};
    const double wt[4] = {(1 - ax) * (1 - ay), ax * (1 - ay), (1 - ax) * ay, ax * ay};
    const double v = wt[0] * (g.v0 + g.dv[idx[0]]) + wt[1] * (g.v0 + g.dv[idx[1]]) +
                     wt[2] * (g.v0 + g.dv[idx[2]]) + wt[3] * (g.v0 + g.dv[idx[3]]);
    acc += ray.dl * (1.0 - g.v0 / v);
    const double f = ray.dl * g.v0 / (v * v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int q = idx[k];
      const double wx = g.ox + (q % g.W) * g.pitch, wy = g.oy + (q / g.W) * g.pitch;
      if (!(hypot(wx - g.mcx, wy - g.mcy) <= g.mr)) continue;  // CircularMask::contains
      if (!COUNT) {
        pixel[pos] = q;
        dwdv[pos] = static_cast<float>(f * wt[k]);
        ++pos;
      }
      ++cnt;
    }
  }
  if (COUNT) {
    row_len[r] = cnt;
  } else if (w_out) {
    w_out[r] = acc;
  }
}

// Exclusive scan of n row lengths into row_start[0..n] (one block; the row
// count is patches x angles, so a sequential pass per thread tile is enough).
__global__ void __launch_bounds__(1024) scan64_kernel(const int64_t* __restrict__ len, int n,
                                                      int64_t* __restrict__ start) {
  __shared__ int64_t s_sum[1024];
  const int per = (n + 1023) / 1024, lo = threadIdx.x * per, hi = min(n, lo + per);
  int64_t sum = 0;
  for (int i = lo; i < hi; ++i) sum += len[i];
  s_sum[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int t = 0; t < 1024; ++t) {
      const int64_t v = s_sum[t];
      s_sum[t] = run;
      run += v;
    }
    start[n] = run;
  }
  __syncthreads();
  int64_t run = s_sum[threadIdx.x];
  for (int i = lo; i < hi; ++i) {
    start[i] = run;
    run += len[i];
  }
}

// ---- accumulate_wavefront_grad (aberration.hpp:316-326) --------------------
__global__ void accumulate_jt64_kernel(int64_t n_rows, const int64_t* __restrict__ row_start,
                                       const int* __restrict__ pixel, const float* __restrict__ dwdv,
                                       const double* __restrict__ dw, double* __restrict__ grad_v) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const double g = dw[r];
  if (g == 0.0) return;
  for (int64_t e = row_start[r]; e < row_start[r + 1]; ++e)
    atomicAdd(grad_v + pixel[e], g * static_cast<double>(dwdv[e]));
}

// ---- psf_from_transfer (aberration.hpp:407-445), batched, fp64 ----------
// Stats per spectrum (atomicMax on the bit patterns of non-negative doubles,
// which order like unsigned integers): [max |S|, max asymmetry, max |Re|, max |Im|].
__device__ __forceinline__ void dmax(double* p, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(__double_as_longlong(v)));
}

// pass 1, one thread per (spectrum, bin): symmetry statistics, and the row
// transform R[y][x] = sum_k S[y][k] e^{+2 pi i k x / P} (fft::inverse_2d
// transforms rows first, fft.hpp:107-115)
__global__ void psf_rows64_kernel(const double2* __restrict__ S, int P, double2* __restrict__ R,
                                  double* __restrict__ stats) {
  const int P2 = P * P, e = blockIdx.x * blockDim.x + threadIdx.x, n = blockIdx.y;
  if (e >= P2) return;
  const int y = e / P, x = e - y * P;
  const double2* s = S + static_cast<size_t>(n) * P2;
  const double2 a = s[e], b = s[((P - y) % P) * P + (P - x) % P];
  dmax(stats + 4 * n, hypot(a.x, a.y));
  dmax(stats + 4 * n + 1, hypot(a.x - b.x, a.y + b.y));  // |S_i - conj(S_j)|
  double re = 0.0, im = 0.0;
  for (int k = 0; k < P; ++k) {
    double sn, cs;
    sincospi(2.0 * ((k * x) % P) / P, &sn, &cs);
    const double2 v = s[y * P + k];
    re += v.x * cs - v.y * sn;
    im += v.x * sn + v.y * cs;
  }
  R[static_cast<size_t>(n) * P2 + e] = make_double2(re, im);
}

// pass 2: the column transform, the 1 / P^2 scale, the residue statistics and
// the centred placement psf[(y + P/2) % P][(x + P/2) % P] = Re
__global__ void psf_cols64_kernel(const double2* __restrict__ R, int P, double* __restrict__ psf,
                                  double* __restrict__ stats) {
  const int P2 = P * P, e = blockIdx.x * blockDim.x + threadIdx.x, n = blockIdx.y;
  if (e >= P2) return;
  const int y = e / P, x = e - y * P;
  const double2* r = R + static_cast<size_t>(n) * P2;
  double re = 0.0, im = 0.0;
  for (int k = 0; k < P; ++k) {
    double sn, cs;
    sincospi(2.0 * ((k * y) % P) / P, &sn, &cs);
    const double2 v = r[k * P + x];
    re += v.x * cs - v.y * sn;
    im += v.x * sn + v.y * cs;
  }
  const double inv = 1.0 / (static_cast<double>(P) * P);
  re *= inv;
  im *= inv;
  dmax(stats + 4 * n + 2, fabs(re));
  dmax(stats + 4 * n + 3, fabs(im));
  psf[static_cast<size_t>(n) * P2 + ((y + P / 2) % P) * P + (x + P / 2) % P] = re;
}

}  // namespace
}  // namespace pactgpu

using namespace pactgpu;

namespace {

Status upload_small(pact_ctx* ctx, int slot, const void* host, size_t bytes, void** dev) {
  PACT_TRY_S(scratch_get(ctx, slot, bytes, dev));
  return cuda_status(cudaMemcpyAsync(*dev, host, bytes, cudaMemcpyHostToDevice, ctx->stream),
                     "cudaMemcpyAsync");
}

}  // namespace

extern "C" int pact_multichannel_deconvolve(pact_ctx* ctx, int32_t n_patches, int32_t K, int32_t P,
                                            const double* Y, const double* H, double eps,
                                            double* X) {
  if (!ctx || !Y || !H || !X) return validation("pact_multichannel_deconvolve: null argument").code;
  if (K < 1) return validation("deconvolve: no channels").code;
  if (n_patches < 1 || P < 1) return validation("pact_multichannel_deconvolve: empty input").code;
  const int P2 = P * P;
  deconvolve64_kernel<<<dim3(div_up(P2, 256), n_patches), 256, 0, ctx->stream>>>(
      reinterpret_cast<const double2*>(Y), reinterpret_cast<const double2*>(H), K, P2,
      eps * K, reinterpret_cast<double2*>(X));
  PACT_TRY(after_launch(ctx, "deconvolve64_kernel"));
  return PACT_OK;
}

extern "C" int pact_deconv_jacobian_H(pact_ctx* ctx, int32_t K, int32_t P, const double* Y,
                                      const double* H, double eps, int32_t n_queries,
                                      const int32_t* queries, double* out) {
  if (!ctx || !Y || !H || !queries || !out)
    return validation("pact_deconv_jacobian_H: null argument").code;
  if (K < 1 || P < 1 || n_queries < 0) return validation("pact_deconv_jacobian_H: empty input").code;
  if (n_queries == 0) return PACT_OK;
  deconv_jacobian64_kernel<<<div_up(n_queries, 128), 128, 0, ctx->stream>>>(
      reinterpret_cast<const double2*>(Y), reinterpret_cast<const double2*>(H), K, P * P, eps * K,
      queries, n_queries, reinterpret_cast<double2*>(out));
  PACT_TRY(after_launch(ctx, "deconv_jacobian64_kernel"));
  return PACT_OK;
}

namespace {

Status launch_patch_loss(pact_ctx* ctx, int n_patches, int K, int P, double pitch,
                         const double* Y, const double* H, double eps, double scale, int implicit,
                         double* loss_per_patch, double* total, double* grad_h) {
  if (K < 1) return validation("data_loss: no channels");
  if (n_patches < 1) return validation("data_loss: no patches");
  if (P < 1 || !(pitch > 0.0)) return validation("data_loss: bad patch geometry");
  BinTab64 t;
  PACT_TRY_S(bin_table(ctx, P, pitch, 0, t));
  const int n_parts = div_up(P * P, kLB);
  void* part = nullptr;
  PACT_TRY_S(scratch_get(ctx, kScratchGeneric2, sizeof(double) * (n_parts * n_patches + 1), &part));
  patch_loss64_kernel<<<dim3(n_parts, n_patches), kLB, 0, ctx->stream>>>(
      t, reinterpret_cast<const double2*>(Y), reinterpret_cast<const double2*>(H), K, eps * K, scale,
      implicit, reinterpret_cast<double2*>(grad_h), static_cast<double*>(part), n_parts);
  PACT_TRY_S(after_launch(ctx, "patch_loss64_kernel"));
  double* dtotal = static_cast<double*>(part) + n_parts * n_patches;
  loss_sum64_kernel<<<1, 32, 0, ctx->stream>>>(static_cast<double*>(part), n_parts, n_patches,
                                               loss_per_patch, dtotal);
  PACT_TRY_S(after_launch(ctx, "loss_sum64_kernel"));
  if (total) {
    PACT_CUDA_S(cudaMemcpyAsync(total, dtotal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    PACT_CUDA_S(cudaStreamSynchronize(ctx->stream));
  }
  return {};
}

}  // namespace

extern "C" int pact_patch_data_loss(pact_ctx* ctx, int32_t n_patches, int32_t K, int32_t P,
                                    double pitch, const double* Y, const double* H, double eps,
                                    double scale, int32_t implicit, double* loss_per_patch,
                                    double* grad_h) {
  if (!ctx || !Y || !H || !loss_per_patch || !grad_h)
    return validation("pact_patch_data_loss: null argument").code;
  PACT_TRY(launch_patch_loss(ctx, n_patches, K, P, pitch, Y, H, eps, scale, implicit,
                             loss_per_patch, nullptr, grad_h));
  return PACT_OK;
}

extern "C" int pact_data_loss(pact_ctx* ctx, int32_t n_patches, int32_t K, int32_t P, double pitch,
                              const double* Y, const double* H, double eps, int32_t implicit,
                              double* value, double* loss_per_patch, double* grad_h) {
  if (!ctx || !Y || !H || !value || !grad_h) return validation("pact_data_loss: null argument").code;
  if (n_patches < 1) return validation("data_loss: no patches").code;
  if (K < 1) return validation("data_loss: no channels").code;
  if (P < 1) return validation("data_loss: bad patch geometry").code;
  // normalised by N * M * P^2 (optimize.hpp:342)
  const double scale = 1.0 / (static_cast<double>(n_patches) * K * P * P);
  PACT_TRY(launch_patch_loss(ctx, n_patches, K, P, pitch, Y, H, eps, scale, implicit,
                             loss_per_patch, value, grad_h));
  return PACT_OK;
}

extern "C" int pact_transfer_grad_to_wavefront(pact_ctx* ctx, int32_t n_patches, const double* w,
                                               int32_t n_angles, const double* delays, int32_t K,
                                               int32_t P, double pitch, const double* grad_h,
                                               double* dw) {
  if (!ctx || !w || !grad_h || !dw || (!delays && K > 0))
    return validation("pact_transfer_grad_to_wavefront: null argument").code;
  if (n_patches < 1 || n_angles < 1 || K < 1 || P < 1 || !(pitch > 0.0))
    return validation("pact_transfer_grad_to_wavefront: empty input").code;
  BinTab64 t;
  PACT_TRY(bin_table(ctx, P, pitch, n_angles, t));
  void* dd = nullptr;
  PACT_TRY(upload_small(ctx, kScratchGeneric3, delays, sizeof(double) * K, &dd));
  void* G = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric2, sizeof(double2) * n_patches * P * P, &G));
  tgw64_bins_kernel<<<dim3(div_up(P * P, kLB), n_patches), kLB, 0, ctx->stream>>>(
      t, w, static_cast<const double*>(dd), K, reinterpret_cast<const double2*>(grad_h),
      static_cast<double2*>(G));
  PACT_TRY(after_launch(ctx, "tgw64_bins_kernel"));
  tgw64_angles_kernel<<<div_up(n_patches * n_angles, 128), 128, 0, ctx->stream>>>(
      t, static_cast<const double2*>(G), n_patches, dw);
  PACT_TRY(after_launch(ctx, "tgw64_angles_kernel"));
  return PACT_OK;
}

extern "C" int pact_wavefront_jacobian(pact_ctx* ctx, const pact_ring* ring, const pact_grid* grid,
                                       const float* sos_dev, double v0, const pact_mask* mask,
                                       int32_t n_centers, const double* centers, int32_t n_angles,
                                       double step, double* w, int64_t* row_start, int32_t* pixel,
                                       float* dw_dv, int64_t capacity, int64_t* n_entries) {
  if (!ctx || !ring || !grid || !sos_dev || !mask || !centers || !row_start || !n_entries)
    return validation("pact_wavefront_jacobian: null argument").code;
  // wavefront_profile's validation (aberration.hpp:138-142)
  if (ring->n_transducers < 1) return validation("ring: need at least one transducer").code;
  if (!(ring->radius > 0.0)) return validation("ring: radius must be > 0").code;
  if (n_angles < 4) return validation("wavefront_profile: need at least 4 angles").code;
  if (!(step > 0.0)) return validation("wavefront_profile: step must be > 0").code;
  for (int i = 0; i < n_centers; ++i)
    if (std::hypot(centers[2 * i], centers[2 * i + 1]) >= ring->radius)
      return validation("wavefront_profile: patch center outside the transducer ring").code;
  if (n_centers < 1) return validation("pact_wavefront_jacobian: no centers").code;
  const int n_rays = n_centers * n_angles;
  void* dc = nullptr;
  PACT_TRY(upload_small(ctx, kScratchGeneric3, centers, sizeof(double) * 2 * n_centers, &dc));
  void* len = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric2, sizeof(int64_t) * n_rays, &len));
  JacArgs a{sos_dev, grid->width, grid->height, grid->origin_x, grid->origin_y, grid->pitch,
            v0, ring->radius, mask->center_x, mask->center_y, mask->radius, step, n_angles,
            n_rays, static_cast<const double2*>(dc)};
  const int nb = div_up(n_rays, 128);
  jacobian64_kernel<true><<<nb, 128, 0, ctx->stream>>>(a, nullptr, static_cast<int64_t*>(len),
                                                       nullptr, nullptr, nullptr);
  PACT_TRY(after_launch(ctx, "jacobian64_kernel<count>"));
  scan64_kernel<<<1, 1024, 0, ctx->stream>>>(static_cast<const int64_t*>(len), n_rays, row_start);
  PACT_TRY(after_launch(ctx, "scan64_kernel"));
  PACT_CUDA(cudaMemcpyAsync(n_entries, row_start + n_rays, sizeof(int64_t), cudaMemcpyDeviceToHost,
                            ctx->stream));
  PACT_CUDA(cudaStreamSynchronize(ctx->stream));
  if (!pixel || !dw_dv) return PACT_OK;  // sizing call: row_start and *n_entries only
  if (capacity < *n_entries) return validation("pact_wavefront_jacobian: entry buffers too small").code;
  jacobian64_kernel<false><<<nb, 128, 0, ctx->stream>>>(a, w, nullptr, row_start, pixel, dw_dv);
  PACT_TRY(after_launch(ctx, "jacobian64_kernel<fill>"));
  return PACT_OK;
}

extern "C" int pact_accumulate_wavefront_grad(pact_ctx* ctx, int64_t n_rows,
                                              const int64_t* row_start, const int32_t* pixel,
                                              const float* dw_dv, const double* dw,
                                              double* grad_v) {
  if (!ctx || !row_start || !dw || !grad_v)
    return validation("pact_accumulate_wavefront_grad: null argument").code;
  if (n_rows < 1) return PACT_OK;
  accumulate_jt64_kernel<<<static_cast<unsigned>((n_rows + 255) / 256), 256, 0, ctx->stream>>>(
      n_rows, row_start, pixel, dw_dv, dw, grad_v);
  PACT_TRY(after_launch(ctx, "accumulate_jt64_kernel"));
  return PACT_OK;
}

extern "C" int pact_psf_from_transfer(pact_ctx* ctx, int32_t n_spectra, int32_t P,
                                      const double* spectra, double* psf) {
  if (!ctx || !spectra || !psf) return validation("pact_psf_from_transfer: null argument").code;
  if (P < 1 || n_spectra < 0) return validation("psf_from_transfer: spectrum size mismatch").code;
  if (n_spectra == 0) return PACT_OK;
  const int P2 = P * P;
  void* st = nullptr;
  void* R = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric3, sizeof(double) * 4 * n_spectra, &st));
  PACT_TRY(scratch_get(ctx, kScratchGeneric2, sizeof(double2) * static_cast<size_t>(n_spectra) * P2,
                       &R));
  PACT_CUDA(cudaMemsetAsync(st, 0, sizeof(double) * 4 * n_spectra, ctx->stream));
  const dim3 g(div_up(P2, 128), n_spectra);
  psf_rows64_kernel<<<g, 128, 0, ctx->stream>>>(reinterpret_cast<const double2*>(spectra), P,
                                                static_cast<double2*>(R), static_cast<double*>(st));
  PACT_TRY(after_launch(ctx, "psf_rows64_kernel"));
  psf_cols64_kernel<<<g, 128, 0, ctx->stream>>>(static_cast<const double2*>(R), P, psf,
                                                static_cast<double*>(st));
  PACT_TRY(after_launch(ctx, "psf_cols64_kernel"));
  std::vector<double> h(4 * static_cast<size_t>(n_spectra));
  PACT_CUDA(cudaMemcpyAsync(h.data(), st, sizeof(double) * h.size(), cudaMemcpyDeviceToHost,
                            ctx->stream));
  PACT_CUDA(cudaStreamSynchronize(ctx->stream));
  // the reference's checks and messages, spectrum by spectrum in order
  for (int i = 0; i < n_spectra; ++i) {
    const double max_mag = h[4 * i], asym = h[4 * i + 1], max_real = h[4 * i + 2],
                 max_imag = h[4 * i + 3];
    if (asym > 1e-9 * std::max(1.0, max_mag)) {
      set_error("psf_from_transfer: spectrum not conjugate-symmetric, max asymmetry %f", asym);
      return PACT_E_VALIDATION;
    }
    if (max_real > 0.0 && max_imag > 1e-9 * max_real) {
      set_error("psf_from_transfer: imaginary residue %f exceeds 1e-9 of max %f", max_imag, max_real);
      return PACT_E_NUMERICAL;
    }
  }
  return PACT_OK;
}
