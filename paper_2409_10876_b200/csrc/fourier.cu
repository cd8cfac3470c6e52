// Part 2/3 Fourier-domain kernels: transfer stacks H_j(k) from the wavefront
// profiles, the fused |k|-weighted multichannel loss with its gradient pulled
// back to dL/dw, and the Wiener (pseudo-inverse) deconvolution epilogue.
//
//   transfer_stack                aberration.hpp:236-265
//   conj_symmetrize_nyquist       aberration.hpp:203-218
//   detail::fused_patch_loss_grad optimize.hpp:234-325
//   multichannel_deconvolve       deconv.hpp:78-96
//
// One thread owns one frequency bin of one patch and walks the M delay
// channels (coalesced over bins: Y is [patch][M][P][P]).  Bins on the Nyquist
// row/column (even P) also evaluate their conjugate partner so the reference's
// symmetrisation of H and of dL/dH is reproduced without a second pass.
// dL/dw is accumulated per bin, then gathered per angle through a static CSR
// table (deterministic; no atomics).  The loss is reduced per patch in fp64.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <memory>
#include <mutex>

#include "fourier.cuh"
#include "tc.cuh"

namespace pactgpu {

void fourier_table_free(FourierTable& t) {
  pool_free(t.dev, t.stream);
  t.dev = nullptr;
  t.host.reset();
  t.bytes = 0;
  t.P = 0;
}

namespace {

// Host image of the tables for (P, pitch, A, delays): one byte buffer with
// 16-byte aligned sections.  Cached per process (the tables depend only on
// the layout and the delays), so repeated reconstructions only upload.
struct HostFourier {
  std::vector<char> bytes;
  size_t o_kmag, o_idx, o_frac, o_mirror, o_dp, o_start, o_slot, o_rho;
  int fin_span = 0;
  bool uniform;
};

std::shared_ptr<const HostFourier> build_host_fourier(int P, double pitch, int A,
                                                      const double* delays, int K) {
  const int P2 = P * P;
  const double tau = 2.0 * M_PI;
  std::vector<float> kmag(P2);
  std::vector<int4> idx(P2);
  std::vector<float2> frac(P2);
  std::vector<int> mirror(P2, -1);
  std::vector<float2> dp(static_cast<size_t>(K) * P2);
  // evenly spaced delays (make_delays, beamform.hpp:113-120): phase recurrence
  double dd = K > 1 ? (delays[K - 1] - delays[0]) / (K - 1) : 0.0, dmax = 0.0;
  for (int j = 0; j < K; ++j) dmax = std::max(dmax, std::fabs(delays[j]));
  bool uniform = K > 1;
  for (int j = 0; j < K && uniform; ++j)
    uniform = std::fabs(delays[j] - (delays[0] + j * dd)) <= 1e-12 * (1.0 + dmax);
  std::vector<float2> rho(P2);
  // PatchBinTable::make, aberration.hpp:373-401
  auto interp = [&](double theta, int& i0, int& i1, double& f) {
    double pos = std::fmod(theta, tau);
    if (pos < 0) pos += tau;
    pos = pos / tau * A;
    i0 = static_cast<int>(pos) % A;
    f = pos - std::floor(pos);
    i1 = (i0 + 1) % A;
  };
  const double scale = 2.0 * M_PI / (P * pitch);
  const int half = P / 2;
  for (int by = 0; by < P; ++by)
    for (int bx = 0; bx < P; ++bx) {
      int b = by * P + bx;
      double kx = scale * (bx <= P / 2 ? bx : bx - P);
      double ky = scale * (by <= P / 2 ? by : by - P);
      double k = std::hypot(kx, ky), ang = std::atan2(ky, kx);
      int a0, a1, b0, b1;
      double f1, f2;
      interp(ang, a0, a1, f1);
      interp(ang + M_PI, b0, b1, f2);
      kmag[b] = static_cast<float>(k);
      idx[b] = make_int4(a0, a1, b0, b1);
      frac[b] = make_float2(static_cast<float>(f1), static_cast<float>(f2));
      if (P % 2 == 0 && (bx == half || by == half))
        mirror[b] = ((P - by) % P) * P + (P - bx) % P;
      rho[b] = make_float2(static_cast<float>(std::cos(-k * dd)), static_cast<float>(std::sin(-k * dd)));
      for (int j = 0; j < K; ++j) {
        // make_delay_phases, optimize.hpp:229: polar(1, -|k| d_j)
        double ph = -k * delays[j];
        dp[static_cast<size_t>(j) * P2 + b] =
            make_float2(static_cast<float>(std::cos(ph)), static_cast<float>(std::sin(ph)));
      }
    }
  // the (bin, branch) pairs sorted by lower interpolation angle: the scatter
  // of fused_patch_loss_grad (optimize.hpp:318-321) as contiguous segments
  std::vector<int> start(A + 1, 0);
  for (int b = 0; b < P2; ++b) {
    start[idx[b].x + 1]++;
    start[idx[b].z + 1]++;
  }
  for (int a = 0; a < A; ++a) start[a + 1] += start[a];
  int fin_span = 0;
  for (int a0 = 0; a0 < A; a0 += kFinishAngles)
    fin_span = std::max(fin_span, start[std::min(a0 + kFinishAngles, A)] - start[a0 > 0 ? a0 - 1 : 0]);
  std::vector<int2> slot(P2);
  {
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (int b = 0; b < P2; ++b) {  // ascending bin within an angle
      slot[b].x = fill[idx[b].x]++;
      slot[b].y = fill[idx[b].z]++;
    }
  }
  // one device allocation, 16-byte aligned sections
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  size_t o_kmag = 0, o_idx = al(o_kmag + 4 * P2), o_frac = al(o_idx + 16 * P2),
         o_mirror = al(o_frac + 8 * P2), o_dp = al(o_mirror + 4 * P2),
         o_start = al(o_dp + 8 * static_cast<size_t>(K) * P2), o_slot = al(o_start + 4 * (A + 1)),
         o_rho = al(o_slot + 8 * P2), total = al(o_rho + 8 * P2);
  auto hf = std::make_shared<HostFourier>();
  std::vector<char>& host = hf->bytes;
  host.assign(total, 0);
  std::memcpy(host.data() + o_kmag, kmag.data(), 4 * P2);
  std::memcpy(host.data() + o_idx, idx.data(), 16 * P2);
  std::memcpy(host.data() + o_frac, frac.data(), 8 * P2);
  std::memcpy(host.data() + o_mirror, mirror.data(), 4 * P2);
  std::memcpy(host.data() + o_dp, dp.data(), 8 * dp.size());
  std::memcpy(host.data() + o_start, start.data(), 4 * (A + 1));
  std::memcpy(host.data() + o_slot, slot.data(), 8 * P2);
  std::memcpy(host.data() + o_rho, rho.data(), 8 * P2);
  hf->o_kmag = o_kmag;
  hf->o_idx = o_idx;
  hf->o_frac = o_frac;
  hf->o_mirror = o_mirror;
  hf->o_dp = o_dp;
  hf->o_start = o_start;
  hf->o_slot = o_slot;
  hf->o_rho = o_rho;
  hf->uniform = uniform;
  hf->fin_span = fin_span;
  return hf;
}

std::shared_ptr<const HostFourier> host_fourier(int P, double pitch, int A, const double* delays,
                                                int K) {
  struct Entry {
    int P, A;
    double pitch;
    std::vector<double> delays;
    std::shared_ptr<const HostFourier> hf;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& e : cache)
      if (e.P == P && e.A == A && e.pitch == pitch && static_cast<int>(e.delays.size()) == K &&
          std::equal(e.delays.begin(), e.delays.end(), delays))
        return e.hf;
  }
  auto hf = build_host_fourier(P, pitch, A, delays, K);
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() >= 4) cache.erase(cache.begin());
  cache.push_back({P, A, pitch, std::vector<double>(delays, delays + K), hf});
  return hf;
}

}  // namespace

Status fourier_table(pact_ctx* ctx, FourierTable& t, int P, double pitch, int A,
                     const double* delays, int K) {
  if (t.dev && t.P == P && t.pitch == pitch && t.A == A && t.K == K &&
      std::equal(t.delays.begin(), t.delays.end(), delays))
    return {};
  const auto hf = host_fourier(P, pitch, A, delays, K);
  const size_t total = hf->bytes.size();
  const int P2 = P * P;
  if (t.dev && t.bytes < total) fourier_table_free(t);
  if (!t.dev) {
    PACT_TRY_S(pool_alloc(&t.dev, total, ctx->stream));
    t.stream = ctx->stream;
    t.bytes = total;
  }
  // the cached host image outlives the copy (held by the cache and by `t`)
  PACT_CUDA_S(cudaMemcpyAsync(t.dev, hf->bytes.data(), total, cudaMemcpyHostToDevice,
                              ctx->stream));
  t.host = hf;
  char* d = static_cast<char*>(t.dev);
  t.P = P;
  t.A = A;
  t.K = K;
  t.pitch = pitch;
  t.delays.assign(delays, delays + K);
  t.tab.P = P;
  t.tab.P2 = P2;
  t.tab.A = A;
  t.tab.K = K;
  t.tab.kmag = reinterpret_cast<const float*>(d + hf->o_kmag);
  t.tab.idx = reinterpret_cast<const int4*>(d + hf->o_idx);
  t.tab.frac = reinterpret_cast<const float2*>(d + hf->o_frac);
  t.tab.mirror = reinterpret_cast<const int*>(d + hf->o_mirror);
  t.tab.dp = reinterpret_cast<const float2*>(d + hf->o_dp);
  t.tab.sstart = reinterpret_cast<const int*>(d + hf->o_start);
  t.tab.slot = reinterpret_cast<const int2*>(d + hf->o_slot);
  t.tab.rho = hf->uniform ? reinterpret_cast<const float2*>(d + hf->o_rho) : nullptr;
  t.tab.fin_span = hf->fin_span;
  return {};
}

namespace {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // conj(a) * b
  return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// e1 = exp(+i|k| w(angle)), e2 = exp(-i|k| w(angle + pi)) for bin b
// (optimize.hpp:261-265), w interpolated from the patch profile in smem.
__device__ __forceinline__ void bin_phases(const FourierTab& t, const float* __restrict__ w, int b,
                                           float2& e1, float2& e2) {
  float k = t.kmag[b];
  int4 ix = t.idx[b];
  float2 fr = t.frac[b];
  float w1 = (1.f - fr.x) * w[ix.x] + fr.x * w[ix.y];
  float w2 = (1.f - fr.y) * w[ix.z] + fr.y * w[ix.w];
  float s, c;
  sincosf(k * w1, &s, &c);
  e1 = make_float2(c, s);
  sincosf(k * w2, &s, &c);
  e2 = make_float2(c, -s);
}

// h_j = 1/2 (dp_j e1 + conj(dp_j) e2)   (optimize.hpp:270-271)
__device__ __forceinline__ float2 h_of(float2 dp, float2 e1, float2 e2) {
  float2 a = cmul(dp, e1), b = cmul(conjf2(dp), e2);
  return make_float2(0.5f * (a.x + b.x), 0.5f * (a.y + b.y));
}

// Symmetrised H_j at bin b (partner m = -1 for ordinary bins).
__device__ __forceinline__ float2 h_sym(const FourierTab& t, int j, int b, int m, float2 e1b,
                                        float2 e2b, float2 e1m, float2 e2m) {
  float2 hb = h_of(t.dp[j * t.P2 + b], e1b, e2b);
  if (m < 0) return hb;
  float2 hm = h_of(t.dp[j * t.P2 + m], e1m, e2m);
  return make_float2(0.5f * (hb.x + hm.x), 0.5f * (hb.y - hm.y));  // (h_b + conj h_m)/2
}

__global__ void transfer_stack_kernel(FourierTab t, const float* __restrict__ w_all, int n_patches,
                                      float2* __restrict__ H) {
  extern __shared__ float s_w[];
  const int patch = blockIdx.y;
  for (int a = threadIdx.x; a < t.A; a += blockDim.x) s_w[a] = w_all[patch * t.A + a];
  __syncthreads();
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= t.P2) return;
  float2 e1b, e2b, e1m = {}, e2m = {};
  bin_phases(t, s_w, b, e1b, e2b);
  int m = t.mirror[b];
  if (m >= 0) bin_phases(t, s_w, m, e1m, e2m);
  float2* out = H + static_cast<size_t>(patch) * t.K * t.P2 + b;
  for (int j = 0; j < t.K; ++j) out[j * t.P2] = h_sym(t, j, b, m, e1b, e2b, e1m, e2m);
}

// (dL/dw1, dL/dw2) of bin b -> the interpolation weights' shares at the
// bin's two sorted slots (FourierTab::slot); u is the patch's [2 P2] block.
__device__ __forceinline__ void put_g(const FourierTab& t, float2* __restrict__ u, int b, float G1,
                                      float G2) {
  const int2 s = t.slot[b];
  const float2 fr = t.frac[b];
  u[s.x] = make_float2((1.f - fr.x) * G1, fr.x * G1);
  u[s.y] = make_float2((1.f - fr.y) * G2, fr.y * G2);
}

// Per-bin state of the loss chain (optimize.hpp:275-311).
struct BinLoss {
  float2 x;    // X-hat
  float den;   // sum |h|^2 + eps M
  float inv;   // 1 / den
  float2 G;    // sum conj(r_j) h_j
  float gx;    // Re(G X)
  float wk;    // |k| * scale
};

// dL/dH_j at bin b before symmetrisation (explicit + implicit terms,
// optimize.hpp:290-311).
__device__ __forceinline__ float2 bin_grad(const BinLoss& L, float2 h, float2 y, bool implicit) {
  float2 hx = cmul(h, L.x);
  float2 r = make_float2(y.x - hx.x, y.y - hx.y);
  float2 z = cmulc(r, L.x);
  float2 g = make_float2(-2.f * L.wk * z.x, 2.f * L.wk * z.y);
  if (implicit && L.den > 0.f) {
    float2 gy = cmul(L.G, y);
    g.x += (-2.f * L.wk * gy.x + 4.f * L.wk * L.gx * h.x) * L.inv;
    g.y += (-2.f * L.wk * gy.y + 4.f * L.wk * L.gx * h.y) * L.inv;
  }
  return g;
}

// dL/dH -> (G1, G2) through t1 = dp e1 / 2, t2 = conj(dp) e2 / 2 (optimize.hpp:314-317)
__device__ __forceinline__ void pullback(float2 g, float2 dp, float2 e1, float2 e2, float k,
                                         float& G1, float& G2) {
  float2 t1 = cmul(dp, e1), t2 = cmul(conjf2(dp), e2);
  G1 += 0.5f * k * (g.x * -t1.y + g.y * t1.x);
  G2 += 0.5f * k * (g.x * t2.y - g.y * t2.x);
}

// Slot of a Nyquist bin (even P) in the per-patch exchange buffer: the
// by == P/2 row (P slots), then the bx == P/2 column without that row (P - 1).
__device__ __forceinline__ int nyq_slot(int b, int P) {
  const int by = b / P, bx = b - by * P, half = P / 2;
  if (by == half) return bx;
  return P + (by < half ? by : by - 1);
}

__device__ __forceinline__ int nyq_bin(int s, int P) {
  const int half = P / 2;
  if (s < P) return half * P + s;
  int by = s - P;
  by = by < half ? by : by + 1;
  return by * P + half;
}

// The per-bin chain of the fused loss (optimize.hpp:275-317) for bin b with
// its K spectra y(j).  SYM: a Nyquist bin (even P) whose H_j is symmetrised
// with its conjugate partner m; its unsymmetrised dL/dH_j go to `nyq_out`
// (the partner's pullback happens in kernel B).  Otherwise (G1, G2) are
// returned.  Returns the bin's weighted residual energy.
template <bool SYM, class YF>
__device__ __forceinline__ double bin_chain(const FourierTab& t, const float* __restrict__ s_w, int b,
                                            int m, float eps_m, float scale, bool impl, YF y_of,
                                            float& G1, float& G2, float2* __restrict__ nyq_out) {
  const int K = t.K, P2 = t.P2;
  G1 = G2 = 0.f;
  BinLoss L;
  L.wk = t.kmag[b] * scale;
  if (L.wk == 0.f) {
    if (SYM)
      for (int j = 0; j < K; ++j) nyq_out[j] = make_float2(0.f, 0.f);
    return 0.0;
  }
  float2 e1b, e2b, e1m = {}, e2m = {};
  bin_phases(t, s_w, b, e1b, e2b);
  if (SYM) bin_phases(t, s_w, m, e1m, e2m);
  // delay phases dp_j at b (and m): the recurrence dp_{j+1} = dp_j rho for
  // evenly spaced delays, table loads otherwise
  const bool walk = t.rho != nullptr;
  const float2 rb = walk ? t.rho[b] : make_float2(1.f, 0.f);
  const float2 rm = SYM && walk ? t.rho[m] : make_float2(1.f, 0.f);
  const float2 db0 = t.dp[b], dm0 = SYM ? t.dp[m] : make_float2(1.f, 0.f);
  auto next = [&](int j, float2& db, float2& dm) {  // phases of delay j + 1
    if (walk) {
      db = cmul(db, rb);
      if (SYM) dm = cmul(dm, rm);
    } else if (j + 1 < K) {
      db = t.dp[(j + 1) * P2 + b];
      if (SYM) dm = t.dp[(j + 1) * P2 + m];
    }
  };
  // h_j = (t1 + t2) / 2, t1 = dp e1, t2 = conj(dp) e2 (optimize.hpp:270-271)
  auto h_at = [&](float2 db, float2 dm, float2& t1, float2& t2) {
    t1 = cmul(db, e1b);
    t2 = cmul(conjf2(db), e2b);
    float2 hb = make_float2(0.5f * (t1.x + t2.x), 0.5f * (t1.y + t2.y));
    if (!SYM) return hb;
    float2 hm = h_of(dm, e1m, e2m);
    return make_float2(0.5f * (hb.x + hm.x), 0.5f * (hb.y - hm.y));  // (h_b + conj h_m)/2
  };
  // pass 1: X-hat = num / den
  float2 num = make_float2(0.f, 0.f);
  float den = eps_m;
  {
    float2 db = db0, dm = dm0;
#pragma unroll 4
    for (int j = 0; j < K; ++j) {
      float2 t1, t2;
      const float2 h = h_at(db, dm, t1, t2);
      const float2 c = cmulc(h, y_of(j));
      num.x += c.x;
      num.y += c.y;
      den += h.x * h.x + h.y * h.y;
      next(j, db, dm);
    }
  }
  L.den = den;
  L.inv = den > 0.f ? 1.f / den : 0.f;
  L.x = make_float2(num.x * L.inv, num.y * L.inv);
  // G = sum_j conj(r_j) h_j = conj(num) - conj(X) sum|h_j|^2 = conj(num) eps M / den
  // (optimize.hpp:287-294; closed form, no cancellation)
  L.G = make_float2(num.x * (eps_m * L.inv), -num.y * (eps_m * L.inv));
  L.gx = L.G.x * L.x.x - L.G.y * L.x.y;
  // pass 2: residuals (the loss) and dL/dH, pulled back through t1, t2
  // (optimize.hpp:296-317)
  const float hk = 0.5f * t.kmag[b];
  float acc = 0.f;
  {
    float2 db = db0, dm = dm0;
#pragma unroll 4
    for (int j = 0; j < K; ++j) {
      float2 t1, t2;
      const float2 h = h_at(db, dm, t1, t2);
      const float2 y = y_of(j);
      const float2 hx = cmul(h, L.x);
      const float2 r = make_float2(y.x - hx.x, y.y - hx.y);
      acc += r.x * r.x + r.y * r.y;
      const float2 g = bin_grad(L, h, y, impl);
      if (SYM) {
        nyq_out[j] = g;
      } else {
        G1 += hk * (g.y * t1.x - g.x * t1.y);
        G2 += hk * (g.x * t2.y - g.y * t2.x);
      }
      next(j, db, dm);
    }
  }
  return static_cast<double>(L.wk) * acc;
}

// Ordinary (non-Nyquist) bins in closed form.  With e1 = exp(+i|k|w1),
// e2 = exp(-i|k|w2) and dp_j = exp(-i|k|d_j) (optimize.hpp:261-271),
//   h_j = (dp_j e1 + conj(dp_j) e2) / 2 = phi c_j,  phi = exp(i|k|(w1 - w2)/2),
//   c_j = cos(|k|(d_j - wbar)) real, wbar = (w1 + w2) / 2.
// |phi| = 1 cancels from the Wiener estimate and every residual:
//   X' = sum_j c_j y_j / (sum_j c_j^2 + eps M),  r_j = y_j - c_j X',
// so the loss needs only c_j, and (with the implicit X' term,
// optimize.hpp:290-311)
//   dL/dc_j = -2 wk [Re(conj(r_j) X') + a Re(conj(X') y_j) - 2 a |X'|^2 c_j],
//   a = eps M / den,   dc_j/dwbar = |k| sin(|k|(d_j - wbar)),
// and w1, w2 each receive half of dL/dwbar.  About a third of the complex
// arithmetic of the general chain; same quantities.
// PAIR: the delays are split between this lane and lane ^ 16 (delays
// [0, K/2) in lanes 0-15, [K/2, K) in lanes 16-31 of the warp); the pass sums
// are combined with one fixed xor-16 shuffle, so both lanes end with the
// bin's values.  Twice the warps per bin chunk, half the dependent chain.
template <bool PAIR = false, class YF>
__device__ __forceinline__ double bin_chain_real(const FourierTab& t, const float* __restrict__ s_w,
                                                 int b, float eps_m, float scale, bool impl,
                                                 YF y_of, float& G) {
  const int P2 = t.P2;
  const int half = PAIR ? (threadIdx.x >> 4) & 1 : 0;
  const int j0 = PAIR ? half * (t.K / 2) : 0, j1 = PAIR ? (half ? t.K : t.K / 2) : t.K;
  auto pair_sum = [&](float v) {
    return PAIR ? v + __shfl_xor_sync(0xffffffffu, v, 16) : v;
  };
  G = 0.f;
  const float k = t.kmag[b];
  const float wk = k * scale;
  if (!PAIR && wk == 0.f) return 0.0;  // (paired lanes stay converged for the shuffles)
  const int4 ix = t.idx[b];
  const float2 fr = t.frac[b];
  const float w1 = (1.f - fr.x) * s_w[ix.x] + fr.x * s_w[ix.y];
  const float w2 = (1.f - fr.y) * s_w[ix.z] + fr.y * s_w[ix.w];
  float sn, cs;
  sincosf(k * (0.5f * (w1 + w2)), &sn, &cs);
  const float2 ew = make_float2(cs, -sn);  // exp(-i|k| wbar)
  // z_j = conj(dp_j) exp(-i|k| wbar) = exp(i|k|(d_j - wbar)): c_j = Re z_j, s_j = Im z_j
  const bool walk = t.rho != nullptr;
  const float2 rr = walk ? conjf2(t.rho[b]) : make_float2(1.f, 0.f);
  const float2 z0 = cmul(conjf2(t.dp[j0 * P2 + b]), ew);
  auto next = [&](int j, float2& z) {
    if (walk)
      z = cmul(z, rr);
    else if (j + 1 < j1)
      z = cmul(conjf2(t.dp[(j + 1) * P2 + b]), ew);
  };
  float2 S = make_float2(0.f, 0.f);
  float den = 0.f;
  {
    float2 z = z0;
#pragma unroll 4
    for (int j = j0; j < j1; ++j) {
      const float2 y = y_of(j);
      S.x = fmaf(z.x, y.x, S.x);
      S.y = fmaf(z.x, y.y, S.y);
      den = fmaf(z.x, z.x, den);
      next(j, z);
    }
  }
  S.x = pair_sum(S.x);
  S.y = pair_sum(S.y);
  den = eps_m + pair_sum(den);
  const float inv = den > 0.f ? 1.f / den : 0.f;
  const float2 X = make_float2(S.x * inv, S.y * inv);
  const float al = impl && den > 0.f ? eps_m * inv : 0.f;
  const float be = 2.f * al * (X.x * X.x + X.y * X.y);
  float acc = 0.f, gs = 0.f;
  {
    float2 z = z0;
#pragma unroll 4
    for (int j = j0; j < j1; ++j) {
      const float2 y = y_of(j);
      const float rx = fmaf(-z.x, X.x, y.x), ry = fmaf(-z.x, X.y, y.y);
      acc = fmaf(rx, rx, fmaf(ry, ry, acc));
      const float dc = fmaf(rx, X.x, ry * X.y) + al * fmaf(X.x, y.x, X.y * y.y) - be * z.x;
      gs = fmaf(dc, z.y, gs);
      next(j, z);
    }
  }
  acc = pair_sum(acc);
  gs = pair_sum(gs);
  if (wk == 0.f) return 0.0;
  G = -wk * k * gs;  // = (1/2) dL/dwbar, for w1 and for w2
  return static_cast<double>(wk) * acc;
}

__device__ __forceinline__ void block_sum_store(double value, double* s_red, double* out) {
  for (int o = 16; o > 0; o >>= 1) value += __shfl_xor_sync(0xffffffffu, value, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = value;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) v += s_red[q];
    *out = v;
  }
}

// Kernel A of the fused loss: ordinary bins, one thread per (patch, bin),
// grid (patch, bin chunk of LB).  The chunk's K spectra are staged in shared
// memory with coalesced 16-B loads ([j][bin], conflict free), so the passes
// over the delays are rolled loops.  Nyquist bins are skipped here (their
// lanes idle) and handled by kernel A'.
constexpr int LB = 128;

// Persistent, two-stage pipelined form (P^2 a multiple of LB): each CTA walks
// the (patch, bin chunk) work list with stride gridDim.x; while it computes a
// chunk, the next chunk's K rows of LB spectra (1 KB each) and its patch's
// wavefront profile arrive by cp.async.bulk into the other stage.  The loss
// partial of every chunk goes to its fixed slot (deterministic).
__global__ void __launch_bounds__(2 * LB) loss_bins_kernel(FourierTab t, const float2* __restrict__ Y_all,
                                                       const float* __restrict__ w_all, float eps_m,
                                                       float scale, int implicit,
                                                       float2* __restrict__ gbuf,
                                                       double* __restrict__ loss_part, int n_parts,
                                                       int n_patches) {
  extern __shared__ __align__(16) float smem[];
  const int K = t.K, P2 = t.P2, A = t.A;
  const int chunks = P2 / LB, total = n_patches * chunks;
  const int stage_floats = 2 * K * LB + ((A + 3) & ~3);
  __shared__ double s_red[2 * LB / 32];
  __shared__ __align__(8) uint64_t bar[2];
  // 2 LB threads: warp w, lane l -> bin w * 16 + (l & 15) of the chunk, delay
  // half l >> 4 (conflict-free 8-B smem rows per half-warp)
  const int bl = (threadIdx.x >> 5) * 16 + (threadIdx.x & 15);
  const bool lead = (threadIdx.x & 16) == 0;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int c, int st) {  // thread 0 arms, threads < K + 1 copy
    const int patch = c / chunks, b0 = (c - patch * chunks) * LB;
    float* base = smem + st * stage_floats;
    tc::fence_proxy_async();  // the stage's generic reads (before the barrier) vs the async refill
    if (threadIdx.x == 0)
      tc::mbar_expect_tx(&bar[st], static_cast<uint32_t>(K * LB * 8 + A * 4));
    __syncwarp();
    for (int j = threadIdx.x; j <= K; j += 32) {
      if (j < K)
        tc::bulk_load(base + 2 * j * LB, Y_all + (static_cast<size_t>(patch) * K + j) * P2 + b0,
                      LB * 8, &bar[st]);
      else
        tc::bulk_load(base + 2 * K * LB, w_all + static_cast<size_t>(patch) * A, A * 4, &bar[st]);
    }
  };
  int i = 0;
  if (threadIdx.x < 32 && blockIdx.x < total) issue(blockIdx.x, 0);
  for (int c = blockIdx.x; c < total; c += gridDim.x, ++i) {
    const int st = i & 1;
    if (threadIdx.x < 32 && c + static_cast<int>(gridDim.x) < total) issue(c + gridDim.x, st ^ 1);
    tc::mbar_wait(&bar[st], (i >> 1) & 1);
    const float* base = smem + st * stage_floats;
    const float2* s_y = reinterpret_cast<const float2*>(base);
    const float* s_w = base + 2 * K * LB;
    const int patch = c / chunks, cb = c - patch * chunks;
    const int b = cb * LB + bl;
    // every lane runs the chain (the pair shuffles need the whole warp); the
    // Nyquist bins' lanes (kernel A') discard their result
    const bool ordinary = t.mirror[b] < 0;
    float G;
    const float2* yb = s_y + bl;
    double value = bin_chain_real<true>(t, s_w, b, eps_m, scale, implicit != 0,
                                        [&](int j) { return yb[j * LB]; }, G);
    if (ordinary && lead) put_g(t, gbuf + static_cast<size_t>(patch) * 2 * P2, b, G, G);
    if (!ordinary || !lead) value = 0.0;
    block_sum_store(value, s_red, loss_part + patch * n_parts + cb);
    __syncthreads();  // stage st is free for chunk i + 2; s_red is reusable
  }
}

// Register form of kernel A (K = NS * JPL): NS lanes share a bin, each holding
// JPL of its K spectra in registers, loaded straight from HBM with streaming
// loads (no shared-memory stage, so occupancy is set by registers only and
// every warp keeps JPL 128-B loads in flight).  Lane l of a warp: bin
// l % (32 / NS), delay group l / (32 / NS); a group's lanes read consecutive
// bins of one delay row (coalesced 128-B lines).  The per-bin chain is
// bin_chain_real's closed form with the group sums combined by fixed xor
// shuffles.  Nyquist bins' lanes idle; for even P the Nyquist pairs run in
// the blocks past the ordinary chunks (nyq_pairs).
//
// Even P: half spectrum.  The patch stack is real, so Y(-k) = conj(Y(k)); with
// H(-k) = conj(H(k)) (transfer_stack, aberration.hpp:236-265) the bin -k has
// the same c_j, conj(X'), conj(r_j), the same loss term and the same (1/2)
// dL/dwbar as k, at the same two wavefront stencils (angle(k) and
// angle(k) + pi swap).  Kernel A therefore reads only rows 0 .. P/2 of each
// spectrum: every ordinary bin k there (row 0: 0 < bx < P/2) counts twice in
// the loss and writes its shares to its own and to -k's slots; the Nyquist
// pairs run in the blocks past the ordinary chunks (nyq_pairs).  Half of Y's
// HBM traffic.
//
// Nyquist bins (even P) come in conjugate pairs (b, m = -b) -- the Nyquist
// row and column, three of them self-paired -- and the reference symmetrises
// H over each pair (conj_symmetrize_nyquist, aberration.hpp:203-218) and the
// pullback of dL/dH alike (optimize.hpp:306-308).  With Y(m) = conj(Y(b)) the
// pair's unsymmetrised gradients are g and conj(g), so the symmetrised
// gradient is g at b and conj(g) at m (Re g for a self-paired bin): one unit
// of NS lanes evaluates the pair -- no exchange, no second kernel.
template <int NS, int JPL>
__device__ __forceinline__ void nyq_pairs(const FourierTab& t, const float2* __restrict__ Y_all,
                                          const float* __restrict__ w_all, float eps_m, float scale,
                                          bool impl, float2* __restrict__ gbuf, double* s_red,
                                          double* __restrict__ loss_out, int patch, int u0) {
  constexpr int K = NS * JPL;
  const int P = t.P, P2 = t.P2, hp = P / 2;
  const int unit = u0 + static_cast<int>(threadIdx.x) / NS, q = threadIdx.x % NS;
  const bool valid = unit <= P;  // P + 1 pairs
  const int uu = valid ? unit : 0;
  int b, m;
  if (uu <= hp) {  // Nyquist row: (P/2, bx) with (P/2, P - bx)
    b = hp * P + uu;
    m = hp * P + (P - uu) % P;
  } else {  // Nyquist column: (by, P/2) with (P - by, P/2), by < P/2
    const int by = uu - hp - 1;
    b = by * P + hp;
    m = ((P - by) % P) * P + hp;
  }
  const bool self = b == m;
  const float* w = w_all + static_cast<size_t>(patch) * t.A;
  float2 e1b, e2b, e1m, e2m;
  bin_phases(t, w, b, e1b, e2b);
  bin_phases(t, w, m, e1m, e2m);
  const float k = t.kmag[b];
  const int j0 = q * JPL;
  const bool walk = t.rho != nullptr;
  const float2 rb = walk ? t.rho[b] : make_float2(1.f, 0.f);
  const float2 rm = walk ? t.rho[m] : make_float2(1.f, 0.f);
  const float2 db0 = t.dp[j0 * P2 + b], dm0 = t.dp[j0 * P2 + m];
  auto next = [&](int j, float2& db, float2& dm) {
    if (walk) {
      db = cmul(db, rb);
      dm = cmul(dm, rm);
    } else if (j + 1 < K) {
      db = t.dp[(j + 1) * P2 + b];
      dm = t.dp[(j + 1) * P2 + m];
    }
  };
  auto h_sym = [&](float2 db, float2 dm) {  // (h_b + conj h_m) / 2
    const float2 hb = h_of(db, e1b, e2b), hm = h_of(dm, e1m, e2m);
    return make_float2(0.5f * (hb.x + hm.x), 0.5f * (hb.y - hm.y));
  };
  auto usum = [&](float v) {  // the unit's NS consecutive lanes
#pragma unroll
    for (int o = 1; o < NS; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  // (the spectra are read in both passes, not held: registers stay with the
  // ordinary chunks' budget)
  const float2* Y = Y_all + (static_cast<size_t>(patch) * K + j0) * P2 + b;
  float nx = 0.f, ny = 0.f, dd = 0.f;
  {
    float2 db = db0, dm = dm0;
#pragma unroll 4
    for (int u = 0; u < JPL; ++u) {
      const float2 h = h_sym(db, dm);
      const float2 c = cmulc(h, __ldg(Y + static_cast<size_t>(u) * P2));
      nx += c.x;
      ny += c.y;
      dd += h.x * h.x + h.y * h.y;
      next(j0 + u, db, dm);
    }
  }
  BinLoss L;
  L.wk = k * scale;
  L.den = eps_m + usum(dd);
  L.inv = L.den > 0.f ? 1.f / L.den : 0.f;
  const float2 num = make_float2(usum(nx), usum(ny));
  L.x = make_float2(num.x * L.inv, num.y * L.inv);
  L.G = make_float2(num.x * (eps_m * L.inv), -num.y * (eps_m * L.inv));
  L.gx = L.G.x * L.x.x - L.G.y * L.x.y;
  float acc = 0.f, G1b = 0.f, G2b = 0.f, G1m = 0.f, G2m = 0.f;
  {
    float2 db = db0, dm = dm0;
#pragma unroll 4
    for (int u = 0; u < JPL; ++u) {
      const float2 h = h_sym(db, dm), y = __ldg(Y + static_cast<size_t>(u) * P2);
      const float2 hx = cmul(h, L.x);
      const float2 r = make_float2(y.x - hx.x, y.y - hx.y);
      acc += r.x * r.x + r.y * r.y;
      const float2 g = bin_grad(L, h, y, impl);
      pullback(g, db, e1b, e2b, k, G1b, G2b);
      pullback(conjf2(g), dm, e1m, e2m, k, G1m, G2m);
      next(j0 + u, db, dm);
    }
  }
  acc = usum(acc);
  G1b = usum(G1b);
  G2b = usum(G2b);
  G1m = usum(G1m);
  G2m = usum(G2m);
  const bool live = valid && L.wk != 0.f;
  if (self) {  // symmetrised gradient Re g: (pullback(g) + pullback(conj g)) / 2
    G1b = 0.5f * (G1b + G1m);
    G2b = 0.5f * (G2b + G2m);
  }
  if (valid && q == 0) {
    float2* ub = gbuf + static_cast<size_t>(patch) * 2 * P2;
    put_g(t, ub, b, live ? G1b : 0.f, live ? G2b : 0.f);
    if (!self) put_g(t, ub, m, live ? G1m : 0.f, live ? G2m : 0.f);
  }
  const double value = live && q == 0 ? (self ? 1.0 : 2.0) * static_cast<double>(L.wk) * acc : 0.0;
  block_sum_store(value, s_red, loss_out);
}

template <int NS, int JPL>
__global__ void __launch_bounds__(256, 4) loss_reg_kernel(FourierTab t, const float2* __restrict__ Y_all,
                                                       const float* __restrict__ w_all, float eps_m,
                                                       float scale, int implicit,
                                                       float2* __restrict__ gbuf,
                                                       double* __restrict__ loss_part, int n_parts,
                                                       int n_patches) {
  constexpr int BPW = 32 / NS, BPB = 8 * BPW, K = NS * JPL;
  __shared__ double s_red[8];
  const int P2 = t.P2, P = t.P, lane = threadIdx.x & 31;
  const bool half = (P & 1) == 0;
  const int n_bins = half ? (P / 2 + 1) * P : P2;  // bins this kernel reads
  const int grp = lane / BPW, bi = lane - grp * BPW;
  const int chunks = (n_bins + BPB - 1) / BPB;
  // the Nyquist pair blocks first (their chains are the longest), then the chunks
  constexpr int UPB = 256 / NS;
  const int nb = half ? (P + 1 + UPB - 1) / UPB : 0;
  if (static_cast<int>(blockIdx.x) < n_patches * nb) {
    const int patch = blockIdx.x / nb, part = blockIdx.x - patch * nb;
    nyq_pairs<NS, JPL>(t, Y_all, w_all, eps_m, scale, implicit != 0, gbuf, s_red,
                       loss_part + patch * n_parts + chunks + part, patch, part * UPB);
    return;
  }
  const int blk = blockIdx.x - n_patches * nb;
  const int patch = blk / chunks, cb = blk - patch * chunks;
  const int b0 = cb * BPB + (threadIdx.x >> 5) * BPW + bi;
  const bool valid = b0 < n_bins;
  const int b = valid ? b0 : n_bins - 1;
  const int j0 = grp * JPL;
  // the bin's table entries and wavefront samples first (a dependent
  // idx -> w chain of L2 hits), so they are back before the spectra from HBM
  const int m = t.mirror[b];
  const float k = t.kmag[b];
  const int4 ix = t.idx[b];
  const float2 fr = t.frac[b];
  const float* w = w_all + static_cast<size_t>(patch) * t.A;
  const float wa = __ldg(w + ix.x), wb = __ldg(w + ix.y), wc = __ldg(w + ix.z), wd = __ldg(w + ix.w);
  const float2* Y = Y_all + (static_cast<size_t>(patch) * K + j0) * P2 + b;
  float2 y[JPL];
#pragma unroll
  for (int u = 0; u < JPL; ++u) y[u] = __ldcs(Y + static_cast<size_t>(u) * P2);
  auto gsum = [&](float v) {
#pragma unroll
    for (int o = BPW; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  const float wk = k * scale;
  const float w1 = (1.f - fr.x) * wa + fr.x * wb;
  const float w2 = (1.f - fr.y) * wc + fr.y * wd;
  float sn, cs;
  sincosf(k * (0.5f * (w1 + w2)), &sn, &cs);
  const float2 ew = make_float2(cs, -sn);  // exp(-i|k| wbar)
  // z_j = conj(dp_j) exp(-i|k| wbar) = exp(i|k|(d_j - wbar)): c_j = Re z_j, s_j = Im z_j
  const bool walk = t.rho != nullptr;
  const float2 rr = walk ? conjf2(t.rho[b]) : make_float2(1.f, 0.f);
  // the phases are walked twice (pass 1, pass 2) rather than kept: registers
  // hold the spectra only
  const float2 z0 = cmul(conjf2(t.dp[j0 * P2 + b]), ew);
  auto znext = [&](int u, float2 z) {
    return walk ? cmul(z, rr) : cmul(conjf2(t.dp[(j0 + u + 1) * P2 + b]), ew);
  };
  float Sx = 0.f, Sy = 0.f, den = 0.f;
  {
    float2 z = z0;
#pragma unroll
    for (int u = 0; u < JPL; ++u) {
      Sx = fmaf(z.x, y[u].x, Sx);
      Sy = fmaf(z.x, y[u].y, Sy);
      den = fmaf(z.x, z.x, den);
      if (u + 1 < JPL) z = znext(u, z);
    }
  }
  Sx = gsum(Sx);
  Sy = gsum(Sy);
  den = eps_m + gsum(den);
  const float inv = den > 0.f ? 1.f / den : 0.f;
  const float2 X = make_float2(Sx * inv, Sy * inv);
  const float al = implicit && den > 0.f ? eps_m * inv : 0.f;
  const float be = 2.f * al * (X.x * X.x + X.y * X.y);
  const float al1 = 1.f + al, xb = X.x * X.x + X.y * X.y + be;
  float acc = 0.f, gs = 0.f;
  {
    float2 z = z0;
#pragma unroll
    for (int u = 0; u < JPL; ++u) {
      const float rx = fmaf(-z.x, X.x, y[u].x), ry = fmaf(-z.x, X.y, y[u].y);
      acc = fmaf(rx, rx, fmaf(ry, ry, acc));
      // dc = Re(conj(r) X) + al Re(conj(X) y) - be c = (1 + al) (X . y) - (|X|^2 + be) c
      const float q = fmaf(X.x, y[u].x, X.y * y[u].y);
      const float dc = fmaf(al1, q, -xb * z.x);
      gs = fmaf(dc, z.y, gs);
      if (u + 1 < JPL) z = znext(u, z);
    }
  }
  acc = gsum(acc);
  gs = gsum(gs);
  // half spectrum: row 0 keeps 0 < bx < P/2; the partner -k of every kept bin
  const int by = b / P, bx = b - by * P;
  const bool kept = valid && m < 0 && !(half && by == 0 && bx > P / 2);
  const bool ordinary = kept && wk != 0.f;
  if (grp == 0 && kept) {
    const float G = ordinary ? -wk * k * gs : 0.f;  // (1/2) dL/dwbar, for w1 and for w2
    float2* u = gbuf + static_cast<size_t>(patch) * 2 * P2;
    put_g(t, u, b, G, G);
    if (half) put_g(t, u, ((P - by) % P) * P + (P - bx) % P, G, G);
  }
  const double value = ordinary && grp == 0 ? (half ? 2.0 : 1.0) * static_cast<double>(wk) * acc : 0.0;
  block_sum_store(value, s_red, loss_part + patch * n_parts + cb);
}

// Small patches (P^2 < LB or not a multiple of LB): one CTA per (patch, chunk).
__global__ void __launch_bounds__(LB) loss_bins_small_kernel(FourierTab t, const float2* __restrict__ Y_all,
                                                             const float* __restrict__ w_all,
                                                             float eps_m, float scale, int implicit,
                                                             float2* __restrict__ gbuf,
                                                             double* __restrict__ loss_part,
                                                             int n_parts) {
  extern __shared__ __align__(16) float smem[];
  const int K = t.K, P2 = t.P2;
  float2* s_y = reinterpret_cast<float2*>(smem);  // [K][LB]
  float* s_w = smem + 2 * K * LB;                 // [A]
  __shared__ double s_red[LB / 32];
  const int patch = blockIdx.x, b0 = blockIdx.y * LB;
  const float2* Y = Y_all + static_cast<size_t>(patch) * K * P2;
  for (int a = threadIdx.x; a < t.A; a += LB) s_w[a] = w_all[patch * t.A + a];
  const int nb = min(LB, P2 - b0);
  for (int e = threadIdx.x; e < K * LB; e += LB) {
    const int j = e / LB, q = e - j * LB;
    s_y[e] = q < nb ? Y[static_cast<size_t>(j) * P2 + b0 + q] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  double value = 0.0;
  const int b = b0 + threadIdx.x;
  if (b < P2 && t.mirror[b] < 0) {
    float G;
    const float2* yb = s_y + threadIdx.x;
    value = bin_chain_real(t, s_w, b, eps_m, scale, implicit != 0,
                           [&](int j) { return yb[j * LB]; }, G);
    put_g(t, gbuf + static_cast<size_t>(patch) * 2 * P2, b, G, G);
  }
  block_sum_store(value, s_red, loss_part + patch * n_parts + blockIdx.y);
}

// The fixed-order sum of a patch's loss partials.
__device__ __forceinline__ double patch_loss(const double* __restrict__ loss_part, int patch,
                                             int n_parts) {
  double v = 0.0;
  for (int c = 0; c < n_parts; ++c) v += loss_part[patch * n_parts + c];
  return v;
}

// Kernel A': the Nyquist bins (even P), one block per patch, kTps threads per
// exchange slot (2P - 1 of them).  Each slot's unsymmetrised dL/dH_j goes to
// the exchange buffer; after the barrier every slot pulls back the
// symmetrised g = (dL/dH_b + conj(dL/dH_m)) / 2 (optimize.hpp:306-308).
constexpr int kTps = 4;

__global__ void __launch_bounds__(1024) loss_nyquist_kernel(FourierTab t, const float2* __restrict__ Y_all,
                                                            const float* __restrict__ w_all,
                                                            float eps_m, float scale, int implicit,
                                                            const float2* __restrict__ ynyq,
                                                            float2* __restrict__ nyq_all,
                                                            float2* __restrict__ gbuf,
                                                            double* __restrict__ loss_part,
                                                            int n_parts, int part0, int stage_y,
                                                            int stage_g) {
  extern __shared__ __align__(16) float smem[];
  __shared__ double s_red[32];
  const int patch = blockIdx.x, K = t.K, P2 = t.P2, S = 2 * t.P - 1;
  // shared memory: [A] profile | [K][S] spectra (stage_y) | [S][K] exchange
  // (stage_g); large K x S (cfg5: P = 128, K = 64) falls back to L2 for either
  float* s_w = smem;
  float2* s_y = reinterpret_cast<float2*>(smem + ((t.A + 1) & ~1));
  float2* s_g = stage_g ? s_y + (stage_y ? K * S : 0)
                        : nyq_all + static_cast<size_t>(patch) * S * K;
  for (int a = threadIdx.x; a < t.A; a += blockDim.x) s_w[a] = w_all[patch * t.A + a];
  const float2* Y = Y_all + static_cast<size_t>(patch) * K * P2;
  // the slots' spectra: from the compact [slot][K] copy kernel A made, or
  // (other kernel A forms) gathered from Y, eight loads in flight per thread
  // (kernel A's half-spectrum form copies the Nyquist bins of rows 0 .. P/2:
  // a column slot below the Nyquist row, by > P/2, reads conj of its
  // partner's, by' = P - by: Y(-k) = conj(Y(k)) for the real patch stack)
  const float2* Yc = ynyq ? ynyq + static_cast<size_t>(patch) * S * K : nullptr;
  const int half = t.P / 2;
  auto yc = [&](int slot, int j) {
    if (slot >= t.P + half) {  // column bin by = slot - P + 1 > P/2
      const float2 v = Yc[static_cast<size_t>(t.P + t.P - (slot - t.P + 1)) * K + j];
      return make_float2(v.x, -v.y);
    }
    return Yc[static_cast<size_t>(slot) * K + j];
  };
  const int kshift = (K & (K - 1)) == 0 ? __ffs(K) - 1 : -1;  // e / K as a shift
  for (int e0 = threadIdx.x; Yc && stage_y && e0 < K * S; e0 += 8 * blockDim.x) {
    float2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < K * S) {
        const int q = kshift >= 0 ? e >> kshift : e / K;
        v[u] = yc(q, e - q * K);
      } else {
        v[u] = make_float2(0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < K * S) {
        const int q = kshift >= 0 ? e >> kshift : e / K, j = e - q * K;
        s_y[j * S + q] = v[u];
      }
    }
  }
  for (int e0 = threadIdx.x; !Yc && stage_y && e0 < K * S; e0 += 8 * blockDim.x) {
    float2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      const int j = e / S, q = e - j * S;
      v[u] = e < K * S ? Y[static_cast<size_t>(j) * P2 + nyq_bin(q, t.P)] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (e0 + u * blockDim.x < K * S) s_y[e0 + u * blockDim.x] = v[u];
  }
  __syncthreads();
  // kTps threads per slot (consecutive lanes), each walking K / kTps delays;
  // the per-bin sums are combined with a fixed xor-shuffle tree
  const int slot = threadIdx.x / kTps, q = threadIdx.x % kTps;
  const bool active = slot < S;
  const int b = nyq_bin(active ? slot : 0, t.P), m = t.mirror[b];
  const int j0 = q * K / kTps, j1 = (q + 1) * K / kTps;
  const float k = t.kmag[b];
  const bool live = active && k * scale != 0.f;
  auto y_of = [&](int j) {
    return stage_y ? s_y[j * S + slot] : (Yc ? yc(slot, j) : Y[static_cast<size_t>(j) * P2 + b]);
  };
  auto group_sum = [&](float v) {
#pragma unroll
    for (int o = 1; o < kTps; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  float2 e1b, e2b, e1m, e2m;
  bin_phases(t, s_w, b, e1b, e2b);
  bin_phases(t, s_w, m, e1m, e2m);
  const bool walk = t.rho != nullptr;
  const float2 rb = walk ? t.rho[b] : make_float2(1.f, 0.f);
  const float2 rm = walk ? t.rho[m] : make_float2(1.f, 0.f);
  const float2 db0 = t.dp[j0 * P2 + b], dm0 = t.dp[j0 * P2 + m];
  auto next = [&](int j, float2& db, float2& dm) {
    if (walk) {
      db = cmul(db, rb);
      dm = cmul(dm, rm);
    } else if (j + 1 < K) {
      db = t.dp[(j + 1) * P2 + b];
      dm = t.dp[(j + 1) * P2 + m];
    }
  };
  auto h_sym = [&](float2 db, float2 dm) {  // (h_b + conj h_m) / 2, conj_symmetrize_nyquist
    const float2 hb = h_of(db, e1b, e2b), hm = h_of(dm, e1m, e2m);
    return make_float2(0.5f * (hb.x + hm.x), 0.5f * (hb.y - hm.y));
  };
  // pass 1: X-hat = num / den
  float nx = 0.f, ny = 0.f, dd = 0.f;
  {
    float2 db = db0, dm = dm0;
    for (int j = j0; j < j1; ++j) {
      const float2 h = h_sym(db, dm);
      const float2 c = cmulc(h, y_of(j));
      nx += c.x;
      ny += c.y;
      dd += h.x * h.x + h.y * h.y;
      next(j, db, dm);
    }
  }
  BinLoss L;
  L.wk = k * scale;
  L.den = eps_m + group_sum(dd);
  L.inv = L.den > 0.f ? 1.f / L.den : 0.f;
  const float2 num = make_float2(group_sum(nx), group_sum(ny));
  L.x = make_float2(num.x * L.inv, num.y * L.inv);
  L.G = make_float2(num.x * (eps_m * L.inv), -num.y * (eps_m * L.inv));
  L.gx = L.G.x * L.x.x - L.G.y * L.x.y;
  // pass 2: residuals and the unsymmetrised dL/dH_j -> exchange
  float acc = 0.f;
  {
    float2 db = db0, dm = dm0;
    for (int j = j0; j < j1; ++j) {
      const float2 h = h_sym(db, dm), y = y_of(j);
      const float2 hx = cmul(h, L.x);
      const float2 r = make_float2(y.x - hx.x, y.y - hx.y);
      acc += r.x * r.x + r.y * r.y;
      const float2 g = bin_grad(L, h, y, implicit != 0);
      if (active) s_g[static_cast<size_t>(j) * S + slot] = live ? g : make_float2(0.f, 0.f);
      next(j, db, dm);
    }
  }
  acc = group_sum(acc);
  const double value = live && q == 0 ? static_cast<double>(L.wk) * acc : 0.0;
  block_sum_store(value, s_red, loss_part + patch * n_parts + part0);
  __syncthreads();  // the exchange buffer of every slot is complete
  // symmetrised pullback g = (dL/dH_b + conj(dL/dH_m)) / 2 over this lane's delays
  float G1 = 0.f, G2 = 0.f;
  if (live) {
    const int sm = nyq_slot(m, t.P);
    float2 db = db0, dm = dm0;
    for (int j = j0; j < j1; ++j) {
      const float2 gb = s_g[j * S + slot], gm = s_g[j * S + sm];
      const float2 gs = make_float2(0.5f * (gb.x + gm.x), 0.5f * (gb.y - gm.y));
      pullback(gs, db, e1b, e2b, k, G1, G2);
      next(j, db, dm);
    }
  }
  G1 = group_sum(G1);
  G2 = group_sum(G2);
  if (active && q == 0) put_g(t, gbuf + static_cast<size_t>(patch) * 2 * P2, b, G1, G2);
}

// Kernel B: dL/dw of every (patch, angle) from the angle-sorted slots
// (FourierTab::slot): the .x shares of angle a's segment plus the .y shares of
// angle a - 1's, each a contiguous run summed in order (deterministic); the
// angle-0 thread also sums the patch's loss partials.  A block takes
// kFinishAngles angles of one patch and first stages their slot span in
// shared memory with coalesced loads (the runs are ~2 P^2 / A slots each).
__global__ void __launch_bounds__(kFinishAngles) loss_finish_kernel(
    FourierTab t, const float2* __restrict__ u_all, const double* __restrict__ loss_part, int n_parts,
    int n_patches, double* __restrict__ loss_out, float* __restrict__ dw_out) {
  extern __shared__ float2 s_u[];
  const int A = t.A, groups = (A + kFinishAngles - 1) / kFinishAngles;
  const int patch = blockIdx.x / groups, a0 = (blockIdx.x - patch * groups) * kFinishAngles;
  const int a1 = min(a0 + kFinishAngles, A);
  const int lo = __ldg(t.sstart + (a0 > 0 ? a0 - 1 : 0)), hi = __ldg(t.sstart + a1);
  const float2* u = u_all + static_cast<size_t>(patch) * 2 * t.P2;
  for (int s0 = lo + threadIdx.x; s0 < hi; s0 += 4 * kFinishAngles) {
    float2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int s = s0 + q * kFinishAngles;
      v[q] = s < hi ? __ldcs(u + s) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (s0 + q * kFinishAngles < hi) s_u[s0 + q * kFinishAngles - lo] = v[q];
  }
  __syncthreads();
  const int a = a0 + threadIdx.x;
  if (a >= A) return;
  const int am = a == 0 ? A - 1 : a - 1;
  // eight partial sums (element s - start goes to partial (s - start) % 8),
  // combined in a fixed tree
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int s0 = __ldg(t.sstart + a), s1 = __ldg(t.sstart + a + 1);
  for (int s = s0; s < s1; s += 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (s + q < s1) acc[q] += s_u[s + q - lo].x;
  }
  const int r0 = __ldg(t.sstart + am), r1 = __ldg(t.sstart + am + 1);
  for (int s = r0; s < r1; s += 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (s + q < r1) acc[q] += a == 0 ? u[s + q].y : s_u[s + q - lo].y;  // angle A - 1 wraps
  }
  dw_out[static_cast<size_t>(patch) * A + a] =
      ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  if (a == 0) loss_out[patch] = patch_loss(loss_part, patch, n_parts);
}

// X = sum_j conj(H_j) Y_j / (sum_j |H_j|^2 + eps M), 0 where den == 0
// (multichannel_deconvolve, deconv.hpp:78-96), H from the wavefront profile.
// HALF: the patch stack is real, so Y(-k) = conj Y(k), H(-k) = conj H(k) (as in
// the fused loss) and the estimate X is Hermitian: only the bins of rows
// 0 .. P/2 are evaluated (half of Y's traffic) and rows 1 .. P/2 - 1 also
// store conj X at -k (rows 0 and P/2 hold their own mirrors).
template <bool HALF>
__global__ void wiener_kernel(FourierTab t, const float2* __restrict__ Y_all,
                              const float* __restrict__ w_all, float eps_m,
                              float2* __restrict__ X_all) {
  extern __shared__ float s_w[];
  const int patch = blockIdx.y;
  for (int a = threadIdx.x; a < t.A; a += blockDim.x) s_w[a] = w_all[patch * t.A + a];
  __syncthreads();
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= (HALF ? (t.P / 2 + 1) * t.P : t.P2)) return;
  float2 e1b, e2b, e1m = {}, e2m = {};
  bin_phases(t, s_w, b, e1b, e2b);
  int m = t.mirror[b];
  if (m >= 0) bin_phases(t, s_w, m, e1m, e2m);
  const float2* Y = Y_all + static_cast<size_t>(patch) * t.K * t.P2;
  float2 num = make_float2(0.f, 0.f);
  float den = eps_m;
#pragma unroll 4
  for (int j = 0; j < t.K; ++j) {
    float2 h = h_sym(t, j, b, m, e1b, e2b, e1m, e2m);
    float2 c = cmulc(h, __ldcs(Y + static_cast<size_t>(j) * t.P2 + b));
    num.x += c.x;
    num.y += c.y;
    den += h.x * h.x + h.y * h.y;
  }
  const float2 x = den > 0.f ? make_float2(num.x / den, num.y / den) : make_float2(0.f, 0.f);
  float2* X = X_all + static_cast<size_t>(patch) * t.P2;
  X[b] = x;
  if (HALF) {
    const int by = b / t.P, bx = b - by * t.P;
    if (by >= 1 && by < t.P / 2) X[(t.P - by) * t.P + (t.P - bx) % t.P] = make_float2(x.x, -x.y);
  }
}

}  // namespace

Status launch_transfer_stack(pact_ctx* ctx, const FourierTab& t, const float* w, int n_patches,
                             float2* H) {
  dim3 g(div_up(t.P2, 256), n_patches);
  transfer_stack_kernel<<<g, 256, t.A * sizeof(float), ctx->stream>>>(t, w, n_patches, H);
  return after_launch(ctx, "transfer_stack_kernel");
}

// Kernel A of the register form for (NS, JPL) with K = NS * JPL, or null.
using LossRegFn = void (*)(FourierTab, const float2*, const float*, float, float, int, float2*,
                           double*, int, int);
LossRegFn loss_reg_for(int K, int& ns) {
  // PACT_LOSS_STAGED=1 selects the shared-memory staged kernel A (comparisons)
  static const bool staged = [] {
    const char* e = std::getenv("PACT_LOSS_STAGED");
    return e && e[0] == '1';
  }();
  if (staged) return nullptr;
  switch (K) {
    case 4: ns = 1; return loss_reg_kernel<1, 4>;
    case 8: ns = 1; return loss_reg_kernel<1, 8>;
    case 16: ns = 1; return loss_reg_kernel<1, 16>;
    case 32: ns = 2; return loss_reg_kernel<2, 16>;
    case 64: ns = 4; return loss_reg_kernel<4, 16>;
    default: return nullptr;
  }
}

Status launch_loss_grad(pact_ctx* ctx, const FourierTab& t, const float2* Y, const float* w,
                        int n_patches, double eps, double scale, bool implicit, double* loss,
                        float* dw) {
  const size_t smem = sizeof(float) * t.A;
  int ns = 0;
  const LossRegFn reg = loss_reg_for(t.K, ns);
  const int bpb = reg ? 8 * 32 / ns : LB;  // bins per kernel-A block
  // the register form reads rows 0 .. P/2 only for even P (half spectrum)
  const bool even = t.P % 2 == 0;
  const int chunks = div_up(reg && even ? (t.P / 2 + 1) * t.P : t.P2, bpb);
  // Nyquist: the register form's pair blocks (256 / ns units each), else kernel A'
  const int nyq_chunks = !even ? 0 : reg ? div_up(t.P + 1, 256 / ns) : 1;
  const int n_parts = chunks + nyq_chunks;  // per-patch loss partials, summed in order
  // scratch: Nyquist dL/dH exchange [patch][2P-1][K] | compact Nyquist spectra
  // [patch][2P-1][K] | (G1, G2) [patch][P2] | chunk losses
  const size_t n_nyq = static_cast<size_t>(n_patches) * (2 * t.P) * t.K;
  const size_t n_g = static_cast<size_t>(n_patches) * 2 * t.P2;  // slot shares
  void* base = nullptr;
  PACT_TRY_S(scratch_get(ctx, kScratchNyq,
                         sizeof(float2) * (2 * n_nyq + n_g) + sizeof(double) * n_patches * n_parts +
                             256,
                         &base));
  float2* nyq = static_cast<float2*>(base);
  float2* ynyq = nyq + n_nyq;
  float2* gbuf = ynyq + n_nyq;
  double* part = reinterpret_cast<double*>(gbuf + n_g);
  const float eps_m = static_cast<float>(eps * t.K), sc = static_cast<float>(scale);
  if (reg) {
    reg<<<n_patches * (chunks + (even ? nyq_chunks : 0)), 256, 0, ctx->stream>>>(
        t, Y, w, eps_m, sc, implicit, gbuf, part, n_parts, n_patches);
  } else if (t.P2 % LB == 0 && t.K * LB * 8 <= 96 * 1024) {
    const size_t stage = sizeof(float) * (2 * t.K * LB + ((t.A + 3) & ~3));
    const size_t smem_bins = 2 * stage;
    PACT_TRY_S(smem_optin(loss_bins_kernel, smem_bins));
    const int per_sm = std::max(1, static_cast<int>((227 * 1024 - 4096) / smem_bins));
    const int grid = std::min(n_patches * chunks, ctx->num_sms * per_sm);
    loss_bins_kernel<<<grid, 2 * LB, smem_bins, ctx->stream>>>(t, Y, w, eps_m, sc, implicit, gbuf,
                                                                part, n_parts, n_patches);
  } else {
    const size_t smem_bins = sizeof(float2) * t.K * LB + smem;
    if (smem_bins > 200 * 1024) return validation("fused loss: too many delays for one bin chunk");
    PACT_TRY_S(smem_optin(loss_bins_small_kernel, smem_bins));
    loss_bins_small_kernel<<<dim3(n_patches, chunks), LB, smem_bins, ctx->stream>>>(
        t, Y, w, eps_m, sc, implicit, gbuf, part, n_parts);
  }
  PACT_TRY_S(after_launch(ctx, reg ? "loss_reg_kernel" : "loss_bins_kernel"));
  if (even && !reg) {
    const int S = 2 * t.P - 1, nt = div_up(S * kTps, 32) * 32;
    if (nt > 1024) return validation("fused loss: patch size too large for the Nyquist kernel");
    const size_t plane = sizeof(float2) * t.K * S, base = sizeof(float) * ((t.A + 1) & ~1);
    const int stage_y = base + 2 * plane <= 200 * 1024;
    const int stage_g = base + (stage_y ? 2 : 1) * plane <= 200 * 1024;
    const size_t smem_nyq = base + (stage_y + stage_g) * plane;
    PACT_TRY_S(smem_optin(loss_nyquist_kernel, smem_nyq));
    loss_nyquist_kernel<<<n_patches, nt, smem_nyq, ctx->stream>>>(
        t, Y, w, eps_m, sc, implicit, nullptr, nyq, gbuf, part, n_parts, chunks, stage_y, stage_g);
    PACT_TRY_S(after_launch(ctx, "loss_nyquist_kernel"));
  }
  const size_t fin_smem = sizeof(float2) * std::max(t.fin_span, 1);
  PACT_TRY_S(smem_optin(loss_finish_kernel, fin_smem));
  loss_finish_kernel<<<n_patches * div_up(t.A, kFinishAngles), kFinishAngles, fin_smem, ctx->stream>>>(
      t, gbuf, part, n_parts, n_patches, loss, dw);
  return after_launch(ctx, "loss_finish_kernel");
}

Status launch_wiener(pact_ctx* ctx, const FourierTab& t, const float2* Y, const float* w,
                     int n_patches, double eps, float2* X) {
  // PACT_WIENER_FULL=1: every bin evaluated (the A/B reference of the half spectrum)
  static const bool full = [] {
    const char* e = std::getenv("PACT_WIENER_FULL");
    return e && e[0] == '1';
  }();
  const float eps_m = static_cast<float>(eps * t.K);
  if (!full && t.P % 2 == 0) {
    dim3 g(div_up((t.P / 2 + 1) * t.P, 256), n_patches);
    wiener_kernel<true><<<g, 256, t.A * sizeof(float), ctx->stream>>>(t, Y, w, eps_m, X);
  } else {
    dim3 g(div_up(t.P2, 256), n_patches);
    wiener_kernel<false><<<g, 256, t.A * sizeof(float), ctx->stream>>>(t, Y, w, eps_m, X);
  }
  return after_launch(ctx, "wiener_kernel");
}

}  // namespace pactgpu

using namespace pactgpu;

namespace {
// Table cache of the standalone entry points, one per context (it is
// rewritten in place when P, the pitch, the angles or the delays change, so it
// must not be shared with another context's stream or device).
struct ApiFourier {
  FourierTable tab;
  ~ApiFourier() { fourier_table_free(tab); }
};

FourierTable& api_table(pact_ctx* ctx) { return ctx_ext<ApiFourier>(ctx, kExtFourier)->tab; }
}  // namespace

extern "C" int pact_transfer_stack(pact_ctx* ctx, int32_t n_patches, const float* w,
                                   int32_t n_angles, const double* delays, int32_t K, int32_t P,
                                   double pitch, float* H) {
  if (!ctx || !w || !H || (!delays && K > 0))
    return validation("pact_transfer_stack: null argument").code;
  if (P < 1) return validation("transfer_stack: patch_pixels must be >= 1").code;
  if (!(pitch > 0.0)) return validation("transfer_stack: pitch must be > 0").code;
  if (n_angles < 1 || K < 1 || n_patches < 1) return validation("transfer_stack: empty input").code;
  FourierTable& tab = api_table(ctx);
  PACT_TRY(fourier_table(ctx, tab, P, pitch, n_angles, delays, K));
  PACT_TRY(launch_transfer_stack(ctx, tab.tab, w, n_patches, reinterpret_cast<float2*>(H)));
  return PACT_OK;
}

extern "C" int pact_loss_grad(pact_ctx* ctx, int32_t n_patches, const float* Y, const float* w,
                              int32_t n_angles, const double* delays, int32_t K, int32_t P,
                              double pitch, double eps, double scale, int32_t implicit,
                              double* loss_per_patch, float* dw) {
  if (!ctx || !Y || !w || !loss_per_patch || !dw || (!delays && K > 0))
    return validation("pact_loss_grad: null argument").code;
  if (K < 1) return validation("data_loss: no channels").code;
  if (n_patches < 1) return validation("data_loss: no patches").code;
  if (P < 1 || !(pitch > 0.0) || n_angles < 1) return validation("pact_loss_grad: bad geometry").code;
  FourierTable& tab = api_table(ctx);
  PACT_TRY(fourier_table(ctx, tab, P, pitch, n_angles, delays, K));
  PACT_TRY(launch_loss_grad(ctx, tab.tab, reinterpret_cast<const float2*>(Y), w, n_patches,
                            eps, scale, implicit != 0, loss_per_patch, dw));
  return PACT_OK;
}
