// SIREN coordinate network (part 2's SOS field and part 3's last gradient
// link), nfield.hpp:110-233:
//   forward   a_0 = W_0 c + b_0,  a_l = W_l sin(w0 a_{l-1}) + b_l,
//             v = v0 + out_scale (w_L . sin(w0 a_{L-1}) + b_L)
//   backward  reverse mode of sum_m g_m v(m) (backprop_sos, nfield.hpp:166-233)
//
// B200 design: per-layer fp32 SIMT GEMMs (128-pixel x 128-unit tiles, 8x8
// register micro-tiles, 256 threads) with the sine / cosine folded into the
// operand loaders and epilogues, so no z_l = sin(w0 a_l) tensor is ever
// stored: only the pre-activations a_l (needed for the cosine of the
// backward) are written.  Weight gradients are split over pixel chunks and
// reduced in a fixed order in fp64 (bitwise deterministic).  TF32/BF16 tensor
// cores fail the 1e-4 PSF tolerance for this network, so the
// dense layers stay on the FP32 pipe here.  Hidden widths that are not a
// multiple of 64 (unit-test networks) take a per-pixel path.
#include <cmath>
#include <memory>
#include <mutex>
#include <cstdlib>
#include <random>

#include "siren.cuh"

namespace pactgpu {

namespace {

MaskedPixels build_masked_pixels(const pact_grid& g, const pact_mask& m) {
  MaskedPixels mp;
  mp.idx.reserve(static_cast<size_t>(g.width) * g.height);
  mp.coords.reserve(2 * static_cast<size_t>(g.width) * g.height);
  for (int iy = 0; iy < g.height; ++iy)
    for (int ix = 0; ix < g.width; ++ix) {
      double px = g.origin_x + ix * g.pitch, py = g.origin_y + iy * g.pitch;
      if (!(std::hypot(px - m.center_x, py - m.center_y) <= m.radius)) continue;
      mp.idx.push_back(iy * g.width + ix);
      mp.coords.push_back(static_cast<float>((px - m.center_x) / m.radius));
      mp.coords.push_back(static_cast<float>((py - m.center_y) / m.radius));
    }
  mp.n = static_cast<int>(mp.idx.size());
  return mp;
}

}  // namespace

// The list depends only on (grid, mask): recent results are cached per
// process, so repeated reconstructions of the same geometry skip the host loop.
MaskedPixels masked_pixels(const pact_grid& g, const pact_mask& m) {
  struct Entry {
    pact_grid g;
    pact_mask m;
    std::shared_ptr<const MaskedPixels> mp;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  auto same = [&](const Entry& e) {
    return e.g.width == g.width && e.g.height == g.height && e.g.pitch == g.pitch &&
           e.g.origin_x == g.origin_x && e.g.origin_y == g.origin_y &&
           e.m.center_x == m.center_x && e.m.center_y == m.center_y && e.m.radius == m.radius;
  };
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& e : cache)
      if (same(e)) return *e.mp;
  }
  auto mp = std::make_shared<const MaskedPixels>(build_masked_pixels(g, m));
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() >= 4) cache.erase(cache.begin());
  cache.push_back({g, m, mp});
  return *mp;
}

namespace {

constexpr int BM = 128, BK = 16, NT = 256;

// the argument reduction of every SIREN kernel (siren.cuh)
__device__ __forceinline__ float red2pi(float x) { return sine_reduce(x); }
__device__ __forceinline__ float sinw(float a, float w0) { return __sinf(red2pi(w0 * a)); }
__device__ __forceinline__ float dsinw(float a, float w0) { return w0 * __cosf(red2pi(w0 * a)); }
__device__ __forceinline__ void sincosw(float a, float w0, float* s, float* c) {
  __sincosf(red2pi(w0 * a), s, c);
}

// ---- tiled GEMM core: acc[8 rows][TN cols] += As[kk][rows] * Bs[kk][cols] ----
template <int BN>
struct TileShape {
  static constexpr int TN = BN / 16;  // 8 (BN=128) or 4 (BN=64)
};

// column owned by thread tx, slot j (interleaved so a warp's LDS.128 are contiguous)
template <int BN>
__device__ __forceinline__ int tcol(int tx, int j) {
  return BN == 128 ? ((j < 4) ? tx * 4 + j : 64 + tx * 4 + (j - 4)) : tx * 4 + j;
}

template <int BN>
__device__ __forceinline__ void mma_tile(const float* __restrict__ As, const float* __restrict__ Bs,
                                         float (&acc)[8][TileShape<BN>::TN], int ty, int tx) {
  constexpr int TN = TileShape<BN>::TN;
#pragma unroll
  for (int kk = 0; kk < BK; ++kk) {
    float a[8], b[TN];
    float4 a0 = *reinterpret_cast<const float4*>(As + kk * BM + ty * 8);
    float4 a1 = *reinterpret_cast<const float4*>(As + kk * BM + ty * 8 + 4);
    a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
    a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
    float4 b0 = *reinterpret_cast<const float4*>(Bs + kk * BN + tx * 4);
    b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
    if constexpr (TN == 8) {
      float4 b1 = *reinterpret_cast<const float4*>(Bs + kk * BN + 64 + tx * 4);
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
  }
}

// Operand tiles are fetched into registers one k-step ahead (load), then
// transformed and written to the other shared-memory buffer (store) after the
// current step's FMAs: one barrier per k-step, global latency hidden behind math.
//
// TileT: R rows x 16 cols of row-major X (leading dim ld) at (r0, c0), stored
// transposed S[kk][r].  Rows >= rmax are zero.  SIN: store sin(w0 x).
template <int R, bool SIN>
struct TileT {
  static constexpr int PER = R * BK / NT;  // 8 (R = 128) or 4 (R = 64)
  float v[PER];
  __device__ __forceinline__ void load(const float* __restrict__ X, int ld, int r0, int c0,
                                       int rmax) {
    const int t = threadIdx.x, r = t / (BK / PER), kk0 = (t % (BK / PER)) * PER;
    if (r0 + r < rmax) {
      const float* src = X + static_cast<size_t>(r0 + r) * ld + c0 + kk0;
#pragma unroll
      for (int q = 0; q < PER; q += 4) {
        float4 x = *reinterpret_cast<const float4*>(src + q);
        v[q] = x.x; v[q + 1] = x.y; v[q + 2] = x.z; v[q + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < PER; ++q) v[q] = 0.f;
    }
  }
  __device__ __forceinline__ void store(float* __restrict__ S, float w0) const {
    const int t = threadIdx.x, r = t / (BK / PER), kk0 = (t % (BK / PER)) * PER;
#pragma unroll
    for (int q = 0; q < PER; ++q) S[(kk0 + q) * R + r] = SIN ? sinw(v[q], w0) : v[q];
  }
};

// TileD: 16 rows x C cols of row-major X at (r0, c0), stored directly S[kk][c].
template <int C, bool SIN>
struct TileD {
  static constexpr int PER = C * BK / NT;  // 8 or 4
  float v[PER];
  __device__ __forceinline__ void load(const float* __restrict__ X, int ld, int r0, int c0,
                                       int rmax) {
    const int t = threadIdx.x, kk = t / (C / PER), cc = (t % (C / PER)) * PER;
    if (r0 + kk < rmax) {
      const float* src = X + static_cast<size_t>(r0 + kk) * ld + c0 + cc;
#pragma unroll
      for (int q = 0; q < PER; q += 4) {
        float4 x = *reinterpret_cast<const float4*>(src + q);
        v[q] = x.x; v[q + 1] = x.y; v[q + 2] = x.z; v[q + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < PER; ++q) v[q] = 0.f;
    }
  }
  __device__ __forceinline__ void store(float* __restrict__ S, float w0) const {
    const int t = threadIdx.x, kk = t / (C / PER), cc = (t % (C / PER)) * PER;
#pragma unroll
    for (int q = 0; q < PER; q += 4) {
      float4 o = SIN ? make_float4(sinw(v[q], w0), sinw(v[q + 1], w0), sinw(v[q + 2], w0),
                                   sinw(v[q + 3], w0))
                     : make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
      *reinterpret_cast<float4*>(S + kk * C + cc + q) = o;
    }
  }
};

// a_0[m][n] = b_0[n] + W_0[n][0] c_x + W_0[n][1] c_y     (nfield.hpp:117-121, l = 0)
// One thread per 4 consecutive features of a pixel (float4 store).
__global__ void siren_first_kernel(const float2* __restrict__ coords, const float* __restrict__ W0,
                                   const float* __restrict__ b0, int n, int H,
                                   float* __restrict__ A0) {
  const int q4 = H / 4;
  const size_t total = static_cast<size_t>(n) * q4;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / q4), k = static_cast<int>(i - static_cast<size_t>(m) * q4) * 4;
    const float2 c = coords[m];
    const float4 wa = *reinterpret_cast<const float4*>(W0 + 2 * k);
    const float4 wb = *reinterpret_cast<const float4*>(W0 + 2 * k + 4);
    const float4 b = *reinterpret_cast<const float4*>(b0 + k);
    *reinterpret_cast<float4*>(A0 + i * 4) =
        make_float4(fmaf(wa.y, c.y, fmaf(wa.x, c.x, b.x)), fmaf(wa.w, c.y, fmaf(wa.z, c.x, b.y)),
                    fmaf(wb.y, c.y, fmaf(wb.x, c.x, b.z)), fmaf(wb.w, c.y, fmaf(wb.z, c.x, b.w)));
  }
}

// a_l = W_l sin(w0 a_{l-1}) + b_l        grid (ceil(n/128), H/BN)
template <int BN>
__global__ void __launch_bounds__(NT, 2)
siren_fwd_kernel(const float* __restrict__ Ain, const float* __restrict__ W,
                 const float* __restrict__ b, int n, int H, float w0, float* __restrict__ Aout) {
  constexpr int TN = TileShape<BN>::TN;
  __shared__ __align__(16) float As[2][BK * BM];
  __shared__ __align__(16) float Bs[2][BK * BN];
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  float acc[8][TN] = {};
  TileT<BM, true> ta;    // As[kk][m] = sin(w0 a_{l-1}[m0+m][k0+kk])
  TileT<BN, false> tb;   // Bs[kk][n] = W[n0+n][k0+kk]
  ta.load(Ain, H, m0, 0, n);
  tb.load(W, H, n0, 0, H);
  ta.store(As[0], w0);
  tb.store(Bs[0], w0);
  __syncthreads();
  const int nk = H / BK;
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) {
      ta.load(Ain, H, m0, (kt + 1) * BK, n);
      tb.load(W, H, n0, (kt + 1) * BK, H);
    }
    mma_tile<BN>(As[cur], Bs[cur], acc, ty, tx);
    if (kt + 1 < nk) {
      ta.store(As[cur ^ 1], w0);
      tb.store(Bs[cur ^ 1], w0);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int m = m0 + ty * 8 + i;
    if (m >= n) break;
#pragma unroll
    for (int j = 0; j < TN; j += 4) {
      int c = n0 + tcol<BN>(tx, j);
      float4 o = make_float4(acc[i][j] + b[c], acc[i][j + 1] + b[c + 1], acc[i][j + 2] + b[c + 2],
                             acc[i][j + 3] + b[c + 3]);
      *reinterpret_cast<float4*>(Aout + static_cast<size_t>(m) * H + c) = o;
    }
  }
}

// dv[idx[m]] = out_scale (b_L + sum_k w_L[k] sin(w0 a_{L-1}[m][k]))
// Eight threads per pixel (H/8 features each, float4 loads), 3-step shuffle sum.
__global__ void siren_out_kernel(const float* __restrict__ A, const float* __restrict__ wL,
                                 const float* __restrict__ bL, const int* __restrict__ idx, int n,
                                 int H, float w0, float out_scale, float* __restrict__ dv) {
  const int sub = threadIdx.x & 7;
  const int per = H / 8;  // features per thread, multiple of 4 (H % 32 == 0)
  for (int m = (blockIdx.x * blockDim.x + threadIdx.x) >> 3; m < ((n + 3) & ~3);
       m += (gridDim.x * blockDim.x) >> 3) {
    float s = 0.f;
    if (m < n) {
      const float* row = A + static_cast<size_t>(m) * H + sub * 4;
      for (int k = 0; k < per; k += 4) {
        const float4 a = *reinterpret_cast<const float4*>(row + k * 8);
        const float4 w = *reinterpret_cast<const float4*>(wL + sub * 4 + k * 8);
        s = fmaf(w.x, sinw(a.x, w0), s);
        s = fmaf(w.y, sinw(a.y, w0), s);
        s = fmaf(w.z, sinw(a.z, w0), s);
        s = fmaf(w.w, sinw(a.w, w0), s);
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (sub == 0 && m < n) dv[idx[m]] = out_scale * (bL[0] + s);
  }
}

// Top of the backward: g_m = out_scale (gv[idx m] + gmask[m]);
//   dA_{L-1}[m][k] = g_m w_L[k] w0 cos(w0 a)      (nfield.hpp:198-200)
//   partial gW_L[k] += g_m sin(w0 a), gb_L += g_m (nfield.hpp:194-197)
// grid.x = pixel chunks of `rows` pixels.  A row is H/4 threads with one
// float4 each (coalesced 16-B loads / stores); TOP_RP rows per pass; each
// thread keeps TOP_U rows in flight and prefetches the next batch into a
// second register set before computing the current one (the kernel streams
// 2 x 134 MB at cfg3, so it lives on memory-level parallelism).
template <int H>
struct TopShape {
  static constexpr int TPR = H / 4;             // threads per row
  static constexpr int RP = 256 / TPR;          // rows per pass
  static constexpr int NTH = TPR * RP;          // block size
  static constexpr int U = 4;                   // rows in flight per thread
};

template <int H>
__global__ void __launch_bounds__(TopShape<H>::NTH)
siren_top_kernel(const float* __restrict__ A, const float* __restrict__ wL,
                 const double* __restrict__ gv, const float* __restrict__ gmask,
                 const int* __restrict__ idx, int n, int rows, float w0, float out_scale,
                 float* __restrict__ dA, float* __restrict__ partial) {
  using T = TopShape<H>;
  constexpr int TPR = T::TPR, RP = T::RP, U = T::U;
  __shared__ float s_part[RP][H + 1];
  const int c4 = threadIdx.x % TPR, rl = threadIdx.x / TPR;
  const int m_begin = blockIdx.x * rows, m_end = min(n, m_begin + rows);
  const float4 wk = reinterpret_cast<const float4*>(wL)[c4];
  float4 gw = make_float4(0.f, 0.f, 0.f, 0.f);
  float gb = 0.f;
  float4 a0[U], a1[U];
  float g0[U], g1[U];
  auto load = [&](int m0, float4 (&av)[U], float (&gvv)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = m0 + rl + RP * u;
      const bool ok = m < m_end;
      const int mm = ok ? m : m_begin;
      av[u] = reinterpret_cast<const float4*>(A + static_cast<size_t>(mm) * H)[c4];
      float gg = 0.f;
      if (gv) gg += static_cast<float>(gv[idx[mm]]);
      if (gmask) gg += gmask[mm];
      gvv[u] = ok ? gg * out_scale : 0.f;
    }
  };
  auto body = [&](int m0, const float4 (&av)[U], const float (&gvv)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = m0 + rl + RP * u;
      const float gg = gvv[u];
      const float4 x = av[u];
      float4 sn, cs, d;
      sincosw(x.x, w0, &sn.x, &cs.x);
      sincosw(x.y, w0, &sn.y, &cs.y);
      sincosw(x.z, w0, &sn.z, &cs.z);
      sincosw(x.w, w0, &sn.w, &cs.w);
      const float gw0 = gg * w0;
      d.x = gw0 * wk.x * cs.x;
      d.y = gw0 * wk.y * cs.y;
      d.z = gw0 * wk.z * cs.z;
      d.w = gw0 * wk.w * cs.w;
      if (m < m_end) reinterpret_cast<float4*>(dA + static_cast<size_t>(m) * H)[c4] = d;
      gw.x = fmaf(gg, sn.x, gw.x);
      gw.y = fmaf(gg, sn.y, gw.y);
      gw.z = fmaf(gg, sn.z, gw.z);
      gw.w = fmaf(gg, sn.w, gw.w);
      gb += gg;
    }
  };
  // two register sets: the next batch is in flight while one is computed
  constexpr int STEP = RP * U;
  if (m_begin < m_end) load(m_begin, a0, g0);
  for (int m0 = m_begin; m0 < m_end; m0 += 2 * STEP) {
    if (m0 + STEP < m_end) load(m0 + STEP, a1, g1);
    body(m0, a0, g0);
    if (m0 + STEP >= m_end) break;
    if (m0 + 2 * STEP < m_end) load(m0 + 2 * STEP, a0, g0);
    body(m0 + STEP, a1, g1);
  }
  // fixed-order sums over the row lanes
  s_part[rl][4 * c4] = gw.x;
  s_part[rl][4 * c4 + 1] = gw.y;
  s_part[rl][4 * c4 + 2] = gw.z;
  s_part[rl][4 * c4 + 3] = gw.w;
  if (c4 == 0) s_part[rl][H] = gb;
  __syncthreads();
  float* out = partial + static_cast<size_t>(blockIdx.x) * (H + 1);
  for (int k = threadIdx.x; k <= H; k += T::NTH) {
    float t = 0.f;
    for (int q = 0; q < RP; ++q) t += s_part[q][k];
    out[k] = t;
  }
}

// dA_{l-1}[m][k] = (sum_r dA_l[m][r] W_l[r][k]) w0 cos(w0 a_{l-1}[m][k])   (nfield.hpp:207-227)
template <int BN>
__global__ void __launch_bounds__(NT, 2)
siren_dgrad_kernel(const float* __restrict__ dAl, const float* __restrict__ W,
                   const float* __restrict__ Aprev, int n, int H, float w0,
                   float* __restrict__ dAprev) {
  constexpr int TN = TileShape<BN>::TN;
  __shared__ __align__(16) float As[2][BK * BM];
  __shared__ __align__(16) float Bs[2][BK * BN];
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  float acc[8][TN] = {};
  TileT<BM, false> ta;  // As[rr][m] = dA_l[m0+m][r0+rr]
  TileD<BN, false> tb;  // Bs[rr][k] = W[r0+rr][n0+k]
  ta.load(dAl, H, m0, 0, n);
  tb.load(W, H, 0, n0, H);
  ta.store(As[0], w0);
  tb.store(Bs[0], w0);
  __syncthreads();
  const int nk = H / BK;
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) {
      ta.load(dAl, H, m0, (kt + 1) * BK, n);
      tb.load(W, H, (kt + 1) * BK, n0, H);
    }
    mma_tile<BN>(As[cur], Bs[cur], acc, ty, tx);
    if (kt + 1 < nk) {
      ta.store(As[cur ^ 1], w0);
      tb.store(Bs[cur ^ 1], w0);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int m = m0 + ty * 8 + i;
    if (m >= n) break;
#pragma unroll
    for (int j = 0; j < TN; j += 4) {
      int c = n0 + tcol<BN>(tx, j);
      size_t off = static_cast<size_t>(m) * H + c;
      float4 a = *reinterpret_cast<const float4*>(Aprev + off);
      float4 o = make_float4(acc[i][j] * dsinw(a.x, w0), acc[i][j + 1] * dsinw(a.y, w0),
                             acc[i][j + 2] * dsinw(a.z, w0), acc[i][j + 3] * dsinw(a.w, w0));
      *reinterpret_cast<float4*>(dAprev + off) = o;
    }
  }
}

// Split-M weight gradient of a hidden layer l >= 1:
//   partial[chunk][r][k] = sum_{m in chunk} dA_l[m][r] sin(w0 a_{l-1}[m][k]),
//   partial bias[chunk][r] = sum_m dA_l[m][r]
// grid (n_chunks, H/BN (rows r), H/BN (cols k)); the tile is BN x BN with
// BN/16 x BN/16 outputs per thread.
template <int BN>
__global__ void __launch_bounds__(NT, 2)
siren_wgrad_kernel(const float* __restrict__ dAl, const float* __restrict__ Aprev, int n, int H,
                   int rows, float w0, float* __restrict__ partial) {
  constexpr int T = BN / 16;  // outputs per thread along each axis (8 or 4)
  __shared__ __align__(16) float As[2][BK * BN];
  __shared__ __align__(16) float Bs[2][BK * BN];
  const int chunk = blockIdx.x;
  const int r0 = blockIdx.y * BN, k0 = blockIdx.z * BN;
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  const int m_begin = chunk * rows, m_end = min(n, m_begin + rows);
  float acc[T][T] = {};
  float bias[T] = {};
  const bool do_bias = (blockIdx.z == 0 && tx == 0);
  TileD<BN, false> ta;  // As[mm][r] = dA[mb+mm][r0+r]
  TileD<BN, true> tb;   // Bs[mm][k] = sin(w0 a_{l-1}[mb+mm][k0+k])
  if (m_begin < m_end) {
    ta.load(dAl, H, m_begin, r0, m_end);
    tb.load(Aprev, H, m_begin, k0, m_end);
    ta.store(As[0], w0);
    tb.store(Bs[0], w0);
  }
  __syncthreads();
  int cur = 0;
  for (int mb = m_begin; mb < m_end; mb += BK) {
    const bool more = mb + BK < m_end;
    if (more) {
      ta.load(dAl, H, mb + BK, r0, m_end);
      tb.load(Aprev, H, mb + BK, k0, m_end);
    }
    const float* A_ = As[cur];
    const float* B_ = Bs[cur];
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[T], b[T];
#pragma unroll
      for (int q = 0; q < T; q += 4) {
        float4 x = *reinterpret_cast<const float4*>(A_ + kk * BN + ty * T + q);
        a[q] = x.x; a[q + 1] = x.y; a[q + 2] = x.z; a[q + 3] = x.w;
        float4 y = *reinterpret_cast<const float4*>(B_ + kk * BN + (q == 0 ? tx * 4 : 64 + tx * 4));
        b[q] = y.x; b[q + 1] = y.y; b[q + 2] = y.z; b[q + 3] = y.w;
      }
#pragma unroll
      for (int i = 0; i < T; ++i)
#pragma unroll
        for (int j = 0; j < T; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      if (do_bias) {
#pragma unroll
        for (int i = 0; i < T; ++i) bias[i] += a[i];
      }
    }
    if (more) {
      ta.store(As[cur ^ 1], w0);
      tb.store(Bs[cur ^ 1], w0);
    }
    __syncthreads();
    cur ^= 1;
  }
  // partial layout per chunk: [H rows][H cols] weights then [H] bias
  float* out = partial + static_cast<size_t>(chunk) * (static_cast<size_t>(H) * H + H);
#pragma unroll
  for (int i = 0; i < T; ++i) {
    int r = r0 + ty * T + i;
#pragma unroll
    for (int j = 0; j < T; ++j) out[static_cast<size_t>(r) * H + k0 + tcol<BN>(tx, j)] = acc[i][j];
    if (do_bias) out[static_cast<size_t>(H) * H + r] = bias[i];
  }
}

// Layer-0 gradient partials: gW_0[r][c] += dA_0[m][r] c_m[c], gb_0[r] += dA_0[m][r].
// Same streaming shape as siren_top_kernel: float4 rows, two register sets.
template <int H>
__global__ void __launch_bounds__(TopShape<H>::NTH)
siren_wgrad0_kernel(const float* __restrict__ dA0, const float2* __restrict__ coords, int n,
                    int rows, float* __restrict__ partial) {
  using T = TopShape<H>;
  constexpr int TPR = T::TPR, RP = T::RP, U = T::U;
  __shared__ float s_part[3][RP][H + 1];
  const int c4 = threadIdx.x % TPR, rl = threadIdx.x / TPR;
  const int m_begin = blockIdx.x * rows, m_end = min(n, m_begin + rows);
  float4 gx = make_float4(0.f, 0.f, 0.f, 0.f), gy = gx, gb = gx;
  float4 d0[U], d1[U];
  float2 c0[U], c1[U];
  auto load = [&](int m0, float4 (&dv)[U], float2 (&cv)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = m0 + rl + RP * u;
      const bool ok = m < m_end;
      const int mm = ok ? m : m_begin;
      dv[u] = reinterpret_cast<const float4*>(dA0 + static_cast<size_t>(mm) * H)[c4];
      const float2 c = coords[mm];
      cv[u] = ok ? c : make_float2(0.f, 0.f);
      if (!ok) dv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto body = [&](const float4 (&dv)[U], const float2 (&cv)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float4 d = dv[u];
      const float2 c = cv[u];
      gx.x = fmaf(d.x, c.x, gx.x);
      gx.y = fmaf(d.y, c.x, gx.y);
      gx.z = fmaf(d.z, c.x, gx.z);
      gx.w = fmaf(d.w, c.x, gx.w);
      gy.x = fmaf(d.x, c.y, gy.x);
      gy.y = fmaf(d.y, c.y, gy.y);
      gy.z = fmaf(d.z, c.y, gy.z);
      gy.w = fmaf(d.w, c.y, gy.w);
      gb.x += d.x;
      gb.y += d.y;
      gb.z += d.z;
      gb.w += d.w;
    }
  };
  constexpr int STEP = RP * U;
  if (m_begin < m_end) load(m_begin, d0, c0);
  for (int m0 = m_begin; m0 < m_end; m0 += 2 * STEP) {
    if (m0 + STEP < m_end) load(m0 + STEP, d1, c1);
    body(d0, c0);
    if (m0 + STEP >= m_end) break;
    if (m0 + 2 * STEP < m_end) load(m0 + 2 * STEP, d0, c0);
    body(d1, c1);
  }
  const float4* acc[3] = {&gx, &gy, &gb};
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    s_part[q][rl][4 * c4] = acc[q]->x;
    s_part[q][rl][4 * c4 + 1] = acc[q]->y;
    s_part[q][rl][4 * c4 + 2] = acc[q]->z;
    s_part[q][rl][4 * c4 + 3] = acc[q]->w;
  }
  __syncthreads();
  float* out = partial + static_cast<size_t>(blockIdx.x) * (3 * H);
  for (int r = threadIdx.x; r < H; r += T::NTH) {
    float tx = 0.f, ty = 0.f, tb = 0.f;
    for (int q = 0; q < RP; ++q) {
      tx += s_part[0][q][r];
      ty += s_part[1][q][r];
      tb += s_part[2][q][r];
    }
    out[2 * r] = tx;  // W_0 row-major [r][c]
    out[2 * r + 1] = ty;
    out[2 * H + r] = tb;
  }
}

// grad[off + p] = sum_chunk partial[chunk][p]   (fixed order, fp64)
// All of one backward pass's partial-sum reductions in one launch: segment
// s sums partial rows [n_chunks][per] of src into dst.  A block is
// (64 params) x (4 chunk groups); group y sums its contiguous quarter of the
// chunks with four interleaved accumulators (every thread has ~n_chunks / 4
// independent coalesced loads in flight: one wave of latency, not one per
// chunk), then a fixed-order fold over the groups (deterministic).  Block b
// belongs to the segment whose cumulative block range holds b.
constexpr int kMaxSeg = 8;
constexpr int kRedP = 64, kRedG = 4;
struct ReduceSegs {
  const float* src[kMaxSeg];
  double* dst[kMaxSeg];
  int n_chunks[kMaxSeg], per[kMaxSeg], block_end[kMaxSeg];
  int n;
};

__global__ void __launch_bounds__(kRedP * kRedG) reduce_segments_kernel(ReduceSegs sg) {
  __shared__ double s_sum[kRedG][kRedP];
  int seg = 0;
  while (seg + 1 < sg.n && blockIdx.x >= static_cast<unsigned>(sg.block_end[seg])) ++seg;
  const int b = blockIdx.x - (seg ? sg.block_end[seg - 1] : 0);
  const float* __restrict__ partial = sg.src[seg];
  const int per_chunk = sg.per[seg], n_chunks = sg.n_chunks[seg];
  const int p = b * kRedP + threadIdx.x;
  const int q = (n_chunks + kRedG - 1) / kRedG;
  const int c0 = threadIdx.y * q, c1 = min(n_chunks, c0 + q);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (p < per_chunk) {
    const float* src = partial + p;
    int c = c0;
#pragma unroll 4
    for (; c + 3 < c1; c += 4) {
      a0 += src[static_cast<size_t>(c) * per_chunk];
      a1 += src[static_cast<size_t>(c + 1) * per_chunk];
      a2 += src[static_cast<size_t>(c + 2) * per_chunk];
      a3 += src[static_cast<size_t>(c + 3) * per_chunk];
    }
    for (; c < c1; ++c) a0 += src[static_cast<size_t>(c) * per_chunk];
  }
  s_sum[threadIdx.y][threadIdx.x] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (threadIdx.y == 0 && p < per_chunk) {
    double t = 0.0;
    for (int y = 0; y < kRedG; ++y) t += s_sum[y][threadIdx.x];
    sg.dst[seg][p] = t;
  }
}

// ---- per-pixel path for small / odd hidden widths (unit-test networks) ----
// Forward: a_l stored as in the tiled path; output written into dv.
__global__ void siren_fwd_small_kernel(const float* __restrict__ th, const float2* __restrict__ coords,
                                       const int* __restrict__ idx, int n, int H, int L, float w0,
                                       float out_scale, float* __restrict__ acts,
                                       float* __restrict__ dv, size_t layer_stride) {
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  float2 c = coords[m];
  const float* W0 = th;
  const float* b0 = th + 2 * H;
  float* a0 = acts + static_cast<size_t>(m) * H;
  for (int k = 0; k < H; ++k) a0[k] = fmaf(W0[2 * k + 1], c.y, fmaf(W0[2 * k], c.x, b0[k]));
  size_t off = 3 * H;
  for (int l = 1; l < L; ++l) {
    const float* W = th + off;
    const float* b = W + static_cast<size_t>(H) * H;
    const float* ap = acts + (l - 1) * layer_stride + static_cast<size_t>(m) * H;
    float* ao = acts + l * layer_stride + static_cast<size_t>(m) * H;
    for (int r = 0; r < H; ++r) {
      float s = b[r];
      for (int k = 0; k < H; ++k) s = fmaf(W[r * H + k], sinw(ap[k], w0), s);
      ao[r] = s;
    }
    off += static_cast<size_t>(H) * H + H;
  }
  const float* wL = th + off;
  const float* ap = acts + (L - 1) * layer_stride + static_cast<size_t>(m) * H;
  float s = 0.f;
  for (int k = 0; k < H; ++k) s = fmaf(wL[k], sinw(ap[k], w0), s);
  dv[idx[m]] = out_scale * (wL[H] + s);
}

// Backward per pixel into contrib[m][param] (reduced afterwards in fixed order).
__global__ void siren_bwd_small_kernel(const float* __restrict__ th, const float2* __restrict__ coords,
                                       const int* __restrict__ idx, int n, int H, int L, float w0,
                                       float out_scale, const float* __restrict__ acts,
                                       size_t layer_stride, const double* __restrict__ gv,
                                       const float* __restrict__ gmask, float* __restrict__ delta,
                                       float* __restrict__ contrib, int n_params) {
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  float* cg = contrib + static_cast<size_t>(m) * n_params;
  float g = 0.f;
  if (gv) g += static_cast<float>(gv[idx[m]]);
  if (gmask) g += gmask[m];
  g *= out_scale;
  float* d = delta + static_cast<size_t>(m) * 2 * H;  // [delta | delta_prev]
  float* dp = d + H;
  size_t offL = 3 * H + static_cast<size_t>(L - 1) * (static_cast<size_t>(H) * H + H);
  const float* wL = th + offL;
  const float* aL = acts + (L - 1) * layer_stride + static_cast<size_t>(m) * H;
  for (int k = 0; k < H; ++k) {
    cg[offL + k] = g * sinw(aL[k], w0);
    d[k] = g * wL[k];
  }
  cg[offL + H] = g;
  for (int l = L - 1; l >= 0; --l) {
    size_t off = l == 0 ? 0 : 3 * H + static_cast<size_t>(l - 1) * (static_cast<size_t>(H) * H + H);
    int cols = l == 0 ? 2 : H;
    const float* W = th + off;
    const float* al = acts + l * layer_stride + static_cast<size_t>(m) * H;
    const float* ap = l > 0 ? acts + (l - 1) * layer_stride + static_cast<size_t>(m) * H : nullptr;
    float2 c = coords[m];
    for (int k = 0; k < H; ++k) dp[k] = 0.f;
    for (int r = 0; r < H; ++r) {
      float da = d[r] * dsinw(al[r], w0);
      cg[off + static_cast<size_t>(H) * cols + r] = da;
      for (int q = 0; q < cols; ++q) {
        float zin = l == 0 ? (q == 0 ? c.x : c.y) : sinw(ap[q], w0);
        cg[off + static_cast<size_t>(r) * cols + q] = da * zin;
        if (l > 0) dp[q] = fmaf(da, W[r * cols + q], dp[q]);
      }
    }
    for (int k = 0; k < H; ++k) d[k] = dp[k];
  }
}

__global__ void reduce_rows_kernel(const float* __restrict__ contrib, int n, int n_params,
                                   double* __restrict__ grad) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_params) return;
  double s = 0.0;
  for (int m = 0; m < n; ++m) s += contrib[static_cast<size_t>(m) * n_params + p];
  grad[p] = s;
}

}  // namespace

// The fused per-layer backward (siren_bwd.cu) serves hidden width 128 on
// tcgen05; PACT_SIREN_FUSED_BWD=0 selects the per-op kernels.  When it runs,
// the forward skips storing a_0 (the backward recomputes it).
bool siren_fused_bwd(const SirenShape& s) {
  static const bool on = [] {
    const char* e = std::getenv("PACT_SIREN_FUSED_BWD");
    return !(e && e[0] == '0');
  }();
  return on && s.hidden == 128 && s.layers >= 2 && siren_use_tc(s.hidden);
}

// Hidden width 256 on the streamed tcgen05 GEMMs (siren_wide.cu);
// PACT_SIREN_SIMT=1 also forces the SIMT tiles here.
bool siren_use_wide(int hidden) {
  static const bool simt = [] {
    const char* e = std::getenv("PACT_SIREN_SIMT");
    return e && e[0] == '1';
  }();
  return !simt && siren_wide_supported(hidden);
}

bool siren_use_tc(int hidden) {
  static const bool simt = [] {
    const char* e = std::getenv("PACT_SIREN_SIMT");
    return e && e[0] == '1';
  }();
  return !simt && siren_tc_supported(hidden);
}

namespace {

bool tiled(const SirenShape& s) { return s.hidden % 64 == 0 && s.hidden <= 256 && s.in_dim == 2; }

int chunk_rows(int n, int tiles, int num_sms) {
  int chunks = std::max(1, (2 * num_sms) / std::max(1, tiles));
  int rows = div_up(n, chunks);
  rows = div_up(rows, BK) * BK;
  return std::max(rows, BK);
}

}  // namespace

Status siren_work_alloc(SirenWork& w, const MaskedPixels& mp, const SirenShape& s,
                        cudaStream_t stream) {
  siren_work_free(w);
  w.n = mp.n;
  w.hidden = s.hidden;
  w.layers = s.layers;
  size_t nh = static_cast<size_t>(std::max(1, mp.n)) * s.hidden;
  w.stream = stream;
  PACT_TRY_S(pool_alloc(reinterpret_cast<void**>(&w.idx), sizeof(int) * std::max(1, mp.n), stream));
  PACT_TRY_S(pool_alloc(reinterpret_cast<void**>(&w.coords), sizeof(float2) * std::max(1, mp.n),
                        stream));
  PACT_TRY_S(pool_alloc(reinterpret_cast<void**>(&w.acts), sizeof(float) * nh * s.layers, stream));
  PACT_TRY_S(pool_alloc(reinterpret_cast<void**>(&w.dA), sizeof(float) * nh * 2, stream));
  PACT_TRY_S(pool_alloc(reinterpret_cast<void**>(&w.dB), sizeof(float) * nh, stream));
  if (mp.n > 0) {
    PACT_CUDA_S(cudaMemcpyAsync(w.idx, mp.idx.data(), sizeof(int) * mp.n, cudaMemcpyHostToDevice,
                                stream));
    // (pageable sources are staged by the copy call; callers keep `mp` alive anyway)
    PACT_CUDA_S(cudaMemcpyAsync(w.coords, mp.coords.data(), sizeof(float2) * mp.n,
                                cudaMemcpyHostToDevice, stream));
  }
  return {};
}

void siren_work_free(SirenWork& w) {
  pool_free(w.idx, w.stream);
  pool_free(w.coords, w.stream);
  pool_free(w.acts, w.stream);
  pool_free(w.wide_planes, w.stream);
  w.wide_planes = nullptr;
  w.wide_planes_floats = 0;
  pool_free(w.dA, w.stream);
  pool_free(w.dB, w.stream);
  pool_free(w.partial, w.stream);
  pool_free(w.wplanes, w.stream);
  w = SirenWork{};
}

static Status ensure_partial(SirenWork& w, size_t floats, cudaStream_t stream) {
  if (w.partial_floats >= floats) return {};
  pool_free(w.partial, stream);
  w.partial = nullptr;
  PACT_TRY_S(pool_alloc(reinterpret_cast<void**>(&w.partial), sizeof(float) * floats, stream));
  w.stream = stream;
  w.partial_floats = floats;
  return {};
}

// W (transposed = false) or W^T planes of every hidden layer into w.wide_planes:
// layer l (1 .. L-1) at (l - 1) * 2 + transposed planes slots.
static Status wide_planes(pact_ctx* ctx, const SirenShape& s, const float* theta, SirenWork& w,
                          bool transposed) {
  const size_t per = tc_wide_plane_floats();
  const size_t need = per * 2 * static_cast<size_t>(s.layers - 1);
  if (w.wide_planes_floats < need) {
    pool_free(w.wide_planes, w.stream ? w.stream : ctx->stream);
    w.wide_planes = nullptr;
    w.wide_planes_floats = 0;
    PACT_TRY_S(pool_alloc(reinterpret_cast<void**>(&w.wide_planes), sizeof(float) * need, ctx->stream));
    w.wide_planes_floats = need;
  }
  for (int l = 1; l < s.layers; ++l)
    PACT_TRY_S(tc_wide_planes(ctx, theta + s.offset(l), transposed,
                              w.wide_planes + per * (2 * (l - 1) + (transposed ? 1 : 0))));
  return {};
}

Status siren_forward(pact_ctx* ctx, const SirenShape& s, const float* theta, SirenWork& w,
                     float* dv) {
  const int n = w.n, H = s.hidden, L = s.layers;
  if (n == 0) return {};
  const float w0 = static_cast<float>(s.omega0);
  const size_t stride = static_cast<size_t>(n) * H;
  cudaStream_t st = ctx->stream;
  if (!tiled(s)) {
    siren_fwd_small_kernel<<<div_up(n, 128), 128, 0, st>>>(theta, w.coords, w.idx, n, H, L, w0,
                                                           static_cast<float>(s.out_scale), w.acts,
                                                           dv, stride);
    return after_launch(ctx, "siren_fwd_small_kernel");
  }
  // hidden width 128 on tcgen05: the whole network in one kernel
  // (PACT_SIREN_CHAIN=0 selects the per-layer kernels, for comparison)
  static const bool chain = [] {
    const char* e = std::getenv("PACT_SIREN_CHAIN");
    return !(e && e[0] == '0');
  }();
  if (chain && H == 128 && L >= 2 && siren_use_tc(H))
    return tc_forward_chain(ctx, s, theta, w, dv, !siren_fused_bwd(s));
  siren_first_kernel<<<ctx->num_sms * 8, 256, 0, st>>>(
      w.coords, theta + s.offset(0), theta + s.offset(0) + 2 * H, n, H, w.acts);
  PACT_TRY_S(after_launch(ctx, "siren_first_kernel"));
  const bool wide = siren_use_wide(H);
  if (wide) PACT_TRY_S(wide_planes(ctx, s, theta, w, false));
  for (int l = 1; l < L; ++l) {
    const float* W = theta + s.offset(l);
    const float* b = W + static_cast<size_t>(H) * H;
    const float* Ain = w.acts + (l - 1) * stride;
    float* Aout = w.acts + l * stride;
    if (wide) {
      PACT_TRY_S(tc_wide_forward_layer(ctx, Ain,
                                       w.wide_planes + tc_wide_plane_floats() * 2 * (l - 1), b, n,
                                       w0, Aout));
      continue;
    }
    if (siren_use_tc(H)) {
      SirenHead head;
      if (l == L - 1) {  // the output layer rides on the last layer's epilogue
        head.w = theta + s.offset(L);
        head.b = head.w + H;
        head.idx = w.idx;
        head.dv = dv;
        head.scale = static_cast<float>(s.out_scale);
      }
      PACT_TRY_S(tc_forward_layer(ctx, H, Ain, W, b, n, w0, Aout, head));
      continue;
    }
    if (H == 64) {
      siren_fwd_kernel<64><<<dim3(div_up(n, BM), 1), NT, 0, st>>>(Ain, W, b, n, H, w0, Aout);
    } else {
      siren_fwd_kernel<128><<<dim3(div_up(n, BM), H / 128), NT, 0, st>>>(Ain, W, b, n, H, w0, Aout);
    }
    PACT_TRY_S(after_launch(ctx, "siren_fwd_kernel"));
  }
  if (L >= 2 && siren_use_tc(H)) return {};  // output layer fused (tc_forward_layer)
  const float* wL = theta + s.offset(L);
  siren_out_kernel<<<std::min(div_up(n, 32), ctx->num_sms * 8), 256, 0, st>>>(w.acts + (L - 1) * stride, wL, wL + H,
                                                             w.idx, n, H, w0,
                                                             static_cast<float>(s.out_scale), dv);
  return after_launch(ctx, "siren_out_kernel");
}

Status siren_backward(pact_ctx* ctx, const SirenShape& s, const float* theta, SirenWork& w,
                      const double* gv, const float* gmask, double* grad) {
  const int n = w.n, H = s.hidden, L = s.layers;
  const int P = static_cast<int>(s.count());
  cudaStream_t st = ctx->stream;
  if (n == 0) {
    PACT_CUDA_S(cudaMemsetAsync(grad, 0, sizeof(double) * P, st));
    return {};
  }
  const float w0 = static_cast<float>(s.omega0);
  const float osc = static_cast<float>(s.out_scale);
  const size_t stride = static_cast<size_t>(n) * H;
  if (!tiled(s)) {
    PACT_TRY_S(ensure_partial(w, static_cast<size_t>(n) * P, st));
    siren_bwd_small_kernel<<<div_up(n, 128), 128, 0, st>>>(theta, w.coords, w.idx, n, H, L, w0, osc,
                                                           w.acts, stride, gv, gmask, w.dA,
                                                           w.partial, P);
    PACT_TRY_S(after_launch(ctx, "siren_bwd_small_kernel"));
    reduce_rows_kernel<<<div_up(P, 128), 128, 0, st>>>(w.partial, n, P, grad);
    return after_launch(ctx, "reduce_rows_kernel");
  }
  if (L + 1 > kMaxSeg) return validation("siren: too many layers for the segmented reduction");
  auto al64 = [](size_t x) { return (x + 63) & ~size_t(63); };
  ReduceSegs segs{};
  auto add_seg = [&](const float* src, int chunks, int per, double* dst) {
    const int k = segs.n++;
    segs.src[k] = src;
    segs.dst[k] = dst;
    segs.n_chunks[k] = chunks;
    segs.per[k] = per;
    segs.block_end[k] = (k ? segs.block_end[k - 1] : 0) + div_up(per, kRedP);
  };
  // hidden width 128 on tcgen05: one fused kernel per hidden layer (data +
  // weight gradient; the output layer folded into the top one, layer 0 into
  // the bottom one).  PACT_SIREN_FUSED_BWD=0 selects the per-op kernels.
  if (siren_fused_bwd(s)) {
    const int grid = tc_bwd_grid(ctx, n);
    const size_t per_w = static_cast<size_t>(H) * H + H;
    const size_t sz_w = al64(static_cast<size_t>(grid) * per_w),
                 sz_top = al64(static_cast<size_t>(grid) * (H + 1)),
                 sz_0 = static_cast<size_t>(grid) * 3 * H;
    const bool f16 = tc_bwd_f16();
    PACT_TRY_S(ensure_partial(w, sz_top + (L - 1) * sz_w + sz_0 + kMaxSeg, st));
    float* part_top = w.partial;
    float* part_w = part_top + sz_top;
    float* part_0 = part_w + (L - 1) * sz_w;
    // split fp16: the per-layer maxima that set the dA scales (siren_bwd16.cu)
    unsigned* mx = reinterpret_cast<unsigned*>(part_0 + sz_0);
    if (f16) PACT_CUDA_S(cudaMemsetAsync(mx, 0, sizeof(unsigned) * L, st));
    float* cur = w.dA;
    float* nxt = w.dB;
    for (int l = L - 1; l >= 1; --l) {
      const bool top = l == L - 1, bottom = l == 1;
      TcBwdLayer a;
      a.X = top ? w.acts + (L - 1) * stride : cur;
      a.Aprev = bottom ? nullptr : w.acts + (l - 1) * stride;
      a.W = theta + s.offset(l);
      a.gv = gv;
      a.gmask = gmask;
      a.idx = w.idx;
      a.wL = theta + s.offset(L);
      a.gpx = w.dA;  // free until the middle layer writes dA_{L-2} into it
      a.coords = w.coords;
      a.W0 = theta + s.offset(0);
      a.b0 = a.W0 + 2 * H;
      a.out_scale = osc;
      a.w0 = w0;
      a.n = n;
      a.Y = bottom ? nullptr : nxt;
      a.part_w = part_w + (l - 1) * sz_w;
      a.part_top = part_top;
      a.part_0 = part_0;
      if (f16)
        PACT_TRY_S(tc_bwd16_layer(ctx, top, bottom, a, mx + (L - 1 - l), mx + (L - l)));
      else
        PACT_TRY_S(tc_bwd_layer(ctx, top, bottom, a));
      add_seg(a.part_w, grid, static_cast<int>(per_w), grad + s.offset(l));
      std::swap(cur, nxt);
    }
    add_seg(part_top, grid, H + 1, grad + s.offset(L));
    add_seg(part_0, grid, 3 * H, grad + s.offset(0));
    reduce_segments_kernel<<<segs.block_end[segs.n - 1], dim3(kRedP, kRedG), 0, st>>>(segs);
    return after_launch(ctx, "reduce_segments_kernel");
  }
  // chunking for the split-M reductions
  const int tilesW = (H / 128 > 0 ? H / 128 : 1) * (H / 128 > 0 ? H / 128 : 1);
  const int rows_top = chunk_rows(n, 1, 4 * ctx->num_sms);
  const int n_top = div_up(n, rows_top);
  const bool use_tc = siren_use_tc(H), wide = siren_use_wide(H);
  int rows_w = chunk_rows(n, tilesW, ctx->num_sms);
  if (use_tc) rows_w = tc_wgrad_rows(ctx, n);
  if (wide) {
    rows_w = tc_wide_wgrad_rows(ctx, n);
    PACT_TRY_S(wide_planes(ctx, s, theta, w, true));  // W^T for the data gradients
  }
  const int n_w = div_up(n, rows_w);
  // one partial slice per reduction (top, each hidden layer, layer 0), summed
  // by a single segmented launch at the end
  // (slices start on 256-B boundaries: the weight-gradient kernels store vectors)
  const size_t per_w = static_cast<size_t>(H) * H + H;
  const size_t sz_top = al64(static_cast<size_t>(n_top) * (H + 1)),
               sz_w = al64(static_cast<size_t>(n_w) * per_w), sz_0 = static_cast<size_t>(n_top) * 3 * H;
  PACT_TRY_S(ensure_partial(w, sz_top + (L - 1) * sz_w + sz_0, st));
  float* part_top = w.partial;
  float* part_w = part_top + sz_top;  // layer l at part_w + (l - 1) sz_w
  float* part_0 = part_w + (L - 1) * sz_w;

  float* cur = w.dA;   // dA_l
  float* nxt = w.dB;   // dA_{l-1}
  // output layer
  const float* wL = theta + s.offset(L);
  {
    const float* aL = w.acts + (L - 1) * stride;
    switch (H) {
      case 64:
        siren_top_kernel<64><<<n_top, TopShape<64>::NTH, 0, st>>>(aL, wL, gv, gmask, w.idx, n,
                                                                  rows_top, w0, osc, cur, part_top);
        break;
      case 128:
        siren_top_kernel<128><<<n_top, TopShape<128>::NTH, 0, st>>>(aL, wL, gv, gmask, w.idx, n,
                                                                    rows_top, w0, osc, cur, part_top);
        break;
      case 192:
        siren_top_kernel<192><<<n_top, TopShape<192>::NTH, 0, st>>>(aL, wL, gv, gmask, w.idx, n,
                                                                    rows_top, w0, osc, cur, part_top);
        break;
      default:
        siren_top_kernel<256><<<n_top, TopShape<256>::NTH, 0, st>>>(aL, wL, gv, gmask, w.idx, n,
                                                                    rows_top, w0, osc, cur, part_top);
    }
  }
  PACT_TRY_S(after_launch(ctx, "siren_top_kernel"));
  add_seg(part_top, n_top, H + 1, grad + s.offset(L));
  for (int l = L - 1; l >= 1; --l) {
    const float* W = theta + s.offset(l);
    const float* Aprev = w.acts + (l - 1) * stride;
    float* part = part_w + (l - 1) * sz_w;
    // weight gradient of layer l
    if (use_tc)
      PACT_TRY_S(tc_wgrad_layer(ctx, H, cur, Aprev, n, rows_w, w0, part, n_w));
    else if (wide)
      PACT_TRY_S(tc_wide_wgrad_layer(ctx, cur, Aprev, n, rows_w, w0, part, n_w));
    else if (H == 64)
      siren_wgrad_kernel<64><<<dim3(n_w, 1, 1), NT, 0, st>>>(cur, Aprev, n, H, rows_w, w0, part);
    else
      siren_wgrad_kernel<128><<<dim3(n_w, H / 128, H / 128), NT, 0, st>>>(cur, Aprev, n, H, rows_w,
                                                                         w0, part);
    if (!use_tc && !wide) PACT_TRY_S(after_launch(ctx, "siren_wgrad_kernel"));
    add_seg(part, n_w, static_cast<int>(per_w), grad + s.offset(l));
    // delta to layer l-1
    if (use_tc)
      PACT_TRY_S(tc_dgrad_layer(ctx, H, cur, W, Aprev, n, w0, nxt));
    else if (wide)
      PACT_TRY_S(tc_wide_dgrad_layer(ctx, cur,
                                     w.wide_planes + tc_wide_plane_floats() * (2 * (l - 1) + 1),
                                     Aprev, n, w0, nxt));
    else if (H == 64)
      siren_dgrad_kernel<64><<<dim3(div_up(n, BM), 1), NT, 0, st>>>(cur, W, Aprev, n, H, w0, nxt);
    else
      siren_dgrad_kernel<128><<<dim3(div_up(n, BM), H / 128), NT, 0, st>>>(cur, W, Aprev, n, H, w0,
                                                                          nxt);
    if (!use_tc && !wide) PACT_TRY_S(after_launch(ctx, "siren_dgrad_kernel"));
    std::swap(cur, nxt);
  }
  switch (H) {
    case 64:
      siren_wgrad0_kernel<64><<<n_top, TopShape<64>::NTH, 0, st>>>(cur, w.coords, n, rows_top, part_0);
      break;
    case 128:
      siren_wgrad0_kernel<128><<<n_top, TopShape<128>::NTH, 0, st>>>(cur, w.coords, n, rows_top, part_0);
      break;
    case 192:
      siren_wgrad0_kernel<192><<<n_top, TopShape<192>::NTH, 0, st>>>(cur, w.coords, n, rows_top, part_0);
      break;
    default:
      siren_wgrad0_kernel<256><<<n_top, TopShape<256>::NTH, 0, st>>>(cur, w.coords, n, rows_top, part_0);
  }
  PACT_TRY_S(after_launch(ctx, "siren_wgrad0_kernel"));
  add_seg(part_0, n_top, 3 * H, grad + s.offset(0));
  reduce_segments_kernel<<<segs.block_end[segs.n - 1], dim3(kRedP, kRedG), 0, st>>>(segs);
  return after_launch(ctx, "reduce_segments_kernel");
}

}  // namespace pactgpu
