// Part 1 of the hot path: the multi-delay delay-and-sum stack.
//
// Reference semantics (das_stack, beamform.hpp:77-110; SignalSet::sample,
// core.hpp:296-304):  for pixel r and delay d_j
//     y_j(r) = sum_n S_n(s),  s = (1e-3 (|r - r_n| - d_j) / v0 - t0) / dt
// with S_n(s) linear interpolation of channel n, 0 for s < 0 or s > T-1 and the
// last sample at exactly s = T-1.
//
// B200 design:
//  * CTA = 16x16 pixel tile, one pixel per thread, KB delay accumulators in
//    registers.  Transducers are walked in chunks; for each (tile, transducer)
//    the time window that any tap of the tile can touch is computed
//    analytically (closest/farthest point of the tile rectangle) and staged in
//    shared memory, zero-filled outside [0, T-1].  Every tap is then two LDS.
//  * Index precision: the sample index reaches ~10^4, so fp32 |r - r_n| would
//    cost ~1e-4 relative L2.  |r - r_n| and the base index are
//    computed in fp64 once per (pixel, transducer); the K per-delay offsets are
//    fp32 fractions relative to that integer base, and floor() is done with the
//    1.5*2^23 magic-add so a tap costs ~10 FP32/INT issue slots.
//  * Out-of-window taps (edge semantics) take an exact per-tap path; with the
//    benchmark configs every tap is in-window and the fast path always runs.
//  * Small grids are split over transducer ranges (grid.z) so the launch fills
//    the 148 SMs; partial stacks are summed in a fixed order (deterministic).
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "simd.cuh"

namespace pactgpu {
namespace {

constexpr int kTile = 16;
constexpr int kThreads = kTile * kTile;
constexpr uint32_t kMagicIndexBias = 0x4B400000u;  // bits(2^23) + 2^22
constexpr float kMagic = 12582912.0f;                // 1.5 * 2^23
// Shared-memory window: interleaved (x[i], x[i+1] - x[i]) entries, so a tap
// is ONE 64-bit shared load (LDS.64) and one FFMA.
constexpr int kPlaneFloats = 6144;  // entries per window
constexpr size_t kWindowSmem = 8 * kPlaneFloats;

// (x[i], x[i+1] - x[i]) of window entry i: one LDS.64 (a half-warp per
// shared-memory wavefront; see the pixel mapping in das_stack_kernel).
__device__ __forceinline__ float2 lds_xd(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

template <int KB>
struct DelayConsts {
  float g[KB];  // -frac(c_j)
  float m[KB];  // 1.5*2^23 - floor(c_j)   (integer-valued, exact in fp32)
  int ci[KB];   // floor(c_j)
};

struct DasArgs {
  const float* sig;
  const double2* pos;
  int n_tx, n_samples;
  int width, height;
  double ox, oy, pitch;
  int row0;       // first grid row of the computed band (its rows are 0..height-1 here)
  double k_dist;  // samples per mm of path: 1e-3 / (v0 dt)
  double s_off;   // t0 / dt
  double cmin, cmax;
  int n_delays;   // delays in this block (<= KB)
  int cap;        // staged entries per transducer
  int chunk;      // transducers per staging round
  int tx_per_split;
  // 8 * (bits(2^23) + 2^22): runtime value so ptxas keeps one LEA per tap
  uint32_t bias8;
  float* out;     // [split][K_block][H][W]
  size_t split_stride;
  size_t plane;   // H*W
};

__device__ __forceinline__ double rect_min_dist(double px, double py, double x0, double x1,
                                                double y0, double y1) {
  double cx = fmin(fmax(px, x0), x1);
  double cy = fmin(fmax(py, y0), y1);
  double dx = px - cx, dy = py - cy;
  return sqrt(dx * dx + dy * dy);
}

__device__ __forceinline__ double rect_max_dist(double px, double py, double x0, double x1,
                                                double y0, double y1) {
  double dx = fmax(fabs(px - x0), fabs(px - x1));
  double dy = fmax(fabs(py - y0), fabs(py - y1));
  return sqrt(dx * dx + dy * dy);
}

// Window entry i is (x[i], x[i+1] - x[i]) so two LDS.32 and one FFMA produce
// the interpolated tap a + f*d.  Each warp covers an 8x4 pixel block, which
// keeps the sample spread of a warp under 32 words (one smem wavefront per
// LDS).  Index math runs two delays at a time in FADD2.
template <int KB>
__global__ void __launch_bounds__(kThreads, (KB <= 32 ? 3 : 2))
das_stack_kernel(DasArgs a, DelayConsts<KB> dc) {
  extern __shared__ float2 s_win[];  // [chunk][cap] (x, dx) entries
  __shared__ int s_lo[128];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  // warp = 8 x 4 pixels as two 4 x 4 half-warps: a 64-bit shared load is
  // served per half-warp, and a 4 x 4 block's samples of one transducer span
  // < 16 window entries at pitch <= 0.1 mm (conflict-free LDS.64)
  const int lx = (warp & 1) * 8 + (lane >> 4) * 4 + (lane & 3);
  const int ly = (warp >> 1) * 4 + ((lane >> 2) & 3);
  const int x0 = blockIdx.x * kTile, y0 = blockIdx.y * kTile;
  const int px = x0 + lx, py = y0 + ly;
  const bool active = px < a.width && py < a.height;
  const int xe = min(x0 + kTile, a.width) - 1, ye = min(y0 + kTile, a.height) - 1;

  const double rx0 = a.ox + x0 * a.pitch, rx1 = a.ox + xe * a.pitch;
  const double ry0 = a.oy + (y0 + a.row0) * a.pitch, ry1 = a.oy + (ye + a.row0) * a.pitch;
  // Pixel world position, GridSpec::world (core.hpp:71), in the full grid's
  // coordinates (a band of rows gives bit-identical values to the full stack).
  const double wx = a.ox + px * a.pitch, wy = a.oy + (py + a.row0) * a.pitch;

  const int n_begin = blockIdx.z * a.tx_per_split;
  const int n_end = min(a.n_tx, n_begin + a.tx_per_split);
  const int T = a.n_samples;
  const uint32_t smem_base = static_cast<uint32_t>(__cvta_generic_to_shared(s_win));

  f32x2 acc[KB / 2];
#pragma unroll
  for (int j = 0; j < KB / 2; ++j) acc[j] = 0ull;

  for (int n0 = n_begin; n0 < n_end; n0 += a.chunk) {
    const int cnt = min(a.chunk, n_end - n0);
    if (tid < cnt) {
      double2 p = __ldg(&a.pos[n0 + tid]);
      double dmin = rect_min_dist(p.x, p.y, rx0, rx1, ry0, ry1);
      double dmax = rect_max_dist(p.x, p.y, rx0, rx1, ry0, ry1);
      double smin = dmin * a.k_dist - a.s_off - a.cmax;
      double smax = dmax * a.k_dist - a.s_off - a.cmin;
      long lo = static_cast<long>(floor(smin)) - 2;
      long hi = static_cast<long>(floor(smax)) + 2;
      if (hi < 0 || lo > T - 1)
        s_lo[tid] = INT_MIN;  // every tap of the tile is out of window
      else
        s_lo[tid] = static_cast<int>(lo < 0 ? 0 : lo);
    }
    __syncthreads();
    // Stage the windows: contiguous per transducer, coalesced, zero outside [0, T-1].
    const int total = cnt * a.cap;
    // (nl, off) of entry e = nl * cap + off, advanced incrementally (no
    // integer division per staged entry)
    int nl = tid / a.cap, off = tid - nl * a.cap;
    for (int e = tid; e < total; e += kThreads) {
      int lo = s_lo[nl];
      float v0 = 0.f, v1 = 0.f;
      if (lo != INT_MIN) {
        int idx = lo + off;
        const float* row = a.sig + static_cast<size_t>(n0 + nl) * T;
        if (idx < T) v0 = __ldg(row + idx);
        if (idx + 1 < T) v1 = __ldg(row + idx + 1);
      }
      s_win[e] = make_float2(v0, v1 - v0);
      off += kThreads;
      while (off >= a.cap) {
        off -= a.cap;
        ++nl;
      }
    }
    __syncthreads();

    if (active) {
      for (int nl = 0; nl < cnt; ++nl) {
        const int lo = s_lo[nl];
        if (lo == INT_MIN) continue;
        double2 p = __ldg(&a.pos[n0 + nl]);
        double dx = wx - p.x, dy = wy - p.y;
        double dist = sqrt(dx * dx + dy * dy);
        double sb = dist * a.k_dist - a.s_off;
        double ibd = floor(sb);
        int ib = static_cast<int>(ibd);
        float fb = static_cast<float>(sb - ibd);
        const f32x2 fb2 = pack2(fb, fb);
        // byte address of tap j: 8*bits(t_j) + cbase (uint32 wrap-around)
        const uint32_t cbase =
            smem_base + 8u * static_cast<uint32_t>(ib - lo + nl * a.cap) - a.bias8;
        const bool fast = (sb - a.cmax >= 0.0) && (sb - a.cmin <= static_cast<double>(T - 1));
        if (fast) {
#pragma unroll
          for (int j = 0; j < KB; j += 2) {
            f32x2 m2 = pack2(dc.m[j], dc.m[j + 1]);
            f32x2 x2 = add2(fb2, pack2(dc.g[j], dc.g[j + 1]));
            f32x2 t2 = add2_rm(x2, m2);           // m_j + floor(x_j)
            f32x2 f2 = sub2(x2, sub2(t2, m2));    // frac
            float t0, t1, f0, f1;
            unpack2(t2, t0, t1);
            unpack2(f2, f0, f1);
            float2 v0 = lds_xd(mad_u32(__float_as_uint(t0), 8u, cbase));
            float2 v1 = lds_xd(mad_u32(__float_as_uint(t1), 8u, cbase));
            acc[j / 2] = add2(acc[j / 2], pack2(fmaf(f0, v0.y, v0.x), fmaf(f1, v1.y, v1.x)));
          }
        } else {
          // Exact SignalSet::sample edge semantics (core.hpp:296-304).
#pragma unroll
          for (int j = 0; j < KB; j += 2) {
            f32x2 m2 = pack2(dc.m[j], dc.m[j + 1]);
            f32x2 x2 = add2(fb2, pack2(dc.g[j], dc.g[j + 1]));
            f32x2 t2 = add2_rm(x2, m2);
            f32x2 r2 = sub2(t2, m2);
            f32x2 f2 = sub2(x2, r2);
            float t[2], f[2], r[2];
            unpack2(t2, t[0], t[1]);
            unpack2(f2, f[0], f[1]);
            unpack2(r2, r[0], r[1]);
            float val[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              int i = ib - dc.ci[j + h] + static_cast<int>(r[h]);
              bool valid = (i >= 0) && (i < T - 1 || (i == T - 1 && f[h] == 0.f));
              val[h] = 0.f;
              if (valid) {
                float2 v = lds_xd(mad_u32(__float_as_uint(t[h]), 8u, cbase));
                val[h] = fmaf(f[h], v.y, v.x);
              }
            }
            acc[j / 2] = add2(acc[j / 2], pack2(val[0], val[1]));
          }
        }
      }
    }
    __syncthreads();
  }

  if (active) {
    float* o = a.out + blockIdx.z * a.split_stride + static_cast<size_t>(py) * a.width + px;
#pragma unroll
    for (int j = 0; j < KB; j += 2) {
      float v0, v1;
      unpack2(acc[j / 2], v0, v1);
      if (j < a.n_delays) o[j * a.plane] = v0;
      if (j + 1 < a.n_delays) o[(j + 1) * a.plane] = v1;
    }
  }
}

// Fixed-order sum of the per-split partial stacks (deterministic).
__global__ void das_reduce_kernel(const float* __restrict__ part, int nsplit, size_t split_stride,
                                  size_t count, float* __restrict__ out) {
  size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (; i < count; i += stride) {
    float s = part[i];
    for (int k = 1; k < nsplit; ++k) s += part[k * split_stride + i];
    out[i] = s;
  }
}

template <int KB>
Status launch_block(pact_ctx* ctx, DasArgs a, const double* c, int nsplit, dim3 grid,
                    size_t smem) {
  DelayConsts<KB> dc;
  for (int j = 0; j < KB; ++j) {
    double cj = c[j < a.n_delays ? j : a.n_delays - 1];
    double fl = std::floor(cj);
    dc.ci[j] = static_cast<int>(fl);
    dc.g[j] = static_cast<float>(-(cj - fl));
    dc.m[j] = kMagic - static_cast<float>(fl);
  }
  PACT_TRY_S(smem_optin(das_stack_kernel<KB>, kWindowSmem));
  grid.z = nsplit;
  das_stack_kernel<KB><<<grid, kThreads, smem, ctx->stream>>>(a, dc);
  return after_launch(ctx, "das_stack_kernel");
}

}  // namespace

Status das_stack_device(pact_ctx* ctx, const pact_ring& ring, const pact_signal_meta& meta,
                        const float* signals, const pact_grid& full_grid, double v0,
                        const double* delays, int K, float* out, int row0, int rows) {
  // Validation order follows das_stack (beamform.hpp:79-85).
  if (K < 1) return validation("das_stack: need at least one delay");
  for (int j = 1; j < K; ++j)
    if (!(delays[j] > delays[j - 1]))
      return validation("das_stack: delays must be strictly increasing");
  if (ring.n_transducers < 3) return validation("ring: need at least 3 transducers");
  if (!(ring.radius > 0.0)) return validation("ring: radius must be > 0");
  if (meta.n_samples < 2) return validation("signals: need at least 2 samples");
  if (!(meta.dt > 0.0)) return validation("signals: dt must be > 0");
  if (full_grid.width < 1 || full_grid.height < 1)
    return validation("grid: width and height must be >= 1");
  if (!(full_grid.pitch > 0.0)) return validation("grid: pitch must be > 0");
  if (!(v0 > 0.0)) return validation("das_stack: v0 must be > 0");
  if (!signals || !out) return validation("das_stack: null buffer");
  // the band [row0, row0 + rows) of the grid (rows < 0: all of it)
  if (rows < 0) rows = full_grid.height - row0;
  if (row0 < 0 || rows < 1 || row0 + rows > full_grid.height)
    return internal_error("das_stack_device: bad row band");
  pact_grid grid = full_grid;
  grid.height = rows;

  const int N = ring.n_transducers, T = meta.n_samples;
  // Transducer positions in fp64, RingGeometry::transducer_position (core.hpp:162-165).
  std::vector<double2> pos(N);
  for (int n = 0; n < N; ++n) {
    double ang = 2.0 * M_PI * n / N + ring.angle_offset;
    pos[n] = make_double2(ring.radius * std::cos(ang), ring.radius * std::sin(ang));
  }
  void* dpos = nullptr;
  PACT_TRY_S(scratch_get(ctx, kScratchDasGeom, sizeof(double2) * N, &dpos));
  PACT_CUDA_S(cudaMemcpyAsync(dpos, pos.data(), sizeof(double2) * N, cudaMemcpyHostToDevice,
                              ctx->stream));

  const double k_dist = 1e-3 / (v0 * meta.dt);
  std::vector<double> c(K);
  for (int j = 0; j < K; ++j) c[j] = delays[j] * k_dist;

  const int tiles_x = div_up(grid.width, kTile), tiles_y = div_up(grid.height, kTile);
  const int tiles = tiles_x * tiles_y;
  const int full_tiles = tiles_x * div_up(full_grid.height, kTile);
  (void)tiles;
  const size_t plane = static_cast<size_t>(grid.width) * grid.height;

  DasArgs a{};
  a.sig = signals;
  a.pos = static_cast<const double2*>(dpos);
  a.n_tx = N;
  a.n_samples = T;
  a.width = grid.width;
  a.height = grid.height;
  a.ox = grid.origin_x;
  a.oy = grid.origin_y;
  a.row0 = row0;
  a.pitch = grid.pitch;
  a.k_dist = k_dist;
  a.s_off = meta.t0 / meta.dt;
  a.plane = plane;
  a.bias8 = 8u * kMagicIndexBias;

  const double diag = std::hypot((double)(kTile - 1), (double)(kTile - 1)) * grid.pitch;

  for (int jb = 0; jb < K;) {
    int kb = K - jb;
    int KBsel = kb <= 8 ? 8 : kb <= 16 ? 16 : kb <= 32 ? 32 : 64;
    kb = std::min(kb, 64);
    a.n_delays = kb;
    a.cmin = c[jb];
    a.cmax = c[jb + kb - 1];
    int span = static_cast<int>(std::ceil(diag * k_dist + (a.cmax - a.cmin))) + 12;
    int cap = span;
    int chunk = std::min(64, kPlaneFloats / cap);
    size_t smem = kWindowSmem;
    if (chunk < 1) {
      return validation("das_stack: per-tile time window exceeds shared memory "
                        "(pitch x tile diagonal + delay span too large)");
    }
    a.cap = cap;
    a.chunk = chunk;
    // Split the transducer range so the launch covers >= 2 waves of CTAs.
    // The split (and so the partial-sum order) follows the FULL grid's tile
    // count, so a row band's pixels are bit-identical to the full stack's.
    // Among the splits from there up, take the first whose CTA count fills
    // its last wave of resident CTAs (>= 95 %; else the fullest): cfg3's 1024
    // tiles are 2.3 waves of 3 x 148 CTAs unsplit, 6.9 waves split in three.
    const int want = div_up(2 * ctx->num_sms * 2, full_tiles);
    const int max_split = div_up(N, chunk);
    const double slots = static_cast<double>(ctx->num_sms) * (KBsel <= 32 ? 3 : 2);
    int nsplit = 1, per = N;
    double best = -1.0;
    for (int s = std::max(1, std::min(want, max_split)); s <= std::min(want + 5, max_split); ++s) {
      int p = div_up(div_up(N, s), chunk) * chunk;
      int ns = div_up(N, p);
      double waves = static_cast<double>(full_tiles) * ns / slots;
      double fill = waves / std::ceil(waves);
      if (fill > best + 1e-9) {
        best = fill;
        nsplit = ns;
        per = p;
      }
      if (fill >= 0.95) break;
    }
    a.tx_per_split = per;
    float* dst = out + static_cast<size_t>(jb) * plane;
    void* part = nullptr;
    if (nsplit > 1) {
      PACT_TRY_S(scratch_get(ctx, kScratchDasPartial,
                             sizeof(float) * plane * kb * static_cast<size_t>(nsplit), &part));
      a.out = static_cast<float*>(part);
      a.split_stride = plane * kb;
    } else {
      a.out = dst;
      a.split_stride = 0;
    }
    dim3 g(tiles_x, tiles_y, 1);
    const double* cb = c.data() + jb;
    Status st;
    switch (KBsel) {
      case 8: st = launch_block<8>(ctx, a, cb, nsplit, g, smem); break;
      case 16: st = launch_block<16>(ctx, a, cb, nsplit, g, smem); break;
      case 32: st = launch_block<32>(ctx, a, cb, nsplit, g, smem); break;
      default: st = launch_block<64>(ctx, a, cb, nsplit, g, smem); break;
    }
    PACT_TRY_S(st);
    if (nsplit > 1) {
      size_t count = plane * kb;
      int blocks = static_cast<int>(std::min<size_t>(div_up((int)std::min<size_t>(count, 1u << 30), 256),
                                                     ctx->num_sms * 8));
      das_reduce_kernel<<<blocks, 256, 0, ctx->stream>>>(static_cast<float*>(part), nsplit,
                                                        plane * kb, count, dst);
      PACT_TRY_S(after_launch(ctx, "das_reduce_kernel"));
    }
    jb += kb;
  }
  return {};
}

}  // namespace pactgpu

extern "C" int pact_das_stack(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                              const float* signals, const pact_grid* grid, double v0,
                              const double* delays, int32_t n_delays, float* out) {
  if (!ctx || !ring || !meta || !grid || (!delays && n_delays > 0))
    return pactgpu::validation("pact_das_stack: null argument").code;
  if (n_delays < 1) return pactgpu::validation("das_stack: need at least one delay").code;
  return pactgpu::das_stack_device(ctx, *ring, *meta, signals, *grid, v0, delays, n_delays, out, 0, -1)
      .code;
}
