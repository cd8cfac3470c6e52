// Part 2 (ray half) of the hot path: per-patch wavefront error profiles
// w(theta) by a straight-ray march through the SOS raster, and the adjoint
// scatter of dL/dw back onto the raster.
//
//   wavefront_profile    aberration.hpp:134-186
//   wavefront_grad_trace aberration.hpp:333-361
//
// B200 design: one thread per ray (patch, angle); a warp is 32 consecutive
// angles of one patch so its rays have near-equal lengths.  Ray setup is fp64
// (identical step counts to the reference); positions are fp64 per step and
// the bilinear stencil runs in fp32 on the *deviation* raster dv = v - v0,
// which keeps full relative precision of the integrand
// 1 - v0/v = dv / (v0 + dv).  The SOS raster (<= 16 MB) is L2-resident and
// read through the read-only path.
//
// The backward pass coalesces consecutive steps that share a stencil cell in
// registers (a step is 0.05 mm, a pixel 0.05-0.2 mm, and steps beyond the grid
// clamp onto one border cell for long runs) and flushes, skipping zero-weight
// corners, into 64-bit FIXED-POINT accumulators (integer RED.ADD.64): integer
// addition is associative, so the result is bitwise identical for any atomic
// order (deterministic by construction), and the integer reduction is faster
// than RED.ADD.F64 on B200 (scripts/probes/red_rate.cu).  The quantum 2^-S is
// set per launch from a deterministic bound on any pixel's total
// (ray_bound_kernel: max |dL/dw|, max 1/v^2 over the raster, the ray count and
// the longest possible ray), so no sum can overflow and the resolution is
// ~1e-10 of the largest single deposit; fix_to_grad_kernel converts to fp64.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "geom.cuh"
#include "train_ops.cuh"

// RAY_EXP (experiments only, never set in the product build): 1 = interior
// carries without atomics, 2 = interior without carries.
#ifndef RAY_EXP
#define RAY_EXP 0
#endif
// steps in flight per thread in the interior loops (texture gathers issued
// back to back before their results are used)
#ifndef RAY_FWD_UNROLL
#define RAY_FWD_UNROLL 8
#endif
#ifndef WF_MINB
#define WF_MINB 8  // 32 registers: 8 blocks per SM (0.181 vs 0.195 ms at 39 registers)
#endif
#ifndef CELL_MINB
#define CELL_MINB 3  // the tile tables (up to ~62 KB at cfg3) allow three 512-thread blocks per SM
#endif
#ifndef RAY_BWD_BATCH
#define RAY_BWD_BATCH 4
#endif
constexpr int kRayFwdUnroll = RAY_FWD_UNROLL;
#define RAY_NO_INT_ATOM (RAY_EXP == 1 || RAY_EXP == 6)
#define RAY_NO_LINE_ATOM (RAY_EXP == 5 || RAY_EXP == 6)

namespace pactgpu {

namespace {

// The grid border (left/right columns, bottom/top rows) cached in shared
// memory: every step beyond the grid samples only border pixels (the stencil
// clamps, aberration.hpp:49-55), which is most steps when the mask is the ring.
struct Border {
  float* colL;  // x = 0      [H]
  float* colR;  // x = W - 1  [H]
  float* rowB;  // y = 0      [W]
  float* rowT;  // y = H - 1  [W]
};

__device__ __forceinline__ Border load_border(const RayArgs& a, float* sm) {
  const int W = a.W, H = a.H;
  Border b{sm, sm + H, sm + 2 * H, sm + 2 * H + W};
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    b.colL[i] = __ldg(a.dv + static_cast<size_t>(i) * W);
    b.colR[i] = __ldg(a.dv + static_cast<size_t>(i) * W + W - 1);
  }
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    b.rowB[i] = __ldg(a.dv + i);
    b.rowT[i] = __ldg(a.dv + static_cast<size_t>(H - 1) * W + i);
  }
  __syncthreads();
  return b;
}

// a / b as __fdividef(a, b) computes it for a normal b (the ray integrands'
// denominators are SOS values or their squares): one MUFU.RCP and a multiply,
// without __fdividef's guard for |b| > 2^126.
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Fixed-point deposit target: int64 multiples of 2^-S (see the header).
// v * 2^S is exact in fp32 (a power-of-two scale; |v| 2^S < 2^62 by the
// bound), so one FMUL + F2I.S64 gives the same integer as an fp64 product.
struct Fix {
  unsigned long long* p;
  float scale;  // 2^S
  __device__ __forceinline__ Fix operator+(long long off) const { return {p + off, scale}; }
  __device__ __forceinline__ void add(float v) const {
    atomicAdd(p, static_cast<unsigned long long>(__float2ll_rn(v * scale)));
  }
};

// Per-launch exponent S from the bound statistics (ray_bound_kernel): every
// deposit is |g| dl v0 / v^2 * beta <= |g|max * step * v0 * max(1/v^2), and a
// pixel receives at most n_rays * max_steps of them; S keeps that below 2^62.
__device__ __forceinline__ int fix_exponent(const unsigned long long* stats, double step, double v0,
                                            double max_steps_total) {
  const double gmax = __longlong_as_double(static_cast<long long>(stats[0]));
  const double ivmax = __longlong_as_double(static_cast<long long>(stats[1]));
  const double B = gmax * step * v0 * ivmax * max_steps_total;
  if (!(B > 0.0) || !isfinite(B)) return 0;
  int e;
  frexp(B, &e);  // B < 2^e
  return min(max(62 - e, -126), 127);  // 2^S is a normal fp32 number
}

// The most deposits any pixel can receive in one launch: every ray's steps
// (a ray from inside the ring is at most one ring diameter long).
__host__ __device__ __forceinline__ double max_steps_total(const RayArgs& a) {
  return static_cast<double>(a.n_rays) * (ceil(2.0 * a.ring_r / a.step) + 1.0);
}

// One midpoint step: the clamped stencil of detail::bilinear_stencil and the
// four raster values under it, fetched from the cheapest source.
struct Step {
  int ix, iy;
  float w00, w01, w10, w11;
  float d;      // interpolated deviation
  bool corner;  // both coordinates clamped: the stencil is a single pixel from here on
};

template <bool TEX>
__device__ __forceinline__ Step step_at(const RayArgs& a, const Border& bd, float fxr, float fyr) {
  const int W = a.W, H = a.H;
  const float Wm1 = static_cast<float>(W - 1), Hm1 = static_cast<float>(H - 1);
  const bool xo = !(fxr >= 0.f && fxr <= Wm1), yo = !(fyr >= 0.f && fyr <= Hm1);
  const float fx = fminf(fmaxf(fxr, 0.f), Wm1), fy = fminf(fmaxf(fyr, 0.f), Hm1);
  Step s;
  s.ix = min(static_cast<int>(fx), max(W - 2, 0));
  s.iy = min(static_cast<int>(fy), max(H - 2, 0));
  const float ax = fx - s.ix, ay = fy - s.iy;
  s.w00 = (1.f - ax) * (1.f - ay);
  s.w01 = ax * (1.f - ay);
  s.w10 = (1.f - ax) * ay;
  s.w11 = ax * ay;
  s.corner = xo && yo;
  if (xo || yo) {
    // clamped: weights vanish off the border line (ax or ay is exactly 0 or 1)
    if (xo && !yo) {
      const float* col = fx == 0.f ? bd.colL : bd.colR;
      s.d = (1.f - ay) * col[s.iy] + ay * col[min(s.iy + 1, H - 1)];
    } else if (yo && !xo) {
      const float* row = fy == 0.f ? bd.rowB : bd.rowT;
      s.d = (1.f - ax) * row[s.ix] + ax * row[min(s.ix + 1, W - 1)];
    } else {
      const float* col = fx == 0.f ? bd.colL : bd.colR;
      s.d = col[fy == 0.f ? 0 : H - 1];
    }
  } else if (TEX) {
    // texel (i, j) centre at (i + 0.5, j + 0.5): the gather footprint of
    // (ix + 1, iy + 1) is exactly {ix, ix+1} x {iy, iy+1}
    float4 g = tex2Dgather<float4>(a.tex, s.ix + 1.f, s.iy + 1.f, 0);
    s.d = s.w00 * g.w + s.w01 * g.z + s.w10 * g.x + s.w11 * g.y;
  } else {
    const int ix1 = min(s.ix + 1, W - 1), iy1 = min(s.iy + 1, H - 1);
    s.d = s.w00 * __ldg(a.dv + s.iy * W + s.ix) + s.w01 * __ldg(a.dv + s.iy * W + ix1) +
          s.w10 * __ldg(a.dv + iy1 * W + s.ix) + s.w11 * __ldg(a.dv + iy1 * W + ix1);
  }
  return s;
}

// Pixel coordinates of the midpoint steps, f_i = f_s + i * df (GridSpec::pixel,
// core.hpp:75, of p_i = c + u (t0 + (i + 0.5) dl)): the start and increment
// are formed in fp64 once per ray; per step one FFMA (error ~1e-5 px), and the
// index from which both coordinates are off the grid (the corner regime).
struct RayPix {
  float fxs, fys, dfx, dfy;
  int i_corner;  // first step index with both coordinates outside (>= n: never)
};

__device__ __forceinline__ RayPix ray_pixels(const RayArgs& a, double cx, double cy, const Ray& ray) {
  const double fx0 = (cx - a.ox) * a.inv_pitch, fy0 = (cy - a.oy) * a.inv_pitch;
  const double sx = ray.ux * a.inv_pitch, sy = ray.uy * a.inv_pitch;
  const double s0 = ray.t0 + 0.5 * ray.dl;
  const double fxs = fx0 + s0 * sx, fys = fy0 + s0 * sy;
  const double dx = ray.dl * sx, dy = ray.dl * sy;
  auto exit_index = [](double f, double d, double hi) -> double {
    if (d > 0.0) return floor((hi - f) / d) + 1.0;
    if (d < 0.0) return floor(-f / d) + 1.0;
    return 1e30;
  };
  double ic = fmax(exit_index(fxs, dx, a.W - 1.0), exit_index(fys, dy, a.H - 1.0));
  RayPix p;
  p.fxs = static_cast<float>(fxs);
  p.fys = static_cast<float>(fys);
  p.dfx = static_cast<float>(dx);
  p.dfy = static_cast<float>(dy);
  p.i_corner = ic > 2e9 ? INT_MAX : static_cast<int>(fmax(ic, 0.0));
  return p;
}

// ---- generic per-step marches (any start position; the reference's branch
// structure step by step) ---------------------------------------------------
template <bool TEX>
__device__ float march_forward_generic(const RayArgs& a, const Border& bd, const RayPix& rp,
                                       int n, float v0) {
  float acc = 0.f;
  // steps that cannot be in the corner regime: no early exit, unrolled
  const int i_main = max(0, min(n, rp.i_corner - 2));
  int i = 0;
#pragma unroll 4
  for (; i < i_main; ++i) {
    Step st = step_at<TEX>(a, bd, fmaf(static_cast<float>(i), rp.dfx, rp.fxs),
                           fmaf(static_cast<float>(i), rp.dfy, rp.fys));
    acc += st.d / (v0 + st.d);  // (1 - v0/v), v = v0 + d
  }
  for (; i < n; ++i) {
    Step st = step_at<TEX>(a, bd, fmaf(static_cast<float>(i), rp.dfx, rp.fxs),
                           fmaf(static_cast<float>(i), rp.dfy, rp.fys));
    float term = st.d / (v0 + st.d);
    if (st.corner) {  // the ray moves outward: every remaining step is identical
      acc += static_cast<float>(n - i) * term;
      break;
    }
    acc += term;
  }
  return acc;
}

__device__ __forceinline__ void flush_cell(Fix g, int W, int H, int ix, int iy, const float acc[4]) {
  int ix1 = min(ix + 1, W - 1), iy1 = min(iy + 1, H - 1);
  if (acc[0] != 0.f) (g + (iy * W + ix)).add(acc[0]);
  if (acc[1] != 0.f) (g + (iy * W + ix1)).add(acc[1]);
  if (acc[2] != 0.f) (g + (iy1 * W + ix)).add(acc[2]);
  if (acc[3] != 0.f) (g + (iy1 * W + ix1)).add(acc[3]);
}

// Per-ray accumulators of the current stencil cell's pixels (cx + i, cy + j):
// a{j}{i}.  A pixel collects a handful of steps in fp32 before its fp64 flush;
// on a move, pixels shared with the new cell stay in registers (halves the
// atomics of a horizontal/vertical move).
struct CellAcc {
  int cx = -1, cy = -1;
  float a00 = 0.f, a01 = 0.f, a10 = 0.f, a11 = 0.f;

  __device__ __forceinline__ void move(Fix grad, int W, int ix, int iy) {
    if (ix == cx && iy == cy) return;
    if (cx >= 0) {
      const int dx = ix - cx, dy = iy - cy;
      float n00 = 0.f, n01 = 0.f, n10 = 0.f, n11 = 0.f;
      const float old[4] = {a00, a01, a10, a11};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ox = (q & 1) - dx, oy = (q >> 1) - dy;  // old pixel in the new cell
        const float val = old[q];
        if (ox >= 0 && ox <= 1 && oy >= 0 && oy <= 1) {
          const int t = oy * 2 + ox;
          n00 += t == 0 ? val : 0.f;
          n01 += t == 1 ? val : 0.f;
          n10 += t == 2 ? val : 0.f;
          n11 += t == 3 ? val : 0.f;
        } else if (val != 0.f && !RAY_NO_INT_ATOM) {
          (grad + ((cy + (q >> 1)) * W + cx + (q & 1))).add(val);
        }
      }
      a00 = n00;
      a01 = n01;
      a10 = n10;
      a11 = n11;
    }
    cx = ix;
    cy = iy;
  }
  // Interior move by at most one cell per axis (a step is <= 1 px): the
  // remap is a fixed select network and the evictions are predicated atomics
  // (no loop); larger jumps take the general path.
  __device__ __forceinline__ void move_unit(Fix grad, int W, int ix, int iy) {
    if (ix == cx && iy == cy) return;
    const int dx = ix - cx, dy = iy - cy;
    if (cx < 0 || dx < -1 || dx > 1 || dy < -1 || dy > 1) {
      move(grad, W, ix, iy);
      return;
    }
    // old slot (i, j) [x i, y j] survives iff (i - dx, j - dy) is in the new cell
    const bool keep_x0 = dx <= 0, keep_x1 = dx >= 0, keep_y0 = dy <= 0, keep_y1 = dy >= 0;
    if (!RAY_NO_INT_ATOM) {
      const Fix p = grad + (cy * W + cx);
      if (!(keep_x0 && keep_y0) && a00 != 0.f) p.add(a00);
      if (!(keep_x1 && keep_y0) && a01 != 0.f) (p + 1).add(a01);
      if (!(keep_x0 && keep_y1) && a10 != 0.f) (p + W).add(a10);
      if (!(keep_x1 && keep_y1) && a11 != 0.f) (p + (W + 1)).add(a11);
    }
    // x shift within each old row j: new x0 <- old (dx == 0 ? x0 : dx == 1 ? x1 : none)
    const float r00 = dx == 0 ? a00 : (dx == 1 ? a01 : 0.f);
    const float r01 = dx == 0 ? a01 : (dx == -1 ? a00 : 0.f);
    const float r10 = dx == 0 ? a10 : (dx == 1 ? a11 : 0.f);
    const float r11 = dx == 0 ? a11 : (dx == -1 ? a10 : 0.f);
    // then the y shift
    a00 = dy == 0 ? r00 : (dy == 1 ? r10 : 0.f);
    a01 = dy == 0 ? r01 : (dy == 1 ? r11 : 0.f);
    a10 = dy == 0 ? r10 : (dy == -1 ? r00 : 0.f);
    a11 = dy == 0 ? r11 : (dy == -1 ? r01 : 0.f);
    cx = ix;
    cy = iy;
  }
  __device__ __forceinline__ void flush(Fix grad, int W, int H) {
    if (cx < 0) return;
    const float fin[4] = {a00, a01, a10, a11};
    flush_cell(grad, W, H, cx, cy, fin);
    cx = cy = -1;
    a00 = a01 = a10 = a11 = 0.f;
  }
};

template <bool TEX>
__device__ void march_backward_generic(const RayArgs& a, const Border& bd, const RayPix& rp, int n,
                                       float v0, float gscale, Fix grad) {
  CellAcc c;
  for (int i = 0; i < n; ++i) {
    Step st = step_at<TEX>(a, bd, fmaf(static_cast<float>(i), rp.dfx, rp.fxs),
                           fmaf(static_cast<float>(i), rp.dfy, rp.fys));
    float v = v0 + st.d;
    float f = gscale / (v * v);
    const bool corner = st.corner && i >= rp.i_corner - 2;
    if (corner) f *= static_cast<float>(n - i);  // all remaining steps, same pixel
    c.move(grad, a.W, st.ix, st.iy);
    c.a00 = fmaf(f, st.w00, c.a00);
    c.a01 = fmaf(f, st.w01, c.a01);
    c.a10 = fmaf(f, st.w10, c.a10);
    c.a11 = fmaf(f, st.w11, c.a11);
    if (corner) break;
  }
  c.flush(grad, a.W, a.H);
}

// ---- regime-split marches (texture path, ray starts inside the grid) -------
// A ray from an interior point moves monotonically away in each coordinate,
// so its steps fall into three contiguous ranges: interior [0, i_side), one
// coordinate clamped (a 1-D interpolation along a border line) up to
// i_corner, and the corner (both clamped: one pixel) for the rest.  Each range
// is a branch-free loop; the range ends come from the same fp32 position
// formula the steps use, so the regime of every step matches step_at.
struct Regimes {
  int i_side, i_corner;
  bool x_first;  // x leaves the grid first: the side range runs along a column
};

__device__ __forceinline__ bool out_at(int i, float fs, float df, float hi) {
  const float f = fmaf(static_cast<float>(i), df, fs);
  return !(f >= 0.f && f <= hi);
}

// First step index in [0, n] whose coordinate is off [0, hi] (n: never).
__device__ int first_out(float fs, float df, float hi, int n) {
  double g;
  if (df > 0.f)
    g = floor((static_cast<double>(hi) - fs) / df) + 1.0;
  else if (df < 0.f)
    g = floor(-static_cast<double>(fs) / df) + 1.0;
  else
    g = static_cast<double>(n);
  int i = static_cast<int>(fmin(fmax(g, 0.0), static_cast<double>(n)));
  while (i > 0 && out_at(i - 1, fs, df, hi)) --i;
  while (i < n && !out_at(i, fs, df, hi)) ++i;
  return i;
}

__device__ __forceinline__ Regimes regimes(const RayPix& rp, int n, float Wm1, float Hm1) {
  const int ix = first_out(rp.fxs, rp.dfx, Wm1, n), iy = first_out(rp.fys, rp.dfy, Hm1, n);
  return {min(ix, iy), max(ix, iy), ix < iy};
}

// The border line a ray runs along once one coordinate has left the grid:
// the moving coordinate f = fs + i df and its line in the smem border
// [colL H | colR H | rowB W | rowT W] (offset off, cells 0..qmax).
struct SideLine {
  float fs, df;
  int off, qmax;
};

__device__ __forceinline__ SideLine side_line(const Regimes& rg, const RayPix& rp, int W, int H) {
  SideLine s;
  if (rg.x_first) {
    s.fs = rp.fys;
    s.df = rp.dfy;
    s.off = rp.dfx > 0.f ? H : 0;
    s.qmax = H - 2;
  } else {
    s.fs = rp.fxs;
    s.df = rp.dfx;
    s.off = 2 * H + (rp.dfy > 0.f ? W : 0);
    s.qmax = W - 2;
  }
  return s;
}


__device__ __forceinline__ float interior_d(cudaTextureObject_t tex, float fx, float fy, int W,
                                            int H, float& ax, float& ay, int& ix, int& iy) {
  ix = min(static_cast<int>(fx), W - 2);
  iy = min(static_cast<int>(fy), H - 2);
  ax = fx - ix;
  ay = fy - iy;
  // texel (i, j) centre at (i + 0.5, j + 0.5): the gather footprint of
  // (ix + 1, iy + 1) is {ix, ix+1} x {iy, iy+1}: w=(ix,iy) z=(ix+1,iy) x=(ix,iy+1) y=(ix+1,iy+1)
  const float4 g = tex2Dgather<float4>(tex, ix + 1.f, iy + 1.f, 0);
  const float top = fmaf(ax, g.z - g.w, g.w);
  const float bot = fmaf(ax, g.y - g.x, g.x);
  return fmaf(ay, bot - top, top);
}

// 1-D carry along a border line: pixels (line position q, q + 1).
struct LineAcc {
  int q = -1;
  float b0 = 0.f, b1 = 0.f;
  __device__ __forceinline__ void move(Fix grad, int nq, int stride, int base) {
    if (nq == q) return;
    if (q >= 0 && !RAY_NO_LINE_ATOM) {
      if (nq == q + 1) {
        if (b0 != 0.f) (grad + (base + q * stride)).add(b0);
        b0 = b1;
        b1 = 0.f;
      } else if (nq == q - 1) {
        if (b1 != 0.f) (grad + (base + (q + 1) * stride)).add(b1);
        b1 = b0;
        b0 = 0.f;
      } else {
        if (b0 != 0.f) (grad + (base + q * stride)).add(b0);
        if (b1 != 0.f) (grad + (base + (q + 1) * stride)).add(b1);
        b0 = b1 = 0.f;
      }
    }
    q = nq;
  }
  __device__ __forceinline__ void flush(Fix grad, int stride, int base) {
    if (q < 0) return;
    if (b0 != 0.f) (grad + (base + q * stride)).add(b0);
    if (b1 != 0.f) (grad + (base + (q + 1) * stride)).add(b1);
  }
};

// Border deposits: every ray of every patch that leaves the grid deposits on
// the same 2(W + H) border pixels (and 4 corners), so global atomics there
// contend.  They go to one of kBorderReplicas copies of the border (by block)
// and border_reduce_kernel folds the copies into the raster afterwards in a
// fixed order.  Replica layout: [R][colL H | colR H | rowB W | rowT W].
#ifndef RAY_REPLICAS
#define RAY_REPLICAS 32
#endif
constexpr int kBorderReplicas = RAY_REPLICAS;

// ---- planned marches -------------------------------------------------------
// The ray geometry (centres, angles, mask, grid) is fixed for a whole
// reconstruction; only the raster changes.  ray_plan_get therefore computes
// once per geometry each ray's record (fp64 setup, regime boundaries) and a
// work list: each ray's interior and border-line step ranges cut into chunks
// of at most kRayChunk steps, sorted by (regime, length) so that the 32 lanes
// of a warp run equal trip counts of the same loop.  Block b takes items
// [256 b, 256 b + 256), longest work first; consecutive items are adjacent
// rays at the same distance, so an SM's resident warps march one neighbourhood
// of the raster (texture-cache locality).  (A persistent variant with a work
// counter measured slower: 0.73 vs 0.53 ms for the cfg3 adjoint, and it
// starves the concurrent frames' kernels.)  The forward pass writes one
// partial sum per item and ray_finish_kernel adds each ray's partials in a
// fixed order; the adjoint flushes its carries per item.
constexpr int kRecGeneric = 1;  // starts outside the grid: per-step generic march
constexpr int kRecXFirst = 2;   // x leaves the grid first

enum ItemKind { kItemInterior = 0, kItemSide = 1, kItemGeneric = 2 };
// item = {ray, lo, hi, slot | kind << 28 | corner << 30}
__device__ __forceinline__ int item_kind(int w) { return (w >> 28) & 3; }
__device__ __forceinline__ bool item_corner(int w) { return (w >> 30) & 1; }
__device__ __forceinline__ int item_slot(int w) { return w & 0x0fffffff; }

__global__ void ray_plan_kernel(RayArgs a, RayRec* __restrict__ rec) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n_rays) return;
  const int patch = r / a.n_angles, ang = r - patch * a.n_angles;
  const double2 c = a.centers[patch];
  const Ray ray = make_ray(c.x, c.y, ang, a.n_angles, a.ring_r, a.mcx, a.mcy, a.mr, a.step);
  RayRec o{};
  o.n = ray.n;
  o.dl = ray.dl;
  if (ray.n > 0) {
    const RayPix rp = ray_pixels(a, c.x, c.y, ray);
    o.fxs = rp.fxs;
    o.fys = rp.fys;
    o.dfx = rp.dfx;
    o.dfy = rp.dfy;
    const float Wm1 = static_cast<float>(a.W - 1), Hm1 = static_cast<float>(a.H - 1);
    if (out_at(0, rp.fxs, rp.dfx, Wm1) || out_at(0, rp.fys, rp.dfy, Hm1)) {
      o.flags = kRecGeneric;
      o.i_corner = rp.i_corner;
    } else {
      const Regimes rg = regimes(rp, ray.n, Wm1, Hm1);
      o.i_side = rg.i_side;
      o.i_corner = rg.i_corner;
      o.flags = rg.x_first ? kRecXFirst : 0;
    }
  }
  rec[r] = o;
}

__device__ __forceinline__ RayPix rec_pixels(const RayRec& r) {
  return {r.fxs, r.fys, r.dfx, r.dfy, r.i_corner};
}

__device__ __forceinline__ Regimes rec_regimes(const RayRec& r) {
  return {r.i_side, r.i_corner, (r.flags & kRecXFirst) != 0};
}

template <bool kSeries>
__global__ void __launch_bounds__(256, WF_MINB) wavefront_plan_kernel(RayArgs a) {
  extern __shared__ float s_border[];
  const Border bd = load_border(a, s_border);
  const int W = a.W, H = a.H;
  const float v0 = static_cast<float>(a.v0);
  {
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= a.n_items) return;
    const int4 item = a.items[it];
    const RayRec rr = a.rec[item.x];
    const int lo = item.y, hi = item.z, kind = item_kind(item.w);
    float acc = 0.f;
    if (kind == kItemInterior) {
#pragma unroll kRayFwdUnroll
      for (int i = lo; i < hi; ++i) {
        float ax, ay;
        int ix, iy;
        const float d = interior_d(a.tex, fmaf(static_cast<float>(i), rr.dfx, rr.fxs),
                                   fmaf(static_cast<float>(i), rr.dfy, rr.fys), W, H, ax, ay, ix,
                                   iy);
        acc += d * rcp_approx(v0 + d);
      }
    } else if (kind == kItemSide) {
      // border line: one loop for both orientations; the line is a slice of
      // the smem border
      const SideLine sl = side_line(rec_regimes(rr), rec_pixels(rr), W, H);
      if (kSeries) {
        // Run by run: inside one border cell d is linear in the step index,
        // d_i = dm + beta k about the run's centre, v_i = vm (1 + u k), and
        //   sum_i d_i / v_i = (dm n - v0 (u^2 S2 + u^4 S4)) / vm,  S2 = sum k^2, S4 = sum k^4
        // (odd power sums vanish; |u k| <= |c1 - c0| / (2 vm); u^6 dropped:
        // < 1e-6 of the sum while |u| n <= 0.2, else the steps are summed).
        // A step on a cell boundary may count for either cell: d is continuous.
        const float adf = fabsf(sl.df);
        const float rdf = adf > 0.f ? rcp_approx(adf) : 0.f;
        int i = lo;
        while (i < hi) {
          const float f = fmaf(static_cast<float>(i), sl.df, sl.fs);
          const int q = min(static_cast<int>(f), sl.qmax);
          const float fa = f - q;
          const float room = sl.df > 0.f ? 1.f - fa : fa;  // to the cell's far boundary
          // steps left in the cell, >= 1 (the conversion saturates; NaN -> 0)
          const int n = adf > 0.f ? min(static_cast<int>(fmaxf(room, 0.f) * rdf), hi - i - 1) + 1 : hi - i;
          const float nf = static_cast<float>(n);
          const float c0 = s_border[sl.off + q], dc = s_border[sl.off + q + 1] - c0;
          const float dm = fmaf(fmaf(0.5f * (nf - 1.f), sl.df, fa), dc, c0);
          const float rv = rcp_approx(v0 + dm);
          const float u = dc * sl.df * rv;
          if (fabsf(u) * nf <= 0.2f) {
            const float n2 = nf * nf, u2 = u * u;
            const float S2 = nf * (n2 - 1.f) * (1.f / 12.f);
            const float S4 = S2 * fmaf(3.f, n2, -7.f) * (1.f / 20.f);
            acc = fmaf(rv, fmaf(dm, nf, -v0 * u2 * fmaf(u2, S4, S2)), acc);
          } else {
            for (int j = i; j < i + n; ++j) {
              const float d = fmaf(fmaf(static_cast<float>(j), sl.df, sl.fs) - q, dc, c0);
              acc += d * rcp_approx(v0 + d);
            }
          }
          i += n;
        }
      } else {
#pragma unroll 4
        for (int i = lo; i < hi; ++i) {
          const float f = fmaf(static_cast<float>(i), sl.df, sl.fs);
          const int q = min(static_cast<int>(f), sl.qmax);
          const float c0 = s_border[sl.off + q];
          const float d = fmaf(f - q, s_border[sl.off + q + 1] - c0, c0);
          acc += d * rcp_approx(v0 + d);
        }
      }
    } else {
      acc = march_forward_generic<true>(a, bd, rec_pixels(rr), rr.n, v0);
    }
    if (item_corner(item.w)) {  // both coordinates clamped: one pixel to the end
      const float* col = rr.dfx > 0.f ? bd.colR : bd.colL;
      const float d = col[rr.dfy > 0.f ? H - 1 : 0];
      acc += static_cast<float>(rr.n - rr.i_corner) * __fdividef(d, v0 + d);
    }
    a.partial[item_slot(item.w)] = acc;
  }
}

// w[r] = dl * (sum of the ray's item partials, in item order).
__global__ void ray_finish_kernel(RayArgs a, float* __restrict__ w) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n_rays) return;
  const int2 sl = a.ray_slots[r];
  float acc = 0.f;
  for (int k = 0; k < sl.y; ++k) acc += a.partial[sl.x + k];
  w[r] = static_cast<float>(a.rec[r].dl) * acc;
}

// (256, 4): at most 64 registers, four blocks per SM (0.53 vs 0.56 ms at 68)
// Items [skip_lo, skip_lo + skip_n) (the interior items, when the cell gather
// takes them) are not run: thread t takes item t, or t + skip_n past skip_lo.
__global__ void __launch_bounds__(256, 4) ray_backward_plan_kernel(RayArgs a, const float* __restrict__ dw,
                                                                  unsigned long long* __restrict__ acc,
                                                                  unsigned long long* __restrict__ border_rep,
                                                                  const unsigned long long* __restrict__ stats,
                                                                  int skip_lo, int skip_n) {
  extern __shared__ float s_border[];
  const Border bd = load_border(a, s_border);
  const int W = a.W, H = a.H;
  const float v0 = static_cast<float>(a.v0);
  const float scale = ldexpf(1.f, fix_exponent(stats, a.step, a.v0, max_steps_total(a)));
  const Fix grad{acc, scale};
  const Fix rep{border_rep + static_cast<size_t>(blockIdx.x % kBorderReplicas) * 2 * (W + H), scale};
  {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int it = t < skip_lo ? t : t + skip_n;
    if (it >= a.n_items) return;
    const int4 item = a.items[it];
    const float gr = dw[item.x];
    if (gr == 0.f) return;  // aberration.hpp:340
    const RayRec rr = a.rec[item.x];
    // f = g * dl * v0 / v^2 per step (aberration.hpp:354-355)
    const float gscale = static_cast<float>(static_cast<double>(gr) * rr.dl * a.v0);
    const int lo = item.y, hi = item.z, kind = item_kind(item.w);
    if (kind == kItemInterior) {
      // gathers issued RAY_BWD_BATCH steps at a time, then the carries
      CellAcc cell;
      constexpr int NB = RAY_BWD_BATCH;
      for (int i = lo; i < hi; i += NB) {
        float4 gt[NB];
        float ax[NB], ay[NB];
        int ix[NB], iy[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const float k = static_cast<float>(min(i + u, hi - 1));
          const float fx = fmaf(k, rr.dfx, rr.fxs), fy = fmaf(k, rr.dfy, rr.fys);
          ix[u] = min(static_cast<int>(fx), W - 2);
          iy[u] = min(static_cast<int>(fy), H - 2);
          ax[u] = fx - ix[u];
          ay[u] = fy - iy[u];
          gt[u] = tex2Dgather<float4>(a.tex, ix[u] + 1.f, iy[u] + 1.f, 0);
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          if (i + u < hi) {
            // gather order: w=(ix,iy) z=(ix+1,iy) x=(ix,iy+1) y=(ix+1,iy+1)
            const float top = fmaf(ax[u], gt[u].z - gt[u].w, gt[u].w);
            const float bot = fmaf(ax[u], gt[u].y - gt[u].x, gt[u].x);
            const float v = v0 + fmaf(ay[u], bot - top, top);
            const float f = __fdividef(gscale, v * v);
            if (RAY_EXP != 2) cell.move_unit(grad, W, ix[u], iy[u]);
            const float fy1 = f * ay[u], fy0 = f - fy1;  // f (1 - ay), f ay
            cell.a00 = fmaf(-fy0, ax[u], cell.a00 + fy0);
            cell.a01 = fmaf(fy0, ax[u], cell.a01);
            cell.a10 = fmaf(-fy1, ax[u], cell.a10 + fy1);
            cell.a11 = fmaf(fy1, ax[u], cell.a11);
          }
        }
      }
      cell.flush(grad, W, H);
    } else if (kind == kItemSide) {
      // border line (one loop for both orientations); the replica slice has
      // the smem border's layout
      const SideLine sl = side_line(rec_regimes(rr), rec_pixels(rr), W, H);
      const Fix dst = rep + sl.off;
      // The carry of LineAcc without its branches: a step moves the cell by
      // at most one (|df| <= 1 px per step; larger jumps take LineAcc::move),
      // so the eviction is a select and one predicated atomic.
      LineAcc line;
      line.q = min(static_cast<int>(fmaf(static_cast<float>(lo), sl.df, sl.fs)), sl.qmax);
      float b0 = 0.f, b1 = 0.f;
      int lq = line.q;
      for (int i = lo; i < hi; ++i) {
        const float f = fmaf(static_cast<float>(i), sl.df, sl.fs);
        const int q = min(static_cast<int>(f), sl.qmax);
        const float fa = f - q, c0 = s_border[sl.off + q];
        const float v = v0 + fmaf(fa, s_border[sl.off + q + 1] - c0, c0);
        const float gv = gscale * rcp_approx(v * v);
        const int dq = q - lq;
        if (dq > 1 || dq < -1) {  // rare: the general move
          line.q = lq;
          line.b0 = b0;
          line.b1 = b1;
          line.move(dst, q, 1, 0);
          b0 = line.b0;
          b1 = line.b1;
        } else {
          const bool up = dq == 1, dn = dq == -1;
          const float ev = up ? b0 : (dn ? b1 : 0.f);
          if (ev != 0.f && !RAY_NO_LINE_ATOM) (dst + (up ? lq : lq + 1)).add(ev);
          const float n0 = up ? b1 : (dn ? 0.f : b0), n1 = up ? 0.f : (dn ? b0 : b1);
          b0 = n0;
          b1 = n1;
        }
        lq = q;
        const float g1 = gv * fa;
        b0 += gv - g1;
        b1 += g1;
      }
      line.q = lq;
      line.b0 = b0;
      line.b1 = b1;
      line.flush(dst, 1, 0);
    } else {
      march_backward_generic<true>(a, bd, rec_pixels(rr), rr.n, v0, gscale, grad);
    }
    if (item_corner(item.w)) {
      const int px = rr.dfx > 0.f ? W - 1 : 0, py = rr.dfy > 0.f ? H - 1 : 0;
      const float* col = rr.dfx > 0.f ? bd.colR : bd.colL;
      const float v = v0 + col[py];
      const float f = __fdividef(gscale, v * v) * static_cast<float>(rr.n - rr.i_corner);
      if (f != 0.f) (rep + ((px == 0 ? 0 : H) + py)).add(f);
    }
  }
}

// Border replicas -> the raster accumulator: one thread per border slot
// ([colL H | colR H | rowB W | rowT W]; consecutive threads, consecutive
// slots), its kBorderReplicas loads issued back to back; the integer sum is
// exact, so folding it into acc with an integer atomic keeps the result
// order-independent.  Slots are reset.
// With a side plan the border cells' sums (side_gather_kernel<true>) join in:
// slot s takes the lower pixel sum of cell s and the upper of cell s - 1 (same
// line).
__global__ void border_fold_kernel(unsigned long long* __restrict__ rep, int W, int H,
                                   const unsigned long long* __restrict__ side_cells,
                                   unsigned long long* __restrict__ acc) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_slots = 2 * (W + H);
  if (slot >= n_slots) return;
  const size_t stride = static_cast<size_t>(n_slots);
  unsigned long long part[kBorderReplicas];
#pragma unroll
  for (int r = 0; r < kBorderReplicas; ++r) part[r] = rep[r * stride + slot];
  unsigned long long v = 0ull;
#pragma unroll
  for (int r = 0; r < kBorderReplicas; ++r) {
    v += part[r];
    if (part[r]) rep[r * stride + slot] = 0ull;
  }
  if (side_cells) {
    const int len = slot < 2 * H ? H : W;
    const int pos = slot < H ? slot : slot < 2 * H ? slot - H : slot < 2 * H + W ? slot - 2 * H : slot - 2 * H - W;
    if (pos <= len - 2) v += side_cells[2 * slot];
    if (pos >= 1) v += side_cells[2 * (slot - 1) + 1];
  }
  if (v == 0ull) return;
  int px, py;
  if (slot < 2 * H) {
    px = slot < H ? 0 : W - 1;
    py = slot < H ? slot : slot - H;
  } else {
    const int q = slot - 2 * H;
    px = q < W ? q : q - W;
    py = q < W ? 0 : H - 1;
  }
  atomicAdd(acc + static_cast<size_t>(py) * W + px, v);
}

// grad[p] += (acc[p] + the pixel's four cell-gather corners) 2^-S, one thread
// per pixel (exact integer sums); the accumulator is reset for the next
// launch, so the raster needs no per-launch memset.
__global__ void fix_to_grad_kernel(unsigned long long* __restrict__ acc, int W, int H,
                                   const unsigned long long* __restrict__ stats, double step,
                                   double v0, double max_steps,
                                   const unsigned long long* __restrict__ cells,
                                   double* __restrict__ grad) {
  const int S = fix_exponent(stats, step, v0, max_steps);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W * H) return;
  unsigned long long v = acc[i];
  if (v != 0ull) acc[i] = 0ull;
  if (cells) {  // cell (x, y) holds corners [(x,y), (x+1,y), (x,y+1), (x+1,y+1)]
    const int y = i / W, x = i - y * W, Wc = W - 1, Hc = H - 1;
    if (x < Wc && y < Hc) v += cells[4 * (y * Wc + x) + 0];
    if (x > 0 && y < Hc) v += cells[4 * (y * Wc + x - 1) + 1];
    if (x < Wc && y > 0) v += cells[4 * ((y - 1) * Wc + x) + 2];
    if (x > 0 && y > 0) v += cells[4 * ((y - 1) * Wc + x - 1) + 3];
  }
  if (v != 0ull) grad[i] += ldexp(static_cast<double>(static_cast<long long>(v)), -S);
}

// Bound statistics of one adjoint launch (exact maxima, order-independent):
// stats[0] = max |dL/dw| over the rays, stats[1] = max 1 / v^2 over the
// raster = 1 / min(v)^2 (non-negative doubles order like their bit patterns).
// With a cell plan it also writes each ray's deposit scale
// gsc[r] = dL/dw[r] dl v0 (aberration.hpp:354-355; 0 for rays the reference
// skips, aberration.hpp:340).
__global__ void __launch_bounds__(256) ray_bound_kernel(const float* __restrict__ dw, int n_rays,
                                                        const float* __restrict__ dv, int npx,
                                                        float v0, const RayRec* __restrict__ rec,
                                                        double v0d, float* __restrict__ gsc,
                                                        unsigned long long* __restrict__ stats) {
  __shared__ float s_g[8], s_v[8];
  float g = 0.f, vmin = INFINITY;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_rays; i += stride) {
    const float d = dw[i], x = fabsf(d);
    g = x != x ? INFINITY : fmaxf(g, x);  // NaN -> infinite bound
    if (gsc) gsc[i] = d == 0.f ? 0.f : static_cast<float>(static_cast<double>(d) * rec[i].dl * v0d);
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npx; i += stride) {
    const float x = dv[i];
    vmin = x != x ? -INFINITY : fminf(vmin, x);
  }
  for (int o = 16; o > 0; o >>= 1) {
    g = fmaxf(g, __shfl_xor_sync(0xffffffffu, g, o));
    vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
  }
  if ((threadIdx.x & 31) == 0) {
    s_g[threadIdx.x >> 5] = g;
    s_v[threadIdx.x >> 5] = vmin;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
    g = fmaxf(g, s_g[w]);
    vmin = fminf(vmin, s_v[w]);
  }
  const double v = static_cast<double>(v0) + static_cast<double>(vmin);
  const double iv = v > 0.0 ? 1.0 / (v * v) : INFINITY;
  // the statistics only grow: skip the atomic when they already exceed ours
  const auto gb = static_cast<unsigned long long>(__double_as_longlong(static_cast<double>(g)));
  const auto ib = static_cast<unsigned long long>(__double_as_longlong(iv));
  if (g != 0.f && *reinterpret_cast<volatile unsigned long long*>(stats) < gb) atomicMax(stats, gb);
  if (*reinterpret_cast<volatile unsigned long long*>(stats + 1) < ib) atomicMax(stats + 1, ib);
}

// ---- cell-gather adjoint of the interior steps -------------------------------
// The interior adjoint as a gather.  The plan (build_cell_plan) lists, per
// stencil cell, every interior step (ray, step index) whose stencil is that
// cell, sorted by (ray, step).  One block per tile of cell_t x cell_t cells
// first stages the line and deposit scale of every ray crossing the tile in
// shared memory; then half a warp per cell walks the cell's list with the
// cell's four raster values in registers, so a step is arithmetic on shared
// operands -- no texture gather, no carry, no atomic -- on exactly the
// positions, stencil values and weights of the per-ray march.  A cell's lanes
// sum their steps in fp32 and combine them by a fixed shuffle tree; the four
// corner sums go to `cells` in the 64-bit fixed-point quantum of fix_exponent,
// and fix_to_grad_kernel adds each pixel's four corners as integers, so the
// result is deterministic by construction.
constexpr int kCellBatch = 4;  // list entries per lane whose loads are in flight together
constexpr int LPC = 8;         // lanes per cell

struct CellTiles {  // tile-major cell numbering
  int T, tx, Wc, Hc;
  __host__ __device__ __forceinline__ int cell(int cx, int cy) const {
    return ((cy / T) * tx + cx / T) * T * T + (cy % T) * T + cx % T;
  }
  __host__ __device__ __forceinline__ int tile(int cx, int cy) const { return (cy / T) * tx + cx / T; }
};

__device__ __forceinline__ void cell_xy(const RayRec& q, int i, int W, int H, int& cx, int& cy) {
  cx = min(static_cast<int>(fmaf(static_cast<float>(i), q.dfx, q.fxs)), W - 2);
  cy = min(static_cast<int>(fmaf(static_cast<float>(i), q.dfy, q.fys)), H - 2);
}

__device__ __forceinline__ int interior_steps(const RayRec& q) {
  return q.n > 0 && !(q.flags & kRecGeneric) ? q.i_side : 0;
}

// Pass A (per ray): its interior steps' keys cell << 32 | r << sb | i at
// keys[off[r] ..], the (tile, ray) pairs of the tiles it crosses (a straight
// line crosses a convex tile once) at tkeys[toff[r] ..] or, with tkeys null,
// their count in tcnt[r]; and the ray's line in geo.
__global__ void cell_steps_kernel(const RayRec* __restrict__ rec, int n_rays, int W, int H, int sb,
                                  CellTiles ct, const unsigned long long* __restrict__ off,
                                  unsigned long long* __restrict__ keys,
                                  const unsigned long long* __restrict__ toff,
                                  unsigned long long* __restrict__ tkeys, unsigned* __restrict__ tcnt,
                                  float4* __restrict__ geo) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const RayRec q = rec[r];
  if (geo) geo[r] = make_float4(q.fxs, q.fys, q.dfx, q.dfy);
  const int n_int = interior_steps(q);
  int prev = -1;
  unsigned nt = 0;
  for (int i = 0; i < n_int; ++i) {
    int cx, cy;
    cell_xy(q, i, W, H, cx, cy);
    if (keys)
      keys[off[r] + i] = (static_cast<unsigned long long>(ct.cell(cx, cy)) << 32) |
                         (static_cast<unsigned long long>(r) << sb) | static_cast<unsigned>(i);
    const int t = ct.tile(cx, cy);
    if (t != prev) {
      if (tkeys) tkeys[toff[r] + nt] = (static_cast<unsigned long long>(t) << 32) | static_cast<unsigned>(r);
      ++nt;
      prev = t;
    }
  }
  if (tcnt) tcnt[r] = nt;
}

// Sorted keys (group << shift | value) -> the per-group ranges
// start[0 .. n_groups] and (shift 32, val non-null) the 32-bit values.
__global__ void group_bounds_kernel(const unsigned long long* __restrict__ keys, unsigned n,
                                    int n_groups, int shift, unsigned* __restrict__ start,
                                    unsigned* __restrict__ val) {
  const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const unsigned long long key = keys[k];
  const int c = static_cast<int>(key >> shift);
  if (val) val[k] = static_cast<unsigned>(key);
  const int prev = k == 0 ? -1 : static_cast<int>(keys[k - 1] >> shift);
  for (int q = prev + 1; q <= c; ++q) start[q] = k;
  if (k == n - 1)
    for (int q = c + 1; q <= n_groups; ++q) start[q] = n;
}

// Pass B (per entry): the ray id -> its index in the tile's sorted ray list.
__global__ void cell_localize_kernel(const unsigned long long* __restrict__ keys, unsigned n, int sb,
                                     int T, const unsigned* __restrict__ tile_start,
                                     const unsigned* __restrict__ tile_rays,
                                     unsigned* __restrict__ ent) {
  const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const unsigned long long key = keys[k];
  const int t = static_cast<int>(key >> 32) / (T * T);
  const unsigned e = static_cast<unsigned>(key), r = e >> sb;
  unsigned lo = tile_start[t], hi = tile_start[t + 1];
  while (lo < hi) {  // lower bound (r is present)
    const unsigned mid = (lo + hi) >> 1;
    if (tile_rays[mid] < r) lo = mid + 1; else hi = mid;
  }
  ent[k] = ((lo - tile_start[t]) << sb) | (e & ((1u << sb) - 1u));
}

__device__ __forceinline__ float cell_sum(float v) {  // fixed xor tree over the cell's lanes
#pragma unroll
  for (int o = LPC / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One block (kCellThreads) per tile of T x T cells; dynamic smem: tile_max ray
// lines (float4) + deposit scales (float).
constexpr int kCellThreads = 512;

template <int T>
__global__ void __launch_bounds__(kCellThreads, CELL_MINB) cell_gather_kernel(RayArgs a, const float* __restrict__ gsc,
                                                          const unsigned long long* __restrict__ stats,
                                                          unsigned long long* __restrict__ cells) {
  extern __shared__ float4 s_geo[];
  float* s_g = reinterpret_cast<float*>(s_geo + a.tile_max);
  const int W = a.W, H = a.H, Wc = W - 1, Hc = H - 1;
  const int tile = blockIdx.x, tx = (Wc + T - 1) / T;
  const int tile_x0 = (tile % tx) * T, tile_y0 = (tile / tx) * T;
  const unsigned r0 = a.tile_start[tile], nr = a.tile_start[tile + 1] - r0;
  for (unsigned j = threadIdx.x; j < nr; j += blockDim.x) {
    const unsigned r = __ldg(a.tile_rays + r0 + j);
    s_geo[j] = __ldg(a.cell_geo + r);
    s_g[j] = __ldg(gsc + r);
  }
  __syncthreads();
  const float scale = ldexpf(1.f, fix_exponent(stats, a.step, a.v0, max_steps_total(a)));
  const float v0 = static_cast<float>(a.v0);
  const int sb = a.cell_sb;
  const unsigned smask = (1u << sb) - 1u;
  const int lane = threadIdx.x & 31, l16 = lane % LPC, half = threadIdx.x / LPC;
  const int halves = blockDim.x / LPC;
  for (int lc = half; lc < T * T; lc += halves) {  // uniform per half-warp; rounds uniform per warp
    const int cx = tile_x0 + lc % T, cy = tile_y0 + lc / T;
    const bool live = cx < Wc && cy < Hc;
    const int ccx = min(cx, Wc - 1), ccy = min(cy, Hc - 1);
    const float q00 = __ldg(a.dv + ccy * W + ccx), q01 = __ldg(a.dv + ccy * W + ccx + 1);
    const float q10 = __ldg(a.dv + (ccy + 1) * W + ccx), q11 = __ldg(a.dv + (ccy + 1) * W + ccx + 1);
    const float dtop = q01 - q00, dbot = q11 - q10;
    const float fcx = static_cast<float>(ccx), fcy = static_cast<float>(ccy);
    const int c = tile * T * T + lc;
    const unsigned e0 = live ? a.cell_start[c] : 0u, e1 = live ? a.cell_start[c + 1] : 0u;
    // the four moments of the cell's deposits f = g / v^2 (the corner sums
    // follow from them after the loop: five instructions per step, not eight)
    float F = 0.f, Fx = 0.f, Fy = 0.f, Fxy = 0.f;
    // software pipeline: the next batch of entries loads while this one runs.
    // Lanes past the list re-read its last entry with g = 0: every lane
    // evaluates a real step of this cell (v > 0), so f needs no guard.
    unsigned nx[kCellBatch];
#pragma unroll
    for (int u = 0; u < kCellBatch; ++u) {
      const unsigned q = e0 + l16 + LPC * u;
      nx[u] = e1 > e0 ? __ldg(a.cell_ent + min(q, e1 - 1u)) : 0u;
    }
    for (unsigned e = e0 + l16; e < e1; e += LPC * kCellBatch) {
      unsigned en[kCellBatch];
#pragma unroll
      for (int u = 0; u < kCellBatch; ++u) {
        en[u] = nx[u];
        const unsigned q = e + LPC * (kCellBatch + u);
        nx[u] = __ldg(a.cell_ent + min(q, e1 - 1u));
      }
#pragma unroll
      for (int u = 0; u < kCellBatch; ++u) {
        // the per-ray march's interior_d arithmetic, operand for operand
        const unsigned j = en[u] >> sb;
        const float4 geo = s_geo[j];
        const float g = e + LPC * u < e1 ? s_g[j] : 0.f;  // (0 too for rays the reference skips, aberration.hpp:340)
        const float fi = static_cast<float>(en[u] & smask);
        const float ax = fmaf(fi, geo.z, geo.x) - fcx, ay = fmaf(fi, geo.w, geo.y) - fcy;
        const float top = fmaf(ax, dtop, q00), bot = fmaf(ax, dbot, q10);
        const float v = v0 + fmaf(ay, bot - top, top);
        const float f = g * rcp_approx(v * v);
        const float fy = f * ay;
        F += f;
        Fy += fy;
        Fx = fmaf(f, ax, Fx);
        Fxy = fmaf(fy, ax, Fxy);
      }
    }
    F = cell_sum(F);
    Fx = cell_sum(Fx);
    Fy = cell_sum(Fy);
    Fxy = cell_sum(Fxy);
    // corner sums: sum f (1-ax)(1-ay), f ax (1-ay), f (1-ax) ay, f ax ay
    const float r11 = Fxy, r10 = Fy - Fxy, r01 = Fx - Fxy, r00 = (F - Fy) - r01;
    if (live && l16 == 0) {
      unsigned long long* o = cells + 4 * static_cast<size_t>(cy * Wc + cx);
      o[0] = static_cast<unsigned long long>(__float2ll_rn(r00 * scale));
      o[1] = static_cast<unsigned long long>(__float2ll_rn(r01 * scale));
      o[2] = static_cast<unsigned long long>(__float2ll_rn(r10 * scale));
      o[3] = static_cast<unsigned long long>(__float2ll_rn(r11 * scale));
    }
  }
}

// ---- border-line (side) steps as a gather --------------------------------------
// Once one coordinate has left the grid the stencil clamps onto a border line,
// so a ray's side steps are a 1-D march along that line: runs of steps in
// one border cell (two raster values).  The plan lists every run under its
// border cell, sorted by length (so a warp's lanes run near-equal loops);
// one block per border cell holds the cell's two values in registers and
// walks its runs: the per-ray adjoint's step arithmetic operand for operand,
// without the smem border cache, the carry or the atomics; each run's two
// pixel sums are converted to the fixed-point quantum once and reduced per
// cell as integers.  (The forward keeps its per-ray border-line items: with
// no carry they cost about the same per step, and a ray's sum stays whole.)
constexpr int kSideThreads = 256;
constexpr int kSideMaxRun = 255;
constexpr int kSideBatch = 4;  // runs per thread whose loads are in flight together

__device__ __forceinline__ int side_range(const RayRec& q, int& i1) {
  const bool ok = q.n > 0 && !(q.flags & kRecGeneric);
  i1 = ok ? min(q.i_corner, q.n) : 0;
  return ok ? q.i_side : 0;
}

// Runs of ray r's side steps: count (pass 0, keys null) or the keys at
// keys[off[r] ..] (pass 1); and the ray's border line.
__global__ void side_runs_kernel(const RayRec* __restrict__ rec, int n_rays, int W, int H,
                                 const unsigned long long* __restrict__ off,
                                 unsigned long long* __restrict__ keys, unsigned* __restrict__ cnt,
                                 float2* __restrict__ geo) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const RayRec q = rec[r];
  int i1;
  const int i0 = side_range(q, i1);
  const SideLine sl = side_line(rec_regimes(q), rec_pixels(q), W, H);
  if (geo) geo[r] = make_float2(sl.fs, sl.df);
  unsigned m = 0;
  int prev = -1, first = i0;
  auto emit = [&](int slot, int a0, int a1) {
    for (int b = a0; b < a1; b += kSideMaxRun) {  // long runs in pieces of <= 255 steps
      const int c = min(kSideMaxRun, a1 - b);
      if (keys)
        keys[off[r] + m] = (static_cast<unsigned long long>(slot) << 48) |
                           (static_cast<unsigned long long>(kSideMaxRun - c) << 40) |
                           (static_cast<unsigned long long>(r) << 20) |
                           (static_cast<unsigned long long>(b) << 8);
      ++m;
    }
  };
  for (int i = i0; i < i1; ++i) {
    const int slot = sl.off + min(static_cast<int>(fmaf(static_cast<float>(i), sl.df, sl.fs)), sl.qmax);
    if (slot != prev) {
      if (prev >= 0) emit(prev, first, i);
      prev = slot;
      first = i;
    }
  }
  if (prev >= 0) emit(prev, first, i1);
  if (cnt) cnt[r] = m;
}

// Raster index of border slot s ([colL H | colR H | rowB W | rowT W]).
__device__ __forceinline__ int border_pixel(int s, int W, int H) {
  if (s < 2 * H) return (s < H ? s : s - H) * W + (s < H ? 0 : W - 1);
  const int q = s - 2 * H;
  return (q < W ? 0 : H - 1) * W + (q < W ? q : q - W);
}

// One block per border cell (slot): cell_out[slot] = the cell's two pixel
// sums (lower, upper) in the fixed-point quantum.
template <bool kSideSeries>
__global__ void __launch_bounds__(kSideThreads) side_gather_kernel(RayArgs a, const float* __restrict__ gsc,
                                                                   const unsigned long long* __restrict__ stats,
                                                                   unsigned long long* __restrict__ cell_out) {
  const int slot = blockIdx.x, W = a.W, H = a.H;
  const unsigned e0 = a.side_start[slot], e1 = a.side_start[slot + 1];
  if (e0 == e1) {  // (empty cell: zeros, so the fold reads no stale value)
    if (threadIdx.x == 0) cell_out[2 * slot] = cell_out[2 * slot + 1] = 0ull;
    return;
  }
  const int q = slot < 2 * H ? (slot < H ? slot : slot - H) : (slot - 2 * H < W ? slot - 2 * H : slot - 2 * H - W);
  const float c0 = __ldg(a.dv + border_pixel(slot, W, H)), c1 = __ldg(a.dv + border_pixel(slot + 1, W, H));
  const float dc = c1 - c0, fq = static_cast<float>(q), v0 = static_cast<float>(a.v0);
  const float scale = ldexpf(1.f, fix_exponent(stats, a.step, a.v0, max_steps_total(a)));
  long long s0 = 0, s1 = 0;
  // kSideBatch runs per thread in flight: the entries, then the rays' scales
  // and lines (scattered L2 gathers), then the arithmetic
  for (unsigned k = e0 + threadIdx.x; k < e1; k += kSideThreads * kSideBatch) {
    unsigned long long ent[kSideBatch];
    float gs[kSideBatch];
    float2 geos[kSideBatch];
#pragma unroll
    for (int t = 0; t < kSideBatch; ++t) {
      const unsigned kk = k + t * kSideThreads;
      ent[t] = kk < e1 ? __ldg(a.side_ent + kk) : 0ull;
    }
#pragma unroll
    for (int t = 0; t < kSideBatch; ++t) {
      const unsigned kk = k + t * kSideThreads;
      const int r = static_cast<int>((ent[t] >> 20) & 0xfffffu);
      gs[t] = kk < e1 ? __ldg(gsc + r) : 0.f;
      geos[t] = __ldg(a.side_geo + r);
    }
#pragma unroll
    for (int t = 0; t < kSideBatch; ++t) {
      const unsigned long long e = ent[t];
      const int i0 = static_cast<int>((e >> 8) & 0xfffu);
      const int cnt = kSideMaxRun - static_cast<int>((e >> 40) & 0xffu);
      const float g = gs[t];
      if (g == 0.f) continue;  // aberration.hpp:340
      const float2 geo = geos[t];
      float b0 = 0.f, b1 = 0.f;
      // Inside one border cell v is linear in the step index: v_i = vm (1 + u k),
      // k = i - (the run's centre), so the run's two deposits
      //   sum_i g / v_i^2 (1 - fa_i),  sum_i g / v_i^2 fa_i        (fa_i = fam + k geo.y)
      // are power series in u k with the odd power sums gone by symmetry:
      //   sum 1/v_i^2 = (n + 3 u^2 S2 + 5 u^4 S4) / vm^2,  S2 = sum k^2, S4 = sum k^4
      //   sum k/v_i^2 = -(2 u S2 + 4 u^3 S4) / vm^2
      // |u k| <= |c1 - c0| / (2 vm) (a run stays in its cell), so the u^6 term
      // dropped is < 1e-6 of the sum while |u| n <= 0.2; beyond that (a field
      // with a > 20 % jump between border neighbours) the steps are summed.
      const float nf = static_cast<float>(cnt);
      const float ic = static_cast<float>(i0) + 0.5f * (nf - 1.f);
      const float fam = fmaf(ic, geo.y, geo.x - fq);
      const float rv = rcp_approx(v0 + fmaf(fam, dc, c0));
      const float u = dc * geo.y * rv;
      if (kSideSeries && fabsf(u) * nf <= 0.2f) {
        const float n2 = nf * nf, u2 = u * u;
        const float S2 = nf * (n2 - 1.f) * (1.f / 12.f);
        const float S4 = S2 * fmaf(3.f, n2, -7.f) * (1.f / 20.f);
        const float T0 = fmaf(u2, fmaf(5.f * u2, S4, 3.f * S2), nf);
        const float T1 = -u * fmaf(4.f * u2, S4, 2.f * S2);
        const float gr = g * rv * rv;
        b1 = gr * fmaf(geo.y, T1, fam * T0);
        b0 = fmaf(gr, T0, -b1);
      } else {
        // the per-ray border-line march's arithmetic (ray_backward_plan_kernel)
        for (int i = i0; i < i0 + cnt; ++i) {
          const float fa = fmaf(static_cast<float>(i), geo.y, geo.x) - fq;
          const float v = v0 + fmaf(fa, dc, c0);
          const float gv = g * rcp_approx(v * v);
          const float g1 = gv * fa;
          b0 += gv - g1;
          b1 += g1;
        }
      }
      s0 += __float2ll_rn(b0 * scale);
      s1 += __float2ll_rn(b1 * scale);
    }
  }
  // integer block sums: exact, so the order does not matter
  __shared__ long long r0[kSideThreads / 32], r1[kSideThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    r0[threadIdx.x >> 5] = s0;
    r1[threadIdx.x >> 5] = s1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t0 = 0, t1 = 0;
    for (int w = 0; w < kSideThreads / 32; ++w) {
      t0 += r0[w];
      t1 += r1[w];
    }
    cell_out[2 * slot] = static_cast<unsigned long long>(t0);
    cell_out[2 * slot + 1] = static_cast<unsigned long long>(t1);
  }
}

// The corner runs of the adjoint (both coordinates clamped: every remaining
// step on one corner pixel), one thread per ray, into the border replicas.
__global__ void corner_adjoint_kernel(RayArgs a, const float* __restrict__ gsc,
                                      const unsigned long long* __restrict__ stats,
                                      unsigned long long* __restrict__ border_rep) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n_rays) return;
  const RayRec rr = a.rec[r];
  if (rr.n <= 0 || (rr.flags & kRecGeneric) || rr.i_corner >= rr.n) return;
  const float g = gsc[r];
  if (g == 0.f) return;
  const int W = a.W, H = a.H;
  const int px = rr.dfx > 0.f ? W - 1 : 0, py = rr.dfy > 0.f ? H - 1 : 0;
  const float v = static_cast<float>(a.v0) + __ldg(a.dv + py * W + px);
  const float f = __fdividef(g, v * v) * static_cast<float>(rr.n - rr.i_corner);
  if (f == 0.f) return;
  const float scale = ldexpf(1.f, fix_exponent(stats, a.step, a.v0, max_steps_total(a)));
  unsigned long long* rep = border_rep + static_cast<size_t>(r % kBorderReplicas) * 2 * (W + H);
  atomicAdd(rep + (px == 0 ? 0 : H) + py, static_cast<unsigned long long>(__float2ll_rn(f * scale)));
}

// Generic kernels (plain loads, no texture): one per-step march per ray.
template <bool TEX>
__global__ void __launch_bounds__(256) wavefront_kernel(RayArgs a, float* __restrict__ w) {
  extern __shared__ float s_border[];
  const Border bd = load_border(a, s_border);
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n_rays) return;
  int patch = r / a.n_angles, ang = r - patch * a.n_angles;
  double2 c = a.centers[patch];
  Ray ray = make_ray(c.x, c.y, ang, a.n_angles, a.ring_r, a.mcx, a.mcy, a.mr, a.step);
  const RayPix rp = ray_pixels(a, c.x, c.y, ray);
  const float acc = march_forward_generic<TEX>(a, bd, rp, ray.n, static_cast<float>(a.v0));
  w[r] = static_cast<float>(ray.dl) * acc;
}

template <bool TEX>
__global__ void __launch_bounds__(256) ray_backward_kernel(RayArgs a, const float* __restrict__ dw,
                                                           unsigned long long* __restrict__ acc,
                                                           const unsigned long long* __restrict__ stats) {
  extern __shared__ float s_border[];
  const Border bd = load_border(a, s_border);
  const Fix grad{acc, ldexpf(1.f, fix_exponent(stats, a.step, a.v0, max_steps_total(a)))};
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n_rays) return;
  const float gr = dw[r];
  if (gr == 0.f) return;  // aberration.hpp:340
  int patch = r / a.n_angles, ang = r - patch * a.n_angles;
  double2 c = a.centers[patch];
  Ray ray = make_ray(c.x, c.y, ang, a.n_angles, a.ring_r, a.mcx, a.mcy, a.mr, a.step);
  if (ray.n == 0) return;
  const RayPix rp = ray_pixels(a, c.x, c.y, ray);
  const float gscale = static_cast<float>(static_cast<double>(gr) * ray.dl * a.v0);
  march_backward_generic<TEX>(a, bd, rp, ray.n, static_cast<float>(a.v0), gscale, grad);
}

}  // namespace

bool make_raster_texture(const float* dv, int W, int H, cudaTextureObject_t* out) {
  *out = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  int align = 0;
  if (cudaDeviceGetAttribute(&align, cudaDevAttrTexturePitchAlignment, dev) != cudaSuccess)
    return false;
  const size_t pitch = sizeof(float) * static_cast<size_t>(W);
  if (W < 2 || H < 2 || align <= 0 || pitch % align != 0 ||
      reinterpret_cast<uintptr_t>(dv) % align != 0)
    return false;
  cudaResourceDesc res{};
  res.resType = cudaResourceTypePitch2D;
  res.res.pitch2D.devPtr = const_cast<float*>(dv);
  res.res.pitch2D.desc = cudaCreateChannelDesc<float>();
  res.res.pitch2D.width = W;
  res.res.pitch2D.height = H;
  res.res.pitch2D.pitchInBytes = pitch;
  cudaTextureDesc td{};
  td.addressMode[0] = cudaAddressModeClamp;
  td.addressMode[1] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  if (cudaCreateTextureObject(out, &res, &td, nullptr) != cudaSuccess) {
    cudaGetLastError();
    *out = 0;
    return false;
  }
  return true;
}

Status ray_args(const pact_ring& ring, const pact_grid& grid, double v0, const pact_mask& mask,
                int n_angles, double step, RayArgs& a) {
  if (ring.n_transducers < 3) return validation("ring: need at least 3 transducers");
  if (!(ring.radius > 0.0)) return validation("ring: radius must be > 0");
  if (n_angles < 4) return validation("wavefront_profile: need at least 4 angles");
  if (!(step > 0.0)) return validation("wavefront_profile: step must be > 0");
  if (grid.width < 1 || grid.height < 1) return validation("grid: width and height must be >= 1");
  if (!(grid.pitch > 0.0)) return validation("grid: pitch must be > 0");
  a.W = grid.width;
  a.H = grid.height;
  a.ox = grid.origin_x;
  a.oy = grid.origin_y;
  a.inv_pitch = 1.0 / grid.pitch;
  a.v0 = v0;
  a.ring_r = ring.radius;
  a.mcx = mask.center_x;
  a.mcy = mask.center_y;
  a.mr = mask.radius;
  a.step = step;
  a.n_angles = n_angles;
  return {};
}

Status validate_centers(const pact_ring& ring, int n, const double* centers) {
  for (int i = 0; i < n; ++i)
    if (std::hypot(centers[2 * i], centers[2 * i + 1]) >= ring.radius)
      return validation("wavefront_profile: patch center outside the transducer ring");
  return {};
}

// ---- ray plans ---------------------------------------------------------------
namespace {

constexpr int kRayChunk = 128;  // max steps per work item (PACT_RAY_CHUNK overrides)
constexpr int kPlanBlock = 256;
constexpr int kLenBucket = 32;

int ray_chunk() {
  static const int c = [] {
    const char* e = std::getenv("PACT_RAY_CHUNK");
    const int v = e ? std::atoi(e) : 0;
    return v >= 8 ? v : kRayChunk;
  }();
  return c;
}

}  // namespace

// Immutable part of a plan, shared by every owner of the same geometry.
struct RayPlanData {
  void* mem = nullptr;  // rec | items | ray_slots (cudaMalloc)
  const RayRec* rec = nullptr;
  const int4* items = nullptr;
  const int2* ray_slots = nullptr;
  int n_items = 0;
  int n_gen = 0, n_int = 0;  // items are sorted generic | interior | side
  // cell-gather plan of the interior adjoint (null: none, see build_cell_plan)
  void* cell_mem = nullptr;
  void* tile_mem = nullptr;
  const unsigned* cell_start = nullptr;
  const unsigned* cell_ent = nullptr;
  const unsigned* tile_start = nullptr;
  const unsigned* tile_rays = nullptr;
  const float4* cell_geo = nullptr;
  int cell_sb = 0, cell_t = 0, tile_max = 0, n_tiles = 0;
  // border-line (side) plan (null: none, see build_side_plan)
  void* side_mem = nullptr;
  const unsigned long long* side_ent = nullptr;
  const unsigned* side_start = nullptr;
  const float2* side_geo = nullptr;
  unsigned n_side = 0;
  std::vector<double> key;
  ~RayPlanData() {
    if (mem) cudaFree(mem);
    if (cell_mem) cudaFree(cell_mem);
    if (tile_mem) cudaFree(tile_mem);
    if (side_mem) cudaFree(side_mem);
  }
};

namespace {

std::vector<double> plan_key(const RayArgs& a, const double* centers, int n_centers) {
  std::vector<double> key = {static_cast<double>(a.W), static_cast<double>(a.H), a.ox, a.oy,
                             a.inv_pitch, a.ring_r, a.mcx, a.mcy, a.mr, a.step,
                             static_cast<double>(a.n_angles), static_cast<double>(a.n_rays)};
  key.insert(key.end(), centers, centers + 2 * n_centers);
  return key;
}

bool cells_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PACT_RAY_CELLS");
    return !(e && e[0] == '0');
  }();
  return on;
}

int bits_for(unsigned long long v) {  // bits to hold 0..v
  int b = 0;
  while (b < 64 && (v >> b) != 0ull) ++b;
  return std::max(b, 1);
}

// The cell-gather plan (see cell_gather_kernel), built once per geometry:
// every interior step of every ray keyed (cell, ray, step) and radix-sorted;
// per tile, the sorted list of rays crossing it; each entry's ray replaced by
// its index in its tile's list.  The tile edge is 16 cells, or 8 when a
// tile's ray table would not fit in shared memory.  Skipped (the interior
// items stay on the per-ray kernel) when an entry does not fit 32 bits or
// PACT_RAY_CELLS=0.  Synchronous.
constexpr size_t kCellSmemMax = 160 * 1024;

Status build_cell_plan(pact_ctx* ctx, cudaStream_t s, const RayArgs& a, RayPlanData& p) {
  if (!cells_enabled() || p.n_int == 0 || a.W < 2 || a.H < 2) return {};
  const int nr = a.n_rays, Wc = a.W - 1, Hc = a.H - 1;
  std::vector<unsigned long long> ho(nr + 1, 0);
  int max_side = 0;
  {
    std::vector<RayRec> rec(nr);
    PACT_CUDA_S(cudaMemcpyAsync(rec.data(), p.rec, sizeof(RayRec) * nr, cudaMemcpyDeviceToHost, s));
    PACT_CUDA_S(cudaStreamSynchronize(s));
    for (int r = 0; r < nr; ++r) {
      const RayRec& q = rec[r];
      const int n_int = q.n > 0 && !(q.flags & kRecGeneric) ? q.i_side : 0;
      max_side = std::max(max_side, n_int);
      ho[r + 1] = ho[r] + static_cast<unsigned long long>(n_int);
    }
  }
  const int sb = bits_for(static_cast<unsigned long long>(std::max(max_side - 1, 0)));
  const unsigned long long total = ho[nr];
  if (total == 0 || total >= (1ull << 31) || sb > 20) return {};
  const unsigned n = static_cast<unsigned>(total);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  auto hold = [](void* q) { return std::unique_ptr<void, void (*)(void*)>(q, [](void* x) { cudaFree(x); }); };
  unsigned long long* null_keys = nullptr;
  // per-ray counts and offsets
  void* small = nullptr;
  PACT_CUDA_S(cudaMalloc(&small, al(sizeof(unsigned long long) * (nr + 1)) * 2 + al(sizeof(unsigned) * nr)));
  auto hold_small = hold(small);
  auto* off = static_cast<unsigned long long*>(small);
  auto* toff = reinterpret_cast<unsigned long long*>(static_cast<char*>(small) + al(sizeof(unsigned long long) * (nr + 1)));
  auto* tcnt = reinterpret_cast<unsigned*>(static_cast<char*>(small) + 2 * al(sizeof(unsigned long long) * (nr + 1)));
  PACT_CUDA_S(cudaMemcpyAsync(off, ho.data(), sizeof(unsigned long long) * nr, cudaMemcpyHostToDevice, s));
  // 1. the tile size and the per-tile ray lists
  int T = 0, tile_max = 0, n_tiles = 0;
  CellTiles ct{};
  void* tmem = nullptr;  // tile_start [n_tiles + 1] | tile_rays [nt]
  for (int cand : {16, 8}) {
    ct = CellTiles{cand, (Wc + cand - 1) / cand, Wc, Hc};
    const int nti = ct.tx * ((Hc + cand - 1) / cand);
    cell_steps_kernel<<<div_up(nr, 256), 256, 0, s>>>(p.rec, nr, a.W, a.H, sb, ct, nullptr, nullptr,
                                                      nullptr, nullptr, tcnt, nullptr);
    PACT_TRY_S(after_launch(ctx, "cell_steps_kernel"));
    std::vector<unsigned> hc(nr);
    PACT_CUDA_S(cudaMemcpyAsync(hc.data(), tcnt, sizeof(unsigned) * nr, cudaMemcpyDeviceToHost, s));
    PACT_CUDA_S(cudaStreamSynchronize(s));
    std::vector<unsigned long long> hto(nr);
    unsigned long long tt = 0;
    for (int r = 0; r < nr; ++r) {
      hto[r] = tt;
      tt += hc[r];
    }
    if (tt == 0 || tt >= (1ull << 31)) return {};
    const unsigned ntc = static_cast<unsigned>(tt);
    PACT_CUDA_S(cudaMemcpyAsync(toff, hto.data(), sizeof(unsigned long long) * nr, cudaMemcpyHostToDevice, s));
    size_t ttemp = 0;
    const int tend = 32 + bits_for(static_cast<unsigned long long>(nti - 1));
    PACT_CUDA_S(cub::DeviceRadixSort::SortKeys(nullptr, ttemp, null_keys, null_keys, ntc, 0, tend, s));
    void* tscratch = nullptr;
    PACT_CUDA_S(cudaMalloc(&tscratch, al(16ull * ntc) + std::max<size_t>(ttemp, 16)));
    auto hold_ts = hold(tscratch);
    auto* tkeys = static_cast<unsigned long long*>(tscratch);
    cell_steps_kernel<<<div_up(nr, 256), 256, 0, s>>>(p.rec, nr, a.W, a.H, sb, ct, nullptr, nullptr,
                                                      toff, tkeys, nullptr, nullptr);
    PACT_TRY_S(after_launch(ctx, "cell_steps_kernel"));
    PACT_CUDA_S(cub::DeviceRadixSort::SortKeys(static_cast<char*>(tscratch) + al(16ull * ntc), ttemp,
                                               tkeys, tkeys + ntc, ntc, 0, tend, s));
    void* tm = nullptr;
    const size_t o_rays = al(sizeof(unsigned) * (nti + 1));
    PACT_CUDA_S(cudaMalloc(&tm, o_rays + sizeof(unsigned) * ntc));
    auto hold_tm = hold(tm);
    auto* ts = static_cast<unsigned*>(tm);
    group_bounds_kernel<<<div_up(static_cast<int>(ntc), 256), 256, 0, s>>>(
        tkeys + ntc, ntc, nti, 32, ts, reinterpret_cast<unsigned*>(static_cast<char*>(tm) + o_rays));
    PACT_TRY_S(after_launch(ctx, "group_bounds_kernel"));
    std::vector<unsigned> hts(nti + 1);
    PACT_CUDA_S(cudaMemcpyAsync(hts.data(), ts, sizeof(unsigned) * (nti + 1), cudaMemcpyDeviceToHost, s));
    PACT_CUDA_S(cudaStreamSynchronize(s));
    int mx = 0;
    for (int t = 0; t < nti; ++t) mx = std::max(mx, static_cast<int>(hts[t + 1] - hts[t]));
    if (static_cast<size_t>(mx) * (sizeof(float4) + sizeof(float)) <= kCellSmemMax &&
        bits_for(static_cast<unsigned long long>(std::max(mx - 1, 0))) + sb <= 32) {
      T = cand;
      tile_max = std::max(mx, 1);
      n_tiles = nti;
      tmem = hold_tm.release();
      break;
    }
  }
  if (!T) return {};
  auto hold_tmem = hold(tmem);
  // 2. the step entries, sorted by (tile-major cell, ray, step), then localised
  const int n_cells = n_tiles * T * T;
  const size_t o_ent = al(sizeof(unsigned) * (n_cells + 1)), o_geo = al(o_ent + sizeof(unsigned) * n),
               bytes = o_geo + sizeof(float4) * nr;
  void* mem = nullptr;
  PACT_CUDA_S(cudaMalloc(&mem, bytes));
  auto hold_mem = hold(mem);
  char* b = static_cast<char*>(mem);
  auto* start = reinterpret_cast<unsigned*>(b);
  auto* ent = reinterpret_cast<unsigned*>(b + o_ent);
  auto* geo = reinterpret_cast<float4*>(b + o_geo);
  const int end_bit = 32 + bits_for(static_cast<unsigned long long>(n_cells - 1));
  size_t temp = 0;
  PACT_CUDA_S(cub::DeviceRadixSort::SortKeys(nullptr, temp, null_keys, null_keys, n, 0, end_bit, s));
  void* scratch = nullptr;
  PACT_CUDA_S(cudaMalloc(&scratch, al(16ull * n) + std::max<size_t>(temp, 16)));
  auto hold_scratch = hold(scratch);
  auto* keys = static_cast<unsigned long long*>(scratch);
  cell_steps_kernel<<<div_up(nr, 256), 256, 0, s>>>(p.rec, nr, a.W, a.H, sb, ct, off, keys, nullptr,
                                                    nullptr, nullptr, geo);
  PACT_TRY_S(after_launch(ctx, "cell_steps_kernel"));
  PACT_CUDA_S(cub::DeviceRadixSort::SortKeys(static_cast<char*>(scratch) + al(16ull * n), temp, keys,
                                             keys + n, n, 0, end_bit, s));
  group_bounds_kernel<<<div_up(static_cast<int>(n), 256), 256, 0, s>>>(keys + n, n, n_cells, 32, start,
                                                                       nullptr);
  PACT_TRY_S(after_launch(ctx, "group_bounds_kernel"));
  auto* tstart = static_cast<unsigned*>(tmem);
  auto* trays = reinterpret_cast<unsigned*>(static_cast<char*>(tmem) + al(sizeof(unsigned) * (n_tiles + 1)));
  cell_localize_kernel<<<div_up(static_cast<int>(n), 256), 256, 0, s>>>(keys + n, n, sb, T, tstart,
                                                                       trays, ent);
  PACT_TRY_S(after_launch(ctx, "cell_localize_kernel"));
  PACT_CUDA_S(cudaStreamSynchronize(s));  // the host offsets and the scratch die here
  p.cell_mem = hold_mem.release();
  p.tile_mem = hold_tmem.release();
  p.cell_start = start;
  p.cell_ent = ent;
  p.cell_geo = geo;
  p.tile_start = tstart;
  p.tile_rays = trays;
  p.cell_sb = sb;
  p.cell_t = T;
  p.tile_max = tile_max;
  p.n_tiles = n_tiles;
  return {};
}

bool side_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PACT_RAY_SIDE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// PACT_SIDE_SERIES=0: the border cells' runs summed step by step (the A/B
// reference of the closed-form run sums in side_gather_kernel).
bool side_series_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PACT_SIDE_SERIES");
    return !(e && e[0] == '0');
  }();
  return on;
}

// The side plan (see side_gather_kernel): every run of every ray's border-line
// steps, keyed (slot, length, ray, first step) and radix-sorted.  Skipped
// (the adjoint's side items stay per ray) when a field does not fit or
// PACT_RAY_SIDE=0.  Synchronous.
Status build_side_plan(pact_ctx* ctx, cudaStream_t s, const RayArgs& a, RayPlanData& p) {
  const int nr = a.n_rays, n_slots = 2 * (a.W + a.H);
  if (!side_enabled() || a.W < 2 || a.H < 2 || nr > (1 << 20) || n_slots >= (1 << 16)) return {};
  {
    std::vector<RayRec> rec(nr);
    PACT_CUDA_S(cudaMemcpyAsync(rec.data(), p.rec, sizeof(RayRec) * nr, cudaMemcpyDeviceToHost, s));
    PACT_CUDA_S(cudaStreamSynchronize(s));
    for (const RayRec& q : rec)
      if (q.n > 0 && !(q.flags & kRecGeneric) && std::min(q.i_corner, q.n) > 4096) return {};
  }
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  auto hold = [](void* q) { return std::unique_ptr<void, void (*)(void*)>(q, [](void* x) { cudaFree(x); }); };
  void* small = nullptr;
  PACT_CUDA_S(cudaMalloc(&small, al(sizeof(unsigned long long) * (nr + 1)) + al(sizeof(unsigned) * nr)));
  auto hold_small = hold(small);
  auto* off = static_cast<unsigned long long*>(small);
  auto* cnt = reinterpret_cast<unsigned*>(static_cast<char*>(small) + al(sizeof(unsigned long long) * (nr + 1)));
  side_runs_kernel<<<div_up(nr, 256), 256, 0, s>>>(p.rec, nr, a.W, a.H, nullptr, nullptr, cnt, nullptr);
  PACT_TRY_S(after_launch(ctx, "side_runs_kernel"));
  std::vector<unsigned> hc(nr);
  PACT_CUDA_S(cudaMemcpyAsync(hc.data(), cnt, sizeof(unsigned) * nr, cudaMemcpyDeviceToHost, s));
  PACT_CUDA_S(cudaStreamSynchronize(s));
  std::vector<unsigned long long> ho(nr);
  unsigned long long total = 0;
  for (int r = 0; r < nr; ++r) {
    ho[r] = total;
    total += hc[r];
  }
  if (total == 0 || total >= (1ull << 31)) return {};
  const unsigned n = static_cast<unsigned>(total);
  PACT_CUDA_S(cudaMemcpyAsync(off, ho.data(), sizeof(unsigned long long) * nr, cudaMemcpyHostToDevice, s));
  // the plan's memory: ent [n] | start [n_slots + 1] | geo [nr]
  const size_t o_start = al(sizeof(unsigned long long) * n), o_geo = al(o_start + sizeof(unsigned) * (n_slots + 1)),
               bytes = o_geo + sizeof(float2) * nr;
  void* mem = nullptr;
  PACT_CUDA_S(cudaMalloc(&mem, bytes));
  auto hold_mem = hold(mem);
  char* b = static_cast<char*>(mem);
  auto* ent = reinterpret_cast<unsigned long long*>(b);
  auto* start = reinterpret_cast<unsigned*>(b + o_start);
  auto* geo = reinterpret_cast<float2*>(b + o_geo);
  unsigned long long* nk = nullptr;
  const int end_bit = 48 + bits_for(static_cast<unsigned long long>(n_slots - 1));
  size_t temp = 0;
  PACT_CUDA_S(cub::DeviceRadixSort::SortKeys(nullptr, temp, nk, nk, n, 0, end_bit, s));
  void* scratch = nullptr;
  PACT_CUDA_S(cudaMalloc(&scratch, al(8ull * n) + std::max<size_t>(temp, 16)));
  auto hold_scratch = hold(scratch);
  auto* keys = static_cast<unsigned long long*>(scratch);
  side_runs_kernel<<<div_up(nr, 256), 256, 0, s>>>(p.rec, nr, a.W, a.H, off, keys, nullptr, geo);
  PACT_TRY_S(after_launch(ctx, "side_runs_kernel"));
  PACT_CUDA_S(cub::DeviceRadixSort::SortKeys(static_cast<char*>(scratch) + al(8ull * n), temp, keys, ent, n, 0,
                                             end_bit, s));
  group_bounds_kernel<<<div_up(static_cast<int>(n), 256), 256, 0, s>>>(ent, n, n_slots, 48, start, nullptr);
  PACT_TRY_S(after_launch(ctx, "group_bounds_kernel"));
  PACT_CUDA_S(cudaStreamSynchronize(s));
  p.side_mem = hold_mem.release();
  p.side_ent = ent;
  p.side_start = start;
  p.side_geo = geo;
  p.n_side = n;
  return {};
}

// Builds the shared plan of a's geometry (a.centers on the device).  Synchronous.
Status build_plan_data(pact_ctx* ctx, cudaStream_t s, const RayArgs& a, RayPlanData& p) {
  const int nr = a.n_rays;
  void* rec_d = nullptr;
  PACT_CUDA_S(cudaMalloc(&rec_d, sizeof(RayRec) * nr));
  p.mem = rec_d;  // freed by ~RayPlanData on any failure below
  ray_plan_kernel<<<div_up(nr, 256), 256, 0, s>>>(a, static_cast<RayRec*>(rec_d));
  PACT_TRY_S(after_launch(ctx, "ray_plan_kernel"));
  std::vector<RayRec> rec(nr);
  PACT_CUDA_S(cudaMemcpyAsync(rec.data(), rec_d, sizeof(RayRec) * nr, cudaMemcpyDeviceToHost, s));
  PACT_CUDA_S(cudaStreamSynchronize(s));
  // work items in ray order (slot = index) with their sort keys
  const int C = ray_chunk();
  std::vector<int4> items;
  std::vector<int> key;
  std::vector<int2> slots(nr);
  items.reserve(static_cast<size_t>(nr) * 8);
  key.reserve(static_cast<size_t>(nr) * 8);
  int max_bucket = 0, max_chunk = 0;
  auto push = [&](int r, int lo, int hi, int kind, int chunk) {
    const int slot = static_cast<int>(items.size());
    items.push_back(make_int4(r, lo, hi, slot | (kind << 28)));
    const int bucket = (hi - lo + kLenBucket - 1) / kLenBucket;
    max_bucket = std::max(max_bucket, bucket);
    max_chunk = std::max(max_chunk, chunk);
    key.push_back(kind == kItemGeneric ? 0 : kind == kItemInterior ? 1 : 2);  // rank
    key.push_back(bucket);
    key.push_back(chunk);
  };
  for (int r = 0; r < nr; ++r) {
    const RayRec& q = rec[r];
    const int first = static_cast<int>(items.size());
    if (q.n > 0) {
      if (q.flags & kRecGeneric) {
        push(r, 0, q.n, kItemGeneric, 0);
      } else {
        const int side_end = std::min(q.i_corner, q.n);
        for (int i = 0; i < q.i_side; i += C)
          push(r, i, std::min(q.i_side, i + C), kItemInterior, i / C);
        for (int i = q.i_side; i < side_end; i += C)
          push(r, i, std::min(side_end, i + C), kItemSide, (i - q.i_side) / C);
        if (q.i_corner < q.n && static_cast<int>(items.size()) > first) {
          // the ray's last item adds the corner run; an empty border-line item
          // carries it when the ray has none (the adjoint's interior items may
          // run in the cell gather, which has no corner logic)
          if (((items.back().w >> 28) & 3) == kItemInterior) push(r, side_end, side_end, kItemSide, 0);
          items.back().w |= 1 << 30;
        }
      }
    }
    slots[r] = make_int2(first, static_cast<int>(items.size()) - first);
  }
  const int ni = static_cast<int>(items.size());
  if (ni >= (1 << 28)) return validation("ray plan: too many work items");
  // Schedule: longest work first -- generic rays, interior chunks (a gather
  // and a carry per step), border-line chunks -- lengths in buckets of
  // kLenBucket steps (at most kLenBucket - 1 idle steps per lane), then by
  // chunk index, then ray, so a warp holds adjacent angles at the same
  // distance.  A stable counting sort on (rank, -bucket, chunk) keeps ray order.
  const int nb = max_bucket + 1, nc = max_chunk + 1;
  const size_t n_keys = static_cast<size_t>(3) * nb * nc;
  std::vector<int> start(n_keys + 1, 0);
  std::vector<int> ck(ni);
  for (int k = 0; k < ni; ++k) {
    const int* kk = &key[3 * static_cast<size_t>(k)];
    ck[k] = (kk[0] * nb + (nb - 1 - kk[1])) * nc + kk[2];
    ++start[ck[k] + 1];
  }
  for (size_t k = 0; k < n_keys; ++k) start[k + 1] += start[k];
  const size_t per_rank = static_cast<size_t>(nb) * nc;
  p.n_gen = start[per_rank];
  p.n_int = start[2 * per_rank] - start[per_rank];
  std::vector<int4> sorted(std::max(ni, 1));
  for (int k = 0; k < ni; ++k) sorted[start[ck[k]]++] = items[k];
  // one allocation: rec | items | slots
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t o_items = al(sizeof(RayRec) * nr), o_slots = al(o_items + sizeof(int4) * sorted.size()),
               total = o_slots + sizeof(int2) * nr;
  void* mem = nullptr;
  PACT_CUDA_S(cudaMalloc(&mem, total));
  char* b = static_cast<char*>(mem);
  Status st = cuda_status(cudaMemcpyAsync(b, rec_d, sizeof(RayRec) * nr, cudaMemcpyDeviceToDevice,
                                          s), "ray plan");
  if (st.ok())
    st = cuda_status(cudaMemcpyAsync(b + o_items, sorted.data(), sizeof(int4) * sorted.size(),
                                     cudaMemcpyHostToDevice, s), "ray plan");
  if (st.ok())
    st = cuda_status(cudaMemcpyAsync(b + o_slots, slots.data(), sizeof(int2) * nr,
                                     cudaMemcpyHostToDevice, s), "ray plan");
  if (st.ok()) st = cuda_status(cudaStreamSynchronize(s), "ray plan");  // host vectors die here
  cudaFree(rec_d);
  p.mem = mem;
  if (!st.ok()) return st;
  p.rec = reinterpret_cast<const RayRec*>(b);
  p.items = reinterpret_cast<const int4*>(b + o_items);
  p.ray_slots = reinterpret_cast<const int2*>(b + o_slots);
  p.n_items = ni;
  PACT_TRY_S(build_cell_plan(ctx, s, a, p));
  return build_side_plan(ctx, s, a, p);
}

// Plans of one context, by geometry (most recent first, a few kept).
struct RayPlanCache {
  std::mutex mu;
  std::vector<std::shared_ptr<RayPlanData>> plans;
  RayPlan scratch;  // the standalone entry points' partials
};
constexpr size_t kPlanCacheSize = 4;

RayPlanCache& plan_cache(pact_ctx* ctx) {
  static std::mutex init_mu;
  std::lock_guard<std::mutex> lk(init_mu);
  if (!ctx->rays) {
    ctx->rays = new RayPlanCache();
    ctx->rays_free = [](void* p) {
      auto* c = static_cast<RayPlanCache*>(p);
      ray_plan_release(c->scratch, nullptr);
      delete c;
    };
  }
  return *static_cast<RayPlanCache*>(ctx->rays);
}

}  // namespace

static void set_cell_args(RayArgs& a, const RayPlanData& d) {
  a.side_ent = d.side_ent;
  a.side_start = d.side_start;
  a.side_geo = d.side_geo;
  a.cell_start = d.cell_start;
  a.cell_ent = d.cell_ent;
  a.cell_sb = d.cell_sb;
  a.tile_start = d.tile_start;
  a.tile_rays = d.tile_rays;
  a.cell_geo = d.cell_geo;
  a.cell_t = d.cell_t;
  a.tile_max = d.tile_max;
  a.n_gen_items = d.n_gen;
  a.n_int_items = d.n_int;
}

Status ray_plan_get(pact_ctx* cache_ctx, pact_ctx* ctx, RayArgs& a, const double* centers,
                    int n_centers, RayPlan& out) {
  ray_plan_release(out, ctx->stream);
  a.cell_start = nullptr;
  a.cell_ent = nullptr;
  a.side_ent = nullptr;
  a.rec = nullptr;
  a.items = nullptr;
  a.ray_slots = nullptr;
  a.partial = nullptr;
  a.n_items = 0;
  if (!a.tex || a.n_rays <= 0) return {};
  std::vector<double> key = plan_key(a, centers, n_centers);
  RayPlanCache& c = plan_cache(cache_ctx);
  std::shared_ptr<RayPlanData> data;
  {
    std::lock_guard<std::mutex> lk(c.mu);
    for (auto& p : c.plans)
      if (p->key == key) data = p;
    if (!data) {
      auto fresh = std::make_shared<RayPlanData>();
      PACT_TRY_S(build_plan_data(ctx, ctx->stream, a, *fresh));
      fresh->key = std::move(key);
      c.plans.insert(c.plans.begin(), fresh);
      if (c.plans.size() > kPlanCacheSize) c.plans.pop_back();
      data = fresh;
    }
  }
  void* part = nullptr;
  PACT_TRY_S(pool_alloc(&part, sizeof(float) * std::max(data->n_items, 1), ctx->stream));
  out.data = data;
  out.partial = static_cast<float*>(part);
  a.rec = data->rec;
  a.items = data->items;
  a.ray_slots = data->ray_slots;
  a.partial = out.partial;
  a.n_items = data->n_items;
  set_cell_args(a, *data);
  return {};
}

void ray_plan_release(RayPlan& p, cudaStream_t s) {
  if (p.partial) pool_free(p.partial, s);
  p.partial = nullptr;
  p.data.reset();
}

Status ray_plan_cached(pact_ctx* ctx, RayArgs& a, const double* centers, int n_centers) {
  if (!a.tex) return {};
  RayPlanCache& c = plan_cache(ctx);
  RayPlan& p = c.scratch;
  if (p.data && p.data->key == plan_key(a, centers, n_centers)) {
    a.rec = p.data->rec;
    a.items = p.data->items;
    a.ray_slots = p.data->ray_slots;
    a.partial = p.partial;
    a.n_items = p.data->n_items;
    set_cell_args(a, *p.data);
    return {};
  }
  return ray_plan_get(ctx, ctx, a, centers, n_centers, p);
}

static size_t border_smem(const RayArgs& a) { return sizeof(float) * 2 * (a.W + a.H); }

Status launch_wavefront(pact_ctx* ctx, const RayArgs& a, float* w) {
  const size_t smem = border_smem(a);
  if (a.tex) {  // make_raster_texture requires W, H >= 2
    if (!a.rec) return internal_error("launch_wavefront: ray plan missing");
    // (the forward keeps its border-line items: without a carry they are as
    // cheap per step as the side gather, and a ray's sum stays in one place)
    if (a.n_items > 0) {
      if (side_series_enabled()) {
        PACT_TRY_S(smem_optin(wavefront_plan_kernel<true>, smem));
        wavefront_plan_kernel<true><<<div_up(a.n_items, kPlanBlock), kPlanBlock, smem, ctx->stream>>>(a);
      } else {
        PACT_TRY_S(smem_optin(wavefront_plan_kernel<false>, smem));
        wavefront_plan_kernel<false><<<div_up(a.n_items, kPlanBlock), kPlanBlock, smem, ctx->stream>>>(a);
      }
      PACT_TRY_S(after_launch(ctx, "wavefront_plan_kernel"));
    }
    ray_finish_kernel<<<div_up(a.n_rays, 256), 256, 0, ctx->stream>>>(a, w);
    return after_launch(ctx, "ray_finish_kernel");
  }
  PACT_TRY_S(smem_optin(wavefront_kernel<false>, smem));
  wavefront_kernel<false><<<div_up(a.n_rays, 256), 256, smem, ctx->stream>>>(a, w);
  return after_launch(ctx, "wavefront_kernel");
}

Status launch_ray_backward(pact_ctx* ctx, const RayArgs& a, const float* dw, double* grad) {
  const size_t smem = border_smem(a);
  if (a.n_rays == 0) return {};
  // fixed-point accumulators: raster [H W] | border replicas | bound statistics,
  // zero between launches (fix_to_grad_kernel resets what it reads); with a
  // cell / side plan also the per-ray deposit scales, the cell corner sums
  // and the border cells' sums
  const size_t npx = static_cast<size_t>(a.W) * a.H;
  const int n_slots = 2 * (a.W + a.H);
  const size_t rep_n = static_cast<size_t>(kBorderReplicas) * n_slots;
  const bool cells = a.tex && a.rec && a.cell_start;
  const bool side = a.tex && a.rec && a.side_ent;
  const size_t n_cells = cells ? static_cast<size_t>(a.W - 1) * (a.H - 1) : 0;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t fix_bytes = sizeof(unsigned long long) * (npx + rep_n + 2);
  const size_t gsc_off = al(fix_bytes);
  const size_t cell_off = al(gsc_off + sizeof(float) * (cells || side ? a.n_rays : 0));
  const size_t side_off = al(cell_off + 4 * sizeof(unsigned long long) * n_cells);
  const size_t bytes = side_off + 2 * sizeof(unsigned long long) * (side ? n_slots : 0);
  pact_scratch& sc = ctx->scratch[kScratchRayBorder];
  const void* before = sc.ptr;
  void* base = nullptr;
  PACT_TRY_S(scratch_get(ctx, kScratchRayBorder, bytes, &base));
  if (base != before) PACT_CUDA_S(cudaMemsetAsync(base, 0, sc.bytes, ctx->stream));
  auto* acc = static_cast<unsigned long long*>(base);
  auto* rep = acc + npx;
  auto* stats = rep + rep_n;
  char* cb = static_cast<char*>(base);
  float* gsc = cells || side ? reinterpret_cast<float*>(cb + gsc_off) : nullptr;
  auto* cell_sums = cells ? reinterpret_cast<unsigned long long*>(cb + cell_off) : nullptr;
  auto* side_cells = side ? reinterpret_cast<unsigned long long*>(cb + side_off) : nullptr;
  PACT_CUDA_S(cudaMemsetAsync(stats, 0, 2 * sizeof(unsigned long long), ctx->stream));
  const int nb = std::max(1, div_up(std::max(static_cast<int>(npx), a.n_rays), 256 * 4));
  ray_bound_kernel<<<nb, 256, 0, ctx->stream>>>(dw, a.n_rays, a.dv, static_cast<int>(npx),
                                                static_cast<float>(a.v0), a.rec, a.v0, gsc, stats);
  PACT_TRY_S(after_launch(ctx, "ray_bound_kernel"));
  if (a.tex) {
    if (!a.rec) return internal_error("launch_ray_backward: ray plan missing");
    // the interior items go to the cell gather, the side items to the side
    // gather, when there are such plans (items: generic | interior | side)
    const int lo = cells ? a.n_gen_items : a.n_gen_items + a.n_int_items;
    const int hi = side ? a.n_items : a.n_gen_items + a.n_int_items;
    const int skip_lo = cells || side ? lo : a.n_items, skip_n = cells || side ? std::max(0, hi - lo) : 0;
    const int n_run = a.n_items - skip_n;
    if (n_run > 0) {
      PACT_TRY_S(smem_optin(ray_backward_plan_kernel, smem));
      ray_backward_plan_kernel<<<div_up(n_run, kPlanBlock), kPlanBlock, smem, ctx->stream>>>(
          a, dw, acc, rep, stats, skip_lo, skip_n);
      PACT_TRY_S(after_launch(ctx, "ray_backward_plan_kernel"));
    }
    if (cells) {
      const int T = a.cell_t, n_tiles = ((a.W - 1 + T - 1) / T) * ((a.H - 1 + T - 1) / T);
      const size_t cs = static_cast<size_t>(a.tile_max) * (sizeof(float4) + sizeof(float));
      if (T == 16) {
        PACT_TRY_S(smem_optin(cell_gather_kernel<16>, cs));
        cell_gather_kernel<16><<<n_tiles, kCellThreads, cs, ctx->stream>>>(a, gsc, stats, cell_sums);
      } else {
        PACT_TRY_S(smem_optin(cell_gather_kernel<8>, cs));
        cell_gather_kernel<8><<<n_tiles, kCellThreads, cs, ctx->stream>>>(a, gsc, stats, cell_sums);
      }
      PACT_TRY_S(after_launch(ctx, "cell_gather_kernel"));
    }
    if (side) {
      if (side_series_enabled())
        side_gather_kernel<true><<<n_slots, kSideThreads, 0, ctx->stream>>>(a, gsc, stats, side_cells);
      else
        side_gather_kernel<false><<<n_slots, kSideThreads, 0, ctx->stream>>>(a, gsc, stats, side_cells);
      PACT_TRY_S(after_launch(ctx, "side_gather_kernel"));
      corner_adjoint_kernel<<<div_up(a.n_rays, 256), 256, 0, ctx->stream>>>(a, gsc, stats, rep);
      PACT_TRY_S(after_launch(ctx, "corner_adjoint_kernel"));
    }
  } else {
    PACT_TRY_S(smem_optin(ray_backward_kernel<false>, smem));
    ray_backward_kernel<false><<<div_up(a.n_rays, 256), 256, smem, ctx->stream>>>(a, dw, acc, stats);
    PACT_TRY_S(after_launch(ctx, "ray_backward_kernel"));
  }
  if (a.tex) {
    border_fold_kernel<<<div_up(n_slots, 128), 128, 0, ctx->stream>>>(rep, a.W, a.H, side_cells, acc);
    PACT_TRY_S(after_launch(ctx, "border_fold_kernel"));
  }
  fix_to_grad_kernel<<<div_up(static_cast<int>(npx), 256), 256, 0, ctx->stream>>>(
      acc, a.W, a.H, stats, a.step, a.v0, max_steps_total(a), cell_sums, grad);
  return after_launch(ctx, "fix_to_grad_kernel");
}

// Standalone entry points: a texture over the caller's raster for the
// duration of one (synchronised) launch.
struct ScopedTexture {
  cudaTextureObject_t t = 0;
  pact_ctx* ctx;
  ScopedTexture(pact_ctx* c, const float* dv, int W, int H) : ctx(c) {
    make_raster_texture(dv, W, H, &t);
  }
  ~ScopedTexture() {
    if (t) {
      cudaStreamSynchronize(ctx->stream);
      cudaDestroyTextureObject(t);
    }
  }
};

}  // namespace pactgpu

using namespace pactgpu;

extern "C" int pact_wavefront(pact_ctx* ctx, const pact_ring* ring, const pact_grid* grid,
                              const float* sos_dev, double v0, const pact_mask* mask,
                              int32_t n_centers, const double* centers, int32_t n_angles,
                              double step, float* w) {
  if (!ctx || !ring || !grid || !mask || !centers || !sos_dev || !w)
    return validation("pact_wavefront: null argument").code;
  RayArgs a{};
  PACT_TRY(ray_args(*ring, *grid, v0, *mask, n_angles, step, a));
  PACT_TRY(validate_centers(*ring, n_centers, centers));
  if (n_centers <= 0) return PACT_OK;
  void* dc = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric3, sizeof(double2) * n_centers, &dc));
  PACT_CUDA(cudaMemcpyAsync(dc, centers, sizeof(double2) * n_centers, cudaMemcpyHostToDevice,
                            ctx->stream));
  a.dv = sos_dev;
  a.centers = static_cast<const double2*>(dc);
  a.n_rays = n_centers * n_angles;
  ScopedTexture tex(ctx, sos_dev, grid->width, grid->height);
  a.tex = tex.t;
  PACT_TRY(ray_plan_cached(ctx, a, centers, n_centers));
  PACT_TRY(launch_wavefront(ctx, a, w));
  return PACT_OK;
}

extern "C" int pact_ray_backward(pact_ctx* ctx, const pact_ring* ring, const pact_grid* grid,
                                 const float* sos_dev, double v0, const pact_mask* mask,
                                 int32_t n_centers, const double* centers, int32_t n_angles,
                                 double step, const float* dw, double* grad_v) {
  if (!ctx || !ring || !grid || !mask || !centers || !sos_dev || !dw || !grad_v)
    return validation("pact_ray_backward: null argument").code;
  RayArgs a{};
  PACT_TRY(ray_args(*ring, *grid, v0, *mask, n_angles, step, a));
  if (n_centers <= 0) return PACT_OK;
  void* dc = nullptr;
  PACT_TRY(scratch_get(ctx, kScratchGeneric3, sizeof(double2) * n_centers, &dc));
  PACT_CUDA(cudaMemcpyAsync(dc, centers, sizeof(double2) * n_centers, cudaMemcpyHostToDevice,
                            ctx->stream));
  a.dv = sos_dev;
  a.centers = static_cast<const double2*>(dc);
  a.n_rays = n_centers * n_angles;
  ScopedTexture tex(ctx, sos_dev, grid->width, grid->height);
  a.tex = tex.t;
  PACT_TRY(ray_plan_cached(ctx, a, centers, n_centers));
  PACT_TRY(launch_ray_backward(ctx, a, dw, grad_v));
  return PACT_OK;
}
