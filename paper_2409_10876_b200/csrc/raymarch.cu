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
// clamp onto one border cell for long runs) and flushes with fp64 atomics,
// skipping zero-weight corners; fp64 accumulation makes the result
// reproducible to fp32 output precision regardless of atomic order.
#include "common.cuh"
#include "geom.cuh"

// RAY_EXP (experiments only, never set in the product build): 1 = interior
// carries without atomics, 2 = interior without carries.
#ifndef RAY_EXP
#define RAY_EXP 0
#endif

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

__device__ __forceinline__ void flush_cell(double* __restrict__ g, int W, int H, int ix, int iy,
                                           const double acc[4]) {
  int ix1 = min(ix + 1, W - 1), iy1 = min(iy + 1, H - 1);
  if (acc[0] != 0.0) atomicAdd(g + iy * W + ix, acc[0]);
  if (acc[1] != 0.0) atomicAdd(g + iy * W + ix1, acc[1]);
  if (acc[2] != 0.0) atomicAdd(g + iy1 * W + ix, acc[2]);
  if (acc[3] != 0.0) atomicAdd(g + iy1 * W + ix1, acc[3]);
}

// Per-ray accumulators of the current stencil cell's pixels (cx + i, cy + j):
// a{j}{i}.  A pixel collects a handful of steps in fp32 before its fp64 flush;
// on a move, pixels shared with the new cell stay in registers (halves the
// atomics of a horizontal/vertical move).
struct CellAcc {
  int cx = -1, cy = -1;
  float a00 = 0.f, a01 = 0.f, a10 = 0.f, a11 = 0.f;

  __device__ __forceinline__ void move(double* __restrict__ grad, int W, int ix, int iy) {
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
        } else if (val != 0.f && RAY_EXP == 0) {
          atomicAdd(grad + (cy + (q >> 1)) * W + cx + (q & 1), static_cast<double>(val));
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
  __device__ __forceinline__ void move_unit(double* __restrict__ grad, int W, int ix, int iy) {
    if (ix == cx && iy == cy) return;
    const int dx = ix - cx, dy = iy - cy;
    if (cx < 0 || dx < -1 || dx > 1 || dy < -1 || dy > 1) {
      move(grad, W, ix, iy);
      return;
    }
    // old slot (i, j) [x i, y j] survives iff (i - dx, j - dy) is in the new cell
    const bool keep_x0 = dx <= 0, keep_x1 = dx >= 0, keep_y0 = dy <= 0, keep_y1 = dy >= 0;
    if (RAY_EXP == 0) {
      double* p = grad + cy * W + cx;
      if (!(keep_x0 && keep_y0) && a00 != 0.f) atomicAdd(p, static_cast<double>(a00));
      if (!(keep_x1 && keep_y0) && a01 != 0.f) atomicAdd(p + 1, static_cast<double>(a01));
      if (!(keep_x0 && keep_y1) && a10 != 0.f) atomicAdd(p + W, static_cast<double>(a10));
      if (!(keep_x1 && keep_y1) && a11 != 0.f) atomicAdd(p + W + 1, static_cast<double>(a11));
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
  __device__ __forceinline__ void flush(double* __restrict__ grad, int W, int H) {
    if (cx < 0) return;
    const double fin[4] = {a00, a01, a10, a11};
    flush_cell(grad, W, H, cx, cy, fin);
    cx = cy = -1;
    a00 = a01 = a10 = a11 = 0.f;
  }
};

template <bool TEX>
__device__ void march_backward_generic(const RayArgs& a, const Border& bd, const RayPix& rp, int n,
                                       float v0, float gscale, double* __restrict__ grad) {
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

// Threads per ray in the split kernels: each ray's steps are cut into SEG
// contiguous segments of about equal cost (an interior step costs ~2 border
// steps, corner steps are free), one lane each; the lanes of a ray are
// adjacent in the warp (forward partial sums are shuffled in a fixed order).
constexpr int SEG = 1;
// Blocks of the split kernels: one wave, evenly loaded.  All rays are
// resident at once (115k rays at cfg3 vs 148 x 2048 thread slots), so the
// kernel time is set by the most loaded SM: ceil(n_rays / SMs) rounded to a
// warp, one block per SM.  (Measured at cfg3: 256-thread blocks leave 4 blocks
// on some SMs, 0.855 ms; 800-thread blocks 0.820 ms.)  The wavefront pass is
// fastest with two whole patches (1024 rays) per block when that still fills
// most SMs (texture-cache locality: 0.252 vs 0.293 ms).
constexpr int kRayBlockMax = 1024;

int ray_block(const RayArgs& a, int num_sms, bool wavefront) {
  if (wavefront && a.n_rays >= kRayBlockMax * (num_sms / 2)) return kRayBlockMax;
  const int per_sm = div_up(a.n_rays, std::max(1, num_sms));
  return std::min(kRayBlockMax, std::max(256, div_up(per_sm, 32) * 32));
}

struct Segment {
  int lo, hi;
};

__device__ __forceinline__ Segment segment_of(const Regimes& rg, int n, int seg) {
  const int side_end = min(rg.i_corner, n);
  const int cost = 2 * rg.i_side + (side_end - rg.i_side);
  auto at_cost = [&](int c) {  // first step index whose cumulative cost reaches c
    return c <= 2 * rg.i_side ? (c + 1) / 2 : min(side_end, rg.i_side + (c - 2 * rg.i_side));
  };
  const int lo = seg == 0 ? 0 : at_cost(cost * seg / SEG);
  const int hi = seg == SEG - 1 ? n : at_cost(cost * (seg + 1) / SEG);
  return {lo, hi};
}

__global__ void __launch_bounds__(kRayBlockMax) wavefront_split_kernel(RayArgs a, float* __restrict__ w) {
  extern __shared__ float s_border[];
  const Border bd = load_border(a, s_border);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = t / SEG, seg = t % SEG;
  float acc = 0.f;
  double dl = 0.0;
  if (r < a.n_rays) {
    int patch = r / a.n_angles, ang = r - patch * a.n_angles;
    double2 c = a.centers[patch];
    Ray ray = make_ray(c.x, c.y, ang, a.n_angles, a.ring_r, a.mcx, a.mcy, a.mr, a.step);
    dl = ray.dl;
    const RayPix rp = ray_pixels(a, c.x, c.y, ray);
    const float v0 = static_cast<float>(a.v0);
    const int W = a.W, H = a.H, n = ray.n;
    const float Wm1 = static_cast<float>(W - 1), Hm1 = static_cast<float>(H - 1);
    if (n > 0 && (out_at(0, rp.fxs, rp.dfx, Wm1) || out_at(0, rp.fys, rp.dfy, Hm1))) {
      if (seg == 0) acc = march_forward_generic<true>(a, bd, rp, n, v0);
    } else if (n > 0) {
      const Regimes rg = regimes(rp, n, Wm1, Hm1);
      const Segment sg = segment_of(rg, n, seg);
      const int i1 = min(rg.i_side, sg.hi);
#pragma unroll 4
      for (int i = sg.lo; i < i1; ++i) {
        float ax, ay;
        int ix, iy;
        const float d = interior_d(a.tex, fmaf(static_cast<float>(i), rp.dfx, rp.fxs),
                                   fmaf(static_cast<float>(i), rp.dfy, rp.fys), W, H, ax, ay, ix,
                                   iy);
        acc += __fdividef(d, v0 + d);
      }
      const int s0 = max(rg.i_side, sg.lo), s1 = min(rg.i_corner, sg.hi);
      if (rg.x_first) {
        const float* col = rp.dfx > 0.f ? bd.colR : bd.colL;
#pragma unroll 4
        for (int i = s0; i < s1; ++i) {
          const float fy = fmaf(static_cast<float>(i), rp.dfy, rp.fys);
          const int iy = min(static_cast<int>(fy), H - 2);
          const float c0 = col[iy];
          const float d = fmaf(fy - iy, col[iy + 1] - c0, c0);
          acc += __fdividef(d, v0 + d);
        }
      } else {
        const float* row = rp.dfy > 0.f ? bd.rowT : bd.rowB;
#pragma unroll 4
        for (int i = s0; i < s1; ++i) {
          const float fx = fmaf(static_cast<float>(i), rp.dfx, rp.fxs);
          const int ix = min(static_cast<int>(fx), W - 2);
          const float c0 = row[ix];
          const float d = fmaf(fx - ix, row[ix + 1] - c0, c0);
          acc += __fdividef(d, v0 + d);
        }
      }
      const int n_corner = sg.hi - max(rg.i_corner, sg.lo);
      if (n_corner > 0) {
        const float* col = rp.dfx > 0.f ? bd.colR : bd.colL;
        const float d = col[rp.dfy > 0.f ? H - 1 : 0];
        acc += static_cast<float>(n_corner) * __fdividef(d, v0 + d);
      }
    }
  }
  // fixed-order sum of the ray's segments (lanes r*SEG .. r*SEG + SEG - 1)
#pragma unroll
  for (int o = 1; o < SEG; o <<= 1) {
    const float other = __shfl_down_sync(0xffffffffu, acc, o, SEG);
    acc += other;
  }
  if (r < a.n_rays && seg == 0) w[r] = static_cast<float>(dl) * acc;
}

// 1-D carry along a border line: pixels (line position q, q + 1).
struct LineAcc {
  int q = -1;
  float b0 = 0.f, b1 = 0.f;
  __device__ __forceinline__ void move(double* __restrict__ grad, int nq, int stride, int base) {
    if (nq == q) return;
    if (q >= 0 && RAY_EXP != 5) {
      if (nq == q + 1) {
        if (b0 != 0.f) atomicAdd(grad + base + q * stride, static_cast<double>(b0));
        b0 = b1;
        b1 = 0.f;
      } else if (nq == q - 1) {
        if (b1 != 0.f) atomicAdd(grad + base + (q + 1) * stride, static_cast<double>(b1));
        b1 = b0;
        b0 = 0.f;
      } else {
        if (b0 != 0.f) atomicAdd(grad + base + q * stride, static_cast<double>(b0));
        if (b1 != 0.f) atomicAdd(grad + base + (q + 1) * stride, static_cast<double>(b1));
        b0 = b1 = 0.f;
      }
    }
    q = nq;
  }
  __device__ __forceinline__ void flush(double* __restrict__ grad, int stride, int base) {
    if (q < 0) return;
    if (b0 != 0.f) atomicAdd(grad + base + q * stride, static_cast<double>(b0));
    if (b1 != 0.f) atomicAdd(grad + base + (q + 1) * stride, static_cast<double>(b1));
  }
};

// Border deposits: every ray of every patch that leaves the grid deposits on
// the same 2(W + H) border pixels (and 4 corners), so global atomics there
// contend.  They go to one of kBorderReplicas copies of the border (by block)
// and border_reduce_kernel folds the copies into the raster afterwards in a
// fixed order.  Replica layout: [R][colL H | colR H | rowB W | rowT W].
constexpr int kBorderReplicas = 32;

__global__ void __launch_bounds__(kRayBlockMax) ray_backward_split_kernel(RayArgs a, const float* __restrict__ dw,
                                                                 double* __restrict__ grad,
                                                                 double* __restrict__ border_rep) {
  extern __shared__ float s_border[];
  const Border bd = load_border(a, s_border);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = t / SEG, seg = t % SEG;
  if (r >= a.n_rays) return;
  const float gr = dw[r];
  if (gr == 0.f) return;  // aberration.hpp:340
  int patch = r / a.n_angles, ang = r - patch * a.n_angles;
  double2 c = a.centers[patch];
  Ray ray = make_ray(c.x, c.y, ang, a.n_angles, a.ring_r, a.mcx, a.mcy, a.mr, a.step);
  if (ray.n == 0) return;
  const RayPix rp = ray_pixels(a, c.x, c.y, ray);
  const float v0 = static_cast<float>(a.v0);
  // f = g * dl * v0 / v^2 per step (aberration.hpp:354-355)
  const float gscale = static_cast<float>(static_cast<double>(gr) * ray.dl * a.v0);
  const int W = a.W, H = a.H, n = ray.n;
  const float Wm1 = static_cast<float>(W - 1), Hm1 = static_cast<float>(H - 1);
  if (out_at(0, rp.fxs, rp.dfx, Wm1) || out_at(0, rp.fys, rp.dfy, Hm1)) {
    if (seg == 0) march_backward_generic<true>(a, bd, rp, n, v0, gscale, grad);
    return;
  }
  const Regimes rg = regimes(rp, n, Wm1, Hm1);
  const Segment sg = segment_of(rg, n, seg);
  {
    // interior: gathers issued four steps at a time, then the carries
    CellAcc cell;
    const int i1 = min(rg.i_side, sg.hi);
    int i = sg.lo;
    for (; i < i1; i += 4) {
      float4 g[4];
      float ax[4], ay[4];
      int ix[4], iy[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float fx = fmaf(static_cast<float>(min(i + u, i1 - 1)), rp.dfx, rp.fxs);
        const float fy = fmaf(static_cast<float>(min(i + u, i1 - 1)), rp.dfy, rp.fys);
        ix[u] = min(static_cast<int>(fx), W - 2);
        iy[u] = min(static_cast<int>(fy), H - 2);
        ax[u] = fx - ix[u];
        ay[u] = fy - iy[u];
        g[u] = tex2Dgather<float4>(a.tex, ix[u] + 1.f, iy[u] + 1.f, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i + u < i1) {
          // gather order: w=(ix,iy) z=(ix+1,iy) x=(ix,iy+1) y=(ix+1,iy+1)
          const float top = fmaf(ax[u], g[u].z - g[u].w, g[u].w);
          const float bot = fmaf(ax[u], g[u].y - g[u].x, g[u].x);
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
  }
  const int s0 = max(rg.i_side, sg.lo), s1 = min(rg.i_corner, sg.hi);
  if (s0 < s1) {
    LineAcc line;
    double* rep = border_rep + static_cast<size_t>(blockIdx.x % kBorderReplicas) * 2 * (W + H);
    if (rg.x_first) {
      const float* col = rp.dfx > 0.f ? bd.colR : bd.colL;
      double* dst = rep + (rp.dfx > 0.f ? H : 0);
      for (int i = s0; i < s1; ++i) {
        const float fy = fmaf(static_cast<float>(i), rp.dfy, rp.fys);
        const int iy = min(static_cast<int>(fy), H - 2);
        const float ay = fy - iy, c0 = col[iy];
        const float v = v0 + fmaf(ay, col[iy + 1] - c0, c0);
        const float f = __fdividef(gscale, v * v);
        line.move(dst, iy, 1, 0);
        const float f1 = f * ay;
        line.b0 += f - f1;
        line.b1 += f1;
      }
      line.flush(dst, 1, 0);
    } else {
      const float* row = rp.dfy > 0.f ? bd.rowT : bd.rowB;
      double* dst = rep + 2 * H + (rp.dfy > 0.f ? W : 0);
      for (int i = s0; i < s1; ++i) {
        const float fx = fmaf(static_cast<float>(i), rp.dfx, rp.fxs);
        const int ix = min(static_cast<int>(fx), W - 2);
        const float ax = fx - ix, c0 = row[ix];
        const float v = v0 + fmaf(ax, row[ix + 1] - c0, c0);
        const float f = __fdividef(gscale, v * v);
        line.move(dst, ix, 1, 0);
        const float f1 = f * ax;
        line.b0 += f - f1;
        line.b1 += f1;
      }
      line.flush(dst, 1, 0);
    }
  }
  const int n_corner = sg.hi - max(rg.i_corner, sg.lo);
  if (n_corner > 0) {
    const int px = rp.dfx > 0.f ? W - 1 : 0, py = rp.dfy > 0.f ? H - 1 : 0;
    const float* col = rp.dfx > 0.f ? bd.colR : bd.colL;
    const float v = v0 + col[py];
    const float f = __fdividef(gscale, v * v) * static_cast<float>(n_corner);
    double* rep = border_rep + static_cast<size_t>(blockIdx.x % kBorderReplicas) * 2 * (W + H);
    if (f != 0.f) atomicAdd(rep + (px == 0 ? 0 : H) + py, static_cast<double>(f));
  }
}

// grad[p] += sum over replicas of the slot(s) of border pixel p (fixed order).
// One thread per border pixel: left / right columns, then the bottom / top
// rows without their corners.
__global__ void border_reduce_kernel(const double* __restrict__ rep, int W, int H,
                                     double* __restrict__ grad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_in = max(W - 2, 0);
  if (i >= 2 * H + 2 * n_in) return;
  int px, py;
  if (i < 2 * H) {
    px = i < H ? 0 : W - 1;
    py = i < H ? i : i - H;
  } else {
    const int k = i - 2 * H;
    px = 1 + (k < n_in ? k : k - n_in);
    py = k < n_in ? 0 : H - 1;
  }
  const int col = px == 0 ? py : (px == W - 1 ? H + py : -1);
  const int row = py == 0 ? 2 * H + px : (py == H - 1 ? 2 * H + W + px : -1);
  const size_t stride = 2 * static_cast<size_t>(W + H);
  double s = 0.0;
  for (int r = 0; r < kBorderReplicas; ++r) {
    if (col >= 0) s += rep[r * stride + col];
    if (row >= 0) s += rep[r * stride + row];
  }
  if (s != 0.0) grad[static_cast<size_t>(py) * W + px] += s;
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
                                                           double* __restrict__ grad) {
  extern __shared__ float s_border[];
  const Border bd = load_border(a, s_border);
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

static size_t border_smem(const RayArgs& a) { return sizeof(float) * 2 * (a.W + a.H); }

template <typename K>
static Status allow_smem(K kernel, size_t smem) {
  if (smem > 48 * 1024)
    PACT_CUDA_S(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  return {};
}

Status launch_wavefront(pact_ctx* ctx, const RayArgs& a, float* w) {
  int blocks = div_up(a.n_rays, 256);
  size_t smem = border_smem(a);
  if (a.tex) {  // make_raster_texture requires W, H >= 2
    PACT_TRY_S(allow_smem(wavefront_split_kernel, smem));
    const int rb = ray_block(a, ctx->num_sms, true);
    wavefront_split_kernel<<<div_up(a.n_rays * SEG, rb), rb, smem, ctx->stream>>>(a, w);
  } else {
    PACT_TRY_S(allow_smem(wavefront_kernel<false>, smem));
    wavefront_kernel<false><<<blocks, 256, smem, ctx->stream>>>(a, w);
  }
  return after_launch(ctx, a.tex ? "wavefront_split_kernel" : "wavefront_kernel");
}

Status launch_ray_backward(pact_ctx* ctx, const RayArgs& a, const float* dw, double* grad) {
  int blocks = div_up(a.n_rays, 256);
  size_t smem = border_smem(a);
  if (a.tex) {
    const int rb = ray_block(a, ctx->num_sms, false);
    blocks = div_up(a.n_rays * SEG, rb);
    const size_t rep_n = static_cast<size_t>(kBorderReplicas) * 2 * (a.W + a.H);
    void* rep = nullptr;
    PACT_TRY_S(scratch_get(ctx, kScratchRayBorder, sizeof(double) * rep_n, &rep));
    PACT_CUDA_S(cudaMemsetAsync(rep, 0, sizeof(double) * rep_n, ctx->stream));
    PACT_TRY_S(allow_smem(ray_backward_split_kernel, smem));
    ray_backward_split_kernel<<<blocks, rb, smem, ctx->stream>>>(a, dw, grad,
                                                                   static_cast<double*>(rep));
    PACT_TRY_S(after_launch(ctx, "ray_backward_split_kernel"));
    const int nbp = 2 * a.H + 2 * std::max(a.W - 2, 0);
    border_reduce_kernel<<<div_up(nbp, 256), 256, 0, ctx->stream>>>(static_cast<double*>(rep), a.W,
                                                                     a.H, grad);
    return after_launch(ctx, "border_reduce_kernel");
  } else {
    PACT_TRY_S(allow_smem(ray_backward_kernel<false>, smem));
    ray_backward_kernel<false><<<blocks, 256, smem, ctx->stream>>>(a, dw, grad);
  }
  return after_launch(ctx, "ray_backward_kernel");
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
  PACT_TRY(launch_ray_backward(ctx, a, dw, grad_v));
  return PACT_OK;
}
