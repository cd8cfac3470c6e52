// Device/host geometry shared by the ray-march, PSF and TV kernels.  Each
// helper restates one reference routine (file:line) with identical
// branch structure; ray setup stays in fp64 like the reference so step counts
// n = max(1, ceil((t1 - t0)/step)) match exactly.
#pragma once

#include <cuda_runtime.h>

#include <cmath>

#include "pact_cuda.h"

namespace pactgpu {

#define PACT_HD __host__ __device__ __forceinline__

// segment_circle_intersection, core.hpp:184-204.  Returns false for an empty
// interval (the reference's {1, 0}).
PACT_HD bool seg_circle(double ax, double ay, double bx, double by, double cx, double cy,
                        double r, double& t0, double& t1) {
  double dx = bx - ax, dy = by - ay;
  double len = hypot(dx, dy);
  if (len == 0.0) {
    bool inside = hypot(ax - cx, ay - cy) <= r;
    t0 = inside ? 0.0 : 1.0;
    t1 = 0.0;
    return t0 <= t1 && inside;
  }
  double ux = dx * (1.0 / len), uy = dy * (1.0 / len);
  double mx = ax - cx, my = ay - cy;
  double bq = mx * ux + my * uy;
  double cq = (mx * mx + my * my) - r * r;
  double disc = bq * bq - cq;
  if (disc < 0.0) {
    t0 = 1.0;
    t1 = 0.0;
    return false;
  }
  double s = sqrt(disc);
  t0 = fmax(-bq - s, 0.0);
  t1 = fmin(-bq + s, len);
  if (t0 > t1) {
    t0 = 1.0;
    t1 = 0.0;
    return false;
  }
  return true;
}

// Ray of wavefront_profile / wavefront_grad_trace (aberration.hpp:153-171):
// direction theta = 2 pi a / n_angles from `center` to the ring, clipped to
// the mask disc.  Marching positions are p_i = center + u (t0 + (i + 0.5) dl).
struct Ray {
  double ux, uy;  // direction
  double t0;      // first arclength of the clipped segment
  double dl;      // step
  int n;          // number of midpoint steps (0 = no contribution)
};

PACT_HD Ray make_ray(double cx, double cy, int a, int n_angles, double ring_r, double mcx,
                     double mcy, double mr, double step) {
  Ray ray;
  double theta = 2.0 * M_PI * a / n_angles;  // WavefrontProfile::angle, aberration.hpp:116
  ray.ux = cos(theta);
  ray.uy = sin(theta);
  double b = cx * ray.ux + cy * ray.uy;
  double c = (cx * cx + cy * cy) - ring_r * ring_r;
  double t_ring = -b + sqrt(b * b - c);
  double ex = cx + ray.ux * t_ring, ey = cy + ray.uy * t_ring;
  double t0, t1;
  seg_circle(cx, cy, ex, ey, mcx, mcy, mr, t0, t1);
  ray.n = 0;
  ray.t0 = 0.0;
  ray.dl = 0.0;
  if (t0 >= t1) return ray;  // aberration.hpp:163
  int n = static_cast<int>(ceil((t1 - t0) / step));
  ray.n = n < 1 ? 1 : n;
  ray.dl = (t1 - t0) / ray.n;
  ray.t0 = t0;
  return ray;
}

// Clamped bilinear stencil, detail::bilinear_stencil (aberration.hpp:41-72),
// in fp32 relative to the grid origin (fx, fy are pixel coordinates).
struct Stencil {
  int i00, i01, i10, i11;  // idx[0..3]
  float w00, w01, w10, w11;
};

__device__ __forceinline__ Stencil stencil_at(float fx, float fy, int W, int H) {
  fx = fminf(fmaxf(fx, 0.f), static_cast<float>(W - 1));
  fy = fminf(fmaxf(fy, 0.f), static_cast<float>(H - 1));
  int ix = min(static_cast<int>(fx), max(W - 2, 0));
  int iy = min(static_cast<int>(fy), max(H - 2, 0));
  float ax = fx - ix, ay = fy - iy;
  int ix1 = min(ix + 1, W - 1), iy1 = min(iy + 1, H - 1);
  Stencil s;
  s.i00 = iy * W + ix;
  s.i01 = iy * W + ix1;
  s.i10 = iy1 * W + ix;
  s.i11 = iy1 * W + ix1;
  s.w00 = (1.f - ax) * (1.f - ay);
  s.w01 = ax * (1.f - ay);
  s.w10 = (1.f - ax) * ay;
  s.w11 = ax * ay;
  return s;
}

// Per-ray record of a ray plan (raymarch.cu: ray_plan_kernel), computed once
// per geometry.
struct RayRec {
  float fxs, fys, dfx, dfy;  // midpoint pixel coordinates f_i = f_s + i df
  double dl;                 // step length
  int n;                     // steps
  int i_side, i_corner;      // regime boundaries or, generic rays, the fp64 corner index
  int flags;
};

// Arguments of the ray-march kernels (raymarch.cu).
struct RayArgs {
  const float* dv;  // SOS deviation raster v - v0, [H][W]
  int W, H;
  double ox, oy, inv_pitch;
  double v0;
  double ring_r;
  double mcx, mcy, mr;
  double step;
  int n_angles;
  int n_rays;
  const double2* centers;  // [n_centers]
  // Optional pitch-2D texture over dv (0: plain loads).  Interior stencils are
  // then one tex2Dgather instead of four scattered loads.
  cudaTextureObject_t tex;
  // Work plan of the texture path (ray_plan_get, raymarch.cu): per-ray
  // records, the sorted chunk list, each ray's partial-sum slots and the
  // owner's forward partials.
  const RayRec* rec;
  const int4* items;
  const int2* ray_slots;
  float* partial;
  int n_items;
  // Cell-gather plan of the interior adjoint (raymarch.cu; null: interior
  // items go through the per-ray kernel).  Stencil cells (W-1 x H-1) are
  // grouped in tiles of cell_t x cell_t, numbered tile-major (tile, then
  // row-major inside the tile, padded); cell c's interior steps are
  // cell_ent[cell_start[c] .. cell_start[c+1]), each local ray << cell_sb |
  // step, where local ray j of tile t is tile_rays[tile_start[t] + j].
  // cell_geo[r] = (fxs, fys, dfx, dfy) of ray r.  The items are sorted
  // generic | interior | side, so the adjoint skips [n_gen, n_gen + n_int).
  const unsigned* cell_start;
  const unsigned* cell_ent;
  const unsigned* tile_start;
  const unsigned* tile_rays;
  const float4* cell_geo;
  int cell_sb, cell_t, tile_max;
  int n_gen_items, n_int_items;
  // Border-line (side) plan of the adjoint (raymarch.cu; null: side items per
  // ray): every run of a ray's border-line steps in one border cell (<= 255
  // steps), as side_ent[k] = slot << 48 | (255 - steps) << 40 | ray << 20 |
  // first step << 8, sorted by (slot, steps desc, ray); slot = the border
  // cell's index in the [colL H | colR H | rowB W | rowT W] layout;
  // side_start[slot] its range; side_geo[r] = (fs, df) of ray r's border line.
  // The adjoint skips the side items [n_gen + n_int, n_items).
  const unsigned long long* side_ent;
  const unsigned* side_start;
  const float2* side_geo;
};

// Creates a point-sampled, clamped pitch-2D texture over a row-major fp32
// raster; returns false (and leaves *out = 0) when the row pitch does not meet
// the device's texture pitch alignment.
bool make_raster_texture(const float* dv, int W, int H, cudaTextureObject_t* out);

// freq_index, fft.hpp:35
PACT_HD int freq_index(int i, int n) { return i <= n / 2 ? i : i - n; }

}  // namespace pactgpu
