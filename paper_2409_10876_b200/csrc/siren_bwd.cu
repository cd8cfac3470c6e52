// SIREN backward for hidden width 128 on tcgen05 (3xTF32, tc.cuh): ONE kernel
// per hidden layer l computes both gradients of the layer from a single pass
// over its inputs (backprop_sos, nfield.hpp:190-230):
//
//   dA_{l-1} = (W_l^T dA_l) * w0 cos(w0 a_{l-1})          data gradient
//   gW_l    += dA_l^T sin(w0 a_{l-1}),  gb_l += sum dA_l    weight gradient
//
// TOP (l = L-1): dA_l is formed on the fly from a_l and the pixel gradient g
//   (the output layer, nfield.hpp:194-205: dA = g s w0 w_L cos(w0 a_l)), and
//   the head partials gw_L = sum g s sin(w0 a_l), gb_L = sum g s are kept.
// BOTTOM (l = 1): dA_0 is not stored; its layer-0 partials
//   gW_0 = sum dA_0 c^T, gb_0 = sum dA_0 (nfield.hpp:228-232) are accumulated
//   in the epilogue.  a_0 = W_0 c + b_0 is recomputed from the pixel
//   coordinates (two FMAs, the forward's expression) instead of being stored
//   by the forward and streamed back (-2 x 4 B per pixel and feature).
// So a 4-layer network's backward is 3 launches reading a_1..a_3 once each
// plus dA_2, dA_1 (written once, read once) instead of 8 kernels.
//
// Per 32-pixel tile (persistent CTAs, tile t = blockIdx + i * grid):
//   TMEM  W_l^T hi [0,128) lo [128,256) (lane = input feature k, column = j);
//         weight-gradient accumulator D_w [256,384) (lane = j, column = k,
//         summed over every tile of the CTA); dA^T of the tile hi [384,416)
//         lo [416,448) (lane = j, column = pixel: the weight gradient's A);
//         data-gradient accumulators D_g[buf] [448 + 32 buf, +32)
//         (lane = k, column = pixel).
//   smem  ND buffers of dA planes (rows = pixel, K = j; SW128: the data
//         gradient's B) -- the hi plane is the dA_l tile itself, written by
//         TMA tensor loads in that swizzle (kind::tf32 ignores the low 13
//         mantissa bits), so producers only add the lo plane; NZ buffers of z
//         planes (rows = k, K = pixel, z = sin(w0 a_{l-1}): the weight
//         gradient's B); NR slots of raw a_{l-1} tiles (cp.async.bulk).
//   weight grad.   D_w[j][k] += sum_p dA^T[j][p] z[p][k]  (TS MMA, K = pixels)
//   data gradient  D_g[k][p]  = sum_j W^T[k][j] dA[p][j] (TS MMA, N = 32 pixels)
// (kind::tf32 has no MN-major operands -- a transposed descriptor yields
// zeros -- so each operand is written in its K-major orientation by the
// producer thread that owns the feature.)
// Roles: warps 0-7 own dA (thread = feature j, 16 pixels), warps 8-15 own
// a_{l-1} (thread = feature k, 16 pixels, from the raw slots), warp 16
// issues the MMAs (one elected lane), warps 17-24 drain D_g (lane = feature:
// coalesced 128-B stores of dA_{l-1}; the cosine factor from the raw slot)
// and issue the loads (a buffer is refilled as soon as its consumers are done:
// both inputs stream ND - 1 / NR - 1 tiles ahead).  With the planes double-buffered the producers
// build tile i + 1 while the tensor core runs tile i; only the dA^T columns
// are single (TMEM is full) and wait for the previous weight gradient.
// Partials are per CTA and reduced in fp64 in a fixed order by the caller
// (deterministic).
#include <cstdint>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "siren.cuh"

// BWD_EXP (timing experiments only, wrong results; never set in the product
// build): 1 = dA^T store does not wait for the previous weight gradient,
// 2 = no weight-gradient MMAs, 3 = no data-gradient MMAs, 4 = no MMAs,
// 5 = store-only timeline of CTA 0 of the middle-layer kernel (read by
// pact_debug_bwd_trace).
#ifndef BWD_EXP
#define BWD_EXP 0
#endif
#if BWD_EXP == 5
#ifndef BWD_TRACE_MODE
#define BWD_TRACE_MODE 0
#endif
__device__ unsigned long long g_btrace[16][512];
#define BTRACE(cond, tag, idx)                                                      \
  do {                                                                              \
    if (MODE == BWD_TRACE_MODE && blockIdx.x == 0 && (cond) && (idx) < 512) {      \
      unsigned long long t_;                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
      g_btrace[tag][idx] = t_;                                                      \
    }                                                                               \
  } while (0)
#else
#define BTRACE(cond, tag, idx)
#endif
#include "tc.cuh"

namespace pactgpu {
namespace {

constexpr int BH = 128;                 // hidden width
constexpr int BT = 32;                  // pixels per tile
#ifndef BWD_ND
#define BWD_ND 4
#endif
#ifndef BWD_NZ
#define BWD_NZ 1
#endif
#ifndef BWD_NR
#define BWD_NR 3
#endif
constexpr int ND = BWD_ND;              // dA plane buffers (TMA-filled hi plane)
constexpr int NZ = BWD_NZ;              // z plane buffers
constexpr int NR = BWD_NR;              // raw a_{l-1} slots (z producers, epilogue)
constexpr uint32_t kRaw = BT * BH;      // floats of one raw tile: 16 KB
constexpr uint32_t kDa = BT * BH;       // floats of one dA plane (rows = pixel): 16 KB
constexpr uint32_t kZ = BH * BT;        // floats of one z plane (rows = feature): 16 KB
constexpr int kDW = 8, kZW = 8, kEpiW = 8;    // warps per role
constexpr int kMmaWarp = kDW + kZW;           // 16
constexpr int kThr = 32 * (kDW + kZW + 1 + kEpiW);  // 800
constexpr uint32_t kColWlo = 128, kColDw = 256, kColT = 384, kColDg = 448;

enum : int { kTop = 1, kBottom = 2 };

struct BwdArgs {
  const float* X;       // dA_l [n][128]; TOP: a_l
  const float* Aprev;   // a_{l-1} [n][128]
  const float* W;       // W_l [128][128] row-major
  const double* gv;     // TOP: fp64 gradient raster (may be null)
  const float* gmask;   // TOP: per-masked-pixel gradient (may be null)
  const int* idx;       // TOP: masked pixel -> raster index
  const float* wL;      // TOP: head weights [128]
  const float* gpx;     // TOP: g s per masked pixel [n] (gather_g_kernel)
  const float2* coords; // BOTTOM
  const float* W0;      // BOTTOM: layer 0 [128][2], b0 [128] (a_0 = W_0 c + b_0)
  const float* b0;
  float out_scale, w0;
  int n;
  float* Y;         // dA_{l-1} [n][128] (not BOTTOM)
  float* part_w;    // [grid][128 * 128 + 128]
  float* part_top;  // TOP: [grid][129]
  float* part_0;    // BOTTOM: [grid][3 * 128]
};

struct BwdBars {
  uint64_t xfull[ND];  // dA_l tile landed in the hi plane of buffer x (TMA)
  uint64_t rfull[NR];  // raw a_{l-1} tile landed (bulk copy)
  uint64_t rfree[NR];  // raw tile read (z producers + epilogue)
  uint64_t zready[NZ]; // z planes of buffer z written (z producers)
  uint64_t wfree[NZ];  // weight-gradient MMAs of buffer z done (commit)
  uint64_t tready;     // dA^T columns written (dA producers)
  uint64_t tfree;      // weight-gradient MMAs done with the dA^T columns (commit)
  uint64_t gready[ND]; // dA planes of buffer x complete (dA producers)
  uint64_t dfull[2];   // D_g[b] ready (commit; also frees the dA buffer)
  uint64_t dfree[2];   // D_g[b] drained (epilogue)
  uint64_t acc;        // D_w final (commit)
  uint32_t tslot;
};

__device__ __forceinline__ float red2pi_b(float x) { return sine_reduce(x); }
__device__ __forceinline__ void sincos_w(float a, float w0, float* s, float* c) {
  __sincosf(red2pi_b(w0 * a), s, c);
}

__device__ __forceinline__ uint32_t saddr_b(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// SW128 K-major float offset of (row, k) in a plane of 128-B rows (32 fp32 of K)
__device__ __forceinline__ uint32_t sw128(int row, int k) {
  return static_cast<uint32_t>(row * 32 + ((((k >> 2) ^ (row & 7))) << 2) + (k & 3));
}

// g s per masked pixel (the output layer's input gradient, nfield.hpp:194-197):
// the gather through the pixel index happens once here, not per tile.
__global__ void gather_g_kernel(const double* __restrict__ gv, const float* __restrict__ gmask,
                                const int* __restrict__ idx, int n, float scale, float* __restrict__ out) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  float gg = 0.f;
  if (gv) gg += static_cast<float>(gv[idx[m]]);
  if (gmask) gg += gmask[m];
  out[m] = gg * scale;
}

template <int MODE>
__global__ void __launch_bounds__(kThr, 1)
tc_bwd_kernel(BwdArgs a, const __grid_constant__ CUtensorMap tmap_x) {
  constexpr bool TOP = (MODE & kTop) != 0, BOTTOM = (MODE & kBottom) != 0;
  extern __shared__ unsigned char smem_dyn[];
  // pda[x]: dA hi [4 chunks][BT][32] | dA lo;  pz[z]: z hi [BH][BT] | z lo  (SW128)
  // raw[r]: a_{l-1} tile [BT][BH] (contiguous rows)
  float* pda = tc::smem_align1024<float>(smem_dyn);
  float* pz = pda + ND * 2 * kDa;
  float* raw = pz + NZ * 2 * kZ;
  float* red = raw + NR * kRaw;  // [2][BH] bias, [2][BH] head, [2] gb, pad; then [3][BH] fp64
  float* wst = pda;              // prologue: W staged [BH][BH + 1] over the dA buffers
  __shared__ BwdBars sb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tc::tmem_alloc<512>(&sb.tslot);
  if (tid == 0) {
    for (int i = 0; i < ND; ++i) {
      tc::mbar_init(&sb.xfull[i], 1);
      tc::mbar_init(&sb.gready[i], 32 * kDW);
    }
    for (int i = 0; i < NR; ++i) {
      tc::mbar_init(&sb.rfull[i], 1);
      tc::mbar_init(&sb.rfree[i], 32 * (kZW + kEpiW));
    }
    for (int i = 0; i < NZ; ++i) {
      tc::mbar_init(&sb.zready[i], 32 * kZW);
      tc::mbar_init(&sb.wfree[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sb.dfull[i], 1);
      tc::mbar_init(&sb.dfree[i], 32 * kEpiW);
    }
    tc::mbar_init(&sb.tready, 32 * kDW);
    tc::mbar_init(&sb.tfree, 1);
    tc::mbar_init(&sb.acc, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int n = a.n;
  const int n_tiles = (n + BT - 1) / BT;
  const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto tile_m0 = [&](int i) { return (blockIdx.x + i * gridDim.x) * BT; };
  // raw a_{l-1} tile i (rows m0.., contiguous) -> raw[i % NR] (one thread)
  auto load_raw = [&](int i) {
    const int m0 = tile_m0(i);
    const uint32_t bytes = static_cast<uint32_t>(min(BT, n - m0)) * BH * 4;
    uint64_t* bar = &sb.rfull[i % NR];
    tc::mbar_expect_tx(bar, bytes);
    tc::bulk_load(raw + (i % NR) * kRaw, a.Aprev + static_cast<size_t>(m0) * BH, bytes, bar);
  };
  // dA_l (TOP: a_l) tile i -> hi plane of buffer i % ND: four 32 x 32 SW128
  // boxes (rows >= n zero-filled) (one thread)
  auto load_x = [&](int i) {
    const int m0 = tile_m0(i);
    uint64_t* bar = &sb.xfull[i % ND];
    tc::mbar_expect_tx(bar, 4 * BT * 32 * 4);
    float* d = pda + (i % ND) * 2 * kDa;
#pragma unroll
    for (int c = 0; c < 4; ++c) tc::tma_load_2d(d + c * BT * 32, &tmap_x, 32 * c, m0, bar);
  };
  if (tid == 0 && !BOTTOM)
    for (int i = 0; i < NR && i < my_tiles; ++i) load_raw(i);
  // W_l -> TMEM as the data gradient's A operand: A[k][j] = W[j][k] (lane k)
  for (int e = tid; e < BH * BH / 4; e += kThr) {
    const float4 w4 = reinterpret_cast<const float4*>(a.W)[e];
    float* d = wst + (e / (BH / 4)) * (BH + 1) + (e % (BH / 4)) * 4;
    d[0] = w4.x;
    d[1] = w4.y;
    d[2] = w4.z;
    d[3] = w4.w;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t t0 = sb.tslot;
  // 16 (lane quarter, plane, K half) pieces, piece = warp (quarter = warp % 4:
  // a warp may only touch TMEM lanes 32 (warp % 4) ..)
  if (warp < 16) {
    const bool lo_plane = warp >= 8;
    const int row = 32 * (warp & 3) + lane;
    const uint32_t lb = t0 + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + (lo_plane ? kColWlo : 0);
    const int kb = ((warp >> 2) & 1) * (BH / 2);
#pragma unroll 1
    for (int k0 = kb; k0 < kb + BH / 2; k0 += 32) {
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        float hi, lo;
        tc::split_tf32(wst[(k0 + i) * (BH + 1) + row], hi, lo);
        v[i] = lo_plane ? lo : hi;
      }
      tc::tmem_st32(lb + k0, v);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    tc::fence_proxy_async();  // the W staging reads precede the TMA writes over it
    for (int i = 0; i < ND && i < my_tiles; ++i) load_x(i);
  }

  const float w0 = a.w0;
  constexpr int HP = BT / 2;  // pixels per producer / epilogue thread

  if (warp < kDW) {
    // ---- dA producers: thread = feature j, pixels [16 h, 16 h + 16) ----
    const int q = warp & 3, h = warp >> 2, j = 32 * q + lane, pb = HP * h;
    const float wlj = TOP ? a.wL[j] : 0.f;
    float bacc = 0.f, hacc = 0.f, gbacc = 0.f;
    // TOP: lane t < 16 holds g s of pixel pb + t of the tile (shuffled when
    // used), from the compact per-pixel array (one coalesced load)
    auto load_g = [&](int i) {
      const int m = tile_m0(i) + pb + (lane & (HP - 1));
      return m < n ? a.gpx[m] : 0.f;
    };
    float gnext = (TOP && my_tiles > 0) ? load_g(0) : 0.f;
    for (int i = 0; i < my_tiles; ++i) {
      const int bx = i % ND;
      const int rows = min(BT, n - tile_m0(i));
      const float gr = gnext;
      if (TOP && i + 1 < my_tiles) gnext = load_g(i + 1);
      tc::mbar_wait(&sb.xfull[bx], (i / ND) & 1);
      BTRACE(tid == 0, 1, i);
      // this thread's column of the hi plane (chunk q, feature lane)
      float* dh = pda + bx * 2 * kDa + q * (BT * 32);
      float* dl = dh + kDa;
      // all loads of the column first (the stores below cannot alias them)
      float hi[HP], lo[HP];
#pragma unroll
      for (int t = 0; t < HP; ++t) hi[t] = dh[sw128(pb + t, lane)];
      BTRACE(tid == 0, 12, i);
#pragma unroll
      for (int t = 0; t < HP; ++t) {
        float v = hi[t];
        if (TOP) {
          // output layer (nfield.hpp:194-205), the expression of siren_top_kernel
          const float gg = __shfl_sync(0xffffffffu, gr, t);
          float sx, cx;
          sincos_w(v, w0, &sx, &cx);
          v = gg * w0 * wlj * cx;
          if (pb + t < rows) hacc = fmaf(gg, sx, hacc);
          if (j == 0) gbacc += gg;
        }
        // rows past n arrive as zeros (TMA bounds); TOP gives them g = 0
        bacc += v;
        tc::split_tf32_trunc(v, hi[t], lo[t]);
      }
      BTRACE(tid == 0, 14, i);
      // dA^T into TMEM first (the weight gradient's A: lane = j, column =
      // pixel; the critical path) once the previous weight gradient is done
      if (i >= 1 && BWD_EXP != 1) tc::mbar_wait(&sb.tfree, (i - 1) & 1);
      BTRACE(tid == 0, 3, i);
      tc::fence_after_sync();
      const uint32_t lb = t0 + (static_cast<uint32_t>(32 * q) << 16) + kColT + pb;
      tc::tmem_st16_nowait(lb, hi);
      tc::tmem_st16_nowait(lb + BT, lo);
      tc::tmem_wait_st();
      tc::fence_before_sync();
      tc::mbar_arrive(&sb.tready);
      BTRACE(tid == 0, 4, i);
      // then the lo plane (TOP: and the hi plane) for the data gradient
#pragma unroll
      for (int t = 0; t < HP; ++t) {
        const uint32_t o = sw128(pb + t, lane);
        if (TOP) dh[o] = hi[t];
        dl[o] = lo[t];
      }
      BTRACE(tid == 0, 13, i);
      tc::fence_proxy_async();
      tc::mbar_arrive(&sb.gready[bx]);
      BTRACE(tid == 0, 2, i);
    }
    red[h * BH + j] = bacc;
    if (TOP) {
      red[2 * BH + h * BH + j] = hacc;
      if (j == 0) red[4 * BH + h] = gbacc;
    }
    tc::named_sync(1, 32 * kDW);
    if (h == 0) {
      a.part_w[static_cast<size_t>(blockIdx.x) * (BH * BH + BH) + BH * BH + j] = red[j] + red[BH + j];
      if (TOP) {
        float* pt = a.part_top + static_cast<size_t>(blockIdx.x) * (BH + 1);
        pt[j] = red[2 * BH + j] + red[3 * BH + j];
        if (j == 0) pt[BH] = red[4 * BH] + red[4 * BH + 1];
      }
    }
  } else if (warp < kDW + kZW) {
    // ---- a_{l-1} producers: thread = feature k, pixels [16 h, 16 h + 16) ----
    const int q = warp & 3, h = (warp - kDW) >> 2, k = 32 * q + lane, pb = HP * h;
    // BOTTOM: a_0 = W_0 c + b_0 from the coordinates (lane t < 16 holds pixel
    // pb + t of the tile, one tile ahead)
    float w0x = 0.f, w0y = 0.f, b0k = 0.f;
    float2 cnext = make_float2(0.f, 0.f);
    auto load_c = [&](int i) {
      return a.coords[min(tile_m0(i) + pb + (lane & (HP - 1)), n - 1)];
    };
    if (BOTTOM) {
      w0x = a.W0[2 * k];
      w0y = a.W0[2 * k + 1];
      b0k = a.b0[k];
      if (my_tiles > 0) cnext = load_c(0);
    }
    for (int i = 0; i < my_tiles; ++i) {
      const int bz = i % NZ, r = i % NR;
      const int rows = min(BT, n - tile_m0(i));
      const float2 cc = cnext;
      if (BOTTOM && i + 1 < my_tiles) cnext = load_c(i + 1);
      if (!BOTTOM) tc::mbar_wait(&sb.rfull[r], (i / NR) & 1);
      BTRACE(warp == kDW && lane == 0, 5, i);
      const float* ar = raw + r * kRaw + pb * BH + k;
      float zh4[HP], zl4[HP];
#pragma unroll
      for (int t = 0; t < HP; ++t) {
        const float av = BOTTOM ? fmaf(w0y, __shfl_sync(0xffffffffu, cc.y, t),
                                       fmaf(w0x, __shfl_sync(0xffffffffu, cc.x, t), b0k))
                                : ar[t * BH];
        float z = __sinf(red2pi_b(w0 * av));
        if (pb + t >= rows) z = 0.f;
        tc::split_tf32_trunc(z, zh4[t], zl4[t]);
      }
      if (!BOTTOM) tc::mbar_arrive(&sb.rfree[r]);
      // z planes (the weight gradient's B: row = k, K = pixel) of buffer bz
      if (i >= NZ) tc::mbar_wait(&sb.wfree[bz], ((i - NZ) / NZ) & 1);
      BTRACE(warp == kDW && lane == 0, 6, i);
      float* zh = pz + bz * 2 * kZ;
      float* zl = zh + kZ;
#pragma unroll
      for (int t = 0; t < HP; t += 4) {
        const uint32_t o = sw128(k, pb + t);
        *reinterpret_cast<float4*>(zh + o) = make_float4(zh4[t], zh4[t + 1], zh4[t + 2], zh4[t + 3]);
        *reinterpret_cast<float4*>(zl + o) = make_float4(zl4[t], zl4[t + 1], zl4[t + 2], zl4[t + 3]);
      }
      BTRACE(warp == kDW && lane == 0, 11, i);
      tc::fence_proxy_async();
      tc::mbar_arrive(&sb.zready[bz]);
      BTRACE(warp == kDW && lane == 0, 7, i);
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issue: the weight gradient of tile i (frees its z buffer and
    // the dA^T columns), then its data gradient (frees its dA buffer) ----
    constexpr uint32_t idesc_w = tc::idesc_tf32(BH, BH);
    constexpr uint32_t idesc_g = tc::idesc_tf32(BH, BT);
    // data gradient of tile i (buffer i % ND -> D_g[i & 1])
    auto dgrad = [&](int i) {
      const int b = i & 1, bx = i % ND;
      tc::mbar_wait(&sb.gready[bx], (i / ND) & 1);
      if (i >= 2) tc::mbar_wait(&sb.dfree[b], ((i - 2) >> 1) & 1);
      BTRACE(lane == 0, 9, i);
      tc::fence_after_sync();
      const uint32_t dah = saddr_b(pda + bx * 2 * kDa), dal = dah + 4 * kDa;
      if (tc::elect_one()) {
        const uint32_t dcol = t0 + kColDg + BT * b;
#pragma unroll
        for (int c = 0; c < (BWD_EXP == 3 || BWD_EXP == 4 ? 0 : BH / 32); ++c)
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const uint32_t ka = c * 32 + 8 * s;
            const uint64_t bh = tc::smem_desc_sw128(dah + c * BT * 128 + 32 * s);
            const uint64_t bl = tc::smem_desc_sw128(dal + c * BT * 128 + 32 * s);
            tc::mma_tf32_ts(dcol, t0 + kColWlo + ka, bh, idesc_g, (c | s) != 0);
            tc::mma_tf32_ts(dcol, t0 + ka, bl, idesc_g, 1u);
            tc::mma_tf32_ts(dcol, t0 + ka, bh, idesc_g, 1u);
          }
        tc::mma_commit(&sb.dfull[b]);
        if (i + 1 == my_tiles) tc::mma_commit(&sb.acc);
      }
      __syncwarp();
    };
    // issue order wgrad(0), wgrad(1), dgrad(0), wgrad(2), dgrad(1), ...: the
    // data gradient of tile i - 1 runs while the producers put tile i + 1's
    // dA^T into TMEM, so the tensor core always has the next MMAs queued
    for (int i = 0; i < my_tiles; ++i) {
      const int bz = i % NZ;
      tc::mbar_wait(&sb.zready[bz], (i / NZ) & 1);
      tc::mbar_wait(&sb.tready, i & 1);
      BTRACE(lane == 0, 8, i);
      tc::fence_after_sync();
      const uint32_t zh = saddr_b(pz + bz * 2 * kZ), zl = zh + 4 * kZ;
      if (tc::elect_one()) {
#pragma unroll
        for (int s = 0; s < (BWD_EXP == 2 || BWD_EXP == 4 ? 0 : BT / 8); ++s) {
          const uint32_t ta = t0 + kColT + 8 * s;
          const uint64_t bh = tc::smem_desc_sw128(zh + 32 * s);
          const uint64_t bl = tc::smem_desc_sw128(zl + 32 * s);
          tc::mma_tf32_ts(t0 + kColDw, ta + BT, bh, idesc_w, (i | s) != 0);
          tc::mma_tf32_ts(t0 + kColDw, ta, bl, idesc_w, 1u);
          tc::mma_tf32_ts(t0 + kColDw, ta, bh, idesc_w, 1u);
        }
        tc::mma_commit(&sb.tfree);
        tc::mma_commit(&sb.wfree[bz]);
      }
      __syncwarp();
      if (i >= 1) dgrad(i - 1);
    }
    if (my_tiles > 0) dgrad(my_tiles - 1);
  } else {
    // ---- epilogue: lane = input feature k, pixels [16 h, 16 h + 16) ----
    const int e = warp - kMmaWarp - 1;
    const int q = warp & 3, h = e >> 2, k = 32 * q + lane, pb = HP * h;
    const uint32_t lb = t0 + (static_cast<uint32_t>(32 * q) << 16);
    const bool loader = warp == kThr / 32 - 1 && lane == 0;  // issues the loads i + NR, i + ND
    double gx = 0.0, gy = 0.0, gb = 0.0;
    float w0x = 0.f, w0y = 0.f, b0k = 0.f;
    float2 cnext = make_float2(0.f, 0.f);
    auto load_c = [&](int i) {
      return a.coords[min(tile_m0(i) + pb + (lane & (HP - 1)), n - 1)];
    };
    if (BOTTOM) {
      w0x = a.W0[2 * k];
      w0y = a.W0[2 * k + 1];
      b0k = a.b0[k];
      if (my_tiles > 0) cnext = load_c(0);
    }
    for (int i = 0; i < my_tiles; ++i) {
      const int b = i & 1, r = i % NR;
      const int m0 = tile_m0(i), rows = min(BT, n - m0);
      const float2 cme = cnext;
      if (BOTTOM && i + 1 < my_tiles) cnext = load_c(i + 1);
      float cw[HP];
      if (BOTTOM) {
        // a_0 = W_0 c + b_0 (the forward's expression)
#pragma unroll
        for (int t = 0; t < HP; ++t) {
          const float av = fmaf(w0y, __shfl_sync(0xffffffffu, cme.y, t),
                                fmaf(w0x, __shfl_sync(0xffffffffu, cme.x, t), b0k));
          cw[t] = w0 * __cosf(red2pi_b(w0 * av));
        }
      } else {
        // the cosine factor from the raw a_{l-1} tile
        tc::mbar_wait(&sb.rfull[r], (i / NR) & 1);
        const float* ar = raw + r * kRaw + pb * BH + k;
#pragma unroll
        for (int t = 0; t < HP; ++t) cw[t] = w0 * __cosf(red2pi_b(w0 * ar[t * BH]));
        tc::mbar_arrive(&sb.rfree[r]);
        if (loader && i + NR < my_tiles) {
          tc::mbar_wait(&sb.rfree[r], (i / NR) & 1);
          tc::fence_proxy_async();  // generic reads of the slot before the refill
          load_raw(i + NR);
        }
      }
      __syncwarp();
      tc::mbar_wait(&sb.dfull[b], (i >> 1) & 1);
      BTRACE(warp == kMmaWarp + 1 && lane == 0, 10, i);
      // dA buffer i % ND is free (its data gradient is done): refill it
      if (loader && i + ND < my_tiles) load_x(i + ND);
      tc::fence_after_sync();
      float v[HP];
      tc::tmem_ld16(lb + kColDg + BT * b + pb, v);
      tc::fence_before_sync();
      tc::mbar_arrive(&sb.dfree[b]);
      if (!BOTTOM) {
        float* y = a.Y + static_cast<size_t>(m0 + pb) * BH + k;
#pragma unroll
        for (int t = 0; t < HP; ++t)
          if (pb + t < rows) y[static_cast<size_t>(t) * BH] = v[t] * cw[t];
      } else {
        // fp32 sums over the tile's 16 pixels, then one fp64 add per tile
        float sx = 0.f, sy = 0.f, s1 = 0.f;
#pragma unroll
        for (int t = 0; t < HP; ++t) {
          const float out = pb + t < rows ? v[t] * cw[t] : 0.f;
          sx = fmaf(out, __shfl_sync(0xffffffffu, cme.x, t), sx);
          sy = fmaf(out, __shfl_sync(0xffffffffu, cme.y, t), sy);
          s1 += out;
        }
        gx += static_cast<double>(sx);
        gy += static_cast<double>(sy);
        gb += static_cast<double>(s1);
      }
    }
    if (BOTTOM) {
      // fixed-order sum of the two pixel halves
      double* rd = reinterpret_cast<double*>(red + 4 * BH + 8);  // [3][BH]
      if (h == 1) {
        rd[k] = gx;
        rd[BH + k] = gy;
        rd[2 * BH + k] = gb;
      }
      tc::named_sync(2, 32 * kEpiW);
      if (h == 0) {
        float* p0 = a.part_0 + static_cast<size_t>(blockIdx.x) * (3 * BH);
        p0[2 * k] = static_cast<float>(gx + rd[k]);
        p0[2 * k + 1] = static_cast<float>(gy + rd[BH + k]);
        p0[2 * BH + k] = static_cast<float>(gb + rd[2 * BH + k]);
      }
    }
    // weight-gradient accumulator -> this CTA's partial (row j = lane; the
    // two warps of a lane quarter take half the columns each)
    float* out = a.part_w + static_cast<size_t>(blockIdx.x) * (BH * BH + BH) + static_cast<size_t>(k) * BH;
    if (my_tiles > 0) {
      tc::mbar_wait(&sb.acc, 0);
      tc::fence_after_sync();
#pragma unroll 1
      for (int c0 = h * (BH / 2); c0 < (h + 1) * (BH / 2); c0 += 32) {
        float w[32];
        tc::tmem_ld32(lb + kColDw + c0, w);
#pragma unroll
        for (int jj = 0; jj < 32; jj += 4)
          *reinterpret_cast<float4*>(out + c0 + jj) = make_float4(w[jj], w[jj + 1], w[jj + 2], w[jj + 3]);
      }
    } else {
      for (int c = h * (BH / 2); c < (h + 1) * (BH / 2); ++c) out[c] = 0.f;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(t0);
}

constexpr size_t kBwdSmem = 1024 + sizeof(float) * (ND * 2 * kDa + NZ * 2 * kZ + NR * kRaw + 10 * BH + 8);

template <int MODE>
Status launch_bwd(pact_ctx* ctx, const BwdArgs& a, int grid) {
  PACT_TRY_S(smem_optin(tc_bwd_kernel<MODE>, kBwdSmem));
  // X = dA_l (TOP: a_l) as a 2-D tensor [n][128] fp32, 32 x 32 SW128 boxes
  static PFN_cuTensorMapEncodeTiled encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }();
  if (!encode) return internal_error("tc_bwd_layer: cuTensorMapEncodeTiled unavailable");
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(BH), static_cast<cuuint64_t>(a.n)};
  const cuuint64_t strides[1] = {sizeof(float) * BH};
  const cuuint32_t box[2] = {32, BT}, estr[2] = {1, 1};
  if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.X), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return internal_error("tc_bwd_layer: tensor map encoding failed");
  tc_bwd_kernel<MODE><<<grid, kThr, kBwdSmem, ctx->stream>>>(a, tmap);
  return after_launch(ctx, "tc_bwd_kernel");
}

}  // namespace

int tc_bwd_grid(pact_ctx* ctx, int n) { return std::max(1, std::min(ctx->num_sms, div_up(n, BT))); }

Status tc_bwd_layer(pact_ctx* ctx, bool top, bool bottom, const TcBwdLayer& L) {
  BwdArgs a{};
  a.X = L.X;
  a.Aprev = L.Aprev;
  a.W = L.W;
  a.gv = L.gv;
  a.gmask = L.gmask;
  a.idx = L.idx;
  a.wL = L.wL;
  a.gpx = L.gpx;
  if (top) {
    if (!L.gpx) return internal_error("tc_bwd_layer: top layer needs the g scratch");
    gather_g_kernel<<<div_up(L.n, 256), 256, 0, ctx->stream>>>(L.gv, L.gmask, L.idx, L.n, L.out_scale,
                                                              L.gpx);
    PACT_TRY_S(after_launch(ctx, "gather_g_kernel"));
  }
  a.coords = L.coords;
  a.W0 = L.W0;
  a.b0 = L.b0;
  a.out_scale = L.out_scale;
  a.w0 = L.w0;
  a.n = L.n;
  a.Y = L.Y;
  a.part_w = L.part_w;
  a.part_top = L.part_top;
  a.part_0 = L.part_0;
  const int grid = tc_bwd_grid(ctx, L.n);
  if (top && bottom) return launch_bwd<kTop | kBottom>(ctx, a, grid);
  if (top) return launch_bwd<kTop>(ctx, a, grid);
  if (bottom) return launch_bwd<kBottom>(ctx, a, grid);
  return launch_bwd<0>(ctx, a, grid);
}

}  // namespace pactgpu

#if BWD_EXP == 5
extern "C" int pact_debug_bwd_trace(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (out) cudaMemcpyFromSymbol(out, g_btrace, sizeof(unsigned long long) * 16 * 512);
  if (reset) {
    static unsigned long long zero[16 * 512];
    cudaMemcpyToSymbol(g_btrace, zero, sizeof(zero));
  }
  return 512;
}
#endif
