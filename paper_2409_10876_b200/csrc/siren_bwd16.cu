// SIREN backward for hidden width 128 on kind::f16 tcgen05 MMAs with split-fp16
// operands: the same fused per-layer kernel as siren_bwd.cu (one launch per
// hidden layer computes both gradients, backprop_sos, nfield.hpp:190-230),
//
//   dA_{l-1} = (W_l^T dA_l) * w0 cos(w0 a_{l-1})          data gradient
//   gW_l    += dA_l^T sin(w0 a_{l-1}),  gb_l += sum dA_l    weight gradient
//
// with every operand held as fp16 hi + lo (tc::split_f16x2; hi*hi + hi*lo +
// lo*hi carries the 22 significant bits of the 3xTF32 split) at twice the
// TF32 tensor rate and half the operand bytes.
//
// fp16 has a narrow exponent range, so each operand is scaled by a power of
// two (exact, undone in the epilogues):
//   z = sin(.) in [-1, 1]                 unscaled
//   W_l            * sw, sw = 2^(14 - e) with max|W_l| < 2^e   (computed in the prologue)
//   dA_l           * sd, sd = 2^(14 - e) with bound(|dA_l|) < 2^e, where the bound is
//     TOP:   max|g s| * w0 * max|w_L|   (max|g s| from gather_g16_kernel)
//     other: max|dA_l| measured exactly by the previous launch's epilogue
//            (it produces dA_l: a per-warp max and one atomicMax on its bits).
// Scaled magnitudes stay below 2^14 < 65504; terms below the fp16 normal
// range keep an absolute error <= 2^-25 of the scaled unit (2^-39 of the
// tensor's maximum).
//
// Per 32-pixel tile (persistent CTAs, tile t = blockIdx + i * grid):
//   TMEM  W_l^T hi [0,64) lo [64,128) (lane = input feature k, two output
//         features j per column); D_w [128,256) (lane = j, column = k, summed
//         over the CTA's tiles); D_g[b] [256 + 32b, +32) (lane = k, column = pixel).
//   smem  NX raw dA_l (TOP: a_l) slots and NR raw a_{l-1} slots (bulk copies,
//         rows contiguous); ND dA plane buffers (row = pixel, 64 features per
//         128-B row in two chunks, hi then lo); NZ z plane buffers (row = k: 32
//         pixels of hi then 32 of lo in one 128-B row).  All SWIZZLE_128B.
//   weight grad.   D_w[j][k] += sum_p dA[p][j] z[p][k]: A = the dA planes read
//                  MN-major (M = j), B = the z planes (K-major); 2 K steps x 3 MMAs
//   data gradient  D_g[k][p]  = sum_j W^T[k][j] dA[p][j]: A = W^T (TMEM),
//                  B = the same dA planes K-major (K = j); 8 K steps x 3 MMAs
// So each dA value is converted and stored once, by a thread owning (pixel,
// 8 features) -- no transposition in the producers.  The raw dA_l slot is
// refilled as soon as the producers have read it, and the MMAs of a tile
// issue in order (wgrad(i), dgrad(i)).
// Roles: warps 0-7 own dA (thread = pixel and 8 features), warps 8-15 own
// a_{l-1} (thread = feature k, 16 pixels: z = sin(w0 a) and the epilogue's
// factor w0 cos(w0 a) from one argument reduction; they issue the raw a_{l-1}
// loads), warp 16 issues the MMAs, warps 17-24 drain D_g (thread = feature
// k: coalesced stores of dA_{l-1}).  Partials are per CTA, reduced in fixed
// orders here and in fp64 by the caller (deterministic).
#include <cstdint>
#include <cstdlib>

#include "siren.cuh"
#include "tc.cuh"

// BWD16_TRACE (timing experiments only; never set in the product build):
// globaltimer stamps per role and tile of CTA 0 of the middle-layer kernel,
// read by pact_debug_bwd_trace (scripts/bwd_trace.py).
#ifndef BWD16_SERIAL
#define BWD16_SERIAL 0
#endif
#ifndef BWD16_TRACE
#define BWD16_TRACE 0
#endif
#if BWD16_TRACE
__device__ unsigned long long g_btrace[16][512];
#define BTRACE(cond, tag, idx)                                                 \
  do {                                                                         \
    if (MODE == 0 && blockIdx.x == 0 && (cond) && (idx) < 512) {               \
      unsigned long long t_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
      g_btrace[tag][idx] = t_;                                                 \
    }                                                                          \
  } while (0)
#else
#define BTRACE(cond, tag, idx)
#endif

namespace pactgpu {
namespace {

constexpr int BH = 128;  // hidden width
constexpr int BT = 32;   // pixels per tile
constexpr int HP = BT / 2;
#ifndef BWD16_NX
#define BWD16_NX 3
#endif
#ifndef BWD16_ND
#define BWD16_ND 2
#endif
#ifndef BWD16_NZ
#define BWD16_NZ 2
#endif
#ifndef BWD16_NR
#define BWD16_NR 3
#endif
#ifndef BWD16_NC
#define BWD16_NC 2
#endif
constexpr int NX = BWD16_NX, ND = BWD16_ND, NZ = BWD16_NZ, NR = BWD16_NR, NC = BWD16_NC;
constexpr uint32_t kRaw = BT * BH;          // floats of a raw tile (16 KB)
constexpr uint32_t kPlane = BT * BH;        // 32-bit words of one dA buffer: hi 2 x 4 KB | lo 2 x 4 KB
constexpr uint32_t kZPlane = BH * 32;       // 32-bit words of one z buffer (16 KB)
constexpr uint32_t kCw = BT * BH;           // floats of one cosine-factor buffer (16 KB)
constexpr int kDW = 8, kZW = 8, kEpiW = 8;  // warps per role
constexpr int kMmaWarp = kDW + kZW;         // 16
constexpr int kThr = 32 * (kDW + kZW + 1 + kEpiW);  // 800
constexpr uint32_t kColWlo = 64, kColDw = 128, kColDg = 256;

enum : int { kTop = 1, kBottom = 2 };

struct Bwd16Args {
  const float* X;       // dA_l [n][128]; TOP: a_l
  const float* Aprev;   // a_{l-1} [n][128]
  const float* W;       // W_l [128][128] row-major
  const float* wL;      // TOP: head weights [128]
  const float* gpx;     // TOP: g s per masked pixel [n]
  const float2* coords; // BOTTOM
  const float* W0;      // BOTTOM: layer 0 [128][2], b0 [128]
  const float* b0;
  const unsigned* mx_in;  // bits of max|g s| (TOP) or max|dA_l|
  unsigned* mx_out;       // bits of max|dA_{l-1}| (atomicMax; not BOTTOM)
  float w0;
  int n;
  float* Y;         // dA_{l-1} [n][128] (not BOTTOM)
  float* part_w;    // [grid][128 * 128 + 128]
  float* part_top;  // TOP: [grid][129]
  float* part_0;    // BOTTOM: [grid][3 * 128]
};

struct Bwd16Bars {
  uint64_t xfull[NX], xfree[NX];  // raw dA_l slot landed / read (dA producers)
  uint64_t rfull[NR], rfree[NR];  // raw a_{l-1} slot landed / read (z producers)
  uint64_t cready[NC], cfree[NC]; // cosine factors written (z producers) / read (epilogue)
  uint64_t zready[NZ], zfree[NZ]; // z planes written / weight-gradient MMAs done with them
  uint64_t gready[ND], pfree[ND]; // dA planes written / data-gradient MMAs done with them
  uint64_t dfull[2], dfree[2];    // D_g[b] ready (commit) / drained (epilogue)
  uint64_t acc;                   // D_w final (commit)
  uint32_t tslot;
  unsigned wmax, lmax;            // prologue: bits of max|W_l|, max|w_L|
};

__device__ __forceinline__ void sincos_w(float a, float w0, float* s, float* c) {
  __sincosf(sine_reduce(w0 * a), s, c);
}

__device__ __forceinline__ uint32_t saddr16(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// MN-major SWIZZLE_128B descriptor of a dA plane as the weight gradient's A
// (M = feature: 64 per 128-B row, the second 64 one chunk = 4 KB on (LBO);
// K = pixel rows in 8-row atoms 1 KB apart (SBO)); scripts/probes/f16_mn_probe.cu
__device__ __forceinline__ uint64_t mn_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(4096 >> 4) << 16;  // LBO: next 64 features
  d |= static_cast<uint64_t>(1024 >> 4) << 32;  // SBO: next 8 pixel rows
  d |= static_cast<uint64_t>(1) << 46;          // version
  d |= static_cast<uint64_t>(2) << 61;          // SWIZZLE_128B
  return d;
}

// 2^(14 - e) for max|x| < 2^e (max = 0: 1): scaled magnitudes stay below 2^14
__device__ __forceinline__ float pow2_scale(float mx) {
  if (!(mx > 0.f)) return 1.f;
  int e;
  frexpf(mx, &e);  // mx = f 2^e, f in [0.5, 1)
  return ldexpf(1.f, 14 - e);
}

// g s per masked pixel (nfield.hpp:194-197) and the bits of its max |.|
__global__ void gather_g16_kernel(const double* __restrict__ gv, const float* __restrict__ gmask,
                                  const int* __restrict__ idx, int n, float scale,
                                  float* __restrict__ out, unsigned* __restrict__ mx) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  float gg = 0.f;
  if (m < n) {
    if (gv) gg += static_cast<float>(gv[idx[m]]);
    if (gmask) gg += gmask[m];
    gg *= scale;
    out[m] = gg;
  }
  // one atomic per block (a same-address atomic per warp serialises)
  __shared__ unsigned wm[8];
  const unsigned b = __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(gg)));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned c = __reduce_max_sync(0xffffffffu, threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0u);
    if (threadIdx.x == 0 && c) atomicMax(mx, c);
  }
}

// 32-bit word offset of the fp16 pair (row, kk..kk+1), kk even in [0, 64), in a
// SW128 K-major plane of 128-B rows (16-B granule kk/8 XOR row % 8)
__device__ __forceinline__ uint32_t sw128h(int row, int kk) {
  return static_cast<uint32_t>(row * 32 + ((((kk >> 3) ^ (row & 7))) << 2) + ((kk & 7) >> 1));
}

template <int MODE>
__global__ void __launch_bounds__(kThr, 1) tc_bwd16_kernel(Bwd16Args a) {
  constexpr bool TOP = (MODE & kTop) != 0, BOTTOM = (MODE & kBottom) != 0;
  extern __shared__ unsigned char smem_dyn[];
  uint32_t* pda = tc::smem_align1024<uint32_t>(smem_dyn);  // [ND][hi c0 | hi c1 | lo c0 | lo c1][32][32]
  uint32_t* pz = pda + ND * kPlane;                          // [NZ][128 rows][hi 16 | lo 16 words]
  float* xr = reinterpret_cast<float*>(pz + NZ * kZPlane);   // [NX][BT][BH]
  float* raw = xr + NX * kRaw;                               // [NR][BT][BH]
  float* pc = raw + NR * kRaw;   // [NC][2 h][BH k][16 t] w0 cos(w0 a_{l-1}) (16-B chunks swizzled)
  float* red = pc + NC * kCw;    // [8][BH] bias, [8][BH] head, [8] gb, pad; then [3][BH] fp64
  float* wst = reinterpret_cast<float*>(pda);  // prologue: W staged [BH][BH + 1] over planes + xr
  __shared__ Bwd16Bars sb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tc::tmem_alloc<512>(&sb.tslot);
  if (tid == 0) {
    for (int i = 0; i < NX; ++i) {
      tc::mbar_init(&sb.xfull[i], 1);
      tc::mbar_init(&sb.xfree[i], 32 * kDW);
    }
    for (int i = 0; i < NR; ++i) {
      tc::mbar_init(&sb.rfull[i], 1);
      tc::mbar_init(&sb.rfree[i], 32 * kZW);
    }
    for (int i = 0; i < NC; ++i) {
      tc::mbar_init(&sb.cready[i], 32 * kZW);
      tc::mbar_init(&sb.cfree[i], 32 * kEpiW);
    }
    for (int i = 0; i < NZ; ++i) {
      tc::mbar_init(&sb.zready[i], 32 * kZW);
      tc::mbar_init(&sb.zfree[i], 1);
    }
    for (int i = 0; i < ND; ++i) {
      tc::mbar_init(&sb.gready[i], 32 * kDW);
      tc::mbar_init(&sb.pfree[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sb.dfull[i], 1);
      tc::mbar_init(&sb.dfree[i], 32 * kEpiW);
    }
    tc::mbar_init(&sb.acc, 1);
    sb.wmax = 0u;
    sb.lmax = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int n = a.n;
  const int n_tiles = (n + BT - 1) / BT;
  const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto tile_m0 = [&](int i) { return (blockIdx.x + i * gridDim.x) * BT; };
  auto load_raw = [&](int i) {
    const int m0 = tile_m0(i);
    const uint32_t bytes = static_cast<uint32_t>(min(BT, n - m0)) * BH * 4;
    uint64_t* bar = &sb.rfull[i % NR];
    tc::mbar_expect_tx(bar, bytes);
    tc::bulk_load(raw + (i % NR) * kRaw, a.Aprev + static_cast<size_t>(m0) * BH, bytes, bar);
  };
  auto load_x = [&](int i) {
    const int m0 = tile_m0(i);
    const uint32_t bytes = static_cast<uint32_t>(min(BT, n - m0)) * BH * 4;
    uint64_t* bar = &sb.xfull[i % NX];
    tc::mbar_expect_tx(bar, bytes);
    tc::bulk_load(xr + (i % NX) * kRaw, a.X + static_cast<size_t>(m0) * BH, bytes, bar);
  };
  __syncthreads();  // barrier init and the max slots
  if (tid == 0 && !BOTTOM)
    for (int i = 0; i < NR && i < my_tiles; ++i) load_raw(i);
  // W_l -> smem [j][k] (row j padded), with max|W_l| (and TOP: max|w_L|)
  {
    float m = 0.f;
    for (int e = tid; e < BH * BH / 4; e += kThr) {
      const float4 w4 = reinterpret_cast<const float4*>(a.W)[e];
      float* d = wst + (e / (BH / 4)) * (BH + 1) + (e % (BH / 4)) * 4;
      d[0] = w4.x;
      d[1] = w4.y;
      d[2] = w4.z;
      d[3] = w4.w;
      m = fmaxf(m, fmaxf(fmaxf(fabsf(w4.x), fabsf(w4.y)), fmaxf(fabsf(w4.z), fabsf(w4.w))));
    }
    const unsigned b = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
    if (lane == 0) atomicMax(&sb.wmax, b);
    if (TOP && tid < BH) {
      const unsigned bl = __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(a.wL[tid])));
      if (lane == 0) atomicMax(&sb.lmax, bl);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const float sw = pow2_scale(__uint_as_float(sb.wmax));
  const float w0 = a.w0;
  const float mx_in = __uint_as_float(*a.mx_in);
  const float sd = pow2_scale(TOP ? mx_in * w0 * __uint_as_float(sb.lmax) : mx_in);
  const uint32_t t0 = sb.tslot;
  // W^T hi / lo -> TMEM: warp = (lane quarter q = warp % 4, j quarter), row k,
  // two output features per column
  if (warp < 16) {
    const int row = 32 * (warp & 3) + lane;
    const uint32_t lb = t0 + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
    const int jq = warp >> 2;  // features [32 jq, 32 jq + 32) -> columns [16 jq, 16 jq + 16)
    uint32_t hi[16], lo[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int j = 32 * jq + 2 * c;
      tc::split_f16x2(sw * wst[j * (BH + 1) + row], sw * wst[(j + 1) * (BH + 1) + row], hi[c], lo[c]);
    }
    tc::tmem_st16u_nowait(lb + 16 * jq, hi);
    tc::tmem_st16u_nowait(lb + kColWlo + 16 * jq, lo);
    tc::tmem_wait_st();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0)
    for (int i = 0; i < NX && i < my_tiles; ++i) load_x(i);

  if (warp < kDW) {
    // ---- dA producers: thread = (pixel, 8 features): features [4 fg, 4 fg + 4)
    // and [64 + 4 fg, 64 + 4 fg + 4) of pixels pr and pr + 16 of the tile ----
    const int fg = lane & 15, pr = 2 * warp + (lane >> 4);
    float wl[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) wl[e] = TOP ? a.wL[(e >> 2) * 64 + 4 * fg + (e & 3)] : 0.f;
    float bacc[8], hacc[8], gbacc = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) bacc[e] = hacc[e] = 0.f;
    auto load_g = [&](int i, int p) {
      const int m = tile_m0(i) + p;
      return m < n ? a.gpx[m] : 0.f;
    };
    float gn0 = 0.f, gn1 = 0.f;
    if (TOP && my_tiles > 0) {
      gn0 = load_g(0, pr);
      gn1 = load_g(0, pr + 16);
    }
    for (int i = 0; i < my_tiles; ++i) {
      const int xs = i % NX, bx = i % ND;
      const int rows = min(BT, n - tile_m0(i));
      const float gg[2] = {gn0, gn1};
      if (TOP && i + 1 < my_tiles) {
        gn0 = load_g(i + 1, pr);
        gn1 = load_g(i + 1, pr + 16);
      }
      tc::mbar_wait(&sb.xfull[xs], (i / NX) & 1);
      BTRACE(tid == 0, 1, i);
      float v[2][8];
#pragma unroll
      for (int ps = 0; ps < 2; ++ps) {
        const float* xt = xr + xs * kRaw + (pr + 16 * ps) * BH + 4 * fg;
        const float4 x0 = *reinterpret_cast<const float4*>(xt);
        const float4 x1 = *reinterpret_cast<const float4*>(xt + 64);
        v[ps][0] = x0.x; v[ps][1] = x0.y; v[ps][2] = x0.z; v[ps][3] = x0.w;
        v[ps][4] = x1.x; v[ps][5] = x1.y; v[ps][6] = x1.z; v[ps][7] = x1.w;
      }
      tc::mbar_arrive(&sb.xfree[xs]);
      BTRACE(tid == 0, 12, i);
      if (tid == 0 && i + NX < my_tiles) {
        tc::mbar_wait(&sb.xfree[xs], (i / NX) & 1);
        // the slot's generic reads (every producer) before the async-proxy
        // refill: without this fence the copy can land under late reads
        tc::fence_proxy_async();
        load_x(i + NX);
      }
      uint32_t hw[2][4], lw[2][4];
#pragma unroll
      for (int ps = 0; ps < 2; ++ps) {
        // rows past n: the slot holds stale rows -> 0 (and g = 0 there), so
        // everything below is computed unconditionally (a condition on the
        // result would become one branch per value)
        const bool valid = pr + 16 * ps < rows;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float d = valid ? v[ps][e] : 0.f;
          if (TOP) {
            // output layer (nfield.hpp:194-205)
            float sx, cx;
            sincos_w(d, w0, &sx, &cx);
            d = gg[ps] * w0 * wl[e] * cx;
            hacc[e] = fmaf(gg[ps], sx, hacc[e]);
          }
          bacc[e] += d;
          v[ps][e] = d * sd;
        }
        if (TOP && fg == 0) gbacc += gg[ps];
#pragma unroll
        for (int u = 0; u < 4; ++u) tc::split_f16x2(v[ps][2 * u], v[ps][2 * u + 1], hw[ps][u], lw[ps][u]);
      }
      BTRACE(tid == 0, 14, i);
      if (i >= ND) tc::mbar_wait(&sb.pfree[bx], ((i - ND) / ND) & 1);
      BTRACE(tid == 0, 13, i);
      // row p, chunk c: the two words of pairs (4 fg, 4 fg + 2) (one 8-B store)
      uint32_t* ph = pda + bx * kPlane;
      uint32_t* pl = ph + 2 * BT * 32;
#pragma unroll
      for (int ps = 0; ps < 2; ++ps) {
        const uint32_t o = sw128h(pr + 16 * ps, 4 * fg);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          *reinterpret_cast<uint2*>(ph + c * (BT * 32) + o) = make_uint2(hw[ps][2 * c], hw[ps][2 * c + 1]);
          *reinterpret_cast<uint2*>(pl + c * (BT * 32) + o) = make_uint2(lw[ps][2 * c], lw[ps][2 * c + 1]);
        }
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&sb.gready[bx]);
      BTRACE(tid == 0, 2, i);
    }
    // per-feature sums: lanes fg and fg + 16, then the 8 warps in a fixed order
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      bacc[e] += __shfl_xor_sync(0xffffffffu, bacc[e], 16);
      if (TOP) hacc[e] += __shfl_xor_sync(0xffffffffu, hacc[e], 16);
    }
    if (TOP) gbacc += __shfl_xor_sync(0xffffffffu, gbacc, 16);
    if (lane < 16) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int f = (e >> 2) * 64 + 4 * fg + (e & 3);
        red[warp * BH + f] = bacc[e];
        if (TOP) red[8 * BH + warp * BH + f] = hacc[e];
      }
      if (TOP && lane == 0) red[16 * BH + warp] = gbacc;
    }
    tc::named_sync(1, 32 * kDW);
    if (tid < BH) {
      float sb_ = 0.f, sh = 0.f;
#pragma unroll
      for (int w = 0; w < kDW; ++w) {
        sb_ += red[w * BH + tid];
        if (TOP) sh += red[8 * BH + w * BH + tid];
      }
      a.part_w[static_cast<size_t>(blockIdx.x) * (BH * BH + BH) + BH * BH + tid] = sb_;
      if (TOP) {
        float* pt = a.part_top + static_cast<size_t>(blockIdx.x) * (BH + 1);
        pt[tid] = sh;
        if (tid == 0) {
          float g = 0.f;
          for (int w = 0; w < kDW; ++w) g += red[16 * BH + w];
          pt[BH] = g;
        }
      }
    }
  } else if (warp < kDW + kZW) {
    // ---- z producers: thread = feature k, pixels [16 h, 16 h + 16) ----
    const int q = warp & 3, h = (warp - kDW) >> 2, k = 32 * q + lane, pb = HP * h;
    float w0x = 0.f, w0y = 0.f, b0k = 0.f;
    float2 cnext = make_float2(0.f, 0.f);
    auto load_c = [&](int i) { return a.coords[min(tile_m0(i) + pb + (lane & (HP - 1)), n - 1)]; };
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
      float z[HP], cw[HP];
#pragma unroll
      for (int t = 0; t < HP; ++t) {
        const float av = BOTTOM ? fmaf(w0y, __shfl_sync(0xffffffffu, cc.y, t),
                                       fmaf(w0x, __shfl_sync(0xffffffffu, cc.x, t), b0k))
                                : ar[t * BH];
        // z = sin(w0 a) for the weight gradient and the epilogue's factor
        // w0 cos(w0 a) from one argument reduction; computed for every row,
        // then selected (a conditional evaluation becomes a branch per pixel)
        float sz, cz;
        __sincosf(sine_reduce(w0 * av), &sz, &cz);
        z[t] = pb + t < rows ? sz : 0.f;
        cw[t] = w0 * cz;
      }
      if (!BOTTOM) {
        tc::mbar_arrive(&sb.rfree[r]);
        if (tid == 32 * kDW && i + NR < my_tiles) {  // the raw loader
          tc::mbar_wait(&sb.rfree[r], (i / NR) & 1);
          tc::fence_proxy_async();  // generic reads of the slot before the refill
          load_raw(i + NR);
        }
      }
      uint32_t hw[HP / 2], lw[HP / 2];
#pragma unroll
      for (int u = 0; u < HP / 2; ++u) tc::split_f16x2(z[2 * u], z[2 * u + 1], hw[u], lw[u]);
      if (i >= NZ) tc::mbar_wait(&sb.zfree[bz], ((i - NZ) / NZ) & 1);
      BTRACE(warp == kDW && lane == 0, 6, i);
      // row k: hi granules 2h, 2h + 1, lo granules 4 + 2h, 5 + 2h (XOR k % 8)
      uint32_t* zr = pz + bz * kZPlane + k * 32;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        *reinterpret_cast<uint4*>(zr + (((2 * h + g) ^ (k & 7)) << 2)) =
            make_uint4(hw[4 * g], hw[4 * g + 1], hw[4 * g + 2], hw[4 * g + 3]);
        *reinterpret_cast<uint4*>(zr + (((4 + 2 * h + g) ^ (k & 7)) << 2)) =
            make_uint4(lw[4 * g], lw[4 * g + 1], lw[4 * g + 2], lw[4 * g + 3]);
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&sb.zready[bz]);
      BTRACE(warp == kDW && lane == 0, 7, i);
      // cosine factors -> buffer i % NC, row (h, k) of 16 floats, 16-B chunk c
      // at c ^ (k / 2 % 4): 8 consecutive lanes cover all banks
      const int cs = i % NC;
      if (i >= NC) tc::mbar_wait(&sb.cfree[cs], ((i - NC) / NC) & 1);
      float* cr = pc + cs * kCw + (h * BH + k) * 16;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<float4*>(cr + ((c ^ ((k >> 1) & 3)) << 2)) =
            make_float4(cw[4 * c], cw[4 * c + 1], cw[4 * c + 2], cw[4 * c + 3]);
      tc::mbar_arrive(&sb.cready[cs]);
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issue, in tile order: wgrad(i) then dgrad(i) ----
    constexpr uint32_t idesc_w = tc::idesc_f16(BH, BH) | (1u << 15);  // A MN-major
    constexpr uint32_t idesc_g = tc::idesc_f16(BH, BT);
    for (int i = 0; i < my_tiles; ++i) {
      const int bz = i % NZ, bx = i % ND, b = i & 1;
      tc::mbar_wait(&sb.zready[bz], (i / NZ) & 1);
      tc::mbar_wait(&sb.gready[bx], (i / ND) & 1);
      BTRACE(lane == 0, 8, i);
      tc::fence_after_sync();
      const uint32_t zrow = saddr16(pz + bz * kZPlane);
      const uint32_t dah = saddr16(pda + bx * kPlane), dal = dah + 2 * BT * 128;
      if (tc::elect_one()) {
#pragma unroll
        for (int s = 0; s < BT / 16; ++s) {
          // A = dA^T straight from the planes, MN-major (M = j: 64 per 128-B
          // row, chunk stride LBO = 4 KB; K = pixel: 8-row groups SBO = 1 KB)
          const uint64_t ah = mn_desc(dah + 2048 * s), al = mn_desc(dal + 2048 * s);
          const uint64_t bh = tc::smem_desc_sw128(zrow + 32 * s);
          const uint64_t bl = tc::smem_desc_sw128(zrow + 64 + 32 * s);
          tc::mma_f16(t0 + kColDw, al, bh, idesc_w, (i | s) != 0);
          tc::mma_f16(t0 + kColDw, ah, bl, idesc_w, 1u);
          tc::mma_f16(t0 + kColDw, ah, bh, idesc_w, 1u);
        }
        tc::mma_commit(&sb.zfree[bz]);
      }
      __syncwarp();
#if BWD16_SERIAL
      tc::mbar_wait(&sb.zfree[bz], (i / NZ) & 1);
#endif
      if (i >= 2) tc::mbar_wait(&sb.dfree[b], ((i - 2) >> 1) & 1);
      BTRACE(lane == 0, 9, i);
      tc::fence_after_sync();
      if (tc::elect_one()) {
        const uint32_t dcol = t0 + kColDg + BT * b;
#pragma unroll
        for (int s = 0; s < BH / 16; ++s) {
          const uint32_t off = (s >> 2) * (BT * 128) + 32 * (s & 3);
          const uint64_t bh = tc::smem_desc_sw128(dah + off);
          const uint64_t bl = tc::smem_desc_sw128(dal + off);
          tc::mma_f16_ts(dcol, t0 + kColWlo + 8 * s, bh, idesc_g, s != 0);
          tc::mma_f16_ts(dcol, t0 + 8 * s, bl, idesc_g, 1u);
          tc::mma_f16_ts(dcol, t0 + 8 * s, bh, idesc_g, 1u);
        }
        tc::mma_commit(&sb.dfull[b]);
        tc::mma_commit(&sb.pfree[bx]);
        if (i + 1 == my_tiles) tc::mma_commit(&sb.acc);
      }
      __syncwarp();
#if BWD16_SERIAL
      tc::mbar_wait(&sb.pfree[bx], (i / ND) & 1);
#endif
    }
  } else {
    // ---- epilogue: thread = input feature k, pixels [16 h, 16 h + 16) ----
    const int e = warp - kMmaWarp - 1;
    const int q = warp & 3, h = e >> 2, k = 32 * q + lane, pb = HP * h;
    const uint32_t lb = t0 + (static_cast<uint32_t>(32 * q) << 16);
    const float ds = 1.f / (sw * sd);                         // D_g scale (exact)
    double gx = 0.0, gy = 0.0, gb = 0.0;
    float ymax = 0.f;
    float2 cnext = make_float2(0.f, 0.f);  // BOTTOM: the pixel coordinates (layer-0 gradient)
    auto load_c = [&](int i) { return a.coords[min(tile_m0(i) + pb + (lane & (HP - 1)), n - 1)]; };
    if (BOTTOM && my_tiles > 0) cnext = load_c(0);
    for (int i = 0; i < my_tiles; ++i) {
      const int b = i & 1;
      const int m0 = tile_m0(i), rows = min(BT, n - m0);
      const float2 cme = cnext;
      if (BOTTOM && i + 1 < my_tiles) cnext = load_c(i + 1);
      // the cosine factors of this thread's (feature, pixels) from the z producers
      float cw[HP];
      const int cs = i % NC;
      tc::mbar_wait(&sb.cready[cs], (i / NC) & 1);
      const float* cr = pc + cs * kCw + (h * BH + k) * 16;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 f = *reinterpret_cast<const float4*>(cr + ((c ^ ((k >> 1) & 3)) << 2));
        cw[4 * c] = f.x;
        cw[4 * c + 1] = f.y;
        cw[4 * c + 2] = f.z;
        cw[4 * c + 3] = f.w;
      }
      tc::mbar_arrive(&sb.cfree[cs]);
      tc::mbar_wait(&sb.dfull[b], (i >> 1) & 1);
      BTRACE(warp == kMmaWarp + 1 && lane == 0, 10, i);
      tc::fence_after_sync();
      float v[HP];
      tc::tmem_ld16(lb + kColDg + BT * b + pb, v);
      tc::fence_before_sync();
      tc::mbar_arrive(&sb.dfree[b]);
      if (!BOTTOM) {
        float* y = a.Y + static_cast<size_t>(m0 + pb) * BH + k;
#pragma unroll
        for (int t = 0; t < HP; ++t)
          if (pb + t < rows) {
            const float o = v[t] * ds * cw[t];
            y[static_cast<size_t>(t) * BH] = o;
            ymax = fmaxf(ymax, fabsf(o));
          }
      } else {
        float sx = 0.f, sy = 0.f, s1 = 0.f;
#pragma unroll
        for (int t = 0; t < HP; ++t) {
          const float out = pb + t < rows ? v[t] * ds * cw[t] : 0.f;
          sx = fmaf(out, __shfl_sync(0xffffffffu, cme.x, t), sx);
          sy = fmaf(out, __shfl_sync(0xffffffffu, cme.y, t), sy);
          s1 += out;
        }
        gx += static_cast<double>(sx);
        gy += static_cast<double>(sy);
        gb += static_cast<double>(s1);
      }
    }
    if (!BOTTOM) {
      const unsigned bm = __reduce_max_sync(0xffffffffu, __float_as_uint(ymax));
      if (lane == 0 && bm) atomicMax(a.mx_out, bm);
    } else {
      double* rd = reinterpret_cast<double*>(red + 16 * BH + 16);  // [3][BH]
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
    // D_w (lane = j = k here, column = input feature) -> this CTA's partial
    const float dw = 1.f / sd;
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
          *reinterpret_cast<float4*>(out + c0 + jj) =
              make_float4(w[jj] * dw, w[jj + 1] * dw, w[jj + 2] * dw, w[jj + 3] * dw);
      }
    } else {
      for (int c = h * (BH / 2); c < (h + 1) * (BH / 2); ++c) out[c] = 0.f;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(t0);
}

constexpr size_t kBwd16Smem =
    1024 + sizeof(float) * (ND * kPlane + NZ * kZPlane + (NX + NR) * kRaw + NC * kCw + 22 * BH + 16);
static_assert(kBwd16Smem <= 227 * 1024, "tc_bwd16_kernel: shared memory budget");
// W is staged [BH][BH + 1] over the planes and the raw dA_l slots (filled after it)
static_assert(ND * kPlane + NZ * kZPlane + NX * kRaw >= BH * (BH + 1), "tc_bwd16_kernel: W staging");

template <int MODE>
Status launch_bwd16(pact_ctx* ctx, const Bwd16Args& a, int grid) {
  PACT_TRY_S(smem_optin(tc_bwd16_kernel<MODE>, kBwd16Smem));
  tc_bwd16_kernel<MODE><<<grid, kThr, kBwd16Smem, ctx->stream>>>(a);
  return after_launch(ctx, "tc_bwd16_kernel");
}

}  // namespace

// PACT_SIREN_BWD_F16=0 keeps the 3xTF32 backward (siren_bwd.cu); default split fp16.
bool tc_bwd_f16() {
  static const bool on = [] {
    const char* e = std::getenv("PACT_SIREN_BWD_F16");
    return !(e && e[0] == '0');
  }();
  return on;
}

Status tc_bwd16_layer(pact_ctx* ctx, bool top, bool bottom, const TcBwdLayer& L, unsigned* mx_in,
                      unsigned* mx_out) {
  Bwd16Args a{};
  a.X = L.X;
  a.Aprev = L.Aprev;
  a.W = L.W;
  a.wL = L.wL;
  a.gpx = L.gpx;
  if (top) {
    if (!L.gpx) return internal_error("tc_bwd16_layer: top layer needs the g scratch");
    gather_g16_kernel<<<div_up(L.n, 256), 256, 0, ctx->stream>>>(L.gv, L.gmask, L.idx, L.n,
                                                                  L.out_scale, L.gpx, mx_in);
    PACT_TRY_S(after_launch(ctx, "gather_g16_kernel"));
  }
  a.coords = L.coords;
  a.W0 = L.W0;
  a.b0 = L.b0;
  a.mx_in = mx_in;
  a.mx_out = mx_out;
  a.w0 = L.w0;
  a.n = L.n;
  a.Y = L.Y;
  a.part_w = L.part_w;
  a.part_top = L.part_top;
  a.part_0 = L.part_0;
  const int grid = tc_bwd_grid(ctx, L.n);
  if (top && bottom) return launch_bwd16<kTop | kBottom>(ctx, a, grid);
  if (top) return launch_bwd16<kTop>(ctx, a, grid);
  if (bottom) return launch_bwd16<kBottom>(ctx, a, grid);
  return launch_bwd16<0>(ctx, a, grid);
}

}  // namespace pactgpu

#if BWD16_TRACE
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
