// SIREN hidden layers of width 256 (cfg5, 2 -> 256 x 4 -> 1) on tcgen05,
// 3xTF32 (tc.cuh).  At this width a layer's hi/lo weight planes (512 KB) fit
// neither TMEM nor shared memory, so these are classic streamed GEMMs with
// both operands in shared memory (SS MMAs), one kernel per layer and mode:
//
//   forward  a_l[p][o]  = sum_k W_l[o][k] sin(w0 a_{l-1}[p][k]) + b_l[o]      (nfield.hpp:117-124)
//   dgrad    dA_{l-1}[p][k] = (sum_o dA_l[p][o] W_l[o][k]) w0 cos(w0 a_{l-1}[p][k])
//   wgrad    gW_l[o][k] += sum_p dA_l[p][o] sin(w0 a_{l-1}[p][k]),  gb_l[o] += sum_p dA_l[p][o]
//                                                                              (nfield.hpp:190-230)
//
// Forward / dgrad (tc_wide_layer_kernel, 2-CTA clusters: the pair streams
// the same weight chunks, each CTA loads one plane and multicasts it into
// both, halving the weight traffic from L2): 128-pixel tiles, N = 256 output
// features in one MMA, K streamed in 16 chunks of 16 through a 4-stage ring
// (SWIZZLE_64B: 64-B rows, so a stage is 48 KB and four fit; the weight
// chunks come from L2 for every tile, and a deep ring hides that latency).
// A stage holds the A chunk (rows = pixel, 16 K; its hi plane is the input
// tile itself, written by a TMA tensor load in the SW64 layout -- kind::tf32
// ignores the low 13 mantissa bits; producers add the lo plane, and for the
// forward first replace hi by sin(w0 a)) and the B chunk (precomputed hi/lo
// planes of W or W^T, 32 KB, one bulk copy).  Two 256-column TMEM
// accumulators alternate between tiles so the epilogue (bias or cosine,
// coalesced float4 row stores) of tile i overlaps the MMAs of tile i + 1.
//
// Weight gradient (tc_wide_wgrad_kernel): M = output feature (two blocks of
// 128), N = 256 input features, K = 32-pixel chunks; both operands are the
// transposes of the row-major activations, so producer threads that own a
// feature read its column from a raw bulk-copied chunk and write their row of
// the K-major planes.  D (2 x 256 columns) accumulates over the CTA's pixel
// range; per-CTA partials are reduced in fixed order in fp64 by the caller.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "siren.cuh"
#include "tc.cuh"

// WIDE_EXP (timing experiments only, wrong results): 1 = the layer
// epilogue neither loads a_{l-1} nor stores its output.
#ifndef WIDE_EXP
#define WIDE_EXP 0
#endif

namespace pactgpu {
namespace {

constexpr int WH = 256;               // hidden width
constexpr int WT = 128;               // pixels per tile (MMA M)
constexpr int WKC = 16;               // K per chunk (one 64-B SW64 row)
constexpr int WNK = WH / WKC;         // 16 K-chunks
constexpr int WNS = 4;                // ring stages
constexpr uint32_t kAPlane = WT * WKC;   // floats of one A plane (8 KB)
constexpr uint32_t kBPlane = WH * WKC;   // floats of one B plane (16 KB)
constexpr uint32_t kStage = 2 * kAPlane + 2 * kBPlane;  // 48 KB
constexpr int kWideThreads = 32 * 18;  // loader, MMA, 8 producer warps, 8 epilogue warps

enum : int { kWideFwd = 0, kWideDgrad = 1 };

__device__ __forceinline__ float red2pi_w(float x) { return sine_reduce(x); }

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- 2-CTA clusters: the two CTAs of a pair stream the same weight chunks,
// so each loads one of the chunk's two planes and multicasts it into both
// (half the L2 traffic for the weights) ----
constexpr int kPair = 2;
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t n_clusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// bulk copy global -> the same smem offset in every CTA of `mask`, completing
// on the mbarrier at the same offset in each
__device__ __forceinline__ void bulk_load_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
          sa(dst)),
      "l"(src), "r"(bytes), "r"(sa(bar)), "h"(mask)
      : "memory");
}
// all prior MMAs of this thread arrive on `bar` in every CTA of `mask`
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   sa(bar)),
               "h"(mask)
               : "memory");
}

// K-major SWIZZLE_64B: 8-row x 64-B atoms (16 fp32 of K per row), 16-B chunk
// index XOR (row / 2) % 4, atoms stacked at SBO = 512 B; K step s of 8
// advances the start address by 32 s bytes.
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;            // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(512 >> 4) << 32;     // SBO
  d |= static_cast<uint64_t>(1) << 46;            // version
  d |= static_cast<uint64_t>(4) << 61;            // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ int sw64(int row, int k) {
  return row * 16 + ((((k >> 2) ^ ((row >> 1) & 3))) << 2) + (k & 3);
}

// Weight planes [chunk c][hi | lo][row r][16] (SW64) of W (row r = output
// feature, K = input feature) or of W^T (row r = input feature, K = output).
__global__ void wide_planes_kernel(const float* __restrict__ W, int transposed, float* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= WH * WH) return;
  const int r = e / WH, k = e % WH;  // plane row, K index
  const int c = k / WKC, kk = k % WKC;
  const float v = transposed ? W[static_cast<size_t>(k) * WH + r] : W[static_cast<size_t>(r) * WH + k];
  float hi, lo;
  tc::split_tf32(v, hi, lo);
  float* pl = out + static_cast<size_t>(c) * 2 * kBPlane;
  const int o = sw64(r, kk);
  pl[o] = hi;
  pl[kBPlane + o] = lo;
}

struct WideBars {
  uint64_t full[WNS], ready[WNS], empty[WNS];
  uint64_t dfull[2], dfree[2];
  uint64_t abox[8];  // dgrad: a_{l-1} block landed in epilogue warp e's box
  uint32_t tslot;
};

template <int MODE>
__global__ void __launch_bounds__(kWideThreads, 1)
tc_wide_layer_kernel(const __grid_constant__ CUtensorMap tmap_in,
                     const __grid_constant__ CUtensorMap tmap_out,
                     const __grid_constant__ CUtensorMap tmap_prev, const float* __restrict__ planes,
                     const float* __restrict__ bias, const float* __restrict__ Aprev, int n, float w0,
                     float* __restrict__ Y) {
  extern __shared__ unsigned char smem_dyn[];
  float* st = tc::smem_align1024<float>(smem_dyn);  // [WNS][kStage]
  float* s_bias = st + WNS * kStage;                                    // [WH]
  float* s_box = s_bias + WH;  // [8 epilogue warps][32 x 32] SW128 output boxes (1024-aligned)
  __shared__ WideBars sb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tc::tmem_alloc<512>(&sb.tslot);
  if (tid == 0) {
    for (int i = 0; i < WNS; ++i) {
      tc::mbar_init(&sb.full[i], 1);
      tc::mbar_init(&sb.ready[i], 256);
      tc::mbar_init(&sb.empty[i], kPair);  // both CTAs' MMAs are done with the stage
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sb.dfull[i], 1);
      tc::mbar_init(&sb.dfree[i], 256);
    }
    for (int i = 0; i < 8; ++i) tc::mbar_init(&sb.abox[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (MODE == kWideFwd)
    for (int i = tid; i < WH; i += kWideThreads) s_bias[i] = bias[i];
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync_all();  // the peer's barriers exist before any multicast reaches them
  tc::fence_after_sync();
  const uint32_t t0 = sb.tslot;
  // tiles go to the pair together: pair step i covers tiles 2 (cid + i ncl) + rank
  // (a tile past the end loads zeros and stores nothing; both CTAs run the
  // same number of steps, as the shared weight chunks require)
  const uint32_t rank = cluster_rank(), cid = cluster_id_x(), ncl = n_clusters_x();
  const int n_tiles = (n + WT - 1) / WT, n_pairs = (n_tiles + 1) / 2;
  const int my_tiles = static_cast<int>(cid) < n_pairs ? (n_pairs - 1 - static_cast<int>(cid)) / static_cast<int>(ncl) + 1 : 0;
  const int n_g = my_tiles * WNK;  // (tile, K-chunk) steps
  auto tile_m0 = [&](int i) { return (2 * (static_cast<int>(cid) + i * static_cast<int>(ncl)) + static_cast<int>(rank)) * WT; };

  if (warp == 0) {
    // ---- loader: A chunk (TMA box 16 x 128, rows >= n zero) + B chunk ----
    if (lane == 0) {
      for (int g = 0; g < n_g; ++g) {
        const int s = g % WNS, i = g / WNK, c = g % WNK;
        if (g >= WNS) tc::mbar_wait_sleep(&sb.empty[s], ((g - WNS) / WNS) & 1);
        float* stg = st + s * kStage;
        tc::mbar_expect_tx(&sb.full[s], 4 * (kAPlane + 2 * kBPlane));
        tc::tma_load_2d(stg, &tmap_in, WKC * c, tile_m0(i), &sb.full[s]);
        // this CTA's plane of the weight chunk (rank 0: hi, rank 1: lo), into both
        bulk_load_mc(stg + 2 * kAPlane + rank * kBPlane,
                     planes + static_cast<size_t>(c) * 2 * kBPlane + rank * kBPlane, 4 * kBPlane,
                     &sb.full[s], 0x3);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issue: per chunk 2 K-steps x 3 products, M = 128, N = 256 ----
    constexpr uint32_t idesc = tc::idesc_tf32(WT, WH);
    for (int g = 0; g < n_g; ++g) {
      const int s = g % WNS, i = g / WNK, c = g % WNK;
      tc::mbar_wait(&sb.ready[s], (g / WNS) & 1);
      if (c == 0 && i >= 2) tc::mbar_wait(&sb.dfree[i & 1], ((i - 2) >> 1) & 1);
      tc::fence_after_sync();
      if (tc::elect_one()) {
        const uint32_t ah = sa(st + s * kStage), al = ah + 4 * kAPlane;
        const uint32_t bh = ah + 8 * kAPlane, bl = bh + 4 * kBPlane;
        const uint32_t d = t0 + WH * (i & 1);
#pragma unroll
        for (int k = 0; k < WKC / 8; ++k) {
          const uint64_t dah = desc_sw64(ah + 32 * k), dal = desc_sw64(al + 32 * k);
          const uint64_t dbh = desc_sw64(bh + 32 * k), dbl = desc_sw64(bl + 32 * k);
          tc::mma_tf32(d, dal, dbh, idesc, (c | k) != 0);
          tc::mma_tf32(d, dah, dbl, idesc, 1u);
          tc::mma_tf32(d, dah, dbh, idesc, 1u);
        }
        mma_commit_mc(&sb.empty[s], 0x3);  // frees the stage in both CTAs
        if (c == WNK - 1) tc::mma_commit(&sb.dfull[i & 1]);
      }
      __syncwarp();
    }
  } else if (warp < 10) {
    // ---- producers: row p = t / 2, granules 2 h, 2 h + 1 of the 64-B row ----
    const int t = tid - 64, p = t >> 1, h = t & 1;
    for (int g = 0; g < n_g; ++g) {
      const int s = g % WNS;
      tc::mbar_wait(&sb.full[s], (g / WNS) & 1);
      float* hi = st + s * kStage;
      float* lo = hi + kAPlane;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int o = p * WKC + (((2 * h + j) ^ ((p >> 1) & 3)) << 2);
        float4 x = *reinterpret_cast<const float4*>(hi + o);
        if (MODE == kWideFwd) {
          // sin(w0 a_{l-1}); rows past n arrive as zeros and stay zero
          x = make_float4(__sinf(red2pi_w(w0 * x.x)), __sinf(red2pi_w(w0 * x.y)),
                          __sinf(red2pi_w(w0 * x.z)), __sinf(red2pi_w(w0 * x.w)));
          *reinterpret_cast<float4*>(hi + o) = x;
        }
        float4 hv, lv;
        tc::split_tf32_trunc(x.x, hv.x, lv.x);
        tc::split_tf32_trunc(x.y, hv.y, lv.y);
        tc::split_tf32_trunc(x.z, hv.z, lv.z);
        tc::split_tf32_trunc(x.w, hv.w, lv.w);
        *reinterpret_cast<float4*>(lo + o) = lv;
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&sb.ready[s]);
    }
  } else {
    // ---- epilogue: lane = pixel (quarter warp % 4), half ch of the 256 columns;
    // each 32 x 32 output block goes through this warp's SW128 box and one
    // TMA tensor store (coalesced; rows >= n clipped by the tensor bounds).
    // The data gradient first TMA-loads the matching a_{l-1} block into the
    // box and overwrites it in place with the result ----
    const int e = warp - 10, q = warp & 3, ch = e >> 2;
    const uint32_t lb = t0 + (static_cast<uint32_t>(32 * q) << 16);
    float* box = s_box + e * 32 * 32;
    uint32_t nst = 0;
    for (int i = 0; i < my_tiles; ++i) {
      const int r0 = tile_m0(i) + 32 * q;  // this warp's 32 rows
      tc::mbar_wait(&sb.dfull[i & 1], (i >> 1) & 1);
      tc::fence_after_sync();
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        const int col = 128 * ch + 32 * cc;
        if (nst > 0) {  // the box's previous store has read it
          if (lane == 0) tc::bulk_wait_read<0>();
          __syncwarp();
        }
        if (MODE == kWideDgrad && lane == 0) {
          tc::mbar_expect_tx(&sb.abox[e], 32 * 32 * 4);
          tc::tma_load_2d(box, &tmap_prev, col, r0, &sb.abox[e]);
        }
        float v[32];
        tc::tmem_ld32(lb + WH * (i & 1) + col, v);
        if (MODE == kWideDgrad) tc::mbar_wait(&sb.abox[e], nst & 1);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float* bp = box + lane * 32 + ((j ^ (lane & 7)) << 2);
          float4 o;
          if (MODE == kWideFwd) {
            o = make_float4(v[4 * j] + s_bias[col + 4 * j], v[4 * j + 1] + s_bias[col + 4 * j + 1],
                            v[4 * j + 2] + s_bias[col + 4 * j + 2], v[4 * j + 3] + s_bias[col + 4 * j + 3]);
          } else {
            const float4 av = *reinterpret_cast<const float4*>(bp);
            o = make_float4(v[4 * j] * (w0 * __cosf(red2pi_w(w0 * av.x))),
                            v[4 * j + 1] * (w0 * __cosf(red2pi_w(w0 * av.y))),
                            v[4 * j + 2] * (w0 * __cosf(red2pi_w(w0 * av.z))),
                            v[4 * j + 3] * (w0 * __cosf(red2pi_w(w0 * av.w))));
          }
          *reinterpret_cast<float4*>(bp) = o;
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0 && WIDE_EXP != 1) {
          tc::tma_store_2d(&tmap_out, box, col, r0);
          tc::bulk_commit();
        }
        ++nst;
      }
      tc::fence_before_sync();
      tc::mbar_arrive(&sb.dfree[i & 1]);
    }
    if (lane == 0) tc::bulk_wait_all();  // the stores are complete before exit
  }
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync_all();  // no multicast copy or commit still targets this CTA
  if (warp == 0) tc::tmem_free<512>(t0);
}

// ---- weight gradient ---------------------------------------------------------
constexpr int WP = 32;                       // pixels per chunk (K)
constexpr uint32_t kRawW = WP * WH;          // floats of one raw chunk (32 KB)
constexpr uint32_t kTPlane = WH * WP;        // floats of one transposed plane (32 KB)
constexpr uint32_t kWSlot = 4 * kTPlane;     // dA^T hi, lo, z^T hi, lo (128 KB)

struct WgBars {
  uint64_t rfull, rfree;     // raw chunk landed / read (512 producers)
  uint64_t ready[1], empty[1];
  uint64_t acc;
  uint32_t tslot;
};

__global__ void __launch_bounds__(kWideThreads, 1)
tc_wide_wgrad_kernel(const float* __restrict__ dA, const float* __restrict__ Aprev, int n, int rows,
                     float w0, float* __restrict__ partial) {
  extern __shared__ unsigned char smem_dyn[];
  float* pl = tc::smem_align1024<float>(smem_dyn);  // [kWSlot]
  float* raw = pl + kWSlot;                                             // dA [WP][WH] | a [WP][WH]
  __shared__ WgBars sb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tc::tmem_alloc<512>(&sb.tslot);
  if (tid == 0) {
    tc::mbar_init(&sb.rfull, 1);
    tc::mbar_init(&sb.rfree, 512);
    tc::mbar_init(&sb.ready[0], 512);
    tc::mbar_init(&sb.empty[0], 1);
    tc::mbar_init(&sb.acc, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t t0 = sb.tslot;
  const int m_begin = blockIdx.x * rows, m_end = min(n, m_begin + rows);
  const int n_ch = m_end > m_begin ? (m_end - m_begin + WP - 1) / WP : 0;
  auto load = [&](int i) {
    const int p0 = m_begin + i * WP;
    const uint32_t bytes = static_cast<uint32_t>(min(WP, m_end - p0)) * WH * 4;
    tc::fence_proxy_async();  // the producers' generic reads before the async refill
    tc::mbar_expect_tx(&sb.rfull, 2 * bytes);
    tc::bulk_load(raw, dA + static_cast<size_t>(p0) * WH, bytes, &sb.rfull);
    tc::bulk_load(raw + kRawW, Aprev + static_cast<size_t>(p0) * WH, bytes, &sb.rfull);
  };
  if (warp == 0) {
    // ---- loader: the next chunk as soon as the producers have read this one ----
    if (lane == 0) {
      for (int i = 0; i < n_ch; ++i) {
        if (i >= 1) tc::mbar_wait_sleep(&sb.rfree, (i - 1) & 1);
        load(i);
      }
    }
  } else if (warp == 1) {
    // ---- MMA: two 128-row blocks of D_w, K = 32 pixels ----
    constexpr uint32_t idesc = tc::idesc_tf32(128, WH);
    for (int i = 0; i < n_ch; ++i) {
      tc::mbar_wait(&sb.ready[0], i & 1);
      tc::fence_after_sync();
      if (tc::elect_one()) {
        const uint32_t ah = sa(pl), al = ah + 4 * kTPlane, bh = ah + 8 * kTPlane, bl = bh + 4 * kTPlane;
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {
          const uint32_t d = t0 + WH * mb, ro = mb * 128 * 128;  // rows 128 mb.. of the A planes
#pragma unroll
          for (int k = 0; k < WP / 8; ++k) {
            const uint64_t dah = tc::smem_desc_sw128(ah + ro + 32 * k), dal = tc::smem_desc_sw128(al + ro + 32 * k);
            const uint64_t dbh = tc::smem_desc_sw128(bh + 32 * k), dbl = tc::smem_desc_sw128(bl + 32 * k);
            tc::mma_tf32(d, dal, dbh, idesc, (i | k) != 0);
            tc::mma_tf32(d, dah, dbl, idesc, 1u);
            tc::mma_tf32(d, dah, dbh, idesc, 1u);
          }
        }
        tc::mma_commit(&sb.empty[0]);
        if (i + 1 == n_ch) tc::mma_commit(&sb.acc);
      }
      __syncwarp();
    }
  } else if (warp < 18) {
    // ---- producers: warps 2-9 own dA (thread = output feature o), 10-17 own
    // a_{l-1} (thread = input feature k); each writes its row of the
    // transposed K-major planes (row = feature, K = the chunk's 32 pixels) ----
    const bool is_z = warp >= 10;
    const int f = tid - (is_z ? 320 : 64);  // feature 0..255
    const float* src = raw + (is_z ? kRawW : 0) + f;
    float* ph = pl + (is_z ? 2 * kTPlane : 0);
    float* plo = ph + kTPlane;
    float bacc = 0.f;
    for (int i = 0; i < n_ch; ++i) {
      const int valid = min(WP, m_end - (m_begin + i * WP));
      tc::mbar_wait(&sb.rfull, i & 1);
      float v[WP];
#pragma unroll
      for (int p = 0; p < WP; ++p) v[p] = src[p * WH];
      tc::mbar_arrive(&sb.rfree);
#pragma unroll
      for (int p = 0; p < WP; ++p) {
        float x = v[p];
        if (is_z) x = __sinf(red2pi_w(w0 * x));
        x = p < valid ? x : 0.f;  // stale rows of a partial chunk
        if (!is_z) bacc += x;
        v[p] = x;
      }
      if (i >= 1) tc::mbar_wait(&sb.empty[0], (i - 1) & 1);
#pragma unroll
      for (int gq = 0; gq < WP / 4; ++gq) {
        float4 hv, lv;
        tc::split_tf32_trunc(v[4 * gq], hv.x, lv.x);
        tc::split_tf32_trunc(v[4 * gq + 1], hv.y, lv.y);
        tc::split_tf32_trunc(v[4 * gq + 2], hv.z, lv.z);
        tc::split_tf32_trunc(v[4 * gq + 3], hv.w, lv.w);
        const int o = f * WP + ((gq ^ (f & 7)) << 2);
        *reinterpret_cast<float4*>(ph + o) = hv;
        *reinterpret_cast<float4*>(plo + o) = lv;
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&sb.ready[0]);
    }
    float* out = partial + static_cast<size_t>(blockIdx.x) * (WH * WH + WH);
    if (!is_z) {
      out[WH * WH + f] = bacc;
      // D_w rows: warp w reads TMEM lane quarter w % 4 of block (w - 2) / 4
      const int mb = (warp - 2) >> 2, q = warp & 3, r = 128 * mb + 32 * q + lane;
      float* orow = out + static_cast<size_t>(r) * WH;
      if (n_ch > 0) {
        tc::mbar_wait(&sb.acc, 0);
        tc::fence_after_sync();
        const uint32_t lb = t0 + (static_cast<uint32_t>(32 * q) << 16) + WH * mb;
#pragma unroll 1
        for (int c0 = 0; c0 < WH; c0 += 32) {
          float w[32];
          tc::tmem_ld32(lb + c0, w);
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(orow + c0 + j) = make_float4(w[j], w[j + 1], w[j + 2], w[j + 3]);
        }
      } else {
        for (int c = 0; c < WH; ++c) orow[c] = 0.f;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(t0);
}

constexpr size_t kWideSmem = 1024 + sizeof(float) * (WNS * kStage + WH + 8 * 32 * 32);
constexpr size_t kWgradSmemW = 1024 + sizeof(float) * (kWSlot + 2 * kRawW);

PFN_cuTensorMapEncodeTiled tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }();
  return encode;
}

template <int MODE>
Status launch_wide(pact_ctx* ctx, const float* in, const float* planes, const float* bias,
                   const float* Aprev, int n, float w0, float* Y) {
  PACT_TRY_S(smem_optin(tc_wide_layer_kernel<MODE>, kWideSmem));
  auto encode = tensor_map_encoder();
  if (!encode) return internal_error("tc_wide_layer: cuTensorMapEncodeTiled unavailable");
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(WH), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[1] = {sizeof(float) * WH};
  const cuuint32_t box[2] = {WKC, WT}, estr[2] = {1, 1};
  if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(in), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return internal_error("tc_wide_layer: tensor map encoding failed");
  CUtensorMap tmap_out, tmap_prev;
  const cuuint32_t obox[2] = {32, 32};
  if (encode(&tmap_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, dims, strides, obox, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return internal_error("tc_wide_layer: output tensor map encoding failed");
  tmap_prev = tmap_out;  // forward: unused
  if (MODE == kWideDgrad &&
      encode(&tmap_prev, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(Aprev), dims, strides,
             obox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return internal_error("tc_wide_layer: a_{l-1} tensor map encoding failed");
  // 2-CTA clusters (the pair shares the weight chunks by multicast)
  const int pairs = std::max(1, std::min(ctx->num_sms / kPair, div_up(div_up(n, WT), kPair)));
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(kPair * pairs);
  lc.blockDim = dim3(kWideThreads);
  lc.dynamicSmemBytes = kWideSmem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  PACT_CUDA_S(cudaLaunchKernelEx(&lc, tc_wide_layer_kernel<MODE>, tmap, tmap_out, tmap_prev, planes, bias,
                                 Aprev, n, w0, Y));
  return after_launch(ctx, MODE == kWideFwd ? "tc_wide_layer_kernel<forward>"
                                            : "tc_wide_layer_kernel<dgrad>");
}

}  // namespace

bool siren_wide_supported(int hidden) { return hidden == WH; }

size_t tc_wide_plane_floats() { return static_cast<size_t>(WNK) * 2 * kBPlane; }

Status tc_wide_planes(pact_ctx* ctx, const float* W, bool transposed, float* planes) {
  wide_planes_kernel<<<div_up(WH * WH, 256), 256, 0, ctx->stream>>>(W, transposed ? 1 : 0, planes);
  return after_launch(ctx, "wide_planes_kernel");
}

Status tc_wide_forward_layer(pact_ctx* ctx, const float* Ain, const float* planes, const float* b,
                             int n, float w0, float* Aout) {
  if (n == 0) return {};
  return launch_wide<kWideFwd>(ctx, Ain, planes, b, nullptr, n, w0, Aout);
}

Status tc_wide_dgrad_layer(pact_ctx* ctx, const float* dAl, const float* planes_t,
                           const float* Aprev, int n, float w0, float* dAprev) {
  if (n == 0) return {};
  return launch_wide<kWideDgrad>(ctx, dAl, planes_t, nullptr, Aprev, n, w0, dAprev);
}

int tc_wide_wgrad_rows(pact_ctx* ctx, int n) {
  return std::max(WP, div_up(div_up(n, ctx->num_sms), WP) * WP);
}

Status tc_wide_wgrad_layer(pact_ctx* ctx, const float* dAl, const float* Aprev, int n, int rows,
                           float w0, float* partial, int n_chunks) {
  PACT_TRY_S(smem_optin(tc_wide_wgrad_kernel, kWgradSmemW));
  tc_wide_wgrad_kernel<<<n_chunks, kWideThreads, kWgradSmemW, ctx->stream>>>(dAl, Aprev, n, rows, w0,
                                                                              partial);
  return after_launch(ctx, "tc_wide_wgrad_kernel");
}

}  // namespace pactgpu
