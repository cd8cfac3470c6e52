// The SIREN forward as ONE kernel (hidden width 128): first layer, every
// tcgen05 hidden layer and the output head per 128-pixel tile, with the
// activations kept on chip between layers (nfield.hpp:110-162, render_sos).
//
//   a_0 = W_0 c + b_0                       (CUDA cores, per pixel)
//   a_l = W_l sin(w0 a_{l-1}) + b_l         (tcgen05 3xTF32, l = 1 .. L-1)
//   v   = v0 + s (w_L . sin(w0 a_{L-1}) + b_L)
//
// Layout (one CTA per SM, persistent over tiles):
//   TMEM  A_hi [0,128) A_lo [128,256): the MMA's A operand = sin(w0 a_{l-1})
//         of the tile (lane = pixel, column = feature), written by the
//         epilogue with tcgen05.st; D0 [256,384), D1 [384,512): accumulators
//         of alternate layers (lane = pixel, column = output feature).
//   smem  a 3-stage ring of weight K-chunks (B operand: W_l[n][32 j .. 32 j+31]
//         as SW128 K-major hi / lo planes, 32 KB per chunk, prepared once per
//         call by chain_wplanes_kernel and streamed from L2 by cp.async.bulk);
//         per-warp transpose tiles for coalesced activation stores.
// Roles: warp 0 streams weight chunks, warp 1 issues the MMAs (one elected
// lane), warps 2-9 are the epilogue (2 per TMEM lane quarter; pixel = lane,
// half h of the features = K-chunks 2h, 2h+1).  The epilogue of layer l
// writes layer l+1's A one 32-feature chunk at a time and signals it, so the
// tensor core starts layer l+1 while the rest of layer l drains.  The
// pre-activations a_1 .. a_{L-1} go to HBM (row-major [n][128], the
// backward's input; a_0 too unless the fused backward recomputes it from the
// coordinates); the per-layer re-read of the separate-kernel forward does not.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "siren.cuh"
#include "tc.cuh"

// CHAIN_EXP (timing experiments only, wrong results): 1 = weight chunks are
// loaded once per ring stage and then reused (no L2 weight stream)
#ifndef CHAIN_EXP
#define CHAIN_EXP 0
#endif
// CHAIN_EXP 3: no activation stores (timing only).
// CHAIN_EXP 2: store-only timeline of CTA 0 (roles: MMA warp, epilogue warps
// (q 0, chunk 0) and (q 0, chunk 3)) read by pact_debug_chain_trace.
#if CHAIN_EXP == 2
__device__ unsigned long long g_ctrace[3][1024][3];
#define CTRACE(role, tag, idx)                                                      \
  do {                                                                              \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) {                               \
      unsigned long long t_;                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
      const unsigned k_ = s_ct[role]++ & 1023;                                      \
      g_ctrace[role][k_][0] = (tag);                                                \
      g_ctrace[role][k_][1] = (idx);                                                \
      g_ctrace[role][k_][2] = t_;                                                   \
    }                                                                               \
  } while (0)
#else
#define CTRACE(role, tag, idx)
#endif

namespace pactgpu {
namespace {

constexpr int CH = 128;           // hidden width
constexpr int CT = 128;           // pixels per tile (MMA M)
constexpr int CKC = 32;           // features per K-chunk
constexpr int NCH = CH / CKC;     // K-chunks per layer
constexpr int WS = NCH;           // weight stages: one layer's 4 K-chunks (both N-halves read them)
constexpr uint32_t kPlaneFloats = CH * CKC;          // one of hi / lo
constexpr uint32_t kChunkBytes = 2 * kPlaneFloats * 4;  // 32 KB
constexpr int kMaxHidden = 8;
constexpr int kEpiWarps = 16, kEpi0 = 64, kThreads = kEpi0 + 32 * kEpiWarps;  // 576
constexpr uint32_t kColAlo = 128, kColD = 256;
constexpr uint32_t kBoxBytes = 32 * 128;  // TMA store box: 32 pixels x 32 features, SW128

struct ChainArgs {
  const float2* coords;
  const int* idx;
  int n;
  const float* W0;  // [128][2]
  const float* b0;  // [128]
  const float* bias[kMaxHidden];  // b_l, l = 1 .. nl
  const float* wplanes;           // [nl][NCH][hi, lo][128][32] SW128
  int nl;                         // hidden tcgen05 layers (L - 1)
  const float* wL;
  const float* bL;
  float scale, w0;
  float* acts;  // [L][n][128]
  float* dv;
  int store_a0;  // 0: a_0 is not written (the fused backward recomputes it)
};

__device__ __forceinline__ float red2pi_c(float x) { return sine_reduce(x); }
__device__ __forceinline__ float sinw(float a, float w0) { return __sinf(red2pi_c(w0 * a)); }

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct ChainBars {
  uint64_t wfull[WS], wempty[WS];  // weight stage j: K-chunk j of the current layer
  uint64_t ardy[NCH];              // A chunk j of the next layer written (128 threads)
  uint64_t dfull[2][2], dfree[2][2];  // [D buffer][N-half]: ready (MMA commit) / drained (256 threads)
  uint32_t tslot;
};

// Weight planes of every hidden layer: [l][j][hi | lo][n][kk] with the SW128
// swizzle of a 128-B K-major row (16-B granule kk/4 XOR n % 8).
struct LayerOffsets {
  long long off[kMaxHidden];  // theta offset of hidden tcgen05 layer l (network layer l + 1)
};

// F16: the planes hold fp16 hi / lo of W * 2^kF16Shift (|W| ~ 1e-2 for a
// SIREN: the scaled weights sit in fp16's normal range), 64 features per
// 128-B row: [l][j < 2][hi | lo][n][kk] with 16-B granule kk/8 XOR n % 8.
constexpr float kF16Scale = 256.f;

template <bool F16>
__global__ void chain_wplanes_kernel(const float* __restrict__ theta, LayerOffsets lo_, int nl,
                                     float* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nl * CH * CH) return;
  const int l = e / (CH * CH), r = (e / CH) % CH, k = e % CH;
  if (F16) {
    if (k & 1) return;  // one thread per feature pair
    const int j = k / 64, kk = k % 64;
    const float* w = theta + lo_.off[l] + static_cast<size_t>(r) * CH + k;
    uint32_t hi, lo;
    tc::split_f16x2(kF16Scale * w[0], kF16Scale * w[1], hi, lo);
    uint32_t* pl = reinterpret_cast<uint32_t*>(out + static_cast<size_t>(l * 2 + j) * 2 * kPlaneFloats);
    const int o = r * 32 + ((((kk >> 3) ^ (r & 7))) << 2) + ((kk & 7) >> 1);  // 32-bit words
    pl[o] = hi;
    pl[kPlaneFloats + o] = lo;
    return;
  }
  const int j = k / CKC, kk = k % CKC;
  float hi, lo;
  tc::split_tf32(theta[lo_.off[l] + static_cast<size_t>(r) * CH + k], hi, lo);
  float* pl = out + static_cast<size_t>(l * NCH + j) * 2 * kPlaneFloats;
  const int o = r * CKC + ((((kk >> 2) ^ (r & 7))) << 2) + (kk & 3);
  pl[o] = hi;
  pl[kPlaneFloats + o] = lo;
}

// F16: the MMAs run kind::f16 on split-fp16 operands (tc::split_f16x2): K-chunks
// of 64 features (two per layer), A packed two features per TMEM column (hi
// [0, 64), lo [64, 128)), weights scaled by kF16Scale (undone in the
// epilogue, an exact power of two).
template <bool F16>
__global__ void __launch_bounds__(kThreads, 1)
siren_chain_fwd_kernel(ChainArgs a, const __grid_constant__ CUtensorMap tmap_acts) {
  constexpr int KCH = F16 ? 2 : NCH;                 // K-chunks (weight stages) per layer
  constexpr uint32_t kAlo = F16 ? 64u : kColAlo;     // TMEM column of A lo
  constexpr float kDs = F16 ? 1.f / kF16Scale : 1.f;  // accumulator scale
  extern __shared__ unsigned char smem_dyn[];
  float* wring = tc::smem_align1024<float>(smem_dyn);  // [WS][2][128][32]
  float* s_tr = wring + WS * 2 * kPlaneFloats;  // [16 warps] SW128 store boxes (1024-aligned)
  float* s_w0 = s_tr + kEpiWarps * kBoxBytes / 4;                          // [128][2]
  float* s_b0 = s_w0 + 2 * CH;                                             // [128]
  float* s_wl = s_b0 + CH;                                                 // [128]
  float* s_bias = s_wl + CH;                                               // [nl][128]
  float* s_head = s_bias + kMaxHidden * CH;                                // [4][128]
  __shared__ ChainBars sb;
#if CHAIN_EXP == 2
  __shared__ unsigned s_ct[3];
  if (threadIdx.x < 3) s_ct[threadIdx.x] = 0;
#endif
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tc::tmem_alloc<512>(&sb.tslot);
  if (tid == 0) {
    for (int i = 0; i < KCH; ++i) {
      tc::mbar_init(&sb.wfull[i], 1);
      tc::mbar_init(&sb.wempty[i], 1);
    }
    for (int j = 0; j < KCH; ++j) tc::mbar_init(&sb.ardy[j], CT * (NCH / KCH));  // its epilogue warps
    for (int b = 0; b < 2; ++b)
      for (int nh = 0; nh < 2; ++nh) {
        tc::mbar_init(&sb.dfull[b][nh], 1);
        tc::mbar_init(&sb.dfree[b][nh], 32 * kEpiWarps / 2);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 2 * CH; i += kThreads) s_w0[i] = a.W0[i];
  for (int i = tid; i < CH; i += kThreads) {
    s_b0[i] = a.b0[i];
    s_wl[i] = a.wL[i];
  }
  for (int l = 0; l < a.nl; ++l)
    for (int i = tid; i < CH; i += kThreads) s_bias[l * CH + i] = a.bias[l][i];
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t t0 = sb.tslot;
  const int n_tiles = (a.n + CT - 1) / CT;
  const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int nl = a.nl;

  if (warp == 0) {
    // ---- weight chunks: K-chunk j of each (tile, layer) into stage j, once
    // both N-halves of the previous layer are done with it ----
    if (lane == 0) {
      uint32_t u = 0;  // layer uses
      for (int i = 0; i < my_tiles; ++i)
        for (int l = 0; l < nl; ++l, ++u)
          for (int j = 0; j < KCH; ++j) {
            if (u > 0) tc::mbar_wait_sleep(&sb.wempty[j], (u - 1) & 1);
            if (CHAIN_EXP == 1 && u > 0) {
              tc::mbar_arrive(&sb.wfull[j]);
              continue;
            }
            tc::mbar_expect_tx(&sb.wfull[j], kChunkBytes);
            tc::bulk_load(wring + j * 2 * kPlaneFloats,
                          a.wplanes + static_cast<size_t>(l * KCH + j) * 2 * kPlaneFloats,
                          kChunkBytes, &sb.wfull[j]);
          }
    }
  } else if (warp == 1) {
    // ---- MMA issue: layer l of tile i in two N-halves (64 output features
    // each), so the epilogue drains half 0 while the tensor core computes
    // half 1, and half 0 of the next layer starts on the first A chunks ----
    constexpr uint32_t idesc = F16 ? tc::idesc_f16(CT, CH / 2) : tc::idesc_tf32(CT, CH / 2);
    for (int i = 0; i < my_tiles; ++i)
      for (int l = 0; l < nl; ++l) {
        const uint32_t lc = static_cast<uint32_t>(i * nl + l), b = lc & 1;
        for (int nh = 0; nh < 2; ++nh) {
          const uint32_t dcol = t0 + kColD + b * CH + nh * (CH / 2);
          if (lc >= 2) tc::mbar_wait_sleep(&sb.dfree[b][nh], ((lc - 2) >> 1) & 1);
          CTRACE(0, 1, lc * 2 + nh);
          for (int j = 0; j < KCH; ++j) {
            if (nh == 0) {
              tc::mbar_wait_sleep(&sb.ardy[j], lc & 1);
              CTRACE(0, 2, lc * 4 + j);
              tc::mbar_wait_sleep(&sb.wfull[j], lc & 1);
              CTRACE(0, 3, lc * 4 + j);
            }
            tc::fence_after_sync();
            // rows [64 nh, 64 nh + 64) of the chunk's planes: 8 SW128 atoms in
            const uint32_t sh = saddr(wring + j * 2 * kPlaneFloats) + nh * (CH / 2) * 128,
                           sl = sh + kPlaneFloats * 4;
            if (tc::elect_one()) {
#pragma unroll
              // four K steps per 128-B row: 8 tf32 or 16 fp16 features, 8 TMEM
              // columns and 32 B of the row each
              for (int s = 0; s < 4; ++s) {
                const uint32_t ka = j * 32 + 8 * s;
                const uint64_t dh = tc::smem_desc_sw128(sh + 32 * s);
                const uint64_t dl = tc::smem_desc_sw128(sl + 32 * s);
                if (F16) {
                  tc::mma_f16_ts(dcol, t0 + kAlo + ka, dh, idesc, (j | s) != 0);
                  tc::mma_f16_ts(dcol, t0 + ka, dl, idesc, 1u);
                  tc::mma_f16_ts(dcol, t0 + ka, dh, idesc, 1u);
                } else {
                  tc::mma_tf32_ts(dcol, t0 + kAlo + ka, dh, idesc, (j | s) != 0);
                  tc::mma_tf32_ts(dcol, t0 + ka, dl, idesc, 1u);
                  tc::mma_tf32_ts(dcol, t0 + ka, dh, idesc, 1u);
                }
              }
              if (nh == 1) tc::mma_commit(&sb.wempty[j]);
              if (j == KCH - 1) tc::mma_commit(&sb.dfull[b][nh]);
            }
            __syncwarp();
          }
          CTRACE(0, 4, lc * 2 + nh);
        }
      }
  } else if (warp >= kEpi0 / 32) {
    // ---- epilogue: 16 warps, warp = (TMEM lane quarter q = warp % 4, K-chunk
    // j); pixel = lane, features [32 j, 32 j + 32) in two 16-column halves ----
    const int q = warp & 3, ew = warp - kEpi0 / 32, j = ew >> 2;
    const int p = 32 * q + lane, kb = CKC * j;
    const uint32_t lb = t0 + (static_cast<uint32_t>(32 * q) << 16);
    float* box0 = s_tr + ew * kBoxBytes / 4;  // this warp's store box
    const int hN = j >> 1;                    // the accumulator N-half holding its features
    const float w0 = a.w0;
    uint32_t nst = 0;  // store boxes issued by this warp
    float* box = box0;
    // the store box is free (its previous TMA store has read it)
    auto open_box = [&]() {
      if (nst >= 1) {
        if (lane == 0) tc::bulk_wait_read<0>();
        __syncwarp();
      }
    };
    // 16 features (half hf) of this pixel into the SW128 box row
    auto put_box = [&](const float (&v)[16], int hf) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int g = 4 * hf + c;
        *reinterpret_cast<float4*>(box + lane * 32 + ((g ^ (lane & 7)) << 2)) =
            make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
      }
    };
    // the box -> acts[l] rows [r0, r0 + 32) (rows >= n clipped by the tensor bounds)
    auto store_box = [&](int l, int r0) {
      if (CHAIN_EXP == 3) return;  // experiment: no activation stores
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tc::tma_store_3d(&tmap_acts, box, kb, r0, l);
        tc::bulk_commit();
      }
      ++nst;
    };
    // sin(w0 v) -> this chunk's A columns (hi, lo) of the next layer
    auto put_a = [&](const float (&v)[16], int hf, bool valid) {
      if (F16) {
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          tc::split_f16x2(valid ? sinw(v[2 * k], w0) : 0.f, valid ? sinw(v[2 * k + 1], w0) : 0.f, hi[k],
                          lo[k]);
        tc::tmem_st8u_nowait(lb + (kb + 16 * hf) / 2, hi);
        tc::tmem_st8u_nowait(lb + kAlo + (kb + 16 * hf) / 2, lo);
      } else {
        float hi[16], lo[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) tc::split_tf32_trunc(valid ? sinw(v[k], w0) : 0.f, hi[k], lo[k]);
        tc::tmem_st16_nowait(lb + kb + 16 * hf, hi);
        tc::tmem_st16_nowait(lb + kAlo + kb + 16 * hf, lo);
      }
    };
    const int jr = F16 ? j >> 1 : j;  // the K-chunk this warp's features belong to
    auto a_ready = [&]() {
      tc::tmem_wait_st();
      tc::fence_before_sync();
      tc::mbar_arrive(&sb.ardy[jr]);
    };
    auto tile_m0 = [&](int t) { return (blockIdx.x + t * gridDim.x) * CT; };
    // first layer of tile t (CUDA cores): a_0 = W_0 c + b_0 -> acts[0], A
    auto first_layer = [&](int t) {
      const int m0t = tile_m0(t);
      const bool vt = p < min(CT, a.n - m0t);
      const float2 c = vt ? a.coords[m0t + p] : make_float2(0.f, 0.f);
      if (a.store_a0) open_box();
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int f = kb + 16 * hf + k;
          v[k] = fmaf(s_w0[2 * f + 1], c.y, fmaf(s_w0[2 * f], c.x, s_b0[f]));
        }
        if (a.store_a0) put_box(v, hf);
        put_a(v, hf, vt);
      }
      if (a.store_a0) store_box(0, m0t + 32 * q);
      a_ready();
    };
    const int role = (q == 0 && (j == 0 || j == 3)) ? (j == 0 ? 1 : 2) : -1;
    if (my_tiles > 0) first_layer(0);
    for (int i = 0; i < my_tiles; ++i) {
      const int m0 = tile_m0(i);
      const int rows = min(CT, a.n - m0);
      const bool valid = p < rows;
      if (role > 0) CTRACE(role, 10, i);
      float hp = 0.f;  // head partial over this chunk's features
      for (int l = 0; l < nl; ++l) {
        const uint32_t lc = static_cast<uint32_t>(i * nl + l), b = lc & 1;
        const bool last = l == nl - 1;
        if (!last) {
          tc::mbar_wait(&sb.dfull[b][hN], (lc >> 1) & 1);
        } else if (i + 1 < my_tiles) {
          // the next tile's first layer, computed (and stored) while the
          // tensor core finishes this tile's last layer; its A columns go in
          // as soon as every MMA of that layer is done, so the tensor core
          // restarts while this tile's last layer and head drain
          const int m1 = tile_m0(i + 1);
          const bool v1 = p < min(CT, a.n - m1);
          const float2 c = v1 ? a.coords[m1 + p] : make_float2(0.f, 0.f);
          float ahi[32], alo[32];
          if (a.store_a0) open_box();
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            float v[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const int f = kb + 16 * hf + k;
              v[k] = fmaf(s_w0[2 * f + 1], c.y, fmaf(s_w0[2 * f], c.x, s_b0[f]));
            }
            if (a.store_a0) put_box(v, hf);
            if (F16) {
              uint32_t* h = reinterpret_cast<uint32_t*>(ahi) + 8 * hf;
              uint32_t* o = reinterpret_cast<uint32_t*>(alo) + 8 * hf;
#pragma unroll
              for (int k = 0; k < 8; ++k)
                tc::split_f16x2(v1 ? sinw(v[2 * k], w0) : 0.f, v1 ? sinw(v[2 * k + 1], w0) : 0.f, h[k], o[k]);
            } else {
#pragma unroll
              for (int k = 0; k < 16; ++k)
                tc::split_tf32_trunc(v1 ? sinw(v[k], w0) : 0.f, ahi[16 * hf + k], alo[16 * hf + k]);
            }
          }
          if (a.store_a0) store_box(0, m1 + 32 * q);
          tc::mbar_wait(&sb.dfull[b][1], (lc >> 1) & 1);
          tc::fence_after_sync();
          if (F16) {
            tc::tmem_st16u_nowait(lb + kb / 2, reinterpret_cast<const uint32_t(&)[16]>(ahi));
            tc::tmem_st16u_nowait(lb + kAlo + kb / 2, reinterpret_cast<const uint32_t(&)[16]>(alo));
            tc::tmem_wait_st();
          } else {
            tc::tmem_st32(lb + kb, ahi);
            tc::tmem_st32(lb + kAlo + kb, alo);
          }
          tc::fence_before_sync();
          tc::mbar_arrive(&sb.ardy[jr]);
          if (role > 0) CTRACE(role, 11, i + 1);
        } else {
          tc::mbar_wait(&sb.dfull[b][1], (lc >> 1) & 1);
        }
        if (role > 0) CTRACE(role, 12, lc);
        tc::fence_after_sync();
        open_box();
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
          float v[16];
          tc::tmem_ld16(lb + kColD + b * CH + kb + 16 * hf, v);
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = fmaf(v[k], kDs, s_bias[l * CH + kb + 16 * hf + k]);
          put_box(v, hf);
          if (last) {
#pragma unroll
            for (int k = 0; k < 16; ++k) hp = fmaf(s_wl[kb + 16 * hf + k], sinw(v[k], w0), hp);
          } else {
            put_a(v, hf, valid);
          }
        }
        tc::fence_before_sync();
        tc::mbar_arrive(&sb.dfree[b][hN]);  // D_b half read; the next layer's A is in flight
        if (role > 0) CTRACE(role, 13, lc);
        store_box(l + 1, m0 + 32 * q);
        if (!last) a_ready();
        if (role > 0) CTRACE(role, 14, lc);
      }
      // output head: the four chunks of a pixel in a fixed order
      s_head[j * CT + p] = hp;
      tc::named_sync(1, 32 * kEpiWarps);
      if (j == 0 && valid)
        a.dv[a.idx[m0 + p]] =
            a.scale * (a.bL[0] + (((s_head[p] + s_head[CT + p]) + s_head[2 * CT + p]) + s_head[3 * CT + p]));
      tc::named_sync(1, 32 * kEpiWarps);
      if (role > 0) CTRACE(role, 15, i);
    }
    if (lane == 0) tc::bulk_wait_all();  // the activation stores are complete before exit
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(t0);
}

// ---- split-fp16 forward with two tiles in flight ------------------------------
// With fp16 operands a tile's A (hi + lo, two features per column) takes 128
// TMEM columns, so two tiles fit beside one accumulator each:
//   TMEM  slot t = 0, 1: A hi [128 t, 128 t + 64), lo [128 t + 64, 128 t + 128),
//         D [256 + 128 t, 256 + 128 t + 128).
// The tensor core alternates the slots layer by layer -- (tile a, l), (tile
// b, l), (tile a, l + 1), ... -- so one tile's epilogue (TMEM -> sin ->
// next-layer A, activation stores) runs while the tensor core computes the
// other tile's layer, instead of the single-tile MMA -> epilogue -> MMA
// hand-off.  Roles, weight ring, stores and the head are those of
// siren_chain_fwd_kernel (F16); a group is the CTA's tiles 2g, 2g + 1.
struct PairBars {
  uint64_t wfull[2], wempty[2];  // weight stage j: K-chunk j (64 features) of the current layer
  uint64_t ardy[2][2];           // [slot][K-chunk] A written (256 threads)
  uint64_t dfull[2][2], dfree[2][2];  // [slot][N-half]: ready (MMA commit) / drained (256 threads)
  uint32_t tslot;
};

__global__ void __launch_bounds__(kThreads, 1)
siren_chain_pair_kernel(ChainArgs a, const __grid_constant__ CUtensorMap tmap_acts) {
  constexpr float kDs = 1.f / kF16Scale;
  extern __shared__ unsigned char smem_dyn[];
  float* wring = tc::smem_align1024<float>(smem_dyn);  // [2][2][128][64 fp16]
  float* s_tr = wring + WS * 2 * kPlaneFloats;  // [16 warps] SW128 store boxes (1024-aligned)
  float* s_w0 = s_tr + kEpiWarps * kBoxBytes / 4;                          // [128][2]
  float* s_b0 = s_w0 + 2 * CH;                                             // [128]
  float* s_wl = s_b0 + CH;                                                 // [128]
  float* s_bias = s_wl + CH;                                               // [nl][128]
  float* s_head = s_bias + kMaxHidden * CH;                                // [2 slots][4][128]
  __shared__ PairBars sb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tc::tmem_alloc<512>(&sb.tslot);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sb.wfull[i], 1);
      tc::mbar_init(&sb.wempty[i], 1);
    }
    for (int t = 0; t < 2; ++t)
      for (int h = 0; h < 2; ++h) {
        tc::mbar_init(&sb.ardy[t][h], 2 * CT);
        tc::mbar_init(&sb.dfull[t][h], 1);
        tc::mbar_init(&sb.dfree[t][h], 32 * kEpiWarps / 2);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 2 * CH; i += kThreads) s_w0[i] = a.W0[i];
  for (int i = tid; i < CH; i += kThreads) {
    s_b0[i] = a.b0[i];
    s_wl[i] = a.wL[i];
  }
  for (int l = 0; l < a.nl; ++l)
    for (int i = tid; i < CH; i += kThreads) s_bias[l * CH + i] = a.bias[l][i];
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t t0 = sb.tslot;
  const int n_tiles = (a.n + CT - 1) / CT;
  const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int n_groups = (my_tiles + 1) / 2;
  const int nl = a.nl;
  auto group_tiles = [&](int g) { return min(2, my_tiles - 2 * g); };

  if (warp == 0) {
    // ---- weights: chunk j of (group, layer) into stage j once both slots'
    // MMAs of the previous (group, layer) are done with it ----
    if (lane == 0) {
      uint32_t u = 0;
      for (int g = 0; g < n_groups; ++g)
        for (int l = 0; l < nl; ++l, ++u)
          for (int j = 0; j < 2; ++j) {
            if (u > 0) tc::mbar_wait_sleep(&sb.wempty[j], (u - 1) & 1);
            tc::mbar_expect_tx(&sb.wfull[j], kChunkBytes);
            tc::bulk_load(wring + j * 2 * kPlaneFloats,
                          a.wplanes + static_cast<size_t>(l * 2 + j) * 2 * kPlaneFloats, kChunkBytes,
                          &sb.wfull[j]);
          }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::idesc_f16(CT, CH / 2);
    for (int g = 0; g < n_groups; ++g) {
      const int nt = group_tiles(g);
      for (int l = 0; l < nl; ++l) {
        const uint32_t u = static_cast<uint32_t>(g * nl + l);  // use of every slot buffer
        for (int t = 0; t < nt; ++t)
          for (int nh = 0; nh < 2; ++nh) {
            const uint32_t dcol = t0 + 256 + 128 * t + nh * (CH / 2), acol = t0 + 128 * t;
            if (u >= 1) tc::mbar_wait_sleep(&sb.dfree[t][nh], (u - 1) & 1);
            for (int j = 0; j < 2; ++j) {
              if (nh == 0) {
                tc::mbar_wait_sleep(&sb.ardy[t][j], u & 1);
                tc::mbar_wait_sleep(&sb.wfull[j], u & 1);
              }
              tc::fence_after_sync();
              const uint32_t sh = saddr(wring + j * 2 * kPlaneFloats) + nh * (CH / 2) * 128,
                             sl = sh + kPlaneFloats * 4;
              if (tc::elect_one()) {
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                  const uint32_t ka = j * 32 + 8 * s;
                  const uint64_t dh = tc::smem_desc_sw128(sh + 32 * s);
                  const uint64_t dl = tc::smem_desc_sw128(sl + 32 * s);
                  tc::mma_f16_ts(dcol, acol + 64 + ka, dh, idesc, (j | s) != 0);
                  tc::mma_f16_ts(dcol, acol + ka, dl, idesc, 1u);
                  tc::mma_f16_ts(dcol, acol + ka, dh, idesc, 1u);
                }
                if (t == nt - 1 && nh == 1) tc::mma_commit(&sb.wempty[j]);
                if (j == 1) tc::mma_commit(&sb.dfull[t][nh]);
              }
              __syncwarp();
            }
          }
      }
    }
  } else if (warp >= kEpi0 / 32) {
    // ---- epilogue: 16 warps, warp = (TMEM lane quarter q, feature chunk j of
    // 32); pixel = lane ----
    const int q = warp & 3, ew = warp - kEpi0 / 32, j = ew >> 2;
    const int p = 32 * q + lane, kb = CKC * j;
    const uint32_t lb = t0 + (static_cast<uint32_t>(32 * q) << 16);
    float* box = s_tr + ew * kBoxBytes / 4;
    const int hN = j >> 1, jr = j >> 1;  // the accumulator N-half = the next layer's K-chunk
    const float w0 = a.w0;
    uint32_t nst = 0;
    auto open_box = [&]() {
      if (nst >= 1) {
        if (lane == 0) tc::bulk_wait_read<0>();
        __syncwarp();
      }
    };
    auto put_box = [&](const float (&v)[16], int hf) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int gq = 4 * hf + c;
        *reinterpret_cast<float4*>(box + lane * 32 + ((gq ^ (lane & 7)) << 2)) =
            make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
      }
    };
    auto store_box = [&](int l, int r0) {
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tc::tma_store_3d(&tmap_acts, box, kb, r0, l);
        tc::bulk_commit();
      }
      ++nst;
    };
    // (rows past n carry the coordinates (0, 0): finite values in every layer,
    // never stored -- the TMA store clips them and the head skips them -- so A
    // needs no masking)
    auto put_a = [&](int t, const float (&v)[16], int hf, bool) {
      uint32_t hi[8], lo[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        tc::split_f16x2(sinw(v[2 * k], w0), sinw(v[2 * k + 1], w0), hi[k], lo[k]);
      tc::tmem_st8u_nowait(lb + 128 * t + (kb + 16 * hf) / 2, hi);
      tc::tmem_st8u_nowait(lb + 128 * t + 64 + (kb + 16 * hf) / 2, lo);
    };
    auto a_ready = [&](int t) {
      tc::tmem_wait_st();
      tc::fence_before_sync();
      tc::mbar_arrive(&sb.ardy[t][jr]);
    };
    auto tile_m0 = [&](int i) { return (blockIdx.x + i * gridDim.x) * CT; };
    // first layer of tile i (CUDA cores): a_0 = W_0 c + b_0 -> acts[0], A of slot t
    auto first_layer = [&](int i, int t) {
      const int m0t = tile_m0(i);
      const bool vt = p < min(CT, a.n - m0t);
      const float2 c = vt ? a.coords[m0t + p] : make_float2(0.f, 0.f);
      if (a.store_a0) open_box();
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int f = kb + 16 * hf + k;
          v[k] = fmaf(s_w0[2 * f + 1], c.y, fmaf(s_w0[2 * f], c.x, s_b0[f]));
        }
        if (a.store_a0) put_box(v, hf);
        put_a(t, v, hf, vt);
      }
      if (a.store_a0) store_box(0, m0t + 32 * q);
      a_ready(t);
    };
    if (n_groups > 0)
      for (int t = 0; t < group_tiles(0); ++t) first_layer(t, t);
    float hp[2] = {0.f, 0.f};  // head partials of the slots
    for (int g = 0; g < n_groups; ++g) {
      const int nt = group_tiles(g);
      for (int l = 0; l < nl; ++l) {
        const uint32_t u = static_cast<uint32_t>(g * nl + l);
        const bool last = l == nl - 1;
        for (int t = 0; t < nt; ++t) {
          const int i = 2 * g + t, m0 = tile_m0(i);
          const bool valid = p < min(CT, a.n - m0);
          if (!last) {
            tc::mbar_wait(&sb.dfull[t][hN], u & 1);
          } else {
            // every MMA of this slot's last layer is done (both halves): its A
            // columns take the next group's tile of this slot (first layer)
            tc::mbar_wait(&sb.dfull[t][1], u & 1);
            if (g + 1 < n_groups && t < group_tiles(g + 1)) {
              tc::fence_after_sync();
              first_layer(i + 2, t);
            }
          }
          tc::fence_after_sync();
          open_box();
          if (l == 0) hp[t] = 0.f;
#pragma unroll 1
          for (int hf = 0; hf < 2; ++hf) {
            float v[16];
            tc::tmem_ld16(lb + 256 + 128 * t + kb + 16 * hf, v);
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = fmaf(v[k], kDs, s_bias[l * CH + kb + 16 * hf + k]);
            put_box(v, hf);
            if (last) {
#pragma unroll
              for (int k = 0; k < 16; ++k) hp[t] = fmaf(s_wl[kb + 16 * hf + k], sinw(v[k], w0), hp[t]);
            } else {
              put_a(t, v, hf, valid);
            }
          }
          tc::fence_before_sync();
          tc::mbar_arrive(&sb.dfree[t][hN]);
          store_box(l + 1, m0 + 32 * q);
          if (!last) a_ready(t);
        }
      }
      // output heads of the group's tiles: the four chunks of a pixel in a fixed order
      for (int t = 0; t < nt; ++t) s_head[(t * NCH + j) * CT + p] = hp[t];
      tc::named_sync(1, 32 * kEpiWarps);
      if (j < nt) {
        const int t = j, m0 = tile_m0(2 * g + t);
        if (p < min(CT, a.n - m0)) {
          const float* h = s_head + t * NCH * CT;
          a.dv[a.idx[m0 + p]] =
              a.scale * (a.bL[0] + (((h[p] + h[CT + p]) + h[2 * CT + p]) + h[3 * CT + p]));
        }
      }
      tc::named_sync(1, 32 * kEpiWarps);
    }
    if (lane == 0) tc::bulk_wait_all();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(t0);
}

}  // namespace

// PACT_SIREN_F16=0 keeps the 3xTF32 MMAs (comparisons); default split fp16.
static bool chain_f16() {
  static const bool on = [] {
    const char* e = std::getenv("PACT_SIREN_F16");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Forward of the whole network for hidden width 128 with >= 1 tcgen05 layer.
Status tc_forward_chain(pact_ctx* ctx, const SirenShape& s, const float* theta, SirenWork& w,
                        float* dv, bool store_a0) {
  const int n = w.n, L = s.layers, nl = L - 1;
  if (s.hidden != CH || nl < 1 || nl > kMaxHidden || s.in_dim != 2)
    return validation("tc_forward_chain: unsupported network shape");
  if (n == 0) return {};
  cudaStream_t st = ctx->stream;
  const size_t plane_floats = static_cast<size_t>(nl) * NCH * 2 * kPlaneFloats;
  if (w.wplanes_floats < plane_floats) {
    pool_free(w.wplanes, st);
    w.wplanes = nullptr;
    w.wplanes_floats = 0;
    PACT_TRY_S(pool_alloc(reinterpret_cast<void**>(&w.wplanes), sizeof(float) * plane_floats + 256,
                          st));
    w.wplanes_floats = plane_floats;
  }
  // layer offsets into theta travel in the launch arguments (graph-capturable)
  LayerOffsets lo{};
  for (int l = 0; l < nl; ++l) lo.off[l] = static_cast<long long>(s.offset(l + 1));
  const bool f16 = chain_f16();
  if (f16)
    chain_wplanes_kernel<true><<<div_up(nl * CH * CH, 256), 256, 0, st>>>(theta, lo, nl, w.wplanes);
  else
    chain_wplanes_kernel<false><<<div_up(nl * CH * CH, 256), 256, 0, st>>>(theta, lo, nl, w.wplanes);
  PACT_TRY_S(after_launch(ctx, "chain_wplanes_kernel"));
  ChainArgs a{};
  a.coords = w.coords;
  a.idx = w.idx;
  a.n = n;
  a.W0 = theta + s.offset(0);
  a.b0 = a.W0 + 2 * CH;
  for (int l = 0; l < nl; ++l) a.bias[l] = theta + s.offset(l + 1) + static_cast<size_t>(CH) * CH;
  a.wplanes = w.wplanes;
  a.nl = nl;
  a.wL = theta + s.offset(L);
  a.bL = a.wL + CH;
  a.scale = static_cast<float>(s.out_scale);
  a.w0 = static_cast<float>(s.omega0);
  a.acts = w.acts;
  a.dv = dv;
  a.store_a0 = store_a0 ? 1 : 0;
  // acts as a 3-D tensor [L][n][128] fp32 for the epilogue's TMA stores
  static PFN_cuTensorMapEncodeTiled encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }();
  if (!encode) return internal_error("tc_forward_chain: cuTensorMapEncodeTiled unavailable");
  CUtensorMap tmap;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(CH), static_cast<cuuint64_t>(n),
                              static_cast<cuuint64_t>(L)};
  const cuuint64_t strides[2] = {sizeof(float) * CH, sizeof(float) * CH * static_cast<cuuint64_t>(n)};
  const cuuint32_t box[3] = {32, 32, 1}, estr[3] = {1, 1, 1};
  if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, w.acts, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return internal_error("tc_forward_chain: tensor map encoding failed");
  const size_t smem = 1024 + sizeof(float) * (WS * 2 * kPlaneFloats + kEpiWarps * kBoxBytes / 4 +
                                               2 * CH + CH + CH + kMaxHidden * CH + NCH * CT);
  const int grid = std::min(ctx->num_sms, div_up(n, CT));
  if (f16) {
    const size_t smem2 = smem + sizeof(float) * NCH * CT;  // s_head of the second slot
    PACT_CUDA_S(cudaFuncSetAttribute(siren_chain_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem2)));
    siren_chain_pair_kernel<<<grid, kThreads, smem2, st>>>(a, tmap);
  } else {
    PACT_CUDA_S(cudaFuncSetAttribute(siren_chain_fwd_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    siren_chain_fwd_kernel<false><<<grid, kThreads, smem, st>>>(a, tmap);
  }
  return after_launch(ctx, "siren_chain_fwd_kernel");
}

}  // namespace pactgpu

#if CHAIN_EXP == 2
extern "C" int pact_debug_chain_trace(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (out) cudaMemcpyFromSymbol(out, g_ctrace, sizeof(unsigned long long) * 3 * 1024 * 3);
  if (reset) {
    static unsigned long long zero[3 * 1024 * 3];
    cudaMemcpyToSymbol(g_ctrace, zero, sizeof(zero));
  }
  return 1024;
}
#endif
