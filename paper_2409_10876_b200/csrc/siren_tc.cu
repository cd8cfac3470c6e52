// SIREN hidden layers on the 5th-generation tensor cores (tcgen05, sm_100a),
// 3xTF32 split precision (tc.cuh), hidden width 128 (cfg3, cfg4):
//   forward   a_l = W_l sin(w0 a_{l-1}) + b_l                  (nfield.hpp:164-180)
//   backward  dA_{l-1} = (W_l^T dA_l) * w0 cos(w0 a_{l-1})     (nfield.hpp:190-230)
//   weights   gW_l = sum_m dA_l[m] sin(w0 a_{l-1}[m])^T, gb_l = sum_m dA_l[m]
//
// Layer kernels (forward / dgrad): persistent, one CTA of 128 threads per SM.
// The layer matrix is the MMA's A operand and lives in TMEM for the whole
// kernel (hi and lo TF32 planes, lane = output feature); pixels are the MMA's
// N.  Each 128-pixel tile of activations arrives by cp.async.bulk (one 512-B
// row per copy, padded rows so the re-layout is bank-conflict free) one tile
// ahead of use; the CTA re-lays a 32-wide K-chunk into K-major hi/lo planes
// (fusing the sine), one thread issues the chunk's 12 MMAs, and the commit
// frees the chunk buffer.  Two TMEM accumulators alternate so the epilogue of
// tile i-1 (bias or cosine, coalesced stores: lane = feature) runs while the
// tensor core works on tile i.
//
// Weight gradient: split over pixel ranges (one CTA per SM), accumulator
// D[r][k] in TMEM with K = pixels.  dA^T enters TMEM directly from registers
// (tcgen05.st, lane = r), sin(w0 a_{l-1})^T goes through shared-memory planes;
// both raw tiles (64 pixels) arrive by bulk copies one tile ahead.  Partials
// are reduced in a fixed order in fp64 by the caller (deterministic).
#include <cstdint>

#include "siren.cuh"
#include "tc.cuh"

// TC_EXP (experiments only, never set in the product build): 1 = no MMA
// issue, 2 = no raw reads / sine (zero planes), 3 = no epilogue stores,
// 4 = 1 + 2 (bulk loads, barriers and epilogue only).
#ifndef TC_EXP
#define TC_EXP 0
#endif

#if TC_EXP == 5 || TC_EXP == 6
// Timeline trace of CTA 0 (experiments only): {tag, tile/chunk, globaltimer ns},
// one region per tracing role, store-only (no atomics on the traced path).
__device__ unsigned long long g_trace[3 * 4096];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ void trace(int tag, int idx) {
  if (blockIdx.x != 0) return;
  static __shared__ unsigned int s_cnt[3];
  const int role = tag <= 4 ? 0 : tag == 5 ? 1 : 2;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const unsigned k = role * 1365 + (s_cnt[role]++ % 1365);
  g_trace[3 * k] = tag;
  g_trace[3 * k + 1] = idx;
  g_trace[3 * k + 2] = t;
}
#define TRACE(tag, idx) trace(tag, idx)
#else
#define TRACE(tag, idx)
#endif

namespace pactgpu {
namespace {

constexpr int H = 128;    // hidden width handled here
constexpr int TP = 128;   // pixels per layer tile (MMA N)
constexpr int KC = 32;    // K per staged chunk

__device__ __forceinline__ float red2pi_tc(float x) { return sine_reduce(x); }
__device__ __forceinline__ float sin_w(float a, float w0) { return __sinf(red2pi_tc(w0 * a)); }
__device__ __forceinline__ float dsin_w(float a, float w0) {
  return w0 * __cosf(red2pi_tc(w0 * a));
}

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void sync_tc() {
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

// 4 consecutive-K values (k % 4 == 0) of one row into K-major hi/lo planes.
__device__ __forceinline__ void put4(float* hi, float* lo, int row, int k, int R, float4 v) {
  float4 h, l;
  tc::split_tf32_trunc(v.x, h.x, l.x);
  tc::split_tf32_trunc(v.y, h.y, l.y);
  tc::split_tf32_trunc(v.z, h.z, l.z);
  tc::split_tf32_trunc(v.w, h.w, l.w);
  const uint32_t o = tc::kmajor_offset(row, k, R) >> 2;
  *reinterpret_cast<float4*>(hi + o) = h;
  *reinterpret_cast<float4*>(lo + o) = l;
}

__device__ __forceinline__ uint32_t lane_base(uint32_t t0, int warp) {
  return t0 + (static_cast<uint32_t>(32 * warp) << 16);
}

// ---- layer kernels (forward, dgrad) ---------------------------------------
enum Mode { kForward = 0, kDgrad = 1 };

// Lane j of the warp receives sum over the warp's lanes of z[j] (fixed
// butterfly order: deterministic).  31 shuffles for 32 sums.
__device__ __forceinline__ float transpose_reduce32(float (&z)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const float send = up ? z[i] : z[i + off];
      const float keep = up ? z[i + off] : z[i];
      z[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return z[0];
}

struct LayerBars {
  uint64_t raw[2];    // raw tile landed (bulk copies)
  uint64_t ready[2];  // chunk planes written (256 producer threads)
  uint64_t buf[2];    // chunk planes free (MMA commit)
  uint64_t full[2];   // accumulator ready (MMA commit)
  uint64_t empty[2];  // accumulator drained (128 epilogue threads)
  uint32_t tslot;
};

// TMEM columns: A_hi [0,128), A_lo [128,256), D0 [256,384), D1 [384,512)
constexpr uint32_t kColAlo = 128, kColD = 256;
// warps 0-7 stage the chunks, warp 8 issues the MMAs (one elected lane, warp-
// uniform descriptors), warps 9-16 drain the accumulators
constexpr int LPROD = 256;  // producer threads
constexpr int LEPI = 256;   // epilogue threads
// The forward has a dedicated MMA warp (544 threads, 96 registers); the dgrad,
// whose cosine epilogue needs the registers, issues from producer thread 0
// after a per-chunk producer barrier (512 threads, 128 registers).
template <int MODE>
struct LayerRoles {
  static constexpr bool kMmaWarp = MODE == 0;
  static constexpr int kThreads = LPROD + (kMmaWarp ? 32 : 0) + LEPI;
  static constexpr int kEpi0 = LPROD + (kMmaWarp ? 32 : 0);  // first epilogue thread
};
constexpr int kWarpMma = LPROD / 32;  // 8
constexpr int WNTH = 416;  // weight gradient: warps 0-3 dA^T, 4-11 sine planes, 12 MMA

template <int MODE>
__global__ void __launch_bounds__(LayerRoles<MODE>::kThreads, 1)
tc_layer_kernel(const float* __restrict__ X,      // [n][H] MMA input rows (a_{l-1} or dA_l)
                const float* __restrict__ W,      // [H][H] layer matrix, row-major
                const float* __restrict__ bias,   // forward: [H]
                const float* __restrict__ Aprev,  // dgrad: a_{l-1} for the cosine
                int n, float w0, float* __restrict__ Y, SirenHead head) {
  extern __shared__ unsigned char smem_dyn[];
  // 1024-B alignment: the 128-B swizzle is a function of the address bits
  float* raw = tc::smem_align1024<float>(smem_dyn);  // [2][TP][H]
  float* zh = raw + 2 * TP * H;                                         // [2][TP][KC] SW128
  float* zl = zh + 2 * TP * KC;                                         // [2][TP][KC] SW128
  float* wst = raw + TP * H;  // prologue only: W staged [H][H + 1] over raw[1] and the planes
  __shared__ LayerBars sb;
  __shared__ float s_out[2][4][TP];  // fused output layer: per-quarter partial sums
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & 127;  // TMEM lane of this thread (warp % 4 quarter)
  if (warp == 0) tc::tmem_alloc<512>(&sb.tslot);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sb.raw[i], 1);
      tc::mbar_init(&sb.ready[i], LPROD);
      tc::mbar_init(&sb.buf[i], 1);
      tc::mbar_init(&sb.full[i], 1);
      tc::mbar_init(&sb.empty[i], LEPI);
    }
    fence_mbar_init();
  }
  sync_tc();
  const uint32_t t0 = sb.tslot;
  const int n_tiles = (n + TP - 1) / TP;
  const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  // Bulk-load local tile i (rows m0.., contiguous) into raw[i & 1] (thread 0).
  auto load_tile = [&](int i) {
    const int m0 = (blockIdx.x + i * gridDim.x) * TP;
    const uint32_t bytes = static_cast<uint32_t>(min(TP, n - m0)) * H * 4;
    tc::fence_proxy_async();  // the buffer's generic reads before the async refill
    tc::mbar_expect_tx(&sb.raw[i & 1], bytes);
    tc::bulk_load(raw + (i & 1) * TP * H, X + static_cast<size_t>(m0) * H, bytes, &sb.raw[i & 1]);
  };
  if (tid == 0 && my_tiles > 0) load_tile(0);

  // Layer matrix -> TMEM A (lane = output row).  W is staged through shared
  // memory with an odd row stride (coalesced loads, conflict-free reads);
  // warp w writes lane quarter w % 4, plane (w / 8) and K half (w / 4) % 2.
  // Forward A[r][k] = W[r][k]; dgrad A[k][r] = W[r][k].
  constexpr int NTHR = LayerRoles<MODE>::kThreads, EPI0 = LayerRoles<MODE>::kEpi0;
  constexpr bool MW = LayerRoles<MODE>::kMmaWarp;
  for (int e = tid; e < H * H / 4; e += NTHR) {
    const float4 w4 = reinterpret_cast<const float4*>(W)[e];
    float* d = wst + (e / (H / 4)) * (H + 1) + (e % (H / 4)) * 4;
    d[0] = w4.x;
    d[1] = w4.y;
    d[2] = w4.z;
    d[3] = w4.w;
  }
  __syncthreads();
  if (warp < 16) {
    const bool lo_plane = warp >= 8;
    const uint32_t lb = lane_base(t0, warp & 3) + (lo_plane ? kColAlo : 0);
#pragma unroll 1
    for (int k0 = ((warp >> 2) & 1) * (H / 2); k0 < ((warp >> 2) & 1) * (H / 2) + H / 2; k0 += 32) {
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float w = MODE == kForward ? wst[row * (H + 1) + k0 + i] : wst[(k0 + i) * (H + 1) + row];
        float hi, lo;
        tc::split_tf32(w, hi, lo);
        v[i] = lo_plane ? lo : hi;
      }
      tc::tmem_st32(lb + k0, v);
    }
  }
  sync_tc();

  if (tid < LPROD) {
    // ---- producers: re-layout K-chunks into the chunk planes ----
    const int c4 = tid & 7, p0 = tid >> 3;  // 16-B chunk of the K-chunk row, first row
    uint32_t g = 0;  // chunks staged so far (chunk buffer g & 1)
    for (int i = 0; i < my_tiles; ++i) {
      const int m0 = (blockIdx.x + i * gridDim.x) * TP;
      const int rows = min(TP, n - m0);
      if (tid == 0 && i + 1 < my_tiles) load_tile(i + 1);
      if (tid == 0) TRACE(1, i);
      tc::mbar_wait(&sb.raw[i & 1], (i >> 1) & 1);
      if (tid == 0) TRACE(2, i);
      const float* rt = raw + (i & 1) * TP * H;
#pragma unroll 1
      for (int kc0 = 0; kc0 < H; kc0 += KC, ++g) {
        const int b = g & 1;
        if (g >= 2) tc::mbar_wait(&sb.buf[b], ((g - 2) >> 1) & 1);
        if (tid == 0) TRACE(3, g);
        float* bh = zh + b * TP * KC;
        float* bl = zl + b * TP * KC;
        // Rows >= `rows` of the raw tile hold stale bytes: load them anyway
        // (keeps the eight loads independent) and select zero afterwards.
        // Eight threads read one 128-B row segment and write one swizzled
        // 128-B plane row: both conflict free.
        constexpr int PJ = TP / (LPROD / 8);
        float4 v[PJ];
#pragma unroll
        for (int j = 0; j < PJ; ++j)
          v[j] = (TC_EXP == 2 || TC_EXP == 4) ? make_float4(0.f, 0.f, 0.f, 0.f)
                             : *reinterpret_cast<const float4*>(rt + (p0 + (LPROD / 8) * j) * H +
                                                                kc0 + 4 * c4);
#pragma unroll
        for (int j = 0; j < PJ; ++j) {
          const int p = p0 + (LPROD / 8) * j;
          float4 z = v[j];
          if (MODE == kForward && TC_EXP != 2 && TC_EXP != 4)
            z = make_float4(sin_w(z.x, w0), sin_w(z.y, w0), sin_w(z.z, w0), sin_w(z.w, w0));
          if (p >= rows) z = make_float4(0.f, 0.f, 0.f, 0.f);
          float4 h, l;
          tc::split_tf32_trunc(z.x, h.x, l.x);
          tc::split_tf32_trunc(z.y, h.y, l.y);
          tc::split_tf32_trunc(z.z, h.z, l.z);
          tc::split_tf32_trunc(z.w, h.w, l.w);
          const int o = p * KC + ((c4 ^ (p & 7)) << 2);
          *reinterpret_cast<float4*>(bh + o) = h;
          *reinterpret_cast<float4*>(bl + o) = l;
        }
        tc::fence_proxy_async();
        if (MW) {
          tc::mbar_arrive(&sb.ready[b]);
          if (tid == 0) TRACE(4, g);
        } else {
          tc::named_sync(1, LPROD);
          if (tid == 0) {
            constexpr uint32_t idesc = tc::idesc_tf32(H, TP);
            const uint32_t dcol = t0 + kColD + (i & 1) * TP;
            if (kc0 == 0 && i >= 2) tc::mbar_wait(&sb.empty[i & 1], ((i - 2) >> 1) & 1);
            tc::fence_after_sync();
            const uint32_t sbh = saddr(bh), sbl = saddr(bl);
#pragma unroll
            for (int s = 0; s < KC / 8; ++s) {
              const uint32_t ka = kc0 + 8 * s;
              const uint64_t dh = tc::smem_desc_sw128(sbh + 32 * s);
              const uint64_t dl = tc::smem_desc_sw128(sbl + 32 * s);
              tc::mma_tf32_ts(dcol, t0 + kColAlo + ka, dh, idesc, (kc0 | s) != 0);
              tc::mma_tf32_ts(dcol, t0 + ka, dl, idesc, 1u);
              tc::mma_tf32_ts(dcol, t0 + ka, dh, idesc, 1u);
            }
            tc::mma_commit(&sb.buf[b]);
            if (kc0 + KC == H) tc::mma_commit(&sb.full[i & 1]);
          }
        }
      }
      // every producer is done reading raw[i & 1] before tile i + 2 is loaded into
      // it (without the MMA warp the per-chunk barrier already orders this)
      if (MW) tc::named_sync(1, LPROD);
    }
  } else if (MW && warp == kWarpMma) {
    // ---- the MMA warp: waits for a staged chunk, issues its 12 MMAs ----
    constexpr uint32_t idesc = tc::idesc_tf32(H, TP);
    uint32_t g = 0;
    for (int i = 0; i < my_tiles; ++i) {
      const uint32_t dcol = t0 + kColD + (i & 1) * TP;
#pragma unroll 1
      for (int kc0 = 0; kc0 < H; kc0 += KC, ++g) {
        const int b = g & 1;
        tc::mbar_wait(&sb.ready[b], (g >> 1) & 1);
        if (kc0 == 0 && i >= 2) tc::mbar_wait(&sb.empty[i & 1], ((i - 2) >> 1) & 1);
        tc::fence_after_sync();
        if ((tid & 31) == 0) TRACE(5, g);
        const uint32_t sbh = saddr(zh + b * TP * KC), sbl = saddr(zl + b * TP * KC);
        if (tc::elect_one()) {
#pragma unroll
          for (int s = 0; s < (TC_EXP == 1 || TC_EXP == 4 || TC_EXP == 6 ? 0 : KC / 8); ++s) {
            const uint32_t ka = kc0 + 8 * s;
            const uint64_t dh = tc::smem_desc_sw128(sbh + 32 * s);
            const uint64_t dl = tc::smem_desc_sw128(sbl + 32 * s);
            tc::mma_tf32_ts(dcol, t0 + kColAlo + ka, dh, idesc, (kc0 | s) != 0);
            tc::mma_tf32_ts(dcol, t0 + ka, dl, idesc, 1u);
            tc::mma_tf32_ts(dcol, t0 + ka, dh, idesc, 1u);
          }
          tc::mma_commit(&sb.buf[b]);
          if (kc0 + KC == H) tc::mma_commit(&sb.full[i & 1]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---- epilogue: lane = output feature, columns = pixels of the tile;
    // warps 8-11 and 12-15 share the TMEM lane quarters and split the columns ----
    const float brow = MODE == kForward ? bias[row] : 0.f;
    const int cb = ((warp - EPI0 / 32) >> 2) * (TP / 2);
    const bool fuse_out = MODE == kForward && head.w != nullptr;
    const float wrow = fuse_out ? head.w[row] : 0.f;
    for (int i = 0; i < my_tiles; ++i) {
      const int m0 = (blockIdx.x + i * gridDim.x) * TP;
      const int rows = min(TP, n - m0);
      // a_{l-1} for the cosine (dgrad) does not depend on the accumulator: all
      // 64 columns of this thread are fetched before the wait
      float av[TP / 2];
      if (MODE == kDgrad) {
        const float* a = Aprev + static_cast<size_t>(m0) * H + row;
#pragma unroll
        for (int j = 0; j < TP / 2; ++j) av[j] = a[min(cb + j, rows - 1) * H];
      }
      if (tid == EPI0) TRACE(6, i);
      tc::mbar_wait(&sb.full[i & 1], (i >> 1) & 1);
      if (tid == EPI0) TRACE(7, i);
      tc::fence_after_sync();
      const uint32_t d = lane_base(t0, warp & 3) + kColD + (i & 1) * TP;
      float* y = Y + static_cast<size_t>(m0) * H + row;
#pragma unroll
      for (int h = 0; MODE == kDgrad && h < TP / 2; h += 32) {
        float v[32];
        tc::tmem_ld32(d + cb + h, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int c = cb + h + j;
          const float out = v[j] * dsin_w(av[h + j], w0);  // unconditional: predicated store
          if (c < rows && TC_EXP != 3) y[c * H] = out;
        }
      }
#pragma unroll
      for (int h = 0; MODE == kForward && h < TP / 2; h += 32) {
        float v[32];
        tc::tmem_ld32(d + cb + h, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int c = cb + h + j;
          const float out = v[j] + brow;
          if (c < rows && (TC_EXP != 3 || out == 12345.f)) y[c * H] = out;
          v[j] = out;
        }
        if (fuse_out) {
          // output layer w_L . sin(w0 a_{L-1}) (nfield.hpp:126-130): this warp's
          // 32 features per pixel, lane j <- pixel cb + h + j
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = wrow * sin_w(v[j], w0);
          const float part = transpose_reduce32(v, tid & 31);
          s_out[i & 1][warp & 3][cb + h + (tid & 31)] = part;
        }
      }
      tc::fence_before_sync();
      tc::mbar_arrive(&sb.empty[i & 1]);
      if (tid == EPI0) TRACE(8, i);
      if (fuse_out) {
        tc::named_sync(2, LEPI);
        const int c = tid - EPI0;
        if (c < rows) {
          const float* so = &s_out[i & 1][0][0];
          const float s = ((so[c] + so[TP + c]) + so[2 * TP + c]) + so[3 * TP + c];
          head.dv[head.idx[m0 + c]] = head.scale * (head.b[0] + s);
        }
      }
    }
  }
  sync_tc();
  if (warp == 0) tc::tmem_free<512>(t0);
}

// ---- weight gradient --------------------------------------------------------
constexpr int WP = 64;  // pixels per raw tile

struct WgradBars {
  uint64_t raw[2];
  uint64_t ready[2];  // chunk staged (384 producer threads)
  uint64_t buf[2];    // chunk consumed (MMA commit)
  uint64_t acc;
  uint32_t tslot;
};

// TMEM: D [0,128); A chunk b: hi [128 + 64b, +32), lo [160 + 64b, +32).
// Warps 0-3 put dA^T into TMEM (lane r), warps 4-11 build the sine planes,
// warp 12 issues the MMAs (one elected lane).
constexpr int WPROD = 384;
__global__ void __launch_bounds__(WNTH, 1)
tc_wgrad_kernel(const float* __restrict__ dA, const float* __restrict__ Aprev, int n, int rows,
                float w0, float* __restrict__ partial) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* rda = reinterpret_cast<float*>(smem);  // [2][WP][H]
  float* rap = rda + 2 * WP * H;                // [2][WP][H]
  float* zh = rap + 2 * WP * H;                 // [2][H * KC]
  float* zl = zh + 2 * H * KC;                  // [2][H * KC]
  __shared__ WgradBars sb;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int r = tid & 127;
  if (warp == 0) tc::tmem_alloc<256>(&sb.tslot);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sb.raw[i], 1);
      tc::mbar_init(&sb.ready[i], WPROD);
      tc::mbar_init(&sb.buf[i], 1);
    }
    tc::mbar_init(&sb.acc, 1);
    fence_mbar_init();
  }
  sync_tc();
  const uint32_t t0 = sb.tslot;
  const int m_begin = blockIdx.x * rows, m_end = min(n, m_begin + rows);
  const int n_raw = m_end > m_begin ? (m_end - m_begin + WP - 1) / WP : 0;
  const int n_chunks = n_raw * (WP / KC);

  auto load_tile = [&](int i) {
    const int p0 = m_begin + i * WP;
    const uint32_t bytes = static_cast<uint32_t>(min(WP, m_end - p0)) * H * 4;
    uint64_t* bar = &sb.raw[i & 1];
    tc::fence_proxy_async();  // the buffer's generic reads before the async refill
    tc::mbar_expect_tx(bar, 2 * bytes);
    tc::bulk_load(rda + (i & 1) * WP * H, dA + static_cast<size_t>(p0) * H, bytes, bar);
    tc::bulk_load(rap + (i & 1) * WP * H, Aprev + static_cast<size_t>(p0) * H, bytes, bar);
  };
  if (tid == 0 && n_raw > 0) load_tile(0);

  float bias_acc = 0.f;
  if (tid < WPROD) {
    // ---- producers ----
    uint32_t g = 0;
    for (int i = 0; i < n_raw; ++i) {
      const int p0 = m_begin + i * WP;
      const int valid = min(WP, m_end - p0);
      if (tid == 0 && i + 1 < n_raw) load_tile(i + 1);
      tc::mbar_wait(&sb.raw[i & 1], (i >> 1) & 1);
      const float* ta = rda + (i & 1) * WP * H;
      const float* tz = rap + (i & 1) * WP * H;
#pragma unroll 1
      for (int q0 = 0; q0 < WP; q0 += KC, ++g) {
        const int b = g & 1;
        if (g >= 2) tc::mbar_wait(&sb.buf[b], ((g - 2) >> 1) & 1);
        if (warp < 4) {
          // dA^T chunk -> TMEM (lane r, column = pixel)
          float hi[32], lo[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) hi[j] = ta[(q0 + j) * H + r];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x = q0 + j < valid ? hi[j] : 0.f;
            bias_acc += x;
            tc::split_tf32_trunc(x, hi[j], lo[j]);
          }
          const uint32_t lb = lane_base(t0, warp) + 128 + 64 * b;
          tc::tmem_st32(lb, hi);
          tc::tmem_st32(lb + 32, lo);
          tc::fence_before_sync();
        } else {
          // sin(w0 a_{l-1})^T chunk -> planes (row k = r, K = pixel); warps
          // 4-7 take pixels [0, 16) of the chunk, warps 8-11 pixels [16, 32).
          // Stale rows past `valid` are read and zeroed after the sine (no
          // branch around the MUFU).
          constexpr int HK = KC / 2;
          const int j0 = warp >= 8 ? HK : 0;
          float a[HK];
          float* bh = zh + b * H * KC;
          float* bl = zl + b * H * KC;
#pragma unroll
          for (int j = 0; j < HK; ++j) a[j] = tz[(q0 + j0 + j) * H + r];
#pragma unroll
          for (int j = 0; j < HK; ++j) {
            const float z = sin_w(a[j], w0);
            a[j] = q0 + j0 + j < valid ? z : 0.f;
          }
#pragma unroll
          for (int j = 0; j < HK; j += 4)
            put4(bh, bl, r, j0 + j, H, make_float4(a[j], a[j + 1], a[j + 2], a[j + 3]));
          tc::fence_proxy_async();
        }
        tc::mbar_arrive(&sb.ready[b]);
      }
      // every producer is done reading raw[i & 1] before tile i + 2 is loaded into it
      tc::named_sync(1, WPROD);
    }
  } else if (warp == WPROD / 32) {
    // ---- the MMA warp ----
    constexpr uint32_t LBO = (H / 8) * 128;
    constexpr uint32_t idesc = tc::idesc_tf32(H, H);
    for (int g = 0; g < n_chunks; ++g) {
      const int b = g & 1;
      tc::mbar_wait(&sb.ready[b], (g >> 1) & 1);
      tc::fence_after_sync();
      const uint32_t sbh = saddr(zh + b * H * KC), sbl = saddr(zl + b * H * KC);
      const uint32_t ah = t0 + 128 + 64 * b, al = ah + 32;
      if (tc::elect_one()) {
#pragma unroll
        for (int s = 0; s < KC / 8; ++s) {
          const uint64_t dh = tc::smem_desc(sbh + 2 * s * LBO, LBO, 128);
          const uint64_t dl = tc::smem_desc(sbl + 2 * s * LBO, LBO, 128);
          tc::mma_tf32_ts(t0, al + 8 * s, dh, idesc, (g | s) != 0);
          tc::mma_tf32_ts(t0, ah + 8 * s, dl, idesc, 1u);
          tc::mma_tf32_ts(t0, ah + 8 * s, dh, idesc, 1u);
        }
        tc::mma_commit(&sb.buf[b]);
        if (g + 1 == n_chunks) tc::mma_commit(&sb.acc);
      }
      __syncwarp();
    }
  }
  float* out = partial + static_cast<size_t>(blockIdx.x) * (static_cast<size_t>(H) * H + H);
  if (n_chunks > 0) {
    tc::mbar_wait(&sb.acc, 0);
    tc::fence_after_sync();
    // warps w and w + 4 (w < 4) share TMEM lanes; each drains half the columns
    const uint32_t lb = lane_base(t0, warp & 3);
    const int cbeg = warp < 4 ? 0 : H / 2;
    if (warp < 8) {
#pragma unroll 1
      for (int c0 = cbeg; c0 < cbeg + H / 2; c0 += 32) {
        float v[32];
        tc::tmem_ld32(lb + c0, v);
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(out + static_cast<size_t>(r) * H + c0 + j) =
              make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
  } else if (warp < 8) {
    for (int c = (warp < 4 ? 0 : H / 2); c < (warp < 4 ? H / 2 : H); ++c)
      out[static_cast<size_t>(r) * H + c] = 0.f;
  }
  if (warp < 4) out[static_cast<size_t>(H) * H + r] = bias_acc;
  sync_tc();
  if (warp == 0) tc::tmem_free<256>(t0);
}

constexpr size_t kLayerSmem = sizeof(float) * (2 * TP * H + 4 * TP * KC) + 1024;
constexpr size_t kWgradSmem = sizeof(float) * (4 * WP * H + 4 * H * KC);

template <class K>
Status set_smem(K kernel, size_t bytes) {
  PACT_CUDA_S(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(bytes)));
  return {};
}

int layer_grid(pact_ctx* ctx, int n) {
  return std::max(1, std::min((n + TP - 1) / TP, ctx->num_sms));
}

Status unsupported_width() {
  set_error("tcgen05 SIREN layers need hidden == %d", H);
  return {PACT_E_UNSUPPORTED};
}

}  // namespace

bool siren_tc_supported(int hidden) { return hidden == H; }

int tc_wgrad_rows(pact_ctx* ctx, int n) {
  return std::max(WP, div_up(div_up(n, ctx->num_sms), WP) * WP);
}

Status tc_forward_layer(pact_ctx* ctx, int hidden, const float* Ain, const float* W,
                        const float* b, int n, float w0, float* Aout, const SirenHead& head) {
  if (hidden != H) return unsupported_width();
  PACT_TRY_S(smem_optin(tc_layer_kernel<kForward>, kLayerSmem));
  tc_layer_kernel<kForward><<<layer_grid(ctx, n), LayerRoles<kForward>::kThreads, kLayerSmem,
                              ctx->stream>>>(
      Ain, W, b, nullptr, n, w0, Aout, head);
  return after_launch(ctx, "tc_layer_kernel<forward>");
}

Status tc_dgrad_layer(pact_ctx* ctx, int hidden, const float* dAl, const float* W,
                      const float* Aprev, int n, float w0, float* dAprev) {
  if (hidden != H) return unsupported_width();
  PACT_TRY_S(smem_optin(tc_layer_kernel<kDgrad>, kLayerSmem));
  tc_layer_kernel<kDgrad><<<layer_grid(ctx, n), LayerRoles<kDgrad>::kThreads, kLayerSmem,
                            ctx->stream>>>(
      dAl, W, nullptr, Aprev, n, w0, dAprev, SirenHead{});
  return after_launch(ctx, "tc_layer_kernel<dgrad>");
}

Status tc_wgrad_layer(pact_ctx* ctx, int hidden, const float* dAl, const float* Aprev, int n,
                      int rows, float w0, float* partial, int n_chunks) {
  if (hidden != H) return unsupported_width();
  PACT_TRY_S(smem_optin(tc_wgrad_kernel, kWgradSmem));
  tc_wgrad_kernel<<<n_chunks, WNTH, kWgradSmem, ctx->stream>>>(dAl, Aprev, n, rows, w0, partial);
  return after_launch(ctx, "tc_wgrad_kernel");
}

}  // namespace pactgpu

#if TC_EXP == 5 || TC_EXP == 6
extern "C" int pact_debug_trace(unsigned long long* out, int n, int reset) {
  cudaDeviceSynchronize();
  if (out) cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * 3 * std::min(n, 4095));
  if (reset) {
    static unsigned long long zero[3 * 4096];
    cudaMemcpyToSymbol(g_trace, zero, sizeof(zero));
  }
  return 4095;
}
#endif
