// SIREN dense layers on the 5th-generation tensor cores (tcgen05, sm_100a),
// 3xTF32 split precision (tc.cuh): the hidden-layer GEMMs of nfield.hpp
// (forward a_l = W_l z + b, backward dA_{l-1} = (dA_l W_l) * w0 cos(w0 a_{l-1}),
// weight gradient dA_l^T z_{l-1}) for hidden widths 64 and 128.
//
// Persistent CTAs (one per SM, 128 threads).  The layer weights are split into
// TF32 hi/lo planes once per CTA and stay resident in shared memory; the
// activation operand streams through two 32-wide K-chunk buffers.  The whole
// CTA stages a chunk (global -> sine / split -> core-matrix layout), one
// thread issues the 12 MMAs of the chunk (4 k-steps x {hi*hi, hi*lo, lo*hi})
// into a TMEM accumulator, and the commit of chunk c frees its buffer for
// chunk c + 2 while the tensor core runs.  Epilogues read TMEM row-per-thread
// (tcgen05.ld 32x32b) and fuse bias / cosine.
#include <cstdint>

#include "siren.cuh"
#include "tc.cuh"

namespace pactgpu {
namespace {

constexpr int TM = 128;   // pixel rows per tile (MMA M)
constexpr int KC = 32;    // K per staged chunk
constexpr int NTH = 128;  // threads per CTA

__device__ __forceinline__ float red2pi_tc(float x) {
  const float k = rintf(x * 0.159154943091895336f);
  return fmaf(-k, -1.74845553146951720e-07f, fmaf(-k, 6.28318548202514648f, x));
}
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

// Store 4 consecutive-K values (k % 4 == 0) of one row into the hi/lo planes.
__device__ __forceinline__ void put4(float* hi, float* lo, int row, int k, int R, float4 v) {
  float4 h, l;
  tc::split_tf32(v.x, h.x, l.x);
  tc::split_tf32(v.y, h.y, l.y);
  tc::split_tf32(v.z, h.z, l.z);
  tc::split_tf32(v.w, h.w, l.w);
  const uint32_t o = tc::kmajor_offset(row, k, R) >> 2;
  *reinterpret_cast<float4*>(hi + o) = h;
  *reinterpret_cast<float4*>(lo + o) = l;
}

// Resident weight planes: B[n][k] (N rows, K = H) from row-major W.
//   TRANS = false: B[n][k] = W[n][k] (forward: a = z W^T)
//   TRANS = true : B[n][k] = W[k][n] (backward: dA_{l-1} = dA_l W)
template <int H, bool TRANS>
__device__ void load_weights(const float* __restrict__ W, float* wh, float* wl) {
  for (int e = threadIdx.x; e < H * H / 4; e += NTH) {
    const int n = e / (H / 4), k = (e % (H / 4)) * 4;
    float4 v;
    if (!TRANS) {
      v = *reinterpret_cast<const float4*>(W + n * H + k);
    } else {
      v = make_float4(W[k * H + n], W[(k + 1) * H + n], W[(k + 2) * H + n], W[(k + 3) * H + n]);
    }
    put4(wh, wl, n, k, H, v);
  }
}

// Issue the 12 MMAs of one K-chunk: A planes (TM x KC, chunk-local), B planes
// resident (H x H) at K offset kc0.
template <int H>
__device__ __forceinline__ void issue_chunk(uint32_t taddr, const float* ah, const float* al,
                                            const float* bh, const float* bl, int kc0,
                                            bool first) {
  constexpr uint32_t LBO_A = (TM / 8) * 128, LBO_B = (H / 8) * 128;
  constexpr uint32_t idesc = tc::idesc_tf32(TM, H);
  const uint32_t a_hi = saddr(ah), a_lo = saddr(al), b_hi = saddr(bh), b_lo = saddr(bl);
#pragma unroll
  for (int s = 0; s < KC / 8; ++s) {
    const uint32_t qa = 2 * s * LBO_A, qb = (kc0 / 4 + 2 * s) * LBO_B;
    const uint64_t dah = tc::smem_desc(a_hi + qa, LBO_A, 128);
    const uint64_t dal = tc::smem_desc(a_lo + qa, LBO_A, 128);
    const uint64_t dbh = tc::smem_desc(b_hi + qb, LBO_B, 128);
    const uint64_t dbl = tc::smem_desc(b_lo + qb, LBO_B, 128);
    tc::mma_tf32(taddr, dal, dbh, idesc, (first && s == 0) ? 0u : 1u);
    tc::mma_tf32(taddr, dah, dbl, idesc, 1u);
    tc::mma_tf32(taddr, dah, dbh, idesc, 1u);
  }
}

struct TcShared {
  uint64_t bar_buf[2];
  uint64_t bar_acc;
  uint32_t tslot;
};

// One persistent GEMM over pixel tiles:  ACC[m][n] = sum_k Aop(m, k) B[n][k]
// with Aop(m, k) = SIN ? sin(w0 X[m][k]) : X[m][k], then the epilogue
// EPI(row m, columns c0..c0+31, values).
template <int H, bool SIN, bool TRANS_W, class Epi>
__device__ void gemm_tiles(const float* __restrict__ X, const float* __restrict__ W, int n,
                           float w0, Epi epi) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* wh = reinterpret_cast<float*>(smem);
  float* wl = wh + H * H;
  float* ah = wl + H * H;           // [2][TM * KC]
  float* al = ah + 2 * TM * KC;     // [2][TM * KC]
  __shared__ TcShared sh;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc<H>(&sh.tslot);
  if (tid == 0) {
    tc::mbar_init(&sh.bar_buf[0], 1);
    tc::mbar_init(&sh.bar_buf[1], 1);
    tc::mbar_init(&sh.bar_acc, 1);
    fence_mbar_init();
  }
  load_weights<H, TRANS_W>(W, wh, wl);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t taddr = sh.tslot;
  const int n_tiles = (n + TM - 1) / TM;
  uint32_t g = 0;          // chunks staged so far (buffer = g & 1)
  uint32_t acc_phase = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int m0 = tile * TM;
    const int row = m0 + tid;  // this thread stages and drains row `row`
    for (int kc0 = 0; kc0 < H; kc0 += KC, ++g) {
      const int b = g & 1;
      if (g >= 2) tc::mbar_wait(&sh.bar_buf[b], ((g - 2) >> 1) & 1);
      float* bh_ = ah + b * TM * KC;
      float* bl_ = al + b * TM * KC;
#pragma unroll
      for (int k = 0; k < KC; k += 4) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < n) {
          v = *reinterpret_cast<const float4*>(X + static_cast<size_t>(row) * H + kc0 + k);
          if (SIN) v = make_float4(sin_w(v.x, w0), sin_w(v.y, w0), sin_w(v.z, w0), sin_w(v.w, w0));
        }
        put4(bh_, bl_, tid, k, TM, v);
      }
      tc::fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
        issue_chunk<H>(taddr, bh_, bl_, wh, wl, kc0, kc0 == 0);
        tc::mma_commit(&sh.bar_buf[b]);
      }
    }
    if (tid == 0) tc::mma_commit(&sh.bar_acc);
    tc::mbar_wait(&sh.bar_acc, acc_phase);
    acc_phase ^= 1;
    tc::fence_after_sync();
#pragma unroll 1
    for (int c0 = 0; c0 < H; c0 += 32) {
      float v[32];
      tc::tmem_ld32(taddr + (static_cast<uint32_t>(32 * warp) << 16) + c0, v);
      if (row < n) epi(row, c0, v);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_free<H>(taddr);
}

// a_l[m][:] = W_l sin(w0 a_{l-1}[m][:]) + b_l
template <int H>
__global__ void __launch_bounds__(NTH, 1)
tc_fwd_kernel(const float* __restrict__ Ain, const float* __restrict__ W,
              const float* __restrict__ bias, int n, float w0, float* __restrict__ Aout) {
  gemm_tiles<H, true, false>(Ain, W, n, w0, [&](int m, int c0, const float (&v)[32]) {
    float* o = Aout + static_cast<size_t>(m) * H + c0;
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      *reinterpret_cast<float4*>(o + i) = make_float4(v[i] + bias[c0 + i], v[i + 1] + bias[c0 + i + 1],
                                                      v[i + 2] + bias[c0 + i + 2],
                                                      v[i + 3] + bias[c0 + i + 3]);
  });
}

// dA_{l-1}[m][k] = (sum_r dA_l[m][r] W_l[r][k]) w0 cos(w0 a_{l-1}[m][k])
template <int H>
__global__ void __launch_bounds__(NTH, 1)
tc_dgrad_kernel(const float* __restrict__ dAl, const float* __restrict__ W,
                const float* __restrict__ Aprev, int n, float w0, float* __restrict__ dAprev) {
  gemm_tiles<H, false, true>(dAl, W, n, w0, [&](int m, int c0, const float (&v)[32]) {
    const float* a = Aprev + static_cast<size_t>(m) * H + c0;
    float* o = dAprev + static_cast<size_t>(m) * H + c0;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      float4 x = *reinterpret_cast<const float4*>(a + i);
      *reinterpret_cast<float4*>(o + i) =
          make_float4(v[i] * dsin_w(x.x, w0), v[i + 1] * dsin_w(x.y, w0),
                      v[i + 2] * dsin_w(x.z, w0), v[i + 3] * dsin_w(x.w, w0));
    }
  });
}

// Split-M weight gradient: partial[chunk][r][k] = sum_{m in chunk} dA_l[m][r] sin(w0 a_{l-1}[m][k]),
// partial bias[chunk][r] = sum_m dA_l[m][r].  The GEMM's M is r (= H rows of
// TMEM), its N is k, its K is the pixel chunk.  Thread t owns r = t (H = 128)
// or r = t % 64 with two pixel halves (H = 64).
template <int H>
__global__ void __launch_bounds__(NTH, 1)
tc_wgrad_kernel(const float* __restrict__ dAl, const float* __restrict__ Aprev, int n, int rows,
                float w0, float* __restrict__ partial) {
  extern __shared__ __align__(1024) unsigned char smem[];
  // A planes: [2][TM=H-padded-to-128 rows r][KC pixels];  B planes: [2][H rows k][KC pixels]
  float* ah = reinterpret_cast<float*>(smem);
  float* al = ah + 2 * TM * KC;
  float* bh = al + 2 * TM * KC;
  float* bl = bh + 2 * H * KC;
  __shared__ TcShared sh;
  __shared__ float s_bias[2][H];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tc::tmem_alloc<H>(&sh.tslot);
  if (tid == 0) {
    tc::mbar_init(&sh.bar_buf[0], 1);
    tc::mbar_init(&sh.bar_buf[1], 1);
    tc::mbar_init(&sh.bar_acc, 1);
    fence_mbar_init();
  }
  // zero the A planes once: rows r >= H (H = 64) stay zero
  for (int e = tid; e < 4 * TM * KC; e += NTH) ah[e] = 0.f;
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t taddr = sh.tslot;
  constexpr uint32_t LBO_A = (TM / 8) * 128, LBO_B = (H / 8) * 128;
  constexpr uint32_t idesc = tc::idesc_tf32(TM, H);
  const int m_begin = blockIdx.x * rows, m_end = min(n, m_begin + rows);
  // thread -> (r or k index, pixel sub-range) for staging
  constexpr int GROUPS = NTH / H;      // 1 (H = 128) or 2 (H = 64)
  const int idx = tid % H, grp = tid / H;
  float bias_acc = 0.f;
  uint32_t g = 0;
  for (int p0 = m_begin; p0 < m_end; p0 += KC, ++g) {
    const int b = g & 1;
    if (g >= 2) tc::mbar_wait(&sh.bar_buf[b], ((g - 2) >> 1) & 1);
    float* ah_ = ah + b * TM * KC;
    float* al_ = al + b * TM * KC;
    float* bh_ = bh + b * H * KC;
    float* bl_ = bl + b * H * KC;
    // pixels p0 + [grp * KC/GROUPS, (grp+1) * KC/GROUPS), four at a time
#pragma unroll
    for (int q = grp * (KC / GROUPS); q < (grp + 1) * (KC / GROUPS); q += 4) {
      float4 da, z;
      float* dav = &da.x;
      float* zv = &z.x;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int m = p0 + q + u;
        float x = 0.f, y = 0.f;
        if (m < m_end) {
          x = dAl[static_cast<size_t>(m) * H + idx];
          y = sin_w(Aprev[static_cast<size_t>(m) * H + idx], w0);
        }
        dav[u] = x;
        zv[u] = y;
        bias_acc += x;
      }
      put4(ah_, al_, idx, q, TM, da);
      put4(bh_, bl_, idx, q, H, z);
    }
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after_sync();
      const uint32_t a_hi = saddr(ah_), a_lo = saddr(al_), b_hi = saddr(bh_), b_lo = saddr(bl_);
#pragma unroll
      for (int s = 0; s < KC / 8; ++s) {
        const uint32_t qa = 2 * s * LBO_A, qb = 2 * s * LBO_B;
        const uint64_t dah = tc::smem_desc(a_hi + qa, LBO_A, 128);
        const uint64_t dal = tc::smem_desc(a_lo + qa, LBO_A, 128);
        const uint64_t dbh = tc::smem_desc(b_hi + qb, LBO_B, 128);
        const uint64_t dbl = tc::smem_desc(b_lo + qb, LBO_B, 128);
        tc::mma_tf32(taddr, dal, dbh, idesc, (g == 0 && s == 0) ? 0u : 1u);
        tc::mma_tf32(taddr, dah, dbl, idesc, 1u);
        tc::mma_tf32(taddr, dah, dbh, idesc, 1u);
      }
      tc::mma_commit(&sh.bar_buf[b]);
    }
  }
  s_bias[grp][idx] = bias_acc;
  float* out = partial + static_cast<size_t>(blockIdx.x) * (static_cast<size_t>(H) * H + H);
  if (g > 0) {
    if (tid == 0) tc::mma_commit(&sh.bar_acc);
    tc::mbar_wait(&sh.bar_acc, 0);
    tc::fence_after_sync();
    // TMEM lane r holds row r of the (r x k) accumulator; rows >= H are padding
    const int r = 32 * warp + lane;
#pragma unroll 1
    for (int c0 = 0; c0 < H; c0 += 32) {
      float v[32];
      tc::tmem_ld32(taddr + (static_cast<uint32_t>(32 * warp) << 16) + c0, v);
      if (r < H) {
#pragma unroll
        for (int i = 0; i < 32; ++i) out[static_cast<size_t>(r) * H + c0 + i] = v[i];
      }
    }
  } else {
    for (int e = tid; e < H * H; e += NTH) out[e] = 0.f;
  }
  __syncthreads();
  if (tid < H) {
    float t = 0.f;
    for (int q = 0; q < GROUPS; ++q) t += s_bias[q][tid];
    out[static_cast<size_t>(H) * H + tid] = t;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<H>(taddr);
}

template <int H>
size_t gemm_smem() {
  return sizeof(float) * (2 * H * H + 4 * TM * KC);
}
template <int H>
size_t wgrad_smem() {
  return sizeof(float) * (4 * TM * KC + 4 * H * KC);
}

template <class K>
Status set_smem(K kernel, size_t bytes) {
  PACT_CUDA_S(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(bytes)));
  return {};
}

}  // namespace

bool siren_tc_supported(int hidden) { return hidden == 64 || hidden == 128; }

Status tc_forward_layer(pact_ctx* ctx, int H, const float* Ain, const float* W, const float* b,
                        int n, float w0, float* Aout) {
  const int tiles = (n + TM - 1) / TM;
  const int grid = std::max(1, std::min(tiles, ctx->num_sms));
  if (H == 128) {
    static bool cfg = false;
    if (!cfg) PACT_TRY_S(set_smem(tc_fwd_kernel<128>, gemm_smem<128>()));
    cfg = true;
    tc_fwd_kernel<128><<<grid, NTH, gemm_smem<128>(), ctx->stream>>>(Ain, W, b, n, w0, Aout);
  } else {
    static bool cfg = false;
    if (!cfg) PACT_TRY_S(set_smem(tc_fwd_kernel<64>, gemm_smem<64>()));
    cfg = true;
    tc_fwd_kernel<64><<<grid, NTH, gemm_smem<64>(), ctx->stream>>>(Ain, W, b, n, w0, Aout);
  }
  return after_launch(ctx, "tc_fwd_kernel");
}

Status tc_dgrad_layer(pact_ctx* ctx, int H, const float* dAl, const float* W, const float* Aprev,
                      int n, float w0, float* dAprev) {
  const int tiles = (n + TM - 1) / TM;
  const int grid = std::max(1, std::min(tiles, ctx->num_sms));
  if (H == 128) {
    static bool cfg = false;
    if (!cfg) PACT_TRY_S(set_smem(tc_dgrad_kernel<128>, gemm_smem<128>()));
    cfg = true;
    tc_dgrad_kernel<128><<<grid, NTH, gemm_smem<128>(), ctx->stream>>>(dAl, W, Aprev, n, w0, dAprev);
  } else {
    static bool cfg = false;
    if (!cfg) PACT_TRY_S(set_smem(tc_dgrad_kernel<64>, gemm_smem<64>()));
    cfg = true;
    tc_dgrad_kernel<64><<<grid, NTH, gemm_smem<64>(), ctx->stream>>>(dAl, W, Aprev, n, w0, dAprev);
  }
  return after_launch(ctx, "tc_dgrad_kernel");
}

// Returns the number of pixel chunks (partials) written.
Status tc_wgrad_layer(pact_ctx* ctx, int H, const float* dAl, const float* Aprev, int n, int rows,
                      float w0, float* partial, int n_chunks) {
  if (H == 128) {
    static bool cfg = false;
    if (!cfg) PACT_TRY_S(set_smem(tc_wgrad_kernel<128>, wgrad_smem<128>()));
    cfg = true;
    tc_wgrad_kernel<128><<<n_chunks, NTH, wgrad_smem<128>(), ctx->stream>>>(dAl, Aprev, n, rows, w0,
                                                                           partial);
  } else {
    static bool cfg = false;
    if (!cfg) PACT_TRY_S(set_smem(tc_wgrad_kernel<64>, wgrad_smem<64>()));
    cfg = true;
    tc_wgrad_kernel<64><<<n_chunks, NTH, wgrad_smem<64>(), ctx->stream>>>(dAl, Aprev, n, rows, w0,
                                                                         partial);
  }
  return after_launch(ctx, "tc_wgrad_kernel");
}

}  // namespace pactgpu
