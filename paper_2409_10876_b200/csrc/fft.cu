// Patch FFTs (part 3): forward 2-D FFT of every (patch, delay) window of the
// DAS stack (extract_patch_spectra, deconv.hpp:45-74) and inverse 2-D FFT of
// the deconvolved patch spectra (deconvolve_image, deconv.hpp:193-196), with
// the reference conventions (fft.hpp:86-115): forward e^{-i}, unscaled;
// inverse e^{+i}, scaled by 1/(w h); rows first, then columns.
//
// P = 64 and P = 128 run register-resident radix-4 transforms (below); other
// sizes one CTA per transform with the P x P complex tile in shared memory:
// power-of-two P an in-place radix-2 Cooley-Tukey with fp64-accurate fp32
// twiddles, other sizes the direct DFT like the reference.  The patch gather is fused into the load
// (no separate crop pass) and the inverse keeps only the real part.
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace pactgpu {
namespace {

__device__ __forceinline__ int bitrev(int x, int logn) { return __brev(x) >> (32 - logn); }

__device__ __forceinline__ float2 cm(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// In-place 2-D transform of buf[P][P] (row-major). sign = -1 forward, +1 inverse.
// tw[q] = exp(sign * 2 pi i q / P) for q < P.  scratch: P*P float2 (DFT path only).
__device__ void fft2d(float2* buf, float2* scratch, const float2* tw, int P, int logP) {
  const int P2 = P * P;
  const int nt = blockDim.x;
  if (logP >= 0) {
    // rows: bit-reverse within each row, then butterflies
    for (int pass = 0; pass < 2; ++pass) {
      // pass 0: rows (stride 1 within row, rows at stride P); pass 1: columns
      const int es = pass == 0 ? 1 : P, ls = pass == 0 ? P : 1;
      for (int e = threadIdx.x; e < P2; e += nt) {
        // consecutive threads -> consecutive addresses in both passes
        int line = pass == 0 ? e / P : e % P, i = pass == 0 ? e % P : e / P;
        int j = bitrev(i, logP);
        if (i < j) {
          float2* a = buf + line * ls + i * es;
          float2* b = buf + line * ls + j * es;
          float2 t = *a;
          *a = *b;
          *b = t;
        }
      }
      __syncthreads();
      for (int len = 2; len <= P; len <<= 1) {
        const int half = len >> 1, tstep = P / len;
        for (int e = threadIdx.x; e < P2 / 2; e += nt) {
          int line = pass == 0 ? e / (P / 2) : e % P;
          int bf = pass == 0 ? e % (P / 2) : e / P;
          int grp = bf / half, k = bf - grp * half;
          int i0 = grp * len + k;
          float2* base = buf + line * ls;
          float2 u = base[i0 * es];
          float2 v = cm(base[(i0 + half) * es], tw[k * tstep]);
          base[i0 * es] = make_float2(u.x + v.x, u.y + v.y);
          base[(i0 + half) * es] = make_float2(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
      }
    }
  } else {
    // direct DFT (fft.hpp:60-71), rows then columns
    for (int pass = 0; pass < 2; ++pass) {
      const int es = pass == 0 ? 1 : P, ls = pass == 0 ? P : 1;
      for (int e = threadIdx.x; e < P2; e += nt) {
        int line = pass == 0 ? e / P : e % P, k = pass == 0 ? e % P : e / P;
        const float2* src = buf + line * ls;
        float2 acc = make_float2(0.f, 0.f);
        for (int m = 0; m < P; ++m) {
          float2 p = cm(src[m * es], tw[(k * m) % P]);
          acc.x += p.x;
          acc.y += p.y;
        }
        scratch[line * ls + k * es] = acc;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < P2; e += nt) buf[e] = scratch[e];
      __syncthreads();
    }
  }
}

__device__ void make_twiddles(float2* tw, int P, double sign) {
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    double s, c;
    sincospi(sign * 2.0 * q / P, &s, &c);
    tw[q] = make_float2(static_cast<float>(c), static_cast<float>(s));
  }
}

// ---- register-resident radix-4 transforms (P = 64) -------------------------
// A 64-point DFT held in one thread's registers: three radix-4 DIF stages,
// fully unrolled, twiddles from a __constant__ table at compile-time indices
// (uniform reads: FFMA constant-bank operands), output in base-4
// digit-reversed register order (renamed away by rev4 at compile time).  A
// 2-D transform is 64 threads: column FFTs straight from the coalesced patch
// load, a padded shared-memory transpose, row FFTs, and a shared-memory pass
// so the complex output is stored coalesced.  No per-stage barriers.
__constant__ float2 c_tw64[64];  // exp(-2 pi i q / 64), fp64-accurate

__host__ __device__ constexpr int rev4_3(int k) {  // reverse 3 base-4 digits
  return ((k & 3) << 4) | (k & 12) | ((k >> 4) & 3);
}

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }  // -i a

// forward (e^{-i}) 64-point DFT in place; a[rev4_3(k)] = X[k] afterwards
__device__ __forceinline__ void fft64_regs(float2 (&a)[64]) {
#pragma unroll
  for (int L = 64; L >= 4; L >>= 2) {
    const int Q = L >> 2, stride = 64 / L;
#pragma unroll
    for (int base = 0; base < 64; base += L) {
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        const float2 x0 = a[base + j], x1 = a[base + j + Q], x2 = a[base + j + 2 * Q],
                     x3 = a[base + j + 3 * Q];
        const float2 t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3),
                     t3 = mul_mi(csub(x1, x3));
        a[base + j] = cadd(t0, t2);
        const float2 y1 = cadd(t1, t3), y2 = csub(t0, t2), y3 = csub(t1, t3);
        if (j == 0) {
          a[base + j + Q] = y1;
          a[base + j + 2 * Q] = y2;
          a[base + j + 3 * Q] = y3;
        } else {
          a[base + j + Q] = cm(y1, c_tw64[(stride * j) & 63]);
          a[base + j + 2 * Q] = cm(y2, c_tw64[(stride * 2 * j) & 63]);
          a[base + j + 3 * Q] = cm(y3, c_tw64[(stride * 3 * j) & 63]);
        }
      }
    }
  }
}

struct LayoutDev {
  int P, nx, ny, stride, last_x, last_y, W, H;
};

// patch_offsets_1d (core.hpp:232-241): offsets 0, s, 2s, ... then the clamped last
__device__ __forceinline__ int patch_offset(int i, int n, int stride, int last) {
  return i == n - 1 ? last : i * stride;
}

// Y[patch][j] = FFT2(stack[j][oy:oy+P, ox:ox+P])       grid (n_patches, K)
__global__ void patch_fft_kernel(LayoutDev L, const float* __restrict__ stack, int K, int logP,
                                 float2* __restrict__ Y, int p_lo, int row0, int rows) {
  extern __shared__ float2 sm[];
  const int P = L.P, P2 = P * P;
  float2* buf = sm;
  float2* tw = sm + P2;
  float2* scratch = tw + P;
  const int patch = p_lo + blockIdx.x, j = blockIdx.y;  // Y is indexed from p_lo
  const int px = patch % L.nx, py = patch / L.nx;
  const int ox = patch_offset(px, L.nx, L.stride, L.last_x);
  const int oy = patch_offset(py, L.ny, L.stride, L.last_y);
  make_twiddles(tw, P, -1.0);
  const float* img = stack + static_cast<size_t>(j) * L.W * rows;
  for (int e = threadIdx.x; e < P2; e += blockDim.x) {
    int y = e / P, x = e - y * P;
    buf[e] = make_float2(img[static_cast<size_t>(oy + y - row0) * L.W + ox + x], 0.f);
  }
  __syncthreads();
  fft2d(buf, scratch, tw, P, logP);
  float2* out = Y + (static_cast<size_t>(blockIdx.x) * K + j) * P2;
  for (int e = threadIdx.x; e < P2; e += blockDim.x) out[e] = buf[e];
}

// Y[patch][j] = FFT2(stack[j][oy:oy+P, ox:ox+P]) for P = 64, 64 threads per
// transform (thread c: column c, then row c).                 grid (n_patches, K)
__global__ void __launch_bounds__(64) patch_fft64_kernel(LayoutDev L, const float* __restrict__ stack,
                                                         int K, float2* __restrict__ Y, int p_lo,
                                                         int row0, int rows) {
  __shared__ float2 s[64][65];
  const int c = threadIdx.x;
  const int patch = p_lo + blockIdx.x, j = blockIdx.y;
  const int px = patch % L.nx, py = patch / L.nx;
  const int ox = patch_offset(px, L.nx, L.stride, L.last_x);
  const int oy = patch_offset(py, L.ny, L.stride, L.last_y);
  const float* img = stack + static_cast<size_t>(j) * L.W * rows +
                     static_cast<size_t>(oy - row0) * L.W + ox + c;
  float2 a[64];
#pragma unroll
  for (int y = 0; y < 64; ++y) a[y] = make_float2(__ldcs(img + static_cast<size_t>(y) * L.W), 0.f);
  fft64_regs(a);  // columns: a[rev(ky)] = Z[ky][c]
#pragma unroll
  for (int ky = 0; ky < 64; ++ky) s[ky][c] = a[rev4_3(ky)];
  __syncthreads();
#pragma unroll
  for (int kx = 0; kx < 64; ++kx) a[kx] = s[c][kx];  // row ky = c
  fft64_regs(a);  // rows: a[rev(kx)] = Y[c][kx]
  __syncthreads();
#pragma unroll
  for (int kx = 0; kx < 64; ++kx) s[c][kx] = a[rev4_3(kx)];
  __syncthreads();
  float2* out = Y + (static_cast<size_t>(blockIdx.x) * K + j) * 4096 + c;
#pragma unroll
  for (int ky = 0; ky < 64; ++ky) __stcs(out + ky * 64, s[ky][c]);
}

// out[patch] = Re(IFFT2(X[patch])) / 64^2 = Re(FFT2(conj X)) / 64^2 (the
// reference's inverse_2d, fft.hpp:107-115, real part kept), P = 64.
__global__ void __launch_bounds__(64) patch_ifft64_real_kernel(const float2* __restrict__ X,
                                                               float* __restrict__ out) {
  __shared__ float2 s[64][65];
  const int c = threadIdx.x;
  const float2* x = X + static_cast<size_t>(blockIdx.x) * 4096 + c;
  float2 a[64];
#pragma unroll
  for (int y = 0; y < 64; ++y) {
    const float2 v = x[y * 64];
    a[y] = make_float2(v.x, -v.y);
  }
  fft64_regs(a);
#pragma unroll
  for (int ky = 0; ky < 64; ++ky) s[ky][c] = a[rev4_3(ky)];
  __syncthreads();
#pragma unroll
  for (int kx = 0; kx < 64; ++kx) a[kx] = s[c][kx];
  fft64_regs(a);
  __syncthreads();
  float* sr = reinterpret_cast<float*>(&s[0][0]);  // [64][65] real plane
#pragma unroll
  for (int kx = 0; kx < 64; ++kx) sr[c * 65 + kx] = a[rev4_3(kx)].x;
  __syncthreads();
  float* o = out + static_cast<size_t>(blockIdx.x) * 4096 + c;
  const float inv = 1.f / 4096.f;
#pragma unroll
  for (int y = 0; y < 64; ++y) o[y * 64] = sr[y * 65 + c] * inv;
}

// ---- P = 128: two threads per 128-point line (radix-2 over the 64-point
// register DFT) ------------------------------------------------------------
// X[k] = E[k] + w^k O[k], X[k + 64] = E[k] - w^k O[k] with E, O the 64-point
// DFTs of the even / odd samples (w = exp(-2 pi i / 128)).  Thread (line,
// h) transforms the samples of parity h in registers (fft64_regs), takes its
// partner's result (lane ^ 16) by shuffles and keeps output half h.  A 2-D
// transform is 256 threads (warp w: lines 16 w .. 16 w + 15): columns
// straight from the coalesced load, a padded shared-memory transpose, rows,
// and a shared-memory pass for coalesced stores.  132 KB of shared memory
// (the [128][129] tile), one transform per CTA.
__constant__ float2 c_tw128[64];  // exp(-2 pi i q / 128), q < 64

// a[] holds this thread's 64-point DFT (digit-reversed order); on return
// a[k] (natural order, k < 64) = X[k + 64 h] of the 128-point line.
__device__ __forceinline__ void combine128(float2 (&a)[64], int h) {
  float2 o[64];
#pragma unroll
  for (int k = 0; k < 64; ++k) {
    const float2 own = a[rev4_3(k)];
    const float2 other = make_float2(__shfl_xor_sync(0xffffffffu, own.x, 16),
                                     __shfl_xor_sync(0xffffffffu, own.y, 16));
    const float2 e = h ? other : own, od = h ? own : other;
    const float2 t = cm(od, c_tw128[k]);
    o[k] = h ? csub(e, t) : cadd(e, t);
  }
#pragma unroll
  for (int k = 0; k < 64; ++k) a[k] = o[k];
}

constexpr int kP128Pad = 129;

// FWD: Y[patch][j] = FFT2(stack[j][oy:oy+128, ox:ox+128])    grid (n_patches, K)
// !FWD: out[patch] = Re(IFFT2(X[patch])) / 128^2 = Re(FFT2(conj X)) / 128^2
template <bool FWD>
__global__ void __launch_bounds__(256) patch_fft128_kernel(LayoutDev L, const float* __restrict__ stack,
                                                           int K, float2* __restrict__ Y, int p_lo,
                                                           int row0, int rows,
                                                           const float2* __restrict__ X,
                                                           float* __restrict__ out) {
  extern __shared__ float2 s128[];  // [128][kP128Pad]
  const int lane = threadIdx.x & 31, h = lane >> 4;
  const int line = (threadIdx.x >> 5) * 16 + (lane & 15);
  float2 a[64];
  if (FWD) {
    const int patch = p_lo + blockIdx.x, j = blockIdx.y;
    const int px = patch % L.nx, py = patch / L.nx;
    const int ox = patch_offset(px, L.nx, L.stride, L.last_x);
    const int oy = patch_offset(py, L.ny, L.stride, L.last_y);
    const float* img = stack + static_cast<size_t>(j) * L.W * rows +
                       static_cast<size_t>(oy - row0 + h) * L.W + ox + line;
#pragma unroll
    for (int y = 0; y < 64; ++y) a[y] = make_float2(__ldcs(img + static_cast<size_t>(2 * y) * L.W), 0.f);
  } else {
    const float2* x = X + static_cast<size_t>(blockIdx.x) * 16384 + h * 128 + line;
#pragma unroll
    for (int y = 0; y < 64; ++y) {
      const float2 v = x[y * 256];
      a[y] = make_float2(v.x, -v.y);
    }
  }
  fft64_regs(a);
  combine128(a, h);  // column `line`: a[k] = Z[k + 64 h][line]
#pragma unroll
  for (int k = 0; k < 64; ++k) s128[(k + 64 * h) * kP128Pad + line] = a[k];
  __syncthreads();
#pragma unroll
  for (int x = 0; x < 64; ++x) a[x] = s128[line * kP128Pad + 2 * x + h];  // row `line`, parity h
  fft64_regs(a);
  combine128(a, h);  // row `line`: a[k] = Y[line][k + 64 h]
  __syncthreads();
  if (FWD) {
#pragma unroll
    for (int k = 0; k < 64; ++k) s128[line * kP128Pad + k + 64 * h] = a[k];
    __syncthreads();
    float2* o = Y + (static_cast<size_t>(blockIdx.x) * K + blockIdx.y) * 16384;
#pragma unroll 8
    for (int q = 0; q < 64; ++q) {
      const int e = q * 256 + threadIdx.x;
      __stcs(o + e, s128[(e >> 7) * kP128Pad + (e & 127)]);
    }
  } else {
    float* sr = reinterpret_cast<float*>(s128);  // [128][kP128Pad] real plane
#pragma unroll
    for (int k = 0; k < 64; ++k) sr[line * kP128Pad + k + 64 * h] = a[k].x;
    __syncthreads();
    float* o = out + static_cast<size_t>(blockIdx.x) * 16384;
    const float inv = 1.f / 16384.f;
#pragma unroll 8
    for (int q = 0; q < 64; ++q) {
      const int e = q * 256 + threadIdx.x;
      o[e] = sr[(e >> 7) * kP128Pad + (e & 127)] * inv;
    }
  }
}

// out[patch][P2] = Re(IFFT2(X[patch])) / (P*P)           grid (n_patches)
__global__ void patch_ifft_real_kernel(int P, int logP, const float2* __restrict__ X,
                                       float* __restrict__ out) {
  extern __shared__ float2 sm[];
  const int P2 = P * P;
  float2* buf = sm;
  float2* tw = sm + P2;
  float2* scratch = tw + P;
  make_twiddles(tw, P, +1.0);
  const float2* src = X + static_cast<size_t>(blockIdx.x) * P2;
  for (int e = threadIdx.x; e < P2; e += blockDim.x) buf[e] = src[e];
  __syncthreads();
  fft2d(buf, scratch, tw, P, logP);
  const float inv = 1.f / static_cast<float>(P2);
  float* o = out + static_cast<size_t>(blockIdx.x) * P2;
  for (int e = threadIdx.x; e < P2; e += blockDim.x) o[e] = buf[e].x * inv;
}

// merge_patches (deconv.hpp:142-164) in gather form: every pixel sums the
// windowed values of the (<= 3x3) patches covering it in layout order.
// patches holds the patches [p_lo, p_hi) (indexed from p_lo); with num/den set
// the kernel writes the accumulators sum w x, sum w of those patches instead
// of the image (a partitioned merge, reduced across ranks by the caller).
__global__ void merge_kernel(LayoutDev L, const float* __restrict__ patches,
                             const float* __restrict__ win, float* __restrict__ img, int p_lo,
                             int p_hi, float* __restrict__ num, float* __restrict__ den) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.W * L.H) return;
  int y = i / L.W, x = i - y * L.W;
  const int P = L.P;
  float acc = 0.f, ws = 0.f;
  // Patches covering (x, y), ascending index per axis (= the reference's
  // row-major accumulation order): offsets i*s for i < n-1, then the last.
  const int ylo = y - P + 1 <= 0 ? 0 : (y - P + 1 + L.stride - 1) / L.stride;
  const int yhi = min(y / L.stride, L.ny - 2);
  const int xlo = x - P + 1 <= 0 ? 0 : (x - P + 1 + L.stride - 1) / L.stride;
  const int xhi = min(x / L.stride, L.nx - 2);
  const bool ylast = L.last_y <= y && y < L.last_y + P;
  const bool xlast = L.last_x <= x && x < L.last_x + P;
  for (int py = min(ylo, yhi + 1); py <= yhi + 1; ++py) {
    if (py == yhi + 1) {
      if (!ylast) break;
      py = L.ny - 1;
    }
    const int oy = patch_offset(py, L.ny, L.stride, L.last_y);
    for (int px = min(xlo, xhi + 1); px <= xhi + 1; ++px) {
      if (px == xhi + 1) {
        if (!xlast) break;
        px = L.nx - 1;
      }
      const int ox = patch_offset(px, L.nx, L.stride, L.last_x);
      const int pi = py * L.nx + px;
      if (pi < p_lo || pi >= p_hi) continue;
      const int q = (y - oy) * P + (x - ox);
      const float w = win[q];
      acc += w * patches[static_cast<size_t>(pi - p_lo) * P * P + q];
      ws += w;
    }
  }
  if (num) {
    num[i] = acc;
    den[i] = ws;
  } else {
    img[i] = ws > 0.f ? acc / ws : 0.f;
  }
}

int ilog2_exact(int P) {
  int l = 0;
  while ((1 << l) < P) ++l;
  return (1 << l) == P ? l : -1;
}

size_t fft_smem(int P, int logP) {
  size_t P2 = static_cast<size_t>(P) * P;
  return sizeof(float2) * (P2 + P + (logP >= 0 ? 0 : P2));
}

LayoutDev layout_dev(const pact_layout& l) {
  LayoutDev d;
  d.P = l.patch_pixels;
  d.nx = l.nx;
  d.ny = l.ny;
  d.stride = l.stride_pixels;
  d.last_x = l.last_x;
  d.last_y = l.last_y;
  d.W = l.grid.width;
  d.H = l.grid.height;
  return d;
}

// c_tw64 / c_tw128 once per device (the constant bank is per device context)
Status twiddles64() {
  int dev = 0;
  PACT_CUDA_S(cudaGetDevice(&dev));
  static std::once_flag once[64];
  static cudaError_t err[64];
  std::call_once(once[dev & 63], [dev] {
    float2 tw[64], tw2[64];
    for (int q = 0; q < 64; ++q) {
      const double ang = -2.0 * M_PI * q / 64.0, ang2 = -2.0 * M_PI * q / 128.0;
      tw[q] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
      tw2[q] = make_float2(static_cast<float>(std::cos(ang2)), static_cast<float>(std::sin(ang2)));
    }
    err[dev & 63] = cudaMemcpyToSymbol(c_tw64, tw, sizeof(tw));
    if (err[dev & 63] == cudaSuccess) err[dev & 63] = cudaMemcpyToSymbol(c_tw128, tw2, sizeof(tw2));
  });
  return cuda_status(err[dev & 63], "cudaMemcpyToSymbol(c_tw64)");
}

constexpr size_t kSmem128 = sizeof(float2) * 128 * kP128Pad;

bool fft64_enabled() {
  static const bool off = [] {  // PACT_FFT_SMEM=1: the shared-memory radix-2 kernels
    const char* e = std::getenv("PACT_FFT_SMEM");
    return e && e[0] == '1';
  }();
  return !off;
}

}  // namespace

Status launch_patch_fft(pact_ctx* ctx, const pact_layout& lay, const float* stack, int K,
                        float2* Y, int p_lo, int p_hi, int row0, int stack_rows) {
  if (p_hi < 0) p_hi = lay.nx * lay.ny;
  if (stack_rows < 0) stack_rows = lay.grid.height - row0;
  if (lay.patch_pixels == 64 && fft64_enabled()) {
    PACT_TRY_S(twiddles64());
    if (p_hi <= p_lo) return {};
    patch_fft64_kernel<<<dim3(p_hi - p_lo, K), 64, 0, ctx->stream>>>(layout_dev(lay), stack, K, Y,
                                                                     p_lo, row0, stack_rows);
    return after_launch(ctx, "patch_fft64_kernel");
  }
  if (lay.patch_pixels == 128 && fft64_enabled()) {
    PACT_TRY_S(twiddles64());
    PACT_TRY_S(smem_optin(patch_fft128_kernel<true>, kSmem128));
    if (p_hi <= p_lo) return {};
    patch_fft128_kernel<true><<<dim3(p_hi - p_lo, K), 256, kSmem128, ctx->stream>>>(
        layout_dev(lay), stack, K, Y, p_lo, row0, stack_rows, nullptr, nullptr);
    return after_launch(ctx, "patch_fft128_kernel");
  }
  const int P = lay.patch_pixels, logP = ilog2_exact(P);
  size_t smem = fft_smem(P, logP);
  if (smem > 220 * 1024) return validation("extract_patch_spectra: patch too large for the device FFT");
  PACT_TRY_S(smem_optin(patch_fft_kernel, smem));
  if (p_hi <= p_lo) return {};
  dim3 g(p_hi - p_lo, K);
  patch_fft_kernel<<<g, 512, smem, ctx->stream>>>(layout_dev(lay), stack, K, logP, Y, p_lo, row0,
                                                   stack_rows);
  return after_launch(ctx, "patch_fft_kernel");
}

Status launch_patch_ifft_real(pact_ctx* ctx, int P, int n_patches, const float2* X, float* out) {
  if (P == 64 && fft64_enabled()) {
    PACT_TRY_S(twiddles64());
    patch_ifft64_real_kernel<<<n_patches, 64, 0, ctx->stream>>>(X, out);
    return after_launch(ctx, "patch_ifft64_real_kernel");
  }
  if (P == 128 && fft64_enabled()) {
    PACT_TRY_S(twiddles64());
    PACT_TRY_S(smem_optin(patch_fft128_kernel<false>, kSmem128));
    patch_fft128_kernel<false><<<n_patches, 256, kSmem128, ctx->stream>>>(LayoutDev{}, nullptr, 0,
                                                                          nullptr, 0, 0, 0, X, out);
    return after_launch(ctx, "patch_fft128_kernel");
  }
  const int logP = ilog2_exact(P);
  size_t smem = fft_smem(P, logP);
  PACT_TRY_S(smem_optin(patch_ifft_real_kernel, smem));
  patch_ifft_real_kernel<<<n_patches, 512, smem, ctx->stream>>>(P, logP, X, out);
  return after_launch(ctx, "patch_ifft_real_kernel");
}

Status launch_merge(pact_ctx* ctx, const pact_layout& lay, const float* patches, const float* win,
                    float* img) {
  int n = lay.grid.width * lay.grid.height;
  merge_kernel<<<div_up(n, 256), 256, 0, ctx->stream>>>(layout_dev(lay), patches, win, img, 0,
                                                         lay.nx * lay.ny, nullptr, nullptr);
  return after_launch(ctx, "merge_kernel");
}

Status launch_merge_partial(pact_ctx* ctx, const pact_layout& lay, const float* patches,
                            const float* win, int p_lo, int p_hi, float* num, float* den) {
  int n = lay.grid.width * lay.grid.height;
  merge_kernel<<<div_up(n, 256), 256, 0, ctx->stream>>>(layout_dev(lay), patches, win, nullptr,
                                                         p_lo, p_hi, num, den);
  return after_launch(ctx, "merge_kernel");
}

}  // namespace pactgpu
