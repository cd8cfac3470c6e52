// Probe 2 (+ SW128 variant) of the tcgen05 building blocks: A operand in TMEM (tcgen05.st from
// registers, lane = row), B staged with one cp.async.bulk into shared memory
// and re-laid out into K-major hi/lo planes; 3xTF32 via the TS form of
// tcgen05.mma.  C[128][N] = A[128][K] . B[N][K]^T against fp64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2409_10876_b200/csrc \
//        scripts/tc_probe2.cu -o build/tc_probe2 && build/tc_probe2
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "tc.cuh"

using namespace pactgpu;

template <int N, int K>
__global__ void probe(const float* A, const float* B, float* C) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* raw = reinterpret_cast<float*>(smem);  // [N][K]
  float* b_hi = raw + N * K;                    // K-major planes, full K
  float* b_lo = b_hi + N * K;
  __shared__ uint64_t bar_ld, bar_mma;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  // TMEM: A_hi [0,K), A_lo [K,2K), D [2K, 2K+N)
  constexpr int NC = 2 * K + N <= 256 ? 256 : 512;
  if (warp == 0) tc::tmem_alloc<NC>(&tslot);
  if (tid == 0) {
    tc::mbar_init(&bar_ld, 1);
    tc::mbar_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t t0 = tslot;
  if (tid == 0) {
    tc::mbar_expect_tx(&bar_ld, N * K * 4);
    tc::bulk_load(raw, B, N * K * 4, &bar_ld);
  }
  // A rows -> TMEM
  for (int k0 = 0; k0 < K; k0 += 32) {
    float hi[32], lo[32];
    for (int i = 0; i < 32; ++i) tc::split_tf32(A[tid * K + k0 + i], hi[i], lo[i]);
    const uint32_t lane_base = t0 + (static_cast<uint32_t>(32 * warp) << 16);
    tc::tmem_st32(lane_base + k0, hi);
    tc::tmem_st32(lane_base + K + k0, lo);
  }
  tc::mbar_wait(&bar_ld, 0);
  for (int e = tid; e < N * K / 4; e += 128) {
    const int n = e / (K / 4), k = (e % (K / 4)) * 4;
    float4 v = *reinterpret_cast<float4*>(raw + n * K + k);
    float4 h, l;
    tc::split_tf32(v.x, h.x, l.x);
    tc::split_tf32(v.y, h.y, l.y);
    tc::split_tf32(v.z, h.z, l.z);
    tc::split_tf32(v.w, h.w, l.w);
    const uint32_t o = tc::kmajor_offset(n, k, N) >> 2;
    *reinterpret_cast<float4*>(b_hi + o) = h;
    *reinterpret_cast<float4*>(b_lo + o) = l;
  }
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  constexpr uint32_t LBO = (N / 8) * 128;
  constexpr uint32_t idesc = tc::idesc_tf32(128, N);
  if (tid == 0) {
    const uint32_t sh = static_cast<uint32_t>(__cvta_generic_to_shared(b_hi));
    const uint32_t sl = static_cast<uint32_t>(__cvta_generic_to_shared(b_lo));
    const uint32_t d = t0 + 2 * K;
    for (int s = 0; s < K / 8; ++s) {
      const uint64_t bh = tc::smem_desc(sh + 2 * s * LBO, LBO, 128);
      const uint64_t bl = tc::smem_desc(sl + 2 * s * LBO, LBO, 128);
      tc::mma_tf32_ts(d, t0 + K + 8 * s, bh, idesc, s != 0);  // lo * hi
      tc::mma_tf32_ts(d, t0 + 8 * s, bl, idesc, 1);           // hi * lo
      tc::mma_tf32_ts(d, t0 + 8 * s, bh, idesc, 1);           // hi * hi
    }
    tc::mma_commit(&bar_mma);
  }
  tc::mbar_wait(&bar_mma, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(t0 + 2 * K + (static_cast<uint32_t>(32 * warp) << 16) + c0, v);
    for (int i = 0; i < 32; ++i) C[tid * N + c0 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<NC>(t0);
}

// B planes as SWIZZLE_128B K-major chunks of 32 (one 128-B row per n).
template <int N, int K>
__global__ void probe_sw(const float* A, const float* B, float* C) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* b_hi = reinterpret_cast<float*>(smem);  // [K/32][N][32]
  float* b_lo = b_hi + N * K;
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  constexpr int NC = 2 * K + N <= 256 ? 256 : 512;
  if (warp == 0) tc::tmem_alloc<NC>(&tslot);
  if (tid == 0) {
    tc::mbar_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t t0 = tslot;
  for (int k0 = 0; k0 < K; k0 += 32) {
    float hi[32], lo[32];
    for (int i = 0; i < 32; ++i) tc::split_tf32(A[tid * K + k0 + i], hi[i], lo[i]);
    const uint32_t lane_base = t0 + (static_cast<uint32_t>(32 * warp) << 16);
    tc::tmem_st32(lane_base + k0, hi);
    tc::tmem_st32(lane_base + K + k0, lo);
  }
  for (int e = tid; e < N * K / 4; e += 128) {
    const int n = e / (K / 4), k = (e % (K / 4)) * 4;
    float4 v = *reinterpret_cast<const float4*>(B + n * K + k);
    float4 h, l;
    tc::split_tf32(v.x, h.x, l.x);
    tc::split_tf32(v.y, h.y, l.y);
    tc::split_tf32(v.z, h.z, l.z);
    tc::split_tf32(v.w, h.w, l.w);
    const int chunk = k / 32, c = (k % 32) / 4;
    const int o = chunk * N * 32 + n * 32 + ((c ^ (n & 7)) * 4);
    *reinterpret_cast<float4*>(b_hi + o) = h;
    *reinterpret_cast<float4*>(b_lo + o) = l;
  }
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  constexpr uint32_t idesc = tc::idesc_tf32(128, N);
  if (tid == 0) {
    const uint32_t sh = static_cast<uint32_t>(__cvta_generic_to_shared(b_hi));
    const uint32_t sl = static_cast<uint32_t>(__cvta_generic_to_shared(b_lo));
    const uint32_t d = t0 + 2 * K;
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t off = (s / 4) * N * 128 + (s % 4) * 32;
      const uint64_t bh = tc::smem_desc_sw128(sh + off);
      const uint64_t bl = tc::smem_desc_sw128(sl + off);
      tc::mma_tf32_ts(d, t0 + K + 8 * s, bh, idesc, s != 0);
      tc::mma_tf32_ts(d, t0 + 8 * s, bl, idesc, 1);
      tc::mma_tf32_ts(d, t0 + 8 * s, bh, idesc, 1);
    }
    tc::mma_commit(&bar_mma);
  }
  tc::mbar_wait(&bar_mma, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(t0 + 2 * K + (static_cast<uint32_t>(32 * warp) << 16) + c0, v);
    for (int i = 0; i < 32; ++i) C[tid * N + c0 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<NC>(t0);
}

template <int N, int K>
int run() {
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<float> u(-1, 1);
  std::vector<float> A(128 * K), B(N * K), C(128 * N);
  for (auto& x : A) x = u(rng);
  for (auto& x : B) x = u(rng) * 0.01f;
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = 3 * N * K * 4;
  cudaFuncSetAttribute(probe<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaMemset(dC, 0, C.size() * 4);
  static int variant = 0;
  if (variant++ % 2 == 0) {
    probe<N, K><<<1, 128, smem>>>(dA, dB, dC);
  } else {
    const size_t sm2 = 2 * N * K * 4 + 1024;
    cudaFuncSetAttribute(probe_sw<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    probe_sw<N, K><<<1, 128, sm2>>>(dA, dB, dC);
    printf("[SW128] ");
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d K=%d launch error %s\n", N, K, cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  double num = 0, den = 0, numf = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      float f32 = 0;
      for (int k = 0; k < K; ++k) {
        ref += (double)A[m * K + k] * B[n * K + k];
        f32 = fmaf(A[m * K + k], B[n * K + k], f32);
      }
      num += (C[m * N + n] - ref) * (C[m * N + n] - ref);
      numf += (f32 - ref) * (f32 - ref);
      den += ref * ref;
    }
  double err = std::sqrt(num / den);
  printf("TS N=%d K=%d 3xTF32: rel L2 vs fp64 %.3e (fp32 FMA %.3e)\n", N, K, err,
         std::sqrt(numf / den));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  return err > 1e-5;
}

int main() {
  int bad = 0;
  for (int rep = 0; rep < 2; ++rep) bad += run<128, 128>() + run<64, 64>() + run<128, 32>();
  printf(bad ? "PROBE2 FAILED\n" : "PROBE2 OK\n");
  return bad;
}
