// Probe: tcgen05.mma kind::f16 with A MN-major (SWIZZLE_128B), as the fused
// backward's dA planes would feed the weight gradient: A[m][k] stored row = k
// (pixel), 64 consecutive m (feature) per 128-B row, two 64-m chunks of 32 rows.
// B K-major (row = n, 32 K per 64-B half row, as the z planes).  Candidate
// LBO / SBO assignments are compared with a host reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2409_10876_b200/csrc \
//        scripts/probes/f16_mn_probe.cu -o build/f16_mn_probe && build/f16_mn_probe
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "tc.cuh"

using namespace pactgpu;

constexpr int M = 128, N = 128, K = 32;

__device__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__global__ void probe(const __half* A, const __half* B, float* C, int nvar) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = tc::smem_align1024<unsigned char>(smem_raw);
  __half* amn = reinterpret_cast<__half*>(sm);          // [2 chunks][32 k][64 m] SW128
  __half* bk = reinterpret_cast<__half*>(sm + 8192);     // [128 n][32 k] + pad to 128-B rows
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&tslot);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = tid; e < M * K; e += 128) {
    const int k = e / M, m = e % M;  // A[m][k] given as A[k * M + m]
    const int c = m / 64, mm = m % 64;
    // 16-B granule mm / 8 XOR k % 8 of row k
    const int o = c * (32 * 64) + k * 64 + (((mm >> 3) ^ (k & 7)) << 3) + (mm & 7);
    amn[o] = A[e];
  }
  for (int e = tid; e < N * K; e += 128) {
    const int n = e / K, k = e % K;  // B[n][k]
    const int o = n * 64 + ((((k >> 3) ^ (n & 7))) << 3) + (k & 7);
    bk[o] = B[e];
  }
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t t0 = tslot;
  if (tid == 0) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(amn));
    const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(bk));
    const uint32_t id_k = tc::idesc_f16(M, N);
    const uint32_t id_amn = id_k | (1u << 15);
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t bd = tc::smem_desc_sw128(sb + 32 * s);
      // K step s = 16 rows of A = two 8-row atoms: start + 2048 s
      tc::mma_f16(t0 + 0, desc(sa + 2048 * s, 4096, 1024), bd, id_amn, s != 0);
      tc::mma_f16(t0 + 128, desc(sa + 2048 * s, 1024, 4096), bd, id_amn, s != 0);
      tc::mma_f16(t0 + 256, desc(sa + 2048 * s, 4096, 2048), bd, id_amn, s != 0);
      tc::mma_f16(t0 + 384, desc(sa + 2048 * s, 2048, 4096), bd, id_amn, s != 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  const uint32_t lb = t0 + (static_cast<uint32_t>(32 * warp) << 16);
  for (int v = 0; v < nvar; ++v)
    for (int c0 = 0; c0 < N; c0 += 32) {
      float r[32];
      tc::tmem_ld32(lb + 128 * v + c0, r);
      for (int j = 0; j < 32; ++j) C[(v * M + tid) * N + c0 + j] = r[j];
    }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(t0);
}

int main() {
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<__half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K);
  for (int i = 0; i < M * K; ++i) {
    A[i] = __float2half(U(rng));
    Af[i] = __half2float(A[i]);
  }
  for (int i = 0; i < N * K; ++i) {
    B[i] = __float2half(U(rng));
    Bf[i] = __half2float(B[i]);
  }
  __half *dA, *dB;
  float* dC;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dC, 4 * M * N * 4);
  cudaMemset(dC, 0, 4 * M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 8192 + 128 * 128 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dA, dB, dC, 4);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> C(4 * M * N);
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  for (int v = 0; v < 4; ++v) {
    double num = 0, den = 0, mx = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += double(Af[k * M + m]) * Bf[n * K + k];
        const double g = C[(v * M + m) * N + n];
        num += (g - r) * (g - r);
        den += r * r;
        mx = std::fmax(mx, std::fabs(g));
      }
    printf("variant %d: rel L2 %.3e  max|C| %.3e\n", v, std::sqrt(num / den), mx);
  }
  return 0;
}
