// Probe: tcgen05.mma kind::tf32 with both operands MN-major (SWIZZLE_128B)
// against a K-major control.  C[m][n] = sum_k A[k][m] B[k][n], M = N = 128,
// K = 32 (data stored row = k, as the fused backward's pixel-row planes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2409_10876_b200/csrc \
//        scripts/tc_probe_mn.cu -o build/tc_probe_mn -lcuda && build/tc_probe_mn
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "tc.cuh"

using namespace pactgpu;

constexpr int M = 128, N = 128, K = 32;

__device__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__global__ void probe(const float* A, const float* B, float* C, int nvar) {
  extern __shared__ unsigned char smem_raw[];
  float* sm = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* amn = sm;             // [4 chunks of m][32 k][32 m]
  float* bmn = amn + M * K;    // [4 chunks of n][32 k][32 n]
  float* ak = bmn + N * K;     // [128 m][32 k] K-major
  float* bk = ak + M * K;      // [128 n][32 k]
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&tslot);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = tid; e < M * K; e += 128) {
    const int k = e / M, m = e % M;  // A[k][m]
    const float va = A[e], vb = B[e];
    const int c = m / 32, mm = m % 32;
    const int omn = c * 1024 + k * 32 + (((mm >> 2) ^ (k & 7)) << 2) + (mm & 3);
    amn[omn] = va;
    bmn[omn] = vb;
    const int ok = m * 32 + (((k >> 2) ^ (m & 7)) << 2) + (k & 3);
    ak[ok] = va;
    bk[ok] = vb;
  }
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t t0 = tslot;
  if (tid == 0) {
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const uint32_t samn = base, sbmn = base + 4 * M * K, sak = base + 8 * M * K, sbk = base + 12 * M * K;
    const uint32_t id_k = tc::idesc_tf32(M, N);
    const uint32_t id_mn = id_k | (1u << 15) | (1u << 16);
    for (int s = 0; s < K / 8; ++s) {
      // variant 0: MN-major, LBO = MN atom stride (4096), SBO = 1024
      tc::mma_tf32(t0 + 0, desc_mn(samn + 1024 * s, 4096, 1024), desc_mn(sbmn + 1024 * s, 4096, 1024), id_mn, s != 0);
      // variant 1: MN-major with LBO / SBO swapped
      tc::mma_tf32(t0 + 128, desc_mn(samn + 1024 * s, 1024, 4096), desc_mn(sbmn + 1024 * s, 1024, 4096), id_mn, s != 0);
      // variant 2: K-major control
      tc::mma_tf32(t0 + 256, tc::smem_desc_sw128(sak + 32 * s), tc::smem_desc_sw128(sbk + 32 * s), id_k, s != 0);
      // variant 3: MN-major data, but MN bits in the other order (A only MN)
      tc::mma_tf32(t0 + 384, desc_mn(samn + 1024 * s, 4096, 1024), tc::smem_desc_sw128(sbk + 32 * s), id_k | (1u << 15), s != 0);
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
  std::vector<float> A(M * K), B(N * K);
  for (auto& x : A) x = U(rng);
  for (auto& x : B) x = U(rng);
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dC, 4 * M * N * 4);
  cudaMemset(dC, 0, 4 * M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 4 * M * K * 4 + 1024;
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
        for (int k = 0; k < K; ++k) r += double(A[k * M + m]) * B[k * N + n];
        // variant 3: A MN-major (A[k][m]), B K-major from bk (bk holds B[k][n] at row n) -> same product
        const double g = C[(v * M + m) * N + n];
        num += (g - r) * (g - r);
        den += r * r;
        mx = std::fmax(mx, std::fabs(g));
      }
    printf("variant %d: rel L2 %.3e  max|C| %.3e\n", v, std::sqrt(num / den), mx);
  }
  return 0;
}
