// Probe of the tcgen05 building blocks (paper_2409_10876_b200/csrc/tc.cuh):
// C[M=128][N] = A[128][K] . B[N][K]^T with kind::tf32, 1xTF32 and 3xTF32,
// against an fp64 host reference.  Build on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2409_10876_b200/csrc \
//        scripts/tc_probe.cu -o build/tc_probe && build/tc_probe
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "tc.cuh"

using namespace pactgpu;

template <int N>
__global__ void probe(const float* A, const float* B, float* C, int K, int three) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* a_hi = reinterpret_cast<float*>(smem);
  float* a_lo = a_hi + 128 * 32;
  float* b_hi = a_lo + 128 * 32;
  float* b_lo = b_hi + N * 32;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NC = N < 32 ? 32 : N;
  if (warp == 0) tc::tmem_alloc<NC>(&tslot);
  if (tid == 0) tc::mbar_init(&bar, 1);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t taddr = tslot;
  constexpr uint32_t LBO_A = (128 / 8) * 128, LBO_B = (N / 8) * 128;
  constexpr uint32_t idesc = tc::idesc_tf32(128, N);
  uint32_t phase = 0;
  for (int kc = 0; kc < K / 32; ++kc) {
    for (int k = 0; k < 32; ++k) {
      float hi, lo;
      tc::split_tf32(A[tid * K + kc * 32 + k], hi, lo);
      if (!three) hi = A[tid * K + kc * 32 + k];  // plain TF32: hardware truncation
      uint32_t o = tc::kmajor_offset(tid, k, 128) / 4;
      a_hi[o] = hi;
      a_lo[o] = lo;
    }
    for (int n = tid; n < N; n += 128)
      for (int k = 0; k < 32; ++k) {
        float hi, lo;
        tc::split_tf32(B[n * K + kc * 32 + k], hi, lo);
        if (!three) hi = B[n * K + kc * 32 + k];
        uint32_t o = tc::kmajor_offset(n, k, N) / 4;
        b_hi[o] = hi;
        b_lo[o] = lo;
      }
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after_sync();
      const uint32_t sa_hi = static_cast<uint32_t>(__cvta_generic_to_shared(a_hi));
      const uint32_t sa_lo = static_cast<uint32_t>(__cvta_generic_to_shared(a_lo));
      const uint32_t sb_hi = static_cast<uint32_t>(__cvta_generic_to_shared(b_hi));
      const uint32_t sb_lo = static_cast<uint32_t>(__cvta_generic_to_shared(b_lo));
      for (int s = 0; s < 4; ++s) {
        uint64_t ah = tc::smem_desc(sa_hi + 2 * s * LBO_A, LBO_A, 128);
        uint64_t al = tc::smem_desc(sa_lo + 2 * s * LBO_A, LBO_A, 128);
        uint64_t bh = tc::smem_desc(sb_hi + 2 * s * LBO_B, LBO_B, 128);
        uint64_t bl = tc::smem_desc(sb_lo + 2 * s * LBO_B, LBO_B, 128);
        uint32_t acc = (kc | s) != 0;
        tc::mma_tf32(taddr, ah, bh, idesc, acc);
        if (three) {
          tc::mma_tf32(taddr, ah, bl, idesc, 1);
          tc::mma_tf32(taddr, al, bh, idesc, 1);
        }
      }
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
  }
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(taddr + (static_cast<uint32_t>(32 * warp) << 16) + c0, v);
    int row = 32 * warp + lane;
    for (int i = 0; i < 32; ++i) C[row * N + c0 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<NC>(taddr);
}

template <int N>
int run(int K) {
  std::mt19937_64 rng(1);
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
  size_t smem = (2 * 128 * 32 + 2 * N * 32) * 4;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bad = 0;
  for (int three = 0; three < 2; ++three) {
    cudaMemset(dC, 0, C.size() * 4);
    probe<N><<<1, 128, smem>>>(dA, dB, dC, K, three);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("N=%d launch error %s\n", N, cudaGetErrorString(e));
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
    printf("N=%d K=%d %s: rel L2 vs fp64 %.3e (fp32 FMA reference %.3e)\n", N, K,
           three ? "3xTF32" : "1xTF32", err, std::sqrt(numf / den));
    if (three && err > 1e-5) bad = 1;
    if (!three && err > 1e-2) bad = 1;
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  return bad;
}

int main() {
  int bad = run<128>(128) + run<64>(64) + run<256>(128);
  printf(bad ? "PROBE FAILED\n" : "PROBE OK\n");
  return bad;
}
