// Throughput probe of tcgen05.mma kind::tf32 (M = 128): TS (A in TMEM) vs SS
// (A in shared memory), N = 64/128/256.  One CTA per SM, one elected thread
// issues `iters` MMAs back to back into one accumulator; CUDA events time it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2409_10876_b200/csrc scripts/tc_rate.cu -o build/tc_rate
#include <cstdio>

#include "tc.cuh"

using namespace pactgpu;

template <int N, bool TS>
__global__ void rate(int iters, float* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&tslot);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t t0 = tslot;
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  constexpr uint32_t idesc = tc::idesc_tf32(128, N);
  if (warp == 0 && tc::elect_one()) {
    for (int i = 0; i < iters; ++i) {
      const uint64_t db = tc::smem_desc_sw128(sa + 16384 + 32 * (i & 3));
      if (TS) {
        tc::mma_tf32_ts(t0 + 256, t0 + 8 * (i & 15), db, idesc, i != 0);
      } else {
        const uint64_t da = tc::smem_desc_sw128(sa + 32 * (i & 3));
        tc::mma_tf32(t0 + 256, da, db, idesc, i != 0);
      }
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  if (warp == 0) {
    float v[32];
    tc::tmem_ld32(t0 + 256, v);
    if (v[0] == 12345.f) sink[0] = v[1];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(t0);
}

template <int N, bool TS>
void run() {
  float* sink;
  cudaMalloc(&sink, 4);
  const int iters = 4096, smem = 64 * 1024;
  cudaFuncSetAttribute(rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rate<N, TS><<<148, 128, smem>>>(iters, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  rate<N, TS><<<148, 128, smem>>>(iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double flop = 2.0 * 128 * N * 8 * iters * 148;
  printf("%s N=%3d: %.3f ms, %.1f TFLOP/s (tf32), %.1f ns per MMA per SM\n", TS ? "TS" : "SS", N, ms,
         flop / (ms * 1e-3) / 1e12, ms * 1e6 / iters);
  cudaFree(sink);
}

int main() {
  run<16, true>();
  run<32, true>();
  run<64, true>();
  run<128, true>();
  run<256, true>();
  run<64, false>();
  run<128, false>();
  run<256, false>();
  return 0;
}
