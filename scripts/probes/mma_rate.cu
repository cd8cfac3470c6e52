// Probe: tcgen05.mma issue-to-completion rate per SM for the shapes of the
// SIREN kernels (A from TMEM, B from SW128 shared memory), kind::tf32 (K = 8)
// and kind::f16 (K = 16), M = 128, N = 32 .. 256.  Garbage operands: timing only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2409_10876_b200/csrc \
//        scripts/probes/mma_rate.cu -o build/mma_rate && build/mma_rate
#include <cstdio>

#include "tc.cuh"

using namespace pactgpu;

__device__ float g_sink;

// LOAD: warps 1..15 stream 16-B shared loads over a 64 KB region while warp 0 issues
template <bool F16, int N, bool LOAD = false>
__global__ void rate(int iters, long long* cyc) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                       ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (LOAD ? 2 * 256 * 128 : 256 * 128) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 7);
  if (warp == 0) tc::tmem_alloc<512>(&tslot);
  if (tid == 0) {
    *reinterpret_cast<unsigned*>(sm + 65536 + 32768) = 0u;
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  tc::fence_proxy_async();
  const uint32_t t0 = tslot;
  if (warp == 0) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const uint64_t bd = tc::smem_desc_sw128(sa);
    constexpr uint32_t idesc = F16 ? tc::idesc_f16(128, N) : tc::idesc_tf32(128, N);
    long long c0 = clock64();
    if (tc::elect_one()) {
      for (int i = 0; i < iters; ++i) {
        if (F16)
          tc::mma_f16_ts(t0, t0 + 256 + 8 * (i & 3), bd + 2 * (i & 3), idesc, 1u);
        else
          tc::mma_tf32_ts(t0, t0 + 256 + 8 * (i & 3), bd + 2 * (i & 3), idesc, 1u);
      }
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, 0);
    long long c1 = clock64();
    if (tid == 0 && blockIdx.x == 0) *cyc = c1 - c0;
    if (LOAD && tid == 0) atomicExch(reinterpret_cast<unsigned*>(sm + 65536 + 32768), 1u);
  } else if (LOAD) {
    volatile unsigned* stop = reinterpret_cast<volatile unsigned*>(sm + 65536 + 32768);
    const float4* src = reinterpret_cast<const float4*>(sm + 32768);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int j = tid;
    while (*stop == 0u) {
#pragma unroll 8
      for (int u = 0; u < 32; ++u) {
        const float4 v = src[(j + u * 128) & 2047];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      j += 7;
    }
    if (acc.x == 12345.f) g_sink = acc.y + acc.z + acc.w;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(t0);
}

template <bool F16, int N, bool LOAD = false>
void run(long long* d) {
  const int smem = 256 * 128 * 4 + 1024;
  cudaFuncSetAttribute(rate<F16, N, LOAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int iters : {256, 4096}) {
    rate<F16, N, LOAD><<<148, LOAD ? 512 : 128, smem>>>(iters, d);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double macs = 128.0 * N * (F16 ? 16 : 8);
    std::printf("%s%s N=%3d iters=%5d: %7.1f clk/MMA  %7.0f MAC/clk\n", LOAD ? "+lds " : "", F16 ? "f16 " : "tf32", N, iters,
                double(c) / iters, macs * iters / double(c));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<false, 32>(d);
  run<false, 64>(d);
  run<false, 128>(d);
  run<false, 256>(d);
  run<true, 32>(d);
  run<true, 64>(d);
  run<true, 128>(d);
  run<true, 256>(d);
  run<false, 32, true>(d);
  run<false, 128, true>(d);
  run<true, 32, true>(d);
  run<true, 128, true>(d);
  std::printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
