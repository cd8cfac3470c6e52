// Microbenchmark: L2 reduction (RED) throughput on B200 for the ray adjoint's
// scatter pattern — each lane of a warp walks its own "ray" through a 2-MB
// raster, depositing into the pixel it is on (scattered across lanes,
// sequential per lane).  Compares RED.F64, RED.U64 (fixed point), RED.F32,
// RED.V2.F32.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 red_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int W = 512, H = 512, STEPS = 1024;

template <int MODE>
__global__ void scatter(void* g, int n_rays, float ang0) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  float th = ang0 + r * 0.0123f;
  float dx = cosf(th) * 0.5f, dy = sinf(th) * 0.5f;
  float x = 256.f + (r % 15) * 8.f - 56.f, y = 256.f + ((r / 15) % 15) * 8.f - 56.f;
  for (int i = 0; i < STEPS; ++i) {
    x += dx; y += dy;
    if (x < 0.f) x += W; if (x >= W - 1) x -= W - 1;
    if (y < 0.f) y += H; if (y >= H - 1) y -= H - 1;
    int ix = (int)x, iy = (int)y;
    int p = iy * W + ix;
    float v = 1e-3f * (i & 7);
    if (MODE == 0) atomicAdd((double*)g + p, (double)v);
    else if (MODE == 1) atomicAdd((unsigned long long*)g + p, (unsigned long long)(v * 1e6f));
    else if (MODE == 2) atomicAdd((float*)g + p, v);
    else if (MODE == 3) {
      float2* q = (float2*)g + (p >> 1);
      atomicAdd(q, make_float2(v, v));
    } else if (MODE == 4) {  // no atomic: plain store (bandwidth reference)
      ((float*)g)[p] = v;
    }
  }
}

int main() {
  void* g;
  cudaMalloc(&g, (size_t)W * H * 8);
  cudaMemset(g, 0, (size_t)W * H * 8);
  const int n_rays = 115200;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"RED.F64", "RED.U64", "RED.F32", "RED.V2.F32", "ST.F32"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      switch (mode) {
        case 0: scatter<0><<<n_rays / 256, 256>>>(g, n_rays, 0.1f); break;
        case 1: scatter<1><<<n_rays / 256, 256>>>(g, n_rays, 0.1f); break;
        case 2: scatter<2><<<n_rays / 256, 256>>>(g, n_rays, 0.1f); break;
        case 3: scatter<3><<<n_rays / 256, 256>>>(g, n_rays, 0.1f); break;
        case 4: scatter<4><<<n_rays / 256, 256>>>(g, n_rays, 0.1f); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2)
        printf("%-11s %.3f ms  %.2f G ops/s\n", names[mode], ms, (double)n_rays * STEPS / ms / 1e6);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
