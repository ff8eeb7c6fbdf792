// FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a: 8 independent
// chains per thread, 4096 iterations, 148*8 CTAs of 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ u64 f2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__global__ void k1(float* out, float s, int iters) {
  float a[16];
  for (int j = 0; j < 16; j++) a[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int j = 0; j < 16; j++) a[j] = fmaf(a[j], s, 0.5f);
  float t = 0; for (int j = 0; j < 16; j++) t += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k2(float* out, float s, int iters) {
  u64 a[8];
  for (int j = 0; j < 8; j++) a[j] = pk(threadIdx.x * 1e-3f + 2 * j, threadIdx.x * 1e-3f + 2 * j + 1);
  const u64 ss = pk(s, s), h = pk(0.5f, 0.5f);
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = f2(a[j], ss, h);
  float t = 0;
  for (int j = 0; j < 8; j++) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[j])); t += x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 8192;
  for (int rep = 0; rep < 2; rep++) {
    for (int v = 0; v < 2; v++) {
      cudaEventRecord(e0);
      if (v == 0) k1<<<148 * 8, 256>>>(o, 0.999f, iters); else k2<<<148 * 8, 256>>>(o, 0.999f, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * iters * 148.0 * 8 * 256;
      printf("%s: %.3f ms, %.1f TFLOP/s\n", v ? "FFMA2" : "FFMA ", ms, flops / ms / 1e9);
    }
  }
  return 0;
}
