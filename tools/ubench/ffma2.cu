// Microbenchmark: FP32 FFMA vs packed FFMA2 (fma.rn.f32x2, sm_100a) throughput on one B200.
// Each thread runs 8 independent dependency chains; reports lane-FMA/s for both forms.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__global__ void k_ffma(float* out, int iters, float s, float t) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  float b = s + threadIdx.x * 1e-7f, c = t;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], c, b);
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_ffma2(float* out, int iters, float s, float t) {
  u64 a[8];
  for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f); a[i] = *(u64*)&v; }
  float2 bv = make_float2(s + threadIdx.x * 1e-7f, s), cv = make_float2(t, t * 0.9f);
  u64 b = *(u64*)&bv, c = *(u64*)&cv;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ffma2(a[i], b, c);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ffma2(a[i], c, b);
  }
  float r = 0; for (int i = 0; i < 8; ++i) { float2 v = *(float2*)&a[i]; r += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_mufu(float* out, int iters, float s) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i + s;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float y; asm volatile("sin.approx.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y; }
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  const int blocks = 148 * 8, nt = 256, iters = 4096;
  float* out; cudaMalloc(&out, blocks * nt * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k_ffma<<<blocks, nt>>>(out, iters, 0.999f, 1e-3f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * nt * iters * 16;
    printf("{\"test\": \"ffma\", \"ms\": %.3f, \"lane_fma_per_s\": %.4e, \"tflops\": %.2f}\n", ms, fma / ms * 1e3, 2 * fma / ms * 1e-9);
    cudaEventRecord(e0); k_ffma2<<<blocks, nt>>>(out, iters, 0.999f, 1e-3f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fma = (double)blocks * nt * iters * 32;
    printf("{\"test\": \"ffma2\", \"ms\": %.3f, \"lane_fma_per_s\": %.4e, \"tflops\": %.2f}\n", ms, fma / ms * 1e3, 2 * fma / ms * 1e-9);
    cudaEventRecord(e0); k_mufu<<<blocks, nt>>>(out, iters / 4, 0.5f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double mu = (double)blocks * nt * (iters / 4) * 8;
    printf("{\"test\": \"mufu_sin\", \"ms\": %.3f, \"per_s\": %.4e, \"per_sm_per_clk_at_1965\": %.2f}\n", ms, mu / ms * 1e3, mu / ms * 1e3 / 148 / 1.965e9);
  }
  return 0;
}
