// Microbenchmark: FFMA vs packed FFMA2 (fma.rn.f32x2) issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void k_ffma(float* out, int iters, float s) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 0.001f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], s, 0.5f);
  }
  float t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_ffma2(float* out, int iters, float s) {
  unsigned long long a[8];
  float2 sv = make_float2(s, s), hv = make_float2(0.5f, 0.5f);
  unsigned long long sr = *(unsigned long long*)&sv, hr = *(unsigned long long*)&hv;
#pragma unroll
  for (int j = 0; j < 8; ++j) { float2 v = make_float2(threadIdx.x * 0.001f + j, j + 0.5f); a[j] = *(unsigned long long*)&v; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = f2fma(a[j], sr, hr);
  }
  float t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { float2 v = *(float2*)&a[j]; t += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 20000;
  float* out;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_ffma<<<blocks, threads>>>(out, iters, 0.999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms1;
    cudaEventElapsedTime(&ms1, e0, e1);
    cudaEventRecord(e0);
    k_ffma2<<<blocks, threads>>>(out, iters, 0.999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms2;
    cudaEventElapsedTime(&ms2, e0, e1);
    const double fl1 = 2.0 * blocks * threads * (double)iters * 8, fl2 = 2 * fl1;
    printf("FFMA  %.3f ms  %.1f TFLOP/s (warp-instr/clk/SM %.2f)\n", ms1, fl1 / ms1 / 1e9,
           (fl1 / 64) / (ms1 * 1e-3) / sms / 1.965e9);
    printf("FFMA2 %.3f ms  %.1f TFLOP/s (warp-instr/clk/SM %.2f)\n", ms2, fl2 / ms2 / 1e9,
           (fl2 / 128) / (ms2 * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
