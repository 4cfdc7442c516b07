// Microbenchmark: FP32 FMA throughput per SM with scalar FFMA vs packed
// FFMA2 (fma.rn.f32x2, sm_100a).  Each thread runs 16 independent FMA chains
// (scalar) or 8 independent FFMA2 chains (= 16 FMAs).  Prints TFLOP/s.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, int iters, float m) {
  float a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], m, 0.5f);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, int iters, float m) {
  uint64_t a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float lo = threadIdx.x * 1e-3f + j, hi = lo + 0.25f;
    asm("mov.b64 %0, {%1,%2};" : "=l"(a[j]) : "f"(lo), "f"(hi));
  }
  uint64_t mm, hh;
  asm("mov.b64 %0, {%1,%1};" : "=l"(mm) : "f"(m));
  const float half = 0.5f;
  asm("mov.b64 %0, {%1,%1};" : "=l"(hh) : "f"(half));
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(mm), "l"(hh));
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float lo, hi;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[j]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FP64: 8 independent DFMA chains per thread (the f64 parity path's pipe)
__global__ void k_dfma(double* out, int iters, double m) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], m, 0.5);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 20000;
  float* out;
  cudaMalloc(&out, blocks * threads * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int pass = 0; pass < 2; ++pass) {
    for (int v = 0; v < 2; ++v) {
      cudaEventRecord(e0);
      if (v == 0) k_ffma<<<blocks, threads>>>(out, iters, 0.999f);
      else k_ffma2<<<blocks, threads>>>(out, iters, 0.999f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 16 * (double)iters * blocks * threads;
      if (pass == 1) printf("%s: %.3f ms  %.1f TFLOP/s\n", v ? "FFMA2" : "FFMA ", ms, flops / ms / 1e9);
    }
  }
  double* dout;
  cudaMalloc(&dout, blocks * threads * sizeof(double));
  for (int pass = 0; pass < 2; ++pass) {
    const int diters = iters / 4;
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(dout, diters, 0.999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * (double)diters * blocks * threads;
    if (pass == 1) printf("DFMA : %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  return 0;
}
