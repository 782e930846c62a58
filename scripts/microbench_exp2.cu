// Microbenchmark: MUFU.EX2 vs FMA-pipe polynomial exp2 throughput on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_exp2.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Cody-Waite split + degree-5 minimax polynomial for 2^f, f in [-0.5, 0.5]
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -127.f);
  const float t = x + 12582912.f;          // round to nearest integer (1.5*2^23)
  const float j = t - 12582912.f;
  const float f = x - j;
  float p = 1.3333558146428443e-3f;
  p = fmaf(p, f, 9.6181291076284772e-3f);
  p = fmaf(p, f, 5.5504108664821580e-2f);
  p = fmaf(p, f, 2.4022650695910071e-1f);
  p = fmaf(p, f, 6.9314718055994531e-1f);
  p = fmaf(p, f, 1.0f);
  const int e = __float_as_int(t) << 23;   // integer part into the exponent
  return __int_as_float(__float_as_int(p) + e);
}

template <int MODE>
__global__ void k(float* out, int iters, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i) + seed;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float e = MODE == 0 ? ex2(a[i]) : ex2_poly(a[i]);
      acc += e;
      a[i] = a[i] * 0.999f - 1e-4f;
    }
  }
  if (acc == 12345.f) out[threadIdx.x] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 4096);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode) {
    for (int threads : {256, 512, 1024}) {
      dim3 grid(sms * (2048 / threads));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<grid, threads>>>(out, iters, 0.5f);
        else k<1><<<grid, threads>>>(out, iters, 0.5f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      double n = double(grid.x) * threads * iters * 8;
      double per_s = n / (ms * 1e-3);
      printf("%s threads=%d: %.3f ms, %.3e exp2/s, %.2f exp2/clk/SM (at %d MHz nominal)\n",
             mode == 0 ? "MUFU.EX2" : "poly    ", threads, ms, per_s, per_s / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
