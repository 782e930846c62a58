// Issue cost of the conversions the e-store loss schedule uses, per SM, on sm_100a:
// fp16x2 -> 2 x fp32 (cvt.f32.f16, HADD2.F32), bf16x2 unpack (shift/and),
// MUFU.EX2, fp32x2 -> fp16x2 / bf16x2 pack (F2FP). Dependent chains of 8
// independent streams per thread, 32 warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_11554_b200/csrc -o scripts/mb_cvt scripts/microbench_cvt.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tm_device.cuh"

using namespace sftm;

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(uint32_t* out, int iters, uint32_t seed) {
  uint32_t w[8];
  float f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    w[i] = seed * (threadIdx.x + 7 * i + 1) | 0x3c003c00u;
    f[i] = __uint_as_float(w[i] & 0x3fffffffu);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {  // fp16x2 -> fp32 pair -> back (keeps a dependent chain)
        const float2 v = unpack_f16x2(w[i]);
        w[i] = __float_as_uint(v.x) ^ __float_as_uint(v.y);
      } else if (MODE == 1) {  // bf16x2 unpack
        const float a = bf16lo(w[i]), b = bf16hi(w[i]);
        w[i] = __float_as_uint(a) ^ __float_as_uint(b);
      } else if (MODE == 2) {  // two MUFU.EX2
        f[i] = ex2(f[i]) + ex2(-f[i]);
      } else if (MODE == 3) {  // fp16x2 pack
        w[i] = pack_f16x2(__uint_as_float(w[i]), __uint_as_float(w[i] >> 1));
      } else {  // bf16x2 pack
        w[i] = pack_bf16x2(__uint_as_float(w[i]), __uint_as_float(w[i] >> 1));
      }
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r ^= w[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  cudaMalloc(&out, sizeof(uint32_t) * sms * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  const char* names[] = {"f16x2->2xf32 (cvt.f32.f16)", "bf16x2 unpack (shift/and)", "2x MUFU.EX2", "f32x2->f16x2 pack", "f32x2->bf16x2 pack"};
  void (*ks[])(uint32_t*, int, uint32_t) = {k<0>, k<1>, k<2>, k<3>, k<4>};
  for (int m = 0; m < 5; ++m) {
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      ks[m]<<<sms, 1024>>>(out, iters, 12345u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ops = double(sms) * 1024 * iters * 8;  // element-pair operations
    printf("%-30s %8.3f ms  %7.1f pair-ops/clk/SM (at %d MHz max)\n", names[m], ms, ops / (ms * 1e-3) / sms / (clk * 1e3),
           clk / 1000);
  }
  return 0;
}
