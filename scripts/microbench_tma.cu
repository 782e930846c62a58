// Read-streaming microbenchmark on sm_100a: TMA 1-D bulk ring vs LDG.128.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_11554_b200/csrc -o mb_tma scripts/microbench_tma.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tm_device.cuh"

using namespace sftm;

__device__ __forceinline__ bool try_wait_nohint(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}

// One CTA per SM: a producer lane streams `chunk`-byte bulk copies of this CTA's
// contiguous share into an `ns`-slot ring; 8 consumer warps wait, touch 16 B, release.
__global__ void __launch_bounds__(288, 1) tma_stream(const char* src, size_t bytes, int chunk, int ns, int hint,
                                                     unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[64], empty[64];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t per = (bytes / gridDim.x) / 65536 * 65536;
  const char* base = src + per * blockIdx.x;
  const int nchunk = static_cast<int>(per / chunk);
  if (tid == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t rb = smem_u32(ring);
  if (warp == 8) {
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      uint32_t slot = 0, ph = 0;
      for (int k = 0; k < nchunk; ++k) {
        if (hint) mbar_wait(smem_u32(&empty[slot]), ph ^ 1u);
        else while (!try_wait_nohint(smem_u32(&empty[slot]), ph ^ 1u)) {}
        mbar_arrive_expect_tx(smem_u32(&full[slot]), chunk);
        bulk_g2s(rb + slot * chunk, base + static_cast<size_t>(k) * chunk, chunk, smem_u32(&full[slot]), pol);
        if (++slot == static_cast<uint32_t>(ns)) { slot = 0; ph ^= 1u; }
      }
    }
  } else {
    uint32_t slot = 0, ph = 0, acc = 0;
    for (int k = 0; k < nchunk; ++k) {
      if (hint) mbar_wait(smem_u32(&full[slot]), ph);
      else while (!try_wait_nohint(smem_u32(&full[slot]), ph)) {}
      const uint4 v = lds128(rb + slot * chunk + (tid * 16) % chunk);
      acc ^= v.x;
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[slot]));
      if (++slot == static_cast<uint32_t>(ns)) { slot = 0; ph ^= 1u; }
    }
    if (acc == 0x12345678u) sink[0] = acc;
  }
}

__global__ void ldg_stream(const uint4* src, size_t n16, unsigned* sink) {
  uint32_t acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride), d = __ldcs(src + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  const size_t bytes = size_t(32) << 30;
  char* buf;
  unsigned* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, bytes);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int chunk, ns, hint, ctas_per_sm; };
  Cfg cfgs[] = {{12288, 17, 1, 1}, {12288, 17, 0, 1}, {8192, 26, 0, 1}, {16384, 13, 0, 1}, {32768, 6, 0, 1},
                {4096, 52, 0, 1}, {65536, 3, 0, 1}, {12288, 8, 0, 2}, {8192, 12, 0, 2}};
  for (auto c : cfgs) {
    const int grid = sms * c.ctas_per_sm;
    const size_t smem = static_cast<size_t>(c.chunk) * c.ns;
    if (smem > 220 * 1024) continue;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      tma_stream<<<grid, 288, smem>>>(buf, bytes, c.chunk, c.ns, c.hint, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("TMA chunk=%6d slots=%2d hint=%d ctas/SM=%d : %7.0f GB/s  (%s)\n", c.chunk, c.ns, c.hint, c.ctas_per_sm,
           bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  for (int blocks_per_sm : {4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      ldg_stream<<<sms * blocks_per_sm, 256>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("LDG.128 x4 unroll, %2d CTAs/SM x 256 thr : %7.0f GB/s\n", blocks_per_sm, bytes / ms / 1e6);
  }
  return 0;
}
