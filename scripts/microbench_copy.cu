// Read+write streaming patterns on sm_100a: does the fused loss's memory
// pattern (per-CTA row streams: TMA read ring -> STG write, writes lagging the
// reads) reach the bandwidth of a grid-stride copy?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_11554_b200/csrc -o scripts/mb_copy scripts/microbench_copy.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tm_device.cuh"

using namespace sftm;

__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// Rows of `row_bytes`; CTA b handles rows b, b+grid, ... (the loss kernel's
// order). Producer lane: TMA 1-D reads of `chunk` bytes into an ns-slot ring.
// mode 0: 8 consumer warps LDS.128 + STG.128 the chunk to dst (same offset)
// mode 1: consumer warp 0 lane 0 bulk-stores the slot (TMA s2g), waits .read
// mode 2: like 0 but STG goes to the chunk `lag` chunks behind (different row)
__global__ void __launch_bounds__(288, 1) row_copy(const char* src, char* dst, size_t rows, size_t row_bytes,
                                                   int chunk, int ns, int mode, int lag) {
  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[64], empty[64];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cpr = static_cast<int>(row_bytes / chunk);
  if (tid == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), mode == 1 ? 1 : 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t rb = smem_u32(ring);
  if (warp == 8) {
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      uint32_t slot = 0, ph = 0;
      for (size_t r = blockIdx.x; r < rows; r += gridDim.x)
        for (int k = 0; k < cpr; ++k) {
          mbar_wait(smem_u32(&empty[slot]), ph ^ 1u);
          mbar_arrive_expect_tx(smem_u32(&full[slot]), chunk);
          bulk_g2s(rb + slot * chunk, src + r * row_bytes + static_cast<size_t>(k) * chunk, chunk,
                   smem_u32(&full[slot]), pol);
          if (++slot == static_cast<uint32_t>(ns)) { slot = 0; ph ^= 1u; }
        }
    }
  } else {
    uint32_t slot = 0, ph = 0;
    size_t gk = 0;  // this CTA's running chunk index
    for (size_t r = blockIdx.x; r < rows; r += gridDim.x)
      for (int k = 0; k < cpr; ++k, ++gk) {
        mbar_wait(smem_u32(&full[slot]), ph);
        if (mode == 1) {
          if (tid == 0) {
            bulk_s2g(dst + r * row_bytes + static_cast<size_t>(k) * chunk, rb + slot * chunk, chunk);
            bulk_commit();
            bulk_wait_read<0>();
            mbar_arrive(smem_u32(&empty[slot]));
          }
        } else {
          size_t doff = r * row_bytes + static_cast<size_t>(k) * chunk;
          if (mode == 2 && gk >= static_cast<size_t>(lag)) {
            const size_t g2 = gk - lag;  // this CTA's chunk g2 -> row/blk
            const size_t r2 = blockIdx.x + (g2 / cpr) * gridDim.x;
            doff = r2 * row_bytes + (g2 % cpr) * chunk;
          }
          for (int o = tid * 16; o < chunk; o += 256 * 16) {
            const uint4 v = lds128(rb + slot * chunk + o);
            if (mode == 3)
              *reinterpret_cast<uint4*>(dst + doff + o) = v;
            else
              __stcs(reinterpret_cast<uint4*>(dst + doff + o), v);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&empty[slot]));
        }
        if (++slot == static_cast<uint32_t>(ns)) { slot = 0; ph ^= 1u; }
      }
  }
}

__global__ void ldg_copy(const uint4* src, uint4* dst, size_t n16) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16; i += stride)
    __stcs(dst + i, __ldcs(src + i));
}

int main(int argc, char** argv) {
  // default: one CTA's half row at C=2 (bf16); argv[1] overrides (bytes)
  const size_t row_bytes = argc > 1 ? static_cast<size_t>(atol(argv[1])) : size_t(151936) * 2 / 2;
  const size_t rows = (size_t(16) << 30) / row_bytes;
  const size_t bytes = rows * row_bytes;
  char *src, *dst;
  cudaMalloc(&src, bytes);
  cudaMalloc(&dst, bytes);
  cudaMemset(src, 1, bytes);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(row_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int bpsm : {1, 4, 8}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      ldg_copy<<<sms * bpsm, 256>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), bytes / 16);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid-stride LDG/STG copy %d CTA/SM     : %7.0f GB/s (r+w)\n", bpsm, 2.0 * bytes / ms / 1e6);
  }
  struct Cfg { int chunk, ns, mode, lag; const char* what; };
  // row_bytes = 151936 B = 12.37 x 12 KB; use chunks dividing it loosely (tail dropped)
  Cfg cfgs[] = {{12288, 17, 0, 0, "TMA ring -> STG same chunk"},
                {12288, 17, 3, 0, "TMA ring -> STG (no .cs)"},
                {12288, 8, 0, 0, "TMA ring -> STG 8 slots"},
                {12288, 8, 1, 0, "TMA ring -> bulk store 8sl"},
                {8192, 26, 0, 0, "TMA ring -> STG same chunk"},
                {12288, 17, 1, 0, "TMA ring -> TMA bulk store"},
                {8192, 26, 1, 0, "TMA ring -> TMA bulk store"},
                {12288, 17, 2, static_cast<int>(row_bytes / 12288), "TMA ring -> STG lag 1 row"},
                {12288, 17, 2, static_cast<int>(2 * (row_bytes / 12288)), "TMA ring -> STG lag 2 rows"}};
  for (auto c : cfgs) {
    const size_t rb = row_bytes / c.chunk * c.chunk;
    const size_t nrows = bytes / rb;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      row_copy<<<sms, 288, static_cast<size_t>(c.chunk) * c.ns>>>(src, dst, nrows, rb, c.chunk, c.ns, c.mode, c.lag);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s chunk=%5d slots=%2d lag=%2d: %7.0f GB/s (r+w)  %s\n", c.what, c.chunk, c.ns, c.lag,
           2.0 * nrows * rb / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
