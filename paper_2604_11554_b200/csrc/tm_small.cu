// SPDX-License-Identifier: Apache-2.0
//
// Latency-bound per-sequence kernels of the hot path:
//   a6  varlen packing metadata (cu_seqlens, token->sequence, loss mask,
//       token->group) — bit-exact integer work;
//   a3  GRPO group advantage keyed on arbitrary int32 group ids (groups need
//       not be contiguous: the bus delivers in readiness order,
//       proj/src/transfer_queue.cpp:162-175);
//   a4  prologue: per-token advantage and loss weight w_t = mask_t * inv_norm_t;
//   synthetic logits for the bench, generated on device from the reference's
//       SplitMix64 (proj/include/staleflow/rng.hpp:17-39) evaluated at an index.
// All reductions are fixed-order (no float atomics) so results are bitwise
// reproducible run to run.

#include <cuda_runtime.h>

#include "tm_device.cuh"
#include "tm_internal.h"

namespace sftm {

// ------------------------------------------------------------------ a6
constexpr int kScanT = 1024;

// Single-CTA exclusive scan of seq_lens -> cu_seqlens[B+1]; total -> d_total.
__global__ void __launch_bounds__(kScanT)
    scan_lens_kernel(const int32_t* __restrict__ lens, int64_t B, int32_t* __restrict__ cu,
                     int32_t* __restrict__ d_total) {
  __shared__ int32_t wsum[kScanT / 32];
  __shared__ int32_t carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < B; base += kScanT) {
    const int64_t i = base + tid;
    const int32_t v = (i < B) ? lens[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int32_t s = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const int32_t incl = x + (warp > 0 ? wsum[warp - 1] : 0) + carry;
    if (i < B) cu[i] = incl - v;
    __syncthreads();
    if (tid == kScanT - 1) carry = incl;
    __syncthreads();
  }
  if (tid == 0) {
    cu[B] = carry;
    if (d_total) *d_total = carry;
  }
}

__global__ void fill_tokens_kernel(const int32_t* __restrict__ cu, const int32_t* __restrict__ plens,
                                   const int32_t* __restrict__ gids, int64_t B, int64_t T,
                                   int32_t* __restrict__ seq_id, uint8_t* __restrict__ mask,
                                   int32_t* __restrict__ tok_group) {
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    const int64_t s = cu[b], e = cu[b + 1];
    const int32_t pl = plens ? plens[b] : 0;
    const int32_t g = gids ? gids[b] : 0;
    for (int64_t t = s + threadIdx.x; t < e && t < T; t += blockDim.x) {
      if (seq_id) seq_id[t] = static_cast<int32_t>(b);
      if (mask) mask[t] = (t - s) >= pl ? 1 : 0;
      if (tok_group) tok_group[t] = g;
    }
  }
}

int launch_varlen_meta(const int32_t* seq_lens, const int32_t* prompt_lens,
                       const int32_t* group_ids, int64_t B, int64_t T, int32_t* cu_seqlens,
                       int32_t* seq_id, uint8_t* mask, int32_t* tok_group, int32_t* d_total,
                       cudaStream_t s, int* launches) {
  scan_lens_kernel<<<1, kScanT, 0, s>>>(seq_lens, B, cu_seqlens, d_total);
  int n = 1;
  if (T > 0 && B > 0 && (seq_id || mask || tok_group)) {
    int64_t grid = B < 4096 ? B : 4096;
    fill_tokens_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(
        cu_seqlens, prompt_lens, group_ids, B, T, seq_id, mask, tok_group);
    ++n;
  }
  if (launches) *launches += n;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a3
// One warp per sample; lanes stride over all samples, fixed shuffle tree.
__global__ void grpo_adv_kernel(const float* __restrict__ r, const int32_t* __restrict__ gid,
                                int64_t B, float eps, int std_mode, float* __restrict__ out,
                                int32_t* __restrict__ gsize) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t i = blockIdx.x * wpb + (threadIdx.x >> 5); i < B; i += gridDim.x * wpb) {
    const int32_t gi = gid[i];
    int n = 0;
    double sum = 0.0;
    float mn = INFINITY, mx = -INFINITY;
    for (int64_t j = lane; j < B; j += 32) {
      if (gid[j] == gi) {
        const float v = r[j];
        ++n;
        sum += static_cast<double>(v);
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      n += __shfl_xor_sync(0xffffffffu, n, o);
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const double mean = sum / static_cast<double>(n);
    double ss = 0.0;
    if (std_mode != 2) {
      for (int64_t j = lane; j < B; j += 32) {
        if (gid[j] == gi) {
          const double d = static_cast<double>(r[j]) - mean;
          ss += d * d;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if (lane == 0) {
      double A;
      if (mx == mn) {
        A = 0.0;  // P3: zero-variance group (includes singletons) -> exactly 0
      } else {
        const double d = static_cast<double>(r[i]) - mean;
        if (std_mode == 2) {
          A = d;
        } else {
          const double var = (std_mode == 0) ? ss / static_cast<double>(n - 1)
                                              : ss / static_cast<double>(n);
          A = d / (sqrt(var) + static_cast<double>(eps));
        }
      }
      out[i] = static_cast<float>(A);
      if (gsize) gsize[i] = n;
    }
  }
}

// O(B log B) form for B <= kSortB (one CTA): bitonic sort of (group id, sample)
// keys in shared memory, then one thread per run of equal ids computes the
// group's n / mean / min / max / sum of squares in sample-index order (fixed
// order: deterministic) and writes every member's advantage. The O(B^2) kernel
// above (one warp per sample scanning all ids) stays for larger B.
constexpr int kSortB = 16384;
constexpr int kSortT = 1024;

__global__ void __launch_bounds__(kSortT)
    grpo_adv_sorted_kernel(const float* __restrict__ r, const int32_t* __restrict__ gid, int B, int n2, float eps,
                           int std_mode, float* __restrict__ out, int32_t* __restrict__ gsize) {
  extern __shared__ unsigned long long keys[];  // n2 (power of two >= B) sort keys
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    keys[i] = i < B ? ((static_cast<unsigned long long>(static_cast<uint32_t>(gid[i]) ^ 0x80000000u) << 32) |
                       static_cast<uint32_t>(i))
                    : ~0ull;  // padding sorts last
  }
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long a = keys[i], b = keys[l];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // runs of equal group ids; within a run the sample indices ascend
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    const uint32_t g = static_cast<uint32_t>(keys[i] >> 32);
    if (i > 0 && static_cast<uint32_t>(keys[i - 1] >> 32) == g) continue;  // not a run head
    int e = i + 1;
    while (e < B && static_cast<uint32_t>(keys[e] >> 32) == g) ++e;
    const int n = e - i;
    double sum = 0.0;
    float mn = INFINITY, mx = -INFINITY;
    for (int q = i; q < e; ++q) {
      const float v = r[static_cast<uint32_t>(keys[q])];
      sum += static_cast<double>(v);
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    }
    const double mean = sum / static_cast<double>(n);
    double ss = 0.0;
    if (std_mode != 2)
      for (int q = i; q < e; ++q) {
        const double d = static_cast<double>(r[static_cast<uint32_t>(keys[q])]) - mean;
        ss += d * d;
      }
    double den = 1.0;
    if (std_mode != 2) {
      const double var = (std_mode == 0) ? ss / static_cast<double>(n - 1) : ss / static_cast<double>(n);
      den = sqrt(var) + static_cast<double>(eps);
    }
    for (int q = i; q < e; ++q) {
      const uint32_t s_ = static_cast<uint32_t>(keys[q]);
      double A = 0.0;  // P3: zero-variance group (includes singletons) -> exactly 0
      if (mx != mn) A = (static_cast<double>(r[s_]) - mean) / den;
      out[s_] = static_cast<float>(A);
      if (gsize) gsize[s_] = n;
    }
  }
}

int launch_grpo_advantage(const float* rewards, const int32_t* group_ids, int64_t B, float eps,
                          int std_mode, float* out_adv, int32_t* out_group_size, cudaStream_t s,
                          int* launches) {
  if (B <= kSortB) {
    int n2 = 1;
    while (n2 < B) n2 <<= 1;
    const size_t smem = sizeof(unsigned long long) * static_cast<size_t>(n2);
    static PerDevice opted;
    if (opted() < 0) {
      cudaFuncSetAttribute(grpo_adv_sorted_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(unsigned long long) * kSortB));
      opted() = 1;
    }
    grpo_adv_sorted_kernel<<<1, kSortT, smem, s>>>(rewards, group_ids, static_cast<int>(B), n2, eps, std_mode,
                                                   out_adv, out_group_size);
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  const int threads = 256;
  int64_t grid = (B + 7) / 8;
  if (grid > 4096) grid = 4096;
  if (grid < 1) grid = 1;
  grpo_adv_kernel<<<static_cast<unsigned>(grid), threads, 0, s>>>(rewards, group_ids, B, eps,
                                                                   std_mode, out_adv,
                                                                   out_group_size);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a5 transport
// The rollout records routed experts per token ("routed_experts" bus field:
// token-major [T, L, k]); the gate consumes them
// layer-major [L, T, k]. After ONE host->device copy of the concatenated
// payloads, a 32 x 32 record tile goes through shared memory per CTA: reads
// are contiguous along layers, writes contiguous along tokens. Records move
// as whole 4- or 8-byte words when their size allows (k u8 indices, or k
// int32), else bytewise. Bit-exact by construction.
template <typename W>
__global__ void __launch_bounds__(256)
    rec_transpose_kernel(const W* __restrict__ src, W* __restrict__ dst, int64_t Tn, int64_t L, int wpr) {
  extern __shared__ __align__(16) unsigned char tile_raw[];
  W* tile = reinterpret_cast<W*>(tile_raw);  // [32 t][32 l][wpr] (+1 word pad per t row)
  const int pitch = 32 * wpr + 1;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * 32, l0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int nw = 32 * wpr;  // words per tile row
  for (int i = threadIdx.x; i < 32 * nw; i += blockDim.x) {
    const int tt = i / nw, r = i % nw;  // token row of the tile, word within its 32 layers
    const int64_t t = t0 + tt, l = l0 + r / wpr;
    if (t < Tn && l < L) tile[tt * pitch + r] = src[(t * L + l) * wpr + r % wpr];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * nw; i += blockDim.x) {
    const int ll = i / nw, r = i % nw;  // layer row of the tile, word within its 32 tokens
    const int64_t l = l0 + ll, t = t0 + r / wpr;
    if (t < Tn && l < L) dst[(l * Tn + t) * wpr + r % wpr] = tile[(r / wpr) * pitch + ll * wpr + r % wpr];
  }
}

int launch_rec_layer_major(const void* rec_tok, int idx_dtype, int64_t T, int64_t L, int64_t k, void* rec_layer,
                           cudaStream_t s, int* launches) {
  const int64_t rb = k * (idx_dtype == 1 ? 1 : 4);  // bytes per (token, layer) record
  const uintptr_t al = reinterpret_cast<uintptr_t>(rec_tok) | reinterpret_cast<uintptr_t>(rec_layer);
  const dim3 grid(static_cast<unsigned>((T + 31) / 32), static_cast<unsigned>((L + 31) / 32));
  auto go = [&](auto w) {
    using Wt = decltype(w);
    const int wpr = static_cast<int>(rb / static_cast<int64_t>(sizeof(Wt)));
    const size_t smem = sizeof(Wt) * 32 * static_cast<size_t>(32 * wpr + 1);  // <= 129 KB (k = 32 int32)
    static PerDevice opted;  // per instantiation and device: allow > 48 KB dynamic smem
    if (opted() < 0) {
      cudaFuncSetAttribute(rec_transpose_kernel<Wt>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
      opted() = 1;
    }
    rec_transpose_kernel<Wt><<<grid, 256, smem, s>>>(static_cast<const Wt*>(rec_tok), static_cast<Wt*>(rec_layer),
                                                     T, L, wpr);
  };
  if (rb % 8 == 0 && al % 8 == 0) {
    go(uint64_t{});
  } else if (rb % 4 == 0 && al % 4 == 0) {
    go(uint32_t{});
  } else {
    go(uint8_t{});
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a4 prologue
// Pass 1: active-token count per sequence; the last block reduces the totals
// (sum of counts, number of sequences with >= 1 active token) in seq order.
__global__ void seq_count_kernel(const int32_t* __restrict__ cu, int64_t B,
                                 const uint8_t* __restrict__ mask, int32_t* __restrict__ cnt,
                                 unsigned* __restrict__ ticket, int64_t* __restrict__ tot) {
  __shared__ int32_t wsum[8];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    const int64_t s = cu[b], e = cu[b + 1];
    int32_t c = 0;
    if (mask) {
      for (int64_t t = s + threadIdx.x; t < e; t += blockDim.x) c += mask[t] ? 1 : 0;
    } else if (threadIdx.x == 0) {
      c = static_cast<int32_t>(e - s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) wsum[warp] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int32_t t = 0;
      for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += wsum[i];
      cnt[b] = t;
    }
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (last) {
    __threadfence();
    int64_t total = 0, nonempty = 0;
    const volatile int32_t* vc = cnt;
    for (int64_t b = threadIdx.x; b < B; b += blockDim.x) {
      const int32_t v = vc[b];
      total += v;
      nonempty += v > 0 ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      total += __shfl_xor_sync(0xffffffffu, total, o);
      nonempty += __shfl_xor_sync(0xffffffffu, nonempty, o);
    }
    __shared__ int64_t ws[2][8];
    if (lane == 0) {
      ws[0][warp] = total;
      ws[1][warp] = nonempty;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t a = 0, n = 0;
      for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) {
        a += ws[0][i];
        n += ws[1][i];
      }
      tot[0] = a;
      tot[1] = n;
      *ticket = 0u;
    }
  }
}

__global__ void token_weights_kernel(const int32_t* __restrict__ cu, int64_t B,
                                     const float* __restrict__ adv, const uint8_t* __restrict__ mask,
                                     int64_t T, int norm_mode, float inv_norm,
                                     const int32_t* __restrict__ cnt,
                                     const int64_t* __restrict__ tot, float* __restrict__ adv_tok,
                                     float* __restrict__ w_tok) {
  const int64_t total = tot[0], nonempty = tot[1];
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    const int64_t s = cu[b], e = cu[b + 1];
    float wseq;
    if (norm_mode == 0) {
      wseq = total > 0 ? static_cast<float>(1.0 / static_cast<double>(total)) : 0.f;
    } else if (norm_mode == 1) {
      const int32_t c = cnt[b];
      wseq = c > 0 ? static_cast<float>(1.0 / (static_cast<double>(c) * static_cast<double>(nonempty)))
                   : 0.f;
    } else {
      wseq = inv_norm;
    }
    const float A = adv ? adv[b] : 0.f;
    for (int64_t t = s + threadIdx.x; t < e && t < T; t += blockDim.x) {
      const bool on = mask ? (mask[t] != 0) : true;
      w_tok[t] = on ? wseq : 0.f;
      adv_tok[t] = A;
    }
  }
}

int launch_token_weights(const int32_t* cu_seqlens, int64_t B, const float* adv_seq,
                         const uint8_t* mask, int64_t T, int norm_mode, float inv_norm,
                         float* out_adv_tok, float* out_w_tok, int32_t* scratch_cnt,
                         unsigned* scratch_ticket, int64_t* scratch_tot, cudaStream_t s,
                         int* launches) {
  int64_t grid = B < 2048 ? B : 2048;
  if (grid < 1) grid = 1;
  seq_count_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(cu_seqlens, B, mask, scratch_cnt,
                                                              scratch_ticket, scratch_tot);
  token_weights_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(
      cu_seqlens, B, adv_seq, mask, T, norm_mode, inv_norm, scratch_cnt, scratch_tot, out_adv_tok,
      out_w_tok);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ synthetic logits
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// i-th output (0-based) of staleflow::SplitMix64(seed) (rng.hpp:21-26).
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t i) {
  return mix64(seed + (i + 1ull) * 0x9e3779b97f4a7c15ull);
}
__device__ __forceinline__ float u24(uint32_t x) {  // (0,1)
  return (static_cast<float>(x >> 8) + 0.5f) * (1.0f / 16777216.0f);
}

template <typename T>
__global__ void synth_logits_kernel(T* __restrict__ out, int64_t Tn, int64_t V, int64_t ld,
                                    uint64_t seed, float sigma, const int32_t* __restrict__ peak,
                                    float plo, float phi, float ofrac) {
  const uint64_t s_out = mix64(seed ^ 0x6f75746c69657273ull);
  const uint64_t s_pk = mix64(seed ^ 0x7065616b7065616bull);
  const int64_t n = Tn * V;
  const uint32_t othr = static_cast<uint32_t>(static_cast<double>(ofrac) * 4294967296.0);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / V, v = i - t * V;
    const uint64_t h = splitmix_at(seed, static_cast<uint64_t>(i));
    const float u1 = u24(static_cast<uint32_t>(h)), u2 = u24(static_cast<uint32_t>(h >> 32));
    float x = sigma * sqrtf(-2.f * __logf(u1)) * __cosf(6.283185307179586f * u2);
    if (othr) {
      const uint64_t h2 = splitmix_at(s_out, static_cast<uint64_t>(i));
      if (static_cast<uint32_t>(h2) < othr) x = (h2 >> 63) ? 30.f : -30.f;
    }
    if (peak && v == peak[t]) {
      const uint64_t h3 = splitmix_at(s_pk, static_cast<uint64_t>(t));
      x += plo + (phi - plo) * u24(static_cast<uint32_t>(h3));
    }
    if constexpr (sizeof(T) == 2) {
      out[t * ld + v] = f32_to_bf16(x);
    } else {
      out[t * ld + v] = x;
    }
  }
}

int launch_synth_logits(void* logits, int dtype, int64_t T, int64_t V, int64_t ld, uint64_t seed,
                        float sigma, const int32_t* peak_id, float peak_lo, float peak_hi,
                        float outlier_frac, cudaStream_t s, int* launches) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = static_cast<unsigned>(sms * 16);
  if (dtype == 1)
    synth_logits_kernel<uint16_t><<<grid, 256, 0, s>>>(static_cast<uint16_t*>(logits), T, V, ld,
                                                       seed, sigma, peak_id, peak_lo, peak_hi,
                                                       outlier_frac);
  else
    synth_logits_kernel<float><<<grid, 256, 0, s>>>(static_cast<float*>(logits), T, V, ld, seed,
                                                    sigma, peak_id, peak_lo, peak_hi,
                                                    outlier_frac);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace sftm
