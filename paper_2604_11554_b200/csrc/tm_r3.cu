// SPDX-License-Identifier: Apache-2.0
//
// a5: R3 Rollout Routing Replay gate (paper §5.5). The
// trainer re-applies the top-k expert indices recorded at rollout time to its
// own router logits instead of re-selecting them:
//   renorm=1 (P8): w_j = softmax_j(z[e_j]) over the k recorded experts;
//   renorm=0:      w_j = softmax(z)[e_j] over all E experts.
// The replayed indices are passed through bit-exactly, and the trainer's own
// top-k set (ties -> lowest expert index, P9) is compared with the recorded
// set per token to count routing mismatches per layer.
//
// Layout: rows are (layer, token) pairs, layer-major [L*T, E]. One warp per
// row; expert e lives in lane e%32, register e/32 (coalesced row loads).
// Each warp owns a contiguous row range so mismatch counts are flushed with
// one integer atomic per (warp, layer) — integer atomics keep the count exact.

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "tm_device.cuh"
#include "tm_internal.h"

namespace sftm {

template <typename T>
__device__ __forceinline__ float r3_load(const T* p, int64_t i);
template <>
__device__ __forceinline__ float r3_load<float>(const float* p, int64_t i) {
  return __ldg(p + i);
}
template <>
__device__ __forceinline__ float r3_load<uint16_t>(const uint16_t* p, int64_t i) {
  return bf16_to_f32(__ldg(reinterpret_cast<const unsigned short*>(p) + i));
}
__device__ __forceinline__ int32_t r3_idx(const void* p, int idx_dtype, int64_t i) {
  if (idx_dtype == 1) return static_cast<int32_t>(__ldg(static_cast<const uint8_t*>(p) + i));
  return __ldg(static_cast<const int32_t*>(p) + i);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T, int NPL>
__global__ void __launch_bounds__(256)
    r3_fwd_kernel(const T* __restrict__ logits, int64_t L, int64_t Tn, int E, int k,
                  const void* __restrict__ rec, int idx_dtype, int renorm, float* __restrict__ out_w,
                  int32_t* __restrict__ out_idx, uint32_t* __restrict__ mismatch) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t rows = L * Tn;
  const int64_t per = (rows + nw - 1) / nw;
  const int64_t r0 = gw * per;
  int64_t r1 = r0 + per;
  if (r1 > rows) r1 = rows;
  int64_t cur_layer = -1;
  uint32_t cur_cnt = 0;

  for (int64_t row = r0; row < r1; ++row) {
    const int64_t layer = row / Tn;
    if (layer != cur_layer) {
      if (cur_cnt && lane == 0 && mismatch) {
        atomicAdd(mismatch + cur_layer, cur_cnt);
        atomicAdd(mismatch + L, cur_cnt);
      }
      cur_layer = layer;
      cur_cnt = 0;
    }
    float z[NPL];
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int e = i * 32 + lane;
      z[i] = (e < E) ? r3_load(logits, row * E + e) : -INFINITY;
    }
    int32_t my_e = -1;
    if (lane < k) my_e = r3_idx(rec, idx_dtype, row * k + lane);
    // gather z at my recorded expert
    float zr = -INFINITY;
    {
      const int src = my_e & 31, reg = my_e >> 5;
#pragma unroll
      for (int i = 0; i < NPL; ++i) {
        const float v = __shfl_sync(0xffffffffu, z[i], src);
        if (reg == i) zr = v;
      }
      if (my_e < 0 || my_e >= E) zr = (lane < k) ? __int_as_float(0x7fc00000) : -INFINITY;
    }
    float wj;
    if (renorm) {
      const float mx = warp_max(lane < k ? zr : -INFINITY);
      const float ez = (lane < k) ? expf(zr - mx) : 0.f;
      const float sum = warp_sum(ez);
      wj = ez / sum;
    } else {
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < NPL; ++i) mx = fmaxf(mx, z[i]);
      mx = warp_max(mx);
      float se = 0.f;
#pragma unroll
      for (int i = 0; i < NPL; ++i) se += expf(z[i] - mx);
      se = warp_sum(se);
      wj = expf(zr - mx) / se;
    }
    if (lane < k) {
      out_w[row * k + lane] = wj;
      if (out_idx) out_idx[row * k + lane] = my_e;
    }
    if (mismatch) {
      // trainer top-k, ties -> lowest expert index (P9)
      uint32_t taken = 0;
      for (int r = 0; r < k; ++r) {
        float bv = -INFINITY;
        int be = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < NPL; ++i) {
          const int e = i * 32 + lane;
          if (e < E && !((taken >> i) & 1u)) {
            if (z[i] > bv || (z[i] == bv && e < be)) {
              bv = z[i];
              be = e;
            }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oe = __shfl_xor_sync(0xffffffffu, be, o);
          if (ov > bv || (ov == bv && oe < be)) {
            bv = ov;
            be = oe;
          }
        }
        if (be != 0x7fffffff && (be & 31) == lane) taken |= 1u << (be >> 5);
      }
      uint32_t recm = 0;
      for (int j = 0; j < k; ++j) {
        const int e = __shfl_sync(0xffffffffu, my_e, j);
        if (e >= 0 && e < E && (e & 31) == lane) recm |= 1u << (e >> 5);
      }
      if (__any_sync(0xffffffffu, recm != taken)) ++cur_cnt;
    }
  }
  if (cur_cnt && lane == 0 && mismatch) {
    atomicAdd(mismatch + cur_layer, cur_cnt);
    atomicAdd(mismatch + L, cur_cnt);
  }
}

template <typename T>
__device__ __forceinline__ void r3_store(T* p, int64_t i, float v);
template <>
__device__ __forceinline__ void r3_store<float>(float* p, int64_t i, float v) {
  p[i] = v;
}
template <>
__device__ __forceinline__ void r3_store<uint16_t>(uint16_t* p, int64_t i, float v) {
  p[i] = f32_to_bf16(v);
}

template <typename T, int NPL>
__global__ void __launch_bounds__(256)
    r3_bwd_kernel(const T* __restrict__ logits, int64_t rows, int E, int k,
                  const void* __restrict__ rec, int idx_dtype, int renorm,
                  const float* __restrict__ w, const float* __restrict__ dw, T* __restrict__ dz) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t row = gw; row < rows; row += nw) {
    int32_t my_e = -1;
    float wj = 0.f, dwj = 0.f;
    if (lane < k) {
      my_e = r3_idx(rec, idx_dtype, row * k + lane);
      wj = w[row * k + lane];
      dwj = dw[row * k + lane];
    }
    const float S = warp_sum(wj * dwj);
    float out[NPL];
    if (renorm) {
      const float val = wj * (dwj - S);
#pragma unroll
      for (int i = 0; i < NPL; ++i) out[i] = 0.f;
      for (int j = 0; j < k; ++j) {
        const int e = __shfl_sync(0xffffffffu, my_e, j);
        const float v = __shfl_sync(0xffffffffu, val, j);
        if (e >= 0 && e < E && (e & 31) == lane) {
#pragma unroll
          for (int i = 0; i < NPL; ++i)
            if ((e >> 5) == i) out[i] += v;
        }
      }
    } else {
      float z[NPL], mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < NPL; ++i) {
        const int e = i * 32 + lane;
        z[i] = (e < E) ? r3_load(logits, row * E + e) : -INFINITY;
        mx = fmaxf(mx, z[i]);
      }
      mx = warp_max(mx);
      float se = 0.f;
#pragma unroll
      for (int i = 0; i < NPL; ++i) se += expf(z[i] - mx);
      se = warp_sum(se);
      float D[NPL];
#pragma unroll
      for (int i = 0; i < NPL; ++i) D[i] = 0.f;
      for (int j = 0; j < k; ++j) {
        const int e = __shfl_sync(0xffffffffu, my_e, j);
        const float v = __shfl_sync(0xffffffffu, dwj, j);
        if (e >= 0 && e < E && (e & 31) == lane) {
#pragma unroll
          for (int i = 0; i < NPL; ++i)
            if ((e >> 5) == i) D[i] += v;
        }
      }
#pragma unroll
      for (int i = 0; i < NPL; ++i) out[i] = expf(z[i] - mx) / se * (D[i] - S);
    }
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int e = i * 32 + lane;
      if (e < E) r3_store(dz, row * E + e, out[i]);
    }
  }
}


// ---------------------------------------------------------------------------
// Fast path (E % 64 == 0, E <= 256, k <= 16): 16-lane groups, two rows per warp
// instruction. Lane l of a group owns experts {i*64 + 4l + c : c < 4} for
// i < E/64 (two float4 loads per 64 experts -> fully coalesced rows).
// The trainer top-k set equals the recorded set iff the best non-recorded expert
// ranks below the worst recorded one under the order (logit desc, index asc):
// one min and one max reduction (plus an index tie-break only on equal logits)
// instead of k argmax rounds.
// ---------------------------------------------------------------------------
constexpr unsigned kG = 16;  // lanes per row group

__device__ __forceinline__ float gmaxf(float v) {
#pragma unroll
  for (int o = kG / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o, kG));
  return v;
}
__device__ __forceinline__ float gsumf(float v) {
#pragma unroll
  for (int o = kG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, kG);
  return v;
}
__device__ __forceinline__ int gsumi(int v) {
#pragma unroll
  for (int o = kG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, kG);
  return v;
}

template <typename T>
__device__ __forceinline__ void r3_load4(const T* p, float (&z)[4]);
template <>
__device__ __forceinline__ void r3_load4<float>(const float* p, float (&z)[4]) {
  const float4 v = __ldg(reinterpret_cast<const float4*>(p));
  z[0] = v.x; z[1] = v.y; z[2] = v.z; z[3] = v.w;
}
template <>
__device__ __forceinline__ void r3_load4<uint16_t>(const uint16_t* p, float (&z)[4]) {
  const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
  z[0] = bf16lo(v.x); z[1] = bf16hi(v.x); z[2] = bf16lo(v.y); z[3] = bf16hi(v.y);
}

// Group reductions over G lanes (G = 8 or 16).
template <int G>
__device__ __forceinline__ float gmaxf_g(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o, G));
  return v;
}
template <int G>
__device__ __forceinline__ float gsumf_g(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
  return v;
}
template <int G>
__device__ __forceinline__ int gsumi_g(int v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
  return v;
}

// One (layer, token) row per G-lane group, R = 32 / G rows per warp step; lane
// gl of a group holds experts i * 4G + 4 gl + c (i < NV, c < 4). G = 8 halves
// the per-row cost of the group reductions and of the per-row bookkeeping
// (used when k <= 8); G = 16 covers k <= 16.
template <typename T, int E, int G>
__global__ void __launch_bounds__(256, (E / G <= 16) ? 4 : 2)
    r3_fwd_fast(const T* __restrict__ logits, int64_t L, int64_t Tn, int k, const void* __restrict__ rec,
                int idx_dtype, int renorm, float* __restrict__ out_w, int32_t* __restrict__ out_idx,
                uint32_t* __restrict__ mismatch) {
  constexpr int R = 32 / G;            // rows per warp step
  constexpr int W = 4 * G;             // experts per float4 stripe of the group
  constexpr int NV = E / W;            // float4 per lane
  constexpr unsigned GM = (1u << G) - 1u;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);       // lane within the row group
  const int gi = lane / G;             // row of the step
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t rows = L * Tn;
  const int64_t steps = (rows + R - 1) / R;
  const int64_t per = (steps + nw - 1) / nw;  // contiguous step range per warp
  int64_t p0 = gw * per, p1 = p0 + per;
  if (p1 > steps) p1 = steps;
  int64_t cur_layer = 0, layer_end = -1;  // forces a (single) division on the first row
  uint32_t cur_cnt = 0;
  // the recorded index is prefetched one step ahead: the recorded logit's load
  // depends on it, and waiting for it was the kernel's main stall (ncu source page)
  auto idx_of = [&](int64_t q) {
    const int64_t r = R * q + gi;
    return gl < k ? r3_idx(rec, idx_dtype, (r < rows ? r : rows - 1) * k + gl) : -1;
  };
  int e_next = p0 < p1 ? idx_of(p0) : -1;
  for (int64_t pr = p0; pr < p1; ++pr) {
    const int64_t row = R * pr + gi;
    const bool valid = row < rows;
    const int64_t rowc = valid ? row : rows - 1;
    float z[NV][4];
    // no software prefetch of the logits: a lean register budget keeps 4 CTAs
    // (32 warps) per SM resident, which hides their latency better (0.62 vs 0.76 ms)
#pragma unroll
    for (int i = 0; i < NV; ++i) r3_load4(logits + rowc * E + i * W + 4 * gl, z[i]);
    const int my_e = e_next;
    if (pr + 1 < p1) e_next = idx_of(pr + 1);
    float zr = -INFINITY;
    if (gl < k) {
      // the recorded logit: an L1 hit (the row's lines were just loaded)
      zr = (my_e >= 0 && my_e < E) ? r3_load(logits, rowc * E + my_e) : __int_as_float(0x7fc00000);
    }
    // gate weights
    float wj;
    if (renorm) {
      const float mx = gmaxf_g<G>(gl < k ? zr : -INFINITY);
      const float ez = gl < k ? __expf(zr - mx) : 0.f;
      wj = __fdividef(ez, gsumf_g<G>(ez));
    } else {
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) mx = fmaxf(mx, z[i][c]);
      mx = gmaxf_g<G>(mx);
      float se = 0.f;
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) se += __expf(z[i][c] - mx);
      wj = __fdividef(__expf(zr - mx), gsumf_g<G>(se));
    }
    if (valid && gl < k) {
      out_w[row * k + gl] = wj;
      if (out_idx) out_idx[row * k + gl] = my_e;
    }
    if (mismatch) {
      // Recorded set R (k distinct valid experts) equals the trainer's top-k iff no
      // expert outside R beats in_min = min over R under (logit desc, index asc).
      // Counting the experts >= in_min decides the common case without knowing
      // which lane holds which recorded expert; a further expert >= in_min (a
      // mismatch or an exact tie) goes to the per-expert slow path.
      const bool bad_e = gl < k && !(my_e >= 0 && my_e < E);
      const unsigned key = (gl < k && !bad_e) ? ((static_cast<unsigned>(gi) << 16) | static_cast<unsigned>(my_e))
                                              : (0x80000000u | static_cast<unsigned>(lane));
      const unsigned same = __match_any_sync(0xffffffffu, key);  // every lane (no short-circuit)
      const bool dup = gl < k && __popc(same) > 1;
      const unsigned badb = __ballot_sync(0xffffffffu, bad_e || dup);
      const bool grp_bad = ((badb >> (gi * G)) & GM) != 0u;
      float in_min = (gl < k && !bad_e) ? zr : INFINITY;
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) in_min = fminf(in_min, __shfl_xor_sync(0xffffffffu, in_min, o, G));
      int n_ge = 0;
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) n_ge += z[i][c] >= in_min ? 1 : 0;
      n_ge = gsumi_g<G>(n_ge);
      bool mm = grp_bad;
      const bool slow = !grp_bad && n_ge > k;
      // At most k - 1 recorded experts lie strictly above in_min (one of them is
      // the minimum), so k experts strictly above it prove a mismatch: no
      // membership needed. Only exact ties at in_min take the per-expert path.
      bool tie = false;
      if (__any_sync(0xffffffffu, slow)) {
        int n_gt = 0;
#pragma unroll
        for (int i = 0; i < NV; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) n_gt += z[i][c] > in_min ? 1 : 0;
        n_gt = gsumi_g<G>(n_gt);
        if (slow && n_gt >= k) mm = true;
        tie = slow && n_gt < k;
      }
      if (__any_sync(0xffffffffu, tie)) {
        // membership of my experts in the recorded set (k <= G, unrolled)
        uint32_t mine = 0;
#pragma unroll
        for (int j = 0; j < G; ++j) {
          if (j < k) {
            const int e = __shfl_sync(0xffffffffu, my_e, j, G);
            if (e >= 0 && e < E && ((e % W) >> 2) == gl) mine |= 1u << ((e / W) * 4 + (e & 3));
          }
        }
        // best non-recorded logit; on an exact tie the trainer prefers the lower index
        float out_max = -INFINITY;
#pragma unroll
        for (int i = 0; i < NV; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (!((mine >> (i * 4 + c)) & 1u)) out_max = fmaxf(out_max, z[i][c]);
        out_max = gmaxf_g<G>(out_max);
        int in_hi = -1, out_lo = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < NV; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int e = i * W + 4 * gl + c;
            const bool rin = (mine >> (i * 4 + c)) & 1u;
            if (rin && z[i][c] == in_min) in_hi = max(in_hi, e);
            if (!rin && z[i][c] == in_min) out_lo = min(out_lo, e);
          }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          in_hi = max(in_hi, __shfl_xor_sync(0xffffffffu, in_hi, o, G));
          out_lo = min(out_lo, __shfl_xor_sync(0xffffffffu, out_lo, o, G));
        }
        if (tie && (out_max > in_min || (out_max == in_min && out_lo < in_hi))) mm = true;
      }
      // per-layer counts; the layer boundary advances incrementally (no 64-bit division per row)
      const unsigned bal = __ballot_sync(0xffffffffu, valid && mm && gl == 0);
      if (R * pr + (R - 1) < layer_end && R * pr + (R - 1) < rows) {
        cur_cnt += __popc(bal);  // all rows of the step in the current layer (only gl == 0 bits)
      } else {
#pragma unroll
        for (int h = 0; h < R; ++h) {
          const int64_t rr = R * pr + h;
          if (rr >= rows) continue;
          if (rr >= layer_end) {
            if (cur_cnt && lane == 0) {
              atomicAdd(mismatch + cur_layer, cur_cnt);
              atomicAdd(mismatch + L, cur_cnt);
            }
            cur_layer = rr / Tn;
            layer_end = (cur_layer + 1) * Tn;
            cur_cnt = 0;
          }
          if ((bal >> (h * G)) & 1u) ++cur_cnt;
        }
      }
    }
  }
  if (mismatch && cur_cnt && lane == 0) {
    atomicAdd(mismatch + cur_layer, cur_cnt);
    atomicAdd(mismatch + L, cur_cnt);
  }
}

template <typename T, int NB>
__global__ void __launch_bounds__(256)
    r3_bwd_fast(int64_t rows, int k, const void* __restrict__ rec, int idx_dtype, const float* __restrict__ w,
                const float* __restrict__ dw, T* __restrict__ dz) {
  constexpr int E = NB * 64;
  __shared__ __align__(16) float buf[8][2][E];  // per warp: the two rows of a pair
  const int lane = threadIdx.x & 31;
  const int gl = lane & (kG - 1);
  const int half = lane >> 4;
  float* rb = buf[threadIdx.x >> 5][half];
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  // the next pair's (index, w, dw) are loaded one iteration ahead
  int en = -1;
  float wn = 0.f, dwn = 0.f;
  if (2 * gw < rows && gl < k) {
    const int64_t r = 2 * gw + half < rows ? 2 * gw + half : rows - 1;
    en = r3_idx(rec, idx_dtype, r * k + gl);
    wn = w[r * k + gl];
    dwn = dw[r * k + gl];
  }
  for (int64_t pr = gw; 2 * pr < rows; pr += nw) {
    const int64_t row = 2 * pr + half;
    const bool valid = row < rows;
    const int my_e = en;
    const float wj = wn, dwj = dwn;
    if (2 * (pr + nw) < rows && gl < k) {
      const int64_t r = 2 * (pr + nw) + half < rows ? 2 * (pr + nw) + half : rows - 1;
      en = r3_idx(rec, idx_dtype, r * k + gl);
      wn = w[r * k + gl];
      dwn = dw[r * k + gl];
    }
    const float S = gsumf(wj * dwj);
#pragma unroll
    for (int i = 0; i < NB; ++i) *reinterpret_cast<float4*>(rb + i * 64 + 4 * gl) = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    // dz[e_j] += w_j (dw_j - S); duplicates of a recorded expert accumulate
    if (gl < k && my_e >= 0 && my_e < E) atomicAdd(rb + my_e, wj * (dwj - S));
    __syncwarp();
    if (valid) {
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const float4 o = *reinterpret_cast<const float4*>(rb + i * 64 + 4 * gl);
        T* d = dz + row * E + i * 64 + 4 * gl;
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<float4*>(d) = o;
        } else {
          *reinterpret_cast<uint2*>(d) = make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
        }
      }
    }
    __syncwarp();
  }
}

// k = 8 backward: the loop body has no global loads. A warp takes chunks of 16
// rows; their (index, w, dw) are one 16-B load each per lane (lane l holds
// row l/2, entries 4(l&1)..+3), prefetched a whole chunk (8 two-row
// iterations) ahead. Each iteration the four lanes holding the two rows add
// w_j (dw_j - S) into two zeroed smem row buffers, every lane stores its 16-B
// vectors, and the scattering lanes reset only the entries they set (measured:
// 0.625 ms vs 0.667 ms re-zeroing the whole rows; also tried and slower: an
// LDS only for touched vectors, 0.650 ms).
template <typename T, int NB>
__global__ void __launch_bounds__(256)
    r3_bwd_k8(int64_t rows, const void* __restrict__ rec, int idx_dtype, const float* __restrict__ w,
              const float* __restrict__ dw, T* __restrict__ dz) {
  constexpr int E = NB * 64;
  __shared__ __align__(16) float buf[8][2][E];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gl = lane & 15, half = lane >> 4;
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t nchunk = (rows + 15) / 16;
  auto load = [&](int64_t c, float4& wv, float4& dv, int4& ev) {
    const int64_t r = c * 16 + (lane >> 1);
    if (c < nchunk && r < rows) {
      const int64_t o = r * 8 + 4 * (lane & 1);
      wv = __ldg(reinterpret_cast<const float4*>(w + o));
      dv = __ldg(reinterpret_cast<const float4*>(dw + o));
      if (idx_dtype == 1) {
        const uint32_t u = __ldg(reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(rec) + o));
        ev = make_int4(u & 255u, (u >> 8) & 255u, (u >> 16) & 255u, u >> 24);
      } else {
        ev = __ldg(reinterpret_cast<const int4*>(static_cast<const int32_t*>(rec) + o));
      }
    } else {
      wv = dv = make_float4(0.f, 0.f, 0.f, 0.f);
      ev = make_int4(-1, -1, -1, -1);
    }
  };
  float* rb = buf[wid][half];
  float* tb = buf[wid][(lane >> 1) & 1];  // the buffer of the row this lane's entries belong to
#pragma unroll
  for (int i = 0; i < NB; ++i) *reinterpret_cast<float4*>(rb + i * 64 + 4 * gl) = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncwarp();
  float4 wv, dv;
  int4 ev;
  load(gw, wv, dv, ev);
  for (int64_t c = gw; c < nchunk; c += nw) {
    float4 wn, dn;
    int4 en;
    load(c + nw, wn, dn, en);
    float S = wv.x * dv.x + wv.y * dv.y + wv.z * dv.z + wv.w * dv.w;
    S += __shfl_xor_sync(0xffffffffu, S, 1);
    const float v0 = wv.x * (dv.x - S), v1 = wv.y * (dv.y - S), v2 = wv.z * (dv.z - S), v3 = wv.w * (dv.w - S);
    const bool ok0 = ev.x >= 0 && ev.x < E, ok1 = ev.y >= 0 && ev.y < E, ok2 = ev.z >= 0 && ev.z < E,
               ok3 = ev.w >= 0 && ev.w < E;
#pragma unroll 1
    for (int it = 0; it < 8; ++it) {
      const int64_t row = c * 16 + 2 * it + half;
      const bool mine = (lane >> 2) == it;
      // plain read-add-write, the row's two lanes one after the other: duplicates of
      // a recorded expert accumulate without shared-memory float atomics (a CAS loop
      // on sm_100a)
#pragma unroll
      for (int ph = 0; ph < 2; ++ph) {
        if (mine && (lane & 1) == ph) {
          if (ok0) tb[ev.x] += v0;
          if (ok1) tb[ev.y] += v1;
          if (ok2) tb[ev.z] += v2;
          if (ok3) tb[ev.w] += v3;
        }
        __syncwarp();
      }
      if (row < rows) {
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const float4 o = *reinterpret_cast<const float4*>(rb + i * 64 + 4 * gl);
          T* d = dz + row * E + i * 64 + 4 * gl;
          if constexpr (sizeof(T) == 4) {
            *reinterpret_cast<float4*>(d) = o;
          } else {
            *reinterpret_cast<uint2*>(d) = make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
          }
        }
      }
      __syncwarp();
      if (mine) {
        if (ok0) tb[ev.x] = 0.f;
        if (ok1) tb[ev.y] = 0.f;
        if (ok2) tb[ev.z] = 0.f;
        if (ok3) tb[ev.w] = 0.f;
      }
      __syncwarp();
    }
    wv = wn;
    dv = dn;
    ev = en;
  }
}

namespace {
int r3_grid(int64_t rows) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t g = (rows + 7) / 8;
  const int64_t cap = static_cast<int64_t>(sms) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}
}  // namespace

#define SFTM_R3_NPL(E, X) \
  ((E) <= 32 ? X(1) : (E) <= 64 ? X(2) : (E) <= 128 ? X(4) : (E) <= 256 ? X(8) : X(16))

int launch_r3_fwd(const void* logits, int dtype, int64_t L, int64_t T, int64_t E, int64_t k,
                  const void* rec_idx, int idx_dtype, int renorm, float* out_w, int32_t* out_idx,
                  uint32_t* out_mismatch, cudaStream_t s, int* launches) {
  if (E % 64 == 0 && E <= 256 && k <= 16) {
    const bool g8 = k <= 8 && E % 32 == 0;  // 8-lane groups: 4 rows per warp step
    const int grid = r3_grid((L * T + (g8 ? 3 : 1)) / (g8 ? 4 : 2));
#define LAUNCH_FF(EE, GG)                                                                              \
  if (dtype == 1)                                                                                      \
    r3_fwd_fast<uint16_t, EE, GG><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(logits), L, T,     \
                                                       static_cast<int>(k), rec_idx, idx_dtype, renorm, \
                                                       out_w, out_idx, out_mismatch);                  \
  else                                                                                                 \
    r3_fwd_fast<float, EE, GG><<<grid, 256, 0, s>>>(static_cast<const float*>(logits), L, T,           \
                                                    static_cast<int>(k), rec_idx, idx_dtype, renorm,    \
                                                    out_w, out_idx, out_mismatch);
    switch (E / 64) {
      case 1: if (g8) { LAUNCH_FF(64, 8) } else { LAUNCH_FF(64, 16) } break;
      case 2: if (g8) { LAUNCH_FF(128, 8) } else { LAUNCH_FF(128, 16) } break;
      case 3: if (g8) { LAUNCH_FF(192, 8) } else { LAUNCH_FF(192, 16) } break;
      default: if (g8) { LAUNCH_FF(256, 8) } else { LAUNCH_FF(256, 16) } break;
    }
#undef LAUNCH_FF
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  const int grid = r3_grid(L * T);
#define LAUNCH_F(NPL)                                                                           \
  (dtype == 1 ? (r3_fwd_kernel<uint16_t, NPL><<<grid, 256, 0, s>>>(                             \
                     static_cast<const uint16_t*>(logits), L, T, static_cast<int>(E),          \
                     static_cast<int>(k), rec_idx, idx_dtype, renorm, out_w, out_idx,          \
                     out_mismatch),                                                             \
                 0)                                                                             \
              : (r3_fwd_kernel<float, NPL><<<grid, 256, 0, s>>>(                                \
                     static_cast<const float*>(logits), L, T, static_cast<int>(E),             \
                     static_cast<int>(k), rec_idx, idx_dtype, renorm, out_w, out_idx,          \
                     out_mismatch),                                                             \
                 0))
  (void)SFTM_R3_NPL(E, LAUNCH_F);
#undef LAUNCH_F
  if (launches) *launches += 1;
  return cudaGetLastError();
}

int launch_r3_bwd(const void* logits, int dtype, int64_t L, int64_t T, int64_t E, int64_t k,
                  const void* rec_idx, int idx_dtype, int renorm, const float* w, const float* dw,
                  void* dlogits, cudaStream_t s, int* launches) {
  const int64_t rows = L * T;
  const bool al = (reinterpret_cast<uintptr_t>(w) % 16 == 0) && (reinterpret_cast<uintptr_t>(dw) % 16 == 0) &&
                  (reinterpret_cast<uintptr_t>(rec_idx) % (idx_dtype == 1 ? 4 : 16) == 0);
  if (renorm && k == 8 && E % 64 == 0 && E <= 256 && al) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // one resident wave (grid-stride over 16-row chunks): no tail wave
    auto grid_for = [&](const void* fn) {
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
      int64_t g = ((rows + 15) / 16 + 7) / 8;
      if (g > static_cast<int64_t>(sms) * per_sm) g = static_cast<int64_t>(sms) * per_sm;
      return static_cast<int>(g < 1 ? 1 : g);
    };
#define LAUNCH_B8(NB)                                                                              \
  if (dtype == 1)                                                                                  \
    r3_bwd_k8<uint16_t, NB><<<grid_for(reinterpret_cast<const void*>(&r3_bwd_k8<uint16_t, NB>)), \
                              256, 0, s>>>(rows, rec_idx, idx_dtype, w, dw,                        \
                                           static_cast<uint16_t*>(dlogits));                       \
  else                                                                                             \
    r3_bwd_k8<float, NB><<<grid_for(reinterpret_cast<const void*>(&r3_bwd_k8<float, NB>)), 256, 0, \
                           s>>>(rows, rec_idx, idx_dtype, w, dw, static_cast<float*>(dlogits));
    switch (E / 64) {
      case 1: LAUNCH_B8(1) break;
      case 2: LAUNCH_B8(2) break;
      case 3: LAUNCH_B8(3) break;
      default: LAUNCH_B8(4) break;
    }
#undef LAUNCH_B8
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  if (renorm && E % 64 == 0 && E <= 256 && k <= 16) {
    const int g2 = r3_grid((rows + 1) / 2);
#define LAUNCH_BF(NB)                                                                                  \
  if (dtype == 1)                                                                                      \
    r3_bwd_fast<uint16_t, NB><<<g2, 256, 0, s>>>(rows, static_cast<int>(k), rec_idx, idx_dtype, w, dw, \
                                                 static_cast<uint16_t*>(dlogits));                     \
  else                                                                                                 \
    r3_bwd_fast<float, NB><<<g2, 256, 0, s>>>(rows, static_cast<int>(k), rec_idx, idx_dtype, w, dw,    \
                                              static_cast<float*>(dlogits));
    switch (E / 64) {
      case 1: LAUNCH_BF(1) break;
      case 2: LAUNCH_BF(2) break;
      case 3: LAUNCH_BF(3) break;
      default: LAUNCH_BF(4) break;
    }
#undef LAUNCH_BF
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  const int grid = r3_grid(rows);
#define LAUNCH_B(NPL)                                                                           \
  (dtype == 1 ? (r3_bwd_kernel<uint16_t, NPL><<<grid, 256, 0, s>>>(                             \
                     static_cast<const uint16_t*>(logits), rows, static_cast<int>(E),          \
                     static_cast<int>(k), rec_idx, idx_dtype, renorm, w, dw,                   \
                     static_cast<uint16_t*>(dlogits)),                                          \
                 0)                                                                             \
              : (r3_bwd_kernel<float, NPL><<<grid, 256, 0, s>>>(                                \
                     static_cast<const float*>(logits), rows, static_cast<int>(E),             \
                     static_cast<int>(k), rec_idx, idx_dtype, renorm, w, dw,                   \
                     static_cast<float*>(dlogits)),                                             \
                 0))
  (void)SFTM_R3_NPL(E, LAUNCH_B);
#undef LAUNCH_B
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace sftm
