// SPDX-License-Identifier: Apache-2.0
//
// Vocab-row kernels of the train-math hot path
// and the dispatch that picks one per call (launch_rows, bottom of this file):
//
//   loss_tmem_kernel (tm_loss.cu)  — fused loss fwd+bwd (kModeFwdBwd), any
//                        element-aligned rows (16-B aligned, or in sector
//                        coordinates when not) whose slice fits the row store.
//   fwd_stream_kernel (tm_fwd.cu)  — forward only (kModeFwd, kModeVpStats).
//   rows_ring_kernel   — a TMA-ring streaming kernel with 16 compute warps: the
//                        two-pass vocab-parallel shard backward (kModeVpBwd), and
//                        the forward modes when the streaming kernel cannot take them.
//   rows_generic_kernel — fallback for what the above cannot take (dlogits at a
//                        different 16-B phase than the logits, rows too wide
//                        for any row store, unaligned rows in kModeVpBwd): two
//                        passes over global memory (the second served from L2),
//                        same math, same outputs.
//
// The per-row math (lse, entropy, logp, DAPO/GRPO surrogate, k3 KL, gradients)
// is pinned in DESIGN.md §2 and restated in fp64 by oracle/sf_oracle.c
// (orc_pg_loss_fwd_bwd). The reference has no implementation of this path:
// it is the latency stub at proj/src/sim_runtime.cpp:441 /
// proj/src/wall_runtime.cpp:197 (see include/staleflow/train_math.h).

#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <string>

#include "tm_rowmath.cuh"

namespace sftm {

constexpr int kCW = 16;                   // compute warps
constexpr int kCT = kCW * 32;             // compute threads
constexpr int kThreads = kCT + 32;        // + one TMA producer warp
constexpr int kEPT = 8;                   // elements per thread per chunk
constexpr int kChunkElems = kCT * kEPT;   // 4096 elements per ring chunk
constexpr int kMaxSlots = 32;
constexpr int kStreamRingBytes = 96 * 1024;

// ===========================================================================
// The TMA-ring kernel.
// ===========================================================================
template <typename T, int C, int MODE, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    rows_ring_kernel(const RowArgs a, int64_t slice_elems, int nslots) {
  constexpr int es = Elem<T>::es;
  constexpr int CB = kChunkElems * es;  // chunk bytes
  constexpr bool kLoss = (MODE == kModeFwdBwd || MODE == kModeVpBwd);
  constexpr bool kResident = (MODE == kModeFwdBwd);

  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ __align__(8) uint64_t full_bar[kMaxSlots];
  __shared__ __align__(8) uint64_t empty_bar[kMaxSlots];
  __shared__ __align__(8) uint64_t mail_bar[2];
  __shared__ __align__(16) float4 mail[2][8];
  __shared__ __align__(16) float4 red[kCW];

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const uint32_t crank = (C > 1) ? cluster_ctarank() : 0u;
  const int64_t cid = (C > 1) ? static_cast<int64_t>(cluster_id_x()) : blockIdx.x;
  const int64_t ncl = (C > 1) ? static_cast<int64_t>(nclusters_x()) : gridDim.x;
  const int64_t slice_start = static_cast<int64_t>(crank) * slice_elems;
  int64_t slice_len = a.V - slice_start;
  if (slice_len > slice_elems) slice_len = slice_elems;
  if (slice_len < 0) slice_len = 0;
  const int nck = static_cast<int>((slice_len + kChunkElems - 1) / kChunkElems);
  const uint32_t ring_base = smem_u32(ring);

  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), kCW);
    }
    mbar_init(smem_u32(&mail_bar[0]), C);
    mbar_init(smem_u32(&mail_bar[1]), C);
    fence_mbar_init();
  }
  if (C > 1) {
    cluster_sync_all();
  } else {
    __syncthreads();
  }

  const T* logits = static_cast<const T*>(a.logits);

  if (warp == kCW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      uint32_t slot = 0, ph = 0;
      for (int64_t t = cid; t < a.T; t += ncl) {
        if (kLoss) {
          if (__ldg(a.w_tok + t) == 0.f) continue;
        }
        const T* row = logits + t * a.ld + slice_start;
        for (int k = 0; k < nck; ++k) {
          int64_t ce = slice_len - static_cast<int64_t>(k) * kChunkElems;
          if (ce > kChunkElems) ce = kChunkElems;
          const uint32_t bytes = static_cast<uint32_t>(ce) * es;
          mbar_wait(smem_u32(&empty_bar[slot]), ph ^ 1u);
          mbar_arrive_expect_tx(smem_u32(&full_bar[slot]), bytes);
          bulk_g2s(ring_base + slot * CB, row + static_cast<int64_t>(k) * kChunkElems, bytes,
                   smem_u32(&full_bar[slot]), pol);
          if (++slot == static_cast<uint32_t>(nslots)) {
            slot = 0;
            ph ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ consumers
    const float c = a.inv_tau * kLog2e;
    const LossParamsDev P{a.eps_lo, a.eps_hi, a.dual_c, a.beta, a.ent_coef, a.kl_mode};
    uint32_t slot = 0, ph = 0, nrow = 0;
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const bool leader = (crank == 0 && tid == 0);
    const int e0 = tid * kEPT;

    for (int64_t t = cid; t < a.T; t += ncl) {
      float w = 1.f, A = 0.f, old = 0.f, ref = 0.f;
      if (kLoss) {
        w = __ldg(a.w_tok + t);
        if (w == 0.f) {
          if (!a.masked_skip) {
            uint8_t* drow = static_cast<uint8_t*>(a.dlogits) + (t * a.ld_d + slice_start) * es;
            const int64_t nb = slice_len * es;
            for (int64_t off = static_cast<int64_t>(tid) * 16; off < nb; off += kCT * 16)
              stg128_cs(drow + off, make_uint4(0, 0, 0, 0));
          }
          if (leader) {
            if (a.out_logp) a.out_logp[t] = 0.f;
            if (a.out_entropy) a.out_entropy[t] = 0.f;
          }
          continue;
        }
        A = __ldg(a.adv_tok + t);
        old = __ldg(a.old_logp + t);
        ref = __ldg(a.ref_logp + t);
      }
      const int64_t y = static_cast<int64_t>(__ldg(a.targets + t));
      const int64_t yl = y - a.vocab_start;  // column of the target in this kernel's rows
      float zy = __int_as_float(0x7fc00000);   // NaN: target not in these columns
      if (MODE != kModeVpBwd) {
        if (yl >= 0 && yl < a.V) zy = ldg_elem(logits, t * a.ld + yl) * a.inv_tau;
      }

      Stats st;
      const uint32_t s0 = slot;
      if (MODE != kModeVpBwd) {
        Stats my = stats_empty();
        for (int k = 0; k < nck; ++k) {
          mbar_wait(smem_u32(&full_bar[slot]), ph);
          int64_t ce = slice_len - static_cast<int64_t>(k) * kChunkElems;
          if (ce > kChunkElems) ce = kChunkElems;
          if (e0 < ce) {
            float x[8];
            lds8(logits, ring_base + slot * CB + e0 * es, x);
            if (e0 + kEPT > ce) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (e0 + j >= ce) x[j] = -INFINITY;
            }
            accum8(my, x, c);
          }
          if (!kResident) {
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&empty_bar[slot]));
          }
          if (++slot == static_cast<uint32_t>(nslots)) {
            slot = 0;
            ph ^= 1u;
          }
        }
        // CTA reduction, then cluster exchange through DSMEM mailboxes.
        my = warp_merge(my);
        if (lane == 0) red[warp] = make_float4(my.m2, my.s, my.w, 0.f);
        named_bar_sync(1, kCT);
        const uint32_t b = nrow & 1u;
        if (warp == 0) {
          Stats v = stats_empty();
          if (lane < kCW) {
            const float4 r = red[lane];
            v = Stats{r.x, r.y, r.z};
          }
          v = warp_merge(v);
          if (lane == 0) {
            if (C == 1) {
              mail[b][0] = make_float4(v.m2, v.s, v.w, 0.f);
              mbar_arrive(smem_u32(&mail_bar[b]));
            } else {
              const uint32_t my_slot = smem_u32(&mail[b][crank]);
              const uint32_t my_bar = smem_u32(&mail_bar[b]);
#pragma unroll
              for (int q = 0; q < C; ++q) {
                st_cluster_v4(mapa(my_slot, q), v.m2, v.s, v.w, 0.f);
                mbar_arrive_remote(mapa(my_bar, q));
              }
            }
          }
        }
        const uint32_t par = (nrow >> 1) & 1u;
        if (C == 1) {
          mbar_wait(smem_u32(&mail_bar[b]), par);
        } else {
          mbar_wait_cluster(smem_u32(&mail_bar[b]), par);
        }
        st = stats_empty();
#pragma unroll
        for (int q = 0; q < C; ++q) {
          const float4 mv = mail[b][q];
          st = stats_merge(st, Stats{mv.x, mv.y, mv.z});
        }
        if (MODE == kModeVpStats) {
          if (tid == 0) {
            reinterpret_cast<float4*>(a.out_stats)[t] =
                make_float4(st.m2 * kLn2, st.s, st.w * kLn2, zy);
          }
          ++nrow;
          continue;
        }
      } else {
        // kModeVpBwd: merge the all-gathered per-shard statistics in rank order.
        st = stats_empty();
        for (int p = 0; p < a.P; ++p) {
          const float4 g = __ldg(reinterpret_cast<const float4*>(a.gathered) + p * a.T + t);
          st = stats_merge(st, Stats{g.x * kLog2e, g.y, g.z * kLog2e});
          if (!(g.w != g.w)) zy = g.w;
        }
      }

      float lse2, lse, H, logp;
      row_scalars(st, zy, lse2, lse, H, logp);
      if (MODE == kModeFwd) {
        if (tid == 0) {
          if (a.out_logp) a.out_logp[t] = logp;
          if (a.out_entropy) a.out_entropy[t] = H;
          if (a.out_lse) a.out_lse[t] = lse;
        }
        ++nrow;
        continue;
      }

      float g, gH, m[8];
      loss_terms(logp, H, w, A, old, ref, P, g, gH, m);
      if (leader) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += static_cast<double>(m[i]);
        if (a.out_logp) a.out_logp[t] = logp;
        if (a.out_entropy) a.out_entropy[t] = H;
      }
      // dlogits_v = g/tau*[v==y] - p_v*(c0 + c1*a_v),  a_v = (z_v - lse)*log2e.
      const float gt = a.inv_tau * g;
      const float c0 = a.inv_tau * (g + gH * H);
      const float c1 = a.inv_tau * gH * kLn2;
      const int64_t kt = yl - slice_start;
      int ck = -1, tt = -1, jt = 0;
      if (kt >= 0 && kt < slice_len) {
        ck = static_cast<int>(kt / kChunkElems);
        const int r = static_cast<int>(kt % kChunkElems);
        tt = r / kEPT;
        jt = r % kEPT;
      }
      T* drow = static_cast<T*>(a.dlogits) + t * a.ld_d + slice_start;
      uint32_t bslot = s0;
      for (int k = 0; k < nck; ++k) {
        uint32_t use;
        if (kResident) {
          use = bslot;
          if (++bslot == static_cast<uint32_t>(nslots)) bslot = 0;
        } else {
          mbar_wait(smem_u32(&full_bar[slot]), ph);
          use = slot;
          if (++slot == static_cast<uint32_t>(nslots)) {
            slot = 0;
            ph ^= 1u;
          }
        }
        int64_t ce = slice_len - static_cast<int64_t>(k) * kChunkElems;
        if (ce > kChunkElems) ce = kChunkElems;
        if (e0 < ce) {
          float x[8], gr[8];
          lds8(logits, ring_base + use * CB + e0 * es, x);
          if (c1 == 0.f) {
#pragma unroll
            for (int j = 0; j < 8; ++j) gr[j] = -ex2(fmaf(x[j], c, -lse2)) * c0;
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float av = fmaxf(fmaf(x[j], c, -lse2), -127.f);
              gr[j] = -ex2(av) * fmaf(c1, av, c0);
            }
          }
          if (k == ck && tid == tt) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j == jt) gr[j] += gt;
          }
          T* dst = drow + static_cast<int64_t>(k) * kChunkElems + e0;
          if (e0 + kEPT <= ce) {
            st8(dst, gr);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (e0 + j < ce) st1(dst + j, gr[j]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty_bar[use]));
      }
      ++nrow;
    }
    if (kLoss && leader) finish_metrics(a, cid, ncl, acc);
  }

  if (C > 1) {
    __syncwarp();
    cluster_sync_all();
  }
}

// ===========================================================================
// Generic two-pass kernel (any alignment / width). 256 threads, one row per
// block iteration; second pass re-reads the row (L2-resident at this size).
// ===========================================================================
constexpr int kGT = 256;

template <typename T, int MODE>
__global__ void __launch_bounds__(kGT) rows_generic_kernel(const RowArgs a) {
  constexpr bool kLoss = (MODE == kModeFwdBwd || MODE == kModeVpBwd);
  __shared__ float4 red[kGT / 32];
  __shared__ float4 bc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const T* logits = static_cast<const T*>(a.logits);
  const float c = a.inv_tau * kLog2e;
  const LossParamsDev P{a.eps_lo, a.eps_hi, a.dual_c, a.beta, a.ent_coef, a.kl_mode};
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};

  for (int64_t t = blockIdx.x; t < a.T; t += gridDim.x) {
    float w = 1.f, A = 0.f, old = 0.f, ref = 0.f;
    if (kLoss) {
      w = a.w_tok[t];
      if (w == 0.f) {
        if (!a.masked_skip) {
          T* drow = static_cast<T*>(a.dlogits) + t * a.ld_d;
          for (int64_t v = tid; v < a.V; v += kGT) st1(drow + v, 0.f);
        }
        if (tid == 0) {
          if (a.out_logp) a.out_logp[t] = 0.f;
          if (a.out_entropy) a.out_entropy[t] = 0.f;
        }
        continue;
      }
      A = a.adv_tok[t];
      old = a.old_logp[t];
      ref = a.ref_logp[t];
    }
    const T* row = logits + t * a.ld;
    const int64_t yl = static_cast<int64_t>(a.targets[t]) - a.vocab_start;
    float zy = __int_as_float(0x7fc00000);
    Stats st;
    if (MODE != kModeVpBwd) {
      if (yl >= 0 && yl < a.V) zy = ldg_elem(logits, t * a.ld + yl) * a.inv_tau;
      Stats my = stats_empty();
      for (int64_t v0 = static_cast<int64_t>(tid) * 8; v0 < a.V; v0 += kGT * 8) {
        float x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = (v0 + j < a.V) ? ldg_elem(row, v0 + j) : -INFINITY;
        accum8(my, x, c);
      }
      my = warp_merge(my);
      if (lane == 0) red[warp] = make_float4(my.m2, my.s, my.w, 0.f);
      __syncthreads();
      if (warp == 0) {
        Stats v = stats_empty();
        if (lane < kGT / 32) v = Stats{red[lane].x, red[lane].y, red[lane].z};
        v = warp_merge(v);
        if (lane == 0) bc = make_float4(v.m2, v.s, v.w, 0.f);
      }
      __syncthreads();
      st = Stats{bc.x, bc.y, bc.z};
      __syncthreads();  // bc / red reused next row
      if (MODE == kModeVpStats) {
        if (tid == 0)
          reinterpret_cast<float4*>(a.out_stats)[t] =
              make_float4(st.m2 * kLn2, st.s, st.w * kLn2, zy);
        continue;
      }
    } else {
      st = stats_empty();
      for (int p = 0; p < a.P; ++p) {
        const float4 g = reinterpret_cast<const float4*>(a.gathered)[p * a.T + t];
        st = stats_merge(st, Stats{g.x * kLog2e, g.y, g.z * kLog2e});
        if (!(g.w != g.w)) zy = g.w;
      }
    }
    float lse2, lse, H, logp;
    row_scalars(st, zy, lse2, lse, H, logp);
    if (MODE == kModeFwd) {
      if (tid == 0) {
        if (a.out_logp) a.out_logp[t] = logp;
        if (a.out_entropy) a.out_entropy[t] = H;
        if (a.out_lse) a.out_lse[t] = lse;
      }
      continue;
    }
    float g, gH, m[8];
    loss_terms(logp, H, w, A, old, ref, P, g, gH, m);
    if (tid == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += static_cast<double>(m[i]);
      if (a.out_logp) a.out_logp[t] = logp;
      if (a.out_entropy) a.out_entropy[t] = H;
    }
    const float gt = a.inv_tau * g;
    const float c0 = a.inv_tau * (g + gH * H);
    const float c1 = a.inv_tau * gH * kLn2;
    T* drow = static_cast<T*>(a.dlogits) + t * a.ld_d;
    for (int64_t v = tid; v < a.V; v += kGT) {
      const float x = ldg_elem(row, v);
      const float av = fmaxf(fmaf(x, c, -lse2), -127.f);
      float gr = -ex2(av) * fmaf(c1, av, c0);
      if (v == yl) gr += gt;
      st1(drow + v, gr);
    }
  }
  if (kLoss && tid == 0) finish_metrics(a, blockIdx.x, gridDim.x, acc);
}

// ===========================================================================
// Host-side launch logic.
// ===========================================================================
int launch_loss_tmem(const RowArgs& a, cudaStream_t s, LaunchInfo* info);  // tm_loss.cu

namespace {

std::atomic<bool> g_force_generic{false};
std::mutex g_mu;

struct DevInfo {
  int sms = 0;
};

DevInfo dev_info() {
  int dev = 0;
  cudaGetDevice(&dev);
  DevInfo d;
  cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
  return d;
}

template <typename T, int C, int MODE, int MINB>
int launch_ring(const RowArgs& a, int64_t slice_elems, int nslots, int ring_bytes,
                cudaStream_t s, LaunchInfo* info) {
  auto kern = rows_ring_kernel<T, C, MODE, MINB>;
  static PerDevice cache;  // per instantiation and device
  int& max_active = cache();
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (max_active < 0) {
      cudaError_t e =
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ring_bytes);
      if (e != cudaSuccess) return e;
      if (C > 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C * 256);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = ring_bytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
        if (e != cudaSuccess) return e;
        max_active = n;
      } else {
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, ring_bytes);
        if (e != cudaSuccess) return e;
        max_active = per_sm * dev_info().sms;
      }
      if (max_active <= 0) return cudaErrorInvalidConfiguration;
    }
  }
  int64_t ncl = a.T < max_active ? a.T : max_active;
  if (ncl > a.max_partial_blocks) ncl = a.max_partial_blocks;
  if (ncl < 1) ncl = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(ncl * C));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = ring_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (C > 1) ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, slice_elems, nslots);
  if (info) {
    info->kernel = 0;
    info->cluster = C;
    info->grid = static_cast<int>(ncl * C);
    info->launches = 1;
  }
  return e;
}

template <typename T, int MODE>
int launch_generic(const RowArgs& a, cudaStream_t s, LaunchInfo* info) {
  int64_t grid = dev_info().sms * 8;
  if (grid > a.T) grid = a.T;
  if (grid > a.max_partial_blocks) grid = a.max_partial_blocks;
  if (grid < 1) grid = 1;
  rows_generic_kernel<T, MODE><<<static_cast<unsigned>(grid), kGT, 0, s>>>(a);
  if (info) {
    info->kernel = 1;
    info->cluster = 1;
    info->grid = static_cast<int>(grid);
    info->launches = 1;
  }
  return cudaGetLastError();
}

template <typename T>
int dispatch(const RowArgs& a, int mode, cudaStream_t s, std::string* err, LaunchInfo* info) {
  constexpr int es = Elem<T>::es;
  const bool aligned_in = (reinterpret_cast<uintptr_t>(a.logits) % 16 == 0) &&
                          ((a.ld * es) % 16 == 0) && ((a.V * es) % 16 == 0);
  bool aligned_out = true;
  if (mode == kModeFwdBwd || mode == kModeVpBwd)
    aligned_out = (reinterpret_cast<uintptr_t>(a.dlogits) % 16 == 0) && ((a.ld_d * es) % 16 == 0);
  const bool ring_ok = !g_force_generic && aligned_in && aligned_out;
  const int CB = kChunkElems * es;
  // The fused loss also takes rows off 16-B boundaries (odd vocabularies or
  // strides) as long as dlogits rows sit at the same sector phase as the logits
  // rows (same base alignment mod 16, stride difference a multiple of 16 B).
  const uintptr_t lb = reinterpret_cast<uintptr_t>(a.logits), db = reinterpret_cast<uintptr_t>(a.dlogits);
  const bool ua_ok = !g_force_generic && mode == kModeFwdBwd && lb % es == 0 && db % es == 0 &&
                     (lb % 16) == (db % 16) && (((a.ld_d - a.ld) * es) % 16 == 0);

  // forward-only modes: any element-aligned rows (unaligned ones in sector coordinates)
  const bool fwd_ok = !g_force_generic && (mode == kModeFwd || mode == kModeVpStats) && lb % es == 0;
  if (ring_ok || ua_ok || fwd_ok) {
    if (mode == kModeFwdBwd) {
      const int e = launch_loss_tmem(a, s, info);
      if (e != -2) return e;  // -2: slice too wide for TMEM residency -> generic
    } else {
      // forward-only modes: the 24-warp streaming kernel (tm_fwd.cu)
      if (mode == kModeFwd || mode == kModeVpStats) {
        const int e = launch_fwd_stream(a, mode, s, info);
        if (e != -2) return e;
      }
      const int nslots = kStreamRingBytes / CB;
      const int ring_bytes = nslots * CB;
      if (ring_ok) {  // the ring kernel needs 16-B aligned rows
        switch (mode) {
          case kModeFwd: return launch_ring<T, 1, kModeFwd, 2>(a, a.V, nslots, ring_bytes, s, info);
          case kModeVpStats:
            return launch_ring<T, 1, kModeVpStats, 2>(a, a.V, nslots, ring_bytes, s, info);
          case kModeVpBwd:
            return launch_ring<T, 1, kModeVpBwd, 2>(a, a.V, nslots, ring_bytes, s, info);
        }
      }
    }
  }
  switch (mode) {
    case kModeFwd: return launch_generic<T, kModeFwd>(a, s, info);
    case kModeFwdBwd: return launch_generic<T, kModeFwdBwd>(a, s, info);
    case kModeVpStats: return launch_generic<T, kModeVpStats>(a, s, info);
    case kModeVpBwd: return launch_generic<T, kModeVpBwd>(a, s, info);
  }
  if (err) *err = "unknown row mode";
  return -1;
}

}  // namespace

void set_force_generic(bool on) { g_force_generic = on; }

namespace {
unsigned long long* g_dbg = nullptr;
}
void set_debug_counters(unsigned long long* p) { g_dbg = p; }
unsigned long long* debug_counters() { return g_dbg; }

int launch_rows(const RowArgs& a, int mode, cudaStream_t s, std::string* err, LaunchInfo* info) {
  if (a.dtype == 1) return dispatch<uint16_t>(a, mode, s, err, info);
  return dispatch<float>(a, mode, s, err, info);
}

}  // namespace sftm
