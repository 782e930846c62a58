// SPDX-License-Identifier: Apache-2.0
//
// Forward-only streaming pass (SURVEY.md §8 row a1, and pass 1 of the two-pass
// vocab-parallel form, a7): per token logp / entropy / lse, or the shard's
// partial statistics — one read of each logits row (2V bytes per bf16 token),
// nothing written but per-token scalars.
//
// sm_100a structure (one CTA per SM, persistent, rows grid-strided):
//   warp 24      TMA producer: cp.async.bulk 12 KB chunks of each row into two
//                8-slot smem rings (192 KB), chunk k of row r into ring (k + r) % 2
//                (rows alternate which group starts, balancing odd chunk counts),
//                L2 evict-first, running ahead across rows.
//   warps 0..23  two groups of 12 forward warps; group g consumes ring g in
//                order (a plain single-consumer ring per group). Each thread folds its 16 elements per chunk into an
//                online softmax state with packed FFMA2/FADD2 + MUFU.EX2 around
//                a fixed exponent base (its first chunk's max); non-finite
//                partials are repaired by re-reading the thread's elements.
//   warps 25,26  control (alternating rows): merge the 24 per-warp partials,
//                read z_target, write logp / H / lse (or the shard stats).
// No barrier spans the CTA: per-row partials travel through a 4-deep
// flow-controlled smem ring, as in the fused kernel (tm_loss.cu).
//
// Replaces: the ActorFwd / RefLogP stage stubs (proj/src/sim_runtime.cpp:322-334,
// proj/src/wall_runtime.cpp:126-129), whose payloads are these logp fields.

#include <cuda_runtime.h>

#include <mutex>
#include <type_traits>

#include "tm_rowmath.cuh"

namespace sftm {
namespace fwd {

constexpr int kGW = 12;                      // warps per forward group
constexpr int kFW = 2 * kGW;                 // forward warps
constexpr int kGT = kGW * 32;                // threads per group (384)
constexpr int kProd = kFW;                   // producer warp
constexpr int kCtl = kFW + 1;                // control warps (2)
constexpr int kThreads = (kFW + 3) * 32;     // 864
constexpr int kCB = kGT * 32;                // chunk bytes: two 16-B vectors per group thread = 12 KB
constexpr int kSlots = 8;                    // slots per group ring
constexpr int kRingBytes = 2 * kSlots * kCB; // 192 KB
constexpr int kRD = 4;                       // per-row partial ring depth

template <typename T>
struct Geo {
  static constexpr int es = sizeof(T);
  static constexpr int CE = kCB / es;
  static constexpr int HALF = CE / 2;
  static constexpr int EV = 16 / es;
  static constexpr int NE = 2 * EV;
};

__device__ __forceinline__ void unpack(const float*, uint4 a, uint4 b, float (&x)[8]) {
  x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y);
  x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
  x[4] = __uint_as_float(b.x); x[5] = __uint_as_float(b.y);
  x[6] = __uint_as_float(b.z); x[7] = __uint_as_float(b.w);
}
__device__ __forceinline__ void unpack(const uint16_t*, uint4 a, uint4 b, float (&x)[16]) {
  x[0] = bf16lo(a.x); x[1] = bf16hi(a.x); x[2] = bf16lo(a.y); x[3] = bf16hi(a.y);
  x[4] = bf16lo(a.z); x[5] = bf16hi(a.z); x[6] = bf16lo(a.w); x[7] = bf16hi(a.w);
  x[8] = bf16lo(b.x); x[9] = bf16hi(b.x); x[10] = bf16lo(b.y); x[11] = bf16hi(b.y);
  x[12] = bf16lo(b.z); x[13] = bf16hi(b.z); x[14] = bf16lo(b.w); x[15] = bf16hi(b.w);
}

template <typename T>
__device__ __forceinline__ int elem_off(int tid, int j) {
  using G = Geo<T>;
  return (j < G::EV) ? (G::EV * tid + j) : (G::HALF + G::EV * tid + (j - G::EV));
}

// UA: rows off 16-B boundaries (odd vocabulary / stride), handled in sector
// coordinates exactly as the fused kernel does (tm_loss.cu): a row starts
// `mis` elements into its first sector; front/tail chunks are masked; the last
// row's final partial sector is loaded by the producer element-wise.
template <typename T, int MODE, bool UA>
__global__ void __launch_bounds__(kThreads, 1) fwd_stream_kernel(const RowArgs a) {
  using G = Geo<T>;
  constexpr int CE = G::CE;
  constexpr int NE = G::NE;
  constexpr int EV = G::EV;

  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ __align__(8) uint64_t full_bar[2][kSlots], empty_bar[2][kSlots];
  __shared__ __align__(16) float4 red[kRD][kFW];
  __shared__ __align__(8) uint64_t red_bar[kRD], red_free[kRD];
  __shared__ uint32_t sink_sh[kFW];

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int64_t cid = blockIdx.x, ncl = gridDim.x;
  const int V = static_cast<int>(a.V);
  const int nck = (V + CE - 1) / CE;
  const uint32_t ring_base = smem_u32(ring);
  const T* logits = static_cast<const T*>(a.logits);
  auto row_mis = [&](int64_t t) -> int {
    if constexpr (UA) {
      return static_cast<int>((reinterpret_cast<uintptr_t>(logits + t * a.ld) & 15u) / G::es);
    } else {
      (void)t;
      return 0;
    }
  };

  if (tid == 0) {
    for (int g = 0; g < 2; ++g)
      for (int i = 0; i < kSlots; ++i) {
        mbar_init(smem_u32(&full_bar[g][i]), 1);
        mbar_init(smem_u32(&empty_bar[g][i]), kGT);  // every thread of the consuming group
      }
    for (int i = 0; i < kRD; ++i) {
      mbar_init(smem_u32(&red_bar[i]), kFW);  // lane 0 of each forward warp
      mbar_init(smem_u32(&red_free[i]), 1);   // lane 0 of the control warp that read it
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kProd) {
    // ================================================================ producer
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      uint32_t slot[2] = {0, 0}, ph[2] = {0, 0};
      uint32_t nrow = 0;
      for (int64_t t = cid; t < a.T; t += ncl, ++nrow) {
        const int mis = row_mis(t);
        const int span = V + mis;
        const int nck_r = UA ? (span + CE - 1) / CE : nck;
        const T* row = logits + t * a.ld - mis;
        for (int k = 0; k < nck_r; ++k) {
          const int g = (k + static_cast<int>(nrow)) & 1;  // alternate the first group per row
          const int rem = span - k * CE;
          uint32_t bytes = static_cast<uint32_t>(rem < CE ? rem : CE) * G::es;
          int tail = 0;
          if constexpr (UA) {
            if ((bytes & 15u) && t == a.T - 1 && k == nck_r - 1) {
              tail = static_cast<int>((bytes & 15u) / G::es);  // never read past the tensor
              bytes &= ~15u;
            } else {
              bytes = (bytes + 15u) & ~15u;
            }
          }
          mbar_wait(smem_u32(&empty_bar[g][slot[g]]), ph[g] ^ 1u);
          if constexpr (UA) {
            const T* tp = row + static_cast<int64_t>(k) * CE + bytes / G::es;
            T* td = reinterpret_cast<T*>(ring + (g * kSlots + slot[g]) * kCB + bytes);
            for (int j = 0; j < tail; ++j) td[j] = tp[j];
          }
          mbar_arrive_expect_tx(smem_u32(&full_bar[g][slot[g]]), bytes);
          if (bytes)
            bulk_g2s(ring_base + (g * kSlots + slot[g]) * kCB, row + static_cast<int64_t>(k) * CE, bytes,
                     smem_u32(&full_bar[g][slot[g]]), pol);
          if (++slot[g] == kSlots) {
            slot[g] = 0;
            ph[g] ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < kFW) {
    // ================================================================ forward
    const int grp = warp / kGW;           // chunk parity this group consumes
    const int gtid = tid - grp * kGT;     // 0..kGT-1 within the group
    const float c = a.inv_tau * kLog2e;
    const uint32_t ring_t = ring_base + grp * kSlots * kCB + 16u * gtid;
    const uint32_t full0 = smem_u32(&full_bar[grp][0]), empty0 = smem_u32(&empty_bar[grp][0]);
    const uint32_t sink_a = smem_u32(&sink_sh[warp]);
    uint32_t slot = 0, ph = 0, nrow = 0;
    for (int64_t t = cid; t < a.T; t += ncl) {
      const int mis = row_mis(t);
      const int span = V + mis;
      const int nck_r = UA ? (span + CE - 1) / CE : nck;
      float m2 = 0.f;
      bool have = false;
      float2 s2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      float2 w2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const int k0 = (grp + static_cast<int>(nrow)) & 1;  // rows alternate which group starts
      for (int k = k0; k < nck_r; k += 2) {
        mbar_wait(full0 + 8u * slot, ph);
        const uint32_t sa = ring_t + slot * kCB;
        const uint4 v0 = lds128(sa);
        const uint4 v1 = lds128(sa + kCB / 2);
        float x[NE];
        unpack(logits, v0, v1, x);
        const int rem = span - k * CE;
        const int lo = (UA && k == 0) ? mis : 0;
        const bool partial = rem < CE || lo > 0;
        if (!have) {
          // exponent base: this thread's max of its first chunk in the row
          float xm = -INFINITY;
#pragma unroll
          for (int j = 0; j < NE; ++j) {
            const int pj = elem_off<T>(gtid, j);
            if (!partial || (pj >= lo && pj < rem)) xm = fmaxf(xm, x[j]);
          }
          m2 = xm * c;
          if (!(m2 > -INFINITY)) m2 = 0.f;
          have = true;
        }
        const float2 c2 = make_float2(c, c), nm2 = make_float2(-m2, -m2);
        if (!partial) {
#pragma unroll
          for (int p = 0; p < NE / 2; ++p) {
            const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nm2);
            const float2 e = make_float2(ex2(av.x), ex2(av.y));
            s2[p & 1] = __fadd2_rn(s2[p & 1], e);
            w2[p & 1] = __ffma2_rn(e, av, w2[p & 1]);
          }
        } else if (UA) {
          // packed math on vectors wholly inside the row, element masks on the
          // (at most two) boundary vectors
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int p0 = v * G::HALF + EV * gtid;
            if (p0 >= lo && p0 + EV <= rem) {
#pragma unroll
              for (int q = 0; q < EV / 2; ++q) {
                const int p = v * (EV / 2) + q;
                const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nm2);
                const float2 e = make_float2(ex2(av.x), ex2(av.y));
                s2[p & 1] = __fadd2_rn(s2[p & 1], e);
                w2[p & 1] = __ffma2_rn(e, av, w2[p & 1]);
              }
            } else if (p0 + EV > lo && p0 < rem) {
#pragma unroll
              for (int j = 0; j < EV; ++j) {
                const int pj = p0 + j;
                if (pj >= lo && pj < rem && x[v * EV + j] != -INFINITY) {
                  const float av = fmaf(x[v * EV + j], c, -m2);
                  const float e = ex2(av);
                  s2[0].x += e;
                  w2[0].x = fmaf(e, av, w2[0].x);
                }
              }
            }
          }
        } else {
          // vector-granular tail (slice lengths are multiples of the 16-B vector)
          const bool ok0 = EV * gtid < rem, ok1 = G::HALF + EV * gtid < rem;
#pragma unroll
          for (int p = 0; p < NE / 2; ++p) {
            if ((2 * p < EV) ? ok0 : ok1) {
              const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nm2);
              const float2 e = make_float2(ex2(av.x), ex2(av.y));
              s2[p & 1] = __fadd2_rn(s2[p & 1], e);
              w2[p & 1] = __ffma2_rn(e, av, w2[p & 1]);
            }
          }
        }
        // release the slot only after the loaded values fed a store (the arrive
        // would otherwise issue ahead of the LDS; see tm_loss.cu)
        sink_u32(sink_a, __float_as_uint(s2[0].x) ^ __float_as_uint(w2[1].y));
        mbar_arrive(empty0 + 8u * slot);
        if (++slot == kSlots) {
          slot = 0;
          ph ^= 1u;
        }
      }
      Stats my{m2, (s2[0].x + s2[1].x) + (s2[0].y + s2[1].y), (w2[0].x + w2[1].x) + (w2[0].y + w2[1].y)};
      if (!have) my = stats_empty();
      // Repair (rare): -inf logits or an exponent overflow made s or w non-finite:
      // recompute this thread's partials exactly from global memory.
      const bool bad = !(fabsf(my.s) <= 3.0e38f) || !(fabsf(my.w) <= 3.0e38f);
      if (__any_sync(0xffffffffu, bad)) {
        const T* row = logits + t * a.ld - mis;  // sector coordinates
        float mx = -INFINITY;
        for (int k = k0; k < nck_r; k += 2) {
          const int rem = span - k * CE, lo = (UA && k == 0) ? mis : 0;
#pragma unroll
          for (int j = 0; j < NE; ++j) {
            const int o = elem_off<T>(gtid, j);
            if (o >= lo && o < rem) mx = fmaxf(mx, ldg_elem(row, static_cast<int64_t>(k) * CE + o));
          }
        }
        const float mb2 = (mx == -INFINITY) ? -INFINITY : mx * c;
        float sr = 0.f, wr = 0.f;
        for (int k = k0; k < nck_r; k += 2) {
          const int rem = span - k * CE, lo = (UA && k == 0) ? mis : 0;
#pragma unroll
          for (int j = 0; j < NE; ++j) {
            const int o = elem_off<T>(gtid, j);
            if (o >= lo && o < rem) {
              const float xv = ldg_elem(row, static_cast<int64_t>(k) * CE + o);
              if (xv != -INFINITY) {
                const float av = fmaf(xv, c, -mb2);
                const float e = ex2(av);
                sr += e;
                wr = fmaf(e, av, wr);
              }
            }
          }
        }
        if (bad) my = Stats{mb2, sr, wr};
      }
      if (my.s == 0.f) my = stats_empty();
      my = warp_merge(my);
      if (lane == 0) {
        mbar_wait(smem_u32(&red_free[nrow % kRD]), ((nrow / kRD) & 1u) ^ 1u);
        red[nrow % kRD][warp] = make_float4(my.m2, my.s, my.w, 0.f);
        mbar_arrive(smem_u32(&red_bar[nrow % kRD]));
      }
      ++nrow;
    }
  } else {
    // ================================================================ control
    const int ci = warp - kCtl;
    uint32_t nrow = 0;
    for (int64_t t = cid; t < a.T; t += ncl, ++nrow) {
      if (static_cast<int>(nrow & 1u) != ci) continue;
      const uint32_t rs = nrow % kRD;
      const int64_t yl = static_cast<int64_t>(__ldg(a.targets + t)) - a.vocab_start;
      float zy = __int_as_float(0x7fc00000);
      if (yl >= 0 && yl < a.V) zy = ldg_elem(logits, t * a.ld + yl) * a.inv_tau;
      mbar_wait(smem_u32(&red_bar[rs]), (nrow / kRD) & 1u);
      Stats v = stats_empty();
      if (lane < kFW) {
        const float4 r = red[rs][lane];
        v = Stats{r.x, r.y, r.z};
      }
      v = warp_merge(v);
      if (lane == 0) {
        mbar_arrive(smem_u32(&red_free[rs]));  // the shuffles consumed every lane's read
        if (MODE == kModeVpStats) {
          reinterpret_cast<float4*>(a.out_stats)[t] = make_float4(v.m2 * kLn2, v.s, v.w * kLn2, zy);
        } else {
          float lse2, lse, H, logp;
          row_scalars(v, zy, lse2, lse, H, logp);
          if (a.out_logp) a.out_logp[t] = logp;
          if (a.out_entropy) a.out_entropy[t] = H;
          if (a.out_lse) a.out_lse[t] = lse;
        }
      }
    }
  }
}

std::mutex g_mu;

template <typename T, int MODE, bool UA>
int launch(const RowArgs& a, cudaStream_t s, LaunchInfo* info) {
  auto kern = fwd_stream_kernel<T, MODE, UA>;
  static PerDevice cache;  // per instantiation and device
  int& sms = cache();
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (sms < 0) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingBytes);
      if (e != cudaSuccess) return e;
      int dev = 0, n = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
      sms = n;
    }
  }
  const int grid = static_cast<int>(a.T < sms ? a.T : sms);
  if (grid < 1) return cudaSuccess;
  kern<<<grid, kThreads, kRingBytes, s>>>(a);
  if (info) {
    info->kernel = 5;
    info->cluster = 1;
    info->grid = grid;
    info->launches = 1;
  }
  return cudaGetLastError();
}

}  // namespace fwd

// Forward-only streaming pass for kModeFwd / kModeVpStats; rows off 16-B
// boundaries run in sector coordinates (UA).
int launch_fwd_stream(const RowArgs& a, int mode, cudaStream_t s, LaunchInfo* info) {
  if (a.V > (int64_t(1) << 30)) return -2;
  const int es = a.dtype == 1 ? 2 : 4;
  const uintptr_t base = reinterpret_cast<uintptr_t>(a.logits);
  if (base % es) return -2;
  const bool ua = (base % 16) || ((a.ld * es) % 16) || ((a.V * es) % 16);
  auto go = [&](auto tag, auto ua_c) -> int {
    using T = decltype(tag);
    constexpr bool U = decltype(ua_c)::value;
    return mode == kModeVpStats ? fwd::launch<T, kModeVpStats, U>(a, s, info) : fwd::launch<T, kModeFwd, U>(a, s, info);
  };
  if (a.dtype == 1) return ua ? go(uint16_t{}, std::true_type{}) : go(uint16_t{}, std::false_type{});
  return ua ? go(float{}, std::true_type{}) : go(float{}, std::false_type{});
}

}  // namespace sftm
