// SPDX-License-Identifier: Apache-2.0
//
// Fused hot path, v3 schedule (SURVEY.md §8 rows a1 + a4 + a2): same math and
// single-HBM-pass contract as tm_loss.cu, different warp schedule.
//
//   warp 16     TMA producer (cp.async.bulk 16 KB chunks -> 12-slot smem ring)
//   warp 17     control: per row, merge the 16 warp partials, exchange with the
//               cluster through DSMEM mailboxes, load z_target from HBM, compute
//               the loss scalars once and publish them in smem
//   warps 0..15 compute, EVERY warp does both halves of the row math,
//               software-pipelined by chunk: step n runs
//                 for k: backward(row n-1, chunk k-D)   (tcgen05.ld its own
//                        TMEM words -> dlogits -> HBM)
//                        forward(row n, chunk k)       (smem -> tcgen05.st its
//                        own TMEM words -> online softmax partials)
//               so a warp only ever re-reads the TMEM columns it wrote itself
//               (no cross-warp TMEM hand-off, no tfull/tempty barriers), the
//               MUFU work of both halves interleaves inside every warp, and the
//               D-chunk lag hides the row-statistics exchange of row n-1.
//
// TMEM holds 16 slots x 16 KB (all 512 columns): a 2-CTA Qwen3 bf16 row slice is
// 10 slots, so D = min(4, 16 - nck) chunks of lag fit.
//
// Seam replaced and math: see tm_loss.cu / DESIGN.md §2 (fp64 twin in
// oracle/sf_oracle.c orc_pg_loss_fwd_bwd).

#include <cuda_runtime.h>

#include <mutex>

#include "tm_rowmath.cuh"

namespace sftm {
namespace loss3 {

constexpr int kCW = 16;                        // compute warps (4 per SM sub-partition)
constexpr int kCT = kCW * 32;                  // 512 compute threads
constexpr int kProd = kCW;                     // producer warp
constexpr int kCtl = kCW + 1;                  // control warp
constexpr int kThreads = (kCW + 2) * 32;       // 576
constexpr int kCB = kCT * 32;                  // 16 KB chunk: two 16-B vectors per thread
constexpr int kSlots = 12;                     // smem ring (192 KB)
constexpr int kRingBytes = kSlots * kCB;
constexpr int kSlotCols = kCB / (128 * 4);     // 32 TMEM columns per chunk slot
constexpr int kTSlots = 512 / kSlotCols;       // 16 TMEM slots = 256 KB
constexpr int kTCols = 512;
constexpr int kMailD = 8;
constexpr int kRD = 4;
constexpr int kMaxLag = 4;
constexpr int kMinLag = 2;

template <typename T>
struct Geo {
  static constexpr int es = sizeof(T);
  static constexpr int CE = kCB / es;   // elements per chunk
  static constexpr int HALF = CE / 2;   // a thread's second vector starts here
  static constexpr int EV = 16 / es;    // elements per 16-B vector
  static constexpr int NE = 2 * EV;     // elements per thread per chunk
};

struct RowScal {
  float lse2, lse2f, c0, c1, gt;
  int yl;
  uint32_t sgn;
  float pad;
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
__device__ __forceinline__ void store_vec(float* p, const float* g) {
  stg128_cs(p, make_uint4(__float_as_uint(g[0]), __float_as_uint(g[1]), __float_as_uint(g[2]),
                          __float_as_uint(g[3])));
}
__device__ __forceinline__ void store_vec(uint16_t* p, const float* g) {
  stg128_cs(p, make_uint4(pack_bf16x2(g[0], g[1]), pack_bf16x2(g[2], g[3]),
                          pack_bf16x2(g[4], g[5]), pack_bf16x2(g[6], g[7])));
}

// Next row >= t of this cluster's strided row sequence with w != 0 (or T).
// Warp-collective: 32 rows are probed per load round.
__device__ __forceinline__ int64_t next_active(const float* __restrict__ w, int64_t t, int64_t ncl,
                                               int64_t T, int lane) {
  while (t < T) {
    const int64_t tl = t + lane * ncl;
    const bool act = tl < T && __ldg(w + tl) != 0.f;
    const unsigned b = __ballot_sync(0xffffffffu, act);
    if (b) return t + static_cast<int64_t>(__ffs(b) - 1) * ncl;
    t += 32 * ncl;
  }
  return T;
}

template <typename T, int C>
__global__ void __launch_bounds__(kThreads, 1)
    loss_v3_kernel(const RowArgs a, int64_t slice_elems, int lag) {
  using G = Geo<T>;
  constexpr int CE = G::CE;
  constexpr int NE = G::NE;
  constexpr int EV = G::EV;

  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ __align__(8) uint64_t full_bar[kSlots];
  __shared__ __align__(8) uint64_t empty_bar[kSlots];
  __shared__ __align__(8) uint64_t mail_bar[kMailD];
  __shared__ __align__(16) float4 mail[kMailD][8];
  __shared__ __align__(16) float4 red[kRD][kCW];
  __shared__ __align__(8) uint64_t red_bar[kRD];
  __shared__ __align__(16) RowScal scal[kRD];
  __shared__ __align__(8) uint64_t scal_bar[kRD];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const uint32_t crank = (C > 1) ? cluster_ctarank() : 0u;
  const int64_t cid = (C > 1) ? static_cast<int64_t>(cluster_id_x()) : blockIdx.x;
  const int64_t ncl = (C > 1) ? static_cast<int64_t>(nclusters_x()) : gridDim.x;
  const int64_t slice_start = static_cast<int64_t>(crank) * slice_elems;
  int64_t sl64 = a.V - slice_start;
  if (sl64 > slice_elems) sl64 = slice_elems;
  if (sl64 < 0) sl64 = 0;
  const int slice_len = static_cast<int>(sl64);
  const int nck = (slice_len + CE - 1) / CE;
  const int nfull = slice_len / CE;
  const uint32_t ring_base = smem_u32(ring);
  const T* logits = static_cast<const T*>(a.logits);

  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), kCT);
    }
    for (int i = 0; i < kMailD; ++i) mbar_init(smem_u32(&mail_bar[i]), C);
    for (int i = 0; i < kRD; ++i) {
      mbar_init(smem_u32(&red_bar[i]), kCW);
      mbar_init(smem_u32(&scal_bar[i]), 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base_sh), kTCols);
  tc_fence_before();
  if (C > 1) {
    cluster_sync_all();
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tbase = tmem_base_sh;

  if (warp == kProd) {
    // ================================================================ producer
    int64_t t = next_active(a.w_tok, cid, ncl, a.T, lane);
    const uint64_t pol = l2_evict_first_policy();
    uint32_t slot = 0, ph = 0;
    while (t < a.T) {
      if (lane == 0) {
        const T* row = logits + t * a.ld + slice_start;
        for (int k = 0; k < nck; ++k) {
          const int rem = slice_len - k * CE;
          const uint32_t bytes = static_cast<uint32_t>(rem < CE ? rem : CE) * G::es;
          mbar_wait(smem_u32(&empty_bar[slot]), ph ^ 1u);
          mbar_arrive_expect_tx(smem_u32(&full_bar[slot]), bytes);
          bulk_g2s(ring_base + slot * kCB, row + static_cast<int64_t>(k) * CE, bytes,
                   smem_u32(&full_bar[slot]), pol);
          if (++slot == kSlots) {
            slot = 0;
            ph ^= 1u;
          }
        }
      }
      t = next_active(a.w_tok, t + ncl, ncl, a.T, lane);
    }
  } else if (warp == kCtl) {
    // ================================================================ control
    const LossParamsDev P{a.eps_lo, a.eps_hi, a.dual_c, a.beta, a.ent_coef, a.kl_mode};
    const bool leader = (crank == 0 && lane == 0);
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t nrow = 0;
    // per-row inputs (incl. the raw target logit) prefetched one row ahead
    float wn = 0.f, An = 0.f, oldn = 0.f, refn = 0.f;
    int32_t yn = 0;
    auto fetch = [&](int64_t tt) {
      wn = __ldg(a.w_tok + tt);
      An = __ldg(a.adv_tok + tt);
      oldn = __ldg(a.old_logp + tt);
      refn = __ldg(a.ref_logp + tt);
      yn = __ldg(a.targets + tt);
    };
    if (cid < a.T) fetch(cid);
    for (int64_t t = cid; t < a.T; t += ncl) {
      const float w = wn, A = An, old = oldn, ref = refn;
      const int32_t y = yn;
      // z_target straight from HBM (before any dlogits of this row is written,
      // so in-place dlogits is safe); issued now, consumed after the merge
      const int64_t yg = static_cast<int64_t>(y) - a.vocab_start;
      float zraw = __int_as_float(0x7fc00000);
      if (w != 0.f && yg >= 0 && yg < a.V) {
        if (sizeof(T) == 2)
          zraw = bf16_to_f32(__ldg(reinterpret_cast<const unsigned short*>(logits) + t * a.ld + yg));
        else
          zraw = __ldg(reinterpret_cast<const float*>(logits) + t * a.ld + yg);
      }
      if (t + ncl < a.T) fetch(t + ncl);
      if (w == 0.f) {
        if (leader) {
          if (a.out_logp) a.out_logp[t] = 0.f;
          if (a.out_entropy) a.out_entropy[t] = 0.f;
        }
        continue;
      }
      const uint32_t rs = nrow % kRD;
      mbar_wait(smem_u32(&red_bar[rs]), (nrow / kRD) & 1u);
      Stats v = stats_empty();
      if (lane < kCW) {
        const float4 r = red[rs][lane];
        v = Stats{r.x, r.y, r.z};
      }
      v = warp_merge(v);
      const uint32_t mb = nrow % kMailD;
      Stats st;
      if (C == 1) {
        st = v;
      } else {
        if (lane == 0) {
          const uint32_t my_slot = smem_u32(&mail[mb][crank]);
          const uint32_t my_bar = smem_u32(&mail_bar[mb]);
#pragma unroll
          for (int q = 0; q < C; ++q) {
            st_cluster_v4(mapa(my_slot, q), v.m2, v.s, v.w, 0.f);
            mbar_arrive_remote(mapa(my_bar, q));
          }
        }
        mbar_wait_cluster_lite(smem_u32(&mail_bar[mb]), (nrow / kMailD) & 1u);
        st = stats_empty();
#pragma unroll
        for (int q = 0; q < C; ++q) {
          const float4 mv = mail[mb][q];
          st = stats_merge(st, Stats{mv.x, mv.y, mv.z});
        }
      }
      float lse2, lse, H, logp;
      row_scalars(st, zraw * a.inv_tau, lse2, lse, H, logp);
      float g, gH, m[8];
      loss_terms(logp, H, w, A, old, ref, P, g, gH, m);
      if (leader) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += static_cast<double>(m[i]);
        if (a.out_logp) a.out_logp[t] = logp;
        if (a.out_entropy) a.out_entropy[t] = H;
      }
      if (lane == 0) {
        RowScal r;
        r.lse2 = lse2;
        r.gt = a.inv_tau * g;
        r.c0 = a.inv_tau * (g + gH * H);
        r.c1 = a.inv_tau * gH * kLn2;
        r.lse2f = lse2 - log2f(fabsf(r.c0));
        r.sgn = r.c0 > 0.f ? 0x80008000u : 0u;
        const int64_t yl = yg - slice_start;
        r.yl = (yl >= 0 && yl < slice_len) ? static_cast<int>(yl) : -1;
        r.pad = 0.f;
        scal[rs] = r;
        mbar_arrive(smem_u32(&scal_bar[rs]));
      }
      ++nrow;
    }
    if (leader) finish_metrics(a, cid, ncl, acc);
  } else {
    // ================================================================ compute
    const uint32_t tm_t = tbase + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                          8u * static_cast<uint32_t>(warp >> 2);
    const uint32_t ring_t = ring_base + 16u * tid;
    const uint32_t full0 = smem_u32(&full_bar[0]), empty0 = smem_u32(&empty_bar[0]);
    const float c = a.inv_tau * kLog2e;
    uint32_t slot = 0, ph = 0;  // smem ring position (forward consumption order)
    uint32_t rel_slot = 0;      // ring slot whose release waits for the TMEM store
    uint32_t n = 0;             // active-row counter of the forward row
    int64_t F = next_active(a.w_tok, cid, ncl, a.T, lane);  // forward row of this step
    int64_t B = -1;                                         // backward row of this step
    int64_t zf = cid;  // next row that may need a zero-fill (masked rows)
    while (F < a.T || B >= 0) {
      const bool hasF = F < a.T, hasB = B >= 0;
      // masked rows before F: dense zero-fill of this CTA's slice (P7)
      if (!a.masked_skip) {
        const int64_t lim = hasF ? F : a.T;
        for (; zf < lim; zf += ncl) {
          if (__ldg(a.w_tok + zf) != 0.f) continue;
          uint8_t* drow = reinterpret_cast<uint8_t*>(static_cast<T*>(a.dlogits) + zf * a.ld_d + slice_start);
          const int nb = slice_len * G::es;
          for (int off = tid * 16; off < nb; off += kCT * 16) stg128_cs(drow + off, make_uint4(0, 0, 0, 0));
        }
        if (hasF) zf = F + ncl;
      }
      // prefetch the window that locates the next forward row
      const int64_t tw = hasF ? F + ncl : a.T;
      const int64_t twl = tw + lane * ncl;
      const float wwin = (twl < a.T) ? __ldg(a.w_tok + twl) : 0.f;

      const uint32_t nb_ = n - 1;  // active-row index of B
      RowScal rsc;
      float lse2 = 0.f, lse2f = 0.f, c0 = 0.f, c1 = 0.f, gt = 0.f;
      uint32_t sgn = 0u;
      bool neg = false;
      int ck = -1, jt = 0;
      T* drow = hasB ? static_cast<T*>(a.dlogits) + B * a.ld_d + slice_start : nullptr;
      float m2 = 0.f;
      float2 s2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      float2 w2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const int kF = hasF ? nck : 0;
      const int kB = hasB ? nck + lag : 0;
      const int K = kF > kB ? kF : kB;
      for (int k = 0; k < K; ++k) {
        const bool doB = hasB && k >= lag;
        const bool doF = hasF && k < nck;
        const int kb = k - lag;
        // ---- issue both loads first: TMEM (backward) and smem (forward)
        uint4 w0, w1, v0, v1;
        if (doB) {
          if (kb == 0) {
            const uint32_t rs = nb_ % kRD;
            mbar_wait(smem_u32(&scal_bar[rs]), (nb_ / kRD) & 1u);
            rsc = scal[rs];
            lse2 = rsc.lse2;
            lse2f = rsc.lse2f;
            c0 = rsc.c0;
            c1 = rsc.c1;
            gt = rsc.gt;
            sgn = rsc.sgn;
            neg = sgn != 0u;
            if (rsc.yl >= 0) {
              const int r = rsc.yl % CE;
              const int v = r >= G::HALF ? 1 : 0;
              const int rr = r - v * G::HALF;
              if (rr / EV == tid) {
                ck = rsc.yl / CE;
                jt = v * EV + rr % EV;
              }
            }
          }
          const uint32_t tsb = (nb_ * static_cast<uint32_t>(nck) + kb) % kTSlots;
          tmem_ld8(tm_t + tsb * kSlotCols, w0, w1);
        }
        if (doF) {
          mbar_wait(full0 + 8u * slot, ph);
          const uint32_t sa = ring_t + slot * kCB;
          v0 = lds128(sa);
          v1 = lds128(sa + kCB / 2);
          rel_slot = slot;  // released after tcgen05.st consumed v0/v1 (LDS returned)
          if (++slot == kSlots) {
            slot = 0;
            ph ^= 1u;
          }
        }
        // ---------------- backward(row B, chunk k - lag)
        if (doB) {
          tmem_wait_ld(w0, w1);
          float x[NE], gr[NE];
          unpack(logits, w0, w1, x);
          T* dst = drow + kb * CE;
          const bool full = kb < nfull;
          bool done = false;
          if (G::es == 2 && c1 == 0.f) {
            const float2 c2 = make_float2(c, c), nl2 = make_float2(-lse2f, -lse2f);
#pragma unroll
            for (int p = 0; p < NE / 2; ++p) {
              const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nl2);
              gr[2 * p] = ex2(av.x);
              gr[2 * p + 1] = ex2(av.y);
            }
            if (kb == ck) {
              const float gts = neg ? -gt : gt;
#pragma unroll
              for (int j = 0; j < NE; ++j)
                if (j == jt) gr[j] += gts;
            }
            if (full) {
              uint4 p0, p1;
              p0.x = pack_bf16x2(gr[0], gr[1]) ^ sgn;
              p0.y = pack_bf16x2(gr[2], gr[3]) ^ sgn;
              p0.z = pack_bf16x2(gr[4], gr[5]) ^ sgn;
              p0.w = pack_bf16x2(gr[6], gr[7]) ^ sgn;
              p1.x = pack_bf16x2(gr[8], gr[9]) ^ sgn;
              p1.y = pack_bf16x2(gr[10], gr[11]) ^ sgn;
              p1.z = pack_bf16x2(gr[12], gr[13]) ^ sgn;
              p1.w = pack_bf16x2(gr[14], gr[15]) ^ sgn;
              stg128_cs(dst + EV * tid, p0);
              stg128_cs(dst + G::HALF + EV * tid, p1);
              done = true;
            } else {
#pragma unroll
              for (int j = 0; j < NE; ++j) gr[j] = neg ? -gr[j] : gr[j];
            }
          } else if (c1 == 0.f) {
            const float2 c2 = make_float2(c, c), nl2 = make_float2(-lse2, -lse2);
            const float2 mc0 = make_float2(-c0, -c0);
#pragma unroll
            for (int p = 0; p < NE / 2; ++p) {
              const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nl2);
              const float2 g2 = __fmul2_rn(make_float2(ex2(av.x), ex2(av.y)), mc0);
              gr[2 * p] = g2.x;
              gr[2 * p + 1] = g2.y;
            }
            if (kb == ck) {
#pragma unroll
              for (int j = 0; j < NE; ++j)
                if (j == jt) gr[j] += gt;
            }
          } else {
#pragma unroll
            for (int j = 0; j < NE; ++j) {
              const float av = fmaxf(fmaf(x[j], c, -lse2), -127.f);
              gr[j] = -ex2(av) * fmaf(c1, av, c0);
            }
            if (kb == ck) {
#pragma unroll
              for (int j = 0; j < NE; ++j)
                if (j == jt) gr[j] += gt;
            }
          }
          if (!done) {
            if (full) {
              store_vec(dst + EV * tid, gr);
              store_vec(dst + G::HALF + EV * tid, gr + EV);
            } else {
              const int rem = slice_len - kb * CE;
#pragma unroll
              for (int j = 0; j < NE; ++j) {
                const int off = elem_off<T>(tid, j);
                if (off < rem) st1(dst + off, gr[j]);
              }
            }
          }
        }
        // ---------------- forward(row F, chunk k)
        if (doF) {
          const uint32_t tsf = (n * static_cast<uint32_t>(nck) + k) % kTSlots;
          tmem_st8(tm_t + tsf * kSlotCols, v0, v1);
          mbar_arrive(empty0 + 8u * rel_slot);
          float x[NE];
          unpack(logits, v0, v1, x);
          if (k == 0) {
            float xm = -INFINITY;
#pragma unroll
            for (int j = 0; j < NE; ++j)
              if (elem_off<T>(tid, j) < slice_len) xm = fmaxf(xm, x[j]);
            m2 = xm * c;
            if (!(m2 > -INFINITY)) m2 = 0.f;
          }
          if (k < nfull) {
            const float2 c2 = make_float2(c, c), nm2 = make_float2(-m2, -m2);
#pragma unroll
            for (int p = 0; p < NE / 2; ++p) {
              const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nm2);
              const float2 e = make_float2(ex2(av.x), ex2(av.y));
              s2[p & 1] = __fadd2_rn(s2[p & 1], e);
              w2[p & 1] = __ffma2_rn(e, av, w2[p & 1]);
            }
          } else {
            const int rem = slice_len - k * CE;
#pragma unroll
            for (int j = 0; j < NE; ++j) {
              if (elem_off<T>(tid, j) < rem && x[j] != -INFINITY) {
                const float av = fmaf(x[j], c, -m2);
                const float e = ex2(av);
                s2[0].x += e;
                w2[0].x = fmaf(e, av, w2[0].x);
              }
            }
          }
          tmem_wait_st(v0, v1);
        }
      }
      if (hasF) {
        Stats my{m2, (s2[0].x + s2[1].x) + (s2[0].y + s2[1].y), (w2[0].x + w2[1].x) + (w2[0].y + w2[1].y)};
        // repair (rare): -inf logits or exponent overflow -> exact recompute from own TMEM words
        const bool bad = !(fabsf(my.s) <= 3.0e38f) || !(fabsf(my.w) <= 3.0e38f);
        if (__any_sync(0xffffffffu, bad)) {
          float mx = -INFINITY;
          for (int k = 0; k < nck; ++k) {
            uint4 q0, q1;
            tmem_ld8(tm_t + ((n * static_cast<uint32_t>(nck) + k) % kTSlots) * kSlotCols, q0, q1);
            tmem_wait_ld(q0, q1);
            float x[NE];
            unpack(logits, q0, q1, x);
            const int rem = slice_len - k * CE;
#pragma unroll
            for (int j = 0; j < NE; ++j)
              if (elem_off<T>(tid, j) < rem) mx = fmaxf(mx, x[j]);
          }
          const float mb2 = (mx == -INFINITY) ? -INFINITY : mx * c;
          float sr = 0.f, wr = 0.f;
          for (int k = 0; k < nck; ++k) {
            uint4 q0, q1;
            tmem_ld8(tm_t + ((n * static_cast<uint32_t>(nck) + k) % kTSlots) * kSlotCols, q0, q1);
            tmem_wait_ld(q0, q1);
            float x[NE];
            unpack(logits, q0, q1, x);
            const int rem = slice_len - k * CE;
#pragma unroll
            for (int j = 0; j < NE; ++j) {
              if (elem_off<T>(tid, j) < rem && x[j] != -INFINITY) {
                const float av = fmaf(x[j], c, -mb2);
                const float e = ex2(av);
                sr += e;
                wr = fmaf(e, av, wr);
              }
            }
          }
          if (bad) my = Stats{mb2, sr, wr};
        }
        if (my.s == 0.f) my = stats_empty();
        my = warp_merge(my);
        if (lane == 0) {
          red[n % kRD][warp] = make_float4(my.m2, my.s, my.w, 0.f);
          mbar_arrive(smem_u32(&red_bar[n % kRD]));
        }
      }
      // advance: B <- F, F <- next active row (window prefetched at step start)
      B = hasF ? F : -1;
      if (hasF) {
        ++n;
        const unsigned bal = __ballot_sync(0xffffffffu, wwin != 0.f);
        F = bal ? tw + static_cast<int64_t>(__ffs(bal) - 1) * ncl
                : next_active(a.w_tok, tw + 32 * ncl, ncl, a.T, lane);
      } else {
        F = a.T;
      }
    }
    // trailing masked rows
    if (!a.masked_skip) {
      for (; zf < a.T; zf += ncl) {
        if (__ldg(a.w_tok + zf) != 0.f) continue;
        uint8_t* drow = reinterpret_cast<uint8_t*>(static_cast<T*>(a.dlogits) + zf * a.ld_d + slice_start);
        const int nb = slice_len * G::es;
        for (int off = tid * 16; off < nb; off += kCT * 16) stg128_cs(drow + off, make_uint4(0, 0, 0, 0));
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, kTCols);
  if (C > 1) cluster_sync_all();
}

std::mutex g_mu;

template <typename T, int C>
int launch_c(const RowArgs& a, int64_t slice, int lag, cudaStream_t s, LaunchInfo* info) {
  auto kern = loss_v3_kernel<T, C>;
  static PerDevice cache;  // per instantiation and device
  int& max_active = cache();
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (max_active < 0) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingBytes);
      if (e != cudaSuccess) return e;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C * 256);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = kRingBytes;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = C;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int ncl = 0;
      e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
      if (e != cudaSuccess) return e;
      max_active = ncl;
      if (max_active <= 0) return cudaErrorInvalidConfiguration;
    }
  }
  int64_t ncl = a.T < max_active ? a.T : max_active;
  if (ncl > a.max_partial_blocks) ncl = a.max_partial_blocks;
  if (ncl < 1) ncl = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(ncl * C));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kRingBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, slice, lag);
  if (info) {
    info->kernel = 3;
    info->cluster = C;
    info->grid = static_cast<int>(ncl * C);
    info->launches = 1;
  }
  return e;
}

template <typename T>
int launch_t(const RowArgs& a, cudaStream_t s, LaunchInfo* info) {
  using G = Geo<T>;
  for (int C : {1, 2, 4, 8}) {
    int64_t slice = (a.V + C - 1) / C;
    slice = (slice + G::EV - 1) / G::EV * G::EV;
    const int64_t nck = (slice + G::CE - 1) / G::CE;
    const int64_t lag = (kTSlots - nck) < kMaxLag ? (kTSlots - nck) : kMaxLag;
    if (lag < kMinLag) continue;
    switch (C) {
      case 1: return launch_c<T, 1>(a, slice, static_cast<int>(lag), s, info);
      case 2: return launch_c<T, 2>(a, slice, static_cast<int>(lag), s, info);
      case 4: return launch_c<T, 4>(a, slice, static_cast<int>(lag), s, info);
      case 8: return launch_c<T, 8>(a, slice, static_cast<int>(lag), s, info);
    }
  }
  return -2;
}

}  // namespace loss3

int launch_loss_v3(const RowArgs& a, cudaStream_t s, LaunchInfo* info) {
  if (a.dtype == 1) return loss3::launch_t<uint16_t>(a, s, info);
  return loss3::launch_t<float>(a, s, info);
}

}  // namespace sftm
