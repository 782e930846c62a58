// SPDX-License-Identifier: Apache-2.0
// Shared per-row math of the vocab-row kernels (tm_rows.cu, tm_loss.cu):
// element access, online-softmax accumulation, the per-row scalars
// (lse, entropy, logp), the DAPO/GRPO/KL loss terms and their gradients, and
// the deterministic metric reduction. Pinned in DESIGN.md §2; fp64 twin in
// oracle/sf_oracle.c (orc_pg_loss_fwd_bwd).
#pragma once

#include "tm_device.cuh"
#include "tm_internal.h"

namespace sftm {

template <typename T>
struct Elem;
template <>
struct Elem<float> {
  static constexpr int es = 4;
};
template <>
struct Elem<uint16_t> {
  static constexpr int es = 2;
};

// 8 consecutive elements from shared memory -> fp32.
__device__ __forceinline__ void lds8(const float*, uint32_t addr, float x[8]) {
  const uint4 a = lds128(addr), b = lds128(addr + 16);
  x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y);
  x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
  x[4] = __uint_as_float(b.x); x[5] = __uint_as_float(b.y);
  x[6] = __uint_as_float(b.z); x[7] = __uint_as_float(b.w);
}
__device__ __forceinline__ void lds8(const uint16_t*, uint32_t addr, float x[8]) {
  const uint4 a = lds128(addr);
  x[0] = bf16lo(a.x); x[1] = bf16hi(a.x); x[2] = bf16lo(a.y); x[3] = bf16hi(a.y);
  x[4] = bf16lo(a.z); x[5] = bf16hi(a.z); x[6] = bf16lo(a.w); x[7] = bf16hi(a.w);
}

__device__ __forceinline__ float ldg_elem(const float* p, int64_t i) { return __ldg(p + i); }
__device__ __forceinline__ float ldg_elem(const uint16_t* p, int64_t i) {
  return bf16_to_f32(__ldg(reinterpret_cast<const unsigned short*>(p) + i));
}

__device__ __forceinline__ void st8(float* p, const float g[8]) {
  stg128_cs(p, make_uint4(__float_as_uint(g[0]), __float_as_uint(g[1]), __float_as_uint(g[2]),
                          __float_as_uint(g[3])));
  stg128_cs(p + 4, make_uint4(__float_as_uint(g[4]), __float_as_uint(g[5]),
                              __float_as_uint(g[6]), __float_as_uint(g[7])));
}
__device__ __forceinline__ void st8(uint16_t* p, const float g[8]) {
  stg128_cs(p, make_uint4(pack_bf16x2(g[0], g[1]), pack_bf16x2(g[2], g[3]),
                          pack_bf16x2(g[4], g[5]), pack_bf16x2(g[6], g[7])));
}
__device__ __forceinline__ void st1(float* p, float g) { *p = g; }
__device__ __forceinline__ void st1(uint16_t* p, float g) { *p = f32_to_bf16(g); }

// Online-softmax update with 8 new elements (z = x * inv_tau; c = inv_tau*log2e).
// One rescale exp per 8 elements at most, and only when this thread's max grows.
__device__ __forceinline__ void accum8(Stats& st, const float x[8], float c) {
  const float xm = fmaxf(fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3])),
                         fmaxf(fmaxf(x[4], x[5]), fmaxf(x[6], x[7])));
  const float cm = xm * c;
  if (cm > st.m2) {
    if (st.m2 != -INFINITY) {
      const float d = st.m2 - cm;
      const float f = ex2(d);
      st.w = f * fmaf(st.s, d, st.w);
      st.s *= f;
    }
    st.m2 = cm;
  }
  float s0 = 0.f, s1 = 0.f, w0 = 0.f, w1 = 0.f;
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float a0 = fmaxf(fmaf(x[j], c, -st.m2), -127.f);
    const float a1 = fmaxf(fmaf(x[j + 1], c, -st.m2), -127.f);
    const float e0 = ex2(a0), e1 = ex2(a1);
    s0 += e0;
    s1 += e1;
    w0 = fmaf(e0, a0, w0);
    w1 = fmaf(e1, a1, w1);
  }
  st.s += s0 + s1;
  st.w += w0 + w1;
}

struct LossParamsDev {
  float eps_lo, eps_hi, dual_c, beta, ent;
  int kl_mode = 0;  // SF_TM_KL_*: 0 k3, 1 k1, 2 k2, 3 abs
};

// Per-row scalars from merged statistics. Decision P1: z = x / tau.
__device__ __forceinline__ void row_scalars(const Stats& st, float zy, float& lse2, float& lse,
                                            float& H, float& logp) {
  const float log2S = log2f(st.s);
  lse2 = st.m2 + log2S;
  lse = lse2 * kLn2;
  H = (log2S - st.w / st.s) * kLn2;
  logp = zy - lse;
}

// DAPO decoupled clip (+dual clip), k3 KL, entropy bonus; g = dL/dlogp, gH = dL/dH.
// m[] receives the w-weighted metric contributions (SF_TM_M_* order).
__device__ __forceinline__ void loss_terms(float logp, float H, float w, float A, float old,
                                           float ref, const LossParamsDev& P, float& g, float& gH,
                                           float m[8]) {
  const float ratio = expf(logp - old);
  const bool clip_hi = (A > 0.f) && (ratio > 1.f + P.eps_hi);
  const bool clip_lo = (A < 0.f) && (ratio < 1.f - P.eps_lo);
  const float rc = fminf(fmaxf(ratio, 1.f - P.eps_lo), 1.f + P.eps_hi);
  float pg = fmaxf(-ratio * A, -rc * A);
  float gpg = (clip_hi || clip_lo) ? 0.f : -A * ratio;
  bool clipped = clip_hi || clip_lo;
  if (P.dual_c > 1.f && A < 0.f) {
    const float cap = -P.dual_c * A;
    if (pg > cap) {
      pg = cap;
      gpg = 0.f;
      clipped = true;
    }
  }
  const float d = ref - logp;
  // KL estimator and its derivative in logp (d = ref - logp): k3 e^d - d - 1
  // (1 - e^d), k1 -d (1), k2 d^2/2 (-d), abs |d| (-sign d)
  float kl, dkl;
  if (P.kl_mode == 1) {
    kl = -d;
    dkl = 1.f;
  } else if (P.kl_mode == 2) {
    kl = 0.5f * d * d;
    dkl = -d;
  } else if (P.kl_mode == 3) {
    kl = fabsf(d);
    dkl = d > 0.f ? -1.f : (d < 0.f ? 1.f : 0.f);
  } else {
    const float er = expf(d);
    kl = er - d - 1.f;
    dkl = 1.f - er;
  }
  // beta == 0 must drop the KL terms entirely: e^(ref - logp) overflows fp32 for
  // rows the policy gives far less mass than the reference (0 * inf = NaN)
  const bool has_kl = P.beta != 0.f;
  const float gkl = has_kl ? P.beta * dkl : 0.f;
  const float l = pg + (has_kl ? P.beta * kl : 0.f) - P.ent * H;
  g = w * (gpg + gkl);
  gH = -w * P.ent;
  m[0] = w * l;
  m[1] = w * pg;
  m[2] = w * kl;
  m[3] = w * H;
  m[4] = clipped ? w : 0.f;
  m[5] = w * ratio;
  m[6] = 1.f;
  m[7] = w * (old - logp);
}

// Deterministic metric finalisation: every block (cluster leader) deposits its
// row-ordered fp64 partials; the last to arrive sums them in block order.
__device__ __forceinline__ void finish_metrics(const RowArgs& a, int64_t blk, int64_t nblk,
                                               const double acc[8]) {
  double* part = a.partials + blk * 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) part[i] = acc[i];
  __threadfence();
  const unsigned prev = atomicAdd(a.ticket, 1u);
  if (prev == static_cast<unsigned>(nblk - 1)) {
    __threadfence();
    double tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const volatile double* vp = a.partials;
    for (int64_t q = 0; q < nblk; ++q) {
#pragma unroll
      for (int i = 0; i < 8; ++i) tot[i] += vp[q * 8 + i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) a.out_metrics[i] = static_cast<float>(tot[i]);
    *a.ticket = 0u;
  }
}


}  // namespace sftm
