/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH (the timed CPU baseline).
 *
 * The "fast" CPU variant of BASELINE.md §3: the fused DAPO/GRPO loss fwd+bwd
 * for bf16 logits with fp32 arithmetic, vectorised (OpenMP simd + the vector
 * libm under -ffast-math, one clone per ISA chosen at run time) and OpenMP over
 * rows. It is what bench.py reports as the CPU baseline; the fp64 restatement
 * in sf_oracle.c stays the parity truth (tests check this variant against it).
 * Same math as orc_pg_loss_fwd_bwd, three passes over a row
 * (max, sums, gradient), each row cache-resident.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "sf_oracle.h"

static inline float bf16f(uint16_t u) {
  union { uint32_t i; float f; } c;
  c.i = (uint32_t)u << 16;
  return c.f;
}
static inline uint16_t f2bf16(float f) {  /* round to nearest even (finite inputs) */
  union { uint32_t i; float f; } c;
  c.f = f;
  const uint32_t lsb = (c.i >> 16) & 1u;
  return (uint16_t)((c.i + 0x7fffu + lsb) >> 16);
}

#if defined(__x86_64__) && defined(__GNUC__) && !defined(__clang__)
#define SF_CLONES __attribute__((target_clones("avx512f", "avx2", "default")))
#else
#define SF_CLONES
#endif

SF_CLONES static void row_pass(const uint16_t* x, int64_t V, float c, float* out_m, float* out_s, float* out_w) {
  float m = -INFINITY;
#pragma omp simd reduction(max : m)
  for (int64_t v = 0; v < V; ++v) m = fmaxf(m, bf16f(x[v]) * c);
  float s = 0.f, w = 0.f;
#pragma omp simd reduction(+ : s, w)
  for (int64_t v = 0; v < V; ++v) {
    const float a = bf16f(x[v]) * c - m;
    const float e = expf(a);
    s += e;
    w += e * a;
  }
  *out_m = m;
  *out_s = s;
  *out_w = w;
}

SF_CLONES static void row_grad(const uint16_t* x, int64_t V, float c, float L, float g, float gH, float H, float tau1,
                               uint16_t* dl) {
#pragma omp simd
  for (int64_t v = 0; v < V; ++v) {
    const float z = bf16f(x[v]) * c;
    const float pv = expf(z - L);
    const float gr = -g * pv - gH * pv * (z - L + H);
    dl[v] = f2bf16(tau1 * gr);
  }
}

int orc_pg_loss_fwd_bwd_fast(const uint16_t* logits, int64_t T, int64_t V, int64_t ld, const int32_t* targets,
                             const float* old_logp, const float* ref_logp, const float* adv_tok, const float* w_tok,
                             const orc_params* p, uint16_t* dlogits, double* metrics) {
  double* rowm = (double*)calloc((size_t)(T > 0 ? T : 1) * 8, sizeof(double));
  if (!rowm) return 1;
  const float c = (float)p->inv_tau;
  int64_t t;
#pragma omp parallel for schedule(dynamic, 4) num_threads(orc_get_threads())
  for (t = 0; t < T; ++t) {
    const float w = w_tok[t];
    uint16_t* dl = dlogits + t * V;
    if (w == 0.f) {
      memset(dl, 0, (size_t)V * sizeof(uint16_t));
      continue;
    }
    const uint16_t* x = logits + t * ld;
    float m, s, ws;
    row_pass(x, V, c, &m, &s, &ws);
    const float L = m + logf(s);
    const float H = logf(s) - ws / s;
    const int32_t y = targets[t];
    const float zy = (y >= 0 && y < V) ? bf16f(x[y]) * c : NAN;
    const float lp = zy - L;
    const float A = adv_tok[t], old = old_logp[t], ref = ref_logp[t];
    const float ratio = expf(lp - old);
    const int clip_hi = (A > 0.f) && (ratio > 1.f + (float)p->eps_hi);
    const int clip_lo = (A < 0.f) && (ratio < 1.f - (float)p->eps_lo);
    const float rc = fminf(fmaxf(ratio, 1.f - (float)p->eps_lo), 1.f + (float)p->eps_hi);
    float pg = fmaxf(-ratio * A, -rc * A);
    float gpg = (clip_hi || clip_lo) ? 0.f : -A * ratio;
    int clipped = clip_hi || clip_lo;
    if (p->dual_c > 1.0 && A < 0.f) {
      const float cap = -(float)p->dual_c * A;
      if (pg > cap) {
        pg = cap;
        gpg = 0.f;
        clipped = 1;
      }
    }
    const int has_kl = p->beta != 0.0;
    const float d = ref - lp;
    float kl, dkl;
    if (p->kl_mode == 1) {
      kl = -d;
      dkl = 1.f;
    } else if (p->kl_mode == 2) {
      kl = 0.5f * d * d;
      dkl = -d;
    } else if (p->kl_mode == 3) {
      kl = fabsf(d);
      dkl = d > 0.f ? -1.f : (d < 0.f ? 1.f : 0.f);
    } else {
      const float er = expf(d);
      kl = er - d - 1.f;
      dkl = 1.f - er;
    }
    const float g = w * (gpg + (has_kl ? (float)p->beta * dkl : 0.f));
    const float gH = -w * (float)p->ent_coef;
    double* mr = rowm + t * 8;
    mr[0] = w * (pg + (has_kl ? (float)p->beta * kl : 0.f) - (float)p->ent_coef * H);
    mr[1] = w * pg;
    mr[2] = w * kl;
    mr[3] = w * H;
    mr[4] = clipped ? w : 0.f;
    mr[5] = w * ratio;
    mr[6] = 1.0;
    mr[7] = w * (old - lp);
    row_grad(x, V, c, L, g, gH, H, c, dl);
    if (y >= 0 && y < V) dl[y] = f2bf16(c * (g * (1.f - expf(zy - L)) - gH * expf(zy - L) * (zy - L + H)));
  }
  if (metrics) {
    for (int i = 0; i < 8; ++i) metrics[i] = 0.0;
    for (int64_t r = 0; r < T; ++r)
      for (int i = 0; i < 8; ++i) metrics[i] += rowm[r * 8 + i];
  }
  free(rowm);
  return 0;
}
