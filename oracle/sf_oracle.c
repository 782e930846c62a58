/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH (see sf_oracle.h).
 *
 * fp64 restatement of the train-math hot path, row-parallel with OpenMP.
 * Every function cites what it restates. The reference has no code for this
 * math; the algorithm anchors are the paper sections the survey
 * names: GRPO group baselines, DAPO
 * decoupled clip, loss only over assistant tokens
 * (PAPER.md:332), cu_seqlens packing, R3 replay
 * (PAPER.md:563-565), with the P1-P9 decisions of DESIGN.md §2.
 *
 * Parity status: math parity unpinned against the reference, because the
 * reference has no implementation, test, fixture or golden vector for it
 * (SURVEY.md §8c). The restatement is pinned instead by hand-derived known
 * answers and by golden vectors from an independent torch-float64 autograd
 * implementation (tests/golden/make_golden.py); its seeded RNG and digest
 * helpers are pinned bit-exactly against the reference's own rng.cpp /
 * hash.hpp compiled in oracle/_ref.
 */
#include "sf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 0;

void orc_set_threads(int n) { g_threads = n; }
int orc_get_threads(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------ bf16 */
double orc_bf16_to_f64(uint16_t u) {
  uint32_t b = ((uint32_t)u) << 16;
  float f;
  memcpy(&f, &b, 4);
  return (double)f;
}

/* Round-to-nearest-even of the exact double value to bf16 (no double rounding). */
uint16_t orc_f64_to_bf16(double x) {
  if (isnan(x)) return 0x7fc0;
  float f = (float)x; /* may round; fix up below using the exact double */
  uint32_t b;
  memcpy(&b, &f, 4);
  uint32_t lo = b & 0xffff0000u;
  uint32_t hi = lo + 0x10000u;
  float flo, fhi;
  memcpy(&flo, &lo, 4);
  memcpy(&fhi, &hi, 4);
  /* candidates: truncation toward zero (lo) and next away (hi) of |f| */
  double dlo = fabs((double)flo), dhi = fabs((double)fhi), ax = fabs(x);
  if (isinf(f)) return (uint16_t)(b >> 16);
  if (!(ax >= dlo)) { /* f rounded away from the bf16 interval: step down */
    lo -= 0x10000u;
    hi -= 0x10000u;
    memcpy(&flo, &lo, 4);
    memcpy(&fhi, &hi, 4);
    dlo = fabs((double)flo);
    dhi = fabs((double)fhi);
  }
  double elo = ax - dlo, ehi = dhi - ax;
  uint32_t pick;
  if (elo < ehi)
    pick = lo;
  else if (ehi < elo)
    pick = hi;
  else
    pick = ((lo >> 16) & 1u) ? hi : lo;
  return (uint16_t)(pick >> 16);
}

static inline double elem(const void* p, int dtype, int64_t i) {
  if (dtype == 1) return orc_bf16_to_f64(((const uint16_t*)p)[i]);
  if (dtype == 2) return ((const double*)p)[i];
  return (double)((const float*)p)[i];
}

static inline void put(void* p, int dtype, int64_t i, double v) {
  if (dtype == 1)
    ((uint16_t*)p)[i] = orc_f64_to_bf16(v);
  else if (dtype == 2)
    ((double*)p)[i] = v;
  else
    ((float*)p)[i] = (float)v;
}

/* Row statistics: m = max z, s = sum e^(z-m), w = sum e^(z-m)(z-m), z = x*inv_tau. */
static void row_stats(const void* logits, int dtype, int64_t off, int64_t V, double inv_tau,
                      double* m_out, double* s_out, double* w_out) {
  double m = -INFINITY;
  for (int64_t v = 0; v < V; ++v) {
    double z = elem(logits, dtype, off + v) * inv_tau;
    if (z > m) m = z;
  }
  double s = 0.0, w = 0.0;
  if (m != -INFINITY) {
    for (int64_t v = 0; v < V; ++v) {
      double z = elem(logits, dtype, off + v) * inv_tau;
      if (z == -INFINITY) continue;
      double e = exp(z - m);
      s += e;
      w += e * (z - m);
    }
  }
  *m_out = m;
  *s_out = s;
  *w_out = w;
}

/* a1: lse = m + ln s; H = ln s - w/s (= -sum p ln p); logp = z_y - lse. */
int orc_logprob_fwd(const void* logits, int dtype, int64_t T, int64_t V, int64_t ld,
                    const int32_t* targets, double inv_tau, double* logp, double* ent,
                    double* lse) {
  int64_t t;
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
  for (t = 0; t < T; ++t) {
    double m, s, w;
    row_stats(logits, dtype, t * ld, V, inv_tau, &m, &s, &w);
    double L = m + log(s);
    double H = log(s) - w / s;
    int64_t y = targets[t];
    double zy = (y >= 0 && y < V) ? elem(logits, dtype, t * ld + y) * inv_tau : NAN;
    if (logp) logp[t] = zy - L;
    if (ent) ent[t] = H;
    if (lse) lse[t] = L;
  }
  return 0;
}

/* a6: exclusive scan of lengths; per token: sequence, loss mask (position >=
 * prompt length, the assistant-token mask of PAPER.md:332), group id. */
int orc_varlen_meta(const int32_t* lens, const int32_t* plens, const int32_t* gids, int64_t B,
                    int32_t* cu, int32_t* seq_id, uint8_t* mask, int32_t* tok_group) {
  int32_t acc = 0;
  for (int64_t b = 0; b < B; ++b) {
    cu[b] = acc;
    acc += lens[b];
  }
  cu[B] = acc;
  for (int64_t b = 0; b < B; ++b) {
    for (int64_t t = cu[b]; t < cu[b + 1]; ++t) {
      if (seq_id) seq_id[t] = (int32_t)b;
      if (mask) mask[t] = (t - cu[b]) >= (plens ? plens[b] : 0) ? 1 : 0;
      if (tok_group) tok_group[t] = gids ? gids[b] : 0;
    }
  }
  return 0;
}

/* a3: GRPO group normalisation ("baselines from group-level
 * statistics"). P2: std_mode 0 unbiased (N-1), 1 population, 2 none
 * (Dr.GRPO). P3: groups whose rewards are all equal (incl. singletons) -> 0. */
int orc_grpo_advantage(const float* r, const int32_t* gid, int64_t B, double eps, int std_mode,
                       double* adv, int32_t* gsize) {
  int64_t i;
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
  for (i = 0; i < B; ++i) {
    int64_t n = 0;
    double sum = 0.0, mn = INFINITY, mx = -INFINITY;
    for (int64_t j = 0; j < B; ++j)
      if (gid[j] == gid[i]) {
        ++n;
        sum += r[j];
        if (r[j] < mn) mn = r[j];
        if (r[j] > mx) mx = r[j];
      }
    double mean = sum / (double)n, ss = 0.0;
    for (int64_t j = 0; j < B; ++j)
      if (gid[j] == gid[i]) ss += ((double)r[j] - mean) * ((double)r[j] - mean);
    double A;
    if (mx == mn) {
      A = 0.0;
    } else if (std_mode == 2) {
      A = (double)r[i] - mean;
    } else {
      double var = std_mode == 0 ? ss / (double)(n - 1) : ss / (double)n;
      A = ((double)r[i] - mean) / (sqrt(var) + eps);
    }
    adv[i] = A;
    if (gsize) gsize[i] = (int32_t)n;
  }
  return 0;
}

/* a4 prologue: w_t = mask_t * inv_norm_t. norm 0: DAPO token
 * mean 1/sum(mask); 1: GRPO seq-mean of token-means 1/(n_b * #nonempty);
 * 2: explicit. */
int orc_token_weights(const int32_t* cu, int64_t B, const float* adv_seq, const uint8_t* mask,
                      int64_t T, int norm_mode, double inv_norm, double* adv_tok, double* w_tok) {
  int64_t total = 0, nonempty = 0;
  int64_t* cnt = (int64_t*)calloc((size_t)(B > 0 ? B : 1), sizeof(int64_t));
  for (int64_t b = 0; b < B; ++b) {
    for (int64_t t = cu[b]; t < cu[b + 1] && t < T; ++t) cnt[b] += mask ? (mask[t] != 0) : 1;
    total += cnt[b];
    nonempty += cnt[b] > 0;
  }
  for (int64_t b = 0; b < B; ++b) {
    double ws;
    if (norm_mode == 0)
      ws = total > 0 ? 1.0 / (double)total : 0.0;
    else if (norm_mode == 1)
      ws = cnt[b] > 0 ? 1.0 / ((double)cnt[b] * (double)nonempty) : 0.0;
    else
      ws = inv_norm;
    for (int64_t t = cu[b]; t < cu[b + 1] && t < T; ++t) {
      int on = mask ? (mask[t] != 0) : 1;
      w_tok[t] = on ? ws : 0.0;
      adv_tok[t] = adv_seq ? (double)adv_seq[b] : 0.0;
    }
  }
  free(cnt);
  return 0;
}

/* a1+a4+a2:
 *   ratio = e^(logp-old); pg = -min(ratio*A, clip(ratio,1-eps_lo,1+eps_hi)*A)
 *   (PAPER.md:122 decoupled clip) with optional dual clip min(pg, -c*A) for A<0;
 *   kl = e^(ref-logp) - (ref-logp) - 1 (k3); l = pg + beta*kl - ent_coef*H;
 *   loss = sum_t w_t l_t.
 *   g = dL/dlogp = w*(gpg + beta*(1 - e^(ref-logp))), gpg = -A*ratio unless the
 *   clipped branch is active; gH = dL/dH = -w*ent_coef;
 *   dL/dx_v = inv_tau*[g*(1[v=y] - p_v) - gH*p_v*(z_v - lse + H)]. */
int orc_pg_loss_fwd_bwd(const void* logits, int dtype, int64_t T, int64_t V, int64_t ld,
                        const int32_t* targets, const float* old_logp, const float* ref_logp,
                        const float* adv_tok, const float* w_tok, const orc_params* p,
                        int masked_skip, void* dlogits, int dl_dtype, double* logp, double* ent,
                        double* metrics, double* g_out) {
  double* rowm = (double*)calloc((size_t)(T > 0 ? T : 1) * 8, sizeof(double));
  int64_t t;
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
  for (t = 0; t < T; ++t) {
    const double w = w_tok[t];
    double* mrow = rowm + t * 8;
    if (w == 0.0) {
      if (dlogits && !masked_skip)
        for (int64_t v = 0; v < V; ++v) put(dlogits, dl_dtype, t * V + v, 0.0);
      if (logp) logp[t] = 0.0;
      if (ent) ent[t] = 0.0;
      if (g_out) g_out[t] = 0.0;
      continue;
    }
    const double A = adv_tok[t], old = old_logp[t], ref = ref_logp[t];
    double m, s, ws;
    row_stats(logits, dtype, t * ld, V, p->inv_tau, &m, &s, &ws);
    const double L = m + log(s);
    const double H = log(s) - ws / s;
    const int64_t y = targets[t];
    const double zy = (y >= 0 && y < V) ? elem(logits, dtype, t * ld + y) * p->inv_tau : NAN;
    const double lp = zy - L;
    const double ratio = exp(lp - old);
    const int clip_hi = (A > 0.0) && (ratio > 1.0 + p->eps_hi);
    const int clip_lo = (A < 0.0) && (ratio < 1.0 - p->eps_lo);
    double rc = ratio;
    if (rc < 1.0 - p->eps_lo) rc = 1.0 - p->eps_lo;
    if (rc > 1.0 + p->eps_hi) rc = 1.0 + p->eps_hi;
    double pg = fmax(-ratio * A, -rc * A);
    double gpg = (clip_hi || clip_lo) ? 0.0 : -A * ratio;
    int clipped = clip_hi || clip_lo;
    if (p->dual_c > 1.0 && A < 0.0) {
      const double cap = -p->dual_c * A;
      if (pg > cap) {
        pg = cap;
        gpg = 0.0;
        clipped = 1;
      }
    }
    /* KL estimators (d = ref - logp) and their derivative in logp: k3 e^d-d-1
     * (1-e^d), k1 -d (1), k2 d^2/2 (-d), abs |d| (-sign d); beta = 0 drops them */
    const double d = ref - lp;
    double kl, dkl;
    if (p->kl_mode == 1) {
      kl = -d;
      dkl = 1.0;
    } else if (p->kl_mode == 2) {
      kl = 0.5 * d * d;
      dkl = -d;
    } else if (p->kl_mode == 3) {
      kl = fabs(d);
      dkl = d > 0.0 ? -1.0 : (d < 0.0 ? 1.0 : 0.0);
    } else {
      const double er = exp(d);
      kl = er - d - 1.0;
      dkl = 1.0 - er;
    }
    const int has_kl = p->beta != 0.0;
    const double gkl = has_kl ? p->beta * dkl : 0.0;
    const double l = pg + (has_kl ? p->beta * kl : 0.0) - p->ent_coef * H;
    const double g = w * (gpg + gkl);
    const double gH = -w * p->ent_coef;
    mrow[0] = w * l;
    mrow[1] = w * pg;
    mrow[2] = w * kl;
    mrow[3] = w * H;
    mrow[4] = clipped ? w : 0.0;
    mrow[5] = w * ratio;
    mrow[6] = 1.0;
    mrow[7] = w * (old - lp);
    if (logp) logp[t] = lp;
    if (ent) ent[t] = H;
    if (g_out) g_out[t] = g;
    if (dlogits) {
      for (int64_t v = 0; v < V; ++v) {
        const double z = elem(logits, dtype, t * ld + v) * p->inv_tau;
        const double pv = (z == -INFINITY) ? 0.0 : exp(z - L);
        double gr = -g * pv;
        if (gH != 0.0 && pv != 0.0) gr -= gH * pv * (z - L + H);
        if (v == y) gr += g;
        put(dlogits, dl_dtype, t * V + v, p->inv_tau * gr);
      }
    }
  }
  if (metrics) {
    for (int i = 0; i < 8; ++i) metrics[i] = 0.0;
    for (int64_t r = 0; r < T; ++r)
      for (int i = 0; i < 8; ++i) metrics[i] += rowm[r * 8 + i];
  }
  free(rowm);
  return 0;
}

static inline int64_t idx_at(const void* rec, int idx_dtype, int64_t i) {
  return idx_dtype == 1 ? (int64_t)((const uint8_t*)rec)[i] : (int64_t)((const int32_t*)rec)[i];
}

/* a5: R3 replay gate. P8 renorm: softmax over the recorded
 * experts; renorm=0: full softmax gathered at the recorded experts. P9: the
 * trainer's top-k orders by (logit desc, expert index asc). */
int orc_r3_gate_fwd(const void* logits, int dtype, int64_t L, int64_t T, int64_t E, int64_t k,
                    const void* rec, int idx_dtype, int renorm, double* w, int32_t* idx,
                    uint32_t* mismatch) {
  const int64_t rows = L * T;
  uint8_t* mm = (uint8_t*)calloc((size_t)(rows > 0 ? rows : 1), 1);
  int64_t r;
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
  for (r = 0; r < rows; ++r) {
    double* z = (double*)malloc(sizeof(double) * (size_t)E);
    uint8_t* sel = (uint8_t*)calloc((size_t)E, 1);
    uint8_t* rm = (uint8_t*)calloc((size_t)E, 1);
    for (int64_t e = 0; e < E; ++e) z[e] = elem(logits, dtype, r * E + e);
    if (renorm) {
      double m = -INFINITY, s = 0.0;
      for (int64_t j = 0; j < k; ++j) {
        int64_t e = idx_at(rec, idx_dtype, r * k + j);
        double v = (e >= 0 && e < E) ? z[e] : NAN;
        if (v > m) m = v;
      }
      for (int64_t j = 0; j < k; ++j) {
        int64_t e = idx_at(rec, idx_dtype, r * k + j);
        s += exp(((e >= 0 && e < E) ? z[e] : NAN) - m);
      }
      for (int64_t j = 0; j < k; ++j) {
        int64_t e = idx_at(rec, idx_dtype, r * k + j);
        w[r * k + j] = exp(((e >= 0 && e < E) ? z[e] : NAN) - m) / s;
      }
    } else {
      double m = -INFINITY, s = 0.0;
      for (int64_t e = 0; e < E; ++e)
        if (z[e] > m) m = z[e];
      for (int64_t e = 0; e < E; ++e) s += exp(z[e] - m);
      for (int64_t j = 0; j < k; ++j) {
        int64_t e = idx_at(rec, idx_dtype, r * k + j);
        w[r * k + j] = exp(((e >= 0 && e < E) ? z[e] : NAN) - m) / s;
      }
    }
    for (int64_t j = 0; j < k; ++j) {
      int64_t e = idx_at(rec, idx_dtype, r * k + j);
      if (idx) idx[r * k + j] = (int32_t)e;
      if (e >= 0 && e < E) rm[e] = 1;
    }
    for (int64_t round = 0; round < k; ++round) {
      int64_t best = -1;
      for (int64_t e = 0; e < E; ++e) {
        if (sel[e]) continue;
        if (best < 0 || z[e] > z[best]) best = e; /* strict > keeps the lowest index on ties */
      }
      if (best >= 0) sel[best] = 1;
    }
    int diff = 0;
    for (int64_t e = 0; e < E; ++e)
      if (sel[e] != rm[e]) diff = 1;
    mm[r] = (uint8_t)diff;
    free(z);
    free(sel);
    free(rm);
  }
  if (mismatch) {
    for (int64_t l = 0; l <= L; ++l) mismatch[l] = 0;
    for (int64_t q = 0; q < rows; ++q)
      if (mm[q]) {
        mismatch[q / T] += 1;
        mismatch[L] += 1;
      }
  }
  free(mm);
  return 0;
}

/* Backward: renorm: dz[e_j] += w_j (dw_j - S), S = sum_i w_i dw_i;
 * renorm=0: dz_e = p_e (D_e - S), D_e = sum_{j: e_j = e} dw_j. */
int orc_r3_gate_bwd(const void* logits, int dtype, int64_t L, int64_t T, int64_t E, int64_t k,
                    const void* rec, int idx_dtype, int renorm, const float* w, const float* dw,
                    double* dz) {
  const int64_t rows = L * T;
  int64_t r;
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
  for (r = 0; r < rows; ++r) {
    double S = 0.0;
    for (int64_t j = 0; j < k; ++j) S += (double)w[r * k + j] * (double)dw[r * k + j];
    for (int64_t e = 0; e < E; ++e) dz[r * E + e] = 0.0;
    if (renorm) {
      for (int64_t j = 0; j < k; ++j) {
        int64_t e = idx_at(rec, idx_dtype, r * k + j);
        if (e >= 0 && e < E) dz[r * E + e] += (double)w[r * k + j] * ((double)dw[r * k + j] - S);
      }
    } else {
      double m = -INFINITY, s = 0.0;
      for (int64_t e = 0; e < E; ++e) {
        double v = elem(logits, dtype, r * E + e);
        if (v > m) m = v;
      }
      for (int64_t e = 0; e < E; ++e) s += exp(elem(logits, dtype, r * E + e) - m);
      for (int64_t j = 0; j < k; ++j) {
        int64_t e = idx_at(rec, idx_dtype, r * k + j);
        if (e >= 0 && e < E) dz[r * E + e] += (double)dw[r * k + j];
      }
      for (int64_t e = 0; e < E; ++e) {
        double pe = exp(elem(logits, dtype, r * E + e) - m) / s;
        dz[r * E + e] = pe * (dz[r * E + e] - S);
      }
    }
  }
  return 0;
}

/* a7: per-shard statistics for the vocab-parallel combine. */
int orc_vp_partial_stats(const void* shard, int dtype, int64_t T, int64_t Vp, int64_t ld,
                         int64_t vocab_start, const int32_t* targets, double inv_tau,
                         double* stats) {
  int64_t t;
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
  for (t = 0; t < T; ++t) {
    double m, s, w;
    row_stats(shard, dtype, t * ld, Vp, inv_tau, &m, &s, &w);
    int64_t yl = (int64_t)targets[t] - vocab_start;
    stats[t * 4 + 0] = m;
    stats[t * 4 + 1] = s;
    stats[t * 4 + 2] = w;
    stats[t * 4 + 3] = (yl >= 0 && yl < Vp) ? elem(shard, dtype, t * ld + yl) * inv_tau : NAN;
  }
  return 0;
}

/* ------------------------------------------------------------ RNG / digest */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* i-th output of SplitMix64(seed): state advanced i+1 times (rng.hpp:21-26). */
uint64_t orc_splitmix_at(uint64_t seed, uint64_t i) {
  return mix64(seed + (i + 1ull) * 0x9e3779b97f4a7c15ull);
}

/* FNV-1a 64 (hash.hpp:14-31). */
uint64_t orc_fnv1a64(const uint8_t* data, uint64_t len) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < len; ++i) {
    h ^= data[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* derive_seed: FNV over (seed LE8, tag bytes, idx LE8) then one SplitMix64
 * step (rng.cpp:10-21). */
uint64_t orc_derive_seed(uint64_t seed, const char* tag, uint64_t tag_len, uint64_t idx) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (int i = 0; i < 8; ++i) {
    h ^= (uint8_t)(seed >> (8 * i));
    h *= 0x100000001b3ull;
  }
  for (uint64_t i = 0; i < tag_len; ++i) {
    h ^= (uint8_t)tag[i];
    h *= 0x100000001b3ull;
  }
  for (int i = 0; i < 8; ++i) {
    h ^= (uint8_t)(idx >> (8 * i));
    h *= 0x100000001b3ull;
  }
  return orc_splitmix_at(h, 0);
}
