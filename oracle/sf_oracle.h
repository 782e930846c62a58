/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH.
 *
 * fp64 CPU oracle for the staleflow train-math hot path. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it, and only as the checker or the timed CPU baseline.
 *
 * Parity status: math parity unpinned against the reference. The reference
 * (/root/reference) contains NO implementation of
 * this math (SPEC.md:8 puts GRPO/DAPO losses and R3 internals out of scope;
 * the compute is a latency stub at proj/src/sim_runtime.cpp:441 and
 * proj/src/wall_runtime.cpp:118,174,197). The oracle is therefore a
 * restatement of the published algorithms pinned in DESIGN.md §2 (P1-P9),
 * cross-checked against (a) hand-derived known answers, (b) golden vectors
 * produced by an independent torch-float64 autograd implementation
 * (tests/golden/make_golden.py), and (c) for the seeded-RNG / digest
 * helpers, bit-exactly against the reference's own rng.cpp / hash.hpp compiled
 * into oracle/_ref (oracle/Makefile, target `ref`).
 */
#ifndef SF_ORACLE_H_
#define SF_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_params {
  double eps_lo, eps_hi, dual_c, beta, ent_coef, inv_tau;
  int32_t kl_mode; /* 0 k3, 1 k1, 2 k2, 3 abs (SF_TM_KL_*) */
} orc_params;

/* dtype: 0 = f32, 1 = bf16 (raw uint16), 2 = f64 (oracle outputs only) */

void orc_set_threads(int n);
int orc_get_threads(void);

/* a1 */
int orc_logprob_fwd(const void* logits, int dtype, int64_t T, int64_t V, int64_t ld,
                    const int32_t* targets, double inv_tau, double* logp, double* ent,
                    double* lse);

/* a6 */
int orc_varlen_meta(const int32_t* lens, const int32_t* plens, const int32_t* gids, int64_t B,
                    int32_t* cu, int32_t* seq_id, uint8_t* mask, int32_t* tok_group);

/* a3 */
int orc_grpo_advantage(const float* r, const int32_t* gid, int64_t B, double eps, int std_mode,
                       double* adv, int32_t* gsize);

/* a4 prologue */
int orc_token_weights(const int32_t* cu, int64_t B, const float* adv_seq, const uint8_t* mask,
                      int64_t T, int norm_mode, double inv_norm, double* adv_tok, double* w_tok);

/* a1+a4+a2. adv_tok / w_tok are the float inputs the GPU kernel consumes.
 * dl_dtype: 0 f32, 1 bf16, 2 f64; dlogits may be NULL; masked rows are
 * zero-filled unless masked_skip. metrics[8] in SF_TM_M_* order. Also returns
 * per-row g (dL/dlogp) if g_out != NULL. */
int orc_pg_loss_fwd_bwd(const void* logits, int dtype, int64_t T, int64_t V, int64_t ld,
                        const int32_t* targets, const float* old_logp, const float* ref_logp,
                        const float* adv_tok, const float* w_tok, const orc_params* p,
                        int masked_skip, void* dlogits, int dl_dtype, double* logp, double* ent,
                        double* metrics, double* g_out);

/* The timed CPU baseline ("fast" variant, sf_cpu_fast.c): bf16 logits -> bf16
 * dlogits [T, V], fp32 arithmetic, vectorised, OpenMP over rows; finite logits.
 * Same math as orc_pg_loss_fwd_bwd; checked against it in tests/test_oracle.py. */
int orc_pg_loss_fwd_bwd_fast(const uint16_t* logits, int64_t T, int64_t V, int64_t ld, const int32_t* targets,
                             const float* old_logp, const float* ref_logp, const float* adv_tok,
                             const float* w_tok, const orc_params* p, uint16_t* dlogits, double* metrics);

/* a5 */
int orc_r3_gate_fwd(const void* logits, int dtype, int64_t L, int64_t T, int64_t E, int64_t k,
                    const void* rec, int idx_dtype, int renorm, double* w, int32_t* idx,
                    uint32_t* mismatch);
int orc_r3_gate_bwd(const void* logits, int dtype, int64_t L, int64_t T, int64_t E, int64_t k,
                    const void* rec, int idx_dtype, int renorm, const float* w, const float* dw,
                    double* dz);

/* a7: stats[T*4] = {max z, sum e^(z-max), sum e^(z-max)(z-max), z_target or NaN} */
int orc_vp_partial_stats(const void* shard, int dtype, int64_t T, int64_t Vp, int64_t ld,
                         int64_t vocab_start, const int32_t* targets, double inv_tau,
                         double* stats);

/* seeded-input and digest helpers restated from proj/include/staleflow/rng.hpp:17-39,
 * proj/src/rng.cpp:10-21 and proj/include/staleflow/hash.hpp:14-31 */
uint64_t orc_splitmix_at(uint64_t seed, uint64_t i);
uint64_t orc_derive_seed(uint64_t seed, const char* tag, uint64_t tag_len, uint64_t idx);
uint64_t orc_fnv1a64(const uint8_t* data, uint64_t len);

/* bf16 helpers (round-to-nearest-even) */
uint16_t orc_f64_to_bf16(double x);
double orc_bf16_to_f64(uint16_t u);

#ifdef __cplusplus
}
#endif

#endif /* SF_ORACLE_H_ */
