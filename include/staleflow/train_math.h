/* SPDX-License-Identifier: Apache-2.0
 *
 * staleflow train-math C-ABI — the per-token training-math hot path of Relax
 * (arXiv 2604.11554) on B200 (sm_100a).
 *
 * This header is the drop-in boundary. The reference (`/root/reference/proj`)
 * models this compute as synthetic latency at its role-compute seams; every
 * entry point below names the seam it replaces:
 *
 *   - Actor loss fwd+bwd ........ trainer_compute_batch  proj/src/sim_runtime.cpp:431-463
 *                                 (latency draw at :441, draw_train_micro :142-145)
 *                                 trainer_thread         proj/src/wall_runtime.cpp:136-232
 *                                 (sleep_units at :174 and :197)
 *   - ActorFwd / RefLogP stages . stage_run_batch        proj/src/sim_runtime.cpp:304-350
 *                                 (payload stub :328-333), stage_thread wall_runtime.cpp:103-134
 *                                 (sleep at :118, stub payload :126-129); field contract
 *                                 controller.cpp:76-77 ("logp", "ref_logp")
 *   - Advantages stage .......... same seams, field "reward" -> "advantage" (controller.cpp:79)
 *   - R3 routing replay ......... a new data-declared field (config.cpp:127-148); paper §5.5
 *
 * Conventions (mirroring proj/include/staleflow/result.hpp:14-47 and :62-63):
 *   - every function returns an int that is static_cast<uint16_t>(staleflow::Errc):
 *       0  = Ok
 *       21 = ConfigError  (bad shape, dtype, pointer, alignment or parameter)
 *       26 = Internal     (CUDA launch / runtime failure)
 *     the message for the last failure on a handle is in sf_tm_last_error().
 *     No C++ exception crosses this ABI.
 *   - all device pointers are caller-owned; the handle owns only scratch
 *     (grown once, reused; no allocation in a steady-state call).
 *   - every call is stream-ordered and asynchronous on `stream`
 *     (a cudaStream_t passed as void*; NULL = legacy default stream).
 *   - handles are thread-compatible: one handle per role thread, or external
 *     synchronisation (the reference runs one thread per role,
 *     wall_runtime.cpp:296-315). The handle's scratch (metric partials,
 *     host-call staging) is shared by its calls, so calls on one handle must
 *     be ordered: one stream per handle, or a handle per concurrent stream.
 *
 * The math (decisions P1-P9 of SURVEY.md §8) is pinned in DESIGN.md §2 and
 * restated in fp64 by oracle/sf_oracle.c.
 */
#ifndef STALEFLOW_TRAIN_MATH_H_
#define STALEFLOW_TRAIN_MATH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SF_TM_ABI_VERSION 1

/* Error codes: numerically identical to staleflow::Errc (result.hpp:14-47). */
#define SF_TM_OK 0
#define SF_TM_CONFIG_ERROR 21
#define SF_TM_INTERNAL 26

/* Element types of the V-wide logits / router-logit rows. */
#define SF_TM_F32 0
#define SF_TM_BF16 1

/* Element types of recorded expert indices (R3). */
#define SF_TM_IDX_I32 0
#define SF_TM_IDX_U8 1

/* GRPO group-std modes (decision P2/P3). */
#define SF_TM_STD_UNBIASED 0   /* sample std, N-1 (veRL) */
#define SF_TM_STD_POPULATION 1 /* N */
#define SF_TM_STD_NONE 2       /* Dr.GRPO: A = r - mean */

/* Loss normalisation modes. */
#define SF_TM_NORM_TOKEN_MEAN 0     /* DAPO: 1 / sum(mask) over the launch  */
#define SF_TM_NORM_SEQ_MEAN 1       /* GRPO: mean over seqs of token-means   */
#define SF_TM_NORM_EXPLICIT 2       /* caller-supplied inv_norm (version-level N) */

/* Masked-row contract for dlogits (decision P7). */
#define SF_TM_MASKED_ZERO_FILL 0 /* dense: masked rows of dlogits are written as 0 */
#define SF_TM_MASKED_SKIP 1      /* sparse: masked rows of dlogits are left untouched */

/* Metrics written by the loss (device float[SF_TM_NUM_METRICS]); each is a
 * w-weighted sum with w_t = mask_t * inv_norm_t, i.e. a masked token-mean
 * under SF_TM_NORM_TOKEN_MEAN. */
#define SF_TM_M_LOSS 0      /* sum w*(pg + beta*kl - ent_coef*H)         */
#define SF_TM_M_PG 1        /* sum w*pg                                  */
#define SF_TM_M_KL 2        /* sum w*kl_k3(ref || cur)                   */
#define SF_TM_M_ENTROPY 3   /* sum w*H                                   */
#define SF_TM_M_CLIPFRAC 4  /* sum w*[clipped]                           */
#define SF_TM_M_RATIO 5     /* sum w*ratio                               */
#define SF_TM_M_ACTIVE 6    /* number of loss-active tokens (w != 0)     */
#define SF_TM_M_PPO_KL 7    /* sum w*(old_logp - logp)                   */
#define SF_TM_NUM_METRICS 8

typedef struct sf_tm_handle* sf_tm_t;

typedef struct sf_tm_loss_params {
  float clip_eps_low;    /* P4: 0.2                                  */
  float clip_eps_high;   /* P4: 0.28 (DAPO clip-higher)              */
  float dual_clip_c;     /* P4: 0 = off, else > 1 (e.g. 3)           */
  float kl_beta;         /* P5: 0 = pure DAPO                         */
  float entropy_coef;    /* P6: 0 = entropy is a metric only          */
  float inv_temperature; /* P1: 1/tau, 1.0 = no temperature           */
  int32_t norm_mode;     /* SF_TM_NORM_*                              */
  float inv_norm;        /* used when norm_mode == SF_TM_NORM_EXPLICIT */
  int32_t masked_rows;   /* SF_TM_MASKED_*                            */
  int32_t kl_mode;       /* P5: SF_TM_KL_* estimator (0 = k3, default) */
} sf_tm_loss_params;

/* KL estimators, d = ref_logp - logp (veRL's kl_loss_type names in brackets):
 * K3 e^d - d - 1 [low_var_kl], K1 -d [kl], K2 d^2/2 [mse], ABS |d| [abs]. */
#define SF_TM_KL_K3 0
#define SF_TM_KL_K1 1
#define SF_TM_KL_K2 2
#define SF_TM_KL_ABS 3

/* Fills the DAPO defaults above (eps 0.2/0.28, no dual clip, beta 0,
 * ent 0, tau 1, token-mean, zero-fill). */
void sf_tm_default_loss_params(sf_tm_loss_params* p);

/* ---- handle ------------------------------------------------------------ */
int sf_tm_create(int device, sf_tm_t* out);
int sf_tm_destroy(sf_tm_t h);
const char* sf_tm_last_error(sf_tm_t h);
int sf_tm_abi_version(void);
/* Number of kernel launches issued on this handle since creation (evidence for
 * the bench's gpu_launches count). */
uint64_t sf_tm_launch_count(sf_tm_t h);
/* Which row kernel the last row-kernel call on this handle launched:
 * *kernel 0 = streaming TMA ring, 1 = generic two-pass, 2 = fused TMEM/smem
 * row-store loss kernel, 4 = the fused vocab-parallel (peer-mailbox) kernel,
 * 5 = the forward-only streaming kernel; *cluster = CTAs
 * per row; *grid = CTAs launched. Any pointer may be NULL. */
int sf_tm_last_launch(sf_tm_t h, int32_t* kernel, int32_t* cluster, int32_t* grid);
/* Row streams of the last fused-loss launch (kernel 2 or 4): 1, 2 or 4 rows of
 * a CTA in flight side by side, chosen from the row slice width (narrow
 * vocab-parallel shards run 2 or 4; the environment variable SFTM_LOSS_NS
 * forces a count for tuning). 1 for every other kernel. */
int sf_tm_last_launch_streams(sf_tm_t h, int32_t* streams);

/* ---- a6: varlen packing metadata --------------------------------------
 * seq_lens[B] (>= 0), prompt_lens[B] (optional; tokens [0, prompt_len) of a
 * sequence are loss-masked), group_ids[B] (optional).
 * Out: cu_seqlens[B+1] (exclusive scan, int32), seq_id[T] (optional),
 * mask[T] u8 (optional, needs prompt_lens or gives all-ones), tok_group[T]
 * (optional, needs group_ids). T = sum(seq_lens) must be passed and match.
 * Bit-exact against the oracle. Anchor: MicroBatch per-sample keys
 * types.hpp:48-59; packing is a reference non-goal. */
int sf_tm_varlen_meta(sf_tm_t h, const int32_t* seq_lens, const int32_t* prompt_lens,
                      const int32_t* group_ids, int64_t B, int64_t T, int32_t* cu_seqlens,
                      int32_t* seq_id, uint8_t* mask, int32_t* tok_group, void* stream);

/* ---- a3: GRPO group advantage ------------------------------------------
 * A_i = (r_i - mean_g(i)) / (std_g(i) + eps); groups keyed by arbitrary int32
 * ids (need not be contiguous: the bus delivers in readiness order,
 * transfer_queue.cpp:162-175). Groups whose rewards are all equal give A = 0
 * exactly (P3). Optional out_group_size[B] (int32, bit-exact).
 * Replaces the Advantages stage stub (controller.cpp:79, sim_runtime.cpp:304-350). */
int sf_tm_grpo_advantage(sf_tm_t h, const float* rewards, const int32_t* group_ids, int64_t B,
                         float eps, int32_t std_mode, float* out_adv, int32_t* out_group_size,
                         void* stream);

/* ---- a1: fused log-softmax gather, forward only -------------------------
 * logits[T, V] row stride ld (elements), dtype SF_TM_F32 / SF_TM_BF16;
 * targets[T] in [0, V). Out (each optional): logp[T], entropy[T], lse[T] fp32.
 * One HBM pass (2V or 4V bytes/token). Producer of the "logp"/"ref_logp"
 * fields (controller.cpp:76-77). */
int sf_tm_logprob_fwd(sf_tm_t h, const void* logits, int32_t dtype, int64_t T, int64_t V,
                      int64_t ld, const int32_t* targets, float inv_temperature, float* out_logp,
                      float* out_entropy, float* out_lse, void* stream);

/* Host-buffer forms for the stage seams (include/staleflow/train_math_seam.hpp):
 * ActorFwd / RefLogP put a `logp` / `ref_logp` payload per sample
 * (proj/src/sim_runtime.cpp:322-334, proj/src/wall_runtime.cpp:126-129) and the
 * Advantages stage an `advantage` (controller.cpp:79). Inputs and outputs are
 * host arrays (pinned for asynchronous copies); logits stay on the device.
 * Results are valid once `stream` is synchronised. */
/* Blocks until all work queued on `stream` (by this library or not) is done. */
int sf_tm_sync(sf_tm_t h, void* stream);
int sf_tm_logprob_fwd_host(sf_tm_t h, const void* logits, int32_t dtype, int64_t T, int64_t V, int64_t ld,
                           const int32_t* h_targets, float inv_temperature, float* h_logp, float* h_entropy,
                           void* stream);
int sf_tm_grpo_advantage_host(sf_tm_t h, const float* h_rewards, const int32_t* h_group_ids, int64_t B, float eps,
                              int32_t std_mode, float* h_adv, void* stream);

/* ---- a4 prologue: per-token advantage and loss weight --------------------
 * From cu_seqlens[B+1], adv_seq[B], mask[T] (u8, NULL = all active):
 * out_adv_tok[T] = adv_seq[seq(t)], out_w_tok[T] = mask_t * inv_norm_t. */
int sf_tm_token_weights(sf_tm_t h, const int32_t* cu_seqlens, int64_t B, const float* adv_seq,
                        const uint8_t* mask, int64_t T, int32_t norm_mode, float inv_norm,
                        float* out_adv_tok, float* out_w_tok, void* stream);

/* ---- a1+a4+a2: the fused hot path ---------------------------------------
 * Per token t with weight w_t (0 = masked) and advantage A_t:
 *   logp, H from the logits row; ratio = exp(logp - old_logp);
 *   pg = -min(ratio*A, clip(ratio, 1-eps_lo, 1+eps_hi)*A)  (+ dual clip);
 *   kl = exp(ref - logp) - (ref - logp) - 1;  l = pg + beta*kl - ent_coef*H;
 *   loss = sum_t w_t * l_t;  dlogits = d loss / d logits.
 * adv_tok/w_tok come from sf_tm_token_weights. dlogits has the logits dtype,
 * row stride ld_d; dlogits == logits (in place) is supported. out_metrics is
 * device float[SF_TM_NUM_METRICS] (deterministic fixed-order reduction).
 * out_logp / out_entropy optional. Replaces the trainer seam latency
 * (sim_runtime.cpp:441, wall_runtime.cpp:197).
 * Kernel choice (transparent): any element-aligned rows take the single-pass
 * kernel when dlogits rows sit at the same 16-byte phase as the logits rows
 * (same base alignment mod 16, stride difference a multiple of 16 bytes) and
 * a row slice fits the row store; otherwise a two-pass kernel computes the
 * same outputs. Narrow rows (a row taking a few 12 KB chunks, e.g. a
 * vocab-parallel shard) run 2 or 4 rows side by side per CTA ("row streams").
 * sf_tm_last_launch / sf_tm_last_launch_streams report which ran. */
int sf_tm_pg_loss_fwd_bwd(sf_tm_t h, const void* logits, int32_t dtype, int64_t T, int64_t V,
                          int64_t ld, const int32_t* targets, const float* old_logp,
                          const float* ref_logp, const float* adv_tok, const float* w_tok,
                          const sf_tm_loss_params* params, void* dlogits, int64_t ld_d,
                          float* out_metrics, float* out_logp, float* out_entropy, void* stream);

/* ---- whole trainer micro-batch from HOST buffers (the seam call) --------
 * Copies the bus fields of one MicroBatch (types.hpp:48-59; trainer field set
 * [advantage, logp, ref_logp, response, reward], controller.cpp:80) from host
 * memory (pinned for async DMA), runs varlen meta -> GRPO advantage -> token
 * weights -> fused loss fwd+bwd on device-resident logits (the LM-head output,
 * which never crosses the bus), and copies the metrics back to h_metrics
 * (valid after `stream` is synchronised).
 *   h_targets[T], h_old_logp[T], h_ref_logp[T]: packed per-token fields;
 *   h_seq_lens[B], h_prompt_lens[B] (optional), h_rewards[B], h_group_ids[B];
 *   h_mask[T] (optional; overrides prompt_lens-derived mask).
 * If adv_eps < 0 the rewards are taken as precomputed advantages.
 * Pipelined: the H2D copies and the varlen / GRPO / token-weight kernels run on
 * a handle-owned side stream (two alternating scratch stages), overlapping the
 * previous call's fused loss on `stream`; `stream` waits for them before the
 * loss. Back-to-back calls need no synchronisation between them, but the host
 * input buffers stay in use until sf_tm_wait_host_inputs returns (or `stream`
 * is synchronised). */
int sf_tm_pg_step_host(sf_tm_t h, const void* logits, int32_t dtype, int64_t T, int64_t V,
                       int64_t ld, const int32_t* h_targets, const float* h_old_logp,
                       const float* h_ref_logp, const uint8_t* h_mask, const int32_t* h_seq_lens,
                       const int32_t* h_prompt_lens, const float* h_rewards,
                       const int32_t* h_group_ids, int64_t B, float adv_eps, int32_t std_mode,
                       const sf_tm_loss_params* params, void* dlogits, int64_t ld_d,
                       float* h_metrics, void* stream);

/* Blocks until the host input buffers of every sf_tm_pg_step_host call made
 * on this handle so far have been read (their H2D copies are complete), so the
 * caller may refill them. Does not wait for the loss itself. */
int sf_tm_wait_host_inputs(sf_tm_t h);

/* ---- a5: R3 rollout routing replay gate ---------------------------------
 * router_logits[L*T, E] (dtype), rec_idx[L*T, k] (SF_TM_IDX_I32 / _U8).
 * renorm = 1: w_j = softmax over the k recorded experts (P8, norm_topk_prob);
 * renorm = 0: w_j = softmax over all E, gathered at the recorded experts.
 * out_w[L*T, k] fp32; out_idx[L*T, k] int32 bit-exact copy of the replayed
 * indices (optional); out_mismatch (optional, device uint32[L+1]): per layer
 * the number of tokens whose trainer top-k set (ties -> lowest index, P9)
 * differs from the recorded set, and the total in [L]. L = layers, rows are
 * layer-major. */
int sf_tm_r3_gate_fwd(sf_tm_t h, const void* router_logits, int32_t dtype, int64_t L, int64_t T,
                      int64_t E, int64_t k, const void* rec_idx, int32_t idx_dtype, int32_t renorm,
                      float* out_w, int32_t* out_idx, uint32_t* out_mismatch, void* stream);

/* Backward of sf_tm_r3_gate_fwd: given w (its output) and dw[L*T, k], writes
 * dlogits[L*T, E] (router-logit dtype); non-recorded experts get 0 when
 * renorm = 1. renorm = 0 re-reads router_logits. */
int sf_tm_r3_gate_bwd(sf_tm_t h, const void* router_logits, int32_t dtype, int64_t L, int64_t T,
                      int64_t E, int64_t k, const void* rec_idx, int32_t idx_dtype, int32_t renorm,
                      const float* w, const float* dw, void* dlogits, void* stream);

/* R3 transport ("GPU-resident"): the
 * rollout's routed_experts bus field is token-major, rec_token_major[T, L, k]
 * (the concatenated per-sample payloads, copied to the device once); this
 * writes the gate's layer-major operand rec_layer_major[L, T, k] on the
 * device, bit-exactly, so the record never makes a host transpose pass.
 * Out of place. idx_dtype SF_TM_IDX_U8 / _I32. */
int sf_tm_r3_record_layer_major(sf_tm_t h, const void* rec_token_major, int32_t idx_dtype, int64_t T, int64_t L,
                                int64_t k, void* rec_layer_major, void* stream);

/* ---- a7: vocab-parallel (logits sharded over P ranks by vocab) ----------
 * Pass 1 (local): per-row partial stats of this rank's shard
 * [vocab_start, vocab_start + Vp): out_stats[T*4] = {max z, sum e^(z-max),
 * sum e^(z-max)(z-max), z_target or NaN if the target is not in the shard}.
 * The caller all-gathers stats over ranks (NCCL) into gathered[P*T*4]. */
int sf_tm_vp_partial_stats(sf_tm_t h, const void* logits_shard, int32_t dtype, int64_t T,
                           int64_t Vp, int64_t ld, int64_t vocab_start, const int32_t* targets,
                           float inv_temperature, float* out_stats, void* stream);

/* Pass 2: combine gathered stats of all P shards, compute the loss exactly as
 * sf_tm_pg_loss_fwd_bwd (metrics are identical on every rank: each rank
 * computes the full per-row scalars) and write this shard's dlogits. */
int sf_tm_vp_loss_fwd_bwd(sf_tm_t h, const void* logits_shard, int32_t dtype, int64_t T,
                          int64_t Vp, int64_t ld, int64_t vocab_start, const float* gathered_stats,
                          int32_t P, const int32_t* targets, const float* old_logp,
                          const float* ref_logp, const float* adv_tok, const float* w_tok,
                          const sf_tm_loss_params* params, void* dlogits, int64_t ld_d,
                          float* out_metrics, float* out_logp, float* out_entropy, void* stream);

/* ---- a7 fused: vocab-parallel with the exchange inside the kernel --------
 * The two-pass path above reads each shard row twice (stats, then backward:
 * 6V/P bytes per token per rank) with an NCCL all_gather in between. The
 * fused path reads it once (4V/P): every rank runs one persistent kernel on
 * its shard with the same row schedule, and the per-row partial statistics
 * travel between the ranks' control warps through peer-mapped mailboxes
 * (NVLink P2P stores with system-scope release/acquire).
 *
 * Setup, once per process group (any transport for the 64-byte handles):
 *   sf_tm_vp_mailbox_create(h, P, rank, my_handle);        // allocates + exports
 *   all-gather the P handles in rank order (P * SF_TM_IPC_HANDLE_BYTES bytes);
 *   sf_tm_vp_mailbox_open(h, all_handles);                 // maps the peers
 * Then every rank calls sf_tm_vp_fused_loss_fwd_bwd with the same T, w_tok and
 * call sequence (calls are matched by order). Outputs are as
 * sf_tm_vp_loss_fwd_bwd; metrics, logp and entropy are identical on all ranks.
 * A call that returns an error before launching does not advance the call
 * sequence; since shapes and pointers may differ per rank, a caller should
 * first agree on sf_tm_vp_fused_check across the group (e.g. an all-reduce
 * of the result) and use the two-pass form on every rank if any rank fails.
 * A launch whose peers never launch stops waiting after SF_TM_XP_TIMEOUT_S
 * seconds (environment, default 300), finishes with invalid outputs and
 * flags the handle: every later fused call on it returns SF_TM_INTERNAL. The
 * CUDA context stays usable (no trap). */
#define SF_TM_IPC_HANDLE_BYTES 64
int sf_tm_vp_mailbox_create(sf_tm_t h, int32_t P, int32_t rank, void* ipc_handle_out);
int sf_tm_vp_mailbox_open(sf_tm_t h, const void* ipc_handles);
int sf_tm_vp_fused_loss_fwd_bwd(sf_tm_t h, const void* logits_shard, int32_t dtype, int64_t T, int64_t Vp,
                                int64_t ld, int64_t vocab_start, const int32_t* targets, const float* old_logp,
                                const float* ref_logp, const float* adv_tok, const float* w_tok,
                                const sf_tm_loss_params* params, void* dlogits, int64_t ld_d, float* out_metrics,
                                float* out_logp, float* out_entropy, void* stream);

/* The checks sf_tm_vp_fused_loss_fwd_bwd makes on its shard (mailboxes open
 * and healthy, dtype, element-aligned rows with the dlogits rows at the logits
 * rows' 16-B phase — an odd shard width or stride runs in 16-B sector
 * coordinates —, shard row fits one CTA's row store), with no side effect.
 * Ok or ConfigError / Internal. */
int sf_tm_vp_fused_check(sf_tm_t h, const void* logits_shard, int32_t dtype, int64_t T, int64_t Vp, int64_t ld,
                         const void* dlogits, int64_t ld_d);

/* ---- pinned host staging (for the C++ seam adapter) ----------------------
 * Page-locked host memory so the seam's H2D copies are asynchronous DMA.
 * Returns ConfigError for bytes == 0 or out == NULL, Internal on CUDA errors. */
int sf_tm_host_alloc(size_t bytes, void** out);
int sf_tm_host_free(void* p);
/* Asynchronous host -> device copy on `stream` (a DMA when src is pinned). */
int sf_tm_h2d(sf_tm_t h, void* dst, const void* src, size_t bytes, void* stream);

/* ---- synthetic inputs (bench / tests) ------------------------------------
 * Counter-based, seeded with the reference's SplitMix64 (rng.hpp:17-39)
 * evaluated at element index: u_i = mix64(seed + (i+1)*0x9e3779b97f4a7c15),
 * i.e. the i-th output of staleflow::SplitMix64(seed).
 * Logits row t: N(0, sigma^2) (Box-Muller), plus a peak logit +U(peak_lo,
 * peak_hi) at id peak_id[t] (optional), plus a fraction `outlier_frac` of
 * entries set to +-30; rounded to the dtype. */
int sf_tm_synth_logits(sf_tm_t h, void* logits, int32_t dtype, int64_t T, int64_t V, int64_t ld,
                       uint64_t seed, float sigma, const int32_t* peak_id, float peak_lo,
                       float peak_hi, float outlier_frac, void* stream);

/* ---- testing hook ---------------------------------------------------------
 * on != 0 routes all row kernels to the generic two-pass (non-TMA) kernel so
 * tests can cover both code paths; process-wide. Not for production use. */
int sf_tm_debug_force_generic(int on);

/* Wires P handles on ONE device into an in-process vocab-parallel group
 * (rank r = handles[r]) without CUDA IPC, and caps each rank's exchange grid
 * at grid_per_rank CTAs (0 = no cap) so the P ranks' kernels, launched on P
 * streams, are co-resident on the GPU. Emulates P GPUs on one for tests and
 * the narrow-shard measurement; not for production use. */
int sf_tm_debug_vp_local_group(sf_tm_t* handles, int32_t P, int32_t grid_per_rank);

/* on a non-NULL device buffer of 16 uint64 (zeroed by the caller), the fused
 * loss kernel accumulates per-role clock64 cycle sums: for role r in
 * {producer, forward, control, backward}: [3r] active, [3r+1] and [3r+2] the
 * two wait classes, [12+r] warp count. NULL turns it off. Debug/tuning only. */
int sf_tm_debug_wait_counters(void* dev_counters);

#ifdef __cplusplus
}
#endif

#endif /* STALEFLOW_TRAIN_MATH_H_ */
