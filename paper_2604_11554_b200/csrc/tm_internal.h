// SPDX-License-Identifier: Apache-2.0
// Internal interfaces between the C-ABI layer (tm_api.cu) and the kernel
// translation units. Nothing here crosses the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace sftm {

enum RowMode : int {
  kModeFwd = 0,      // a1: logp / entropy / lse, one streaming pass
  kModeFwdBwd = 1,   // a1+a4+a2: fused loss fwd+bwd, row resident in (cluster) smem
  kModeVpStats = 2,  // a7 pass 1: partial stats of a vocab shard
  kModeVpBwd = 3,    // a7 pass 2: combine gathered stats, loss, shard dlogits
};

struct RowArgs {
  const void* logits = nullptr;
  int dtype = 0;  // SF_TM_F32 / SF_TM_BF16
  int64_t T = 0, V = 0, ld = 0;
  int64_t vocab_start = 0;
  const int32_t* targets = nullptr;
  float inv_tau = 1.f;
  // loss inputs
  const float* old_logp = nullptr;
  const float* ref_logp = nullptr;
  const float* adv_tok = nullptr;
  const float* w_tok = nullptr;
  float eps_lo = 0.2f, eps_hi = 0.28f, dual_c = 0.f, beta = 0.f, ent_coef = 0.f;
  int masked_skip = 0;
  int kl_mode = 0;  // SF_TM_KL_*
  void* dlogits = nullptr;
  int64_t ld_d = 0;
  // outputs
  float* out_logp = nullptr;
  float* out_entropy = nullptr;
  float* out_lse = nullptr;
  float* out_stats = nullptr;  // VpStats: [T,4]
  const float* gathered = nullptr;  // VpBwd: [P,T,4]
  int P = 1;
  float* out_metrics = nullptr;
  // fused vocab-parallel exchange (sf_tm_vp_fused_loss_fwd_bwd): every rank's
  // peer-mapped mailbox buffer, indexed by rank (xp_mail[xp_rank] is local)
  void* xp_mail[8] = {};
  int xp_rank = 0, xp_P = 0;
  unsigned long long xp_epoch = 0;  // launch sequence number, identical on all ranks
  int* xp_err = nullptr;    // host-mapped: set to 1 when a launch gave up waiting for a peer
  int* xp_abort = nullptr;  // device: first CTA to time out tells the others to stop waiting
  unsigned long long xp_timeout_ns = 300000000000ull;  // SF_TM_XP_TIMEOUT_S (default 300 s)
  int xp_grid = 0;          // > 0: cap the exchange grid (emulated ranks sharing one GPU)
  // optional wait-time instrumentation (debug only): per-role clock64 sums
  unsigned long long* dbg = nullptr;
  // workspace (owned by the handle)
  double* partials = nullptr;  // [max_blocks * 8]
  unsigned* ticket = nullptr;
  int max_partial_blocks = 0;
};

// Peer mailbox geometry (fused vocab-parallel). One message = 4 x 64-bit words
// {m2, s, w, z_target|NaN}, each word = (32-bit tag << 32) | float bits, tag =
// epoch << 20 | row + 1. Every word is written and read with single-copy-atomic
// 8-byte accesses, so a reader that sees all four tags match has the whole
// message: no fences on either side (a system-scope release per row cost more
// than the row's HBM time at narrow shards).
constexpr int kXpMaxP = 8;
constexpr int kXpMaxCtas = 256;
#ifndef SFTM_XP_MAILD
#define SFTM_XP_MAILD 16
#endif
constexpr int kXpMailD = SFTM_XP_MAILD;
struct alignas(32) XpMsg {
  unsigned long long w[4];
};
// halves alternate by epoch parity so a rank one launch ahead never overwrites
// messages a slower peer has not read yet
constexpr size_t kXpMailboxBytes = size_t(2) * kXpMaxCtas * kXpMailD * kXpMaxP * sizeof(XpMsg);
__host__ __device__ inline size_t xp_index(unsigned long long epoch, int cta, int slot, int src) {
  return ((static_cast<size_t>(epoch & 1) * kXpMaxCtas + cta) * kXpMailD + slot) * kXpMaxP + src;
}

// One-time launch setup (cudaFuncSetAttribute, occupancy queries) is per
// device: a process may drive several GPUs. Indexed by the current device.
struct PerDevice {
  int v[64];
  PerDevice() {
    for (int& x : v) x = -1;
  }
  int& operator()() {
    int d = 0;
    cudaGetDevice(&d);
    return v[d & 63];
  }
};

struct LaunchInfo {
  int kernel = 0;  // 0 = ring (TMA) kernel, 1 = generic two-pass kernel
  int cluster = 1;
  int grid = 0;
  int launches = 0;
  int streams = 1;  // row streams of the fused loss kernel (1 = one row at a time per CTA)
};

// Launches the row kernel for `mode`. Returns 0 or a cudaError_t value; on a
// config problem returns -1 with *err set.
int launch_rows(const RowArgs& a, int mode, cudaStream_t s, std::string* err, LaunchInfo* info);
// Fused vocab-parallel loss (one CTA per SM, peer-mailbox exchange); -2 if the
// shard is not eligible (then the caller reports a config error).
int launch_loss_xp(const RowArgs& a, cudaStream_t s, LaunchInfo* info);
// Whether a shard row of Vp elements fits one CTA's row store (the fused
// vocab-parallel kernel runs one CTA per row per rank).
bool loss_xp_eligible(int dtype, int64_t Vp, bool unaligned);
// One-time setup of every peer-exchange kernel instantiation on the current
// device (called when the mailboxes are wired, before any rank can be waiting
// in a launch). Returns a cudaError_t value.
int prepare_loss_xp();
// Forward-only streaming pass (kModeFwd / kModeVpStats) on 16-B aligned rows (tm_fwd.cu).
int launch_fwd_stream(const RowArgs& a, int mode, cudaStream_t s, LaunchInfo* info);

// Forces the generic (non-TMA) kernel; used by tests to cover both paths.
void set_force_generic(bool on);
// Debug: device buffer of kDbgCounters u64 that the fused loss kernel fills with
// per-role busy/wait cycle sums (nullptr = off).
constexpr int kDbgCounters = 16;
void set_debug_counters(unsigned long long* dev_ptr);
unsigned long long* debug_counters();

int launch_varlen_meta(const int32_t* seq_lens, const int32_t* prompt_lens,
                       const int32_t* group_ids, int64_t B, int64_t T, int32_t* cu_seqlens,
                       int32_t* seq_id, uint8_t* mask, int32_t* tok_group, int32_t* d_total,
                       cudaStream_t s, int* launches);

int launch_grpo_advantage(const float* rewards, const int32_t* group_ids, int64_t B, float eps,
                          int std_mode, float* out_adv, int32_t* out_group_size, cudaStream_t s,
                          int* launches);

int launch_token_weights(const int32_t* cu_seqlens, int64_t B, const float* adv_seq,
                         const uint8_t* mask, int64_t T, int norm_mode, float inv_norm,
                         float* out_adv_tok, float* out_w_tok, int32_t* scratch_cnt,
                         unsigned* scratch_ticket, int64_t* scratch_tot, cudaStream_t s,
                         int* launches);

int launch_r3_fwd(const void* logits, int dtype, int64_t L, int64_t T, int64_t E, int64_t k,
                  const void* rec_idx, int idx_dtype, int renorm, float* out_w, int32_t* out_idx,
                  uint32_t* out_mismatch, cudaStream_t s, int* launches);

int launch_r3_bwd(const void* logits, int dtype, int64_t L, int64_t T, int64_t E, int64_t k,
                  const void* rec_idx, int idx_dtype, int renorm, const float* w, const float* dw,
                  void* dlogits, cudaStream_t s, int* launches);

// routed_experts record, token-major [T, L, k] -> layer-major [L, T, k] (bit-exact)
int launch_rec_layer_major(const void* rec_tok, int idx_dtype, int64_t T, int64_t L, int64_t k, void* rec_layer,
                           cudaStream_t s, int* launches);

int launch_synth_logits(void* logits, int dtype, int64_t T, int64_t V, int64_t ld, uint64_t seed,
                        float sigma, const int32_t* peak_id, float peak_lo, float peak_hi,
                        float outlier_frac, cudaStream_t s, int* launches);

}  // namespace sftm
