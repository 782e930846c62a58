// SPDX-License-Identifier: Apache-2.0
//
// C-ABI layer of include/staleflow/train_math.h: argument validation, error
// mapping onto staleflow::Errc (proj/include/staleflow/result.hpp:14-47: Ok=0,
// ConfigError=21, Internal=26), handle-owned scratch, and the host-buffer
// trainer-seam call sf_tm_pg_step_host. No exception crosses this boundary.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "staleflow/train_math.h"
#include "tm_internal.h"

struct sf_tm_handle {
  int device = 0;
  std::string err;
  uint64_t launches = 0;
  sftm::LaunchInfo last;  // last row-kernel launch (sf_tm_last_launch)
  // fused vocab-parallel peer mailboxes (sf_tm_vp_mailbox_*)
  void* xp_local = nullptr;
  void* xp_mail[sftm::kXpMaxP] = {};
  int xp_P = 0, xp_rank = -1;
  bool xp_ready = false;
  bool xp_local_group = false;  // peers wired in-process (sf_tm_debug_vp_local_group)
  unsigned long long xp_epoch = 0;
  int* xp_err_h = nullptr;  // host-mapped launch-failure word (peer timeout)
  int* xp_err_d = nullptr;  // its device alias
  int* xp_abort = nullptr;  // device: stop-waiting flag shared by a launch's CTAs
  int xp_grid = 0;
  // metric partials for the deterministic row-kernel reduction
  double* partials = nullptr;
  unsigned* ticket = nullptr;
  int max_partial_blocks = 0;
  // token-weight scratch
  int32_t* cnt = nullptr;
  int64_t cnt_cap = 0;
  unsigned* ticket2 = nullptr;
  int64_t* tot = nullptr;
  // sf_tm_pg_step_host scratch
  int64_t tcap = 0, bcap = 0;
  int32_t* d_targets = nullptr;
  float* d_old = nullptr;
  float* d_ref = nullptr;
  uint8_t* d_mask = nullptr;
  float* d_advtok = nullptr;
  float* d_wtok = nullptr;
  int32_t* d_lens = nullptr;
  int32_t* d_plens = nullptr;
  float* d_rewards = nullptr;
  int32_t* d_gids = nullptr;
  int32_t* d_cu = nullptr;
  float* d_adv = nullptr;
  int32_t* d_total = nullptr;
  float* d_metrics = nullptr;
  // sf_tm_pg_step_host pipeline: two prologue stages (bus-field H2D, varlen,
  // GRPO, token weights) run on `side` while the caller's stream runs the
  // previous micro-batch's fused loss; each stage is reused two calls later,
  // after the loss that read it (free_ev).
  struct HostStage {
    int64_t tcap = 0, bcap = 0;
    int32_t* targets = nullptr;
    float* old = nullptr;
    float* ref = nullptr;
    uint8_t* mask = nullptr;
    float* advtok = nullptr;
    float* wtok = nullptr;
    int32_t* lens = nullptr;
    int32_t* plens = nullptr;
    float* rewards = nullptr;
    int32_t* gids = nullptr;
    int32_t* cu = nullptr;
    float* adv = nullptr;
    int32_t* cnt = nullptr;
    int32_t* total = nullptr;
    unsigned* ticket = nullptr;
    int64_t* tot = nullptr;
    cudaEvent_t ready_ev = nullptr;
    cudaEvent_t free_ev = nullptr;
  } st[2];
  int st_next = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t h2d_ev = nullptr;  // after the latest call's host-input copies (side stream)
};

namespace {

constexpr int kMaxPartialBlocks = 4096;

int fail(sf_tm_t h, int code, const std::string& msg) {
  if (h) h->err = msg;
  return code;
}

int cuda_fail(sf_tm_t h, int e, const char* where) {
  if (e == -1) return fail(h, SF_TM_CONFIG_ERROR, std::string(where) + ": " + h->err);
  const cudaError_t ce = static_cast<cudaError_t>(e);
  return fail(h, SF_TM_INTERNAL,
              std::string(where) + ": " + cudaGetErrorName(ce) + ": " + cudaGetErrorString(ce));
}

int check_cuda(sf_tm_t h, int e, const char* where) {
  if (e == 0) return SF_TM_OK;
  return cuda_fail(h, e, where);
}

int use_device(sf_tm_t h) {
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != h->device) {
    const cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return cuda_fail(h, e, "cudaSetDevice");
  }
  return SF_TM_OK;
}

bool bad_dtype(int32_t d) { return d != SF_TM_F32 && d != SF_TM_BF16; }

template <typename P>
int grow(sf_tm_t h, P** p, int64_t n, const char* what) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  if (n <= 0) return SF_TM_OK;
  const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), static_cast<size_t>(n) * sizeof(P));
  if (e != cudaSuccess) return cuda_fail(h, e, what);
  return SF_TM_OK;
}

int ensure_cnt(sf_tm_t h, int64_t B) {
  if (B <= h->cnt_cap) return SF_TM_OK;
  int64_t cap = B < 1024 ? 1024 : B;
  int rc = grow(h, &h->cnt, cap, "scratch cnt");
  if (rc) return rc;
  h->cnt_cap = cap;
  return SF_TM_OK;
}

int check_loss_params(sf_tm_t h, const sf_tm_loss_params* p) {
  if (!p) return fail(h, SF_TM_CONFIG_ERROR, "params is NULL");
  if (!(p->clip_eps_low >= 0.f && p->clip_eps_low < 1.f))
    return fail(h, SF_TM_CONFIG_ERROR, "clip_eps_low must be in [0, 1)");
  if (!(p->clip_eps_high >= 0.f && std::isfinite(p->clip_eps_high)))
    return fail(h, SF_TM_CONFIG_ERROR, "clip_eps_high must be >= 0");
  if (!(p->dual_clip_c == 0.f || p->dual_clip_c > 1.f))
    return fail(h, SF_TM_CONFIG_ERROR, "dual_clip_c must be 0 (off) or > 1");
  if (!std::isfinite(p->kl_beta) || !std::isfinite(p->entropy_coef))
    return fail(h, SF_TM_CONFIG_ERROR, "kl_beta / entropy_coef must be finite");
  if (!(p->inv_temperature > 0.f && std::isfinite(p->inv_temperature)))
    return fail(h, SF_TM_CONFIG_ERROR, "inv_temperature must be > 0");
  if (p->norm_mode < 0 || p->norm_mode > 2)
    return fail(h, SF_TM_CONFIG_ERROR, "norm_mode must be SF_TM_NORM_*");
  if (p->norm_mode == SF_TM_NORM_EXPLICIT && !(std::isfinite(p->inv_norm) && p->inv_norm >= 0.f))
    return fail(h, SF_TM_CONFIG_ERROR, "inv_norm must be finite and >= 0");
  if (p->masked_rows != SF_TM_MASKED_ZERO_FILL && p->masked_rows != SF_TM_MASKED_SKIP)
    return fail(h, SF_TM_CONFIG_ERROR, "masked_rows must be SF_TM_MASKED_*");
  if (p->kl_mode < SF_TM_KL_K3 || p->kl_mode > SF_TM_KL_ABS)
    return fail(h, SF_TM_CONFIG_ERROR, "kl_mode must be SF_TM_KL_*");
  return SF_TM_OK;
}

int check_rows(sf_tm_t h, const void* logits, int32_t dtype, int64_t T, int64_t V, int64_t ld,
               const int32_t* targets) {
  if (bad_dtype(dtype)) return fail(h, SF_TM_CONFIG_ERROR, "dtype must be SF_TM_F32 or SF_TM_BF16");
  if (T < 0) return fail(h, SF_TM_CONFIG_ERROR, "T must be >= 0");
  if (V <= 0 || V > (int64_t(1) << 31) - 1) return fail(h, SF_TM_CONFIG_ERROR, "V out of range");
  if (ld < V) return fail(h, SF_TM_CONFIG_ERROR, "ld must be >= V");
  if (T > 0 && (!logits || !targets))
    return fail(h, SF_TM_CONFIG_ERROR, "logits and targets are required");
  return SF_TM_OK;
}

void fill_loss(sftm::RowArgs& a, const sf_tm_loss_params* p) {
  a.eps_lo = p->clip_eps_low;
  a.eps_hi = p->clip_eps_high;
  a.dual_c = p->dual_clip_c;
  a.beta = p->kl_beta;
  a.ent_coef = p->entropy_coef;
  a.inv_tau = p->inv_temperature;
  a.masked_skip = p->masked_rows == SF_TM_MASKED_SKIP ? 1 : 0;
  a.kl_mode = p->kl_mode;
}

int run_rows(sf_tm_t h, sftm::RowArgs& a, int mode, cudaStream_t s, const char* where) {
  a.partials = h->partials;
  a.ticket = h->ticket;
  a.max_partial_blocks = h->max_partial_blocks;
  sftm::LaunchInfo info;
  const int e = sftm::launch_rows(a, mode, s, &h->err, &info);
  h->launches += static_cast<uint64_t>(info.launches);
  if (info.launches) h->last = info;
  return check_cuda(h, e, where);
}

}  // namespace

namespace {
// Grow-once host-call scratch (per-token and per-sample device buffers).
int ensure_tscratch(sf_tm_t h, int64_t T) {
  if (T <= h->tcap) return SF_TM_OK;
  int rc = 0;
  if ((rc = grow(h, &h->d_targets, T, "scratch")) || (rc = grow(h, &h->d_old, T, "scratch")) ||
      (rc = grow(h, &h->d_ref, T, "scratch")) || (rc = grow(h, &h->d_mask, T, "scratch")) ||
      (rc = grow(h, &h->d_advtok, T, "scratch")) || (rc = grow(h, &h->d_wtok, T, "scratch")))
    return rc;
  h->tcap = T;
  return SF_TM_OK;
}
int ensure_bscratch(sf_tm_t h, int64_t B) {
  if (B <= h->bcap) return SF_TM_OK;
  int rc = 0;
  if ((rc = grow(h, &h->d_lens, B, "scratch")) || (rc = grow(h, &h->d_plens, B, "scratch")) ||
      (rc = grow(h, &h->d_rewards, B, "scratch")) || (rc = grow(h, &h->d_gids, B, "scratch")) ||
      (rc = grow(h, &h->d_cu, B + 1, "scratch")) || (rc = grow(h, &h->d_adv, B, "scratch")))
    return rc;
  h->bcap = B;
  return SF_TM_OK;
}

// Stage buffers for sf_tm_pg_step_host (grow-once; the first use creates the
// side stream, the events and the per-stage counters).
int ensure_stage(sf_tm_t h, sf_tm_handle::HostStage& g, int64_t T, int64_t B) {
  if (!h->side) {
    cudaError_t e = cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->h2d_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(h, e, "pg_step_host side stream");
  }
  if (!g.ready_ev) {
    cudaError_t e = cudaEventCreateWithFlags(&g.ready_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g.free_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&g.ticket, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMalloc(&g.tot, sizeof(int64_t) * 2);
    if (e == cudaSuccess) e = cudaMalloc(&g.total, sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemset(g.ticket, 0, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();  // the zeroed ticket before any side-stream use
    if (e != cudaSuccess) return cuda_fail(h, e, "pg_step_host stage");
  }
  int rc = 0;
  if (T > g.tcap) {
    // a grow frees buffers a pending launch may still read
    if (cudaError_t e = cudaEventSynchronize(g.free_ev)) return cuda_fail(h, e, "pg_step_host stage");
    if ((rc = grow(h, &g.targets, T, "scratch")) || (rc = grow(h, &g.old, T, "scratch")) ||
        (rc = grow(h, &g.ref, T, "scratch")) || (rc = grow(h, &g.mask, T, "scratch")) ||
        (rc = grow(h, &g.advtok, T, "scratch")) || (rc = grow(h, &g.wtok, T, "scratch")))
      return rc;
    g.tcap = T;
  }
  if (B > g.bcap) {
    if (cudaError_t e = cudaEventSynchronize(g.free_ev)) return cuda_fail(h, e, "pg_step_host stage");
    const int64_t cap = B < 1024 ? 1024 : B;
    if ((rc = grow(h, &g.lens, cap, "scratch")) || (rc = grow(h, &g.plens, cap, "scratch")) ||
        (rc = grow(h, &g.rewards, cap, "scratch")) || (rc = grow(h, &g.gids, cap, "scratch")) ||
        (rc = grow(h, &g.cu, cap + 1, "scratch")) || (rc = grow(h, &g.adv, cap, "scratch")) ||
        (rc = grow(h, &g.cnt, cap, "scratch")))
      return rc;
    g.bcap = cap;
  }
  return SF_TM_OK;
}

void free_stages(sf_tm_t h) {
  if (h->side) cudaStreamSynchronize(h->side);
  for (auto& g : h->st) {
    void* ptrs[] = {g.targets, g.old, g.ref, g.mask, g.advtok, g.wtok, g.lens, g.plens, g.rewards,
                    g.gids, g.cu, g.adv, g.cnt, g.total, g.ticket, g.tot};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    if (g.ready_ev) cudaEventDestroy(g.ready_ev);
    if (g.free_ev) cudaEventDestroy(g.free_ev);
  }
  if (h->h2d_ev) cudaEventDestroy(h->h2d_ev);
  if (h->side) cudaStreamDestroy(h->side);
}

// This rank's mailbox, the host-mapped failure word and the abort flag.
int alloc_mailbox(sf_tm_t h, int32_t P, int32_t rank) {
  cudaError_t e = cudaMalloc(&h->xp_local, sftm::kXpMailboxBytes);
  if (e == cudaSuccess) e = cudaMemset(h->xp_local, 0, sftm::kXpMailboxBytes);
  if (e == cudaSuccess) e = cudaMalloc(&h->xp_abort, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(h->xp_abort, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&h->xp_err_h), sizeof(int), cudaHostAllocMapped);
  if (e == cudaSuccess) {
    *h->xp_err_h = 0;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->xp_err_d), h->xp_err_h, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return check_cuda(h, e, "peer mailbox");
  h->xp_P = P;
  h->xp_rank = rank;
  h->xp_mail[rank] = h->xp_local;
  return SF_TM_OK;
}

// Everything sf_tm_vp_fused_loss_fwd_bwd checks before it consumes a launch
// epoch: a call that fails here has no effect on the peers' call sequence.
int vp_fused_check(sf_tm_t h, const void* logits_shard, int32_t dtype, int64_t T, int64_t Vp, int64_t ld,
                   const void* dlogits, int64_t ld_d) {
  if (!h->xp_ready) return fail(h, SF_TM_CONFIG_ERROR, "peer mailboxes not open (sf_tm_vp_mailbox_open)");
  if (*h->xp_err_h)
    return fail(h, SF_TM_INTERNAL,
                "an earlier fused vocab-parallel launch timed out waiting for a peer (its outputs are invalid); "
                "the peer exchange of this handle is disabled, use sf_tm_vp_loss_fwd_bwd");
  if (bad_dtype(dtype)) return fail(h, SF_TM_CONFIG_ERROR, "dtype must be SF_TM_F32 or SF_TM_BF16");
  if (T < 0 || Vp <= 0 || ld < Vp || ld_d < Vp) return fail(h, SF_TM_CONFIG_ERROR, "bad shard shape or stride");
  const int64_t es = dtype == SF_TM_BF16 ? 2 : 4;
  const uintptr_t lb = reinterpret_cast<uintptr_t>(logits_shard), db = reinterpret_cast<uintptr_t>(dlogits);
  // Rows off 16-B boundaries (an odd shard width or stride) run in sector
  // coordinates, which needs the dlogits rows at the same 16-B phase as the
  // logits rows (same base phase, stride difference a multiple of 16 B).
  if (lb % es || db % es || (lb % 16) != (db % 16) || ((ld_d - ld) * es) % 16)
    return fail(h, SF_TM_CONFIG_ERROR,
                "fused vocab-parallel needs element-aligned shard rows with dlogits at the logits' 16-B phase");
  const bool ua = (lb % 16) || (ld * es) % 16 || (Vp * es) % 16;
  if (!sftm::loss_xp_eligible(dtype, Vp, ua))
    return fail(h, SF_TM_CONFIG_ERROR, "shard row too wide for the fused vocab-parallel kernel");
  return SF_TM_OK;
}

}  // namespace

extern "C" {

void sf_tm_default_loss_params(sf_tm_loss_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->clip_eps_low = 0.2f;
  p->clip_eps_high = 0.28f;
  p->dual_clip_c = 0.f;
  p->kl_beta = 0.f;
  p->entropy_coef = 0.f;
  p->inv_temperature = 1.f;
  p->norm_mode = SF_TM_NORM_TOKEN_MEAN;
  p->inv_norm = 0.f;
  p->masked_rows = SF_TM_MASKED_ZERO_FILL;
}

int sf_tm_abi_version(void) { return SF_TM_ABI_VERSION; }

int sf_tm_create(int device, sf_tm_t* out) {
  if (!out) return SF_TM_CONFIG_ERROR;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) return SF_TM_INTERNAL;
  if (device < 0 || device >= n) return SF_TM_CONFIG_ERROR;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (major != 10 || minor != 0) return SF_TM_CONFIG_ERROR;  // built for sm_100a only
  sf_tm_t h = new (std::nothrow) sf_tm_handle();
  if (!h) return SF_TM_INTERNAL;
  h->device = device;
  if (use_device(h) != SF_TM_OK) {
    delete h;
    return SF_TM_INTERNAL;
  }
  h->max_partial_blocks = kMaxPartialBlocks;
  if (cudaMalloc(&h->partials, sizeof(double) * 8 * kMaxPartialBlocks) != cudaSuccess ||
      cudaMalloc(&h->ticket, sizeof(unsigned) * 2) != cudaSuccess ||
      cudaMalloc(&h->tot, sizeof(int64_t) * 2) != cudaSuccess ||
      cudaMalloc(&h->d_total, sizeof(int32_t)) != cudaSuccess ||
      cudaMalloc(&h->d_metrics, sizeof(float) * SF_TM_NUM_METRICS) != cudaSuccess ||
      cudaMemset(h->ticket, 0, sizeof(unsigned) * 2) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    sf_tm_destroy(h);
    return SF_TM_INTERNAL;
  }
  h->ticket2 = h->ticket + 1;
  *out = h;
  return SF_TM_OK;
}

int sf_tm_destroy(sf_tm_t h) {
  if (!h) return SF_TM_OK;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != h->device) cudaSetDevice(h->device);
  void* ptrs[] = {h->partials, h->ticket,  h->cnt,     h->tot,    h->d_targets, h->d_old,
                  h->d_ref,    h->d_mask,  h->d_advtok, h->d_wtok, h->d_lens,    h->d_plens,
                  h->d_rewards, h->d_gids, h->d_cu,    h->d_adv,  h->d_total,   h->d_metrics};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  free_stages(h);
  if (!h->xp_local_group)
    for (int q = 0; q < h->xp_P; ++q)
      if (q != h->xp_rank && h->xp_mail[q]) cudaIpcCloseMemHandle(h->xp_mail[q]);
  if (h->xp_local) cudaFree(h->xp_local);
  if (h->xp_abort) cudaFree(h->xp_abort);
  if (h->xp_err_h) cudaFreeHost(h->xp_err_h);
  delete h;
  return SF_TM_OK;
}

const char* sf_tm_last_error(sf_tm_t h) { return h ? h->err.c_str() : "null handle"; }

uint64_t sf_tm_launch_count(sf_tm_t h) { return h ? h->launches : 0; }

int sf_tm_last_launch(sf_tm_t h, int32_t* kernel, int32_t* cluster, int32_t* grid) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (kernel) *kernel = h->last.kernel;
  if (cluster) *cluster = h->last.cluster;
  if (grid) *grid = h->last.grid;
  return SF_TM_OK;
}

int sf_tm_last_launch_streams(sf_tm_t h, int32_t* streams) {
  if (!h || !streams) return SF_TM_CONFIG_ERROR;
  *streams = h->last.streams;
  return SF_TM_OK;
}

int sf_tm_varlen_meta(sf_tm_t h, const int32_t* seq_lens, const int32_t* prompt_lens,
                      const int32_t* group_ids, int64_t B, int64_t T, int32_t* cu_seqlens,
                      int32_t* seq_id, uint8_t* mask, int32_t* tok_group, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (B < 0 || T < 0) return fail(h, SF_TM_CONFIG_ERROR, "B and T must be >= 0");
  if (!cu_seqlens || (B > 0 && !seq_lens))
    return fail(h, SF_TM_CONFIG_ERROR, "seq_lens and cu_seqlens are required");
  if (tok_group && !group_ids) return fail(h, SF_TM_CONFIG_ERROR, "tok_group needs group_ids");
  int n = 0;
  const int e = sftm::launch_varlen_meta(seq_lens, prompt_lens, group_ids, B, T, cu_seqlens,
                                         seq_id, mask, tok_group, h->d_total,
                                         static_cast<cudaStream_t>(stream), &n);
  h->launches += n;
  return check_cuda(h, e, "sf_tm_varlen_meta");
}

int sf_tm_grpo_advantage(sf_tm_t h, const float* rewards, const int32_t* group_ids, int64_t B,
                         float eps, int32_t std_mode, float* out_adv, int32_t* out_group_size,
                         void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (B < 0) return fail(h, SF_TM_CONFIG_ERROR, "B must be >= 0");
  if (std_mode < 0 || std_mode > 2) return fail(h, SF_TM_CONFIG_ERROR, "std_mode must be SF_TM_STD_*");
  if (!(eps >= 0.f && std::isfinite(eps))) return fail(h, SF_TM_CONFIG_ERROR, "eps must be >= 0");
  if (B == 0) return SF_TM_OK;
  if (!rewards || !group_ids || !out_adv)
    return fail(h, SF_TM_CONFIG_ERROR, "rewards, group_ids and out_adv are required");
  int n = 0;
  const int e = sftm::launch_grpo_advantage(rewards, group_ids, B, eps, std_mode, out_adv,
                                            out_group_size, static_cast<cudaStream_t>(stream), &n);
  h->launches += n;
  return check_cuda(h, e, "sf_tm_grpo_advantage");
}

int sf_tm_logprob_fwd(sf_tm_t h, const void* logits, int32_t dtype, int64_t T, int64_t V,
                      int64_t ld, const int32_t* targets, float inv_temperature, float* out_logp,
                      float* out_entropy, float* out_lse, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (int rc = check_rows(h, logits, dtype, T, V, ld, targets)) return rc;
  if (!(inv_temperature > 0.f && std::isfinite(inv_temperature)))
    return fail(h, SF_TM_CONFIG_ERROR, "inv_temperature must be > 0");
  if (T == 0) return SF_TM_OK;
  sftm::RowArgs a;
  a.logits = logits;
  a.dtype = dtype;
  a.T = T;
  a.V = V;
  a.ld = ld;
  a.targets = targets;
  a.inv_tau = inv_temperature;
  a.out_logp = out_logp;
  a.out_entropy = out_entropy;
  a.out_lse = out_lse;
  return run_rows(h, a, sftm::kModeFwd, static_cast<cudaStream_t>(stream), "sf_tm_logprob_fwd");
}

int sf_tm_token_weights(sf_tm_t h, const int32_t* cu_seqlens, int64_t B, const float* adv_seq,
                        const uint8_t* mask, int64_t T, int32_t norm_mode, float inv_norm,
                        float* out_adv_tok, float* out_w_tok, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (B < 0 || T < 0) return fail(h, SF_TM_CONFIG_ERROR, "B and T must be >= 0");
  if (norm_mode < 0 || norm_mode > 2) return fail(h, SF_TM_CONFIG_ERROR, "norm_mode must be SF_TM_NORM_*");
  if (B == 0 || T == 0) return SF_TM_OK;
  if (!cu_seqlens || !out_adv_tok || !out_w_tok)
    return fail(h, SF_TM_CONFIG_ERROR, "cu_seqlens, out_adv_tok and out_w_tok are required");
  if (int rc = ensure_cnt(h, B)) return rc;
  int n = 0;
  const int e = sftm::launch_token_weights(cu_seqlens, B, adv_seq, mask, T, norm_mode, inv_norm,
                                           out_adv_tok, out_w_tok, h->cnt, h->ticket2, h->tot,
                                           static_cast<cudaStream_t>(stream), &n);
  h->launches += n;
  return check_cuda(h, e, "sf_tm_token_weights");
}

int sf_tm_pg_loss_fwd_bwd(sf_tm_t h, const void* logits, int32_t dtype, int64_t T, int64_t V,
                          int64_t ld, const int32_t* targets, const float* old_logp,
                          const float* ref_logp, const float* adv_tok, const float* w_tok,
                          const sf_tm_loss_params* params, void* dlogits, int64_t ld_d,
                          float* out_metrics, float* out_logp, float* out_entropy, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (int rc = check_rows(h, logits, dtype, T, V, ld, targets)) return rc;
  if (int rc = check_loss_params(h, params)) return rc;
  if (!out_metrics) return fail(h, SF_TM_CONFIG_ERROR, "out_metrics is required");
  if (ld_d < V) return fail(h, SF_TM_CONFIG_ERROR, "ld_d must be >= V");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (T == 0) {
    return check_cuda(h, cudaMemsetAsync(out_metrics, 0, sizeof(float) * SF_TM_NUM_METRICS, s),
                      "sf_tm_pg_loss_fwd_bwd");
  }
  if (!old_logp || !ref_logp || !adv_tok || !w_tok || !dlogits)
    return fail(h, SF_TM_CONFIG_ERROR,
                "old_logp, ref_logp, adv_tok, w_tok and dlogits are required");
  if (dlogits == logits && ld_d != ld)
    return fail(h, SF_TM_CONFIG_ERROR, "in-place dlogits needs ld_d == ld");
  sftm::RowArgs a;
  a.logits = logits;
  a.dtype = dtype;
  a.T = T;
  a.V = V;
  a.ld = ld;
  a.targets = targets;
  a.old_logp = old_logp;
  a.ref_logp = ref_logp;
  a.adv_tok = adv_tok;
  a.w_tok = w_tok;
  fill_loss(a, params);
  a.dlogits = dlogits;
  a.ld_d = ld_d;
  a.out_metrics = out_metrics;
  a.out_logp = out_logp;
  a.out_entropy = out_entropy;
  return run_rows(h, a, sftm::kModeFwdBwd, s, "sf_tm_pg_loss_fwd_bwd");
}

int sf_tm_pg_step_host(sf_tm_t h, const void* logits, int32_t dtype, int64_t T, int64_t V,
                       int64_t ld, const int32_t* h_targets, const float* h_old_logp,
                       const float* h_ref_logp, const uint8_t* h_mask, const int32_t* h_seq_lens,
                       const int32_t* h_prompt_lens, const float* h_rewards,
                       const int32_t* h_group_ids, int64_t B, float adv_eps, int32_t std_mode,
                       const sf_tm_loss_params* params, void* dlogits, int64_t ld_d,
                       float* h_metrics, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (int rc = check_rows(h, logits, dtype, T, V, ld, h_targets)) return rc;
  if (int rc = check_loss_params(h, params)) return rc;
  if (B <= 0) return fail(h, SF_TM_CONFIG_ERROR, "B must be > 0");
  if (!h_seq_lens || !h_rewards || !h_metrics || !h_old_logp || !h_ref_logp || !dlogits)
    return fail(h, SF_TM_CONFIG_ERROR, "missing required host buffer");
  if (ld_d < V) return fail(h, SF_TM_CONFIG_ERROR, "ld_d must be >= V");
  if (dlogits == logits && ld_d != ld)
    return fail(h, SF_TM_CONFIG_ERROR, "in-place dlogits needs ld_d == ld");
  if (adv_eps >= 0.f && !h_group_ids)
    return fail(h, SF_TM_CONFIG_ERROR, "group ids are required to compute advantages");
  if (std_mode < 0 || std_mode > 2) return fail(h, SF_TM_CONFIG_ERROR, "std_mode must be SF_TM_STD_*");
  int64_t tsum = 0;
  for (int64_t b = 0; b < B; ++b) {
    if (h_seq_lens[b] < 0) return fail(h, SF_TM_CONFIG_ERROR, "negative sequence length");
    tsum += h_seq_lens[b];
  }
  if (tsum != T) return fail(h, SF_TM_CONFIG_ERROR, "sum(seq_lens) != T");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Pipelined prologue: the H2D of this micro-batch's bus fields and its
  // varlen / GRPO / token-weight kernels run on the side stream, into the stage
  // the loss two calls back has released, so they overlap the fused loss of
  // the previous call on `s`; `s` then waits only for this stage to be ready.
  sf_tm_handle::HostStage& g = h->st[h->st_next];
  if (int rc = ensure_stage(h, g, T, B)) return rc;
  cudaStream_t q = h->side;
  cudaError_t e = cudaStreamWaitEvent(q, g.free_ev, 0);
  if (e != cudaSuccess) return cuda_fail(h, e, "sf_tm_pg_step_host");
  auto h2d = [&](void* d, const void* src, size_t bytes) {
    return cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, q);
  };
  if ((e = h2d(g.targets, h_targets, sizeof(int32_t) * T)) ||
      (e = h2d(g.old, h_old_logp, sizeof(float) * T)) ||
      (e = h2d(g.ref, h_ref_logp, sizeof(float) * T)) ||
      (e = h2d(g.lens, h_seq_lens, sizeof(int32_t) * B)) ||
      (e = h2d(g.rewards, h_rewards, sizeof(float) * B)))
    return cuda_fail(h, e, "sf_tm_pg_step_host H2D");
  if (h_group_ids && (e = h2d(g.gids, h_group_ids, sizeof(int32_t) * B)))
    return cuda_fail(h, e, "sf_tm_pg_step_host H2D");
  if (h_prompt_lens && (e = h2d(g.plens, h_prompt_lens, sizeof(int32_t) * B)))
    return cuda_fail(h, e, "sf_tm_pg_step_host H2D");
  if (h_mask && (e = h2d(g.mask, h_mask, sizeof(uint8_t) * T)))
    return cuda_fail(h, e, "sf_tm_pg_step_host H2D");
  if ((e = cudaEventRecord(h->h2d_ev, q))) return cuda_fail(h, e, "sf_tm_pg_step_host H2D");

  int n = 0;
  int rc = sftm::launch_varlen_meta(g.lens, h_prompt_lens ? g.plens : nullptr, nullptr, B, T, g.cu,
                                    nullptr, (!h_mask && h_prompt_lens) ? g.mask : nullptr, nullptr,
                                    g.total, q, &n);
  h->launches += n;
  if (rc) return cuda_fail(h, rc, "sf_tm_pg_step_host varlen");
  const uint8_t* mask = (h_mask || h_prompt_lens) ? g.mask : nullptr;
  const float* adv = g.rewards;
  if (adv_eps >= 0.f) {
    n = 0;
    rc = sftm::launch_grpo_advantage(g.rewards, g.gids, B, adv_eps, std_mode, g.adv, nullptr, q, &n);
    h->launches += n;
    if (rc) return cuda_fail(h, rc, "sf_tm_pg_step_host advantage");
    adv = g.adv;
  }
  n = 0;
  rc = sftm::launch_token_weights(g.cu, B, adv, mask, T, params->norm_mode, params->inv_norm, g.advtok,
                                  g.wtok, g.cnt, g.ticket, g.tot, q, &n);
  h->launches += n;
  if (rc) return cuda_fail(h, rc, "sf_tm_pg_step_host token weights");
  if ((e = cudaEventRecord(g.ready_ev, q)) || (e = cudaStreamWaitEvent(s, g.ready_ev, 0)))
    return cuda_fail(h, e, "sf_tm_pg_step_host");
  sftm::RowArgs a;
  a.logits = logits;
  a.dtype = dtype;
  a.T = T;
  a.V = V;
  a.ld = ld;
  a.targets = g.targets;
  a.old_logp = g.old;
  a.ref_logp = g.ref;
  a.adv_tok = g.advtok;
  a.w_tok = g.wtok;
  fill_loss(a, params);
  a.dlogits = dlogits;
  a.ld_d = ld_d;
  a.out_metrics = h->d_metrics;
  if (int r2 = run_rows(h, a, sftm::kModeFwdBwd, s, "sf_tm_pg_step_host loss")) return r2;
  if ((e = cudaEventRecord(g.free_ev, s)))
    return cuda_fail(h, e, "sf_tm_pg_step_host");
  h->st_next ^= 1;
  e = cudaMemcpyAsync(h_metrics, h->d_metrics, sizeof(float) * SF_TM_NUM_METRICS,
                      cudaMemcpyDeviceToHost, s);
  return check_cuda(h, e, "sf_tm_pg_step_host D2H");
}

int sf_tm_wait_host_inputs(sf_tm_t h) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (!h->h2d_ev) return SF_TM_OK;  // no pg_step_host call yet
  if (int rc = use_device(h)) return rc;
  return check_cuda(h, cudaEventSynchronize(h->h2d_ev), "sf_tm_wait_host_inputs");
}

int sf_tm_sync(sf_tm_t h, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  return check_cuda(h, cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sf_tm_sync");
}

int sf_tm_logprob_fwd_host(sf_tm_t h, const void* logits, int32_t dtype, int64_t T, int64_t V, int64_t ld,
                           const int32_t* h_targets, float inv_temperature, float* h_logp, float* h_entropy,
                           void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (int rc = check_rows(h, logits, dtype, T, V, ld, h_targets)) return rc;
  if (!(inv_temperature > 0.f && std::isfinite(inv_temperature)))
    return fail(h, SF_TM_CONFIG_ERROR, "inv_temperature must be > 0");
  if (T == 0) return SF_TM_OK;
  if (!h_logp) return fail(h, SF_TM_CONFIG_ERROR, "h_logp is required");
  if (int rc = ensure_tscratch(h, T)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(h->d_targets, h_targets, sizeof(int32_t) * T, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "sf_tm_logprob_fwd_host H2D");
  sftm::RowArgs a;
  a.logits = logits;
  a.dtype = dtype;
  a.T = T;
  a.V = V;
  a.ld = ld;
  a.targets = h->d_targets;
  a.inv_tau = inv_temperature;
  a.out_logp = h->d_old;
  a.out_entropy = h_entropy ? h->d_ref : nullptr;
  if (int rc = run_rows(h, a, sftm::kModeFwd, s, "sf_tm_logprob_fwd_host")) return rc;
  e = cudaMemcpyAsync(h_logp, h->d_old, sizeof(float) * T, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && h_entropy)
    e = cudaMemcpyAsync(h_entropy, h->d_ref, sizeof(float) * T, cudaMemcpyDeviceToHost, s);
  return check_cuda(h, e, "sf_tm_logprob_fwd_host D2H");
}

int sf_tm_grpo_advantage_host(sf_tm_t h, const float* h_rewards, const int32_t* h_group_ids, int64_t B, float eps,
                              int32_t std_mode, float* h_adv, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (B < 0) return fail(h, SF_TM_CONFIG_ERROR, "B must be >= 0");
  if (std_mode < 0 || std_mode > 2) return fail(h, SF_TM_CONFIG_ERROR, "std_mode must be SF_TM_STD_*");
  if (!(eps >= 0.f && std::isfinite(eps))) return fail(h, SF_TM_CONFIG_ERROR, "eps must be >= 0");
  if (B == 0) return SF_TM_OK;
  if (!h_rewards || !h_group_ids || !h_adv)
    return fail(h, SF_TM_CONFIG_ERROR, "h_rewards, h_group_ids and h_adv are required");
  if (int rc = ensure_bscratch(h, B)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(h->d_rewards, h_rewards, sizeof(float) * B, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->d_gids, h_group_ids, sizeof(int32_t) * B, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(h, e, "sf_tm_grpo_advantage_host H2D");
  int n = 0;
  const int rc = sftm::launch_grpo_advantage(h->d_rewards, h->d_gids, B, eps, std_mode, h->d_adv, nullptr, s, &n);
  h->launches += n;
  if (rc) return cuda_fail(h, rc, "sf_tm_grpo_advantage_host");
  e = cudaMemcpyAsync(h_adv, h->d_adv, sizeof(float) * B, cudaMemcpyDeviceToHost, s);
  return check_cuda(h, e, "sf_tm_grpo_advantage_host D2H");
}

int sf_tm_r3_gate_fwd(sf_tm_t h, const void* router_logits, int32_t dtype, int64_t L, int64_t T,
                      int64_t E, int64_t k, const void* rec_idx, int32_t idx_dtype, int32_t renorm,
                      float* out_w, int32_t* out_idx, uint32_t* out_mismatch, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (bad_dtype(dtype)) return fail(h, SF_TM_CONFIG_ERROR, "dtype must be SF_TM_F32 or SF_TM_BF16");
  if (idx_dtype != SF_TM_IDX_I32 && idx_dtype != SF_TM_IDX_U8)
    return fail(h, SF_TM_CONFIG_ERROR, "idx_dtype must be SF_TM_IDX_*");
  if (L < 0 || T < 0) return fail(h, SF_TM_CONFIG_ERROR, "L and T must be >= 0");
  if (E < 1 || E > 512) return fail(h, SF_TM_CONFIG_ERROR, "E must be in [1, 512]");
  if (k < 1 || k > 32 || k > E) return fail(h, SF_TM_CONFIG_ERROR, "k must be in [1, min(32, E)]");
  if (idx_dtype == SF_TM_IDX_U8 && E > 256)
    return fail(h, SF_TM_CONFIG_ERROR, "u8 indices need E <= 256");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (out_mismatch) {
    cudaError_t e = cudaMemsetAsync(out_mismatch, 0, sizeof(uint32_t) * (L + 1), s);
    if (e != cudaSuccess) return cuda_fail(h, e, "sf_tm_r3_gate_fwd");
  }
  if (L * T == 0) return SF_TM_OK;
  if (!router_logits || !rec_idx || !out_w)
    return fail(h, SF_TM_CONFIG_ERROR, "router_logits, rec_idx and out_w are required");
  int n = 0;
  const int e = sftm::launch_r3_fwd(router_logits, dtype, L, T, E, k, rec_idx, idx_dtype, renorm,
                                    out_w, out_idx, out_mismatch, s, &n);
  h->launches += n;
  return check_cuda(h, e, "sf_tm_r3_gate_fwd");
}

int sf_tm_r3_gate_bwd(sf_tm_t h, const void* router_logits, int32_t dtype, int64_t L, int64_t T,
                      int64_t E, int64_t k, const void* rec_idx, int32_t idx_dtype, int32_t renorm,
                      const float* w, const float* dw, void* dlogits, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (bad_dtype(dtype)) return fail(h, SF_TM_CONFIG_ERROR, "dtype must be SF_TM_F32 or SF_TM_BF16");
  if (idx_dtype != SF_TM_IDX_I32 && idx_dtype != SF_TM_IDX_U8)
    return fail(h, SF_TM_CONFIG_ERROR, "idx_dtype must be SF_TM_IDX_*");
  if (L < 0 || T < 0) return fail(h, SF_TM_CONFIG_ERROR, "L and T must be >= 0");
  if (E < 1 || E > 512) return fail(h, SF_TM_CONFIG_ERROR, "E must be in [1, 512]");
  if (k < 1 || k > 32 || k > E) return fail(h, SF_TM_CONFIG_ERROR, "k must be in [1, min(32, E)]");
  if (L * T == 0) return SF_TM_OK;
  if (!rec_idx || !w || !dw || !dlogits || (!renorm && !router_logits))
    return fail(h, SF_TM_CONFIG_ERROR, "missing required pointer");
  int n = 0;
  const int e = sftm::launch_r3_bwd(router_logits, dtype, L, T, E, k, rec_idx, idx_dtype, renorm,
                                    w, dw, dlogits, static_cast<cudaStream_t>(stream), &n);
  h->launches += n;
  return check_cuda(h, e, "sf_tm_r3_gate_bwd");
}

int sf_tm_r3_record_layer_major(sf_tm_t h, const void* rec_token_major, int32_t idx_dtype, int64_t T, int64_t L,
                                int64_t k, void* rec_layer_major, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (idx_dtype != SF_TM_IDX_I32 && idx_dtype != SF_TM_IDX_U8)
    return fail(h, SF_TM_CONFIG_ERROR, "idx_dtype must be SF_TM_IDX_*");
  if (T < 0 || L < 0) return fail(h, SF_TM_CONFIG_ERROR, "T and L must be >= 0");
  if (k < 1 || k > 32) return fail(h, SF_TM_CONFIG_ERROR, "k must be in [1, 32]");
  if (T > 65535LL * 32 * 1024 || L > 65535LL * 32) return fail(h, SF_TM_CONFIG_ERROR, "T or L too large");
  if (T * L == 0) return SF_TM_OK;
  if (!rec_token_major || !rec_layer_major) return fail(h, SF_TM_CONFIG_ERROR, "record pointers are required");
  if (rec_token_major == rec_layer_major) return fail(h, SF_TM_CONFIG_ERROR, "the transpose is out of place");
  int n = 0;
  const int e = sftm::launch_rec_layer_major(rec_token_major, idx_dtype, T, L, k, rec_layer_major,
                                             static_cast<cudaStream_t>(stream), &n);
  h->launches += n;
  return check_cuda(h, e, "sf_tm_r3_record_layer_major");
}

int sf_tm_vp_partial_stats(sf_tm_t h, const void* logits_shard, int32_t dtype, int64_t T,
                           int64_t Vp, int64_t ld, int64_t vocab_start, const int32_t* targets,
                           float inv_temperature, float* out_stats, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (int rc = check_rows(h, logits_shard, dtype, T, Vp, ld, targets)) return rc;
  if (!(inv_temperature > 0.f && std::isfinite(inv_temperature)))
    return fail(h, SF_TM_CONFIG_ERROR, "inv_temperature must be > 0");
  if (vocab_start < 0) return fail(h, SF_TM_CONFIG_ERROR, "vocab_start must be >= 0");
  if (T == 0) return SF_TM_OK;
  if (!out_stats) return fail(h, SF_TM_CONFIG_ERROR, "out_stats is required");
  sftm::RowArgs a;
  a.logits = logits_shard;
  a.dtype = dtype;
  a.T = T;
  a.V = Vp;
  a.ld = ld;
  a.vocab_start = vocab_start;
  a.targets = targets;
  a.inv_tau = inv_temperature;
  a.out_stats = out_stats;
  return run_rows(h, a, sftm::kModeVpStats, static_cast<cudaStream_t>(stream),
                  "sf_tm_vp_partial_stats");
}

int sf_tm_vp_loss_fwd_bwd(sf_tm_t h, const void* logits_shard, int32_t dtype, int64_t T,
                          int64_t Vp, int64_t ld, int64_t vocab_start, const float* gathered_stats,
                          int32_t P, const int32_t* targets, const float* old_logp,
                          const float* ref_logp, const float* adv_tok, const float* w_tok,
                          const sf_tm_loss_params* params, void* dlogits, int64_t ld_d,
                          float* out_metrics, float* out_logp, float* out_entropy, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (int rc = check_rows(h, logits_shard, dtype, T, Vp, ld, targets)) return rc;
  if (int rc = check_loss_params(h, params)) return rc;
  if (P < 1) return fail(h, SF_TM_CONFIG_ERROR, "P must be >= 1");
  if (vocab_start < 0) return fail(h, SF_TM_CONFIG_ERROR, "vocab_start must be >= 0");
  if (!out_metrics) return fail(h, SF_TM_CONFIG_ERROR, "out_metrics is required");
  if (ld_d < Vp) return fail(h, SF_TM_CONFIG_ERROR, "ld_d must be >= Vp");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (T == 0) {
    return check_cuda(h, cudaMemsetAsync(out_metrics, 0, sizeof(float) * SF_TM_NUM_METRICS, s),
                      "sf_tm_vp_loss_fwd_bwd");
  }
  if (!gathered_stats || !old_logp || !ref_logp || !adv_tok || !w_tok || !dlogits)
    return fail(h, SF_TM_CONFIG_ERROR, "missing required pointer");
  sftm::RowArgs a;
  a.logits = logits_shard;
  a.dtype = dtype;
  a.T = T;
  a.V = Vp;
  a.ld = ld;
  a.vocab_start = vocab_start;
  a.targets = targets;
  a.gathered = gathered_stats;
  a.P = P;
  a.old_logp = old_logp;
  a.ref_logp = ref_logp;
  a.adv_tok = adv_tok;
  a.w_tok = w_tok;
  fill_loss(a, params);
  a.dlogits = dlogits;
  a.ld_d = ld_d;
  a.out_metrics = out_metrics;
  a.out_logp = out_logp;
  a.out_entropy = out_entropy;
  return run_rows(h, a, sftm::kModeVpBwd, s, "sf_tm_vp_loss_fwd_bwd");
}

int sf_tm_vp_mailbox_create(sf_tm_t h, int32_t P, int32_t rank, void* ipc_handle_out) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (P < 1 || P > sftm::kXpMaxP) return fail(h, SF_TM_CONFIG_ERROR, "P must be in [1, 8]");
  if (rank < 0 || rank >= P) return fail(h, SF_TM_CONFIG_ERROR, "rank must be in [0, P)");
  if (!ipc_handle_out) return fail(h, SF_TM_CONFIG_ERROR, "ipc_handle_out is required");
  if (h->xp_local) return fail(h, SF_TM_CONFIG_ERROR, "mailbox already created on this handle");
  if (int rc = alloc_mailbox(h, P, rank)) return rc;
  cudaIpcMemHandle_t ih;
  const cudaError_t e = cudaIpcGetMemHandle(&ih, h->xp_local);
  if (e != cudaSuccess) return check_cuda(h, e, "sf_tm_vp_mailbox_create");
  std::memcpy(ipc_handle_out, &ih, SF_TM_IPC_HANDLE_BYTES);
  return SF_TM_OK;
}

int sf_tm_vp_mailbox_open(sf_tm_t h, const void* ipc_handles) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (!h->xp_local) return fail(h, SF_TM_CONFIG_ERROR, "sf_tm_vp_mailbox_create first");
  if (h->xp_ready) return fail(h, SF_TM_CONFIG_ERROR, "mailboxes already open (or wired as a local group)");
  if (!ipc_handles) return fail(h, SF_TM_CONFIG_ERROR, "ipc_handles is required");
  const uint8_t* hb = static_cast<const uint8_t*>(ipc_handles);
  for (int q = 0; q < h->xp_P; ++q) {
    if (q == h->xp_rank) continue;
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, hb + static_cast<size_t>(q) * SF_TM_IPC_HANDLE_BYTES, SF_TM_IPC_HANDLE_BYTES);
    const cudaError_t e = cudaIpcOpenMemHandle(&h->xp_mail[q], ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      h->xp_mail[q] = nullptr;
      return check_cuda(h, e, "sf_tm_vp_mailbox_open (cudaIpcOpenMemHandle)");
    }
  }
  if (const int e = sftm::prepare_loss_xp()) return check_cuda(h, static_cast<cudaError_t>(e), "sf_tm_vp_mailbox_open");
  h->xp_ready = true;
  return SF_TM_OK;
}

int sf_tm_vp_fused_loss_fwd_bwd(sf_tm_t h, const void* logits_shard, int32_t dtype, int64_t T, int64_t Vp,
                                int64_t ld, int64_t vocab_start, const int32_t* targets, const float* old_logp,
                                const float* ref_logp, const float* adv_tok, const float* w_tok,
                                const sf_tm_loss_params* params, void* dlogits, int64_t ld_d, float* out_metrics,
                                float* out_logp, float* out_entropy, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (int rc = vp_fused_check(h, logits_shard, dtype, T, Vp, ld, dlogits, ld_d)) return rc;
  if (int rc = check_rows(h, logits_shard, dtype, T, Vp, ld, targets)) return rc;
  if (int rc = check_loss_params(h, params)) return rc;
  if (vocab_start < 0) return fail(h, SF_TM_CONFIG_ERROR, "vocab_start must be >= 0");
  if (!out_metrics) return fail(h, SF_TM_CONFIG_ERROR, "out_metrics is required");
  if (T > 0 && (!old_logp || !ref_logp || !adv_tok || !w_tok || !dlogits))
    return fail(h, SF_TM_CONFIG_ERROR, "missing required pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Every argument check is above this line: a rank's launch epoch advances
  // only for a call that launches (or, for T == 0, that every rank makes with
  // the same T), so the peers' epochs stay in step.
  ++h->xp_epoch;
  if (T == 0) {
    return check_cuda(h, cudaMemsetAsync(out_metrics, 0, sizeof(float) * SF_TM_NUM_METRICS, s),
                      "sf_tm_vp_fused_loss_fwd_bwd");
  }
  sftm::RowArgs a;
  a.logits = logits_shard;
  a.dtype = dtype;
  a.T = T;
  a.V = Vp;
  a.ld = ld;
  a.vocab_start = vocab_start;
  a.targets = targets;
  a.old_logp = old_logp;
  a.ref_logp = ref_logp;
  a.adv_tok = adv_tok;
  a.w_tok = w_tok;
  fill_loss(a, params);
  a.dlogits = dlogits;
  a.ld_d = ld_d;
  a.out_metrics = out_metrics;
  a.out_logp = out_logp;
  a.out_entropy = out_entropy;
  for (int q = 0; q < h->xp_P; ++q) a.xp_mail[q] = h->xp_mail[q];
  a.xp_P = h->xp_P;
  a.xp_rank = h->xp_rank;
  a.xp_epoch = h->xp_epoch;
  a.xp_err = h->xp_err_d;
  a.xp_abort = h->xp_abort;
  a.xp_grid = h->xp_grid;
  static const unsigned long long timeout_ns = [] {
    const char* v = getenv("SF_TM_XP_TIMEOUT_S");
    const double sec = v ? atof(v) : 300.0;
    return static_cast<unsigned long long>((sec > 0 ? sec : 300.0) * 1e9);
  }();
  a.xp_timeout_ns = timeout_ns;
  a.partials = h->partials;
  a.ticket = h->ticket;
  a.max_partial_blocks = h->max_partial_blocks;
  sftm::LaunchInfo info;
  const int e = sftm::launch_loss_xp(a, s, &info);
  if (e == -2) return fail(h, SF_TM_INTERNAL, "fused vocab-parallel eligibility changed after the check");
  h->launches += static_cast<uint64_t>(info.launches);
  if (info.launches) h->last = info;
  return check_cuda(h, e, "sf_tm_vp_fused_loss_fwd_bwd");
}

int sf_tm_vp_fused_check(sf_tm_t h, const void* logits_shard, int32_t dtype, int64_t T, int64_t Vp, int64_t ld,
                         const void* dlogits, int64_t ld_d) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  return vp_fused_check(h, logits_shard, dtype, T, Vp, ld, dlogits, ld_d);
}

int sf_tm_debug_vp_local_group(sf_tm_t* handles, int32_t P, int32_t grid_per_rank) {
  if (!handles || P < 1 || P > sftm::kXpMaxP || grid_per_rank < 0) return SF_TM_CONFIG_ERROR;
  for (int r = 0; r < P; ++r) {
    sf_tm_t h = handles[r];
    if (!h || h->device != handles[0]->device) return SF_TM_CONFIG_ERROR;
    if (h->xp_local) return fail(h, SF_TM_CONFIG_ERROR, "mailbox already created on this handle");
  }
  for (int r = 0; r < P; ++r) {
    if (int rc = use_device(handles[r])) return rc;
    if (int rc = alloc_mailbox(handles[r], P, r)) return rc;
  }
  if (const int e = sftm::prepare_loss_xp())
    return check_cuda(handles[0], static_cast<cudaError_t>(e), "sf_tm_debug_vp_local_group");
  for (int r = 0; r < P; ++r) {
    sf_tm_t h = handles[r];
    for (int q = 0; q < P; ++q) h->xp_mail[q] = handles[q]->xp_local;
    h->xp_grid = grid_per_rank;
    h->xp_local_group = true;
    h->xp_ready = true;
  }
  return SF_TM_OK;
}

int sf_tm_synth_logits(sf_tm_t h, void* logits, int32_t dtype, int64_t T, int64_t V, int64_t ld,
                       uint64_t seed, float sigma, const int32_t* peak_id, float peak_lo,
                       float peak_hi, float outlier_frac, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (bad_dtype(dtype)) return fail(h, SF_TM_CONFIG_ERROR, "dtype must be SF_TM_F32 or SF_TM_BF16");
  if (T < 0 || V <= 0 || ld < V) return fail(h, SF_TM_CONFIG_ERROR, "bad shape");
  if (!(outlier_frac >= 0.f && outlier_frac <= 1.f))
    return fail(h, SF_TM_CONFIG_ERROR, "outlier_frac must be in [0, 1]");
  if (T == 0) return SF_TM_OK;
  if (!logits) return fail(h, SF_TM_CONFIG_ERROR, "logits is NULL");
  int n = 0;
  const int e = sftm::launch_synth_logits(logits, dtype, T, V, ld, seed, sigma, peak_id, peak_lo,
                                          peak_hi, outlier_frac, static_cast<cudaStream_t>(stream),
                                          &n);
  h->launches += n;
  return check_cuda(h, e, "sf_tm_synth_logits");
}

int sf_tm_host_alloc(size_t bytes, void** out) {
  if (!out || bytes == 0) return SF_TM_CONFIG_ERROR;
  *out = nullptr;
  return cudaMallocHost(out, bytes) == cudaSuccess ? SF_TM_OK : SF_TM_INTERNAL;
}

int sf_tm_host_free(void* p) {
  if (!p) return SF_TM_OK;
  return cudaFreeHost(p) == cudaSuccess ? SF_TM_OK : SF_TM_INTERNAL;
}

int sf_tm_h2d(sf_tm_t h, void* dst, const void* src, size_t bytes, void* stream) {
  if (!h) return SF_TM_CONFIG_ERROR;
  if (int rc = use_device(h)) return rc;
  if (bytes == 0) return SF_TM_OK;
  if (!dst || !src) return fail(h, SF_TM_CONFIG_ERROR, "sf_tm_h2d: NULL pointer");
  return check_cuda(h, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)),
                    "sf_tm_h2d");
}

int sf_tm_debug_force_generic(int on) {
  sftm::set_force_generic(on != 0);
  return SF_TM_OK;
}

int sf_tm_debug_wait_counters(void* dev_counters) {
  sftm::set_debug_counters(static_cast<unsigned long long*>(dev_counters));
  return SF_TM_OK;
}

}  // extern "C"
