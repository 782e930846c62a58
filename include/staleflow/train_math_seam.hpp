// SPDX-License-Identifier: Apache-2.0
//
// C++ trainer-seam adapter over the train-math C-ABI (staleflow/train_math.h).
//
// It turns one trainer MicroBatch, as delivered by the reference's bus
// (proj/include/staleflow/types.hpp:48-59, StreamLoader::next_micro_batch,
// stream_loader.cpp:77-91), into one fused loss fwd+bwd on the device-resident
// LM-head logits. This is the drop-in for the latency stub at
// proj/src/sim_runtime.cpp:441 / proj/src/wall_runtime.cpp:197.
//
// Header-only and templated on the MicroBatch type, so it compiles against the
// reference's own staleflow::MicroBatch without changing proj/include. Required
// members: field_set (sorted std::vector<std::string>), sample_ids, and
// payloads[i][j] (bytes of field_set[j] for sample i).
//
// Field codecs (little-endian, SURVEY.md §8b "Payload / ownership"):
//   response   int32[L_i]    token ids; logits row j scores response[j]
//   logp       float32[L_i]  behaviour-policy log-probs (ActorFwd)
//   ref_logp   float32[L_i]  reference-model log-probs (RefLogP)
//   advantage  float32       per-sample GRPO advantage (Advantages stage)
//   reward     float32       per-sample reward (used when there is no advantage
//                            field: GRPO is then computed here over `group`)
//   loss_mask  uint8[L_i]    optional; default all ones
//   group      int32         optional group id; default (sample_id-1)/group_size
//   routed_experts uint8[L_i * layers * k]  R3 record, token-major (token, layer, slot);
//                            decoded by pack_routed_experts into the gate's
//                            layer-major [layers, T, k] operand
// Staleness tags pass through from MicroBatch.producer_versions:
// staleness = v_trainer - v_producer per sample, as StalenessGate::staleness_of
// (proj/src/staleness.cpp:169-173) defines it for the batch minimum.
#pragma once

#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "staleflow/train_math.h"

namespace staleflow {
namespace train_math {

// Host arrays of one packed micro-batch (samples concatenated in bus order).
struct PackedBatch {
  int64_t T = 0, B = 0;
  std::vector<int32_t> targets;
  std::vector<float> logp, ref_logp;
  std::vector<uint8_t> mask;
  bool has_mask = false;
  std::vector<int32_t> seq_lens, group_ids;
  std::vector<float> per_sample;  // advantages, or rewards when !has_advantage
  bool has_advantage = false;
  std::vector<int64_t> producer_versions;  // per sample (MicroBatch.producer_versions)
};

// Per-sample staleness histogram {v_trainer - v_producer: count} and the batch
// staleness v_trainer - min(v_producer) (StalenessGate::staleness_of).
inline std::map<int64_t, uint64_t> staleness_histogram(const PackedBatch& p, int64_t v_trainer,
                                                       int64_t* batch_staleness = nullptr) {
  std::map<int64_t, uint64_t> h;
  int64_t vmin = v_trainer;
  for (int64_t v : p.producer_versions) {
    ++h[v_trainer - v];
    if (v < vmin) vmin = v;
  }
  if (batch_staleness) *batch_staleness = v_trainer - vmin;
  return h;
}

// GRPO is only correct on complete groups: every group id of the
// batch must occur exactly group_size times. SF_TM_OK or SF_TM_CONFIG_ERROR.
inline int check_complete_groups(const PackedBatch& p, int group_size, std::string* err) {
  if (group_size <= 0) return SF_TM_OK;
  std::map<int32_t, int> n;
  for (int32_t g : p.group_ids) ++n[g];
  for (const auto& kv : n)
    if (kv.second != group_size) {
      if (err) *err = "group " + std::to_string(kv.first) + " has " + std::to_string(kv.second) + " of " +
                      std::to_string(group_size) + " samples in this micro-batch";
      return SF_TM_CONFIG_ERROR;
    }
  return SF_TM_OK;
}

namespace detail {
inline int find_field(const std::vector<std::string>& fs, const char* name) {
  for (size_t j = 0; j < fs.size(); ++j)
    if (fs[j] == name) return static_cast<int>(j);
  return -1;
}
template <class Bytes, class T>
bool append(const Bytes& b, std::vector<T>& out, size_t n) {
  if (b.size() != n * sizeof(T)) return false;
  const size_t old = out.size();
  out.resize(old + n);
  if (n) std::memcpy(out.data() + old, b.data(), b.size());
  return true;
}
}  // namespace detail

// Decode a trainer MicroBatch into PackedBatch. Returns SF_TM_OK or
// SF_TM_CONFIG_ERROR with *err (missing field, ragged payload sizes).
template <class MicroBatchT>
int pack_trainer_batch(const MicroBatchT& b, int group_size, PackedBatch& out, std::string* err) {
  using detail::find_field;
  const auto& fs = b.field_set;
  const int jr = find_field(fs, "response"), jl = find_field(fs, "logp"), jf = find_field(fs, "ref_logp");
  const int ja = find_field(fs, "advantage"), jw = find_field(fs, "reward"), jm = find_field(fs, "loss_mask");
  const int jg = find_field(fs, "group");
  if (jr < 0 || jl < 0 || jf < 0 || (ja < 0 && jw < 0)) {
    if (err) *err = "trainer field set needs response, logp, ref_logp and advantage or reward";
    return SF_TM_CONFIG_ERROR;
  }
  if (jg < 0 && ja < 0 && group_size <= 0) {
    if (err) *err = "group ids: no 'group' field and no group_size";
    return SF_TM_CONFIG_ERROR;
  }
  out = PackedBatch{};
  out.B = static_cast<int64_t>(b.sample_ids.size());
  out.has_advantage = ja >= 0;
  out.has_mask = jm >= 0;
  if (b.payloads.size() != b.sample_ids.size()) {
    if (err) *err = "payloads missing (fetch with with_payload=true)";
    return SF_TM_CONFIG_ERROR;
  }
  for (size_t i = 0; i < b.sample_ids.size(); ++i) {
    const auto& row = b.payloads[i];
    if (row.size() != fs.size()) {
      if (err) *err = "payload row size != field_set size";
      return SF_TM_CONFIG_ERROR;
    }
    const size_t L = row[jr].size() / sizeof(int32_t);
    bool ok = row[jr].size() % sizeof(int32_t) == 0 && detail::append(row[jr], out.targets, L) &&
              detail::append(row[jl], out.logp, L) && detail::append(row[jf], out.ref_logp, L) &&
              detail::append(row[ja >= 0 ? ja : jw], out.per_sample, 1);
    if (ok && jm >= 0) ok = detail::append(row[jm], out.mask, L);
    if (ok && jg >= 0) ok = detail::append(row[jg], out.group_ids, 1);
    if (!ok) {
      if (err) *err = "sample " + std::to_string(b.sample_ids[i]) + ": payload sizes do not match response";
      return SF_TM_CONFIG_ERROR;
    }
    if (jg < 0) out.group_ids.push_back(group_size > 0 ? static_cast<int32_t>((b.sample_ids[i] - 1) / group_size) : 0);
    out.seq_lens.push_back(static_cast<int32_t>(L));
    out.T += static_cast<int64_t>(L);
  }
  if (b.producer_versions.size() == b.sample_ids.size())
    out.producer_versions.assign(b.producer_versions.begin(), b.producer_versions.end());
  return SF_TM_OK;
}

// Decode the "routed_experts" field of every sample into the R3 gate's recorded
// index operand, layer-major uint8 [layers, T, k] with T = sum of the samples'
// response lengths in bus order (the same token order as pack_trainer_batch).
// Returns SF_TM_OK or SF_TM_CONFIG_ERROR (missing field, size not L_i*layers*k).
template <class MicroBatchT>
int pack_routed_experts(const MicroBatchT& b, int layers, int k, std::vector<uint8_t>& out, int64_t* T_out,
                        std::string* err) {
  const int jr = detail::find_field(b.field_set, "response");
  const int je = detail::find_field(b.field_set, "routed_experts");
  if (jr < 0 || je < 0 || layers <= 0 || k <= 0) {
    if (err) *err = "routed_experts needs the response and routed_experts fields and layers, k > 0";
    return SF_TM_CONFIG_ERROR;
  }
  if (b.payloads.size() != b.sample_ids.size()) {
    if (err) *err = "payloads missing (fetch with with_payload=true)";
    return SF_TM_CONFIG_ERROR;
  }
  int64_t T = 0;
  for (size_t i = 0; i < b.payloads.size(); ++i) {
    const size_t L = b.payloads[i][jr].size() / sizeof(int32_t);
    if (b.payloads[i][je].size() != L * static_cast<size_t>(layers) * k) {
      if (err) *err = "sample " + std::to_string(b.sample_ids[i]) + ": routed_experts is not L*layers*k bytes";
      return SF_TM_CONFIG_ERROR;
    }
    T += static_cast<int64_t>(L);
  }
  out.assign(static_cast<size_t>(layers) * T * k, 0);
  int64_t t0 = 0;
  for (size_t i = 0; i < b.payloads.size(); ++i) {
    const auto& src = b.payloads[i][je];
    const int64_t L = static_cast<int64_t>(b.payloads[i][jr].size() / sizeof(int32_t));
    for (int64_t t = 0; t < L; ++t)
      for (int l = 0; l < layers; ++l)
        std::memcpy(out.data() + ((static_cast<size_t>(l) * T + t0 + t) * k),
                    src.data() + ((static_cast<size_t>(t) * layers + l) * k), static_cast<size_t>(k));
    t0 += L;
  }
  if (T_out) *T_out = T;
  return SF_TM_OK;
}

// One Actor role's device-side loss: owns the sf_tm handle and pinned staging.
class ActorLossSeam {
 public:
  explicit ActorLossSeam(int device = 0) { rc_ = sf_tm_create(device, &h_); }
  ~ActorLossSeam() {
    for (void* p : pin_) sf_tm_host_free(p);
    if (h_) sf_tm_destroy(h_);
  }
  ActorLossSeam(const ActorLossSeam&) = delete;
  ActorLossSeam& operator=(const ActorLossSeam&) = delete;

  int status() const { return rc_; }
  const char* last_error() const { return h_ ? sf_tm_last_error(h_) : "sf_tm_create failed"; }
  sf_tm_t handle() const { return h_; }

  // Decode `batch`, copy its bus fields through pinned staging, and run the
  // fused DAPO/GRPO loss fwd+bwd on `d_logits` [T, V] (row stride V). Writes
  // dlogits and the metrics (valid once `stream` is synchronised; steps may be
  // issued back to back, the next one overlapping this one's loss). When the
  // batch carries rewards (GRPO computed here), every group must be complete
  // in the micro-batch unless allow_partial_groups.
  template <class MicroBatchT>
  int step(const MicroBatchT& batch, const void* d_logits, int32_t dtype, int64_t V, void* d_dlogits,
           const sf_tm_loss_params& params, float* h_metrics, void* stream, int group_size = 0,
           float adv_eps = 1e-6f, int32_t std_mode = SF_TM_STD_UNBIASED, bool allow_partial_groups = false) {
    if (rc_ != SF_TM_OK) return rc_;
    std::string err;
    int rc = pack_trainer_batch(batch, group_size, packed_, &err);
    if (rc == SF_TM_OK && !packed_.has_advantage && !allow_partial_groups)
      rc = check_complete_groups(packed_, group_size, &err);
    if (rc != SF_TM_OK) {
      err_ = err;
      return rc;
    }
    const PackedBatch& p = packed_;
    // the previous step's H2D may still be reading the pinned staging (calls
    // are pipelined; no stream sync is required between steps)
    if ((rc = sf_tm_wait_host_inputs(h_))) return rc;
    if ((rc = stage(0, p.targets.data(), p.targets.size() * 4)) || (rc = stage(1, p.logp.data(), p.T * 4)) ||
        (rc = stage(2, p.ref_logp.data(), p.T * 4)) || (rc = stage(3, p.seq_lens.data(), p.B * 4)) ||
        (rc = stage(4, p.per_sample.data(), p.B * 4)) || (rc = stage(5, p.group_ids.data(), p.B * 4)))
      return rc;
    if (p.has_mask && (rc = stage(6, p.mask.data(), p.T))) return rc;
    return sf_tm_pg_step_host(h_, d_logits, dtype, p.T, V, V, static_cast<const int32_t*>(pin_[0]),
                              static_cast<const float*>(pin_[1]), static_cast<const float*>(pin_[2]),
                              p.has_mask ? static_cast<const uint8_t*>(pin_[6]) : nullptr,
                              static_cast<const int32_t*>(pin_[3]), nullptr, static_cast<const float*>(pin_[4]),
                              static_cast<const int32_t*>(pin_[5]), p.B, p.has_advantage ? -1.f : adv_eps,
                              std_mode, &params, d_dlogits, V, h_metrics, stream);
  }
  const PackedBatch& packed() const { return packed_; }
  const std::string& pack_error() const { return err_; }

 private:
  // Copy into the i-th pinned staging buffer (grown on demand; reused).
  int stage(int i, const void* src, size_t bytes) {
    if (bytes == 0) return SF_TM_OK;
    if (pin_cap_[i] < bytes) {
      if (pin_[i]) sf_tm_host_free(pin_[i]);
      pin_[i] = nullptr;
      const size_t cap = bytes + bytes / 4;
      if (int rc = sf_tm_host_alloc(cap, &pin_[i])) return rc;
      pin_cap_[i] = cap;
    }
    std::memcpy(pin_[i], src, bytes);
    return SF_TM_OK;
  }

  sf_tm_t h_ = nullptr;
  int rc_ = SF_TM_OK;
  PackedBatch packed_;
  std::string err_;
  void* pin_[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t pin_cap_[7] = {0, 0, 0, 0, 0, 0, 0};
};

// Pinned staging buffers, grown on demand and reused (used by the seams below).
class PinnedStage {
 public:
  PinnedStage() = default;
  PinnedStage(const PinnedStage&) = delete;
  PinnedStage& operator=(const PinnedStage&) = delete;
  ~PinnedStage() {
    for (auto& b : buf_)
      if (b.p) sf_tm_host_free(b.p);
  }
  // Returns a pinned buffer of >= bytes for slot i (contents not preserved).
  void* get(int i, size_t bytes, int* rc) {
    if (static_cast<size_t>(i) >= buf_.size()) buf_.resize(i + 1);
    Buf& b = buf_[i];
    if (b.cap < bytes) {
      if (b.p) sf_tm_host_free(b.p);
      b.p = nullptr;
      b.cap = 0;
      const size_t cap = bytes + bytes / 4 + 64;
      if ((*rc = sf_tm_host_alloc(cap, &b.p)) != SF_TM_OK) return nullptr;
      b.cap = cap;
    }
    *rc = SF_TM_OK;
    return b.p;
  }

 private:
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  std::vector<Buf> buf_;
};

// ActorFwd / RefLogP stage producer (the payload stub at proj/src/sim_runtime.cpp:322-334,
// proj/src/wall_runtime.cpp:126-129): the per-sample `logp` (or `ref_logp`) payload,
// fp32[L_i] = log-prob of each response token under the stage model, from that
// model's device logits [T, V] (samples concatenated in bus order). Synchronous:
// `payloads[i]` is ready for Bus::put_field when run returns.
class LogpStageSeam {
 public:
  explicit LogpStageSeam(int device = 0) { rc_ = sf_tm_create(device, &h_); }
  ~LogpStageSeam() {
    if (h_) sf_tm_destroy(h_);
  }
  LogpStageSeam(const LogpStageSeam&) = delete;
  LogpStageSeam& operator=(const LogpStageSeam&) = delete;
  int status() const { return rc_; }
  sf_tm_t handle() const { return h_; }
  const std::string& error() const { return err_; }

  template <class MicroBatchT, class BytesT>
  int run(const MicroBatchT& b, const void* d_logits, int32_t dtype, int64_t V, float inv_temperature,
          std::vector<BytesT>& payloads, void* stream) {
    if (rc_ != SF_TM_OK) return rc_;
    const int jr = detail::find_field(b.field_set, "response");
    if (jr < 0 || b.payloads.size() != b.sample_ids.size()) {
      err_ = "the stage needs the response field with payloads";
      return SF_TM_CONFIG_ERROR;
    }
    int64_t T = 0;
    for (const auto& row : b.payloads) {
      if (row[jr].size() % sizeof(int32_t)) {
        err_ = "response payload is not int32[L]";
        return SF_TM_CONFIG_ERROR;
      }
      T += static_cast<int64_t>(row[jr].size() / sizeof(int32_t));
    }
    int rc = SF_TM_OK;
    auto* tg = static_cast<uint8_t*>(pin_.get(0, static_cast<size_t>(T) * 4 + 4, &rc));
    if (rc) return rc;
    auto* lp = static_cast<float*>(pin_.get(1, static_cast<size_t>(T) * 4 + 4, &rc));
    if (rc) return rc;
    size_t off = 0;
    for (const auto& row : b.payloads) {
      if (!row[jr].empty()) std::memcpy(tg + off, row[jr].data(), row[jr].size());
      off += row[jr].size();
    }
    if ((rc = sf_tm_logprob_fwd_host(h_, d_logits, dtype, T, V, V, reinterpret_cast<const int32_t*>(tg),
                                     inv_temperature, lp, nullptr, stream)) ||
        (rc = sf_tm_sync(h_, stream))) {
      err_ = sf_tm_last_error(h_);
      return rc;
    }
    payloads.assign(b.payloads.size(), BytesT{});
    off = 0;
    for (size_t i = 0; i < b.payloads.size(); ++i) {
      const size_t L = b.payloads[i][jr].size() / sizeof(int32_t);
      payloads[i].resize(L * sizeof(float));
      if (L) std::memcpy(payloads[i].data(), lp + off, L * sizeof(float));
      off += L;
    }
    return SF_TM_OK;
  }

 private:
  sf_tm_t h_ = nullptr;
  int rc_ = SF_TM_OK;
  std::string err_;
  PinnedStage pin_;
};

// Advantages stage producer (controller.cpp:79 reward -> advantage): GRPO over
// the micro-batch's groups (field `group`, else (sample_id - 1) / group_size);
// every group must be complete. payloads[i] = fp32 advantage.
class AdvantageStageSeam {
 public:
  explicit AdvantageStageSeam(int device = 0) { rc_ = sf_tm_create(device, &h_); }
  ~AdvantageStageSeam() {
    if (h_) sf_tm_destroy(h_);
  }
  AdvantageStageSeam(const AdvantageStageSeam&) = delete;
  AdvantageStageSeam& operator=(const AdvantageStageSeam&) = delete;
  int status() const { return rc_; }
  const std::string& error() const { return err_; }

  template <class MicroBatchT, class BytesT>
  int run(const MicroBatchT& b, int group_size, float eps, int32_t std_mode, std::vector<BytesT>& payloads,
          void* stream) {
    if (rc_ != SF_TM_OK) return rc_;
    const int jw = detail::find_field(b.field_set, "reward"), jg = detail::find_field(b.field_set, "group");
    if (jw < 0 || b.payloads.size() != b.sample_ids.size() || (jg < 0 && group_size <= 0)) {
      err_ = "the stage needs the reward field with payloads and a group field or group_size";
      return SF_TM_CONFIG_ERROR;
    }
    const int64_t B = static_cast<int64_t>(b.sample_ids.size());
    PackedBatch p;
    for (int64_t i = 0; i < B; ++i) {
      const auto& row = b.payloads[i];
      if (!detail::append(row[jw], p.per_sample, 1) || (jg >= 0 && !detail::append(row[jg], p.group_ids, 1))) {
        err_ = "sample " + std::to_string(b.sample_ids[i]) + ": reward/group payload is not 4 bytes";
        return SF_TM_CONFIG_ERROR;
      }
      if (jg < 0) p.group_ids.push_back(static_cast<int32_t>((b.sample_ids[i] - 1) / group_size));
    }
    int rc = check_complete_groups(p, jg < 0 ? group_size : 0, &err_);
    if (rc) return rc;
    auto* rw = static_cast<float*>(pin_.get(0, static_cast<size_t>(B) * 4 + 4, &rc));
    if (rc) return rc;
    auto* gi = static_cast<int32_t*>(pin_.get(1, static_cast<size_t>(B) * 4 + 4, &rc));
    if (rc) return rc;
    auto* ad = static_cast<float*>(pin_.get(2, static_cast<size_t>(B) * 4 + 4, &rc));
    if (rc) return rc;
    if (B) {
      std::memcpy(rw, p.per_sample.data(), static_cast<size_t>(B) * 4);
      std::memcpy(gi, p.group_ids.data(), static_cast<size_t>(B) * 4);
    }
    if ((rc = sf_tm_grpo_advantage_host(h_, rw, gi, B, eps, std_mode, ad, stream)) ||
        (rc = sf_tm_sync(h_, stream))) {
      err_ = sf_tm_last_error(h_);
      return rc;
    }
    payloads.assign(static_cast<size_t>(B), BytesT(sizeof(float)));
    for (int64_t i = 0; i < B; ++i) std::memcpy(payloads[i].data(), ad + i, sizeof(float));
    return SF_TM_OK;
  }

 private:
  sf_tm_t h_ = nullptr;
  int rc_ = SF_TM_OK;
  std::string err_;
  PinnedStage pin_;
};


// ---------------------------------------------------------------------------
// Group-completion batching. The bus hands samples
// out FIFO by readiness (proj/src/transfer_queue.cpp:162-175) and sample ids
// are sequential per permit (proj/src/staleness.cpp:102-106), so a fetched
// micro-batch can hold any mix of partial groups. GRPO is only defined over a
// whole group: the Advantages stage (and a trainer that computes GRPO itself)
// feeds every fetched micro-batch in here and takes back micro-batches made
// of complete groups only, in the order the groups completed. Group of a
// sample: its int32 "group" field, else (sample_id - 1) / group_size.
template <class MicroBatchT>
class GroupAssembler {
 public:
  explicit GroupAssembler(int group_size) : gs_(group_size) {}

  // Buffer every sample of `b` (payloads required). SF_TM_OK, or
  // SF_TM_CONFIG_ERROR (no payloads, a field set that differs from earlier
  // batches, a group that receives more than group_size samples).
  int feed(const MicroBatchT& b, std::string* err) {
    if (gs_ <= 0) return fail(err, "group_size must be > 0");
    if (b.payloads.size() != b.sample_ids.size()) return fail(err, "payloads missing (fetch with with_payload=true)");
    if (fields_.empty()) {
      fields_ = b.field_set;
      jg_ = detail::find_field(fields_, "group");
    } else if (b.field_set != fields_) {
      return fail(err, "field set changed between micro-batches");
    }
    for (size_t i = 0; i < b.sample_ids.size(); ++i) {
      int64_t g;
      if (jg_ >= 0) {
        int32_t v = 0;
        if (b.payloads[i][jg_].size() != sizeof(v)) return fail(err, "group payload is not int32");
        std::memcpy(&v, b.payloads[i][jg_].data(), sizeof(v));
        g = v;
      } else {
        g = static_cast<int64_t>((b.sample_ids[i] - 1) / static_cast<uint64_t>(gs_));
      }
      auto& bucket = partial_[g];
      Sample smp{b.sample_ids[i], i < b.producer_versions.size() ? b.producer_versions[i] : Version{},
                 i < b.global_steps.size() ? b.global_steps[i] : Step{}, b.payloads[i]};
      bucket.push_back(std::move(smp));
      if (static_cast<int>(bucket.size()) > gs_)
        return fail(err, "group " + std::to_string(g) + " received more than " + std::to_string(gs_) + " samples");
      if (static_cast<int>(bucket.size()) == gs_) {
        ready_.push_back(std::move(bucket));
        partial_.erase(g);
        ready_samples_ += static_cast<size_t>(gs_);
      }
    }
    return SF_TM_OK;
  }

  // Move up to max_samples samples of complete groups (whole groups only, in
  // completion order) into `out`. Returns the number of samples moved (0 when
  // no group is complete or max_samples < group_size).
  size_t pop(MicroBatchT& out, size_t max_samples) {
    out = MicroBatchT{};
    out.batch_id = ++batches_;
    out.field_set = fields_;
    size_t n = 0;
    while (!ready_.empty() && n + static_cast<size_t>(gs_) <= max_samples) {
      for (auto& smp : ready_.front()) {
        out.sample_ids.push_back(smp.id);
        out.producer_versions.push_back(smp.version);
        out.global_steps.push_back(smp.step);
        out.payloads.push_back(std::move(smp.row));
      }
      ready_.pop_front();
      n += static_cast<size_t>(gs_);
    }
    ready_samples_ -= n;
    return n;
  }

  size_t ready_samples() const { return ready_samples_; }
  size_t pending_groups() const { return partial_.size(); }
  size_t pending_samples() const {
    size_t n = 0;
    for (const auto& kv : partial_) n += kv.second.size();
    return n;
  }

 private:
  using Version = typename std::decay_t<decltype(std::declval<MicroBatchT>().producer_versions)>::value_type;
  using Step = typename std::decay_t<decltype(std::declval<MicroBatchT>().global_steps)>::value_type;
  using SampleId = typename std::decay_t<decltype(std::declval<MicroBatchT>().sample_ids)>::value_type;
  using Row = typename std::decay_t<decltype(std::declval<MicroBatchT>().payloads)>::value_type;
  struct Sample {
    SampleId id;
    Version version;
    Step step;
    Row row;
  };
  static int fail(std::string* err, const std::string& m) {
    if (err) *err = m;
    return SF_TM_CONFIG_ERROR;
  }
  int gs_;
  int jg_ = -1;
  std::vector<std::string> fields_;
  std::map<int64_t, std::vector<Sample>> partial_;
  std::deque<std::vector<Sample>> ready_;
  size_t ready_samples_ = 0;
  uint64_t batches_ = 0;
};

// ---------------------------------------------------------------------------
// Version-boundary normalisation (the trainer's version boundary
// fires once consumed_in_version >= G samples, proj/src/sim_runtime.cpp:453-454,
// 514-557). The DAPO token-mean divides by N = the loss-active tokens of the
// whole version, which is unknown while its micro-batches stream in. Each
// micro-batch therefore runs with micro_params() (explicit inv_norm = 1: its
// dlogits and metrics are unnormalised sums, so the trainer's parameter
// gradients accumulate unnormalised too); at the boundary close() returns the
// scale 1/N for the accumulated gradients and the normalised step metrics.
// By linearity this equals running every micro-batch with inv_norm = 1/N.
class VersionAccumulator {
 public:
  explicit VersionAccumulator(uint64_t global_batch_size) : G_(global_batch_size) {}

  static sf_tm_loss_params micro_params(sf_tm_loss_params p) {
    p.norm_mode = SF_TM_NORM_EXPLICIT;
    p.inv_norm = 1.f;
    return p;
  }
  // One micro-batch's metrics (computed with micro_params) and its sample count.
  void add(const float* h_metrics, uint64_t samples) {
    for (int i = 0; i < SF_TM_NUM_METRICS; ++i) sum_[i] += static_cast<double>(h_metrics[i]);
    consumed_ += samples;
    ++micro_batches_;
  }
  bool at_boundary() const { return consumed_ >= G_; }
  uint64_t consumed() const { return consumed_; }

  struct Closed {
    uint64_t samples = 0, micro_batches = 0;
    double active_tokens = 0.0;
    double grad_scale = 0.0;  // multiply the version's accumulated gradients by this (1/N)
    double metrics[SF_TM_NUM_METRICS] = {};  // token-means over the version; [SF_TM_M_ACTIVE] = N
  };
  Closed close() {
    Closed c;
    c.samples = consumed_;
    c.micro_batches = micro_batches_;
    c.active_tokens = sum_[SF_TM_M_ACTIVE];
    c.grad_scale = c.active_tokens > 0 ? 1.0 / c.active_tokens : 0.0;
    for (int i = 0; i < SF_TM_NUM_METRICS; ++i)
      c.metrics[i] = (i == SF_TM_M_ACTIVE) ? sum_[i] : sum_[i] * c.grad_scale;
    for (double& v : sum_) v = 0.0;
    consumed_ = 0;
    micro_batches_ = 0;
    return c;
  }

 private:
  uint64_t G_;
  uint64_t consumed_ = 0, micro_batches_ = 0;
  double sum_[SF_TM_NUM_METRICS] = {};
};

// ---------------------------------------------------------------------------
// R3 routed-experts transport (the paper keeps the record
// GPU-resident). The samples' routed_experts payloads are
// token-major, so their bus-order concatenation IS the token-major record
// [T, layers, k]: it is staged with one memcpy per sample (no per-byte host
// transpose, unlike pack_routed_experts), copied to the device once, and
// transposed to the gate's layer-major operand there
// (sf_tm_r3_record_layer_major). d_tok: caller-owned device scratch of
// T * layers * k bytes; d_rec: the layer-major u8 [layers, T, k] output.
class RoutedExpertsSeam {
 public:
  explicit RoutedExpertsSeam(int device = 0) { rc_ = sf_tm_create(device, &h_); }
  ~RoutedExpertsSeam() {
    if (h_) sf_tm_destroy(h_);
  }
  RoutedExpertsSeam(const RoutedExpertsSeam&) = delete;
  RoutedExpertsSeam& operator=(const RoutedExpertsSeam&) = delete;
  int status() const { return rc_; }
  sf_tm_t handle() const { return h_; }
  const std::string& error() const { return err_; }

  // Token count of the batch's record (sum of response lengths), or -1 with error().
  template <class MicroBatchT>
  int64_t tokens(const MicroBatchT& b, int layers, int k) {
    const int jr = detail::find_field(b.field_set, "response");
    const int je = detail::find_field(b.field_set, "routed_experts");
    if (jr < 0 || je < 0 || layers <= 0 || k <= 0 || b.payloads.size() != b.sample_ids.size()) {
      err_ = "routed_experts needs the response and routed_experts fields (with payloads) and layers, k > 0";
      return -1;
    }
    int64_t T = 0;
    for (size_t i = 0; i < b.payloads.size(); ++i) {
      const size_t L = b.payloads[i][jr].size() / sizeof(int32_t);
      if (b.payloads[i][je].size() != L * static_cast<size_t>(layers) * k) {
        err_ = "sample " + std::to_string(b.sample_ids[i]) + ": routed_experts is not L*layers*k bytes";
        return -1;
      }
      T += static_cast<int64_t>(L);
    }
    return T;
  }

  // Stage + copy + device transpose; asynchronous on `stream` (the pinned
  // staging is reused by the next call only after this one's copy finished).
  template <class MicroBatchT>
  int upload(const MicroBatchT& b, int layers, int k, void* d_tok, void* d_rec, int64_t* T_out, void* stream) {
    if (rc_ != SF_TM_OK) return rc_;
    const int64_t T = tokens(b, layers, k);
    if (T < 0) return SF_TM_CONFIG_ERROR;
    if (T_out) *T_out = T;
    const size_t bytes = static_cast<size_t>(T) * layers * k;
    if (bytes == 0) return SF_TM_OK;
    int rc = sf_tm_sync(h_, stream);  // the previous upload's copy has read the staging
    if (rc) return rc;
    auto* st = static_cast<uint8_t*>(pin_.get(0, bytes, &rc));
    if (rc) return rc;
    const int je = detail::find_field(b.field_set, "routed_experts");
    size_t off = 0;
    for (const auto& row : b.payloads) {
      std::memcpy(st + off, row[je].data(), row[je].size());
      off += row[je].size();
    }
    if ((rc = sf_tm_h2d(h_, d_tok, st, bytes, stream)) ||
        (rc = sf_tm_r3_record_layer_major(h_, d_tok, SF_TM_IDX_U8, T, layers, k, d_rec, stream))) {
      err_ = sf_tm_last_error(h_);
      return rc;
    }
    return SF_TM_OK;
  }

 private:
  sf_tm_t h_ = nullptr;
  int rc_ = SF_TM_OK;
  std::string err_;
  PinnedStage pin_;
};

}  // namespace train_math
}  // namespace staleflow
