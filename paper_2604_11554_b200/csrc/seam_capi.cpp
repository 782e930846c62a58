// SPDX-License-Identifier: Apache-2.0
//
// C-ABI of include/staleflow/train_math_seam_c.h: the C++ ActorLossSeam
// (include/staleflow/train_math_seam.hpp) over a MicroBatch with the member
// layout of proj/include/staleflow/types.hpp:48-59. Host code only; it calls
// the CUDA kernels through libsf_train_math.so.
#include "staleflow/train_math_seam_c.h"

#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "staleflow/train_math_seam.hpp"

namespace {
using Bytes = std::vector<std::uint8_t>;
struct MicroBatch {  // member names and types as staleflow::MicroBatch (types.hpp:48-59)
  std::uint64_t batch_id = 0;
  std::vector<std::uint64_t> sample_ids;
  std::vector<std::string> field_set;
  std::vector<std::int64_t> producer_versions;
  std::vector<std::int64_t> global_steps;
  std::vector<std::vector<Bytes>> payloads;
};
template <class T>
Bytes enc(const T* v, size_t n) {
  Bytes b(n * sizeof(T));
  if (n) std::memcpy(b.data(), v, b.size());
  return b;
}
}  // namespace

struct sf_seam {
  explicit sf_seam(int device) : seam(device) {}
  staleflow::train_math::ActorLossSeam seam;
  std::string err;
};
struct sf_seam_batch {
  MicroBatch mb;
};

extern "C" {

int sf_seam_create(int device, sf_seam_t* out) {
  if (!out) return SF_TM_CONFIG_ERROR;
  *out = nullptr;
  sf_seam_t s = new (std::nothrow) sf_seam(device);
  if (!s) return SF_TM_INTERNAL;
  if (int rc = s->seam.status()) {
    delete s;
    return rc;
  }
  *out = s;
  return SF_TM_OK;
}

int sf_seam_destroy(sf_seam_t s) {
  delete s;
  return SF_TM_OK;
}

const char* sf_seam_last_error(sf_seam_t s) {
  if (!s) return "null seam";
  if (!s->err.empty()) return s->err.c_str();
  return s->seam.last_error();
}

int sf_seam_batch_build(int64_t B, const int32_t* seq_lens, const int32_t* targets, const float* logp,
                        const float* ref_logp, const float* per_sample, int32_t has_advantage, const uint8_t* loss_mask,
                        const uint64_t* sample_ids, const int64_t* producer_versions, sf_seam_batch_t* out) {
  if (!out || B < 0 || (B > 0 && (!seq_lens || !targets || !logp || !ref_logp || !per_sample || !sample_ids)))
    return SF_TM_CONFIG_ERROR;
  *out = nullptr;
  sf_seam_batch_t b = new (std::nothrow) sf_seam_batch();
  if (!b) return SF_TM_INTERNAL;
  MicroBatch& mb = b->mb;
  // sorted trainer field set (TransferQueue::get_ready_batch sorts it, transfer_queue.cpp:183)
  mb.field_set = {has_advantage ? "advantage" : "reward", "logp", "ref_logp", "response"};
  if (loss_mask) mb.field_set.push_back("loss_mask");
  std::sort(mb.field_set.begin(), mb.field_set.end());
  int64_t off = 0;
  for (int64_t i = 0; i < B; ++i) {
    if (seq_lens[i] < 0) {
      delete b;
      return SF_TM_CONFIG_ERROR;
    }
    const size_t L = static_cast<size_t>(seq_lens[i]);
    std::vector<Bytes> row;
    for (const auto& f : mb.field_set) {
      if (f == "advantage" || f == "reward") row.push_back(enc(per_sample + i, 1));
      else if (f == "logp") row.push_back(enc(logp + off, L));
      else if (f == "ref_logp") row.push_back(enc(ref_logp + off, L));
      else if (f == "response") row.push_back(enc(targets + off, L));
      else row.push_back(enc(loss_mask + off, L));
    }
    mb.payloads.push_back(std::move(row));
    mb.sample_ids.push_back(sample_ids[i]);
    mb.producer_versions.push_back(producer_versions ? producer_versions[i] : 0);
    mb.global_steps.push_back(0);
    off += static_cast<int64_t>(L);
  }
  *out = b;
  return SF_TM_OK;
}

int sf_seam_batch_free(sf_seam_batch_t b) {
  delete b;
  return SF_TM_OK;
}

int sf_seam_batch_staleness(sf_seam_batch_t b, int64_t v_trainer, int64_t* batch_staleness, uint64_t* hist,
                            int32_t n_hist) {
  if (!b || n_hist < 0 || (n_hist > 0 && !hist)) return SF_TM_CONFIG_ERROR;
  staleflow::train_math::PackedBatch p;
  p.producer_versions = b->mb.producer_versions;
  int64_t bs = 0;
  const auto h = staleflow::train_math::staleness_histogram(p, v_trainer, &bs);
  if (batch_staleness) *batch_staleness = bs;
  for (const auto& kv : h)
    if (kv.first >= 0 && kv.first < n_hist) hist[kv.first] += kv.second;
  return SF_TM_OK;
}

int sf_seam_step(sf_seam_t s, sf_seam_batch_t b, const void* logits, int32_t dtype, int64_t V, void* dlogits,
                 const sf_tm_loss_params* params, float* h_metrics, void* stream, int32_t group_size) {
  if (!s || !b || !params) return SF_TM_CONFIG_ERROR;
  s->err.clear();
  const int rc = s->seam.step(b->mb, logits, dtype, V, dlogits, *params, h_metrics, stream, group_size);
  if (rc && !s->seam.pack_error().empty()) s->err = s->seam.pack_error();
  return rc;
}

}  // extern "C"
