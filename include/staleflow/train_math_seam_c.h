/* SPDX-License-Identifier: Apache-2.0
 *
 * C-ABI over the C++ trainer seam (include/staleflow/train_math_seam.hpp), for
 * callers that are not C++ (the Python bench's end-to-end leg): one trainer
 * MicroBatch (proj/include/staleflow/types.hpp:48-59) in its bus encoding —
 * per-sample payload bytes of the sorted trainer field set, as
 * TransferQueue::get_ready_batch deep-copies them (transfer_queue.cpp:202-207)
 * — and ActorLossSeam::step on it: payload decode, pinned staging, H2D,
 * GRPO / token weights, fused loss fwd+bwd, D2H metrics. Errors are
 * staleflow::Errc values as in train_math.h.
 */
#ifndef STALEFLOW_TRAIN_MATH_SEAM_C_H_
#define STALEFLOW_TRAIN_MATH_SEAM_C_H_

#include <stdint.h>

#include "staleflow/train_math.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sf_seam* sf_seam_t;          /* one Actor role's ActorLossSeam */
typedef struct sf_seam_batch* sf_seam_batch_t; /* one MicroBatch with payloads */

int sf_seam_create(int device, sf_seam_t* out);
int sf_seam_destroy(sf_seam_t s);
const char* sf_seam_last_error(sf_seam_t s);

/* Encode B samples as a trainer MicroBatch: fields response (int32[L_i]),
 * logp, ref_logp (float32[L_i]), advantage (float32, has_advantage != 0) or
 * reward (float32), loss_mask (uint8[L_i], optional). Arrays are packed in
 * sample order (seq_lens[i] tokens each); sample_ids / producer_versions are
 * the bus keys (producer_versions optional). */
int sf_seam_batch_build(int64_t B, const int32_t* seq_lens, const int32_t* targets, const float* logp,
                        const float* ref_logp, const float* per_sample, int32_t has_advantage, const uint8_t* loss_mask,
                        const uint64_t* sample_ids, const int64_t* producer_versions, sf_seam_batch_t* out);
int sf_seam_batch_free(sf_seam_batch_t b);

/* Staleness tags of the batch: *batch_staleness = v_trainer -
 * min producer_version (StalenessGate::staleness_of, staleness.cpp:169-173) and
 * hist[s] += number of samples with v_trainer - producer_version == s for
 * 0 <= s < n_hist (others are not counted). */
int sf_seam_batch_staleness(sf_seam_batch_t b, int64_t v_trainer, int64_t* batch_staleness, uint64_t* hist,
                            int32_t n_hist);

/* ActorLossSeam::step on `b` (logits [T, V] row stride V, device-resident).
 * group_size: GRPO group size when the batch carries rewards. h_metrics is
 * host float[SF_TM_NUM_METRICS], valid after `stream` is synchronised. */
int sf_seam_step(sf_seam_t s, sf_seam_batch_t b, const void* logits, int32_t dtype, int64_t V, void* dlogits,
                 const sf_tm_loss_params* params, float* h_metrics, void* stream, int32_t group_size);

#ifdef __cplusplus
}
#endif

#endif /* STALEFLOW_TRAIN_MATH_SEAM_C_H_ */
