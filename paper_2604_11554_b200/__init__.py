# SPDX-License-Identifier: Apache-2.0
"""staleflow train-math on B200: the per-token training-math hot path of Relax
(arXiv 2604.11554) — fused log-softmax gather with dlogits, GRPO advantage,
DAPO/KL masked token-mean loss, R3 replay gate, vocab-parallel combine — as
hand-written sm_100a CUDA behind the C-ABI in include/staleflow/train_math.h.

`train_math` is the Python mirror of that C-ABI (torch tensors in, raw device
pointers out); `vocab_parallel` adds the multi-GPU vocabulary-sharded loss
(in-kernel peer exchange, or the two-pass NCCL form). There is no CPU
implementation in this package: without the CUDA library every call raises.
"""
__all__ = ["train_math", "vocab_parallel"]
