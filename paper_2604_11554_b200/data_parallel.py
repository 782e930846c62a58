# SPDX-License-Identifier: Apache-2.0
"""Sequence sharding across ranks (SURVEY.md §8e partitioning A).

Each rank owns whole packed sequences of the step; the rows are independent, so
the data path has no collective. The DAPO token-mean, though, divides by the
loss-active tokens of the WHOLE step: the ranks agree on
N = sum over ranks of their active tokens (one 8-byte all-reduce before the
step), every rank weights its tokens by 1/N, and the SUM all-reduce of the
per-rank metric sums after the step is then exactly the single-GPU token-mean
of the union batch. The reference has no counterpart (no collectives,
SPEC.md:8); its trainer consumes the global batch one micro-batch at a time
(proj/src/sim_runtime.cpp:431-463).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def _initialized() -> bool:
    return dist.is_available() and dist.is_initialized()


def global_active_tokens(local_active: int, group=None, device: Optional[torch.device] = None) -> int:
    """Sum of the ranks' loss-active token counts (identical on every rank)."""
    if not _initialized() or dist.get_world_size(group) == 1:
        return int(local_active)
    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([int(local_active)], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def global_inv_norm(local_active: int, group=None, device: Optional[torch.device] = None) -> float:
    """1 / (global loss-active tokens): the explicit inv_norm every rank passes
    (SF_TM_NORM_EXPLICIT) so the per-rank sums add up to the global token-mean."""
    n = global_active_tokens(local_active, group, device)
    return 1.0 / n if n > 0 else 0.0


def reduce_step_metrics(metrics: torch.Tensor, group=None) -> torch.Tensor:
    """SUM all-reduce (in place) of per-rank metric sums [.., SF_TM_NUM_METRICS]
    computed with global_inv_norm weights: the result is the global step's."""
    if _initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(metrics, op=dist.ReduceOp.SUM, group=group)
    return metrics
