# SPDX-License-Identifier: Apache-2.0
"""Vocab-parallel fused loss (SURVEY.md §8 row a7, §8e partitioning B).

Rank p of P holds logits[:, vs_p : vs_p + Vp] (the natural output of a
vocab-parallel LM head). One step is:

  1. sf_tm_vp_partial_stats on the local shard -> stats[T, 4] =
     {max z, sum e^(z - max), sum e^(z - max)(z - max), z_target or NaN};
  2. all_gather of stats over the group (NCCL over NVLink; 16 B/token/rank,
     versus 4V/P B/token of HBM traffic per rank);
  3. sf_tm_vp_loss_fwd_bwd: every rank merges the P partials in rank order
     (identical lse/entropy/logp/loss on every rank) and writes its shard's
     dlogits.

`vp_fused_pg_loss_fwd_bwd` is the single-pass form (compute
fused with its collective): one persistent kernel per rank, the per-row
partials exchanged between the ranks' control warps through peer-mapped
mailboxes over NVLink, so each shard row is read once (4V/P B/token/rank
instead of 6V/P). `open_peer_exchange(group)` sets it up once per group.

The exchange is a single collective (all_gather) instead of the MAX then SUM
all-reduce pair; it carries the same information and lets every rank merge in
the same fixed order, so the per-token scalars are bitwise identical across
ranks. The reference has no counterpart (no NCCL anywhere; the
paper's GPU-resident transport is PAPER.md:250,577).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from . import train_math as tm
from ._lib import LossParams


def shard_bounds(V: int, P: int, align: int = 8) -> list[int]:
    """Vocab shard boundaries [b0=0, ..., bP=V] with every shard start aligned
    to `align` elements (16 B for bf16) so each shard row can be TMA-streamed."""
    if P < 1 or V < 1:
        raise ValueError("need V >= 1 and P >= 1")
    b = [((V * p) // P) // align * align for p in range(P)] + [V]
    for i in range(P):
        if b[i + 1] <= b[i]:
            raise ValueError(f"vocab {V} too small for {P} aligned shards")
    return b


def gather_stats(local_stats: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather per-rank [T, 4] partial statistics into [P, T, 4] (rank order)."""
    P = dist.get_world_size(group)
    T = local_stats.shape[0]
    out = torch.empty((P * T,) + tuple(local_stats.shape[1:]), dtype=local_stats.dtype, device=local_stats.device)
    dist.all_gather_into_tensor(out, local_stats.contiguous(), group=group)
    return out.view((P, T) + tuple(local_stats.shape[1:]))


def vp_pg_loss_fwd_bwd(shard: torch.Tensor, vocab_start: int, targets, old_logp, ref_logp, adv_tok, w_tok,
                       params: Optional[LossParams] = None, dlogits=None, group=None, want_logp: bool = False,
                       inv_temperature: Optional[float] = None):
    """Fused DAPO/GRPO loss fwd+bwd on a vocab shard; returns
    (metrics, dlogits_shard, logp, entropy) — metrics identical on every rank."""
    if params is None:
        params = tm.default_loss_params()
    it = params.inv_temperature if inv_temperature is None else inv_temperature
    stats = tm.vp_partial_stats(shard, targets, vocab_start, it)
    gathered = gather_stats(stats, group)
    return tm.vp_loss_fwd_bwd(shard, vocab_start, gathered, targets, old_logp, ref_logp, adv_tok, w_tok, params,
                              dlogits=dlogits, want_logp=want_logp)


_peer_groups: dict = {}   # (device, group's global ranks) -> agreed outcome
_bound: dict = {}         # device -> group key its handle's mailbox is bound to


def _group_key(group):
    ranks = tuple(dist.get_process_group_ranks(group)) if group is not None else \
        tuple(range(dist.get_world_size()))
    return ranks


def open_peer_exchange(group=None) -> bool:
    """Create this rank's peer mailbox, all-gather the 64-byte CUDA IPC handles
    over `group` (any backend) and map the peers. The outcome is agreed on by
    all ranks: if any rank cannot map its peers (no P2P path), every rank
    reports False and the callers use the two-pass NCCL form. Cached per
    (device, group); a handle's mailbox serves one group only, so a second
    group on the same device gets False (two-pass) on every rank."""
    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    key = (dev, _group_key(group))
    if key in _peer_groups:
        return _peer_groups[key]
    P = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ok = True
    mine = None
    if dev in _bound:
        ok = False  # this device's handle is already bound to another group
    else:
        try:
            mine = tm.vp_mailbox_create(P, rank, dev)
            _bound[dev] = key
        except tm.TrainMathError:
            ok = False
    handles = [None] * P
    dist.all_gather_object(handles, mine, group=group)
    if ok and all(h is not None for h in handles):
        try:
            tm.vp_mailbox_open(handles, dev)
        except tm.TrainMathError:
            ok = False
    else:
        ok = False
    flags = [None] * P
    dist.all_gather_object(flags, ok, group=group)
    _peer_groups[key] = all(flags)
    return _peer_groups[key]


def _all_ok(ok: bool, device, group) -> bool:
    """Agree on a per-rank flag (MIN over the group, one 4-byte all-reduce)."""
    f = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device)
    dist.all_reduce(f, op=dist.ReduceOp.MIN, group=group)
    return bool(f.item())


def vp_fused_pg_loss_fwd_bwd(shard: torch.Tensor, vocab_start: int, targets, old_logp, ref_logp, adv_tok, w_tok,
                             params: Optional[LossParams] = None, dlogits=None, group=None, want_logp: bool = False,
                             metrics=None):
    """Single-pass vocab-parallel fused loss (exchange inside the kernel over
    NVLink peer memory); same outputs as vp_pg_loss_fwd_bwd, which it falls back
    to on every rank when the ranks cannot map each other's memory or when any
    rank's shard is not eligible (shape, alignment, row-store size) -- the
    eligibility is agreed before the kernel launches, so no rank is left
    waiting for a peer that did not launch."""
    use = open_peer_exchange(group)
    if use:
        rc, _ = tm.vp_fused_check(shard, dlogits)
        use = _all_ok(rc == 0, shard.device, group)
    if not use:
        met, dl, lp, ent = vp_pg_loss_fwd_bwd(shard, vocab_start, targets, old_logp, ref_logp, adv_tok, w_tok, params,
                                              dlogits=dlogits, group=group, want_logp=want_logp)
        if metrics is not None:
            metrics.copy_(met)
            met = metrics
        return met, dl, lp, ent
    return tm.vp_fused_loss_fwd_bwd(shard, vocab_start, targets, old_logp, ref_logp, adv_tok, w_tok, params,
                                    dlogits=dlogits, want_logp=want_logp, metrics=metrics)
