# SPDX-License-Identifier: Apache-2.0
"""Python host mirror of the staleflow train-math C-ABI (include/staleflow/train_math.h).

Each function here calls exactly one C-ABI entry point of the same name with raw
device pointers taken from torch tensors; torch is only device memory and the
current CUDA stream. Argument meaning and error behaviour are the C-ABI's:
a non-Ok staleflow::Errc (result.hpp:14-47) raises TrainMathError with the
handle's last_error message. There is no CPU path.

Seam map (reference file:line, see the header for the full list):
  logprob_fwd      -> ActorFwd / RefLogP stage stub, proj/src/sim_runtime.cpp:304-350
  grpo_advantage   -> Advantages stage (controller.cpp:79)
  pg_loss_fwd_bwd  -> trainer_compute_batch latency, proj/src/sim_runtime.cpp:441
  pg_step_host     -> trainer_thread micro-batch, proj/src/wall_runtime.cpp:178-198
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _lib
from ._lib import LossParams, TrainMathError, default_loss_params  # noqa: F401

_DT = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16}


def _p(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Handle:
    """Owns an sf_tm_t (scratch + error state) for one device."""

    def __init__(self, device: int = 0):
        self.device = device
        self._h = _lib._H()
        rc = _lib.lib().sf_tm_create(device, ctypes.byref(self._h))
        if rc != 0:
            raise TrainMathError(rc, f"sf_tm_create(device={device}) failed (sm_100a B200 required)")

    @property
    def ptr(self):
        return self._h

    def check(self, rc: int, what: str):
        if rc != 0:
            msg = _lib.lib().sf_tm_last_error(self._h)
            raise TrainMathError(rc, f"{what}: {msg.decode() if msg else ''}")

    def launch_count(self) -> int:
        return int(_lib.lib().sf_tm_launch_count(self._h))

    def last_launch(self) -> dict:
        """The last row-kernel launch: kernel name, CTAs per row, grid."""
        k, c, g = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        self.check(_lib.lib().sf_tm_last_launch(self._h, ctypes.byref(k), ctypes.byref(c), ctypes.byref(g)),
                   "sf_tm_last_launch")
        names = {0: "rows_ring_kernel", 1: "rows_generic_kernel", 2: "loss_tmem_kernel",
                 4: "loss_tmem_kernel[peer-exchange]", 5: "fwd_stream_kernel"}
        ns = ctypes.c_int32()
        self.check(_lib.lib().sf_tm_last_launch_streams(self._h, ctypes.byref(ns)), "sf_tm_last_launch_streams")
        return {"kernel": names.get(k.value, str(k.value)), "cluster": c.value, "grid": g.value,
                "streams": ns.value}

    def close(self):
        if self._h:
            _lib.lib().sf_tm_destroy(self._h)
            self._h = _lib._H()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_handles: dict[int, Handle] = {}


def handle(device: Optional[int] = None) -> Handle:
    if device is None:
        device = torch.cuda.current_device()
    h = _handles.get(device)
    if h is None:
        h = Handle(device)
        _handles[device] = h
    return h


def _dev(t: torch.Tensor) -> int:
    if not t.is_cuda:
        raise TrainMathError(_lib.CONFIG_ERROR, "tensors must live on a CUDA device (no CPU path)")
    return t.device.index


def _rows(logits: torch.Tensor):
    if logits.dim() != 2 or logits.stride(1) != 1:
        raise TrainMathError(_lib.CONFIG_ERROR, "logits must be 2-D with unit column stride")
    if logits.dtype not in _DT:
        raise TrainMathError(_lib.CONFIG_ERROR, "logits dtype must be float32 or bfloat16")
    T, V = logits.shape
    return _DT[logits.dtype], T, V, logits.stride(0)


def set_force_generic(on: bool):
    _lib.lib().sf_tm_debug_force_generic(1 if on else 0)


# ---------------------------------------------------------------------- a6
def varlen_meta(seq_lens: torch.Tensor, prompt_lens=None, group_ids=None, T: Optional[int] = None,
                want=("cu", "seq_id", "mask", "tok_group")):
    d = _dev(seq_lens)
    h = handle(d)
    B = seq_lens.numel()
    if T is None:
        T = int(seq_lens.sum().item())
    cu = torch.empty(B + 1, dtype=torch.int32, device=seq_lens.device)
    seq_id = torch.empty(T, dtype=torch.int32, device=seq_lens.device) if "seq_id" in want else None
    mask = torch.empty(T, dtype=torch.uint8, device=seq_lens.device) if "mask" in want else None
    tg = (torch.empty(T, dtype=torch.int32, device=seq_lens.device)
          if ("tok_group" in want and group_ids is not None) else None)
    rc = _lib.lib().sf_tm_varlen_meta(h.ptr, _p(seq_lens), _p(prompt_lens), _p(group_ids), B, T,
                                      _p(cu), _p(seq_id), _p(mask), _p(tg), _stream(d))
    h.check(rc, "sf_tm_varlen_meta")
    return cu, seq_id, mask, tg


# ---------------------------------------------------------------------- a3
def grpo_advantage(rewards: torch.Tensor, group_ids: torch.Tensor, eps: float = 1e-6,
                   std_mode: int = _lib.STD_UNBIASED, want_group_size: bool = False):
    d = _dev(rewards)
    h = handle(d)
    B = rewards.numel()
    adv = torch.empty(B, dtype=torch.float32, device=rewards.device)
    gs = torch.empty(B, dtype=torch.int32, device=rewards.device) if want_group_size else None
    rc = _lib.lib().sf_tm_grpo_advantage(h.ptr, _p(rewards), _p(group_ids), B, eps, std_mode,
                                         _p(adv), _p(gs), _stream(d))
    h.check(rc, "sf_tm_grpo_advantage")
    return (adv, gs) if want_group_size else adv


# ---------------------------------------------------------------------- a1
def logprob_fwd(logits: torch.Tensor, targets: torch.Tensor, inv_temperature: float = 1.0):
    d = _dev(logits)
    h = handle(d)
    dt, T, V, ld = _rows(logits)
    logp = torch.empty(T, dtype=torch.float32, device=logits.device)
    ent = torch.empty_like(logp)
    lse = torch.empty_like(logp)
    rc = _lib.lib().sf_tm_logprob_fwd(h.ptr, _p(logits), dt, T, V, ld, _p(targets), inv_temperature,
                                      _p(logp), _p(ent), _p(lse), _stream(d))
    h.check(rc, "sf_tm_logprob_fwd")
    return logp, ent, lse


# ---------------------------------------------------------------------- a4 prologue
def token_weights(cu_seqlens: torch.Tensor, adv_seq: torch.Tensor, mask: Optional[torch.Tensor], T: int,
                  norm_mode: int = _lib.NORM_TOKEN_MEAN, inv_norm: float = 0.0):
    d = _dev(cu_seqlens)
    h = handle(d)
    B = cu_seqlens.numel() - 1
    adv_tok = torch.empty(T, dtype=torch.float32, device=cu_seqlens.device)
    w_tok = torch.empty_like(adv_tok)
    rc = _lib.lib().sf_tm_token_weights(h.ptr, _p(cu_seqlens), B, _p(adv_seq), _p(mask), T, norm_mode,
                                        inv_norm, _p(adv_tok), _p(w_tok), _stream(d))
    h.check(rc, "sf_tm_token_weights")
    return adv_tok, w_tok


# ---------------------------------------------------------------------- a1+a4+a2
def pg_loss_fwd_bwd(logits, targets, old_logp, ref_logp, adv_tok, w_tok, params: Optional[LossParams] = None,
                    dlogits: Optional[torch.Tensor] = None, in_place: bool = False,
                    want_logp: bool = False, metrics: Optional[torch.Tensor] = None):
    d = _dev(logits)
    h = handle(d)
    dt, T, V, ld = _rows(logits)
    if params is None:
        params = default_loss_params()
    if in_place:
        dlogits = logits
    elif dlogits is None:
        dlogits = torch.empty_like(logits)
    if metrics is None:
        metrics = torch.empty(_lib.NUM_METRICS, dtype=torch.float32, device=logits.device)
    logp = torch.empty(T, dtype=torch.float32, device=logits.device) if want_logp else None
    ent = torch.empty(T, dtype=torch.float32, device=logits.device) if want_logp else None
    rc = _lib.lib().sf_tm_pg_loss_fwd_bwd(h.ptr, _p(logits), dt, T, V, ld, _p(targets), _p(old_logp),
                                          _p(ref_logp), _p(adv_tok), _p(w_tok), ctypes.byref(params),
                                          _p(dlogits), dlogits.stride(0), _p(metrics), _p(logp), _p(ent),
                                          _stream(d))
    h.check(rc, "sf_tm_pg_loss_fwd_bwd")
    return metrics, dlogits, logp, ent


def pg_step_host(logits, h_targets, h_old, h_ref, h_seq_lens, h_rewards, h_group_ids=None,
                 h_prompt_lens=None, h_mask=None, adv_eps: float = 1e-6, std_mode: int = _lib.STD_UNBIASED,
                 params: Optional[LossParams] = None, dlogits=None, h_metrics=None):
    """Trainer seam call with HOST (ideally pinned) per-token/per-sample buffers."""
    d = _dev(logits)
    h = handle(d)
    dt, T, V, ld = _rows(logits)
    if params is None:
        params = default_loss_params()
    if dlogits is None:
        dlogits = torch.empty_like(logits)
    if h_metrics is None:
        h_metrics = torch.empty(_lib.NUM_METRICS, dtype=torch.float32).pin_memory()
    for t in (h_targets, h_old, h_ref, h_seq_lens, h_rewards):
        if t.is_cuda:
            raise TrainMathError(_lib.CONFIG_ERROR, "pg_step_host takes host tensors")
    B = h_seq_lens.numel()
    rc = _lib.lib().sf_tm_pg_step_host(h.ptr, _p(logits), dt, T, V, ld, _p(h_targets), _p(h_old), _p(h_ref),
                                       _p(h_mask), _p(h_seq_lens), _p(h_prompt_lens), _p(h_rewards),
                                       _p(h_group_ids), B, adv_eps, std_mode, ctypes.byref(params),
                                       _p(dlogits), dlogits.stride(0), _p(h_metrics), _stream(d))
    h.check(rc, "sf_tm_pg_step_host")
    return h_metrics, dlogits


# ---------------------------------------------------------------------- a5
def r3_gate_fwd(router_logits, rec_idx, renorm: bool = True, want_idx: bool = True, want_mismatch: bool = True,
                out=None):
    """router_logits [L, T, E] (f32/bf16), rec_idx [L, T, k] (int32/uint8).
    out: optional preallocated (w, idx, mismatch) to reuse."""
    d = _dev(router_logits)
    h = handle(d)
    L, T, E = router_logits.shape
    k = rec_idx.shape[-1]
    dt = _DT[router_logits.dtype]
    it = _lib.IDX_U8 if rec_idx.dtype == torch.uint8 else _lib.IDX_I32
    if out is not None:
        w, idx, mm = out
    else:
        w = torch.empty(L, T, k, dtype=torch.float32, device=router_logits.device)
        idx = torch.empty(L, T, k, dtype=torch.int32, device=router_logits.device) if want_idx else None
        mm = torch.empty(L + 1, dtype=torch.int32, device=router_logits.device) if want_mismatch else None
    rc = _lib.lib().sf_tm_r3_gate_fwd(h.ptr, _p(router_logits.contiguous()), dt, L, T, E, k,
                                      _p(rec_idx.contiguous()), it, 1 if renorm else 0, _p(w), _p(idx), _p(mm),
                                      _stream(d))
    h.check(rc, "sf_tm_r3_gate_fwd")
    return w, idx, mm


def r3_gate_bwd(router_logits, rec_idx, w, dw, renorm: bool = True, out=None):
    d = _dev(router_logits)
    h = handle(d)
    L, T, E = router_logits.shape
    k = rec_idx.shape[-1]
    dt = _DT[router_logits.dtype]
    it = _lib.IDX_U8 if rec_idx.dtype == torch.uint8 else _lib.IDX_I32
    dz = torch.empty_like(router_logits) if out is None else out
    rc = _lib.lib().sf_tm_r3_gate_bwd(h.ptr, _p(router_logits), dt, L, T, E, k, _p(rec_idx), it,
                                      1 if renorm else 0, _p(w), _p(dw), _p(dz), _stream(d))
    h.check(rc, "sf_tm_r3_gate_bwd")
    return dz


def r3_record_layer_major(rec_token_major: torch.Tensor, out: Optional[torch.Tensor] = None):
    """routed_experts record [T, L, k] (token-major, as on the bus) -> the gate's
    layer-major [L, T, k], on the device, bit-exact."""
    d = _dev(rec_token_major)
    h = handle(d)
    T, L, k = rec_token_major.shape
    it = _lib.IDX_U8 if rec_token_major.dtype == torch.uint8 else _lib.IDX_I32
    src = rec_token_major.contiguous()
    if out is None:
        out = torch.empty(L, T, k, dtype=rec_token_major.dtype, device=rec_token_major.device)
    rc = _lib.lib().sf_tm_r3_record_layer_major(h.ptr, _p(src), it, T, L, k, _p(out), _stream(d))
    h.check(rc, "sf_tm_r3_record_layer_major")
    return out


# ---------------------------------------------------------------------- a7
def vp_partial_stats(shard, targets, vocab_start: int, inv_temperature: float = 1.0):
    d = _dev(shard)
    h = handle(d)
    dt, T, Vp, ld = _rows(shard)
    stats = torch.empty(T, 4, dtype=torch.float32, device=shard.device)
    rc = _lib.lib().sf_tm_vp_partial_stats(h.ptr, _p(shard), dt, T, Vp, ld, vocab_start, _p(targets),
                                           inv_temperature, _p(stats), _stream(d))
    h.check(rc, "sf_tm_vp_partial_stats")
    return stats


def vp_loss_fwd_bwd(shard, vocab_start: int, gathered_stats, targets, old_logp, ref_logp, adv_tok, w_tok,
                    params: Optional[LossParams] = None, dlogits=None, want_logp: bool = False, metrics=None):
    d = _dev(shard)
    h = handle(d)
    dt, T, Vp, ld = _rows(shard)
    P = gathered_stats.shape[0]
    if params is None:
        params = default_loss_params()
    if dlogits is None:
        dlogits = torch.empty_like(shard)
    if metrics is None:
        metrics = torch.empty(_lib.NUM_METRICS, dtype=torch.float32, device=shard.device)
    logp = torch.empty(T, dtype=torch.float32, device=shard.device) if want_logp else None
    ent = torch.empty(T, dtype=torch.float32, device=shard.device) if want_logp else None
    rc = _lib.lib().sf_tm_vp_loss_fwd_bwd(h.ptr, _p(shard), dt, T, Vp, ld, vocab_start, _p(gathered_stats), P,
                                          _p(targets), _p(old_logp), _p(ref_logp), _p(adv_tok), _p(w_tok),
                                          ctypes.byref(params), _p(dlogits), dlogits.stride(0), _p(metrics),
                                          _p(logp), _p(ent), _stream(d))
    h.check(rc, "sf_tm_vp_loss_fwd_bwd")
    return metrics, dlogits, logp, ent


def vp_mailbox_create(P: int, rank: int, device: Optional[int] = None) -> bytes:
    """Allocate this rank's peer mailbox; returns its 64-byte CUDA IPC handle."""
    h = handle(device)
    buf = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
    h.check(_lib.lib().sf_tm_vp_mailbox_create(h.ptr, P, rank, buf), "sf_tm_vp_mailbox_create")
    return buf.raw


def vp_mailbox_open(handles: list, device: Optional[int] = None):
    """Map the peers' mailboxes (handles: every rank's 64-byte handle, rank order)."""
    h = handle(device)
    blob = b"".join(handles)
    buf = ctypes.create_string_buffer(blob, len(blob))
    h.check(_lib.lib().sf_tm_vp_mailbox_open(h.ptr, buf), "sf_tm_vp_mailbox_open")


def vp_fused_check(shard, dlogits=None) -> tuple[int, str]:
    """sf_tm_vp_fused_check: (Errc, message) for this rank's shard, no side effect."""
    d = _dev(shard)
    h = handle(d)
    dt, T, Vp, ld = _rows(shard)
    ld_d = ld if dlogits is None else dlogits.stride(0)
    ptr = _p(shard) if dlogits is None else _p(dlogits)
    rc = _lib.lib().sf_tm_vp_fused_check(h.ptr, _p(shard), dt, T, Vp, ld, ptr, ld_d)
    msg = _lib.lib().sf_tm_last_error(h.ptr) if rc else b""
    return int(rc), (msg.decode() if msg else "")


def vp_local_group(handles: list, grid_per_rank: int = 0):
    """Wire P handles of one device into an in-process vocab-parallel group
    (sf_tm_debug_vp_local_group): P ranks emulated on one GPU."""
    arr = (_lib._H * len(handles))(*[hh.ptr.value for hh in handles])
    rc = _lib.lib().sf_tm_debug_vp_local_group(arr, len(handles), grid_per_rank)
    if rc != 0:
        raise TrainMathError(rc, "sf_tm_debug_vp_local_group failed")


def vp_fused_loss_fwd_bwd(shard, vocab_start: int, targets, old_logp, ref_logp, adv_tok, w_tok,
                          params: Optional[LossParams] = None, dlogits=None, want_logp: bool = False, metrics=None,
                          h: Optional[Handle] = None, stream=None):
    """Single-pass vocab-parallel loss: the exchange happens inside the kernel.
    `h`: the rank's Handle (default: the device's shared handle; emulated
    in-process groups pass their own)."""
    d = _dev(shard)
    h = handle(d) if h is None else h
    dt, T, Vp, ld = _rows(shard)
    if params is None:
        params = default_loss_params()
    if dlogits is None:
        dlogits = torch.empty_like(shard)
    if metrics is None:
        metrics = torch.empty(_lib.NUM_METRICS, dtype=torch.float32, device=shard.device)
    logp = torch.empty(T, dtype=torch.float32, device=shard.device) if want_logp else None
    ent = torch.empty(T, dtype=torch.float32, device=shard.device) if want_logp else None
    rc = _lib.lib().sf_tm_vp_fused_loss_fwd_bwd(h.ptr, _p(shard), dt, T, Vp, ld, vocab_start, _p(targets),
                                                _p(old_logp), _p(ref_logp), _p(adv_tok), _p(w_tok),
                                                ctypes.byref(params), _p(dlogits), dlogits.stride(0), _p(metrics),
                                                _p(logp), _p(ent),
                                                _stream(d) if stream is None else ctypes.c_void_p(stream.cuda_stream))
    h.check(rc, "sf_tm_vp_fused_loss_fwd_bwd")
    return metrics, dlogits, logp, ent


# ---------------------------------------------------------------------- synthetic inputs
def synth_logits(logits: torch.Tensor, seed: int, sigma: float = 2.0, peak_id=None, peak_lo: float = 5.0,
                 peak_hi: float = 25.0, outlier_frac: float = 1e-3):
    d = _dev(logits)
    h = handle(d)
    dt, T, V, ld = _rows(logits)
    rc = _lib.lib().sf_tm_synth_logits(h.ptr, _p(logits), dt, T, V, ld, seed & 0xFFFFFFFFFFFFFFFF, sigma,
                                       _p(peak_id), peak_lo, peak_hi, outlier_frac, _stream(d))
    h.check(rc, "sf_tm_synth_logits")
    return logits
