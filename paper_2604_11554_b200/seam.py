# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of include/staleflow/train_math_seam_c.h: the C++ trainer seam
(ActorLossSeam, include/staleflow/train_math_seam.hpp) on one MicroBatch in its
bus encoding. The bench's end-to-end leg times sf_seam_step — payload decode,
pinned staging, H2D, GRPO/weights, fused loss fwd+bwd, D2H metrics — which is
the call the reference's trainer seam (proj/src/sim_runtime.cpp:441,
proj/src/wall_runtime.cpp:197) makes per micro-batch."""
from __future__ import annotations

import ctypes
import os
import re
from typing import Optional

import numpy as np
import torch

from . import _lib

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libsf_seam.so")
HEADER_PATH = os.path.join(os.path.dirname(_lib.HEADER_PATH), "train_math_seam_c.h")

_vp, _i32, _i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_SIGS = {
    "sf_seam_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "sf_seam_destroy": (ctypes.c_int, [_vp]),
    "sf_seam_last_error": (ctypes.c_char_p, [_vp]),
    "sf_seam_batch_build": (ctypes.c_int, [_i64, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "sf_seam_batch_free": (ctypes.c_int, [_vp]),
    "sf_seam_batch_staleness": (ctypes.c_int, [_vp, _i64, ctypes.POINTER(_i64), _vp, _i32]),
    "sf_seam_step": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i64, _vp, ctypes.POINTER(_lib.LossParams), _vp, _vp, _i32]),
}
_l = None


def header_functions() -> list[str]:
    src = re.sub(r"/\*.*?\*/", "", open(HEADER_PATH).read(), flags=re.S)
    return sorted(set(re.findall(r"\b(sf_seam_[a-z0-9_]+)\s*\(", src)))


def lib() -> ctypes.CDLL:
    global _l
    if _l is None:
        _lib.lib()  # libsf_train_math.so first (the seam library links it)
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing (make -C paper_2604_11554_b200/csrc)")
        l = ctypes.CDLL(LIB_PATH)
        for n, (r, a) in _SIGS.items():
            f = getattr(l, n)
            f.restype, f.argtypes = r, a
        _l = l
    return _l


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class MicroBatch:
    """One trainer MicroBatch with payloads (the bus encoding, built once)."""

    def __init__(self, seq_lens, targets, logp, ref_logp, per_sample, has_advantage: bool,
                 loss_mask=None, sample_ids=None, producer_versions=None):
        c = lambda a, dt: None if a is None else np.ascontiguousarray(a, dtype=dt)
        self._keep = [c(seq_lens, np.int32), c(targets, np.int32), c(logp, np.float32), c(ref_logp, np.float32),
                      c(per_sample, np.float32), c(loss_mask, np.uint8)]
        B = len(self._keep[0])
        ids = c(sample_ids if sample_ids is not None else np.arange(1, B + 1), np.uint64)
        pv = c(producer_versions, np.int64)
        self._keep += [ids, pv]
        self.T = int(self._keep[0].sum())
        self.B = B
        self._b = _vp()
        rc = lib().sf_seam_batch_build(B, *[_ptr(a) for a in self._keep[:5]], 1 if has_advantage else 0,
                                       _ptr(self._keep[5]), _ptr(ids), _ptr(pv), ctypes.byref(self._b))
        if rc:
            raise _lib.TrainMathError(rc, "sf_seam_batch_build failed")

    def staleness(self, v_trainer: int, hist: np.ndarray) -> int:
        """Adds this batch's per-sample staleness counts into hist (uint64[n]);
        returns the batch staleness v_trainer - min producer version."""
        assert hist.dtype == np.uint64 and hist.flags.c_contiguous
        bs = _i64()
        rc = lib().sf_seam_batch_staleness(self._b, v_trainer, ctypes.byref(bs), _ptr(hist), len(hist))
        if rc:
            raise _lib.TrainMathError(rc, "sf_seam_batch_staleness failed")
        return int(bs.value)

    def __del__(self):
        try:
            if self._b:
                lib().sf_seam_batch_free(self._b)
        except Exception:
            pass


class ActorLossSeam:
    """The Actor role's trainer seam (C++ ActorLossSeam) on device `device`."""

    def __init__(self, device: int = 0):
        self._s = _vp()
        rc = lib().sf_seam_create(device, ctypes.byref(self._s))
        if rc:
            raise _lib.TrainMathError(rc, f"sf_seam_create(device={device}) failed")

    def step(self, batch: MicroBatch, logits: torch.Tensor, dlogits: torch.Tensor, params, h_metrics: torch.Tensor,
             group_size: int = 0):
        dt = _lib.BF16 if logits.dtype == torch.bfloat16 else _lib.F32
        rc = lib().sf_seam_step(self._s, batch._b, ctypes.c_void_p(logits.data_ptr()), dt, logits.shape[1],
                                ctypes.c_void_p(dlogits.data_ptr()), ctypes.byref(params),
                                ctypes.c_void_p(h_metrics.data_ptr()),
                                ctypes.c_void_p(torch.cuda.current_stream(logits.device).cuda_stream), group_size)
        if rc:
            msg = lib().sf_seam_last_error(self._s)
            raise _lib.TrainMathError(rc, f"sf_seam_step: {msg.decode() if msg else ''}")

    def __del__(self):
        try:
            if self._s:
                lib().sf_seam_destroy(self._s)
        except Exception:
            pass
