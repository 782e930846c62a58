# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of the C-ABI in include/staleflow/train_math.h.

The shared library is built in-tree (paper_2604_11554_b200/lib/libsf_train_math.so,
see csrc/Makefile and __graft_entry__.build). There is no fallback: if the
library is missing, importing a compute entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libsf_train_math.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "staleflow", "train_math.h")

# staleflow::Errc values (proj/include/staleflow/result.hpp:14-47)
OK = 0
CONFIG_ERROR = 21
INTERNAL = 26
ERRC_NAMES = {OK: "Ok", CONFIG_ERROR: "ConfigError", INTERNAL: "Internal"}

F32 = 0
BF16 = 1
IDX_I32 = 0
IDX_U8 = 1
STD_UNBIASED, STD_POPULATION, STD_NONE = 0, 1, 2
NORM_TOKEN_MEAN, NORM_SEQ_MEAN, NORM_EXPLICIT = 0, 1, 2
MASKED_ZERO_FILL, MASKED_SKIP = 0, 1
METRIC_NAMES = ["loss", "pg_loss", "kl", "entropy", "clipfrac", "ratio", "n_active", "ppo_kl"]
NUM_METRICS = 8


class TrainMathError(RuntimeError):
    """A non-Ok staleflow::Errc returned through the C-ABI."""

    def __init__(self, code: int, message: str):
        self.code = code
        super().__init__(f"{ERRC_NAMES.get(code, code)} ({code}): {message}")


class LossParams(ctypes.Structure):
    _fields_ = [
        ("clip_eps_low", ctypes.c_float),
        ("clip_eps_high", ctypes.c_float),
        ("dual_clip_c", ctypes.c_float),
        ("kl_beta", ctypes.c_float),
        ("entropy_coef", ctypes.c_float),
        ("inv_temperature", ctypes.c_float),
        ("norm_mode", ctypes.c_int32),
        ("inv_norm", ctypes.c_float),
        ("masked_rows", ctypes.c_int32),
        ("kl_mode", ctypes.c_int32),
    ]


IPC_HANDLE_BYTES = 64  # SF_TM_IPC_HANDLE_BYTES
KL_K3, KL_K1, KL_K2, KL_ABS = 0, 1, 2, 3  # SF_TM_KL_*

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f32 = ctypes.c_float
_u64 = ctypes.c_uint64
_H = ctypes.c_void_p  # sf_tm_t

_SIGS = {
    "sf_tm_default_loss_params": (None, [ctypes.POINTER(LossParams)]),
    "sf_tm_abi_version": (ctypes.c_int, []),
    "sf_tm_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_H)]),
    "sf_tm_destroy": (ctypes.c_int, [_H]),
    "sf_tm_last_error": (ctypes.c_char_p, [_H]),
    "sf_tm_launch_count": (_u64, [_H]),
    "sf_tm_last_launch": (_i32, [_H, _vp, _vp, _vp]),
    "sf_tm_last_launch_streams": (_i32, [_H, _vp]),
    "sf_tm_varlen_meta": (ctypes.c_int, [_H, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "sf_tm_grpo_advantage": (ctypes.c_int, [_H, _vp, _vp, _i64, _f32, _i32, _vp, _vp, _vp]),
    "sf_tm_logprob_fwd": (ctypes.c_int, [_H, _vp, _i32, _i64, _i64, _i64, _vp, _f32, _vp, _vp, _vp, _vp]),
    "sf_tm_token_weights": (ctypes.c_int, [_H, _vp, _i64, _vp, _vp, _i64, _i32, _f32, _vp, _vp, _vp]),
    "sf_tm_pg_loss_fwd_bwd": (
        ctypes.c_int,
        [_H, _vp, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(LossParams), _vp, _i64, _vp, _vp, _vp, _vp],
    ),
    "sf_tm_pg_step_host": (
        ctypes.c_int,
        [_H, _vp, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _f32, _i32,
         ctypes.POINTER(LossParams), _vp, _i64, _vp, _vp],
    ),
    "sf_tm_r3_gate_fwd": (ctypes.c_int, [_H, _vp, _i32, _i64, _i64, _i64, _i64, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "sf_tm_r3_gate_bwd": (ctypes.c_int, [_H, _vp, _i32, _i64, _i64, _i64, _i64, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "sf_tm_r3_record_layer_major": (ctypes.c_int, [_H, _vp, _i32, _i64, _i64, _i64, _vp, _vp]),
    "sf_tm_vp_partial_stats": (ctypes.c_int, [_H, _vp, _i32, _i64, _i64, _i64, _i64, _vp, _f32, _vp, _vp]),
    "sf_tm_vp_loss_fwd_bwd": (
        ctypes.c_int,
        [_H, _vp, _i32, _i64, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _vp, _vp, _vp,
         ctypes.POINTER(LossParams), _vp, _i64, _vp, _vp, _vp, _vp],
    ),
    "sf_tm_sync": (ctypes.c_int, [_H, _vp]),
    "sf_tm_wait_host_inputs": (ctypes.c_int, [_H]),
    "sf_tm_logprob_fwd_host": (ctypes.c_int, [_H, _vp, _i32, _i64, _i64, _i64, _vp, _f32, _vp, _vp, _vp]),
    "sf_tm_grpo_advantage_host": (ctypes.c_int, [_H, _vp, _vp, _i64, _f32, _i32, _vp, _vp]),
    "sf_tm_vp_mailbox_create": (ctypes.c_int, [_H, _i32, _i32, _vp]),
    "sf_tm_vp_mailbox_open": (ctypes.c_int, [_H, _vp]),
    "sf_tm_vp_fused_loss_fwd_bwd": (
        ctypes.c_int,
        [_H, _vp, _i32, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp,
         ctypes.POINTER(LossParams), _vp, _i64, _vp, _vp, _vp, _vp],
    ),
    "sf_tm_vp_fused_check": (ctypes.c_int, [_H, _vp, _i32, _i64, _i64, _i64, _vp, _i64]),
    "sf_tm_debug_vp_local_group": (ctypes.c_int, [ctypes.POINTER(_H), _i32, _i32]),
    "sf_tm_synth_logits": (ctypes.c_int, [_H, _vp, _i32, _i64, _i64, _i64, _u64, _f32, _vp, _f32, _f32, _f32, _vp]),
    "sf_tm_host_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(_vp)]),
    "sf_tm_host_free": (ctypes.c_int, [_vp]),
    "sf_tm_h2d": (ctypes.c_int, [_H, _vp, _vp, ctypes.c_size_t, _vp]),
    "sf_tm_debug_force_generic": (ctypes.c_int, [ctypes.c_int]),
    "sf_tm_debug_wait_counters": (ctypes.c_int, [_vp]),
}

_lib = None


def header_functions(path: str = HEADER_PATH) -> list[str]:
    """Names of every function declared in include/staleflow/train_math.h."""
    src = open(path).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sf_tm_[a-z0-9_]+)\s*\(", src)))


def lib() -> ctypes.CDLL:
    """Load libsf_train_math.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA extension is not built "
                "(run `python -c 'import __graft_entry__ as g; g.build()'` or `make -C paper_2604_11554_b200/csrc`)"
            )
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def default_loss_params(**kw) -> LossParams:
    p = LossParams()
    lib().sf_tm_default_loss_params(ctypes.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise TypeError(f"unknown loss param {k}")
        setattr(p, k, v)
    return p
