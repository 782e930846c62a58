# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE — ctypes/numpy front-end of the fp64 CPU oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or as the timed
CPU baseline. It never backs a product call.

Parity status (see sf_oracle.h and DESIGN.md §3): math parity unpinned against
the reference — the reference has no code for this math, so the oracle
restates the published algorithms with the P1-P9 decisions; it is pinned by hand-derived known answers and by golden vectors
from an independent torch-float64 autograd implementation
(tests/golden/make_golden.py). The seeded RNG and digest helpers are pinned
bit-exactly against the reference's own rng.cpp / hash.hpp (oracle/_ref).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libsf_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libsfref.so")

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_d = ctypes.c_double
_u64 = ctypes.c_uint64


class OrcParams(ctypes.Structure):
    _fields_ = [("eps_lo", _d), ("eps_hi", _d), ("dual_c", _d), ("beta", _d), ("ent_coef", _d), ("inv_tau", _d),
                ("kl_mode", ctypes.c_int32)]


_lib = None
_ref = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        l = ctypes.CDLL(LIB_PATH)
        sig = {
            "orc_set_threads": (None, [_i32]),
            "orc_get_threads": (_i32, []),
            "orc_logprob_fwd": (_i32, [_vp, _i32, _i64, _i64, _i64, _vp, _d, _vp, _vp, _vp]),
            "orc_varlen_meta": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
            "orc_grpo_advantage": (_i32, [_vp, _vp, _i64, _d, _i32, _vp, _vp]),
            "orc_token_weights": (_i32, [_vp, _i64, _vp, _vp, _i64, _i32, _d, _vp, _vp]),
            "orc_pg_loss_fwd_bwd": (_i32, [_vp, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp,
                                           ctypes.POINTER(OrcParams), _i32, _vp, _i32, _vp, _vp, _vp, _vp]),
            "orc_pg_loss_fwd_bwd_fast": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp,
                                                ctypes.POINTER(OrcParams), _vp, _vp]),
            "orc_r3_gate_fwd": (_i32, [_vp, _i32, _i64, _i64, _i64, _i64, _vp, _i32, _i32, _vp, _vp, _vp]),
            "orc_r3_gate_bwd": (_i32, [_vp, _i32, _i64, _i64, _i64, _i64, _vp, _i32, _i32, _vp, _vp, _vp]),
            "orc_vp_partial_stats": (_i32, [_vp, _i32, _i64, _i64, _i64, _i64, _vp, _d, _vp]),
            "orc_splitmix_at": (_u64, [_u64, _u64]),
            "orc_derive_seed": (_u64, [_u64, ctypes.c_char_p, _u64, _u64]),
            "orc_fnv1a64": (_u64, [_vp, _u64]),
            "orc_f64_to_bf16": (ctypes.c_uint16, [_d]),
            "orc_bf16_to_f64": (_d, [ctypes.c_uint16]),
        }
        for n, (r, a) in sig.items():
            f = getattr(l, n)
            f.restype = r
            f.argtypes = a
        _lib = l
    return _lib


def ref_lib():
    """The reference's own rng.cpp/hash.hpp (oracle/_ref), or None if not built."""
    global _ref
    if _ref is None and os.path.exists(REF_PATH):
        l = ctypes.CDLL(REF_PATH)
        l.sfref_splitmix_seq.argtypes = [_u64, _u64, _vp]
        l.sfref_splitmix_seq.restype = None
        l.sfref_derive_seed.argtypes = [_u64, ctypes.c_char_p, _u64, _u64]
        l.sfref_derive_seed.restype = _u64
        l.sfref_fnv1a64.argtypes = [_vp, _u64]
        l.sfref_fnv1a64.restype = _u64
        l.sfref_inverse_normal_cdf.argtypes = [_d]
        l.sfref_inverse_normal_cdf.restype = _d
        _ref = l
    return _ref


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return 0
    if a.dtype == np.uint16:  # raw bf16 bits
        return 1
    if a.dtype == np.float64:
        return 2
    raise TypeError(a.dtype)


def set_threads(n: int):
    lib().orc_set_threads(n)


def threads() -> int:
    return lib().orc_get_threads()


# ---------------------------------------------------------------- bf16 (numpy)
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bits (same as cvt.rn.bf16.f32)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    r = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    out = r.astype(np.uint16)
    nan = np.isnan(x)
    out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(u: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(u, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def to_f64(logits: np.ndarray) -> np.ndarray:
    if logits.dtype == np.uint16:
        return bf16_bits_to_f32(logits).astype(np.float64)
    return logits.astype(np.float64)


# ---------------------------------------------------------------- wrappers
def logprob_fwd(logits: np.ndarray, targets: np.ndarray, inv_tau: float = 1.0):
    logits = np.ascontiguousarray(logits)
    T, V = logits.shape
    t = np.ascontiguousarray(targets, dtype=np.int32)
    logp, ent, lse = (np.empty(T) for _ in range(3))
    lib().orc_logprob_fwd(_ptr(logits), _dtype_code(logits), T, V, V, _ptr(t), inv_tau, _ptr(logp), _ptr(ent), _ptr(lse))
    return logp, ent, lse


def varlen_meta(lens, plens=None, gids=None):
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    B = lens.size
    T = int(lens.sum())
    cu = np.empty(B + 1, np.int32)
    sid = np.empty(T, np.int32)
    mask = np.empty(T, np.uint8)
    tg = np.empty(T, np.int32)
    pl = None if plens is None else np.ascontiguousarray(plens, dtype=np.int32)
    g = None if gids is None else np.ascontiguousarray(gids, dtype=np.int32)
    lib().orc_varlen_meta(_ptr(lens), _ptr(pl), _ptr(g), B, _ptr(cu), _ptr(sid), _ptr(mask), _ptr(tg))
    return cu, sid, mask, tg


def grpo_advantage(rewards, gids, eps=1e-6, std_mode=0):
    r = np.ascontiguousarray(rewards, dtype=np.float32)
    g = np.ascontiguousarray(gids, dtype=np.int32)
    B = r.size
    adv = np.empty(B)
    gs = np.empty(B, np.int32)
    lib().orc_grpo_advantage(_ptr(r), _ptr(g), B, eps, std_mode, _ptr(adv), _ptr(gs))
    return adv, gs


def token_weights(cu, adv_seq, mask, T, norm_mode=0, inv_norm=0.0):
    cu = np.ascontiguousarray(cu, dtype=np.int32)
    B = cu.size - 1
    a = None if adv_seq is None else np.ascontiguousarray(adv_seq, dtype=np.float32)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    adv_tok = np.empty(T)
    w_tok = np.empty(T)
    lib().orc_token_weights(_ptr(cu), B, _ptr(a), _ptr(m), T, norm_mode, inv_norm, _ptr(adv_tok), _ptr(w_tok))
    return adv_tok, w_tok


def params(eps_lo=0.2, eps_hi=0.28, dual_c=0.0, beta=0.0, ent_coef=0.0, inv_tau=1.0, kl_mode=0) -> OrcParams:
    return OrcParams(eps_lo, eps_hi, dual_c, beta, ent_coef, inv_tau, kl_mode)


def pg_loss_fwd_bwd(logits, targets, old, ref, adv_tok, w_tok, p: OrcParams = None, masked_skip=False,
                    want_dlogits=True, dl_dtype=2):
    """dl_dtype: 0 f32, 1 bf16 bits, 2 f64. Returns metrics, dlogits, logp, ent, g."""
    if p is None:
        p = params()
    logits = np.ascontiguousarray(logits)
    T, V = logits.shape
    args = [np.ascontiguousarray(a, dtype=dt) for a, dt in
            ((targets, np.int32), (old, np.float32), (ref, np.float32), (adv_tok, np.float32), (w_tok, np.float32))]
    dl = None
    if want_dlogits:
        dl = np.empty((T, V), dtype={0: np.float32, 1: np.uint16, 2: np.float64}[dl_dtype])
    logp = np.empty(T)
    ent = np.empty(T)
    g = np.empty(T)
    met = np.empty(8)
    lib().orc_pg_loss_fwd_bwd(_ptr(logits), _dtype_code(logits), T, V, V, *[_ptr(a) for a in args], ctypes.byref(p),
                              1 if masked_skip else 0, _ptr(dl), dl_dtype, _ptr(logp), _ptr(ent), _ptr(met), _ptr(g))
    return met, dl, logp, ent, g


def pg_loss_fwd_bwd_fast(logits_bits, targets, old, ref, adv_tok, w_tok, p: OrcParams = None):
    """The timed CPU baseline (sf_cpu_fast.c): bf16 bits in, bf16 bits out, fp32
    arithmetic. Returns (metrics, dlogits_bits)."""
    if p is None:
        p = params()
    x = np.ascontiguousarray(logits_bits, dtype=np.uint16)
    T, V = x.shape
    args = [np.ascontiguousarray(a, dtype=dt) for a, dt in
            ((targets, np.int32), (old, np.float32), (ref, np.float32), (adv_tok, np.float32), (w_tok, np.float32))]
    dl = np.empty((T, V), np.uint16)
    met = np.empty(8)
    lib().orc_pg_loss_fwd_bwd_fast(_ptr(x), T, V, V, *[_ptr(a) for a in args], ctypes.byref(p), _ptr(dl), _ptr(met))
    return met, dl


def r3_gate_fwd(logits, rec, renorm=True):
    """logits [L,T,E] f32 or bf16 bits, rec [L,T,k] int32/uint8."""
    logits = np.ascontiguousarray(logits)
    rec = np.ascontiguousarray(rec)
    L, T, E = logits.shape
    k = rec.shape[-1]
    w = np.empty((L, T, k))
    idx = np.empty((L, T, k), np.int32)
    mm = np.empty(L + 1, np.uint32)
    lib().orc_r3_gate_fwd(_ptr(logits), _dtype_code(logits), L, T, E, k, _ptr(rec), 1 if rec.dtype == np.uint8 else 0,
                          1 if renorm else 0, _ptr(w), _ptr(idx), _ptr(mm))
    return w, idx, mm


def r3_gate_bwd(logits, rec, w, dw, renorm=True):
    logits = np.ascontiguousarray(logits)
    rec = np.ascontiguousarray(rec)
    L, T, E = logits.shape
    k = rec.shape[-1]
    w = np.ascontiguousarray(w, dtype=np.float32)
    dw = np.ascontiguousarray(dw, dtype=np.float32)
    dz = np.empty((L, T, E))
    lib().orc_r3_gate_bwd(_ptr(logits), _dtype_code(logits), L, T, E, k, _ptr(rec), 1 if rec.dtype == np.uint8 else 0,
                          1 if renorm else 0, _ptr(w), _ptr(dw), _ptr(dz))
    return dz


def vp_partial_stats(shard, targets, vocab_start, inv_tau=1.0):
    shard = np.ascontiguousarray(shard)
    T, Vp = shard.shape
    t = np.ascontiguousarray(targets, dtype=np.int32)
    st = np.empty((T, 4))
    lib().orc_vp_partial_stats(_ptr(shard), _dtype_code(shard), T, Vp, Vp, vocab_start, _ptr(t), inv_tau, _ptr(st))
    return st


def splitmix_at(seed: int, i: int) -> int:
    return int(lib().orc_splitmix_at(seed & (2**64 - 1), i))


def derive_seed(seed: int, tag: str, idx: int = 0) -> int:
    b = tag.encode()
    return int(lib().orc_derive_seed(seed & (2**64 - 1), b, len(b), idx & (2**64 - 1)))


def fnv1a64(data: bytes) -> int:
    buf = np.frombuffer(data, dtype=np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
    return int(lib().orc_fnv1a64(_ptr(buf), len(data)))


def digest(a: np.ndarray) -> int:
    """FNV-1a64 of an array's bytes (hash.hpp:14-31) — used for bit-exact checks."""
    return fnv1a64(np.ascontiguousarray(a).tobytes())


# ---------------------------------------------------------------- seeded inputs
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix_vec(seed: int, idx: np.ndarray) -> np.ndarray:
    """Vectorised i-th SplitMix64 outputs: mix64(seed + (i+1)*gamma) (rng.hpp:21-26)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & (2**64 - 1)) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """(0,1) doubles from the reference generator's stream (53-bit, rng.hpp:29-36)."""
    u = (splitmix_vec(seed, np.arange(offset, offset + n)) >> np.uint64(11)).astype(np.float64) * 2.0**-53
    u[u == 0.0] = 2.0**-53
    return u


def normal(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """Standard normals by Box-Muller over the reference stream."""
    u1 = uniform(seed, n, offset)
    u2 = uniform(seed ^ 0x5DEECE66D, n, offset)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2 * np.pi * u2)


def synth_problem(seed: int, lens, V: int, dtype: str = "bf16", prompt_max: int = 64, sigma: float = 2.0,
                  G: int = 8, outlier_frac: float = 1e-3):
    """A seeded packed micro-batch (SURVEY.md §8d 'Synthetic inputs'), CPU-generated.

    Returns dict with logits (f32 or bf16 bits), targets, old/ref logp (derived
    from the fp64 oracle logp + noise), rewards, group ids, prompt lens.
    """
    lens = np.asarray(lens, dtype=np.int32)
    B = lens.size
    T = int(lens.sum())
    s = derive_seed(seed, "logits")
    x = normal(s, T * V).reshape(T, V) * sigma
    peak = (splitmix_vec(derive_seed(seed, "peak"), np.arange(T)) % np.uint64(V)).astype(np.int64)
    amp = 5.0 + 20.0 * uniform(derive_seed(seed, "peak_amp"), T)
    x[np.arange(T), peak] += amp
    if outlier_frac > 0:
        u = uniform(derive_seed(seed, "outlier"), T * V).reshape(T, V)
        sgn = np.where(uniform(derive_seed(seed, "outlier_sign"), T * V).reshape(T, V) < 0.5, -30.0, 30.0)
        x = np.where(u < outlier_frac, sgn, x)
    x32 = x.astype(np.float32)
    logits = f32_to_bf16_bits(x32) if dtype == "bf16" else x32
    coin = uniform(derive_seed(seed, "target_coin"), T) < 0.5
    rnd = (splitmix_vec(derive_seed(seed, "target"), np.arange(T)) % np.uint64(V)).astype(np.int64)
    targets = np.where(coin, peak, rnd).astype(np.int32)
    logp, _, _ = logprob_fwd(logits, targets)
    old = (logp + 0.05 * normal(derive_seed(seed, "old"), T)).astype(np.float32)
    ref = (logp + 0.1 * normal(derive_seed(seed, "ref"), T)).astype(np.float32)
    rewards = (uniform(derive_seed(seed, "reward"), B) < 0.5).astype(np.float32)
    gids = (np.arange(B) // G).astype(np.int32)
    plens = np.minimum((splitmix_vec(derive_seed(seed, "prompt"), np.arange(B)) % np.uint64(prompt_max + 1)).astype(np.int32),
                       lens)
    return dict(logits=logits, targets=targets, old=old, ref=ref, rewards=rewards, gids=gids, lens=lens,
                plens=plens, T=T, V=V, B=B, dtype=dtype)
