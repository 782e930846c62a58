# SPDX-License-Identifier: Apache-2.0
"""Comparison helpers with the tolerances of DESIGN.md §3 written out."""
import numpy as np

# logp / entropy / lse / loss vs the fp64 oracle: |d| <= ATOL + RTOL*|ref|
ATOL = 1e-5
RTOL = 1e-5


def assert_close(got, ref, atol=ATOL, rtol=RTOL, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(got - ref)
    lim = atol + rtol * np.abs(ref)
    bad = ~(err <= lim)
    if bad.any():
        i = np.flatnonzero(bad.ravel())[:5]
        raise AssertionError(f"{what}: {bad.sum()} / {bad.size} out of tolerance; e.g. idx {i} got "
                             f"{got.ravel()[i]} ref {ref.ravel()[i]} (atol {atol}, rtol {rtol})")


def bf16_ulp(v: np.ndarray) -> np.ndarray:
    """Spacing of the bf16 grid at |v| (8 significant bits)."""
    a = np.abs(v)
    e = np.floor(np.log2(np.maximum(a, 1e-38)))
    return np.exp2(e - 7)


def assert_grad_close(got, ref, row_scale, dtype, what="dlogits", rows_ok=None):
    """dlogits: bf16 -> within 1 bf16 ulp of the exact value (plus a row-scale
    floor for cancellation at the target entry); f32 -> rel 1e-5.
    row_scale[t] ~ |dL/dlogp_t| * inv_tau (+ entropy term scale)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    floor = 4e-6 * np.asarray(row_scale, dtype=np.float64)[:, None] + 1e-30
    if dtype == "bf16":
        lim = bf16_ulp(ref) + floor
    else:
        lim = 1e-5 * np.abs(ref) + floor
    bad = ~(np.abs(got - ref) <= lim)
    if rows_ok is not None:
        bad &= rows_ok[:, None]
    if bad.any():
        r, c = np.nonzero(bad)
        raise AssertionError(f"{what}: {bad.sum()} entries out of tolerance in rows {np.unique(r)[:8]}; "
                             f"e.g. ({r[0]},{c[0]}) got {got[r[0], c[0]]!r} ref {ref[r[0], c[0]]!r}")


def near_clip_rows(logp_ref, old, adv, eps_lo, eps_hi, dual_c=0.0, tol=1e-5):
    """Rows whose ratio sits within tol of a clip decision boundary, where an
    fp32 kernel and the fp64 oracle may legitimately take different branches."""
    r = np.exp(np.asarray(logp_ref) - np.asarray(old, dtype=np.float64))
    a = np.asarray(adv, dtype=np.float64)
    near = (np.abs(r - (1 + eps_hi)) < tol * (1 + eps_hi)) | (np.abs(r - (1 - eps_lo)) < tol)
    if dual_c > 1:
        near |= (a < 0) & (np.abs(r - dual_c) < tol * dual_c)
    return near


def loss_row_scale(og, w, a, olp, old, ref, beta=0.0, kl_mode=0, ent=0.0, inv_tau=1.0):
    """Per-row gradient magnitude before cancellation: |g| can be far smaller than
    the policy and KL terms it is the sum of (fp32 error follows the terms)."""
    w = np.abs(np.asarray(w, np.float64))
    ratio = np.exp(np.asarray(olp, np.float64) - np.asarray(old, np.float64))
    d = np.asarray(ref, np.float64) - np.asarray(olp, np.float64)
    # k3's derivative 1 - e^d is a difference of two O(1) terms: an fp32 logp
    # error eps moves it by ~eps * e^d however small |1 - e^d| is
    dkl = {0: 1 + np.exp(np.minimum(d, 80)), 1: np.ones_like(d), 2: np.abs(d), 3: np.ones_like(d)}[kl_mode]
    terms = np.abs(np.asarray(a, np.float64)) * ratio + abs(beta) * dkl
    return (np.abs(og) + w * terms + w * abs(ent) * 60.0) * inv_tau


def metrics_from_rows(logp, ent, old, ref, adv, w, eps_lo=0.2, eps_hi=0.28, dual_c=0.0, beta=0.0, ent_coef=0.0,
                      kl_mode=0):
    """The step metrics [loss, pg, kl, entropy, clipfrac, ratio, n_active, ppo_kl]
    as fp64 sums over rows, from per-row logp / entropy: a numpy restatement of
    the per-row terms of orc_pg_loss_fwd_bwd (oracle/sf_oracle.c), pinned
    against it in tests/test_oracle.py. Lets a full-size GPU run check its
    reduction from its own per-row outputs when the oracle cannot hold every
    row."""
    f = lambda a: np.asarray(a, np.float64)
    lp, H, o, r, A, w = f(logp), f(ent), f(old), f(ref), f(adv), f(w)
    act = w != 0
    lp, H, o, r, A, w = lp[act], H[act], o[act], r[act], A[act], w[act]
    ratio = np.exp(lp - o)
    clip_hi = (A > 0) & (ratio > 1 + eps_hi)
    clip_lo = (A < 0) & (ratio < 1 - eps_lo)
    rc = np.clip(ratio, 1 - eps_lo, 1 + eps_hi)
    pg = np.maximum(-ratio * A, -rc * A)
    clipped = clip_hi | clip_lo
    if dual_c > 1:
        cap = -dual_c * A
        dc = (A < 0) & (pg > cap)
        pg = np.where(dc, cap, pg)
        clipped |= dc
    d = r - lp
    kl = {0: np.exp(d) - d - 1, 1: -d, 2: 0.5 * d * d, 3: np.abs(d)}[kl_mode]
    loss = pg + (beta * kl if beta != 0 else 0.0) - ent_coef * H
    return np.array([(w * loss).sum(), (w * pg).sum(), (w * kl).sum(), (w * H).sum(), (w * clipped).sum(),
                     (w * ratio).sum(), float(act.sum()), (w * (o - lp)).sum()])
