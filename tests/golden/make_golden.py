# SPDX-License-Identifier: Apache-2.0
"""Generate golden vectors for the train-math oracle from an INDEPENDENT
implementation: torch float64 autograd (log_softmax / softmax / clamp / min
written the usual way, gradients by autograd, not by the hand-derived formulas
the oracle and the kernels use).

The reference (/root/reference) has no implementation of this math
(SPEC.md:8), so these vectors are the pin for the oracle.
Run from the repo root:  python tests/golden/make_golden.py
Writes tests/golden/golden_*.npz (small, committed).
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

torch.set_default_dtype(torch.float64)


def bf16_round(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).to(torch.float32).numpy()


def loss_torch(logits, targets, old, ref, adv, w, eps_lo, eps_hi, dual_c, beta, ent_coef, inv_tau):
    """The DAPO/GRPO token loss as commonly written (veRL-style), float64."""
    z = logits * inv_tau
    lsm = torch.log_softmax(z, dim=-1)
    logp = lsm.gather(1, targets[:, None]).squeeze(1)
    p = lsm.exp()
    ent = -(p * lsm).sum(-1)
    ratio = torch.exp(logp - old)
    pg1 = -adv * ratio
    pg2 = -adv * torch.clamp(ratio, 1 - eps_lo, 1 + eps_hi)
    pg = torch.maximum(pg1, pg2)
    if dual_c > 1:
        pg3 = -adv * dual_c
        pg = torch.where(adv < 0, torch.minimum(pg, pg3), pg)
    d = ref - logp
    kl = torch.exp(d) - d - 1
    l = pg + beta * kl - ent_coef * ent
    loss = (w * l).sum()
    return loss, logp, ent, ratio, kl, pg


def case_loss(name, seed, T, V, dtype, **kw):
    rng = np.random.default_rng(seed)
    x = rng.normal(0, 2.0, size=(T, V))
    peak = rng.integers(0, V, size=T)
    x[np.arange(T), peak] += rng.uniform(5, 25, size=T)
    x[rng.random((T, V)) < 0.01] = 30.0
    x = bf16_round(x) if dtype == "bf16" else x.astype(np.float32)
    targets = np.where(rng.random(T) < 0.5, peak, rng.integers(0, V, size=T)).astype(np.int64)
    lt = torch.tensor(x.astype(np.float64), requires_grad=True)
    with torch.no_grad():
        lp0 = torch.log_softmax(lt * kw.get("inv_tau", 1.0), -1).gather(1, torch.tensor(targets)[:, None]).squeeze(1).numpy()
    old = (lp0 + rng.normal(0, 0.3, size=T)).astype(np.float32)
    ref = (lp0 + rng.normal(0, 0.3, size=T)).astype(np.float32)
    adv = rng.normal(0, 1, size=T).astype(np.float32)
    mask = (rng.random(T) < 0.8).astype(np.float64)
    w = (mask / max(mask.sum(), 1)).astype(np.float32)
    p = dict(eps_lo=0.2, eps_hi=0.28, dual_c=0.0, beta=0.0, ent_coef=0.0, inv_tau=1.0)
    p.update(kw)
    loss, logp, ent, ratio, kl, pg = loss_torch(lt, torch.tensor(targets), torch.tensor(old.astype(np.float64)),
                                                 torch.tensor(ref.astype(np.float64)), torch.tensor(adv.astype(np.float64)),
                                                 torch.tensor(w.astype(np.float64)), **p)
    loss.backward()
    # exclude rows whose ratio sits within 1e-9 of a clip boundary (autograd tie split)
    r = ratio.detach().numpy()
    near = (np.abs(r - (1 + p["eps_hi"])) < 1e-9) | (np.abs(r - (1 - p["eps_lo"])) < 1e-9)
    assert not near.any()
    wd = torch.tensor(w.astype(np.float64))
    a64 = adv.astype(np.float64)
    pgmax = np.maximum(-a64 * r, -a64 * np.clip(r, 1 - p["eps_lo"], 1 + p["eps_hi"]))
    clip_reg = ((a64 > 0) & (r > 1 + p["eps_hi"])) | ((a64 < 0) & (r < 1 - p["eps_lo"]))
    dual = (p["dual_c"] > 1) & (a64 < 0) & (pgmax > -a64 * p["dual_c"])
    clipped = clip_reg | dual
    metrics = np.array([
        loss.item(), (wd * pg).sum().item(), (wd * kl).sum().item(), (wd * ent).sum().item(),
        float(np.sum(np.where(clipped, w.astype(np.float64), 0.0))),
        (wd * ratio).sum().item(), float((w != 0).sum()), (wd * (torch.tensor(old.astype(np.float64)) - logp)).sum().item(),
    ])
    np.savez_compressed(os.path.join(HERE, f"golden_{name}.npz"), logits=x, targets=targets.astype(np.int32), old=old,
                        ref=ref, adv=adv, w=w, dlogits=lt.grad.numpy(), logp=logp.detach().numpy(),
                        ent=ent.detach().numpy(), metrics=metrics, dtype=np.array(dtype),
                        params=np.array([p["eps_lo"], p["eps_hi"], p["dual_c"], p["beta"], p["ent_coef"], p["inv_tau"]]))


def case_grpo(seed):
    rng = np.random.default_rng(seed)
    B = 96
    gids = rng.integers(0, 12, size=B).astype(np.int32)  # non-contiguous groups
    r = (rng.random(B) < 0.5).astype(np.float32)
    r[gids == 3] = 1.0  # an all-equal group
    r[:5] = rng.normal(size=5).astype(np.float32)
    out = {}
    for mode, name in ((0, "unbiased"), (1, "population"), (2, "none")):
        rt = torch.tensor(r.astype(np.float64))
        A = torch.zeros(B)
        for g in np.unique(gids):
            idx = torch.tensor(np.nonzero(gids == g)[0])
            x = rt[idx]
            if x.max() == x.min():
                A[idx] = 0.0
                continue
            mean = x.mean()
            if mode == 2:
                A[idx] = x - mean
            else:
                std = x.std(unbiased=(mode == 0))
                A[idx] = (x - mean) / (std + 1e-6)
        out[name] = A.numpy()
    np.savez_compressed(os.path.join(HERE, "golden_grpo.npz"), rewards=r, gids=gids, **out)


def case_r3(seed):
    rng = np.random.default_rng(seed)
    L, T, E, k = 3, 40, 64, 6
    z = bf16_round(rng.normal(0, 1, size=(L, T, E)) * 2)  # bf16 grid -> many ties
    z[0, :4, :] = 0.0  # fully tied rows: P9 picks experts 0..k-1
    # trainer top-k with ties -> lowest index
    order = np.lexsort((np.broadcast_to(np.arange(E), z.shape), -z), axis=-1)
    topk = order[..., :k]
    rec = topk.copy()
    flip = rng.random((L, T)) < 0.2
    for l, t in zip(*np.nonzero(flip)):
        others = np.setdiff1d(np.arange(E), rec[l, t])
        rec[l, t, rng.integers(0, k)] = rng.choice(others)
    mism = np.array([(np.sort(topk[l], -1) != np.sort(rec[l], -1)).any(-1).sum() for l in range(L)])
    zt = torch.tensor(z.astype(np.float64), requires_grad=True)
    rect = torch.tensor(rec)
    g = zt.gather(-1, rect)
    w_re = torch.softmax(g, -1)
    w_full = torch.softmax(zt, -1).gather(-1, rect)
    dw = torch.tensor(rng.normal(size=(L, T, k)).astype(np.float32).astype(np.float64))
    (w_re * dw).sum().backward()
    dz_re = zt.grad.numpy().copy()
    zt.grad = None
    (w_full * dw).sum().backward()
    dz_full = zt.grad.numpy().copy()
    np.savez_compressed(os.path.join(HERE, "golden_r3.npz"), z=z.astype(np.float32), rec=rec.astype(np.int32),
                        topk=topk.astype(np.int32), mismatch=np.concatenate([mism, [mism.sum()]]).astype(np.uint32),
                        w_re=w_re.detach().numpy(), w_full=w_full.detach().numpy(), dw=dw.numpy().astype(np.float32),
                        dz_re=dz_re, dz_full=dz_full)


if __name__ == "__main__":
    case_loss("loss_bf16_v1000", 1, T=24, V=1000, dtype="bf16")
    case_loss("loss_f32_v257", 2, T=16, V=257, dtype="f32")
    case_loss("loss_bf16_kl_ent_tau", 3, T=20, V=640, dtype="bf16", beta=0.05, ent_coef=0.01, inv_tau=1.0 / 0.7)
    case_loss("loss_f32_dualclip", 4, T=32, V=320, dtype="f32", dual_c=3.0, eps_lo=0.1, eps_hi=0.15)
    case_grpo(5)
    case_r3(6)
    print("golden vectors written to", HERE)
