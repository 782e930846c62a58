# SPDX-License-Identifier: Apache-2.0
"""CPU: pin the fp64 oracle before trusting it.

1. seeded-RNG / digest helpers vs the reference's own rng.cpp + hash.hpp
   compiled into oracle/_ref (bit-exact);
2. hand-derived known answers;
3. golden vectors from an independent torch-float64 autograd implementation
   (tests/golden/make_golden.py).
"""
import glob
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- 1. reference pins
def _ref_or_skip(orc):
    r = orc.ref_lib()
    if r is None:
        pytest.skip("oracle/_ref not built (needs /root/reference; `make -C oracle ref`)")
    return r


def test_splitmix_matches_reference(orc):
    import ctypes

    r = _ref_or_skip(orc)
    for seed in (0, 1, 42, 0xDEADBEEFCAFEBABE, 2**64 - 1):
        n = 257
        out = np.zeros(n, np.uint64)
        r.sfref_splitmix_seq(seed, n, ctypes.c_void_p(out.ctypes.data))
        mine = [orc.splitmix_at(seed, i) for i in range(n)]
        assert mine == [int(v) for v in out]
        assert np.array_equal(orc.splitmix_vec(seed, np.arange(n)), out)


def test_derive_seed_and_fnv_match_reference(orc):
    import ctypes

    r = _ref_or_skip(orc)
    for seed in (0, 42, 7, 2**63 + 5):
        for tag in ("", "train", "logits", "rollout.sample", "stage.actor_fwd", "x" * 100):
            for idx in (0, 1, 31, 2**40 + 3):
                b = tag.encode()
                assert orc.derive_seed(seed, tag, idx) == r.sfref_derive_seed(seed, b, len(b), idx)
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 64, 1000):
        buf = rng.integers(0, 256, size=max(n, 1), dtype=np.uint8)
        assert orc.fnv1a64(buf[:n].tobytes()) == r.sfref_fnv1a64(ctypes.c_void_p(buf.ctypes.data), n)


def test_fnv_known_answers(orc):
    # published FNV-1a 64 test vectors
    assert orc.fnv1a64(b"") == 0xCBF29CE484222325
    assert orc.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert orc.fnv1a64(b"foobar") == 0x85944171F73967E8


def test_bf16_rounding_matches_torch(orc):
    import torch

    rng = np.random.default_rng(1)
    x = np.concatenate([rng.normal(0, 10, 20000), rng.normal(0, 1e-3, 2000), [0.0, -0.0, 1.0, 65504.0, 3e38]])
    x32 = x.astype(np.float32)
    want = torch.from_numpy(x32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(orc.f32_to_bf16_bits(x32), want)
    got = np.array([orc.lib().orc_f64_to_bf16(float(v)) for v in x32.astype(np.float64)], np.uint16)
    assert np.array_equal(got, want)


# ---------------------------------------------------------------- 2. known answers
def test_uniform_logits_known_answer(orc):
    V = 1000
    x = np.zeros((3, V), np.float32)
    logp, ent, lse = orc.logprob_fwd(x, np.array([0, 5, 999]))
    assert np.allclose(logp, -math.log(V), atol=1e-13)
    assert np.allclose(ent, math.log(V), atol=1e-12)
    assert np.allclose(lse, math.log(V), atol=1e-13)


def test_dominant_logit_known_answer(orc):
    V = 500
    x = np.zeros((1, V), np.float32)
    x[0, 17] = 40.0
    logp, ent, _ = orc.logprob_fwd(x, np.array([17]))
    assert abs(logp[0]) < 1e-15 + V * math.exp(-40)
    assert 0 <= ent[0] < 1e-13


def test_ratio_one_loss_is_minus_weighted_advantage(orc):
    rng = np.random.default_rng(3)
    T, V = 16, 300
    x = rng.normal(size=(T, V)).astype(np.float32)
    y = rng.integers(0, V, T).astype(np.int32)
    logp, _, _ = orc.logprob_fwd(x, y)
    adv = rng.normal(size=T).astype(np.float32)
    w = np.full(T, 1.0 / T, np.float32)
    old = logp.astype(np.float32)  # ratio ~ 1 (to fp32 rounding of old)
    met, dl, lp, _, g = orc.pg_loss_fwd_bwd(x, y, old, old, adv, w)
    assert abs(met[0] - float(-(w.astype(np.float64) * adv * np.exp(lp - old)).sum())) < 1e-12
    assert abs(met[0] - float(-(w * adv).sum())) < 1e-6
    # gradient: d/dlogits of -A*ratio*w = -w*A*ratio*(onehot - p)
    p = np.exp(x.astype(np.float64) - np.log(np.exp(x.astype(np.float64)).sum(1, keepdims=True)))
    oh = np.zeros_like(p)
    oh[np.arange(T), y] = 1
    want = (g[:, None]) * (oh - p)
    assert np.allclose(dl, want, atol=1e-14)
    assert np.allclose(g, -w * adv * np.exp(lp - old), atol=1e-14)


@pytest.mark.parametrize("A,delta,on", [(1.0, 0.279, True), (1.0, 0.281, False), (-1.0, -0.199, True),
                                         (-1.0, -0.201, False), (1.0, -0.5, True), (-1.0, 0.5, True)])
def test_clip_boundary_gradient_on_off(orc, A, delta, on):
    V = 64
    x = np.zeros((1, V), np.float32)
    logp = -math.log(V)
    old = np.array([logp - math.log(1.0 + delta)], np.float32)  # ratio = 1 + delta
    _, _, _, _, g = orc.pg_loss_fwd_bwd(x, np.array([3]), old, old, np.array([A], np.float32), np.array([1.0], np.float32))
    ratio = math.exp(logp - float(old[0]))
    assert (abs(g[0]) > 0) == on
    if on:
        assert abs(g[0] - (-A * ratio)) < 1e-12


def test_equal_rewards_give_zero_advantage(orc):
    r = np.array([1, 1, 1, 1, 0, 1, 0, 1, 0.5, 0.5], np.float32)
    g = np.array([0, 0, 0, 0, 1, 1, 1, 1, 2, 2], np.int32)
    for mode in (0, 1, 2):
        adv, gs = orc.grpo_advantage(r, g, 1e-6, mode)
        assert np.all(adv[:4] == 0.0) and np.all(adv[8:] == 0.0)
        assert list(gs) == [4] * 8 + [2, 2]
    adv, _ = orc.grpo_advantage(np.array([3.0], np.float32), np.array([9], np.int32))
    assert adv[0] == 0.0  # singleton group


def test_r3_recorded_equals_topk_gives_normal_gate(orc):
    rng = np.random.default_rng(4)
    L, T, E, k = 2, 10, 128, 8
    z = rng.normal(size=(L, T, E)).astype(np.float32)
    top = np.argsort(-z, axis=-1, kind="stable")[..., :k].astype(np.int32)
    w, idx, mm = orc.r3_gate_fwd(z, top, renorm=True)
    assert mm.sum() == 0 and np.array_equal(idx, top)
    zz = np.take_along_axis(z.astype(np.float64), top, -1)
    want = np.exp(zz - zz.max(-1, keepdims=True))
    want /= want.sum(-1, keepdims=True)
    assert np.allclose(w, want, atol=1e-15)


def test_varlen_meta_known_answer(orc):
    cu, sid, mask, tg = orc.varlen_meta([3, 0, 2], plens=[1, 0, 5], gids=[7, 8, 9])
    assert list(cu) == [0, 3, 3, 5]
    assert list(sid) == [0, 0, 0, 2, 2]
    assert list(mask) == [0, 1, 1, 0, 0]
    assert list(tg) == [7, 7, 7, 9, 9]


# ---------------------------------------------------------------- 3. golden vectors
@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "golden_loss_*.npz"))))
def test_oracle_matches_torch_autograd_golden(orc, path):
    d = np.load(path)
    eps_lo, eps_hi, dual_c, beta, ent_coef, inv_tau = d["params"]
    x = d["logits"]
    logits = orc.f32_to_bf16_bits(x) if str(d["dtype"]) == "bf16" else x
    p = orc.params(eps_lo, eps_hi, dual_c, beta, ent_coef, inv_tau)
    met, dl, lp, ent, _ = orc.pg_loss_fwd_bwd(logits, d["targets"], d["old"], d["ref"], d["adv"], d["w"], p)
    act = d["w"] != 0
    assert np.allclose(lp[act], d["logp"][act], rtol=0, atol=1e-12)
    assert np.allclose(ent[act], d["ent"][act], rtol=0, atol=1e-12)
    assert np.allclose(dl, d["dlogits"], rtol=1e-10, atol=1e-15)
    assert np.allclose(met, d["metrics"], rtol=1e-11, atol=1e-14)


def test_oracle_grpo_matches_golden(orc):
    d = np.load(os.path.join(GOLD, "golden_grpo.npz"))
    for mode, name in ((0, "unbiased"), (1, "population"), (2, "none")):
        adv, _ = orc.grpo_advantage(d["rewards"], d["gids"], 1e-6, mode)
        assert np.allclose(adv, d[name], rtol=1e-12, atol=1e-15), name


def test_oracle_r3_matches_golden(orc):
    d = np.load(os.path.join(GOLD, "golden_r3.npz"))
    w, idx, mm = orc.r3_gate_fwd(d["z"], d["rec"], renorm=True)
    assert np.array_equal(idx, d["rec"])
    assert np.array_equal(mm, d["mismatch"])
    assert np.allclose(w, d["w_re"], atol=1e-14)
    w2, _, mm2 = orc.r3_gate_fwd(d["z"], d["rec"], renorm=False)
    assert np.allclose(w2, d["w_full"], atol=1e-14)
    assert np.array_equal(mm2, d["mismatch"])
    dz = orc.r3_gate_bwd(d["z"], d["rec"], d["w_re"].astype(np.float32), d["dw"], renorm=True)
    # golden dz uses fp64 w; oracle uses the fp32 w the GPU sees -> fp32-level agreement
    assert np.allclose(dz, d["dz_re"], atol=2e-7)
    dz2 = orc.r3_gate_bwd(d["z"], d["rec"], d["w_full"].astype(np.float32), d["dw"], renorm=False)
    assert np.allclose(dz2, d["dz_full"], atol=2e-7)


def test_vp_partial_stats_combine_equals_full_row(orc):
    rng = np.random.default_rng(7)
    T, V, P = 9, 1003, 4
    x = (rng.normal(size=(T, V)) * 3).astype(np.float32)
    y = rng.integers(0, V, T).astype(np.int32)
    logp, ent, lse = orc.logprob_fwd(x, y)
    bounds = np.linspace(0, V, P + 1).astype(int)
    st = [orc.vp_partial_stats(np.ascontiguousarray(x[:, a:b]), y, a) for a, b in zip(bounds[:-1], bounds[1:])]
    m = np.max([s[:, 0] for s in st], 0)
    S = sum(s[:, 1] * np.exp(s[:, 0] - m) for s in st)
    W = sum(np.exp(s[:, 0] - m) * (s[:, 2] + s[:, 1] * (s[:, 0] - m)) for s in st)
    zy = np.nansum([s[:, 3] for s in st], 0)
    L = m + np.log(S)
    assert np.allclose(L, lse, atol=1e-12)
    assert np.allclose(np.log(S) - W / S, ent, atol=1e-12)
    assert np.allclose(zy - L, logp, atol=1e-12)


def test_fast_cpu_baseline_matches_fp64_oracle(orc):
    """The fp32 'fast' CPU variant timed as the CPU baseline computes the same
    loss: metrics within fp32 tolerance, dlogits within 2 bf16 ulp."""
    prob = orc.synth_problem(13, [20, 17], 5000, "bf16", prompt_max=4)
    T = prob["T"]
    rng = np.random.default_rng(2)
    a = rng.normal(size=T).astype(np.float32)
    w = (rng.random(T) < 0.8).astype(np.float32) / T
    p = orc.params(beta=0.05, ent_coef=0.01)
    om, odl, olp, oent, og = orc.pg_loss_fwd_bwd(prob["logits"], prob["targets"], prob["old"], prob["ref"], a, w, p)
    fm, fdl = orc.pg_loss_fwd_bwd_fast(prob["logits"], prob["targets"], prob["old"], prob["ref"], a, w, p)
    assert np.allclose(fm[:6], om[:6], rtol=1e-4, atol=1e-6) and fm[6] == om[6]
    g = orc.bf16_bits_to_f32(fdl.ravel()).reshape(fdl.shape).astype(np.float64)
    ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(odl), 1e-38))) - 7)
    err = np.abs(g - odl) - 2 * ulp - 1e-6 * np.abs(og)[:, None]
    assert (err <= 0).mean() > 0.999


@pytest.mark.parametrize("kl_mode", [0, 1, 2, 3])
def test_kl_estimators_known_answer(orc, kl_mode):
    """The four KL estimators (d = ref - logp): k3 e^d - d - 1, k1 -d, k2 d^2/2,
    abs |d|; metric 2 is sum w*kl and g_t = w*(g_pg + beta*dkl/dlogp)."""
    prob = orc.synth_problem(17, [9, 8], 600, "f32", prompt_max=0)
    T = prob["T"]
    a = np.zeros(T, np.float32)  # no policy term: g is the KL gradient alone
    w = np.full(T, 1.0 / T, np.float32)
    beta = 0.3
    om, _, olp, _, og = orc.pg_loss_fwd_bwd(prob["logits"], prob["targets"], prob["old"], prob["ref"], a, w,
                                            orc.params(beta=beta, kl_mode=kl_mode))
    d = prob["ref"].astype(np.float64) - olp
    kl, dkl = {0: (np.exp(d) - d - 1, 1 - np.exp(d)), 1: (-d, np.ones_like(d)), 2: (0.5 * d * d, -d),
               3: (np.abs(d), -np.sign(d))}[kl_mode]
    w64 = w.astype(np.float64)
    assert np.isclose(om[2], (w64 * kl).sum(), rtol=1e-10, atol=1e-14)
    assert np.isclose(om[0], beta * (w64 * kl).sum(), rtol=1e-10, atol=1e-14)
    assert np.allclose(og, w64 * beta * dkl, rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("pkw", [{}, {"beta": 0.05}, {"dual_c": 3.0, "ent_coef": 0.01}, {"beta": 0.1, "kl_mode": 2}])
def test_metrics_from_rows_matches_oracle(orc, pkw):
    """tests/_cmp.metrics_from_rows (used by the full-size GPU tests to check the
    kernel's reduction from its own per-row outputs) restates the oracle's
    per-row terms exactly."""
    from tests._cmp import metrics_from_rows

    prob = orc.synth_problem(91, [40, 25, 33], 3000, "f32", prompt_max=10)
    rng = np.random.default_rng(5)
    T = prob["T"]
    a = rng.normal(size=T).astype(np.float32)
    w = np.where(rng.random(T) < 0.8, 1.0 / T, 0.0).astype(np.float32)
    p = orc.params(**{k: v for k, v in pkw.items()})
    om, _, olp, oent, _ = orc.pg_loss_fwd_bwd(prob["logits"], prob["targets"], prob["old"], prob["ref"], a, w, p)
    got = metrics_from_rows(olp, oent, prob["old"], prob["ref"], a, w, p.eps_lo, p.eps_hi, p.dual_c, p.beta,
                            p.ent_coef, p.kl_mode)
    assert np.allclose(got, om, rtol=1e-12, atol=1e-15)
