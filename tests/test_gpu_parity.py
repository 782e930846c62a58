# SPDX-License-Identifier: Apache-2.0
"""GPU parity: every C-ABI entry point vs the fp64 oracle on the same seeded
inputs. Bit-exact for integer/index work (cu_seqlens, seq ids,
masks, group ids/sizes, replayed expert indices, mismatch counts); stated
tolerances (tests/_cmp.py) for floating point."""
import zlib

import numpy as np
import pytest

from tests._cmp import assert_close, assert_grad_close, loss_row_scale, near_clip_rows

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def tm():
    from paper_2604_11554_b200 import train_math

    train_math.handle(0)
    return train_math


def to_dev_logits(prob):
    x = prob["logits"]
    if x.dtype == np.uint16:
        return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(x).cuda()


def grad_to_np(dl):
    if dl.dtype == torch.bfloat16:
        from oracle.oracle import bf16_bits_to_f32

        return bf16_bits_to_f32(dl.view(torch.int16).cpu().numpy().view(np.uint16)).astype(np.float64)
    return dl.cpu().numpy().astype(np.float64)


def i32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def f32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def gpu_pipeline(tm, prob, norm_mode=0, adv_eps=1e-6, std_mode=0):
    lens = i32(prob["lens"])
    cu, sid, mask, _ = tm.varlen_meta(lens, i32(prob["plens"]), T=prob["T"])
    adv = tm.grpo_advantage(f32(prob["rewards"]), i32(prob["gids"]), adv_eps, std_mode)
    adv_tok, w_tok = tm.token_weights(cu, adv, mask, prob["T"], norm_mode)
    return cu, sid, mask, adv, adv_tok, w_tok


def check_loss_case(tm, orc, prob, pkw=None, generic=False, in_place=False, masked_skip=False, norm_mode=0):
    pkw = dict(pkw or {})
    from paper_2604_11554_b200 import _lib

    params = _lib.default_loss_params(**pkw)
    params.norm_mode = norm_mode
    if masked_skip:
        params.masked_rows = _lib.MASKED_SKIP
    logits = to_dev_logits(prob)
    cu, sid, mask, adv, adv_tok, w_tok = gpu_pipeline(tm, prob, norm_mode)
    tm.set_force_generic(generic)
    try:
        sentinel = None
        if masked_skip:
            dl = torch.full_like(logits, 7.0)
            sentinel = 7.0
        else:
            dl = None
        met, dl, logp, ent = tm.pg_loss_fwd_bwd(logits, i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"]),
                                                adv_tok, w_tok, params, dlogits=dl, in_place=in_place, want_logp=True)
        torch.cuda.synchronize()
    finally:
        tm.set_force_generic(False)
    w = w_tok.cpu().numpy()
    a = adv_tok.cpu().numpy()
    op = orc.params(params.clip_eps_low, params.clip_eps_high, params.dual_clip_c, params.kl_beta,
                    params.entropy_coef, params.inv_temperature, params.kl_mode)
    om, odl, olp, oent, og = orc.pg_loss_fwd_bwd(prob["logits"], prob["targets"], prob["old"], prob["ref"], a, w, op,
                                                 masked_skip=masked_skip)
    act = w != 0
    gl = logp.cpu().numpy()
    ge = ent.cpu().numpy()
    assert_close(gl[act], olp[act], what="logp")
    assert_close(ge[act], oent[act], what="entropy")
    gm = met.cpu().numpy()
    near = near_clip_rows(olp, prob["old"], a, params.clip_eps_low, params.clip_eps_high, params.dual_clip_c)
    near &= act
    scale = loss_row_scale(og, w, a, olp, prob["old"], prob["ref"], params.kl_beta, params.kl_mode,
                           params.entropy_coef, params.inv_temperature)
    gdl = grad_to_np(dl)
    if masked_skip:
        assert np.all(gdl[~act] == sentinel)
        rows = act & ~near
    else:
        rows = ~near
    assert_grad_close(gdl, odl, scale, prob["dtype"], rows_ok=rows)
    if not near.any():
        tol = 1e-5 * (np.abs(w) * (np.abs(a) * 2 + 1)).sum() + 1e-6
        for i, name in enumerate(["loss", "pg", "kl", "entropy", "clipfrac", "ratio", "n_active", "ppo_kl"]):
            if name == "n_active":
                assert gm[i] == om[i]
            else:
                t = tol * (30 if name in ("kl", "entropy") else 1) + 1e-5 * abs(om[i])
                assert abs(gm[i] - om[i]) <= t, (name, gm[i], om[i])
    return gm, gdl


# ---------------------------------------------------------------------------- a6 / a3 / a4 prologue
def test_varlen_meta_bit_exact(tm, orc):
    rng = np.random.default_rng(11)
    lens = rng.integers(0, 300, size=257).astype(np.int32)
    lens[[0, 5, 100]] = 0
    plens = rng.integers(0, 400, size=257).astype(np.int32)
    gids = rng.integers(-5, 50, size=257).astype(np.int32)
    cu, sid, mask, tg = tm.varlen_meta(i32(lens), i32(plens), i32(gids), T=int(lens.sum()))
    ocu, osid, omask, otg = orc.varlen_meta(lens, plens, gids)
    for g, o in ((cu, ocu), (sid, osid), (mask, omask), (tg, otg)):
        g = g.cpu().numpy()
        assert orc.digest(g) == orc.digest(o)


def test_varlen_meta_large_b(tm, orc):
    lens = (np.arange(5000) % 7).astype(np.int32)
    cu, _, _, _ = tm.varlen_meta(i32(lens), T=int(lens.sum()), want=("cu",))
    assert orc.digest(cu.cpu().numpy()) == orc.digest(orc.varlen_meta(lens)[0])


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_grpo_advantage_golden(tm, orc, mode):
    import os

    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_grpo.npz"))
    adv, gs = tm.grpo_advantage(f32(d["rewards"]), i32(d["gids"]), 1e-6, mode, want_group_size=True)
    oadv, ogs = orc.grpo_advantage(d["rewards"], d["gids"], 1e-6, mode)
    assert np.array_equal(gs.cpu().numpy(), ogs)
    got = adv.cpu().numpy()
    assert_close(got, oadv, atol=1e-6, rtol=1e-6, what="advantage")
    eq = oadv == 0.0
    assert np.all(got[eq] == 0.0)  # P3: zero-variance groups are exactly 0


def test_grpo_advantage_large_noncontiguous(tm, orc):
    rng = np.random.default_rng(12)
    B = 4096
    gids = rng.permutation(np.repeat(np.arange(256), 16)).astype(np.int32)
    r = rng.random(B).astype(np.float32)
    adv, gs = tm.grpo_advantage(f32(r), i32(gids), 1e-6, 0, want_group_size=True)
    oadv, ogs = orc.grpo_advantage(r, gids)
    assert np.array_equal(gs.cpu().numpy(), ogs)
    assert_close(adv.cpu().numpy(), oadv, atol=1e-6, rtol=1e-6, what="advantage")


@pytest.mark.parametrize("norm_mode", [0, 1, 2])
def test_token_weights(tm, orc, norm_mode):
    rng = np.random.default_rng(13)
    lens = rng.integers(0, 50, size=40).astype(np.int32)
    T = int(lens.sum())
    cu = orc.varlen_meta(lens)[0]
    mask = (rng.random(T) < 0.7).astype(np.uint8)
    adv = rng.normal(size=40).astype(np.float32)
    at, wt = tm.token_weights(i32(cu), f32(adv), torch.from_numpy(mask).cuda(), T, norm_mode, 0.125)
    oat, owt = orc.token_weights(cu, adv, mask, T, norm_mode, 0.125)
    assert np.array_equal(at.cpu().numpy(), oat.astype(np.float32))
    assert_close(wt.cpu().numpy(), owt, atol=0, rtol=1e-7, what="w_tok")


# ---------------------------------------------------------------------------- a1
@pytest.mark.parametrize("dtype,V,T,generic", [("bf16", 151936, 40, False), ("bf16", 151936, 40, True),
                                               ("f32", 32000, 64, False), ("bf16", 1001, 33, False),
                                               ("f32", 151936, 9, False), ("bf16", 8, 5, False),
                                               ("bf16", 50257, 37, False), ("f32", 32001, 21, False),
                                               ("bf16", 13, 7, False)])
def test_logprob_fwd(tm, orc, dtype, V, T, generic):
    """bf16 1001 / 50257 / 13 and f32 32001 rows start off 16-B boundaries:
    the streaming kernel runs them in sector coordinates."""
    lens = [T]
    prob = orc.synth_problem(100 + V % 97, lens, V, dtype)
    logits = to_dev_logits(prob)
    tm.set_force_generic(generic)
    try:
        logp, ent, lse = tm.logprob_fwd(logits, i32(prob["targets"]))
        torch.cuda.synchronize()
    finally:
        tm.set_force_generic(False)
    olp, oent, olse = orc.logprob_fwd(prob["logits"], prob["targets"])
    assert_close(logp.cpu().numpy(), olp, what="logp")
    assert_close(ent.cpu().numpy(), oent, what="entropy")
    assert_close(lse.cpu().numpy(), olse, what="lse")


def test_logprob_fwd_odd_stride_uses_streaming_kernel(tm, orc):
    prob = orc.synth_problem(5, [45], 4099, "bf16")
    T, V = 45, 4099
    base = torch.zeros(T, V + 5, dtype=torch.bfloat16, device="cuda")
    view = base[:, 3:3 + V]
    view.copy_(to_dev_logits(prob))
    logp, ent, lse = tm.logprob_fwd(view, i32(prob["targets"]))
    torch.cuda.synchronize()
    assert tm.handle().last_launch()["kernel"] == "fwd_stream_kernel"
    olp, oent, olse = orc.logprob_fwd(prob["logits"], prob["targets"])
    assert_close(logp.cpu().numpy(), olp, what="logp")
    assert_close(ent.cpu().numpy(), oent, what="entropy")
    assert_close(lse.cpu().numpy(), olse, what="lse")


def test_logprob_fwd_temperature_and_strided_rows(tm, orc):
    prob = orc.synth_problem(5, [24], 32000, "bf16")
    big = torch.zeros(24, 32064, dtype=torch.bfloat16, device="cuda")
    big[:, :32000] = to_dev_logits(prob)
    view = big[:, :32000]
    logp, ent, lse = tm.logprob_fwd(view, i32(prob["targets"]), inv_temperature=1 / 0.6)
    olp, oent, olse = orc.logprob_fwd(prob["logits"], prob["targets"], 1 / 0.6)
    assert_close(logp.cpu().numpy(), olp, what="logp")
    assert_close(ent.cpu().numpy(), oent, what="entropy")


# ---------------------------------------------------------------------------- a1+a4+a2 fused
LOSS_CASES = [
    # id, dtype, V, lens, params, kwargs
    ("qwen_bf16_c2", "bf16", 151936, [17, 9, 30, 8], {}, {}),
    ("qwen_bf16_generic", "bf16", 151936, [17, 9, 30, 8], {}, {"generic": True}),
    ("cfg1_f32", "f32", 32000, [40, 3, 21], {}, {}),
    ("kl_ent_tau_bf16", "bf16", 32000, [20, 20], {"kl_beta": 0.05, "entropy_coef": 0.01, "inv_temperature": 1 / 0.7}, {}),
    ("dualclip_f32", "f32", 4096, [30, 30], {"dual_clip_c": 3.0, "clip_eps_low": 0.1, "clip_eps_high": 0.15}, {}),
    ("inplace_bf16", "bf16", 151936, [12, 12], {}, {"in_place": True}),
    ("masked_skip_bf16", "bf16", 32000, [25, 25], {}, {"masked_skip": True}),
    ("seq_mean_bf16", "bf16", 32000, [25, 5, 25], {}, {"norm_mode": 1}),
    ("f32_wide_c4", "f32", 151936, [6, 4], {}, {}),
    ("bf16_c8_262k", "bf16", 262144, [5], {}, {}),
    ("bf16_odd_vocab", "bf16", 50257, [10, 7, 40, 3], {}, {}),
    ("f32_odd_vocab_kl_ent", "f32", 32001, [20, 13], {"kl_beta": 0.05, "entropy_coef": 0.01}, {}),
    ("bf16_odd_vocab_ent_inplace", "bf16", 50257, [9, 30], {"entropy_coef": 0.02}, {"in_place": True}),
    ("bf16_odd_vocab_skip", "bf16", 20011, [25, 25], {}, {"masked_skip": True}),
    ("bf16_odd_tiny", "bf16", 13, [9, 9], {}, {}),
    ("bf16_tiny_vocab", "bf16", 16, [9, 9], {"kl_beta": 0.1}, {}),
    ("kl_k1_f32", "f32", 4096, [20, 11], {"kl_beta": 0.1, "kl_mode": 1}, {}),
    ("kl_k2_bf16", "bf16", 32000, [17, 9], {"kl_beta": 0.1, "kl_mode": 2}, {}),
    ("kl_abs_bf16_odd", "bf16", 20011, [13, 15], {"kl_beta": 0.1, "kl_mode": 3}, {}),
    # vocab-parallel shard widths (P = 8 / 4 of Qwen3): the row-stream kernels (4 / 2 streams),
    # row counts that leave the last group of a CTA partial
    ("vp8_shard_bf16_streams4", "bf16", 18992, [40, 33, 17, 9, 51], {}, {}),
    ("vp4_shard_kl_ent_streams2", "bf16", 37984, [30, 21, 7], {"kl_beta": 0.05, "entropy_coef": 0.01}, {}),
    ("vp8_shard_f32_streams2", "f32", 18992, [19, 23, 5], {"kl_beta": 0.05}, {}),
    ("vp8_shard_inplace", "bf16", 18992, [21, 14], {}, {"in_place": True}),
    ("vp8_shard_masked_skip", "bf16", 18992, [17, 30, 2], {}, {"masked_skip": True}),
    # unaligned rows (16-B sector coordinates) through the row streams: each row of a
    # group has its own sector phase, so rows of one group take different chunk counts
    ("odd_shard_bf16_streams4", "bf16", 18993, [30, 27, 11], {"entropy_coef": 0.01}, {}),
    ("odd_32001_bf16_streams2_inplace", "bf16", 32001, [14, 23], {}, {"in_place": True}),
    ("odd_9497_f32_streams2_skip", "f32", 9497, [19, 8, 25], {"kl_beta": 0.05}, {"masked_skip": True}),
]


@pytest.mark.parametrize("case", LOSS_CASES, ids=[c[0] for c in LOSS_CASES])
def test_pg_loss_fwd_bwd(tm, orc, case):
    _, dtype, V, lens, pkw, kw = case
    prob = orc.synth_problem(zlib.crc32(case[0].encode()) % 1000, lens, V, dtype, prompt_max=8)  # stable per case
    check_loss_case(tm, orc, prob, pkw, **kw)


def test_pg_loss_unaligned_rows_use_fused_kernel(tm, orc):
    """Odd vocabularies and odd row strides run the fused single-pass kernel
    (rows handled in 16-B sector coordinates), not the two-pass fallback; a
    dlogits buffer at a different sector phase falls back and still agrees."""
    from paper_2604_11554_b200 import _lib

    prob = orc.synth_problem(9, [33, 20, 51], 4099, "bf16", prompt_max=8)
    T, V = len(prob["targets"]), 4099
    base = torch.zeros(T, V + 5, dtype=torch.bfloat16, device="cuda")
    view = base[:, 3:3 + V]  # odd stride (V + 5) and a 6-byte row offset
    view.copy_(to_dev_logits(prob))
    cu, sid, mask, adv, adv_tok, w_tok = gpu_pipeline(tm, prob, 0)
    params = _lib.default_loss_params()
    dbase = torch.full_like(base, 7.0)  # guard columns around every dlogits row
    dl = dbase[:, 3:3 + V]
    met, dl, logp, ent = tm.pg_loss_fwd_bwd(view, i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"]),
                                            adv_tok, w_tok, params, dlogits=dl, want_logp=True)
    torch.cuda.synchronize()
    assert tm.handle().last_launch()["kernel"] == "loss_tmem_kernel"
    assert torch.all(dbase[:, :3] == 7.0) and torch.all(dbase[:, 3 + V:] == 7.0), "dlogits written out of row bounds"
    om, odl, olp, oent, og = orc.pg_loss_fwd_bwd(prob["logits"], prob["targets"], prob["old"], prob["ref"],
                                                 adv_tok.cpu().numpy(), w_tok.cpu().numpy(), orc.params())
    act = w_tok.cpu().numpy() != 0
    assert_close(logp.cpu().numpy()[act], olp[act], what="logp")
    near = near_clip_rows(olp, prob["old"], adv_tok.cpu().numpy(), 0.2, 0.28)
    assert_grad_close(grad_to_np(dl), odl, np.abs(og), "bf16", rows_ok=~near)
    # dlogits at another sector phase: generic fallback, same answer
    dl2 = torch.zeros(T, V + 1, dtype=torch.bfloat16, device="cuda")[:, :V]
    met2, dl2, _, _ = tm.pg_loss_fwd_bwd(view, i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"]),
                                         adv_tok, w_tok, params, dlogits=dl2)
    torch.cuda.synchronize()
    assert tm.handle().last_launch()["kernel"] == "rows_generic_kernel"
    assert_grad_close(grad_to_np(dl2), odl, np.abs(og), "bf16", rows_ok=~near)
    assert np.allclose(met2.cpu().numpy()[:6], met.cpu().numpy()[:6], rtol=1e-5, atol=1e-7)


def test_pg_loss_deterministic(tm, orc):
    prob = orc.synth_problem(77, [64, 64], 151936, "bf16")
    m1, d1 = check_loss_case(tm, orc, prob)
    m2, d2 = check_loss_case(tm, orc, prob)
    assert np.array_equal(m1, m2)
    assert np.array_equal(d1, d2)


def test_vocab_padding_columns_are_inert(tm, orc):
    """padding an odd vocabulary to a multiple of 8 * P with a
    large finite negative logit (-1e4) leaves logp, entropy, the metrics and the
    real columns' dlogits unchanged and gives the padding columns dlogits of
    exactly 0 (their probability underflows to 0; no repair path)."""
    from paper_2604_11554_b200 import _lib

    V, Vpad = 50257, 50272
    prob = orc.synth_problem(41, [33, 20, 51], V, "bf16", prompt_max=8)
    T = prob["T"]
    logits = to_dev_logits(prob)
    padded = torch.full((T, Vpad), -1e4, dtype=torch.bfloat16, device="cuda")
    padded[:, :V] = logits
    cu, sid, mask, adv, adv_tok, w_tok = gpu_pipeline(tm, prob, 0)
    params = _lib.default_loss_params(kl_beta=0.05, entropy_coef=0.01)
    args = (i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"]), adv_tok, w_tok, params)
    m0, d0, lp0, e0 = tm.pg_loss_fwd_bwd(logits, *args, want_logp=True)
    m1, d1, lp1, e1 = tm.pg_loss_fwd_bwd(padded, *args, want_logp=True)
    torch.cuda.synchronize()
    assert tm.handle().last_launch()["kernel"] == "loss_tmem_kernel"
    assert torch.all(d1[:, V:] == 0)
    act = w_tok != 0
    assert torch.allclose(lp1[act], lp0[act], atol=2e-6, rtol=2e-6)
    assert torch.allclose(e1[act], e0[act], atol=2e-5, rtol=2e-5)
    assert torch.allclose(m1[:6], m0[:6], atol=2e-6, rtol=2e-5)
    g0, g1 = d0.float(), d1[:, :V].float()
    assert torch.all((g1 - g0).abs() <= 2.0 ** -7 * g0.abs() + 1e-9)


@pytest.mark.parametrize("dtype,V", [("bf16", 3000), ("f32", 5000)])
def test_pg_loss_deep_runahead(tm, orc, dtype, V):
    """Many short rows: a row slice is one chunk, so the forward warps can run
    up to the whole row store (31 rows) ahead of the backward warps. The
    partial/scalar rings and the cluster mailboxes must stay flow-controlled."""
    prob = orc.synth_problem(5, [300, 257, 400, 311, 280], V, dtype, prompt_max=30)
    check_loss_case(tm, orc, prob)


@pytest.mark.parametrize("dtype,T,V", [("bf16", 20000, 151936), ("bf16", 8000, 75968), ("f32", 5000, 16000),
                                       ("bf16", 9001, 18992), ("bf16", 6007, 37984), ("bf16", 7001, 18993)])
def test_fused_all_rows_vs_streaming_forward(tm, dtype, T, V):
    """Race regression: every loss-active row's logp/entropy from the fused
    kernel equals the streaming forward kernel's, over repeated launches at
    full row counts (a ring slot released before its LDS returned once let
    the next TMA fill corrupt ~1e-3 of the rows)."""
    g = torch.Generator(device="cpu").manual_seed(7)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    lg = (torch.randn(T, V, generator=g) * 3).to(tdt).cuda()
    tg = torch.randint(0, V, (T,), generator=g, dtype=torch.int32).cuda()
    o = (-4 + torch.randn(T, generator=g)).cuda()
    r = (o + 0.1 * torch.randn(T, generator=g).cuda()).float()
    a = torch.randn(T, generator=g).cuda()
    w = (torch.rand(T, generator=g) < 0.8).float().cuda() / T
    lp_ref, ent_ref, _ = tm.logprob_fwd(lg, tg)
    act = w != 0
    # row streams by shard width (SFTM_LOSS_NS unset): 4 at 18,992 bf16, 2 at 37,984 bf16 / 16,000 f32
    want_ns = {18992: 4, 37984: 2, 16000: 2, 18993: 4}.get(V, 1)
    for _ in range(4):
        _, _, lp, ent = tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, want_logp=True)
        torch.cuda.synchronize()
        env = __import__("os").environ
        if "SFTM_LOSS_NS" not in env and "SFTM_LOSS_C" not in env:
            assert tm.handle().last_launch()["streams"] == want_ns
        bad = ((lp - lp_ref).abs() > 2e-5 + 2e-6 * lp_ref.abs()) & act
        bad |= ((ent - ent_ref).abs() > 2e-5 + 2e-5 * ent_ref.abs()) & act
        assert int(bad.sum()) == 0, f"{int(bad.sum())} rows differ, e.g. {torch.nonzero(bad)[:5].flatten().tolist()}"


@pytest.mark.parametrize("dtype,V,generic", [("f32", 8192, False), ("bf16", 20011, False), ("bf16", 151936, False),
                                             ("f32", 8192, True)])
def test_neg_inf_logits_and_exponent_overflow(tm, orc, dtype, V, generic):
    """-inf logits (masked vocabulary entries), a row whose first chunk is far
    below a later logit (the fixed exponent base overflows) and a row with a
    single finite logit: the kernels' repair paths must match the oracle."""
    from paper_2604_11554_b200 import _lib

    prob = orc.synth_problem(31, [7, 6], V, "f32", prompt_max=0)
    x = prob["logits"].copy()
    rng = np.random.default_rng(3)
    x[rng.random(x.shape) < 0.1] = -np.inf
    x[0, :V // 2] = -100.0
    x[0, V // 2 + 5] = 100.0
    x[1, :] = -np.inf
    x[1, 7] = 2.0
    t = prob["targets"].copy()
    t[1] = 7
    for r in range(x.shape[0]):
        if not np.isfinite(x[r, t[r]]):
            x[r, t[r]] = 0.5
    if dtype == "bf16":
        xb = orc.f32_to_bf16_bits(x).reshape(x.shape)
        x = orc.bf16_bits_to_f32(xb).reshape(x.shape)
        xin, xt = xb, torch.from_numpy(xb.view(np.int16)).view(torch.bfloat16).cuda()
    else:
        xin, xt = x, torch.from_numpy(x).cuda()
    T = x.shape[0]
    w = np.full(T, 1.0 / T, np.float32)
    a = np.linspace(-1, 1, T).astype(np.float32)
    tm.set_force_generic(generic)
    try:
        met, dl, logp, ent = tm.pg_loss_fwd_bwd(xt, i32(t), f32(prob["old"]), f32(prob["ref"]), f32(a), f32(w),
                                                want_logp=True)
        lp2, ent2, _ = tm.logprob_fwd(xt, i32(t))
        torch.cuda.synchronize()
    finally:
        tm.set_force_generic(False)
    om, odl, olp, oent, og = orc.pg_loss_fwd_bwd(xin, t, prob["old"], prob["ref"], a, w)
    assert_close(logp.cpu().numpy(), olp, what="fused logp")
    assert_close(ent.cpu().numpy(), oent, what="fused entropy")
    assert_close(lp2.cpu().numpy(), olp, what="forward logp")
    assert_close(ent2.cpu().numpy(), oent, what="forward entropy")
    g = grad_to_np(dl)
    assert np.isfinite(g).all()
    near = near_clip_rows(olp, prob["old"], a, 0.2, 0.28)
    assert_grad_close(g, odl, np.abs(og), dtype, rows_ok=~near)


def test_pg_loss_all_masked_and_empty(tm, orc):
    from paper_2604_11554_b200 import _lib

    prob = orc.synth_problem(3, [6], 4096, "bf16")
    logits = to_dev_logits(prob)
    z = torch.zeros(6, device="cuda")
    met, dl, _, _ = tm.pg_loss_fwd_bwd(logits, i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"]), z, z)
    assert torch.all(met == 0) and torch.all(dl == 0)
    e = torch.empty(0, 4096, dtype=torch.bfloat16, device="cuda")
    ei = torch.empty(0, dtype=torch.int32, device="cuda")
    ef = torch.empty(0, device="cuda")
    met, _, _, _ = tm.pg_loss_fwd_bwd(e, ei, ef, ef, ef, ef)
    assert torch.all(met.cpu() == 0)
    with pytest.raises(_lib.TrainMathError) as ex:
        tm.pg_loss_fwd_bwd(logits, i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"]), z, z,
                           _lib.default_loss_params(inv_temperature=0.0))
    assert ex.value.code == _lib.CONFIG_ERROR


def test_config_errors_are_reported(tm, orc):
    """Bad arguments return ConfigError (21) with a message, never a launch."""
    from paper_2604_11554_b200 import _lib

    prob = orc.synth_problem(4, [5], 4096, "bf16")
    x = to_dev_logits(prob)
    t, o, r = i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"])
    z = torch.zeros(5, device="cuda")
    bad = [dict(kl_mode=7), dict(norm_mode=9), dict(masked_rows=5), dict(inv_temperature=-1.0),
           dict(kl_beta=float("nan"))]
    for kw in bad:
        with pytest.raises(_lib.TrainMathError) as ex:
            tm.pg_loss_fwd_bwd(x, t, o, r, z, z, _lib.default_loss_params(**kw))
        assert ex.value.code == _lib.CONFIG_ERROR and str(ex.value), kw
    with pytest.raises(_lib.TrainMathError) as ex:  # the fused vocab-parallel call needs open mailboxes
        tm.vp_fused_loss_fwd_bwd(x, 0, t, o, r, z, z)
    assert ex.value.code == _lib.CONFIG_ERROR
    with pytest.raises(_lib.TrainMathError) as ex:  # no CPU path
        tm.pg_loss_fwd_bwd(x.cpu(), t, o, r, z, z)
    assert ex.value.code == _lib.CONFIG_ERROR


def test_pg_step_host_matches_oracle_pipeline(tm, orc):
    from paper_2604_11554_b200 import _lib

    prob = orc.synth_problem(21, [50, 40, 33, 61, 12, 70, 8, 30], 32000, "bf16", prompt_max=20, G=4)
    logits = to_dev_logits(prob)
    pin = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).pin_memory()
    hm, dl = tm.pg_step_host(logits, pin(prob["targets"], np.int32), pin(prob["old"], np.float32),
                             pin(prob["ref"], np.float32), pin(prob["lens"], np.int32), pin(prob["rewards"], np.float32),
                             pin(prob["gids"], np.int32), h_prompt_lens=pin(prob["plens"], np.int32))
    torch.cuda.synchronize()
    cu, _, mask, _ = orc.varlen_meta(prob["lens"], prob["plens"])
    adv, _ = orc.grpo_advantage(prob["rewards"], prob["gids"])
    at, wt = orc.token_weights(cu, adv.astype(np.float32), mask, prob["T"])
    om, odl, olp, _, og = orc.pg_loss_fwd_bwd(prob["logits"], prob["targets"], prob["old"], prob["ref"],
                                              at.astype(np.float32), wt.astype(np.float32))
    near = near_clip_rows(olp, prob["old"], at, 0.2, 0.28) & (wt != 0)
    assert_grad_close(grad_to_np(dl), odl, np.abs(og), "bf16", rows_ok=~near)
    gm = hm.numpy()
    assert gm[_lib.NUM_METRICS - 2] == om[6]
    if not near.any():
        assert_close(gm[:6], om[:6], atol=2e-5, rtol=1e-4, what="metrics")


def test_pg_step_host_pipelined_calls_match_synced(tm, orc):
    """Back-to-back seam calls (no sync between them) overlap each call's H2D and
    prologue with the previous call's loss in two alternating stages; results
    must equal the same calls made one at a time (stage reuse, stage growth,
    masks on/off, precomputed advantages)."""
    pin = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).pin_memory()
    probs = [orc.synth_problem(40 + i, lens, 32000, "bf16", prompt_max=20, G=2)
             for i, lens in enumerate([[30, 22], [64, 40, 9, 17], [300, 210, 5, 90, 77, 64], [12, 12],
                                       [500, 400], [33, 1, 70, 2]])]

    def call(i, p, x):
        args = [pin(p["targets"], np.int32), pin(p["old"], np.float32), pin(p["ref"], np.float32),
                pin(p["lens"], np.int32), pin(p["rewards"], np.float32), pin(p["gids"], np.int32)]
        kw = dict(h_prompt_lens=pin(p["plens"], np.int32)) if i % 3 != 2 else {}
        eps = -1.0 if i == 3 else 1e-6  # call 3: rewards taken as precomputed advantages
        return tm.pg_step_host(x, *args, adv_eps=eps, **kw)

    xs = [to_dev_logits(p) for p in probs]
    ref = []
    for i, (p, x) in enumerate(zip(probs, xs)):
        hm, dl = call(i, p, x)
        torch.cuda.synchronize()
        ref.append((hm.clone(), dl.clone()))
    for rep in range(2):
        outs = [call(i, p, x) for i, (p, x) in enumerate(zip(probs, xs))]
        torch.cuda.synchronize()
        for i, ((hm, dl), (rm, rd)) in enumerate(zip(outs, ref)):
            assert torch.equal(hm, rm), (rep, i)
            assert torch.equal(dl, rd), (rep, i)


# ---------------------------------------------------------------------------- a7 vocab parallel (1-GPU emulation)
@pytest.mark.parametrize("P", [2, 4])
def test_vocab_parallel_matches_fused(tm, orc, P):
    prob = orc.synth_problem(31, [20, 12], 151936, "bf16", prompt_max=4)
    logits = to_dev_logits(prob)
    cu, sid, mask, adv, adv_tok, w_tok = gpu_pipeline(tm, prob)
    tg = i32(prob["targets"])
    old, ref = f32(prob["old"]), f32(prob["ref"])
    met_f, dl_f, lp_f, _ = tm.pg_loss_fwd_bwd(logits, tg, old, ref, adv_tok, w_tok, want_logp=True)
    V = prob["V"]
    b = np.linspace(0, V, P + 1).astype(int) // 8 * 8
    b[-1] = V
    shards = [logits[:, b[i]:b[i + 1]].contiguous() for i in range(P)]
    stats = torch.stack([tm.vp_partial_stats(s, tg, int(b[i])) for i, s in enumerate(shards)])
    # partial stats vs oracle
    for i, s in enumerate(shards):
        ost = orc.vp_partial_stats(prob["logits"][:, b[i]:b[i + 1]], prob["targets"], int(b[i]))
        g = stats[i].cpu().numpy()
        assert_close(g[:, 0], ost[:, 0], what="m")
        assert_close(g[:, 1], ost[:, 1], atol=0, rtol=2e-6, what="s")
        assert np.array_equal(np.isnan(g[:, 3]), np.isnan(ost[:, 3]))
    dls, mets = [], []
    for i, s in enumerate(shards):
        m, d, lp, _ = tm.vp_loss_fwd_bwd(s, int(b[i]), stats, tg, old, ref, adv_tok, w_tok, want_logp=True)
        dls.append(d)
        mets.append(m)
        assert_close(lp.cpu().numpy(), lp_f.cpu().numpy(), atol=2e-6, rtol=2e-6, what="vp logp")
    dl = torch.cat(dls, 1)
    a = adv_tok.cpu().numpy()
    w = w_tok.cpu().numpy()
    om, odl, olp, _, og = orc.pg_loss_fwd_bwd(prob["logits"], prob["targets"], prob["old"], prob["ref"], a, w)
    near = near_clip_rows(olp, prob["old"], a, 0.2, 0.28)
    assert_grad_close(grad_to_np(dl), odl, np.abs(og), "bf16", rows_ok=~near)
    for m in mets[1:]:
        assert torch.equal(m, mets[0])  # identical on every rank
    assert_close(mets[0].cpu().numpy()[:6], met_f.cpu().numpy()[:6], atol=2e-6, rtol=2e-5, what="vp metrics")


# ---------------------------------------------------------------------------- a5 R3
@pytest.mark.parametrize("dtype,idx_dtype,renorm,E,k", [("f32", "i32", True, 128, 8), ("bf16", "u8", True, 128, 8),
                                                        ("f32", "i32", False, 128, 8), ("bf16", "i32", False, 128, 8),
                                                        ("f32", "u8", True, 64, 12), ("bf16", "i32", True, 256, 16),
                                                        ("f32", "i32", True, 192, 4)])
def test_r3_gate(tm, orc, dtype, idx_dtype, renorm, E, k):
    """k <= 8 runs 8-lane row groups, k <= 16 16-lane groups (E % 64 == 0)."""
    rng = np.random.default_rng(41)
    L, T = 4, 301  # L*T not a multiple of the 16-row backward chunk
    z = (rng.normal(size=(L, T, E)) * 2).astype(np.float32)
    if dtype == "bf16":
        zb = orc.f32_to_bf16_bits(z).reshape(L, T, E)
        z = orc.bf16_bits_to_f32(zb).reshape(L, T, E)
        zin, zt = zb, torch.from_numpy(zb.view(np.int16)).view(torch.bfloat16).cuda()
    else:
        zin, zt = z, torch.from_numpy(z).cuda()
    z[1, :3] = 0.0  # fully tied rows (P9)
    z[3, 100:200] = np.round(z[3, 100:200] / 2)  # coarse logits: many exact ties at the k-th value
    if dtype == "bf16":
        zin[1, :3] = 0
        zt[1, :3] = 0
        zin[3, 100:200] = orc.f32_to_bf16_bits(z[3, 100:200]).reshape(100, E)
        zt[3, 100:200] = torch.from_numpy(z[3, 100:200]).to(torch.bfloat16).cuda()
    else:
        zt[1, :3] = 0
        zt[3, 100:200] = torch.from_numpy(z[3, 100:200]).cuda()
    order = np.lexsort((np.broadcast_to(np.arange(E), z.shape), -z), axis=-1)
    rec = order[..., :k].copy()
    flip = rng.random((L, T)) < 0.05
    for l, t in zip(*np.nonzero(flip)):
        others = np.setdiff1d(np.arange(E), rec[l, t])
        rec[l, t, rng.integers(0, k)] = rng.choice(others)
    rec[2, :4, 1] = rec[2, :4, 0]  # duplicated recorded expert: not a top-k set (mismatch)
    rec[1, 3:6] = order[1, 3:6, 1:k + 1]  # shifted by one: a boundary swap
    rec[3, 100:200:3, k - 1] = order[3, 100:200:3, k]  # tied rows: swap in the next expert in
    # (logit desc, index asc) order -- an equal logit at a higher index is still a mismatch (P9)
    rec = rec.astype(np.uint8 if idx_dtype == "u8" else np.int32)
    rt = torch.from_numpy(rec).cuda()
    w, idx, mm = tm.r3_gate_fwd(zt, rt, renorm=renorm)
    ow, oidx, omm = orc.r3_gate_fwd(zin, rec, renorm=renorm)
    assert orc.digest(idx.cpu().numpy()) == orc.digest(oidx)  # replayed indices bit-exact
    assert np.array_equal(mm.cpu().numpy().astype(np.uint32), omm)
    assert omm[L] >= flip.sum()
    assert_close(w.cpu().numpy(), ow, atol=1e-6, rtol=1e-5, what="r3 w")
    dw = rng.normal(size=(L, T, k)).astype(np.float32)
    wg = w.cpu().numpy()
    dz = tm.r3_gate_bwd(zt, rt, w, torch.from_numpy(dw).cuda(), renorm=renorm)
    odz = orc.r3_gate_bwd(zin, rec, wg, dw, renorm=renorm)
    g = grad_to_np(dz.reshape(L * T, E)).reshape(L, T, E)
    if dtype == "bf16":
        from tests._cmp import bf16_ulp

        assert np.all(np.abs(g - odz) <= bf16_ulp(odz) + 1e-6)
    else:
        assert_close(g, odz, atol=1e-6, rtol=1e-5, what="r3 dz")


# ---------------------------------------------------------------------------- full-size properties
def test_full_vocab_large_batch_properties(tm, orc):
    """Config-2 width at a large row count: sampled rows vs the oracle, and
    size-independent properties on all rows (finite, masked rows zero, each
    row's gradient sums to ~0 since sum_v (onehot - p) = 0)."""
    from paper_2604_11554_b200 import _lib

    T, V = 8192, 151936
    logits = torch.empty(T, V, dtype=torch.bfloat16, device="cuda")
    g = torch.Generator(device="cpu").manual_seed(0)
    peak = torch.randint(0, V, (T,), generator=g).to(torch.int32).cuda()
    tm.synth_logits(logits, seed=1234, sigma=2.0, peak_id=peak)
    targets = torch.where(torch.rand(T, generator=g).cuda() < 0.5, peak,
                          torch.randint(0, V, (T,), generator=g).to(torch.int32).cuda()).to(torch.int32)
    logp0, _, _ = tm.logprob_fwd(logits, targets)
    old = (logp0 + 0.05 * torch.randn(T, generator=g).cuda()).float()
    ref = (logp0 + 0.1 * torch.randn(T, generator=g).cuda()).float()
    adv_tok = torch.randn(T, generator=g).cuda()
    w_tok = (torch.rand(T, generator=g).cuda() < 0.9).float() / T
    met, dl, logp, ent = tm.pg_loss_fwd_bwd(logits, targets, old, ref, adv_tok, w_tok, want_logp=True)
    torch.cuda.synchronize()
    act = (w_tok != 0)
    assert torch.all(dl[~act] == 0)
    rs = dl.float().sum(1)
    assert torch.all(rs.abs() <= 2e-3 * (torch.abs(w_tok) * 4 * (adv_tok.abs() + 1)) + 1e-7)
    assert torch.isfinite(met).all()
    assert met[_lib.NUM_METRICS - 2].item() == act.sum().item()
    rows = torch.randperm(T, generator=g)[:12].sort().values
    sub = logits[rows.cuda()].contiguous()
    sub_bits = sub.view(torch.int16).cpu().numpy().view(np.uint16)
    tg = targets[rows.cuda()].cpu().numpy()
    a = adv_tok[rows.cuda()].cpu().numpy()
    w = w_tok[rows.cuda()].cpu().numpy()
    o, r = old[rows.cuda()].cpu().numpy(), ref[rows.cuda()].cpu().numpy()
    om, odl, olp, oent, og = orc.pg_loss_fwd_bwd(sub_bits, tg, o, r, a, w)
    actn = w != 0
    assert_close(logp[rows.cuda()].cpu().numpy()[actn], olp[actn], what="logp")
    assert_close(ent[rows.cuda()].cpu().numpy()[actn], oent[actn], what="entropy")
    near = near_clip_rows(olp, o, a, 0.2, 0.28)
    assert_grad_close(grad_to_np(dl[rows.cuda()]), odl, np.abs(og), "bf16", rows_ok=~near)
    # metrics self-consistency: recompute sum w*H from per-row outputs
    wh = float((w_tok.double() * ent.double()).sum())
    assert abs(met[3].item() - wh) <= 1e-5 * abs(wh) + 1e-6


@pytest.mark.parametrize("NS", [1, 2, 4])
def test_row_stream_count_parity(NS):
    """Every row-stream count of the fused kernel (SFTM_LOSS_NS forces one where
    a row fits; the default picks by width) meets the same parity bar on the
    loss cases, the deep run-ahead cases (many one-chunk rows, partial last
    groups) and the all-rows race regression."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, SFTM_LOSS_NS=str(NS))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_parity.py", "-k",
                          "test_pg_loss_fwd_bwd or deep_runahead or all_rows or neg_inf",
                          "--timeout", "120"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]


@pytest.mark.parametrize("C", [2, 3, 4])
def test_cluster_size_parity(C):
    """Every multi-CTA cluster size the fused kernel can pick (SFTM_LOSS_C forces
    one; C = 1 is the default and runs in the main session) meets the same
    parity bar, including the deep run-ahead cases."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, SFTM_LOSS_C=str(C))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_parity.py", "-k",
                          "test_pg_loss_fwd_bwd or test_pg_loss_deterministic or deep_runahead or step_host or all_rows",
                          "--timeout", "120"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
