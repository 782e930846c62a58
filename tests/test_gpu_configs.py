# SPDX-License-Identifier: Apache-2.0
"""GPU parity at the BASELINE.json config shapes and for the vocab-parallel
kernel on ONE GPU (the driver's GPU tier has one device):

- the fused vocab-parallel kernel (peer-mailbox exchange inside the kernel) at
  P = 1 (self-exchange) and P = 2 / 4 / 8 ranks emulated on one GPU (P handles
  wired as an in-process group, one stream per rank, the exchange grid capped
  so the P kernels are co-resident): every dlogits entry, logp and the metrics
  against the fp64 oracle, three launches in a row (both mailbox halves);
- a rank whose peer never launches: the kernel stops waiting, the handle
  reports Internal, the CUDA context stays usable;
- config 3 exactly as benchmarked: fp32 router logits, u8 recorded indices,
  48 layers x 128 experts, top-8;
- config 4 at its shape: 8 x 16,384-token sequences, prompt + 3 image/audio
  spans masked, DAPO + k3 KL (beta 0.05), Qwen3 vocabulary bf16.
All seeds are fixed constants.
"""
import numpy as np
import pytest

from tests._cmp import assert_close, assert_grad_close, loss_row_scale, metrics_from_rows, near_clip_rows

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def tm():
    from paper_2604_11554_b200 import train_math

    train_math.handle(0)
    return train_math


def to_dev(prob):
    x = prob["logits"]
    if x.dtype == np.uint16:
        return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(x).cuda()


def grad_np(dl):
    if dl.dtype == torch.bfloat16:
        from oracle.oracle import bf16_bits_to_f32

        return bf16_bits_to_f32(dl.view(torch.int16).cpu().numpy().view(np.uint16)).astype(np.float64)
    return dl.cpu().numpy().astype(np.float64)


i32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()
f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


# ---------------------------------------------------------------------------- a7 fused, emulated ranks
def _vp_group(tm, P):
    hs = [tm.Handle(0) for _ in range(P)]
    tm.vp_local_group(hs, 0 if P == 1 else 148 // P)
    return hs


@pytest.mark.parametrize("P,dtype,V,pkw", [(1, "bf16", 151936, {}), (1, "f32", 32000, {"kl_beta": 0.05}),
                                           (2, "bf16", 151936, {"entropy_coef": 0.01}), (4, "bf16", 151936, {}),
                                           (8, "bf16", 151936, {"kl_beta": 0.05}), (2, "f32", 32000, {}),
                                           # odd vocabularies: the last shard's rows are off 16-B boundaries
                                           # (sector coordinates) while the others are aligned
                                           (4, "bf16", 50257, {"entropy_coef": 0.01}), (8, "bf16", 50257, {}),
                                           (2, "f32", 32001, {"kl_beta": 0.05})])
def test_vp_fused_emulated_ranks(tm, orc, P, dtype, V, pkw):
    from paper_2604_11554_b200 import _lib
    from paper_2604_11554_b200.vocab_parallel import shard_bounds

    prob = orc.synth_problem(600 + 10 * P + len(pkw), [37, 20, 51, 9], V, dtype, prompt_max=6, G=2)
    T = prob["T"]
    logits = to_dev(prob)
    lens = i32(prob["lens"])
    cu, _, mask, _ = tm.varlen_meta(lens, i32(prob["plens"]), T=T, want=("cu", "mask"))
    adv = tm.grpo_advantage(f32(prob["rewards"]), i32(prob["gids"]))
    adv_tok, w_tok = tm.token_weights(cu, adv, mask, T)
    tg, old, ref = i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"])
    params = _lib.default_loss_params(**pkw)
    b = shard_bounds(V, P, 8 if dtype == "bf16" else 4)
    shards = [logits[:, b[r]:b[r + 1]].contiguous() for r in range(P)]
    hs = _vp_group(tm, P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    a, w = adv_tok.cpu().numpy(), w_tok.cpu().numpy()
    op = orc.params(params.clip_eps_low, params.clip_eps_high, params.dual_clip_c, params.kl_beta,
                    params.entropy_coef, params.inv_temperature, params.kl_mode)
    om, odl, olp, oent, og = orc.pg_loss_fwd_bwd(prob["logits"], prob["targets"], prob["old"], prob["ref"], a, w, op)
    act = w != 0
    near = near_clip_rows(olp, prob["old"], a, 0.2, 0.28) & act
    scale = loss_row_scale(og, w, a, olp, prob["old"], prob["ref"], params.kl_beta, params.kl_mode,
                           params.entropy_coef)
    cur = torch.cuda.current_stream()
    for launch in range(3):  # both mailbox halves, then the first again
        outs = []
        for s in streams:
            s.wait_stream(cur)
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                outs.append(tm.vp_fused_loss_fwd_bwd(shards[r], b[r], tg, old, ref, adv_tok, w_tok, params,
                                                     want_logp=True, h=hs[r], stream=streams[r]))
        torch.cuda.synchronize()
        assert hs[0].last_launch()["kernel"].startswith("loss_tmem_kernel[peer")
        for r in range(1, P):  # identical per-row scalars and metrics on every rank
            assert torch.equal(outs[r][0], outs[0][0]), (launch, r)
            assert torch.equal(outs[r][2], outs[0][2]), (launch, r)
        assert_close(outs[0][2].cpu().numpy()[act], olp[act], what=f"logp (P={P}, launch {launch})")
        assert_close(outs[0][3].cpu().numpy()[act], oent[act], what=f"entropy (P={P}, launch {launch})")
        dl = torch.cat([o[1] for o in outs], 1)
        assert_grad_close(grad_np(dl), odl, scale, dtype, rows_ok=~near, what=f"dlogits (P={P}, launch {launch})")
        gm = outs[0][0].cpu().numpy()
        assert gm[6] == om[6]
        if not near.any():
            tol = 1e-5 * (np.abs(w) * (np.abs(a) * 2 + 1)).sum() + 1e-6
            for i in (0, 1, 2, 3, 5, 7):
                assert abs(gm[i] - om[i]) <= tol * (30 if i in (2, 3) else 1) + 1e-5 * abs(om[i]), (i, gm[i], om[i])
    for hh in hs:
        hh.close()


def test_vp_fused_peer_timeout_is_an_error_not_a_trap(tm, orc):
    """Rank 1 of an emulated P = 2 group never launches: rank 0's kernel stops
    waiting after SF_TM_XP_TIMEOUT_S (tests/conftest.py: 10 s), completes, and
    every later fused call on its handle returns Internal; the context (and
    other handles) keep working."""
    from paper_2604_11554_b200 import _lib

    prob = orc.synth_problem(77, [8], 4096, "bf16", prompt_max=0)
    logits = to_dev(prob)
    T = prob["T"]
    w = torch.full((T,), 1.0 / T, device="cuda")
    a = torch.zeros(T, device="cuda")
    hs = _vp_group(tm, 2)
    half = logits[:, :2048].contiguous()
    tm.vp_fused_loss_fwd_bwd(half, 0, i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"]), a, w, h=hs[0])
    torch.cuda.synchronize()  # returns: no hang, no sticky CUDA error
    with pytest.raises(_lib.TrainMathError) as ex:
        tm.vp_fused_loss_fwd_bwd(half, 0, i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"]), a, w, h=hs[0])
    assert ex.value.code == _lib.INTERNAL and "timed out" in str(ex.value)
    met, _, _, _ = tm.pg_loss_fwd_bwd(logits, i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"]), a, w)
    torch.cuda.synchronize()
    assert met[6].item() == T
    for hh in hs:
        hh.close()


# ---------------------------------------------------------------------------- config 3 exactly
def test_config3_r3_exact_shape(tm, orc):
    """BASELINE configs[2] as bench.py --config 3 runs it: fp32 router logits,
    u8 recorded indices, L = 48, E = 128, k = 8 (here 2,048 tokens per layer)."""
    L, T, E, k = 48, 2048, 128, 8
    rng = np.random.default_rng(303)
    z = (rng.normal(size=(L, T, E)) * 2).astype(np.float32)
    order = np.argsort(-z, axis=-1, kind="stable")
    rec = order[..., :k].copy()
    swap = rng.random((L, T)) < 0.05
    for l, t in zip(*np.nonzero(swap)):
        rec[l, t, k - 1] = order[l, t, k + int(rng.integers(0, E - k))]
    rec = rec.astype(np.uint8)
    zt, rt = torch.from_numpy(z).cuda(), torch.from_numpy(rec).cuda()
    w, idx, mm = tm.r3_gate_fwd(zt, rt, renorm=True)
    ow, oidx, omm = orc.r3_gate_fwd(z, rec, renorm=True)
    assert orc.digest(idx.cpu().numpy()) == orc.digest(oidx)
    assert np.array_equal(mm.cpu().numpy().astype(np.uint32), omm)
    assert omm[L] == swap.sum()
    assert_close(w.cpu().numpy(), ow, atol=1e-6, rtol=1e-5, what="r3 w")
    dw = rng.normal(size=(L, T, k)).astype(np.float32)
    dz = tm.r3_gate_bwd(zt, rt, w, torch.from_numpy(dw).cuda(), renorm=True)
    odz = orc.r3_gate_bwd(z, rec, w.cpu().numpy(), dw, renorm=True)
    assert_close(dz.cpu().numpy(), odz, atol=1e-6, rtol=1e-5, what="r3 dz")


# ---------------------------------------------------------------------------- config 4 at its shape
def test_config4_omni_long_sequences(tm, orc):
    """BASELINE configs[3]: 8 packed 16,384-token sequences (131,072 rows x
    151,936 bf16 in one launch), prompt + 3 image/audio spans masked, DAPO +
    k3 KL (beta 0.05). Packing metadata and weights bit-exact; sampled rows
    (every dlogits entry) against the fp64 oracle; every row's logp/entropy
    against the streaming forward kernel; the step metrics against a fp64
    re-reduction of the kernel's own per-row outputs; every masked row zero
    and every active row's gradient summing to ~0."""
    from bench_extra import _varlen_batch
    from paper_2604_11554_b200 import _lib

    V, beta = 151936, 0.05
    rng = np.random.default_rng(404)
    T, lens, plens, mask, rewards, gids = _varlen_batch(rng, 8, 0, 0, 8, spans=3, fixed_len=16384)
    logits = torch.empty(T, V, dtype=torch.bfloat16, device="cuda")
    peak = rng.integers(0, V, size=T).astype(np.int32)
    tm.synth_logits(logits, seed=4040, sigma=2.0, peak_id=i32(peak))
    targets = np.where(rng.random(T) < 0.5, peak, rng.integers(0, V, size=T)).astype(np.int32)
    tg = i32(targets)
    lp0, ent0, _ = tm.logprob_fwd(logits, tg)
    g = torch.Generator(device="cuda").manual_seed(404)
    old = (lp0 + 0.05 * torch.randn(T, device="cuda", generator=g)).float()
    ref = (lp0 + 0.1 * torch.randn(T, device="cuda", generator=g)).float()
    cu, _, pmask, _ = tm.varlen_meta(i32(lens), i32(plens), T=T, want=("cu", "mask"))
    ocu, _, opmask, _ = orc.varlen_meta(lens, plens)
    assert orc.digest(cu.cpu().numpy()) == orc.digest(ocu)
    assert orc.digest(pmask.cpu().numpy()) == orc.digest(opmask)
    adv = tm.grpo_advantage(f32(rewards), i32(gids))
    oadv, _ = orc.grpo_advantage(rewards, gids)
    assert_close(adv.cpu().numpy(), oadv, atol=1e-6, rtol=1e-6, what="advantage")
    d_mask = torch.from_numpy(mask).cuda()
    adv_tok, w_tok = tm.token_weights(cu, adv, d_mask, T)
    oat, owt = orc.token_weights(ocu, adv.cpu().numpy(), mask, T)
    assert np.array_equal(adv_tok.cpu().numpy(), oat.astype(np.float32))
    assert np.array_equal(w_tok.cpu().numpy(), owt.astype(np.float32))
    params = _lib.default_loss_params(kl_beta=beta)
    met, dl, logp, ent = tm.pg_loss_fwd_bwd(logits, tg, old, ref, adv_tok, w_tok, params, want_logp=True)
    torch.cuda.synchronize()
    act_t = w_tok != 0
    act = act_t.cpu().numpy()
    # every row vs the streaming forward kernel
    bad = ((logp - lp0).abs() > 2e-5 + 2e-6 * lp0.abs()) & act_t
    bad |= ((ent - ent0).abs() > 2e-5 + 2e-5 * ent0.abs()) & act_t
    assert int(bad.sum()) == 0
    # metrics: the kernel's deterministic reduction vs fp64 over its own rows
    gm = met.cpu().numpy()
    rm = metrics_from_rows(logp.cpu().numpy(), ent.cpu().numpy(), old.cpu().numpy(), ref.cpu().numpy(),
                           adv_tok.cpu().numpy(), w_tok.cpu().numpy(), beta=beta)
    assert gm[6] == rm[6] == int(mask.sum())
    for i in (0, 1, 2, 3, 4, 5, 7):
        assert abs(gm[i] - rm[i]) <= 1e-5 * abs(rm[i]) + 1e-7, (i, gm[i], rm[i])
    # every row: masked rows zero-filled, active rows' gradients sum to ~0
    wt, at = w_tok, adv_tok
    for c0 in range(0, T, 8192):
        blk = dl[c0:c0 + 8192]
        m = act_t[c0:c0 + 8192]
        assert not bool((blk[~m] != 0).any())
        rs = blk.float().sum(1)
        lim = 2e-3 * (wt[c0:c0 + 8192].abs() * 4 * (at[c0:c0 + 8192].abs() + 1 + 10 * beta)) + 1e-7
        assert bool((rs.abs() <= lim).all())
    # sampled rows, every entry, vs the fp64 oracle (span / prompt boundaries included)
    edges = np.flatnonzero(np.diff(mask.astype(np.int8)) != 0)
    pick = np.unique(np.concatenate([edges[:8], edges[:8] + 1, rng.choice(T, 8, replace=False)]))
    pick = pick[pick < T]
    rows = torch.from_numpy(pick).cuda()
    sub = logits[rows].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    o, r = old[rows].cpu().numpy(), ref[rows].cpu().numpy()
    a, w = adv_tok[rows].cpu().numpy(), w_tok[rows].cpu().numpy()
    om, odl, olp, oent, og = orc.pg_loss_fwd_bwd(sub, targets[pick], o, r, a, w, orc.params(beta=beta))
    an = w != 0
    assert_close(logp[rows].cpu().numpy()[an], olp[an], what="logp")
    assert_close(ent[rows].cpu().numpy()[an], oent[an], what="entropy")
    near = near_clip_rows(olp, o, a, 0.2, 0.28)
    scale = loss_row_scale(og, w, a, olp, o, r, beta)
    assert_grad_close(grad_np(dl[rows]), odl, scale, "bf16", rows_ok=~near)
    del logits, dl
    torch.cuda.empty_cache()


# ---------------------------------------------------------------------------- a5 transport (f4)
@pytest.mark.parametrize("T,L,k,dt", [(2048, 48, 8, "u8"), (301, 5, 3, "u8"), (77, 33, 16, "i32"), (1000, 7, 32, "i32"),
                                      (33, 48, 1, "u8"), (4096, 48, 8, "i32")])
def test_r3_record_token_to_layer_major_bit_exact(tm, orc, T, L, k, dt):
    """The routed_experts record as the bus carries it (token-major [T, L, k])
    transposed on the device to the gate's layer-major [L, T, k]: FNV digest
    equal to the host transpose, and the gate on it equal to the gate on the
    host-transposed record."""
    rng = np.random.default_rng(T + L + k)
    npdt = np.uint8 if dt == "u8" else np.int32
    rec_tok = rng.integers(0, 128, size=(T, L, k)).astype(npdt)
    out = tm.r3_record_layer_major(torch.from_numpy(rec_tok).cuda())
    host = np.ascontiguousarray(rec_tok.transpose(1, 0, 2))
    assert orc.digest(out.cpu().numpy()) == orc.digest(host)
    if k <= 16 and dt == "u8":
        z = torch.from_numpy((rng.normal(size=(L, T, 128)) * 2).astype(np.float32)).cuda()
        w1, i1, m1 = tm.r3_gate_fwd(z, out)
        w2, i2, m2 = tm.r3_gate_fwd(z, torch.from_numpy(host).cuda())
        assert torch.equal(w1, w2) and torch.equal(i1, i2) and torch.equal(m1, m2)


# ---------------------------------------------------------------------------- argument checks / bounds
def test_pg_step_host_rejects_bad_dlogits_stride(tm, orc):
    """the host seam call validates ld_d >= V and the in-place stride
    like the device call (ConfigError before any copy is issued)."""
    from paper_2604_11554_b200 import _lib

    prob = orc.synth_problem(8, [6, 5], 4096, "bf16", prompt_max=2, G=2)
    x = to_dev(prob)
    pin = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).pin_memory()
    args = [pin(prob["targets"], np.int32), pin(prob["old"], np.float32), pin(prob["ref"], np.float32),
            pin(prob["lens"], np.int32), pin(prob["rewards"], np.float32), pin(prob["gids"], np.int32)]
    narrow = torch.empty(prob["T"], 4000, dtype=torch.bfloat16, device="cuda")  # ld_d = 4000 < V
    with pytest.raises(_lib.TrainMathError) as ex:
        tm.pg_step_host(x, *args, dlogits=narrow)
    assert ex.value.code == _lib.CONFIG_ERROR and "ld_d" in str(ex.value)
    wide = torch.zeros(prob["T"], 4104, dtype=torch.bfloat16, device="cuda")
    wide[:, :4096] = x
    view = wide[:, :4096]
    h = tm.handle(0)
    params = _lib.default_loss_params()
    met = torch.empty(_lib.NUM_METRICS).pin_memory()
    # dlogits == logits but with another row stride: refused
    rc = _lib.lib().sf_tm_pg_step_host(h.ptr, tm._p(view), _lib.BF16, prob["T"], 4096, 4104, tm._p(args[0]),
                                       tm._p(args[1]), tm._p(args[2]), None, tm._p(args[3]), None, tm._p(args[4]),
                                       tm._p(args[5]), len(prob["lens"]), 1e-6, 0, ctypes_byref(params),
                                       tm._p(view), 4096, tm._p(met), tm._stream(0))
    assert rc == _lib.CONFIG_ERROR


def ctypes_byref(p):
    import ctypes

    return ctypes.byref(p)


def test_kernels_write_nothing_outside_their_outputs(tm, orc):
    """A bounds check in place of compute-sanitizer (closed on this pool): every
    output buffer of every kernel family is allocated with sentinel guard
    regions before and after (and guard columns around strided rows), and the
    guards must be untouched after the call."""
    from paper_2604_11554_b200 import _lib

    G = 4096  # guard elements on each side

    def guarded(n, dtype, fill):
        buf = torch.full((n + 2 * G,), fill, dtype=dtype, device="cuda")
        return buf, buf[G:G + n]

    def check(buf, fill, what):
        torch.cuda.synchronize()
        assert torch.all(buf[:G] == fill) and torch.all(buf[-G:] == fill), f"{what}: write outside the output"

    cases = [("bf16", 151936, [9, 4]), ("bf16", 262144, [3]), ("bf16", 50257, [7, 5]), ("f32", 32000, [6, 6]),
             ("bf16", 18992, [40, 33])]
    for dt, V, lens in cases:
        prob = orc.synth_problem(V % 1000, lens, V, dt, prompt_max=3)
        x = to_dev(prob)
        T = prob["T"]
        tdt = x.dtype
        buf, dl = guarded(T * V, tdt, 7.0)
        dl = dl.view(T, V)
        cu, _, mask, _ = tm.varlen_meta(i32(prob["lens"]), i32(prob["plens"]), T=T, want=("cu", "mask"))
        adv = tm.grpo_advantage(f32(prob["rewards"]), i32(prob["gids"]))
        at, wt = tm.token_weights(cu, adv, mask, T)
        mbuf, met = guarded(_lib.NUM_METRICS, torch.float32, -5.0)
        lbuf, lp = guarded(T, torch.float32, -5.0)
        ebuf, en = guarded(T, torch.float32, -5.0)
        rc = _lib.lib().sf_tm_pg_loss_fwd_bwd(tm.handle(0).ptr, tm._p(x), _lib.BF16 if dt == "bf16" else _lib.F32, T, V,
                                              V, tm._p(i32(prob["targets"])), tm._p(f32(prob["old"])),
                                              tm._p(f32(prob["ref"])), tm._p(at), tm._p(wt),
                                              ctypes_byref(_lib.default_loss_params()), tm._p(dl), V, tm._p(met),
                                              tm._p(lp), tm._p(en), tm._stream(0))
        assert rc == 0
        for b_, f_, w_ in ((buf, 7.0, "dlogits"), (mbuf, -5.0, "metrics"), (lbuf, -5.0, "logp"), (ebuf, -5.0, "H")):
            check(b_, f_, f"{w_} {dt} V={V}")
        # forward-only outputs
        for b_, f_ in ((lbuf, -5.0), (ebuf, -5.0)):
            b_.fill_(f_)
        rc = _lib.lib().sf_tm_logprob_fwd(tm.handle(0).ptr, tm._p(x), _lib.BF16 if dt == "bf16" else _lib.F32, T, V,
                                          V, tm._p(i32(prob["targets"])), 1.0, tm._p(lp), tm._p(en), None,
                                          tm._stream(0))
        assert rc == 0
        check(lbuf, -5.0, "fwd logp")
        check(ebuf, -5.0, "fwd entropy")
    # R3 outputs and the record transpose
    L, T, E, k = 3, 301, 128, 8
    z = torch.randn(L, T, E, device="cuda")
    rec = torch.topk(z, k, dim=-1).indices.to(torch.uint8)
    wbuf, w = guarded(L * T * k, torch.float32, -5.0)
    ibuf, idx = guarded(L * T * k, torch.int32, -5)
    mmb, mm = guarded(L + 1, torch.int32, -5)
    tm.r3_gate_fwd(z, rec, out=(w.view(L, T, k), idx.view(L, T, k), mm))
    for b_, f_, n_ in ((wbuf, -5.0, "r3 w"), (ibuf, -5, "r3 idx"), (mmb, -5, "r3 mismatch")):
        check(b_, f_, n_)
    dzb, dz = guarded(L * T * E, torch.float32, -5.0)
    tm.r3_gate_bwd(z, rec, w.view(L, T, k), torch.randn(L, T, k, device="cuda"), out=dz.view(L, T, E))
    check(dzb, -5.0, "r3 dz")
    rb, r = guarded(L * T * k, torch.uint8, 201)
    tm.r3_record_layer_major(rec.permute(1, 0, 2).contiguous(), out=r.view(L, T, k))
    check(rb, 201, "record transpose")


@pytest.mark.parametrize("B,G", [(1, 1), (7, 3), (4096, 16), (16384, 8), (16385, 5), (20000, 16)])
def test_grpo_advantage_sizes(tm, orc, B, G):
    """The sorted single-CTA GRPO kernel (B <= 16,384) and the per-sample scan
    kernel beyond it: group sizes bit-exact, advantages vs the fp64 oracle,
    zero-variance groups exactly 0, groups in arbitrary (readiness) order."""
    rng = np.random.default_rng(B)
    gids = rng.permutation(np.arange(B) // G).astype(np.int32) * 7 - 3  # non-contiguous, negative ids too
    r = (rng.random(B) < 0.5).astype(np.float32)
    r[: min(B, 40)] = 1.0  # some all-equal groups
    adv, gs = tm.grpo_advantage(f32(r), i32(gids), 1e-6, 0, want_group_size=True)
    oadv, ogs = orc.grpo_advantage(r, gids)
    assert np.array_equal(gs.cpu().numpy(), ogs)
    got = adv.cpu().numpy()
    assert_close(got, oadv, atol=1e-6, rtol=1e-6, what="advantage")
    assert np.all(got[oadv == 0.0] == 0.0)
