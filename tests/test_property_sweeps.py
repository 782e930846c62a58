# SPDX-License-Identifier: Apache-2.0
"""Property sweeps (hypothesis) over shapes, dtypes, strides, masks and loss
parameters (SURVEY.md §8c asks for them next to the fixed parity cases).

CPU: invariants of the oracle and of the host logic (GRPO zero-mean/unit-std
groups, varlen offsets, shard bounds). GPU: the fused loss, the forward pass
and GRPO on random problems against the fp64 oracle, through whichever kernel
the dispatch picks (aligned, unaligned / sector-coordinate rows, clusters)."""
import numpy as np
import pytest

from tests._cmp import assert_close, assert_grad_close, loss_row_scale, near_clip_rows

hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

from oracle import oracle as orc  # noqa: E402

CPU = settings(max_examples=40, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])
GPU = settings(max_examples=60, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])


# ---------------------------------------------------------------------------- CPU
@CPU
@given(rewards=st.lists(st.sampled_from([0.0, 0.5, 1.0, 2.0]), min_size=2, max_size=40),
       G=st.integers(1, 8), mode=st.sampled_from([0, 1]))
def test_grpo_oracle_group_invariants(rewards, G, mode):
    r = np.asarray(rewards, np.float32)
    g = (np.arange(len(r)) // G).astype(np.int32)
    a, _ = orc.grpo_advantage(r, g, 1e-6, mode)
    for gid in np.unique(g):
        sel = g == gid
        if np.all(r[sel] == r[sel][0]):
            assert np.all(a[sel] == 0)  # P3: zero-variance groups give exactly 0
        else:
            assert abs(a[sel].mean()) < 1e-6
            n = sel.sum()
            sd = a[sel].std(ddof=1 if mode == 0 else 0) if n > 1 else 0
            assert abs(sd - 1) < 1e-4


@CPU
@given(lens=st.lists(st.integers(0, 50), min_size=1, max_size=30))
def test_varlen_oracle_offsets(lens):
    lens = np.asarray(lens, np.int32)
    cu, sid, mask, tg = orc.varlen_meta(lens)
    assert cu[0] == 0 and np.all(np.diff(cu) == lens) and cu[-1] == lens.sum()
    for b in range(len(lens)):
        assert np.all(sid[cu[b]:cu[b + 1]] == b)


@CPU
@given(V=st.integers(64, 300000), P=st.sampled_from([1, 2, 4, 8]))
def test_shard_bounds_properties(V, P):
    from paper_2604_11554_b200.vocab_parallel import shard_bounds

    b = shard_bounds(V, P)
    assert b[0] == 0 and b[-1] == V and all(b[i] < b[i + 1] for i in range(P))
    assert all(x % 8 == 0 for x in b[:-1])
    w = np.diff(b)
    assert w.max() - w.min() <= 8 + V % 8  # balanced to the alignment


# ---------------------------------------------------------------------------- GPU
def _torch():
    import torch

    return torch


@pytest.mark.gpu
@GPU
@given(seed=st.integers(0, 10 ** 6),
       V=st.sampled_from([16, 1000, 4099, 6144, 12289, 32000, 50257, 65536, 151936]),
       dtype=st.sampled_from(["bf16", "f32"]),
       nseq=st.integers(1, 5), L=st.integers(1, 40),
       pad=st.sampled_from([0, 0, 3, 8]),
       beta=st.sampled_from([0.0, 0.05]), ent=st.sampled_from([0.0, 0.01]),
       tau=st.sampled_from([1.0, 0.7]), dual=st.sampled_from([0.0, 3.0]), klm=st.sampled_from([0, 1, 2, 3]))
def test_fused_loss_sweep(seed, V, dtype, nseq, L, pad, beta, ent, tau, dual, klm):
    torch = _torch()
    from paper_2604_11554_b200 import _lib, train_math as tm

    rng = np.random.default_rng(seed)
    lens = rng.integers(1, L + 1, size=nseq)
    prob = orc.synth_problem(seed % 100000, lens, V, dtype, prompt_max=4)
    T = prob["T"]
    x = prob["logits"]
    # a row stride of V + pad elements (pad 3: rows off 16-B boundaries)
    if dtype == "bf16":
        base = torch.zeros(T, V + pad, dtype=torch.bfloat16, device="cuda")
        base[:, :V] = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
    else:
        base = torch.zeros(T, V + pad, dtype=torch.float32, device="cuda")
        base[:, :V] = torch.from_numpy(x).cuda()
    logits = base[:, :V]
    i32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()
    f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    a = rng.normal(size=T).astype(np.float32)
    w = (rng.random(T) < 0.85).astype(np.float32) / T
    p = _lib.default_loss_params(kl_beta=beta, entropy_coef=ent, inv_temperature=1 / tau, dual_clip_c=dual,
                                 kl_mode=klm)
    met, dl, logp, entr = tm.pg_loss_fwd_bwd(logits, i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"]),
                                             f32(a), f32(w), p, want_logp=True)
    lp2, ent2, _ = tm.logprob_fwd(logits, i32(prob["targets"]), inv_temperature=1 / tau)
    torch.cuda.synchronize()
    op = orc.params(p.clip_eps_low, p.clip_eps_high, p.dual_clip_c, p.kl_beta, p.entropy_coef, p.inv_temperature,
                    p.kl_mode)
    om, odl, olp, oent, og = orc.pg_loss_fwd_bwd(x, prob["targets"], prob["old"], prob["ref"], a, w, op)
    olp2, oent2, _ = orc.logprob_fwd(x, prob["targets"], 1 / tau)
    act = w != 0
    assert_close(logp.cpu().numpy()[act], olp[act], what="logp")
    assert_close(entr.cpu().numpy()[act], oent[act], what="entropy")
    assert_close(lp2.cpu().numpy(), olp2, what="forward logp")
    assert_close(ent2.cpu().numpy(), oent2, what="forward entropy")
    if dtype == "bf16":
        from oracle.oracle import bf16_bits_to_f32

        g = bf16_bits_to_f32(dl.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)).astype(np.float64)
    else:
        g = dl.cpu().numpy().astype(np.float64)
    near = near_clip_rows(olp, prob["old"], a, 0.2, 0.28, dual)
    scale = loss_row_scale(og, w, a, olp, prob["old"], prob["ref"], beta, klm, ent, 1 / tau)
    assert_grad_close(g, odl, scale, dtype, rows_ok=~near)
    assert met.cpu().numpy()[6] == om[6]


@pytest.mark.gpu
@GPU
@given(rewards=st.lists(st.sampled_from([0.0, 1.0, 0.25, 3.0]), min_size=1, max_size=300),
       G=st.integers(1, 16), mode=st.sampled_from([0, 1, 2]), shuffle=st.booleans())
def test_grpo_sweep(rewards, G, mode, shuffle):
    torch = _torch()
    from paper_2604_11554_b200 import train_math as tm

    r = np.asarray(rewards, np.float32)
    g = (np.arange(len(r)) // G).astype(np.int32)
    if shuffle:  # readiness order: groups interleaved, ids non-contiguous
        perm = np.random.default_rng(len(r)).permutation(len(r))
        r, g = r[perm], g[perm] * 7 + 3
    adv = tm.grpo_advantage(torch.from_numpy(r).cuda(), torch.from_numpy(g).cuda(), 1e-6, mode)
    oadv, _ = orc.grpo_advantage(r, g, 1e-6, mode)
    assert_close(adv.cpu().numpy(), oadv, atol=1e-6, rtol=1e-5, what="advantage")
