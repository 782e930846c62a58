# SPDX-License-Identifier: Apache-2.0
"""CPU, world_size 2 over gloo: the multi-GPU protocols of SURVEY.md §8e.

 * vocab-parallel (partitioning B): each rank computes its shard's partial
   statistics, the [P, T, 4] exchange runs through
   paper_2604_11554_b200.vocab_parallel.gather_stats, and the rank-order merge
   reproduces the full-row lse / entropy / logp on every rank;
 * sequence sharding (partitioning A, what bench.py --gpus N does): per-rank
   metric sums all-reduced equal the metrics of the union batch.
The per-rank compute here is the fp64 oracle (test infrastructure); the GPU
path runs the same protocol with the CUDA kernels (tests/test_gpu_parity.py).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _work(rank, world, q)
    except Exception as e:  # surface worker failures instead of a queue timeout
        q.put((rank, repr(e), False))
        raise
    finally:
        dist.destroy_process_group()


def _work(rank, world, q):
    from oracle import oracle as orc
    from paper_2604_11554_b200.vocab_parallel import gather_stats, shard_bounds

    orc.set_threads(1)
    # ---- vocab parallel
    prob = orc.synth_problem(5, [7, 6], 4000, "bf16", prompt_max=2)
    b = shard_bounds(prob["V"], world)
    a, e = b[rank], b[rank + 1]
    st = orc.vp_partial_stats(np.ascontiguousarray(prob["logits"][:, a:e]), prob["targets"], a)
    g = gather_stats(torch.from_numpy(st.astype(np.float64)))
    g = g.numpy()
    m = g[:, :, 0].max(0)
    S = (g[:, :, 1] * np.exp(g[:, :, 0] - m)).sum(0)
    W = (np.exp(g[:, :, 0] - m) * (g[:, :, 2] + g[:, :, 1] * (g[:, :, 0] - m))).sum(0)
    zy = np.nansum(g[:, :, 3], 0)
    lse = m + np.log(S)
    lp, ent, olse = orc.logprob_fwd(prob["logits"], prob["targets"])
    ok_vp = bool(np.allclose(lse, olse, atol=1e-12) and np.allclose(np.log(S) - W / S, ent, atol=1e-12)
                 and np.allclose(zy - lse, lp, atol=1e-12))
    # ---- sequence sharding: each rank owns half of the sequences
    full = orc.synth_problem(9, [5, 9, 4, 8], 512, "bf16", prompt_max=0)
    T = full["T"]
    w = np.full(T, 1.0 / T, np.float32)
    adv = np.linspace(-1, 1, T).astype(np.float32)
    cu = np.concatenate([[0], np.cumsum(full["lens"])])
    mine = np.arange(cu[2 * rank], cu[2 * rank + 2])
    met, _, _, _, _ = orc.pg_loss_fwd_bwd(full["logits"][mine], full["targets"][mine], full["old"][mine],
                                          full["ref"][mine], adv[mine], w[mine], want_dlogits=False)
    t = torch.from_numpy(met)
    dist.all_reduce(t)
    ref, _, _, _, _ = orc.pg_loss_fwd_bwd(full["logits"], full["targets"], full["old"], full["ref"], adv, w,
                                          want_dlogits=False)
    ok_dp = bool(np.allclose(t.numpy(), ref, rtol=1e-12, atol=1e-15))
    # ---- sequence sharding with UNEQUAL per-rank masks: the DAPO token-mean is
    # over the global batch, so every rank weights by 1 / (sum of all ranks'
    # active tokens) (data_parallel.global_inv_norm), not 1 / its own count
    from paper_2604_11554_b200 import data_parallel as dp

    full2 = orc.synth_problem(13, [6, 9, 7, 12], 512, "bf16", prompt_max=0)
    cu2 = np.concatenate([[0], np.cumsum(full2["lens"])])
    mask = np.ones(full2["T"], np.uint8)
    plen = [1, 5, 0, 3]  # ranks end up with 9+? active tokens each, unequal
    for s_ in range(4):
        mask[cu2[s_]:cu2[s_] + plen[s_]] = 0
    adv2 = np.linspace(-1, 1, full2["T"]).astype(np.float32)
    mine2 = np.arange(cu2[2 * rank], cu2[2 * rank + 2])
    local_active = int(mask[mine2].sum())
    inv = dp.global_inv_norm(local_active)
    w_loc = (mask[mine2] * inv).astype(np.float32)
    met2, _, _, _, _ = orc.pg_loss_fwd_bwd(full2["logits"][mine2], full2["targets"][mine2], full2["old"][mine2],
                                           full2["ref"][mine2], adv2[mine2], w_loc, want_dlogits=False)
    t2 = dp.reduce_step_metrics(torch.from_numpy(met2))
    w_all = (mask / mask.sum()).astype(np.float32)
    ref2, _, _, _, _ = orc.pg_loss_fwd_bwd(full2["logits"], full2["targets"], full2["old"], full2["ref"], adv2, w_all,
                                           want_dlogits=False)
    ok_dp2 = bool(np.allclose(t2.numpy(), ref2, rtol=1e-6, atol=1e-12))
    # the per-rank normaliser (round 1's bench) would not be the global token-mean
    w_bad = (mask[mine2] / max(local_active, 1)).astype(np.float32)
    met3, _, _, _, _ = orc.pg_loss_fwd_bwd(full2["logits"][mine2], full2["targets"][mine2], full2["old"][mine2],
                                           full2["ref"][mine2], adv2[mine2], w_bad, want_dlogits=False)
    t3 = dp.reduce_step_metrics(torch.from_numpy(met3))
    ok_dp2 = ok_dp2 and not np.allclose(t3.numpy()[5], ref2[5], rtol=1e-3)  # ratio ~ world x the mean
    q.put((rank, ok_vp, ok_dp and ok_dp2))


def test_two_rank_gloo_protocols():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_vp, ok_dp in res:
        assert ok_vp is True, f"vocab-parallel merge mismatch on rank {rank}: {ok_vp}"
        assert ok_dp, f"sequence-shard metric all-reduce mismatch on rank {rank}"


def _agree_worker(rank, world, port, q, fail_rank):
    """open_peer_exchange's collective decision with a (mocked) mailbox layer:
    one rank failing to map its peers makes every rank fall back."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_11554_b200 import train_math as tm
        from paper_2604_11554_b200 import vocab_parallel as vp

        opened = []
        tm.vp_mailbox_create = lambda P, r, dev=None: bytes([r]) * 64
        def _open(handles, dev=None):
            if rank == fail_rank:
                raise tm.TrainMathError(26, "no peer access (mock)")
            opened.append(len(handles))
        tm.vp_mailbox_open = _open
        ok = vp.open_peer_exchange()
        again = vp.open_peer_exchange()  # idempotent, no second exchange
        q.put((rank, ok, again, opened))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_peer_exchange_agreement(fail_rank):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, world, port, q, fail_rank)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = fail_rank < 0
    for rank, ok, again, opened in res:
        assert ok is want and again is want, (rank, ok, again)
        if rank != fail_rank:
            assert opened == [world]


def test_shard_bounds():
    from paper_2604_11554_b200.vocab_parallel import shard_bounds

    for V in (151936, 32000, 50257, 1000):
        for P in (1, 2, 4, 8):
            b = shard_bounds(V, P)
            assert b[0] == 0 and b[-1] == V and len(b) == P + 1
            assert all(x % 8 == 0 for x in b[:-1]) and all(b[i] < b[i + 1] for i in range(P))
    with pytest.raises(ValueError):
        shard_bounds(8, 4)
