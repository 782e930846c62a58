# SPDX-License-Identifier: Apache-2.0
"""Bench lines for the other BASELINE.json configs (bench.py --config N).

The driver's headline is configs[1] (bench.py default). These modes measure the
remaining SURVEY.md §8 rows on their own BASELINE shapes, with the same JSON
line layout (value, e2e where a host seam exists, roofline of the dominant
kernel, clocks):

  --config 1  CPU-ref GRPO step math: 16 prompts x 8 rollouts, <=1k tok packed
              varlen, vocab 32k fp32 logits (a1+a3+a4+a2+a6, one launch per step)
  --config 3  Qwen3-30B-A3B R3 replay: 128 experts top-8, 48 layers, recorded vs
              trainer router (a5 fwd+bwd over the config-2 micro-batch tokens)
  --config 4  Qwen3-Omni long packed sequences: 16k tokens, prompt + image/audio
              spans masked, DAPO + KL (beta 0.05), Qwen vocab bf16
  --config 5  vocab-parallel fused loss over P = n_gpus ranks: one single-pass
              kernel per rank, per-row partials exchanged in-kernel through
              NVLink peer mailboxes (--vp-two-pass: stats kernel + NCCL
              all_gather + backward kernel), 4 micro-batches of 32 x 4096
              tokens per step, staleness-tagged samples
"""
from __future__ import annotations

import json
import os
import time

import numpy as np

METRIC_LOSS = "tokens/s fused logprob+GRPO loss fwd+bwd (Qwen3-4B vocab); % HBM roofline"


def _peak():
    from bench import ROOT

    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _timed(fn, steps, warmup, dev, world, dist, stream):
    import torch

    from bench import ClockSampler

    for _ in range(warmup):
        fn(False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(dev.index)
    clk.start()
    time.sleep(0.25)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    kms = []
    for _ in range(steps):
        kms += fn(True)
    t1.record(stream)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    ms = torch.tensor([t0.elapsed_time(t1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    kt = [a.elapsed_time(b) for a, b in kms]
    return float(ms.item()) / steps, float(np.mean(kt)) if kt else None, clocks


def _line(args, world, metric, value, ms_step, dtype, config, roofline, clocks, launches, e2e=None, extra=None):
    d = {"metric": metric, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
         "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
         "scaling": config.pop("_scaling", "weak"), "vs_baseline": None, "dtype": dtype,
         "data": "synthetic (seeded)", "config": config, "roofline": roofline, "cpu_baseline": None,
         "e2e": e2e, "gpu_launches": launches, "clocks": clocks}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)


def _varlen_batch(rng, n_seq, lmin, lmax, G, spans=0, span_lo=256, span_hi=2048, fixed_len=None):
    lens = (np.full(n_seq, fixed_len) if fixed_len else rng.integers(lmin, lmax + 1, size=n_seq)).astype(np.int32)
    plens = np.minimum(rng.integers(32, 513, size=n_seq), lens - 1).astype(np.int32)
    T = int(lens.sum())
    mask = np.ones(T, np.uint8)
    cu = np.concatenate([[0], np.cumsum(lens)])
    for b in range(n_seq):
        mask[cu[b]:cu[b] + plens[b]] = 0
        for _ in range(spans):  # image/audio token spans (omni, config 4)
            L = int(rng.integers(span_lo, span_hi + 1))
            s0 = int(rng.integers(plens[b], max(plens[b] + 1, lens[b] - L)))
            mask[cu[b] + s0:cu[b] + min(lens[b], s0 + L)] = 0
    rewards = (rng.random(n_seq) < 0.5).astype(np.float32)
    gids = (np.arange(n_seq) // G).astype(np.int32)
    return T, lens, plens, mask, rewards, gids


def run_loss_config(args, cfg, world, rank, dev, dist):
    """Configs 1 and 4: the fused loss on their own shapes (single-GPU per rank)."""
    import torch

    from paper_2604_11554_b200 import _lib, train_math as tm

    rng = np.random.default_rng(2000 + rank)
    if cfg == 1:
        V, dt, es = 32000, torch.float32, 4
        T, lens, plens, mask, rewards, gids = _varlen_batch(rng, 16 * 8, 64, 1024, 8)
        M, beta, workload = 1, 0.0, "CPU-ref GRPO step: 16 prompts x 8 rollouts, <=1k tok packed varlen, V=32000 fp32"
        T_mb = T
    else:
        V, dt, es = 151936, torch.bfloat16, 2
        T, lens, plens, mask, rewards, gids = _varlen_batch(rng, 32, 0, 0, 8, spans=3, fixed_len=16384)
        M, beta = 4, 0.05
        workload = "Qwen3-Omni long packed: 4 x (8 seqs x 16384 tok), prompt + 3 image/audio spans masked, DAPO+KL"
        T_mb = T // M
    logits = torch.empty(T_mb, V, dtype=dt, device=dev)
    dlogits = torch.empty_like(logits)
    peak = torch.from_numpy(rng.integers(0, V, size=T_mb).astype(np.int32)).to(dev)
    tm.synth_logits(logits, seed=77 + rank, sigma=2.0, peak_id=peak)
    targets = torch.from_numpy(np.where(rng.random(T) < 0.5, np.tile(peak.cpu().numpy(), M),
                                        rng.integers(0, V, size=T)).astype(np.int32)).to(dev)
    logp0 = torch.empty(T, device=dev)
    for m in range(M):
        logp0[m * T_mb:(m + 1) * T_mb] = tm.logprob_fwd(logits, targets[m * T_mb:(m + 1) * T_mb])[0]
    g = torch.Generator(device=dev).manual_seed(11 + rank)
    old = (logp0 + 0.05 * torch.randn(T, device=dev, generator=g)).float()
    ref = (logp0 + 0.1 * torch.randn(T, device=dev, generator=g)).float()
    d_lens, d_rw, d_g = (torch.from_numpy(x).to(dev) for x in (lens, rewards, gids))
    d_mask = torch.from_numpy(mask).to(dev)
    from paper_2604_11554_b200 import data_parallel as dp

    n_act_local = int(mask.sum())
    n_act = dp.global_active_tokens(n_act_local, device=dev)  # global token-mean over the ranks
    params = _lib.default_loss_params(norm_mode=_lib.NORM_EXPLICIT, inv_norm=1.0 / n_act, kl_beta=beta)
    metrics = torch.zeros(M, _lib.NUM_METRICS, device=dev)
    stream = torch.cuda.current_stream(dev)
    h = tm.handle(dev.index)

    def step(rec):
        cu, _, _, _ = tm.varlen_meta(d_lens, T=T, want=("cu",))
        adv = tm.grpo_advantage(d_rw, d_g)
        adv_tok, w_tok = tm.token_weights(cu, adv, d_mask, T, _lib.NORM_EXPLICIT, 1.0 / n_act)
        ev = []
        for m in range(M):
            sl = slice(m * T_mb, (m + 1) * T_mb)
            e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) if rec else None
            if rec:
                e[0].record(stream)
            tm.pg_loss_fwd_bwd(logits, targets[sl], old[sl], ref[sl], adv_tok[sl], w_tok[sl], params,
                               dlogits=dlogits, metrics=metrics[m])
            if rec:
                e[1].record(stream)
                ev.append(e)
        return ev

    l0 = h.launch_count()
    ms_step, kms, clocks = _timed(step, args.steps, args.warmup, dev, world, dist, stream)
    launches = h.launch_count() - l0
    pk, src = _peak()
    act_mb = [int(mask[m * T_mb:(m + 1) * T_mb].sum()) for m in range(M)]  # this rank's rows
    by = float(np.mean([a * 2 * V * es + (T_mb - a) * V * es + 20 * T_mb for a in act_mb]))
    ach = by / (kms / 1e3) / 1e9
    _line(args, world, METRIC_LOSS if cfg == 4 else METRIC_LOSS.replace("(Qwen3-4B vocab)", "(32k vocab, fp32)"),
          n_act / (ms_step / 1e3), ms_step, "bf16" if es == 2 else "f32",
          {"workload": workload, "config_index": cfg, "vocab": V, "tokens_per_step": world * T,
           "loss_active_tokens_per_step": n_act, "value_counts": "loss-active tokens",
           "value_all_tokens": world * T / (ms_step / 1e3), "micro_batches": M, "kl_beta": beta,
           "l2": "inputs >> L2 (no flush)", "parallelism": f"dp{world}"},
          {"bound": "hbm", "achieved": ach, "peak": pk, "unit": "GB/s", "frac": ach / pk, "traffic": None,
           "peak_source": src, "algorithmic_bytes_per_launch": by, "avg_launch_ms": kms,
           "kernel": "{kernel}<{t},C={cluster}> grid {grid}".format(t="bf16" if es == 2 else "f32",
                                                                    **h.last_launch())}, clocks, int(launches))


def run_fwd_only(args, world, rank, dev, dist):
    """a1 forward only: per-token logp + entropy + lse of every token (the
    ActorFwd / RefLogP stage payloads), config-2 shape: 16 micro-batches of
    32 x 4096 tokens, Qwen3 vocab bf16. 2V bytes per token."""
    import torch

    from paper_2604_11554_b200 import train_math as tm

    V, M, T_mb = args.vocab, args.micro_batches, args.seqs_per_mb * args.seq_len
    logits = torch.empty(T_mb, V, dtype=torch.bfloat16, device=dev)
    tm.synth_logits(logits, seed=11 + rank, sigma=2.0)
    g = torch.Generator(device=dev).manual_seed(3 + rank)
    targets = torch.randint(0, V, (M * T_mb,), device=dev, dtype=torch.int32, generator=g)
    out_lp = torch.empty(M * T_mb, device=dev)
    out_h = torch.empty(M * T_mb, device=dev)
    stream = torch.cuda.current_stream(dev)
    h = tm.handle(dev.index)

    def step(rec):
        ev = []
        for m in range(M):
            sl = slice(m * T_mb, (m + 1) * T_mb)
            e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) if rec else None
            if rec:
                e[0].record(stream)
            lp, ent, _ = tm.logprob_fwd(logits, targets[sl])
            out_lp[sl].copy_(lp)
            out_h[sl].copy_(ent)
            if rec:
                e[1].record(stream)
                ev.append(e)
        return ev

    l0 = h.launch_count()
    ms_step, kms, clocks = _timed(step, args.steps, args.warmup, dev, world, dist, stream)
    launches = h.launch_count() - l0
    pk, src = _peak()
    by = T_mb * V * 2 + T_mb * 16
    ach = by / (kms / 1e3) / 1e9
    _line(args, world, "tokens/s fused logprob+entropy forward (ActorFwd/RefLogP, Qwen3-4B vocab)",
          world * M * T_mb / (ms_step / 1e3), ms_step, "bf16",
          {"workload": f"a1 forward only: {M} x ({args.seqs_per_mb} x {args.seq_len} tok), vocab {V} bf16",
           "tokens_per_step": world * M * T_mb, "vocab": V, "parallelism": f"dp{world}",
           "l2": "inputs >> L2 (no flush)"},
          {"bound": "hbm", "achieved": ach, "peak": pk, "unit": "GB/s", "frac": ach / pk, "traffic": None,
           "peak_source": src + " (copy = read+write; a read-only stream can exceed it)",
           "algorithmic_bytes_per_launch": by, "avg_launch_ms": kms,
           "kernel": "{kernel}<bf16,C={cluster}> grid {grid}".format(**h.last_launch()),
           "bytes_model": "2V B per token read + 16 B/token scalars"}, clocks, int(launches))


def run_r3(args, world, rank, dev, dist):
    """Config 3: R3 replay gate fwd+bwd, 48 layers x 128 experts top-8, fp32 router logits."""
    import torch

    from paper_2604_11554_b200 import train_math as tm

    L, E, k = 48, 128, 8
    T = 32 * 4096
    g = torch.Generator(device=dev).manual_seed(5 + rank)
    z = torch.randn(L, T, E, device=dev, generator=g) * 2
    top = torch.topk(z, k, dim=-1).indices
    swap = torch.rand(L, T, device=dev, generator=g) < 0.05  # 5% tokens: one expert replaced
    alt = (top[..., 0] + 1 + torch.randint(0, E - 1, (L, T), device=dev, generator=g)) % E
    rec = top.clone()
    rec[..., k - 1] = torch.where(swap & (alt[..., None] != top).all(-1), alt, top[..., k - 1])
    rec = rec.to(torch.uint8)
    dw = torch.randn(L, T, k, device=dev, generator=g)
    stream = torch.cuda.current_stream(dev)
    h = tm.handle(dev.index)
    out = {}
    # outputs preallocated once (a trainer reuses its buffers); the timed region
    # holds the two kernels and the mismatch-count reset
    bufs = (torch.empty(L, T, k, device=dev), torch.empty(L, T, k, dtype=torch.int32, device=dev),
            torch.empty(L + 1, dtype=torch.int32, device=dev), torch.empty_like(z))

    def step(rec_ev):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if rec_ev else None
        if rec_ev:
            e[0].record(stream)
        w, idx, mm = tm.r3_gate_fwd(z, rec, renorm=True, out=bufs[:3])
        if rec_ev:
            e[1].record(stream)
        tm.r3_gate_bwd(z, rec, w, dw, renorm=True, out=bufs[3])
        if rec_ev:
            e[2].record(stream)
        out["mm"] = mm
        return [(e[0], e[1]), (e[1], e[2])] if rec_ev else []

    l0 = h.launch_count()
    ms_step, kms, clocks = _timed(step, args.steps, args.warmup, dev, world, dist, stream)
    launches = h.launch_count() - l0
    pk, src = _peak()
    per_lt = (4 * E + k + 4 * k + 4 * k) + (k + 4 * k + 4 * k + 4 * E)  # fwd + bwd bytes per (layer, token)
    by = per_lt * L * T / 2  # per launch (fwd or bwd), averaged
    ach = by / (kms / 1e3) / 1e9
    mm = out["mm"].cpu().numpy()
    _line(args, world, "tokens/s R3 routing-replay gate fwd+bwd (48 layers x 128 experts, top-8)",
          world * T / (ms_step / 1e3), ms_step, "f32",
          {"workload": "Qwen3-30B-A3B R3 replay: L=48, E=128, k=8, recorded u8 indices vs trainer router, "
                       "32 x 4096 tokens", "config_index": 3, "tokens_per_step": world * T,
           "bytes_per_token_fwd_bwd": per_lt * L, "parallelism": f"dp{world}", "l2": "inputs >> L2"},
          {"bound": "hbm", "achieved": ach, "peak": pk, "unit": "GB/s", "frac": ach / pk, "traffic": None,
           "peak_source": src, "algorithmic_bytes_per_launch": by, "avg_launch_ms": kms,
           "kernel": "r3_fwd_kernel / r3_bwd_kernel"}, clocks, int(launches),
          extra={"r3_mismatch_tokens": int(mm[L]), "r3_mismatch_frac": float(mm[L]) / (L * T)})


def run_vocab_parallel(args, world, rank, dev, dist):
    """Config 5 as BASELINE.json states it: the vocab-parallel loss over P = world
    ranks (strong scaling: every rank holds a 1/P vocab shard of the SAME tokens)
    for one global step of 256 prompts x 16 rollouts = 4,096 packed sequences of
    1,024 tokens (4,194,304 tokens; 32 micro-batches of 128 sequences), GRPO over
    the 256 groups of 16, DAPO token-mean over the step, staleness-tagged samples
    (producer versions v_t - {0, 1, 2}; the per-micro-batch staleness histogram
    and batch staleness come from the C++ seam, staleness_histogram =
    StalenessGate::staleness_of, proj/src/staleness.cpp:169-173)."""
    import torch

    from paper_2604_11554_b200 import _lib, seam, train_math as tm
    from paper_2604_11554_b200.vocab_parallel import gather_stats, open_peer_exchange, shard_bounds

    V, P = args.vocab, world  # Qwen3's 151,936 unless --vocab (e.g. an odd vocabulary's last shard)
    b = shard_bounds(V, P)
    vs, Vp = b[rank], b[rank + 1] - b[rank]
    prompts, G, Ls, S = 256, 16, 1024, 128
    n_seq = prompts * G
    M = n_seq // S
    T_mb = S * Ls
    T = M * T_mb
    rng = np.random.default_rng(3000)  # same token data on every rank
    shard = torch.empty(T_mb, Vp, dtype=torch.bfloat16, device=dev)
    tm.synth_logits(shard, seed=900 + rank, sigma=2.0)
    targets = torch.from_numpy(rng.integers(0, V, size=T).astype(np.int32)).to(dev)
    plens = rng.integers(32, 257, size=n_seq)
    mask = np.ones(T, np.uint8)
    for s_ in range(n_seq):
        mask[s_ * Ls:s_ * Ls + plens[s_]] = 0
    n_act = int(mask.sum())
    rewards = (rng.random(n_seq) < 0.5).astype(np.float32)
    gids = (np.arange(n_seq) // G).astype(np.int32)
    # staleness tags (a8): producer versions of the samples vs trainer version v_t
    v_t = 10
    prod_ver = (v_t - rng.choice([0, 0, 0, 1, 1, 2], size=n_seq)).astype(np.int64)
    hist = np.zeros(8, np.uint64)
    batch_stale = []
    zeros_tok = np.zeros(T_mb, np.float32)
    for m in range(M):
        ss = slice(m * S, (m + 1) * S)
        mb = seam.MicroBatch(np.full(S, Ls), np.zeros(T_mb, np.int32), zeros_tok, zeros_tok, rewards[ss], False,
                             sample_ids=np.arange(m * S, (m + 1) * S) + 1, producer_versions=prod_ver[ss])
        batch_stale.append(mb.staleness(v_t, hist))
    stale_hist = {int(k): int(v) for k, v in enumerate(hist) if v}
    g = torch.Generator(device=dev).manual_seed(17)
    old = (-3.0 + 0.5 * torch.randn(T, device=dev, generator=g)).float()
    ref = (old + 0.1 * torch.randn(T, device=dev, generator=g)).float()
    cu, _, _, _ = tm.varlen_meta(torch.full((n_seq,), Ls, dtype=torch.int32, device=dev), T=T, want=("cu",))
    adv = tm.grpo_advantage(torch.from_numpy(rewards).to(dev), torch.from_numpy(gids).to(dev))  # G = 16
    adv_tok, w_tok = tm.token_weights(cu, adv, torch.from_numpy(mask).to(dev), T, _lib.NORM_EXPLICIT, 1.0 / n_act)
    params = _lib.default_loss_params(norm_mode=_lib.NORM_EXPLICIT, inv_norm=1.0 / n_act)
    dsh = torch.empty_like(shard)
    metrics = torch.zeros(M, _lib.NUM_METRICS, device=dev)
    stream = torch.cuda.current_stream(dev)
    h = tm.handle(dev.index)

    fused = not args.vp_two_pass
    if fused and P > 1 and not open_peer_exchange():
        fused = False  # no P2P path between the ranks: the two-pass NCCL form

    def step(rec):
        ev = []
        for m in range(M):
            sl = slice(m * T_mb, (m + 1) * T_mb)
            if fused:
                e = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if rec else None
                if rec:
                    e[0].record(stream)
                if P > 1:
                    tm.vp_fused_loss_fwd_bwd(shard, vs, targets[sl], old[sl], ref[sl], adv_tok[sl], w_tok[sl],
                                             params, dlogits=dsh, metrics=metrics[m])
                else:
                    tm.pg_loss_fwd_bwd(shard, targets[sl], old[sl], ref[sl], adv_tok[sl], w_tok[sl], params,
                                       dlogits=dsh, metrics=metrics[m])
                if rec:
                    e[1].record(stream)
                    ev.append((e[0], e[1]))
                continue
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if rec else None
            if rec:
                e[0].record(stream)
            st = tm.vp_partial_stats(shard, targets[sl], vs)
            if rec:
                e[1].record(stream)
            gathered = gather_stats(st) if P > 1 else st[None]
            if rec:
                e[2].record(stream)
            tm.vp_loss_fwd_bwd(shard, vs, gathered, targets[sl], old[sl], ref[sl], adv_tok[sl], w_tok[sl], params,
                               dlogits=dsh, metrics=metrics[m])
            if rec:
                e[3].record(stream)
                ev += [(e[0], e[1]), (e[2], e[3])]
        return ev

    l0 = h.launch_count()
    ms_step, kms, clocks = _timed(step, args.steps, args.warmup, dev, world, dist, stream)
    launches = h.launch_count() - l0
    pk, src = _peak()
    act_mb = n_act / M
    # algorithmic (minimum) bytes per rank per micro-batch: read the shard once, write its dlogits once
    by_min = act_mb * 4 * Vp + (T_mb - act_mb) * 2 * Vp
    # two-pass: the two kernels read the active shard rows twice (stats, then backward)
    by_design = by_min if fused else act_mb * 6 * Vp + (T_mb - act_mb) * 2 * Vp
    per_mb_ms = kms if fused else kms * 2  # two-pass: kms averages the two kernels
    ach = by_min / (per_mb_ms / 1e3) / 1e9
    if rank == 0:
        _line(args, world, "tokens/s vocab-parallel fused logprob+GRPO loss fwd+bwd (Qwen3-4B vocab)",
              n_act / (ms_step / 1e3), ms_step, "bf16",
              {"workload": f"vocab-parallel P={P}: 256 prompts x 16 rollouts x {Ls} tok ({M} micro-batches of "
                           f"{S} seqs), GRPO G=16, shard V/P={Vp}, staleness-tagged samples",
               "config_index": 5, "tokens_per_step": T, "loss_active_tokens_per_step": n_act,
               "value_counts": "loss-active tokens", "value_all_tokens": T / (ms_step / 1e3),
               "vocab": V, "vocab_shard": Vp, "batch_staleness_max": int(max(batch_stale)),
               "parallelism": (f"vocab-parallel tp{P} (" + ("in-kernel peer-mailbox exchange over NVLink, 32 B/row/peer"
                                                             if fused else "NCCL all-gather 16 B/token/rank") + ")"),
               "_scaling": "strong",
               "staleness_hist": stale_hist},
              {"bound": "hbm", "achieved": ach, "peak": pk, "unit": "GB/s", "frac": ach / pk, "traffic": None,
               "peak_source": src, "algorithmic_bytes_per_launch_pair": by_min, "design_bytes": by_design,
               "avg_kernel_ms": kms,
               "kernel": ("{kernel}<bf16,C={cluster}> grid {grid}".format(**h.last_launch()) if fused
                          else "rows_ring_kernel<bf16, VpStats|VpBwd>"),
               "bytes_model": "algorithmic 4V/P per active token (read+write once)" +
                              ("" if fused else "; the two-pass design reads the shard twice")},
              clocks, int(launches))
