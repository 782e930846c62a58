# SPDX-License-Identifier: Apache-2.0
"""Benchmark of the fused logprob + GRPO/DAPO loss fwd+bwd hot path on B200.

Metric (BASELINE.json): "tokens/s fused logprob+GRPO loss fwd+bwd (Qwen3-4B
vocab); % HBM roofline". Workload = BASELINE.json configs[1] (the Qwen3-4B
shape): one step is the whole global batch of 64 prompts x 8 rollouts = 512
packed sequences of 4,096 tokens (2,097,152 tokens, vocab 151,936, bf16 logits,
fp32 accumulation), processed as 16 trainer micro-batches of 32 sequences
(StreamLoader micro_batch_size 32, proj/include/staleflow/stream_loader.hpp:19).
Per step: varlen packing metadata, GRPO group advantages over the 512 rollouts,
per-token loss weights (DAPO token-mean over the step), then per
micro-batch the fused loss fwd+bwd writing dlogits. The per-micro-batch logits
(39.8 GB bf16) stay resident in HBM — in the trainer they are the LM-head
output, which never crosses the bus — and are far larger than L2 (126 MB), so
no L2 flush is needed between steps. Data are synthetic (seeded SplitMix64).

`value` counts loss-active tokens (mask = 1); `value_all_tokens`
adds the masked prompt rows. `e2e` is the same metric through the C++ trainer
seam (ActorLossSeam::step via libsf_seam.so) on MicroBatch payloads as the bus
delivers them, host->device copies included.

Multi-GPU: one process per GPU (torchrun), weak scaling — each rank processes
its own global batch of sequences; before the step the ranks sum their
loss-active token counts (one 8-byte all-reduce) so every rank weights by the
global token-mean, and after it one all-reduce of the step metrics.

`--impl reference`: the reference has no implementation of this path
(SPEC.md:8); its CPU arm is the repo's fp32 port of the oracle (oracle/), run on
all host threads on 4,096 rows of the same workload per step (>= 10 s timed),
with the CPU model and a one-thread rate recorded.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

V_QWEN3 = 151936
METRIC = "tokens/s fused logprob+GRPO loss fwd+bwd (Qwen3-4B vocab); % HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--seqs-per-mb", type=int, default=32)
    ap.add_argument("--micro-batches", type=int, default=16)
    ap.add_argument("--seq-len", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=V_QWEN3)
    ap.add_argument("--group", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline sample duration")
    ap.add_argument("--generic", action="store_true", help="force the generic two-pass kernel (comparison)")
    ap.add_argument("--fwd-only", action="store_true",
                    help="a1 forward only (ActorFwd / RefLogP logp+entropy) on the config-2 micro-batch shape")
    ap.add_argument("--vp-two-pass", action="store_true",
                    help="config 5: stats kernel + NCCL all_gather + backward kernel instead of the fused "
                         "single-pass kernel with the in-kernel peer exchange (comparison)")
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (1-based); 2 = the headline (default)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ workload
def make_step_inputs(rng: np.random.Generator, n_seq: int, L: int, V: int, G: int):
    """Per-step host-side bus fields for n_seq packed sequences of length L."""
    T = n_seq * L
    lens = np.full(n_seq, L, np.int32)
    plens = rng.integers(32, 513, size=n_seq).astype(np.int32)  # prompt prefix masked
    rewards = (rng.random(n_seq) < 0.5).astype(np.float32)
    gids = (np.arange(n_seq) // G).astype(np.int32)
    return T, lens, plens, rewards, gids


def cpu_model() -> str:
    """The host CPU model (the CPU baseline depends on it; boxes differ)."""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def _time_cpu(run, target_s: float):
    """Repeat run() until ~target_s of CPU time has been measured; (passes, seconds)."""
    run()  # warm (page-in, thread pool)
    reps, dt = 0, 0.0
    while dt < target_s or reps == 0:
        t0 = time.perf_counter()
        run()
        dt += time.perf_counter() - t0
        reps += 1
    return reps, dt


def cpu_rate_one_thread(orc, smp, target_s: float = 3.0):
    """Tokens/s of the same CPU port on ONE thread (a slice of the sample)."""
    cores = os.cpu_count() or 1
    rows = max(1, min(len(smp[0]), 16))
    sub = tuple(a[:rows] for a in smp)
    orc.set_threads(1)
    try:
        reps, dt = _time_cpu(lambda: orc.pg_loss_fwd_bwd_fast(*sub, orc.params()), target_s)
    finally:
        orc.set_threads(cores)
    return rows * reps / dt


def run_reference(args, rank: int):
    """CPU arm: the oracle's fp32 CPU port (the reference has no implementation of
    this path) on all host threads, on rows of the same workload
    (V = 151,936 bf16, every row loss-active). Each step is 4,096 rows -- the
    cpu_baseline leg's sample -- repeated so the timed steps hold >= 10 s of CPU
    work in total; the run stays within a few minutes."""
    if rank != 0:
        return
    from oracle import oracle as orc

    orc.lib()
    cores = os.cpu_count() or 1
    orc.set_threads(cores)
    rows = 4096
    prob = orc.synth_problem(7, [rows], args.vocab, "bf16", prompt_max=0)
    a = np.random.default_rng(0).normal(size=rows).astype(np.float32)
    w = np.full(rows, 1.0 / rows, np.float32)
    smp = (prob["logits"], prob["targets"], prob["old"], prob["ref"], a, w)
    p = orc.params()
    one = lambda: orc.pg_loss_fwd_bwd_fast(*smp, p)
    one()  # warm
    t0 = time.perf_counter()
    one()
    t_pass = time.perf_counter() - t0
    passes = max(1, int(np.ceil(10.0 / max(args.steps, 1) / t_pass)))  # >= 10 s over the timed steps
    budget = 240.0 / max(1, args.steps + args.warmup)  # the whole run within a few minutes
    passes = max(1, min(passes, int(budget / t_pass)))

    def step():
        for _ in range(passes):
            one()

    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    sec = float(np.mean(ts))
    tok_s = rows * passes / sec
    one_thread = cpu_rate_one_thread(orc, smp)
    sample = (f"{rows} loss-active rows x V={args.vocab} bf16, x {passes} passes per step "
              f"({sum(ts):.1f} s timed), fused loss fwd+bwd, fp32 vectorised CPU port (oracle/sf_cpu_fast.c), OpenMP")
    out = {
        "impl": "reference", "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded SplitMix64)",
        "config": {"workload": "Qwen3-4B shape (BASELINE configs[1]) row sample, every row loss-active",
                   "vocab": args.vocab, "rows_per_step": rows * passes, "logits": "bf16"},
        "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model(), "value_1thread": one_thread},
        "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "note": "the reference has no implementation of this path (SPEC.md:8); the timed CPU arm is the fp32 "
                "vectorised port of the oracle (the fp64 oracle is the parity truth)",
    }
    print(json.dumps(out), flush=True)


def cpu_baseline_leg(tm, logits, targets, old, ref, adv_tok, w_tok, vocab, target_s):
    """Time the CPU port on loss-active rows copied from the device workload
    (same data): all host threads, and one thread."""
    import torch
    from oracle import oracle as orc

    orc.lib()
    cores = os.cpu_count() or 1
    orc.set_threads(cores)
    act = torch.nonzero(w_tok != 0).flatten()

    def sample(n):
        idx = act[:n]
        sub = logits[idx].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        return (sub, targets[idx].cpu().numpy(), old[idx].cpu().numpy(), ref[idx].cpu().numpy(),
                adv_tok[idx].cpu().numpy(), w_tok[idx].cpu().numpy())

    n = 4096  # <= 2.5 GB of host logits + dlogits
    s = sample(n)
    reps, dt = _time_cpu(lambda: orc.pg_loss_fwd_bwd_fast(*s, orc.params()), target_s)
    one_thread = cpu_rate_one_thread(orc, s)
    return {"value": n * reps / dt, "unit": "tokens/s", "cores": cores, "kind": "port",
            "sample": f"{n} loss-active rows of the timed workload (V={vocab} bf16) x {reps} passes, fused fwd+bwd "
                      f"with the fp32 vectorised CPU port (oracle/sf_cpu_fast.c), {dt:.1f} s on {cores} threads",
            "cpu_model": cpu_model(), "value_1thread": one_thread}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2604_11554_b200 import _lib, data_parallel as dp, train_math as tm

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.config != 2 or args.fwd_only:
        import bench_extra

        if args.fwd_only:
            bench_extra.run_fwd_only(args, world, rank, dev, dist)
        elif args.config in (1, 4):
            bench_extra.run_loss_config(args, args.config, world, rank, dev, dist)
        elif args.config == 3:
            bench_extra.run_r3(args, world, rank, dev, dist)
        else:
            bench_extra.run_vocab_parallel(args, world, rank, dev, dist)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    h = tm.handle(local)
    V, L, S, M, G = args.vocab, args.seq_len, args.seqs_per_mb, args.micro_batches, args.group
    n_seq = S * M
    rng = np.random.default_rng(1000 + rank)
    T_step, lens, plens, rewards, gids = make_step_inputs(rng, n_seq, L, V, G)
    T_mb = S * L

    # resident per-micro-batch logits + dlogits (LM-head output and its gradient)
    logits = torch.empty(T_mb, V, dtype=torch.bfloat16, device=dev)
    dlogits = torch.empty_like(logits)
    peak = torch.from_numpy(rng.integers(0, V, size=T_mb).astype(np.int32)).to(dev)
    tm.synth_logits(logits, seed=42 + rank, sigma=2.0, peak_id=peak)
    coin = torch.from_numpy(rng.random(T_step) < 0.5).to(dev)
    rnd = torch.from_numpy(rng.integers(0, V, size=T_step).astype(np.int32)).to(dev)
    targets = torch.where(coin, peak.repeat(M), rnd).to(torch.int32)
    logp0 = torch.empty(T_step, device=dev)
    for m in range(M):
        lp, _, _ = tm.logprob_fwd(logits, targets[m * T_mb:(m + 1) * T_mb])
        logp0[m * T_mb:(m + 1) * T_mb] = lp
    g = torch.Generator(device=dev).manual_seed(7 + rank)
    old = (logp0 + 0.05 * torch.randn(T_step, device=dev, generator=g)).float()
    ref = (logp0 + 0.1 * torch.randn(T_step, device=dev, generator=g)).float()
    d_lens = torch.from_numpy(lens).to(dev)
    d_plens = torch.from_numpy(plens).to(dev)
    d_rewards = torch.from_numpy(rewards).to(dev)
    d_gids = torch.from_numpy(gids).to(dev)
    n_active = int((lens - np.minimum(plens, lens)).sum())
    # DAPO token-mean over the whole GLOBAL step (H5: exact): every rank weights
    # its tokens by 1 / (loss-active tokens summed over the ranks)
    n_active_global = dp.global_active_tokens(n_active, device=dev)
    inv_norm = 1.0 / n_active_global
    params = _lib.default_loss_params(norm_mode=_lib.NORM_EXPLICIT, inv_norm=inv_norm)
    if args.generic:
        tm.set_force_generic(True)
    metrics = torch.zeros(M, _lib.NUM_METRICS, device=dev)
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(M)]

    def device_step(record: bool):
        cu, _, mask, _ = tm.varlen_meta(d_lens, d_plens, T=T_step, want=("cu", "mask"))
        adv = tm.grpo_advantage(d_rewards, d_gids, 1e-6, _lib.STD_UNBIASED)
        adv_tok, w_tok = tm.token_weights(cu, adv, mask, T_step, _lib.NORM_EXPLICIT, inv_norm)
        for m in range(M):
            sl = slice(m * T_mb, (m + 1) * T_mb)
            if record:
                ev[m][0].record(stream)
            tm.pg_loss_fwd_bwd(logits, targets[sl], old[sl], ref[sl], adv_tok[sl], w_tok[sl], params,
                               dlogits=dlogits, metrics=metrics[m])
            if record:
                ev[m][1].record(stream)
        return adv_tok, w_tok

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---------------- device-resident timed region (value)
    for _ in range(args.warmup):
        device_step(False)
    barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.25)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    launches0 = h.launch_count()
    t0.record(stream)
    per_launch = []
    for _ in range(args.steps):
        device_step(True)
        # collect this step's kernel times lazily (events are on the launching stream)
        per_launch.append([e for e in ev])
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(M)]
    t1.record(stream)
    barrier()
    clocks = clk.stop()
    launches = h.launch_count() - launches0
    ms = t0.elapsed_time(t1)
    kms = [a.elapsed_time(b) for step in per_launch for (a, b) in step]
    tmax = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    ms_step = ms_max / args.steps
    value = n_active_global / (ms_step / 1e3)  # loss-active tokens of all ranks
    value_all = world * T_step / (ms_step / 1e3)  # every token, masked prompt rows included

    # roofline of the dominant kernel (fused loss fwd+bwd), algorithmic bytes per launch
    es = 2
    metrics.zero_()
    adv_last, w_last = device_step(False)
    torch.cuda.synchronize(dev)
    act_per_mb = [int((w_last[m * T_mb:(m + 1) * T_mb] != 0).sum().item()) for m in range(M)]
    small = 5 * 4  # targets, old, ref, adv_tok, w_tok per token (fp32/int32)
    bytes_per_mb = [a * 2 * V * es + (T_mb - a) * V * es + T_mb * small for a in act_per_mb]
    avg_bytes = float(np.mean(bytes_per_mb))
    avg_kms = float(np.mean(kms))
    ll = h.last_launch()
    kname = f"{ll['kernel']}<bf16,C={ll['cluster']}> grid {ll['grid']}"
    achieved = avg_bytes / (avg_kms / 1e3) / 1e9
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak_gbs, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        peak_gbs = float(json.load(open(peaks_path))["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    traffic = None
    prof = os.path.join(ROOT, "profiles", "fused_loss_traffic.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            if pj.get("vocab") == V and pj.get("rows") == T_mb:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    kernel_share = sum(kms) / ms if ms > 0 else None

    # ---------------- end-to-end through the C++ trainer seam (e2e): per micro-batch
    # ActorLossSeam::step (include/staleflow/train_math_seam.hpp) on the MicroBatch
    # as the bus delivers it (payload bytes of the trainer field set, built once
    # outside the timed region): payload decode, pinned staging, H2D, GRPO over the
    # micro-batch's complete groups, token weights, fused loss, D2H metrics.
    e2e = None
    if not args.no_e2e:
        from paper_2604_11554_b200 import seam

        actor = seam.ActorLossSeam(local)
        h_t, h_o, h_r = targets.cpu().numpy(), old.cpu().numpy(), ref.cpu().numpy()
        tok_mask = np.ones(T_step, np.uint8)
        for b_ in range(n_seq):
            tok_mask[b_ * L:b_ * L + min(int(plens[b_]), L)] = 0
        batches = []
        for m in range(M):
            sl = slice(m * T_mb, (m + 1) * T_mb)
            ss = slice(m * S, (m + 1) * S)
            batches.append(seam.MicroBatch(lens[ss], h_t[sl], h_o[sl], h_r[sl], rewards[ss], False,
                                           loss_mask=tok_mask[sl], sample_ids=np.arange(m * S, (m + 1) * S) + 1))
        h_met = torch.zeros(M, _lib.NUM_METRICS).pin_memory()

        def e2e_step():
            for m in range(M):
                actor.step(batches[m], logits, dlogits, params, h_met[m], group_size=G)

        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        barrier()
        ems = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e_step = float(ems.item()) / args.steps
        h2d = T_step * (4 + 4 + 4 + 1) + n_seq * (4 + 4 + 4)  # targets, logp, ref_logp, loss_mask; lens, reward, group
        d2h = M * _lib.NUM_METRICS * 4
        # the seam's metrics equal the device path's (same groups, same weights)
        e_met = h_met.sum(0)
        e2e = {"value": n_active_global / (e_step / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e_step,
               "value_all_tokens": world * T_step / (e_step / 1e3),
               "loss_matches_device_path": bool(abs(float(e_met[0]) - float(metrics.sum(0)[0].item())) <=
                                                1e-5 * abs(float(e_met[0])) + 1e-7),
               "path": "C++ ActorLossSeam::step per micro-batch via libsf_seam.so (MicroBatch payload bytes of "
                       "the trainer field set -> decode -> pinned staging -> H2D -> varlen/GRPO/weights/fused "
                       "loss -> D2H metrics); logits device-resident (LM-head output)"}

    # step metrics all-reduce (the one real DP exchange); metrics of the last device step,
    # weighted by the global token count, so the SUM is the global token-mean
    step_metrics = dp.reduce_step_metrics(metrics.sum(0))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_leg(tm, logits, targets[:T_mb], old[:T_mb], ref[:T_mb], adv_last[:T_mb],
                                   w_last[:T_mb], V, args.cpu_seconds)
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {ex!r}"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded SplitMix64 logits, device-resident)",
            "config": {"workload": "Qwen3-4B shape, BASELINE configs[1]: 64 prompts x 8 rollouts x 4096 tok per rank",
                       "vocab": V, "global_batch_seqs": world * n_seq, "seq_len": L,
                       "micro_batches": M, "seqs_per_micro_batch": S, "tokens_per_step": world * T_step,
                       "loss_active_tokens_per_step": n_active_global,
                       "value_counts": "loss-active tokens (mask = 1, SURVEY.md §8d); value_all_tokens adds the "
                                       "masked prompt rows",
                       "parallelism": f"dp{world} (sequence sharding, global token-mean)",
                       "l2": "no flush: 39.8 GB resident logits per launch >> 126 MB L2",
                       "loss": "DAPO decoupled clip 0.2/0.28, token-mean over step, beta=0",
                       "kernel": "generic two-pass" if args.generic else
                       "fused single pass: TMA ring -> TMEM + smem row store, warp-specialised"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                         "frac": achieved / peak_gbs, "traffic": traffic, "peak_source": peak_src,
                         "kernel": kname, "algorithmic_bytes_per_launch": avg_bytes,
                         "avg_launch_ms": avg_kms, "kernel_share_of_step": kernel_share,
                         "bytes_model": "4V B per loss-active row (bf16 read + dlogits write), 2V B per masked row "
                                        "(zero-filled dlogits), + 20 B/token scalars"},
            "value_all_tokens": value_all,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "step_metrics": {n: float(v) for n, v in zip(_lib.METRIC_NAMES, step_metrics.tolist())},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
