# Per-micro-batch cost of the host-buffer seam call (pg_step_host) against the
# device-resident fused call, on the bench's config-2 micro-batch shape:
#   fused   : pg_loss_fwd_bwd only (prologue outputs precomputed)
#   serial  : device prologue (varlen, GRPO, token weights) + fused, one stream
#   seam    : pg_step_host (pinned host fields; pipelined prologue)
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import _lib, train_math as tm

dev = torch.device("cuda", 0)
S, L, V, M = 32, 4096, 151936, 16
T = S * L
lg = torch.empty(T, V, dtype=torch.bfloat16, device=dev)
tm.synth_logits(lg, seed=3, sigma=2.0)
rng = np.random.default_rng(0)
tg = rng.integers(0, V, T).astype(np.int32)
old = (-4 + rng.normal(size=T)).astype(np.float32)
ref = (old + 0.1 * rng.normal(size=T)).astype(np.float32)
lens = np.full(S, L, np.int32)
plens = rng.integers(32, 513, S).astype(np.int32)
rew = (rng.random(S) < 0.5).astype(np.float32)
gid = (np.arange(S) // 8).astype(np.int32)
pin = lambda a: torch.from_numpy(a).pin_memory()
h_t, h_o, h_r, h_l, h_p, h_w, h_g = map(pin, (tg, old, ref, lens, plens, rew, gid))
d_t, d_o, d_r, d_l, d_p, d_w, d_g = (x.cuda() for x in (h_t, h_o, h_r, h_l, h_p, h_w, h_g))
dl = torch.empty_like(lg)
hm = torch.zeros(M, _lib.NUM_METRICS).pin_memory()
params = _lib.default_loss_params()


def prologue():
    cu, _, mask, _ = tm.varlen_meta(d_l, d_p, T=T, want=("cu", "mask"))
    adv = tm.grpo_advantage(d_w, d_g, 1e-6, _lib.STD_UNBIASED)
    return tm.token_weights(cu, adv, mask, T, _lib.NORM_TOKEN_MEAN, 0.0)


at, wt = prologue()


def fused():
    for _ in range(M):
        tm.pg_loss_fwd_bwd(lg, d_t, d_o, d_r, at, wt, params, dlogits=dl)


def serial():
    for _ in range(M):
        a, w = prologue()
        tm.pg_loss_fwd_bwd(lg, d_t, d_o, d_r, a, w, params, dlogits=dl)


def seam():
    for m in range(M):
        tm.pg_step_host(lg, h_t, h_o, h_r, h_l, h_w, h_g, h_prompt_lens=h_p, params=params, dlogits=dl,
                        h_metrics=hm[m])


res = {}
for rep in range(2):
    for name, fn in [("fused", fused), ("serial", serial), ("seam", seam)]:
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / M
    print(" ".join(f"{k}={v:.3f}ms" for k, v in res.items()),
          f"seam-fused={1e3 * (res['seam'] - res['fused']):.0f}us serial-fused={1e3 * (res['serial'] - res['fused']):.0f}us",
          flush=True)
