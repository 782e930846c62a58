# Where the host-buffer step (pg_step_host) spends its extra time vs the device-resident fused call.
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import _lib, train_math as tm

dev = torch.device("cuda", 0)
S, L, V = 32, 4096, 151936
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
dl = torch.empty_like(lg)
hm = torch.zeros(_lib.NUM_METRICS).pin_memory()
params = _lib.default_loss_params()
d_t, d_o, d_r = (x.cuda() for x in (h_t, h_o, h_r))
adv = torch.randn(T, device=dev)
w = torch.full((T,), 1.0 / T, device=dev)

def host_step():
    tm.pg_step_host(lg, h_t, h_o, h_r, h_l, h_w, h_g, h_prompt_lens=h_p, params=params, dlogits=dl, h_metrics=hm)

def dev_step():
    tm.pg_loss_fwd_bwd(lg, d_t, d_o, d_r, adv, w, params, dlogits=dl)

for name, fn in [("device", dev_step), ("host", host_step), ("device", dev_step), ("host", host_step)]:
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(8):
        fn()
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 8:.3f} ms/step (host enqueue {1e3 * (t1 - t0) / 8:.3f} ms)", flush=True)
