# Fused loss backward modes: 0 (bf16, no entropy term), 1 (fp32, no entropy), 2 (entropy bonus).
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import _lib, train_math as tm

dev = torch.device("cuda", 0)
T, V = 65536, 151936
lg = torch.empty(T, V, dtype=torch.bfloat16, device=dev)
tm.synth_logits(lg, seed=3, sigma=2.0)
g = torch.Generator(device=dev).manual_seed(1)
tg = torch.randint(0, V, (T,), device=dev, dtype=torch.int32, generator=g)
o = (-4 + torch.randn(T, device=dev, generator=g)).float()
r = (o + 0.1 * torch.randn(T, device=dev, generator=g)).float()
a = torch.randn(T, device=dev, generator=g)
w = (torch.rand(T, device=dev, generator=g) < 0.93).float() / T
dl = torch.empty_like(lg)
by = (w != 0).sum().item() * 4 * V + (w == 0).sum().item() * 2 * V
for name, kw in [("mode0 (no entropy bonus)", {}), ("kl 0.05", {"kl_beta": 0.05}),
                 ("mode2 (entropy 0.01)", {"entropy_coef": 0.01}), ("mode0 again", {})]:
    p = _lib.default_loss_params(**kw)
    for _ in range(2):
        tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, p, dlogits=dl)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, p, dlogits=dl)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name}: {ms:.3f} ms {by / ms / 1e6:.0f} GB/s", flush=True)
