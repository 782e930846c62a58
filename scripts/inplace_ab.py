# Fused loss at the headline micro-batch: separate dlogits vs in place (dlogits aliasing logits).
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import train_math as tm

dev = torch.device("cuda", 0)
T, V = 131072, 151936
lg = torch.empty(T, V, dtype=torch.bfloat16, device=dev)
g = torch.Generator(device=dev).manual_seed(1)
tg = torch.randint(0, V, (T,), device=dev, dtype=torch.int32, generator=g)
o = (-4 + torch.randn(T, device=dev, generator=g)).float()
r = (o + 0.1 * torch.randn(T, device=dev, generator=g)).float()
a = torch.randn(T, device=dev, generator=g)
w = (torch.rand(T, device=dev, generator=g) < 0.93).float() / T
dl = torch.empty_like(lg)
for name in ["separate", "inplace", "separate", "inplace"]:
    ms = []
    for it in range(4):
        tm.synth_logits(lg, seed=3, sigma=2.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if name == "inplace":
            tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, dlogits=lg, in_place=True)
        else:
            tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, dlogits=dl)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    by = (w != 0).sum().item() * 4 * V + (w == 0).sum().item() * 2 * V
    best = min(ms[1:])
    print(f"{name}: {best:.3f} ms  {by / best / 1e6:.0f} GB/s", flush=True)
