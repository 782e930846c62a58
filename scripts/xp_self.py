# Fused vocab-parallel kernel at P=1 (self-exchange through the peer mailbox)
# vs the plain fused kernel: cost of the exchange mechanism without NVLink.
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import train_math as tm

dev = torch.device("cuda", 0)
T = 131072
for V in [151936 // 4, 151936 // 2]:
    lg = torch.empty(T, V, dtype=torch.bfloat16, device=dev)
    tm.synth_logits(lg, seed=3, sigma=2.0)
    g = torch.Generator(device=dev).manual_seed(1)
    tg = torch.randint(0, V, (T,), device=dev, dtype=torch.int32, generator=g)
    o = (-4 + torch.randn(T, device=dev, generator=g)).float()
    r = (o + 0.1 * torch.randn(T, device=dev, generator=g)).float()
    a = torch.randn(T, device=dev, generator=g)
    w = (torch.rand(T, device=dev, generator=g) < 0.93).float() / T
    dl = torch.empty_like(lg)
    if V == 151936 // 4:
        h = tm.vp_mailbox_create(1, 0, 0)
        tm.vp_mailbox_open([h], 0)
    res = {}
    for name, fn in [("plain", lambda: tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, dlogits=dl)),
                     ("xp_self", lambda: tm.vp_fused_loss_fwd_bwd(lg, 0, tg, o, r, a, w, dlogits=dl))]:
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[name] = ms
        by = (w != 0).sum().item() * 4 * V + (w == 0).sum().item() * 2 * V
        print(f"V={V} {name}: {ms:.3f} ms  {by / ms / 1e6:.0f} GB/s  last={tm.handle(0).last_launch()}", flush=True)
