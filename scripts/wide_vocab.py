# Fused loss throughput on vocabularies that need a 2-CTA cluster (C=2).
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import train_math as tm

dev = torch.device("cuda", 0)
for V, dt, T in [(262144, torch.bfloat16, 65536), (151936, torch.float32, 49152), (201088, torch.bfloat16, 65536)]:
    lg = torch.empty(T, V, dtype=dt, device=dev)
    tm.synth_logits(lg, seed=3, sigma=2.0)
    g = torch.Generator(device=dev).manual_seed(1)
    tg = torch.randint(0, V, (T,), device=dev, dtype=torch.int32, generator=g)
    o = (-4 + torch.randn(T, device=dev, generator=g)).float()
    r = (o + 0.1 * torch.randn(T, device=dev, generator=g)).float()
    a = torch.randn(T, device=dev, generator=g)
    w = (torch.rand(T, device=dev, generator=g) < 0.93).float() / T
    dl = torch.empty_like(lg)
    for _ in range(2):
        tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, dlogits=dl)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, dlogits=dl)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    es = lg.element_size()
    by = (w != 0).sum().item() * 2 * es * V + (w == 0).sum().item() * es * V
    print(f"V={V} {dt}: {ms:.3f} ms {by / ms / 1e6:.0f} GB/s {T / ms / 1e3:.2f} M tok/s {tm.handle(0).last_launch()}", flush=True)
    del lg, dl
