# Fused loss time per row vs vocab width: separates per-chunk from per-row costs.
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import train_math as tm

dev = torch.device("cuda", 0)
T = 131072
for V in [int(v) for v in os.environ.get('VS', '18432,24576,30720,36864,37984,43008,49152,75968').split(',')]:
    lg = torch.empty(T, V, dtype=torch.bfloat16, device=dev)
    tm.synth_logits(lg, seed=3, sigma=2.0)
    g = torch.Generator(device=dev).manual_seed(1)
    tg = torch.randint(0, V, (T,), device=dev, dtype=torch.int32, generator=g)
    o = (-4 + torch.randn(T, device=dev, generator=g)).float()
    r = (o + 0.1 * torch.randn(T, device=dev, generator=g)).float()
    a = torch.randn(T, device=dev, generator=g)
    w = torch.full((T,), 1.0 / T, device=dev)
    dl = torch.empty_like(lg)
    for _ in range(2):
        tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, dlogits=dl)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, dlogits=dl)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 4
    per_row_us = ms * 1e3 / (T / 148)
    print(f"V={V:6d} chunks={V / 6144:5.2f}: {ms:.3f} ms  {4 * T * V / ms / 1e6:.0f} GB/s  {per_row_us:.2f} us/row/CTA", flush=True)
    del lg, dl
