# R3 fwd / bwd kernel times separately (config 3 shape), GB/s each.
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import train_math as tm

dev = torch.device("cuda", 0)
L, E, k, T = 48, 128, 8, 32 * 4096
g = torch.Generator(device=dev).manual_seed(5)
z = torch.randn(L, T, E, device=dev, generator=g) * 2
rec = torch.topk(z, k, dim=-1).indices.to(torch.uint8)
dw = torch.randn(L, T, k, device=dev, generator=g)
w, idx, mm = tm.r3_gate_fwd(z, rec, renorm=True)
rows = L * T
for name, fn, by in [("fwd", lambda: tm.r3_gate_fwd(z, rec, renorm=True), rows * (4 * E + k + 4 * k + 4 * k)),
                     ("fwd_noidx", lambda: tm.r3_gate_fwd(z, rec, renorm=True, want_idx=False) if 'want_idx' in tm.r3_gate_fwd.__code__.co_varnames else None, rows * (4 * E + k + 4 * k)),
                     ("bwd", lambda: tm.r3_gate_bwd(z, rec, w, dw, renorm=True), rows * (k + 4 * k + 4 * k + 4 * E)),
                     ("copy", lambda: z.clone(), rows * 8 * E)]:
    if fn() is None:
        continue
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms  {by / ms / 1e6:.0f} GB/s")
