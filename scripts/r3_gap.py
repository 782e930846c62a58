# Why the config-3 bench line's R3 launches are slower than r3_split.py's:
# record pattern (exact top-k vs 5% swapped), alternating fwd/bwd vs repeated.
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import train_math as tm

dev = torch.device("cuda", 0)
L, E, k, T = 48, 128, 8, 32 * 4096
g = torch.Generator(device=dev).manual_seed(5)
z = torch.randn(L, T, E, device=dev, generator=g) * 2
top = torch.topk(z, k, dim=-1).indices
swap = torch.rand(L, T, device=dev, generator=g) < 0.05
alt = (top[..., 0] + 1 + torch.randint(0, E - 1, (L, T), device=dev, generator=g)) % E
rec_sw = top.clone()
rec_sw[..., k - 1] = torch.where(swap & (alt[..., None] != top).all(-1), alt, top[..., k - 1])
recs = {"exact": top.to(torch.uint8), "swapped": rec_sw.to(torch.uint8)}
dw = torch.randn(L, T, k, device=dev, generator=g)
bufs = (torch.empty(L, T, k, device=dev), torch.empty(L, T, k, dtype=torch.int32, device=dev),
        torch.empty(L + 1, dtype=torch.int32, device=dev), torch.empty_like(z))


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for name, rec in recs.items():
    w, _, _ = tm.r3_gate_fwd(z, rec, renorm=True, out=bufs[:3])
    f = timeit(lambda: tm.r3_gate_fwd(z, rec, renorm=True, out=bufs[:3]))
    b = timeit(lambda: tm.r3_gate_bwd(z, rec, w, dw, renorm=True, out=bufs[3]))
    fb = timeit(lambda: (tm.r3_gate_fwd(z, rec, renorm=True, out=bufs[:3]),
                         tm.r3_gate_bwd(z, rec, bufs[0], dw, renorm=True, out=bufs[3])))
    print(f"{name}: fwd {f:.3f} ms  bwd {b:.3f} ms  fwd+bwd alternating {fb:.3f} ms (sum {f + b:.3f})", flush=True)
