# a1 forward-only (logprob + entropy) throughput: rows_ring_kernel mode Fwd.
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import train_math as tm

dev = torch.device("cuda", 0)
T = 131072
for V, dt in [(151936, torch.bfloat16), (32000, torch.float32), (50257, torch.bfloat16)]:
    lg = torch.empty(T, V, dtype=dt, device=dev)
    tm.synth_logits(lg, seed=3, sigma=2.0)
    tg = torch.randint(0, V, (T,), device=dev, dtype=torch.int32)
    for _ in range(3):
        tm.logprob_fwd(lg, tg)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        tm.logprob_fwd(lg, tg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    by = T * V * lg.element_size()
    print(f"V={V} {dt}: {ms:.3f} ms  {by / ms / 1e6:.0f} GB/s  {T / ms / 1e3:.1f} M tok/s  {tm.handle(0).last_launch()}", flush=True)
    del lg
