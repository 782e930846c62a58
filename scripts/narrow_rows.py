# SPDX-License-Identifier: Apache-2.0
"""Narrow rows through the single-GPU fused kernel (the per-row fixed cost of a
vocab-parallel shard, without the exchange): T rows x W bf16. For ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import train_math as tm  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
W = int(sys.argv[2]) if len(sys.argv) > 2 else 18992
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
x = torch.empty(T, W, dtype=torch.bfloat16, device=dev)
tm.synth_logits(x, seed=5, sigma=2.0)
tg = torch.randint(0, W, (T,), device=dev, dtype=torch.int32, generator=g)
old = (-3 + 0.5 * torch.randn(T, device=dev, generator=g)).float()
ref = (old + 0.1 * torch.randn(T, device=dev, generator=g)).float()
adv = torch.randn(T, device=dev, generator=g)
w = torch.full((T,), 1.0 / T, device=dev)
dl = torch.empty_like(x)
for _ in range(3):
    tm.pg_loss_fwd_bwd(x, tg, old, ref, adv, w, dlogits=dl)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    tm.pg_loss_fwd_bwd(x, tg, old, ref, adv, w, dlogits=dl)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"T={T} W={W}: {ms:.3f} ms, {4 * W * T / ms / 1e6:.0f} GB/s")
