# SPDX-License-Identifier: Apache-2.0
"""Tuning aid: per-role wait breakdown of the fused loss kernel (clock64
instrumentation behind sf_tm_debug_wait_counters). Not a benchmark.

  python scripts/wait_profile.py [rows] [vocab]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import _lib, train_math as tm  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
V = int(sys.argv[2]) if len(sys.argv) > 2 else 151936
dev = torch.device("cuda", 0)
logits = torch.empty(T, V, dtype=torch.bfloat16, device=dev)
peak = torch.randint(0, V, (T,), dtype=torch.int32, device=dev)
tm.synth_logits(logits, seed=1, peak_id=peak)
tg = peak.clone()
lp, _, _ = tm.logprob_fwd(logits, tg)
old = lp + 0.05 * torch.randn(T, device=dev)
ref = lp + 0.1 * torch.randn(T, device=dev)
adv = torch.randn(T, device=dev)
w = torch.full((T,), 1.0 / T, device=dev)
dl = torch.empty_like(logits)
for _ in range(2):
    tm.pg_loss_fwd_bwd(logits, tg, old, ref, adv, w, dlogits=dl)
cnt = torch.zeros(16, dtype=torch.int64, device=dev)
_lib.lib().sf_tm_debug_wait_counters(ctypes.c_void_p(cnt.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
tm.pg_loss_fwd_bwd(logits, tg, old, ref, adv, w, dlogits=dl)
e1.record()
torch.cuda.synchronize()
_lib.lib().sf_tm_debug_wait_counters(None)
c = cnt.cpu().tolist()
ms = e0.elapsed_time(e1)
print(f"rows={T} V={V}: {ms:.3f} ms, {4 * V * T / ms / 1e6:.0f} GB/s (instrumented)")
names = ["producer", "forward", "control", "backward"]
waits = [("empty", "-"), ("full", "tempty"), ("red", "mail"), ("scal", "tfull")]
for r, n in enumerate(names):
    nw = max(c[12 + r], 1)
    act = c[3 * r] / nw
    print(f"{n:9s} warps={c[12 + r]:5d} cycles/warp={act:12.0f}  wait[{waits[r][0]}]={c[3 * r + 1] / nw / act * 100:5.1f}%"
          f"  wait[{waits[r][1]}]={c[3 * r + 2] / nw / act * 100:5.1f}%")
