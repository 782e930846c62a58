# SPDX-License-Identifier: Apache-2.0
"""Row-stream debugging aid: the fused loss at a given width/dtype with the
stream count forced (SFTM_LOSS_NS), compared with a reference run of the same
process-independent inputs saved by NS=1. Not a test."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import train_math as tm  # noqa: E402

T, V, dt = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
g = torch.Generator(device="cpu").manual_seed(7)
tdt = torch.bfloat16 if dt == "bf16" else torch.float32
lg = (torch.randn(T, V, generator=g) * 3).to(tdt).cuda()
tg = torch.randint(0, V, (T,), generator=g, dtype=torch.int32).cuda()
o = (-4 + torch.randn(T, generator=g)).cuda()
r = (o + 0.1 * torch.randn(T, generator=g).cuda()).float()
a = torch.randn(T, generator=g).cuda()
w = (torch.rand(T, generator=g) < 0.8).float().cuda() / T
met, dl, lp, ent = tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, want_logp=True)
torch.cuda.synchronize()
print("launch", tm.handle().last_launch())
path = f"/tmp/ns_ref_{T}_{V}_{dt}.pt"
if os.environ.get("SFTM_LOSS_NS", "1") == "1":
    torch.save((dl.cpu(), lp.cpu(), ent.cpu()), path)
else:
    dl0, lp0, ent0 = torch.load(path)
    d = (dl.cpu().float() - dl0.float()).abs()
    rel = d / (dl0.float().abs() + 1e-12)
    bad = rel > 1e-5
    print("dl max abs", d.max().item(), "entries rel>1e-5", int(bad.sum()), "rows", torch.nonzero(bad.any(1)).flatten()[:10].tolist())
    print("lp max", (lp.cpu() - lp0).abs().max().item(), "ent max", (ent.cpu() - ent0).abs().max().item())
    rows = torch.nonzero(((lp.cpu() - lp0).abs() > 1e-6)).flatten()
    print("lp rows differing", rows[:20].tolist(), len(rows))
