# SPDX-License-Identifier: Apache-2.0
"""Every kernel of libsf_train_math.so once, at small shapes, for
compute-sanitizer (scripts/sanitize.sh): the fused loss at every cluster size it
picks (C = 1 Qwen bf16 rows, C = 2 262k-wide rows) and in sector coordinates
(odd vocabulary), the e-store schedule, masked-skip / in-place / entropy
variants, the forward-only streaming kernel, the two-pass generic kernel, the
vocab-parallel stats / backward kernels and the fused peer-exchange kernel at
P = 1 (self-exchange) and P = 2 (emulated on one GPU), the R3 gate fwd/bwd,
the routed-experts transpose, varlen / GRPO / token-weight prologue kernels."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import _lib, train_math as tm  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)


def loss_case(V, T, dtype=torch.bfloat16, **kw):
    x = (torch.randn(T, V, device=dev, generator=g) * 2).to(dtype)
    y = torch.randint(0, V, (T,), device=dev, dtype=torch.int32, generator=g)
    o = (-3 + torch.randn(T, device=dev, generator=g)).float()
    r = o + 0.1
    a = torch.randn(T, device=dev, generator=g)
    w = (torch.rand(T, device=dev, generator=g) < 0.8).float() / T
    tm.pg_loss_fwd_bwd(x, y, o, r, a, w, _lib.default_loss_params(**kw.get("p", {})), in_place=kw.get("inplace", False),
                       want_logp=True)
    tm.logprob_fwd(x, y)
    return x, y, o, r, a, w


loss_case(151936, 12)                       # C = 1, TMEM + smem row store
loss_case(262144, 5)                        # C = 2 cluster (DSMEM exchange)
loss_case(50257, 9)                         # odd vocabulary: sector coordinates
loss_case(32000, 20, torch.float32, p={"entropy_coef": 0.01, "kl_beta": 0.05})
loss_case(4096, 64, p={"masked_rows": _lib.MASKED_SKIP})
loss_case(8192, 16, inplace=True)
tm.set_force_generic(True)
loss_case(8192, 16)                         # the two-pass generic kernel
tm.set_force_generic(False)
# vocab-parallel two-pass kernels and the fused peer-exchange kernel
x, y, o, r, a, w = loss_case(8192, 24)
st = tm.vp_partial_stats(x[:, :4096].contiguous(), y, 0)
tm.vp_loss_fwd_bwd(x[:, :4096].contiguous(), 0, torch.stack([st, st]), y, o, r, a, w)
for P in (1, 2):
    hs = [tm.Handle(0) for _ in range(P)]
    tm.vp_local_group(hs, 0 if P == 1 else 74)
    shards = [x[:, p * (8192 // P):(p + 1) * (8192 // P)].contiguous() for p in range(P)]
    ss = [torch.cuda.Stream() for _ in range(P)]
    torch.cuda.synchronize()
    for p in range(P):
        with torch.cuda.stream(ss[p]):
            tm.vp_fused_loss_fwd_bwd(shards[p], p * (8192 // P), y, o, r, a, w, h=hs[p], stream=ss[p])
    torch.cuda.synchronize()
    for hh in hs:
        hh.close()
# R3
L, Tr, E, k = 3, 70, 128, 8
z = torch.randn(L, Tr, E, device=dev, generator=g)
rec = torch.topk(z, k, dim=-1).indices.to(torch.uint8)
wg, idx, mm = tm.r3_gate_fwd(z, rec)
tm.r3_gate_bwd(z, rec, wg, torch.randn(L, Tr, k, device=dev, generator=g))
tm.r3_gate_fwd(z, rec.to(torch.int32), renorm=False)
tm.r3_record_layer_major(rec.permute(1, 0, 2).contiguous())
# prologue kernels
lens = torch.tensor([5, 0, 9, 3], dtype=torch.int32, device=dev)
cu, sid, mask, tg = tm.varlen_meta(lens, torch.tensor([1, 0, 2, 5], dtype=torch.int32, device=dev),
                                   torch.tensor([0, 0, 1, 1], dtype=torch.int32, device=dev))
adv = tm.grpo_advantage(torch.tensor([1.0, 0.0, 1.0, 1.0], device=dev), torch.tensor([0, 0, 1, 1], dtype=torch.int32,
                                                                                       device=dev))
tm.token_weights(cu, adv, mask, 17)
torch.cuda.synchronize()
# the e-store schedule (opt-in) in a child process: SFTM_ES is read once per process
if os.environ.get("SFTM_ES") != "1":
    import subprocess

    rc = subprocess.run([sys.executable, __file__], env=dict(os.environ, SFTM_ES="1")).returncode
    assert rc == 0
print("sanitize cases done")
