# SPDX-License-Identifier: Apache-2.0
"""Debug aid: emulated vocab-parallel ranks (one GPU) on an odd vocabulary;
per-row logp of every rank vs the fp64 oracle. Test infrastructure only.
  python scripts/xp_ua_debug.py P dtype V"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402
from paper_2604_11554_b200 import _lib, train_math as tm  # noqa: E402
from paper_2604_11554_b200.vocab_parallel import shard_bounds  # noqa: E402

P, dtype, V = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
prob = orc.synth_problem(600 + 10 * P, [37, 20, 51, 9], V, dtype, prompt_max=6, G=2)
T = prob["T"]
x = prob["logits"]
logits = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16) if dtype == "bf16" else torch.from_numpy(x)).cuda()
i32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()
f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
cu, _, mask, _ = tm.varlen_meta(i32(prob["lens"]), i32(prob["plens"]), T=T, want=("cu", "mask"))
adv = tm.grpo_advantage(f32(prob["rewards"]), i32(prob["gids"]))
adv_tok, w_tok = tm.token_weights(cu, adv, mask, T)
tg, old, ref = i32(prob["targets"]), f32(prob["old"]), f32(prob["ref"])
params = _lib.default_loss_params()
b = shard_bounds(V, P, 8 if dtype == "bf16" else 4)
shards = [logits[:, b[r]:b[r + 1]].contiguous() for r in range(P)]
hs = [tm.Handle(0) for _ in range(P)]
tm.vp_local_group(hs, 0 if P == 1 else 148 // P)
dbg = None
if os.environ.get("HANG_DBG"):  # an -DSFTM_HANG_DEBUG build: give-up waits record their sites here
    import ctypes
    dbg = torch.zeros(16 + 3 * 8 * 148 * 32 + 8 * 148 + 8 * 148 * 4, dtype=torch.int64, pin_memory=True)
    _lib.lib().sf_tm_debug_wait_counters(ctypes.c_void_p(dbg.data_ptr()))
streams = [torch.cuda.Stream() for _ in range(P)]
cur = torch.cuda.current_stream()
outs = []
for s in streams:
    s.wait_stream(cur)
for r in range(P):
    with torch.cuda.stream(streams[r]):
        outs.append(tm.vp_fused_loss_fwd_bwd(shards[r], b[r], tg, old, ref, adv_tok, w_tok, params, want_logp=True,
                                             h=hs[r], stream=streams[r]))
try:
    torch.cuda.synchronize()
except Exception as e:  # noqa: BLE001
    print("launch failed:", str(e).splitlines()[0])
if dbg is not None:
    d = dbg.tolist()
    dec = lambda v: dict(line=v & 0xffff, par=(v >> 16) & 0xf, rank=(v >> 20) & 0xf, row=(v >> 24) & 0xffff,
                         cta=(v >> 40) & 0xff, warp=(v >> 56) & 0xff)
    print("gave up:", bool(d[15]), dec(d[0]) if d[15] else "")
    if d[15]:
        first = dec(d[0])
        for rk in range(P):  # the first stuck CTA on every rank
            base = 16 + (rk * 148 + first["cta"]) * 32
            print(f"  rank {rk} cta {first['cta']}:", [(dec(v)["warp"], dec(v)["line"], dec(v)["row"], dec(v)["par"])
                                                      for v in d[base:base + 32] if v])
            lb = 16 + 8 * 148 * 32 + (rk * 148 + first["cta"]) * 32
            late = [(ln, (d[lb + ln] >> 56) & 0xff, (d[lb + ln] >> 48) & 0xff, hex((d[lb + ln] >> 8) & 0xffffffff))
                    for ln in range(32) if d[lb + ln]]
            sp = d[16 + 2 * 8 * 148 * 32 + rk * 148 + first["cta"]]
            TB = 16 + 2 * 8 * 148 * 32 + 8 * 148
            posts = [d[TB + (rk * 148 + first["cta"]) * 4 + q] for q in range(4)]
            waits = [d[16 + 8 * 148 * 32 + 8 * 148 * 32 + 8 * 148 + 8 * 148 * 4 + (rk * 148 + first["cta"]) * 32 + ln]
                     for ln in range(4)]
            print("    post times (ns):", posts, " receiver wait start per peer lane:", waits)
            print(f"    late peer messages (peer, row, epoch, src addr):", late,
                  f" sender: rows {sp & 0xff}, epoch {(sp >> 8) & 0xff}, last dst for peer 0 {hex((sp >> 16) & 0xffffffff)}")
    if d[15]:
        os._exit(0)
a, w = adv_tok.cpu().numpy(), w_tok.cpu().numpy()
om, odl, olp, oent, og = orc.pg_loss_fwd_bwd(prob["logits"], prob["targets"], prob["old"], prob["ref"], a, w, orc.params())
act = w != 0
grid = 148 // P if P > 1 else 148
print("shards", [b[r + 1] - b[r] for r in range(P)], "streams", [h.last_launch()["streams"] for h in hs])
owner = np.searchsorted(np.array(b[1:]), prob["targets"], side="right")
for r in range(P):
    lp = outs[r][2].cpu().numpy()
    bad = np.nonzero(act & (np.abs(lp - olp) > 1e-4 + 1e-4 * np.abs(olp)))[0]
    print(f"rank {r}: {len(bad)} bad rows of {act.sum()}; first:",
          [(int(t), int(t % grid), int(t // grid), int(owner[t]), round(float(lp[t]), 3), round(float(olp[t]), 3))
           for t in bad[:8]])
