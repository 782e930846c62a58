# Stress: the fused kernel's per-row logp/entropy (all rows) against the
# streaming forward kernel, many rows, repeated; prints mismatching rows.
import os, sys
import torch
sys.path.insert(0, os.environ.get("SF_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2604_11554_b200 import train_math as tm

dev = torch.device("cuda", 0)
g = torch.Generator(device="cpu").manual_seed(1)
SHAPES = [(torch.float32, 5000, 16000), (torch.bfloat16, 20000, 151936), (torch.float32, 20000, 4096),
          (torch.bfloat16, 8000, 75968), (torch.bfloat16, 16000, 50257), (torch.bfloat16, 6000, 262144),
          (torch.float32, 6000, 32001)]
if os.environ.get("SHAPES"):
    SHAPES = [SHAPES[int(i)] for i in os.environ["SHAPES"].split(",")]
for (dt, T, V) in SHAPES:
    lg = (torch.randn(T, V, generator=g) * 3).to(dt).to(dev)
    tg = torch.randint(0, V, (T,), generator=g, dtype=torch.int32).to(dev)
    o = (-4 + torch.randn(T, generator=g)).to(dev)
    r = (o + 0.1 * torch.randn(T, generator=g).to(dev)).float()
    a = torch.randn(T, generator=g).to(dev)
    w = (torch.rand(T, generator=g) < 0.8).float().to(dev) / T
    lp_ref, ent_ref, _ = tm.logprob_fwd(lg, tg)
    nbad = 0
    for it in range(int(os.environ.get("ITERS", "10"))):
        m, d, lp, ent = tm.pg_loss_fwd_bwd(lg, tg, o, r, a, w, want_logp=True)
        torch.cuda.synchronize()
        bad = torch.nonzero(((lp - lp_ref).abs() > 1e-4 + 1e-5 * lp_ref.abs()) & (w != 0)).flatten()
        if len(bad):
            nbad += 1
            i = int(bad[0])
            # the dlogits of a bad row against the two-kernel reference p_v (rows with g == 0 carry none)
            print(f"  {dt} T={T} V={V} iter {it}: {len(bad)} bad rows (row//148: {(bad // 148).tolist()[:12]}), "
                  f"e.g. {i}: ref {float(lp_ref[i])} got {float(lp[i])}; ent ref {float(ent_ref[i])} got {float(ent[i])}")
    print(f"{dt} T={T} V={V} C={tm.handle(0).last_launch() if hasattr(tm.handle(0), "last_launch") else "?"}: {nbad} bad iterations", flush=True)
