import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import train_math as tm
dev = torch.device("cuda", 0)
for (L, T) in [(1, 64), (4, 300)]:
    E, k = 128, 8
    z = torch.randn(L, T, E, device=dev)
    rec = torch.topk(z, k, dim=-1).indices.to(torch.int32)
    for renorm in (True, False):
        t0 = time.time()
        w, idx, mm = tm.r3_gate_fwd(z, rec, renorm=renorm)
        torch.cuda.synchronize()
        print(L, T, renorm, "fwd ok", mm.tolist(), f"{time.time() - t0:.3f}s", flush=True)
