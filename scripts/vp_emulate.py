# SPDX-License-Identifier: Apache-2.0
"""Vocab-parallel at P = 1/2/4/8 emulated on ONE B200 (the evidence this pool
allows for the north star's 8-GPU point): P handles wired as an in-process
group (sf_tm_debug_vp_local_group), one stream per rank, each rank's exchange
grid capped at 148 // P CTAs so the P kernels are co-resident; every rank owns
a V/P-wide shard of the same T rows. Reported: the aggregate HBM rate of the P
kernels (all shards' algorithmic bytes / wall time), and, for comparison, the
same narrow rows through the single-GPU fused kernel on the whole GPU (no
exchange) -- the per-row cost of a narrow shard vs the cost of the exchange.

  python scripts/vp_emulate.py [T]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11554_b200 import _lib, train_math as tm  # noqa: E402
from paper_2604_11554_b200.vocab_parallel import shard_bounds  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
V = 151936
dev = torch.device("cuda", 0)
peak = float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
g = torch.Generator(device=dev).manual_seed(3)
tg = torch.randint(0, V, (T,), device=dev, dtype=torch.int32, generator=g)
old = (-3 + 0.5 * torch.randn(T, device=dev, generator=g)).float()
ref = (old + 0.1 * torch.randn(T, device=dev, generator=g)).float()
adv = torch.randn(T, device=dev, generator=g)
w = torch.full((T,), 1.0 / T, device=dev)
res = []
for P in (1, 2, 4, 8):
    b = shard_bounds(V, P)
    shards = [torch.empty(T, b[r + 1] - b[r], dtype=torch.bfloat16, device=dev) for r in range(P)]
    for r, s in enumerate(shards):
        tm.synth_logits(s, seed=10 + r, sigma=2.0)
    dls = [torch.empty_like(s) for s in shards]
    hs = [tm.Handle(0) for _ in range(P)]
    tm.vp_local_group(hs, 0 if P == 1 else 148 // P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    byts = sum(4 * s.shape[1] * T for s in shards)

    def launch():
        cur = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(cur)
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                tm.vp_fused_loss_fwd_bwd(shards[r], b[r], tg, old, ref, adv, w, dlogits=dls[r], h=hs[r],
                                         stream=streams[r])
        for s in streams:
            cur.wait_stream(s)

    for _ in range(2):
        launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        launch()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    # the same shard width through the plain fused kernel on the whole GPU (no exchange)
    s0 = shards[0]
    for _ in range(2):
        tm.pg_loss_fwd_bwd(s0, torch.remainder(tg, s0.shape[1]).to(torch.int32), old, ref, adv, w, dlogits=dls[0])
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        tm.pg_loss_fwd_bwd(s0, torch.remainder(tg, s0.shape[1]).to(torch.int32), old, ref, adv, w, dlogits=dls[0])
    e1.record()
    torch.cuda.synchronize()
    ms1 = e0.elapsed_time(e1) / reps
    r = {"P": P, "shard": b[1] - b[0], "rows": T, "grid_per_rank": 148 if P == 1 else 148 // P,
         "ms": ms, "aggregate_gbs": byts / ms / 1e6, "frac": byts / ms / 1e6 / peak,
         "narrow_rows_no_exchange_gbs": 4 * s0.shape[1] * T / ms1 / 1e6,
         "narrow_rows_no_exchange_frac": 4 * s0.shape[1] * T / ms1 / 1e6 / peak}
    print(json.dumps(r), flush=True)
    res.append(r)
    for hh in hs:
        hh.close()
    del shards, dls
    torch.cuda.empty_cache()
