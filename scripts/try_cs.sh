#!/bin/bash
# Cluster-size A/B on one box: python bench lines for each SFTM_LOSS_C in $CS, twice.
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e $BARGS"
P='import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for i in 1 2; do for C in ${CS:-0}; do echo "== C=$C run $i"; SFTM_LOSS_C=$C timeout 300 $B | python -c "$P"; done; done
