#!/bin/bash
# A/B build variants of the fused kernel on one box (same clocks, same HBM).
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e $BARGS"
P='import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])'
for X in ${XS:-none}; do
  [ "$X" = none ] && X=""
  touch paper_2604_11554_b200/csrc/tm_loss.cu
  make -s -j8 -C paper_2604_11554_b200/csrc EXTRA="$X" > /dev/null 2>&1 || { echo build fail $X; continue; }
  for i in 1 2; do echo "== [$X] run $i"; timeout 300 $B | python -c "$P"; done
done
