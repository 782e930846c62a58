#!/bin/bash
./scripts/mb_copy
for D in 1 3 7; do
  for C in 2 3; do
  echo "== dbg=$D C=$C"; SFTM_DBG_NOCOMPUTE=$D SFTM_LOSS_C=$C timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
  done
done
