#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 > gpurun_out/c3_tests.log 2>&1 || { tail -40 gpurun_out/c3_tests.log; exit 1; }
tail -2 gpurun_out/c3_tests.log
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
P='import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])'
for C in 0 3; do echo "== C=$C config2"; SFTM_LOSS_C=$C timeout 300 $B | python -c "$P"; done
for C in 0 2; do echo "== C=$C config1"; SFTM_LOSS_C=$C timeout 300 $B --config 1 | python -c "$P"; done
echo "== config4"; timeout 300 $B --config 4 | python -c "$P"
