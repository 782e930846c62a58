#!/bin/bash
# every BASELINE config's bench line at N=1 with the current build
mkdir -p gpurun_out/cfg
for c in 1 3 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 2 > gpurun_out/cfg/config$c.json 2>&1; tail -c 900 gpurun_out/cfg/config$c.json; echo; done
timeout 600 python bench.py --fwd-only --steps 5 --warmup 2 > gpurun_out/cfg/fwd_only.json 2>&1; tail -c 700 gpurun_out/cfg/fwd_only.json
