#!/bin/bash
mkdir -p gpurun_out/r2c
timeout 300 ./oracle/_ref/test_bus_seam_gpu bench 16 > gpurun_out/r2c/bus_bench.json 2>&1; cat gpurun_out/r2c/bus_bench.json
timeout 600 python scripts/vp_emulate.py 32768 > gpurun_out/r2c/vp_emulate.jsonl 2>&1; cat gpurun_out/r2c/vp_emulate.jsonl
bash scripts/sanitize.sh memcheck
