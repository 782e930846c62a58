#!/bin/bash
mkdir -p gpurun_out/r2d
SFTM_ES=1 timeout 600 python scripts/vp_emulate.py 32768 > gpurun_out/r2d/vp_emulate_es.jsonl 2>&1; cat gpurun_out/r2d/vp_emulate_es.jsonl
for W in 18992 37984; do python scripts/narrow_rows.py 65536 $W; SFTM_ES=1 python scripts/narrow_rows.py 65536 $W; done
timeout 300 python scripts/narrow_rows.py 16384 18992 > gpurun_out/r2d/narrow_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loss_tmem_kernel -s 3 -c 1 \
   -o gpurun_out/r2d/narrow18992 python scripts/narrow_rows.py 16384 18992 > gpurun_out/r2d/narrow_ncu.log 2>&1
tail -2 gpurun_out/r2d/narrow_ncu.log
