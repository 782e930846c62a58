#!/bin/bash
mkdir -p gpurun_out/r2e
timeout 300 python scripts/narrow_rows.py 16384 18992 > gpurun_out/r2e/narrow_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loss_tmem_kernel -s 3 -c 1 \
   -o gpurun_out/r2e/narrow18992 python scripts/narrow_rows.py 16384 18992 > gpurun_out/r2e/narrow_ncu.log 2>&1
tail -1 gpurun_out/r2e/narrow_ncu.log
timeout 300 python scripts/narrow_rows.py 16384 151936 > gpurun_out/r2e/wide_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loss_tmem_kernel -s 3 -c 1 \
   -o gpurun_out/r2e/wide151936 python scripts/narrow_rows.py 16384 151936 > gpurun_out/r2e/wide_ncu.log 2>&1
tail -1 gpurun_out/r2e/wide_ncu.log
