#!/bin/bash
mkdir -p gpurun_out
./scripts/mb_cvt > gpurun_out/mb_cvt.txt 2>&1; cat gpurun_out/mb_cvt.txt
bash scripts/ncu_full.sh r2_es loss_tmem_kernel
bash scripts/ncu_full.sh r2_raw loss_tmem_kernel SFTM_ES=0
ls -la gpurun_out/*.ncu-rep
