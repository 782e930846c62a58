#!/bin/bash
for W in 18992 37984 50257 151936; do python scripts/narrow_rows.py 65536 $W; done
timeout 600 python scripts/vp_emulate.py 32768 2>&1 | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "pg_loss or all_rows or neg_inf or deep or vp_fused or cluster" --timeout 600 2>&1 | tail -3
