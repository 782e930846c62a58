#!/bin/bash
# Memory-pattern ceiling of the fused loss: copy microbenchmarks and the kernel
# with its math switched off (compile-time SFTM_DBG_MODE, rebuilt on the box).
OUT=gpurun_out/${1:-pattern}
mkdir -p $OUT
for rb in 151936 303872; do echo "== row_bytes $rb"; ./scripts/mb_copy $rb; done > $OUT/mb_copy.txt 2>&1
for D in 0 1 2 3; do
  touch paper_2604_11554_b200/csrc/tm_loss.cu
  make -s -j8 -C paper_2604_11554_b200/csrc EXTRA=-DSFTM_DBG_MODE=$D > /dev/null 2>&1 || exit 1
  echo "== dbg=$D"; timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['clocks'])"
done > $OUT/dbg.txt 2>&1
touch paper_2604_11554_b200/csrc/tm_loss.cu; make -s -j8 -C paper_2604_11554_b200/csrc > /dev/null 2>&1
cat $OUT/mb_copy.txt $OUT/dbg.txt
