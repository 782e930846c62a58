#!/bin/bash
# Instruction count / duration of one fused-loss launch per library variant (ncu, cold serialised launch).
LIB=paper_2604_11554_b200/lib/libsf_train_math.so
cp $LIB /tmp/ncu_ab_orig.so
for v in $VARIANTS; do
  cp _ab/$v/libsf_train_math.so $LIB
  for W in $WIDTHS; do
    timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:loss_tmem_kernel -s 3 -c 1 --csv python scripts/narrow_rows.py 16384 $W 2>/dev/null | grep -E "inst_executed|time_duration|issue_active" | awk -F'","' -v v=$v -v w=$W '{print v, w, $(NF-2), $NF}'
  done
done
cp /tmp/ncu_ab_orig.so $LIB
