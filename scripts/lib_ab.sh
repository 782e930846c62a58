#!/bin/bash
# A/B of prebuilt variants of libsf_train_math.so (built here under _ab/<name>/,
# see DESIGN.md §5): each variant is copied over the in-tree library in turn and
# timed on the same box, interleaved over ROUNDS passes to average out drift.
# Usage: VARIANTS="base nbar" WIDTHS="18992 151936" [CHECK=1] bash scripts/lib_ab.sh
set -u
LIB=paper_2604_11554_b200/lib/libsf_train_math.so
cp $LIB /tmp/lib_ab_orig.so
if [ "${CHECK:-0}" = 1 ]; then
  for v in $VARIANTS; do
    cp _ab/$v/libsf_train_math.so $LIB
    echo "== check $v"
    timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "pg_loss or fused_all_rows or neg_inf or vocab_parallel" 2>&1 | tail -2
    timeout 600 python -m pytest -q -x tests/test_gpu_configs.py -k "vp_fused" 2>&1 | tail -2
  done
fi
for r in $(seq ${ROUNDS:-2}); do
  for v in $VARIANTS; do
    cp _ab/$v/libsf_train_math.so $LIB
    for W in $WIDTHS; do
      T=65536; [ $W -gt 100000 ] && T=32768
      echo -n "r$r $v: "; timeout 300 python scripts/narrow_rows.py $T $W
    done
  done
done
cp /tmp/lib_ab_orig.so $LIB
