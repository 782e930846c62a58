#!/bin/bash
# A/B of prebuilt library variants (_ab/<name>/) on the P = 1/2/4/8 vocab-parallel emulation.
LIB=paper_2604_11554_b200/lib/libsf_train_math.so
cp $LIB /tmp/xp_ab_orig.so
for r in 1 2; do for v in $VARIANTS; do
  cp _ab/$v/libsf_train_math.so $LIB
  echo "== r$r $v"; timeout 300 python scripts/vp_emulate.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['P'], round(d['frac'],3), round(d['narrow_rows_no_exchange_frac'],3))"
done; done
cp /tmp/xp_ab_orig.so $LIB
