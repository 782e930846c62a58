#!/bin/bash
# Headline bench A/B of prebuilt library variants (_ab/<name>/), alternating on one box.
LIB=paper_2604_11554_b200/lib/libsf_train_math.so
cp $LIB /tmp/bench_ab_orig.so
for r in $(seq ${ROUNDS:-2}); do for v in $VARIANTS; do
  cp _ab/$v/libsf_train_math.so $LIB
  timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('r$r', '$v', round(d['value']/1e6,3), 'M tok/s', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
cp /tmp/bench_ab_orig.so $LIB
