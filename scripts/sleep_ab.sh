#!/bin/bash
# A/B of the back-off sleeps (SFTM_SLEEP_BWD / SFTM_SLEEP_CTL, ns) and the row store (SFTM_ES).
OUT=gpurun_out/${1:-sleep}
mkdir -p $OUT
run() {
  echo "== $*"
  env "$@" timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; print('frac %.4f kms %.3f' % (r['frac'], r['avg_launch_ms']), d['clocks'])"
}
{
run SFTM_ES=1
run SFTM_ES=0
run SFTM_ES=1 SFTM_SLEEP_BWD=200
run SFTM_ES=1 SFTM_SLEEP_BWD=500
run SFTM_ES=1 SFTM_SLEEP_BWD=500 SFTM_SLEEP_CTL=100
run SFTM_ES=1 SFTM_SLEEP_BWD=1000 SFTM_SLEEP_CTL=200
run SFTM_ES=0 SFTM_SLEEP_BWD=500 SFTM_SLEEP_CTL=100
run SFTM_ES=0 SFTM_SLEEP_BWD=200
run SFTM_ES=1
} > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
