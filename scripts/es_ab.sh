#!/bin/bash
# bench A/B: e-store vs raw row store (kernel-only, same box)
OUT=gpurun_out/${1:-esab}
mkdir -p $OUT
run() {
  echo "== $*"
  env "$@" timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; print('frac %.4f kms %.3f' % (r['frac'], r['avg_launch_ms']), d['clocks'])"
}
{ run SFTM_ES=1; run SFTM_ES=0; run SFTM_ES=1; run SFTM_ES=0; } > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
[ -n "$2" ] && bash scripts/r2_wait.sh
