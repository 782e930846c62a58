#!/bin/bash
# A/B: backward exponentials partly on the FMA pipe (SFTM_POLY_EXP = pairs of 8
# per thread-chunk through ex2_poly2), headline bench per variant on one box.
for P in ${PS:-0 4 8 0 2 4}; do
  X=""; [ "$P" != 0 ] && X="-DSFTM_POLY_EXP=$P"
  touch paper_2604_11554_b200/csrc/tm_loss.cu
  make -s -j8 -C paper_2604_11554_b200/csrc EXTRA="$X" > /dev/null 2>&1 || { echo build fail $P; continue; }
  echo "== poly=$P"
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value']/1e6,3), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
if [ -n "$TEST_P" ]; then
  touch paper_2604_11554_b200/csrc/tm_loss.cu
  make -s -j8 -C paper_2604_11554_b200/csrc EXTRA="-DSFTM_POLY_EXP=$TEST_P" > /dev/null 2>&1
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
fi
