#!/bin/bash
for W in 18992 37984; do
for cfg in "0 0" "100 0" "300 0" "300 100" "1000 200" "0 200"; do
  set -- $cfg
  echo -n "W=$W bwd=$1 ctl=$2: "; SFTM_SLEEP_BWD=$1 SFTM_SLEEP_CTL=$2 python scripts/narrow_rows.py 65536 $W
done; done
echo -n "qwen bwd=0: "; python scripts/narrow_rows.py 32768 151936
echo -n "qwen bwd=300: "; SFTM_SLEEP_BWD=300 python scripts/narrow_rows.py 32768 151936
