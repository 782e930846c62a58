#!/bin/bash
# A/B build variants of tm_loss.cu: narrow-row (xp_self) and headline timings on one box.
for X in ${XS:-none}; do
  [ "$X" = none ] && X=""
  X=${X//,/ }
  touch paper_2604_11554_b200/csrc/tm_loss.cu
  touch paper_2604_11554_b200/csrc/*.cu; make -s -j8 -C paper_2604_11554_b200/csrc EXTRA="$X" > /dev/null 2>&1 || { echo build fail $X; continue; }
  echo "== [$X]"
  timeout -s KILL 120 python scripts/xp_self.py 2>&1 | grep plain
  CS=0 bash scripts/try_cs.sh 2>&1 | grep -v "==" | head -1
done
