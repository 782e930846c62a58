#!/bin/bash
# Race hunt: stress_logp.py under build variants (EXTRA flags), one box.
for X in ${XS:-none}; do
  [ "$X" = none ] && X=""
  touch paper_2604_11554_b200/csrc/tm_loss.cu
  make -s -j8 -C paper_2604_11554_b200/csrc EXTRA="$X" > /dev/null 2>&1 || { echo build fail $X; continue; }
  echo "== [$X]"; ITERS=${ITERS:-4} SHAPES=${SHAPES:-1} timeout 300 python scripts/stress_logp.py 2>&1 | tail -${TAILN:-3}
done
