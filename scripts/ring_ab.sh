#!/bin/bash
# TMA ring depth A/B (compile-time SFTM_RING_SLOTS; stash slots = 18 - ring)
for R in 8 10 12 6; do
  touch paper_2604_11554_b200/csrc/tm_loss.cu
  make -s -j8 -C paper_2604_11554_b200/csrc EXTRA=-DSFTM_RING_SLOTS=$R > /dev/null 2>&1 || { echo "build $R failed"; continue; }
  echo "== ring $R"
  for W in 18992 37984 151936; do python scripts/narrow_rows.py 65536 $W; done
done
touch paper_2604_11554_b200/csrc/tm_loss.cu; make -s -j8 -C paper_2604_11554_b200/csrc > /dev/null 2>&1
