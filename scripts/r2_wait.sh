#!/bin/bash
# per-role wait breakdown of the fused loss (instrumented build on the box)
touch paper_2604_11554_b200/csrc/tm_loss.cu
make -s -j8 -C paper_2604_11554_b200/csrc EXTRA=-DSFTM_WAIT_PROFILE > /dev/null 2>&1 || exit 1
for V in ${VS:-151936 37984 18992}; do python scripts/wait_profile.py ${ROWS:-32768} $V; done
