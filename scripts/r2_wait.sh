#!/bin/bash
# per-role wait breakdown, e-store vs raw row store (instrumented build on the box)
touch paper_2604_11554_b200/csrc/tm_loss.cu
make -s -j8 -C paper_2604_11554_b200/csrc EXTRA=-DSFTM_WAIT_PROFILE > /dev/null 2>&1 || exit 1
for ES in 1 0; do echo "== SFTM_ES=$ES"; SFTM_ES=$ES python scripts/wait_profile.py 32768 151936; done
