#!/bin/bash
for X in ${XS:-none}; do
  [ "$X" = none ] && X=""
  X=${X//,/ }
  touch paper_2604_11554_b200/csrc/tm_r3.cu
  make -s -j8 -C paper_2604_11554_b200/csrc EXTRA="$X" > /dev/null 2>&1 || { echo build fail $X; continue; }
  echo "== [$X]"; grep -A3 "r3_fwd_fastIfLi128ELi8" paper_2604_11554_b200/lib/obj/tm_r3.ptxas.log | grep -E "registers|spill" | tr '\n' ' '; echo
  timeout -s KILL 120 python scripts/r3_split.py 2>&1 | grep -E "fwd:|bwd:"
done
