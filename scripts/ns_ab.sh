#!/bin/bash
# Row-stream count A/B of the fused loss (SFTM_LOSS_NS forces 1 / 2 / 4 where a row fits).
for r in 1 2; do
  for W in ${WIDTHS:-18992 37984 75968 151936}; do
    T=65536; [ $W -gt 100000 ] && T=32768
    for NS in ${NSS:-1 2 4}; do
      echo -n "r$r NS=$NS: "; SFTM_LOSS_NS=$NS timeout 300 python scripts/narrow_rows.py $T $W
    done
  done
done
