#!/bin/bash
# One full ncu capture of the fused loss kernel on the small config.
# usage: scripts/ncu_full.sh <name> <kernel-regex> [env...]
NAME=$1; RE=$2; shift 2
OUT=gpurun_out
SMALL="python bench.py --seqs-per-mb 4 --micro-batches 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
env "$@" timeout 300 $SMALL > $OUT/${NAME}_plain.log 2>&1 || { cat $OUT/${NAME}_plain.log; exit 1; }
env "$@" timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
   -k regex:$RE -s 1 -c 1 -o $OUT/$NAME $SMALL > $OUT/${NAME}.log 2>&1
tail -3 $OUT/${NAME}.log
