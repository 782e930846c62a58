#!/bin/bash
# One ncu --set full capture of one kernel launch of a command (after a plain run of it).
# usage: scripts/ncu_kernel.sh <name> <kernel-regex> <skip> <command...>
NAME=$1; RE=$2; SKIP=$3; shift 3
OUT=gpurun_out
timeout 300 "$@" > $OUT/${NAME}_plain.log 2>&1 || { tail -5 $OUT/${NAME}_plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
   -k regex:$RE -s $SKIP -c 1 -o $OUT/$NAME "$@" > $OUT/${NAME}.log 2>&1
tail -2 $OUT/${NAME}.log
