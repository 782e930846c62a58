#!/bin/bash
# One compute-sanitizer tool per GPU call (B200_PROFILING.md): TOOL = memcheck | synccheck | racecheck | initcheck
TOOL=${1:-memcheck}
mkdir -p gpurun_out
SF_TM_XP_TIMEOUT_S=20 timeout 1200 compute-sanitizer --tool $TOOL --error-exitcode 9 --print-limit 50 \
   python scripts/sanitize_cases.py > gpurun_out/sanitize_$TOOL.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_$TOOL.log
tail -25 gpurun_out/sanitize_$TOOL.log
