# Round evidence, one ncu per gpurun call (run from the repo root under gpurun):
#   bash scripts/prof_evidence.sh launches   plain bench, then the ncu launch list of the same command
#   bash scripts/prof_evidence.sh full       one --set full capture of the fused kernel (small config)
#   bash scripts/prof_evidence.sh traffic    DRAM bytes of one fused launch at the headline size
# Each ncu runs only after the same command exited 0 without it.
set -x
OUT=gpurun_out
K=${KREGEX:-regex:loss_tmem_kernelItLi1E}
case "$1" in
launches)
  timeout 600 python bench.py > $OUT/ev_plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/ev_launches.csv \
     python bench.py --steps 2 --warmup 1 > $OUT/ev_launches.log 2>&1 ;;
full)
  SMALL="python bench.py --seqs-per-mb 4 --micro-batches 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 300 $SMALL > $OUT/ev_small_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
     -k $K -s 1 -c 1 -o $OUT/ev_full $SMALL > $OUT/ev_full.log 2>&1 ;;
traffic)
  HEAD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 600 $HEAD > $OUT/ev_head_plain.log 2>&1 && \
  timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
     --kernel-name-base mangled -k $K -s 2 -c 1 --csv --log-file $OUT/ev_traffic.csv $HEAD > $OUT/ev_traffic.log 2>&1 ;;
esac
echo "done rc=$?"
