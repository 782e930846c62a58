set -x
SMALL="python bench.py --seqs-per-mb 4 --micro-batches 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $SMALL > gpurun_out/small_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:loss_tmem_kernelItLi2E -s 1 -c 1 -o gpurun_out/prof_fused_r1f $SMALL > gpurun_out/ncu_full_f.log 2>&1
echo done
