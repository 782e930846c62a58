set -x
timeout 300 python bench.py --generic --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_generic.log 2>&1
SMALL="python bench.py --seqs-per-mb 4 --micro-batches 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $SMALL > gpurun_out/small_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:rows_ring_kernelItLi2ELi1E -s 1 -c 1 -o gpurun_out/prof_fused_r1 $SMALL > gpurun_out/ncu_full.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 1 > gpurun_out/plain_default.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launches.log 2>&1
echo done
