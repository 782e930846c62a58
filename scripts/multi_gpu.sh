# Multi-GPU checks and scaling lines (run under gpurun --gpus N from the repo root).
N=${1:-2}
REPS=${REPS:-1}
set -x
for i in $(seq $REPS); do
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/multi_pytest_$N.log 2>&1; echo rc=$? >> gpurun_out/multi_pytest_$N.log
grep -E "^E .*Assert|passed|failed|rc=" gpurun_out/multi_pytest_$N.log
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $R --master-port 29511 bench.py --gpus $N --steps 3 --warmup 2 > gpurun_out/multi_bench_$N.log 2>&1
timeout 900 $R --master-port 29512 bench.py --gpus $N --config 5 --steps 3 --warmup 2 > gpurun_out/multi_vp_$N.log 2>&1
timeout 900 $R --master-port 29513 bench.py --gpus $N --config 5 --vp-two-pass --steps 3 --warmup 2 > gpurun_out/multi_vp2_$N.log 2>&1
for f in multi_bench multi_vp multi_vp2; do tail -1 gpurun_out/${f}_$N.log | cut -c1-400; done
echo done
