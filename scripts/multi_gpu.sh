# Multi-GPU checks and scaling lines (run under gpurun --gpus N from the repo root).
N=${1:-2}
set -x
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/multi_pytest_$N.log 2>&1; echo rc=$? >> gpurun_out/multi_pytest_$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus $N --steps 3 --warmup 2 > gpurun_out/multi_bench_$N.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
   bench.py --gpus $N --config 5 --steps 3 --warmup 2 > gpurun_out/multi_vp_$N.log 2>&1
echo done
