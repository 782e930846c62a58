#!/bin/bash
# Multi-GPU checks and scaling lines (run under gpurun --gpus N from the repo root).
N=${1:-2}
OUT=gpurun_out/multi$N
mkdir -p $OUT
nvidia-smi topo -m > $OUT/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -rf > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
tail -3 $OUT/pytest.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $R --master-port 29511 bench.py --gpus $N --steps 5 --warmup 3 > $OUT/bench.log 2>&1
timeout 900 $R --master-port 29512 bench.py --gpus $N --config 5 --steps 3 --warmup 1 > $OUT/vp.log 2>&1
timeout 900 $R --master-port 29513 bench.py --gpus $N --config 5 --vp-two-pass --steps 3 --warmup 1 > $OUT/vp2.log 2>&1
timeout 600 $R --master-port 29514 bench.py --gpus $N --impl reference --steps 5 --warmup 1 > $OUT/ref.log 2>&1
timeout 900 $R --master-port 29515 bench.py --gpus $N --config 5 --vocab 50257 --steps 3 --warmup 1 > $OUT/vp_odd.log 2>&1
for f in bench vp vp2 ref vp_odd; do echo "== $f"; grep '^{' $OUT/$f.log | tail -1 | cut -c1-600; done
echo done
