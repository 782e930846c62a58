#!/bin/bash
# Peer-exchange variants (_ab/<name>/) on N real GPUs: config 5 at Qwen3 and at an odd vocabulary.
N=${N:-4}
LIB=paper_2604_11554_b200/lib/libsf_train_math.so
cp $LIB /tmp/xp_multi_orig.so
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for W in 12560 12569; do timeout 300 python scripts/narrow_rows.py 65536 $W; done
port=29600
for v in $VARIANTS; do
  cp _ab/$v/libsf_train_math.so $LIB
  for V in 151936 50257; do
    port=$((port+1))
    timeout 600 $R --master-port $port bench.py --gpus $N --config 5 --vocab $V --steps 3 --warmup 1 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', $V, round(d['value']/1e6,2), 'M tok/s', round(d['roofline']['frac'],3))"
  done
done
cp /tmp/xp_multi_orig.so $LIB
