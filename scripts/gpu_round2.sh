#!/bin/bash
# GPU pass: all GPU tests, smoke, the default bench line (+ reference arm),
# the bus-driven C++ trainer e2e, config 5 at P=1.
TAG=${1:-r2b}
OUT=gpurun_out/$TAG
mkdir -p $OUT
lscpu > $OUT/cpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest.log 2>&1; echo "pytest_rc=$?" >> $OUT/pytest.log
tail -15 $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
tail -c 2500 $OUT/bench.json; tail -3 $OUT/bench.err
timeout 400 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/ref.json 2> $OUT/ref.err; echo "rc=$?" >> $OUT/ref.err
tail -c 1500 $OUT/ref.json
timeout 300 ./oracle/_ref/test_bus_seam_gpu bench 16 > $OUT/bus_bench.json 2>&1; cat $OUT/bus_bench.json
timeout 600 python bench.py --config 5 --steps 3 --warmup 1 > $OUT/cfg5_p1.json 2>&1; tail -c 1500 $OUT/cfg5_p1.json
