#!/bin/bash
# One GPU-box pass: GPU tests, smoke, bench (e-store default) and the raw-store A/B.
# usage (via gpurun): bash scripts/gpu_round.sh TAG [pytest -k expr]
TAG=${1:-run}
K=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
lscpu | head -20 > $OUT/cpu.txt 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf -k "$K" --timeout 600 > $OUT/pytest.log 2>&1; echo "pytest_rc=$?" >> $OUT/pytest.log
else
  timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > $OUT/pytest.log 2>&1; echo "pytest_rc=$?" >> $OUT/pytest.log
fi
tail -30 $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke.log
tail -3 $OUT/smoke.log
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_es.json 2> $OUT/bench_es.err; echo "rc=$?" >> $OUT/bench_es.err
SFTM_ES=0 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_raw.json 2> $OUT/bench_raw.err; echo "rc=$?" >> $OUT/bench_raw.err
python - <<'PY' $OUT
import json, sys
o = sys.argv[1]
for n in ("bench_es", "bench_raw"):
    try:
        d = json.loads(open(f"{o}/{n}.json").read().strip().splitlines()[-1])
        r = d["roofline"]
        print(n, "value %.3fM" % (d["value"] / 1e6), "frac %.4f" % r["frac"], "kms %.3f" % r["avg_launch_ms"],
              "clk", d.get("clocks"), "e2e", (d.get("e2e") or {}).get("value"))
    except Exception as ex:
        print(n, "failed", ex)
PY
