#!/bin/bash
# quick perf snapshot: narrow rows, VP emulation, headline bench (kernel-only)
for W in 18992 37984 50257 151936; do python scripts/narrow_rows.py 65536 $W; done
timeout 400 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; print('headline value %.3fM frac %.4f kms %.3f' % (d['value']/1e6, r['frac'], r['avg_launch_ms']), d['clocks'])"
