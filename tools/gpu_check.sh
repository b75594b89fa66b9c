#!/bin/bash
# usage: tools/gpu_check.sh "<pytest -k expr or ALL>" variant...   (runs on the GPU box)
K="$1"; shift
if [ "$K" = "ALL" ]; then timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
elif [ -n "$K" ]; then timeout 900 python -m pytest tests -q -m gpu -x -k "$K" 2>&1 | tail -3; fi
for v in "$@"; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --variant $v 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['config']['workload'], round(d['value']/1e9,2), 'GFVU/s pass_ms', round(r['pass_ms_avg'],4), 'frac', round(r['frac'],3), 'sm_mhz', d['clocks']['sm_mhz'])"
done
