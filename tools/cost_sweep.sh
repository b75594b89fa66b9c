#!/bin/bash
# usage (GPU box): tools/cost_sweep.sh variant "g,m"...  -- pass time with scheduler warp-cost weights STS_COST=g,m
V=$1; shift
for w in "$@"; do
  STS_COST=$w STS_VERBOSE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --variant $V 2>/tmp/err | tail -1 | \
   python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('cost $w', '$V', 'pass_ms', round(r['pass_ms_avg'],4))"; grep "sts:" /tmp/err | head -1
done
