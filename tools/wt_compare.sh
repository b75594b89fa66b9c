#!/bin/bash
# usage (GPU box): tools/wt_compare.sh dir...  -- quick bench of several worktrees (A/B of commits)
for d in "$@"; do
  for v in implicit_upwind implicit_tvd explicit_upwind; do
    (cd $d && timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --variant $v 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$d', '$v', round(d['value']/1e9,2), 'GFVU/s pass_ms', round(r['pass_ms_avg'],4), 'frac', round(r['frac'],3))")
  done
done
