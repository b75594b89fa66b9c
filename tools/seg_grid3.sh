#!/bin/bash
# headline value (graph path, fused kernel) over (Hg, Hr), C3 implicit upwind
run() { timeout 300 python bench.py --steps 60 --warmup 3 --no-cpu --no-e2e 2> /dev/null | tail -1 | \
   python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$1', 'G', round(d['value']/1e9,2))"; }
run auto
for hg in 12 16 24 48 96; do for hr in 64 94; do STS_SEG=$hg,$hr run $hg,$hr; done; done
run auto
