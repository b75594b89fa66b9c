#!/bin/bash
# headline value (graph path) over a (Hg, Hr) grid
V=${1:-implicit_upwind}
run() { timeout 300 python bench.py --steps 60 --warmup 3 --no-cpu --no-e2e --variant $V 2> /tmp/err.txt | tail -1 | \
   python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$1', 'G', round(d['value']/1e9,2), 'ms_step', round(d['ms_per_step'],4), 'stream_pass', round(r['pass_ms_avg'],4))"; }
run auto
for hg in 8 12 16 24; do for hr in 48 64 80 96; do STS_SEG=$hg,$hr run $hg,$hr; done; done
run auto
