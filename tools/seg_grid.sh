#!/bin/bash
# pass time over a (Hg, Hr) grid (STS_SEG=Hg,Hr) and the automatic choice for given model params
V=${1:-implicit_upwind}; W=${2:-C3}
run() { timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --variant $V --workload ${W} 2> /tmp/err.txt | tail -1 | \
   python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$1', 'pass_ms', round(r['pass_ms_avg'],4), 'G', round(d['value']/1e9,2))"; grep "sts: Hg" /tmp/err.txt | head -1; }
export STS_VERBOSE=1
for ov in 0 2 4 8; do STS_CTA_OVH=$ov run auto_ovh$ov; done
for hg in 16 32 48; do for hr in 32 48 64; do STS_SEG=$hg,$hr run $hg,$hr; done; done
