#!/bin/bash
# usage (GPU box): tools/seg_sweep.sh "variant" seg... -- pass time of C3 H200 with forced segment heights (STS_SEG)
V=$1; shift
for sg in "$@"; do
  STS_SEG=$sg timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --variant $V 2>/dev/null | tail -1 | \
   python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('seg $sg', '$V', 'pass_ms', round(r['pass_ms_avg'],4), 'GFVU/s', round(d['value']/1e9,2))"
done
