#!/bin/bash
# pass time vs forced segment height (STS_SEG) for the default workload, regk build
for seg in auto 16 24 32 40 48 64 96; do
  if [ $seg = auto ]; then unset STS_SEG; else export STS_SEG=$seg; fi
  STS_VERBOSE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --variant ${1:-implicit_upwind} 2> /tmp/err.txt | tail -1 | \
   python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$seg', 'pass_ms', round(r['pass_ms_avg'],4), 'frac', round(r['frac'],3))"
  grep "sts: Hg" /tmp/err.txt | head -1
done
