#!/bin/bash
# usage (GPU box): tools/ab.sh "variant..." lib1 lib2 ...  -- pass time of each build/libN.so, interleaved twice
VS=$1; shift
for rep in 1 2; do
for L in "$@"; do for v in $VS; do
  STS_LIB=build/$L.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --variant $v 2>/dev/null | tail -1 | \
   python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$L', '$v', 'pass_ms', round(r['pass_ms_avg'],4), 'frac', round(r['frac'],3))" || echo "$L $v FAILED"
done; done; done
