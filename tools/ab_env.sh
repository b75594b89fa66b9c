#!/bin/bash
# usage (GPU box): tools/ab_env.sh "variant..." "lib[:ENV=VAL]"...  -- headline value + stream pass time
VS=$1; shift
for L in "$@"; do for v in $VS; do
  lib=${L%%:*}; envs=""; [ "$lib" != "$L" ] && envs=${L#*:}
  env $envs STS_LIB=build/$lib.so timeout 300 python bench.py --steps 40 --warmup 3 --no-cpu --no-e2e --variant $v 2>/dev/null | tail -1 | \
   python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$L', '$v', 'G', round(d['value']/1e9,2), 'stream_pass', round(r['pass_ms_avg'],4))" || echo "$L $v FAILED"
done; done
