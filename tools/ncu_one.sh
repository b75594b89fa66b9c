#!/bin/bash
# usage: tools/ncu_one.sh TAG variant...  -- one ncu --set full capture of the pass kernel per variant (GPU box)
T=$1; shift
for v in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 5 -c 1 -o gpurun_out/prof_${T}_$v \
      python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --variant $v > gpurun_out/ncu_${T}_$v.log 2>&1
done
