#!/bin/bash
# usage (GPU box): tools/prof2.sh TAG [variant]  -- serialized per-kernel times of a few passes + one ncu --set full
# capture of the general and the all-regular march kernel of one pass
T=$1; V=${2:-implicit_upwind}
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:march_kernel -c 12 --csv --log-file gpurun_out/klist_${T}_$V.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --variant $V > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 10 -c 2 -o gpurun_out/prof_${T}_$V \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --variant $V > gpurun_out/ncu_${T}_$V.log 2>&1
