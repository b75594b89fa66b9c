#!/bin/bash
# Round profile on the GPU box: default bench + reference arm, launch lists, and one
# ncu --set full capture per variant of both march kernels of a pass (the general
# kernel and the all-regular one).  usage: tools/profile_round.sh TAG
T=${1:-r02}
O=gpurun_out
python bench.py > $O/bench_$T.json 2> $O/bench_$T.err
python bench.py --impl reference > $O/bench_ref_$T.json 2> $O/bench_ref_$T.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_$T.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_${T}_explicit.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --variant explicit_upwind > /dev/null 2>&1
for v in implicit_upwind implicit_tvd explicit_upwind explicit_tvd; do
  ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 6 -c 2 -o $O/prof_${T}_$v \
      python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --variant $v > $O/ncu_${T}_$v.log 2>&1
done
