#!/bin/bash
# Round-2 v10 profile on the GPU box: default bench + reference arm, launch lists, and
# one ncu --set full capture of one pass per variant (march_fused_kernel: one launch;
# implicit TVD: the general + all-regular kernels).  usage: tools/profile_v10.sh TAG
T=${1:-r02v10}
O=gpurun_out
python bench.py > $O/bench_$T.json 2> $O/bench_$T.err
python bench.py --impl reference > $O/bench_ref_$T.json 2> $O/bench_ref_$T.err
for v in implicit_upwind implicit_tvd explicit_upwind explicit_tvd; do
  python bench.py --steps 40 --warmup 3 --no-cpu --variant $v > $O/bench_${T}_$v.json 2> /dev/null
done
python bench.py --steps 20 --warmup 3 --no-cpu --workload C4 > $O/bench_${T}_c4.json 2> /dev/null
python bench.py --steps 10 --warmup 3 --no-cpu --workload C5 > $O/bench_${T}_c5.json 2> /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_$T.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_${T}_explicit.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --variant explicit_upwind > /dev/null 2>&1
for v in implicit_upwind implicit_tvd explicit_upwind explicit_tvd; do
  c=1; [ $v = implicit_tvd ] && c=2
  ncu --set full --clock-control none --import-source on -k regex:"march_" -s 6 -c $c -o $O/prof_${T}_$v \
      python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --variant $v > $O/ncu_${T}_$v.log 2>&1
  ncu -i $O/prof_${T}_$v.ncu-rep --page raw --csv > $O/prof_${T}_$v.raw.csv 2>/dev/null
  [ $v = implicit_upwind ] || rm -f $O/prof_${T}_$v.ncu-rep      # gpurun_out is capped at 64 MiB
done
python tools/sweep.py > $O/sweep_$T.jsonl 2>/dev/null
