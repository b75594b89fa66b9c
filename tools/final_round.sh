#!/bin/bash
# End-of-round evidence on the GPU box: GPU tests + smoke, the profile round, the
# other variants' / workloads' bench lines, the grid sweep.  usage: tools/final_round.sh TAG
T=${1:-r02z}
O=gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > $O/gputests_$T.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$T.log 2>&1
bash tools/profile_round.sh $T
python bench.py --variant implicit_tvd --no-cpu > $O/bench_${T}_implicit_tvd.json 2>/dev/null
python bench.py --variant explicit_upwind --no-cpu > $O/bench_${T}_explicit_upwind.json 2>/dev/null
python bench.py --variant explicit_tvd --steps 40 --no-cpu > $O/bench_${T}_explicit_tvd.json 2>/dev/null
python bench.py --workload C4 --steps 10 --no-cpu --no-e2e > $O/bench_${T}_c4.json 2>/dev/null
python bench.py --workload C5 --steps 5 --no-cpu --no-e2e > $O/bench_${T}_c5.json 2>/dev/null
timeout 600 python tools/sweep.py > $O/sweep_$T.jsonl 2>&1
