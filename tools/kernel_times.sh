#!/bin/bash
# usage (GPU box): tools/kernel_times.sh TAG variant...  -- ncu launch list (cold, serialised) per variant
T=$1; shift
for v in "$@"; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/kt_${T}_$v.csv \
      python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e --variant $v > /dev/null 2>&1
  python - gpurun_out/kt_${T}_$v.csv $v <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; iN = h.index('Kernel Name'); iV = h.index('Metric Value')
t = collections.defaultdict(list)
for r in rows[1:]:
    t[r[iN].split('(')[0]].append(float(r[iV].replace(',', '')))
for k, v in t.items():
    print(sys.argv[2], k[:40], len(v), round(sum(v) / len(v) / 1e3, 1), 'us')
PY
done
