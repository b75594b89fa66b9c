#!/bin/bash
# usage (GPU box): tools/conv_ab.sh -- ncu time of the explicit-plane kernel for two builds (edit the list)
for L in cv1 cv2 cv1 cv2; do for v in explicit_upwind explicit_tvd; do
STS_LIB=build/$L.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_march -c 6 --csv --log-file gpurun_out/kt_$L.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --variant $v > /dev/null 2>&1
python -c "
import csv; rows=[r for r in csv.reader(open('gpurun_out/kt_$L.csv')) if len(r)>10]; h=rows[0]; i=h.index('Metric Value')
v=[float(r[i].replace(',','')) for r in rows[1:]]; print('$L','$v', round(sum(v)/len(v)/1e3,1),'us')"
done; done
