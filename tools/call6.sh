export STS_VERBOSE=1
for r in 1 2; do
timeout 300 python bench.py --steps 100 --warmup 3 --no-cpu --no-e2e 2> /tmp/e.txt | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('C3 auto', 'G', round(d['value']/1e9,2), 'stream_pass', round(r['pass_ms_avg'],4))"; grep "sts: Hg" /tmp/e.txt | head -1
done
python tools/sweep.py > gpurun_out/c6_sweep.jsonl 2>/dev/null; cat gpurun_out/c6_sweep.jsonl
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print({k:d[k] for k in d if k in ('mesh','variant','gfvus','G','value','ny','pass_ms','workload')})
" | head -20
