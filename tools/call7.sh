timeout 600 python -m pytest tests/test_gpu_decomposition.py tests/test_gpu_graph.py -x -q 2>&1 | tail -3
for v in implicit_upwind implicit_tvd explicit_upwind explicit_tvd; do
 for e in "" "STS_NO_FUSED=1"; do
  env $e timeout 300 python bench.py --steps 60 --warmup 3 --no-cpu --no-e2e --variant $v 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$v', '${e:-fused}', 'G', round(d['value']/1e9,2), 'stream_pass', round(r['pass_ms_avg'],4))"
 done
done
