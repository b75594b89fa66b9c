set -x
timeout 600 python -m pytest tests/test_gpu_decomposition.py -x -q -k "regk or allreg or segments or general_instance" > gpurun_out/c2_dec.log 2>&1; tail -3 gpurun_out/c2_dec.log
for v in implicit_upwind implicit_tvd explicit_upwind explicit_tvd; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --variant $v 2>/dev/null | tail -1 > gpurun_out/c2_bench_$v.json
  STS_OLD_REGK=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --variant $v 2>/dev/null | tail -1 > gpurun_out/c2_bench_old_$v.json
done
python - <<'PY'
import json
for v in ["implicit_upwind","implicit_tvd","explicit_upwind","explicit_tvd"]:
    for t in ["","old_"]:
        try:
            d=json.load(open(f"gpurun_out/c2_bench_{t}{v}.json")); r=d["roofline"]
            print(t or "new ", v, round(d["value"]/1e9,2), "G", "pass", round(r["pass_ms_avg"],4), "frac", round(r["frac"],3))
        except Exception as e: print(v,t,"ERR",e)
PY
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/c2_gpu.log 2>&1; tail -3 gpurun_out/c2_gpu.log
