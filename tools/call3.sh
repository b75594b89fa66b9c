python tools/regk_diag.py implicit_upwind explicit_upwind implicit_tvd explicit_tvd 2>&1 | grep -v same | head -20
echo DIAG_DONE
timeout 900 python -m pytest tests/test_gpu_decomposition.py -x -q 2>&1 | tail -3
for v in implicit_upwind implicit_tvd explicit_upwind; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --variant $v 2>/dev/null | tail -1 > gpurun_out/c3_bench_$v.json
  STS_OLD_REGK=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --variant $v 2>/dev/null | tail -1 > gpurun_out/c3_bench_old_$v.json
done
python - <<'PY'
import json
for v in ["implicit_upwind","implicit_tvd","explicit_upwind"]:
    for t in ["","old_"]:
        try:
            d=json.load(open(f"gpurun_out/c3_bench_{t}{v}.json")); r=d["roofline"]
            print(t or "new ", v, round(d["value"]/1e9,2), "G", "pass", round(r["pass_ms_avg"],4), "frac", round(r["frac"],3))
        except Exception as e: print(v,t,"ERR",e)
PY
