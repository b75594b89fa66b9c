set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
tail -1 gpurun_out/c1_bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 6 -c 2 -o gpurun_out/c1_prof python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --variant implicit_upwind > gpurun_out/c1_ncu.log 2>&1
ls -la gpurun_out
