timeout 600 ncu --set full --clock-control none --import-source on -k regex:regk_kernel -s 3 -c 1 -o gpurun_out/c5_regk python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --variant implicit_upwind > gpurun_out/c5_ncu.log 2>&1
tail -2 gpurun_out/c5_ncu.log
