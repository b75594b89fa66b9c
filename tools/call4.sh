timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/c4_gpu.log 2>&1; tail -5 gpurun_out/c4_gpu.log
timeout 300 python bench.py > gpurun_out/c4_bench.json 2> gpurun_out/c4_bench.err; tail -1 gpurun_out/c4_bench.json | cut -c1-400
