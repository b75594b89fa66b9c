#!/bin/bash
# final check of the round's build on the GPU box: the -m gpu suite, smoke, the default bench line
timeout 1700 python -m pytest tests -q -m gpu > gpurun_out/final_gpu.log 2>&1; tail -3 gpurun_out/final_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 300 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.json | cut -c1-200
