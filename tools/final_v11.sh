#!/bin/bash
# final check of the round's build on the GPU box: the -m gpu suite, smoke, the default
# bench line, and a 2-process bench on the one GPU (the N > 1 path: peer halo, pipelined e2e)
timeout 1700 python -m pytest tests -q -m gpu > gpurun_out/final_gpu.log 2>&1; tail -3 gpurun_out/final_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 300 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.json | cut -c1-200
STS_BENCH_ONE_DEVICE=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/final_bench_2proc.json 2> gpurun_out/final_bench_2proc.err
tail -1 gpurun_out/final_bench_2proc.json | cut -c1-300; tail -3 gpurun_out/final_bench_2proc.err
