timeout 900 python -m pytest tests/test_gpu_graph.py -q -m gpu -k "pdl" > gpurun_out/pdl_test.log 2>&1; tail -2 gpurun_out/pdl_test.log
STS_BENCH_ONE_DEVICE=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/final_bench_2proc.json 2> gpurun_out/final_bench_2proc.err
tail -1 gpurun_out/final_bench_2proc.json | cut -c1-400; grep -i "error" gpurun_out/final_bench_2proc.err | head -5
