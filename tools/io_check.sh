#!/bin/bash
# async host-I/O tests + the default bench line (GPU box)
timeout 600 python -m pytest tests/test_gpu_io_async.py tests/test_abi.py -q -m gpu > gpurun_out/io_tests.log 2>&1; tail -3 gpurun_out/io_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/io_smoke.log 2>&1; tail -1 gpurun_out/io_smoke.log
timeout 400 python bench.py > gpurun_out/io_bench.json 2> gpurun_out/io_bench.err; tail -1 gpurun_out/io_bench.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, json.dumps(d['e2e']))"
