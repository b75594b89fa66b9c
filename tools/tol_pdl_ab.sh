#!/bin/bash
# tolerance-mode graphs with / without PDL edges: graph tests, then steps/s (GPU box)
timeout 900 python -m pytest tests/test_gpu_graph.py -q -m gpu -x > gpurun_out/tolpdl_tests.log 2>&1; tail -3 gpurun_out/tolpdl_tests.log
grep -h "without PDL" gpurun_out/tolpdl_tests.log | head -2
for rep in 1 2; do
  timeout 300 python tools/time_tolmode.py 2>&1 | grep -v "^sts: Hg" | sed 's/^/pdl /'
  STS_NO_PDL=1 timeout 300 python tools/time_tolmode.py 2>&1 | grep -v "^sts: Hg" | sed 's/^/nopdl /'
done | tee gpurun_out/tolpdl_ab.txt
