#!/bin/bash
# A/B of programmatic-dependent-launch edges in the fixed-pass step graphs (GPU box):
# graph tests, then the paper's small meshes and C3 with and without PDL (interleaved twice)
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pdl_tests.log 2>&1; tail -2 gpurun_out/pdl_tests.log
for rep in 1 2; do
for H in 10 20 200; do for V in implicit_upwind implicit_tvd explicit_upwind; do
  H=$H V=$V timeout 300 python tools/small_mesh.py "pdl=" "nopdl=STS_NO_PDL:1"
done; done; done 2>&1 | tee gpurun_out/pdl_ab.jsonl
