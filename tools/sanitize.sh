#!/bin/bash
# compute-sanitizer over the CUDA path on small cases (GPU box): memcheck, racecheck (shared-memory
# ring / row buffers), initcheck, synccheck.  usage: tools/sanitize.sh > gpurun_out/sanitize.log
K='test_parity_small_square or test_parity_ragged_tiles or test_parity_periodic or test_slabs_bitwise or test_graph_loop_matches or test_nonuniform_small_square or test_loop3_small_square or test_peer_group_bitwise'
for tool in memcheck racecheck initcheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_parity.py tests/test_gpu_decomposition.py tests/test_gpu_graph.py \
       tests/test_gpu_nonuniform.py tests/test_gpu_loop3.py -q -x -m gpu -k "$K" 2>&1 | \
     grep -E "ERROR SUMMARY|passed|failed|Error|error" | tail -6
  echo "exit ${PIPESTATUS[0]}"
done
