#!/bin/bash
# compute-sanitizer over the CUDA path on small cases (GPU box): memcheck, racecheck (shared-memory
# ring / row buffers), initcheck, synccheck.  usage: tools/sanitize.sh > gpurun_out/sanitize.log
K='test_regk_same_bits or test_allreg_loop_bitwise or test_parity_small_square or test_parity_ragged_tiles or test_parity_periodic or test_slabs_bitwise or test_nonuniform_small_square or test_loop3_small_square or test_peer_group_bitwise'
for tool in memcheck racecheck initcheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_parity.py tests/test_gpu_decomposition.py tests/test_gpu_graph.py \
       tests/test_gpu_nonuniform.py tests/test_gpu_loop3.py -q -x -m gpu -k "$K" 2>&1 | \
     grep -E "ERROR SUMMARY|passed|failed|Error|error" | tail -6
  echo "exit ${PIPESTATUS[0]}"
done
# conditional-WHILE graphs: the tolerance-mode kernels stream-launched (graph instances,
# STS_GRAPH_KERNEL) under synccheck / racecheck, and a minimal conditional graph with
# a trivially correct kernel (tools/cond_graph_probe.cu) to test the tool itself
for tool in synccheck racecheck; do
  echo "== $tool, graph kernel instances stream-launched (tolerance mode, host loop)"
  STS_NO_GRAPH=1 STS_GRAPH_KERNEL=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k test_tolerance_mode_converges 2>&1 | \
     grep -E "ERROR SUMMARY|HAZARD|hazards|passed|failed" | tail -4
  echo "exit ${PIPESTATUS[0]}"
  echo "== $tool, minimal conditional-WHILE graph probe"
  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cond_graph_probe tools/cond_graph_probe.cu && \
    timeout 300 compute-sanitizer --tool $tool --print-limit 5 /tmp/cond_graph_probe 2>&1 | tail -8
  echo "exit ${PIPESTATUS[0]}"
done
