#!/bin/bash
# implicit TVD: one fused launch per pass (STS_ITVD_FUSED=1) vs the two-kernel pass (GPU box)
for rep in 1 2; do for H in 10 20 100 200; do
  H=$H V=implicit_tvd timeout 300 python tools/small_mesh.py "two=" "fused=STS_ITVD_FUSED:1"
done; done 2>&1 | grep -v "^sts:" | tee gpurun_out/itvd_ab.jsonl
