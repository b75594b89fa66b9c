#!/bin/bash
# CTA fixed-cost term of the schedule model (STS_CTA_OVH, row steps per CTA) with the
# PDL step graphs: ms per step on the paper's meshes and C3 (GPU box)
for rep in 1 2; do for H in 10 20 100 200; do for V in implicit_upwind explicit_upwind; do
  H=$H V=$V timeout 300 python tools/small_mesh.py "ovh0=" "ovh1=STS_CTA_OVH:1" "ovh2=STS_CTA_OVH:2" "ovh4=STS_CTA_OVH:4" "ovh8=STS_CTA_OVH:8"
done; done; done 2>&1 | grep -v "^sts:" | tee gpurun_out/ovh_sweep.jsonl
