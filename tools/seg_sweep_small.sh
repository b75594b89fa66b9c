#!/bin/bash
# usage (GPU box): tools/seg_sweep_small.sh H seg... -- ms per step of C3 4032 x (20 H) with forced segment heights
H=$1; shift
for sg in "$@"; do
  STS_SEG=$sg python - <<PY
import os, sys, json, torch
sys.path.insert(0, os.getcwd())
from paper_1802_04243_b200 import simplets as S, workloads as W
case = W.c3($H, "implicit_upwind", passes=10)
g = S.Solver(case, stream=torch.cuda.current_stream().cuda_stream)
g.advance(3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.advance(20); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"H": $H, "seg": "$sg", "ms_per_step": round(ms, 4), "GFVU_s": round(case["nx"] * case["ny"] * 10 / ms / 1e6, 2)}), flush=True)
PY
done
