"""The paper's grid sweep (4032 x {200, 400, 2000, 4000}, flow past
{1, 2, 10, 20} squares) on one B200: FVU/s of each variant, fixed 10 passes per
step, CUDA-event timing of sts_advance (the pass-kernel average from the
library's event profile as well).  usage (GPU box): python tools/sweep.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402

variants = sys.argv[1].split(",") if len(sys.argv) > 1 else list(W.VARIANTS)
for H in (10, 20, 100, 200):
    for v in variants:
        case = W.c3(H, v, passes=10)
        g = S.Solver(case, stream=torch.cuda.current_stream().cuda_stream)
        g.advance(2)
        steps = 10
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st, _ = g.advance(steps, check=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        fv = case["nx"] * case["ny"]
        print(json.dumps({"H": H, "nx": case["nx"], "ny": case["ny"], "variant": v, "ms_per_step": round(ms, 4),
                          "GFVU_s": round(fv * 10 / ms / 1e6, 3), "status": st}), flush=True)
        del g
