"""Raw step time of C3 (H env, default 200) for a build (STS_LIB), ignoring the results
(check=False everywhere): for timing experiments whose numerics are knowingly wrong."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402

H = int(os.environ.get("H", "200"))
v = os.environ.get("V", "implicit_upwind")
case = W.c3(H, v, passes=10)
g = S.Solver(case, stream=torch.cuda.current_stream().cuda_stream)
g.advance(3, check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.advance(20, check=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"lib": os.environ.get("STS_LIB", "in-tree"), "fused": not os.environ.get("STS_NO_FUSED"),
                  "ms_per_step": round(ms, 4), "GFVU_s": round(case["nx"] * case["ny"] * 10 / ms / 1e6, 2)}))
