"""4032 x 200 (the paper's smallest mesh): ms per step of a fixed-pass step
(10 passes) through the graph path, for the env settings given on the command line
as NAME=ENV1:VAL1;ENV2:VAL2 ... (each in a fresh Solver)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402

H = int(os.environ.get("H", "10"))
variant = os.environ.get("V", "implicit_upwind")
for spec in sys.argv[1:] or ["auto="]:
    name, _, envs = spec.partition("=")
    for k in ("STS_SEG", "STS_OLD_REGK", "STS_CTA_OVH", "STS_COST", "STS_NO_PDL", "STS_ITVD_FUSED"):
        os.environ.pop(k, None)
    for kv in filter(None, envs.split(";")):
        k, v = kv.split(":")
        os.environ[k] = v
    case = W.c3(H, variant, passes=10)
    g = S.Solver(case, stream=torch.cuda.current_stream().cuda_stream)
    g.advance(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.advance(20, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(json.dumps({"name": name, "H": H, "variant": variant, "ms_per_step": round(ms, 4),
                      "GFVU_s": round(case["nx"] * case["ny"] * 10 / ms / 1e6, 2)}))
