"""ms per step of the fixed-pass graph path vs the stream path (STS_NO_GRAPH),
C3 H = 200 and H = 10, every variant.  usage (GPU box): python tools/graph_ab.py [lib]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1802_04243_b200 import simplets as S, workloads as W
for H in (200, 10):
    for v in W.VARIANTS:
        out = {"H": H, "variant": v, "lib": os.path.basename(S.LIB_PATH)}
        for mode in ("graph", "stream"):
            if mode == "stream":
                os.environ["STS_NO_GRAPH"] = "1"
            else:
                os.environ.pop("STS_NO_GRAPH", None)
            case = W.c3(H, v, passes=10)
            g = S.Solver(case, stream=torch.cuda.current_stream().cuda_stream)
            g.advance(3)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            steps = 10
            e0.record(); g.advance(steps); e1.record(); torch.cuda.synchronize()
            out[mode + "_ms"] = round(e0.elapsed_time(e1) / steps, 4)
            g.close()
        print(json.dumps(out), flush=True)
os.environ.pop("STS_NO_GRAPH", None)
