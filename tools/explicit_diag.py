"""Why do explicit steps time differently with the event profile on?  (GPU box)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1802_04243_b200 import simplets as S, workloads as W
v = sys.argv[1] if len(sys.argv) > 1 else "explicit_upwind"
for mode in ("profile", "stream", "graph", "profile"):
    if mode == "stream": os.environ["STS_NO_GRAPH"] = "1"
    else: os.environ.pop("STS_NO_GRAPH", None)
    case = W.c3(200, v, passes=10)
    g = S.Solver(case, stream=torch.cuda.current_stream().cuda_stream)
    g.advance(3)
    g.profile(mode == "profile")
    g.profile_read(reset=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); st, stats = g.advance(10, check=False); e1.record(); torch.cuda.synchronize()
    pr = g.profile_read(reset=True)
    print(json.dumps({"mode": mode, "ms_per_step": round(e0.elapsed_time(e1) / 10, 4), "status": st, "prof": pr,
                      "res": stats["res"]}), flush=True)
    g.close()
