"""Passes per time step that loop 2 needs to reach a tolerance on C3 (SURVEY
8(d).1: "report ... the number of passes per step that tol = 1e-8 needs"),
graph-driven loop 2, from the free-stream start.  usage (GPU box):
python tools/passes_to_tol.py [tol] [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402

tol = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for v in W.VARIANTS:
    case = W.c3(200, v, passes=500)
    case["tol"] = tol
    g = S.Solver(case)
    per = []
    t = time.perf_counter()
    for _ in range(steps):
        p0 = g.advance(0)[1]["passes_done"]
        st, stats = g.advance(1, check=False)
        per.append(stats["passes_done"] - p0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(json.dumps({"variant": v, "tol": tol, "steps": steps, "passes_per_step": per,
                      "mean_passes": sum(per) / len(per), "steps_per_s": steps / dt, "status": st}), flush=True)
