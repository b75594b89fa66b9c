"""Loop 3 (N3) vs passes to tolerance: loop-2 passes per step and wall time per step
for loop3 = 1, 2, 3 on the paper's 4032 x 400 mesh (implicit upwind, explicit upwind),
tol = 1e-8, from the free-stream start (host-driven loop 2: loop3 > 1 has no graph).
usage (GPU box): python tools/passes_loop3.py [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
os.environ["STS_NO_GRAPH"] = "1"          # the same (host) driver for every loop3
for v in ("implicit_upwind", "explicit_upwind"):
    for l3 in (1, 2, 3):
        case = W.c3(20, v, passes=500)
        case["tol"], case["loop3"] = 1e-8, l3
        g = S.Solver(case)
        per = []
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(steps):
            p0 = g.advance(0)[1]["passes_done"]
            st, stats = g.advance(1, check=False)
            per.append(stats["passes_done"] - p0)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(json.dumps({"variant": v, "loop3": l3, "mean_passes": sum(per) / len(per), "passes": per,
                          "ms_per_step": 1e3 * dt / steps, "status": st}), flush=True)
        g.close()
