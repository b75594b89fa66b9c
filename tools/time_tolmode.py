"""Tolerance-mode loop 2: time steps per second with the graph-driven loop
(device convergence test, conditional WHILE node) and with the host-driven loop
(STS_NO_GRAPH=1: residual read-back + host test after every pass, as P:707).
usage (GPU box): python tools/time_tolmode.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402


def run(case, graph, steps):
    os.environ.pop("STS_NO_GRAPH", None)
    if not graph:
        os.environ["STS_NO_GRAPH"] = "1"
    g = S.Solver(case)
    g.advance(3, check=False)                       # warm-up: builds the graphs of all 3 snapshot rotations
    torch.cuda.synchronize()
    p0 = g.advance(0)[1]["passes_done"]
    t = time.perf_counter()
    st, stats = g.advance(steps, check=False)
    dt = time.perf_counter() - t
    return {"graph": graph, "steps_per_s": steps / dt, "passes_per_step": (stats["passes_done"] - p0) / steps,
            "ms_per_pass": 1e3 * dt / max(1, stats["passes_done"] - p0), "status": st}


out = []
for name, case, steps in [("C1_implicit_upwind", W.c1("implicit_upwind", passes=100), 200),
                          ("C3_H10_implicit_upwind", W.c3(10, "implicit_upwind", passes=100), 50),
                          ("C3_H200_implicit_upwind", W.c3(200, "implicit_upwind", passes=100), 5)]:
    case["tol"] = 1e-6
    for graph in (True, False):
        r = run(case, graph, steps)
        r["case"] = name
        print(json.dumps(r), flush=True)
        out.append(r)
