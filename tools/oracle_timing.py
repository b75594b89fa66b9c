"""Oracle timing coverage of SURVEY 8(d).4 / BASELINE.md 3 on the GPU box's host
(one core, pinned): the full C1 run of every variant (200 steps x 10 passes),
C2 (4096 x 256) for 20 steps x 10 passes, the paper's four C3 meshes for 3
passes each, and C4 (100.8 M FVs) for 1 pass.  FVU/s = FVs x passes / wall
time.  usage (GPU box or any host): python tools/oracle_timing.py > profiles/..."""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402


def cpu():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def timed(case, steps, label):
    o = oracle.Case(case)
    t0 = time.perf_counter()
    st = o.advance(steps)[0]
    dt = time.perf_counter() - t0
    fvu = case["nx"] * case["ny"] * case["max_passes"] * steps
    print(json.dumps({"run": label, "nx": case["nx"], "ny": case["ny"], "steps": steps, "passes": case["max_passes"],
                      "seconds": round(dt, 2), "FVU_s": round(fvu / dt), "status": st, "cores": 1,
                      "cpu": cpu(), "nproc": os.cpu_count()}), flush=True)


def main():
    try:
        os.sched_setaffinity(0, {min(os.sched_getaffinity(0))})
    except (AttributeError, OSError):
        pass
    oracle.build()
    for v in W.VARIANTS:
        timed(W.c1(v, passes=10), 200, f"C1 {v} full run")
    timed(W.c2(small=False, variant="implicit_upwind", passes=10), 20, "C2 20 x 10")
    for H in (10, 20, 100, 200):
        for v in W.VARIANTS:
            timed(W.c3(H, v, passes=3), 1, f"C3 H{H} {v} 3 passes")
    if "--c4" in sys.argv:
        timed(W.c4("implicit_upwind", passes=1), 1, "C4 implicit_upwind 1 pass")


if __name__ == "__main__":
    main()
