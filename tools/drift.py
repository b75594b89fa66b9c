#!/usr/bin/env python
"""GPU-vs-oracle drift over a run: after every time step, the max relative field
error (reading R31) between the CUDA path and the CPU oracle on the same seeded
input.  One JSON line per step (test infrastructure: calls oracle/).

    python tools/drift.py --case c1|c3h10|c2 --variant V --steps S --passes P [--seed N]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402
from tests.parity_util import FIELDS, rel_errors, seeded_pair  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="c1")
    ap.add_argument("--variant", default="implicit_tvd")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--passes", type=int, default=10)
    ap.add_argument("--seed", type=int, default=-1, help="-1: free-stream start")
    a = ap.parse_args()
    case = {"c1": lambda: W.c1(a.variant, a.passes), "c3h10": lambda: W.c3(10, a.variant, a.passes),
            "c2": lambda: W.c2(False, a.variant, a.passes)}[a.case]()
    if a.seed >= 0:
        g, o = seeded_pair(S, oracle, case, seed=a.seed)
    else:
        g, o = S.Solver(case), oracle.Case(case)
    fluid = o.get_map(0) == 0
    for s in range(1, a.steps + 1):
        t0 = time.time()
        g.advance(1, check=False)
        st = o.advance(1)[0]
        err = rel_errors({k: g.get_field(k) for k in FIELDS}, o.fields(), fluid)
        print(json.dumps({"case": a.case, "variant": a.variant, "step": s, "passes": s * a.passes,
                          "oracle_status": st, "max_rel_err": max(err.values()), "err": err,
                          "oracle_s": round(time.time() - t0, 2)}), flush=True)


if __name__ == "__main__":
    main()
