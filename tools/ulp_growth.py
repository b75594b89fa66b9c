#!/usr/bin/env python
"""Oracle-only conditioning of a run: two oracle runs from states that differ by
one ulp of T everywhere; max relative field difference (R31) after every time
step.  Shows whether GPU-vs-oracle drift is intrinsic to the discrete method
(test infrastructure: calls oracle/ only).

    python tools/ulp_growth.py --case c3h10 --variant implicit_tvd --steps 6
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402
from tests.parity_util import FIELDS, rel_errors  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="c3h10")
    ap.add_argument("--variant", default="implicit_tvd")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--passes", type=int, default=10)
    a = ap.parse_args()
    case = {"c1": lambda: W.c1(a.variant, a.passes), "c3h10": lambda: W.c3(10, a.variant, a.passes)}[a.case]()
    x, y = oracle.Case(case), oracle.Case(case)
    y.set("T", np.nextafter(y.get("T"), 2.0))
    fluid = x.get_map(0) == 0
    for s in range(1, a.steps + 1):
        x.advance(1)
        y.advance(1)
        err = rel_errors(y.fields(), x.fields(), fluid)
        print(json.dumps({"case": a.case, "variant": a.variant, "step": s, "passes": s * a.passes,
                          "max_rel_diff_1ulp": max(err.values())}), flush=True)


if __name__ == "__main__":
    main()
