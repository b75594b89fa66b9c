"""Dump 1-pass results of the default / STS_OLD_REGK / STS_NO_ALLREG runs (debug)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402

F = ("u", "v", "p", "T")
tag = sys.argv[1]
variant = "implicit_upwind"
case = W.channel(520, 96, spacing=0.25, variant=variant, passes=1, squares=[(200, 40, 10, 10)])
res = {}
for name, env in (("def", {"STS_SEG": "16"}), ("old", {"STS_SEG": "16", "STS_OLD_REGK": "1"}),
                  ("gen", {"STS_SEG": "16", "STS_NO_ALLREG": "1"}), ("def_auto", {})):
    for k in ("STS_SEG", "STS_OLD_REGK", "STS_NO_ALLREG"):
        os.environ.pop(k, None)
    os.environ.update(env)
    os.environ["STS_VERBOSE"] = "1"
    g = S.Solver(case)
    st = W.perturbed_state({f: g.get_field(f) for f in F}, W.perturbation(case, seed=9), vscale=0.05)
    for f in ("p", "T", "u", "v"):
        g.set_field(f, st[f])
    g.advance(1)
    for f in F:
        res[name + "_" + f] = g.get_field(f)
    res["init_" + "T"] = st["T"]
np.savez(f"gpurun_out/dump_{tag}.npz", **res)
