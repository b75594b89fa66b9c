"""regk2 (STS_REGK2=1) vs the default path: bitwise after a few steps (debug / A-B)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402

F = ("u", "v", "p", "T")
for variant in sys.argv[1:] or list(W.VARIANTS):
    for seg in ("16", "17", "5"):
        case = W.channel(520, 96, spacing=0.25, variant=variant, passes=3, squares=[(200, 40, 10, 10)])
        out = []
        for env in ({"STS_SEG": seg}, {"STS_SEG": seg, "STS_REGK2": "1"}):
            for k in ("STS_SEG", "STS_REGK2"):
                os.environ.pop(k, None)
            os.environ.update(env)
            g = S.Solver(case)
            st = W.perturbed_state({f: g.get_field(f) for f in F}, W.perturbation(case, seed=9), vscale=0.05)
            for f in ("p", "T", "u", "v"):
                g.set_field(f, st[f])
            g.advance(3)
            out.append({f: g.get_field(f) for f in F})
        for f in F:
            d = out[0][f] != out[1][f]
            print(variant, "seg", seg, f, "same" if not d.any() else f"ndiff {d.sum()} rows {sorted(set(np.nonzero(d)[0].tolist()))[:10]} max {np.abs(out[0][f]-out[1][f]).max()}")
