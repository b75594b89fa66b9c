"""Old vs new all-regular kernel after 1 pass: which fields / cells differ (debug)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402

F = ("u", "v", "p", "T")
for variant in sys.argv[1:] or ["implicit_upwind", "explicit_upwind"]:
    for passes in (1, 2):
        case = W.channel(520, 96, spacing=0.25, variant=variant, passes=passes, squares=[(200, 40, 10, 10)])
        out = []
        for env in ({"STS_SEG": "16"}, {"STS_SEG": "16", "STS_OLD_REGK": "1"}, {"STS_SEG": "16", "STS_NO_ALLREG": "1"}):
            for k in ("STS_SEG", "STS_OLD_REGK", "STS_NO_ALLREG", "STS_NO_FUSE"):
                os.environ.pop(k, None)
            os.environ.update(env)
            os.environ["STS_NO_FUSE"] = "1"
            g = S.Solver(case)
            st = W.perturbed_state({f: g.get_field(f) for f in F}, W.perturbation(case, seed=9), vscale=0.05)
            for f in ("p", "T", "u", "v"):
                g.set_field(f, st[f])
            g.advance(1)
            out.append({f: g.get_field(f) for f in F})
        for name, o in (("old", out[1]), ("gen", out[2])):
            for f in F:
                d = out[0][f] != o[f]
                if d.any():
                    jj, ii = np.nonzero(d)
                    rel = np.abs(out[0][f] - o[f]).max() / np.abs(o[f]).max()
                    print(variant, passes, "new vs", name, f, "ndiff", d.sum(), "rows", sorted(set(jj.tolist()))[:12],
                          "cols", sorted(set(ii.tolist()))[:8], "rel", rel)
                else:
                    print(variant, passes, "new vs", name, f, "same")
