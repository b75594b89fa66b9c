"""Diagnostic: periodic x with k in-process slabs vs one context vs the oracle."""
import sys

import numpy as np

sys.path.insert(0, ".")
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import oracle  # noqa: E402
from paper_1802_04243_b200 import simplets as S  # noqa: E402
from paper_1802_04243_b200 import workloads as W  # noqa: E402

F = ("u", "v", "p", "T")
for passes, steps in ((1, 1), (2, 1), (3, 3)):
    case = W.c2(small=True, variant="implicit_tvd", passes=passes)
    ref = S.Solver(case)
    o = oracle.Case(case)
    st = W.perturbed_state({f: o.get(f) for f in F}, W.perturbation(case, 3), vscale=0.05)
    k = 4
    grp = [S.Solver(case, rank=r, world=k) for r in range(k)]
    for f in ("p", "T", "u", "v"):
        ref.set_field(f, st[f])
        o.set(f, st[f])
        for g in grp:
            g.set_field(f, st[f])
    ref.advance(steps)
    S.advance_group(grp, steps)
    o.advance(steps)
    for f in F:
        a = ref.get_field(f)
        b = np.concatenate([g.get_field(f) for g in grp], axis=1)
        c = o.get(f)
        d1 = np.abs(a - c)
        d2 = np.abs(b - c)
        j1, i1 = np.unravel_index(d1.argmax(), d1.shape)
        j2, i2 = np.unravel_index(d2.argmax(), d2.shape)
        print(f"passes={passes} steps={steps} {f}: ref-vs-oracle {d1.max():.2e} at (j={j1}, i={i1}); "
              f"group-vs-oracle {d2.max():.2e} at (j={j2}, i={i2})")
