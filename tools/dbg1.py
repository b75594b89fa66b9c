import sys, os
sys.path.insert(0, os.getcwd())
from paper_1802_04243_b200 import simplets as S, workloads as W
case = W.periodic_box(377, 20, 0.1, variant="explicit_upwind", passes=4, dt=0.02, Kn=0.02, squares=[(3, 6, 4, 4), (371, 9, 4, 5)])
for tol in (0.0, 1e-3):
    c = dict(case, tol=tol, min_passes=2)
    a = S.Solver(c)
    print("created", tol, flush=True)
    print(a.advance(3, check=False)[0], flush=True)
