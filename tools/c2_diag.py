"""Diagnose GPU-vs-oracle differences on periodic C2-like channels (GPU box)."""
import math, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_1802_04243_b200 import simplets as S, workloads as W
from tests.parity_util import rel_errors, FIELDS

def run(nx, ny, steps, passes=10):
    case = W.c2(small=False, variant="implicit_upwind", passes=passes)
    sp = 1.0 / ny
    case.update(nx=nx, ny=ny, spacing=sp)
    H, N, Kn, gx = 1.0, ny, case["Kn"], case["g_x"]
    B = 5.0 * math.sqrt(math.pi) / 16.0 * Kn
    y = (np.arange(N) + 0.5) * H / N
    x = (np.arange(nx) + 0.5) / nx
    prof = (gx / (2 * B)) * (y * (H - y) + 1.1466 * Kn * H)
    st = {"u": np.repeat(1.05 * prof[:, None], nx + 1, axis=1), "v": np.zeros((N + 1, nx)),
          "p": 1 + 1e-3 * np.sin(2 * np.pi * x)[None, :] * np.ones((N, 1)),
          "T": 1 + 5e-4 * np.outer(np.sin(np.pi * y), np.cos(2 * np.pi * x))}
    g = S.Solver(case); o = oracle.Case(case)
    for k in ("p", "T", "u", "v"):
        g.set_field(k, st[k]); o.set(k, st[k])
    for s in range(steps):
        g.advance(1); o.advance(1)
        fg = {k: g.get_field(k) for k in FIELDS}; fo = o.fields()
        e = rel_errors(fg, fo)
        d = np.abs(fg["u"] - fo["u"])
        cols = np.where(d.max(axis=0) > 1e-12)[0]
        rows = np.where(d.max(axis=1) > 1e-12)[0]
        print(nx, ny, "step", s, {k: float(f"{v:.2e}") for k, v in e.items()}, "cols", cols[:6], cols[-3:], len(cols), "rows", rows[:4], rows[-3:], flush=True)

for nx, ny, steps in ((256, 64, 3), (1024, 256, 2), (4096, 256, 2)):
    run(nx, ny, steps)
