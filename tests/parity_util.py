"""Shared helpers of the GPU parity tests (test infrastructure only)."""
import numpy as np

from paper_1802_04243_b200 import workloads as W

FIELDS = ("u", "v", "p", "T", "rho")
TOL = 1e-9     # north_star: max relative field error (reading R31)


def rel_errors(fg: dict, fo: dict, fluid=None):
    """Max relative error per field (R31): |gpu - oracle| / max|oracle| over the
    field; velocities are normalised by the max speed over u and v."""
    vel = max(np.abs(fo["u"]).max(), np.abs(fo["v"]).max(), 1e-300)
    out = {}
    for k in fg:
        a, b = fg[k], fo[k]
        if fluid is not None and k in ("p", "T", "rho"):
            a, b = a[fluid], b[fluid]
        den = vel if k in ("u", "v", "uexp", "vexp") else max(np.abs(b).max(), 1e-300)
        out[k] = float(np.abs(a - b).max() / den)
    return out


def seeded_pair(S, oracle, case, seed=0, amplitude=0.01, vscale=0.05, stream=None):
    """GPU solver and oracle case set to the same seeded perturbed free stream."""
    g = S.Solver(case, stream=stream)
    o = oracle.Case(case)
    base = {k: o.get(k) for k in ("u", "v", "p", "T")}
    st = W.perturbed_state(base, W.perturbation(case, seed, amplitude), vscale=vscale)
    for k in ("p", "T", "u", "v"):
        g.set_field(k, st[k])
        o.set(k, st[k])
    return g, o
