"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds ONLY case descriptions (geometry in integer cell units, gas
and scheme parameters, as the paper states them) and seeded random
perturbation arrays.  It contains none of the method's arithmetic: both the
CUDA library and the oracle derive every method quantity (u_in, Eq. pl37
constants, fixed faces, ...) themselves from these parameters.

Paper workload: Kn = 0.001, M = 2.43 at the inlet,
gamma = 5/3, Pr = 2/3; channel L_ch = 201.6, square side a = 1 with its front
face at L_a = 5.5, uniform mesh Delta = 0.05, H_ch in {10, 20, 100, 200} with
{1, 2, 10, 20} squares (stacked in y, one per 10-unit band, reading R18).
"""
from __future__ import annotations

import numpy as np

# time / space schemes (same numbering in include/simplets.h and the oracle)
EXPLICIT, IMPLICIT = 0, 1
UPWIND, TVD = 0, 1
X_INOUT, X_PERIODIC = 0, 1
# pressure-work forms of S^T_c (reading R9): C^T3 Dp/Dt (default), +C^T3 p div u
# (as printed), -C^T3 p div u (round-1 reading), -gamma C^T3 p div u
PW_DPDT, PW_PRINTED, PW_NEG, PW_GAMMA = 0, 1, 2, 3

VARIANTS = {
    "explicit_upwind": (EXPLICIT, UPWIND),
    "explicit_tvd": (EXPLICIT, TVD),
    "implicit_upwind": (IMPLICIT, UPWIND),
    "implicit_tvd": (IMPLICIT, TVD),
}

PAPER_GAS = dict(Kn=0.001, mach=2.43, gamma=5.0 / 3.0, p_in=1.0, T_in=1.0,
                 T_wall=1.0, T_square=1.0, g_x=0.0, g_y=0.0, particle_frame=1,
                 pw_form=0)   # reading R9: 0 = C^T3 Dp/Dt of Eq. pl6


def _case(nx, ny, spacing, squares, variant, dt, passes, **kw):
    time, space = VARIANTS[variant]
    c = dict(PAPER_GAS)
    c.update(nx=int(nx), ny=int(ny), spacing=float(spacing), squares=[list(map(int, s)) for s in squares],
             xbc=X_INOUT, time=time, space=space, dt=float(dt), min_passes=1,
             max_passes=int(passes), tol=0.0, variant=variant)
    c.update(kw)
    return c


def supersonic_dt(spacing, variant):
    """Time step of the supersonic cases (reading R12): dt = 0.1 Delta (convective
    CFL (u_in + c) dt / Delta = 0.31); explicit TVD takes half of it (R39: forward
    Euler on the limited convective terms turns non-physical at CFL 0.31 within
    ~50 steps in the oracle and on the GPU alike, stable at 0.16)."""
    return (0.05 if variant == "explicit_tvd" else 0.1) * spacing


def c1(variant="explicit_upwind", passes=10):
    """C1: L = 30, H = 10, Delta = 0.25 -> 120 x 40; one square [5.5,6.5]x[4.5,5.5]
    = cells i 22..25, j 18..21 (centred in y -> mirror symmetric); dt = 0.1 Delta."""
    return _case(120, 40, 0.25, [(22, 18, 4, 4)], variant, supersonic_dt(0.25, variant), passes, name="C1")


def c1_small(variant="implicit_upwind", passes=4):
    """A 48 x 16 cut of C1 (Delta = 0.25, one 4x4 square centred in y) for fast parity."""
    return _case(48, 16, 0.25, [(10, 6, 4, 4)], variant, supersonic_dt(0.25, variant), passes, name="C1s")


def c3(H=200, variant="implicit_upwind", passes=10):
    """C3: the paper's meshes 4032 x {200,400,2000,4000}, Delta = 0.05,
    squares of 20x20 cells at i0 = 110 (L_a/Delta), centred at y = 5 + 10k."""
    ny = int(round(H / 0.05))
    nsq = int(round(H / 10))
    squares = [(110, 90 + 200 * k, 20, 20) for k in range(nsq)]
    return _case(4032, ny, 0.05, squares, variant, supersonic_dt(0.05, variant), passes, name=f"C3_H{H}")


def c3_long(G, variant="implicit_upwind", passes=10):
    """Weak-scaling channel for G GPUs: G copies of the C3 H = 200 mesh laid end to
    end (4032 G x 4000, a column of 20 squares every 201.6 units), one slab per GPU."""
    squares = [(110 + 4032 * m, 90 + 200 * k, 20, 20) for m in range(G) for k in range(20)]
    return _case(4032 * G, 4000, 0.05, squares, variant, supersonic_dt(0.05, variant), passes, name=f"C3L_G{G}")


def c4(variant="implicit_upwind", passes=10):
    """C4: H = 200, L = 201.6, Delta = 0.02 -> 10080 x 10000 (100.8 M FVs);
    20 squares of 50x50 cells at i0 = 275, j0 = 225 + 500k."""
    squares = [(275, 225 + 500 * k, 50, 50) for k in range(20)]
    return _case(10080, 10000, 0.02, squares, variant, supersonic_dt(0.02, variant), passes, name="C4")


def c5(G=1, variant="implicit_upwind", passes=10):
    """C5 weak scaling: H = 200, Delta = 0.05, L = 1875 G -> (37500 G) x 4000;
    a column of 20 squares every 25 units in x so every slab is identical."""
    nx = 37500 * G
    squares = [(110 + 500 * m, 90 + 200 * k, 20, 20) for m in range(nx // 500) for k in range(20)
               if 110 + 500 * m + 20 <= nx - 1]
    return _case(nx, 4000, 0.05, squares, variant, supersonic_dt(0.05, variant), passes, name=f"C5_G{G}")


def channel(nx, ny, spacing=0.25, variant="implicit_upwind", passes=4, squares=(), **kw):
    """Generic inflow/outflow channel of the paper's gas (free-stream checks)."""
    return _case(nx, ny, spacing, list(squares), variant, 0.1 * spacing, passes, name="channel", **kw)


def periodic_box(nx, ny, spacing, variant="implicit_upwind", passes=10, dt=0.01, squares=(), **kw):
    """Periodic-x channel with stationary walls (Couette / Poiseuille / quiescent)."""
    kw.setdefault("mach", 0.0)          # no inflow: the free-stream state is at rest
    c = _case(nx, ny, spacing, list(squares), variant, dt, passes, name="periodic", **kw)
    c.update(xbc=X_PERIODIC, particle_frame=0)
    c.setdefault("u_wall_bottom", 0.0)
    c.setdefault("u_wall_top", 0.0)
    return c


def c2(small=False, variant="implicit_upwind", passes=10):
    """C2: obstacle-free periodic channel, H = 1, L = 16, Delta = 1/256 (4096 x 256),
    stationary slip walls, Kn = 0.05, body force g_x = 9.0114e-3, dt = 0.002.
    small=True: the 64 x 32 oracle-only variant (Delta = 1/32)."""
    if small:
        nx, ny, sp = 64, 32, 1.0 / 32
    else:
        nx, ny, sp = 4096, 256, 1.0 / 256
    c = periodic_box(nx, ny, sp, variant=variant, passes=passes, dt=0.002, g_x=9.0114e-3, Kn=0.05)
    c["name"] = "C2s" if small else "C2"
    return c


# ------------------------------------------------------------ non-uniform meshes (N4)
def smooth_steps(n: int, spacing: float, amplitude: float = 0.3):
    """Steps Delta_k = spacing (1 + amplitude cos(2 pi (k + 1/2) / n)), k < n: a
    smooth stretching, mirror symmetric (Delta_k = Delta_{n-1-k}), mean spacing."""
    k = np.arange(n)
    return spacing * (1.0 + amplitude * np.cos(2 * np.pi * (k + 0.5) / n))


def random_steps(n: int, spacing: float, seed: int, spread: float = 0.4):
    """Seeded rough steps spacing (1 + spread U(-1/2, 1/2)) (every stencil weight differs)."""
    rng = np.random.default_rng(seed)
    return spacing * (1.0 + spread * rng.uniform(-0.5, 0.5, size=n))


def with_mesh(case: dict, dxs=None, dys=None):
    """The case on a non-uniform mesh: per-column steps dxs (nx) and per-row steps
    dys (ny); None keeps that direction at the uniform `spacing`."""
    c = dict(case)
    if dxs is not None:
        c["dxs"] = np.asarray(dxs, dtype=np.float64)
        assert c["dxs"].shape == (c["nx"],)
    if dys is not None:
        c["dys"] = np.asarray(dys, dtype=np.float64)
        assert c["dys"].shape == (c["ny"],)
    c["name"] = c["name"] + "_nu"
    return c


# ------------------------------------------------------------ perturbations
def perturbation(case: dict, seed: int, amplitude: float = 0.01):
    """Seeded multiplicative noise factors (1 + amplitude * U(-1,1)) for u, v
    (additive scale amplitude), p, T in the solver's global field shapes.
    Returned arrays are applied by the caller to a state read back from the
    solver, so no method arithmetic lives here."""
    rng = np.random.default_rng(seed)
    nx, ny = case["nx"], case["ny"]
    return {
        "u": 1.0 + amplitude * rng.uniform(-1, 1, size=(ny, nx + 1)),
        "v": amplitude * rng.uniform(-1, 1, size=(ny + 1, nx)),
        "p": 1.0 + amplitude * rng.uniform(-1, 1, size=(ny, nx)),
        "T": 1.0 + amplitude * rng.uniform(-1, 1, size=(ny, nx)),
    }


def perturbed_state(base: dict, noise: dict, vscale: float):
    """Apply ``perturbation`` factors to a base state {u, v, p, T}: u, p, T are
    scaled, v gets additive noise of size vscale * noise.  Pure data plumbing."""
    return {
        "u": base["u"] * noise["u"],
        "v": base["v"] + vscale * noise["v"],
        "p": base["p"] * noise["p"],
        "T": base["T"] * noise["T"],
    }


def n_fv(case: dict) -> int:
    """Finite volumes of a case (owned fluid + solid cells)."""
    return int(case["nx"]) * int(case["ny"])
