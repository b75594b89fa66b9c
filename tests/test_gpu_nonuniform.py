"""Non-uniform meshes on the GPU: the NU kernel instances
(sts_set_mesh) against the CPU oracle, element by element, and their
decomposition invariance.

The oracle's general-mesh forms are pinned in tests/test_oracle_nonuniform.py.
Inputs: the paper's geometry on rough (seeded random steps, +-20 %) and smoothly
stretched (+-30 %) meshes with seeded +-1 % perturbations."""
import os

import numpy as np
import pytest

from paper_1802_04243_b200 import workloads as W
from tests.parity_util import FIELDS, TOL, rel_errors, seeded_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch
    assert torch.cuda.is_available()
    import __graft_entry__
    __graft_entry__.build()
    from paper_1802_04243_b200 import simplets
    return simplets


def _rough(case, seed):
    return W.with_mesh(case, W.random_steps(case["nx"], case["spacing"], seed),
                       W.random_steps(case["ny"], case["spacing"], seed + 1))


def _compare(S, oracle_mod, case, steps, seed=0, vscale=0.05, extra=()):
    g, o = seeded_pair(S, oracle_mod, case, seed=seed, vscale=vscale)
    g.advance(steps)
    assert o.advance(steps)[0] == 0
    fg = {k: g.get_field(k) for k in FIELDS + tuple(extra)}
    fo = {k: o.get(k) for k in FIELDS + tuple(extra)}
    err = rel_errors(fg, fo, o.get_map(0) == 0)
    assert max(err.values()) <= TOL, err
    return err


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_nonuniform_small_square(S, oracle_mod, variant):
    """48 x 16 channel with a square on a rough mesh, 3 steps x 3 passes, every
    variant; the explicit planes too."""
    case = _rough(W.c1_small(variant, passes=3), seed=20)
    extra = ("uexp", "vexp", "Texp") if variant.startswith("explicit") else ()
    _compare(S, oracle_mod, case, 3, seed=1, extra=extra)


@pytest.mark.parametrize("variant", ["implicit_tvd", "explicit_upwind"])
def test_nonuniform_ragged_squares(S, oracle_mod, variant):
    """Squares touching each other and the walls, ragged strip / segment edges,
    rough mesh in both directions."""
    case = W.channel(75, 37, spacing=0.25, variant=variant, passes=4,
                     squares=[(30, 14, 5, 4), (35, 18, 3, 3), (60, 0, 4, 6), (10, 31, 6, 6)])
    _compare(S, oracle_mod, _rough(case, seed=22), 3, seed=2)


@pytest.mark.parametrize("variant", ["implicit_upwind", "explicit_tvd"])
def test_nonuniform_periodic(S, oracle_mod, variant):
    """Periodic x (wrapped ghost widths) with a body force on a rough mesh."""
    case = _rough(W.c2(small=True, variant=variant, passes=5), seed=24)
    _compare(S, oracle_mod, case, 4, seed=3, vscale=0.001)


@pytest.mark.parametrize("variant", ["implicit_upwind", "implicit_tvd", "explicit_tvd"])
def test_nonuniform_paper_mesh(S, oracle_mod, variant):
    """The paper's 4032 x 200 channel (C3, H = 10) on a smoothly stretched mesh
    (steps +-30 % in y, mirror symmetric; +-20 % rough in x), 1 step x 3 passes in
    the NU launch configuration."""
    case = W.c3(10, variant, passes=3)
    case = W.with_mesh(case, W.random_steps(case["nx"], case["spacing"], seed=26),
                       W.smooth_steps(case["ny"], case["spacing"], 0.3))
    _compare(S, oracle_mod, case, 1, seed=5)


def test_nonuniform_c1_length(S, oracle_mod):
    """C1 at BASELINE configs[0]'s run length on a stretched mesh: 200 steps x 10
    passes of explicit upwind from the free stream."""
    case = W.c1("explicit_upwind", passes=10)
    case = W.with_mesh(case, W.random_steps(case["nx"], case["spacing"], seed=28),
                       W.smooth_steps(case["ny"], case["spacing"], 0.3))
    g = S.Solver(case)
    o = oracle_mod.Case(case)
    g.advance(200)
    assert o.advance(200)[0] == 0
    err = rel_errors({k: g.get_field(k) for k in FIELDS}, o.fields(), o.get_map(0) == 0)
    assert max(err.values()) <= TOL, err


@pytest.mark.parametrize("variant", ["implicit_tvd", "explicit_tvd"])
def test_nonuniform_slabs_bitwise(S, variant):
    """3 in-process x-slabs on a rough mesh reproduce one slab bit for bit (each
    slab builds its column widths, ghost columns included, from the global steps)."""
    case = _rough(W.c1(variant, passes=4), seed=30)
    ref = S.Solver(case)
    st = W.perturbed_state({f: ref.get_field(f) for f in ("u", "v", "p", "T")},
                           W.perturbation(case, 3), vscale=0.05)
    group = [S.Solver(case, rank=r, world=3) for r in range(3)]
    for g in [ref] + group:
        for f in ("p", "T", "u", "v"):
            g.set_field(f, st[f])
    ref.advance(3)
    S.advance_group(group, 3)
    for f in ("u", "v", "p", "T"):
        got = np.concatenate([g.get_field(f) for g in group], axis=1)
        assert np.array_equal(ref.get_field(f), got), f


def test_nonuniform_segments_bitwise(S):
    """1-row y segments of the NU march kernel give the same bits as the scheduled ones."""
    case = _rough(W.c1("implicit_tvd", passes=3), seed=32)
    out = []
    for seg in (None, "1"):
        old = os.environ.pop("STS_SEG", None)
        if seg:
            os.environ["STS_SEG"] = seg
        try:
            g = S.Solver(case)
            st = W.perturbed_state({f: g.get_field(f) for f in ("u", "v", "p", "T")},
                                   W.perturbation(case, 4), vscale=0.05)
            for f in ("p", "T", "u", "v"):
                g.set_field(f, st[f])
            g.advance(2)
            out.append({f: g.get_field(f) for f in ("u", "v", "p", "T")})
        finally:
            os.environ.pop("STS_SEG", None)
            if old is not None:
                os.environ["STS_SEG"] = old
    for f in out[0]:
        assert np.array_equal(out[0][f], out[1][f]), f


def test_nonuniform_tolerance_mode(S, oracle_mod):
    """Tolerance mode (graph-driven loop 2) with the NU kernels: the oracle's pass
    count and fields."""
    case = _rough(W.c1_small("implicit_upwind", passes=200), seed=34)
    case["tol"] = 1e-9
    g, o = seeded_pair(S, oracle_mod, case, seed=6)
    st, stats = g.advance(2, check=False)
    ost, ores, opasses = o.advance(2)
    assert st == 0 and ost == 0 and stats["converged"] == 1
    err = rel_errors({k: g.get_field(k) for k in FIELDS}, o.fields(), o.get_map(0) == 0)
    assert max(err.values()) <= TOL, err


def test_set_mesh_rejects_bad_steps(S):
    case = W.c1_small("implicit_upwind", passes=2)
    g = S.Solver(case)
    bad = np.full(case["nx"], 0.25)
    bad[3] = 0.0
    with pytest.raises(S.StsError):
        g.set_mesh(bad, None)
    with pytest.raises(S.StsError):
        g.set_mesh(np.full(case["nx"] + 1, 0.25), None)
