"""Loop 3 on the GPU (reading R41): passes of k energy /
pressure sweeps (the L3 instances of the march kernel for sweeps 2..k) against
the CPU oracle, element by element, at 1e-9."""
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


def _compare(S, oracle_mod, case, steps, seed=0, vscale=0.05):
    g, o = seeded_pair(S, oracle_mod, case, seed=seed, vscale=vscale)
    _, stats = g.advance(steps)
    ost, ores, _ = o.advance(steps)
    assert ost == 0
    err = rel_errors({k: g.get_field(k) for k in FIELDS}, o.fields(), o.get_map(0) == 0)
    assert max(err.values()) <= TOL, err
    assert np.allclose(stats["res"], ores, rtol=1e-6, atol=1e-14), (stats["res"], ores)


@pytest.mark.parametrize("variant", list(W.VARIANTS))
@pytest.mark.parametrize("l3", [2, 3])
def test_loop3_small_square(S, oracle_mod, variant, l3):
    """48 x 16 channel with a square, 3 steps x 3 passes of l3 sweeps each."""
    case = W.c1_small(variant, passes=3)
    case["loop3"] = l3
    _compare(S, oracle_mod, case, 3, seed=1)


def test_loop3_ragged_and_periodic(S, oracle_mod):
    """Squares touching each other and the walls (general points, outlet ghosts),
    and a periodic channel (wrapped ghost columns of the sweep iterates)."""
    case = W.channel(75, 37, spacing=0.25, variant="implicit_tvd", passes=3,
                     squares=[(30, 14, 5, 4), (35, 18, 3, 3), (60, 0, 4, 6), (10, 31, 6, 6)])
    case["loop3"] = 2
    _compare(S, oracle_mod, case, 2, seed=2)
    case = W.c2(small=True, variant="implicit_upwind", passes=4)
    case["loop3"] = 2
    _compare(S, oracle_mod, case, 3, seed=3, vscale=0.001)


def test_loop3_paper_mesh(S, oracle_mod):
    """The paper's 4032 x 200 mesh, implicit upwind, 2 steps x 4 passes x 2 sweeps,
    in the bench's launch configuration (all-regular + general kernels)."""
    case = W.c3(10, "implicit_upwind", passes=4)
    case["loop3"] = 2
    _compare(S, oracle_mod, case, 2, seed=5)


def test_loop3_tolerance_mode(S, oracle_mod):
    """Tolerance mode (host-driven loop 2) with 2 sweeps: the oracle's pass count."""
    case = W.c1_small("implicit_upwind", passes=200)
    case["tol"], case["loop3"] = 1e-9, 2
    g, o = seeded_pair(S, oracle_mod, case, seed=6)
    st, stats = g.advance(1, check=False)
    ost, ores, opasses = o.advance(1)
    assert st == 0 and ost == 0 and stats["converged"] == 1
    assert stats["passes_done"] == opasses
    err = rel_errors({k: g.get_field(k) for k in FIELDS}, o.fields(), o.get_map(0) == 0)
    assert max(err.values()) <= TOL, err


def test_loop3_rejected_where_unsupported(S):
    """loop3 > 1 runs on single-rank uniform meshes; elsewhere STS_E_CONFIG."""
    case = W.c1_small("implicit_upwind", passes=2)
    case["loop3"] = 2
    g = S.Solver(case)
    with pytest.raises(S.StsError):
        g.set_mesh(np.full(case["nx"], 0.25), None)
    with pytest.raises(S.StsError):
        S.Solver(case, rank=0, world=2)
