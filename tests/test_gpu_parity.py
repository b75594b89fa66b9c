"""GPU (CUDA, sm_100a, through the C ABI) vs CPU oracle, element by element.

Bar (north_star): max relative field error <= 1e-9 on u, v, p, T, rho after a
fixed step/pass count; integer kind maps bit-exact.  Inputs: the paper's
geometry with seeded +-1 % perturbations."""
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


def _run_compare(S, oracle_mod, case, steps, seed=0, vscale=0.05, tol=TOL, extra=()):
    g, o = seeded_pair(S, oracle_mod, case, seed=seed, vscale=vscale)
    st, stats = g.advance(steps)
    ost, ores, _ = o.advance(steps)
    assert ost == 0
    fg = {k: g.get_field(k) for k in FIELDS + tuple(extra)}
    fo = {k: o.get(k) for k in FIELDS + tuple(extra)}
    fluid = o.get_map(0) == 0
    err = rel_errors(fg, fo, fluid)
    assert max(err.values()) <= tol, err
    # residuals of the last pass agree as well (R35)
    assert np.allclose(stats["res"], ores, rtol=1e-6, atol=1e-14), (stats["res"], ores)
    return err


@pytest.mark.parametrize("variant", list(W.VARIANTS))
@pytest.mark.parametrize("pw", [-1.0, 1.0])
def test_parity_small_square(S, oracle_mod, variant, pw):
    """48x16 channel, one square, 3 steps x 3 passes, both pressure-work signs (R9)."""
    case = W.c1_small(variant, passes=3)
    case["pw_sign"] = pw
    extra = ("uexp", "vexp", "Texp") if variant.startswith("explicit") else ()
    _run_compare(S, oracle_mod, case, 3, seed=1, extra=extra)


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_parity_ragged_tiles(S, oracle_mod, variant):
    """nx, ny not multiples of the 32 x 16 tile; squares straddling tile edges and
    touching each other (corner links, fixed faces, TVD stencils cut by solids)."""
    case = W.channel(75, 37, spacing=0.25, variant=variant, passes=4,
                     squares=[(30, 14, 5, 4), (35, 18, 3, 3), (60, 0, 4, 6), (10, 31, 6, 6)])
    _run_compare(S, oracle_mod, case, 3, seed=2)


@pytest.mark.parametrize("variant", ["implicit_upwind", "explicit_tvd"])
def test_parity_periodic_poiseuille(S, oracle_mod, variant):
    """Periodic-x channel with body force (C2 small) -- wrapped ghost columns."""
    case = W.c2(small=True, variant=variant, passes=5)
    _run_compare(S, oracle_mod, case, 4, seed=3, vscale=0.001)


def test_parity_transposition_box(S, oracle_mod):
    """Closed box: a solid column with periodic x (squares touching the walls)."""
    case = W.periodic_box(11, 10, 0.1, variant="implicit_tvd", dt=0.02, passes=3, Kn=0.02, squares=[(0, 0, 1, 10)])
    _run_compare(S, oracle_mod, case, 2, seed=4, vscale=0.3)


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_parity_c1(S, oracle_mod, variant):
    """C1 (120 x 40, Delta = 0.25, supersonic past one square), 20 steps x 10 passes
    from the free stream (explicit TVD: 10 steps, it oscillates later)."""
    case = W.c1(variant, passes=10)
    steps = 10 if variant == "explicit_tvd" else 20
    g = S.Solver(case)
    o = oracle_mod.Case(case)
    g.advance(steps)
    assert o.advance(steps)[0] == 0
    fluid = o.get_map(0) == 0
    err = rel_errors({k: g.get_field(k) for k in FIELDS}, o.fields(), fluid)
    assert max(err.values()) <= TOL, err


def test_maps_bit_exact(S, oracle_mod):
    """Cell / u-face / v-face kind maps equal the oracle's bit for bit."""
    for case in (W.c1("implicit_upwind"), W.channel(75, 37, squares=[(30, 14, 5, 4), (60, 0, 4, 6)]),
                 W.c2(small=True), W.periodic_box(11, 10, 0.1, squares=[(0, 0, 1, 10)])):
        g = S.Solver(case)
        o = oracle_mod.Case(case)
        for which in (0, 1, 2):
            a, b = g.get_map(which), o.get_map(which)
            assert a.shape == b.shape and np.array_equal(a, b), (case["name"], which)


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_free_stream_gpu(S, variant):
    """The obstacle-free channel in the particle frame is an exact fixed point on the GPU too."""
    g = S.Solver(W.channel(130, 20, variant=variant, passes=4))
    u_in = g.constants()["u_in"]
    g.advance(5)
    f = g.fields()
    assert np.abs(f["u"] - u_in).max() < 1e-13 and np.abs(f["v"]).max() < 1e-13
    assert np.abs(f["p"] - 1).max() < 1e-13 and np.abs(f["T"] - 1).max() < 1e-13


def test_constants_match(S, oracle_mod):
    case = W.c1()
    a = S.Solver(case).constants()
    b = oracle_mod.Case(case).constants()
    for k in ("A", "B", "CT1", "CT2", "CT3", "u_in"):
        assert a[k] == pytest.approx(b[k], rel=1e-15)


def test_bad_state_reported(S):
    """A non-positive temperature is reported as STS_E_STATE with the cell index."""
    case = W.c1_small("implicit_upwind", passes=2)
    g = S.Solver(case)
    T = g.get_field("T")
    T[5, 3] = -1.0
    g.set_field("T", T)
    st, stats = g.advance(1, check=False)
    assert st == S.STS_E_STATE
    assert stats["bad_cell"] >= 0


def test_tolerance_mode_converges(S, oracle_mod):
    """tol > 0: loop 2 stops when all residuals < tol; same pass count as the oracle."""
    case = W.c1_small("implicit_upwind", passes=200)
    case["tol"] = 1e-9
    g = S.Solver(case)
    o = oracle_mod.Case(case)
    st, stats = g.advance(2)
    ost, ores, opasses = o.advance(2)
    assert stats["converged"] == 1 and ost == 0
    assert max(stats["res"]) < 1e-9
    err = rel_errors({k: g.get_field(k) for k in FIELDS}, o.fields(), o.get_map(0) == 0)
    assert max(err.values()) <= 1e-8, err


@pytest.mark.parametrize("H", [10])
def test_parity_paper_mesh(S, oracle_mod, H):
    """The paper's 4032 x 200 mesh (C3, H = 10), implicit upwind, 1 step x 3 passes
    in the bench's launch configuration: every element compared."""
    case = W.c3(H, "implicit_upwind", passes=3)
    _run_compare(S, oracle_mod, case, 1, seed=5)
