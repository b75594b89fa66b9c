"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these compares the oracle with itself or with the CUDA path.  Each
check is chosen so that a plausible transcription slip (dropped term, wrong
sign, wrong index, transposed operand) fails at least one of them:

* closed-form values / identities of the scheme functions (Eqs. pl15_1,
  pl15_2, pl15_12), incl. exactness of the TVD face value on
  linear data on NON-uniform meshes;
* Eq. pl37 constants (golden file with citations);
* exact discrete fixed points: free stream in the particle frame (P:686,
  reading R14) and the quiescent gas, all four scheme variants;
* closed forms: plane Couette flow with velocity slip (Eq. pl38) and
  body-force Poiseuille flow with slip (Eqs. pl2, pl38);
* the transposition identity u-equation(transposed input) == v-equation
  (the paper prints only the v-equation);
* the explicit and implicit schemes reach the same steady state (the
  explicit planes pl15_11 / pl31_1 vs the implicit coefficient sets);
* discrete continuity (Eq. pl4) holds cell by cell at loop-2 convergence;
* mirror symmetry of a centred square; solid cells are never read.
"""
import json
import math
import os

import numpy as np
import pytest

from paper_1802_04243_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------- limiter
def test_vanleer_closed_form(oracle_mod):
    """psi(r) = (r+|r|)/(1+r): psi(1)=1, psi(3)=1.5, psi(1/3)=0.5, psi(r<=0)=0."""
    o = oracle_mod
    assert o.vanleer(1.0) == 1.0
    assert o.vanleer(3.0) == 1.5
    assert abs(o.vanleer(1.0 / 3.0) - 0.5) < 1e-16
    for r in (0.0, -0.5, -1.0, -2.0, -1e300):
        assert o.vanleer(r) == 0.0


def test_vanleer_symmetry_and_bounds(oracle_mod):
    """Van Leer is symmetric, psi(r) = r psi(1/r), and 0 <= psi < 2."""
    rng = np.random.default_rng(1)
    for r in np.exp(rng.uniform(-20, 20, 2000)):
        a = oracle_mod.vanleer(r)
        assert 0.0 <= a < 2.0
        assert abs(a - r * oracle_mod.vanleer(1.0 / r)) <= 1e-14 * max(1.0, a)


def test_upwind_tie_rule(oracle_mod):
    """upwind(phi1, phi2, v) = phi1 if v > 0 else phi2; v = 0 -> phi2 (Eq. pl15_12, R7)."""
    assert oracle_mod.upwind(2, 5, 1) == 2
    assert oracle_mod.upwind(2, 5, 0) == 5
    assert oracle_mod.upwind(2, 5, -1) == 5


def test_psi_closed_values(oracle_mod):
    """Uniform mesh: psi_s = +-0.5 psi(r) (Eq. pl15_2) -- note psi_s((0,1,2,3), v<0)
    is -0.5 (SPEC.md S:106 is wrong); psi_c = 0.5 psi (Eq. pl15_1)."""
    o = oracle_mod
    assert o.psi_s(0, 1, 2, 3, 1, 1, 1, 1, +1) == 0.5
    assert o.psi_s(0, 1, 2, 3, 1, 1, 1, 1, -1) == -0.5
    assert o.psi_s(0, 0, 2, 3, 1, 1, 1, 1, +1) == 0.0            # zero numerator
    assert o.psi_s(0, 1, 1, 3, 1, 1, 1, 1, +1) == 0.0            # zero denominator (R6)
    assert o.psi_c(0, 1, 2, 9, 1, 1, 1, +1) == 0.5
    assert o.psi_c(0, 1, 4, 9, 1, 1, 1, +1) == 0.25              # 0.5 psi(1/3)
    assert o.psi_c(5, 1, 4, 9, 1, 1, 1, +1) == 0.0               # r < 0


def _face_value_s(o, f, d, w):
    """Face value of the TVD scheme: upwind(phi2, phi3, w) + psi_s (phi3 - phi2)."""
    return o.upwind(f[1], f[2], w) + o.psi_s(*f, *d, w) * (f[2] - f[1])


def test_psi_s_exact_on_linear_nonuniform(oracle_mod):
    """On linear data over a NON-uniform mesh r = 1, psi = 1 and the TVD face value
    is the exact linear interpolant at the face x^f for both flow
    directions.  A swapped width in either branch breaks this."""
    o = oracle_mod
    rng = np.random.default_rng(2)
    for _ in range(500):
        d = rng.uniform(0.2, 3.0, 4)
        xc = np.concatenate([[0.0], np.cumsum((d[:-1] + d[1:]) / 2)])   # cell centres
        xface = xc[1] + d[1] / 2
        k, b = rng.uniform(-3, 3, 2)
        f = k * xc + b
        exact = k * xface + b
        for w in (1.0, -1.0):
            assert abs(_face_value_s(o, f, d, w) - exact) < 1e-12 * (1 + abs(exact))


def test_psi_c_exact_on_linear_nonuniform(oracle_mod):
    """psi_c interpolates to the cell centre between two face nodes:
    exact on linear data for a non-uniform mesh, both directions."""
    o = oracle_mod
    rng = np.random.default_rng(3)
    for _ in range(500):
        d = rng.uniform(0.2, 3.0, 3)                  # distances between the 4 nodes
        x = np.concatenate([[0.0], np.cumsum(d)])
        k, b = rng.uniform(-3, 3, 2)
        f = k * x + b
        exact = k * (x[1] + x[2]) / 2 + b
        for w in (1.0, -1.0):
            val = o.upwind(f[1], f[2], w) + o.psi_c(*f, *d, w) * (f[2] - f[1])
            assert abs(val - exact) < 1e-12 * (1 + abs(exact))


def test_psi_s_mirror_identity(oracle_mod):
    """Reflecting the stencil and the flow leaves the TVD face value unchanged:
    psi_s(reversed; -w) = -psi_s(original; w), random non-uniform."""
    o = oracle_mod
    rng = np.random.default_rng(4)
    for _ in range(2000):
        f = rng.normal(size=4)
        d = rng.uniform(0.2, 3.0, 4)
        a = o.psi_s(*f, *d, 1.0)
        b = o.psi_s(*f[::-1], *d[::-1], -1.0)
        assert abs(a + b) < 1e-13 * (1 + abs(a))


def test_psi_s_face_value_bounded(oracle_mod):
    """TVD on a uniform mesh: the face value lies between the two neighbouring cell
    values (0 <= 0.5 psi < 1)."""
    o = oracle_mod
    rng = np.random.default_rng(5)
    for _ in range(2000):
        f = rng.normal(size=4)
        d = np.full(4, rng.uniform(0.5, 2.0))
        for w in (1.0, -1.0):
            val = _face_value_s(o, f, d, w)
            lo, hi = min(f[1], f[2]), max(f[1], f[2])
            assert lo - 1e-14 <= val <= hi + 1e-14


# --------------------------------------------------------------- constants
def test_constants_pl37(oracle_mod):
    """Eq. pl37 and u_in = M sqrt(gamma/2) at Kn = 1e-3, M = 2.43."""
    gold = json.load(open(os.path.join(GOLDEN, "constants_pl37.json")))
    case = oracle_mod.Case(W.channel(8, 4))
    k = case.constants()
    for name in ("A", "B", "CT1", "CT2", "CT3", "u_in"):
        assert abs(k[name] - gold[name]["value"]) <= 1e-13 * abs(gold[name]["value"]), name


# ----------------------------------------------------------- fixed points
@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_free_stream_preserved(oracle_mod, variant):
    """Obstacle-free channel in the particle frame (walls at +u_in, R14), inflow state
    as IC: an exact discrete fixed point of every variant."""
    case = oracle_mod.Case(W.channel(40, 12, variant=variant, passes=5))
    u_in = case.constants()["u_in"]
    st, res, _ = case.advance(8)
    assert st == 0
    f = case.fields()
    assert np.abs(f["u"] - u_in).max() < 1e-13
    assert np.abs(f["v"]).max() < 1e-13
    assert np.abs(f["p"] - 1).max() < 1e-13 and np.abs(f["T"] - 1).max() < 1e-13


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_quiescent_fixed_point(oracle_mod, variant):
    """Gas at rest (u = v = 0, p = T = 1) with walls and a square at rest and T_w = 1
    stays at rest for any dt."""
    c = W.periodic_box(20, 10, 0.1, variant=variant, dt=0.37, passes=6, squares=[(6, 3, 3, 4)])
    case = oracle_mod.Case(c)
    st, _, _ = case.advance(5)
    assert st == 0
    f = case.fields()
    assert np.abs(f["u"]).max() == 0 and np.abs(f["v"]).max() == 0
    assert np.abs(f["p"] - 1).max() < 1e-15 and np.abs(f["T"] - 1).max() < 1e-15


# ---------------------------------------------------------- closed forms
def test_couette_slip_closed_form(oracle_mod):
    """Plane Couette flow between walls at -U / +U with velocity slip (Eq. pl38,
    zeta = 1.1466 Kn / rho): u(y) = U (2y - H) / (H + 2 zeta).  The slip wall
    link is exact for linear profiles, so only viscous heating (O(U^2)) is left."""
    U, N, H, Kn = 0.02, 16, 1.0, 0.05
    c = W.periodic_box(4, N, H / N, dt=0.5, passes=2000, Kn=Kn, u_wall_bottom=-U, u_wall_top=U)
    c["tol"] = 1e-12
    case = oracle_mod.Case(c)
    for _ in range(40):
        st, _, _ = case.advance(10)
        assert st == 0
    y = (np.arange(N) + 0.5) * H / N
    zeta = 1.1466 * Kn
    exact = U * (2 * y - H) / (H + 2 * zeta)
    u = case.get("u")
    assert np.abs(u - exact[:, None]).max() < 2e-5 * U
    assert np.abs(case.get("v")).max() < 1e-12


def test_poiseuille_slip_closed_form(oracle_mod):
    """Body-force Poiseuille flow with slip (Eqs. pl2 + pl38): continuum
    u = (g/2B)[y(H-y) + zeta H]; the discrete solution (exact interior second
    differences + the one-sided slip wall link of BC spec 5) is the same parabola
    shifted by (g/2B) dn^2, dn = Delta/2.  Residual differences come from viscous
    heating (T - 1 < 1e-3)."""
    N, H, g, Kn = 32, 1.0, 9.0114e-3, 0.05
    c = W.periodic_box(4, N, H / N, dt=0.5, passes=3000, Kn=Kn, g_x=g)
    c["tol"] = 1e-12
    case = oracle_mod.Case(c)
    B = 5.0 * math.sqrt(math.pi) / 16.0 * Kn
    zeta = 1.1466 * Kn
    y = (np.arange(N) + 0.5) * H / N
    u0 = np.zeros((N, 5))
    u0[:] = ((g / (2 * B)) * (y * (H - y) + zeta * H))[:, None]
    case.set("u", u0)
    for _ in range(40):
        st, _, _ = case.advance(10)
        assert st == 0
    u = case.get("u")[:, 0]
    dn = H / N / 2
    disc = (g / (2 * B)) * (y * (H - y) + zeta * H + dn * dn)
    cont = (g / (2 * B)) * (y * (H - y) + zeta * H)
    assert np.abs(u - disc).max() < 6e-4 * disc.max()
    assert np.abs(u - cont).max() < 1.5e-3 * cont.max()
    assert abs(u.max() - 0.05) < 1e-3          # u_max = 0.05
    assert np.abs(case.get("v")).max() < 1e-12


# ---------------------------------------------------------- transposition
def _transpose_state(f, N):
    """Map a state of the box A onto box B = A transposed.  Box: nx = N+1, ny = N,
    periodic x, solid column i = 0 -> interior cells i = 1..N, j = 0..N-1.
    Cell (i, j) of A <-> cell (j+1, i-1) of B; v_A(i, j) <-> u_B(j+1, i-1);
    u_A(i, j) <-> v_B(j+1, i-1)."""
    g = {k: np.zeros_like(v) for k, v in f.items()}
    for name in ("p", "T"):
        a = f[name]
        for j in range(N):
            for i in range(1, N + 1):
                g[name][i - 1, j + 1] = a[j, i]
        g[name][:, 0] = a[:, 0]                       # the solid column itself
    for j in range(N + 1):
        for i in range(1, N + 1):
            g["u"][i - 1, j + 1] = f["v"][j, i]
    for j in range(N):
        for i in range(1, N + 1):
            g["v"][i - 1, j + 1] = f["u"][j, i]
    return g


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_transposition_symmetry(oracle_mod, variant):
    """The paper prints only the v-equation; the u-equation is its x<->y
    transposition (DESIGN 3.4).  In a closed square box whose channel walls
    (bottom/top) and square walls (left/right, a solid column with periodic x)
    obey the same slip/jump spec, evolving a random state and evolving its
    transpose must give transposed results."""
    N = 10
    c = W.periodic_box(N + 1, N, 0.1, variant=variant, dt=0.02, passes=3, Kn=0.02, squares=[(0, 0, 1, N)])
    A = oracle_mod.Case(c)
    Bc = oracle_mod.Case(c)
    rng = np.random.default_rng(7)
    f = {"u": 0.3 * rng.uniform(-1, 1, (N, N + 2)), "v": 0.3 * rng.uniform(-1, 1, (N + 1, N + 1)),
         "p": 1 + 0.2 * rng.uniform(-1, 1, (N, N + 1)), "T": 1 + 0.2 * rng.uniform(-1, 1, (N, N + 1))}
    for k in ("T", "p", "u", "v"):
        A.set(k, f[k])
    fa = {k: A.get(k) for k in ("u", "v", "p", "T")}      # fixed faces imposed
    fb = _transpose_state(fa, N)
    for k in ("T", "p", "u", "v"):
        Bc.set(k, fb[k])
    assert A.advance(2)[0] == 0 and Bc.advance(2)[0] == 0
    ra = {k: A.get(k) for k in ("u", "v", "p", "T")}
    rb = {k: Bc.get(k) for k in ("u", "v", "p", "T")}
    tb = _transpose_state(ra, N)
    for k in ("u", "v", "p", "T"):
        assert np.abs(tb[k] - rb[k]).max() < 1e-13, k
    # and the state really moved
    assert np.abs(ra["u"] - fa["u"]).max() > 1e-3


# ------------------------------------------------ explicit vs implicit steady
def _steady(oracle_mod, variant):
    c = W.periodic_box(20, 10, 0.1, variant=variant, dt=0.05, passes=500, Kn=0.05, g_x=0.05,
                       squares=[(7, 3, 3, 4)])
    c["tol"] = 1e-12
    case = oracle_mod.Case(c)
    prev = None
    for _ in range(600):
        st, _, _ = case.advance(5)
        assert st == 0
        f = case.fields()
        if prev is not None and max(np.abs(f[k] - prev[k]).max() for k in f) < 2e-12:
            return f
        prev = f
    raise AssertionError("no steady state")


@pytest.mark.parametrize("space", ["upwind", "tvd"])
def test_explicit_implicit_same_steady_state(oracle_mod, space):
    """At a steady state n-1 = old = new, so the explicit planes (Eqs. pl15_11,
    pl31_1 and the transposed u-plane) must reproduce exactly the convective parts
    of the implicit coefficients (Eqs. pl15, pl31): the face-value and coefficient
    forms are algebraically equal.  Low-Re flow past a square, both limiters."""
    fi = _steady(oracle_mod, "implicit_" + space)
    fe = _steady(oracle_mod, "explicit_" + space)
    assert fi["u"].max() > 0.05
    for k in ("u", "v", "p", "T"):
        assert np.abs(fi[k] - fe[k]).max() < 1e-9, k


# ---------------------------------------------------------- conservation
def test_discrete_continuity_at_convergence(oracle_mod):
    """At loop-2 convergence the pressure equation (Eqs. pl23-pl24) with the velocity
    correction (pl18-pl19) and the EOS (pl5) is the discrete continuity equation (pl4):
    (rho - rho^{n-1}) dV + dt sum_faces rho_face u dA = 0 in every fluid cell, with the
    first-order upwind face density (the implicit-upwind variant) -- and summed over the
    channel, the mass change equals the inflow minus the outflow."""
    c = W.channel(30, 10, spacing=0.25, variant="implicit_upwind", passes=400, squares=[(8, 3, 3, 4)])
    c["tol"] = 1e-13
    case = oracle_mod.Case(c)
    assert case.advance(3)[0] in (0, 3)
    before = case.fields()
    st, res, npass = case.advance(1)
    assert st == 0, (res, npass)
    f = case.fields()
    solid = case.get_map(0).astype(bool)
    d, dt = c["spacing"], c["dt"]
    rho, u, v = f["rho"], f["u"], f["v"]
    nx, ny = c["nx"], c["ny"]
    rin = c["p_in"] / c["T_in"]
    worst = 0.0
    for j in range(ny):
        for i in range(nx):
            if solid[j, i]:
                continue
            def flux_x(ii):
                w = u[j, ii]
                left = rin if ii == 0 else rho[j, ii - 1]
                right = rho[j, ii] if ii < nx else rho[j, nx - 1]
                return (left if w > 0 else right) * w * d
            def flux_y(jj):
                w = v[jj, i]
                if jj == 0 or jj == ny:
                    return 0.0
                return (rho[jj - 1, i] if w > 0 else rho[jj, i]) * w * d
            # the outlet face carries u_old(nx-1) (BC spec 3) -- at convergence = u(nx-1)
            fe = flux_x(i + 1) if i + 1 < nx else rho[j, nx - 1] * u[j, nx - 1] * d
            r = (rho[j, i] - before["rho"][j, i]) * d * d + dt * (fe - flux_x(i) + flux_y(j + 1) - flux_y(j))
            worst = max(worst, abs(r))
    assert worst < 1e-11


# ------------------------------------------------------------- symmetry
@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_mirror_symmetry_centred_square(oracle_mod, variant):
    """C1 geometry: the square is centred in y and both walls move at +u_in, so p, T,
    rho, u are even and v odd under y -> H - y."""
    c = W.c1(variant, passes=10)
    case = oracle_mod.Case(c)
    st, _, _ = case.advance(20)
    assert st == 0
    f = case.fields()
    tol = 1e-11 if "upwind" in variant else 1e-9
    for k in ("p", "T", "rho", "u"):
        assert np.abs(f[k] - f[k][::-1]).max() < tol * np.abs(f[k]).max(), k
    assert np.abs(f["v"] + f["v"][::-1]).max() < tol * np.abs(f["u"]).max()


@pytest.mark.parametrize("variant", ["implicit_tvd", "explicit_tvd"])
def test_solid_cells_never_read(oracle_mod, variant):
    """BC spec 1: solid cells are never updated and never read -- poisoning them
    with NaN changes nothing, bit for bit."""
    c = W.c1_small(variant, passes=3)
    a = oracle_mod.Case(c)
    b = oracle_mod.Case(c)
    b.poison_solids()
    assert a.advance(4)[0] == 0
    assert b.advance(4)[0] == 0
    fa, fb = a.fields(), b.fields()
    solid = a.get_map(0).astype(bool)
    for k in ("u", "v"):
        assert np.array_equal(fa[k], fb[k])
    for k in ("p", "T", "rho"):
        assert np.array_equal(fa[k][~solid], fb[k][~solid])


def test_supersonic_square_physical(oracle_mod):
    """C1, implicit upwind: the state stays positive and bounded, and the gas is
    compressed and heated in front of the square (stagnation; reading R9)."""
    c = W.c1("implicit_upwind", passes=10)
    case = oracle_mod.Case(c)
    for _ in range(5):
        assert case.advance(20)[0] == 0
    f = case.fields()
    fluid = ~case.get_map(0).astype(bool)
    u_in = case.constants()["u_in"]
    assert f["p"][fluid].min() > 0 and f["T"][fluid].min() > 0
    assert np.abs(f["u"]).max() <= 2 * u_in
    front = f["T"][18:22, 19:22]            # cells just upstream of the square face i = 22
    assert front.min() > 1.3 and f["p"][18:22, 19:22].min() > 2.0


# --------------------------------------------------- energy equation (R9, R38)
def _acoustic_speed(oracle_mod, form):
    """Standing acoustic wave in a periodic box: u = eps sin(kx) at t = 0, p = T = 1.
    u at the face x = L/4 oscillates as eps cos(omega t); the first zero crossing
    (linear interpolation in t) gives omega = pi / (2 t_1), c = omega / k.  Kn = 1e-5
    makes viscous / conductive effects negligible; implicit upwind, dt = 0.01
    (backward Euler phase error (omega dt)^2 / 3 < 1e-4); 64 cells per wavelength."""
    nx, L, H, dt, eps = 64, 4.0, 1.0, 0.01, 1e-3
    d = L / nx
    ny = int(round(H / d))
    c = W.periodic_box(nx, ny, d, variant="implicit_upwind", dt=dt, passes=8, Kn=1e-5)
    c["pw_form"] = form
    case = oracle_mod.Case(c)
    x = np.arange(nx + 1) * d
    u = np.zeros((ny, nx + 1))
    u[:] = eps * np.sin(2 * math.pi * x / L)[None, :]
    case.set("u", u)
    prev = case.get("u")[:, nx // 4].mean()
    for s in range(1, 250):
        assert case.advance(1)[0] == 0
        cur = case.get("u")[:, nx // 4].mean()
        if prev * cur < 0:
            t1 = dt * (s - 1) + dt * prev / (prev - cur)
            return math.pi / (2 * t1) / (2 * math.pi / L)
        prev = cur
    raise AssertionError("no zero crossing")


@pytest.mark.parametrize("form,passes", [(W.PW_DPDT, True), (W.PW_GAMMA, True),
                                         (W.PW_PRINTED, False), (W.PW_NEG, False)])
def test_acoustic_speed(oracle_mod, form, passes):
    """Speed of sound of the discrete gas.  The continuum model (Eqs. pl2, pl4-pl6,
    P:43-68) linearised about p = T = rho = 1: rho du/dt = -A dp/dx with A = 1/2
    (Eq. pl37), and the energy equation rho DT/Dt = C^T3 Dp/Dt (C^T3 = 2/5 =
    (gamma-1)/gamma, gamma = 5/3) with p = rho T gives dp/drho = gamma T,
    so c = sqrt(gamma T / 2) = 0.9129 (the inflow Mach number of P:669 uses the same
    c, u_in = M sqrt(gamma/2)).  The pressure-work term decides it: C^T3 Dp/Dt
    (R9, default) and -gamma C^T3 p div u give 0.9129; the term as printed
    (+C^T3 p div u) gives sqrt(0.3) = 0.548 and the round-1 reading
    (-C^T3 p div u) sqrt(0.7) = 0.837 -- both rejected by this pin."""
    c = _acoustic_speed(oracle_mod, form)
    c0 = math.sqrt(5.0 / 3.0 / 2.0)
    if passes:
        assert abs(c / c0 - 1) < 2e-3, c
    else:
        assert abs(c / c0 - 1) > 5e-2, c


def _thermal_decay_ratio(oracle_mod, form):
    """Isobaric decay of an entropy mode T = 1 + eps cos(kx), p = 1, gas at rest, in a
    periodic box (L = 1, H = 2, 16 x 32 cells, Kn = 5e-3, dt = 0.02): the amplitude
    at mid-height decays as exp(-lambda t), and lambda divided by the rate of the
    discrete heat equation with the paper's C^T1 (Eq. pl37) is returned."""
    nx, L, H, dt, Kn, eps, steps = 16, 1.0, 2.0, 0.02, 5e-3, 1e-3, 150
    d = L / nx
    ny = int(round(H / d))
    c = W.periodic_box(nx, ny, d, variant="implicit_upwind", dt=dt, passes=20, Kn=Kn)
    c["pw_form"] = form
    case = oracle_mod.Case(c)
    x = (np.arange(nx) + 0.5) * d
    k = 2 * math.pi / L
    case.set("T", 1.0 + eps * np.cos(k * x)[None, :] * np.ones((ny, 1)))
    t, amp = [], []
    for s in range(steps + 1):
        if s:
            assert case.advance(1)[0] == 0
        if s * dt >= 1.0:                       # after the acoustic transient
            Tm = case.get("T")[ny // 2 - 1:ny // 2 + 1].mean(axis=0)
            t.append(s * dt)
            amp.append(2 * np.mean((Tm - 1) * np.cos(k * x)))
    rate = -np.polyfit(np.array(t), np.log(np.array(amp)), 1)[0]
    CT1 = Kn * math.sqrt(225 * math.pi / 1024)
    lam = CT1 * (2 - 2 * math.cos(k * d)) / d ** 2      # discrete Laplacian eigenvalue
    return rate / (math.log(1 + lam * dt) / dt)         # backward-Euler decay per unit time


@pytest.mark.parametrize("form,expected", [(W.PW_DPDT, 1.0), (W.PW_GAMMA, 0.6),
                                           (W.PW_NEG, 1 / 1.4), (W.PW_PRINTED, None)])
def test_isobaric_thermal_diffusion(oracle_mod, form, expected):
    """At rest and at uniform pressure Eq. pl6 is rho dT/dt = C^T1 lap T (C^T1 is the
    c_p-form conductivity: Kn sqrt(225 pi/1024) = (15/32) sqrt(pi) Kn of
    Eq. pl36 over rho0 c_p V0 a), so a temperature mode decays at C^T1 k^2 / rho.
    Only C^T3 Dp/Dt (R9, ratio 1) gets this right; a p div(u) term with
    coefficient kappa makes the decay isobaric-expansion-loaded,
    rho dT/dt (1 - kappa) = C^T1 lap T: -gamma C^T3 -> 1/gamma, -C^T3 -> 1/1.4
    (each measured here within 3 %); +C^T3 (as printed) has c = 0.548, too slow for
    the isobaric limit at this k, and is only required to be far off."""
    r = _thermal_decay_ratio(oracle_mod, form)
    if expected is not None:
        assert abs(r / expected - 1) < 3e-2, r
    if form != W.PW_DPDT:
        assert abs(r - 1) > 0.25, r


def test_poiseuille_temperature_and_jump(oracle_mod):
    """Steady slip Poiseuille flow (C2 geometry, 4 x 16 cells, Kn = 0.05): the energy
    equation reduces to 0 = C^T1 T'' + C^T2 (u')^2 with u' = (g/2B)(H - 2y), so
    T - T_s = (C^T2/C^T1) (g/2B)^2 [H^4 - (H - 2y)^4] / 48 (viscous heating C^T2 Gamma
    Phi and conduction C^T1 of Eqs. pl6-pl7, pl37), and at the walls the temperature
    jump of Eq. pl39: T_s - T_w = tau dT/dn, tau = 2.1904 Kn / rho,
    dT/dn = (C^T2/C^T1)(g/2B)^2 H^3 / 6.  Rise 2.9e-4, jump 2.6e-4; the discrete
    solution is second-order (0.9 % at 16 cells, 0.2 % at 32).  A factor 2 in Phi,
    the slip coefficient 1.1466 in place of 2.1904, or the wall velocity in place
    of the slip velocity at a wall face of S^T_c (R38) each fail it."""
    N, H, g, Kn = 16, 1.0, 9.0114e-3, 0.05
    c = W.periodic_box(4, N, H / N, dt=0.5, passes=3000, Kn=Kn, g_x=g)
    c["tol"] = 1e-12
    case = oracle_mod.Case(c)
    B = 5.0 * math.sqrt(math.pi) / 16.0 * Kn
    CT1 = Kn * math.sqrt(225 * math.pi / 1024)
    CT2 = math.sqrt(math.pi) / 4 * Kn
    zeta = 1.1466 * Kn
    y = (np.arange(N) + 0.5) * H / N
    G = g / (2 * B)
    u0 = np.zeros((N, 5))
    u0[:] = (G * (y * (H - y) + zeta * H))[:, None]
    case.set("u", u0)
    for _ in range(40):
        assert case.advance(10)[0] == 0
    T = case.get("T")
    assert np.abs(T - T[:, :1]).max() < 1e-13                    # uniform in x
    T = T[:, 0]
    jump = 2.1904 * Kn * (CT2 / CT1) * G ** 2 * H ** 3 / 6      # rho = p / T = 1 - O(1e-3)
    rise = (CT2 / CT1) * G ** 2 * (H ** 4 - (H - 2 * y) ** 4) / 48
    exact = 1.0 + jump + rise
    total = exact.max() - 1.0
    assert np.abs(T - exact).max() < 1.5e-2 * total, np.abs(T - exact).max() / total
    assert abs((T[N // 2] - T[0]) - (exact[N // 2] - exact[0])) < 2e-2 * (exact[N // 2] - exact[0])


# ---------------------------------------------------------------- R37 guard
def test_r37_threshold_edges(oracle_mod):
    """R37: |phi3 - phi2| <= 1e-12 (1 + |phi2| + |phi3|) counts as a flat stencil
    (psi = 0); just above the threshold the limiter is evaluated as usual (on
    linear data r = 1, psi_s = 0.5 on a uniform mesh)."""
    o = oracle_mod
    for base in (1.0, 2.5, 100.0):
        thr = 1e-12 * (1 + 2 * base)
        for delta, want in ((0.5 * thr, 0.0), (2.0 * thr, 0.5)):
            f = (base - delta, base, base + delta, base + 2 * delta)
            assert o.psi_s(*f, 1, 1, 1, 1, +1) == pytest.approx(want, abs=1e-3), (base, delta)
            assert o.psi_c(*f, 1, 1, 1, +1) == pytest.approx(want, abs=1e-3), (base, delta)


@pytest.mark.parametrize("r37_off", [0, 1])
def test_r37_conditioning(oracle_mod, r37_off):
    """Why R37 exists: in the implicit coefficient form F psi enters a_0, so on a
    rounding-flat stencil r = noise / noise gives an arbitrary O(1) psi.  C1
    implicit TVD after 19 steps, then one step from that state and from the same
    state with T moved by one ulp everywhere: with the guard the two stay within
    1e-13; without it (test hook r37_off) they differ by > 1e-10 -- the 1e-9
    parity bar would be at the mercy of rounding order."""
    c = W.c1("implicit_tvd", passes=10)
    c["r37_off"] = r37_off
    a = oracle_mod.Case(c)
    assert a.advance(19)[0] == 0
    st = {k: a.get(k) for k in ("u", "v", "p", "T")}
    b1, b2 = oracle_mod.Case(c), oracle_mod.Case(c)
    for k in ("T", "p", "u", "v"):
        b1.set(k, st[k])
        b2.set(k, np.nextafter(st[k], 2.0) if k == "T" else st[k])
    assert b1.advance(1)[0] == 0 and b2.advance(1)[0] == 0
    f1, f2 = b1.fields(), b2.fields()
    diff = max(np.abs(f1[k] - f2[k]).max() for k in ("u", "v", "p", "T"))
    if r37_off:
        assert diff > 1e-10, diff
    else:
        assert diff < 1e-13, diff


@pytest.mark.parametrize("variant", ["implicit_tvd", "explicit_tvd"])
def test_r37_inert_on_real_gradients(oracle_mod, variant):
    """R37 does not touch real gradients: from a +-1 % perturbed state (differences
    ~1e-2, far above 1e-12) the runs with and without the guard are bit-identical."""
    out = []
    for off in (0, 1):
        c = W.c1_small(variant, passes=3)
        c["r37_off"] = off
        case = oracle_mod.Case(c)
        base = {k: case.get(k) for k in ("u", "v", "p", "T")}
        st = W.perturbed_state(base, W.perturbation(c, 21), vscale=0.05)
        for k in ("p", "T", "u", "v"):
            case.set(k, st[k])
        assert case.advance(2)[0] == 0
        out.append(case.fields())
    for k in out[0]:
        assert np.array_equal(out[0][k], out[1][k]), k
