"""Pins of the CPU oracle on NON-uniform meshes.

The paper writes every coefficient for a general staggered mesh with steps
Delta x_i, Delta y_j (Fig. 5; Eqs. pl10-pl16, pl24, pl29-pl33 carry
them explicitly); its test case is uniform.  The oracle's only
additions for a general mesh are the bilinear weights of reading R4 (corner
Gamma, the mid-face velocities of S^T_c).  None of these tests compares the
oracle with itself on the same input or with the CUDA path:

* exact discrete fixed points: free stream on a rough mesh (all variants);
* plane Couette flow with slip is exact for the linear profile on a rough y mesh
  (the y-distances of the tangential links and the wall half-cell);
* slip Poiseuille velocity and temperature (viscous heating through the
  bilinear mid-face velocities of S^T_c, conduction, the Eq. pl39 jump) converge
  at second order to the closed forms on a smoothly stretched mesh -- a weight
  applied to the wrong node makes the heating first order;
* the transposition identity with Delta x <-> Delta y swapped (every Delta in
  the u- and v-equations in the right direction and index);
* mirror symmetry of C1 on a mirror-symmetric y mesh with a rough x mesh;
* cell-wise discrete continuity (Eq. pl4) at loop-2 convergence with the
  cell widths and heights of a rough mesh.
"""
import math

import numpy as np
import pytest

from paper_1802_04243_b200 import workloads as W
from tests.test_oracle_pins import _transpose_state


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_free_stream_nonuniform(oracle_mod, variant):
    """Obstacle-free channel in the particle frame (walls at +u_in, R14) on a
    rough mesh: the uniform state is an exact fixed point of the discrete scheme."""
    c = W.channel(40, 16, variant=variant, passes=4)
    c = W.with_mesh(c, W.random_steps(40, 0.25, seed=1), W.random_steps(16, 0.25, seed=2))
    case = oracle_mod.Case(c)
    u_in = case.constants()["u_in"]
    assert case.advance(5)[0] == 0
    f = case.fields()
    assert np.abs(f["u"] - u_in).max() < 1e-13 and np.abs(f["v"]).max() < 1e-13
    assert np.abs(f["p"] - 1).max() < 1e-13 and np.abs(f["T"] - 1).max() < 1e-13


def test_couette_slip_nonuniform(oracle_mod):
    """Plane Couette flow with slip (Eq. pl38) on a rough y mesh: the tangential
    links use the distance between u-nodes (Delta y_{j-1} + Delta y_j)/2 and the
    wall link the half-cell Delta y_0 / 2, so the linear profile
    u(y) = U (2y - H) / (H + 2 zeta) is exact at the cell centres (up to the
    O(U^2) viscous heating) -- a Delta taken from the wrong row is not."""
    U, N, Kn = 0.02, 16, 0.05
    dys = W.random_steps(N, 1.0 / N, seed=3)
    c = W.periodic_box(4, N, 1.0 / N, dt=0.5, passes=2000, Kn=Kn, u_wall_bottom=-U, u_wall_top=U)
    c["tol"] = 1e-12
    c = W.with_mesh(c, None, dys)
    case = oracle_mod.Case(c)
    for _ in range(40):
        assert case.advance(10)[0] == 0
    H = dys.sum()
    y = np.cumsum(dys) - 0.5 * dys
    zeta = 1.1466 * Kn
    exact = U * (2 * y - H) / (H + 2 * zeta)
    assert np.abs(case.get("u") - exact[:, None]).max() < 2e-5 * U
    assert np.abs(case.get("v")).max() < 1e-12


def _poiseuille_nonuniform(oracle_mod, N):
    """Steady slip Poiseuille flow on the smoothly stretched y mesh of N rows
    (C2 gas, Kn = 0.05); returns (u error / u_max, T error / T rise) against the
    closed forms of test_poiseuille_temperature_and_jump."""
    H, g, Kn = 1.0, 9.0114e-3, 0.05
    dys = W.smooth_steps(N, H / N, 0.3)
    c = W.periodic_box(4, N, H / N, dt=0.5, passes=3000, Kn=Kn, g_x=g)
    c["tol"] = 1e-12
    c = W.with_mesh(c, None, dys)
    case = oracle_mod.Case(c)
    B = 5.0 * math.sqrt(math.pi) / 16.0 * Kn
    CT1 = Kn * math.sqrt(225 * math.pi / 1024)
    CT2 = math.sqrt(math.pi) / 4 * Kn
    zeta = 1.1466 * Kn
    y = np.cumsum(dys) - 0.5 * dys
    G = g / (2 * B)
    u_cf = G * (y * (H - y) + zeta * H)
    case.set("u", np.repeat(u_cf[:, None], 5, axis=1))
    for _ in range(40):
        assert case.advance(10)[0] == 0
    u = case.get("u")[:, 0]
    T = case.get("T")[:, 0]
    jump = 2.1904 * Kn * (CT2 / CT1) * G ** 2 * H ** 3 / 6
    rise = (CT2 / CT1) * G ** 2 * (H ** 4 - (H - 2 * y) ** 4) / 48
    T_cf = 1.0 + jump + rise
    return np.abs(u - u_cf).max() / u_cf.max(), np.abs(T - T_cf).max() / (T_cf.max() - 1.0)


def test_poiseuille_nonuniform_second_order(oracle_mod):
    """Slip Poiseuille velocity and temperature on a smoothly stretched y mesh
    (steps vary by +-30 %): both errors fall at second order from 16 to 32 rows
    (ratio > 3; 4.1 and 4.0 measured).  The temperature is heated through the mid-face velocities of
    S^T_c (bilinear weights, R4) and cooled through the Eq. pl39 jump; a
    bilinear weight on the wrong node leaves an O(Delta) heating error."""
    eu16, eT16 = _poiseuille_nonuniform(oracle_mod, 16)
    eu32, eT32 = _poiseuille_nonuniform(oracle_mod, 32)
    assert eu16 < 8e-3 and eT16 < 3e-2, (eu16, eT16)      # 5.2e-3, 1.7e-2 measured
    assert eu16 / eu32 > 3.0 and eT16 / eT32 > 3.0, (eu16, eu32, eT16, eT32)


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_transposition_nonuniform(oracle_mod, variant):
    """The transposition identity of test_transposition_symmetry on rough meshes:
    box A has column steps (x0, a_1..a_N) and row steps (b_0..b_{N-1}); the
    transposed box B has column steps (x0, b_0..b_{N-1}) and row steps
    (a_1..a_N).  Evolving a random state in A and its transpose in B must give
    transposed results: every Delta x / Delta y of the printed v-equation and of
    its transposition (the u-equation) sits in the right direction and index."""
    N = 10
    a = W.random_steps(N, 0.1, seed=5)
    b = W.random_steps(N, 0.1, seed=6)
    x0 = 0.1
    c = W.periodic_box(N + 1, N, 0.1, variant=variant, dt=0.02, passes=3, Kn=0.02, squares=[(0, 0, 1, N)])
    A = oracle_mod.Case(W.with_mesh(c, np.concatenate([[x0], a]), b))
    Bc = oracle_mod.Case(W.with_mesh(c, np.concatenate([[x0], b]), a))
    rng = np.random.default_rng(7)
    f = {"u": 0.3 * rng.uniform(-1, 1, (N, N + 2)), "v": 0.3 * rng.uniform(-1, 1, (N + 1, N + 1)),
         "p": 1 + 0.2 * rng.uniform(-1, 1, (N, N + 1)), "T": 1 + 0.2 * rng.uniform(-1, 1, (N, N + 1))}
    for k in ("T", "p", "u", "v"):
        A.set(k, f[k])
    fa = {k: A.get(k) for k in ("u", "v", "p", "T")}
    fb = _transpose_state(fa, N)
    for k in ("T", "p", "u", "v"):
        Bc.set(k, fb[k])
    assert A.advance(2)[0] == 0 and Bc.advance(2)[0] == 0
    ra = {k: A.get(k) for k in ("u", "v", "p", "T")}
    rb = {k: Bc.get(k) for k in ("u", "v", "p", "T")}
    tb = _transpose_state(ra, N)
    for k in ("u", "v", "p", "T"):
        assert np.abs(tb[k] - rb[k]).max() < 1e-13, k
    assert np.abs(ra["u"] - fa["u"]).max() > 1e-3


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_mirror_symmetry_nonuniform(oracle_mod, variant):
    """C1 with a mirror-symmetric stretched y mesh (steps +-30 %) and a rough x mesh:
    the square stays centred, both walls move at +u_in, so p, T, rho, u are even and
    v odd under y -> H - y after 20 steps."""
    c = W.c1(variant, passes=10)
    c = W.with_mesh(c, W.random_steps(120, 0.25, seed=8), W.smooth_steps(40, 0.25, 0.3))
    case = oracle_mod.Case(c)
    assert case.advance(20)[0] == 0
    f = case.fields()
    tol = 1e-11 if "upwind" in variant else 1e-9
    for k in ("p", "T", "rho", "u"):
        assert np.abs(f[k] - f[k][::-1]).max() < tol * np.abs(f[k]).max(), k
    assert np.abs(f["v"] + f["v"][::-1]).max() < tol * np.abs(f["u"]).max()
    assert np.abs(f["v"]).max() > 1e-3


def test_discrete_continuity_nonuniform(oracle_mod):
    """Eq. pl4 cell by cell at loop-2 convergence on a rough mesh (implicit upwind):
    (rho - rho^{n-1}) Delta x_i Delta y_j + dt (F_e - F_w + F_n - F_s) = 0 with
    F^x = rho^u u Delta y_j (Eq. pl8), F^y = rho^v v Delta x_i (Eq. pl9)."""
    nx, ny = 30, 10
    dxs = W.random_steps(nx, 0.25, seed=9)
    dys = W.random_steps(ny, 0.25, seed=10)
    c = W.channel(nx, ny, spacing=0.25, variant="implicit_upwind", passes=400, squares=[(8, 3, 3, 4)])
    c["tol"] = 1e-13
    c = W.with_mesh(c, dxs, dys)
    case = oracle_mod.Case(c)
    assert case.advance(3)[0] in (0, 3)
    before = case.fields()
    st, res, npass = case.advance(1)
    assert st == 0, (res, npass)
    f = case.fields()
    solid = case.get_map(0).astype(bool)
    dt = c["dt"]
    rho, u, v = f["rho"], f["u"], f["v"]
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
                return (left if w > 0 else right) * w * dys[j]

            def flux_y(jj):
                w = v[jj, i]
                if jj == 0 or jj == ny:
                    return 0.0
                return (rho[jj - 1, i] if w > 0 else rho[jj, i]) * w * dxs[i]
            fe = flux_x(i + 1) if i + 1 < nx else rho[j, nx - 1] * u[j, nx - 1] * dys[j]
            r = (rho[j, i] - before["rho"][j, i]) * dxs[i] * dys[j] + dt * (fe - flux_x(i) + flux_y(j + 1) - flux_y(j))
            worst = max(worst, abs(r))
    assert worst < 1e-11


@pytest.mark.parametrize("variant", ["explicit_upwind", "explicit_tvd"])
def test_shear_heating_exact_for_linear_velocity(oracle_mod, variant):
    """The mid-face velocities of S^T_c are bilinear interpolations (R4), exact
    for a linear field.  One pass from p = T = 1, v = 0, u = a y (at the u-node
    centres of each mesh): cell row 4 gets the viscous heating C^T2 Gamma a^2 dV of
    the exact shear, and its T-equation coefficients depend on the neighbour rows
    only through the conduction links (explicit scheme: the convective part is the
    T^exp plane, 0 for this x-invariant uniform T) C^T1 Delta x / ((Delta y_4 + Delta y_{4+-1})/2),
    whose sum is the same for the neighbour heights (0.5, 1.5) and (0.875, 0.875)
    (1/1.5 + 1/2.5 = 2/1.875).  So T of row 4 must agree on the two meshes; a
    weight put on the wrong node shifts the interpolated u by a (Delta y_{j+1} -
    Delta y_j)/2 and the two meshes then disagree (planted-bug check, DESIGN 3.7)."""
    d = 0.125
    out = []
    for h1, h2 in ((0.5, 1.5), (0.875, 0.875)):
        dys = d * np.array([1, 1, 1, h1, 1, h2, 1, 1], dtype=float)
        c = W.periodic_box(4, 8, d, variant=variant, dt=0.01, passes=1, Kn=0.05)
        case = oracle_mod.Case(W.with_mesh(c, None, dys))
        y = np.cumsum(dys) - 0.5 * dys
        case.set("u", np.repeat((0.3 * y)[:, None], 5, axis=1))
        assert case.advance(1)[0] == 0
        out.append(case.get("T")[4] - 1.0)
    assert out[0].min() > 1e-7                                 # the heating is there
    assert np.abs(out[0] - out[1]).max() < 1e-12 * out[0].max(), (out[0], out[1])
