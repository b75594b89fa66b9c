/*
 * simplets_oracle.c -- TEST INFRASTRUCTURE ONLY (see simplets_oracle.h).
 *
 * The SIMPLE-TS step of arXiv:1802.04243 written out plainly, in fp64, in the
 * paper's notation and order, single-threaded, compiled with
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 *
 * One loop-2 pass is done as three whole-field phases:
 *   phase A: T (Eq. pl30), u-hat/d^u (Eq. pl20 + transposition, DESIGN 3.4),
 *            v-hat/d^v (Eqs. pl14-pl16, pl21) from loop-2 constants only
 *            (Eqs. pl29_1-pl29_5);
 *   phase B: p (Eqs. pl23-pl24) with T of phase A (Eq. pl29_6);
 *   phase C: u, v (Eqs. pl18-pl19), rho = p/T (Eq. pl5), Gamma = sqrt(T)
 *            (Eq. pl37), residuals.
 * This equals the paper's row sweep because every value in a phase depends
 * only on loop-2 constants or on earlier phases.
 *
 * Boundary handling follows DESIGN.md section 3.5 ("BC spec"), which the
 * paper leaves open; every reading taken is listed in DESIGN.md 3.6 as Rnn.
 * Values that the spec says are never read (solid cells, cells beyond the
 * channel walls) are returned as NaN, so a spec violation poisons the result.
 */
#include "simplets_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

enum { K_FLUID = 0, K_SOLID = 1, K_WALLY = 2, K_INLET = 3, K_OUTLET = 4 };
enum { F_ACTIVE = 0, F_FIXED0 = 1, F_INLET = 2, F_OUTLET = 3, F_WALL = 4, F_NONE = 5 };

typedef struct { double *u, *v, *p, *T, *rho, *gam; } level;

struct orc_case {
    orc_params P;
    int nx, ny;
    double A, B, CT1, CT2, CT3, u_in;
    double PWK;                  /* kappa of the p div(u) forms of R9 */
    unsigned char* solid;        /* nx*ny, 1 = inside a square          */
    level L[3];                  /* 0: time n-1, 1: old iterate, 2: new */
    double *ue, *ve, *Te;        /* explicit planes       */
    double *uh, *du, *vh, *dv;   /* phase-A pseudo-velocities            */
    double *dxs, *dys;           /* per-column / per-row steps, NULL = uniform */
    level L3;                    /* loop 3 (N3): the previous T-p iterate of the pass */
    const level* it3;            /* the level the coupled T-p terms read: OLD, or &L3 */
};

#define N1 (&c->L[0])
#define OLD (&c->L[1])
#define NEW (&c->L[2])
/* The T-p coupled quantities of the energy and pressure equations (reading R41):
 * the old iterate in the GPU column, the previous loop-3 iterate in
 * the CPU column's loop 3. */
#define TP3 (c->it3 ? c->it3 : OLD)

/* ---------------------------------------------------------------- indices */
static int IC(const orc_case* c, int i, int j) { return j * c->nx + i; }
static int IU(const orc_case* c, int i, int j) { return j * (c->nx + 1) + i; }
static int IV(const orc_case* c, int i, int j) { return j * c->nx + i; }
static int wrap(int i, int n) { int r = i % n; return r < 0 ? r + n : r; }
static int periodic(const orc_case* c) { return c->P.xbc == ORC_X_PERIODIC; }
static int tvd(const orc_case* c) { return c->P.space_scheme == ORC_TVD; }
static int implicit_(const orc_case* c) { return c->P.time_scheme == ORC_IMPLICIT; }

/* Grid steps Delta x_i, Delta y_j (Fig. 5).  The mesh of the
 * paper's test case is uniform (the P.dx / P.dy default); orc_set_mesh
 * gives per-column / per-row steps (the general mesh of P:271-280, SURVEY
 * 8(f) N4).  A ghost column takes the step of the column it copies (inflow
 * ghosts: column 0, outflow ghosts: column nx-1, periodic: the wrapped
 * column); rows beyond a wall take the boundary row's step (no stencil that
 * is used reaches them: R17). */
static double DX(const orc_case* c, int i)
{
    if (!c->dxs) return c->P.dx;
    if (periodic(c)) return c->dxs[wrap(i, c->nx)];
    return c->dxs[i < 0 ? 0 : (i >= c->nx ? c->nx - 1 : i)];
}
static double DY(const orc_case* c, int j)
{
    if (!c->dys) return c->P.dy;
    return c->dys[j < 0 ? 0 : (j >= c->ny ? c->ny - 1 : j)];
}
/* Linear-interpolation weight of the node left of a face (reading R4): the
 * face between nodes of widths dl (left) and dr (right) lies dl/2 from the
 * left centre and dr/2 from the right one, so the left node weighs
 * dr / (dl + dr) and the right node dl / (dl + dr) (1/2 each on a uniform
 * mesh, exactly). */
static double wleft(double dl, double dr) { return dr / (dl + dr); }

/* ------------------------------------------------------------ scheme funcs */
/* Van Leer limiter psi(r) = (r+|r|)/(1+r); r <= 0 -> 0 (R6). */
double orc_vanleer(double r)
{
    if (!(r > 0.0)) return 0.0;
    return (r + fabs(r)) / (1.0 + r);
}

/* upwind(phi1, phi2, v), Eq. pl15_12; tie v = 0 -> phi2 (R7). */
double orc_upwind(double f1, double f2, double w) { return w > 0.0 ? f1 : f2; }

/* Reading R37: the ratio r of psi_s / psi_c has the difference phi3 - phi2
 * in its denominator; a difference at the rounding level of O(1)
 * nondimensional fields counts as zero (R6 extended), so a flat stencil
 * never yields an O(1) limiter value from rounding noise. */
static int flat(double f2, double f3)
{
    return fabs(f3 - f2) <= 1e-12 * (1.0 + fabs(f2) + fabs(f3));
}

/* psi_s, Eq. pl15_2, without the R37 flat-stencil guard; a zero
 * denominator gives 0 (R6). */
static double psi_s_raw(double f1, double f2, double f3, double f4,
                        double d1, double d2, double d3, double d4, double w)
{
    if (w > 0.0) {
        double den = (d1 + d2) * (f3 - f2);
        if (den == 0.0) return 0.0;
        double r = (d2 + d3) * (f2 - f1) / den;
        return d2 / (d2 + d3) * orc_vanleer(r);
    } else {
        double den = (d3 + d4) * (f3 - f2);
        if (den == 0.0) return 0.0;
        double r = (d2 + d3) * (f4 - f3) / den;
        return -d3 / (d2 + d3) * orc_vanleer(r);
    }
}

/* psi_c, Eq. pl15_1, without the R37 guard; zero denominator -> 0 (R6). */
static double psi_c_raw(double f1, double f2, double f3, double f4,
                        double d1, double d2, double d3, double w)
{
    if (w > 0.0) {
        double den = d1 * (f3 - f2);
        if (den == 0.0) return 0.0;
        return 0.5 * orc_vanleer(d2 * (f2 - f1) / den);
    } else {
        double den = d3 * (f3 - f2);
        if (den == 0.0) return 0.0;
        return -0.5 * orc_vanleer(d2 * (f4 - f3) / den);
    }
}

/* psi_s / psi_c of the method: the flat-stencil guard R37, then the limiter. */
double orc_psi_s(double f1, double f2, double f3, double f4,
                 double d1, double d2, double d3, double d4, double w)
{
    if (flat(f2, f3)) return 0.0;
    return psi_s_raw(f1, f2, f3, f4, d1, d2, d3, d4, w);
}
double orc_psi_c(double f1, double f2, double f3, double f4,
                 double d1, double d2, double d3, double w)
{
    if (flat(f2, f3)) return 0.0;
    return psi_c_raw(f1, f2, f3, f4, d1, d2, d3, w);
}
/* The case's limiter: R37 on, or off for the conditioning test (test hook). */
static double psi_s_c(const orc_case* c, double f1, double f2, double f3, double f4,
                      double d1, double d2, double d3, double d4, double w)
{
    return c->P.r37_off ? psi_s_raw(f1, f2, f3, f4, d1, d2, d3, d4, w)
                        : orc_psi_s(f1, f2, f3, f4, d1, d2, d3, d4, w);
}
static double psi_c_c(const orc_case* c, double f1, double f2, double f3, double f4,
                      double d1, double d2, double d3, double w)
{
    return c->P.r37_off ? psi_c_raw(f1, f2, f3, f4, d1, d2, d3, w)
                        : orc_psi_c(f1, f2, f3, f4, d1, d2, d3, w);
}

static double max0(double a) { return a > 0.0 ? a : 0.0; }

/* -------------------------------------------------------------- kinds */
static int cell_kind(const orc_case* c, int i, int j)
{
    if (j < 0 || j >= c->ny) return K_WALLY;
    if (periodic(c)) i = wrap(i, c->nx);
    else if (i < 0) return K_INLET;
    else if (i >= c->nx) return K_OUTLET;
    return c->solid[IC(c, i, j)] ? K_SOLID : K_FLUID;
}
static int is_fluid(const orc_case* c, int i, int j) { return cell_kind(c, i, j) == K_FLUID; }
static int is_wallish(const orc_case* c, int i, int j)
{
    int k = cell_kind(c, i, j);
    return k == K_SOLID || k == K_WALLY;
}

/* u-face (i,j) on x^f_i between cells (i-1,j),(i,j). */
static int ukind(const orc_case* c, int i, int j)
{
    if (j < 0 || j >= c->ny) return F_NONE;
    if (periodic(c)) {
        i = wrap(i, c->nx);
        return (is_fluid(c, i - 1, j) && is_fluid(c, i, j)) ? F_ACTIVE : F_FIXED0;
    }
    if (i < 0 || i > c->nx) return F_NONE;
    if (i == 0) return F_INLET;
    if (i == c->nx) return F_OUTLET;
    return (is_fluid(c, i - 1, j) && is_fluid(c, i, j)) ? F_ACTIVE : F_FIXED0;
}
/* v-face (i,j) on y^f_j between cells (i,j-1),(i,j). */
static int vkind(const orc_case* c, int i, int j)
{
    if (j < 0 || j > c->ny) return F_NONE;
    if (j == 0 || j == c->ny) return F_WALL;
    if (periodic(c)) i = wrap(i, c->nx);
    else if (i < 0 || i >= c->nx) return F_NONE;
    return (is_fluid(c, i, j - 1) && is_fluid(c, i, j)) ? F_ACTIVE : F_FIXED0;
}
static int flux_face_u(int k) { return k == F_ACTIVE || k == F_INLET || k == F_OUTLET; }

/* --------------------------------------------------------- field access */
enum { C_P, C_T, C_RHO, C_GAM };
/* Cell value phi_{i,j} at a level, with the ghost rules of BC spec 2-4. */
static double cell(const orc_case* c, const level* s, int f, int i, int j)
{
    int k = cell_kind(c, i, j);
    if (k == K_WALLY || k == K_SOLID) return NAN;      /* never read (BC spec) */
    if (k == K_INLET) {                                 /* inflow state, R12 */
        switch (f) {
        case C_P: return c->P.p_in;
        case C_T: return c->P.T_in;
        case C_RHO: return c->P.p_in / c->P.T_in;
        default: return sqrt(c->P.T_in);
        }
    }
    if (k == K_OUTLET) i = c->nx - 1;                   /* zero gradient */
    if (periodic(c)) i = wrap(i, c->nx);
    int id = IC(c, i, j);
    switch (f) {
    case C_P: return s->p[id];
    case C_T: return s->T[id];
    case C_RHO: return s->rho[id];
    default: return s->gam[id];
    }
}
#define RHO(s, i, j) cell(c, s, C_RHO, i, j)
#define TT(s, i, j) cell(c, s, C_T, i, j)
#define PP(s, i, j) cell(c, s, C_P, i, j)
#define GAM(s, i, j) cell(c, s, C_GAM, i, j)

/* u at face (i,j); beyond the channel walls the wall velocity (BC spec 8). */
static double U(const orc_case* c, const level* s, int i, int j)
{
    if (j < 0) return c->P.u_wall_bottom;
    if (j >= c->ny) return c->P.u_wall_top;
    if (periodic(c)) i = wrap(i, c->nx);
    else if (i < 0) return c->u_in;
    else if (i > c->nx) return NAN;
    return s->u[IU(c, i, j)];
}
/* v at face (i,j); inlet ghost v = 0, outlet ghost copies column nx-1. */
static double V(const orc_case* c, const level* s, int i, int j)
{
    if (j < 0 || j > c->ny) return NAN;
    if (periodic(c)) i = wrap(i, c->nx);
    else if (i < 0) return 0.0;
    else if (i >= c->nx) i = c->nx - 1;
    return s->v[IV(c, i, j)];
}

/* --------------------------------------------- TVD stencil validity (R17) */
static int cells_ok_x(const orc_case* c, int i0, int j)
{ for (int k = 0; k < 4; k++) if (!is_fluid(c, i0 + k, j)) return 0; return 1; }
static int cells_ok_y(const orc_case* c, int i, int j0)
{ for (int k = 0; k < 4; k++) if (!is_fluid(c, i, j0 + k)) return 0; return 1; }
static int ufaces_ok_x(const orc_case* c, int i0, int j)
{ for (int k = 0; k < 4; k++) if (ukind(c, i0 + k, j) != F_ACTIVE) return 0; return 1; }
static int ufaces_ok_y(const orc_case* c, int i, int j0)
{ for (int k = 0; k < 4; k++) if (ukind(c, i, j0 + k) != F_ACTIVE) return 0; return 1; }
static int vfaces_ok_x(const orc_case* c, int i0, int j)
{ for (int k = 0; k < 4; k++) if (vkind(c, i0 + k, j) != F_ACTIVE) return 0; return 1; }
static int vfaces_ok_y(const orc_case* c, int i, int j0)
{ for (int k = 0; k < 4; k++) if (vkind(c, i, j0 + k) != F_ACTIVE) return 0; return 1; }

/* psi_s of a cell-centred scalar (getter f) at u-face i (stencil i-2..i+1). */
static double psis_cell_x(const orc_case* c, const level* s, int f, int i, int j, double w)
{
    if (!tvd(c) || !cells_ok_x(c, i - 2, j)) return 0.0;
    return psi_s_c(c, cell(c, s, f, i - 2, j), cell(c, s, f, i - 1, j), cell(c, s, f, i, j),
                     cell(c, s, f, i + 1, j), DX(c, i - 2), DX(c, i - 1), DX(c, i), DX(c, i + 1), w);
}
/* psi_s of a cell-centred scalar at v-face j (stencil j-2..j+1). */
static double psis_cell_y(const orc_case* c, const level* s, int f, int i, int j, double w)
{
    if (!tvd(c) || !cells_ok_y(c, i, j - 2)) return 0.0;
    return psi_s_c(c, cell(c, s, f, i, j - 2), cell(c, s, f, i, j - 1), cell(c, s, f, i, j),
                     cell(c, s, f, i, j + 1), DY(c, j - 2), DY(c, j - 1), DY(c, j), DY(c, j + 1), w);
}

/* ------------------------------------- face densities, fluxes (pl8-pl11) */
/* rho^u_{i,j} = upwind(rho_{i-1,j}, rho_{i,j}, u_{i,j}) + psi_s (rho_{i,j}-rho_{i-1,j})
 * -- Eq. pl10 read as R1. */
static double rho_u(const orc_case* c, const level* s, int i, int j)
{
    double w = U(c, s, i, j);
    double r1 = RHO(s, i - 1, j), r2 = RHO(s, i, j);
    return orc_upwind(r1, r2, w) + psis_cell_x(c, s, C_RHO, i, j, w) * (r2 - r1);
}
/* rho^v_{i,j}, Eq. pl11 read as R1. */
static double rho_v(const orc_case* c, const level* s, int i, int j)
{
    double w = V(c, s, i, j);
    double r1 = RHO(s, i, j - 1), r2 = RHO(s, i, j);
    return orc_upwind(r1, r2, w) + psis_cell_y(c, s, C_RHO, i, j, w) * (r2 - r1);
}
/* F^x_{i,j} = rho^u u Delta y_j, Eq. pl8; 0 through fixed faces. */
static double Fx(const orc_case* c, const level* s, int i, int j)
{
    if (!flux_face_u(ukind(c, i, j))) return 0.0;
    return rho_u(c, s, i, j) * U(c, s, i, j) * DY(c, j);
}
/* F^y_{i,j} = rho^v v Delta x_i, Eq. pl9; 0 through walls. */
static double Fy(const orc_case* c, const level* s, int i, int j)
{
    if (vkind(c, i, j) != F_ACTIVE) return 0.0;
    return rho_v(c, s, i, j) * V(c, s, i, j) * DX(c, i);
}

/* Corner Gamma at (x^f_i, y^f_j): bilinear interpolation between the 4
 * surrounding cell centres (R4, R5; weights wx * wy of wleft, 1/4 each on a
 * uniform mesh), over the cells that are not solid and not beyond a wall,
 * the weights renormalised to the cells kept (BC spec 8).  On a uniform mesh
 * this is the mean of the cells kept, bit for bit (power-of-two weights). */
static double gam_corner(const orc_case* c, const level* s, int i, int j)
{
    const double wxl = wleft(DX(c, i - 1), DX(c, i)), wxr = 1.0 - wxl;
    const double wyb = wleft(DY(c, j - 1), DY(c, j)), wyt = 1.0 - wyb;
    double sum = 0.0, wsum = 0.0;
    int ii[4] = {i - 1, i, i - 1, i}, jj[4] = {j - 1, j - 1, j, j};
    double w[4] = {wxl * wyb, wxr * wyb, wxl * wyt, wxr * wyt};
    for (int k = 0; k < 4; k++)
        if (!is_wallish(c, ii[k], jj[k])) { sum += w[k] * GAM(s, ii[k], jj[k]); wsum += w[k]; }
    return sum / wsum;
}
/* Harmonic face average of Gamma^lambda, Eq. pl33. */
static double harmonic(double gm, double gp, double dm, double dp)
{
    return (dm + dp) * gm * gp / (dm * gp + dp * gm);
}

/* Slip / jump wall conductances (BC spec 5): Eq. pl38 with
 * zeta = 1.1466 Kn / rho_local, Eq. pl39 with tau = 2.1904 Kn/rho_local
 * (P:696), first-order one-sided normal derivative over dn. */
static double wall_D_mom(const orc_case* c, double gam_adj, double rho_adj, double L, double dn)
{
    double zeta = 1.1466 * c->P.Kn / rho_adj;
    return c->B * gam_adj * L / (dn + zeta);
}
static double wall_D_T(const orc_case* c, double gam_adj, double rho_adj, double L, double dn)
{
    double tau = 2.1904 * c->P.Kn / rho_adj;
    return c->CT1 * gam_adj * L / (dn + tau);
}
static double wall_T_of(const orc_case* c, int i, int j)
{
    return cell_kind(c, i, j) == K_WALLY ? c->P.T_wall : c->P.T_square;
}

/* Face value of a cell-centred scalar on the face between cells a (width da)
 * and b (width db): linear interpolation between the two centres. */
static double face_interp(double fa, double fb, double da, double db)
{
    return (db * fa + da * fb) / (da + db);
}

/* Pressure work of S^T_c per unit volume, reading R9.
 * The continuum energy equation is the enthalpy form with +C^T3 Dp/Dt
 * (Eq. pl6; C^T1, C^T2, C^T3 = (gamma-1)/gamma of Eq. pl37 are its
 * c_p-form coefficients), the printed discrete source is +C^T3 p div(u)
 * (Eq. pl29).  Default ORC_PW_DPDT discretises the continuum term at
 * the old iterate, as the rest of S^T_c:
 *   C^T3 [ (p_{i,j} - p^{n-1}_{i,j}) / dt
 *          + ubar_{i,j} (p_e - p_w) / dx_i + vbar_{i,j} (p_n - p_s) / dy_j ],
 * ubar = (u_{i,j} + u_{i+1,j}) / 2, vbar = (v_{i,j} + v_{i,j+1}) / 2, p_e the
 * face value between cells i and i+1 (linear interpolation), p_e = p_{i,j}
 * when the neighbour is solid or beyond a wall (dp/dn = 0 at a wall, no flow
 * through it); likewise p_w, p_n, p_s.  The other forms are kappa p div(u)
 * with kappa = +C^T3 (as printed), -C^T3 (round-1 reading) or -gamma C^T3. */
static double pressure_work(const orc_case* c, int i, int j, double div)
{
    const level* o = OLD;
    const level* q = TP3;                          /* pressure of the T-p iterate (R41) */
    const double pc = PP(q, i, j);
    if (c->P.pw_form != ORC_PW_DPDT) return c->PWK * pc * div;
    const double dx = DX(c, i), dy = DY(c, j);
    double pe = is_wallish(c, i + 1, j) ? pc : face_interp(pc, PP(q, i + 1, j), dx, DX(c, i + 1));
    double pw = is_wallish(c, i - 1, j) ? pc : face_interp(PP(q, i - 1, j), pc, DX(c, i - 1), dx);
    double pn = is_wallish(c, i, j + 1) ? pc : face_interp(pc, PP(q, i, j + 1), dy, DY(c, j + 1));
    double ps = is_wallish(c, i, j - 1) ? pc : face_interp(PP(q, i, j - 1), pc, DY(c, j - 1), dy);
    double ub = 0.5 * (U(c, o, i, j) + U(c, o, i + 1, j));
    double vb = 0.5 * (V(c, o, i, j) + V(c, o, i, j + 1));
    double dpdt = (pc - PP(N1, i, j)) / c->P.dt;
    return c->CT3 * (dpdt + ub * (pe - pw) / dx + vb * (pn - ps) / dy);
}

/* Tangential wall velocity u_w of the wall cell (i, j): the channel walls
 * move (BC spec 6, R14), the squares are at rest (R15). */
static double wall_u_of(const orc_case* c, int i, int j)
{
    (void)i;
    if (cell_kind(c, i, j) == K_WALLY) return j < 0 ? c->P.u_wall_bottom : c->P.u_wall_top;
    return 0.0;
}
/* Gas velocity at a wall surface from the slip condition Eq. pl38,
 * v_s - v_w = zeta (v_P - v_s) / dn, zeta = 1.1466 Kn / rho_local:
 * v_s = (dn v_w + zeta v_P) / (dn + zeta); v_P = tangential velocity at the
 * centre of the wall-adjacent cell, dn = half its width (reading R38). */
static double slip_velocity(const orc_case* c, double vP, double vw, double rho, double dn)
{
    double zeta = 1.1466 * c->P.Kn / rho;
    return (dn * vw + zeta * vP) / (dn + zeta);
}

/* ===================================================== phase A: energy */
/* Temperature at fluid cell (i,j): Eqs. pl30-pl33, pl28-pl29, pl31_1
 * (P:432-498).  Returns T_{i,j} of this pass. */
static double T_equation(const orc_case* c, int i, int j)
{
    const level* o = OLD;
    const level* n1 = N1;
    const int impl = implicit_(c);
    const double dx = DX(c, i), dy = DY(c, j), dt = c->P.dt;
    const level* q = TP3;                       /* T-p coupled values (R41): old iterate, or loop 3 */
    const double gP = GAM(o, i, j), rP = RHO(o, i, j);
    double a1, a2, a3, a4, T1, T2, T3, T4;
    double FW = 0, FE = 0, FS = 0, FN = 0;

    /* a^T_1: west (Eq. pl31 line 2, D^Tx_{i,j} Eq. pl32) */
    if (is_wallish(c, i - 1, j)) {
        a1 = wall_D_T(c, gP, rP, dy, 0.5 * dx); T1 = wall_T_of(c, i - 1, j);
    } else {
        FW = Fx(c, o, i, j);
        double D = c->CT1 * harmonic(GAM(o, i - 1, j), gP, DX(c, i - 1), dx) * dy / (0.5 * (dx + DX(c, i - 1)));
        a1 = (impl ? max0(FW) - FW * psis_cell_x(c, o, C_T, i, j, U(c, o, i, j)) : 0.0) + D;
        T1 = TT(q, i - 1, j);
    }
    /* a^T_2: east, D^Tx_{i+1,j} */
    if (is_wallish(c, i + 1, j)) {
        a2 = wall_D_T(c, gP, rP, dy, 0.5 * dx); T2 = wall_T_of(c, i + 1, j);
    } else {
        FE = Fx(c, o, i + 1, j);
        double D = c->CT1 * harmonic(gP, GAM(o, i + 1, j), dx, DX(c, i + 1)) * dy / (0.5 * (DX(c, i + 1) + dx));
        a2 = (impl ? max0(-FE) - FE * psis_cell_x(c, o, C_T, i + 1, j, U(c, o, i + 1, j)) : 0.0) + D;
        T2 = TT(q, i + 1, j);
    }
    /* a^T_3: south, D^Ty_{i,j} */
    if (is_wallish(c, i, j - 1)) {
        a3 = wall_D_T(c, gP, rP, dx, 0.5 * dy); T3 = wall_T_of(c, i, j - 1);
    } else {
        FS = Fy(c, o, i, j);
        double D = c->CT1 * harmonic(GAM(o, i, j - 1), gP, DY(c, j - 1), dy) * dx / (0.5 * (dy + DY(c, j - 1)));
        a3 = (impl ? max0(FS) - FS * psis_cell_y(c, o, C_T, i, j, V(c, o, i, j)) : 0.0) + D;
        T3 = TT(q, i, j - 1);
    }
    /* a^T_4: north, D^Ty_{i,j+1} */
    if (is_wallish(c, i, j + 1)) {
        a4 = wall_D_T(c, gP, rP, dx, 0.5 * dy); T4 = wall_T_of(c, i, j + 1);
    } else {
        FN = Fy(c, o, i, j + 1);
        double D = c->CT1 * harmonic(gP, GAM(o, i, j + 1), dy, DY(c, j + 1)) * dx / (0.5 * (DY(c, j + 1) + dy));
        a4 = (impl ? max0(-FN) - FN * psis_cell_y(c, o, C_T, i, j + 1, V(c, o, i, j + 1)) : 0.0) + D;
        T4 = TT(q, i, j + 1);
    }

    double a0;
    const double rq = RHO(q, i, j);             /* rho of the unsteady term: p/T of the T-p iterate */
    if (impl) a0 = dt * (a1 + a2 + a3 + a4 + FE - FW + FN - FS) + rq * dx * dy;   /* pl31 */
    else      a0 = dt * (a1 + a2 + a3 + a4) + rq * dx * dy;                       /* pl31_1 */

    /* S^T_c, Eq. pl29; mid-face velocities by bilinear
     * interpolation between the four neighbouring nodes (R4): the face
     * x^f_{i+1} lies between the v-node columns i and i+1 (weights wleft) and
     * y^v_j halfway between the v-node rows j and j+1 (1/2 each); likewise
     * for u.  Terms summed in node order: on a uniform mesh this is the
     * 4-point mean 0.25 (a + b + c + d) bit for bit. */
    double dudx = (U(c, o, i + 1, j) - U(c, o, i, j)) / dx;
    double dvdy = (V(c, o, i, j + 1) - V(c, o, i, j)) / dy;
    double wE = wleft(dx, DX(c, i + 1)), wW = wleft(DX(c, i - 1), dx);
    double wN = wleft(dy, DY(c, j + 1)), wS = wleft(DY(c, j - 1), dy);
    double vE = 0.5 * wE * V(c, o, i, j) + 0.5 * (1.0 - wE) * V(c, o, i + 1, j)
              + 0.5 * wE * V(c, o, i, j + 1) + 0.5 * (1.0 - wE) * V(c, o, i + 1, j + 1);
    double vW = 0.5 * wW * V(c, o, i - 1, j) + 0.5 * (1.0 - wW) * V(c, o, i, j)
              + 0.5 * wW * V(c, o, i - 1, j + 1) + 0.5 * (1.0 - wW) * V(c, o, i, j + 1);
    double uN = 0.5 * wN * U(c, o, i, j) + 0.5 * wN * U(c, o, i + 1, j)
              + 0.5 * (1.0 - wN) * U(c, o, i, j + 1) + 0.5 * (1.0 - wN) * U(c, o, i + 1, j + 1);
    double uS = 0.5 * wS * U(c, o, i, j - 1) + 0.5 * wS * U(c, o, i + 1, j - 1)
              + 0.5 * (1.0 - wS) * U(c, o, i, j) + 0.5 * (1.0 - wS) * U(c, o, i + 1, j);
    /* A mid-face velocity on a face that lies on a wall is the gas velocity at
     * the surface: the slip velocity of Eq. pl38 (reading R38) */
    if (is_wallish(c, i + 1, j)) vE = slip_velocity(c, 0.5 * (V(c, o, i, j) + V(c, o, i, j + 1)), 0.0, rP, 0.5 * dx);
    if (is_wallish(c, i - 1, j)) vW = slip_velocity(c, 0.5 * (V(c, o, i, j) + V(c, o, i, j + 1)), 0.0, rP, 0.5 * dx);
    if (is_wallish(c, i, j + 1))
        uN = slip_velocity(c, 0.5 * (U(c, o, i, j) + U(c, o, i + 1, j)), wall_u_of(c, i, j + 1), rP, 0.5 * dy);
    if (is_wallish(c, i, j - 1))
        uS = slip_velocity(c, 0.5 * (U(c, o, i, j) + U(c, o, i + 1, j)), wall_u_of(c, i, j - 1), rP, 0.5 * dy);
    double shear = (vE - vW) / dx + (uN - uS) / dy;
    double div = dudx + dvdy;
    double Sc = c->CT2 * gP * (2.0 * (dudx * dudx + dvdy * dvdy) + shear * shear - 2.0 / 3.0 * div * div) * dx * dy
              + pressure_work(c, i, j, div) * dx * dy;

    double Texp = impl ? 0.0 : c->Te[IC(c, i, j)];
    double rhs = dt * (a1 * T1 + a2 * T2 + a3 * T3 + a4 * T4 + Sc + Texp)
               + RHO(n1, i, j) * TT(n1, i, j) * dx * dy;                              /* pl30 */
    return rhs / a0;
}

/* ============================================ phase A: u pseudo-velocity */
/* u-hat_{i,j}, d^u_{i,j} at an active u-face: Eq. pl20 with the
 * coefficients of Eqs. pl14-pl16 / pl15_11 transposed x<->y (DESIGN 3.4). */
static void u_equation(const orc_case* c, int i, int j, double* uhat, double* du)
{
    const level* o = OLD;
    const level* n1 = N1;
    const int impl = implicit_(c);
    const double dxL = DX(c, i - 1), dxR = DX(c, i), dy = DY(c, j), dt = c->P.dt;
    const double rL = RHO(o, i - 1, j), rR = RHO(o, i, j);
    const double gL = GAM(o, i - 1, j), gR = GAM(o, i, j);
    double a1, a2, a3, a4, uW, uE, uS, uN;
    double FbW, FbE, Fs_i = 0, Fs_im1 = 0, Fn_i = 0, Fn_im1 = 0;

    /* normal links: F-bar^x at cell centres (R2 transposed) */
    double ubW = 0.5 * (U(c, o, i - 1, j) + U(c, o, i, j));
    double ubE = 0.5 * (U(c, o, i, j) + U(c, o, i + 1, j));
    FbW = rL * ubW * dy;
    FbE = rR * ubE * dy;
    double Dux_i = c->B * gL * dy / dxL;          /* D^ux_{i,j}   = B Gamma_{i-1,j} dy_j / dx_{i-1} */
    double Dux_ip1 = c->B * gR * dy / dxR;        /* D^ux_{i+1,j} = B Gamma_{i,j} dy_j / dx_i       */
    double psW = 0, psE = 0;
    if (impl && tvd(c)) {
        if (ufaces_ok_x(c, i - 2, j))
            psW = psi_c_c(c, U(c, o, i - 2, j), U(c, o, i - 1, j), U(c, o, i, j), U(c, o, i + 1, j),
                            DX(c, i - 2), DX(c, i - 1), DX(c, i), ubW);
        if (ufaces_ok_x(c, i - 1, j))
            psE = psi_c_c(c, U(c, o, i - 1, j), U(c, o, i, j), U(c, o, i + 1, j), U(c, o, i + 2, j),
                            DX(c, i - 1), DX(c, i), DX(c, i + 1), ubE);
    }
    a1 = (impl ? max0(FbW) - FbW * psW : 0.0) + 4.0 / 3.0 * Dux_i;
    a2 = (impl ? max0(-FbE) - FbE * psE : 0.0) + 4.0 / 3.0 * Dux_ip1;
    uW = U(c, o, i - 1, j);
    uE = U(c, o, i + 1, j);

    /* tangential south link (a^u_3) */
    if (j - 1 < 0 || (cell_kind(c, i - 1, j - 1) == K_SOLID && cell_kind(c, i, j - 1) == K_SOLID)) {
        a3 = wall_D_mom(c, 0.5 * (gL + gR), 0.5 * (rL + rR), 0.5 * (dxL + dxR), 0.5 * dy);
        uS = (j - 1 < 0) ? c->P.u_wall_bottom : 0.0;
    } else {
        Fs_i = Fy(c, o, i, j);
        Fs_im1 = Fy(c, o, i - 1, j);
        double p1 = 0, p2 = 0;
        if (impl && tvd(c) && ufaces_ok_y(c, i, j - 2)) {
            double f1 = U(c, o, i, j - 2), f2 = U(c, o, i, j - 1), f3 = U(c, o, i, j), f4 = U(c, o, i, j + 1);
            p1 = psi_s_c(c, f1, f2, f3, f4, DY(c, j - 2), DY(c, j - 1), DY(c, j), DY(c, j + 1), V(c, o, i, j));
            p2 = psi_s_c(c, f1, f2, f3, f4, DY(c, j - 2), DY(c, j - 1), DY(c, j), DY(c, j + 1), V(c, o, i - 1, j));
        }
        double Duy = c->B * gam_corner(c, o, i, j) * (dxR + dxL) / (dy + DY(c, j - 1));
        a3 = (impl ? 0.5 * (max0(Fs_i) - Fs_i * p1 + max0(Fs_im1) - Fs_im1 * p2) : 0.0) + Duy;
        uS = U(c, o, i, j - 1);
    }
    /* tangential north link (a^u_4) */
    if (j + 1 >= c->ny || (cell_kind(c, i - 1, j + 1) == K_SOLID && cell_kind(c, i, j + 1) == K_SOLID)) {
        a4 = wall_D_mom(c, 0.5 * (gL + gR), 0.5 * (rL + rR), 0.5 * (dxL + dxR), 0.5 * dy);
        uN = (j + 1 >= c->ny) ? c->P.u_wall_top : 0.0;
    } else {
        Fn_i = Fy(c, o, i, j + 1);
        Fn_im1 = Fy(c, o, i - 1, j + 1);
        double p1 = 0, p2 = 0;
        if (impl && tvd(c) && ufaces_ok_y(c, i, j - 1)) {
            double f1 = U(c, o, i, j - 1), f2 = U(c, o, i, j), f3 = U(c, o, i, j + 1), f4 = U(c, o, i, j + 2);
            p1 = psi_s_c(c, f1, f2, f3, f4, DY(c, j - 1), DY(c, j), DY(c, j + 1), DY(c, j + 2), V(c, o, i, j + 1));
            p2 = psi_s_c(c, f1, f2, f3, f4, DY(c, j - 1), DY(c, j), DY(c, j + 1), DY(c, j + 2), V(c, o, i - 1, j + 1));
        }
        double Duy = c->B * gam_corner(c, o, i, j + 1) * (dxR + dxL) / (DY(c, j + 1) + dy);
        a4 = (impl ? 0.5 * (max0(-Fn_i) - Fn_i * p1 + max0(-Fn_im1) - Fn_im1 * p2) : 0.0) + Duy;
        uN = U(c, o, i, j + 1);
    }

    double tterm = (rR * dxR + rL * dxL) * dy / (2.0 * dt);
    double a0;
    if (impl) a0 = a1 + a2 + a3 + a4 + FbE - FbW + 0.5 * (Fn_i - Fs_i + Fn_im1 - Fs_im1) + tterm;
    else      a0 = a1 + a2 + a3 + a4 + tterm;

    /* b^u: transposition of b^v (Eq. pl14) + body force (R22) */
    double prT = PP(n1, i, j) / TT(n1, i, j), prTL = PP(n1, i - 1, j) / TT(n1, i - 1, j);
    double b = (prT * dxR + prTL * dxL) * dy / (2.0 * dt) * n1->u[IU(c, periodic(c) ? wrap(i, c->nx) : i, j)]
             + c->B * (gam_corner(c, o, i, j + 1) * (V(c, o, i, j + 1) - V(c, o, i - 1, j + 1))
                       - gam_corner(c, o, i, j) * (V(c, o, i, j) - V(c, o, i - 1, j))
                       - 2.0 / 3.0 * gR * (V(c, o, i, j + 1) - V(c, o, i, j))
                       + 2.0 / 3.0 * gL * (V(c, o, i - 1, j + 1) - V(c, o, i - 1, j)))
             + c->P.g_x * 0.5 * (rR * dxR + rL * dxL) * dy;

    double uexp = impl ? 0.0 : c->ue[IU(c, periodic(c) ? wrap(i, c->nx) : i, j)];
    *uhat = (a1 * uW + a2 * uE + a3 * uS + a4 * uN + b + uexp) / a0;
    *du = c->A * dy / a0;
}

/* ============================================ phase A: v pseudo-velocity */
/* v-hat_{i,j}, d^v_{i,j} at an active v-face: Eqs. pl14-pl16, pl21, pl15_11
 * with the F-bar / v-bar reading R2. */
static void v_equation(const orc_case* c, int i, int j, double* vhat, double* dv)
{
    const level* o = OLD;
    const level* n1 = N1;
    const int impl = implicit_(c);
    const double dyB = DY(c, j - 1), dyT = DY(c, j), dx = DX(c, i), dt = c->P.dt;
    const double rB = RHO(o, i, j - 1), rT = RHO(o, i, j);
    const double gB = GAM(o, i, j - 1), gT = GAM(o, i, j);
    double a1, a2, a3, a4, vW, vE, vS, vN;
    double Fw_j = 0, Fw_jm1 = 0, Fe_j = 0, Fe_jm1 = 0;

    /* normal links (y): F-bar^y on cell centres (R2) */
    double vbS = 0.5 * (V(c, o, i, j - 1) + V(c, o, i, j));
    double vbN = 0.5 * (V(c, o, i, j) + V(c, o, i, j + 1));
    double FbS = rB * vbS * dx;
    double FbN = rT * vbN * dx;
    double Dvy_j = c->B * gB * dx / dyB;          /* D^vy_{i,j},   Eq. pl16 */
    double Dvy_jp1 = c->B * gT * dx / dyT;        /* D^vy_{i,j+1}          */
    double psS = 0, psN = 0;
    if (impl && tvd(c)) {
        if (vfaces_ok_y(c, i, j - 2))
            psS = psi_c_c(c, V(c, o, i, j - 2), V(c, o, i, j - 1), V(c, o, i, j), V(c, o, i, j + 1),
                            DY(c, j - 2), DY(c, j - 1), DY(c, j), vbS);
        if (vfaces_ok_y(c, i, j - 1))
            psN = psi_c_c(c, V(c, o, i, j - 1), V(c, o, i, j), V(c, o, i, j + 1), V(c, o, i, j + 2),
                            DY(c, j - 1), DY(c, j), DY(c, j + 1), vbN);
    }
    a3 = (impl ? max0(FbS) - FbS * psS : 0.0) + 4.0 / 3.0 * Dvy_j;      /* a^vc_3 + 4/3 D^vy */
    a4 = (impl ? max0(-FbN) - FbN * psN : 0.0) + 4.0 / 3.0 * Dvy_jp1;   /* a^vc_4 + 4/3 D^vy */
    vS = V(c, o, i, j - 1);
    vN = V(c, o, i, j + 1);

    /* tangential west link (a^v_1) */
    if (cell_kind(c, i - 1, j - 1) == K_SOLID && cell_kind(c, i - 1, j) == K_SOLID) {
        a1 = wall_D_mom(c, 0.5 * (gB + gT), 0.5 * (rB + rT), 0.5 * (dyB + dyT), 0.5 * dx);
        vW = 0.0;
    } else {
        Fw_j = Fx(c, o, i, j);
        Fw_jm1 = Fx(c, o, i, j - 1);
        double p1 = 0, p2 = 0;
        if (impl && tvd(c) && vfaces_ok_x(c, i - 2, j)) {
            double f1 = V(c, o, i - 2, j), f2 = V(c, o, i - 1, j), f3 = V(c, o, i, j), f4 = V(c, o, i + 1, j);
            p1 = psi_s_c(c, f1, f2, f3, f4, DX(c, i - 2), DX(c, i - 1), DX(c, i), DX(c, i + 1), U(c, o, i, j));
            p2 = psi_s_c(c, f1, f2, f3, f4, DX(c, i - 2), DX(c, i - 1), DX(c, i), DX(c, i + 1), U(c, o, i, j - 1));
        }
        double Dvx = c->B * gam_corner(c, o, i, j) * (dyT + dyB) / (dx + DX(c, i - 1));
        a1 = (impl ? 0.5 * (max0(Fw_j) - Fw_j * p1 + max0(Fw_jm1) - Fw_jm1 * p2) : 0.0) + Dvx;
        vW = V(c, o, i - 1, j);
    }
    /* tangential east link (a^v_2) */
    if (cell_kind(c, i + 1, j - 1) == K_SOLID && cell_kind(c, i + 1, j) == K_SOLID) {
        a2 = wall_D_mom(c, 0.5 * (gB + gT), 0.5 * (rB + rT), 0.5 * (dyB + dyT), 0.5 * dx);
        vE = 0.0;
    } else {
        Fe_j = Fx(c, o, i + 1, j);
        Fe_jm1 = Fx(c, o, i + 1, j - 1);
        double p1 = 0, p2 = 0;
        if (impl && tvd(c) && vfaces_ok_x(c, i - 1, j)) {
            double f1 = V(c, o, i - 1, j), f2 = V(c, o, i, j), f3 = V(c, o, i + 1, j), f4 = V(c, o, i + 2, j);
            p1 = psi_s_c(c, f1, f2, f3, f4, DX(c, i - 1), DX(c, i), DX(c, i + 1), DX(c, i + 2), U(c, o, i + 1, j));
            p2 = psi_s_c(c, f1, f2, f3, f4, DX(c, i - 1), DX(c, i), DX(c, i + 1), DX(c, i + 2), U(c, o, i + 1, j - 1));
        }
        double Dvx = c->B * gam_corner(c, o, i + 1, j) * (dyT + dyB) / (DX(c, i + 1) + dx);
        a2 = (impl ? 0.5 * (max0(-Fe_j) - Fe_j * p1 + max0(-Fe_jm1) - Fe_jm1 * p2) : 0.0) + Dvx;
        vE = V(c, o, i + 1, j);
    }

    double tterm = (rT * dyT + rB * dyB) * dx / (2.0 * dt);
    double a0;
    if (impl) a0 = a1 + a2 + a3 + a4 + 0.5 * (Fe_j - Fw_j + Fe_jm1 - Fw_jm1) + FbN - FbS + tterm;  /* pl15 */
    else      a0 = a1 + a2 + a3 + a4 + tterm;                                                    /* pl15_11 */

    /* b^v, Eq. pl14 + body force (R22) */
    double prT = PP(n1, i, j) / TT(n1, i, j), prTB = PP(n1, i, j - 1) / TT(n1, i, j - 1);
    int ii = periodic(c) ? wrap(i, c->nx) : i;
    double b = (prT * dyT + prTB * dyB) * dx / (2.0 * dt) * n1->v[IV(c, ii, j)]
             + c->B * (gam_corner(c, o, i + 1, j) * (U(c, o, i + 1, j) - U(c, o, i + 1, j - 1))
                       - gam_corner(c, o, i, j) * (U(c, o, i, j) - U(c, o, i, j - 1))
                       - 2.0 / 3.0 * gT * (U(c, o, i + 1, j) - U(c, o, i, j))
                       + 2.0 / 3.0 * gB * (U(c, o, i + 1, j - 1) - U(c, o, i, j - 1)))
             + c->P.g_y * 0.5 * (rT * dyT + rB * dyB) * dx;

    double vexp = impl ? 0.0 : c->ve[IV(c, ii, j)];
    *vhat = (a1 * vW + a2 * vE + a3 * vS + a4 * vN + b + vexp) / a0;   /* pl21 */
    *dv = c->A * dx / a0;                                                  /* pl14 */
}

/* ============================================ explicit planes (a1 row) */
/* T^explicit_{i,j}, Eq. pl31_1, at time level n-1. */
static double T_explicit(const orc_case* c, int i, int j)
{
    const level* s = N1;
    double e = 0.0;
    if (flux_face_u(ukind(c, i + 1, j))) {
        double F = Fx(c, s, i + 1, j), w = U(c, s, i + 1, j);
        double Ti = TT(s, i, j), Tp = TT(s, i + 1, j);
        e += -F * (orc_upwind(Ti, Tp, w) + (Tp - Ti) * psis_cell_x(c, s, C_T, i + 1, j, w));
    }
    if (flux_face_u(ukind(c, i, j))) {
        double F = Fx(c, s, i, j), w = U(c, s, i, j);
        double Tm = TT(s, i - 1, j), Ti = TT(s, i, j);
        e += F * (orc_upwind(Tm, Ti, w) + (Ti - Tm) * psis_cell_x(c, s, C_T, i, j, w));
    }
    if (vkind(c, i, j + 1) == F_ACTIVE) {
        double F = Fy(c, s, i, j + 1), w = V(c, s, i, j + 1);
        double Tj = TT(s, i, j), Tp = TT(s, i, j + 1);
        e += -F * (orc_upwind(Tj, Tp, w) + (Tp - Tj) * psis_cell_y(c, s, C_T, i, j + 1, w));
    }
    if (vkind(c, i, j) == F_ACTIVE) {
        double F = Fy(c, s, i, j), w = V(c, s, i, j);
        double Tm = TT(s, i, j - 1), Tj = TT(s, i, j);
        e += F * (orc_upwind(Tm, Tj, w) + (Tj - Tm) * psis_cell_y(c, s, C_T, i, j, w));
    }
    return e;
}

/* v^explicit_{i,j}, Eq. pl15_11 with R2, at time level n-1. */
static double v_explicit(const orc_case* c, int i, int j)
{
    const level* s = N1;
    const int tv = tvd(c);
    double e = 0.0;
    double vi = V(c, s, i, j);
    /* east half-faces: -0.5 [F^x_{i+1,j-1}(...) + F^x_{i+1,j}(...)] */
    {
        double vp = V(c, s, i + 1, j);
        int ok = tv && vfaces_ok_x(c, i - 1, j);
        double sum = 0.0;
        for (int h = 0; h < 2; h++) {
            int jj = (h == 0) ? j - 1 : j;
            if (!flux_face_u(ukind(c, i + 1, jj))) continue;
            double F = Fx(c, s, i + 1, jj), w = U(c, s, i + 1, jj);
            double ps = ok ? psi_s_c(c, V(c, s, i - 1, j), vi, vp, V(c, s, i + 2, j),
                                       DX(c, i - 1), DX(c, i), DX(c, i + 1), DX(c, i + 2), w) : 0.0;
            sum += F * (orc_upwind(vi, vp, w) + (vp - vi) * ps);
        }
        e += -0.5 * sum;
    }
    /* west half-faces: +0.5 [F^x_{i,j-1}(...) + F^x_{i,j}(...)] */
    {
        double vm = V(c, s, i - 1, j);
        int ok = tv && vfaces_ok_x(c, i - 2, j);
        double sum = 0.0;
        for (int h = 0; h < 2; h++) {
            int jj = (h == 0) ? j - 1 : j;
            if (!flux_face_u(ukind(c, i, jj))) continue;
            double F = Fx(c, s, i, jj), w = U(c, s, i, jj);
            double ps = ok ? psi_s_c(c, V(c, s, i - 2, j), vm, vi, V(c, s, i + 1, j),
                                       DX(c, i - 2), DX(c, i - 1), DX(c, i), DX(c, i + 1), w) : 0.0;
            sum += F * (orc_upwind(vm, vi, w) + (vi - vm) * ps);
        }
        e += 0.5 * sum;
    }
    /* north: - dx_i rho_{i,j} vbar_N [upwind(v_j, v_{j+1}, vbar_N) + (v_{j+1}-v_j) psi_c] */
    {
        double vp = V(c, s, i, j + 1);
        double vb = 0.5 * (vi + vp);
        double ps = (tv && vfaces_ok_y(c, i, j - 1))
                  ? psi_c_c(c, V(c, s, i, j - 1), vi, vp, V(c, s, i, j + 2), DY(c, j - 1), DY(c, j), DY(c, j + 1), vb) : 0.0;
        e += -DX(c, i) * RHO(s, i, j) * vb * (orc_upwind(vi, vp, vb) + (vp - vi) * ps);
    }
    /* south: + dx_i rho_{i,j-1} vbar_S [upwind(v_{j-1}, v_j, vbar_S) + (v_j - v_{j-1}) psi_c] */
    {
        double vm = V(c, s, i, j - 1);
        double vb = 0.5 * (vm + vi);
        double ps = (tv && vfaces_ok_y(c, i, j - 2))
                  ? psi_c_c(c, V(c, s, i, j - 2), vm, vi, V(c, s, i, j + 1), DY(c, j - 2), DY(c, j - 1), DY(c, j), vb) : 0.0;
        e += DX(c, i) * RHO(s, i, j - 1) * vb * (orc_upwind(vm, vi, vb) + (vi - vm) * ps);
    }
    return e;
}

/* u^explicit_{i,j}: transposition of v^explicit (DESIGN 3.4). */
static double u_explicit(const orc_case* c, int i, int j)
{
    const level* s = N1;
    const int tv = tvd(c);
    double e = 0.0;
    double ui = U(c, s, i, j);
    /* north half-faces: -0.5 [F^y_{i-1,j+1}(...) + F^y_{i,j+1}(...)] */
    {
        double up = U(c, s, i, j + 1);
        int ok = tv && ufaces_ok_y(c, i, j - 1);
        double sum = 0.0;
        for (int h = 0; h < 2; h++) {
            int ii = (h == 0) ? i - 1 : i;
            if (vkind(c, ii, j + 1) != F_ACTIVE) continue;
            double F = Fy(c, s, ii, j + 1), w = V(c, s, ii, j + 1);
            double ps = ok ? psi_s_c(c, U(c, s, i, j - 1), ui, up, U(c, s, i, j + 2),
                                       DY(c, j - 1), DY(c, j), DY(c, j + 1), DY(c, j + 2), w) : 0.0;
            sum += F * (orc_upwind(ui, up, w) + (up - ui) * ps);
        }
        e += -0.5 * sum;
    }
    /* south half-faces: +0.5 [F^y_{i-1,j}(...) + F^y_{i,j}(...)] */
    {
        double um = U(c, s, i, j - 1);
        int ok = tv && ufaces_ok_y(c, i, j - 2);
        double sum = 0.0;
        for (int h = 0; h < 2; h++) {
            int ii = (h == 0) ? i - 1 : i;
            if (vkind(c, ii, j) != F_ACTIVE) continue;
            double F = Fy(c, s, ii, j), w = V(c, s, ii, j);
            double ps = ok ? psi_s_c(c, U(c, s, i, j - 2), um, ui, U(c, s, i, j + 1),
                                       DY(c, j - 2), DY(c, j - 1), DY(c, j), DY(c, j + 1), w) : 0.0;
            sum += F * (orc_upwind(um, ui, w) + (ui - um) * ps);
        }
        e += 0.5 * sum;
    }
    /* east: - dy_j rho_{i,j} ubar_E [...] */
    {
        double up = U(c, s, i + 1, j);
        double ub = 0.5 * (ui + up);
        double ps = (tv && ufaces_ok_x(c, i - 1, j))
                  ? psi_c_c(c, U(c, s, i - 1, j), ui, up, U(c, s, i + 2, j), DX(c, i - 1), DX(c, i), DX(c, i + 1), ub) : 0.0;
        e += -DY(c, j) * RHO(s, i, j) * ub * (orc_upwind(ui, up, ub) + (up - ui) * ps);
    }
    /* west: + dy_j rho_{i-1,j} ubar_W [...] */
    {
        double um = U(c, s, i - 1, j);
        double ub = 0.5 * (um + ui);
        double ps = (tv && ufaces_ok_x(c, i - 2, j))
                  ? psi_c_c(c, U(c, s, i - 2, j), um, ui, U(c, s, i + 1, j), DX(c, i - 2), DX(c, i - 1), DX(c, i), ub) : 0.0;
        e += DY(c, j) * RHO(s, i - 1, j) * ub * (orc_upwind(um, ui, ub) + (ui - um) * ps);
    }
    return e;
}

static void compute_explicit_planes(orc_case* c)
{
    const int nx = c->nx, ny = c->ny;
    for (int j = 0; j < ny; j++)
        for (int i = 0; i < nx; i++)
            c->Te[IC(c, i, j)] = is_fluid(c, i, j) ? T_explicit(c, i, j) : 0.0;
    for (int j = 0; j < ny; j++)
        for (int i = 0; i <= nx; i++)
            c->ue[IU(c, i, j)] = (ukind(c, i, j) == F_ACTIVE && !(periodic(c) && i == nx)) ? u_explicit(c, i, j) : 0.0;
    for (int j = 0; j <= ny; j++)
        for (int i = 0; i < nx; i++)
            c->ve[IV(c, i, j)] = vkind(c, i, j) == F_ACTIVE ? v_explicit(c, i, j) : 0.0;
}

/* ================================================ phase B: pressure */
/* p_{i,j}, Eqs. pl23-pl24, T of this pass (R28). */
static double p_equation(const orc_case* c, int i, int j)
{
    const level* o = OLD;
    const level* n1 = N1;
    const level* nw = NEW;
    const double dx = DX(c, i), dy = DY(c, j), dt = c->P.dt;
    double apW = 0, apE = 0, apS = 0, apN = 0, bpW = 0, bpE = 0, bpS = 0, bpN = 0;
    int nxu = c->nx + 1;
    int iw = periodic(c) ? wrap(i, c->nx) : i, ie = periodic(c) ? wrap(i + 1, c->nx) : i + 1;

    /* x faces: a^px = rho^u d^u dy, b^px = rho^u u-hat dy; boundary faces per BC spec 2,3,9 */
    int kw = ukind(c, i, j), ke = ukind(c, i + 1, j);
    if (kw == F_ACTIVE) { double r = rho_u(c, o, i, j); apW = r * c->du[j * nxu + iw] * dy; bpW = r * c->uh[j * nxu + iw] * dy; }
    else if (kw == F_INLET) { bpW = rho_u(c, o, i, j) * c->u_in * dy; }
    if (ke == F_ACTIVE) { double r = rho_u(c, o, i + 1, j); apE = r * c->du[j * nxu + ie] * dy; bpE = r * c->uh[j * nxu + ie] * dy; }
    else if (ke == F_OUTLET) { bpE = rho_u(c, o, i + 1, j) * U(c, o, c->nx - 1, j) * dy; }
    /* y faces */
    if (vkind(c, i, j) == F_ACTIVE) { double r = rho_v(c, o, i, j); apS = r * c->dv[IV(c, i, j)] * dx; bpS = r * c->vh[IV(c, i, j)] * dx; }
    if (vkind(c, i, j + 1) == F_ACTIVE) { double r = rho_v(c, o, i, j + 1); apN = r * c->dv[IV(c, i, j + 1)] * dx; bpN = r * c->vh[IV(c, i, j + 1)] * dx; }

    double Tn = nw->T[IC(c, i, j)];
    double a0 = 1.0 / Tn * dx * dy + (apW + apE + apS + apN) * dt;
    double bp = PP(n1, i, j) / TT(n1, i, j) * dx * dy - (bpE - bpW + bpN - bpS) * dt;
    /* neighbour p_old only through active faces (BC spec 9: a^p = 0 elsewhere) */
    double sum = 0.0;
    const level* q = TP3;                       /* neighbour pressures: old iterate, or loop 3 (R41) */
    if (kw == F_ACTIVE) sum += apW * PP(q, i - 1, j);
    if (ke == F_ACTIVE) sum += apE * PP(q, i + 1, j);
    if (vkind(c, i, j) == F_ACTIVE) sum += apS * PP(q, i, j - 1);
    if (vkind(c, i, j + 1) == F_ACTIVE) sum += apN * PP(q, i, j + 1);
    return (sum * dt + bp) / a0;
}

/* =================================================== one loop-2 pass */
static double maxd(double a, double b) { return a > b ? a : b; }

static int one_pass(orc_case* c, double* res)
{
    const int nx = c->nx, ny = c->ny;
    level* o = OLD;
    level* nw = NEW;
    const int nxu = nx + 1;

    /* phase A */
    for (int j = 0; j < ny; j++)
        for (int i = 0; i < nx; i++)
            nw->T[IC(c, i, j)] = is_fluid(c, i, j) ? T_equation(c, i, j) : o->T[IC(c, i, j)];
    for (int j = 0; j < ny; j++)
        for (int i = 0; i <= nx; i++) {
            c->uh[j * nxu + i] = 0.0; c->du[j * nxu + i] = 0.0;
            if (ukind(c, i, j) == F_ACTIVE && !(periodic(c) && i == nx))
                u_equation(c, i, j, &c->uh[j * nxu + i], &c->du[j * nxu + i]);
        }
    for (int j = 0; j <= ny; j++)
        for (int i = 0; i < nx; i++) {
            c->vh[IV(c, i, j)] = 0.0; c->dv[IV(c, i, j)] = 0.0;
            if (vkind(c, i, j) == F_ACTIVE) v_equation(c, i, j, &c->vh[IV(c, i, j)], &c->dv[IV(c, i, j)]);
        }
    /* phase B */
    for (int j = 0; j < ny; j++)
        for (int i = 0; i < nx; i++)
            nw->p[IC(c, i, j)] = is_fluid(c, i, j) ? p_equation(c, i, j) : o->p[IC(c, i, j)];
    /* loop 3 of the CPU column (Figs. 1-2, reading R41):
     * sweeps k = 2 .. loop3 repeat the coupled energy / pressure pair with the
     * T-p terms at the previous sweep's iterate (Jacobi): the energy equation's
     * neighbour temperatures, unsteady density p/T and pressure work, and the
     * pressure equation's neighbour pressures; every other coefficient (fluxes,
     * limiters, links, Gamma, viscous heating, u-hat, d) stays the old iterate's. */
    for (int k = 2; k <= c->P.loop3; k++) {
        const size_t nc = (size_t)nx * ny;
        for (size_t e = 0; e < nc; e++) {
            c->L3.p[e] = nw->p[e];
            c->L3.T[e] = nw->T[e];
            c->L3.rho[e] = c->solid[e] ? o->rho[e] : nw->p[e] / nw->T[e];
        }
        c->it3 = &c->L3;
        for (int j = 0; j < ny; j++)
            for (int i = 0; i < nx; i++)
                if (is_fluid(c, i, j)) nw->T[IC(c, i, j)] = T_equation(c, i, j);
        for (int j = 0; j < ny; j++)
            for (int i = 0; i < nx; i++)
                if (is_fluid(c, i, j)) nw->p[IC(c, i, j)] = p_equation(c, i, j);
        c->it3 = NULL;
    }
    /* phase C: velocity correction (pl18, pl19), EOS (pl5), Gamma (pl37) */
    for (int j = 0; j < ny; j++)
        for (int i = 0; i <= nx; i++) {
            int k = ukind(c, i, j);
            double val;
            if (k == F_ACTIVE) {
                int ii = periodic(c) ? wrap(i, nx) : i;
                int im = periodic(c) ? wrap(i - 1, nx) : i - 1;
                val = c->uh[j * nxu + ii] - c->du[j * nxu + ii] * (nw->p[IC(c, ii, j)] - nw->p[IC(c, im, j)]);
            } else if (k == F_INLET) val = c->u_in;
            else if (k == F_OUTLET) val = o->u[IU(c, nx - 1, j)];   /* BC spec 3 */
            else val = 0.0;
            nw->u[IU(c, i, j)] = val;
        }
    for (int j = 0; j <= ny; j++)
        for (int i = 0; i < nx; i++) {
            double val = 0.0;
            if (vkind(c, i, j) == F_ACTIVE)
                val = c->vh[IV(c, i, j)] - c->dv[IV(c, i, j)] * (nw->p[IC(c, i, j)] - nw->p[IC(c, i, j - 1)]);
            nw->v[IV(c, i, j)] = val;
        }
    int bad = 0;
    for (int j = 0; j < ny; j++)
        for (int i = 0; i < nx; i++) {
            int id = IC(c, i, j);
            if (is_fluid(c, i, j)) {
                nw->rho[id] = nw->p[id] / nw->T[id];
                nw->gam[id] = sqrt(nw->T[id]);
                if (!(nw->T[id] > 0.0) || !(nw->p[id] > 0.0) || !isfinite(nw->p[id]) || !isfinite(nw->T[id])) bad = 1;
            } else {
                nw->rho[id] = o->rho[id]; nw->gam[id] = o->gam[id];
            }
        }

    /* residuals (R11): max |phi - phi_old| / max |phi| over updated points */
    double du_ = 0, dv_ = 0, dp_ = 0, dT_ = 0, mvel = 0, mp = 0, mT = 0;
    for (int j = 0; j < ny; j++)
        for (int i = 0; i <= nx; i++)
            if (ukind(c, i, j) == F_ACTIVE) {
                double a = nw->u[IU(c, i, j)];
                if (!isfinite(a)) bad = 1;
                du_ = maxd(du_, fabs(a - o->u[IU(c, i, j)])); mvel = maxd(mvel, fabs(a));
            }
    for (int j = 0; j <= ny; j++)
        for (int i = 0; i < nx; i++)
            if (vkind(c, i, j) == F_ACTIVE) {
                double a = nw->v[IV(c, i, j)];
                if (!isfinite(a)) bad = 1;
                dv_ = maxd(dv_, fabs(a - o->v[IV(c, i, j)])); mvel = maxd(mvel, fabs(a));
            }
    for (int j = 0; j < ny; j++)
        for (int i = 0; i < nx; i++)
            if (is_fluid(c, i, j)) {
                int id = IC(c, i, j);
                dp_ = maxd(dp_, fabs(nw->p[id] - o->p[id])); mp = maxd(mp, fabs(nw->p[id]));
                dT_ = maxd(dT_, fabs(nw->T[id] - o->T[id])); mT = maxd(mT, fabs(nw->T[id]));
            }
    res[0] = mvel > 0 ? du_ / mvel : du_;
    res[1] = mvel > 0 ? dv_ / mvel : dv_;
    res[2] = mp > 0 ? dp_ / mp : dp_;
    res[3] = mT > 0 ? dT_ / mT : dT_;

    /* swap old <-> new */
    level tmp = c->L[1]; c->L[1] = c->L[2]; c->L[2] = tmp;
    return bad ? 4 : 0;
}

static void copy_level(const orc_case* c, level* d, const level* s)
{
    size_t nc = (size_t)c->nx * c->ny, nu = (size_t)(c->nx + 1) * c->ny, nv = (size_t)c->nx * (c->ny + 1);
    memcpy(d->u, s->u, nu * sizeof(double));
    memcpy(d->v, s->v, nv * sizeof(double));
    memcpy(d->p, s->p, nc * sizeof(double));
    memcpy(d->T, s->T, nc * sizeof(double));
    memcpy(d->rho, s->rho, nc * sizeof(double));
    memcpy(d->gam, s->gam, nc * sizeof(double));
}

/* Loop 1 x loop 2 of the GPU column of Figs. 1-2. */
int orc_advance(orc_case* c, int32_t n_steps, double* res, int32_t* passes_out)
{
    double r[4] = {0, 0, 0, 0};
    int status = 0, passes = 0;
    for (int s = 0; s < n_steps; s++) {
        /* "Set the initial condition for the calculated time step":
         * n-1 := current state, first old iterate := n-1.  L[1] holds the
         * current (last converged) state between steps. */
        copy_level(c, N1, OLD);
        if (!implicit_(c)) compute_explicit_planes(c);
        passes = 0;
        int conv = 0;
        for (int k = 0; k < c->P.max_passes; k++) {
            int st = one_pass(c, r);
            passes++;
            if (st) { status = st; break; }
            if (c->P.tol > 0 && passes >= c->P.min_passes &&
                r[0] < c->P.tol && r[1] < c->P.tol && r[2] < c->P.tol && r[3] < c->P.tol) { conv = 1; break; }
        }
        if (status) break;
        if (c->P.tol > 0 && !conv) status = 3;
    }
    if (res) memcpy(res, r, sizeof r);
    if (passes_out) *passes_out = passes;
    return status;
}

/* ------------------------------------------------------- setup / io */
static void alloc_level(orc_case* c, level* l)
{
    size_t nc = (size_t)c->nx * c->ny, nu = (size_t)(c->nx + 1) * c->ny, nv = (size_t)c->nx * (c->ny + 1);
    l->u = calloc(nu, sizeof(double));
    l->v = calloc(nv, sizeof(double));
    l->p = calloc(nc, sizeof(double));
    l->T = calloc(nc, sizeof(double));
    l->rho = calloc(nc, sizeof(double));
    l->gam = calloc(nc, sizeof(double));
}
static void free_level(level* l)
{
    free(l->u); free(l->v); free(l->p); free(l->T); free(l->rho); free(l->gam);
}

orc_case* orc_create(const orc_params* prm, const int32_t* squares, int32_t n_sq)
{
    if (!prm || prm->nx < 1 || prm->ny < 1 || !(prm->dx > 0) || !(prm->dy > 0) || !(prm->Kn > 0) ||
        !(prm->dt > 0) || prm->max_passes < 1 || prm->pw_form < ORC_PW_DPDT || prm->pw_form > ORC_PW_GAMMA ||
        prm->loop3 < 0)
        return NULL;
    orc_case* c = calloc(1, sizeof *c);
    c->P = *prm;
    c->nx = prm->nx;
    c->ny = prm->ny;
    /* Eq. pl37 */
    c->A = 0.5;
    c->B = 5.0 * sqrt(M_PI) / 16.0 * prm->Kn;
    c->CT1 = prm->Kn * sqrt(M_PI * 225.0 / 1024.0);
    c->CT2 = sqrt(M_PI) / 4.0 * prm->Kn;
    c->CT3 = 2.0 / 5.0;
    /* kappa of the p div(u) forms of reading R9 */
    c->PWK = prm->pw_form == ORC_PW_PRINTED ? c->CT3 : prm->pw_form == ORC_PW_NEG ? -c->CT3 : -prm->gamma * c->CT3;
    /* u_in = M sqrt(gamma/2): V0 = sqrt(2 R T0), sound speed sqrt(gamma R T_in) */
    c->u_in = prm->mach * sqrt(prm->gamma / 2.0 * prm->T_in);
    if (prm->particle_frame) {           /* walls move with the gas in the particle frame (R14) */
        c->P.u_wall_bottom = c->u_in;
        c->P.u_wall_top = c->u_in;
    }
    c->solid = calloc((size_t)c->nx * c->ny, 1);
    for (int s = 0; s < n_sq; s++) {
        int i0 = squares[4 * s], j0 = squares[4 * s + 1], ni = squares[4 * s + 2], nj = squares[4 * s + 3];
        if (ni < 1 || nj < 1 || i0 < 0 || j0 < 0 || i0 + ni > c->nx || j0 + nj > c->ny) { free(c->solid); free(c); return NULL; }
        if (prm->xbc == ORC_X_INOUT && (i0 < 1 || i0 + ni > c->nx - 1)) { free(c->solid); free(c); return NULL; }
        for (int j = j0; j < j0 + nj; j++)
            for (int i = i0; i < i0 + ni; i++) c->solid[IC(c, i, j)] = 1;
    }
    for (int k = 0; k < 3; k++) alloc_level(c, &c->L[k]);
    if (prm->loop3 > 1) alloc_level(c, &c->L3);
    size_t nu = (size_t)(c->nx + 1) * c->ny, nv = (size_t)c->nx * (c->ny + 1), nc = (size_t)c->nx * c->ny;
    c->ue = calloc(nu, sizeof(double)); c->ve = calloc(nv, sizeof(double)); c->Te = calloc(nc, sizeof(double));
    c->uh = calloc(nu, sizeof(double)); c->du = calloc(nu, sizeof(double));
    c->vh = calloc(nv, sizeof(double)); c->dv = calloc(nv, sizeof(double));
    orc_init_freestream(c);
    return c;
}

void orc_destroy(orc_case* c)
{
    if (!c) return;
    for (int k = 0; k < 3; k++) free_level(&c->L[k]);
    free_level(&c->L3);
    free(c->ue); free(c->ve); free(c->Te); free(c->uh); free(c->du); free(c->vh); free(c->dv);
    free(c->solid);
    free(c->dxs); free(c->dys);
    free(c);
}

int orc_set_mesh(orc_case* c, const double* dxs, const double* dys)
{
    if (dxs) for (int i = 0; i < c->nx; i++) if (!(dxs[i] > 0.0)) return 1;
    if (dys) for (int j = 0; j < c->ny; j++) if (!(dys[j] > 0.0)) return 1;
    free(c->dxs); free(c->dys);
    c->dxs = c->dys = NULL;
    if (dxs) { c->dxs = malloc((size_t)c->nx * sizeof(double)); memcpy(c->dxs, dxs, (size_t)c->nx * sizeof(double)); }
    if (dys) { c->dys = malloc((size_t)c->ny * sizeof(double)); memcpy(c->dys, dys, (size_t)c->ny * sizeof(double)); }
    return 0;
}

/* Re-impose the fixed faces of BC spec 1-4 on the current state. */
static void impose_fixed_faces(orc_case* c, level* l)
{
    for (int j = 0; j < c->ny; j++)
        for (int i = 0; i <= c->nx; i++) {
            int k = ukind(c, i, j);
            if (k == F_FIXED0) l->u[IU(c, i, j)] = 0.0;
            else if (k == F_INLET) l->u[IU(c, i, j)] = c->u_in;
        }
    if (periodic(c))
        for (int j = 0; j < c->ny; j++) l->u[IU(c, c->nx, j)] = l->u[IU(c, 0, j)];
    for (int j = 0; j <= c->ny; j++)
        for (int i = 0; i < c->nx; i++) {
            int k = vkind(c, i, j);
            if (k == F_FIXED0 || k == F_WALL) l->v[IV(c, i, j)] = 0.0;
        }
}

void orc_init_freestream(orc_case* c)
{
    level* l = OLD;
    size_t nc = (size_t)c->nx * c->ny;
    for (size_t k = 0; k < nc; k++) {
        l->p[k] = c->P.p_in; l->T[k] = c->P.T_in;
        l->rho[k] = c->P.p_in / c->P.T_in; l->gam[k] = sqrt(c->P.T_in);
    }
    for (int j = 0; j < c->ny; j++)
        for (int i = 0; i <= c->nx; i++) l->u[IU(c, i, j)] = c->u_in;
    memset(l->v, 0, (size_t)c->nx * (c->ny + 1) * sizeof(double));
    impose_fixed_faces(c, l);
}

void orc_poison_solids(orc_case* c)
{
    for (int k = 0; k < 3; k++)
        for (int j = 0; j < c->ny; j++)
            for (int i = 0; i < c->nx; i++)
                if (c->solid[IC(c, i, j)]) {
                    int id = IC(c, i, j);
                    c->L[k].p[id] = NAN; c->L[k].T[id] = NAN; c->L[k].rho[id] = NAN; c->L[k].gam[id] = NAN;
                }
}

static int64_t field_size(const orc_case* c, int which)
{
    switch (which) {
    case ORC_U: case ORC_UEXP: return (int64_t)(c->nx + 1) * c->ny;
    case ORC_V: case ORC_VEXP: return (int64_t)c->nx * (c->ny + 1);
    default: return (int64_t)c->nx * c->ny;
    }
}

int orc_set_field(orc_case* c, int32_t which, const double* a, int64_t n)
{
    if (n != field_size(c, which) || which > ORC_T) return 1;
    level* l = OLD;
    double* dst = which == ORC_U ? l->u : which == ORC_V ? l->v : which == ORC_P ? l->p : l->T;
    memcpy(dst, a, (size_t)n * sizeof(double));
    if (which == ORC_P || which == ORC_T) {
        size_t nc = (size_t)c->nx * c->ny;
        for (size_t k = 0; k < nc; k++) { l->rho[k] = l->p[k] / l->T[k]; l->gam[k] = sqrt(l->T[k]); }
    }
    impose_fixed_faces(c, l);
    return 0;
}

int orc_get_field(const orc_case* c, int32_t which, double* a, int64_t n)
{
    if (n != field_size(c, which)) return 1;
    const level* l = &c->L[1];
    const double* src;
    switch (which) {
    case ORC_U: src = l->u; break;
    case ORC_V: src = l->v; break;
    case ORC_P: src = l->p; break;
    case ORC_T: src = l->T; break;
    case ORC_RHO: src = l->rho; break;
    case ORC_GAMMA: src = l->gam; break;
    case ORC_UEXP: src = c->ue; break;
    case ORC_VEXP: src = c->ve; break;
    case ORC_TEXP: src = c->Te; break;
    default: return 1;
    }
    memcpy(a, src, (size_t)n * sizeof(double));
    return 0;
}

int orc_get_map(const orc_case* c, int32_t which, int32_t* a, int64_t n)
{
    if (which == 0) {
        if (n != (int64_t)c->nx * c->ny) return 1;
        for (int64_t k = 0; k < n; k++) a[k] = c->solid[k];
    } else if (which == 1) {
        if (n != (int64_t)(c->nx + 1) * c->ny) return 1;
        for (int j = 0; j < c->ny; j++)
            for (int i = 0; i <= c->nx; i++) a[IU(c, i, j)] = ukind(c, i, j);
    } else if (which == 2) {
        if (n != (int64_t)c->nx * (c->ny + 1)) return 1;
        for (int j = 0; j <= c->ny; j++)
            for (int i = 0; i < c->nx; i++) a[IV(c, i, j)] = vkind(c, i, j);
    } else return 1;
    return 0;
}

void orc_constants(const orc_case* c, double* out)
{
    out[0] = c->A; out[1] = c->B; out[2] = c->CT1; out[3] = c->CT2; out[4] = c->CT3; out[5] = c->u_in; out[6] = 0.0;
}
