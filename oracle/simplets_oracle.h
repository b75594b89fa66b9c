/*
 * simplets_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded fp64 C implementation of one SIMPLE-TS time
 * step (loop 1 x loop 2) exactly as arXiv:1802.04243 (K. S. Shterev) prints
 * it, plus the boundary-condition spec and ambiguity readings of DESIGN.md
 * section 3.  It is the parity oracle for the CUDA path and nothing else:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, table or
 * constant generator with paper_1802_04243_b200/ (the product path).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (the paper's LaTeX),
 * with the equation label the paper uses (pl8 ... pl39).
 */
#ifndef SIMPLETS_ORACLE_H
#define SIMPLETS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Boundary in x: 0 = supersonic inflow at x=0 / zero-gradient outflow at x=L
 * (the paper's channel), 1 = periodic (validation cases only). */
enum { ORC_X_INOUT = 0, ORC_X_PERIODIC = 1 };
/* Time treatment of the convective terms. */
enum { ORC_EXPLICIT = 0, ORC_IMPLICIT = 1 };
/* Space treatment of the convective terms. */
enum { ORC_UPWIND = 0, ORC_TVD = 1 };
/* Pressure-work forms of S^T_c (reading R9). */
enum { ORC_PW_DPDT = 0, ORC_PW_PRINTED = 1, ORC_PW_NEG = 2, ORC_PW_GAMMA = 3 };
/* Field ids for set/get. */
enum { ORC_U = 0, ORC_V = 1, ORC_P = 2, ORC_T = 3, ORC_RHO = 4, ORC_GAMMA = 5,
       ORC_UEXP = 6, ORC_VEXP = 7, ORC_TEXP = 8 };

typedef struct {
    int32_t nx, ny;           /* cells along x, y                              */
    double  dx, dy;           /* uniform spacings Delta x, Delta y     */
    int32_t xbc;              /* ORC_X_INOUT / ORC_X_PERIODIC                  */
    double  Kn, mach, gamma;
    double  p_in, T_in;       /* inflow reference state (=1,1)          */
    double  u_wall_bottom, u_wall_top;  /* tangential wall velocities  */
    double  T_wall, T_square; /* wall temperatures (reading R15)       */
    double  g_x, g_y;         /* body force (Eqs. pl2/pl3)          */
    int32_t particle_frame;   /* 1: both channel walls move at +u_in (P:686,
                                 reading R14); overrides u_wall_bottom/top      */
    int32_t pw_form;          /* pressure-work term of S^T_c (reading R9):
                                 ORC_PW_DPDT  C^T3 Dp/Dt of Eq. pl6 at
                                              the old iterate (default)
                                 ORC_PW_PRINTED  +C^T3 p div(u) (Eq. pl29)
                                 ORC_PW_NEG      -C^T3 p div(u) (round-1 R9)
                                 ORC_PW_GAMMA    -gamma C^T3 p div(u)          */
    int32_t r37_off;          /* test hook: 1 switches the R37 flat-stencil
                                 guard of psi_s / psi_c off (DESIGN R37)       */
    int32_t time_scheme;      /* ORC_EXPLICIT / ORC_IMPLICIT                   */
    int32_t space_scheme;     /* ORC_UPWIND / ORC_TVD                          */
    double  dt;               /* time step                                     */
    int32_t min_passes, max_passes;
    double  tol;              /* <= 0 -> exactly max_passes per step           */
    int32_t loop3;            /* T-p sweeps per pass (loop 3 of the CPU column,
                                 Figs. 1-2, reading R41); 0 or 1 =
                                 the GPU column (one energy / pressure pair)    */
    int32_t reserved;
} orc_params;

typedef struct orc_case orc_case;

/* squares: n_sq rows of (i0, j0, ni, nj) in cell units (solid block). */
orc_case* orc_create(const orc_params* prm, const int32_t* squares, int32_t n_sq);
void      orc_destroy(orc_case* c);
/* p = T = 1 (inflow state), rho = p/T, Gamma = sqrt(T), u = u_in at every
 * u-face, v = 0; faces touching a solid or a wall hold 0. */
void      orc_init_freestream(orc_case* c);
/* Overwrite one field (global shape; u: (nx+1)*ny, v: nx*(ny+1), cells nx*ny,
 * row-major with i fastest).  Setting p or T refreshes rho and Gamma.
 * Fixed faces are re-imposed afterwards. */
int       orc_set_field(orc_case* c, int32_t which, const double* a, int64_t n);
int       orc_get_field(const orc_case* c, int32_t which, double* a, int64_t n);
/* Cell map (0 fluid, 1 solid), u-face kinds, v-face kinds (see .c). */
int       orc_get_map(const orc_case* c, int32_t which, int32_t* a, int64_t n);
/* Advance n_steps time steps.  res[4] gets the last pass' normalised
 * residuals (u, v, p, T); passes_out the loop-2 passes of the last step.
 * Returns 0, or 3 if tol > 0 and a step hit max_passes unconverged,
 * or 4 if a non-finite / non-positive state appeared. */
int       orc_advance(orc_case* c, int32_t n_steps, double* res, int32_t* passes_out);
/* Non-uniform mesh (the general staggered mesh of Fig. 5): dxs[nx]
 * = Delta x_i, dys[ny] = Delta y_j (> 0); NULL keeps that direction uniform
 * (P.dx / P.dy).  Returns 1 on a non-positive step. */
int       orc_set_mesh(orc_case* c, const double* dxs, const double* dys);
/* Debug: fill solid-cell p,T,rho,Gamma with NaN (proves they are never read). */
void      orc_poison_solids(orc_case* c);
/* Derived constants of Eq. pl37 and u_in: out[0..6] =
 * A, B, CT1, CT2, CT3, u_in, (unused 0). */
void      orc_constants(const orc_case* c, double* out);

/* Scheme functions exposed for pinning. */
double orc_vanleer(double r);
double orc_psi_s(double f1, double f2, double f3, double f4,
                 double d1, double d2, double d3, double d4, double w);
double orc_psi_c(double f1, double f2, double f3, double f4,
                 double d1, double d2, double d3, double w);
double orc_upwind(double f1, double f2, double w);

#ifdef __cplusplus
}
#endif
#endif
