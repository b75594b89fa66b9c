// sts_kernels.cuh -- sm_100a fp64 kernels of the SIMPLE-TS loop-2 sweep
// (arXiv:1802.04243).  Written from the paper and DESIGN.md section 3; shares
// no code with oracle/.
//
// Design: one fused kernel per loop-2 pass.  A CTA owns
// a TX x TY tile of cells; it stages the old iterate of u, v, p, T with a
// 3-cell halo in shared memory (rho = p/T and Gamma = sqrt(T) are recomputed
// on load instead of being stored, P:576 stored them because division was
// slow on 2013 GPUs), then runs the paper's dependency order inside the CTA
// (Eqs. pl29_1-pl29_8):
//   stage 1  face densities rho^u, rho^v (Eqs. pl10-pl11, reading R1)
//   stage 2  T (pl30-pl33), u-hat/d^u (pl20 + transposition), v-hat/d^v
//            (pl14-pl16, pl21) on the tile plus a one-cell ring
//   stage 3  p (pl23-pl24) on the tile plus the west/south ring
//   stage 4  u, v correction (pl18-pl19), writes, residual maxima.
// Every intermediate (T, u-hat, d^u, v-hat, d^v, p) lives in shared memory
// only, as the paper kept them in local memory; HBM sees the
// 96 B/FV of DESIGN.md section 6 (implicit) plus the explicit planes.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sts {

// ------------------------------------------------------------ kinds
enum : uint8_t { CK_FLUID = 0, CK_SOLID = 1, CK_INLET = 2, CK_OUTLET = 3, CK_WALLY = 4 };
enum : uint8_t { FK_ACTIVE = 0, FK_FIXED0 = 1, FK_INLET = 2, FK_OUTLET = 3, FK_WALL = 4, FK_NONE = 5 };

// ------------------------------------------------------------ tiling
constexpr int TX = 32;          // owned cells per tile in x (one warp-wide row)
constexpr int TY = 16;          // owned cells per tile in y
constexpr int HH = 3;           // halo: TVD stencil reach of one fused pass (DESIGN 5.2)
constexpr int CW = TX + 2 * HH, CH = TY + 2 * HH;   // cell region
constexpr int UW = CW + 1, UH = CH;                  // u-face region
constexpr int VW = CW, VH = CH + 1;                  // v-face region
constexpr int NT = 256;         // threads per CTA
constexpr int OFF = 4;          // local column of global column gi0 is OFF (ghost columns 0..3)

struct Params {
    // geometry / decomposition
    int nx, ny;                 // global cells
    int gi0, nloc;              // first owned global column of this rank, owned columns
    int pitch;                  // doubles per stored row (all arrays)
    int xbc;                    // 0 inflow/outflow, 1 periodic
    int mirror;                 // 1: single rank periodic -> kernel writes wrapped ghosts
    int last_rank;              // this rank owns global column nx-1
    int first_rank;             // this rank owns global column 0
    // constants
    double dx, dy, dt;
    double A, B, CT1, CT2, CT3, Kn;
    double u_in, p_in, T_in;
    double u_wb, u_wt, T_wall, T_sq, g_x, g_y, pw_sign;
    // fields: old iterate, time level n-1, explicit planes, new iterate
    const double *u_o, *v_o, *p_o, *T_o;
    const double *u_1, *v_1, *p_1, *T_1;
    const double *ue, *ve, *Te;
    double *u_w, *v_w, *p_w, *T_w;
    double *ue_w, *ve_w, *Te_w;  // conv kernel outputs
    const uint8_t *ck, *uk, *vk;  // kind maps (local layout)
    unsigned long long* red;    // residual slots of this pass (9 x u64)
};

__device__ __forceinline__ long long gidx(const Params& k, int gi, int gj)
{
    return (long long)gj * k.pitch + (gi - k.gi0 + OFF);
}
__device__ __forceinline__ bool stored_col(const Params& k, int gi)
{
    int li = gi - k.gi0 + OFF;
    return li >= 0 && li < k.pitch;
}

// Van Leer TVD correction on a uniform mesh (Eqs. pl15_1 / pl15_2 with equal
// widths coincide): w > 0: psi = 0.5 psi_VL(a/b) = a/(a+b) if a b > 0;
// w <= 0: -0.5 psi_VL(c/b) = -c/(c+b) if c b > 0; else 0 (readings R6, R7).
// A denominator difference b at the rounding level counts as zero (R37).
__device__ __forceinline__ double psi_u(double f1, double f2, double f3, double f4, double w)
{
    double b = f3 - f2;
    if (fabs(b) <= 1e-12 * (1.0 + fabs(f2) + fabs(f3))) return 0.0;
    if (w > 0.0) {
        double a = f2 - f1;
        return ((a > 0.0 && b > 0.0) || (a < 0.0 && b < 0.0)) ? a / (a + b) : 0.0;
    } else {
        double c = f4 - f3;
        return ((c > 0.0 && b > 0.0) || (c < 0.0 && b < 0.0)) ? -c / (c + b) : 0.0;
    }
}
// max(0, a) exactly (also for -0 and NaN inputs of either sign' magnitude): clear
// both words when the sign bit is set -- three integer ops, no fp64 compare/select
__device__ __forceinline__ double max0(double a)
{
    const int hi = __double2hiint(a), lo = __double2loint(a);
    const int keep = ~(hi >> 31);
    return __hiloint2double(hi & keep, lo & keep);
}
__device__ __forceinline__ bool flux_face(uint8_t k) { return k == FK_ACTIVE || k == FK_INLET || k == FK_OUTLET; }
__device__ __forceinline__ bool wallish(uint8_t k) { return k == CK_SOLID || k == CK_WALLY; }

struct Smem {
    double P[CH][CW], T[CH][CW], R[CH][CW], G[CH][CW], R1[CH][CW], TN[CH][CW], PN[CH][CW];
    double U[UH][UW], RU[UH][UW], UHAT[UH][UW], DU[UH][UW];
    double V[VH][VW], RV[VH][VW], VHAT[VH][VW], DV[VH][VW];
    uint8_t K[CH][CW], UK[UH][UW], VK[VH][VW];
};

// Stage 0: stage the tile + halo of one snapshot (old, or n-1 for the conv
// kernel) into shared memory.  Rows beyond the channel walls get kind WALLY,
// u = wall velocity (BC spec 8), other values 1 (never used).
template <bool WITH_N1>
__device__ void load_tile(Smem& s, const Params& k, int I0, int J0,
                          const double* u, const double* v, const double* p, const double* T)
{
    const int tid = threadIdx.x;
    for (int e = tid; e < CH * CW; e += NT) {
        int y = e / CW, x = e - y * CW;
        int gi = I0 - HH + x, gj = J0 - HH + y;
        uint8_t kind = CK_WALLY;
        double pv = 1.0, Tv = 1.0, p1 = 1.0, T1 = 1.0;
        if (gj >= 0 && gj < k.ny && stored_col(k, gi)) {
            long long id = gidx(k, gi, gj);
            kind = k.ck[id];
            pv = p[id];
            Tv = T[id];
            if (WITH_N1) { p1 = k.p_1[id]; T1 = k.T_1[id]; }
        }
        s.K[y][x] = kind;
        s.P[y][x] = pv;
        s.T[y][x] = Tv;
        s.R[y][x] = pv / Tv;            // Eq. pl5
        s.G[y][x] = sqrt(Tv);           // Eq. pl37: Gamma = Gamma^lambda = sqrt(T)
        if (WITH_N1) s.R1[y][x] = p1 / T1;
    }
    for (int e = tid; e < UH * UW; e += NT) {
        int y = e / UW, x = e - y * UW;
        int gf = I0 - HH + x, gj = J0 - HH + y;
        double val;
        uint8_t kind = FK_NONE;
        if (gj < 0) val = k.u_wb;
        else if (gj >= k.ny) val = k.u_wt;
        else if (stored_col(k, gf)) { long long id = gidx(k, gf, gj); val = u[id]; kind = k.uk[id]; }
        else val = 0.0;
        s.U[y][x] = val;
        s.UK[y][x] = kind;
    }
    for (int e = tid; e < VH * VW; e += NT) {
        int y = e / VW, x = e - y * VW;
        int gi = I0 - HH + x, gj = J0 - HH + y;
        double val = 0.0;
        uint8_t kind = FK_NONE;
        if (gj >= 0 && gj <= k.ny && stored_col(k, gi)) { long long id = gidx(k, gi, gj); val = v[id]; kind = k.vk[id]; }
        s.V[y][x] = val;
        s.VK[y][x] = kind;
    }
}

// Stage 1: face densities rho^u (u-faces x in [2, TX+4), rows [1, TY+4)) and
// rho^v (v-faces x in [1, TX+4), rows [2, TY+4)); 0 where no mass crosses.
template <bool TVD>
__device__ void face_densities(Smem& s)
{
    const int tid = threadIdx.x;
    constexpr int NXU = TX + 2, NYU = TY + 3;
    for (int e = tid; e < NXU * NYU; e += NT) {
        int y = 1 + e / NXU, x = 2 + e % NXU;
        double ru = 0.0;
        if (flux_face(s.UK[y][x])) {
            double w = s.U[y][x], r1 = s.R[y][x - 1], r2 = s.R[y][x];
            ru = w > 0.0 ? r1 : r2;
            if (TVD && s.K[y][x - 2] == CK_FLUID && s.K[y][x - 1] == CK_FLUID && s.K[y][x] == CK_FLUID &&
                s.K[y][x + 1] == CK_FLUID)
                ru += psi_u(s.R[y][x - 2], r1, r2, s.R[y][x + 1], w) * (r2 - r1);
        }
        s.RU[y][x] = ru;
    }
    constexpr int NXV = TX + 3, NYV = TY + 2;
    for (int e = tid; e < NXV * NYV; e += NT) {
        int y = 2 + e / NXV, x = 1 + e % NXV;
        double rv = 0.0;
        if (s.VK[y][x] == FK_ACTIVE) {
            double w = s.V[y][x], r1 = s.R[y - 1][x], r2 = s.R[y][x];
            rv = w > 0.0 ? r1 : r2;
            if (TVD && s.K[y - 2][x] == CK_FLUID && s.K[y - 1][x] == CK_FLUID && s.K[y][x] == CK_FLUID &&
                s.K[y + 1][x] == CK_FLUID)
                rv += psi_u(s.R[y - 2][x], r1, r2, s.R[y + 1][x], w) * (r2 - r1);
        }
        s.RV[y][x] = rv;
    }
}

// Corner Gamma at (x^f_x, y^f_y): mean over the adjacent cells that are not
// solid and not beyond a wall (readings R4, R5; BC spec 8).
__device__ __forceinline__ double gam_corner(const Smem& s, int x, int y)
{
    double sum = 0.0;
    int n = 0;
    if (!wallish(s.K[y - 1][x - 1])) { sum += s.G[y - 1][x - 1]; n++; }
    if (!wallish(s.K[y - 1][x])) { sum += s.G[y - 1][x]; n++; }
    if (!wallish(s.K[y][x - 1])) { sum += s.G[y][x - 1]; n++; }
    if (!wallish(s.K[y][x])) { sum += s.G[y][x]; n++; }
    return sum / n;
}

// ---------------------------------------------------------------- energy
// Eqs. pl30-pl33, pl28-pl29 (implicit) / pl31_1 (explicit); walls: BC spec 5.
template <bool IMPL, bool TVD>
__device__ double T_equation(const Smem& s, const Params& k, int x, int y, int gi, int gj)
{
    const double dx = k.dx, dy = k.dy, dt = k.dt;
    const double gP = s.G[y][x], rP = s.R[y][x];
    double a1, a2, a3, a4, T1, T2, T3, T4;
    double FW = 0.0, FE = 0.0, FS = 0.0, FN = 0.0;
    const double tau = 2.1904 * k.Kn / rP;    // Eq. pl39

    uint8_t kn = s.K[y][x - 1];
    if (wallish(kn)) {
        a1 = k.CT1 * gP * dy / (0.5 * dx + tau);
        T1 = kn == CK_WALLY ? k.T_wall : k.T_sq;
    } else {
        FW = s.RU[y][x] * s.U[y][x] * dy;
        double gm = s.G[y][x - 1];
        double D = k.CT1 * (2.0 * dx * gm * gP / (dx * gP + dx * gm)) * dy / dx;
        double ps = 0.0;
        if (IMPL && TVD && s.K[y][x - 2] == CK_FLUID && kn == CK_FLUID && s.K[y][x + 1] == CK_FLUID)
            ps = psi_u(s.T[y][x - 2], s.T[y][x - 1], s.T[y][x], s.T[y][x + 1], s.U[y][x]);
        a1 = (IMPL ? max0(FW) - FW * ps : 0.0) + D;
        T1 = s.T[y][x - 1];
    }
    kn = s.K[y][x + 1];
    if (wallish(kn)) {
        a2 = k.CT1 * gP * dy / (0.5 * dx + tau);
        T2 = kn == CK_WALLY ? k.T_wall : k.T_sq;
    } else {
        FE = s.RU[y][x + 1] * s.U[y][x + 1] * dy;
        double gp = s.G[y][x + 1];
        double D = k.CT1 * (2.0 * dx * gP * gp / (dx * gp + dx * gP)) * dy / dx;
        double ps = 0.0;
        if (IMPL && TVD && s.K[y][x - 1] == CK_FLUID && kn == CK_FLUID && s.K[y][x + 2] == CK_FLUID)
            ps = psi_u(s.T[y][x - 1], s.T[y][x], s.T[y][x + 1], s.T[y][x + 2], s.U[y][x + 1]);
        a2 = (IMPL ? max0(-FE) - FE * ps : 0.0) + D;
        T2 = s.T[y][x + 1];
    }
    kn = s.K[y - 1][x];
    if (wallish(kn)) {
        a3 = k.CT1 * gP * dx / (0.5 * dy + tau);
        T3 = kn == CK_WALLY ? k.T_wall : k.T_sq;
    } else {
        FS = s.RV[y][x] * s.V[y][x] * dx;
        double gm = s.G[y - 1][x];
        double D = k.CT1 * (2.0 * dy * gm * gP / (dy * gP + dy * gm)) * dx / dy;
        double ps = 0.0;
        if (IMPL && TVD && s.K[y - 2][x] == CK_FLUID && kn == CK_FLUID && s.K[y + 1][x] == CK_FLUID)
            ps = psi_u(s.T[y - 2][x], s.T[y - 1][x], s.T[y][x], s.T[y + 1][x], s.V[y][x]);
        a3 = (IMPL ? max0(FS) - FS * ps : 0.0) + D;
        T3 = s.T[y - 1][x];
    }
    kn = s.K[y + 1][x];
    if (wallish(kn)) {
        a4 = k.CT1 * gP * dx / (0.5 * dy + tau);
        T4 = kn == CK_WALLY ? k.T_wall : k.T_sq;
    } else {
        FN = s.RV[y + 1][x] * s.V[y + 1][x] * dx;
        double gp = s.G[y + 1][x];
        double D = k.CT1 * (2.0 * dy * gP * gp / (dy * gp + dy * gP)) * dx / dy;
        double ps = 0.0;
        if (IMPL && TVD && s.K[y - 1][x] == CK_FLUID && kn == CK_FLUID && s.K[y + 2][x] == CK_FLUID)
            ps = psi_u(s.T[y - 1][x], s.T[y][x], s.T[y + 1][x], s.T[y + 2][x], s.V[y + 1][x]);
        a4 = (IMPL ? max0(-FN) - FN * ps : 0.0) + D;
        T4 = s.T[y + 1][x];
    }
    const double dV = dx * dy;
    double a0 = IMPL ? dt * (a1 + a2 + a3 + a4 + FE - FW + FN - FS) + rP * dV
                     : dt * (a1 + a2 + a3 + a4) + rP * dV;

    // S^T_c, Eq. pl29 with bilinear (4-point mean) mid-point velocities (R4)
    double dudx = (s.U[y][x + 1] - s.U[y][x]) / dx;
    double dvdy = (s.V[y + 1][x] - s.V[y][x]) / dy;
    double vE = 0.25 * (s.V[y][x] + s.V[y][x + 1] + s.V[y + 1][x] + s.V[y + 1][x + 1]);
    double vW = 0.25 * (s.V[y][x - 1] + s.V[y][x] + s.V[y + 1][x - 1] + s.V[y + 1][x]);
    double uN = 0.25 * (s.U[y][x] + s.U[y][x + 1] + s.U[y + 1][x] + s.U[y + 1][x + 1]);
    double uS = 0.25 * (s.U[y - 1][x] + s.U[y - 1][x + 1] + s.U[y][x] + s.U[y][x + 1]);
    double shear = (vE - vW) / dx + (uN - uS) / dy;
    double div = dudx + dvdy;
    double Sc = k.CT2 * gP * (2.0 * (dudx * dudx + dvdy * dvdy) + shear * shear - 2.0 / 3.0 * div * div) * dV
              + k.pw_sign * k.CT3 * s.P[y][x] * div * dV;

    double Texp = IMPL ? 0.0 : k.Te[gidx(k, gi, gj)];
    double T1n = k.T_1[gidx(k, gi, gj)];
    double rhs = dt * (a1 * T1 + a2 * T2 + a3 * T3 + a4 * T4 + Sc + Texp) + s.R1[y][x] * T1n * dV;
    return rhs / a0;
}

// -------------------------------------------------------- u pseudo-velocity
// Eq. pl20 with the v-coefficients of Eqs. pl14-pl16 / pl15_11 transposed
// x <-> y (DESIGN 3.4).  u-face (x, y) between cells (x-1, y) and (x, y).
template <bool IMPL, bool TVD>
__device__ void u_equation(Smem& s, const Params& k, int x, int y, int gf, int gj)
{
    const double dx = k.dx, dy = k.dy, dt = k.dt;
    const double rL = s.R[y][x - 1], rR = s.R[y][x], gL = s.G[y][x - 1], gR = s.G[y][x];
    double a1, a2, a3, a4, uS, uN;
    double Fs_i = 0.0, Fs_im1 = 0.0, Fn_i = 0.0, Fn_im1 = 0.0;

    const double ubW = 0.5 * (s.U[y][x - 1] + s.U[y][x]);
    const double ubE = 0.5 * (s.U[y][x] + s.U[y][x + 1]);
    const double FbW = rL * ubW * dy, FbE = rR * ubE * dy;
    const double Dux_i = k.B * gL * dy / dx, Dux_ip1 = k.B * gR * dy / dx;
    double psW = 0.0, psE = 0.0;
    if (IMPL && TVD) {
        bool okc = s.UK[y][x - 1] == FK_ACTIVE && s.UK[y][x + 1] == FK_ACTIVE;   // face x itself is active
        if (okc && s.UK[y][x - 2] == FK_ACTIVE)
            psW = psi_u(s.U[y][x - 2], s.U[y][x - 1], s.U[y][x], s.U[y][x + 1], ubW);
        if (okc && s.UK[y][x + 2] == FK_ACTIVE)
            psE = psi_u(s.U[y][x - 1], s.U[y][x], s.U[y][x + 1], s.U[y][x + 2], ubE);
    }
    a1 = (IMPL ? max0(FbW) - FbW * psW : 0.0) + 4.0 / 3.0 * Dux_i;
    a2 = (IMPL ? max0(-FbE) - FbE * psE : 0.0) + 4.0 / 3.0 * Dux_ip1;
    const double uW = s.U[y][x - 1], uE = s.U[y][x + 1];

    const double gadj = 0.5 * (gL + gR), radj = 0.5 * (rL + rR);
    const double zeta = 1.1466 * k.Kn / radj;   // Eq. pl38
    // south (tangential) link
    {
        uint8_t kl = s.K[y - 1][x - 1], kr = s.K[y - 1][x];
        if (kl == CK_WALLY || (kl == CK_SOLID && kr == CK_SOLID)) {
            a3 = k.B * gadj * dx / (0.5 * dy + zeta);
            uS = kl == CK_WALLY ? k.u_wb : 0.0;
        } else {
            Fs_i = s.RV[y][x] * s.V[y][x] * dx;
            Fs_im1 = s.RV[y][x - 1] * s.V[y][x - 1] * dx;
            double p1 = 0.0, p2 = 0.0;
            if (IMPL && TVD && s.UK[y - 2][x] == FK_ACTIVE && s.UK[y - 1][x] == FK_ACTIVE &&
                s.UK[y + 1][x] == FK_ACTIVE) {
                double f1 = s.U[y - 2][x], f2 = s.U[y - 1][x], f3 = s.U[y][x], f4 = s.U[y + 1][x];
                p1 = psi_u(f1, f2, f3, f4, s.V[y][x]);
                p2 = psi_u(f1, f2, f3, f4, s.V[y][x - 1]);
            }
            double Duy = k.B * gam_corner(s, x, y) * dx / dy;
            a3 = (IMPL ? 0.5 * (max0(Fs_i) - Fs_i * p1 + max0(Fs_im1) - Fs_im1 * p2) : 0.0) + Duy;
            uS = s.U[y - 1][x];
        }
    }
    // north (tangential) link
    {
        uint8_t kl = s.K[y + 1][x - 1], kr = s.K[y + 1][x];
        if (kl == CK_WALLY || (kl == CK_SOLID && kr == CK_SOLID)) {
            a4 = k.B * gadj * dx / (0.5 * dy + zeta);
            uN = kl == CK_WALLY ? k.u_wt : 0.0;
        } else {
            Fn_i = s.RV[y + 1][x] * s.V[y + 1][x] * dx;
            Fn_im1 = s.RV[y + 1][x - 1] * s.V[y + 1][x - 1] * dx;
            double p1 = 0.0, p2 = 0.0;
            if (IMPL && TVD && s.UK[y - 1][x] == FK_ACTIVE && s.UK[y + 1][x] == FK_ACTIVE &&
                s.UK[y + 2][x] == FK_ACTIVE) {
                double f1 = s.U[y - 1][x], f2 = s.U[y][x], f3 = s.U[y + 1][x], f4 = s.U[y + 2][x];
                p1 = psi_u(f1, f2, f3, f4, s.V[y + 1][x]);
                p2 = psi_u(f1, f2, f3, f4, s.V[y + 1][x - 1]);
            }
            double Duy = k.B * gam_corner(s, x, y + 1) * dx / dy;
            a4 = (IMPL ? 0.5 * (max0(-Fn_i) - Fn_i * p1 + max0(-Fn_im1) - Fn_im1 * p2) : 0.0) + Duy;
            uN = s.U[y + 1][x];
        }
    }
    const double tterm = (rR * dx + rL * dx) * dy / (2.0 * dt);
    const double a0 = IMPL ? a1 + a2 + a3 + a4 + FbE - FbW + 0.5 * (Fn_i - Fs_i + Fn_im1 - Fs_im1) + tterm
                           : a1 + a2 + a3 + a4 + tterm;
    const long long gid = gidx(k, gf, gj);
    double b = (s.R1[y][x] * dx + s.R1[y][x - 1] * dx) * dy / (2.0 * dt) * k.u_1[gid]
             + k.B * (gam_corner(s, x, y + 1) * (s.V[y + 1][x] - s.V[y + 1][x - 1])
                      - gam_corner(s, x, y) * (s.V[y][x] - s.V[y][x - 1])
                      - 2.0 / 3.0 * gR * (s.V[y + 1][x] - s.V[y][x])
                      + 2.0 / 3.0 * gL * (s.V[y + 1][x - 1] - s.V[y][x - 1]))
             + k.g_x * 0.5 * (rR * dx + rL * dx) * dy;
    const double uexp = IMPL ? 0.0 : k.ue[gid];
    s.UHAT[y][x] = (a1 * uW + a2 * uE + a3 * uS + a4 * uN + b + uexp) / a0;
    s.DU[y][x] = k.A * dy / a0;
}

// -------------------------------------------------------- v pseudo-velocity
// Eqs. pl14-pl16, pl21, pl15_11 with reading R2.  v-face (x, y) between cells
// (x, y-1) and (x, y).
template <bool IMPL, bool TVD>
__device__ void v_equation(Smem& s, const Params& k, int x, int y, int gi, int gj)
{
    const double dx = k.dx, dy = k.dy, dt = k.dt;
    const double rB = s.R[y - 1][x], rT = s.R[y][x], gB = s.G[y - 1][x], gT = s.G[y][x];
    double a1, a2, a3, a4, vW, vE;
    double Fw_j = 0.0, Fw_jm1 = 0.0, Fe_j = 0.0, Fe_jm1 = 0.0;

    const double vbS = 0.5 * (s.V[y - 1][x] + s.V[y][x]);
    const double vbN = 0.5 * (s.V[y][x] + s.V[y + 1][x]);
    const double FbS = rB * vbS * dx, FbN = rT * vbN * dx;
    const double Dvy_j = k.B * gB * dx / dy, Dvy_jp1 = k.B * gT * dx / dy;
    double psS = 0.0, psN = 0.0;
    if (IMPL && TVD) {
        bool okc = s.VK[y - 1][x] == FK_ACTIVE && s.VK[y + 1][x] == FK_ACTIVE;
        if (okc && s.VK[y - 2][x] == FK_ACTIVE)
            psS = psi_u(s.V[y - 2][x], s.V[y - 1][x], s.V[y][x], s.V[y + 1][x], vbS);
        if (okc && s.VK[y + 2][x] == FK_ACTIVE)
            psN = psi_u(s.V[y - 1][x], s.V[y][x], s.V[y + 1][x], s.V[y + 2][x], vbN);
    }
    a3 = (IMPL ? max0(FbS) - FbS * psS : 0.0) + 4.0 / 3.0 * Dvy_j;
    a4 = (IMPL ? max0(-FbN) - FbN * psN : 0.0) + 4.0 / 3.0 * Dvy_jp1;
    const double vS = s.V[y - 1][x], vN = s.V[y + 1][x];

    const double gadj = 0.5 * (gB + gT), radj = 0.5 * (rB + rT);
    const double zeta = 1.1466 * k.Kn / radj;
    // west (tangential) link
    if (s.K[y - 1][x - 1] == CK_SOLID && s.K[y][x - 1] == CK_SOLID) {
        a1 = k.B * gadj * dy / (0.5 * dx + zeta);
        vW = 0.0;
    } else {
        Fw_j = s.RU[y][x] * s.U[y][x] * dy;
        Fw_jm1 = s.RU[y - 1][x] * s.U[y - 1][x] * dy;
        double p1 = 0.0, p2 = 0.0;
        if (IMPL && TVD && s.VK[y][x - 2] == FK_ACTIVE && s.VK[y][x - 1] == FK_ACTIVE &&
            s.VK[y][x + 1] == FK_ACTIVE) {
            double f1 = s.V[y][x - 2], f2 = s.V[y][x - 1], f3 = s.V[y][x], f4 = s.V[y][x + 1];
            p1 = psi_u(f1, f2, f3, f4, s.U[y][x]);
            p2 = psi_u(f1, f2, f3, f4, s.U[y - 1][x]);
        }
        double Dvx = k.B * gam_corner(s, x, y) * dy / dx;
        a1 = (IMPL ? 0.5 * (max0(Fw_j) - Fw_j * p1 + max0(Fw_jm1) - Fw_jm1 * p2) : 0.0) + Dvx;
        vW = s.V[y][x - 1];
    }
    // east (tangential) link
    if (s.K[y - 1][x + 1] == CK_SOLID && s.K[y][x + 1] == CK_SOLID) {
        a2 = k.B * gadj * dy / (0.5 * dx + zeta);
        vE = 0.0;
    } else {
        Fe_j = s.RU[y][x + 1] * s.U[y][x + 1] * dy;
        Fe_jm1 = s.RU[y - 1][x + 1] * s.U[y - 1][x + 1] * dy;
        double p1 = 0.0, p2 = 0.0;
        if (IMPL && TVD && s.VK[y][x - 1] == FK_ACTIVE && s.VK[y][x + 1] == FK_ACTIVE &&
            s.VK[y][x + 2] == FK_ACTIVE) {
            double f1 = s.V[y][x - 1], f2 = s.V[y][x], f3 = s.V[y][x + 1], f4 = s.V[y][x + 2];
            p1 = psi_u(f1, f2, f3, f4, s.U[y][x + 1]);
            p2 = psi_u(f1, f2, f3, f4, s.U[y - 1][x + 1]);
        }
        double Dvx = k.B * gam_corner(s, x + 1, y) * dy / dx;
        a2 = (IMPL ? 0.5 * (max0(-Fe_j) - Fe_j * p1 + max0(-Fe_jm1) - Fe_jm1 * p2) : 0.0) + Dvx;
        vE = s.V[y][x + 1];
    }
    const double tterm = (rT * dy + rB * dy) * dx / (2.0 * dt);
    const double a0 = IMPL ? a1 + a2 + a3 + a4 + 0.5 * (Fe_j - Fw_j + Fe_jm1 - Fw_jm1) + FbN - FbS + tterm
                           : a1 + a2 + a3 + a4 + tterm;
    const long long gid = gidx(k, gi, gj);
    double b = (s.R1[y][x] * dy + s.R1[y - 1][x] * dy) * dx / (2.0 * dt) * k.v_1[gid]
             + k.B * (gam_corner(s, x + 1, y) * (s.U[y][x + 1] - s.U[y - 1][x + 1])
                      - gam_corner(s, x, y) * (s.U[y][x] - s.U[y - 1][x])
                      - 2.0 / 3.0 * gT * (s.U[y][x + 1] - s.U[y][x])
                      + 2.0 / 3.0 * gB * (s.U[y - 1][x + 1] - s.U[y - 1][x]))
             + k.g_y * 0.5 * (rT * dy + rB * dy) * dx;
    const double vexp = IMPL ? 0.0 : k.ve[gid];
    s.VHAT[y][x] = (a1 * vW + a2 * vE + a3 * vS + a4 * vN + b + vexp) / a0;
    s.DV[y][x] = k.A * dx / a0;
}

// ------------------------------------------------------------- pressure
// Eqs. pl23-pl24 with T of this pass (R28); boundary faces BC spec 2, 3, 9.
__device__ double p_equation(const Smem& s, const Params& k, int x, int y)
{
    const double dx = k.dx, dy = k.dy, dt = k.dt;
    double apW = 0.0, apE = 0.0, apS = 0.0, apN = 0.0, bpW = 0.0, bpE = 0.0, bpS = 0.0, bpN = 0.0;
    const uint8_t kw = s.UK[y][x], ke = s.UK[y][x + 1], ks = s.VK[y][x], kn = s.VK[y + 1][x];
    if (kw == FK_ACTIVE) { double r = s.RU[y][x]; apW = r * s.DU[y][x] * dy; bpW = r * s.UHAT[y][x] * dy; }
    else if (kw == FK_INLET) bpW = s.RU[y][x] * k.u_in * dy;
    if (ke == FK_ACTIVE) { double r = s.RU[y][x + 1]; apE = r * s.DU[y][x + 1] * dy; bpE = r * s.UHAT[y][x + 1] * dy; }
    else if (ke == FK_OUTLET) bpE = s.RU[y][x + 1] * s.U[y][x] * dy;
    if (ks == FK_ACTIVE) { double r = s.RV[y][x]; apS = r * s.DV[y][x] * dx; bpS = r * s.VHAT[y][x] * dx; }
    if (kn == FK_ACTIVE) { double r = s.RV[y + 1][x]; apN = r * s.DV[y + 1][x] * dx; bpN = r * s.VHAT[y + 1][x] * dx; }
    const double a0 = 1.0 / s.TN[y][x] * dx * dy + (apW + apE + apS + apN) * dt;
    const double bp = s.R1[y][x] * dx * dy - (bpE - bpW + bpN - bpS) * dt;
    double sum = 0.0;
    if (kw == FK_ACTIVE) sum += apW * s.P[y][x - 1];
    if (ke == FK_ACTIVE) sum += apE * s.P[y][x + 1];
    if (ks == FK_ACTIVE) sum += apS * s.P[y - 1][x];
    if (kn == FK_ACTIVE) sum += apN * s.P[y + 1][x];
    return (sum * dt + bp) / a0;
}

// ------------------------------------------------------- residual helpers
__device__ __forceinline__ double warp_max(double v)
{
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// NaN-propagating max for the residual slots (fmax would drop NaN).
__device__ __forceinline__ double nmax(double a, double b) { return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000LL) : (a > b ? a : b); }

__device__ void reduce_and_publish(double* vals, int n, unsigned long long* red, long long bad, int badf)
{
    __shared__ double part[NT / 32][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int q = 0; q < n; q++) {
        double v = vals[q];
        bool isn = v != v;
        unsigned nanmask = __ballot_sync(0xffffffffu, isn);
        v = warp_max(isn ? 0.0 : v);
        if (nanmask) v = __longlong_as_double(0x7ff8000000000000LL);
        if (lane == 0) part[wid][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < n) {
        double v = 0.0;
        for (int w = 0; w < NT / 32; w++) v = nmax(v, part[w][threadIdx.x]);
        atomicMax(&red[threadIdx.x], (unsigned long long)__double_as_longlong(v));
    }
    if (bad >= 0) {   // first bad cell: max of (LLONG_MAX - flat index)
        atomicMax(&red[7], 0x7fffffffffffffffULL - (unsigned long long)bad);
        red[8] = (unsigned long long)badf;
    }
}

// =================================================================== pass
// One loop-2 pass (P:171-177 explicit, P:227-236 implicit) for one tile.
template <bool IMPL, bool TVD>
__global__ void __launch_bounds__(NT, 2) pass_kernel(Params k)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);
    const int I0 = k.gi0 + blockIdx.x * TX, J0 = blockIdx.y * TY;
    const int tid = threadIdx.x;

    load_tile<true>(s, k, I0, J0, k.u_o, k.v_o, k.p_o, k.T_o);
    __syncthreads();
    face_densities<TVD>(s);
    __syncthreads();

    // stage 2: T on cells [2, TX+3) x [2, TY+3); u-hat on faces [2, TX+4) x [2, TY+3);
    //          v-hat on faces [2, TX+3) x [2, TY+4)
    constexpr int NC = (TX + 1) * (TY + 1);
    constexpr int NU = (TX + 2) * (TY + 1);
    constexpr int NV = (TX + 1) * (TY + 2);
    for (int e = tid; e < NC + NU + NV; e += NT) {
        if (e < NC) {
            int y = 2 + e / (TX + 1), x = 2 + e % (TX + 1);
            int gi = I0 - HH + x, gj = J0 - HH + y;
            s.TN[y][x] = s.K[y][x] == CK_FLUID ? T_equation<IMPL, TVD>(s, k, x, y, gi, gj) : s.T[y][x];
        } else if (e < NC + NU) {
            int q = e - NC;
            int y = 2 + q / (TX + 2), x = 2 + q % (TX + 2);
            if (s.UK[y][x] == FK_ACTIVE) u_equation<IMPL, TVD>(s, k, x, y, I0 - HH + x, J0 - HH + y);
        } else {
            int q = e - NC - NU;
            int y = 2 + q / (TX + 1), x = 2 + q % (TX + 1);
            if (s.VK[y][x] == FK_ACTIVE) v_equation<IMPL, TVD>(s, k, x, y, I0 - HH + x, J0 - HH + y);
        }
    }
    __syncthreads();
    // stage 3: p on cells [2, TX+3) x [2, TY+3)
    for (int e = tid; e < NC; e += NT) {
        int y = 2 + e / (TX + 1), x = 2 + e % (TX + 1);
        s.PN[y][x] = s.K[y][x] == CK_FLUID ? p_equation(s, k, x, y) : s.P[y][x];
    }
    __syncthreads();

    // stage 4: corrections, writes, residual maxima over owned points
    double r_du = 0.0, r_dv = 0.0, r_dp = 0.0, r_dT = 0.0, r_vel = 0.0, r_p = 0.0, r_T = 0.0;
    long long bad = -1;
    int badf = 0;
    const int iend = k.gi0 + k.nloc;
    for (int e = tid; e < TX * TY; e += NT) {
        int y = HH + e / TX, x = HH + e % TX;
        int gi = I0 - HH + x, gj = J0 - HH + y;
        if (gi >= iend || gj >= k.ny) continue;
        const long long id = gidx(k, gi, gj);
        // cell
        if (s.K[y][x] == CK_FLUID) {
            double Tn = s.TN[y][x], pn = s.PN[y][x];
            k.T_w[id] = Tn;
            k.p_w[id] = pn;
            r_dT = nmax(r_dT, fabs(Tn - s.T[y][x]));
            r_dp = nmax(r_dp, fabs(pn - s.P[y][x]));
            r_T = nmax(r_T, fabs(Tn));
            r_p = nmax(r_p, fabs(pn));
            if (!(Tn > 0.0) || !(pn > 0.0) || !isfinite(Tn) || !isfinite(pn)) {
                long long flat = (long long)gj * k.nx + gi;
                if (bad < 0 || flat < bad) { bad = flat; badf = !(Tn > 0.0) || !isfinite(Tn) ? 3 : 2; }
            }
        }
        // u-face x (global face gi)
        {
            uint8_t ku = s.UK[y][x];
            double un;
            if (ku == FK_ACTIVE) {
                un = s.UHAT[y][x] - s.DU[y][x] * (s.PN[y][x] - s.PN[y][x - 1]);
                r_du = nmax(r_du, fabs(un - s.U[y][x]));
                r_vel = nmax(r_vel, fabs(un));
            } else if (ku == FK_INLET) un = k.u_in;
            else un = 0.0;
            k.u_w[id] = un;
            if (gi == k.nx - 1 && k.xbc == 0) k.u_w[id + 1] = s.U[y][x];   // outlet face: u_old(nx-1), BC spec 3
        }
        // v-face (x, y) (global row gj)
        {
            uint8_t kv = s.VK[y][x];
            double vn = 0.0;
            if (kv == FK_ACTIVE) {
                vn = s.VHAT[y][x] - s.DV[y][x] * (s.PN[y][x] - s.PN[y - 1][x]);
                r_dv = nmax(r_dv, fabs(vn - s.V[y][x]));
                r_vel = nmax(r_vel, fabs(vn));
            }
            k.v_w[id] = vn;
        }
        // ghost columns owned by the physical boundary (BC spec 3, 4)
        if (k.xbc == 0) {
            if (gi == k.nx - 1) {
                double pn = k.p_w[id], Tn = k.T_w[id], vn = k.v_w[id];
                for (int g = 1; g <= OFF - 1; g++) { k.p_w[id + g] = pn; k.T_w[id + g] = Tn; k.v_w[id + g] = vn; }
            }
        } else if (k.mirror) {
            int tgt = -1000;
            if (gi < OFF) tgt = gi + k.nx;
            else if (gi >= k.nx - OFF) tgt = gi - k.nx;
            if (tgt > -1000) {
                long long t = gidx(k, tgt, gj);
                k.p_w[t] = k.p_w[id]; k.T_w[t] = k.T_w[id]; k.u_w[t] = k.u_w[id]; k.v_w[t] = k.v_w[id];
            }
            if (gi == 0) k.u_w[gidx(k, k.nx, gj)] = k.u_w[id];   // face nx == face 0 (also covered above)
        }
    }
    double vals[7] = {r_du, r_dv, r_dp, r_dT, r_vel, r_p, r_T};
    reduce_and_publish(vals, 7, k.red, bad, badf);
}

// ================================================================== conv
// Explicit convective planes u^exp, v^exp, T^exp from the n-1 state, once per
// time step (Eqs. pl15_11, pl31_1 and the transposed u-plane).
template <bool TVD>
__global__ void __launch_bounds__(NT, 2) conv_kernel(Params k)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);
    const int I0 = k.gi0 + blockIdx.x * TX, J0 = blockIdx.y * TY;
    const int tid = threadIdx.x;
    load_tile<false>(s, k, I0, J0, k.u_1, k.v_1, k.p_1, k.T_1);
    __syncthreads();
    face_densities<TVD>(s);
    __syncthreads();
    const double dx = k.dx, dy = k.dy;
    const int iend = k.gi0 + k.nloc;
    for (int e = tid; e < TX * TY; e += NT) {
        int y = HH + e / TX, x = HH + e % TX;
        int gi = I0 - HH + x, gj = J0 - HH + y;
        if (gi >= iend || gj >= k.ny) continue;
        const long long id = gidx(k, gi, gj);
        // ---- T^exp (Eq. pl31_1)
        double te = 0.0;
        if (s.K[y][x] == CK_FLUID) {
            const double Ti = s.T[y][x];
            if (flux_face(s.UK[y][x + 1])) {
                double F = s.RU[y][x + 1] * s.U[y][x + 1] * dy, w = s.U[y][x + 1], Tp = s.T[y][x + 1];
                double ps = (TVD && s.K[y][x - 1] == CK_FLUID && s.K[y][x + 1] == CK_FLUID && s.K[y][x + 2] == CK_FLUID)
                          ? psi_u(s.T[y][x - 1], Ti, Tp, s.T[y][x + 2], w) : 0.0;
                te += -F * ((w > 0.0 ? Ti : Tp) + (Tp - Ti) * ps);
            }
            if (flux_face(s.UK[y][x])) {
                double F = s.RU[y][x] * s.U[y][x] * dy, w = s.U[y][x], Tm = s.T[y][x - 1];
                double ps = (TVD && s.K[y][x - 2] == CK_FLUID && s.K[y][x - 1] == CK_FLUID && s.K[y][x + 1] == CK_FLUID)
                          ? psi_u(s.T[y][x - 2], Tm, Ti, s.T[y][x + 1], w) : 0.0;
                te += F * ((w > 0.0 ? Tm : Ti) + (Ti - Tm) * ps);
            }
            if (s.VK[y + 1][x] == FK_ACTIVE) {
                double F = s.RV[y + 1][x] * s.V[y + 1][x] * dx, w = s.V[y + 1][x], Tp = s.T[y + 1][x];
                double ps = (TVD && s.K[y - 1][x] == CK_FLUID && s.K[y + 1][x] == CK_FLUID && s.K[y + 2][x] == CK_FLUID)
                          ? psi_u(s.T[y - 1][x], Ti, Tp, s.T[y + 2][x], w) : 0.0;
                te += -F * ((w > 0.0 ? Ti : Tp) + (Tp - Ti) * ps);
            }
            if (s.VK[y][x] == FK_ACTIVE) {
                double F = s.RV[y][x] * s.V[y][x] * dx, w = s.V[y][x], Tm = s.T[y - 1][x];
                double ps = (TVD && s.K[y - 2][x] == CK_FLUID && s.K[y - 1][x] == CK_FLUID && s.K[y + 1][x] == CK_FLUID)
                          ? psi_u(s.T[y - 2][x], Tm, Ti, s.T[y + 1][x], w) : 0.0;
                te += F * ((w > 0.0 ? Tm : Ti) + (Ti - Tm) * ps);
            }
        }
        k.Te_w[id] = te;
        // ---- u^exp at u-face x (transposed pl15_11)
        double ue = 0.0;
        if (s.UK[y][x] == FK_ACTIVE) {
            const double ui = s.U[y][x];
            {   // north half-faces
                const double up = s.U[y + 1][x];
                const bool ok = TVD && s.UK[y - 1][x] == FK_ACTIVE && s.UK[y + 1][x] == FK_ACTIVE && s.UK[y + 2][x] == FK_ACTIVE;
                double sum = 0.0;
                for (int h = 0; h < 2; h++) {
                    int xx = x - 1 + h;
                    if (s.VK[y + 1][xx] != FK_ACTIVE) continue;
                    double F = s.RV[y + 1][xx] * s.V[y + 1][xx] * dx, w = s.V[y + 1][xx];
                    double ps = ok ? psi_u(s.U[y - 1][x], ui, up, s.U[y + 2][x], w) : 0.0;
                    sum += F * ((w > 0.0 ? ui : up) + (up - ui) * ps);
                }
                ue += -0.5 * sum;
            }
            {   // south half-faces
                const double um = s.U[y - 1][x];
                const bool ok = TVD && s.UK[y - 2][x] == FK_ACTIVE && s.UK[y - 1][x] == FK_ACTIVE && s.UK[y + 1][x] == FK_ACTIVE;
                double sum = 0.0;
                for (int h = 0; h < 2; h++) {
                    int xx = x - 1 + h;
                    if (s.VK[y][xx] != FK_ACTIVE) continue;
                    double F = s.RV[y][xx] * s.V[y][xx] * dx, w = s.V[y][xx];
                    double ps = ok ? psi_u(s.U[y - 2][x], um, ui, s.U[y + 1][x], w) : 0.0;
                    sum += F * ((w > 0.0 ? um : ui) + (ui - um) * ps);
                }
                ue += 0.5 * sum;
            }
            {   // east: cell centre x
                const double up = s.U[y][x + 1], ub = 0.5 * (ui + up);
                const bool ok = TVD && s.UK[y][x - 1] == FK_ACTIVE && s.UK[y][x + 1] == FK_ACTIVE && s.UK[y][x + 2] == FK_ACTIVE;
                double ps = ok ? psi_u(s.U[y][x - 1], ui, up, s.U[y][x + 2], ub) : 0.0;
                ue += -dy * s.R[y][x] * ub * ((ub > 0.0 ? ui : up) + (up - ui) * ps);
            }
            {   // west: cell centre x-1
                const double um = s.U[y][x - 1], ub = 0.5 * (um + ui);
                const bool ok = TVD && s.UK[y][x - 2] == FK_ACTIVE && s.UK[y][x - 1] == FK_ACTIVE && s.UK[y][x + 1] == FK_ACTIVE;
                double ps = ok ? psi_u(s.U[y][x - 2], um, ui, s.U[y][x + 1], ub) : 0.0;
                ue += dy * s.R[y][x - 1] * ub * ((ub > 0.0 ? um : ui) + (ui - um) * ps);
            }
        }
        k.ue_w[id] = ue;
        // ---- v^exp at v-face (x, y) (Eq. pl15_11, R2)
        double ve = 0.0;
        if (s.VK[y][x] == FK_ACTIVE) {
            const double vi = s.V[y][x];
            {   // east half-faces
                const double vp = s.V[y][x + 1];
                const bool ok = TVD && s.VK[y][x - 1] == FK_ACTIVE && s.VK[y][x + 1] == FK_ACTIVE && s.VK[y][x + 2] == FK_ACTIVE;
                double sum = 0.0;
                for (int h = 0; h < 2; h++) {
                    int yy = y - 1 + h;
                    if (!flux_face(s.UK[yy][x + 1])) continue;
                    double F = s.RU[yy][x + 1] * s.U[yy][x + 1] * dy, w = s.U[yy][x + 1];
                    double ps = ok ? psi_u(s.V[y][x - 1], vi, vp, s.V[y][x + 2], w) : 0.0;
                    sum += F * ((w > 0.0 ? vi : vp) + (vp - vi) * ps);
                }
                ve += -0.5 * sum;
            }
            {   // west half-faces
                const double vm = s.V[y][x - 1];
                const bool ok = TVD && s.VK[y][x - 2] == FK_ACTIVE && s.VK[y][x - 1] == FK_ACTIVE && s.VK[y][x + 1] == FK_ACTIVE;
                double sum = 0.0;
                for (int h = 0; h < 2; h++) {
                    int yy = y - 1 + h;
                    if (!flux_face(s.UK[yy][x])) continue;
                    double F = s.RU[yy][x] * s.U[yy][x] * dy, w = s.U[yy][x];
                    double ps = ok ? psi_u(s.V[y][x - 2], vm, vi, s.V[y][x + 1], w) : 0.0;
                    sum += F * ((w > 0.0 ? vm : vi) + (vi - vm) * ps);
                }
                ve += 0.5 * sum;
            }
            {   // north: cell centre (x, y)
                const double vp = s.V[y + 1][x], vb = 0.5 * (vi + vp);
                const bool ok = TVD && s.VK[y - 1][x] == FK_ACTIVE && s.VK[y + 1][x] == FK_ACTIVE && s.VK[y + 2][x] == FK_ACTIVE;
                double ps = ok ? psi_u(s.V[y - 1][x], vi, vp, s.V[y + 2][x], vb) : 0.0;
                ve += -dx * s.R[y][x] * vb * ((vb > 0.0 ? vi : vp) + (vp - vi) * ps);
            }
            {   // south: cell centre (x, y-1)
                const double vm = s.V[y - 1][x], vb = 0.5 * (vm + vi);
                const bool ok = TVD && s.VK[y - 2][x] == FK_ACTIVE && s.VK[y - 1][x] == FK_ACTIVE && s.VK[y + 1][x] == FK_ACTIVE;
                double ps = ok ? psi_u(s.V[y - 2][x], vm, vi, s.V[y + 1][x], vb) : 0.0;
                ve += dx * s.R[y - 1][x] * vb * ((vb > 0.0 ? vm : vi) + (vi - vm) * ps);
            }
        }
        k.ve_w[id] = ve;
        if (k.xbc == 1 && k.mirror) {
            int tgt = -1000;
            if (gi < OFF) tgt = gi + k.nx;
            else if (gi >= k.nx - OFF) tgt = gi - k.nx;
            if (tgt > -1000) {
                long long t = gidx(k, tgt, gj);
                k.Te_w[t] = te; k.ue_w[t] = ue; k.ve_w[t] = ve;
            }
        }
    }
}

}  // namespace sts
