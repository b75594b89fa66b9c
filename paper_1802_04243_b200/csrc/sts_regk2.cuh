// sts_regk2.cuh -- the all-regular march, two rows per row step (round 2, v11).
//
// regk_kernel (sts_regk.cuh) is latency-bound: 12 warps per SM (166 registers),
// "wait" (fixed-latency dependency) the first stall reason, 3 barriers per row.
// Here a row step advances rows j ("lo") and j+1 ("hi") together: the stage
// dependency order of P:550 is kept per row (A, barrier, C, barrier, D, barrier,
// E) but the two rows' stages share each barrier interval, so there are 1.5
// barriers per row and two independent rows of fp64 chains per warp (2 CTAs,
// 8 warps per SM at up to 255 registers).  The hi row consumes the lo row's
// carries inside the step (registers).  Every formula is regk_body's (explicit
// FMA/MUL, same order): the same bits (test_regk_same_bits).
// Shared memory: an 8-slot ring (rows j-1 .. j+4 in use, rows j+5, j+6 in flight:
// TMA issued one step ahead of the derive), 4 flux rows (rows mod 4) and the face
// rows of both rows of the step.
#pragma once

#include "sts_regk.cuh"

namespace sts {

#define STS_LINK(F, ps) (TVD ? FMA(-(F), (ps), max0(F)) : max0(F))

constexpr int RS2 = 8;
struct Regk2Smem {
    RingRow ring[RS2];
    FluxRow fr[4];
    double R1[2][RW];
    double XTW[2][RW], XUW[2][RW], XVW[2][RW], UH[2][RW], DU[2][RW], PN[2][RW];
    unsigned long long mbar[RS2];
};

// Own-column values of one row's stencil (rows M = j-1, O = j, A = j+1, B = j+2,
// C = j+3 relative to the row j being advanced).
struct Own2 {
    double uM, uO, uA, pM, pO, pA, tM, tO, tA, vO, vA, vB, rM, rO, rA, gO, gA;
    double rB, tB, uB, vC;            // TVD only
};
// Carries into a row (from the row below, in registers).
struct Cin2 {
    Carry c;
    double fxO, fxE, ruO, r1O;
};
// Results of a row's stages.
struct Row2 {
    double Fx1, ru, Fy1, rv1, xtw, ytN, ytSn, xe, Fb, upsi1, upsi2, vcN, vcSn, FbN, gcN, xvW, FwSum, r1n;
    double t0W, t0E, u0W, vaW, vaE, fxnE;
    double TN, uhat, du, utSn, FsSumN, vhatN, dvN, p0W, p0E, pn;
};

// stage A of one row (regk_body's, with the row's rings and face rows)
template <bool IMPL, bool TVD>
__device__ __forceinline__ void regk2_A(const MarchParams& m, int lc, const RingRow& R0, const RingRow& Ra,
                                        FluxRow& Fn, double* XTW, double* XUW, double* XVW, const Own2& o,
                                        const Cin2& ci, double p1n, double T1n, Row2& v)
{
    const double dx = m.k.dx, dy = m.k.dy;
    v.r1n = fdiv(p1n, T1n == 0.0 ? 1.0 : T1n);
    const double raW = Ra.R[lc - 1], g0W = R0.G[lc - 1], gaW = Ra.G[lc - 1], u0E = R0.U[lc + 1];
    if (TVD) { v.t0W = R0.T[lc - 1]; v.t0E = R0.T[lc + 1]; v.u0W = R0.U[lc - 1]; v.vaW = Ra.V[lc - 1]; v.vaE = Ra.V[lc + 1]; }
    {
        const double w = o.uA, r1 = raW, r2 = o.rA;
        double ru = w > 0.0 ? r1 : r2;
        if (TVD) ru = FMA(psi_f(Ra.R[lc - 2], r1, r2, Ra.R[lc + 1], w), r2 - r1, ru);
        v.ru = ru;
        v.Fx1 = MUL(MUL(ru, w), dy);
        Fn.RU[lc] = ru;
        Fn.FX[lc] = v.Fx1;
    }
    {
        const double w = o.vA, r1 = o.rO, r2 = o.rA;
        double rv = w > 0.0 ? r1 : r2;
        if (TVD) rv = FMA(psi_f(o.rM, r1, r2, o.rB, w), r2 - r1, rv);
        v.rv1 = rv;
        v.Fy1 = MUL(MUL(rv, w), dx);
        Fn.FY[lc] = v.Fy1;
    }
    {
        const double F = ci.fxO;
        const double g1 = g0W, g2 = o.gO;
        const double hg = MUL(MUL(MUL(2.0, g1), g2), rcp(g1 + g2));
        double ps = 0.0;
        if (IMPL && TVD) ps = psi_f(R0.T[lc - 2], v.t0W, o.tO, v.t0E, o.uO);
        v.xtw = FMA(m.CT1_dydx, hg, IMPL ? STS_LINK(F, ps) : 0.0);
        XTW[lc] = v.xtw;
    }
    {
        const double F = v.Fy1;
        const double g1 = o.gO, g2 = o.gA;
        const double hg = MUL(MUL(MUL(2.0, g1), g2), rcp(g1 + g2));
        double ps = 0.0;
        if (IMPL && TVD) ps = psi_f(o.tM, o.tO, o.tA, o.tB, o.vA);
        v.ytSn = FMA(m.CT1_dxdy, hg, IMPL ? STS_LINK(F, ps) : 0.0);
        v.ytN = IMPL ? v.ytSn - F : v.ytSn;
    }
    {
        const double ub = MUL(0.5, o.uO + u0E);
        v.Fb = MUL(MUL(o.rO, ub), dy);
        double ps = 0.0;
        if (IMPL && TVD) ps = psi_f(v.u0W, o.uO, u0E, R0.U[lc + 2], ub);
        const double xw = FMA(m.B43_dydx, o.gO, IMPL ? STS_LINK(v.Fb, ps) : 0.0);
        v.xe = IMPL ? xw - v.Fb : xw;
        XUW[lc] = xw;
    }
    v.upsi1 = 0.0;
    v.upsi2 = 0.0;
    if (IMPL && TVD) {
        v.upsi1 = psi_f(o.uM, o.uO, o.uA, o.uB, o.vA);
        v.upsi2 = psi_f(o.uM, o.uO, o.uA, o.uB, v.vaW);
    }
    {
        const double vb = MUL(0.5, o.vA + o.vB);
        v.FbN = MUL(MUL(o.rA, vb), dx);
        double ps = 0.0;
        if (IMPL && TVD) ps = psi_f(o.vO, o.vA, o.vB, o.vC, vb);
        v.vcSn = FMA(m.B43_dxdy, o.gA, IMPL ? STS_LINK(v.FbN, ps) : 0.0);
        v.vcN = IMPL ? v.vcSn - v.FbN : v.vcSn;
    }
    v.gcN = MUL(0.25, g0W + o.gO + gaW + o.gA);
    {
        const double F1 = v.Fx1, F2 = ci.fxO;
        double p1 = 0.0, p2 = 0.0;
        if (IMPL && TVD) {
            const double f1 = Ra.V[lc - 2];
            p1 = psi_f(f1, v.vaW, o.vA, v.vaE, o.uA);
            p2 = psi_f(f1, v.vaW, o.vA, v.vaE, o.uO);
        }
        v.FwSum = F1 + F2;
        const double lk = IMPL ? MUL(0.5, STS_LINK(F1, p1) + STS_LINK(F2, p2)) : 0.0;
        v.xvW = FMA(m.B_dydx, v.gcN, lk);
        XVW[lc] = v.xvW;
    }
}

// stage C of one row
template <bool IMPL, bool TVD>
__device__ __forceinline__ void regk2_C(const MarchParams& m, int lc, const RingRow& Rm, const RingRow& R0,
                                        const RingRow& Ra, const FluxRow& Fn, const double* XTW, const double* XUW,
                                        const double* XVW, const double* R1, double* UH, double* DU, const Own2& o,
                                        const Cin2& ci, double T1c, double u1c, double v1n, double Tec, double uec,
                                        double ven, Row2& v)
{
    const Params& k = m.k;
    const double dt = k.dt, dy = k.dy, dV = m.dV;
    if (!TVD) { v.t0W = R0.T[lc - 1]; v.t0E = R0.T[lc + 1]; v.u0W = R0.U[lc - 1]; v.vaW = Ra.V[lc - 1]; v.vaE = Ra.V[lc + 1]; }
    const double u0E = R0.U[lc + 1], g0W = R0.G[lc - 1];
    const double v0W = R0.V[lc - 1], v0E = R0.V[lc + 1];
    const double uaE = Ra.U[lc + 1], umE = Rm.U[lc + 1];
    v.p0W = R0.P[lc - 1];
    v.p0E = R0.P[lc + 1];
    const double xtwE = XTW[lc + 1], fyW = Fn.FY[lc - 1], xuwW = XUW[lc - 1], r1W = R1[lc - 1];
    v.fxnE = Fn.FX[lc + 1];
    const double xvwE = XVW[lc + 1];
    const Carry& c = ci.c;
    {
        const double a1 = v.xtw, FW = ci.fxO, T1 = v.t0W;
        const double FE = ci.fxE, a2 = IMPL ? xtwE - FE : xtwE, T2 = v.t0E;
        const double a3 = c.ytS, FSl = c.FS, T3 = o.tM;
        const double a4 = v.ytN, FNl = v.Fy1, T4 = o.tA;
        const double rq = o.rO;
        const double a0 = IMPL ? FMA(dt, a1 + a2 + a3 + a4 + FE - FW + FNl - FSl, MUL(rq, dV))
                               : FMA(dt, a1 + a2 + a3 + a4, MUL(rq, dV));
        const double dudx = MUL(u0E - o.uO, m.inv_dx);
        const double dvdy = MUL(o.vA - o.vO, m.inv_dy);
        const double shear = FMA((v0E + v.vaE) - (v0W + v.vaW), m.q_dx, MUL((o.uA + uaE) - (o.uM + umE), m.q_dy));
        const double div = dudx + dvdy;
        const double pc = o.pO;
        const double p1 = MUL(ci.r1O, T1c);
        const double dpx = MUL(v.p0E - v.p0W, m.h_dx);
        const double dpy = MUL(o.pA - o.pM, m.h_dy);
        const double ub = MUL(0.5, o.uO + u0E), vb = MUL(0.5, o.vO + o.vA);
        const double pwork = FMA(m.pw_a, FMA(vb, dpy, FMA(ub, dpx, MUL(pc - p1, m.inv_dt))), MUL(MUL(k.pwk, pc), div));
        const double Phi = FMA(MUL(-2.0 / 3.0, div), div, FMA(shear, shear, MUL(2.0, FMA(dvdy, dvdy, MUL(dudx, dudx)))));
        const double Sc = MUL(FMA(MUL(k.CT2, o.gO), Phi, pwork), dV);
        const double sT = FMA(a4, T4, FMA(a3, T3, FMA(a2, T2, MUL(a1, T1))));
        const double rhs = FMA(dt, sT + (IMPL ? Sc : Sc + Tec), MUL(p1, dV));
        v.TN = MUL(rhs, rcp(a0));
    }
    {
        const double F1 = v.Fy1, F2 = fyW;
        v.FsSumN = F1 + F2;
        const double lk = IMPL ? MUL(0.5, STS_LINK(F1, v.upsi1) + STS_LINK(F2, v.upsi2)) : 0.0;
        v.utSn = FMA(m.B_dxdy, v.gcN, lk);
        const double a4p = IMPL ? FMA(-0.5, v.FsSumN, v.utSn) : v.utSn;
        const double rL = R0.R[lc - 1], rR = o.rO, gL = g0W, gR = o.gO;
        const double a1 = xuwW, a2 = v.xe;
        const double FbW = MUL(MUL(rL, MUL(0.5, v.u0W + o.uO)), dy), FbE = v.Fb;
        const double a3 = c.utS, FsS = c.FsSum, uS = o.uM;
        const double a4 = a4p, FnS = v.FsSumN, uN = o.uA;
        const double tterm = MUL(rR + rL, m.c_t);
        const double a0 = IMPL ? FMA(0.5, FnS - FsS, a1 + a2 + a3 + a4 + FbE - FbW) + tterm
                               : a1 + a2 + a3 + a4 + tterm;
        const double bt = MUL(ci.r1O + r1W, m.c_t);
        const double bg = MUL(MUL(k.g_x, rR + rL), m.half_dV);
        const double bv = FMA(MUL(2.0 / 3.0, gL), v.vaW - v0W,
                          FMA(MUL(-2.0 / 3.0, gR), o.vA - o.vO,
                          FMA(-c.gcP, o.vO - v0W, MUL(v.gcN, o.vA - v.vaW))));
        const double b = FMA(k.B, bv, MUL(bt, u1c)) + bg;
        const double r = rcp(a0);
        const double su = FMA(a4, uN, FMA(a3, uS, FMA(a2, u0E, MUL(a1, v.u0W))));
        v.uhat = MUL(su + (IMPL ? b : b + uec), r);
        v.du = MUL(m.A_dy, r);
        UH[lc] = v.uhat;
        DU[lc] = v.du;
    }
    {
        const double rB = o.rO, rT = o.rA, gB = o.gO, gT = o.gA;
        const double a1 = v.xvW, FwS = v.FwSum, vW = v.vaW;
        const double FeS = v.fxnE + ci.fxE, a2 = IMPL ? FMA(-0.5, FeS, xvwE) : xvwE, vE = v.vaE;
        const double gcE = MUL(0.25, o.gO + R0.G[lc + 1] + o.gA + Ra.G[lc + 1]);
        const double a3 = c.vcS, a4 = v.vcN;
        const double tterm = MUL(rT + rB, m.c_t);
        const double a0 = IMPL ? FMA(0.5, FeS - FwS, a1 + a2 + a3 + a4) + v.FbN - c.FbS + tterm
                               : a1 + a2 + a3 + a4 + tterm;
        const double bt = MUL(v.r1n + ci.r1O, m.c_t);
        const double bg = MUL(MUL(k.g_y, rT + rB), m.half_dV);
        const double bv = FMA(MUL(2.0 / 3.0, gB), u0E - o.uO,
                          FMA(MUL(-2.0 / 3.0, gT), uaE - o.uA,
                          FMA(-v.gcN, o.uA - o.uO, MUL(gcE, uaE - u0E))));
        const double b = FMA(k.B, bv, MUL(bt, v1n)) + bg;
        const double r = rcp(a0);
        const double sv = FMA(a4, o.vB, FMA(a3, o.vO, FMA(a2, vE, MUL(a1, vW))));
        v.vhatN = MUL(sv + (IMPL ? b : b + ven), r);
        v.dvN = MUL(m.A_dx, r);
    }
}

// stage D of one row
__device__ __forceinline__ void regk2_D(const MarchParams& m, int lc, const FluxRow& Fc, const double* UH,
                                        const double* DU, double* PN, const Own2& o, const Cin2& ci, Row2& v)
{
    const double dt = m.k.dt, dx = m.k.dx, dy = m.k.dy, dV = m.dV;
    const Carry& c = ci.c;
    const double rw = ci.ruO, re = Fc.RU[lc + 1], rsv = c.rvS, rn = v.rv1;
    const double duE = DU[lc + 1], uhE = UH[lc + 1];
    const double apW = MUL(MUL(rw, v.du), dy), bpW = MUL(MUL(rw, v.uhat), dy);
    const double apE = MUL(MUL(re, duE), dy), bpE = MUL(MUL(re, uhE), dy);
    const double apS = MUL(MUL(rsv, c.dvP), dx), bpS = MUL(MUL(rsv, c.vhatP), dx);
    const double apN = MUL(MUL(rn, v.dvN), dx), bpN = MUL(MUL(rn, v.vhatN), dx);
    const double sum = FMA(apN, o.pA, FMA(apS, o.pM, FMA(apE, v.p0E, MUL(apW, v.p0W))));
    const double bp = FMA(-(bpE - bpW + bpN - bpS), dt, MUL(ci.r1O, dV));
    v.pn = MUL(MUL(v.TN, FMA(sum, dt, bp)), rcp(FMA(MUL(v.TN, dt), apW + apE + apS + apN, dV)));
    PN[lc] = v.pn;
}

template <bool IMPL, bool TVD, bool GRAPH>
__device__ __forceinline__ void regk2_body(const MarchParams m)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Regk2Smem& s = *reinterpret_cast<Regk2Smem*>(smem_raw);
    const Params& k = m.k;
    int stop = 0;
    if (threadIdx.x == 0)
        stop = (GRAPH && *(volatile const int*)m.done) || *(volatile const unsigned long long*)m.bad != 0ull;
    if (__syncthreads_or(stop)) return;
    const int t = threadIdx.x;
    const int4 ce = m.order[blockIdx.x];
    const int strip = ce.x;
    const int I0 = k.gi0 + strip * MW;
    const int wbase = I0 - 4 - k.gi0 + OFF;
    const int shift = wbase & 3;
    const int c0 = wbase - shift;
    const bool tma = c0 + RW <= k.pitch;
    const int lc = t + 2 + shift;
    if (t == 0) {
        for (int q = 0; q < RS2; q++) mbar_init(&s.mbar[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int gi = I0 - 2 + t;
    const int J0 = ce.y, J1 = ce.z;
    const int js = J0 - WARM;
    const bool col_stored = stored_col(k, gi);
    const bool owner = t >= 2 && t < 2 + MW && gi < k.gi0 + k.nloc;
    // ring row r lives in slot (r - js + 1) & 7; its q-th fill completes phase (q >> 3) & 1
    auto RR = [&](int r) -> RingRow& { return s.ring[(r - js + 1) & (RS2 - 1)]; };
    for (int q = 0; q < 6; q++) ring_issue_tma(s, q, m, c0, tma, js - 1 + q, false);   // rows js-1 .. js+4
    cp_wait_all();
    __syncthreads();
    for (int q = 0; q < 4; q++) mbar_wait(&s.mbar[q], 0);                              // rows js-1 .. js+2
    for (int q = 0; q < 4; q++) ring_derive(s.ring[q]);
    __syncthreads();

    const int col = gi - k.gi0 + OFF;
    auto ld = [&](const double* a, int j) -> double {
        return (col_stored && j >= 0 && j < k.ny) ? __ldg(a + (j * k.pitch + col)) : 0.0;
    };
    auto ldv = [&](const double* a, int j) -> double {
        return (col_stored && j >= 0 && j <= k.ny) ? __ldg(a + (j * k.pitch + col)) : 0.0;
    };
    // n-1 values of the step's two rows (j, j+1): p^{n-1}, T^{n-1} of rows j+1, j+2;
    // T^{n-1}, u^{n-1} of rows j, j+1; v^{n-1} of rows j+1, j+2 (explicit: the planes)
    double p1a = ld(k.p_1, js + 1), p1b = ld(k.p_1, js + 2);
    double T1o = ld(k.T_1, js), T1a = ld(k.T_1, js + 1), T1b = ld(k.T_1, js + 2);
    double u1o = ld(k.u_1, js), u1a = ld(k.u_1, js + 1);
    double v1a = ldv(k.v_1, js + 1), v1b = ldv(k.v_1, js + 2);
    double Teo = 0.0, Tea = 0.0, ueo = 0.0, uea = 0.0, vea = 0.0, veb = 0.0;
    if (!IMPL) {
        Teo = ld(k.Te, js); Tea = ld(k.Te, js + 1); ueo = ld(k.ue, js); uea = ld(k.ue, js + 1);
        vea = ldv(k.ve, js + 1); veb = ldv(k.ve, js + 2);
    }
    // own-column registers carried between steps: rows j-1 (M), j (O) of u, p, T;
    // v of rows j, j+1; rho of rows j-1, j; Gamma of row j
    double uM = RR(js - 1).U[lc], uO = RR(js).U[lc];
    double pM = RR(js - 1).P[lc], pO = RR(js).P[lc];
    double tM = RR(js - 1).T[lc], tO = RR(js).T[lc];
    double vO = RR(js).V[lc], vA = RR(js + 1).V[lc];
    double rM = RR(js - 1).R[lc], rO = RR(js).R[lc], gO = RR(js).G[lc];
    Cin2 cl;
    cl.c = Carry{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 1.0, 0.0};
    cl.fxO = cl.fxE = cl.ruO = cl.r1O = 0.0;
    Resid rs{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, -1, 0, false};
    int oj = js * k.pitch + col;

    for (int j = js; j < J1; j += 2) {
        const int hi = j + 1;
        // prefetch the n-1 values of the next step (rows j+2, j+3)
        double np1a = 0.0, np1b = 0.0, nT1a = 0.0, nT1b = 0.0, nu1o = 0.0, nu1a = 0.0, nv1a = 0.0, nv1b = 0.0;
        double nTeo = 0.0, nTea = 0.0, nueo = 0.0, nuea = 0.0, nvea = 0.0, nveb = 0.0;
        {
            const unsigned o2 = (unsigned)(oj + 2 * k.pitch), o3 = o2 + (unsigned)k.pitch, o4 = o3 + (unsigned)k.pitch;
            const bool ok2 = col_stored && (unsigned)(j + 2) < (unsigned)k.ny;
            const bool ok3 = col_stored && (unsigned)(j + 3) < (unsigned)k.ny;
            const bool ok4 = col_stored && (unsigned)(j + 4) < (unsigned)k.ny;
            const bool ok3v = col_stored && (unsigned)(j + 3) <= (unsigned)k.ny;
            const bool ok4v = col_stored && (unsigned)(j + 4) <= (unsigned)k.ny;
            if (ok2) nu1o = __ldg(k.u_1 + o2);
            if (ok3) { np1a = __ldg(k.p_1 + o3); nT1a = __ldg(k.T_1 + o3); nu1a = __ldg(k.u_1 + o3); }
            if (ok4) { np1b = __ldg(k.p_1 + o4); nT1b = __ldg(k.T_1 + o4); }
            if (ok3v) nv1a = __ldg(k.v_1 + o3);
            if (ok4v) nv1b = __ldg(k.v_1 + o4);
            if (!IMPL) {
                if (ok2) { nTeo = __ldg(k.Te + o2); nueo = __ldg(k.ue + o2); }
                if (ok3) { nTea = __ldg(k.Te + o3); nuea = __ldg(k.ue + o3); }
                if (ok3v) nvea = __ldg(k.ve + o3);
                if (ok4v) nveb = __ldg(k.ve + o4);
            }
        }
        {
            // rows j+5, j+6 -> their slots (TMA, one step ahead); rows j+3, j+4 landed -> derive
            const int q = j + 6 - js;          // ring offset of row j+5
            ring_issue_tma(s, q & (RS2 - 1), m, c0, tma, j + 5, false);
            ring_issue_tma(s, (q + 1) & (RS2 - 1), m, c0, tma, j + 6, false);
            mbar_wait(&s.mbar[(q - 2) & (RS2 - 1)], ((q - 2) >> 3) & 1);
            mbar_wait(&s.mbar[(q - 1) & (RS2 - 1)], ((q - 1) >> 3) & 1);
        }
        ring_derive(RR(j + 3));
        ring_derive(RR(j + 4));
        RingRow& Rm = RR(j - 1);
        RingRow& R0 = RR(j);
        RingRow& Ra = RR(j + 1);
        RingRow& Rb = RR(j + 2);
        RingRow& Rc = RR(j + 3);
        FluxRow& F0 = s.fr[j & 3];
        FluxRow& F1 = s.fr[(j + 1) & 3];
        FluxRow& F2 = s.fr[(j + 2) & 3];
        const int bl = j & 1, bh = hi & 1;
        // own values of the step's rows
        Own2 ol, oh;
        ol.uM = uM; ol.uO = uO; ol.uA = Ra.U[lc];
        ol.pM = pM; ol.pO = pO; ol.pA = Ra.P[lc];
        ol.tM = tM; ol.tO = tO; ol.tA = Ra.T[lc];
        ol.vO = vO; ol.vA = vA; ol.vB = Rb.V[lc];
        ol.rM = rM; ol.rO = rO; ol.rA = Ra.R[lc];
        ol.gO = gO; ol.gA = Ra.G[lc];
        oh.uM = uO; oh.uO = ol.uA; oh.uA = Rb.U[lc];
        oh.pM = pO; oh.pO = ol.pA; oh.pA = Rb.P[lc];
        oh.tM = tO; oh.tO = ol.tA; oh.tA = Rb.T[lc];
        oh.vO = vA; oh.vA = ol.vB; oh.vB = Rc.V[lc];
        oh.rM = rO; oh.rO = ol.rA; oh.rA = Rb.R[lc];
        oh.gO = ol.gA; oh.gA = Rb.G[lc];
        if (TVD) {
            ol.rB = oh.rA; ol.tB = oh.tA; ol.uB = oh.uA; ol.vC = oh.vB;
            oh.rB = Rc.R[lc]; oh.tB = Rc.T[lc]; oh.uB = Rc.U[lc]; oh.vC = RR(j + 4).V[lc];
        } else {
            ol.rB = ol.tB = ol.uB = ol.vC = oh.rB = oh.tB = oh.uB = oh.vC = 0.0;
        }

        // ---- stage A of both rows
        Row2 vl, vh;
        regk2_A<IMPL, TVD>(m, lc, R0, Ra, F1, s.XTW[bl], s.XUW[bl], s.XVW[bl], ol, cl, p1a, T1a, vl);
        s.R1[bh][lc] = vl.r1n;                              // (p/T)^{n-1} of row j+1 (read by C of the hi row)
        Cin2 ch;
        ch.fxO = vl.Fx1; ch.ruO = vl.ru; ch.r1O = vl.r1n;
        regk2_A<IMPL, TVD>(m, lc, Ra, Rb, F2, s.XTW[bh], s.XUW[bh], s.XVW[bh], oh, ch, p1b, T1b, vh);
        __syncthreads();                                    // B1
        // ---- stage C of both rows (the hi row takes the lo row's carries)
        regk2_C<IMPL, TVD>(m, lc, Rm, R0, Ra, F1, s.XTW[bl], s.XUW[bl], s.XVW[bl], s.R1[bl], s.UH[bl], s.DU[bl],
                           ol, cl, T1o, u1o, v1a, Teo, ueo, vea, vl);
        ch.fxE = vl.fxnE;
        ch.c.ytS = vl.ytSn; ch.c.FS = vl.Fy1;
        ch.c.utS = vl.utSn; ch.c.FsSum = vl.FsSumN;
        ch.c.vcS = vl.vcSn; ch.c.FbS = vl.FbN;
        ch.c.vhatP = vl.vhatN; ch.c.dvP = vl.dvN;
        ch.c.gcP = vl.gcN; ch.c.rvS = vl.rv1;
        ch.c.pnP = 0.0;                                     // set after the lo row's stage D
        regk2_C<IMPL, TVD>(m, lc, R0, Ra, Rb, F2, s.XTW[bh], s.XUW[bh], s.XVW[bh], s.R1[bh], s.UH[bh], s.DU[bh],
                           oh, ch, T1a, u1a, v1b, Tea, uea, veb, vh);
        __syncthreads();                                    // B2
        // ---- stage D of both rows
        regk2_D(m, lc, F0, s.UH[bl], s.DU[bl], s.PN[bl], ol, cl, vl);
        ch.c.pnP = vl.pn;
        regk2_D(m, lc, F1, s.UH[bh], s.DU[bh], s.PN[bh], oh, ch, vh);
        cp_wait_all();
        __syncthreads();                                    // B3
        // ---- stage E of both rows
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int row = j + h;
            const Own2& o = h ? oh : ol;
            const Cin2& ci = h ? ch : cl;
            const Row2& v = h ? vh : vl;
            const double* PN = s.PN[h ? bh : bl];
            if (row >= J0 && row < J1 && owner) {
                const int id = row * k.pitch + col;
                const double TN = v.TN, pn = v.pn;
                k.T_w[id] = TN;
                k.p_w[id] = pn;
                rs.dT = dmax(rs.dT, fabs(TN - o.tO));
                rs.dp = dmax(rs.dp, fabs(pn - o.pO));
                rs.T = dmax(rs.T, fabs(TN));
                rs.p = dmax(rs.p, fabs(pn));
                if (!(TN > 0.0) || !(pn > 0.0) || !isfinite(TN) || !isfinite(pn)) {
                    const long long flat = (long long)row * k.nx + gi;
                    if (rs.bad < 0 || flat < rs.bad) { rs.bad = flat; rs.badf = (!(TN > 0.0) || !isfinite(TN)) ? 3 : 2; }
                }
                const double un = FMA(-v.du, pn - PN[lc - 1], v.uhat);
                rs.du = dmax(rs.du, fabs(un - o.uO));
                rs.vel = dmax(rs.vel, fabs(un));
                rs.nanv |= un != un;
                k.u_w[id] = un;
                const double vn = FMA(-ci.c.dvP, pn - ci.c.pnP, ci.c.vhatP);
                rs.dv = dmax(rs.dv, fabs(vn - o.vO));
                rs.vel = dmax(rs.vel, fabs(vn));
                rs.nanv |= vn != vn;
                k.v_w[id] = vn;
                if (k.mirror) {
                    int tgt = -1000;
                    if (gi < OFF) tgt = gi + k.nx;
                    else if (gi >= k.nx - OFF) tgt = gi - k.nx;
                    if (tgt > -1000) {
                        const int tt = row * k.pitch + (tgt - k.gi0 + OFF);
                        k.p_w[tt] = pn; k.T_w[tt] = TN;
                        k.u_w[tt] = un;
                        k.v_w[tt] = vn;
                    }
                }
            }
        }
        s.R1[bl][lc] = vh.r1n;                              // (p/T)^{n-1} of row j+2 (C of the next step's lo row)
        // ---- carry rows j+2 (next lo) quantities
        cl.c.ytS = vh.ytSn; cl.c.FS = vh.Fy1;
        cl.c.utS = vh.utSn; cl.c.FsSum = vh.FsSumN;
        cl.c.vcS = vh.vcSn; cl.c.FbS = vh.FbN;
        cl.c.vhatP = vh.vhatN; cl.c.dvP = vh.dvN;
        cl.c.pnP = vh.pn; cl.c.gcP = vh.gcN; cl.c.rvS = vh.rv1;
        cl.fxO = vh.Fx1; cl.fxE = vh.fxnE; cl.ruO = vh.ru; cl.r1O = vh.r1n;
        uM = oh.uO; uO = oh.uA; pM = oh.pO; pO = oh.pA; tM = oh.tO; tO = oh.tA;
        vO = oh.vA; vA = oh.vB; rM = oh.rO; rO = oh.rA; gO = oh.gA;
        p1a = np1a; p1b = np1b;
        T1o = T1b; T1a = nT1a; T1b = nT1b;
        u1o = nu1o; u1a = nu1a;
        v1a = nv1a; v1b = nv1b;
        if (!IMPL) { Teo = nTeo; Tea = nTea; ueo = nueo; uea = nuea; vea = nvea; veb = nveb; }
        oj += 2 * k.pitch;
    }
    // the last step's TMA rows (j+5, j+6) land before the CTA's shared memory is released
    {
        const int jl = js + 2 * ((J1 - js + 1) / 2) - 2;   // lo row of the last step
        const int q = jl + 6 - js;
        mbar_wait(&s.mbar[q & (RS2 - 1)], (q >> 3) & 1);
        mbar_wait(&s.mbar[(q + 1) & (RS2 - 1)], ((q + 1) >> 3) & 1);
    }
    cp_wait_all();
    const double qnan = __longlong_as_double(0x7ff8000000000000LL);
    double vals[7] = {rs.nanv ? qnan : rs.du, rs.nanv ? qnan : rs.dv, rs.dp, rs.dT, rs.vel, rs.p, rs.T};
    __syncthreads();
    __shared__ double part[MX / 32][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int q = 0; q < 7; q++) {
        double val = vals[q];
        const bool isn = val != val;
        const unsigned nanmask = __ballot_sync(0xffffffffu, isn);
        val = warp_max(isn ? 0.0 : val);
        if (nanmask) val = __longlong_as_double(0x7ff8000000000000LL);
        if (lane == 0) part[wid][q] = val;
    }
    __syncthreads();
    if (threadIdx.x < 7) {
        double val = 0.0;
        for (int w = 0; w < MX / 32; w++) val = nmax(val, part[w][threadIdx.x]);
        atomicMax(&k.red[threadIdx.x], (unsigned long long)__double_as_longlong(val));
    }
    if (rs.bad >= 0 || rs.nanv) {
        const long long flat = rs.bad >= 0 ? rs.bad : BAD_NOCELL;
        atomicMax(m.bad, bad_key(m.pass_key, flat, rs.bad >= 0 ? rs.badf : 0));
    }
}

#ifndef STS_REGK2_CTAS
#define STS_REGK2_CTAS 2
#endif
template <bool IMPL, bool TVD, bool GRAPH>
__global__ void __launch_bounds__(MX, STS_REGK2_CTAS) regk2_kernel(MarchParams m)
{
    regk2_body<IMPL, TVD, GRAPH>(m);
}

}  // namespace sts
#undef STS_LINK
