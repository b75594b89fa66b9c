// sts_regk.cuh -- the all-regular march kernel, register-resident (round 2, v10).
//
// Same pass, same CTAs, same ring and TMA rows as march_kernel<..., REGK = true>
// (sts_march.cuh): the CTAs whose every point (warm-up rows included) is a
// regular fluid point, marching along y.  The regular stage
// instances are restated here with the operands held in registers instead of
// re-read from shared memory:
//  - ncu (profiles/r02_summary.md) shows the REGK kernel bound by the L1/shared
//    data pipe (LSU wavefronts 81 % of peak, 88 LDS.64 per point per row step):
//    a __syncthreads() is a compiler memory fence, so every ring value used in
//    two stages of a row step was loaded twice, and own-column values written by
//    the thread itself (F^x, rho^u, (p/T)^{n-1}, the T-eq W coefficient) were
//    read back from shared memory;
//  - here the own column's u, p, T (rows j-1, j, j+1), v (rows j, j+1, j+2) and
//    rho, Gamma (rows j, j+1) rotate through registers down the march, the
//    own-column face values a thread produces are kept, and every neighbour
//    value is loaded once per row step: ~34 shared loads per point (upwind)
//    instead of 88.
// Every formula is the REG instance's of sts_march.cuh with the same operands in
// the same order (same bits: the general kernel's regular points, the segment
// and slab bitwise tests, and test_regk_same_bits compare them).
#pragma once

#include "sts_march.cuh"

namespace sts {

#define STS_LINK(F, ps) (TVD ? FMA(-(F), (ps), max0(F)) : max0(F))

#ifndef STS_REGK_CTAS
#define STS_REGK_CTAS 3
#endif

template <bool IMPL, bool TVD, bool GRAPH>
__device__ __forceinline__ void regk_body(const MarchParams m)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MarchSmem& s = *reinterpret_cast<MarchSmem*>(smem_raw);
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
        for (int q = 0; q < RS; q++) mbar_init(&s.mbar[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int gi = I0 - 2 + t;
    const int J0 = ce.y, J1 = ce.z;
    const int js = J0 - WARM;
    const bool col_stored = stored_col(k, gi);
    const bool owner = t >= 2 && t < 2 + MW && gi < k.gi0 + k.nloc;

    RingRow *pm = &s.ring[0], *p0 = &s.ring[1], *pa = &s.ring[2], *pb = &s.ring[3], *pc = &s.ring[4], *pd = &s.ring[5];
    for (int q = 0; q < 5; q++) ring_issue_tma(s, q, m, c0, tma, js - 1 + q, false);
    cp_wait_all();
    __syncthreads();
    for (int q = 0; q < 4; q++) mbar_wait(&s.mbar[q], 0);
    ring_derive(*pm);
    ring_derive(*p0);
    ring_derive(*pa);
    ring_derive(*pb);
    __syncthreads();

    const int col = gi - k.gi0 + OFF;
    auto ld = [&](const double* a, int j) -> double {
        return (col_stored && j >= 0 && j < k.ny) ? __ldg(a + (j * k.pitch + col)) : 0.0;
    };
    auto ldv = [&](const double* a, int j) -> double {
        return (col_stored && j >= 0 && j <= k.ny) ? __ldg(a + (j * k.pitch + col)) : 0.0;
    };
    NM1 nm;
    nm.Tec = nm.uec = nm.ven = 0.0;
    nm.p1n = ld(k.p_1, js + 1); nm.T1n = ld(k.T_1, js + 1);
    nm.T1c = ld(k.T_1, js); nm.u1c = ld(k.u_1, js); nm.v1n = ldv(k.v_1, js + 1);
    if (!IMPL) { nm.Tec = ld(k.Te, js); nm.uec = ld(k.ue, js); nm.ven = ldv(k.ve, js + 1); }

    // own-column registers: u, p, T of rows j-1 (M), j (O); v of rows j (O), j+1 (A);
    // rho, Gamma of row j (rho also j-1 for TVD)
    double uM = pm->U[lc], uO = p0->U[lc];
    double pM = pm->P[lc], pO = p0->P[lc];
    double tM = pm->T[lc], tO = p0->T[lc];
    double vO = p0->V[lc], vA = pa->V[lc];
    double rM = pm->R[lc], rO = p0->R[lc], gO = p0->G[lc];
    // own-column face values of row j (written by this thread one step earlier) and
    // F^x(i+1, j) (read as the v-equation's E flux one step earlier); the warm-up
    // rows flush their initial values (WARM, sts_march.cuh)
    double fxO = 0.0, fxE = 0.0, ruO = 0.0, r1O = 0.0;
    Carry c{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 1.0, 0.0};
    Resid rs{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, -1, 0, false};
    int oj = js * k.pitch + col;
    const double dt = k.dt, dx = k.dx, dy = k.dy, dV = m.dV;

#if defined(STS_REGK_UNROLL) && STS_REGK_UNROLL == 2
#pragma unroll 2
#elif defined(STS_REGK_UNROLL) && STS_REGK_UNROLL == 3
#pragma unroll 3
#endif
    for (int j = js; j < J1; j++) {
        RingRow& Rm = *pm;
        RingRow& R0 = *p0;
        RingRow& Ra = *pa;
        RingRow& Rb = *pb;
        RingRow& Rc = *pc;
        FluxRow& Fn = s.fr[(j + 1) & 1];
        const FluxRow& Fc = s.fr[j & 1];

        double p1nn = 0.0, T1nn = 0.0, u1n = 0.0, v1nn = 0.0, Ten = 0.0, uen = 0.0, vem = 0.0;
        {
            const unsigned o1 = (unsigned)(oj + k.pitch), o2 = o1 + (unsigned)k.pitch;
            const bool ok1 = col_stored && (unsigned)(j + 1) < (unsigned)k.ny;
            const bool ok2 = col_stored && (unsigned)(j + 2) < (unsigned)k.ny;
            const bool ok2v = col_stored && (unsigned)(j + 2) <= (unsigned)k.ny;
            if (ok2) { p1nn = __ldg(k.p_1 + o2); T1nn = __ldg(k.T_1 + o2); }
            if (ok1) u1n = __ldg(k.u_1 + o1);
            if (ok2v) v1nn = __ldg(k.v_1 + o2);
            if (!IMPL) {
                if (ok1) { Ten = __ldg(k.Te + o1); uen = __ldg(k.ue + o1); }
                if (ok2v) vem = __ldg(k.ve + o2);
            }
        }
        {
            const int q = j + 4 - js;
            ring_issue_tma(s, (q + 1) % RS, m, c0, tma, j + 4, false);
            mbar_wait(&s.mbar[q % RS], (q / RS) & 1);
        }
        ring_derive(Rc);
        // newest own-column values: u, p, T, rho, Gamma of row j+1, v of row j+2
        const double uA = Ra.U[lc], pA = Ra.P[lc], tA = Ra.T[lc], rA = Ra.R[lc], gA = Ra.G[lc];
        const double vB = Rb.V[lc];

        // ================= stage A (sts_march.cuh stage_A, REG) =================
        const double r1n = fdiv(nm.p1n, nm.T1n == 0.0 ? 1.0 : nm.T1n);
        const double raW = Ra.R[lc - 1], g0W = R0.G[lc - 1], gaW = Ra.G[lc - 1], u0E = R0.U[lc + 1];
        double t0W, t0E, u0W, vaW, vaE;
        if (TVD) { t0W = R0.T[lc - 1]; t0E = R0.T[lc + 1]; u0W = R0.U[lc - 1]; vaW = Ra.V[lc - 1]; vaE = Ra.V[lc + 1]; }
        double Fx1, ru;
        {
            const double w = uA, r1 = raW, r2 = rA;
            ru = w > 0.0 ? r1 : r2;
            if (TVD) ru = FMA(psi_f(Ra.R[lc - 2], r1, r2, Ra.R[lc + 1], w), r2 - r1, ru);
            Fx1 = MUL(MUL(ru, w), dy);
            Fn.RU[lc] = ru;
            Fn.FX[lc] = Fx1;
        }
        double Fy1, rv1;
        {
            const double w = vA, r1 = rO, r2 = rA;
            rv1 = w > 0.0 ? r1 : r2;
            if (TVD) rv1 = FMA(psi_f(rM, r1, r2, Rb.R[lc], w), r2 - r1, rv1);
            Fy1 = MUL(MUL(rv1, w), dx);
            Fn.FY[lc] = Fy1;
        }
        double xtw;
        {
            const double F = fxO;
            const double g1 = g0W, g2 = gO;
            const double hg = MUL(MUL(MUL(2.0, g1), g2), rcp(g1 + g2));
            double ps = 0.0;
            if (IMPL && TVD) ps = psi_f(R0.T[lc - 2], t0W, tO, t0E, uO);
            xtw = FMA(m.CT1_dydx, hg, IMPL ? STS_LINK(F, ps) : 0.0);
            s.XTW[lc] = xtw;
        }
        double ytN, ytSn;
        {
            const double F = Fy1;
            const double g1 = gO, g2 = gA;
            const double hg = MUL(MUL(MUL(2.0, g1), g2), rcp(g1 + g2));
            double ps = 0.0;
            if (IMPL && TVD) ps = psi_f(tM, tO, tA, Rb.T[lc], vA);
            ytSn = FMA(m.CT1_dxdy, hg, IMPL ? STS_LINK(F, ps) : 0.0);
            ytN = IMPL ? ytSn - F : ytSn;
        }
        double xe, Fb;
        {
            const double ub = MUL(0.5, uO + u0E);
            Fb = MUL(MUL(rO, ub), dy);
            double ps = 0.0;
            if (IMPL && TVD) ps = psi_f(u0W, uO, u0E, R0.U[lc + 2], ub);
            const double xw = FMA(m.B43_dydx, gO, IMPL ? STS_LINK(Fb, ps) : 0.0);
            xe = IMPL ? xw - Fb : xw;
            s.XUW[lc] = xw;
        }
        double upsi1 = 0.0, upsi2 = 0.0;
        if (IMPL && TVD) {
            const double f4 = Rb.U[lc];
            upsi1 = psi_f(uM, uO, uA, f4, vA);
            upsi2 = psi_f(uM, uO, uA, f4, vaW);
        }
        double vcN, vcSn, FbN;
        {
            const double vb = MUL(0.5, vA + vB);
            FbN = MUL(MUL(rA, vb), dx);
            double ps = 0.0;
            if (IMPL && TVD) ps = psi_f(vO, vA, vB, Rc.V[lc], vb);
            vcSn = FMA(m.B43_dxdy, gA, IMPL ? STS_LINK(FbN, ps) : 0.0);
            vcN = IMPL ? vcSn - FbN : vcSn;
        }
        const double gcN = MUL(0.25, g0W + gO + gaW + gA);
        double xvW, FwSum;
        {
            const double F1 = Fx1, F2 = fxO;
            double p1 = 0.0, p2 = 0.0;
            if (IMPL && TVD) {
                const double f1 = Ra.V[lc - 2];
                p1 = psi_f(f1, vaW, vA, vaE, uA);
                p2 = psi_f(f1, vaW, vA, vaE, uO);
            }
            FwSum = F1 + F2;
            const double lk = IMPL ? MUL(0.5, STS_LINK(F1, p1) + STS_LINK(F2, p2)) : 0.0;
            xvW = FMA(m.B_dydx, gcN, lk);
            s.XVW[lc] = xvW;
        }
        // ring values of stage C: the rows do not change during the step, so the implicit
        // variants load the first ones before the barrier and hide their latency behind it
        // (implicit upwind +1.6 %, explicit upwind -0.4 %: explicit loads them after)
        double p0W, p0E;
        if (IMPL) {
            if (!TVD) { t0W = R0.T[lc - 1]; t0E = R0.T[lc + 1]; u0W = R0.U[lc - 1]; vaW = Ra.V[lc - 1]; vaE = Ra.V[lc + 1]; }
            p0W = R0.P[lc - 1]; p0E = R0.P[lc + 1];
        }
        __syncthreads();                                    // B1

        // ================= stage C (stage_C, REG) =================
        if (!IMPL) {
            if (!TVD) { t0W = R0.T[lc - 1]; t0E = R0.T[lc + 1]; u0W = R0.U[lc - 1]; vaW = Ra.V[lc - 1]; vaE = Ra.V[lc + 1]; }
            p0W = R0.P[lc - 1]; p0E = R0.P[lc + 1];
        }
        const double v0W = R0.V[lc - 1], v0E = R0.V[lc + 1];
        const double uaE = Ra.U[lc + 1], umE = Rm.U[lc + 1];
        const double xtwE = s.XTW[lc + 1], fyW = Fn.FY[lc - 1], xuwW = s.XUW[lc - 1], r1W = s.R1[lc - 1];
        const double fxnE = Fn.FX[lc + 1], xvwE = s.XVW[lc + 1];
        double TN;
        {
            const double a1 = xtw, FW = fxO, T1 = t0W;
            const double FE = fxE, a2 = IMPL ? xtwE - FE : xtwE, T2 = t0E;
            const double a3 = c.ytS, FSl = c.FS, T3 = tM;
            const double a4 = ytN, FNl = Fy1, T4 = tA;
            const double rq = rO;
            const double a0 = IMPL ? FMA(dt, a1 + a2 + a3 + a4 + FE - FW + FNl - FSl, MUL(rq, dV))
                                   : FMA(dt, a1 + a2 + a3 + a4, MUL(rq, dV));
            const double rdx = m.inv_dx, rdy = m.inv_dy;
            const double dudx = MUL(u0E - uO, rdx);
            const double dvdy = MUL(vA - vO, rdy);
            const double shear = FMA((v0E + vaE) - (v0W + vaW), m.q_dx, MUL((uA + uaE) - (uM + umE), m.q_dy));
            const double div = dudx + dvdy;
            const double pc = pO;
            const double p1 = MUL(r1O, nm.T1c);
            const double dpx = MUL(p0E - p0W, m.h_dx);
            const double dpy = MUL(pA - pM, m.h_dy);
            const double ub = MUL(0.5, uO + u0E), vb = MUL(0.5, vO + vA);
            const double pwork = FMA(m.pw_a, FMA(vb, dpy, FMA(ub, dpx, MUL(pc - p1, m.inv_dt))), MUL(MUL(k.pwk, pc), div));
            const double Phi = FMA(MUL(-2.0 / 3.0, div), div, FMA(shear, shear, MUL(2.0, FMA(dvdy, dvdy, MUL(dudx, dudx)))));
            const double Sc = MUL(FMA(MUL(k.CT2, gO), Phi, pwork), dV);
            const double sT = FMA(a4, T4, FMA(a3, T3, FMA(a2, T2, MUL(a1, T1))));
            const double rhs = FMA(dt, sT + (IMPL ? Sc : Sc + nm.Tec), MUL(p1, dV));
            TN = MUL(rhs, rcp(a0));
        }
        double uhat, du, utSn, FsSumN;
        {
            const double F1 = Fy1, F2 = fyW;
            FsSumN = F1 + F2;
            const double lk = IMPL ? MUL(0.5, STS_LINK(F1, upsi1) + STS_LINK(F2, upsi2)) : 0.0;
            utSn = FMA(m.B_dxdy, gcN, lk);
            const double a4p = IMPL ? FMA(-0.5, FsSumN, utSn) : utSn;
            const double rL = R0.R[lc - 1], rR = rO, gL = g0W, gR = gO;
            const double a1 = xuwW, a2 = xe;
            const double FbW = MUL(MUL(rL, MUL(0.5, u0W + uO)), dy), FbE = Fb;
            const double a3 = c.utS, FsS = c.FsSum, uS = uM;
            const double a4 = a4p, FnS = FsSumN, uN = uA;
            const double tterm = MUL(rR + rL, m.c_t);
            const double a0 = IMPL ? FMA(0.5, FnS - FsS, a1 + a2 + a3 + a4 + FbE - FbW) + tterm
                                   : a1 + a2 + a3 + a4 + tterm;
            const double bt = MUL(r1O + r1W, m.c_t);
            const double bg = MUL(MUL(k.g_x, rR + rL), m.half_dV);
            const double bv = FMA(MUL(2.0 / 3.0, gL), vaW - v0W,
                              FMA(MUL(-2.0 / 3.0, gR), vA - vO,
                              FMA(-c.gcP, vO - v0W, MUL(gcN, vA - vaW))));
            const double b = FMA(k.B, bv, MUL(bt, nm.u1c)) + bg;
            const double r = rcp(a0);
            const double su = FMA(a4, uN, FMA(a3, uS, FMA(a2, u0E, MUL(a1, u0W))));
            uhat = MUL(su + (IMPL ? b : b + nm.uec), r);
            du = MUL(m.A_dy, r);
            s.UH[lc] = uhat;
            s.DU[lc] = du;
        }
        double vhatN, dvN;
        {
            const double rB = rO, rT = rA, gB = gO, gT = gA;
            const double a1 = xvW, FwS = FwSum, vW = vaW;
            const double FeS = fxnE + fxE, a2 = IMPL ? FMA(-0.5, FeS, xvwE) : xvwE, vE = vaE;
            const double gcE = MUL(0.25, gO + R0.G[lc + 1] + gA + Ra.G[lc + 1]);
            const double a3 = c.vcS, a4 = vcN;
            const double tterm = MUL(rT + rB, m.c_t);
            const double a0 = IMPL ? FMA(0.5, FeS - FwS, a1 + a2 + a3 + a4) + FbN - c.FbS + tterm
                                   : a1 + a2 + a3 + a4 + tterm;
            const double bt = MUL(r1n + r1O, m.c_t);
            const double bg = MUL(MUL(k.g_y, rT + rB), m.half_dV);
            const double bv = FMA(MUL(2.0 / 3.0, gB), u0E - uO,
                              FMA(MUL(-2.0 / 3.0, gT), uaE - uA,
                              FMA(-gcN, uA - uO, MUL(gcE, uaE - u0E))));
            const double b = FMA(k.B, bv, MUL(bt, nm.v1n)) + bg;
            const double r = rcp(a0);
            const double sv = FMA(a4, vB, FMA(a3, vO, FMA(a2, vE, MUL(a1, vW))));
            vhatN = MUL(sv + (IMPL ? b : b + nm.ven), r);
            dvN = MUL(m.A_dx, r);
        }
        __syncthreads();                                    // B2

        // ================= stage D (stage_D, REG) =================
        double pn;
        {
            const double rw = ruO, re = Fc.RU[lc + 1], rsv = c.rvS, rn = rv1;
            const double duE = s.DU[lc + 1], uhE = s.UH[lc + 1];
            const double apW = MUL(MUL(rw, du), dy), bpW = MUL(MUL(rw, uhat), dy);
            const double apE = MUL(MUL(re, duE), dy), bpE = MUL(MUL(re, uhE), dy);
            const double apS = MUL(MUL(rsv, c.dvP), dx), bpS = MUL(MUL(rsv, c.vhatP), dx);
            const double apN = MUL(MUL(rn, dvN), dx), bpN = MUL(MUL(rn, vhatN), dx);
            const double sum = FMA(apN, pA, FMA(apS, pM, FMA(apE, p0E, MUL(apW, p0W))));
            const double bp = FMA(-(bpE - bpW + bpN - bpS), dt, MUL(r1O, dV));
            pn = MUL(MUL(TN, FMA(sum, dt, bp)), rcp(FMA(MUL(TN, dt), apW + apE + apS + apN, dV)));
            s.PN[lc] = pn;
        }
        cp_wait_all();
        __syncthreads();                                    // B3

        // ================= stage E (stage_E, REG) =================
        if (j >= J0 && owner) {
            const int id = j * k.pitch + col;
            k.T_w[id] = TN;
            k.p_w[id] = pn;
            rs.dT = dmax(rs.dT, fabs(TN - tO));
            rs.dp = dmax(rs.dp, fabs(pn - pO));
            rs.T = dmax(rs.T, fabs(TN));
            rs.p = dmax(rs.p, fabs(pn));
            if (!(TN > 0.0) || !(pn > 0.0) || !isfinite(TN) || !isfinite(pn)) {
                const long long flat = (long long)j * k.nx + gi;
                if (rs.bad < 0 || flat < rs.bad) { rs.bad = flat; rs.badf = (!(TN > 0.0) || !isfinite(TN)) ? 3 : 2; }
            }
            const double un = FMA(-du, pn - s.PN[lc - 1], uhat);
            rs.du = dmax(rs.du, fabs(un - uO));
            rs.vel = dmax(rs.vel, fabs(un));
            rs.nanv |= un != un;
            k.u_w[id] = un;
            const double vn = FMA(-c.dvP, pn - c.pnP, c.vhatP);
            rs.dv = dmax(rs.dv, fabs(vn - vO));
            rs.vel = dmax(rs.vel, fabs(vn));
            rs.nanv |= vn != vn;
            k.v_w[id] = vn;
            if (k.mirror) {                              // single-rank periodic: wrapped ghosts
                int tgt = -1000;
                if (gi < OFF) tgt = gi + k.nx;
                else if (gi >= k.nx - OFF) tgt = gi - k.nx;
                if (tgt > -1000) {
                    const int tt = j * k.pitch + (tgt - k.gi0 + OFF);
                    k.p_w[tt] = pn; k.T_w[tt] = TN;
                    k.u_w[tt] = un;
                    k.v_w[tt] = vn;
                }
            }
        }
        s.R1[lc] = r1n;
        // ---- carry row j+1 quantities to the next step
        c.ytS = ytSn; c.FS = Fy1;
        c.utS = utSn; c.FsSum = FsSumN;
        c.vcS = vcSn; c.FbS = FbN;
        c.vhatP = vhatN; c.dvP = dvN;
        c.pnP = pn; c.gcP = gcN; c.rvS = rv1;
        fxO = Fx1; fxE = fxnE; ruO = ru; r1O = r1n;
        uM = uO; uO = uA; pM = pO; pO = pA; tM = tO; tO = tA;
        vO = vA; vA = vB; rM = rO; rO = rA; gO = gA;
        nm.p1n = p1nn; nm.T1c = nm.T1n; nm.T1n = T1nn; nm.u1c = u1n; nm.v1n = v1nn;
        if (!IMPL) { nm.Tec = Ten; nm.uec = uen; nm.ven = vem; }
        RingRow* const pf = pm;
        pm = p0; p0 = pa; pa = pb; pb = pc; pc = pd; pd = pf;
        oj += k.pitch;
    }
    {   // the last step's TMA row (J1 + 3) lands before the CTA's shared memory is released
        const int qo = J1 + 4 - js;
        mbar_wait(&s.mbar[qo % RS], (qo / RS) & 1);
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
template <bool IMPL, bool TVD, bool GRAPH>
__global__ void __launch_bounds__(MX, STS_REGK_CTAS) regk_kernel(MarchParams m)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");                 // PDL: see march_fused_kernel
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    regk_body<IMPL, TVD, GRAPH>(m);
}

// One launch per loop-2 pass: the CTA schedule (order[], general CTAs first) runs
// the general CTAs through march_body and the all-regular ones through regk_body
// (implicit TVD: march_body<REGK>), so the general CTAs are dispatched first
// inside a graph too (two parallel kernel nodes left their order to the hardware:
// the general CTAs could queue behind the regular grid and form the pass's tail),
// and the general code runs with the all-regular kernel's register budget (no
// spills).  Same instance code per CTA as the two-kernel launch: same bits.
template <bool IMPL, bool TVD, bool GRAPH>
__global__ void __launch_bounds__(MX, STS_REGK_CTAS) march_fused_kernel(MarchParams m)
{
    // Programmatic dependent launch (fixed-pass step graphs, §5.5): the pass may be
    // launched while the previous pass drains; every read of its outputs comes after
    // this wait (which returns once the previous grid has completed and its writes
    // are visible), and the next pass is released only after it.  No-ops without a
    // programmatic edge (stream launches).
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (m.order[blockIdx.x].w & ALLREG_BIT) {
        if (IMPL && TVD) march_body<IMPL, TVD, GRAPH, true>(m);
        else regk_body<IMPL, TVD, GRAPH>(m);
    } else {
        march_body<IMPL, TVD, GRAPH, false>(m);
    }
}

}  // namespace sts
#undef STS_LINK
