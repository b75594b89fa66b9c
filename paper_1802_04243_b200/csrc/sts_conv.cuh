// sts_conv.cuh -- explicit convective planes u^exp, v^exp, T^exp as a y-march
// (once per time step, explicit schemes).
//
// Every plane is a difference of face-value fluxes of the n-1 state
// (Eqs. pl15_11, pl31_1 and the transposed u-plane, DESIGN 3.4):
//   T^exp(i,j) = TX(i,j) - TX(i+1,j) + TY(i,j) - TY(i,j+1),
//     TX(face) = F^x [upwind(T_W, T_E, u) + psi_s (T_E - T_W)], TY likewise;
//   u^exp(i,j) = uX(i-1,j) - uX(i,j) + uY(i,j) - uY(i,j+1),
//     uX(cell c) = dy rho_c ubar_c [upwind(u_c, u_{c+1}, ubar_c) + psi_c (...)],
//     uY(i, y^f_j) = 1/2 sum over the half faces (i-1, j), (i, j) of F^y [...];
//   v^exp(i,j) = vX(i,j) - vX(i+1,j) + vY(i,j-1) - vY(i,j)   (the mirror).
// Each flux is computed once per face (x neighbours through shared memory,
// y neighbours through a carried register), as in the pass kernel.
#pragma once

#include <type_traits>

#include "sts_march.cuh"

namespace sts {

struct RingRowC {                // n-1 row of the conv kernel: no Gamma (the planes need none)
    double U[RW], V[RW], P[RW], T[RW], R[RW];
    uint32_t KK[RW];
};
static_assert(sizeof(RingRowC) % 16 == 0, "TMA rows need 16-byte alignment");
// 43.6 KB: five CTAs (20 warps) per SM
struct ConvSmem {
    RingRowC ring[RS];
    double FX[2][RW], FY[2][RW];     // fluxes rows j (cur) / j+1 (nxt)
    double TX[RW], UX[RW], VX[RW];
    unsigned long long mbar[RS];     // TMA completion barrier of each ring slot
};

template <bool TVD>
__global__ void __launch_bounds__(MX, 5) conv_march_kernel(MarchParams m)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ConvSmem& s = *reinterpret_cast<ConvSmem*>(smem_raw);
    const Params& k = m.k;
    const int t = threadIdx.x;
    const int ow = m.order[blockIdx.x];
    const int cta = ow & (ALLREG_BIT - 1);
    const bool allreg = (ow & ALLREG_BIT) != 0;
    const int strip = cta % m.nstrips, segi = cta / m.nstrips;
    const int I0 = k.gi0 + strip * MW;
    // ring rows by TMA as in march_kernel: ring column 0 = stored column c0 (a multiple of 4)
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
    const int J0 = segi * m.seg;
    const int J1 = min(J0 + m.seg, k.ny);
    const int js = J0 - 2;                              // 2 warm-up rows (carried TY, uY, vY, fluxes)
    const bool owner = t >= 2 && t < 2 + MW && gi < k.gi0 + k.nloc;
    const double dx = k.dx, dy = k.dy;
    // ring fed from the n-1 snapshot
    MarchParams mm = m;
    mm.k.u_o = k.u_1; mm.k.v_o = k.v_1; mm.k.p_o = k.p_1; mm.k.T_o = k.T_1;

    // row r goes to slot(r); its use of that slot is the ((r - js + 1) / RS)-th
    for (int j = js - 1; j <= js + 2; j++) ring_issue_tma(s, slot(j), mm, c0, tma, j);
    cp_wait_all();
    __syncthreads();
    for (int j = js - 1; j <= js + 2; j++) mbar_wait(&s.mbar[slot(j)], 0);
    for (int j = js - 1; j <= js + 2; j++) ring_derive<false>(s.ring[slot(j)]);
    ring_issue_tma(s, slot(js + 3), mm, c0, tma, js + 3);
    int sj = slot(js);

    double TYc = 0.0, uYc = 0.0, vYc = 0.0;          // carried: TY(i,j), uY(i,y^f_j), vY(cell (i,j-1)) for v-face (i,j)
    for (int j = js; j < J1; j++) {
        const int sa = sj + 1 == RS ? 0 : sj + 1, sb = sa + 1 == RS ? 0 : sa + 1;
        const int sc = sb + 1 == RS ? 0 : sb + 1, sd = sc + 1 == RS ? 0 : sc + 1;
        const int sm = sj == 0 ? RS - 1 : sj - 1;
        const RingRowC& Rm = s.ring[sm];
        const RingRowC& R0 = s.ring[sj];
        const RingRowC& Ra = s.ring[sa];
        const RingRowC& Rb = s.ring[sb];
        const int cb = j & 1, nb = (j + 1) & 1;
        cp_wait_all();
        __syncthreads();                                  // B0
        ring_issue_tma(s, sd, mm, c0, tma, j + 4);
        mbar_wait(&s.mbar[sc], ((j + 4 - js) / RS) & 1);   // row j+3
        ring_derive<false>(s.ring[sc]);
        const uint32_t kw0 = R0.KK[lc], kw1 = Ra.KK[lc];
        // per-point instance (REG: the +-3 window of the point is all fluid, so
        // every kind test folds away; same operations as the general instance)
        const bool reg = allreg || (kw0 & REG_BIT) != 0u;
        double Fx1 = 0.0, Fy1 = 0.0, TYn = 0.0, vYn = 0.0, uYn = 0.0;
        auto stageA = [&](auto regc) {
            constexpr bool REG = decltype(regc)::value;
            // ---- stage A: fluxes of row j+1 (Eqs. pl8-pl11 at time level n-1)
            {
                double ru = 0.0;
                if ((REG || flux_face(ukind(kw1)))) {
                    const double w = Ra.U[lc], r1 = Ra.R[lc - 1], r2 = Ra.R[lc];
                    ru = w > 0.0 ? r1 : r2;
                    if (TVD && (REG || ckind(Ra.KK[lc - 2]) == CK_FLUID) && (REG || ckind(Ra.KK[lc - 1]) == CK_FLUID) &&
                        (REG || ckind(kw1) == CK_FLUID) && (REG || ckind(Ra.KK[lc + 1]) == CK_FLUID))
                        ru += psi_f(Ra.R[lc - 2], r1, r2, Ra.R[lc + 1], w) * (r2 - r1);
                    Fx1 = ru * w * dy;
                }
                s.FX[nb][lc] = Fx1;
                double rv = 0.0;
                if ((REG || vkind(kw1) == FK_ACTIVE)) {
                    const double w = Ra.V[lc], r1 = R0.R[lc], r2 = Ra.R[lc];
                    rv = w > 0.0 ? r1 : r2;
                    if (TVD && (REG || ckind(Rm.KK[lc]) == CK_FLUID) && (REG || ckind(kw0) == CK_FLUID) && (REG || ckind(kw1) == CK_FLUID) &&
                        (REG || ckind(Rb.KK[lc]) == CK_FLUID))
                        rv += psi_f(Rm.R[lc], r1, r2, Rb.R[lc], w) * (r2 - r1);
                    Fy1 = rv * w * dx;
                }
                s.FY[nb][lc] = Fy1;
            }
            // TX at u-face (i, j): T flux through x^f_i (pl31_1)
            {
                double tx = 0.0;
                if ((REG || flux_face(ukind(kw0)))) {
                    const double F = s.FX[cb][lc], w = R0.U[lc], Tm = R0.T[lc - 1], Ti = R0.T[lc];
                    const double ps = (TVD && (REG || ckind(R0.KK[lc - 2]) == CK_FLUID) && (REG || ckind(R0.KK[lc - 1]) == CK_FLUID) &&
                                       (REG || ckind(kw0) == CK_FLUID) && (REG || ckind(R0.KK[lc + 1]) == CK_FLUID))
                                    ? psi_f(R0.T[lc - 2], Tm, Ti, R0.T[lc + 1], w) : 0.0;
                    tx = F * ((w > 0.0 ? Tm : Ti) + (Ti - Tm) * ps);
                }
                s.TX[lc] = tx;
            }
            // TY at v-face (i, j+1)
            if ((REG || vkind(kw1) == FK_ACTIVE)) {
                const double w = Ra.V[lc], Tj = R0.T[lc], Tp = Ra.T[lc];
                const double ps = (TVD && (REG || ckind(Rm.KK[lc]) == CK_FLUID) && (REG || ckind(kw0) == CK_FLUID) &&
                                   (REG || ckind(kw1) == CK_FLUID) && (REG || ckind(Rb.KK[lc]) == CK_FLUID))
                                ? psi_f(Rm.T[lc], Tj, Tp, Rb.T[lc], w) : 0.0;
                TYn = Fy1 * ((w > 0.0 ? Tj : Tp) + (Tp - Tj) * ps);
            }
            // uX at cell (i, j): u flux through the cell centre (transposed pl15_11 x-terms)
            {
                double ux = 0.0;
                if ((REG || ckind(kw0) == CK_FLUID) && (REG || ukind(kw0) == FK_ACTIVE) && (REG || ukind(R0.KK[lc + 1]) == FK_ACTIVE)) {
                    const double ui = R0.U[lc], up = R0.U[lc + 1], ub = 0.5 * (ui + up);
                    const bool ok = TVD && (REG || ukind(R0.KK[lc - 1]) == FK_ACTIVE) && (REG || ukind(R0.KK[lc + 2]) == FK_ACTIVE);
                    const double ps = ok ? psi_f(R0.U[lc - 1], ui, up, R0.U[lc + 2], ub) : 0.0;
                    ux = dy * R0.R[lc] * ub * ((ub > 0.0 ? ui : up) + (up - ui) * ps);
                } else if ((REG || ckind(kw0) == CK_FLUID)) {
                    // a fixed / inlet / outlet face on one side: same formula, no limiter
                    const double ui = R0.U[lc], up = R0.U[lc + 1], ub = 0.5 * (ui + up);
                    ux = dy * R0.R[lc] * ub * (ub > 0.0 ? ui : up);
                }
                s.UX[lc] = ux;
            }
            // vX at (u-face column i, v-row j+1): v flux through x^f_i, both half faces
            {
                double vx = 0.0;
                if ((REG || vkind(kw1) == FK_ACTIVE) || (REG || vkind(Ra.KK[lc - 1]) == FK_ACTIVE)) {
                    const double vm = Ra.V[lc - 1], vi = Ra.V[lc];
                    const bool ok = TVD && (REG || vkind(Ra.KK[lc - 2]) == FK_ACTIVE) && (REG || vkind(Ra.KK[lc - 1]) == FK_ACTIVE) &&
                                    (REG || vkind(kw1) == FK_ACTIVE) && (REG || vkind(Ra.KK[lc + 1]) == FK_ACTIVE);
                    double sum = 0.0;
                    if ((REG || flux_face(ukind(kw0)))) {               // lower half: u-face (i, j)
                        const double F = s.FX[cb][lc], w = R0.U[lc];
                        const double ps = ok ? psi_f(Ra.V[lc - 2], vm, vi, Ra.V[lc + 1], w) : 0.0;
                        sum += F * ((w > 0.0 ? vm : vi) + (vi - vm) * ps);
                    }
                    if ((REG || flux_face(ukind(kw1)))) {               // upper half: u-face (i, j+1)
                        const double F = Fx1, w = Ra.U[lc];
                        const double ps = ok ? psi_f(Ra.V[lc - 2], vm, vi, Ra.V[lc + 1], w) : 0.0;
                        sum += F * ((w > 0.0 ? vm : vi) + (vi - vm) * ps);
                    }
                    vx = 0.5 * sum;
                }
                s.VX[lc] = vx;
            }
            // vY at cell (i, j+1): v flux through the cell centre (pl15_11 y-terms)
            if ((REG || ckind(kw1) == CK_FLUID)) {
                const double vi = Ra.V[lc], vp = Rb.V[lc], vb = 0.5 * (vi + vp);
                const bool ok = TVD && (REG || vkind(kw1) == FK_ACTIVE) && (REG || vkind(Rb.KK[lc]) == FK_ACTIVE) &&
                                (REG || vkind(kw0) == FK_ACTIVE) && (REG || vkind(s.ring[sc].KK[lc]) == FK_ACTIVE);
                const double ps = ok ? psi_f(R0.V[lc], vi, vp, s.ring[sc].V[lc], vb) : 0.0;
                vYn = dx * Ra.R[lc] * vb * ((vb > 0.0 ? vi : vp) + (vp - vi) * ps);
            }
        };
        if (reg) stageA(std::true_type{}); else stageA(std::false_type{});
        __syncthreads();                                  // B1
        auto stageC = [&](auto regc) {
            constexpr bool REG = decltype(regc)::value;
            // ---- stage C: uY at (u column i, y^f_{j+1}) and the planes
            {
                const double ui = R0.U[lc], up = Ra.U[lc];
                const bool ok = TVD && (REG || ukind(Rm.KK[lc]) == FK_ACTIVE) && (REG || ukind(kw0) == FK_ACTIVE) &&
                                (REG || ukind(kw1) == FK_ACTIVE) && (REG || ukind(Rb.KK[lc]) == FK_ACTIVE);
                double sum = 0.0;
                for (int h = 0; h < 2; h++) {
                    const int cc = lc - 1 + h;
                    if ((!REG && vkind(Ra.KK[cc]) != FK_ACTIVE)) continue;
                    const double F = s.FY[nb][cc], w = Ra.V[cc];
                    const double ps = ok ? psi_f(Rm.U[lc], ui, up, Rb.U[lc], w) : 0.0;
                    sum += F * ((w > 0.0 ? ui : up) + (up - ui) * ps);
                }
                uYn = 0.5 * sum;
            }
        };
        if (reg) stageC(std::true_type{}); else stageC(std::false_type{});
        if (owner) {
            int tgt = -1000;                               // single-rank periodic: wrapped ghosts
            if (k.xbc == 1 && k.mirror) {
                if (gi < OFF) tgt = gi + k.nx;
                else if (gi >= k.nx - OFF) tgt = gi - k.nx;
            }
            if (j >= J0) {                                 // T^exp, u^exp of row j
                const long long id = gidx(k, gi, j);
                const double te = ckind(kw0) == CK_FLUID ? (s.TX[lc] - s.TX[lc + 1] + TYc - TYn) : 0.0;
                const double ue = ukind(kw0) == FK_ACTIVE ? (s.UX[lc - 1] - s.UX[lc] + uYc - uYn) : 0.0;
                k.Te_w[id] = te;
                k.ue_w[id] = ue;
                if (tgt > -1000) { k.Te_w[gidx(k, tgt, j)] = te; k.ue_w[gidx(k, tgt, j)] = ue; }
            }
            if (j + 1 >= J0 && j + 1 < J1) {               // v^exp of v-face row j+1 (rows J0 .. J1-1)
                const double ve = vkind(kw1) == FK_ACTIVE ? (s.VX[lc] - s.VX[lc + 1] + vYc - vYn) : 0.0;
                k.ve_w[gidx(k, gi, j + 1)] = ve;
                if (tgt > -1000) k.ve_w[gidx(k, tgt, j + 1)] = ve;
            }
        }
        TYc = TYn;
        uYc = uYn;
        vYc = vYn;
        sj = sa;
    }
    cp_wait_all();
}

}  // namespace sts
