// sts_march.cuh -- v2 loop-2 pass kernel: y-marching row sweep (sm_100a, fp64).
//
// The paper's single kernel marches along y inside a work-group with row
// buffers for p, u-hat/d^u, v-hat/d^v in local memory (P:248-253, P:550,
// P:558; Fig. 7).  Re-designed for B200:
//  - a CTA of MX = 128 threads owns a strip of MW = 125 columns (+2 left /
//    +1 right redundant columns, the paper's "halo work-items") and a
//    segment of rows; thread t owns global column I0 - 2 + t for the whole
//    segment;
//  - old-iterate rows of u, v, p, T (+ packed kind codes) stream through a
//    6-row shared-memory ring fed by cp.async one row ahead; rho = p/T and
//    Gamma = sqrt(T) are computed once per ring element (not stored in HBM);
//  - every face quantity (rho^u, F^x, rho^v, F^y, harmonic Gamma, TVD psi,
//    link coefficients) is computed ONCE: x-neighbours read it from a
//    shared-memory row, the y-neighbour gets it through a register carried to
//    the next row step (the S side of row j+1 is the N side of row j);
//  - per row step j: stage A (fluxes and link pieces of row j / j+1),
//    stage C (T_{i,j}, u-hat_{i,j}, v-hat_{i,j+1}: Eqs. pl29_1-pl29_5), stage D
//    (p_{i,j}, Eq. pl29_6), stage E (u_{i,j}, v_{i,j}, Eqs. pl29_7-pl29_8,
//    writes, residual maxima) -- the paper's dependency order;
//  - divisions become MUFU reciprocals + Newton steps; the mesh constants
//    (dy/dx, dx dy/(2 dt), ...) are precomputed on the host.
// A segment starts 4 rows early (warm-up) so that every carried quantity is
// exact when its first output row is reached.
#pragma once

#include "sts_kernels.cuh"

namespace sts {

constexpr int MX = 128;          // threads per CTA = columns handled per strip
constexpr int MW = MX - 3;       // owned columns per strip
constexpr int RW = MX + 8;       // ring row width (global columns I0-4 .. I0-4+RW)
constexpr int RS = 6;            // ring slots
constexpr int WARM = 4;          // warm-up rows per segment

struct MarchParams {
    Params k;                    // v1 parameter block (pointers, constants)
    const uint32_t* kind;        // packed kinds: ck | uk << 8 | vk << 16, (ny+1) x pitch
    int seg;                     // rows per segment
    double inv_dx, inv_dy, CT1_dydx, CT1_dxdy, B_dydx, B_dxdy, c_t, dV, A_dy, A_dx, half_dV;
};

// fp64 reciprocal: MUFU.RCP64H seed + 2 Newton steps (~1 ulp), no slow path.
__device__ __forceinline__ double rcp(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    return r;
}
// a / b with one remainder correction after the reciprocal (~0.5-1 ulp).
__device__ __forceinline__ double fdiv(double a, double b)
{
    double r = rcp(b);
    double q = a * r;
    double rem = fma(-b, q, a);
    return fma(rem, r, q);
}
// sqrt via rsqrt seed + Newton (~1 ulp), x > 0.
__device__ __forceinline__ double fsqrt(double x)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = y * fma(-0.5 * x * y, y, 1.5);
    y = y * fma(-0.5 * x * y, y, 1.5);
    double s = x * y;
    return fma(0.5 * y, fma(-s, s, x), s);
}
// same TVD correction as psi_u, with the reciprocal instead of IEEE division
__device__ __forceinline__ double psi_f(double f1, double f2, double f3, double f4, double w)
{
    double b = f3 - f2;
    if (fabs(b) <= 1e-12 * (1.0 + fabs(f2) + fabs(f3))) return 0.0;   // R37
    if (w > 0.0) {
        double a = f2 - f1;
        return ((a > 0.0 && b > 0.0) || (a < 0.0 && b < 0.0)) ? fdiv(a, a + b) : 0.0;
    } else {
        double c = f4 - f3;
        return ((c > 0.0 && b > 0.0) || (c < 0.0 && b < 0.0)) ? -fdiv(c, c + b) : 0.0;
    }
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

struct MarchSmem {
    // ring of old-iterate rows
    double U[RS][RW], V[RS][RW], P[RS][RW], T[RS][RW], R[RS][RW], G[RS][RW];
    uint32_t KK[RS][RW];
    // per-row face / link pieces (indexed by ring column)
    double RU[2][RW], FX[2][RW], RV[2][RW], FY[2][RW], R1[2][RW];
    double XTW[RW], XTE[RW], XUW[RW], XUE[RW], FBX[RW], XVE[RW], XVF[RW], GC[RW];
    double UH[RW], DU[RW], PN[RW];
};

__device__ __forceinline__ int slot(int j) { return (j + 4 * RS) % RS; }
__device__ __forceinline__ uint8_t ckind(uint32_t w) { return (uint8_t)(w & 0xff); }
__device__ __forceinline__ uint8_t ukind(uint32_t w) { return (uint8_t)((w >> 8) & 0xff); }
__device__ __forceinline__ uint8_t vkind(uint32_t w) { return (uint8_t)((w >> 16) & 0xff); }

// Issue the loads of ring row j (global columns I0-4 .. I0-4+RW).  Rows outside
// [0, ny] and unstored columns are filled directly: kind WALLY / NONE, u = wall
// velocity beyond the walls (BC spec 8), p = T = 1, v = 0.
__device__ __forceinline__ void ring_issue(MarchSmem& s, const MarchParams& m, int I0, int j)
{
    const Params& k = m.k;
    const int sl = slot(j);
    for (int lc = threadIdx.x; lc < RW; lc += MX) {
        const int gi = I0 - 4 + lc;
        const bool col_ok = stored_col(k, gi);
        if (j >= 0 && j < k.ny && col_ok) {
            const long long id = gidx(k, gi, j);
            cp_async8(&s.U[sl][lc], k.u_o + id);
            cp_async8(&s.V[sl][lc], k.v_o + id);
            cp_async8(&s.P[sl][lc], k.p_o + id);
            cp_async8(&s.T[sl][lc], k.T_o + id);
            cp_async4(&s.KK[sl][lc], m.kind + id);
        } else if (j == k.ny && col_ok) {          // top wall row: v = 0 (WALL), no cells
            const long long id = gidx(k, gi, j);
            s.U[sl][lc] = k.u_wt;
            cp_async8(&s.V[sl][lc], k.v_o + id);
            s.P[sl][lc] = 1.0;
            s.T[sl][lc] = 1.0;
            cp_async4(&s.KK[sl][lc], m.kind + id);
        } else {
            s.U[sl][lc] = j < 0 ? k.u_wb : (j >= k.ny ? k.u_wt : 0.0);
            s.V[sl][lc] = 0.0;
            s.P[sl][lc] = 1.0;
            s.T[sl][lc] = 1.0;
            s.KK[sl][lc] = (uint32_t)CK_WALLY | ((uint32_t)FK_NONE << 8) | ((uint32_t)FK_NONE << 16);
        }
    }
    cp_commit();
}
// rho = p/T (Eq. pl5), Gamma = sqrt(T) (Eq. pl37) of ring row j
__device__ __forceinline__ void ring_derive(MarchSmem& s, int j)
{
    const int sl = slot(j);
    for (int lc = threadIdx.x; lc < RW; lc += MX) {
        const double Tv = s.T[sl][lc];
        s.R[sl][lc] = fdiv(s.P[sl][lc], Tv);
        s.G[sl][lc] = fsqrt(Tv);
    }
}

template <bool IMPL, bool TVD>
__global__ void __launch_bounds__(MX, 3) march_kernel(MarchParams m)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MarchSmem& s = *reinterpret_cast<MarchSmem*>(smem_raw);
    const Params& k = m.k;
    const int t = threadIdx.x;
    const int lc = t + 2;                               // ring column of this thread's column
    const int I0 = k.gi0 + blockIdx.x * MW;             // first owned column of the strip
    const int gi = I0 - 2 + t;                          // this thread's global column
    const int J0 = blockIdx.y * m.seg;
    const int J1 = min(J0 + m.seg, k.ny);
    const int js = J0 - WARM;
    const bool col_stored = stored_col(k, gi);
    const bool owner = t >= 2 && t < 2 + MW && gi < k.gi0 + k.nloc;
    const double dt = k.dt, dx = k.dx, dy = k.dy;

    // ---- prologue: ring rows js-1 .. js+2 (synchronous), issue js+3
    for (int j = js - 1; j <= js + 2; j++) ring_issue(s, m, I0, j);
    cp_wait_all();
    __syncthreads();
    for (int j = js - 1; j <= js + 2; j++) ring_derive(s, j);
    ring_issue(s, m, I0, js + 3);

    // ---- n-1 / plane register pipeline (loaded one row step ahead)
    auto ld = [&](const double* a, int j) -> double {
        return (col_stored && j >= 0 && j < k.ny) ? __ldg(a + gidx(k, gi, j)) : 0.0;
    };
    auto ldv = [&](const double* a, int j) -> double {
        return (col_stored && j >= 0 && j <= k.ny) ? __ldg(a + gidx(k, gi, j)) : 0.0;
    };
    double p1n = ld(k.p_1, js + 1), T1n = ld(k.T_1, js + 1);     // row j+1 at step js
    double T1c = ld(k.T_1, js), u1c = ld(k.u_1, js), v1n = ldv(k.v_1, js + 1);
    double Tec = 0.0, uec = 0.0, ven = 0.0;
    if (!IMPL) { Tec = ld(k.Te, js); uec = ld(k.ue, js); ven = ldv(k.ve, js + 1); }

    // ---- carried (row-rotated) quantities, valid after the warm-up
    double ytS = 0.0, FS = 0.0;           // T-eq south link piece / flux at v-face (i, j)
    double utS = 0.0, FsSum = 0.0;        // u-eq south tangential piece / half-flux sum
    double vcS = 0.0, FbS = 0.0;          // v-eq south normal piece (cell (i, j)) / F-bar
    double vhatP = 0.0, dvP = 0.0;        // v-hat, d^v at v-face (i, j)
    double pnP = 1.0;                     // p_new(i, j-1)
    double gcP = 1.0;                     // corner Gamma (i, j)

    double r_du = 0.0, r_dv = 0.0, r_dp = 0.0, r_dT = 0.0, r_vel = 0.0, r_p = 0.0, r_T = 0.0;
    long long bad = -1;
    int badf = 0;

    for (int j = js; j < J1; j++) {
        const int c0 = slot(j), cm = slot(j - 1), c1 = slot(j + 1), c2 = slot(j + 2), c3 = slot(j + 3);
        const int cb = j & 1, nb = (j + 1) & 1;
        const bool out_row = j >= J0;

        // prefetch the next row's n-1 / plane values (consumed one step later)
        double p1nn = ld(k.p_1, j + 2), T1nn = ld(k.T_1, j + 2);
        double u1n = ld(k.u_1, j + 1), v1nn = ldv(k.v_1, j + 2);
        double Ten = 0.0, uen = 0.0, vem = 0.0;
        if (!IMPL) { Ten = ld(k.Te, j + 1); uen = ld(k.ue, j + 1); vem = ldv(k.ve, j + 2); }

        cp_wait_all();
        __syncthreads();                                    // B0: ring row j+3 landed
        ring_issue(s, m, I0, j + 4);

        // ================= stage A: row j+1 fluxes, link pieces =================
        ring_derive(s, j + 3);
        const uint32_t kw0 = s.KK[c0][lc], kw1 = s.KK[c1][lc];
        // (p/T)^{n-1} of row j+1
        s.R1[nb][lc] = fdiv(p1n, T1n == 0.0 ? 1.0 : T1n);
        // F^x, rho^u at u-face (i, j+1)  (Eqs. pl8, pl10, R1)
        double Fx1 = 0.0;
        {
            double ru = 0.0;
            const uint8_t uk = ukind(kw1);
            if (flux_face(uk)) {
                const double w = s.U[c1][lc], r1 = s.R[c1][lc - 1], r2 = s.R[c1][lc];
                ru = w > 0.0 ? r1 : r2;
                if (TVD && ckind(s.KK[c1][lc - 2]) == CK_FLUID && ckind(s.KK[c1][lc - 1]) == CK_FLUID &&
                    ckind(kw1) == CK_FLUID && ckind(s.KK[c1][lc + 1]) == CK_FLUID)
                    ru += psi_f(s.R[c1][lc - 2], r1, r2, s.R[c1][lc + 1], w) * (r2 - r1);
                Fx1 = ru * w * dy;
            }
            s.RU[nb][lc] = ru;
            s.FX[nb][lc] = Fx1;
        }
        // F^y, rho^v at v-face (i, j+1)  (Eqs. pl9, pl11, R1)
        double Fy1 = 0.0;
        {
            double rv = 0.0;
            if (vkind(kw1) == FK_ACTIVE) {
                const double w = s.V[c1][lc], r1 = s.R[c0][lc], r2 = s.R[c1][lc];
                rv = w > 0.0 ? r1 : r2;
                if (TVD && ckind(s.KK[cm][lc]) == CK_FLUID && ckind(kw0) == CK_FLUID && ckind(kw1) == CK_FLUID &&
                    ckind(s.KK[c2][lc]) == CK_FLUID)
                    rv += psi_f(s.R[cm][lc], r1, r2, s.R[c2][lc], w) * (r2 - r1);
                Fy1 = rv * w * dx;
            }
            s.RV[nb][lc] = rv;
            s.FY[nb][lc] = Fy1;
        }
        // T-eq x-face pieces at u-face (i, j): a^T_1 of cell i, a^T_2 of cell i-1 (Eqs. pl31-pl33)
        {
            double pw = 0.0, pe = 0.0;
            const uint8_t kl = ckind(s.KK[c0][lc - 1]), kr = ckind(kw0);
            if (!wallish(kl) && !wallish(kr)) {
                const double F = s.FX[cb][lc];
                const double g1 = s.G[c0][lc - 1], g2 = s.G[c0][lc];
                const double D = m.CT1_dydx * (2.0 * g1 * g2 * rcp(g1 + g2));
                double ps = 0.0;
                if (IMPL && TVD && ckind(s.KK[c0][lc - 2]) == CK_FLUID && kl == CK_FLUID && kr == CK_FLUID &&
                    ckind(s.KK[c0][lc + 1]) == CK_FLUID)
                    ps = psi_f(s.T[c0][lc - 2], s.T[c0][lc - 1], s.T[c0][lc], s.T[c0][lc + 1], s.U[c0][lc]);
                pw = (IMPL ? max0(F) - F * ps : 0.0) + D;
                pe = (IMPL ? max0(-F) - F * ps : 0.0) + D;
            }
            s.XTW[lc] = pw;
            s.XTE[lc] = pe;
        }
        // T-eq y-face piece at v-face (i, j+1): a^T_4 of cell (i, j), a^T_3 of cell (i, j+1)
        double ytN = 0.0, ytSn = 0.0;
        {
            const uint8_t kb = ckind(kw0), kt = ckind(kw1);
            if (!wallish(kb) && !wallish(kt)) {
                const double F = Fy1;
                const double g1 = s.G[c0][lc], g2 = s.G[c1][lc];
                const double D = m.CT1_dxdy * (2.0 * g1 * g2 * rcp(g1 + g2));
                double ps = 0.0;
                if (IMPL && TVD && ckind(s.KK[cm][lc]) == CK_FLUID && kb == CK_FLUID && kt == CK_FLUID &&
                    ckind(s.KK[c2][lc]) == CK_FLUID)
                    ps = psi_f(s.T[cm][lc], s.T[c0][lc], s.T[c1][lc], s.T[c2][lc], s.V[c1][lc]);
                ytN = (IMPL ? max0(-F) - F * ps : 0.0) + D;
                ytSn = (IMPL ? max0(F) - F * ps : 0.0) + D;
            }
        }
        // u-eq x pieces of cell (i, j): a^u_2 of face i, a^u_1 of face i+1 (transposed pl15)
        {
            double xe = 0.0, xw = 0.0, Fb = 0.0;
            if (ckind(kw0) == CK_FLUID) {
                const double ub = 0.5 * (s.U[c0][lc] + s.U[c0][lc + 1]);
                Fb = s.R[c0][lc] * ub * dy;
                const double D = 4.0 / 3.0 * m.B_dydx * s.G[c0][lc];
                double ps = 0.0;
                if (IMPL && TVD && ukind(s.KK[c0][lc - 1]) == FK_ACTIVE && ukind(kw0) == FK_ACTIVE &&
                    ukind(s.KK[c0][lc + 1]) == FK_ACTIVE && ukind(s.KK[c0][lc + 2]) == FK_ACTIVE)
                    ps = psi_f(s.U[c0][lc - 1], s.U[c0][lc], s.U[c0][lc + 1], s.U[c0][lc + 2], ub);
                xe = (IMPL ? max0(-Fb) - Fb * ps : 0.0) + D;
                xw = (IMPL ? max0(Fb) - Fb * ps : 0.0) + D;
            }
            s.XUE[lc] = xe;
            s.XUW[lc] = xw;
            s.FBX[lc] = Fb;
        }
        // u-eq tangential psi at (u column i, y^f_{j+1}) (fluxes need the neighbour: stage C)
        double upsi1 = 0.0, upsi2 = 0.0;
        if (IMPL && TVD && ukind(s.KK[cm][lc]) == FK_ACTIVE && ukind(kw0) == FK_ACTIVE &&
            ukind(kw1) == FK_ACTIVE && ukind(s.KK[c2][lc]) == FK_ACTIVE) {
            const double f1 = s.U[cm][lc], f2 = s.U[c0][lc], f3 = s.U[c1][lc], f4 = s.U[c2][lc];
            upsi1 = psi_f(f1, f2, f3, f4, s.V[c1][lc]);
            upsi2 = psi_f(f1, f2, f3, f4, s.V[c1][lc - 1]);
        }
        // v-eq normal piece of cell (i, j+1): a^v_4 of v-face (i, j+1), a^v_3 of v-face (i, j+2)
        double vcN = 0.0, vcSn = 0.0, FbN = 0.0;
        if (ckind(kw1) == CK_FLUID) {
            const double vb = 0.5 * (s.V[c1][lc] + s.V[c2][lc]);
            FbN = s.R[c1][lc] * vb * dx;
            const double D = 4.0 / 3.0 * m.B_dxdy * s.G[c1][lc];
            double ps = 0.0;
            if (IMPL && TVD && vkind(kw0) == FK_ACTIVE && vkind(kw1) == FK_ACTIVE &&
                vkind(s.KK[c2][lc]) == FK_ACTIVE && vkind(s.KK[c3][lc]) == FK_ACTIVE)
                ps = psi_f(s.V[c0][lc], s.V[c1][lc], s.V[c2][lc], s.V[c3][lc], vb);
            vcN = (IMPL ? max0(-FbN) - FbN * ps : 0.0) + D;
            vcSn = (IMPL ? max0(FbN) - FbN * ps : 0.0) + D;
        }
        // corner Gamma at (x^f_i, y^f_{j+1}) (R4, R5; BC spec 8)
        double gcN;
        {
            double sum = 0.0;
            int n = 0;
            const uint8_t a = ckind(s.KK[c0][lc - 1]), b = ckind(kw0), c = ckind(s.KK[c1][lc - 1]), d = ckind(kw1);
            if (!wallish(a)) { sum += s.G[c0][lc - 1]; n++; }
            if (!wallish(b)) { sum += s.G[c0][lc]; n++; }
            if (!wallish(c)) { sum += s.G[c1][lc - 1]; n++; }
            if (!wallish(d)) { sum += s.G[c1][lc]; n++; }
            gcN = n == 4 ? 0.25 * sum : (n > 0 ? sum / n : 0.0);
            s.GC[lc] = gcN;
        }
        // v-eq tangential pieces at (u-face column i, v-row j+1): a^v_1 of v-face (i, j+1),
        // a^v_2 of v-face (i-1, j+1)
        double xvW, FwSum;
        {
            const double F1 = Fx1, F2 = s.FX[cb][lc];     // rows j+1 (upper half) and j (lower half)
            double p1 = 0.0, p2 = 0.0;
            if (IMPL && TVD && vkind(s.KK[c1][lc - 2]) == FK_ACTIVE && vkind(s.KK[c1][lc - 1]) == FK_ACTIVE &&
                vkind(kw1) == FK_ACTIVE && vkind(s.KK[c1][lc + 1]) == FK_ACTIVE) {
                const double f1 = s.V[c1][lc - 2], f2 = s.V[c1][lc - 1], f3 = s.V[c1][lc], f4 = s.V[c1][lc + 1];
                p1 = psi_f(f1, f2, f3, f4, s.U[c1][lc]);
                p2 = psi_f(f1, f2, f3, f4, s.U[c0][lc]);
            }
            const double D = m.B_dydx * gcN;
            xvW = (IMPL ? 0.5 * (max0(F1) - F1 * p1 + max0(F2) - F2 * p2) : 0.0) + D;
            s.XVE[lc] = (IMPL ? 0.5 * (max0(-F1) - F1 * p1 + max0(-F2) - F2 * p2) : 0.0) + D;
            FwSum = F1 + F2;
            s.XVF[lc] = FwSum;
        }
        __syncthreads();                                    // B1

        // ================= stage C: T_{i,j}, u-hat_{i,j}, v-hat_{i,j+1} =================
        const double rP = s.R[c0][lc], gP = s.G[c0][lc];
        double TN = 0.0;
        if (ckind(kw0) == CK_FLUID) {
            const double tau = 2.1904 * k.Kn * rcp(rP);   // Eq. pl39
            double a1, a2, a3, a4, T1, T2, T3, T4, FW = 0.0, FE = 0.0, FSl = 0.0, FNl = 0.0;
            uint8_t kn = ckind(s.KK[c0][lc - 1]);
            if (wallish(kn)) { a1 = k.CT1 * gP * dy * rcp(0.5 * dx + tau); T1 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a1 = s.XTW[lc]; FW = s.FX[cb][lc]; T1 = s.T[c0][lc - 1]; }
            kn = ckind(s.KK[c0][lc + 1]);
            if (wallish(kn)) { a2 = k.CT1 * gP * dy * rcp(0.5 * dx + tau); T2 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a2 = s.XTE[lc + 1]; FE = s.FX[cb][lc + 1]; T2 = s.T[c0][lc + 1]; }
            kn = ckind(s.KK[cm][lc]);
            if (wallish(kn)) { a3 = k.CT1 * gP * dx * rcp(0.5 * dy + tau); T3 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a3 = ytS; FSl = FS; T3 = s.T[cm][lc]; }
            kn = ckind(kw1);
            if (wallish(kn)) { a4 = k.CT1 * gP * dx * rcp(0.5 * dy + tau); T4 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a4 = ytN; FNl = Fy1; T4 = s.T[c1][lc]; }
            const double a0 = IMPL ? dt * (a1 + a2 + a3 + a4 + FE - FW + FNl - FSl) + rP * m.dV
                                   : dt * (a1 + a2 + a3 + a4) + rP * m.dV;
            // S^T_c, Eq. pl29 (R4 bilinear = 4-point mean; R9 sign)
            const double dudx = (s.U[c0][lc + 1] - s.U[c0][lc]) * m.inv_dx;
            const double dvdy = (s.V[c1][lc] - s.V[c0][lc]) * m.inv_dy;
            const double vE = 0.25 * (s.V[c0][lc] + s.V[c0][lc + 1] + s.V[c1][lc] + s.V[c1][lc + 1]);
            const double vW = 0.25 * (s.V[c0][lc - 1] + s.V[c0][lc] + s.V[c1][lc - 1] + s.V[c1][lc]);
            const double uN = 0.25 * (s.U[c0][lc] + s.U[c0][lc + 1] + s.U[c1][lc] + s.U[c1][lc + 1]);
            const double uS = 0.25 * (s.U[cm][lc] + s.U[cm][lc + 1] + s.U[c0][lc] + s.U[c0][lc + 1]);
            const double shear = (vE - vW) * m.inv_dx + (uN - uS) * m.inv_dy;
            const double div = dudx + dvdy;
            const double Sc = (k.CT2 * gP * (2.0 * (dudx * dudx + dvdy * dvdy) + shear * shear - 2.0 / 3.0 * div * div)
                               + k.pw_sign * k.CT3 * s.P[c0][lc] * div) * m.dV;
            const double rhs = dt * (a1 * T1 + a2 * T2 + a3 * T3 + a4 * T4 + Sc + Tec) + s.R1[cb][lc] * T1c * m.dV;
            TN = rhs * rcp(a0);
        }
        // u-eq at u-face (i, j)
        double uhat = 0.0, du = 0.0;
        double utSn, FsSumN;
        {
            // N tangential link pieces at y^f_{j+1} (both sides; the S side is carried)
            const double F1 = Fy1, F2 = s.FY[nb][lc - 1];
            const double D = m.B_dxdy * gcN;
            const double a4p = (IMPL ? 0.5 * (max0(-F1) - F1 * upsi1 + max0(-F2) - F2 * upsi2) : 0.0) + D;
            utSn = (IMPL ? 0.5 * (max0(F1) - F1 * upsi1 + max0(F2) - F2 * upsi2) : 0.0) + D;
            FsSumN = F1 + F2;
            if (ukind(kw0) == FK_ACTIVE) {
                const double rL = s.R[c0][lc - 1], rR = rP, gL = s.G[c0][lc - 1], gR = gP;
                const double gadj = 0.5 * (gL + gR);
                const double zeta = 1.1466 * k.Kn * rcp(0.5 * (rL + rR));     // Eq. pl38
                const double a1 = s.XUW[lc - 1], a2 = s.XUE[lc];
                const double FbW = s.FBX[lc - 1], FbE = s.FBX[lc];
                double a3, a4, uS, uN, FsS = 0.0, FnS = 0.0;
                const uint8_t kl = ckind(s.KK[cm][lc - 1]), kr = ckind(s.KK[cm][lc]);
                if (kl == CK_WALLY || (kl == CK_SOLID && kr == CK_SOLID)) {
                    a3 = k.B * gadj * dx * rcp(0.5 * dy + zeta); uS = kl == CK_WALLY ? k.u_wb : 0.0;
                } else { a3 = utS; FsS = FsSum; uS = s.U[cm][lc]; }
                const uint8_t ml = ckind(s.KK[c1][lc - 1]), mr = ckind(kw1);
                if (ml == CK_WALLY || (ml == CK_SOLID && mr == CK_SOLID)) {
                    a4 = k.B * gadj * dx * rcp(0.5 * dy + zeta); uN = ml == CK_WALLY ? k.u_wt : 0.0;
                } else { a4 = a4p; FnS = FsSumN; uN = s.U[c1][lc]; }
                const double tterm = (rR + rL) * m.c_t;
                const double a0 = IMPL ? a1 + a2 + a3 + a4 + FbE - FbW + 0.5 * (FnS - FsS) + tterm
                                       : a1 + a2 + a3 + a4 + tterm;
                const double b = (s.R1[cb][lc] + s.R1[cb][lc - 1]) * m.c_t * u1c
                               + k.B * (gcN * (s.V[c1][lc] - s.V[c1][lc - 1]) - gcP * (s.V[c0][lc] - s.V[c0][lc - 1])
                                        - 2.0 / 3.0 * gR * (s.V[c1][lc] - s.V[c0][lc])
                                        + 2.0 / 3.0 * gL * (s.V[c1][lc - 1] - s.V[c0][lc - 1]))
                               + k.g_x * (rR + rL) * m.half_dV;
                const double r = rcp(a0);
                uhat = (a1 * s.U[c0][lc - 1] + a2 * s.U[c0][lc + 1] + a3 * uS + a4 * uN + b + uec) * r;
                du = m.A_dy * r;
            }
            s.UH[lc] = uhat;
            s.DU[lc] = du;
        }
        // v-eq at v-face (i, j+1)
        double vhatN = 0.0, dvN = 0.0;
        if (vkind(kw1) == FK_ACTIVE) {
            const double rB = rP, rT = s.R[c1][lc], gB = gP, gT = s.G[c1][lc];
            const double gadj = 0.5 * (gB + gT);
            const double zeta = 1.1466 * k.Kn * rcp(0.5 * (rB + rT));
            double a1, a2, vW, vE, FwS = 0.0, FeS = 0.0;
            if (ckind(s.KK[c0][lc - 1]) == CK_SOLID && ckind(s.KK[c1][lc - 1]) == CK_SOLID) {
                a1 = k.B * gadj * dy * rcp(0.5 * dx + zeta); vW = 0.0;
            } else { a1 = xvW; FwS = FwSum; vW = s.V[c1][lc - 1]; }
            if (ckind(s.KK[c0][lc + 1]) == CK_SOLID && ckind(s.KK[c1][lc + 1]) == CK_SOLID) {
                a2 = k.B * gadj * dy * rcp(0.5 * dx + zeta); vE = 0.0;
            } else { a2 = s.XVE[lc + 1]; FeS = s.XVF[lc + 1]; vE = s.V[c1][lc + 1]; }
            const double a3 = vcS, a4 = vcN;
            const double tterm = (rT + rB) * m.c_t;
            const double a0 = IMPL ? a1 + a2 + a3 + a4 + 0.5 * (FeS - FwS) + FbN - FbS + tterm
                                   : a1 + a2 + a3 + a4 + tterm;
            const double b = (s.R1[nb][lc] + s.R1[cb][lc]) * m.c_t * v1n
                           + k.B * (s.GC[lc + 1] * (s.U[c1][lc + 1] - s.U[c0][lc + 1]) - gcN * (s.U[c1][lc] - s.U[c0][lc])
                                    - 2.0 / 3.0 * gT * (s.U[c1][lc + 1] - s.U[c1][lc])
                                    + 2.0 / 3.0 * gB * (s.U[c0][lc + 1] - s.U[c0][lc]))
                           + k.g_y * (rT + rB) * m.half_dV;
            const double r = rcp(a0);
            vhatN = (a1 * vW + a2 * vE + a3 * s.V[c0][lc] + a4 * s.V[c2][lc] + b + ven) * r;
            dvN = m.A_dx * r;
        }
        __syncthreads();                                    // B2

        // ================= stage D: p_{i,j} (Eqs. pl23-pl24) =================
        double pn = s.P[c0][lc];
        if (ckind(kw0) == CK_FLUID) {
            double apW = 0.0, apE = 0.0, apS = 0.0, apN = 0.0, bpW = 0.0, bpE = 0.0, bpS = 0.0, bpN = 0.0, sum = 0.0;
            const uint8_t kwf = ukind(kw0), kef = ukind(s.KK[c0][lc + 1]);
            if (kwf == FK_ACTIVE) {
                const double r = s.RU[cb][lc];
                apW = r * du * dy; bpW = r * uhat * dy; sum += apW * s.P[c0][lc - 1];
            } else if (kwf == FK_INLET) bpW = s.RU[cb][lc] * k.u_in * dy;
            if (kef == FK_ACTIVE) {
                const double r = s.RU[cb][lc + 1];
                apE = r * s.DU[lc + 1] * dy; bpE = r * s.UH[lc + 1] * dy; sum += apE * s.P[c0][lc + 1];
            } else if (kef == FK_OUTLET) bpE = s.RU[cb][lc + 1] * s.U[c0][lc] * dy;
            if (vkind(kw0) == FK_ACTIVE) {
                const double r = s.RV[cb][lc];
                apS = r * dvP * dx; bpS = r * vhatP * dx; sum += apS * s.P[cm][lc];
            }
            if (vkind(kw1) == FK_ACTIVE) {
                const double r = s.RV[nb][lc];
                apN = r * dvN * dx; bpN = r * vhatN * dx; sum += apN * s.P[c1][lc];
            }
            const double a0 = m.dV * rcp(TN) + (apW + apE + apS + apN) * dt;
            const double bp = s.R1[cb][lc] * m.dV - (bpE - bpW + bpN - bpS) * dt;
            pn = (sum * dt + bp) * rcp(a0);
        }
        s.PN[lc] = pn;
        __syncthreads();                                    // B3

        // ================= stage E: corrections, writes, residuals =================
        if (out_row && owner) {
            const long long id = gidx(k, gi, j);
            if (ckind(kw0) == CK_FLUID) {
                k.T_w[id] = TN;
                k.p_w[id] = pn;
                r_dT = nmax(r_dT, fabs(TN - s.T[c0][lc]));
                r_dp = nmax(r_dp, fabs(pn - s.P[c0][lc]));
                r_T = nmax(r_T, fabs(TN));
                r_p = nmax(r_p, fabs(pn));
                if (!(TN > 0.0) || !(pn > 0.0) || !isfinite(TN) || !isfinite(pn)) {
                    const long long flat = (long long)j * k.nx + gi;
                    if (bad < 0 || flat < bad) { bad = flat; badf = (!(TN > 0.0) || !isfinite(TN)) ? 3 : 2; }
                }
            }
            const uint8_t ku = ukind(kw0);
            double un;
            if (ku == FK_ACTIVE) {
                un = uhat - du * (pn - s.PN[lc - 1]);
                r_du = nmax(r_du, fabs(un - s.U[c0][lc]));
                r_vel = nmax(r_vel, fabs(un));
            } else if (ku == FK_INLET) un = k.u_in;
            else un = 0.0;
            k.u_w[id] = un;
            if (gi == k.nx - 1 && k.xbc == 0) k.u_w[id + 1] = s.U[c0][lc];   // outlet face (BC spec 3)
            double vn = 0.0;
            if (vkind(kw0) == FK_ACTIVE) {
                vn = vhatP - dvP * (pn - pnP);
                r_dv = nmax(r_dv, fabs(vn - s.V[c0][lc]));
                r_vel = nmax(r_vel, fabs(vn));
            }
            k.v_w[id] = vn;
            if (k.xbc == 0) {
                if (gi == k.nx - 1) {
                    const double pv = ckind(kw0) == CK_FLUID ? pn : s.P[c0][lc];
                    const double Tv = ckind(kw0) == CK_FLUID ? TN : s.T[c0][lc];
                    for (int g = 1; g <= OFF - 1; g++) { k.p_w[id + g] = pv; k.T_w[id + g] = Tv; k.v_w[id + g] = vn; }
                }
            } else if (k.mirror) {
                int tgt = -1000;
                if (gi < OFF) tgt = gi + k.nx;
                else if (gi >= k.nx - OFF) tgt = gi - k.nx;
                if (tgt > -1000) {
                    const long long tt = gidx(k, tgt, j);
                    if (ckind(kw0) == CK_FLUID) { k.p_w[tt] = pn; k.T_w[tt] = TN; }
                    k.u_w[tt] = un;
                    k.v_w[tt] = vn;
                }
            }
        }
        // ---- carry row j+1 quantities to the next step
        ytS = ytSn; FS = Fy1;
        utS = utSn; FsSum = FsSumN;
        vcS = vcSn; FbS = FbN;
        vhatP = vhatN; dvP = dvN;
        pnP = pn; gcP = gcN;
        p1n = p1nn; T1c = T1n; T1n = T1nn; u1c = u1n; v1n = v1nn;
        if (!IMPL) { Tec = Ten; uec = uen; ven = vem; }
    }
    cp_wait_all();
    double vals[7] = {r_du, r_dv, r_dp, r_dT, r_vel, r_p, r_T};
    __syncthreads();
    // reuse the v1 block reduction (NT = 256 there; here MX = 128 threads -> 4 warps)
    __shared__ double part[MX / 32][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int q = 0; q < 7; q++) {
        double v = vals[q];
        const bool isn = v != v;
        const unsigned nanmask = __ballot_sync(0xffffffffu, isn);
        v = warp_max(isn ? 0.0 : v);
        if (nanmask) v = __longlong_as_double(0x7ff8000000000000LL);
        if (lane == 0) part[wid][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < 7) {
        double v = 0.0;
        for (int w = 0; w < MX / 32; w++) v = nmax(v, part[w][threadIdx.x]);
        atomicMax(&k.red[threadIdx.x], (unsigned long long)__double_as_longlong(v));
    }
    if (bad >= 0) {
        atomicMax(&k.red[7], 0x7fffffffffffffffULL - (unsigned long long)bad);
        k.red[8] = (unsigned long long)badf;
    }
}

}  // namespace sts
