// sts_march.cuh -- v3 loop-2 pass kernel: y-marching row sweep (sm_100a, fp64).
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

struct RingRow {                 // one old-iterate row (slot-major: one base address per row)
    double U[RW], V[RW], P[RW], T[RW], R[RW], G[RW];
    uint32_t KK[RW];
};
struct FluxRow {                 // face densities / fluxes of one row, (p/T)^{n-1} of that row
    double RU[RW], FX[RW], RV[RW], FY[RW], R1[RW];
};
struct MarchSmem {
    RingRow ring[RS];
    FluxRow fr[2];
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
__device__ __forceinline__ void ring_issue(MarchSmem& s, const MarchParams& m, int I0, int j, int sl)
{
    const Params& k = m.k;
    RingRow& r = s.ring[sl];
    const long long ro = (long long)j * k.pitch;
    for (int lc = threadIdx.x; lc < RW; lc += MX) {
        const int li = I0 - 4 + lc - k.gi0 + OFF;        // stored local column
        const bool col_ok = li >= 0 && li < k.pitch;
        if (j >= 0 && j < k.ny && col_ok) {
            const long long id = ro + li;
            cp_async8(&r.U[lc], k.u_o + id);
            cp_async8(&r.V[lc], k.v_o + id);
            cp_async8(&r.P[lc], k.p_o + id);
            cp_async8(&r.T[lc], k.T_o + id);
            cp_async4(&r.KK[lc], m.kind + id);
        } else if (j == k.ny && col_ok) {          // top wall row: v = 0 (WALL), no cells
            const long long id = ro + li;
            r.U[lc] = k.u_wt;
            cp_async8(&r.V[lc], k.v_o + id);
            r.P[lc] = 1.0;
            r.T[lc] = 1.0;
            cp_async4(&r.KK[lc], m.kind + id);
        } else {
            r.U[lc] = j < 0 ? k.u_wb : (j >= k.ny ? k.u_wt : 0.0);
            r.V[lc] = 0.0;
            r.P[lc] = 1.0;
            r.T[lc] = 1.0;
            r.KK[lc] = (uint32_t)CK_WALLY | ((uint32_t)FK_NONE << 8) | ((uint32_t)FK_NONE << 16);
        }
    }
    cp_commit();
}
// rho = p/T (Eq. pl5), Gamma = sqrt(T) (Eq. pl37) of ring row j
__device__ __forceinline__ void ring_derive(MarchSmem& s, int sl)
{
    RingRow& r = s.ring[sl];
    for (int lc = threadIdx.x; lc < RW; lc += MX) {
        const double Tv = r.T[lc];
        r.R[lc] = fdiv(r.P[lc], Tv);
        r.G[lc] = fsqrt(Tv);
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
    for (int j = js - 1; j <= js + 2; j++) ring_issue(s, m, I0, j, slot(j));
    cp_wait_all();
    __syncthreads();
    for (int j = js - 1; j <= js + 2; j++) ring_derive(s, slot(j));
    ring_issue(s, m, I0, js + 3, slot(js + 3));
    int sj = slot(js);                                  // ring slot of row j (incremental)

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
        const int sa = sj + 1 == RS ? 0 : sj + 1, sb = sa + 1 == RS ? 0 : sa + 1;
        const int sc = sb + 1 == RS ? 0 : sb + 1, sd = sc + 1 == RS ? 0 : sc + 1;
        const int sm = sj == 0 ? RS - 1 : sj - 1;
        RingRow& Rm = s.ring[sm];
        RingRow& R0 = s.ring[sj];
        RingRow& Ra = s.ring[sa];
        RingRow& Rb = s.ring[sb];
        RingRow& Rc = s.ring[sc];
        FluxRow& Fc = s.fr[j & 1];
        FluxRow& Fn = s.fr[(j + 1) & 1];
        const bool out_row = j >= J0;

        // prefetch the next row's n-1 / plane values (consumed one step later)
        double p1nn = ld(k.p_1, j + 2), T1nn = ld(k.T_1, j + 2);
        double u1n = ld(k.u_1, j + 1), v1nn = ldv(k.v_1, j + 2);
        double Ten = 0.0, uen = 0.0, vem = 0.0;
        if (!IMPL) { Ten = ld(k.Te, j + 1); uen = ld(k.ue, j + 1); vem = ldv(k.ve, j + 2); }

        cp_wait_all();
        __syncthreads();                                    // B0: ring row j+3 landed
        ring_issue(s, m, I0, j + 4, sd);

        // ================= stage A: row j+1 fluxes, link pieces =================
        ring_derive(s, sc);
        const uint32_t kw0 = R0.KK[lc], kw1 = Ra.KK[lc];
        // (p/T)^{n-1} of row j+1
        Fn.R1[lc] = fdiv(p1n, T1n == 0.0 ? 1.0 : T1n);
        // F^x, rho^u at u-face (i, j+1)  (Eqs. pl8, pl10, R1)
        double Fx1 = 0.0;
        {
            double ru = 0.0;
            const uint8_t uk = ukind(kw1);
            if (flux_face(uk)) {
                const double w = Ra.U[lc], r1 = Ra.R[lc - 1], r2 = Ra.R[lc];
                ru = w > 0.0 ? r1 : r2;
                if (TVD && ckind(Ra.KK[lc - 2]) == CK_FLUID && ckind(Ra.KK[lc - 1]) == CK_FLUID &&
                    ckind(kw1) == CK_FLUID && ckind(Ra.KK[lc + 1]) == CK_FLUID)
                    ru += psi_f(Ra.R[lc - 2], r1, r2, Ra.R[lc + 1], w) * (r2 - r1);
                Fx1 = ru * w * dy;
            }
            Fn.RU[lc] = ru;
            Fn.FX[lc] = Fx1;
        }
        // F^y, rho^v at v-face (i, j+1)  (Eqs. pl9, pl11, R1)
        double Fy1 = 0.0;
        {
            double rv = 0.0;
            if (vkind(kw1) == FK_ACTIVE) {
                const double w = Ra.V[lc], r1 = R0.R[lc], r2 = Ra.R[lc];
                rv = w > 0.0 ? r1 : r2;
                if (TVD && ckind(Rm.KK[lc]) == CK_FLUID && ckind(kw0) == CK_FLUID && ckind(kw1) == CK_FLUID &&
                    ckind(Rb.KK[lc]) == CK_FLUID)
                    rv += psi_f(Rm.R[lc], r1, r2, Rb.R[lc], w) * (r2 - r1);
                Fy1 = rv * w * dx;
            }
            Fn.RV[lc] = rv;
            Fn.FY[lc] = Fy1;
        }
        // T-eq x-face pieces at u-face (i, j): a^T_1 of cell i, a^T_2 of cell i-1 (Eqs. pl31-pl33)
        {
            double pw = 0.0, pe = 0.0;
            const uint8_t kl = ckind(R0.KK[lc - 1]), kr = ckind(kw0);
            if (!wallish(kl) && !wallish(kr)) {
                const double F = Fc.FX[lc];
                const double g1 = R0.G[lc - 1], g2 = R0.G[lc];
                const double D = m.CT1_dydx * (2.0 * g1 * g2 * rcp(g1 + g2));
                double ps = 0.0;
                if (IMPL && TVD && ckind(R0.KK[lc - 2]) == CK_FLUID && kl == CK_FLUID && kr == CK_FLUID &&
                    ckind(R0.KK[lc + 1]) == CK_FLUID)
                    ps = psi_f(R0.T[lc - 2], R0.T[lc - 1], R0.T[lc], R0.T[lc + 1], R0.U[lc]);
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
                const double g1 = R0.G[lc], g2 = Ra.G[lc];
                const double D = m.CT1_dxdy * (2.0 * g1 * g2 * rcp(g1 + g2));
                double ps = 0.0;
                if (IMPL && TVD && ckind(Rm.KK[lc]) == CK_FLUID && kb == CK_FLUID && kt == CK_FLUID &&
                    ckind(Rb.KK[lc]) == CK_FLUID)
                    ps = psi_f(Rm.T[lc], R0.T[lc], Ra.T[lc], Rb.T[lc], Ra.V[lc]);
                ytN = (IMPL ? max0(-F) - F * ps : 0.0) + D;
                ytSn = (IMPL ? max0(F) - F * ps : 0.0) + D;
            }
        }
        // u-eq x pieces of cell (i, j): a^u_2 of face i, a^u_1 of face i+1 (transposed pl15)
        {
            double xe = 0.0, xw = 0.0, Fb = 0.0;
            if (ckind(kw0) == CK_FLUID) {
                const double ub = 0.5 * (R0.U[lc] + R0.U[lc + 1]);
                Fb = R0.R[lc] * ub * dy;
                const double D = 4.0 / 3.0 * m.B_dydx * R0.G[lc];
                double ps = 0.0;
                if (IMPL && TVD && ukind(R0.KK[lc - 1]) == FK_ACTIVE && ukind(kw0) == FK_ACTIVE &&
                    ukind(R0.KK[lc + 1]) == FK_ACTIVE && ukind(R0.KK[lc + 2]) == FK_ACTIVE)
                    ps = psi_f(R0.U[lc - 1], R0.U[lc], R0.U[lc + 1], R0.U[lc + 2], ub);
                xe = (IMPL ? max0(-Fb) - Fb * ps : 0.0) + D;
                xw = (IMPL ? max0(Fb) - Fb * ps : 0.0) + D;
            }
            s.XUE[lc] = xe;
            s.XUW[lc] = xw;
            s.FBX[lc] = Fb;
        }
        // u-eq tangential psi at (u column i, y^f_{j+1}) (fluxes need the neighbour: stage C)
        double upsi1 = 0.0, upsi2 = 0.0;
        if (IMPL && TVD && ukind(Rm.KK[lc]) == FK_ACTIVE && ukind(kw0) == FK_ACTIVE &&
            ukind(kw1) == FK_ACTIVE && ukind(Rb.KK[lc]) == FK_ACTIVE) {
            const double f1 = Rm.U[lc], f2 = R0.U[lc], f3 = Ra.U[lc], f4 = Rb.U[lc];
            upsi1 = psi_f(f1, f2, f3, f4, Ra.V[lc]);
            upsi2 = psi_f(f1, f2, f3, f4, Ra.V[lc - 1]);
        }
        // v-eq normal piece of cell (i, j+1): a^v_4 of v-face (i, j+1), a^v_3 of v-face (i, j+2)
        double vcN = 0.0, vcSn = 0.0, FbN = 0.0;
        if (ckind(kw1) == CK_FLUID) {
            const double vb = 0.5 * (Ra.V[lc] + Rb.V[lc]);
            FbN = Ra.R[lc] * vb * dx;
            const double D = 4.0 / 3.0 * m.B_dxdy * Ra.G[lc];
            double ps = 0.0;
            if (IMPL && TVD && vkind(kw0) == FK_ACTIVE && vkind(kw1) == FK_ACTIVE &&
                vkind(Rb.KK[lc]) == FK_ACTIVE && vkind(Rc.KK[lc]) == FK_ACTIVE)
                ps = psi_f(R0.V[lc], Ra.V[lc], Rb.V[lc], Rc.V[lc], vb);
            vcN = (IMPL ? max0(-FbN) - FbN * ps : 0.0) + D;
            vcSn = (IMPL ? max0(FbN) - FbN * ps : 0.0) + D;
        }
        // corner Gamma at (x^f_i, y^f_{j+1}) (R4, R5; BC spec 8)
        double gcN;
        {
            double sum = 0.0;
            int n = 0;
            const uint8_t a = ckind(R0.KK[lc - 1]), b = ckind(kw0), c = ckind(Ra.KK[lc - 1]), d = ckind(kw1);
            if (!wallish(a)) { sum += R0.G[lc - 1]; n++; }
            if (!wallish(b)) { sum += R0.G[lc]; n++; }
            if (!wallish(c)) { sum += Ra.G[lc - 1]; n++; }
            if (!wallish(d)) { sum += Ra.G[lc]; n++; }
            gcN = n == 4 ? 0.25 * sum : (n > 0 ? sum / n : 0.0);
            s.GC[lc] = gcN;
        }
        // v-eq tangential pieces at (u-face column i, v-row j+1): a^v_1 of v-face (i, j+1),
        // a^v_2 of v-face (i-1, j+1)
        double xvW, FwSum;
        {
            const double F1 = Fx1, F2 = Fc.FX[lc];     // rows j+1 (upper half) and j (lower half)
            double p1 = 0.0, p2 = 0.0;
            if (IMPL && TVD && vkind(Ra.KK[lc - 2]) == FK_ACTIVE && vkind(Ra.KK[lc - 1]) == FK_ACTIVE &&
                vkind(kw1) == FK_ACTIVE && vkind(Ra.KK[lc + 1]) == FK_ACTIVE) {
                const double f1 = Ra.V[lc - 2], f2 = Ra.V[lc - 1], f3 = Ra.V[lc], f4 = Ra.V[lc + 1];
                p1 = psi_f(f1, f2, f3, f4, Ra.U[lc]);
                p2 = psi_f(f1, f2, f3, f4, R0.U[lc]);
            }
            const double D = m.B_dydx * gcN;
            xvW = (IMPL ? 0.5 * (max0(F1) - F1 * p1 + max0(F2) - F2 * p2) : 0.0) + D;
            s.XVE[lc] = (IMPL ? 0.5 * (max0(-F1) - F1 * p1 + max0(-F2) - F2 * p2) : 0.0) + D;
            FwSum = F1 + F2;
            s.XVF[lc] = FwSum;
        }
        __syncthreads();                                    // B1

        // ================= stage C: T_{i,j}, u-hat_{i,j}, v-hat_{i,j+1} =================
        const double rP = R0.R[lc], gP = R0.G[lc];
        double TN = 0.0;
        if (ckind(kw0) == CK_FLUID) {
            const double tau = 2.1904 * k.Kn * rcp(rP);   // Eq. pl39
            double a1, a2, a3, a4, T1, T2, T3, T4, FW = 0.0, FE = 0.0, FSl = 0.0, FNl = 0.0;
            uint8_t kn = ckind(R0.KK[lc - 1]);
            if (wallish(kn)) { a1 = k.CT1 * gP * dy * rcp(0.5 * dx + tau); T1 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a1 = s.XTW[lc]; FW = Fc.FX[lc]; T1 = R0.T[lc - 1]; }
            kn = ckind(R0.KK[lc + 1]);
            if (wallish(kn)) { a2 = k.CT1 * gP * dy * rcp(0.5 * dx + tau); T2 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a2 = s.XTE[lc + 1]; FE = Fc.FX[lc + 1]; T2 = R0.T[lc + 1]; }
            kn = ckind(Rm.KK[lc]);
            if (wallish(kn)) { a3 = k.CT1 * gP * dx * rcp(0.5 * dy + tau); T3 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a3 = ytS; FSl = FS; T3 = Rm.T[lc]; }
            kn = ckind(kw1);
            if (wallish(kn)) { a4 = k.CT1 * gP * dx * rcp(0.5 * dy + tau); T4 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a4 = ytN; FNl = Fy1; T4 = Ra.T[lc]; }
            const double a0 = IMPL ? dt * (a1 + a2 + a3 + a4 + FE - FW + FNl - FSl) + rP * m.dV
                                   : dt * (a1 + a2 + a3 + a4) + rP * m.dV;
            // S^T_c, Eq. pl29 (R4 bilinear = 4-point mean; R9 sign)
            const double dudx = (R0.U[lc + 1] - R0.U[lc]) * m.inv_dx;
            const double dvdy = (Ra.V[lc] - R0.V[lc]) * m.inv_dy;
            const double vE = 0.25 * (R0.V[lc] + R0.V[lc + 1] + Ra.V[lc] + Ra.V[lc + 1]);
            const double vW = 0.25 * (R0.V[lc - 1] + R0.V[lc] + Ra.V[lc - 1] + Ra.V[lc]);
            const double uN = 0.25 * (R0.U[lc] + R0.U[lc + 1] + Ra.U[lc] + Ra.U[lc + 1]);
            const double uS = 0.25 * (Rm.U[lc] + Rm.U[lc + 1] + R0.U[lc] + R0.U[lc + 1]);
            const double shear = (vE - vW) * m.inv_dx + (uN - uS) * m.inv_dy;
            const double div = dudx + dvdy;
            const double Sc = (k.CT2 * gP * (2.0 * (dudx * dudx + dvdy * dvdy) + shear * shear - 2.0 / 3.0 * div * div)
                               + k.pw_sign * k.CT3 * R0.P[lc] * div) * m.dV;
            const double rhs = dt * (a1 * T1 + a2 * T2 + a3 * T3 + a4 * T4 + Sc + Tec) + Fc.R1[lc] * T1c * m.dV;
            TN = rhs * rcp(a0);
        }
        // u-eq at u-face (i, j)
        double uhat = 0.0, du = 0.0;
        double utSn, FsSumN;
        {
            // N tangential link pieces at y^f_{j+1} (both sides; the S side is carried)
            const double F1 = Fy1, F2 = Fn.FY[lc - 1];
            const double D = m.B_dxdy * gcN;
            const double a4p = (IMPL ? 0.5 * (max0(-F1) - F1 * upsi1 + max0(-F2) - F2 * upsi2) : 0.0) + D;
            utSn = (IMPL ? 0.5 * (max0(F1) - F1 * upsi1 + max0(F2) - F2 * upsi2) : 0.0) + D;
            FsSumN = F1 + F2;
            if (ukind(kw0) == FK_ACTIVE) {
                const double rL = R0.R[lc - 1], rR = rP, gL = R0.G[lc - 1], gR = gP;
                const double gadj = 0.5 * (gL + gR);
                const double zeta = 1.1466 * k.Kn * rcp(0.5 * (rL + rR));     // Eq. pl38
                const double a1 = s.XUW[lc - 1], a2 = s.XUE[lc];
                const double FbW = s.FBX[lc - 1], FbE = s.FBX[lc];
                double a3, a4, uS, uN, FsS = 0.0, FnS = 0.0;
                const uint8_t kl = ckind(Rm.KK[lc - 1]), kr = ckind(Rm.KK[lc]);
                if (kl == CK_WALLY || (kl == CK_SOLID && kr == CK_SOLID)) {
                    a3 = k.B * gadj * dx * rcp(0.5 * dy + zeta); uS = kl == CK_WALLY ? k.u_wb : 0.0;
                } else { a3 = utS; FsS = FsSum; uS = Rm.U[lc]; }
                const uint8_t ml = ckind(Ra.KK[lc - 1]), mr = ckind(kw1);
                if (ml == CK_WALLY || (ml == CK_SOLID && mr == CK_SOLID)) {
                    a4 = k.B * gadj * dx * rcp(0.5 * dy + zeta); uN = ml == CK_WALLY ? k.u_wt : 0.0;
                } else { a4 = a4p; FnS = FsSumN; uN = Ra.U[lc]; }
                const double tterm = (rR + rL) * m.c_t;
                const double a0 = IMPL ? a1 + a2 + a3 + a4 + FbE - FbW + 0.5 * (FnS - FsS) + tterm
                                       : a1 + a2 + a3 + a4 + tterm;
                const double b = (Fc.R1[lc] + Fc.R1[lc - 1]) * m.c_t * u1c
                               + k.B * (gcN * (Ra.V[lc] - Ra.V[lc - 1]) - gcP * (R0.V[lc] - R0.V[lc - 1])
                                        - 2.0 / 3.0 * gR * (Ra.V[lc] - R0.V[lc])
                                        + 2.0 / 3.0 * gL * (Ra.V[lc - 1] - R0.V[lc - 1]))
                               + k.g_x * (rR + rL) * m.half_dV;
                const double r = rcp(a0);
                uhat = (a1 * R0.U[lc - 1] + a2 * R0.U[lc + 1] + a3 * uS + a4 * uN + b + uec) * r;
                du = m.A_dy * r;
            }
            s.UH[lc] = uhat;
            s.DU[lc] = du;
        }
        // v-eq at v-face (i, j+1)
        double vhatN = 0.0, dvN = 0.0;
        if (vkind(kw1) == FK_ACTIVE) {
            const double rB = rP, rT = Ra.R[lc], gB = gP, gT = Ra.G[lc];
            const double gadj = 0.5 * (gB + gT);
            const double zeta = 1.1466 * k.Kn * rcp(0.5 * (rB + rT));
            double a1, a2, vW, vE, FwS = 0.0, FeS = 0.0;
            if (ckind(R0.KK[lc - 1]) == CK_SOLID && ckind(Ra.KK[lc - 1]) == CK_SOLID) {
                a1 = k.B * gadj * dy * rcp(0.5 * dx + zeta); vW = 0.0;
            } else { a1 = xvW; FwS = FwSum; vW = Ra.V[lc - 1]; }
            if (ckind(R0.KK[lc + 1]) == CK_SOLID && ckind(Ra.KK[lc + 1]) == CK_SOLID) {
                a2 = k.B * gadj * dy * rcp(0.5 * dx + zeta); vE = 0.0;
            } else { a2 = s.XVE[lc + 1]; FeS = s.XVF[lc + 1]; vE = Ra.V[lc + 1]; }
            const double a3 = vcS, a4 = vcN;
            const double tterm = (rT + rB) * m.c_t;
            const double a0 = IMPL ? a1 + a2 + a3 + a4 + 0.5 * (FeS - FwS) + FbN - FbS + tterm
                                   : a1 + a2 + a3 + a4 + tterm;
            const double b = (Fn.R1[lc] + Fc.R1[lc]) * m.c_t * v1n
                           + k.B * (s.GC[lc + 1] * (Ra.U[lc + 1] - R0.U[lc + 1]) - gcN * (Ra.U[lc] - R0.U[lc])
                                    - 2.0 / 3.0 * gT * (Ra.U[lc + 1] - Ra.U[lc])
                                    + 2.0 / 3.0 * gB * (R0.U[lc + 1] - R0.U[lc]))
                           + k.g_y * (rT + rB) * m.half_dV;
            const double r = rcp(a0);
            vhatN = (a1 * vW + a2 * vE + a3 * R0.V[lc] + a4 * Rb.V[lc] + b + ven) * r;
            dvN = m.A_dx * r;
        }
        __syncthreads();                                    // B2

        // ================= stage D: p_{i,j} (Eqs. pl23-pl24) =================
        double pn = R0.P[lc];
        if (ckind(kw0) == CK_FLUID) {
            double apW = 0.0, apE = 0.0, apS = 0.0, apN = 0.0, bpW = 0.0, bpE = 0.0, bpS = 0.0, bpN = 0.0, sum = 0.0;
            const uint8_t kwf = ukind(kw0), kef = ukind(R0.KK[lc + 1]);
            if (kwf == FK_ACTIVE) {
                const double r = Fc.RU[lc];
                apW = r * du * dy; bpW = r * uhat * dy; sum += apW * R0.P[lc - 1];
            } else if (kwf == FK_INLET) bpW = Fc.RU[lc] * k.u_in * dy;
            if (kef == FK_ACTIVE) {
                const double r = Fc.RU[lc + 1];
                apE = r * s.DU[lc + 1] * dy; bpE = r * s.UH[lc + 1] * dy; sum += apE * R0.P[lc + 1];
            } else if (kef == FK_OUTLET) bpE = Fc.RU[lc + 1] * R0.U[lc] * dy;
            if (vkind(kw0) == FK_ACTIVE) {
                const double r = Fc.RV[lc];
                apS = r * dvP * dx; bpS = r * vhatP * dx; sum += apS * Rm.P[lc];
            }
            if (vkind(kw1) == FK_ACTIVE) {
                const double r = Fn.RV[lc];
                apN = r * dvN * dx; bpN = r * vhatN * dx; sum += apN * Ra.P[lc];
            }
            const double a0 = m.dV * rcp(TN) + (apW + apE + apS + apN) * dt;
            const double bp = Fc.R1[lc] * m.dV - (bpE - bpW + bpN - bpS) * dt;
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
                r_dT = nmax(r_dT, fabs(TN - R0.T[lc]));
                r_dp = nmax(r_dp, fabs(pn - R0.P[lc]));
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
                r_du = nmax(r_du, fabs(un - R0.U[lc]));
                r_vel = nmax(r_vel, fabs(un));
            } else if (ku == FK_INLET) un = k.u_in;
            else un = 0.0;
            k.u_w[id] = un;
            if (gi == k.nx - 1 && k.xbc == 0) k.u_w[id + 1] = R0.U[lc];   // outlet face (BC spec 3)
            double vn = 0.0;
            if (vkind(kw0) == FK_ACTIVE) {
                vn = vhatP - dvP * (pn - pnP);
                r_dv = nmax(r_dv, fabs(vn - R0.V[lc]));
                r_vel = nmax(r_vel, fabs(vn));
            }
            k.v_w[id] = vn;
            if (k.xbc == 0) {
                if (gi == k.nx - 1) {
                    const double pv = ckind(kw0) == CK_FLUID ? pn : R0.P[lc];
                    const double Tv = ckind(kw0) == CK_FLUID ? TN : R0.T[lc];
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
        sj = sa;
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
