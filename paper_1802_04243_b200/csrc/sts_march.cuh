// sts_march.cuh -- v4 loop-2 pass kernel: y-marching row sweep (sm_100a, fp64).
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
//  - the paper separates fluid control volumes from wall control volumes
//    (Fig. 9): here every stage has a "regular" instance (REG =
//    true: the +-3 window of the point is all fluid, so no kind test, wall
//    link or TVD-validity test is compiled in) and a general instance; the
//    choice is a per-cell bit precomputed on the host, so it is a function of
//    the cell alone (decomposition-invariant);
//  - divisions become MUFU reciprocals + Newton steps; the mesh constants
//    (dy/dx, dx dy/(2 dt), ...) are precomputed on the host.
// A segment starts 3 rows early (warm-up) so that every carried quantity is
// exact when its first output row is reached.
#pragma once

#include <type_traits>

#include "sts_common.cuh"

namespace sts {

constexpr int MX = 128;          // threads per CTA = columns handled per strip
constexpr int MW = MX - 3;       // owned columns per strip
constexpr int RW = MX + 8;       // ring row width: columns I0-4-shift .. (TMA rows 16-byte aligned, shift in 0..3)
constexpr int RS = 6;            // ring slots
constexpr int WARM = 3;          // warm-up rows per segment: the longest carried chain is
                                 // E(J0) <- D(J0-1) <- C(J0-2) <- A(J0-3); 2 rows fail the bitwise
                                 // segmentation tests, 3 pass them for every variant down to 1-row segments
constexpr uint32_t REG_BIT = 1u << 24;   // kind-word bit: the +-3 window is all fluid
constexpr int ALLREG_BIT = 1;            // launch-order flag (int4 .w): every point of the CTA is regular

struct MarchParams {
    Params k;                    // v1 parameter block (pointers, constants)
    const uint32_t* kind;        // packed kinds: ck | uk << 8 | vk << 16 | regular << 24, (ny+1) x pitch
    const int4* order;           // CTA schedule: blockIdx.x -> {strip, first row J0, end row J1, flags}
    double inv_dx, inv_dy, CT1_dydx, CT1_dxdy, B_dydx, B_dxdy, c_t, dV, A_dy, A_dx, half_dV;
    double B43_dydx, B43_dxdy;   // 4/3 B dy/dx, 4/3 B dx/dy (normal viscous links)
    double q_dx, q_dy;           // 1/(4 dx), 1/(4 dy) (bilinear differences in S^T_c)
    double h_dx, h_dy, inv_dt;   // 1/(2 dx), 1/(2 dy), 1/dt (pressure work, R9)
    double pw_a;                 // C^T3 for the C^T3 Dp/Dt form of R9, else 0
    const int* done;             // graph-driven loop 2 (tolerance mode): loop finished -> the pass is a no-op
    unsigned long long* bad;     // sticky first-bad-state key of the advance call (bad_key)
    int pass_key;                // 0xFFFFF - pass index within the advance call
    // non-uniform mesh (NU instances): Delta x of every stored local
    // column (pitch entries, ghost rules applied by the host) and Delta y of rows
    // -PADY .. ny+PADY-1 at dyp[j + PADY] (rows beyond a wall take the wall row's step)
    const double* dxl;
    const double* dyp;
    // fused halo: the pass epilogue also stores this slab's first /
    // last OFF owned columns of u, v, p, T (the conv kernel: u^exp, v^exp, T^exp)
    // straight into the ghost columns of the left [0] / right [1] neighbour's copy of
    // the same snapshot -- peer-mapped pointers (NVLink P2P, CUDA IPC, or the same
    // device for in-process slabs), null = no such neighbour.  Neighbour element of
    // local (row j, column l): j * nb_pitch + l + nb_shift.
    double* nb_u[2];
    double* nb_v[2];
    double* nb_p[2];
    double* nb_T[2];
    int nb_pitch[2], nb_shift[2];
    // loop 3 (L3 instances, reading R41): the previous T-p sweep's
    // pressure and temperature (local layout) -- the energy equation's neighbour
    // T, unsteady density p/T and pressure work, the pressure equation's neighbour p
    const double* p3;
    const double* T3;
    int force_general;           // test hook (STS_FORCE_GENERAL): every point of the general kernel general
};
// A point's view of the loop-3 iterate: element id = j pitch + local column.
struct Tp3 {
    const double* p;
    const double* T;
    int id, pitch;
    __device__ __forceinline__ double P(int o) const { return __ldg(p + id + o); }
    __device__ __forceinline__ double Tt(int o) const { return __ldg(T + id + o); }
};
constexpr int PADY = 4;

// Store one point's new values into the neighbours' ghost columns (fused halo):
// the first OFF owned columns go left, the last OFF right (both when the slab is
// narrower than 2 OFF).  Cells that are not fluid keep their p, T everywhere.
__device__ __forceinline__ void halo_store(const MarchParams& m, int j, int col, bool fluid,
                                           double u, double v, double p, double T)
{
#pragma unroll
    for (int sd = 0; sd < 2; sd++) {
        if (m.nb_u[sd] && (sd == 0 ? col < 2 * OFF : col >= m.k.nloc)) {
            const long long id = (long long)j * m.nb_pitch[sd] + col + m.nb_shift[sd];
            m.nb_u[sd][id] = u;
            m.nb_v[sd][id] = v;
            if (fluid) { m.nb_p[sd][id] = p; m.nb_T[sd][id] = T; }
        }
    }
}

// Mesh steps around a point of a non-uniform mesh: the column widths of the
// CTA's ring columns (shared memory, ring column index) and the heights of
// rows j-1 .. j+3 of the row step (Fig. 5).
struct Geo {
    const double* dxr;
    double ym, y0, ya, yb, yc;
};

// fp64 reciprocal: MUFU.RCP64H seed (relative error <= 2^-19.9, measured) and
// one third-order step r (1 + e + e^2), e = 1 - x r: error e^3 < 2^-59 plus
// rounding, max 1 ulp over 2e8 samples in [2^-20, 2^20] (tools/rcp_accuracy.cu);
// three dependent fp64 operations instead of the four of two Newton steps.
__device__ __forceinline__ double rcp(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
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
// The two flow directions share one code path (the upstream difference is
// selected); the early exits skip the reciprocal on flat / extremum stencils,
// which dominate the free stream.  (A fully branch-free form that always forms
// the quotient measured 15 % slower on implicit TVD.)
__device__ __forceinline__ double psi_f(double f1, double f2, double f3, double f4, double w)
{
    const double b = f3 - f2;
    if (fabs(b) <= 1e-12 * (1.0 + fabs(f2) + fabs(f3))) return 0.0;   // R37
    const bool up = w > 0.0;
    const double a = up ? f2 - f1 : f4 - f3;
    if (!(a * b > 0.0)) return 0.0;                                    // r <= 0 (R6)
    const double q = fdiv(a, a + b);
    return up ? q : -q;
}

// psi_s of Eq. pl15_2 on a general mesh, Van Leer psi(r) = 2r/(1+r)
// for r > 0 multiplied out: up (v > 0) 2 d2 a / ((d1 + d2) b + (d2 + d3) a),
// a = f2 - f1; down -2 d3 a / ((d3 + d4) b + (d2 + d3) a), a = f4 - f3; b = f3 - f2.
// Same guards as psi_f (R37, R6); equals psi_f's a / (a + b) on a uniform mesh.
__device__ __forceinline__ double psi_s_nu(double f1, double f2, double f3, double f4,
                                           double d1, double d2, double d3, double d4, double w)
{
    const double b = f3 - f2;
    if (fabs(b) <= 1e-12 * (1.0 + fabs(f2) + fabs(f3))) return 0.0;   // R37
    const bool up = w > 0.0;
    const double a = up ? f2 - f1 : f4 - f3;
    if (!(a * b > 0.0)) return 0.0;                                    // r <= 0 (R6)
    const double q = fdiv(2.0 * (up ? d2 : d3) * a, (up ? d1 + d2 : d3 + d4) * b + (d2 + d3) * a);
    return up ? q : -q;
}
// psi_c of Eq. pl15_1: up d2 a / (d1 b + d2 a), down -d2 a / (d3 b + d2 a).
__device__ __forceinline__ double psi_c_nu(double f1, double f2, double f3, double f4,
                                           double d1, double d2, double d3, double w)
{
    const double b = f3 - f2;
    if (fabs(b) <= 1e-12 * (1.0 + fabs(f2) + fabs(f3))) return 0.0;   // R37
    const bool up = w > 0.0;
    const double a = up ? f2 - f1 : f4 - f3;
    if (!(a * b > 0.0)) return 0.0;                                    // r <= 0 (R6)
    const double q = fdiv(d2 * a, (up ? d1 : d3) * b + d2 * a);
    return up ? q : -q;
}
// Linear-interpolation weight of the node left of a face between nodes of
// widths dl, dr (reading R4): dr / (dl + dr).
__device__ __forceinline__ double wleft(double dl, double dr) { return dr / (dl + dr); }

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

// ---- TMA (bulk async copy) rows with mbarrier completion.  Work beyond one
// element per thread is spread over different warps (a CTA advances at the
// pace of its slowest warp): warp 1 derives the ring columns beyond MX, the
// first lane of warp 2 issues the row copies.
constexpr int TMA_THREAD = 64;
constexpr int DERIVE_EXTRA_WARP = 1;
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, int parity)
{
    asm volatile("{\n\t.reg .pred P1;\n"
                 "WAIT:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                 "\t@!P1 bra WAIT;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_row(void* dst, const void* src, unsigned bytes, unsigned long long* b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

struct RingRow {                 // one old-iterate row (slot-major: one base address per row)
    double U[RW], V[RW], P[RW], T[RW], R[RW], G[RW];
    uint32_t KK[RW];
};
static_assert(sizeof(RingRow) % 16 == 0 && (RW * 4) % 16 == 0, "TMA rows need 16-byte alignment");
struct FluxRow {                 // face densities / fluxes of one row
    double RU[RW], FX[RW], FY[RW];   // (rho^v stays in registers: only the own column reads it)
};
// 54.7 KB: four CTAs (16 warps) per SM.  Pieces a neighbour can recompute with
// the same operations (E-side coefficients = W-side - F, F-bar^x, corner Gamma)
// are not stored.
struct MarchSmem {
    RingRow ring[RS];
    FluxRow fr[2];
    double R1[RW];               // (p/T)^{n-1} of row j (row j+1 is written in stage E)
    double XTW[RW];              // T-eq W coefficient of face i (stage C)
    double XUW[RW], XVW[RW];     // (the flux sum F^x(j) + F^x(j+1) of a face is re-read from the flux rows)
    double UH[RW], DU[RW];
    double PN[RW];               // p_new of row j (stages D-E): a row of its own, so no row-start barrier
    unsigned long long mbar[RS]; // TMA completion barrier of each ring slot (u, v, p, T rows)
};
// resident CTAs per SM: 4 (128 registers, 16 warps) for every variant (implicit TVD
// spills 12 B at 128 registers and is still 4 % faster than at 3 CTAs / 154 registers)
#ifndef STS_MARCH_CTAS
#define STS_MARCH_CTAS 4
#endif
constexpr int MARCH_CTAS = STS_MARCH_CTAS;
// max that ignores a NaN operand (NaN u / v are flagged separately, T / p by the bad-state test)
__device__ __forceinline__ double dmax(double m, double x) { return x > m ? x : m; }

__device__ __forceinline__ int slot(int j) { return (j + 4 * RS) % RS; }
__device__ __forceinline__ uint8_t ckind(uint32_t w) { return (uint8_t)(w & 0xff); }
__device__ __forceinline__ uint8_t ukind(uint32_t w) { return (uint8_t)((w >> 8) & 0xff); }
__device__ __forceinline__ uint8_t vkind(uint32_t w) { return (uint8_t)((w >> 16) & 0xff); }

// kind predicates; with REG every one folds to its regular-point value
template <bool REG> __device__ __forceinline__ bool cF(uint32_t w) { return REG || ckind(w) == CK_FLUID; }
template <bool REG> __device__ __forceinline__ bool cW(uint32_t w) { return !REG && wallish(ckind(w)); }
template <bool REG> __device__ __forceinline__ bool uA(uint32_t w) { return REG || ukind(w) == FK_ACTIVE; }
template <bool REG> __device__ __forceinline__ bool uFl(uint32_t w) { return REG || flux_face(ukind(w)); }
template <bool REG> __device__ __forceinline__ bool vA(uint32_t w) { return REG || vkind(w) == FK_ACTIVE; }

// 1/sqrt(x), x > 0: MUFU seed and one third-order step
// y (1 + e/2 + 3 e^2/8), e = 1 - x y^2 (max 2 ulp measured; two Newton steps: 2.9)
__device__ __forceinline__ double frsqrt(double x)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}
// rho = p/T (Eq. pl5), Gamma = sqrt(T) (Eq. pl37) of ring row j from one
// reciprocal square root y = T^(-1/2): Gamma = T y, rho = p y^2 (~2 ulp; the
// explicit planes need no Gamma)
template <bool WITH_GAMMA = true, class ROW = RingRow>
__device__ __forceinline__ void ring_derive(ROW& r)
{
    const int t = threadIdx.x, xl = t - 32 * DERIVE_EXTRA_WARP;
    const int n = (xl >= 0 && xl < RW - MX) ? 2 : 1;
    for (int q = 0; q < n; q++) {
        const int lc = q == 0 ? t : MX + xl;
        const double Tv = r.T[lc];
        // the same rho bits with or without Gamma: the explicit planes computed in the
        // first pass (N2) must equal conv_march_kernel's
        const double y = frsqrt(Tv);
        r.R[lc] = r.P[lc] * (y * y);
        if constexpr (WITH_GAMMA) r.G[lc] = Tv * y;
    }
}
template <bool WITH_GAMMA = true>
__device__ __forceinline__ void ring_derive(MarchSmem& s, int sl)
{
    ring_derive<WITH_GAMMA>(s.ring[sl]);
}

// Quantities carried from row step j-1 to row step j (register rotation).
struct Carry {
    double ytS, FS;       // T-eq south link piece / flux at v-face (i, j)
    double utS, FsSum;    // u-eq south tangential piece / half-flux sum at y^f_j
    double vcS, FbS;      // v-eq south normal piece (cell (i, j)) / F-bar
    double vhatP, dvP;    // v-hat, d^v at v-face (i, j)
    double pnP;           // p_new(i, j-1)
    double gcP;           // corner Gamma (i, j)
    double rvS;           // rho^v at v-face (i, j)
};
// Values passed between the stages of one row step.
struct StepVars {
    double Fx1, Fy1;              // F^x (i, j+1), F^y (i, j+1)
    double ytN, ytSn;             // T-eq y pieces at v-face (i, j+1)
    double upsi1, upsi2;          // u-eq tangential psi at y^f_{j+1}
    double vcN, vcSn, FbN;        // v-eq normal pieces of cell (i, j+1)
    double gcN;                   // corner Gamma (i, j+1)
    double xvW, FwSum;            // v-eq tangential W piece / flux sum at x^f_i, v-row j+1
    double xe, Fb;                // u-eq E coefficient of face i / F-bar^x of cell (i, j)
    double r1n;                   // (p/T)^{n-1} (i, j+1)
    double rv1;                   // rho^v at v-face (i, j+1)
    double TN, uhat, du, utSn, FsSumN, vhatN, dvN, pn;
};
struct NM1 {                      // n-1 state / explicit planes at this thread's points
    double p1n, T1n;              // row j+1
    double T1c, u1c, v1n;         // T^{n-1}(i, j), u^{n-1}(i, j), v^{n-1}(i, j+1)
    double Tec, uec, ven;         // T^exp(i, j), u^exp(i, j), v^exp(i, j+1)
};

// Ring row r into slot sl (march kernel).  c0 = stored column of ring column 0,
// a multiple of 4, so every double and kind row starts 16-byte aligned; `tma` = the CTA's window
// [c0, c0 + RW) lies inside the stored columns.  Rows inside the channel are
// five TMA bulk copies (RW doubles of u, v, p, T; RW packed kind words) issued
// by one thread and completing on the slot's mbarrier.  Every other row (beyond a channel wall, or a window that
// leaves the stored columns) is filled by the threads exactly as ring_issue
// does, and the issuing thread arrives on the mbarrier without bytes, so the
// slot's phase advances either way.
template <class SM>   // MarchSmem or ConvSmem (both hold ring[RS] and mbar[RS])
__device__ __forceinline__ void ring_issue_tma(SM& s, int sl, const MarchParams& m, int c0, bool tma, int r,
                                               bool kinds = true)   // false: an all-regular CTA reads no kinds
{
    const Params& k = m.k;
    auto& R = s.ring[sl];
    const int t = threadIdx.x;
    const bool row_in = (unsigned)r < (unsigned)k.ny;
    if (tma && row_in) {
        const int base = r * k.pitch + c0;
        if (t == TMA_THREAD) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // earlier generic writes of the slot
            mbar_expect_tx(&s.mbar[sl], 4u * RW * 8u + (kinds ? RW * 4u : 0u));
            tma_row(R.U, k.u_o + base, RW * 8, &s.mbar[sl]);
            tma_row(R.V, k.v_o + base, RW * 8, &s.mbar[sl]);
            tma_row(R.P, k.p_o + base, RW * 8, &s.mbar[sl]);
            tma_row(R.T, k.T_o + base, RW * 8, &s.mbar[sl]);
            if (kinds) tma_row(R.KK, m.kind + base, RW * 4, &s.mbar[sl]);
        }
    } else {
        for (int c = t; c < RW; c += MX) {
            const int li = c0 + c;
            const bool col_ok = li >= 0 && li < k.pitch;
            const int id = r * k.pitch + li;
            if (row_in && col_ok) {
                cp_async8(&R.U[c], k.u_o + id);
                cp_async8(&R.V[c], k.v_o + id);
                cp_async8(&R.P[c], k.p_o + id);
                cp_async8(&R.T[c], k.T_o + id);
                cp_async4(&R.KK[c], m.kind + id);
            } else if (r == k.ny && col_ok) {          // top wall row: v = 0 (WALL), no cells
                R.U[c] = k.u_wt;
                cp_async8(&R.V[c], k.v_o + id);
                R.P[c] = 1.0;
                R.T[c] = 1.0;
                cp_async4(&R.KK[c], m.kind + id);
            } else {
                R.U[c] = r < 0 ? k.u_wb : (r >= k.ny ? k.u_wt : 0.0);
                R.V[c] = 0.0;
                R.P[c] = 1.0;
                R.T[c] = 1.0;
                R.KK[c] = (uint32_t)CK_WALLY | ((uint32_t)FK_NONE << 8) | ((uint32_t)FK_NONE << 16);
            }
        }
        if (t == TMA_THREAD) mbar_arrive(&s.mbar[sl]);
    }
    cp_commit();
}

// Convective part of an upwind/TVD link coefficient, max(0, F) - F psi (Eqs. pl15,
// pl31); psi is the constant 0 without TVD, and F * 0 must not be formed
// (IEEE cannot fold it: F * 0 is NaN for F = inf).
#define STS_LINK(F, ps) (TVD ? FMA(-(F), (ps), max0(F)) : max0(F))

// ================= stage A: row j+1 fluxes, link pieces =================
// NU: the non-uniform-mesh instance (general points only): every step of the
// uniform shortcuts is replaced by the printed general-mesh form (Eqs. pl8-pl16,
// pl31-pl33, pl15_1-pl15_2; reading R4 for the corner Gamma).
template <bool IMPL, bool TVD, bool REG, bool NU = false>
__device__ __forceinline__ void stage_A(MarchSmem& s, const MarchParams& m, int lc, const RingRow& Rm,
                                        const RingRow& R0, const RingRow& Ra, const RingRow& Rb,
                                        const RingRow& Rc, const FluxRow& Fc, FluxRow& Fn, const NM1& nm,
                                        StepVars& v, const Geo& g)
{
    static_assert(!(NU && REG), "non-uniform meshes run the general instances only");
    const double dx = NU ? g.dxr[lc] : m.k.dx;
    const double dya = NU ? g.ya : m.k.dy;           // Delta y of row j+1
    const uint32_t kw0 = R0.KK[lc], kw1 = Ra.KK[lc];
    auto X = [&](int o) { return g.dxr[lc + o]; };   // Delta x of the column at ring offset o (NU)
    // (p/T)^{n-1} of row j+1 (to shared memory in stage E)
    v.r1n = fdiv(nm.p1n, nm.T1n == 0.0 ? 1.0 : nm.T1n);
    // F^x, rho^u at u-face (i, j+1)  (Eqs. pl8, pl10, R1)
    {
        double ru = 0.0, F = 0.0;
        if (uFl<REG>(kw1)) {
            const double w = Ra.U[lc], r1 = Ra.R[lc - 1], r2 = Ra.R[lc];
            ru = w > 0.0 ? r1 : r2;
            if (TVD && cF<REG>(Ra.KK[lc - 2]) && cF<REG>(Ra.KK[lc - 1]) && cF<REG>(kw1) && cF<REG>(Ra.KK[lc + 1]))
                ru = FMA(NU ? psi_s_nu(Ra.R[lc - 2], r1, r2, Ra.R[lc + 1], X(-2), X(-1), X(0), X(1), w)
                            : psi_f(Ra.R[lc - 2], r1, r2, Ra.R[lc + 1], w), r2 - r1, ru);
            F = MUL(MUL(ru, w), dya);
        }
        Fn.RU[lc] = ru;
        Fn.FX[lc] = F;
        v.Fx1 = F;
    }
    // F^y, rho^v at v-face (i, j+1)  (Eqs. pl9, pl11, R1)
    {
        double rv = 0.0, F = 0.0;
        if (vA<REG>(kw1)) {
            const double w = Ra.V[lc], r1 = R0.R[lc], r2 = Ra.R[lc];
            rv = w > 0.0 ? r1 : r2;
            if (TVD && cF<REG>(Rm.KK[lc]) && cF<REG>(kw0) && cF<REG>(kw1) && cF<REG>(Rb.KK[lc]))
                rv = FMA(NU ? psi_s_nu(Rm.R[lc], r1, r2, Rb.R[lc], g.ym, g.y0, g.ya, g.yb, w)
                            : psi_f(Rm.R[lc], r1, r2, Rb.R[lc], w), r2 - r1, rv);
            F = MUL(MUL(rv, w), dx);
        }
        v.rv1 = rv;
        Fn.FY[lc] = F;
        v.Fy1 = F;
    }
    // T-eq x-face pieces at u-face (i, j): a^T_1 of cell i, a^T_2 of cell i-1 (Eqs. pl31-pl33)
    // (max(0,-F) = max(0,F) - F: the consumer forms the E-side coefficient as XTW - F)
    {
        double pw = 0.0;
        const uint32_t kl = R0.KK[lc - 1];
        if (!cW<REG>(kl) && !cW<REG>(kw0)) {
            const double F = Fc.FX[lc];
            const double g1 = R0.G[lc - 1], g2 = R0.G[lc];
            // NU: C^T1 Gamma|_{x^f_i} Delta y_j / (0.5 (Delta x_{i-1} + Delta x_i)) with the harmonic
            // Gamma of Eq. pl33 = 2 C^T1 Delta y_j g1 g2 / (Delta x_{i-1} g2 + Delta x_i g1)
            const double hg = MUL(MUL(MUL(2.0, g1), g2), rcp(g1 + g2));      // (uniform mesh)
            double ps = 0.0;
            if (IMPL && TVD && cF<REG>(R0.KK[lc - 2]) && cF<REG>(kl) && cF<REG>(kw0) && cF<REG>(R0.KK[lc + 1]))
                ps = NU ? psi_s_nu(R0.T[lc - 2], R0.T[lc - 1], R0.T[lc], R0.T[lc + 1], X(-2), X(-1), X(0), X(1), R0.U[lc])
                        : psi_f(R0.T[lc - 2], R0.T[lc - 1], R0.T[lc], R0.T[lc + 1], R0.U[lc]);
            pw = NU ? (IMPL ? STS_LINK(F, ps) : 0.0) + 2.0 * m.k.CT1 * g.y0 * g1 * g2 * rcp(X(-1) * g2 + dx * g1)
                    : FMA(m.CT1_dydx, hg, IMPL ? STS_LINK(F, ps) : 0.0);
        }
        s.XTW[lc] = pw;
    }
    // T-eq y-face piece at v-face (i, j+1): a^T_4 of cell (i, j), a^T_3 of cell (i, j+1)
    v.ytN = 0.0;
    v.ytSn = 0.0;
    if (!cW<REG>(kw0) && !cW<REG>(kw1)) {
        const double F = v.Fy1;
        const double g1 = R0.G[lc], g2 = Ra.G[lc];
        const double hg = MUL(MUL(MUL(2.0, g1), g2), rcp(g1 + g2));          // (uniform mesh)
        double ps = 0.0;
        if (IMPL && TVD && cF<REG>(Rm.KK[lc]) && cF<REG>(kw0) && cF<REG>(kw1) && cF<REG>(Rb.KK[lc]))
            ps = NU ? psi_s_nu(Rm.T[lc], R0.T[lc], Ra.T[lc], Rb.T[lc], g.ym, g.y0, g.ya, g.yb, Ra.V[lc])
                    : psi_f(Rm.T[lc], R0.T[lc], Ra.T[lc], Rb.T[lc], Ra.V[lc]);
        v.ytSn = NU ? (IMPL ? STS_LINK(F, ps) : 0.0) + 2.0 * m.k.CT1 * dx * g1 * g2 * rcp(g.y0 * g2 + g.ya * g1)
                    : FMA(m.CT1_dxdy, hg, IMPL ? STS_LINK(F, ps) : 0.0);
        v.ytN = IMPL ? v.ytSn - F : v.ytSn;
    }
    // u-eq x pieces of cell (i, j): a^u_2 of face i, a^u_1 of face i+1 (transposed pl15)
    {
        double xe = 0.0, xw = 0.0, Fb = 0.0;
        if (cF<REG>(kw0)) {
            const double ub = MUL(0.5, R0.U[lc] + R0.U[lc + 1]);
            Fb = MUL(MUL(R0.R[lc], ub), NU ? g.y0 : m.k.dy);
            // NU: 4/3 D^ux = 4/3 B Gamma_i Delta y_j / Delta x_i (transposed Eq. pl16)
            const double D = NU ? 4.0 / 3.0 * m.k.B * R0.G[lc] * g.y0 * rcp(dx) : 0.0;
            double ps = 0.0;
            if (IMPL && TVD && uA<REG>(R0.KK[lc - 1]) && uA<REG>(kw0) && uA<REG>(R0.KK[lc + 1]) &&
                uA<REG>(R0.KK[lc + 2]))
                ps = NU ? psi_c_nu(R0.U[lc - 1], R0.U[lc], R0.U[lc + 1], R0.U[lc + 2], X(-1), X(0), X(1), ub)
                        : psi_f(R0.U[lc - 1], R0.U[lc], R0.U[lc + 1], R0.U[lc + 2], ub);
            xw = NU ? (IMPL ? STS_LINK(Fb, ps) : 0.0) + D : FMA(m.B43_dydx, R0.G[lc], IMPL ? STS_LINK(Fb, ps) : 0.0);
            xe = IMPL ? xw - Fb : xw;
        }
        s.XUW[lc] = xw;              // a^u_1 of face i+1 (neighbour); a^u_2 and F-bar stay here
        v.xe = xe;
        v.Fb = Fb;
    }
    // u-eq tangential psi at (u column i, y^f_{j+1}) (fluxes need the neighbour: stage C)
    v.upsi1 = 0.0;
    v.upsi2 = 0.0;
    if (IMPL && TVD && uA<REG>(Rm.KK[lc]) && uA<REG>(kw0) && uA<REG>(kw1) && uA<REG>(Rb.KK[lc])) {
        const double f1 = Rm.U[lc], f2 = R0.U[lc], f3 = Ra.U[lc], f4 = Rb.U[lc];
        if (NU) {
            v.upsi1 = psi_s_nu(f1, f2, f3, f4, g.ym, g.y0, g.ya, g.yb, Ra.V[lc]);
            v.upsi2 = psi_s_nu(f1, f2, f3, f4, g.ym, g.y0, g.ya, g.yb, Ra.V[lc - 1]);
        } else {
            v.upsi1 = psi_f(f1, f2, f3, f4, Ra.V[lc]);
            v.upsi2 = psi_f(f1, f2, f3, f4, Ra.V[lc - 1]);
        }
    }
    // v-eq normal piece of cell (i, j+1): a^v_4 of v-face (i, j+1), a^v_3 of v-face (i, j+2)
    v.vcN = 0.0;
    v.vcSn = 0.0;
    v.FbN = 0.0;
    if (cF<REG>(kw1)) {
        const double vb = MUL(0.5, Ra.V[lc] + Rb.V[lc]);
        v.FbN = MUL(MUL(Ra.R[lc], vb), dx);
        // NU: 4/3 D^vy_{i,j+2} = 4/3 B Gamma_{i,j+1} Delta x_i / Delta y_{j+1} (Eq. pl16)
        const double D = NU ? 4.0 / 3.0 * m.k.B * Ra.G[lc] * dx * rcp(g.ya) : 0.0;
        double ps = 0.0;
        if (IMPL && TVD && vA<REG>(kw0) && vA<REG>(kw1) && vA<REG>(Rb.KK[lc]) && vA<REG>(Rc.KK[lc]))
            ps = NU ? psi_c_nu(R0.V[lc], Ra.V[lc], Rb.V[lc], Rc.V[lc], g.y0, g.ya, g.yb, vb)
                    : psi_f(R0.V[lc], Ra.V[lc], Rb.V[lc], Rc.V[lc], vb);
        v.vcSn = NU ? (IMPL ? STS_LINK(v.FbN, ps) : 0.0) + D : FMA(m.B43_dxdy, Ra.G[lc], IMPL ? STS_LINK(v.FbN, ps) : 0.0);
        v.vcN = IMPL ? v.vcSn - v.FbN : v.vcSn;
    }
    // corner Gamma at (x^f_i, y^f_{j+1}) (R4, R5; BC spec 8)
    if (REG) {
        v.gcN = MUL(0.25, R0.G[lc - 1] + R0.G[lc] + Ra.G[lc - 1] + Ra.G[lc]);
    } else if (NU) {
        // bilinear weights of the four cell centres, renormalised to the cells kept
        const double wxl = wleft(X(-1), dx), wxr = 1.0 - wxl;
        const double wyb = wleft(g.y0, g.ya), wyt = 1.0 - wyb;
        double sum = 0.0, ws = 0.0;
        if (!wallish(ckind(R0.KK[lc - 1]))) { sum += wxl * wyb * R0.G[lc - 1]; ws += wxl * wyb; }
        if (!wallish(ckind(kw0))) { sum += wxr * wyb * R0.G[lc]; ws += wxr * wyb; }
        if (!wallish(ckind(Ra.KK[lc - 1]))) { sum += wxl * wyt * Ra.G[lc - 1]; ws += wxl * wyt; }
        if (!wallish(ckind(kw1))) { sum += wxr * wyt * Ra.G[lc]; ws += wxr * wyt; }
        v.gcN = ws > 0.0 ? sum / ws : 0.0;
    } else {
        double sum = 0.0;
        int n = 0;
        if (!wallish(ckind(R0.KK[lc - 1]))) { sum += R0.G[lc - 1]; n++; }
        if (!wallish(ckind(kw0))) { sum += R0.G[lc]; n++; }
        if (!wallish(ckind(Ra.KK[lc - 1]))) { sum += Ra.G[lc - 1]; n++; }
        if (!wallish(ckind(kw1))) { sum += Ra.G[lc]; n++; }
        v.gcN = n == 4 ? MUL(0.25, sum) : (n > 0 ? sum / n : 0.0);
    }
    // v-eq tangential pieces at (u-face column i, v-row j+1): a^v_1 of v-face (i, j+1),
    // a^v_2 of v-face (i-1, j+1)
    {
        const double F1 = v.Fx1, F2 = Fc.FX[lc];     // rows j+1 (upper half) and j (lower half)
        double p1 = 0.0, p2 = 0.0;
        if (IMPL && TVD && vA<REG>(Ra.KK[lc - 2]) && vA<REG>(Ra.KK[lc - 1]) && vA<REG>(kw1) &&
            vA<REG>(Ra.KK[lc + 1])) {
            const double f1 = Ra.V[lc - 2], f2 = Ra.V[lc - 1], f3 = Ra.V[lc], f4 = Ra.V[lc + 1];
            if (NU) {
                p1 = psi_s_nu(f1, f2, f3, f4, X(-2), X(-1), X(0), X(1), Ra.U[lc]);
                p2 = psi_s_nu(f1, f2, f3, f4, X(-2), X(-1), X(0), X(1), R0.U[lc]);
            } else {
                p1 = psi_f(f1, f2, f3, f4, Ra.U[lc]);
                p2 = psi_f(f1, f2, f3, f4, R0.U[lc]);
            }
        }
        // NU: D^vx_{i,j+1} = B Gamma|_{x^f_i} (Delta y_j + Delta y_{j+1}) / (Delta x_{i-1} + Delta x_i) (Eq. pl16)
        v.FwSum = F1 + F2;
        const double lk = IMPL ? MUL(0.5, STS_LINK(F1, p1) + STS_LINK(F2, p2)) : 0.0;
        v.xvW = NU ? lk + m.k.B * v.gcN * (g.y0 + g.ya) * rcp(X(-1) + dx) : FMA(m.B_dydx, v.gcN, lk);
        s.XVW[lc] = v.xvW;           // the E side of v-face (i-1, j+1) is XVW - (F^x(j) + F^x(j+1))/2
    }
}

// S^T_c pieces of a general (boundary) point.
// dv/dx + du/dy from mid-face velocities: bilinear interpolation between the four
// neighbouring nodes (R4 -- the 4-point mean on a uniform mesh), or on a face
// that lies on a wall the slip velocity of Eq. pl38 (R38).
template <bool NU>
__device__ __forceinline__ double shear_general(const RingRow& R0, const RingRow& Ra, const RingRow& Rm, int lc,
                                                double rP, const MarchParams& m, const Geo& g)
{
    const Params& k = m.k;
    const double dx = NU ? g.dxr[lc] : k.dx, dy = NU ? g.y0 : k.dy;
    const double zeta = 1.1466 * k.Kn * rcp(rP);
    auto slip = [&](double vP, double vw, double dn) { return (dn * vw + zeta * vP) * rcp(dn + zeta); };
    const double vs = R0.V[lc] + Ra.V[lc], us = R0.U[lc] + R0.U[lc + 1];
    const uint8_t kE = ckind(R0.KK[lc + 1]), kW = ckind(R0.KK[lc - 1]);
    const uint8_t kN = ckind(Ra.KK[lc]), kS = ckind(Rm.KK[lc]);
    double vE, vW, uN, uS;
    if (NU) {
        // node order as the 4-point mean: (i, j), (i+1, j), (i, j+1), (i+1, j+1) etc.
        const double wE = wleft(dx, g.dxr[lc + 1]), wW = wleft(g.dxr[lc - 1], dx);
        const double wN = wleft(dy, g.ya), wS = wleft(g.ym, dy);
        vE = 0.5 * wE * R0.V[lc] + 0.5 * (1.0 - wE) * R0.V[lc + 1] + 0.5 * wE * Ra.V[lc] + 0.5 * (1.0 - wE) * Ra.V[lc + 1];
        vW = 0.5 * wW * R0.V[lc - 1] + 0.5 * (1.0 - wW) * R0.V[lc] + 0.5 * wW * Ra.V[lc - 1] + 0.5 * (1.0 - wW) * Ra.V[lc];
        uN = 0.5 * wN * R0.U[lc] + 0.5 * wN * R0.U[lc + 1] + 0.5 * (1.0 - wN) * Ra.U[lc] + 0.5 * (1.0 - wN) * Ra.U[lc + 1];
        uS = 0.5 * wS * Rm.U[lc] + 0.5 * wS * Rm.U[lc + 1] + 0.5 * (1.0 - wS) * R0.U[lc] + 0.5 * (1.0 - wS) * R0.U[lc + 1];
        if (wallish(kE)) vE = slip(0.5 * vs, 0.0, 0.5 * dx);
        if (wallish(kW)) vW = slip(0.5 * vs, 0.0, 0.5 * dx);
        if (wallish(kN)) uN = slip(0.5 * us, kN == CK_WALLY ? k.u_wt : 0.0, 0.5 * dy);
        if (wallish(kS)) uS = slip(0.5 * us, kS == CK_WALLY ? k.u_wb : 0.0, 0.5 * dy);
    } else {
        // no wall around the point: exactly the regular instance's operations, so a
        // regular point gives the same bits in either instance (warp-uniform dispatch)
        if (!wallish(kE) && !wallish(kW) && !wallish(kN) && !wallish(kS))
            return FMA((R0.V[lc + 1] + Ra.V[lc + 1]) - (R0.V[lc - 1] + Ra.V[lc - 1]), m.q_dx,
                       MUL((Ra.U[lc] + Ra.U[lc + 1]) - (Rm.U[lc] + Rm.U[lc + 1]), m.q_dy));
        vE = wallish(kE) ? slip(0.5 * vs, 0.0, 0.5 * dx) : 0.25 * (vs + (R0.V[lc + 1] + Ra.V[lc + 1]));
        vW = wallish(kW) ? slip(0.5 * vs, 0.0, 0.5 * dx) : 0.25 * ((R0.V[lc - 1] + Ra.V[lc - 1]) + vs);
        uN = wallish(kN) ? slip(0.5 * us, kN == CK_WALLY ? k.u_wt : 0.0, 0.5 * dy)
                         : 0.25 * (us + (Ra.U[lc] + Ra.U[lc + 1]));
        uS = wallish(kS) ? slip(0.5 * us, kS == CK_WALLY ? k.u_wb : 0.0, 0.5 * dy)
                         : 0.25 * ((Rm.U[lc] + Rm.U[lc + 1]) + us);
    }
    return NU ? (vE - vW) * rcp(dx) + (uN - uS) * rcp(dy) : (vE - vW) * m.inv_dx + (uN - uS) * m.inv_dy;
}
// Pressure gradient of the C^T3 Dp/Dt term (R9) at a general point: face
// pressures = linear interpolation between the two cell centres (the mean on a
// uniform mesh), = p of the cell at a wall.
template <bool NU, bool L3 = false>
__device__ __forceinline__ void dp_general(const RingRow& R0, const RingRow& Ra, const RingRow& Rm, int lc,
                                           const MarchParams& m, const Geo& g, double& dpx, double& dpy,
                                           const Tp3& q3 = Tp3{})
{
    const bool nowall = !wallish(ckind(R0.KK[lc + 1])) && !wallish(ckind(R0.KK[lc - 1])) &&
                        !wallish(ckind(Ra.KK[lc])) && !wallish(ckind(Rm.KK[lc]));
    if (!NU && nowall) {                           // the regular instance's operations (same bits)
        dpx = MUL(L3 ? q3.P(1) - q3.P(-1) : R0.P[lc + 1] - R0.P[lc - 1], m.h_dx);
        dpy = MUL(L3 ? q3.P(q3.pitch) - q3.P(-q3.pitch) : Ra.P[lc] - Rm.P[lc], m.h_dy);
        return;
    }
    if (L3) {                                      // loop 3: the pressures of the previous sweep
        const double pc = q3.P(0);
        const double pe = wallish(ckind(R0.KK[lc + 1])) ? pc : 0.5 * (pc + q3.P(1));
        const double pw = wallish(ckind(R0.KK[lc - 1])) ? pc : 0.5 * (q3.P(-1) + pc);
        const double pn = wallish(ckind(Ra.KK[lc])) ? pc : 0.5 * (pc + q3.P(q3.pitch));
        const double ps = wallish(ckind(Rm.KK[lc])) ? pc : 0.5 * (q3.P(-q3.pitch) + pc);
        dpx = (pe - pw) * m.inv_dx;
        dpy = (pn - ps) * m.inv_dy;
        return;
    }
    const double pc = R0.P[lc];
    if (NU) {
        const double dx = g.dxr[lc], dxe = g.dxr[lc + 1], dxw = g.dxr[lc - 1];
        const double pe = wallish(ckind(R0.KK[lc + 1])) ? pc : (dxe * pc + dx * R0.P[lc + 1]) / (dx + dxe);
        const double pw = wallish(ckind(R0.KK[lc - 1])) ? pc : (dx * R0.P[lc - 1] + dxw * pc) / (dxw + dx);
        const double pn = wallish(ckind(Ra.KK[lc])) ? pc : (g.ya * pc + g.y0 * Ra.P[lc]) / (g.y0 + g.ya);
        const double ps = wallish(ckind(Rm.KK[lc])) ? pc : (g.y0 * Rm.P[lc] + g.ym * pc) / (g.ym + g.y0);
        dpx = (pe - pw) * rcp(dx);
        dpy = (pn - ps) * rcp(g.y0);
        return;
    }
    const double pe = wallish(ckind(R0.KK[lc + 1])) ? pc : 0.5 * (pc + R0.P[lc + 1]);
    const double pw = wallish(ckind(R0.KK[lc - 1])) ? pc : 0.5 * (R0.P[lc - 1] + pc);
    const double pn = wallish(ckind(Ra.KK[lc])) ? pc : 0.5 * (pc + Ra.P[lc]);
    const double ps = wallish(ckind(Rm.KK[lc])) ? pc : 0.5 * (Rm.P[lc] + pc);
    dpx = (pe - pw) * m.inv_dx;
    dpy = (pn - ps) * m.inv_dy;
}

// ================= stage C: T_{i,j}, u-hat_{i,j}, v-hat_{i,j+1} =================
template <bool IMPL, bool TVD, bool REG, bool NU = false, bool L3 = false>
__device__ __forceinline__ void stage_C(MarchSmem& s, const MarchParams& m, int lc, const RingRow& Rm,
                                        const RingRow& R0, const RingRow& Ra, const RingRow& Rb,
                                        const FluxRow& Fc, const FluxRow& Fn, const NM1& nm, const Carry& c,
                                        StepVars& v, const Geo& g, const Tp3& q3 = Tp3{})
{
    static_assert(!(NU && L3), "loop 3 runs on uniform meshes");
    const Params& k = m.k;
    const double dt = k.dt;
    const double dx = NU ? g.dxr[lc] : k.dx, dy = NU ? g.y0 : k.dy;
    const double dxw = NU ? g.dxr[lc - 1] : k.dx;                 // Delta x_{i-1}
    const double dV = NU ? dx * dy : m.dV;
    const uint32_t kw0 = R0.KK[lc], kw1 = Ra.KK[lc];
    const double rP = R0.R[lc], gP = R0.G[lc];
    // ---- energy (Eqs. pl30-pl33, pl28-pl29 / pl31_1)
    v.TN = 0.0;
    if (cF<REG>(kw0)) {
        double a1, a2, a3, a4, T1, T2, T3, T4, FW, FE, FSl, FNl;
        // neighbour temperatures: the old iterate, or (loop 3) the previous sweep's
        auto TW = [&] { return L3 ? q3.Tt(-1) : R0.T[lc - 1]; };
        auto TE = [&] { return L3 ? q3.Tt(1) : R0.T[lc + 1]; };
        auto TS = [&] { return L3 ? q3.Tt(-q3.pitch) : Rm.T[lc]; };
        auto TN = [&] { return L3 ? q3.Tt(q3.pitch) : Ra.T[lc]; };
        if (REG) {
            a1 = s.XTW[lc]; FW = Fc.FX[lc]; T1 = TW();
            FE = Fc.FX[lc + 1]; a2 = IMPL ? s.XTW[lc + 1] - FE : s.XTW[lc + 1]; T2 = TE();
            a3 = c.ytS; FSl = c.FS; T3 = TS();
            a4 = v.ytN; FNl = v.Fy1; T4 = TN();
        } else {
            FW = FE = FSl = FNl = 0.0;
            const double tau = 2.1904 * k.Kn * rcp(rP);   // Eq. pl39
            uint8_t kn = ckind(R0.KK[lc - 1]);
            if (wallish(kn)) { a1 = k.CT1 * gP * dy * rcp(0.5 * dx + tau); T1 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a1 = s.XTW[lc]; FW = Fc.FX[lc]; T1 = TW(); }
            kn = ckind(R0.KK[lc + 1]);
            if (wallish(kn)) { a2 = k.CT1 * gP * dy * rcp(0.5 * dx + tau); T2 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { FE = Fc.FX[lc + 1]; a2 = IMPL ? s.XTW[lc + 1] - FE : s.XTW[lc + 1]; T2 = TE(); }
            kn = ckind(Rm.KK[lc]);
            if (wallish(kn)) { a3 = k.CT1 * gP * dx * rcp(0.5 * dy + tau); T3 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a3 = c.ytS; FSl = c.FS; T3 = TS(); }
            kn = ckind(kw1);
            if (wallish(kn)) { a4 = k.CT1 * gP * dx * rcp(0.5 * dy + tau); T4 = kn == CK_WALLY ? k.T_wall : k.T_sq; }
            else { a4 = v.ytN; FNl = v.Fy1; T4 = TN(); }
        }
        // unsteady density: old iterate, or (loop 3) p / T of the previous sweep
        const double rq = L3 ? fdiv(q3.P(0), q3.Tt(0)) : rP;
        const double a0 = IMPL ? FMA(dt, a1 + a2 + a3 + a4 + FE - FW + FNl - FSl, MUL(rq, dV))
                               : FMA(dt, a1 + a2 + a3 + a4, MUL(rq, dV));
        // S^T_c, Eq. pl29 (R4 bilinear = 4-point mean on a uniform mesh); a mid-face
        // velocity on a wall face is the slip velocity of Eq. pl38 (R38)
        const double rdx = NU ? rcp(dx) : m.inv_dx, rdy = NU ? rcp(dy) : m.inv_dy;
        const double dudx = MUL(R0.U[lc + 1] - R0.U[lc], rdx);
        const double dvdy = MUL(Ra.V[lc] - R0.V[lc], rdy);
        double shear;
        if (REG) {
            // dv/dx + du/dy from the bilinear face values (R4): v_E - v_W and u_N - u_S
            // as one difference each (the shared corner values cancel)
            shear = FMA((R0.V[lc + 1] + Ra.V[lc + 1]) - (R0.V[lc - 1] + Ra.V[lc - 1]), m.q_dx,
                        MUL((Ra.U[lc] + Ra.U[lc + 1]) - (Rm.U[lc] + Rm.U[lc + 1]), m.q_dy));
        } else {
            shear = shear_general<NU>(R0, Ra, Rm, lc, rP, m, g);
        }
        const double div = dudx + dvdy;
        // pressure work (R9): C^T3 Dp/Dt of Eq. pl6 at the old iterate --
        // (p - p^{n-1}) / dt + ubar dp/dx + vbar dp/dy with face pressures p_f =
        // linear interpolation of the two cells, = p of the cell at a wall -- or
        // kappa p div(u); branch-free: pw_a = C^T3 or 0, pwk = 0 or kappa.
        // p^{n-1} = rho^{n-1} T^{n-1} (the (p/T)^{n-1} row times T^{n-1}, within
        // 2 ulp of the stored p^{n-1})
        const double pc = L3 ? q3.P(0) : R0.P[lc];
        const double p1 = MUL(s.R1[lc], nm.T1c);
        double dpx, dpy;
        if (REG) {
            dpx = MUL(L3 ? q3.P(1) - q3.P(-1) : R0.P[lc + 1] - R0.P[lc - 1], m.h_dx);
            dpy = MUL(L3 ? q3.P(q3.pitch) - q3.P(-q3.pitch) : Ra.P[lc] - Rm.P[lc], m.h_dy);
        } else {
            dp_general<NU, L3>(R0, Ra, Rm, lc, m, g, dpx, dpy, q3);
        }
        const double ub = MUL(0.5, R0.U[lc] + R0.U[lc + 1]), vb = MUL(0.5, R0.V[lc] + Ra.V[lc]);
        const double pwork = FMA(m.pw_a, FMA(vb, dpy, FMA(ub, dpx, MUL(pc - p1, m.inv_dt))), MUL(MUL(k.pwk, pc), div));
        const double Phi = FMA(MUL(-2.0 / 3.0, div), div, FMA(shear, shear, MUL(2.0, FMA(dvdy, dvdy, MUL(dudx, dudx)))));
        const double Sc = MUL(FMA(MUL(k.CT2, gP), Phi, pwork), dV);
        const double sT = FMA(a4, T4, FMA(a3, T3, FMA(a2, T2, MUL(a1, T1))));
        const double rhs = FMA(dt, sT + (IMPL ? Sc : Sc + nm.Tec), MUL(p1, dV));
        v.TN = MUL(rhs, rcp(a0));
    }
    // ---- u pseudo-velocity at u-face (i, j)
    {
        // N tangential link pieces at y^f_{j+1} (both sides; the S side is carried)
        const double F1 = v.Fy1, F2 = Fn.FY[lc - 1];
        // NU: D^uy = B Gamma|_{corner} (Delta x_{i-1} + Delta x_i) / (Delta y_j + Delta y_{j+1})
        v.FsSumN = F1 + F2;
        const double lk = IMPL ? MUL(0.5, STS_LINK(F1, v.upsi1) + STS_LINK(F2, v.upsi2)) : 0.0;
        v.utSn = NU ? lk + k.B * v.gcN * (dxw + dx) * rcp(dy + g.ya) : FMA(m.B_dxdy, v.gcN, lk);
        const double a4p = IMPL ? FMA(-0.5, v.FsSumN, v.utSn) : v.utSn;
        double uhat = 0.0, du = 0.0;
        if (uA<REG>(kw0)) {
            const double rL = R0.R[lc - 1], rR = rP, gL = R0.G[lc - 1], gR = gP;
            const double a1 = s.XUW[lc - 1], a2 = v.xe;
            // F-bar^x of cell i-1, recomputed with the same operations as its owner
            const double FbW = MUL(MUL(rL, MUL(0.5, R0.U[lc - 1] + R0.U[lc])), dy), FbE = v.Fb;
            double a3, a4, uS, uN, FsS, FnS;
            if (REG) {
                a3 = c.utS; FsS = c.FsSum; uS = Rm.U[lc];
                a4 = a4p; FnS = v.FsSumN; uN = Ra.U[lc];
            } else {
                FsS = FnS = 0.0;
                const double gadj = 0.5 * (gL + gR);
                const double zeta = 1.1466 * k.Kn * rcp(0.5 * (rL + rR));     // Eq. pl38
                const double L = NU ? 0.5 * (dxw + dx) : dx;                    // u-CV width
                const uint8_t kl = ckind(Rm.KK[lc - 1]), kr = ckind(Rm.KK[lc]);
                if (kl == CK_WALLY || (kl == CK_SOLID && kr == CK_SOLID)) {
                    a3 = k.B * gadj * L * rcp(0.5 * dy + zeta); uS = kl == CK_WALLY ? k.u_wb : 0.0;
                } else { a3 = c.utS; FsS = c.FsSum; uS = Rm.U[lc]; }
                const uint8_t ml = ckind(Ra.KK[lc - 1]), mr = ckind(kw1);
                if (ml == CK_WALLY || (ml == CK_SOLID && mr == CK_SOLID)) {
                    a4 = k.B * gadj * L * rcp(0.5 * dy + zeta); uN = ml == CK_WALLY ? k.u_wt : 0.0;
                } else { a4 = a4p; FnS = v.FsSumN; uN = Ra.U[lc]; }
            }
            // unsteady term (rho_i Delta x_i + rho_{i-1} Delta x_{i-1}) Delta y_j / (2 dt) (transposed pl15)
            const double tterm = NU ? (rR * dx + rL * dxw) * dy * (0.5 * m.inv_dt) : MUL(rR + rL, m.c_t);
            const double a0 = IMPL ? FMA(0.5, FnS - FsS, a1 + a2 + a3 + a4 + FbE - FbW) + tterm
                                   : a1 + a2 + a3 + a4 + tterm;
            const double bt = NU ? (s.R1[lc] * dx + s.R1[lc - 1] * dxw) * dy * (0.5 * m.inv_dt)
                                 : MUL(s.R1[lc] + s.R1[lc - 1], m.c_t);
            const double bg = NU ? k.g_x * 0.5 * (rR * dx + rL * dxw) * dy : MUL(MUL(k.g_x, rR + rL), m.half_dV);
            const double bv = FMA(MUL(2.0 / 3.0, gL), Ra.V[lc - 1] - R0.V[lc - 1],
                              FMA(MUL(-2.0 / 3.0, gR), Ra.V[lc] - R0.V[lc],
                              FMA(-c.gcP, R0.V[lc] - R0.V[lc - 1], MUL(v.gcN, Ra.V[lc] - Ra.V[lc - 1]))));
            const double b = FMA(k.B, bv, MUL(bt, nm.u1c)) + bg;
            const double r = rcp(a0);
            const double su = FMA(a4, uN, FMA(a3, uS, FMA(a2, R0.U[lc + 1], MUL(a1, R0.U[lc - 1]))));
            uhat = MUL(su + (IMPL ? b : b + nm.uec), r);
            du = MUL(NU ? k.A * dy : m.A_dy, r);
        }
        v.uhat = uhat;
        v.du = du;
        s.UH[lc] = uhat;
        s.DU[lc] = du;
    }
    // ---- v pseudo-velocity at v-face (i, j+1)
    v.vhatN = 0.0;
    v.dvN = 0.0;
    if (vA<REG>(kw1)) {
        const double rB = rP, rT = Ra.R[lc], gB = gP, gT = Ra.G[lc];
        const double dyT = NU ? g.ya : k.dy;                           // Delta y_{j+1}
        double a1, a2, vW, vE, FwS, FeS;
        if (REG) {
            a1 = v.xvW; FwS = v.FwSum; vW = Ra.V[lc - 1];
            FeS = Fn.FX[lc + 1] + Fc.FX[lc + 1]; a2 = IMPL ? FMA(-0.5, FeS, s.XVW[lc + 1]) : s.XVW[lc + 1]; vE = Ra.V[lc + 1];
        } else {
            FwS = FeS = 0.0;
            const double gadj = 0.5 * (gB + gT);
            const double zeta = 1.1466 * k.Kn * rcp(0.5 * (rB + rT));
            const double L = NU ? 0.5 * (dy + dyT) : dy;                   // v-CV height
            if (ckind(R0.KK[lc - 1]) == CK_SOLID && ckind(Ra.KK[lc - 1]) == CK_SOLID) {
                a1 = k.B * gadj * L * rcp(0.5 * dx + zeta); vW = 0.0;
            } else { a1 = v.xvW; FwS = v.FwSum; vW = Ra.V[lc - 1]; }
            if (ckind(R0.KK[lc + 1]) == CK_SOLID && ckind(Ra.KK[lc + 1]) == CK_SOLID) {
                a2 = k.B * gadj * L * rcp(0.5 * dx + zeta); vE = 0.0;
            } else { FeS = Fn.FX[lc + 1] + Fc.FX[lc + 1]; a2 = IMPL ? FMA(-0.5, FeS, s.XVW[lc + 1]) : s.XVW[lc + 1]; vE = Ra.V[lc + 1]; }
        }
        // corner Gamma (i+1, j+1), recomputed with the same operations as its owner
        double gcE;
        if (REG) {
            gcE = MUL(0.25, R0.G[lc] + R0.G[lc + 1] + Ra.G[lc] + Ra.G[lc + 1]);
        } else if (NU) {
            const double wxl = wleft(dx, g.dxr[lc + 1]), wxr = 1.0 - wxl;
            const double wyb = wleft(dy, dyT), wyt = 1.0 - wyb;
            double sum = 0.0, ws = 0.0;
            if (!wallish(ckind(R0.KK[lc]))) { sum += wxl * wyb * R0.G[lc]; ws += wxl * wyb; }
            if (!wallish(ckind(R0.KK[lc + 1]))) { sum += wxr * wyb * R0.G[lc + 1]; ws += wxr * wyb; }
            if (!wallish(ckind(Ra.KK[lc]))) { sum += wxl * wyt * Ra.G[lc]; ws += wxl * wyt; }
            if (!wallish(ckind(Ra.KK[lc + 1]))) { sum += wxr * wyt * Ra.G[lc + 1]; ws += wxr * wyt; }
            gcE = ws > 0.0 ? sum / ws : 0.0;
        } else {
            double sum = 0.0;
            int n = 0;
            if (!wallish(ckind(R0.KK[lc]))) { sum += R0.G[lc]; n++; }
            if (!wallish(ckind(R0.KK[lc + 1]))) { sum += R0.G[lc + 1]; n++; }
            if (!wallish(ckind(Ra.KK[lc]))) { sum += Ra.G[lc]; n++; }
            if (!wallish(ckind(Ra.KK[lc + 1]))) { sum += Ra.G[lc + 1]; n++; }
            gcE = n == 4 ? MUL(0.25, sum) : (n > 0 ? sum / n : 0.0);
        }
        const double a3 = c.vcS, a4 = v.vcN;
        // unsteady term (rho_{j+1} Delta y_{j+1} + rho_j Delta y_j) Delta x_i / (2 dt) (Eq. pl15)
        const double tterm = NU ? (rT * dyT + rB * dy) * dx * (0.5 * m.inv_dt) : MUL(rT + rB, m.c_t);
        const double a0 = IMPL ? FMA(0.5, FeS - FwS, a1 + a2 + a3 + a4) + v.FbN - c.FbS + tterm
                               : a1 + a2 + a3 + a4 + tterm;
        const double bt = NU ? (v.r1n * dyT + s.R1[lc] * dy) * dx * (0.5 * m.inv_dt) : MUL(v.r1n + s.R1[lc], m.c_t);
        const double bg = NU ? k.g_y * 0.5 * (rT * dyT + rB * dy) * dx : MUL(MUL(k.g_y, rT + rB), m.half_dV);
        const double bv = FMA(MUL(2.0 / 3.0, gB), R0.U[lc + 1] - R0.U[lc],
                          FMA(MUL(-2.0 / 3.0, gT), Ra.U[lc + 1] - Ra.U[lc],
                          FMA(-v.gcN, Ra.U[lc] - R0.U[lc], MUL(gcE, Ra.U[lc + 1] - R0.U[lc + 1]))));
        const double b = FMA(k.B, bv, MUL(bt, nm.v1n)) + bg;
        const double r = rcp(a0);
        const double sv = FMA(a4, Rb.V[lc], FMA(a3, R0.V[lc], FMA(a2, vE, MUL(a1, vW))));
        v.vhatN = MUL(sv + (IMPL ? b : b + nm.ven), r);
        v.dvN = MUL(NU ? k.A * dx : m.A_dx, r);
    }
}

// ================= stage D: p_{i,j} (Eqs. pl23-pl24) =================
template <bool IMPL, bool TVD, bool REG, bool NU = false, bool L3 = false>
__device__ __forceinline__ void stage_D(MarchSmem& s, const MarchParams& m, int lc, const RingRow& Rm,
                                        const RingRow& R0, const RingRow& Ra, const FluxRow& Fc,
                                        const FluxRow& Fn, const Carry& c, StepVars& v, const Geo& g,
                                        const Tp3& q3 = Tp3{})
{
    const Params& k = m.k;
    const double dt = k.dt, dx = NU ? g.dxr[lc] : k.dx, dy = NU ? g.y0 : k.dy;
    const double dV = NU ? dx * dy : m.dV;
    const uint32_t kw0 = R0.KK[lc];
    double pn = R0.P[lc];
    if (cF<REG>(kw0)) {
        double apW = 0.0, apE = 0.0, apS = 0.0, apN = 0.0, bpW = 0.0, bpE = 0.0, bpS = 0.0, bpN = 0.0, sum = 0.0;
        // neighbour pressures: the old iterate, or (loop 3) the previous sweep's
        auto PW = [&] { return L3 ? q3.P(-1) : R0.P[lc - 1]; };
        auto PE = [&] { return L3 ? q3.P(1) : R0.P[lc + 1]; };
        auto PS = [&] { return L3 ? q3.P(-q3.pitch) : Rm.P[lc]; };
        auto PN = [&] { return L3 ? q3.P(q3.pitch) : Ra.P[lc]; };
        if (REG) {
            const double rw = Fc.RU[lc], re = Fc.RU[lc + 1], rs = c.rvS, rn = v.rv1;
            apW = MUL(MUL(rw, v.du), dy); bpW = MUL(MUL(rw, v.uhat), dy);
            apE = MUL(MUL(re, s.DU[lc + 1]), dy); bpE = MUL(MUL(re, s.UH[lc + 1]), dy);
            apS = MUL(MUL(rs, c.dvP), dx); bpS = MUL(MUL(rs, c.vhatP), dx);
            apN = MUL(MUL(rn, v.dvN), dx); bpN = MUL(MUL(rn, v.vhatN), dx);
            sum = FMA(apN, PN(), FMA(apS, PS(), FMA(apE, PE(), MUL(apW, PW()))));
        } else {
            const uint8_t kwf = ukind(kw0), kef = ukind(R0.KK[lc + 1]);
            if (kwf == FK_ACTIVE) {
                const double r = Fc.RU[lc];
                apW = MUL(MUL(r, v.du), dy); bpW = MUL(MUL(r, v.uhat), dy); sum = FMA(apW, PW(), sum);
            } else if (kwf == FK_INLET) bpW = MUL(MUL(Fc.RU[lc], k.u_in), dy);
            if (kef == FK_ACTIVE) {
                const double r = Fc.RU[lc + 1];
                apE = MUL(MUL(r, s.DU[lc + 1]), dy); bpE = MUL(MUL(r, s.UH[lc + 1]), dy); sum = FMA(apE, PE(), sum);
            } else if (kef == FK_OUTLET) bpE = MUL(MUL(Fc.RU[lc + 1], R0.U[lc]), dy);
            if (vkind(kw0) == FK_ACTIVE) {
                const double r = c.rvS;
                apS = MUL(MUL(r, c.dvP), dx); bpS = MUL(MUL(r, c.vhatP), dx); sum = FMA(apS, PS(), sum);
            }
            if (vkind(Ra.KK[lc]) == FK_ACTIVE) {
                const double r = v.rv1;
                apN = MUL(MUL(r, v.dvN), dx); bpN = MUL(MUL(r, v.vhatN), dx); sum = FMA(apN, PN(), sum);
            }
            // four active faces: the regular instance's expression (same bits)
            if (!NU && kwf == FK_ACTIVE && kef == FK_ACTIVE && vkind(kw0) == FK_ACTIVE && vkind(Ra.KK[lc]) == FK_ACTIVE)
                sum = FMA(apN, PN(), FMA(apS, PS(), FMA(apE, PE(), MUL(apW, PW()))));
        }
        // a^p_0 = dV / T_new + dt sum a^p (Eq. pl24, R28); multiplied through by T_new
        // so one reciprocal serves: p = T_new (dt sum + b^p) / (dV + T_new dt sum a^p)
        const double bp = FMA(-(bpE - bpW + bpN - bpS), dt, MUL(s.R1[lc], dV));
        pn = MUL(MUL(v.TN, FMA(sum, dt, bp)), rcp(FMA(MUL(v.TN, dt), apW + apE + apS + apN, dV)));
    }
    v.pn = pn;
    s.PN[lc] = pn;
}

// ================= explicit planes inside the first pass of a step (N2) =================
// In pass 1 of a time step the old iterate IS the n-1 state, so the ring
// rows are exactly what conv_march_kernel reads and stage A's F^x, F^y of row j+1
// are its fluxes.  The planes' face-value fluxes are computed here with the conv
// kernel's operations (sts_conv_loop.inc, same order: same bits) and the planes
// are formed in stage C, used by this pass, and stored for passes 2..N.
// Shared rows (behind MarchSmem): TX (u-face i, row j), UX (cell i, row j), VX
// (u-face column i, v-row j+1).  Carried: TY, uY, vY of the previous row step.
struct ConvRows { double* TX; double* UX; double* VX; };
template <bool TVD, bool REG>
__device__ __forceinline__ void conv_A(const ConvRows& cr, int lc, const RingRow& Rm, const RingRow& R0,
                                       const RingRow& Ra, const RingRow& Rb, const RingRow& Rc,
                                       const FluxRow& Fc, const StepVars& v, double dx, double dy,
                                       double& TYn, double& vYn)
{
    const uint32_t kw0 = R0.KK[lc], kw1 = Ra.KK[lc];
    const double Fx1 = v.Fx1, Fy1 = v.Fy1;
    // TX at u-face (i, j): T flux through x^f_i (pl31_1)
    {
        double tx = 0.0;
        if ((REG || flux_face(ukind(kw0)))) {
            const double F = Fc.FX[lc], w = R0.U[lc], Tm = R0.T[lc - 1], Ti = R0.T[lc];
            const double ps = (TVD && (REG || ckind(R0.KK[lc - 2]) == CK_FLUID) && (REG || ckind(R0.KK[lc - 1]) == CK_FLUID) &&
                               (REG || ckind(kw0) == CK_FLUID) && (REG || ckind(R0.KK[lc + 1]) == CK_FLUID))
                            ? psi_f(R0.T[lc - 2], Tm, Ti, R0.T[lc + 1], w) : 0.0;
            tx = F * ((w > 0.0 ? Tm : Ti) + (Ti - Tm) * ps);
        }
        cr.TX[lc] = tx;
    }
    // TY at v-face (i, j+1)
    TYn = 0.0;
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
            const double ui = R0.U[lc], up = R0.U[lc + 1], ub = 0.5 * (ui + up);
            ux = dy * R0.R[lc] * ub * (ub > 0.0 ? ui : up);
        }
        cr.UX[lc] = ux;
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
                const double F = Fc.FX[lc], w = R0.U[lc];
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
        cr.VX[lc] = vx;
    }
    // vY at cell (i, j+1): v flux through the cell centre (pl15_11 y-terms)
    vYn = 0.0;
    if ((REG || ckind(kw1) == CK_FLUID)) {
        const double vi = Ra.V[lc], vp = Rb.V[lc], vb = 0.5 * (vi + vp);
        const bool ok = TVD && (REG || vkind(kw1) == FK_ACTIVE) && (REG || vkind(Rb.KK[lc]) == FK_ACTIVE) &&
                        (REG || vkind(kw0) == FK_ACTIVE) && (REG || vkind(Rc.KK[lc]) == FK_ACTIVE);
        const double ps = ok ? psi_f(R0.V[lc], vi, vp, Rc.V[lc], vb) : 0.0;
        vYn = dx * Ra.R[lc] * vb * ((vb > 0.0 ? vi : vp) + (vp - vi) * ps);
    }
}
// uY at (u column i, y^f_{j+1}) (needs the neighbour's F^y: after B1), then the
// planes of this point: T^exp(i, j), u^exp(i, j), v^exp(i, j+1).
template <bool TVD, bool REG>
__device__ __forceinline__ void conv_C(const ConvRows& cr, int lc, const RingRow& Rm, const RingRow& R0,
                                       const RingRow& Ra, const RingRow& Rb, const FluxRow& Fn,
                                       double TYc, double TYn, double uYc, double vYc, double vYn,
                                       double& uYn, double& te, double& ue, double& ve)
{
    const uint32_t kw0 = R0.KK[lc], kw1 = Ra.KK[lc];
    {
        const double ui = R0.U[lc], up = Ra.U[lc];
        const bool ok = TVD && (REG || ukind(Rm.KK[lc]) == FK_ACTIVE) && (REG || ukind(kw0) == FK_ACTIVE) &&
                        (REG || ukind(kw1) == FK_ACTIVE) && (REG || ukind(Rb.KK[lc]) == FK_ACTIVE);
        double sum = 0.0;
        for (int h = 0; h < 2; h++) {
            const int cc = lc - 1 + h;
            if ((!REG && vkind(Ra.KK[cc]) != FK_ACTIVE)) continue;
            const double F = Fn.FY[cc], w = Ra.V[cc];
            const double ps = ok ? psi_f(Rm.U[lc], ui, up, Rb.U[lc], w) : 0.0;
            sum += F * ((w > 0.0 ? ui : up) + (up - ui) * ps);
        }
        uYn = 0.5 * sum;
    }
    // (a regular point is a fluid cell with active faces; the all-regular kernel
    // reads no kind words, so REG must not test them)
    te = (REG || ckind(kw0) == CK_FLUID) ? (cr.TX[lc] - cr.TX[lc + 1] + TYc - TYn) : 0.0;
    ue = (REG || ukind(kw0) == FK_ACTIVE) ? (cr.UX[lc - 1] - cr.UX[lc] + uYc - uYn) : 0.0;
    ve = (REG || vkind(kw1) == FK_ACTIVE) ? (cr.VX[lc] - cr.VX[lc + 1] + vYc - vYn) : 0.0;
}

struct Resid { double du, dv, dp, dT, vel, p, T; long long bad; int badf; bool nanv; };
// Sticky bad-state key: bits 63..44 = 0xFFFFF - pass index (earliest pass wins
// the max), 43..2 = 2^42 - 1 - flat cell index j nx + i (lowest cell wins),
// 1..0 = field (sts_field: 0 u, 1 v, 2 p, 3 T).  BAD_NOCELL: a NaN velocity.
constexpr long long BAD_NOCELL = (1LL << 42) - 2;
__host__ __device__ __forceinline__ unsigned long long bad_key(int pass_key, long long flat, int field)
{
    return ((unsigned long long)pass_key << 44) | ((((1ULL << 42) - 1) - (unsigned long long)flat) << 2) |
           (unsigned long long)(field & 3);
}

// ================= stage E: corrections, writes, residuals =================
template <bool IMPL, bool TVD, bool REG, bool HALO = false>
__device__ __forceinline__ void stage_E(MarchSmem& s, const MarchParams& m, int lc, int gi, int j,
                                        const RingRow& R0, const Carry& c, const StepVars& v, Resid& rs)
{
    const Params& k = m.k;
    const int id = j * k.pitch + (gi - k.gi0 + OFF);
    const uint32_t kw0 = R0.KK[lc];
    const bool fluid = cF<REG>(kw0);
    if (fluid) {
        k.T_w[id] = v.TN;
        k.p_w[id] = v.pn;
        rs.dT = dmax(rs.dT, fabs(v.TN - R0.T[lc]));
        rs.dp = dmax(rs.dp, fabs(v.pn - R0.P[lc]));
        rs.T = dmax(rs.T, fabs(v.TN));
        rs.p = dmax(rs.p, fabs(v.pn));
        if (!(v.TN > 0.0) || !(v.pn > 0.0) || !isfinite(v.TN) || !isfinite(v.pn)) {
            const long long flat = (long long)j * k.nx + gi;
            if (rs.bad < 0 || flat < rs.bad) { rs.bad = flat; rs.badf = (!(v.TN > 0.0) || !isfinite(v.TN)) ? 3 : 2; }
        }
    }
    double un = 0.0;
    if (uA<REG>(kw0)) {
        un = FMA(-v.du, v.pn - s.PN[lc - 1], v.uhat);
        rs.du = dmax(rs.du, fabs(un - R0.U[lc]));
        rs.vel = dmax(rs.vel, fabs(un));
        rs.nanv |= un != un;
    } else if (ukind(kw0) == FK_INLET) un = k.u_in;
    k.u_w[id] = un;
    double vn = 0.0;
    if (vA<REG>(kw0)) {
        vn = FMA(-c.dvP, v.pn - c.pnP, c.vhatP);
        rs.dv = dmax(rs.dv, fabs(vn - R0.V[lc]));
        rs.vel = dmax(rs.vel, fabs(vn));
        rs.nanv |= vn != vn;
    }
    k.v_w[id] = vn;
    if (HALO) halo_store(m, j, gi - k.gi0 + OFF, fluid, un, vn, v.pn, v.TN);   // fused halo (N1)
    if (!REG && k.xbc == 0 && gi == k.nx - 1) {
        k.u_w[id + 1] = R0.U[lc];                    // outlet face: u_old(nx-1), BC spec 3
        const double pv = fluid ? v.pn : R0.P[lc];
        const double Tv = fluid ? v.TN : R0.T[lc];
        for (int g = 1; g <= OFF - 1; g++) { k.p_w[id + g] = pv; k.T_w[id + g] = Tv; k.v_w[id + g] = vn; }
    }
    if (k.mirror) {                                  // single-rank periodic: wrapped ghosts
        int tgt = -1000;
        if (gi < OFF) tgt = gi + k.nx;
        else if (gi >= k.nx - OFF) tgt = gi - k.nx;
        if (tgt > -1000) {
            const int tt = j * k.pitch + (tgt - k.gi0 + OFF);
            if (fluid) { k.p_w[tt] = v.pn; k.T_w[tt] = v.TN; }
            k.u_w[tt] = un;
            k.v_w[tt] = vn;
        }
    }
}

// REGK = true: the kernel of the all-regular CTAs (every point of the CTA's rows
// and columns, warm-up rows included, is regular -- host-classified): the row
// loop is compiled with the regular stage instances only, reads no kinds and
// has a register allocation of its own.  REGK = false: every other CTA, with
// the per-point choice between the instances.  A regular point runs the same
// instance code in both kernels, so the split never changes a bit.
// NU = true: the non-uniform-mesh kernel: every point runs the
// general instances in their general-mesh form; the column widths of the ring
// columns sit behind MarchSmem in shared memory, the row heights come from m.dyp.
// HALO = true: the edge-strip kernel of a peer-connected rank (fused halo
// stores in stage E, N1); every other launch compiles them out.
// FUSEC = true: the first pass of an explicit step with the planes computed in
// the pass (N2; single rank, uniform mesh), 3 more shared rows behind MarchSmem.
#ifndef STS_GEN_CTAS
#define STS_GEN_CTAS STS_MARCH_CTAS
#endif
template <bool IMPL, bool TVD, bool GRAPH = false, bool REGK = false, bool NU = false, bool L3 = false,
          bool HALO = false, bool FUSEC = false>
__device__ __forceinline__ void march_body(const MarchParams m)
{
    static_assert(!(FUSEC && (IMPL || NU || L3 || HALO)), "plane fusion: explicit, uniform, single-rank passes");
    static_assert(!(HALO && (REGK || GRAPH || L3)), "fused halo stores: edge strips of the stream path only");
    static_assert(!(NU && REGK), "non-uniform meshes run the general kernel only");
    static_assert(!(NU && L3), "loop 3 runs on uniform meshes");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MarchSmem& s = *reinterpret_cast<MarchSmem*>(smem_raw);
    double* const s_dx = reinterpret_cast<double*>(smem_raw + sizeof(MarchSmem));   // NU only: RW widths
    const ConvRows cr{s_dx, s_dx + RW, s_dx + 2 * RW};                               // FUSEC only
    const Params& k = m.k;
    // Early exit: loop 2 converged earlier in this graph launch, or a bad state
    // earlier in this advance call.  The bad key is written by other CTAs of this
    // very launch (atomicMax at their end), so a per-thread read could differ
    // inside one CTA and split it at the barriers below; thread 0 reads both
    // flags and the CTA takes one decision (__syncthreads_or).
    int stop = 0;
    if (threadIdx.x == 0)
        stop = (GRAPH && *(volatile const int*)m.done) || *(volatile const unsigned long long*)m.bad != 0ull;
    if (__syncthreads_or(stop)) return;
    const int t = threadIdx.x;
    const int4 ce = m.order[blockIdx.x];
    const int strip = ce.x;
    const int I0 = k.gi0 + strip * MW;                  // first owned column of the strip
    // ring column 0 = stored column c0 (a multiple of 4: 16-byte aligned TMA rows); this
    // thread's column sits at ring column lc
    const int wbase = I0 - 4 - k.gi0 + OFF;
    const int shift = wbase & 3;                        // c0 % 4 == 0: double and 4-byte kind rows aligned
    const int c0 = wbase - shift;
    const bool tma = c0 + RW <= k.pitch;
    const int lc = t + 2 + shift;
    if (t == 0) {
        for (int q = 0; q < RS; q++) mbar_init(&s.mbar[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (NU)
        for (int q = t; q < RW; q += MX) s_dx[q] = __ldg(m.dxl + min(max(c0 + q, 0), k.pitch - 1));
    __syncthreads();
    const int gi = I0 - 2 + t;                          // this thread's global column
    const int J0 = ce.y, J1 = ce.z;
    const int js = J0 - WARM;
    const bool col_stored = stored_col(k, gi);
    const bool owner = t >= 2 && t < 2 + MW && gi < k.gi0 + k.nloc;

    // ---- prologue: ring rows js-1 .. js+3 land (there is no row-start barrier: from
    // here on, row j+4 is issued at the start of step j and lands before its B3);
    // ring slots of rows j-1 .. j+4, rotated by one per row step
    RingRow *pm = &s.ring[0], *p0 = &s.ring[1], *pa = &s.ring[2], *pb = &s.ring[3], *pc = &s.ring[4], *pd = &s.ring[5];
    constexpr bool kinds = !REGK;                        // the all-regular loop reads no kinds
    for (int q = 0; q < 5; q++) ring_issue_tma(s, q, m, c0, tma, js - 1 + q, kinds);   // row js-1+q -> slot q
    cp_wait_all();
    __syncthreads();
    for (int q = 0; q < 4; q++) mbar_wait(&s.mbar[q], 0);
    ring_derive(*pm);
    ring_derive(*p0);
    ring_derive(*pa);
    ring_derive(*pb);
    __syncthreads();        // rho, Gamma of rows js-1 .. js+2 before step js reads neighbours' elements

    // ---- n-1 / explicit-plane values of this thread's column.  Prefetched one
    // row step ahead through registers (PREF_L), except in implicit TVD (no
    // registers to spare at 4 CTAs/SM: 16 B of spills and +14 %), which loads them
    // at the start of the row step that uses them
    const int col = gi - k.gi0 + OFF;                   // stored local column of this thread
    auto ld = [&](const double* a, int j) -> double {
        return (col_stored && j >= 0 && j < k.ny) ? __ldg(a + (j * k.pitch + col)) : 0.0;
    };
    auto ldv = [&](const double* a, int j) -> double {
        return (col_stored && j >= 0 && j <= k.ny) ? __ldg(a + (j * k.pitch + col)) : 0.0;
    };
    NM1 nm;
    nm.Tec = nm.uec = nm.ven = 0.0;
    auto nm_prefetch_init = [&]() {
        nm.p1n = ld(k.p_1, js + 1); nm.T1n = ld(k.T_1, js + 1);
        nm.T1c = ld(k.T_1, js); nm.u1c = ld(k.u_1, js); nm.v1n = ldv(k.v_1, js + 1);
        if (!IMPL && !FUSEC) { nm.Tec = ld(k.Te, js); nm.uec = ld(k.ue, js); nm.ven = ldv(k.ve, js + 1); }
    };

    Carry c{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 1.0, 0.0};
    double cTY = 0.0, cuY = 0.0, cvY = 0.0;             // FUSEC: plane fluxes carried from the previous row
    Resid rs{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, -1, 0, false};
    StepVars v;
    int oj = js * k.pitch + col;                        // element offset of (row j, own column), + pitch per step (upwind prefetch)

    // The row loop: the all-regular kernel prefetches the n-1 values of its
    // column one row step ahead through registers; the general kernel of the
    // implicit TVD variant has no registers to spare for it.
    if constexpr (REGK) {
        constexpr bool ALLREG = true;
        constexpr bool PREF_L = true;
        nm_prefetch_init();
#include "sts_march_loop.inc"
    } else {
        constexpr bool ALLREG = false;
        constexpr bool PREF_L = !(IMPL && TVD);
        if (PREF_L) nm_prefetch_init();
#include "sts_march_loop.inc"
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
    // first bad state of the advance call, sticky: one u64 key per context,
    // (earliest pass, then lowest cell, field) ordered so that one atomicMax
    // (and one NCCL MAX allreduce) keeps it; later passes see it and exit
    if (rs.bad >= 0 || rs.nanv) {
        const long long flat = rs.bad >= 0 ? rs.bad : BAD_NOCELL;
        atomicMax(m.bad, bad_key(m.pass_key, flat, rs.bad >= 0 ? rs.badf : 0));
    }
}
template <bool IMPL, bool TVD, bool GRAPH = false, bool REGK = false, bool NU = false, bool L3 = false,
          bool HALO = false, bool FUSEC = false>
__global__ void __launch_bounds__(MX, REGK ? MARCH_CTAS : STS_GEN_CTAS) march_kernel(MarchParams m)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");                 // PDL: see march_fused_kernel
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    march_body<IMPL, TVD, GRAPH, REGK, NU, L3, HALO, FUSEC>(m);
}

}  // namespace sts
#undef STS_LINK
