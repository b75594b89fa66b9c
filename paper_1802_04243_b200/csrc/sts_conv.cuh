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

// NU = true: non-uniform mesh -- general points only, the
// limiters and fluxes in their general-mesh form (Eqs. pl15_1-pl15_2, pl15_11,
// pl31_1); column widths behind ConvSmem, row heights from m.dyp.
template <bool TVD, bool NU = false>
__global__ void __launch_bounds__(MX, 5) conv_march_kernel(MarchParams m)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ConvSmem& s = *reinterpret_cast<ConvSmem*>(smem_raw);
    double* const s_dx = reinterpret_cast<double*>(smem_raw + sizeof(ConvSmem));   // NU only: RW widths
    const Params& k = m.k;
    const int t = threadIdx.x;
    const int4 ce = m.order[blockIdx.x];
    const bool allreg = (ce.w & ALLREG_BIT) != 0;
    const int strip = ce.x;
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
    if (NU)
        for (int q = t; q < RW; q += MX) s_dx[q] = __ldg(m.dxl + min(max(c0 + q, 0), k.pitch - 1));
    __syncthreads();
    const int gi = I0 - 2 + t;
    const int J0 = ce.y, J1 = ce.z;
    const int js = J0 - 2;                              // 2 warm-up rows (carried TY, uY, vY, fluxes)
    const bool owner = t >= 2 && t < 2 + MW && gi < k.gi0 + k.nloc;
    const double dx = NU ? s_dx[lc] : k.dx;
    auto X = [&](int o) { return s_dx[lc + o]; };     // Delta x at ring offset o (NU)
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
    if (allreg && !NU) {
        constexpr bool ALLREG = true;
#include "sts_conv_loop.inc"
    } else {
        constexpr bool ALLREG = false;
#include "sts_conv_loop.inc"
    }
    mbar_wait(&s.mbar[slot(J1 + 3)], ((J1 + 4 - js) / RS) & 1);   // the last TMA row lands before exit
    cp_wait_all();
}

}  // namespace sts
