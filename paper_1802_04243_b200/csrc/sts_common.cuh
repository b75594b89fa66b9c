// sts_common.cuh -- definitions shared by the sm_100a kernels of the SIMPLE-TS
// loop-2 sweep (arXiv:1802.04243): kind codes, the parameter block, small
// exact helpers.  Written from the paper and DESIGN.md section 3; shares no
// code with oracle/.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sts {

// ------------------------------------------------------------ kinds (DESIGN 3.5)
enum : uint8_t { CK_FLUID = 0, CK_SOLID = 1, CK_INLET = 2, CK_OUTLET = 3, CK_WALLY = 4 };
enum : uint8_t { FK_ACTIVE = 0, FK_FIXED0 = 1, FK_INLET = 2, FK_OUTLET = 3, FK_WALL = 4, FK_NONE = 5 };
// pressure-work forms of S^T_c (reading R9; include/simplets.h sts_gas.pw_form)
enum : int { PW_DPDT = 0, PW_PRINTED = 1, PW_NEG = 2, PW_GAMMA = 3 };

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
    int pw_form;                // PW_* (reading R9)
    // constants
    double dx, dy, dt;
    double A, B, CT1, CT2, CT3, Kn;
    double u_in, p_in, T_in;
    double u_wb, u_wt, T_wall, T_sq, g_x, g_y;
    double pwk;                 // kappa of the kappa p div(u) forms of R9
    // fields: old iterate, time level n-1, explicit planes, new iterate
    const double *u_o, *v_o, *p_o, *T_o;
    const double *u_1, *v_1, *p_1, *T_1;
    const double *ue, *ve, *Te;
    double *u_w, *v_w, *p_w, *T_w;
    double *ue_w, *ve_w, *Te_w;  // conv kernel outputs
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

// Explicitly rounded products and fused multiply-adds.  The regular-point
// arithmetic (the uniform-mesh stage expressions of sts_march.cuh and their
// restatement in sts_regk.cuh) is written with these: a product that may feed an
// addition is never a plain `*`, so the compiler has no contraction choice left
// (its FMA-fusion heuristics depend on the surrounding code -- use counts, CSE --
// and two kernels computing the same expression were measured to differ by one
// ulp in ~5 % of the points).  Every kernel that computes a regular point then
// gives the same bits, which the decomposition invariance relies on.
__device__ __forceinline__ double MUL(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double FMA(double a, double b, double c) { return __fma_rn(a, b, c); }

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

// ------------------------------------------------------- residual helpers
__device__ __forceinline__ double warp_max(double v)
{
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// NaN-propagating max for the residual slots (fmax would drop NaN).
__device__ __forceinline__ double nmax(double a, double b) { return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000LL) : (a > b ? a : b); }

}  // namespace sts
