// simplets.cu -- host orchestrator + C ABI of libsimplets.so (include/simplets.h).
//
// Loop 1 x loop 2 of the GPU columns of Figs. 1-2:
// per time step: rotate the snapshot handles (n-1 := current, old := n-1;
// no copies), [explicit] one conv_kernel launch, then loop-2 passes of
// pass_kernel until converged or max_passes.  Only residual maxima cross to
// the host during a run.  Multi-GPU slabs along x: halo exchange over
// NCCL after every pass.
#include "../../include/simplets.h"
#include "sts_common.cuh"
#include "sts_march.cuh"
#include "sts_regk.cuh"
#include "sts_conv.cuh"

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <functional>
#include <mutex>
#include <queue>
#include <vector>

// NVTX ranges (header-only NVTX3: a no-op unless a tool such as nsys / ncu with
// --nvtx is attached) around the ABI calls, every time step and every halo phase,
// so a trace shows loop 1, the state transfers and the comm / compute overlap.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

using namespace sts;

// ------------------------------------------------------------- errors
static thread_local std::string g_err;

struct sts_ctx;
static sts_status fail(sts_ctx* c, sts_status st, const std::string& msg);

#define CU(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? STS_E_OOM : STS_E_CUDA,    \
                        std::string(#call) + ": " + cudaGetErrorString(e_));              \
    } while (0)

// ------------------------------------------------------------- NCCL (dlopen)
typedef struct { char internal[128]; } nccl_uid;
typedef void* nccl_comm;
enum { NCCL_UINT64 = 5, NCCL_FLOAT64 = 8, NCCL_MAX = 2 };
struct NcclApi {
    void* h = nullptr;
    int (*GetUniqueId)(nccl_uid*);
    int (*CommInitRank)(nccl_comm*, int, nccl_uid, int);
    int (*CommDestroy)(nccl_comm);
    int (*GroupStart)();
    int (*GroupEnd)();
    int (*Send)(const void*, size_t, int, int, nccl_comm, cudaStream_t);
    int (*Recv)(void*, size_t, int, int, nccl_comm, cudaStream_t);
    int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t);
    bool load()
    {
        if (h) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) { h = dlopen(n, RTLD_NOW | RTLD_GLOBAL); if (h) break; }
        if (!h) return false;
        GetUniqueId = (int (*)(nccl_uid*))dlsym(h, "ncclGetUniqueId");
        CommInitRank = (int (*)(nccl_comm*, int, nccl_uid, int))dlsym(h, "ncclCommInitRank");
        CommDestroy = (int (*)(nccl_comm))dlsym(h, "ncclCommDestroy");
        GroupStart = (int (*)())dlsym(h, "ncclGroupStart");
        GroupEnd = (int (*)())dlsym(h, "ncclGroupEnd");
        Send = (int (*)(const void*, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclSend");
        Recv = (int (*)(void*, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclRecv");
        AllReduce = (int (*)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllReduce");
        return GetUniqueId && CommInitRank && CommDestroy && GroupStart && GroupEnd && Send && Recv && AllReduce;
    }
};
static NcclApi g_nccl;

// ------------------------------------------------------------- context
struct Snapshot { double *u = nullptr, *v = nullptr, *p = nullptr, *T = nullptr; };

struct sts_ctx {
    // problem
    int nx = 0, ny = 0;
    double spacing = 0;
    sts_gas gas{};
    sts_scheme sch{};
    std::vector<sts_square> squares;
    double A = 0, B = 0, CT1 = 0, CT2 = 0, CT3 = 0, u_in = 0, u_wb = 0, u_wt = 0;
    // decomposition
    int rank = 0, world = 1, device = 0;
    int gi0 = 0, nloc = 0, pitch = 0;
    std::vector<int> col_start;            // world+1 entries
    // device memory
    Snapshot snap[3];
    int cur = 0;                           // index of the current state snapshot
    double *ue = nullptr, *ve = nullptr, *Te = nullptr;
    uint32_t* kind32 = nullptr;            // packed ck | uk << 8 | vk << 16, (ny+1) x pitch
    // non-uniform mesh (sts_set_mesh): Delta x of every stored local
    // column, Delta y of rows -PADY .. ny+PADY-1; nu = the NU kernel instances run
    bool nu = false;
    double *dxl = nullptr, *dyp = nullptr;
    std::vector<uint8_t> h_ck, h_uk, h_vk; // host copies of the local kind maps
    std::vector<uint8_t> h_solid;          // slab-local solid map, ny x sol_w (unwrapped columns from sol_lo)
    int sol_lo = 0, sol_w = 0;
    int march_seg = 0, march_nstrips = 0;   // regular CTA height (Hr), strips
    int* cta_order = nullptr;              // (int4) launch order of the march CTAs: general CTAs (longest
                                           // first), then the all-regular ones
    int n_gen = 0, n_reg = 0;              // CTAs of the general / all-regular march kernel
    int* cta_split = nullptr;              // (int4) multi-GPU split: edge strips first (general kernel),
                                           // then the interior general and all-regular CTAs
    int n_edge = 0;                        // CTAs in the edge strips
    int n_split = 0;                       // entries of cta_split
    int n_split_gen = 0;                   // interior general CTAs of cta_split
    cudaStream_t gstream = nullptr;        // the general CTAs of a pass run here, beside the regular ones
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // halo overlap (multi-GPU): edge strips + pack/NCCL/unpack on a high-priority
    // stream while the interior strips of the next pass run on the pass stream
    cudaStream_t hstream = nullptr;
    cudaEvent_t ev_a[2] = {nullptr, nullptr}, ev_b = nullptr, ev_s = nullptr, ev_h = nullptr;
    unsigned long long* red = nullptr;     // [max_passes][9] residual slots, then the sticky bad key
    unsigned long long* bad = nullptr;     // = red + 9 max_passes: first bad state of the advance call
    // graph-driven loop 2 (tolerance mode, one context without NCCL): one CUDA
    // graph per snapshot rotation, loop 2 as a conditional WHILE node
    cudaGraphExec_t tol_exec[3] = {nullptr, nullptr, nullptr};
    // fixed-pass mode as one CUDA graph per time step and snapshot rotation (no
    // host round trip, no per-launch API cost; the paper's small meshes)
    cudaGraphExec_t fix_exec[3] = {nullptr, nullptr, nullptr};
    unsigned long long* h_badstep = nullptr;   // pinned: the sticky bad key after every step of a call
    int h_badstep_n = 0;
    unsigned long long* red2 = nullptr;    // [2][9] residual slots (even / odd passes)
    struct LoopState* d_ls = nullptr;      // device loop state
    struct LoopState* h_ls = nullptr;      // pinned copy
    unsigned long long* h_red = nullptr;   // pinned, 9 entries
    double* stage = nullptr;               // device scratch of the owned slab (rho read-back)
    size_t stage_elems = 0;
    double* halo = nullptr;                // send/recv buffers (multi-GPU)
    size_t halo_elems = 0;
    cudaStream_t stream = nullptr;
    // multi-GPU
    nccl_comm comm = nullptr;
    // fused halo transport (sts_peer_connect / sts_peer_connect_group):
    // peer-mapped pointers to the left [0] / right [1] neighbour's snapshots and
    // explicit planes, and stream-ordered flags instead of pack / NCCL / unpack
    bool peer = false;
    Snapshot nb_snap[2][3];
    double* nb_pl[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};   // ue, ve, Te
    int nb_pitch[2] = {0, 0}, nb_shift[2] = {0, 0};
    unsigned long long* flags = nullptr;       // [2 world]: [q] last halo phase of rank q, [world+q] its last residual push
    std::vector<unsigned long long*> peer_flags;   // every rank's `flags` (peer-mapped; own at [rank])
    unsigned long long* red_all = nullptr;     // [2][10] residual maxima pushed by every rank (step parity)
    unsigned long long** d_peer_red = nullptr; // device array: every rank's red_all
    unsigned long long seq = 0, rseq = 0;      // halo phases / residual pushes issued so far
    std::vector<void*> ipc_mapped;             // IPC mappings to close
    // loop 3 (N3, sch.loop3 > 1): T-p sweep iterates (ping-pong), a junk target for
    // the u, v of the non-final sweeps, junk residual slots + bad key
    double *l3p[2] = {nullptr, nullptr}, *l3T[2] = {nullptr, nullptr}, *l3junk = nullptr;
    unsigned long long* l3red = nullptr;
    bool local_group = false;              // world > 1 without NCCL: in-process slabs (sts_advance_group)
    // stats / profiling
    sts_stats stats{};
    bool profiling = false;
    long long pass0 = 0;                   // passes_done when the current advance call started
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, int>> ev_used;   // (start idx, kind)
    double prof_pass_n = 0, prof_pass_ms = 0, prof_conv_n = 0, prof_conv_ms = 0, launches = 0;
    std::string err;
    // asynchronous host I/O (sts_stage_field / sts_set_staged / sts_fetch_field / sts_io_sync):
    // per field (u, v, p, T) one device staging slot per direction, copy streams for
    // each direction and the events that order slot reuse against the context stream
    struct IoSlot {
        double* d = nullptr;
        int64_t cap = 0, n = 0;
        cudaEvent_t copied = nullptr, consumed = nullptr;   // H2D / D2H done; slot read / written on `stream`
        bool pending = false;                               // staged, not yet set (in) / fetch in flight (out)
    };
    IoSlot io_in[4], io_out[4];
    cudaStream_t io_h2d = nullptr, io_d2h = nullptr;
};

static sts_status fail(sts_ctx* c, sts_status st, const std::string& msg)
{
    g_err = msg;
    if (c) c->err = msg;
    return st;
}

extern "C" const char* sts_last_error(const sts_ctx* ctx)
{
    if (ctx && !ctx->err.empty()) return ctx->err.c_str();
    return g_err.c_str();
}

// ------------------------------------------------------------- layout helpers
static inline long long lidx(const sts_ctx* c, int gi, int gj) { return (long long)gj * c->pitch + (gi - c->gi0 + OFF); }
static inline size_t cell_elems(const sts_ctx* c) { return (size_t)c->pitch * c->ny; }
static inline size_t v_elems(const sts_ctx* c) { return (size_t)c->pitch * (c->ny + 1); }
static inline bool is_periodic(const sts_ctx* c) { return c->gas.xbc == STS_X_PERIODIC; }

// Host kind maps for the stored local columns [gi0-OFF, gi0-OFF+pitch) (DESIGN 3.5).
// The solid map is slab-local: unwrapped global columns [sol_lo, sol_lo + sol_w)
// = the stored columns plus SOL_M on each side (the +-3 window of the regular
// bit and the face kinds reach them), so host memory grows with the slab, not
// with the channel.
constexpr int SOL_M = 4;
static bool solid_global(const sts_ctx* c, int gi, int gj, const std::vector<uint8_t>& solid)
{
    const int u = gi - c->sol_lo;
    if (u < 0 || u >= c->sol_w) return false;            // never reached for stored columns +- SOL_M
    return solid[(size_t)gj * c->sol_w + u] != 0;
}
static uint8_t cell_kind_g(const sts_ctx* c, int gi, int gj, const std::vector<uint8_t>& solid)
{
    if (gj < 0 || gj >= c->ny) return CK_WALLY;
    if (is_periodic(c)) { /* the slab-local map holds the wrapped columns unwrapped */ }
    else if (gi < 0) return CK_INLET;
    else if (gi >= c->nx) return CK_OUTLET;
    return solid_global(c, gi, gj, solid) ? CK_SOLID : CK_FLUID;
}
static uint8_t u_kind_g(const sts_ctx* c, int gf, int gj, const std::vector<uint8_t>& solid)
{
    if (gj < 0 || gj >= c->ny) return FK_NONE;
    if (!is_periodic(c)) {
        if (gf < 0 || gf > c->nx) return FK_NONE;
        if (gf == 0) return FK_INLET;
        if (gf == c->nx) return FK_OUTLET;
    }
    return (cell_kind_g(c, gf - 1, gj, solid) == CK_FLUID && cell_kind_g(c, gf, gj, solid) == CK_FLUID) ? FK_ACTIVE : FK_FIXED0;
}
static uint8_t v_kind_g(const sts_ctx* c, int gi, int gj, const std::vector<uint8_t>& solid)
{
    if (gj < 0 || gj > c->ny) return FK_NONE;
    if (gj == 0 || gj == c->ny) return FK_WALL;
    if (!is_periodic(c) && (gi < 0 || gi >= c->nx)) return FK_NONE;
    return (cell_kind_g(c, gi, gj - 1, solid) == CK_FLUID && cell_kind_g(c, gi, gj, solid) == CK_FLUID) ? FK_ACTIVE : FK_FIXED0;
}

// ------------------------------------------------------------- field I/O
// Fields move between caller buffers (host or device, global or slab shape)
// and the stored local columns by strided 2-D copies (cudaMemcpy2DAsync, the
// direction inferred from the pointers); finish_kernel then applies the ghost
// rules of DESIGN 3.5 items 2-4 and re-imposes the fixed faces of item 1 from
// the packed kind map, in the local layout.
struct FinishArgs {
    int nx, ny, gi0, nloc, pitch, xbc, field, single;   // field: 0 u, 1 v, 2 p, 3 T; single: one rank
    int fill_left, fill_right;                         // ghost columns filled here (not by a halo exchange)
    double inlet_val, u_in;
};
__global__ void finish_kernel(FinishArgs a, const uint32_t* __restrict__ kind, double* d)
{
    const int rows = a.field == 1 ? a.ny + 1 : a.ny;
    const long long n = (long long)rows * a.pitch;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(e / a.pitch), li = (int)(e - (long long)j * a.pitch);
        const int gi = a.gi0 - OFF + li;
        const long long rowb = (long long)j * a.pitch;
        const bool left = li < OFF, right = li >= OFF + a.nloc + (a.field == 0 && !a.xbc && a.gi0 + a.nloc == a.nx ? 1 : 0);
        if ((left && a.fill_left) || (right && a.fill_right)) {
            double val;
            if (a.xbc == 1) {                            // one periodic rank: wrap to an owned column
                const int w = ((gi % a.nx) + a.nx) % a.nx;
                val = d[rowb + (w - a.gi0 + OFF)];
            } else if (gi < 0) {
                val = a.inlet_val;                         // inflow state (BC spec 2)
            } else if (a.field == 0) {
                val = a.inlet_val;                         // u beyond the outlet face: never read
            } else {
                val = d[rowb + (a.nx - 1 - a.gi0 + OFF)];  // zero-gradient outlet (BC spec 3)
            }
            d[e] = val;
        }
        if (a.field <= 1) {                              // fixed faces (BC spec 1-2)
            const uint32_t w = kind[e];
            const uint8_t fk = (uint8_t)((w >> (a.field == 0 ? 8 : 16)) & 0xff);
            if (fk == FK_FIXED0 || fk == FK_WALL) d[e] = 0.0;
            else if (fk == FK_INLET) d[e] = a.u_in;
        }
    }
}
// rho = p / T of the owned columns into a compact (rows x ncols) buffer (Eq. pl5)
__global__ void ratio_kernel(int rows, int ncols, int pitch, const double* __restrict__ p, const double* __restrict__ T,
                             double* __restrict__ r)
{
    const long long n = (long long)rows * ncols;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(e / ncols), i = (int)(e - (long long)j * ncols);
        const long long id = (long long)j * pitch + OFF + i;
        r[e] = p[id] / T[id];
    }
}
// Free stream (BC spec 1-2, R12) in the local layout of all three snapshots.
__global__ void freestream_kernel(long long n_cells, long long n_v, const uint32_t* __restrict__ kind, double u_in,
                                  double p_in, double T_in, double* u0, double* u1, double* u2, double* v0, double* v1,
                                  double* v2, double* p0, double* p1, double* p2, double* T0, double* T1, double* T2)
{
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n_v; e += (long long)gridDim.x * blockDim.x) {
        v0[e] = 0.0; v1[e] = 0.0; v2[e] = 0.0;
        if (e < n_cells) {
            const uint8_t fk = (uint8_t)((kind[e] >> 8) & 0xff);
            const double uv = fk == FK_FIXED0 ? 0.0 : u_in;
            u0[e] = uv; u1[e] = uv; u2[e] = uv;
            p0[e] = p_in; p1[e] = p_in; p2[e] = p_in;
            T0[e] = T_in; T1[e] = T_in; T2[e] = T_in;
        }
    }
}
// Halo strips for the multi-GPU exchange: columns [c0, c0+OFF) of u, v, p, T.
__global__ void halo_pack_kernel(int ny, int pitch, int c0, const double* u, const double* v, const double* p,
                                 const double* T, double* buf)
{
    const int per = OFF * (ny + 1);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 4 * per; e += gridDim.x * blockDim.x) {
        int f = e / per, r = e - f * per, j = r / OFF, i = r - j * OFF;
        const double* src = f == 0 ? u : f == 1 ? v : f == 2 ? p : T;
        int rows = f == 1 ? ny + 1 : ny;
        buf[e] = j < rows ? src[(long long)j * pitch + c0 + i] : 0.0;
    }
}
__global__ void halo_unpack_kernel(int ny, int pitch, int c0, double* u, double* v, double* p, double* T,
                                   const double* buf)
{
    const int per = OFF * (ny + 1);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 4 * per; e += gridDim.x * blockDim.x) {
        int f = e / per, r = e - f * per, j = r / OFF, i = r - j * OFF;
        double* dst = f == 0 ? u : f == 1 ? v : f == 2 ? p : T;
        int rows = f == 1 ? ny + 1 : ny;
        if (j < rows) dst[(long long)j * pitch + c0 + i] = buf[e];
    }
}

// Fused-halo push (N1) of a whole snapshot outside a pass (slab-shaped field
// input): columns [c0, c0+OFF) of u, v, p, T straight into the neighbour's
// columns [c0 + shift, ...) of its copy (peer-mapped pointers, pitch npitch).
__global__ void halo_push_kernel(int ny, int pitch, int c0, const double* u, const double* v, const double* p,
                                 const double* T, int npitch, int shift, double* nu, double* nv, double* np, double* nT)
{
    const int per = OFF * (ny + 1);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 4 * per; e += gridDim.x * blockDim.x) {
        int f = e / per, r = e - f * per, j = r / OFF, i = r - j * OFF;
        if (j >= (f == 1 ? ny + 1 : ny)) continue;
        const double* src = f == 0 ? u : f == 1 ? v : f == 2 ? p : T;
        double* dst = f == 0 ? nu : f == 1 ? nv : f == 2 ? np : nT;
        dst[(long long)j * npitch + c0 + i + shift] = src[(long long)j * pitch + c0 + i];
    }
}
// Residual maxima of one pass (9 u64 slots + the sticky bad key) pushed into
// every rank's red_all by system-scope atomicMax (exact, order-independent:
// the u64 bit patterns of non-negative doubles order like the doubles).
__global__ void red_push_kernel(const unsigned long long* slot, const unsigned long long* bad,
                                unsigned long long** dst, int world, int par)
{
    const int q = threadIdx.x;
    if (q >= world) return;
    unsigned long long* d = dst[q] + 10 * par;
    for (int e = 0; e < 9; e++) atomicMax_system(d + e, slot[e]);
    atomicMax_system(d + 9, *bad);
}

// ------------------------------------------------------------- kernel table
typedef void (*march_fn)(MarchParams);
// regk: the all-regular kernel (sts_march.cuh); nu: the non-uniform-mesh kernel
// the first pass of an explicit step with the planes computed in the pass (N2)
static march_fn march_fusec_table(int tvd, int regk, int graph)
{
    if (graph) {
        if (regk) return tvd ? march_kernel<false, true, true, true, false, false, false, true> : march_kernel<false, false, true, true, false, false, false, true>;
        return tvd ? march_kernel<false, true, true, false, false, false, false, true> : march_kernel<false, false, true, false, false, false, false, true>;
    }
    if (regk) return tvd ? march_kernel<false, true, false, true, false, false, false, true> : march_kernel<false, false, false, true, false, false, false, true>;
    return tvd ? march_kernel<false, true, false, false, false, false, false, true> : march_kernel<false, false, false, false, false, false, false, true>;
}
static constexpr size_t FUSEC_SMEM = sizeof(MarchSmem) + 3 * RW * sizeof(double);
// the explicit planes inside the first pass of each step: explicit variants on one
// context without a halo, uniform mesh, no loop 3 (STS_NO_FUSE: the separate
// conv kernel, as the paper does)
static bool fuse_conv(const sts_ctx* c)
{
    return c->sch.time == STS_EXPLICIT && !c->nu && c->world == 1 && !c->comm && !c->peer && c->sch.loop3 <= 1 &&
           !getenv("STS_NO_FUSE");
}

// the edge strips of a peer-connected rank: general kernel with the fused halo stores (N1)
static march_fn march_halo_table(int impl, int tvd, int nu)
{
    if (nu) {
        if (impl) return tvd ? march_kernel<true, true, false, false, true, false, true> : march_kernel<true, false, false, false, true, false, true>;
        return tvd ? march_kernel<false, true, false, false, true, false, true> : march_kernel<false, false, false, false, true, false, true>;
    }
    if (impl) return tvd ? march_kernel<true, true, false, false, false, false, true> : march_kernel<true, false, false, false, false, false, true>;
    return tvd ? march_kernel<false, true, false, false, false, false, true> : march_kernel<false, false, false, false, false, false, true>;
}
// the all-regular CTAs run regk_kernel (sts_regk.cuh, register-resident operands),
// except implicit TVD (168 registers, 3 CTAs/SM and spills: 0.81 vs 0.74 ms/pass on
// C3, profiles/r02_summary.md); STS_OLD_REGK=1 selects march_kernel<..., REGK = true>
// for every variant, STS_OLD_REGK=0 regk_kernel for every variant (A/B, bitwise tests)
static bool old_regk(int impl, int tvd)
{
    const char* v = getenv("STS_OLD_REGK");
    if (v != nullptr && *v) return atoi(v) != 0;
    return impl && tvd;
}
// one launch per pass (march_fused_kernel, sts_regk.cuh) for the general + all-regular
// CTAs of a uniform-mesh pass without plane fusion or loop 3; STS_NO_FUSED=1: the two
// kernels as two launches / parallel graph nodes (A/B)
static bool use_fused(const sts_ctx* c, bool fusec, bool l3)
{
    const char* v = getenv("STS_NO_FUSED");
    // implicit TVD: the two-kernel launch (the general kernel at 4 CTAs/SM beside
    // march_kernel<REGK>) measured faster than one launch at 3 CTAs/SM (22.0 vs 20.6 G FVU/s)
    const bool itvd = c->sch.time == STS_IMPLICIT && c->sch.space == STS_TVD_VANLEER && !getenv("STS_ITVD_FUSED");
    return !fusec && !l3 && !c->nu && !itvd && !(v != nullptr && atoi(v) != 0) && !old_regk(0, 0);
}
static march_fn fused_table(int impl, int tvd, int graph)
{
    if (graph) {
        if (impl) return tvd ? march_fused_kernel<true, true, true> : march_fused_kernel<true, false, true>;
        return tvd ? march_fused_kernel<false, true, true> : march_fused_kernel<false, false, true>;
    }
    if (impl) return tvd ? march_fused_kernel<true, true, false> : march_fused_kernel<true, false, false>;
    return tvd ? march_fused_kernel<false, true, false> : march_fused_kernel<false, false, false>;
}
static march_fn march_table(int impl, int tvd, int regk, int nu = 0, int l3 = 0)
{
    if (l3) {                                    // loop-3 sweeps k >= 2 (N3)
        if (regk) {
            if (impl) return tvd ? march_kernel<true, true, false, true, false, true> : march_kernel<true, false, false, true, false, true>;
            return tvd ? march_kernel<false, true, false, true, false, true> : march_kernel<false, false, false, true, false, true>;
        }
        if (impl) return tvd ? march_kernel<true, true, false, false, false, true> : march_kernel<true, false, false, false, false, true>;
        return tvd ? march_kernel<false, true, false, false, false, true> : march_kernel<false, false, false, false, false, true>;
    }
    if (nu) {
        if (impl) return tvd ? march_kernel<true, true, false, false, true> : march_kernel<true, false, false, false, true>;
        return tvd ? march_kernel<false, true, false, false, true> : march_kernel<false, false, false, false, true>;
    }
    if (regk) {
        if (!old_regk(impl, tvd)) {
            if (impl) return tvd ? regk_kernel<true, true, false> : regk_kernel<true, false, false>;
            return tvd ? regk_kernel<false, true, false> : regk_kernel<false, false, false>;
        }
        if (impl) return tvd ? march_kernel<true, true, false, true> : march_kernel<true, false, false, true>;
        return tvd ? march_kernel<false, true, false, true> : march_kernel<false, false, false, true>;
    }
    if (impl) return tvd ? march_kernel<true, true> : march_kernel<true, false>;
    return tvd ? march_kernel<false, true> : march_kernel<false, false>;
}
static march_fn march_graph_table(int impl, int tvd, int regk, int nu = 0)
{
    if (nu) {
        if (impl) return tvd ? march_kernel<true, true, true, false, true> : march_kernel<true, false, true, false, true>;
        return tvd ? march_kernel<false, true, true, false, true> : march_kernel<false, false, true, false, true>;
    }
    if (regk) {
        if (!old_regk(impl, tvd)) {
            if (impl) return tvd ? regk_kernel<true, true, true> : regk_kernel<true, false, true>;
            return tvd ? regk_kernel<false, true, true> : regk_kernel<false, false, true>;
        }
        if (impl) return tvd ? march_kernel<true, true, true, true> : march_kernel<true, false, true, true>;
        return tvd ? march_kernel<false, true, true, true> : march_kernel<false, false, true, true>;
    }
    if (impl) return tvd ? march_kernel<true, true, true> : march_kernel<true, false, true>;
    return tvd ? march_kernel<false, true, true> : march_kernel<false, false, true>;
}
static march_fn conv_march_table(int tvd, int nu = 0)
{
    if (nu) return tvd ? conv_march_kernel<true, true> : conv_march_kernel<false, true>;
    return tvd ? conv_march_kernel<true> : conv_march_kernel<false>;
}
// dynamic shared memory of the march / conv kernels: the NU instances keep the
// column widths of their ring columns behind the struct
static size_t march_smem(const sts_ctx* c) { return sizeof(MarchSmem) + (c->nu ? RW * sizeof(double) : 0); }
// dynamic shared memory of the all-regular kernel of a pass
static size_t regk_smem(const sts_ctx* c, bool fusec, bool l3)
{
    (void)l3;
    return fusec ? sizeof(MarchSmem) + 3 * RW * sizeof(double) : march_smem(c);
}
static size_t conv_smem(const sts_ctx* c) { return sizeof(ConvSmem) + (c->nu ? RW * sizeof(double) : 0); }

// The shared-memory opt-in is a per-device function attribute: one bit per
// device (the caller has made ctx->device current), set once every attribute
// of that device is in place.
static sts_status set_smem_attrs(sts_ctx* ctx)
{
    static std::atomic<unsigned long long> done_mask{0};
    const unsigned long long bit = 1ull << (ctx->device & 63);
    if (done_mask.load() & bit) return STS_OK;
    for (int q = 0; q < 40; q++) {
        const int impl = q & 1, tvd = (q >> 1) & 1, regk = (q >> 2) & 1, graph = (q >> 3) & 1, nu = (q >> 4) & 1;
        const int l3 = q >= 32;                  // q 32..39: the loop-3 instances (no graph, no NU)
        if ((nu && regk) || (l3 && (graph || nu))) continue;
        march_fn f = l3 ? march_table(impl, tvd, regk, 0, 1)
                        : graph ? march_graph_table(impl, tvd, regk, nu) : march_table(impl, tvd, regk, nu);
        CU(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(MarchSmem) + (nu ? RW * sizeof(double) : 0))));
    }
    {
        const march_fn rk[] = {regk_kernel<false, false, false>, regk_kernel<false, true, false>, regk_kernel<true, false, false>,
                               regk_kernel<true, true, false>, regk_kernel<false, false, true>, regk_kernel<false, true, true>,
                               regk_kernel<true, false, true>, regk_kernel<true, true, true>,
                               march_kernel<false, false, false, true>, march_kernel<false, true, false, true>,
                               march_kernel<true, false, false, true>, march_kernel<true, true, false, true>,
                               march_kernel<false, false, true, true>, march_kernel<false, true, true, true>,
                               march_kernel<true, false, true, true>, march_kernel<true, true, true, true>};
        for (march_fn f : rk)
            CU(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MarchSmem)));
        for (int q = 0; q < 8; q++)
            CU(cudaFuncSetAttribute((const void*)fused_table(q & 1, (q >> 1) & 1, q >> 2),
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MarchSmem)));
    }
    for (int q = 0; q < 8; q++) {
        const int impl = q & 1, tvd = (q >> 1) & 1, nu = q >> 2;
        CU(cudaFuncSetAttribute((const void*)march_halo_table(impl, tvd, nu), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(MarchSmem) + (nu ? RW * sizeof(double) : 0))));
    }
    for (int q = 0; q < 8; q++)
        CU(cudaFuncSetAttribute((const void*)march_fusec_table(q & 1, (q >> 1) & 1, q >> 2),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FUSEC_SMEM));
    for (int q = 0; q < 4; q++)
        CU(cudaFuncSetAttribute((const void*)conv_march_table(q & 1, q >> 1), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(ConvSmem) + ((q >> 1) ? RW * sizeof(double) : 0))));
    done_mask.fetch_or(bit);
    return STS_OK;
}

static Params make_params(const sts_ctx* c)
{
    Params k{};
    k.nx = c->nx; k.ny = c->ny; k.gi0 = c->gi0; k.nloc = c->nloc; k.pitch = c->pitch;
    k.xbc = c->gas.xbc; k.mirror = (is_periodic(c) && c->world == 1 && !c->comm) ? 1 : 0;
    k.first_rank = c->rank == 0; k.last_rank = c->rank == c->world - 1;
    k.dx = c->spacing; k.dy = c->spacing; k.dt = c->sch.dt;
    k.A = c->A; k.B = c->B; k.CT1 = c->CT1; k.CT2 = c->CT2; k.CT3 = c->CT3; k.Kn = c->gas.Kn;
    k.u_in = c->u_in; k.p_in = c->gas.p_in; k.T_in = c->gas.T_in;
    k.u_wb = c->u_wb; k.u_wt = c->u_wt; k.T_wall = c->gas.T_wall; k.T_sq = c->gas.T_square;
    k.g_x = c->gas.g_x; k.g_y = c->gas.g_y;
    // pressure-work form of S^T_c (reading R9) and kappa of the p div(u) forms
    k.pw_form = c->gas.pw_form;
    k.pwk = c->gas.pw_form == PW_DPDT ? 0.0 : c->gas.pw_form == PW_PRINTED ? c->CT3
          : c->gas.pw_form == PW_NEG ? -c->CT3 : -c->gas.gamma * c->CT3;
    return k;
}

static MarchParams make_march(const sts_ctx* c, const Params& k)
{
    MarchParams m{};
    m.k = k;
    m.kind = c->kind32;
    m.order = (const int4*)c->cta_order;
    const double dx = c->spacing, dy = c->spacing, dt = c->sch.dt;
    m.inv_dx = 1.0 / dx; m.inv_dy = 1.0 / dy;
    m.CT1_dydx = c->CT1 * dy / dx; m.CT1_dxdy = c->CT1 * dx / dy;
    m.B_dydx = c->B * dy / dx; m.B_dxdy = c->B * dx / dy;
    m.c_t = dx * dy / (2.0 * dt); m.dV = dx * dy; m.half_dV = 0.5 * dx * dy;
    m.A_dy = c->A * dy; m.A_dx = c->A * dx;
    m.B43_dydx = 4.0 / 3.0 * m.B_dydx; m.B43_dxdy = 4.0 / 3.0 * m.B_dxdy;
    m.q_dx = 0.25 / dx; m.q_dy = 0.25 / dy;
    m.h_dx = 0.5 / dx; m.h_dy = 0.5 / dy; m.inv_dt = 1.0 / dt;
    m.pw_a = c->gas.pw_form == PW_DPDT ? c->CT3 : 0.0;
    m.bad = c->bad;
    m.pass_key = 0xFFFFF;
    m.dxl = c->dxl;
    m.dyp = c->dyp;
    m.force_general = getenv("STS_FORCE_GENERAL") ? 1 : 0;
    return m;
}

// CTA schedule of the y-march (DESIGN 5.1).  Every strip of MX columns is cut
// along y into CTAs {strip, J0, J1, flags}.  Row j of a strip can belong to an
// all-regular CTA when every point of rows j-3 .. j (the warm-up reach) in the
// strip's 128 columns is regular; such rows form regular runs, run by the
// all-regular kernel in CTAs of about Hr rows.  The other rows (near the
// channel walls and the squares, the inlet and outlet strips) form general
// runs, cut into CTAs of at most Hg rows: a general row step costs up to 2.35
// regular ones (warps that mix both instances run both), so short general CTAs
// keep them off the critical path.  Cost of a CTA = its rows + WARM warm-up rows,
// each weighted by the slowest warp of the row (regular 1, general 1.35, mixed
// 2.35); Hg and Hr minimise the makespan of a longest-first list schedule onto
// the resident slots (148 SMs x CTAs/SM from the occupancy API).
struct CtaE { int strip, J0, J1, flags; double cost; };

static void choose_segments(sts_ctx* c, const std::vector<uint32_t>& packed)
{
    int dev_sms = 148, per_sm = 3;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
    int nb = 0;
    const void* fn = (const void*)march_table(c->sch.time == STS_IMPLICIT, c->sch.space == STS_TVD_VANLEER, !c->nu, c->nu);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, MX, regk_smem(c, false, false)) == cudaSuccess && nb > 0)
        per_sm = nb;
    const int strips = (c->nloc + MW - 1) / MW;
    const int slots = dev_sms * per_sm;
    const int ny = c->ny;
    // warp costs relative to an all-regular warp: a warp with any general point runs
    // the general instance (warp-uniform dispatch, sts_march_loop.inc)
    // (regk_kernel, v10: a row of a general CTA costs ~3 regk rows -- the general kernel
    // runs the round-2 regular instance at 4 CTAs/SM beside the general one; measured
    // over 4032 x {200, 400, 4000}, profiles/r02_v10_seg_grid.txt)
    double w_gen = 3.0, w_mix = 3.0;
    if (const char* cv = getenv("STS_COST")) sscanf(cv, "%lf,%lf", &w_gen, &w_mix);   // tuning hook
    // every CTA general: test hook, or a non-uniform mesh (the NU kernel has general instances only)
    const bool no_allreg = getenv("STS_NO_ALLREG") != nullptr || c->nu;
    int forced = 0, forced_r = 0;
    if (const char* sv = getenv("STS_SEG")) {                 // test hook: all heights, or "Hg,Hr"
        forced = std::max(0, atoi(sv));
        const char* cm = strchr(sv, ',');
        forced_r = cm ? std::max(0, atoi(cm + 1)) : forced;
    }
    // fixed cost of a CTA in row steps (prologue: 5 ring rows, 4 derives, the
    // residual epilogue, launch) -- tuning hook STS_CTA_OVH
    double ovh = 0.0;
    if (const char* ov = getenv("STS_CTA_OVH")) ovh = atof(ov);
    // per (strip, row): cost of a row step and "all 128 points regular"
    std::vector<double> rcost((size_t)strips * ny);
    std::vector<uint8_t> rreg((size_t)strips * ny);
    for (int st = 0; st < strips; st++)
        for (int j = 0; j < ny; j++) {
            double rc = 1.0;
            int all = 1;
            for (int w = 0; w < MX / 32; w++) {
                int nreg = 0;
                for (int l = 0; l < 32; l++) {
                    const int li = st * MW - 2 + 32 * w + l + OFF;
                    if (li >= 0 && li < c->pitch && (packed[(size_t)j * c->pitch + li] & REG_BIT)) nreg++;
                }
                rc = std::max(rc, nreg == 32 ? 1.0 : (nreg == 0 ? w_gen : w_mix));
                all &= nreg == 32;
            }
            rcost[(size_t)st * ny + j] = rc;
            rreg[(size_t)st * ny + j] = (uint8_t)(all && !no_allreg);
        }
    // row j can be in an all-regular CTA: rows j-WARM .. j all regular
    auto R = [&](int st, int j) {
        if (j < WARM) return false;
        for (int q = j - WARM; q <= j; q++) if (!rreg[(size_t)st * ny + q]) return false;
        return true;
    };
    auto cta_cost = [&](int st, int J0, int J1) {
        double cst = 0.0;
        for (int q = std::max(0, J0 - WARM); q < J1; q++) cst += rcost[(size_t)st * ny + q];
        if (J0 - WARM < 0) cst += (WARM - J0) * rcost[(size_t)st * ny + 0];
        return cst + ovh;
    };
    // the CTAs of one strip for heights (Hg, Hr)
    auto cut = [&](int st, int Hg, int Hr, std::vector<CtaE>& out) {
        int j = 0;
        while (j < ny) {
            const bool reg = R(st, j);
            int e = j;
            while (e < ny && R(st, e) == reg) e++;
            const int len = e - j, H = reg ? Hr : Hg;
            const int n = reg ? std::max(1, (len + H / 2) / H) : (len + H - 1) / H;
            for (int q = 0; q < n; q++) {
                const int a = j + (int)((long long)len * q / n), b = j + (int)((long long)len * (q + 1) / n);
                out.push_back({st, a, b, reg ? ALLREG_BIT : 0, cta_cost(st, a, b) * (reg ? 1.0 : 1.0)});
            }
            j = e;
        }
    };
    auto makespan = [&](std::vector<CtaE>& v) {
        std::stable_sort(v.begin(), v.end(), [](const CtaE& x, const CtaE& y) { return x.cost > y.cost; });
        std::priority_queue<double, std::vector<double>, std::greater<double>> load;
        for (size_t q = 0; q < std::min<size_t>(slots, v.size()); q++) load.push(0.0);
        double ms = 0.0;
        for (auto& q : v) {
            const double l = load.top() + q.cost;
            load.pop();
            load.push(l);
            ms = std::max(ms, l);
        }
        return ms;
    };
    std::vector<CtaE> best, cur;
    double best_ms = 1e300;
    int best_hg = 8, best_hr = 8;
    std::vector<int> hg_c, hr_c;
    if (forced > 0) { hg_c = {forced}; hr_c = {forced_r > 0 ? forced_r : forced}; }
    else {
        hg_c = {4, 6, 8, 12, 16};   // short general CTAs: 24-48 rows measured 3-6 % slower (C3)
        // Hr: 4, 6, ..., 96.  Longer regular CTAs look cheaper to the model (fewer
        // warm-up rows) but measure slower past a point: a slot is not a processor --
        // the CTAs resident on one SM share its issue rate, so a schedule of few long
        // CTAs leaves a long tail (round 2, march_kernel: Hr 252, 501 CTAs 0.630
        // ms/pass, 64 0.614; regk_kernel at 3 CTAs/SM, graph path, C3: Hg 16 with
        // Hr 48 / 64 / 96 29.1 / 29.6 / 29.8 G FVU/s, profiles/r02_v10_seg_grid.txt)
        // (from 4 rows: the paper's 4032 x 200 mesh cannot fill 148 SMs x 4 CTAs with
        // longer segments -- 6-row segments measured 0.63 ms/step, 8-row ones 0.72)
        for (int h = std::min(ny, 4); h <= std::min(ny, 96); h += 2) hr_c.push_back(h);
        if (hr_c.empty()) hr_c.push_back(std::max(1, ny));
    }
    // the longest regular CTAs (then general ones) whose makespan is within 4 % of the best: the model
    // ignores that CTAs sharing an SM share its issue rate, and longer regular CTAs
    // (fewer warm-up rows and prologues) measured faster at equal model makespan
    // (C3: Hr 74 vs 94 at Hg 16, 28.9 vs 29.8 G FVU/s; 4032 x 200: Hr 10 vs 20 at
    // Hg 6, 15.2 vs 15.5 G FVU/s)
    std::vector<std::array<double, 3>> scored;
    for (int hg : hg_c)
        for (int hr : hr_c) {
            cur.clear();
            for (int st = 0; st < strips; st++) cut(st, hg, hr, cur);
            const double ms = makespan(cur);
            scored.push_back({ms, (double)hg, (double)hr});
            best_ms = std::min(best_ms, ms);
        }
    {
        double pick_ms = 1e300;
        best_hr = 0;
        best_hg = 0;
        for (auto& q : scored) {
            if (q[0] > best_ms * 1.04) continue;
            if (q[2] > best_hr || (q[2] == best_hr && q[1] > best_hg)) { best_hr = (int)q[2]; best_hg = (int)q[1]; pick_ms = q[0]; }
        }
        cur.clear();
        for (int st = 0; st < strips; st++) cut(st, best_hg, best_hr, cur);
        best_ms = makespan(cur);
        best = cur;
    }
    c->march_seg = best_hr;
    c->march_nstrips = strips;
    // launch order: general CTAs (longest first), then the all-regular ones
    auto upload = [&](int** dst, const std::vector<int4>& v) {
        cudaFree(*dst);
        *dst = nullptr;
        cudaMalloc(dst, std::max<size_t>(1, v.size()) * sizeof(int4));
        cudaMemcpy(*dst, v.data(), v.size() * sizeof(int4), cudaMemcpyHostToDevice);
    };
    std::vector<int4> order, order_reg;
    for (auto& q : best) ((q.flags & ALLREG_BIT) ? order_reg : order).push_back(make_int4(q.strip, q.J0, q.J1, q.flags));
    c->n_gen = (int)order.size();
    c->n_reg = (int)order_reg.size();
    order.insert(order.end(), order_reg.begin(), order_reg.end());
    if (getenv("STS_VERBOSE"))
        fprintf(stderr, "sts: Hg %d Hr %d, %d general + %d all-regular CTAs, makespan %.0f\n", best_hg, best_hr,
                c->n_gen, c->n_reg, best_ms);
    upload(&c->cta_order, order);
    // Split order for the multi-GPU halo overlap: the CTAs of the edge strips
    // (strip st reads local columns st MW .. st MW + 127 and writes st MW + 2 ..
    // + 126: an edge strip reads a ghost column or writes one of the 4 columns
    // sent to a neighbour), all run by the general kernel and cut ~15 % shorter
    // so that they finish early enough for the halo exchange to hide behind the
    // interior of the next pass; then the interior general and regular CTAs.
    auto edge = [&](int st) { const int I0 = st * MW; return I0 < OFF || I0 + MX >= c->nloc; };
    std::vector<CtaE> ev;
    for (int st = 0; st < strips; st++)
        if (edge(st)) cut(st, std::max(1, (int)(best_hg * 0.85)), std::max(1, std::min(best_hr, (int)(best_hr * 0.85))), ev);
    std::stable_sort(ev.begin(), ev.end(), [](const CtaE& x, const CtaE& y) { return x.cost > y.cost; });
    std::vector<int4> split, split_reg;
    for (auto& q : ev) split.push_back(make_int4(q.strip, q.J0, q.J1, q.flags));
    c->n_edge = (int)split.size();
    for (auto& q : order) {
        if (edge(q.x)) continue;
        ((q.w & ALLREG_BIT) ? split_reg : split).push_back(q);
    }
    c->n_split_gen = (int)split.size() - c->n_edge;
    split.insert(split.end(), split_reg.begin(), split_reg.end());
    c->n_split = (int)split.size();
    upload(&c->cta_split, split);
}

// One loop-2 pass of the march kernels over `order`: the n_gen general CTAs on
// the context's high-priority stream beside the n_reg all-regular CTAs on st
// (fork / join by events; the same calls build the dependencies inside a graph
// capture).  Returns the number of launches.
static int launch_march(sts_ctx* c, const MarchParams& m, bool graph, cudaStream_t st, const int* order,
                        int n_gen, int n_reg, bool l3 = false, bool fusec = false)
{
    const int impl = c->sch.time == STS_IMPLICIT, tvd = c->sch.space == STS_TVD_VANLEER;
    march_fn gen = fusec ? march_fusec_table(tvd, 0, graph)
                 : l3 ? march_table(impl, tvd, 0, 0, 1) : graph ? march_graph_table(impl, tvd, 0, c->nu) : march_table(impl, tvd, 0, c->nu);
    march_fn reg = fusec ? march_fusec_table(tvd, 1, graph)
                 : l3 ? march_table(impl, tvd, 1, 0, 1) : graph ? march_graph_table(impl, tvd, 1) : march_table(impl, tvd, 1);
    const size_t sm = fusec ? FUSEC_SMEM : march_smem(c);
    if (use_fused(c, fusec, l3) && n_gen + n_reg > 0) {
        MarchParams mf = m;
        mf.order = (const int4*)order;
        fused_table(impl, tvd, graph)<<<n_gen + n_reg, MX, sm, st>>>(mf);
        return 1;
    }
    MarchParams mg = m, mr = m;
    mg.order = (const int4*)order;
    mr.order = (const int4*)order + n_gen;
    if (n_gen > 0 && n_reg > 0) {
        cudaEventRecord(c->ev_fork, st);
        cudaStreamWaitEvent(c->gstream, c->ev_fork, 0);
        gen<<<n_gen, MX, sm, c->gstream>>>(mg);
        cudaEventRecord(c->ev_join, c->gstream);
        reg<<<n_reg, MX, regk_smem(c, fusec, l3), st>>>(mr);
        cudaStreamWaitEvent(st, c->ev_join, 0);
        return 2;
    }
    if (n_gen > 0) gen<<<n_gen, MX, sm, st>>>(mg);
    else if (n_reg > 0) reg<<<n_reg, MX, regk_smem(c, fusec, l3), st>>>(mr);
    return (n_gen > 0 || n_reg > 0) ? 1 : 0;
}

// ------------------------------------------------------------- profiling
static cudaEvent_t ev_get(sts_ctx* c, size_t i)
{
    while (c->ev_pool.size() <= i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[i];
}
static void prof_begin(sts_ctx* c, int kind)
{
    if (!c->profiling) return;
    size_t i = 2 * c->ev_used.size();
    cudaEventRecord(ev_get(c, i), c->stream);
    c->ev_used.push_back({(int)i, kind});
}
static void prof_end(sts_ctx* c)
{
    if (!c->profiling) return;
    cudaEventRecord(ev_get(c, c->ev_used.back().first + 1), c->stream);
}
static void prof_collect(sts_ctx* c)
{
    if (c->ev_used.empty()) return;
    cudaEventSynchronize(c->ev_pool[c->ev_used.back().first + 1]);
    for (auto& pr : c->ev_used) {
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev_pool[pr.first], c->ev_pool[pr.first + 1]);
        if (pr.second == 0) { c->prof_pass_n += 1; c->prof_pass_ms += ms; }
        else { c->prof_conv_n += 1; c->prof_conv_ms += ms; }
    }
    c->ev_used.clear();
}

// ------------------------------------------------------------- halo exchange
// Slab halos: my first OFF owned columns go to the left
// neighbour's right ghost columns, my last OFF owned columns to the right
// neighbour's left ghosts; u, v, p, T (or the three explicit planes).
static int left_of(const sts_ctx* c) { return c->rank > 0 ? c->rank - 1 : (is_periodic(c) ? c->world - 1 : -1); }
static int right_of(const sts_ctx* c) { return c->rank < c->world - 1 ? c->rank + 1 : (is_periodic(c) ? 0 : -1); }
static int halo_per(const sts_ctx* c) { return 4 * OFF * (c->ny + 1); }

static sts_status halo_pack(sts_ctx* ctx, const Snapshot& s, cudaStream_t st)
{
    const int per = halo_per(ctx), blocks = (per + 255) / 256;
    if (left_of(ctx) >= 0) { halo_pack_kernel<<<blocks, 256, 0, st>>>(ctx->ny, ctx->pitch, OFF, s.u, s.v, s.p, s.T, ctx->halo); ctx->launches++; }
    if (right_of(ctx) >= 0) { halo_pack_kernel<<<blocks, 256, 0, st>>>(ctx->ny, ctx->pitch, ctx->nloc, s.u, s.v, s.p, s.T, ctx->halo + per); ctx->launches++; }
    CU(cudaGetLastError());
    return STS_OK;
}
static sts_status halo_unpack(sts_ctx* ctx, const Snapshot& s, cudaStream_t st)
{
    const int per = halo_per(ctx), blocks = (per + 255) / 256;
    if (left_of(ctx) >= 0) { halo_unpack_kernel<<<blocks, 256, 0, st>>>(ctx->ny, ctx->pitch, 0, s.u, s.v, s.p, s.T, ctx->halo + 2 * per); ctx->launches++; }
    if (right_of(ctx) >= 0) { halo_unpack_kernel<<<blocks, 256, 0, st>>>(ctx->ny, ctx->pitch, OFF + ctx->nloc, s.u, s.v, s.p, s.T, ctx->halo + 3 * per); ctx->launches++; }
    CU(cudaGetLastError());
    return STS_OK;
}
// NCCL transport: grouped send/recv with both neighbours on the context stream.
static sts_status halo_nccl(sts_ctx* ctx, cudaStream_t st)
{
    const int per = halo_per(ctx);
    const int left = left_of(ctx), right = right_of(ctx);
    // NCCL matches the messages of one (sender, receiver) pair in issue order.
    // When the left and right neighbour are the same rank (2-rank ring, or a
    // periodic single rank talking to itself) every rank must send its RIGHT
    // strip first and receive into its LEFT ghosts first: a rank's left ghosts
    // take its left neighbour's right strip.
    if (g_nccl.GroupStart()) return fail(ctx, STS_E_COMM, "ncclGroupStart");
    if (right >= 0 && g_nccl.Send(ctx->halo + per, per, NCCL_FLOAT64, right, ctx->comm, st))
        return fail(ctx, STS_E_COMM, "ncclSend");
    if (left >= 0 && g_nccl.Send(ctx->halo, per, NCCL_FLOAT64, left, ctx->comm, st))
        return fail(ctx, STS_E_COMM, "ncclSend");
    if (left >= 0 && g_nccl.Recv(ctx->halo + 2 * per, per, NCCL_FLOAT64, left, ctx->comm, st))
        return fail(ctx, STS_E_COMM, "ncclRecv");
    if (right >= 0 && g_nccl.Recv(ctx->halo + 3 * per, per, NCCL_FLOAT64, right, ctx->comm, st))
        return fail(ctx, STS_E_COMM, "ncclRecv");
    if (g_nccl.GroupEnd()) return fail(ctx, STS_E_COMM, "ncclGroupEnd");
    return STS_OK;
}
// One halo exchange of snapshot `which` (0..2 = snapshots, 3 = explicit planes)
// for a group of n contexts (n == 1: this process' rank, NCCL if world > 1;
// n == world: in-process slabs, device-to-device copies on one stream).
static Snapshot pick(sts_ctx* c, int which)
{
    if (which == 3) return Snapshot{c->ue, c->ve, c->Te, c->Te};
    return c->snap[which];
}
static sts_status exchange_group(sts_ctx** cs, int n, const int* which, cudaStream_t st)
{
    NvtxRange nv("halo_exchange");
    if ((cs[0]->world == 1 && !cs[0]->comm) || cs[0]->peer) return STS_OK;   // peers: stored in the epilogues
    for (int r = 0; r < n; r++) { sts_status e = halo_pack(cs[r], pick(cs[r], which[r]), st); if (e) return e; }
    if (n == 1) {
        sts_status e = halo_nccl(cs[0], st);
        if (e) return e;
    } else {
        for (int r = 0; r < n; r++) {
            sts_ctx* ctx = cs[r];
            const int per = halo_per(ctx);
            const int l = left_of(ctx), rr = right_of(ctx);
            if (l >= 0) CU(cudaMemcpyAsync(ctx->halo + 2 * per, cs[l]->halo + per, per * sizeof(double), cudaMemcpyDeviceToDevice, st));
            if (rr >= 0) CU(cudaMemcpyAsync(ctx->halo + 3 * per, cs[rr]->halo, per * sizeof(double), cudaMemcpyDeviceToDevice, st));
        }
    }
    for (int r = 0; r < n; r++) { sts_status e = halo_unpack(cs[r], pick(cs[r], which[r]), st); if (e) return e; }
    return STS_OK;
}

// ------------------------------------------------------------- fused halo (N1)
// Stream-ordered flags over peer memory: every halo phase
// (explicit planes, loop-2 pass) gets a number q.  Before a phase stores into
// its neighbours' ghost columns it waits, on its own stream, until both
// neighbours have finished phase q-1: that covers the neighbour's writes into
// my ghosts (read now) and its reads of the ghosts I am about to overwrite
// (both happened in phase q-1 or earlier; interior strips touch no ghost
// column).  After the phase's edge work the stream writes q into the
// neighbours' flag word for this rank; the write carries a memory barrier, so
// the peer stores of the phase are visible first.  No SM waits, no kernel
// is added, no NCCL call is made.
typedef CUresult (*pfn_memop64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
static pfn_memop64 g_write64 = nullptr, g_wait64 = nullptr;
static bool memops_load()
{
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = cudaDriverEntryPointSymbolNotFound;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", (void**)&g_write64, cudaEnableDefault, &q1) != cudaSuccess ||
            q1 != cudaDriverEntryPointSuccess)
            g_write64 = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue64", (void**)&g_wait64, cudaEnableDefault, &q2) != cudaSuccess ||
            q2 != cudaDriverEntryPointSuccess)
            g_wait64 = nullptr;
    });
    return g_write64 && g_wait64;
}
static sts_status peer_wait_rank(sts_ctx* c, int q, int slot_base, unsigned long long v, cudaStream_t s)
{
    if (v == 0) return STS_OK;
    if (g_wait64((CUstream)s, (CUdeviceptr)(c->flags + slot_base + q), v, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        return fail(c, STS_E_COMM, "cuStreamWaitValue64 failed");
    return STS_OK;
}
static sts_status peer_signal_rank(sts_ctx* c, int q, int slot_base, unsigned long long v, cudaStream_t s)
{
    if (g_write64((CUstream)s, (CUdeviceptr)(c->peer_flags[q] + slot_base + c->rank), v, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
        return fail(c, STS_E_COMM, "cuStreamWriteValue64 failed");
    return STS_OK;
}
// wait until both neighbours finished halo phase v
static sts_status peer_wait(sts_ctx* c, unsigned long long v, cudaStream_t s)
{
    const int l = left_of(c), r = right_of(c);
    if (l >= 0) { sts_status e = peer_wait_rank(c, l, 0, v, s); if (e) return e; }
    if (r >= 0 && r != l) { sts_status e = peer_wait_rank(c, r, 0, v, s); if (e) return e; }
    return STS_OK;
}
// tell both neighbours that this rank finished halo phase v
static sts_status peer_signal(sts_ctx* c, unsigned long long v, cudaStream_t s)
{
    const int l = left_of(c), r = right_of(c);
    if (l >= 0) { sts_status e = peer_signal_rank(c, l, 0, v, s); if (e) return e; }
    if (r >= 0 && r != l) { sts_status e = peer_signal_rank(c, r, 0, v, s); if (e) return e; }
    return STS_OK;
}
// The neighbour pointers of one march / conv launch: snapshot `which` of the
// neighbours (0..2), or their explicit planes (3); none on a physical boundary.
static void peer_params(const sts_ctx* c, int which, MarchParams& m)
{
    for (int sd = 0; sd < 2; sd++) {
        const int nb = sd == 0 ? left_of(c) : right_of(c);
        const bool on = c->peer && nb >= 0;
        if (which == 3) {
            m.nb_u[sd] = on ? c->nb_pl[sd][0] : nullptr; m.nb_v[sd] = on ? c->nb_pl[sd][1] : nullptr;
            m.nb_p[sd] = nullptr; m.nb_T[sd] = on ? c->nb_pl[sd][2] : nullptr;
        } else {
            m.nb_u[sd] = on ? c->nb_snap[sd][which].u : nullptr; m.nb_v[sd] = on ? c->nb_snap[sd][which].v : nullptr;
            m.nb_p[sd] = on ? c->nb_snap[sd][which].p : nullptr; m.nb_T[sd] = on ? c->nb_snap[sd][which].T : nullptr;
        }
        m.nb_pitch[sd] = c->nb_pitch[sd];
        m.nb_shift[sd] = c->nb_shift[sd];
    }
}
// A state write outside a pass (sts_set_field, sts_init_freestream) on a
// peer-connected rank is a halo phase of its own: the neighbours' next pushes
// into my ghost columns must come after it (they wait for this phase), and
// mine after theirs.  Every rank makes the same calls (they are collective).
static sts_status peer_fence(sts_ctx* c)
{
    if (!c->peer) return STS_OK;
    return peer_signal(c, ++c->seq, c->stream);
}
// One collective push of a whole snapshot (slab-shaped field input on a
// peer-connected rank): my edge columns into both neighbours' ghosts, then
// wait until both neighbours have pushed theirs into mine.
static sts_status peer_exchange(sts_ctx* ctx, int which, cudaStream_t st)
{
    NvtxRange nv("halo_peer");
    sts_ctx* const c = ctx;
    const unsigned long long q = ++c->seq;
    sts_status e = peer_wait(c, q - 1, st);
    if (e) return e;
    const Snapshot& s = c->snap[which];
    const int per = 4 * OFF * (c->ny + 1), blocks = (per + 255) / 256;
    for (int sd = 0; sd < 2; sd++) {
        if ((sd == 0 ? left_of(c) : right_of(c)) < 0) continue;
        const Snapshot& n = c->nb_snap[sd][which];
        halo_push_kernel<<<blocks, 256, 0, st>>>(c->ny, c->pitch, sd == 0 ? OFF : c->nloc, s.u, s.v, s.p, s.T,
                                                 c->nb_pitch[sd], c->nb_shift[sd], n.u, n.v, n.p, n.T);
        c->launches++;
    }
    CU(cudaGetLastError());
    e = peer_signal(c, q, st);
    if (!e) e = peer_wait(c, q, st);
    return e;
}

// ------------------------------------------------------------- ABI
extern "C" sts_status sts_nccl_unique_id(void* out128)
{
    sts_ctx* ctx = nullptr;
    if (!out128) return fail(ctx, STS_E_ARG, "null id buffer");
    if (!g_nccl.load()) return fail(ctx, STS_E_COMM, "libnccl.so.2 not loadable");
    nccl_uid id;
    if (g_nccl.GetUniqueId(&id)) return fail(ctx, STS_E_COMM, "ncclGetUniqueId failed");
    memcpy(out128, &id, 128);
    return STS_OK;
}

// Host-only planning, no CUDA call: geometry validation and snapping to
// integer cells, the slab decomposition along x, the slab-local solid map and the
// local cell / u-face / v-face kind maps of this rank (DESIGN 3.5, 7).
// Used by sts_create and by sts_plan (the CPU-testable decomposition).
static sts_status plan_host(const sts_grid* grid, const sts_square* squares, int32_t n_squares, const sts_gas* gas,
                            int world, int rank, sts_ctx* ctx)
{
    if (!(grid->spacing > 0) || !(grid->length_x > 0) || !(grid->length_y > 0)) return fail(nullptr, STS_E_CONFIG, "non-positive grid");
    double fx = grid->length_x / grid->spacing, fy = grid->length_y / grid->spacing;
    int nx = (int)llround(fx), ny = (int)llround(fy);
    if (std::fabs(fx - nx) > 1e-9 || std::fabs(fy - ny) > 1e-9 || nx < 1 || ny < 1)
        return fail(nullptr, STS_E_CONFIG, "channel lengths are not multiples of the spacing");
    if (!(gas->Kn > 0)) return fail(nullptr, STS_E_CONFIG, "Kn must be > 0");
    if (gas->pw_form < PW_DPDT || gas->pw_form > PW_GAMMA) return fail(nullptr, STS_E_CONFIG, "bad pw_form");
    if (gas->xbc != STS_X_INFLOW_OUTFLOW && gas->xbc != STS_X_PERIODIC) return fail(nullptr, STS_E_ARG, "bad xbc");
    if (!(gas->p_in > 0) || !(gas->T_in > 0)) return fail(nullptr, STS_E_CONFIG, "inflow state must be positive");
    if (world < 1 || rank < 0 || rank >= world) return fail(nullptr, STS_E_ARG, "bad rank/world");
    for (int s = 0; s < n_squares; s++) {
        const sts_square& q = squares[s];
        if (q.ni < 1 || q.nj < 1 || q.i0 < 0 || q.j0 < 0 || q.i0 + q.ni > nx || q.j0 + q.nj > ny)
            return fail(nullptr, STS_E_CONFIG, "square outside the channel");
        if (gas->xbc == STS_X_INFLOW_OUTFLOW && (q.i0 < 1 || q.i0 + q.ni > nx - 1))
            return fail(nullptr, STS_E_CONFIG, "square must leave a fluid column at the inlet and outlet");
    }
    ctx->nx = nx; ctx->ny = ny; ctx->spacing = grid->spacing;
    ctx->gas = *gas;
    ctx->squares.assign(squares, squares + n_squares);
    ctx->rank = rank; ctx->world = world;
    // slab decomposition along x: near-equal, remainder to the low ranks
    ctx->col_start.resize(world + 1);
    for (int r = 0, acc = 0; r <= world; r++) {
        ctx->col_start[r] = acc;
        if (r < world) acc += nx / world + (r < nx % world ? 1 : 0);
    }
    ctx->gi0 = ctx->col_start[rank];
    ctx->nloc = ctx->col_start[rank + 1] - ctx->gi0;
    if (world > 1 && ctx->nloc < OFF) return fail(nullptr, STS_E_CONFIG, "slab narrower than the halo");
    ctx->pitch = ((ctx->nloc + 2 * OFF + 1) + 15) / 16 * 16;
    if ((int64_t)ctx->pitch * (ny + 1) >= (int64_t)INT32_MAX)
        return fail(nullptr, STS_E_CONFIG, "slab too large for 32-bit element indices (use more ranks)");
    // slab-local solid map: every square intersected with the covered columns
    // (periodic: with the copies shifted by -nx, 0, +nx)
    ctx->sol_lo = ctx->gi0 - OFF - SOL_M;
    ctx->sol_w = ctx->pitch + 2 * SOL_M;
    ctx->h_solid.assign((size_t)ctx->sol_w * ny, 0);
    std::vector<uint8_t>& solid = ctx->h_solid;
    for (int s = 0; s < n_squares; s++) {
        const sts_square& q = squares[s];
        const bool per = gas->xbc == STS_X_PERIODIC;
        const int sh0 = per ? (int)std::floor((double)ctx->sol_lo / nx) - 1 : 0;
        const int sh1 = per ? (ctx->sol_lo + ctx->sol_w) / nx + 1 : 0;
        for (int sh = sh0; sh <= sh1; sh++) {
            const int a = std::max(q.i0 + sh * nx, ctx->sol_lo), b = std::min(q.i0 + q.ni + sh * nx, ctx->sol_lo + ctx->sol_w);
            for (int j = q.j0; j < q.j0 + q.nj; j++)
                for (int i = a; i < b; i++) solid[(size_t)j * ctx->sol_w + (i - ctx->sol_lo)] = 1;
        }
    }
    // kind maps of the stored local columns [gi0-OFF, gi0-OFF+pitch)
    const size_t nce = (size_t)ctx->pitch * ny, nve = (size_t)ctx->pitch * (ny + 1);
    ctx->h_ck.assign(nce, CK_WALLY); ctx->h_uk.assign(nce, FK_NONE); ctx->h_vk.assign(nve, FK_NONE);
    for (int j = 0; j < ny; j++)
        for (int li = 0; li < ctx->pitch; li++) {
            int gi = ctx->gi0 - OFF + li;
            ctx->h_ck[(size_t)j * ctx->pitch + li] = cell_kind_g(ctx, gi, j, solid);
            ctx->h_uk[(size_t)j * ctx->pitch + li] = u_kind_g(ctx, gi, j, solid);
        }
    for (int j = 0; j <= ny; j++)
        for (int li = 0; li < ctx->pitch; li++)
            ctx->h_vk[(size_t)j * ctx->pitch + li] = v_kind_g(ctx, ctx->gi0 - OFF + li, j, solid);
    return STS_OK;
}

extern "C" sts_status sts_plan(const sts_grid* grid, const sts_square* squares, int32_t n_squares,
                               const sts_gas* gas, int32_t world, int32_t rank, sts_plan_info* out,
                               uint8_t* kinds)
{
    if (!grid || !gas || !out || (n_squares > 0 && !squares)) return fail(nullptr, STS_E_ARG, "null argument");
    sts_ctx c;
    sts_status st = plan_host(grid, squares, n_squares, gas, world, rank, &c);
    if (st != STS_OK) return st;
    const bool per = gas->xbc == STS_X_PERIODIC;
    out->nx = c.nx; out->ny = c.ny;
    out->i0 = c.gi0; out->i1 = c.gi0 + c.nloc;
    out->pitch = c.pitch; out->ghost = OFF;
    out->left = rank > 0 ? rank - 1 : (per && world > 1 ? world - 1 : -1);
    out->right = rank < world - 1 ? rank + 1 : (per && world > 1 ? 0 : -1);
    // first / last OFF owned columns go to the left / right neighbour; the ghost
    // columns [i0-OFF, i0) and [i1, i1+OFF) (unwrapped) come from them
    out->send_left[0] = out->i0; out->send_left[1] = out->i0 + OFF;
    out->send_right[0] = out->i1 - OFF; out->send_right[1] = out->i1;
    out->recv_left[0] = out->i0 - OFF; out->recv_left[1] = out->i0;
    out->recv_right[0] = out->i1; out->recv_right[1] = out->i1 + OFF;
    if (kinds) {
        const size_t nve = (size_t)c.pitch * (c.ny + 1);
        for (size_t e = 0; e < nve; e++) {
            kinds[e] = e < c.h_ck.size() ? c.h_ck[e] : (uint8_t)CK_WALLY;
            kinds[nve + e] = e < c.h_uk.size() ? c.h_uk[e] : (uint8_t)FK_NONE;
            kinds[2 * nve + e] = c.h_vk[e];
        }
    }
    return STS_OK;
}

extern "C" sts_status sts_create(const sts_grid* grid, const sts_square* squares, int32_t n_squares,
                                 const sts_gas* gas, const sts_scheme* scheme, const sts_dist* dist,
                                 sts_ctx** out)
{
    sts_ctx* ctx = nullptr;
    if (!grid || !gas || !scheme || !out || (n_squares > 0 && !squares)) return fail(ctx, STS_E_ARG, "null argument");
    *out = nullptr;
    if ((scheme->time != STS_EXPLICIT && scheme->time != STS_IMPLICIT) || (scheme->space != STS_UPWIND && scheme->space != STS_TVD_VANLEER))
        return fail(ctx, STS_E_ARG, "bad scheme enum");
    if (!(scheme->dt > 0) || scheme->max_passes < 1 || scheme->min_passes < 0) return fail(ctx, STS_E_CONFIG, "bad dt / passes");
    const int world = dist ? dist->world : 1, rank = dist ? dist->rank : 0;
    if (scheme->loop3 < 0 || scheme->reserved != 0 || (scheme->loop3 > 1 && world > 1))
        return fail(ctx, STS_E_CONFIG, "loop3 must be >= 0, and > 1 only on a single-rank context");
    ctx = new sts_ctx();
    {
        sts_status st0 = plan_host(grid, squares, n_squares, gas, world, rank, ctx);
        if (st0 != STS_OK) { delete ctx; return st0; }
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) { delete ctx; return fail(nullptr, STS_E_CUDA, "no CUDA device"); }
    const int nx = ctx->nx, ny = ctx->ny;
    const std::vector<uint8_t>& solid = ctx->h_solid;
    ctx->sch = *scheme;
    ctx->device = dist ? dist->device : 0;
    if (ctx->device < 0 || ctx->device >= ndev) { delete ctx; return fail(nullptr, STS_E_ARG, "bad device"); }
    if (cudaSetDevice(ctx->device) != cudaSuccess) { delete ctx; return fail(nullptr, STS_E_CUDA, "cudaSetDevice"); }
    // Eq. pl37; u_in = M sqrt(gamma T_in / 2) (V0 = sqrt(2 R T0))
    ctx->A = 0.5;
    ctx->B = 5.0 * std::sqrt(M_PI) / 16.0 * gas->Kn;
    ctx->CT1 = gas->Kn * std::sqrt(M_PI * 225.0 / 1024.0);
    ctx->CT2 = std::sqrt(M_PI) / 4.0 * gas->Kn;
    ctx->CT3 = 2.0 / 5.0;
    ctx->u_in = gas->mach * std::sqrt(gas->gamma / 2.0 * gas->T_in);
    ctx->u_wb = gas->particle_frame ? ctx->u_in : gas->u_wall_bottom;   // R14
    ctx->u_wt = gas->particle_frame ? ctx->u_in : gas->u_wall_top;

    sts_status st = set_smem_attrs(ctx);
    if (st != STS_OK) { sts_destroy(ctx); return st; }
    {
        int lo = 0, hi = 0;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess ||
            cudaStreamCreateWithPriority(&ctx->gstream, cudaStreamNonBlocking, hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess) {
            sts_destroy(ctx);
            return fail(nullptr, STS_E_CUDA, "stream / event creation failed");
        }
    }
    size_t nce = cell_elems(ctx), nve = v_elems(ctx);

    auto alloc = [&](double** p, size_t n) -> sts_status {
        CU(cudaMalloc(p, n * sizeof(double)));
        CU(cudaMemset(*p, 0, n * sizeof(double)));
        return STS_OK;
    };
#define ALLOC(p, n) do { sts_status s_ = alloc(&(p), (n)); if (s_ != STS_OK) { sts_destroy(ctx); return s_; } } while (0)
    for (int k = 0; k < 3; k++) {
        ALLOC(ctx->snap[k].u, nce); ALLOC(ctx->snap[k].v, nve); ALLOC(ctx->snap[k].p, nce); ALLOC(ctx->snap[k].T, nce);
    }
    ALLOC(ctx->ue, nce); ALLOC(ctx->ve, nve); ALLOC(ctx->Te, nce);
    if (scheme->loop3 > 1) {                  // loop 3 (N3): sweep iterates and junk targets
        for (int q = 0; q < 2; q++) { ALLOC(ctx->l3p[q], nce); ALLOC(ctx->l3T[q], nce); }
        ALLOC(ctx->l3junk, nve);
        if (cudaMalloc(&ctx->l3red, 10 * sizeof(unsigned long long)) != cudaSuccess) {
            sts_destroy(ctx);
            return fail(nullptr, STS_E_OOM, "device allocation failed");
        }
    }
    ctx->stage_elems = (size_t)ctx->nloc * ny;          // slab-shaped scratch (rho read-back)
    ALLOC(ctx->stage, ctx->stage_elems);
    if (world > 1 || (dist && dist->nccl_id && gas->xbc == STS_X_PERIODIC)) {
        ctx->halo_elems = (size_t)16 * OFF * (ny + 1);
        ALLOC(ctx->halo, ctx->halo_elems);
    }
#undef ALLOC
    if (cudaMalloc(&ctx->red, ((size_t)scheme->max_passes * 9 + 1) * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMallocHost(&ctx->h_red, 10 * sizeof(unsigned long long)) != cudaSuccess) {
        sts_destroy(ctx);
        return fail(nullptr, STS_E_OOM, "device allocation failed");
    }
    ctx->bad = ctx->red + (size_t)scheme->max_passes * 9;
    cudaMemset(ctx->bad, 0, sizeof(unsigned long long));
    {
        std::vector<uint32_t> packed(nve);
        for (size_t e = 0; e < nve; e++) {
            uint32_t ckv = e < nce ? ctx->h_ck[e] : (uint32_t)CK_WALLY;
            uint32_t ukv = e < nce ? ctx->h_uk[e] : (uint32_t)FK_NONE;
            packed[e] = ckv | (ukv << 8) | ((uint32_t)ctx->h_vk[e] << 16);
        }
        // "regular" bit (Fig. 9 split): every cell of the +-3 window is
        // FLUID (separable 7-wide minimum of the fluid mask, x then y)
        const int R = 3, W = ctx->pitch + 2 * R, H = ny + 2 * R;
        std::vector<uint8_t> fl((size_t)W * H), hx((size_t)ctx->pitch * H);
        for (int jj = 0; jj < H; jj++)
            for (int c = 0; c < W; c++)
                fl[(size_t)jj * W + c] = cell_kind_g(ctx, ctx->gi0 - OFF - R + c, jj - R, solid) == CK_FLUID;
        for (int jj = 0; jj < H; jj++)
            for (int li = 0; li < ctx->pitch; li++) {
                uint8_t a = 1;
                for (int d = 0; d <= 2 * R; d++) a &= fl[(size_t)jj * W + li + d];
                hx[(size_t)jj * ctx->pitch + li] = a;
            }
        for (int j = 0; j < ny; j++)
            for (int li = 0; li < ctx->pitch; li++) {
                uint8_t a = 1;
                for (int d = 0; d <= 2 * R; d++) a &= hx[(size_t)(j + d) * ctx->pitch + li];
                if (a) packed[(size_t)j * ctx->pitch + li] |= REG_BIT;
            }
        if (cudaMalloc(&ctx->kind32, nve * sizeof(uint32_t)) != cudaSuccess) { sts_destroy(ctx); return fail(nullptr, STS_E_OOM, "device allocation failed"); }
        cudaMemcpy(ctx->kind32, packed.data(), nve * sizeof(uint32_t), cudaMemcpyHostToDevice);
        choose_segments(ctx, packed);
    }
    if (world > 1 && !dist->nccl_id) {
        ctx->local_group = true;            // slabs of one process, driven by sts_advance_group
    } else if (world > 1 || (dist && dist->nccl_id && gas->xbc == STS_X_PERIODIC)) {
        // NCCL transport; a single periodic rank given an id exchanges its wrapped
        // halo with itself over ncclSend/ncclRecv (exercises the transport on 1 GPU)
        if (!g_nccl.load()) { sts_destroy(ctx); return fail(nullptr, STS_E_COMM, "libnccl.so.2 not loadable"); }
        nccl_uid id;
        memcpy(&id, dist->nccl_id, 128);
        if (g_nccl.CommInitRank(&ctx->comm, world, id, rank)) { sts_destroy(ctx); return fail(nullptr, STS_E_COMM, "ncclCommInitRank failed"); }
    }
    ctx->stats.bad_cell = -1;
    st = sts_init_freestream(ctx);
    if (st != STS_OK) { sts_destroy(ctx); return st; }
    *out = ctx;
    return STS_OK;
}

extern "C" void sts_destroy(sts_ctx* ctx)
{
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    for (int k = 0; k < 3; k++) { cudaFree(ctx->snap[k].u); cudaFree(ctx->snap[k].v); cudaFree(ctx->snap[k].p); cudaFree(ctx->snap[k].T); }
    cudaFree(ctx->ue); cudaFree(ctx->ve); cudaFree(ctx->Te); cudaFree(ctx->stage); cudaFree(ctx->halo);
    cudaFree(ctx->kind32); cudaFree(ctx->cta_order); cudaFree(ctx->cta_split); cudaFree(ctx->red);
    cudaFree(ctx->dxl); cudaFree(ctx->dyp);
    for (void* p : ctx->ipc_mapped) cudaIpcCloseMemHandle(p);
    cudaFree(ctx->flags); cudaFree(ctx->red_all); cudaFree(ctx->d_peer_red);
    for (int q = 0; q < 2; q++) { cudaFree(ctx->l3p[q]); cudaFree(ctx->l3T[q]); }
    cudaFree(ctx->l3junk); cudaFree(ctx->l3red);
    if (ctx->h_red) cudaFreeHost(ctx->h_red);
    for (cudaGraphExec_t& g : ctx->tol_exec) if (g) cudaGraphExecDestroy(g);
    for (cudaGraphExec_t& g : ctx->fix_exec) if (g) cudaGraphExecDestroy(g);
    if (ctx->h_badstep) cudaFreeHost(ctx->h_badstep);
    cudaFree(ctx->red2); cudaFree(ctx->d_ls);
    for (int d = 0; d < 2; d++)
        for (sts_ctx::IoSlot& q : d ? ctx->io_out : ctx->io_in) {
            cudaFree(q.d);
            if (q.copied) cudaEventDestroy(q.copied);
            if (q.consumed) cudaEventDestroy(q.consumed);
        }
    if (ctx->io_h2d) cudaStreamDestroy(ctx->io_h2d);
    if (ctx->io_d2h) cudaStreamDestroy(ctx->io_d2h);
    if (ctx->h_ls) cudaFreeHost(ctx->h_ls);
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : {ctx->ev_a[0], ctx->ev_a[1], ctx->ev_b, ctx->ev_s, ctx->ev_h}) if (e) cudaEventDestroy(e);
    if (ctx->hstream) cudaStreamDestroy(ctx->hstream);
    if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
    for (cudaEvent_t e : {ctx->ev_fork, ctx->ev_join}) if (e) cudaEventDestroy(e);
    if (ctx->comm) g_nccl.CommDestroy(ctx->comm);
    delete ctx;
}

extern "C" sts_status sts_set_stream(sts_ctx* ctx, void* s)
{
    if (!ctx) return fail(ctx, STS_E_ARG, "null ctx");
    ctx->stream = (cudaStream_t)s;
    return STS_OK;
}


static double* field_ptr(const Snapshot& s, int field)
{
    return field == STS_U ? s.u : field == STS_V ? s.v : field == STS_P ? s.p : s.T;
}
static double inlet_value(const sts_ctx* c, int field)
{
    return field == STS_U ? c->u_in : field == STS_V ? 0.0 : field == STS_P ? c->gas.p_in : c->gas.T_in;
}
// Owned-part shape of a field on this rank (sts_shape): the last rank also
// returns u-face nx (the outlet face; periodic: the copy of face 0).
static void owned_shape(const sts_ctx* c, int field, int* rows, int* ncols)
{
    const bool last = c->rank == c->world - 1;
    *rows = (field == STS_V || field == STS_VEXP) ? c->ny + 1 : c->ny;
    *ncols = c->nloc + ((field == STS_U || field == STS_UEXP) && last ? 1 : 0);
}

// One field from a caller buffer (host or device; global shape, or this rank's
// owned slab) into the current snapshot: strided 2-D copies of the stored
// columns, ghost rules + fixed faces (finish_kernel), then device copies into
// the other two snapshots (solid cells and fixed faces must agree in every
// snapshot: they are never rewritten).  Slab-shaped input on a multi-rank
// context ends with one halo exchange (every rank calls it, collectively).
static sts_status set_field_any(sts_ctx* ctx, int field, const double* src, int64_t n)
{
    NvtxRange nv("sts_set_field");
    if (!ctx || !src) return fail(ctx, STS_E_ARG, "null argument");
    if (field < STS_U || field > STS_T) return fail(ctx, STS_E_ARG, "field not settable");
    CU(cudaSetDevice(ctx->device));
    const int rows = field == STS_V ? ctx->ny + 1 : ctx->ny;
    const int gw = field == STS_U ? ctx->nx + 1 : ctx->nx;
    int orows, ncols;
    owned_shape(ctx, field, &orows, &ncols);
    const bool global = n == (int64_t)rows * gw;
    const bool slab = !global && n == (int64_t)orows * ncols;
    if (!global && !slab) return fail(ctx, STS_E_ARG, "wrong buffer size (neither global nor slab shape)");
    if (slab && ctx->local_group) return fail(ctx, STS_E_ARG, "in-process slab groups take global-shape fields");
    const bool per = is_periodic(ctx);
    double* dst = field_ptr(ctx->snap[ctx->cur], field);
    const size_t dp = (size_t)ctx->pitch * sizeof(double);
    FinishArgs f{ctx->nx, ctx->ny, ctx->gi0, ctx->nloc, ctx->pitch, ctx->gas.xbc, field, ctx->world == 1 ? 1 : 0,
                 0, 0, inlet_value(ctx, field), ctx->u_in};
    if (global) {
        // stored unwrapped columns [lo, lo + pitch), periodic: wrapped pieces
        const int lo = ctx->gi0 - OFF, hi = lo + ctx->pitch;
        if (per && ctx->world > 1) {
            for (int u = lo; u < hi;) {
                const int w = ((u % ctx->nx) + ctx->nx) % ctx->nx, len = std::min(hi - u, ctx->nx - w);
                CU(cudaMemcpy2DAsync(dst + (u - lo), dp, src + w, (size_t)gw * sizeof(double), (size_t)len * sizeof(double),
                                     rows, cudaMemcpyDefault, ctx->stream));
                u += len;
            }
        } else {
            const int a = std::max(lo, 0), b = std::min(hi, per ? ctx->nx : gw);
            if (b > a)
                CU(cudaMemcpy2DAsync(dst + (a - lo), dp, src + a, (size_t)gw * sizeof(double), (size_t)(b - a) * sizeof(double),
                                     rows, cudaMemcpyDefault, ctx->stream));
            f.fill_left = ctx->gi0 == 0 || per;
            f.fill_right = ctx->gi0 + ctx->nloc == ctx->nx || per;
        }
        if (per && ctx->world == 1) { f.fill_left = 1; f.fill_right = 1; }
    } else {
        CU(cudaMemcpy2DAsync(dst + OFF, dp, src, (size_t)ncols * sizeof(double), (size_t)ncols * sizeof(double), orows,
                             cudaMemcpyDefault, ctx->stream));
        f.fill_left = !per && ctx->gi0 == 0;
        f.fill_right = !per && ctx->gi0 + ctx->nloc == ctx->nx;
        if (per && ctx->world == 1) { f.fill_left = 1; f.fill_right = 1; }
    }
    finish_kernel<<<592, 256, 0, ctx->stream>>>(f, ctx->kind32, dst);
    ctx->launches++;
    CU(cudaGetLastError());
    for (int k = 0; k < 3; k++)
        if (k != ctx->cur)
            CU(cudaMemcpyAsync(field_ptr(ctx->snap[k], field), dst, (size_t)rows * dp, cudaMemcpyDeviceToDevice, ctx->stream));
    if (slab && ctx->world > 1 && (ctx->comm || ctx->peer)) {
        const int which = ctx->cur;
        sts_ctx* one[1] = {ctx};
        sts_status e = ctx->peer ? peer_exchange(ctx, which, ctx->stream) : exchange_group(one, 1, &which, ctx->stream);
        if (e) return e;
        for (int k = 0; k < 3; k++)        // the exchanged ghost columns into the other snapshots too
            if (k != ctx->cur)
                for (int f2 = 0; f2 < 4; f2++)
                    CU(cudaMemcpyAsync(field_ptr(ctx->snap[k], f2), field_ptr(ctx->snap[ctx->cur], f2),
                                       (size_t)(f2 == STS_V ? ctx->ny + 1 : ctx->ny) * dp, cudaMemcpyDeviceToDevice,
                                       ctx->stream));
    }
    return peer_fence(ctx);
}

extern "C" sts_status sts_set_field(sts_ctx* ctx, int32_t field, const double* host, int64_t n)
{
    sts_status st = set_field_any(ctx, field, host, n);
    if (st != STS_OK) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    return STS_OK;
}

extern "C" sts_status sts_set_field_device(sts_ctx* ctx, int32_t field, const double* dev, int64_t n)
{
    return set_field_any(ctx, field, dev, n);
}

extern "C" sts_status sts_init_freestream(sts_ctx* ctx)
{
    if (!ctx) return fail(ctx, STS_E_ARG, "null ctx");
    CU(cudaSetDevice(ctx->device));
    Snapshot* s = ctx->snap;
    freestream_kernel<<<592, 256, 0, ctx->stream>>>((long long)cell_elems(ctx), (long long)v_elems(ctx), ctx->kind32,
                                                   ctx->u_in, ctx->gas.p_in, ctx->gas.T_in, s[0].u, s[1].u, s[2].u,
                                                   s[0].v, s[1].v, s[2].v, s[0].p, s[1].p, s[2].p, s[0].T, s[1].T, s[2].T);
    ctx->launches++;
    CU(cudaGetLastError());
    CU(cudaMemsetAsync(ctx->ue, 0, cell_elems(ctx) * sizeof(double), ctx->stream));
    CU(cudaMemsetAsync(ctx->ve, 0, v_elems(ctx) * sizeof(double), ctx->stream));
    CU(cudaMemsetAsync(ctx->Te, 0, cell_elems(ctx) * sizeof(double), ctx->stream));
    sts_status e = peer_fence(ctx);
    if (e) return e;
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->cur = 0;
    return STS_OK;
}

// This rank's owned part of a field (sts_shape) into a caller buffer (host or
// device, compact rows x ncols), asynchronously on the context stream.
static sts_status get_field_any(sts_ctx* ctx, int field, double* dst, int64_t n)
{
    NvtxRange nv("sts_get_field");
    if (!ctx || !dst) return fail(ctx, STS_E_ARG, "null argument");
    CU(cudaSetDevice(ctx->device));
    int rows, ncols;
    owned_shape(ctx, field == STS_RHO ? STS_P : field, &rows, &ncols);
    if ((int64_t)rows * ncols != n) return fail(ctx, STS_E_ARG, "wrong buffer size");
    const Snapshot& s = ctx->snap[ctx->cur];
    const double* src;
    switch (field) {
    case STS_U: src = s.u; break;
    case STS_V: src = s.v; break;
    case STS_P: src = s.p; break;
    case STS_T: src = s.T; break;
    case STS_UEXP: src = ctx->ue; break;
    case STS_VEXP: src = ctx->ve; break;
    case STS_TEXP: src = ctx->Te; break;
    case STS_RHO:
        ratio_kernel<<<592, 256, 0, ctx->stream>>>(rows, ncols, ctx->pitch, s.p, s.T, ctx->stage);
        ctx->launches++;
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(dst, ctx->stage, (size_t)n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        return STS_OK;
    default: return fail(ctx, STS_E_ARG, "bad field");
    }
    CU(cudaMemcpy2DAsync(dst, (size_t)ncols * sizeof(double), src + OFF, (size_t)ctx->pitch * sizeof(double),
                         (size_t)ncols * sizeof(double), rows, cudaMemcpyDefault, ctx->stream));
    return STS_OK;
}

extern "C" sts_status sts_get_field(sts_ctx* ctx, int32_t field, double* host, int64_t n)
{
    sts_status st = get_field_any(ctx, field, host, n);
    if (st != STS_OK) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    return STS_OK;
}

extern "C" sts_status sts_get_field_device(sts_ctx* ctx, int32_t field, double* dev, int64_t n)
{
    return get_field_any(ctx, field, dev, n);
}

// ---- asynchronous host I/O: H2D / D2H on their own copy streams, overlapping the
// pass kernels of the context stream (and each other: the two directions of the
// host link are independent).  The staging slots are compact device buffers of the
// caller's shape; set / fetch run the same set_field_any / get_field_any as the
// synchronous calls, from / into the slot.
static sts_status io_slot(sts_ctx* ctx, sts_ctx::IoSlot& q, int64_t n)
{
    sts_ctx* const c = ctx;
    if (!c->io_h2d) {
        CU(cudaStreamCreateWithFlags(&c->io_h2d, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&c->io_d2h, cudaStreamNonBlocking));
    }
    if (!q.copied) {
        CU(cudaEventCreateWithFlags(&q.copied, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&q.consumed, cudaEventDisableTiming));
    }
    if (q.cap < n) {
        if (q.d) { CU(cudaStreamSynchronize(c->stream)); CU(cudaStreamSynchronize(c->io_h2d)); CU(cudaStreamSynchronize(c->io_d2h)); }
        cudaFree(q.d);
        q.d = nullptr;
        q.cap = 0;
        CU(cudaMalloc(&q.d, (size_t)n * sizeof(double)));
        q.cap = n;
    }
    return STS_OK;
}

extern "C" sts_status sts_stage_field(sts_ctx* ctx, int32_t field, const double* host, int64_t n)
{
    NvtxRange nv("sts_stage_field");
    if (!ctx || !host || n <= 0) return fail(ctx, STS_E_ARG, "null argument");
    if (field < STS_U || field > STS_T) return fail(ctx, STS_E_ARG, "field not settable");
    CU(cudaSetDevice(ctx->device));
    sts_ctx::IoSlot& q = ctx->io_in[field];
    sts_status st = io_slot(ctx, q, n);
    if (st) return st;
    CU(cudaStreamWaitEvent(ctx->io_h2d, q.consumed, 0));     // the previous set has read the slot
    CU(cudaMemcpyAsync(q.d, host, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, ctx->io_h2d));
    CU(cudaEventRecord(q.copied, ctx->io_h2d));
    q.n = n;
    q.pending = true;
    return STS_OK;
}

extern "C" sts_status sts_set_staged(sts_ctx* ctx, int32_t field)
{
    if (!ctx) return fail(ctx, STS_E_ARG, "null ctx");
    if (field < STS_U || field > STS_T) return fail(ctx, STS_E_ARG, "field not settable");
    sts_ctx::IoSlot& q = ctx->io_in[field];
    if (!q.pending) return fail(ctx, STS_E_ARG, "no staged copy of this field");
    CU(cudaSetDevice(ctx->device));
    CU(cudaStreamWaitEvent(ctx->stream, q.copied, 0));
    sts_status st = set_field_any(ctx, field, q.d, q.n);
    if (st) return st;
    CU(cudaEventRecord(q.consumed, ctx->stream));
    q.pending = false;
    return STS_OK;
}

extern "C" sts_status sts_fetch_field(sts_ctx* ctx, int32_t field, double* host, int64_t n)
{
    NvtxRange nv("sts_fetch_field");
    if (!ctx || !host || n <= 0) return fail(ctx, STS_E_ARG, "null argument");
    if (field < STS_U || field > STS_T) return fail(ctx, STS_E_ARG, "field not fetchable asynchronously");
    CU(cudaSetDevice(ctx->device));
    sts_ctx::IoSlot& q = ctx->io_out[field];
    sts_status st = io_slot(ctx, q, n);
    if (st) return st;
    CU(cudaStreamWaitEvent(ctx->stream, q.copied, 0));       // the previous D2H has read the slot
    st = get_field_any(ctx, field, q.d, n);
    if (st) return st;
    CU(cudaEventRecord(q.consumed, ctx->stream));
    CU(cudaStreamWaitEvent(ctx->io_d2h, q.consumed, 0));
    CU(cudaMemcpyAsync(host, q.d, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, ctx->io_d2h));
    CU(cudaEventRecord(q.copied, ctx->io_d2h));
    q.pending = true;
    return STS_OK;
}

extern "C" sts_status sts_io_sync(sts_ctx* ctx)
{
    NvtxRange nv("sts_io_sync");
    if (!ctx) return fail(ctx, STS_E_ARG, "null ctx");
    CU(cudaSetDevice(ctx->device));
    if (ctx->io_h2d) CU(cudaStreamSynchronize(ctx->io_h2d));
    if (ctx->io_d2h) CU(cudaStreamSynchronize(ctx->io_d2h));
    for (sts_ctx::IoSlot& q : ctx->io_out) q.pending = false;
    return STS_OK;
}

extern "C" sts_status sts_get_map(sts_ctx* ctx, int32_t which, int32_t* host, int64_t n)
{
    if (!ctx || !host) return fail(ctx, STS_E_ARG, "null argument");
    if (which == 3) {
        if (n != 2 * ctx->world) return fail(ctx, STS_E_ARG, "wrong buffer size");
        for (int r = 0; r < ctx->world; r++) { host[2 * r] = ctx->col_start[r]; host[2 * r + 1] = ctx->col_start[r + 1]; }
        return STS_OK;
    }
    bool last = ctx->rank == ctx->world - 1;
    int rows = which == 2 ? ctx->ny + 1 : ctx->ny;
    int ncols = ctx->nloc + (which == 1 && last ? 1 : 0);
    if (which < 0 || which > 2) return fail(ctx, STS_E_ARG, "bad map");
    if ((int64_t)rows * ncols != n) return fail(ctx, STS_E_ARG, "wrong buffer size");
    const std::vector<uint8_t>& m = which == 0 ? ctx->h_ck : which == 1 ? ctx->h_uk : ctx->h_vk;
    for (int j = 0; j < rows; j++)
        for (int i = 0; i < ncols; i++) {
            uint8_t k = m[(size_t)j * ctx->pitch + OFF + i];
            host[(size_t)j * ncols + i] = which == 0 ? (k == CK_SOLID ? 1 : 0) : k;
        }
    return STS_OK;
}

extern "C" sts_status sts_shape(sts_ctx* ctx, int32_t field, int64_t* nx, int64_t* ny, int64_t* i0, int64_t* ni)
{
    if (!ctx || !nx || !ny || !i0 || !ni) return fail(ctx, STS_E_ARG, "null argument");
    bool last = ctx->rank == ctx->world - 1;
    *nx = ctx->nloc + ((field == STS_U || field == STS_UEXP) && last ? 1 : 0);
    *ny = (field == STS_V || field == STS_VEXP) ? ctx->ny + 1 : ctx->ny;
    *i0 = ctx->gi0;
    *ni = ctx->nloc;
    return STS_OK;
}

extern "C" sts_status sts_constants(sts_ctx* ctx, double* out)
{
    if (!ctx || !out) return fail(ctx, STS_E_ARG, "null argument");
    out[0] = ctx->A; out[1] = ctx->B; out[2] = ctx->CT1; out[3] = ctx->CT2; out[4] = ctx->CT3; out[5] = ctx->u_in; out[6] = ctx->sch.dt;
    return STS_OK;
}

// Non-uniform mesh (Fig. 5): per-column / per-row
// steps of the global mesh.  The stored local columns take the steps of the
// global columns they hold (periodic: wrapped; inflow / outflow ghosts: the
// boundary column's, like their state), rows beyond a wall the wall row's.
extern "C" sts_status sts_set_mesh(sts_ctx* ctx, const double* dx, int64_t nx, const double* dy, int64_t ny)
{
    if (!ctx) return fail(ctx, STS_E_ARG, "null ctx");
    if ((dx && nx != ctx->nx) || (dy && ny != ctx->ny)) return fail(ctx, STS_E_ARG, "wrong mesh array size");
    if (ctx->sch.loop3 > 1) return fail(ctx, STS_E_CONFIG, "loop 3 (loop3 > 1) runs on uniform meshes");
    if (dx) for (int64_t i = 0; i < nx; i++) if (!(dx[i] > 0.0) || !std::isfinite(dx[i])) return fail(ctx, STS_E_CONFIG, "mesh step <= 0");
    if (dy) for (int64_t j = 0; j < ny; j++) if (!(dy[j] > 0.0) || !std::isfinite(dy[j])) return fail(ctx, STS_E_CONFIG, "mesh step <= 0");
    CU(cudaSetDevice(ctx->device));
    CU(cudaStreamSynchronize(ctx->stream));
    std::vector<double> hx(ctx->pitch), hy(ctx->ny + 2 * PADY);
    for (int l = 0; l < ctx->pitch; l++) {
        int gi = ctx->gi0 - OFF + l;
        gi = is_periodic(ctx) ? ((gi % ctx->nx) + ctx->nx) % ctx->nx : std::min(std::max(gi, 0), ctx->nx - 1);
        hx[l] = dx ? dx[gi] : ctx->spacing;
    }
    for (int q = 0; q < ctx->ny + 2 * PADY; q++)
        hy[q] = dy ? dy[std::min(std::max(q - PADY, 0), ctx->ny - 1)] : ctx->spacing;
    if (!ctx->dxl && cudaMalloc(&ctx->dxl, hx.size() * sizeof(double)) != cudaSuccess) return fail(ctx, STS_E_OOM, "mesh");
    if (!ctx->dyp && cudaMalloc(&ctx->dyp, hy.size() * sizeof(double)) != cudaSuccess) return fail(ctx, STS_E_OOM, "mesh");
    CU(cudaMemcpy(ctx->dxl, hx.data(), hx.size() * sizeof(double), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->dyp, hy.data(), hy.size() * sizeof(double), cudaMemcpyHostToDevice));
    ctx->nu = dx || dy;
    // a new CTA schedule (the NU kernel has general instances only) and new graphs
    std::vector<uint32_t> packed((size_t)(ctx->ny + 1) * ctx->pitch);
    CU(cudaMemcpy(packed.data(), ctx->kind32, packed.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    choose_segments(ctx, packed);
    for (cudaGraphExec_t& g : ctx->tol_exec)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    for (cudaGraphExec_t& g : ctx->fix_exec)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    return STS_OK;
}

// ------------------------------------------------------------- fused-halo setup (N1)
// Opaque per-rank description for sts_peer_connect: the slab geometry and CUDA
// IPC handles of the three snapshots (u, v, p, T), the explicit planes, the flag
// words and the pushed residual slots.
struct PeerBlob {
    uint32_t magic, version;
    int32_t rank, world, nloc, pitch, gi0, ny, device, pad;
    cudaIpcMemHandle_t h[17];
};
static constexpr uint32_t PEER_MAGIC = 0x53545331u;   // "STS1"

static sts_status peer_alloc(sts_ctx* ctx)
{
    sts_ctx* const c = ctx;
    if (!memops_load()) return fail(c, STS_E_CUDA, "cuStreamWriteValue64 / cuStreamWaitValue64 unavailable");
    if (!c->flags) {
        CU(cudaMalloc(&c->flags, 2 * (size_t)c->world * sizeof(unsigned long long)));
        CU(cudaMemset(c->flags, 0, 2 * (size_t)c->world * sizeof(unsigned long long)));
    }
    if (!c->red_all) {
        CU(cudaMalloc(&c->red_all, 20 * sizeof(unsigned long long)));
        CU(cudaMemset(c->red_all, 0, 20 * sizeof(unsigned long long)));
    }
    return STS_OK;
}
static sts_status peer_finish(sts_ctx* ctx, const std::vector<unsigned long long*>& reds)
{
    sts_ctx* const c = ctx;
    CU(cudaMalloc(&c->d_peer_red, reds.size() * sizeof(unsigned long long*)));
    CU(cudaMemcpy(c->d_peer_red, reds.data(), reds.size() * sizeof(unsigned long long*), cudaMemcpyHostToDevice));
    c->peer = true;
    c->local_group = false;
    c->seq = c->rseq = 0;
    // the edge / interior split of every pass (edge strips first, ~15 % shorter)
    // needs a schedule with edge strips: choose_segments made it at creation
    return STS_OK;
}

extern "C" sts_status sts_peer_export(sts_ctx* ctx, void* blob, int64_t* nbytes)
{
    if (!ctx || !nbytes) return fail(ctx, STS_E_ARG, "null argument");
    if (!blob) { *nbytes = (int64_t)sizeof(PeerBlob); return STS_OK; }
    if (*nbytes < (int64_t)sizeof(PeerBlob)) return fail(ctx, STS_E_ARG, "blob buffer too small");
    if (ctx->world < 2) return fail(ctx, STS_E_ARG, "peer transport needs world >= 2");
    CU(cudaSetDevice(ctx->device));
    sts_status e = peer_alloc(ctx);
    if (e) return e;
    PeerBlob b{};
    b.magic = PEER_MAGIC; b.version = 1;
    b.rank = ctx->rank; b.world = ctx->world; b.nloc = ctx->nloc; b.pitch = ctx->pitch; b.gi0 = ctx->gi0;
    b.ny = ctx->ny; b.device = ctx->device;
    void* ptrs[17];
    for (int k = 0; k < 3; k++) { ptrs[4 * k] = ctx->snap[k].u; ptrs[4 * k + 1] = ctx->snap[k].v; ptrs[4 * k + 2] = ctx->snap[k].p; ptrs[4 * k + 3] = ctx->snap[k].T; }
    ptrs[12] = ctx->ue; ptrs[13] = ctx->ve; ptrs[14] = ctx->Te; ptrs[15] = ctx->flags; ptrs[16] = ctx->red_all;
    for (int q = 0; q < 17; q++) CU(cudaIpcGetMemHandle(&b.h[q], ptrs[q]));
    memcpy(blob, &b, sizeof b);
    *nbytes = (int64_t)sizeof b;
    return STS_OK;
}

extern "C" sts_status sts_peer_connect(sts_ctx* ctx, const void* blobs, int64_t nbytes_each)
{
    if (!ctx || !blobs) return fail(ctx, STS_E_ARG, "null argument");
    if (nbytes_each != (int64_t)sizeof(PeerBlob)) return fail(ctx, STS_E_ARG, "wrong blob size");
    if (ctx->world < 2 || ctx->comm) return fail(ctx, STS_E_ARG, "peer transport: world >= 2 and no NCCL communicator");
    CU(cudaSetDevice(ctx->device));
    sts_status e = peer_alloc(ctx);
    if (e) return e;
    std::vector<PeerBlob> bl(ctx->world);
    for (int q = 0; q < ctx->world; q++) {
        memcpy(&bl[q], (const char*)blobs + (size_t)q * sizeof(PeerBlob), sizeof(PeerBlob));
        if (bl[q].magic != PEER_MAGIC || bl[q].rank != q || bl[q].world != ctx->world || bl[q].ny != ctx->ny)
            return fail(ctx, STS_E_ARG, "peer blobs must be ranks 0..world-1 of this decomposition");
    }
    auto open = [&](const cudaIpcMemHandle_t& h, void** p) -> sts_status {
        cudaError_t err = cudaIpcOpenMemHandle(p, h, cudaIpcMemLazyEnablePeerAccess);
        if (err != cudaSuccess) return fail(ctx, STS_E_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(err));
        ctx->ipc_mapped.push_back(*p);
        return STS_OK;
    };
    ctx->peer_flags.assign(ctx->world, nullptr);
    std::vector<unsigned long long*> reds(ctx->world, nullptr);
    for (int q = 0; q < ctx->world; q++) {
        if (q == ctx->rank) { ctx->peer_flags[q] = ctx->flags; reds[q] = ctx->red_all; continue; }
        void* p = nullptr;
        if ((e = open(bl[q].h[15], &p))) return e;
        ctx->peer_flags[q] = (unsigned long long*)p;
        if ((e = open(bl[q].h[16], &p))) return e;
        reds[q] = (unsigned long long*)p;
    }
    for (int sd = 0; sd < 2; sd++) {
        const int nb = sd == 0 ? left_of(ctx) : right_of(ctx);
        if (nb < 0) continue;
        if (nb == ctx->rank) return fail(ctx, STS_E_ARG, "a rank cannot be its own neighbour");
        // the neighbour's element of my local column l: l + shift (DESIGN 7)
        ctx->nb_pitch[sd] = bl[nb].pitch;
        ctx->nb_shift[sd] = sd == 0 ? bl[nb].nloc : -ctx->nloc;
        if (sd == 1 && nb == left_of(ctx)) {       // 2-rank ring: both sides are the same rank
            ctx->nb_snap[1][0] = ctx->nb_snap[0][0]; ctx->nb_snap[1][1] = ctx->nb_snap[0][1]; ctx->nb_snap[1][2] = ctx->nb_snap[0][2];
            for (int f = 0; f < 3; f++) ctx->nb_pl[1][f] = ctx->nb_pl[0][f];
            continue;
        }
        void* p[15];
        for (int q = 0; q < 15; q++) if ((e = open(bl[nb].h[q], &p[q]))) return e;
        for (int k = 0; k < 3; k++)
            ctx->nb_snap[sd][k] = Snapshot{(double*)p[4 * k], (double*)p[4 * k + 1], (double*)p[4 * k + 2], (double*)p[4 * k + 3]};
        for (int f = 0; f < 3; f++) ctx->nb_pl[sd][f] = (double*)p[12 + f];
    }
    return peer_finish(ctx, reds);
}

extern "C" sts_status sts_peer_connect_group(sts_ctx** ctxs, int32_t n)
{
    sts_ctx* ctx = nullptr;
    if (!ctxs || n < 2) return fail(ctx, STS_E_ARG, "bad argument");
    for (int r = 0; r < n; r++)
        if (!ctxs[r] || ctxs[r]->world != n || ctxs[r]->rank != r || !ctxs[r]->local_group || ctxs[r]->device != ctxs[0]->device)
            return fail(ctxs[r], STS_E_ARG, "group must be ranks 0..n-1 of one in-process decomposition on one device");
    CU(cudaSetDevice(ctxs[0]->device));
    for (int r = 0; r < n; r++) { sts_status e = peer_alloc(ctxs[r]); if (e) return e; }
    std::vector<unsigned long long*> reds(n), flags(n);
    for (int r = 0; r < n; r++) { reds[r] = ctxs[r]->red_all; flags[r] = ctxs[r]->flags; }
    for (int r = 0; r < n; r++) {
        sts_ctx* c = ctxs[r];
        c->peer_flags = flags;
        for (int sd = 0; sd < 2; sd++) {
            const int nb = sd == 0 ? left_of(c) : right_of(c);
            if (nb < 0) continue;
            c->nb_pitch[sd] = ctxs[nb]->pitch;
            c->nb_shift[sd] = sd == 0 ? ctxs[nb]->nloc : -c->nloc;
            for (int k = 0; k < 3; k++) c->nb_snap[sd][k] = ctxs[nb]->snap[k];
            c->nb_pl[sd][0] = ctxs[nb]->ue; c->nb_pl[sd][1] = ctxs[nb]->ve; c->nb_pl[sd][2] = ctxs[nb]->Te;
        }
        sts_status e = peer_finish(c, reds);
        if (e) return e;
        c->local_group = true;                      // still driven by sts_advance_group
    }
    return STS_OK;
}

extern "C" sts_status sts_profile(sts_ctx* ctx, int32_t enable)
{
    if (!ctx) return fail(ctx, STS_E_ARG, "null ctx");
    ctx->profiling = enable != 0;
    return STS_OK;
}

extern "C" sts_status sts_profile_read(sts_ctx* ctx, double* out, int32_t reset)
{
    if (!ctx || !out) return fail(ctx, STS_E_ARG, "null argument");
    CU(cudaSetDevice(ctx->device));
    prof_collect(ctx);
    out[0] = ctx->prof_pass_n; out[1] = ctx->prof_pass_ms; out[2] = ctx->prof_conv_n; out[3] = ctx->prof_conv_ms; out[4] = ctx->launches;
    if (reset) ctx->prof_pass_n = ctx->prof_pass_ms = ctx->prof_conv_n = ctx->prof_conv_ms = ctx->launches = 0;
    return STS_OK;
}

// residual slots + sticky bad key -> stats (reading R35); returns STS_E_STATE
// on a bad state (the first one of the advance call: pass, cell, field)
static sts_status finish_residuals(sts_ctx* ctx, const unsigned long long* r, unsigned long long key)
{
    double v[7];
    for (int q = 0; q < 7; q++) { long long b = (long long)r[q]; memcpy(&v[q], &b, 8); }
    double vel = v[4], pm = v[5], Tm = v[6];
    ctx->stats.res[0] = vel > 0 ? v[0] / vel : v[0];
    ctx->stats.res[1] = vel > 0 ? v[1] / vel : v[1];
    ctx->stats.res[2] = pm > 0 ? v[2] / pm : v[2];
    ctx->stats.res[3] = Tm > 0 ? v[3] / Tm : v[3];
    bool bad = key != 0;
    for (int q = 0; q < 7; q++) if (!(v[q] == v[q]) || std::isinf(v[q])) bad = true;
    if (bad) {
        ctx->stats.bad_cell = -1;
        ctx->stats.bad_field = STS_U;
        ctx->stats.bad_pass = -1;
        if (key) {
            const long long flat = (long long)(((1ULL << 42) - 1) - ((key >> 2) & ((1ULL << 42) - 1)));
            ctx->stats.bad_cell = flat == BAD_NOCELL ? -1 : flat;
            ctx->stats.bad_field = (int)(key & 3);
            ctx->stats.bad_pass = ctx->pass0 + (0xFFFFF - (long long)(key >> 44));
        }
        return fail(ctx, STS_E_STATE, "non-finite or non-positive state (see sts_stats.bad_cell)");
    }
    return STS_OK;
}

// Max-combine the residual slots of a pass over all slabs: NCCL MAX allreduce
// on the u64 bit patterns (order-independent, exact) or, in-process, on the host.
static sts_status gather_red(sts_ctx** cs, int n, int it, unsigned long long* out, cudaStream_t st)
{
    sts_ctx* ctx = cs[0];
    for (int q = 0; q < 10; q++) out[q] = 0;
    if (n == 1 && ctx->peer) {
        // fused path (N1): push my maxima into every rank's slots (system-scope
        // atomicMax over peer memory), signal every rank, wait for every rank's
        // push, read my slots; slots alternate by parity, zeroed after reading
        const int par = (int)(ctx->rseq & 1);
        const unsigned long long q = ++ctx->rseq;
        red_push_kernel<<<1, 32, 0, st>>>(ctx->red + (size_t)it * 9, ctx->bad, ctx->d_peer_red, ctx->world, par);
        ctx->launches++;
        CU(cudaGetLastError());
        for (int r = 0; r < ctx->world; r++) { sts_status e = peer_signal_rank(ctx, r, ctx->world, q, st); if (e) return e; }
        for (int r = 0; r < ctx->world; r++) { sts_status e = peer_wait_rank(ctx, r, ctx->world, q, st); if (e) return e; }
        CU(cudaMemcpyAsync(ctx->h_red, ctx->red_all + 10 * par, 10 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CU(cudaMemsetAsync(ctx->red_all + 10 * par, 0, 10 * sizeof(unsigned long long), st));
        CU(cudaStreamSynchronize(st));
        for (int q2 = 0; q2 < 10; q2++) out[q2] = ctx->h_red[q2];
        return STS_OK;
    }
    if (n == 1 && ctx->comm) {
        unsigned long long* slot = ctx->red + (size_t)it * 9;
        if (g_nccl.AllReduce(slot, slot, 9, NCCL_UINT64, NCCL_MAX, ctx->comm, st)) return fail(ctx, STS_E_COMM, "ncclAllReduce");
        if (g_nccl.AllReduce(ctx->bad, ctx->bad, 1, NCCL_UINT64, NCCL_MAX, ctx->comm, st)) return fail(ctx, STS_E_COMM, "ncclAllReduce");
    }
    for (int r = 0; r < n; r++) {
        CU(cudaMemcpyAsync(cs[r]->h_red, cs[r]->red + (size_t)it * 9, 9 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(cs[r]->h_red + 9, cs[r]->bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    }
    CU(cudaStreamSynchronize(st));
    for (int r = 0; r < n; r++)
        for (int q = 0; q < 10; q++) out[q] = std::max(out[q], cs[r]->h_red[q]);
    return STS_OK;
}

// ------------------------------------------------------------- graph-driven loop 2
// Tolerance mode on one context without NCCL: the loop-2 convergence test runs
// on the device, so a whole time step is one CUDA graph launch and one 100-byte
// read-back, instead of a host round trip per pass (the paper reads the maximum
// residuals back after every pass).  Graph of snapshot rotation n1
// (a = n1+1, b = n1+2 mod 3):
//   zero slots + loop state; [explicit planes]; pass(n1 -> a); check;
//   WHILE(cond) { pass(a -> b); check; pass(b -> a); check }
// A pass that finds the loop finished returns at once (MarchParams.done), so the
// second pass of a body iteration is a no-op when the first one converged.  The
// check applies exactly the host's test (finish_residuals + the tol comparison,
// same fp64 operations), so both drivers take identical pass counts.
// The general CTAs of a pass (walls, squares, inlet / outlet strips: the long
// critical path of the schedule) run on a high-priority stream on the stream
// path; inside a graph the same priority is a kernel-node attribute.
static cudaError_t graph_node_high_priority(cudaGraphNode_t node)
{
    int lo = 0, hi = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (e != cudaSuccess) return e;
    cudaKernelNodeAttrValue v = {};
    v.priority = hi;
    return cudaGraphKernelNodeSetAttribute(node, cudaKernelNodeAttributePriority, &v);
}

struct LoopState {
    int passes, done, conv, checked;
    unsigned long long red[9];   // residual slots of the last checked pass
    unsigned long long bad;      // sticky bad-state key (the march kernels' MarchParams.bad)
};

// A pass's kernel node; with `programmatic` every edge from the previous pass's
// node(s) is a programmatic (PDL) edge: the node's CTAs may launch once every CTA of
// the previous pass has started, and each waits in griddepcontrol.wait (first
// statement of the march kernels) for the previous pass to complete.
static cudaError_t add_pass_node(cudaGraphNode_t* node, cudaGraph_t g, const std::vector<cudaGraphNode_t>& deps,
                                 const cudaKernelNodeParams& kp, bool programmatic)
{
    if (!programmatic || deps.empty()) return cudaGraphAddKernelNode(node, g, deps.data(), deps.size(), &kp);
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeKernel;
    np.kernel.func = kp.func;
    np.kernel.gridDim = kp.gridDim;
    np.kernel.blockDim = kp.blockDim;
    np.kernel.sharedMemBytes = kp.sharedMemBytes;
    np.kernel.kernelParams = kp.kernelParams;
    std::vector<cudaGraphEdgeData> ed(deps.size());
    for (cudaGraphEdgeData& x : ed) {
        x = cudaGraphEdgeData{};
        x.from_port = cudaGraphKernelNodePortProgrammatic;
        x.type = cudaGraphDependencyTypeProgrammatic;
    }
    return cudaGraphAddNode_v2(node, g, deps.data(), ed.data(), deps.size(), &np);
}
__global__ void loop_check_kernel(unsigned long long* slot, LoopState* ls, cudaGraphConditionalHandle h,
                                  int min_passes, int max_passes, double tol)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");      // PDL (tolerance graphs): after the pass
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x != 0) return;
    if (ls->done) { cudaGraphSetConditional(h, 0); return; }
    const int passes = ls->passes + 1;
    ls->passes = passes;
    bool done = passes >= max_passes;
    const bool bad_state = *(volatile unsigned long long*)&ls->bad != 0;
    if (passes >= min_passes || bad_state) {
        double v[7];
        bool bad = bad_state;
        for (int q = 0; q < 7; q++) {
            v[q] = __longlong_as_double((long long)slot[q]);
            if (!(v[q] == v[q]) || isinf(v[q])) bad = true;
        }
        for (int q = 0; q < 9; q++) ls->red[q] = slot[q];
        ls->checked = 1;
        const double vel = v[4], pm = v[5], Tm = v[6];
        const double r0 = vel > 0 ? v[0] / vel : v[0], r1 = vel > 0 ? v[1] / vel : v[1];
        const double r2 = pm > 0 ? v[2] / pm : v[2], r3 = Tm > 0 ? v[3] / Tm : v[3];
        if (bad) done = true;
        else if (r0 < tol && r1 < tol && r2 < tol && r3 < tol) { ls->conv = 1; done = true; }
    }
    for (int q = 0; q < 9; q++) slot[q] = 0;   // re-armed for the pass two later
    ls->done = done ? 1 : 0;
    cudaGraphSetConditional(h, done ? 0u : 1u);
}

static bool tol_graph_ok(const sts_ctx* c)
{
    return c->sch.tol > 0 && c->world == 1 && !c->comm && !c->profiling && c->sch.loop3 <= 1 && !getenv("STS_NO_GRAPH");
}

#define CG(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    /* the body capture first: its graph belongs to the outer one */ \
    if (cap2) { cudaGraph_t g_ = nullptr; cudaStreamEndCapture(cap2, &g_); cudaStreamDestroy(cap2); } \
    if (cap) { cudaGraph_t g_ = nullptr; cudaStreamEndCapture(cap, &g_); if (g_) cudaGraphDestroy(g_); cudaStreamDestroy(cap); } \
    return fail(c, STS_E_CUDA, std::string("graph build: ") + cudaGetErrorString(e_)); } } while (0)

// the convergence check after a pass; `pdl`: a programmatic edge from the pass
static cudaError_t launch_check(cudaStream_t s, unsigned long long* slot, LoopState* ls, cudaGraphConditionalHandle h,
                                int mn, int mx, double tol, bool pdl)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, loop_check_kernel, slot, ls, h, mn, mx, tol);
}
// pdl: programmatic edges pass -> check -> pass inside the step (the first pass of
// the step and of the WHILE body keep full edges); the caller falls back to pdl =
// false when the driver rejects them
static sts_status build_tol_graph(sts_ctx* c, int n1, bool pdl)
{
    cudaStream_t cap = nullptr, cap2 = nullptr;
    const int impl = c->sch.time == STS_IMPLICIT, tvd = c->sch.space == STS_TVD_VANLEER;
    const int a = (n1 + 1) % 3, b = (n1 + 2) % 3;
    if (!c->red2) {
        CG(cudaMalloc(&c->red2, 18 * sizeof(unsigned long long)));
        CG(cudaMalloc(&c->d_ls, sizeof(LoopState)));
        CG(cudaMallocHost(&c->h_ls, sizeof(LoopState)));
    }
    CG(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    CG(cudaStreamCreateWithFlags(&cap2, cudaStreamNonBlocking));
    Params k = make_params(c);
    k.u_1 = c->snap[n1].u; k.v_1 = c->snap[n1].v; k.p_1 = c->snap[n1].p; k.T_1 = c->snap[n1].T;
    k.ue = c->ue; k.ve = c->ve; k.Te = c->Te;
    const dim3 mgrid(c->n_gen + c->n_reg);                 // the conv kernel: every CTA of the schedule
    const bool fuse = fuse_conv(c);
    auto pass = [&](int o, int w, int sl, cudaStream_t s, bool fz = false, bool pin = false) -> cudaError_t {
        Params q = k;
        if (fz) { q.ue_w = c->ue; q.ve_w = c->ve; q.Te_w = c->Te; }   // pass 1 computes the planes (N2)
        q.u_o = c->snap[o].u; q.v_o = c->snap[o].v; q.p_o = c->snap[o].p; q.T_o = c->snap[o].T;
        q.u_w = c->snap[w].u; q.v_w = c->snap[w].v; q.p_w = c->snap[w].p; q.T_w = c->snap[w].T;
        q.red = c->red2 + sl * 9;
        MarchParams m = make_march(c, q);
        m.done = &c->d_ls->done;
        m.bad = &c->d_ls->bad;
        // the general and the all-regular kernel as two parallel kernel nodes after
        // the capture's current dependencies (no cross-stream fork inside a
        // conditional body)
        cudaStreamCaptureStatus cs;
        cudaGraph_t g;
        const cudaGraphNode_t* dp = nullptr;
        size_t n = 0;
        cudaError_t e = cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &dp, &n);
        if (e != cudaSuccess) return e;
        std::vector<cudaGraphNode_t> deps(dp, dp + n);
        cudaGraphNode_t nodes[2];
        int nn = 0;
        if (use_fused(c, fz, false) && c->n_gen + c->n_reg > 0) {     // one node: general CTAs first
            MarchParams mp = m;
            mp.order = (const int4*)c->cta_order;
            void* args[] = {&mp};
            cudaKernelNodeParams kp = {};
            kp.func = (void*)fused_table(impl, tvd, 1);
            kp.gridDim = dim3(c->n_gen + c->n_reg);
            kp.blockDim = dim3(MX);
            kp.sharedMemBytes = march_smem(c);
            kp.kernelParams = args;
            e = add_pass_node(&nodes[nn], g, deps, kp, pdl && pin);
            if (e != cudaSuccess) return e;
            nn++;
            return cudaStreamUpdateCaptureDependencies(s, nodes, nn, cudaStreamSetCaptureDependencies);
        }
        for (int part = 0; part < 2; part++) {
            const int cnt = part == 0 ? c->n_gen : c->n_reg;
            if (cnt == 0) continue;
            MarchParams mp = m;
            mp.order = (const int4*)c->cta_order + (part ? c->n_gen : 0);
            void* args[] = {&mp};
            cudaKernelNodeParams kp = {};
            kp.func = fz ? (void*)march_fusec_table(tvd, part, 1) : (void*)march_graph_table(impl, tvd, part, part ? 0 : c->nu);
            kp.gridDim = dim3(cnt);
            kp.blockDim = dim3(MX);
            kp.sharedMemBytes = part ? regk_smem(c, fz, false) : (fz ? FUSEC_SMEM : march_smem(c));
            kp.kernelParams = args;
            e = add_pass_node(&nodes[nn], g, deps, kp, pdl && pin);
            if (e != cudaSuccess) return e;
            if (part == 0) e = graph_node_high_priority(nodes[nn]);   // general CTAs first, as on the stream path
            if (e != cudaSuccess) return e;
            nn++;
        }
        return cudaStreamUpdateCaptureDependencies(s, nodes, nn, cudaStreamSetCaptureDependencies);
    };
    const int mn = c->sch.min_passes, mx = c->sch.max_passes;
    const double tol = c->sch.tol;

    CG(cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed));
    cudaStreamCaptureStatus cst;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CG(cudaStreamGetCaptureInfo(cap, &cst, nullptr, &cg, &deps, &nd));
    cudaGraphConditionalHandle h;
    CG(cudaGraphConditionalHandleCreate(&h, cg, 1, cudaGraphCondAssignDefault));
    CG(cudaMemsetAsync(c->red2, 0, 18 * sizeof(unsigned long long), cap));
    CG(cudaMemsetAsync(c->d_ls, 0, sizeof(LoopState), cap));
    if (!impl && !fuse) {                         // a1: explicit planes of this step
        Params q = k;
        q.ue_w = c->ue; q.ve_w = c->ve; q.Te_w = c->Te;
        conv_march_table(tvd, c->nu)<<<mgrid, MX, conv_smem(c), cap>>>(make_march(c, q));
    }
    CG(pass(n1, a, 0, cap, fuse));
    CG(launch_check(cap, c->red2, c->d_ls, h, mn, mx, tol, pdl));
    CG(cudaStreamGetCaptureInfo(cap, &cst, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CG(cudaGraphAddNode(&cn, cg, deps, nd, &cp));
    CG(cudaStreamUpdateCaptureDependencies(cap, &cn, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CG(cudaStreamBeginCaptureToGraph(cap2, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    CG(pass(a, b, 1, cap2));
    CG(launch_check(cap2, c->red2 + 9, c->d_ls, h, mn, mx, tol, pdl));
    CG(pass(b, a, 0, cap2, false, true));
    CG(launch_check(cap2, c->red2, c->d_ls, h, mn, mx, tol, pdl));
    cudaGraph_t bo = nullptr;
    CG(cudaStreamEndCapture(cap2, &bo));
    cudaGraph_t g = nullptr;
    CG(cudaStreamEndCapture(cap, &g));
    cudaStream_t keep = cap;
    cap = nullptr;                                // capture ended: CG must not end it again
    cudaError_t e = cudaGraphInstantiate(&c->tol_exec[n1], g, 0);
    cudaGraphDestroy(g);
    cudaStreamDestroy(keep);
    cudaStreamDestroy(cap2);
    cap2 = nullptr;
    if (e != cudaSuccess) return fail(c, STS_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    return STS_OK;
}
#undef CG

// One time step of loop 1 through the graph of the current rotation.
static sts_status graph_step(sts_ctx* ctx, bool* conv)
{
    sts_ctx* const c = ctx;
    const int n1 = c->cur, a = (n1 + 1) % 3, b = (n1 + 2) % 3;
    for (int r = 0; r < 3; r++)                   // all three rotations at once: no build inside later steps
        if (!c->tol_exec[r]) {
            const bool pdl = !(getenv("STS_NO_PDL") && atoi(getenv("STS_NO_PDL")) != 0);
            sts_status e = build_tol_graph(c, r, pdl);
            if (e && pdl) {                       // programmatic edges rejected: full edges
                fprintf(stderr, "sts: tolerance-mode graph without PDL edges (%s)\n", c->err.c_str());
                cudaGetLastError();
                if (c->tol_exec[r]) { cudaGraphExecDestroy(c->tol_exec[r]); c->tol_exec[r] = nullptr; }
                e = build_tol_graph(c, r, false);
            }
            if (e) return e;
        }
    CU(cudaGraphLaunch(c->tol_exec[n1], c->stream));
    CU(cudaMemcpyAsync(c->h_ls, c->d_ls, sizeof(LoopState), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    const LoopState ls = *c->h_ls;
    c->launches += 2 * ls.passes + (c->sch.time == STS_EXPLICIT && !fuse_conv(c) ? 1 : 0);
    c->cur = (ls.passes & 1) ? a : b;             // pass 1 writes a, pass 2 b, ...
    *conv = ls.conv != 0;
    if (ls.checked) {
        c->pass0 = c->stats.passes_done + ls.passes - 1;   // graph passes carry pass key 0xFFFFF
        sts_status e = finish_residuals(c, ls.red, ls.bad);
        if (e) return e;
    }
    c->stats.steps_done++;
    c->stats.passes_done += ls.passes;
    c->stats.converged = ls.conv ? 1 : 0;
    return STS_OK;
}

// Fixed-pass mode (tol <= 0) on one context without a halo: one time step =
// one graph launch of [zero residual slots; explicit planes; max_passes passes]
// built from the same kernels and launch configuration as the stream path (the
// general and all-regular CTA sets as two parallel kernel nodes per pass).  The
// pass key of a graph pass is its index within the step; the host keeps the
// sticky bad key after every step (one 8-byte async copy) to place a bad state
// in the call.
static bool fix_graph_ok(const sts_ctx* c)
{
    return c->sch.tol <= 0 && c->world == 1 && !c->comm && !c->peer && !c->profiling && c->sch.loop3 <= 1 &&
           !getenv("STS_NO_GRAPH") && !getenv("STS_GRAPH_KERNEL");
}
static sts_status build_fix_graph(sts_ctx* ctx, int n1)
{
    sts_ctx* const c = ctx;
    const int impl = c->sch.time == STS_IMPLICIT, tvd = c->sch.space == STS_TVD_VANLEER;
    const int a = (n1 + 1) % 3, b = (n1 + 2) % 3;
    cudaStream_t cap = nullptr;
    CU(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    Params k = make_params(c);
    k.u_1 = c->snap[n1].u; k.v_1 = c->snap[n1].v; k.p_1 = c->snap[n1].p; k.T_1 = c->snap[n1].T;
    k.ue = c->ue; k.ve = c->ve; k.Te = c->Te;
    const bool fuse = fuse_conv(c);
    cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->red, 0, (size_t)c->sch.max_passes * 9 * sizeof(unsigned long long), cap);
    if (e == cudaSuccess && !impl && !fuse) {
        Params q = k;
        q.ue_w = c->ue; q.ve_w = c->ve; q.Te_w = c->Te;
        conv_march_table(tvd, c->nu)<<<dim3(c->n_gen + c->n_reg), MX, conv_smem(c), cap>>>(make_march(c, q));
        e = cudaGetLastError();
    }
    int old = n1, nw = a;
    // consecutive one-node passes are joined by programmatic edges (PDL): pass k+1's
    // CTAs launch once every CTA of pass k has started and wait on the device for its
    // completion (griddepcontrol.wait in march_fused_kernel) -- the launch latency of a
    // pass hides behind the previous pass's tail.  STS_NO_PDL=1: full edges.
    const bool pdl = !(getenv("STS_NO_PDL") && atoi(getenv("STS_NO_PDL")) != 0);
    for (int it = 0; it < c->sch.max_passes && e == cudaSuccess; it++) {
        Params q = k;
        q.u_o = c->snap[old].u; q.v_o = c->snap[old].v; q.p_o = c->snap[old].p; q.T_o = c->snap[old].T;
        q.u_w = c->snap[nw].u; q.v_w = c->snap[nw].v; q.p_w = c->snap[nw].p; q.T_w = c->snap[nw].T;
        q.red = c->red + (size_t)it * 9;
        const bool fz = fuse && it == 0;                  // pass 1 computes and stores the planes (N2)
        if (fz) { q.ue_w = c->ue; q.ve_w = c->ve; q.Te_w = c->Te; }
        MarchParams m = make_march(c, q);
        m.pass_key = 0xFFFFF - it;
        cudaStreamCaptureStatus cs;
        cudaGraph_t g;
        const cudaGraphNode_t* dp = nullptr;
        size_t nd = 0;
        e = cudaStreamGetCaptureInfo(cap, &cs, nullptr, &g, &dp, &nd);
        if (e != cudaSuccess) break;
        std::vector<cudaGraphNode_t> deps(dp, dp + nd);
        cudaGraphNode_t nodes[2];
        int nn = 0;
        const bool one = use_fused(c, fz, false) && c->n_gen + c->n_reg > 0;
        if (one) {                                        // one node: general CTAs first
            MarchParams mp = m;
            mp.order = (const int4*)c->cta_order;
            void* args[] = {&mp};
            cudaKernelNodeParams kp = {};
            kp.func = (void*)fused_table(impl, tvd, 0);
            kp.gridDim = dim3(c->n_gen + c->n_reg);
            kp.blockDim = dim3(MX);
            kp.sharedMemBytes = march_smem(c);
            kp.kernelParams = args;
            e = add_pass_node(&nodes[nn], g, deps, kp, pdl && it > 0);
            nn++;
        }
        for (int part = 0; part < 2 && e == cudaSuccess && !one; part++) {
            const int cnt = part == 0 ? c->n_gen : c->n_reg;
            if (cnt == 0) continue;
            MarchParams mp = m;
            mp.order = (const int4*)c->cta_order + (part ? c->n_gen : 0);
            void* args[] = {&mp};
            cudaKernelNodeParams kp = {};
            kp.func = fz ? (void*)march_fusec_table(tvd, part, 0) : (void*)march_table(impl, tvd, part, part ? 0 : c->nu);
            kp.gridDim = dim3(cnt);
            kp.blockDim = dim3(MX);
            kp.sharedMemBytes = part ? regk_smem(c, fz, false) : (fz ? FUSEC_SMEM : march_smem(c));
            kp.kernelParams = args;
            e = add_pass_node(&nodes[nn], g, deps, kp, pdl && it > 0);
            if (e == cudaSuccess && part == 0) e = graph_node_high_priority(nodes[nn]);
            nn++;
        }
        if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(cap, nodes, nn, cudaStreamSetCaptureDependencies);
        old = nw;
        nw = nw == a ? b : a;
    }
    cudaGraph_t g = nullptr;
    const cudaError_t e2 = cudaStreamEndCapture(cap, &g);
    if (e == cudaSuccess) e = e2;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&c->fix_exec[n1], g, 0);
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
    if (e != cudaSuccess) return fail(c, STS_E_CUDA, std::string("fixed-pass graph: ") + cudaGetErrorString(e));
    return STS_OK;
}
static sts_status fix_graph_advance(sts_ctx* ctx, int32_t n_steps, sts_stats* out)
{
    sts_ctx* c = ctx;
    for (int r = 0; r < 3; r++)                   // all three rotations at once: no build inside later steps
        if (!c->fix_exec[r]) { sts_status e = build_fix_graph(c, r); if (e) return e; }
    if (c->h_badstep_n < n_steps) {
        if (c->h_badstep) cudaFreeHost(c->h_badstep);
        c->h_badstep = nullptr;
        c->h_badstep_n = 0;
        CU(cudaMallocHost(&c->h_badstep, (size_t)std::max(n_steps, 1) * sizeof(unsigned long long)));
        c->h_badstep_n = std::max(n_steps, 1);
    }
    const long long pass0 = c->stats.passes_done;
    const int P = c->sch.max_passes;
    for (int s = 0; s < n_steps; s++) {
        NvtxRange nv_step("time step");
        const int n1 = c->cur;
        CU(cudaGraphLaunch(c->fix_exec[n1], c->stream));
        CU(cudaMemcpyAsync(c->h_badstep + s, c->bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
        c->cur = (P & 1) ? (n1 + 1) % 3 : (n1 + 2) % 3;          // pass 1 writes n1+1, pass 2 n1+2, ...
        c->launches += 2 * P + (c->sch.time == STS_EXPLICIT && !fuse_conv(c) ? 1 : 0);
        c->stats.steps_done++;
        c->stats.passes_done += P;
        c->stats.converged = 0;
    }
    if (n_steps > 0) {
        unsigned long long red[10];
        sts_status e = gather_red(&c, 1, P - 1, red, c->stream);     // synchronises the stream
        if (e) return e;
        c->pass0 = pass0;
        for (int s = 0; s < n_steps; s++)
            if (c->h_badstep[s]) { c->pass0 = pass0 + (long long)s * P; break; }
        e = finish_residuals(c, red, red[9]);
        if (out) *out = c->stats;
        return e;
    }
    if (out) *out = c->stats;
    return STS_OK;
}

// Loop 1 x loop 2 for a group of slab contexts advanced in lockstep (n == 1
// for the usual one-context-per-process case).
static sts_status drive(sts_ctx** cs, int n, int32_t n_steps, sts_stats* out)
{
    sts_ctx* ctx = cs[0];
    CU(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int impl = ctx->sch.time == STS_IMPLICIT, tvd = ctx->sch.space == STS_TVD_VANLEER;
    // test hook: the graph instances (early exit on a zero `done` flag) launched from the stream
    const bool gk = getenv("STS_GRAPH_KERNEL") != nullptr;
    if (gk && !ctx->red2) {
        CU(cudaMalloc(&ctx->red2, 18 * sizeof(unsigned long long)));
        CU(cudaMalloc(&ctx->d_ls, sizeof(LoopState)));
        CU(cudaMallocHost(&ctx->h_ls, sizeof(LoopState)));
        CU(cudaMemset(ctx->d_ls, 0, sizeof(LoopState)));
    }
    const bool tolmode = ctx->sch.tol > 0;
    sts_status status = STS_OK;
    int last_it = -1;
    std::vector<int> n1(n), a(n), b(n), old(n), nw(n), which(n);
    unsigned long long red[10];
    for (int r = 0; r < n; r++) {                    // a new advance call: clear the sticky bad state
        cs[r]->pass0 = cs[r]->stats.passes_done;
        CU(cudaMemsetAsync(cs[r]->bad, 0, sizeof(unsigned long long), st));
    }
    long long prel = 0;                               // pass index within this advance call
    if (n == 1 && fix_graph_ok(ctx)) return fix_graph_advance(ctx, n_steps, out);
    if (n == 1 && tol_graph_ok(ctx)) {
        for (int step = 0; step < n_steps; step++) {
            NvtxRange nv_step("time step");
            bool conv = false;
            sts_status e = graph_step(ctx, &conv);
            if (e) { if (out) *out = ctx->stats; return e; }
            if (!conv) status = STS_E_NONCONVERGED;
        }
        if (out) *out = ctx->stats;
        if (status == STS_E_NONCONVERGED) return fail(ctx, status, "loop 2 reached max_passes without convergence");
        return STS_OK;
    }
    for (int step = 0; step < n_steps; step++) {
        NvtxRange nv_step("time step");
        for (int r = 0; r < n; r++) {
            sts_ctx* c = cs[r];
            // a0: n-1 := current state; old := n-1; ping-pong between the other two
            n1[r] = c->cur; a[r] = (n1[r] + 1) % 3; b[r] = (n1[r] + 2) % 3;
            old[r] = n1[r]; nw[r] = a[r];
            CU(cudaMemsetAsync(c->red, 0, (size_t)c->sch.max_passes * 9 * sizeof(unsigned long long), st));
        }
        auto base = [&](sts_ctx* c, int r) {
            Params k = make_params(c);
            k.u_1 = c->snap[n1[r]].u; k.v_1 = c->snap[n1[r]].v; k.p_1 = c->snap[n1[r]].p; k.T_1 = c->snap[n1[r]].T;
            k.ue = c->ue; k.ve = c->ve; k.Te = c->Te;
            return k;
        };
        const bool fuse = n == 1 && fuse_conv(ctx);       // a1 inside pass 1 (N2)
        if (!impl && !fuse) {   // a1: explicit planes, once per time step
            for (int r = 0; r < n; r++) {
                sts_ctx* c = cs[r];
                Params k = base(c, r);
                k.ue_w = c->ue; k.ve_w = c->ve; k.Te_w = c->Te;
                prof_begin(c, 1);
                const dim3 mgrid(c->n_gen + c->n_reg);                 // the conv kernel: every CTA of the schedule
                MarchParams mc = make_march(c, k);
                unsigned long long q = 0;
                if (c->peer) {                                         // fused halo: planes stored into the neighbours
                    q = ++c->seq;
                    sts_status e = peer_wait(c, q - 1, st);
                    if (e) return e;
                    peer_params(c, 3, mc);
                }
                conv_march_table(tvd, c->nu)<<<mgrid, MX, conv_smem(c), st>>>(mc);
                if (c->peer) { sts_status e = peer_signal(c, q, st); if (e) return e; }
                prof_end(c);
                c->launches++;
                CU(cudaGetLastError());
                which[r] = 3;
            }
            sts_status e = exchange_group(cs, n, which.data(), st);
            if (e) return e;
        }
        int passes = 0;
        bool conv = false;
        // Halo overlap (one rank per process, a halo to exchange, >= 3 strips):
        // pass p runs its edge strips on the high-priority halo stream, followed
        // there by pack -> NCCL send/recv -> unpack; the interior strips run on the
        // pass stream and need only pass p-1 (edge + interior), never the halo, so
        // the exchange of pass p overlaps the interior of pass p+1.  In-process
        // slab groups launch the same two CTA sets one after the other.
        // a peer-connected rank always splits (its edge strips carry the fused halo
        // stores, which the all-regular kernel does not compile in), even when
        // every strip is an edge strip (an empty interior set)
        const bool split = (ctx->world > 1 || ctx->comm) && ctx->n_edge > 0 &&
                           (ctx->peer || (ctx->n_edge < ctx->n_split && !getenv("STS_NO_SPLIT")));
        const bool overlap = split && n == 1 && (ctx->comm || ctx->peer);
        if (overlap) {
            if (!ctx->hstream) {
                int lo = 0, hi = 0;
                CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
                CU(cudaStreamCreateWithPriority(&ctx->hstream, cudaStreamNonBlocking, hi));
                for (cudaEvent_t* e : {&ctx->ev_a[0], &ctx->ev_a[1], &ctx->ev_b, &ctx->ev_s, &ctx->ev_h})
                    CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            }
            CU(cudaEventRecord(ctx->ev_s, st));                   // red reset, explicit planes, last step
            CU(cudaStreamWaitEvent(ctx->hstream, ctx->ev_s, 0));
        }
        for (int it = 0; it < ctx->sch.max_passes; it++) {
            for (int r = 0; r < n; r++) {
                sts_ctx* c = cs[r];
                Params k = base(c, r);
                k.u_o = c->snap[old[r]].u; k.v_o = c->snap[old[r]].v; k.p_o = c->snap[old[r]].p; k.T_o = c->snap[old[r]].T;
                k.u_w = c->snap[nw[r]].u; k.v_w = c->snap[nw[r]].v; k.p_w = c->snap[nw[r]].p; k.T_w = c->snap[nw[r]].T;
                k.red = c->red + (size_t)it * 9;
                const int pkey = 0xFFFFF - (int)std::min<long long>(prel, 0xFFFFE);
                if (split) {
                    MarchParams ma = make_march(c, k);
                    ma.pass_key = pkey;
                    MarchParams mb = ma;
                    ma.order = (const int4*)c->cta_split;
                    cudaStream_t as = overlap ? c->hstream : st;
                    if (overlap && it > 0) CU(cudaStreamWaitEvent(as, c->ev_b, 0));   // pass it-1 complete
                    prof_begin(c, 0);
                    unsigned long long q = 0;
                    if (c->peer) {              // fused halo: the edge strips store into the neighbours
                        q = ++c->seq;
                        sts_status e = peer_wait(c, q - 1, as);
                        if (e) return e;
                        peer_params(c, nw[r], ma);
                    }
                    march_fn gen = c->peer ? march_halo_table(impl, tvd, c->nu)
                                 : gk ? march_graph_table(impl, tvd, 0, c->nu) : march_table(impl, tvd, 0, c->nu);
                    gen<<<c->n_edge, MX, march_smem(c), as>>>(ma);
                    if (c->peer) { sts_status e = peer_signal(c, q, as); if (e) return e; }
                    if (overlap) CU(cudaEventRecord(c->ev_a[it & 1], as));
                    c->launches += 1 + launch_march(c, mb, gk, st, c->cta_split + 4 * c->n_edge, c->n_split_gen,
                                                    c->n_split - c->n_edge - c->n_split_gen);
                    if (overlap) {
                        CU(cudaStreamWaitEvent(st, c->ev_a[it & 1], 0));   // the pass ends with both sets
                        prof_end(c);
                        CU(cudaEventRecord(c->ev_b, st));
                        if (!c->peer) {
                            sts_status e = halo_pack(c, c->snap[nw[r]], as);
                            if (!e) e = halo_nccl(c, as);
                            if (!e) e = halo_unpack(c, c->snap[nw[r]], as);
                            if (e) return e;
                        }
                    } else {
                        prof_end(c);
                    }
                } else if (c->sch.loop3 > 1) {
                    // loop 3 (N3, reading R41): sweeps 1 .. L3-1 write T, p into the sweep
                    // iterates (u, v, residuals, bad key into junk); sweep k >= 2 reads the
                    // previous sweep's T, p for the coupled terms; the last sweep writes the
                    // new state, the velocity correction and the residuals as usual
                    prof_begin(c, 0);
                    const int L = c->sch.loop3;
                    const size_t cb = cell_elems(c) * sizeof(double);
                    for (int q2 = 0; q2 < 2 && q2 < L - 1; q2++) {   // ghost columns / solid cells: the old iterate's
                        CU(cudaMemcpyAsync(c->l3p[q2], c->snap[old[r]].p, cb, cudaMemcpyDeviceToDevice, st));
                        CU(cudaMemcpyAsync(c->l3T[q2], c->snap[old[r]].T, cb, cudaMemcpyDeviceToDevice, st));
                    }
                    for (int kk = 1; kk <= L; kk++) {
                        Params q = k;
                        const bool last = kk == L;
                        if (!last) {
                            q.p_w = c->l3p[(kk - 1) & 1]; q.T_w = c->l3T[(kk - 1) & 1];
                            q.u_w = c->l3junk; q.v_w = c->l3junk; q.red = c->l3red;
                            CU(cudaMemsetAsync(c->l3red, 0, 10 * sizeof(unsigned long long), st));
                        }
                        MarchParams mk = make_march(c, q);
                        mk.pass_key = pkey;
                        if (!last) mk.bad = c->l3red + 9;
                        if (kk >= 2) { mk.p3 = c->l3p[(kk - 2) & 1]; mk.T3 = c->l3T[(kk - 2) & 1]; }
                        c->launches += launch_march(c, mk, false, st, c->cta_order, c->n_gen, c->n_reg, kk >= 2);
                    }
                    prof_end(c);
                } else {
                    prof_begin(c, 0);
                    MarchParams mk = make_march(c, k);
                    mk.pass_key = pkey;
                    if (gk) mk.done = &c->d_ls->done;
                    if (c->peer) return fail(c, STS_E_ARG, "peer-connected rank without edge strips");
                    const bool fz = fuse && it == 0;       // pass 1 computes and stores the planes
                    if (fz) { mk.k.ue_w = c->ue; mk.k.ve_w = c->ve; mk.k.Te_w = c->Te; }
                    c->launches += launch_march(c, mk, gk, st, c->cta_order, c->n_gen, c->n_reg, false, fz);
                    prof_end(c);
                }
                CU(cudaGetLastError());
                which[r] = nw[r];
            }
            if (!overlap) {
                sts_status e = exchange_group(cs, n, which.data(), st);
                if (e) return e;
            }
            passes++;
            prel++;
            last_it = it;
            for (int r = 0; r < n; r++) { old[r] = nw[r]; nw[r] = (nw[r] == a[r]) ? b[r] : a[r]; }
            if (tolmode && passes >= ctx->sch.min_passes) {
                if (overlap) {                                    // the halo of this pass too
                    CU(cudaEventRecord(ctx->ev_h, ctx->hstream));
                    CU(cudaStreamWaitEvent(st, ctx->ev_h, 0));
                }
                sts_status e = gather_red(cs, n, it, red, st);
                if (e) return e;
                for (int r = 0; r < n; r++) cs[r]->cur = old[r];
                e = finish_residuals(ctx, red, red[9]);
                for (int r = 1; r < n; r++) { cs[r]->stats = ctx->stats; }
                if (e) return e;
                const double* rs = ctx->stats.res;
                if (rs[0] < ctx->sch.tol && rs[1] < ctx->sch.tol && rs[2] < ctx->sch.tol && rs[3] < ctx->sch.tol) { conv = true; break; }
            }
        }
        if (overlap) {                                            // join the halo stream
            CU(cudaEventRecord(ctx->ev_h, ctx->hstream));
            CU(cudaStreamWaitEvent(st, ctx->ev_h, 0));
        }
        for (int r = 0; r < n; r++) {
            sts_ctx* c = cs[r];
            c->cur = old[r];
            c->stats.steps_done++;
            c->stats.passes_done += passes;
            c->stats.converged = conv ? 1 : 0;
        }
        if (tolmode && !conv) status = STS_E_NONCONVERGED;
    }
    if (last_it >= 0 && !tolmode) {
        sts_status e = gather_red(cs, n, last_it, red, st);
        if (e) return e;
        e = finish_residuals(ctx, red, red[9]);
        for (int r = 1; r < n; r++) { cs[r]->stats.res[0] = ctx->stats.res[0]; cs[r]->stats.res[1] = ctx->stats.res[1];
                                      cs[r]->stats.res[2] = ctx->stats.res[2]; cs[r]->stats.res[3] = ctx->stats.res[3]; }
        if (e) { if (out) *out = ctx->stats; return e; }
    }
    if (out) *out = ctx->stats;
    if (status == STS_E_NONCONVERGED) return fail(ctx, status, "loop 2 reached max_passes without convergence");
    return STS_OK;
}

extern "C" sts_status sts_advance(sts_ctx* ctx, int32_t n_steps, sts_stats* out)
{
    NvtxRange nv("sts_advance");
    if (!ctx || n_steps < 0) return fail(ctx, STS_E_ARG, "bad argument");
    if (ctx->local_group) return fail(ctx, STS_E_ARG, "in-process slab contexts advance with sts_advance_group");
    return drive(&ctx, 1, n_steps, out);
}

extern "C" sts_status sts_advance_group(sts_ctx** ctxs, int32_t n, int32_t n_steps, sts_stats* out)
{
    NvtxRange nv("sts_advance_group");
    sts_ctx* ctx = nullptr;
    if (!ctxs || n < 1 || n_steps < 0) return fail(ctx, STS_E_ARG, "bad argument");
    for (int r = 0; r < n; r++) {
        if (!ctxs[r] || ctxs[r]->world != n || ctxs[r]->rank != r || (n > 1 && !ctxs[r]->local_group) ||
            ctxs[r]->device != ctxs[0]->device)
            return fail(ctxs[r], STS_E_ARG, "group must be ranks 0..n-1 of one in-process decomposition on one device");
    }
    return drive(ctxs, n, n_steps, out);
}
