/*
 * simplets.h -- C ABI of libsimplets.so, the B200 (sm_100a) fp64 SIMPLE-TS
 * sweep of K. S. Shterev, "GPU implementation of algorithm SIMPLE-TS for
 * calculation of unsteady, viscous, compressible and heat-conductive gas
 * flows" (arXiv:1802.04243).
 *
 * Citations: P:n = line n of the paper's LaTeX,
 * with the paper's equation labels; DESIGN.md section 3 is the written
 * discrete spec (formulas, boundary-condition spec, readings Rn) that this
 * library implements.
 *
 * Conventions
 *  - Every call returns sts_status; no C++ exception crosses the ABI.  A
 *    message for the last failure is available from sts_last_error().
 *  - The library owns the context and every device allocation it makes; the
 *    caller owns every host buffer it passes and keeps it valid for the call.
 *  - Host buffers are fp64, row-major with i (x) fastest, in the GLOBAL shape
 *    of the field: cells nx*ny, u (nx+1)*ny (u_{i,j} on face x^f_i between
 *    cells (i-1,j) and (i,j)), v nx*(ny+1) (v_{i,j} on face y^f_j between
 *    (i,j-1) and (i,j)) -- P:271-280.  With a multi-GPU context (dist->world
 *    > 1) sts_get_field returns only this rank's owned slab (see sts_shape).
 *  - All device work runs on the context's stream (sts_set_stream); calls that
 *    return host data synchronise that stream.
 *  - There is no CPU fallback: sts_create fails with STS_E_CUDA when no
 *    CUDA device is usable.
 */
#ifndef SIMPLETS_H
#define SIMPLETS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    STS_OK = 0,
    STS_E_ARG = 1,          /* NULL pointer, wrong buffer size, bad enum          */
    STS_E_CONFIG = 2,       /* geometry/gas/scheme rejected (lengths not multiples
                               of the spacing, square outside the channel, Kn<=0) */
    STS_E_NONCONVERGED = 3, /* tol > 0 and a step reached max_passes; state valid */
    STS_E_STATE = 4,        /* NaN / T <= 0 / p <= 0 appeared (see sts_stats)     */
    STS_E_CUDA = 5,         /* CUDA runtime error or no device                    */
    STS_E_COMM = 6,         /* NCCL error (multi-GPU)                             */
    STS_E_OOM = 7           /* device allocation failed                           */
} sts_status;

/* Time treatment of the convective terms: explicit (Forward Euler, separate
 * convective kernel once per step, Fig. 1) or implicit (Backward Euler,
 * one kernel per loop-2 pass, Fig. 2).  P:82-88. */
typedef enum { STS_EXPLICIT = 0, STS_IMPLICIT = 1 } sts_time_scheme;
/* Space treatment: first-order upwind, or TVD with the Van Leer limiter
 * psi(r) = (r+|r|)/(1+r). */
typedef enum { STS_UPWIND = 0, STS_TVD_VANLEER = 1 } sts_space_scheme;
/* x boundaries: supersonic inflow at x = 0 and zero-gradient outflow at x = L
 * (the paper's channel, DESIGN 3.5 items 2-3), or periodic
 * (validation cases, DESIGN 3.5 item 4). */
typedef enum { STS_X_INFLOW_OUTFLOW = 0, STS_X_PERIODIC = 1 } sts_xbc;
/* Pressure-work form of the energy source S^T_c (reading R9). */
typedef enum { STS_PW_DPDT = 0, STS_PW_PRINTED = 1, STS_PW_NEG = 2, STS_PW_GAMMA = 3 } sts_pw_form;
typedef enum {
    STS_U = 0, STS_V = 1, STS_P = 2, STS_T = 3, STS_RHO = 4,
    STS_UEXP = 6, STS_VEXP = 7, STS_TEXP = 8      /* explicit planes (read only) */
} sts_field;

/* Uniform Cartesian grid: nx = round(length_x/spacing), ny likewise;
 * |length/spacing - n| > 1e-9 -> STS_E_CONFIG. */
typedef struct { double length_x, length_y, spacing; } sts_grid;

/* A square particle as a solid block of cells [i0, i0+ni) x [j0, j0+nj)
 * in integer cell coordinates (paper squares: ni = nj = a/spacing).  With
 * inflow/outflow it must leave at least one fluid column at each end. */
typedef struct { int32_t i0, j0, ni, nj; } sts_square;

/* Gas, walls and body force.  Kn (> 0), inlet Mach number and
 * gamma = c_p/c_v set the Eq. pl37 constants A = 0.5,
 * B = 5 sqrt(pi)/16 Kn, C^T1 = Kn sqrt(225 pi/1024), C^T2 = sqrt(pi)/4 Kn,
 * C^T3 = 2/5 and the inlet velocity u_in = M sqrt(gamma T_in / 2)
 * (V0 = sqrt(2 R T0)).  particle_frame = 1 makes both channel walls
 * move at +u_in (reading R14) and overrides u_wall_*.  T_wall is the
 * channel-wall temperature (= reference), T_square the square's
 * (R15).  g_x, g_y: body force of Eqs. pl2/pl3 (R22).  pw_form: the
 * pressure-work term of S^T_c (reading R9): STS_PW_DPDT (0,
 * default) = C^T3 Dp/Dt of the continuum energy equation Eq. pl6 at the
 * old iterate; STS_PW_PRINTED (1) = +C^T3 p div(u) as printed in Eq. pl29
 * (P:479); STS_PW_NEG (2) = -C^T3 p div(u); STS_PW_GAMMA (3) =
 * -gamma C^T3 p div(u).  Any other value -> STS_E_CONFIG. */
typedef struct {
    double Kn, mach, gamma;
    double p_in, T_in;
    double u_wall_bottom, u_wall_top;
    double T_wall, T_square;
    double g_x, g_y;
    int32_t pw_form;             /* sts_pw_form */
    int32_t reserved0;           /* must be 0 */
    int32_t particle_frame;
    int32_t xbc;                 /* sts_xbc */
} sts_gas;

/* Scheme and loop-2 control (Figs. 1-2): time step dt > 0; per time step
 * loop 2 runs until the four residuals (DESIGN R35) are < tol after at least
 * min_passes passes, or exactly max_passes passes when tol <= 0.
 * loop3: energy / pressure sweeps per loop-2 pass -- 0 or 1 is the GPU column
 * of Figs. 1-2; k > 1 adds the CPU column's loop 3 ("calculate the
 * coupled equations for energy and pressure") as
 * k-1 Jacobi sweeps over the T-p coupled terms (reading R41, DESIGN 3.6).
 * loop3 > 1 runs on single-rank, uniform-mesh contexts (else STS_E_CONFIG). */
typedef struct {
    int32_t time;                /* sts_time_scheme  */
    int32_t space;               /* sts_space_scheme */
    double dt;
    int32_t min_passes, max_passes;
    double tol;
    int32_t loop3;               /* T-p sweeps per pass (N3); 0 / 1 = off */
    int32_t reserved;            /* must be 0 */
} sts_scheme;

/* Multi-GPU: one process per GPU; the channel is split into slabs along x
 * (DESIGN section 7).  nccl_id points to the 128-byte ncclUniqueId made by
 * sts_nccl_unique_id on rank 0 and broadcast by the caller.  NULL dist or
 * world == 1 -> single GPU; world > 1 with nccl_id == NULL -> an in-process
 * slab of a group driven by sts_advance_group. */
typedef struct { int32_t rank, world, device; const void* nccl_id; } sts_dist;

/* Statistics of the last sts_advance: steps/passes done (cumulative), last
 * residuals (u, v, p, T), converged flag of the last step.  On STS_E_STATE:
 * the FIRST bad state of the call -- its cell (flat global index j*nx + i, -1
 * for a NaN velocity), field (STS_P / STS_T, STS_U for a NaN velocity) and the
 * cumulative pass index at which it appeared.  The passes after it do no work
 * (a sticky device flag), and the state is undefined. */
typedef struct {
    int64_t steps_done, passes_done;
    double res[4];
    int32_t converged;
    int32_t bad_field;
    int64_t bad_cell;
    int64_t bad_pass;
} sts_stats;

typedef struct sts_ctx sts_ctx;

/* Host-only decomposition plan of one rank (no CUDA call):
 * the channel is cut into `world` slabs of near-equal width along x
 * (remainder to the low ranks).  Rank `rank` owns global columns [i0, i1)
 * and stores `pitch` local columns, local column l <-> global column
 * i0 - ghost + l (periodic: mod nx).  After every pass it sends its first /
 * last `ghost` owned columns to the left / right neighbour (-1: physical
 * boundary) and receives the unwrapped global columns recv_left /
 * recv_right into its ghost columns.  kinds (optional, 3 x (ny+1) x pitch
 * bytes): cell kinds (0 fluid, 1 solid, 2 inlet ghost, 3 outlet ghost,
 * 4 beyond a wall), u-face kinds, v-face kinds (0 active, 1 fixed 0,
 * 2 inlet, 3 outlet, 4 wall, 5 none) of the stored columns. */
typedef struct {
    int32_t nx, ny, i0, i1, pitch, ghost, left, right;
    int32_t send_left[2], send_right[2], recv_left[2], recv_right[2];
} sts_plan_info;
sts_status sts_plan(const sts_grid* grid, const sts_square* squares, int32_t n_squares,
                    const sts_gas* gas, int32_t world, int32_t rank, sts_plan_info* out,
                    uint8_t* kinds);

/* Build the case: validates and snaps the geometry (integer cells), builds
 * the cell / u-face / v-face kind maps (DESIGN 3.5), derives the Eq. pl37
 * constants, allocates three device snapshots (n-1, old, new) of u, v, p, T
 * plus the explicit planes, and sets the free-stream state. */
sts_status sts_create(const sts_grid* grid, const sts_square* squares, int32_t n_squares,
                      const sts_gas* gas, const sts_scheme* scheme, const sts_dist* dist,
                      sts_ctx** out);
void sts_destroy(sts_ctx* ctx);
/* Thread-local message of the last failure (ctx may be NULL). */
const char* sts_last_error(const sts_ctx* ctx);

/* Use this CUDA stream (cudaStream_t as void*, e.g.
 * torch.cuda.current_stream().cuda_stream); NULL = the legacy default stream. */
sts_status sts_set_stream(sts_ctx* ctx, void* cuda_stream);

/* Free-stream state (P:686 test case; reading R12): p = p_in, T = T_in,
 * rho = p/T, u = u_in on every face, v = 0; fixed faces (solid, walls) 0. */
sts_status sts_init_freestream(sts_ctx* ctx);

/* Copy one field (STS_U, STS_V, STS_P or STS_T) from a host buffer of n
 * doubles into the current state (all three snapshots); rho and Gamma follow
 * from p and T (Eqs. pl5, pl37); ghost columns follow the BC spec and fixed
 * faces are re-imposed (DESIGN 3.5).  The buffer is the GLOBAL shape, or on a
 * multi-rank context this rank's owned slab (sts_shape); a slab-shaped input
 * ends with a halo exchange, so every rank makes the call (collective).  On a
 * peer-connected rank every call is a fenced halo phase (DESIGN 7.2).
 * Synchronises the context stream; n of neither shape -> STS_E_ARG. */
sts_status sts_set_field(sts_ctx* ctx, int32_t field, const double* host, int64_t n);
/* Same from a DEVICE buffer (global or slab shape). */
sts_status sts_set_field_device(sts_ctx* ctx, int32_t field, const double* dev, int64_t n);

/* Non-uniform mesh (the general staggered mesh of Fig. 5, with the
 * steps Delta x_i, Delta y_j that every coefficient of Eqs. pl8-pl33 carries;
 * SURVEY 8(f) N4): dx = nx GLOBAL column widths, dy = ny row heights (host
 * buffers, > 0; the caller keeps ownership).  NULL keeps that direction at the
 * uniform sts_grid spacing.  Bilinear interpolation weights per reading R4.  The
 * cell counts and the squares (in cell units) are those of sts_create; the
 * state is kept.  Every point then runs the general-mesh instances of the
 * kernels (no uniform shortcuts), which is slower than the uniform path.
 * Returns STS_E_ARG on a size mismatch, STS_E_CONFIG on a step <= 0. */
sts_status sts_set_mesh(sts_ctx* ctx, const double* dx, int64_t nx, const double* dy, int64_t ny);

/* Loop 1 x loop 2 (Figs. 1-2, GPU columns): n_steps time steps. */
sts_status sts_advance(sts_ctx* ctx, int32_t n_steps, sts_stats* out);

/* Advance n in-process slab contexts in lockstep: contexts created with
 * dist = {rank r, world n, device d, nccl_id = NULL} for r = 0..n-1 on the
 * same device form one x-decomposed domain whose per-pass halo exchange is a
 * device-to-device copy on ctxs[0]'s stream instead of NCCL (same pack /
 * unpack kernels, same halo index maps).  Used to verify the slab
 * decomposition on one GPU; stats are the group's. */
sts_status sts_advance_group(sts_ctx** ctxs, int32_t n, int32_t n_steps, sts_stats* out);

/* Copy this rank's owned part of a field to a host buffer of n doubles
 * (global shape for a single GPU; slab shape per sts_shape otherwise). */
sts_status sts_get_field(sts_ctx* ctx, int32_t field, double* host, int64_t n);
/* Same into a DEVICE buffer (async on the context stream). */
sts_status sts_get_field_device(sts_ctx* ctx, int32_t field, double* dev, int64_t n);

/* Asynchronous host I/O for pipelined time loops (a user's loop 1 of Figs. 1-2,
 * P:165, with its state kept on the host between steps).  Same shapes, same
 * arithmetic and the same resulting state as sts_set_field / sts_get_field; only
 * the copies move to two copy streams of the context (one per direction) so the
 * host<->device transfers of one step overlap the loop-2 passes of another.
 *
 * sts_stage_field: starts the H2D copy of a host buffer of n doubles (global or
 *   slab shape, as sts_set_field; pinned memory for a truly asynchronous copy)
 *   into the context's device staging slot of `field` (STS_U..STS_T) and returns.
 *   The caller keeps ownership and must not modify the buffer until the matching
 *   sts_set_staged has been made and the context stream has passed it (or
 *   sts_io_sync returns).  A second stage of the same field waits (on the device)
 *   until the previous staged copy has been set.
 * sts_set_staged: the context stream waits for that copy, then sets the field
 *   from the slot exactly as sts_set_field_device does.  Does not synchronise.
 *   STS_E_ARG if nothing is staged for the field.
 * sts_fetch_field: on the context stream, copies this rank's owned part of the
 *   current state of `field` (STS_U..STS_T) into a device slot, then starts the
 *   D2H copy of the slot into the host buffer of n doubles (shape as
 *   sts_get_field) and returns; the host buffer is valid after sts_io_sync.
 * sts_io_sync: blocks until every started H2D and D2H copy has completed.
 * Errors as the synchronous calls (STS_E_ARG on sizes, STS_E_CUDA). */
sts_status sts_stage_field(sts_ctx* ctx, int32_t field, const double* host, int64_t n);
sts_status sts_set_staged(sts_ctx* ctx, int32_t field);
sts_status sts_fetch_field(sts_ctx* ctx, int32_t field, double* host, int64_t n);
sts_status sts_io_sync(sts_ctx* ctx);

/* Integer maps, global shape for a single GPU: which = 0 cell kinds
 * (0 fluid, 1 solid), 1 u-face kinds, 2 v-face kinds (0 active, 1 fixed-0,
 * 2 inlet, 3 outlet, 4 wall), 3 the owned global column range of every rank
 * (2*world int32: i0, i1). */
sts_status sts_get_map(sts_ctx* ctx, int32_t which, int32_t* host, int64_t n);

/* Shape of this rank's owned part of a field: nx, ny of the returned
 * buffer and the first owned global column / owned column count. */
sts_status sts_shape(sts_ctx* ctx, int32_t field, int64_t* nx, int64_t* ny,
                     int64_t* i0_owned, int64_t* ni_owned);

/* Derived constants: out[0..6] = A, B, C^T1, C^T2, C^T3, u_in, dt. */
sts_status sts_constants(sts_ctx* ctx, double* out7);

/* Measurement hooks for bench.py: enable per-launch CUDA-event timing of the
 * hot kernels (on the context stream); read the accumulated totals:
 * out[0] = pass-kernel launches, out[1] = their summed ms, out[2] = conv
 * launches, out[3] = their ms, out[4] = all kernel launches of this context
 * since the last reset.  reset != 0 zeroes the counters. */
sts_status sts_profile(sts_ctx* ctx, int32_t enable);
sts_status sts_profile_read(sts_ctx* ctx, double* out5, int32_t reset);

/* Fused halo transport: instead of
 * pack -> NCCL send/recv -> unpack after every pass, the pass kernel's epilogue
 * (and the explicit-plane kernel's) stores this slab's first / last 4 owned
 * columns straight into the neighbours' ghost columns of the same snapshot
 * through peer-mapped memory (NVLink P2P / CUDA IPC), ordered by stream-side
 * flag writes and waits (cuStreamWriteValue64 / cuStreamWaitValue64); the
 * residual maxima go to every rank by system-scope atomicMax.  No NCCL call.
 *  - sts_peer_export: an opaque description of this rank (CUDA IPC handles of
 *    its snapshots, planes, flag and residual words); blob == NULL returns the
 *    size in *nbytes.  The caller moves the blobs between processes.
 *  - sts_peer_connect: blobs = world blobs of nbytes_each bytes, in rank
 *    order (this rank's own included); for contexts created with world > 1 and
 *    no nccl_id (one process per rank).  Afterwards sts_advance and
 *    sts_set_field are collective over the ranks, like the NCCL path.
 *  - sts_peer_connect_group: the same transport for in-process slab contexts of
 *    one device (sts_advance_group), with plain device pointers.
 * Results are bit-identical to the NCCL path and to one slab. */
sts_status sts_peer_export(sts_ctx* ctx, void* blob, int64_t* nbytes);
sts_status sts_peer_connect(sts_ctx* ctx, const void* blobs, int64_t nbytes_each);
sts_status sts_peer_connect_group(sts_ctx** ctxs, int32_t n);

/* rank 0: make the 128-byte NCCL unique id (multi-GPU bootstrap). */
sts_status sts_nccl_unique_id(void* out128);

#ifdef __cplusplus
}
#endif
#endif
