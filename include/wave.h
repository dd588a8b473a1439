/* wave.h -- C ABI of the B200-native 25-point acoustic wave stepper
 * (arXiv 2009.04619, "Accelerating High-Order Stencils on GPUs").
 *
 * The calls follow the paper's problem statement (PAPER.md L255-267,
 * Algorithm 1: data f, result u^n for n = 1..T; L300-301: inner size and PML
 * width are inputs of a simulation): create an nx*ny*nz grid with spacing, dt
 * and a velocity model, inject a source wavelet, step N times, read back the
 * wavefield.  One step computes, at every point of the extended domain,
 *
 *   inner (Eq. 2-3):
 *     u_next = 2u - u_prev + (V dt)^2 Lap8(u)
 *   PML   (25-pt on u + 7-pt star on eta;
 *          formula SPEC.md L152; profile DESIGN.md R2/R3):
 *     u_next = [2u - (1 - eta dt) u_prev + (V dt)^2 (Lap8(u) + grad eta . grad u)]
 *              / (1 + eta dt),   eta = eta_max (d/w)^2, d = Chebyshev distance
 *   then the source (Alg. 1, Eq. 2 RHS):
 *     u_next[src] += fp32((V_src dt)^2 * w[n])
 *
 * in fp32 with every constant computed in fp64 and rounded once (R8).
 *
 * Conventions for every call:
 *  - Pointers: "device" = CUDA device memory of the current device, "host" =
 *    any host memory (pinned memory makes copies asynchronous).  `where`
 *    arguments say which.  `stream` is a cudaStream_t passed as void*; NULL =
 *    the legacy default stream.  All device work is enqueued on `stream`;
 *    calls return before it completes unless stated otherwise.
 *  - Errors: every call returns a wave_status; no exception crosses the ABI.
 *    wave_last_error() returns a thread-local message for the last failure.
 *    Configuration errors are detected before anything is written.
 *    Asynchronous CUDA faults surface at the next synchronising call
 *    (wave_read to host, wave_check_finite) as WAVE_ERR_CUDA.
 *  - Ownership: the caller owns the big device buffers (two wavefield
 *    buffers and the vdt2 buffer, sized by wave_layout), the streams and any
 *    process group.  The plan owns its small device tables, the source
 *    increments, the TMA descriptors, its CUDA graphs and the step counter.
 *    Bound buffers must outlive all enqueued work.  A plan is not
 *    thread-safe; different plans are independent.
 */
#ifndef WAVE25_WAVE_H
#define WAVE25_WAVE_H

#include <stdint.h>

#if defined(__GNUC__)
#define WAVE_API __attribute__((visibility("default")))
#else
#define WAVE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; 0..3 mirror SPEC.md L585 exit codes. */
typedef enum {
    WAVE_OK = 0,
    WAVE_ERR_CONFIG = 1,     /* invalid descriptor / argument, nothing written */
    WAVE_ERR_UNSTABLE = 2,   /* non-finite wavefield        */
    WAVE_ERR_VERIFY = 3,     /* reserved for verification harnesses           */
    WAVE_ERR_CUDA = 4,       /* CUDA runtime / driver error                    */
    WAVE_ERR_ALLOC = 5,      /* host or device allocation failure              */
    WAVE_ERR_STATE = 6,      /* call out of order (e.g. step before bind)       */
    WAVE_ERR_PEER = 7        /* a z-neighbour did not complete its step within
                                the peer-wait bound (wave_peer_check)           */
} wave_status;

typedef enum { WAVE_MEM_HOST = 0, WAVE_MEM_DEVICE = 1 } wave_mem;

/* Kernel family used by wave_step.  STREAM (default) is the production
 * path: TMA-fed z-streaming interior kernel + PML wall kernels + source
 * kernel.  NAIVE is one thread per point with all 25 loads from global memory
 * (the paper's gmem code shape), kept as an ablation /
 * debugging path.  TB2 is two-step temporal blocking (the paper's future
 * work): one interior launch advances two time
 * steps reading u^n, u^{n-1}, vdt2 once (10 B per point-step instead of 16);
 * it needs two extra wavefield buffers (wave_plan_bind_aux) and a single-slab
 * plan, and falls back to STREAM single steps otherwise (odd step counts end
 * with one STREAM step).  All four compute bitwise-identical values. */
typedef enum { WAVE_KERNEL_STREAM = 0, WAVE_KERNEL_NAIVE = 1, WAVE_KERNEL_TB2 = 2, WAVE_KERNEL_PAIR = 3 } wave_kernel;
/* WAVE_KERNEL_PAIR: two steps per interior launch with no
 * redundant work: step-1 blocks publish per-tile, per-z-chunk progress,
 * step-2 blocks of the same launch wait for their own and neighbouring tiles
 * and read u^{n+1} back through L2; CTAs take work units from a ticket
 * counter in start order (deadlock-free); walls run as single steps before
 * and after.  In place (two buffers), single-slab plans only (CONFIG error
 * otherwise), fp32 and fp64, falls back to STREAM single steps with a stored
 * eta.  Bitwise equal to STREAM.  Measured slower than STREAM on B200 (kept
 * as an ablation). */

/* Arithmetic / storage precision of a plan.  FP32 (default): every constant
 * computed in fp64 and rounded once to fp32 (R8), fp32 storage and
 * arithmetic — the production path.  FP64 (SPEC.md L82 verification
 * precision): constants, vdt2, source increments,
 * wavefields and arithmetic in fp64 (the velocity model, dt and the wavelet
 * are still given in fp32); every buffer and every wavefield array crossing
 * the ABI (wave_set_state, wave_read, wave_field_ptr, halo views) holds
 * doubles.  STREAM and NAIVE kernels only. */
typedef enum { WAVE_PREC_FP32 = 0, WAVE_PREC_FP64 = 1 } wave_precision;

/* Problem descriptor.
 *  nx, ny, nz  extended domain (inner + PML on every face) of
 *              THIS plan; x innermost.  nz = planes of this rank's z-slab
 *              (= nz_global on one GPU).                         all >= 1
 *  pml_width   w, uniform on all six faces;
 *              0 <= 2w < min(nx, ny, nz_global), w <= 256
 *              (the kernels' shared PML tables hold 4 (w + 2) entries)
 *  kernel      wave_kernel
 *  hx, hy, hz  spacing (m), > 0 (per-axis, R1)
 *  dt          time step (s) as the fp32 value used; > 0, or 0 = automatic
 *              fp32(0.4 h_min / Vmax) resolved at wave_set_velocity (SPEC.md
 *              L199; single-slab plans only).  Rejected above the Courant
 *              limit dt Vmax sqrt(sum_a 1/h_a^2) <= 2/sqrt(6.5016...)
 *  precision   wave_precision (WAVE_PREC_FP32 = 0 unless stated)
 *  eta_max     PML damping maximum (1/s), >= 0.  Default 4 (stable; SPEC's
 *              100 diverges, R5)
 *  nz_global,  this slab covers global planes [z_offset, z_offset + nz) of
 *  z_offset    nz_global; (nz_global, z_offset) = (nz, 0) on one GPU
 */
typedef struct {
    int64_t nx, ny, nz;
    int32_t pml_width;
    int32_t kernel;
    double hx, hy, hz;
    float dt;
    int32_t precision;      /* wave_precision */
    double eta_max;
    int64_t nz_global, z_offset;
} wave_desc;

/* Device memory layout the caller must allocate (wave_layout).
 * Wavefield buffer: [planes][ny][pitch_x] elements (fp32, or fp64 for fp64
 * plans), planes = nz + 2*ghost_z, starting `origin` elements into the
 * allocation; element (i, j, k) (local k) lives at
 * origin + ((k + ghost_z)*ny + j)*pitch_x + i.  The origin shift puts the
 * first inner column x = pml_width on a 128-B line boundary when rows are
 * whole lines, so wall and inner points never share a line.
 * The ghost_z = 4 planes on each z side are the zero Dirichlet fringe
 * at the global ends and the neighbour's planes (halo) between
 * slabs.  x/y have no stored fringe (TMA out-of-bounds fill supplies zeros).
 * vdt2 buffer: [nz][ny][pitch_x] fp32 holding fp32((V dt)^2), also from `origin`.
 * Base addresses must be aligned to align_bytes. */
typedef struct {
    int64_t pitch_x;      /* floats per row: >= nx, multiple of 4 (16 B TMA stride rule) */
    int64_t ghost_z;      /* 4 = stencil radius R                     */
    int64_t planes;       /* nz + 2*ghost_z                                               */
    int64_t elems_u;      /* floats per wavefield buffer                                  */
    int64_t elems_vdt2;   /* floats in the vdt2 buffer                                    */
    int64_t align_bytes;  /* 128                                                          */
    int64_t elem_bytes;   /* 4 (fp32 plans) or 8 (fp64 plans): buffer element size        */
    int64_t origin;       /* elements before the layout's first element: the 128-B line
                             shift, plus one pad row when `seam` is set                   */
    int64_t seam;         /* 1: the layout admits the seam x-wall variant (both walls of
                             adjacent rows in one line; opt-in, measured
                             slower): one pad row before (in `origin`) and after the
                             buffers; never written, read only into masked lanes          */
} wave_layout_info;

/* One region of the paper's 7-region decomposition (PAPER.md L342-356,
 * Fig. 1; SPEC.md L239-247 axis binding: top/bottom split z, front/back
 * split y, left/right split x). Global coordinates. */
typedef enum {
    WAVE_REGION_INNER = 0, WAVE_REGION_TOP = 1, WAVE_REGION_BOTTOM = 2,
    WAVE_REGION_FRONT = 3, WAVE_REGION_BACK = 4, WAVE_REGION_LEFT = 5, WAVE_REGION_RIGHT = 6
} wave_region_kind;

typedef struct {
    int32_t kind;
    int32_t reserved0;
    int64_t lo[3];        /* x, y, z origin */
    int64_t ext[3];       /* extents (>= 0)  */
} wave_region;

typedef struct wave_plan wave_plan;   /* opaque */

/* ---- host-only calls (no GPU needed) ------------------------------------ */

/* Library version string, e.g. "wave25 0.1.0 sm_100a". Never fails. */
WAVE_API const char *wave_version(void);

/* Thread-local text of the last failure on this thread ("" if none). */
WAVE_API const char *wave_last_error(void);

/* Validate `desc` (all CONFIG rules except the velocity-dependent Courant
 * check) and return the buffer sizes to allocate in *out. */
WAVE_API wave_status wave_layout(const wave_desc *desc, wave_layout_info *out);

/* The 7 regions (inner, top, bottom, front, back, left, right) of the GLOBAL
 * extended domain nx*ny*nz_global.  out must hold 7. */
WAVE_API wave_status wave_decompose(const wave_desc *desc, wave_region *out);

/* The PML divisors of an fp32 plan, B_d = fp32(1 + eta_d dt) for d = 0..w
 * (the denominator of the SPEC.md L152 update), and rB_d = RN(1/B_d), the
 * correctly rounded reciprocal (host arithmetic, exact).  The kernels divide
 * a numerator n by a table B_d as q0 = RN(n rB), q = RN(q0 + RN(n - q0 B) rB)
 * (Markstein's FMA correction) when a plan's exhaustive device check has shown
 * it equal to the IEEE quotient RN(n / B_d) for every fp32 n of the binades
 * covering the range used (see wave_fastdiv; R9).  Uses desc->dt
 * (> 0); B and rB (either may be NULL) hold w + 1 floats.  Host memory. */
WAVE_API wave_status wave_division_table(const wave_desc *desc, float *B, float *rB);

/* 1 if the plan divides by its PML table through the verified Markstein
 * correction, 0 if by the IEEE division (fp64 plans, WAVE25_FASTDIV=0, or a
 * failed check), -1 on NULL. */
WAVE_API int32_t wave_fastdiv(const wave_plan *plan);

/* fp32 constants the plan uses, computed in fp64 and rounded once:
 * c13 = {c_xyz, c_x1..4, c_y1..4, c_z1..4},
 * eta/A/B[w+1] = eta_max (d/w)^2, 1 - eta dt, 1 + eta dt (SPEC.md L152,
 * DESIGN.md R2), inv2h[3] = 1/(2 h_a).  Uses desc->dt (must be > 0).
 * Any output pointer may be NULL.  Host memory. */
WAVE_API wave_status wave_constants(const wave_desc *desc, float *c13, float *eta, float *A,
                           float *B, float *inv2h);

/* ---- plan lifecycle ------------------------------------------------------ */

/* Validate desc and create a plan on the current CUDA device. */
WAVE_API wave_status wave_plan_create(const wave_desc *desc, wave_plan **out);

/* Bind caller-owned DEVICE buffers (sizes from wave_layout).  Zero-fills both
 * wavefield buffers (u^0 = u^{-1} = 0) and the vdt2 buffer,
 * builds TMA descriptors, resets the step counter to 0. */
WAVE_API wave_status wave_plan_bind(wave_plan *plan, float *u0, float *u1, float *vdt2, void *stream);

/* Bind two more caller-owned DEVICE wavefield buffers (same size and
 * alignment as u0/u1) for WAVE_KERNEL_TB2: a two-step launch reads
 * (u^n, u^{n-1}) from two buffers and writes (u^{n+1}, u^{n+2}) to the other
 * two, out of place (neighbouring tiles still read the old levels while the
 * new ones are written).  Zero-fills them; call after wave_plan_bind and
 * before setting the state.  Which buffer holds u^n afterwards is internal:
 * use wave_read / wave_field_ptr. */
WAVE_API wave_status wave_plan_bind_aux(wave_plan *plan, float *u2, float *u3, void *stream);

/* Stored (user-supplied) PML damping field (the
 * paper's smem_eta kernels read eta from memory):
 * bind a caller-owned DEVICE buffer of elems_vdt2 fp32 (vdt2 layout
 * [nz][ny][pitch_x]); zero-filled.  Single-slab plans only. */
WAVE_API wave_status wave_plan_bind_eta(wave_plan *plan, float *eta_buf, void *stream);

/* Install eta (dense [nz][ny][nx] fp32 in `where` memory, finite and >= 0;
 * copied into the bound buffer) instead of the eta_max (d/w)^2 profile; NULL
 * returns to the profile.  The PML region stays geometric (points with
 * Chebyshev distance d > 0 to the inner box take the PML update); there eta
 * is read on the 7-point star from the field (0 outside the domain) and
 * A = 1 - eta dt, B = 1 + eta dt come from the point's own value, computed in
 * fp64 and rounded once (R16).  Inner points ignore eta.  The z-PML
 * caps move from the interior kernel to the wall kernel; two-step blocking is
 * disabled while a field is installed.  Synchronises `stream`. */
WAVE_API wave_status wave_set_eta(wave_plan *plan, const float *eta, int32_t where, void *stream);

/* Destroy the plan (caller synchronises its streams first). NULL is a no-op. */
WAVE_API void wave_plan_destroy(wave_plan *plan);

/* ---- inputs -------------------------------------------------------------- */

/* Velocity model V (m/s), dense [nz][ny][nx] fp32 of THIS slab, all > 0
 * (SPEC.md L118), in `where` memory.  Computes vdt2 = fp32((V dt)^2) on the
 * device.  If desc.dt == 0 resolves dt = fp32(0.4 h_min / Vmax) first (reads
 * V back; synchronises `stream`).  Performs the Courant check (CONFIG).
 * If a source was set, its increments are rebuilt. */
WAVE_API wave_status wave_set_velocity(wave_plan *plan, const float *vel, int32_t where, void *stream);

/* Point source at GLOBAL cell (i, j, k), strictly inside the inner region
 * (SPEC.md L114), with wavelet samples w[0..nsamples) (host fp32, copied);
 * step n injects fp32(vdt2[src] * w[n]) (0 for n >= nsamples).  On a slab
 * that does not own plane k the call only records the source.  Requires
 * wave_set_velocity first. */
WAVE_API wave_status wave_set_source(wave_plan *plan, int64_t i, int64_t j, int64_t k,
                            const float *wavelet, int64_t nsamples, void *stream);

/* Optional initial state: u^{-1} (uprev) and u^0 (ucur), dense [nz][ny][nx]
 * fp32 in `where` memory (either may be NULL = zero).  Resets the step
 * counter to 0 and clears the halo planes.  On a peer-wired plan
 * (wave_set_peers) it also restarts the step-flag protocol (this rank's done
 * count, its flag words and the peer-wait error word): re-initialising a
 * peer-wired run is COLLECTIVE -- every rank calls it after a barrier that
 * follows its last step, then a second barrier, then wave_push_halo(1) for a
 * non-zero state and a third barrier, before anyone steps again
 * (dist.PeerSlabRunner.reset does exactly this). */
WAVE_API wave_status wave_set_state(wave_plan *plan, const float *uprev, const float *ucur,
                           int32_t where, void *stream);

/* ---- stepping ------------------------------------------------------------ */

/* Advance nsteps >= 0 time steps (Algorithm 1 lines 1-5 per step).  Single-
 * slab plans only (multi-slab plans use the split calls below).  Steps are
 * replayed from CUDA graphs captured on first use. */
WAVE_API wave_status wave_step(wave_plan *plan, int64_t nsteps, void *stream);

/* Split step for z-slab decomposition (one step = edges, halo exchange by the
 * caller, interior, finish; any order of edges/interior, same values as
 * wave_step):
 *  edges    : compute u_next on local planes [0, 4) and [nz-4, nz) (+ source
 *             if it lies there) -- the planes the neighbours need
 *  interior : compute u_next on local planes [4, nz-4) (+ source if there)
 *  finish   : role swap and step counter (host-side bookkeeping only) */
WAVE_API wave_status wave_step_edges(wave_plan *plan, void *stream);
WAVE_API wave_status wave_step_interior(wave_plan *plan, void *stream);
WAVE_API wave_status wave_step_finish(wave_plan *plan);

/* Device pointers of the 4-plane blocks to SEND to the lower / upper
 * neighbour (local planes [0,4) and [nz-4,nz)) and of the ghost blocks to
 * RECEIVE into (the 4 planes below / above the slab); each block is *count
 * contiguous floats.  which = 0: in the buffer wave_step_edges writes (the
 * next u^n; valid between wave_step_edges and wave_step_finish); which = 1:
 * in the current u^n (for the initial halo of a non-zero starting state). */
WAVE_API wave_status wave_halo_views(const wave_plan *plan, int32_t which, float **send_lo,
                                     float **send_hi, float **recv_lo, float **recv_hi,
                                     int64_t *count);

/* ---- fused peer-store halo exchange (z-slab runs, one GPU per rank) ------ */

/* Neighbour wiring for wave_step_peer.  All pointers are device pointers valid
 * in this process (peer / IPC mappings of the neighbours' buffers, e.g. opened
 * with cudaIpcOpenMemHandle over NVLink); NULL where there is no neighbour.
 * Every rank must bind its buffers in the same order and step in lockstep so
 * that buffer parity agrees.  Ownership stays with the caller. */
typedef struct {
    float *lo_buf[2];        /* lower (z_offset-1) neighbour's wavefield buffers 0/1 */
    float *hi_buf[2];        /* upper neighbour's wavefield buffers 0/1             */
    int64_t lo_nz;           /* lower neighbour's nz (locates its upper ghosts)    */
    uint64_t *my_flags;      /* this rank's 2 flag words (device, zero-initialised):
                                [0] steps completed by the lower neighbour,
                                [1] steps completed by the upper neighbour        */
    uint64_t *lo_flags;      /* lower neighbour's flag words (peer pointer)       */
    uint64_t *hi_flags;      /* upper neighbour's flag words (peer pointer)       */
} wave_peers;

/* Install (or clear, with NULL) the neighbour wiring.  Resets the step
 * counters used by the flag protocol.  A neighbour pointer that lives on
 * another device needs peer access from the plan's device: it is enabled here
 * (cudaDeviceEnablePeerAccess); CUDA error if the two devices cannot access
 * each other (no NVLink/PCIe P2P path). */
WAVE_API wave_status wave_set_peers(wave_plan *plan, const wave_peers *peers);

/* Cross-process mapping of device buffers for the peer wiring (CUDA IPC; the
 * current device is the caller's).
 *   wave_ipc_export: handle (64 bytes, cudaIpcMemHandle_t) of the allocation
 *     holding dptr and dptr's byte offset inside it (dptr may be an interior
 *     pointer of a caching-allocator block).
 *   wave_ipc_import: opens a handle exported by ANOTHER process on the current
 *     device with lazy peer access (the allocation may live on another GPU);
 *     *base = the mapping (pass to wave_ipc_release), *dptr = base + offset.
 *   wave_ipc_release: unmaps a base returned by wave_ipc_import.
 * CUDA errors (e.g. a handle from the same process, VMM/expandable-segment
 * memory) are returned as WAVE_ERR_CUDA with the driver's message. */
WAVE_API wave_status wave_ipc_export(const void *dptr, void *handle64, int64_t *offset);
WAVE_API wave_status wave_ipc_import(const void *handle64, int64_t offset, void **base, void **dptr);
WAVE_API wave_status wave_ipc_release(void *base);

/* Advance nsteps steps on a z-slab with the halo exchange fused into the
 * compute: every step (a) waits until both neighbours have completed the
 * previous step (acquire loads of my_flags), (b) runs the interior and wall
 * kernels over all local planes; CTAs that compute planes [0,4) / [nz-4,nz)
 * also store them straight into the lower / upper neighbour's ghost planes of
 * the next buffer, (c) adds the source (mirrored into the neighbour's ghost if
 * on an edge plane), (d) publishes its completed-step count to both
 * neighbours (system-scope fence + release stores).  No NCCL in the step;
 * replayed from CUDA graphs. */
WAVE_API wave_status wave_step_peer(wave_plan *plan, int64_t nsteps, void *stream);

/* Bound of each peer wait in device time (default 300 s, or the environment
 * variable WAVE25_PEER_TIMEOUT_S at plan creation).  A wait that expires does
 * not trap: it records which neighbour was late in a device error word, the
 * run continues (its results are invalid) and wave_peer_check reports it.
 * Re-instantiates the peer graphs (call before stepping, on every rank). */
WAVE_API wave_status wave_set_peer_timeout(wave_plan *plan, double seconds);

/* Synchronises `stream` and returns WAVE_ERR_PEER if any peer wait of this
 * plan has expired since wave_set_peers / wave_set_state, else WAVE_OK. */
WAVE_API wave_status wave_peer_check(wave_plan *plan, void *stream);

/* Copy this slab's 4 edge planes of u^n (which = 1) or of the next buffer
 * (which = 0) into the neighbours' ghost planes (for a non-zero initial
 * state); enqueued on `stream`, no flag traffic. */
WAVE_API wave_status wave_push_halo(wave_plan *plan, int32_t which, void *stream);

/* ---- outputs ------------------------------------------------------------- */

/* Copy u^n (which = 0) or u^{n-1} (which = 1) to dst, dense [nz][ny][nx] fp32
 * in `where` memory.  A host destination synchronises `stream` and reports
 * pending asynchronous CUDA errors. */
WAVE_API wave_status wave_read(const wave_plan *plan, int32_t which, float *dst, int32_t where,
                      void *stream);

/* Device pointer to the first element (i,j,k) = (0,0,0) of u^n (which = 0) or
 * u^{n-1} (which = 1) inside its padded buffer; row pitch = pitch_x, plane
 * pitch = ny*pitch_x.  Zero-copy view; valid until the next step. */
WAVE_API wave_status wave_field_ptr(const wave_plan *plan, int32_t which, float **out);

/* max |u^n| into *h_maxabs (host); synchronises `stream`.  Returns
 * WAVE_ERR_UNSTABLE (with the step number in wave_last_error) when any value
 * is non-finite. */
WAVE_API wave_status wave_check_finite(wave_plan *plan, float *h_maxabs, void *stream);

/* Number of completed steps n (u^n is current). -1 on NULL. */
WAVE_API int64_t wave_step_index(const wave_plan *plan);

/* The dt in use (after auto resolution), 0 if unresolved or NULL. */
WAVE_API float wave_get_dt(const wave_plan *plan);

/* Number of kernel launches one wave_step(plan, 1) enqueues (for launch
 * accounting in benchmarks); -1 on NULL. */
WAVE_API int32_t wave_launches_per_step(const wave_plan *plan);

/* Exact number of kernel launches wave_step(plan, nsteps) enqueues from the
 * current state (two-step pairs, plus one single step for an odd count);
 * -1 on NULL or nsteps < 0. */
WAVE_API int64_t wave_launches(const wave_plan *plan, int64_t nsteps);

/* Time steps one interior-kernel launch advances: 2 when wave_step runs
 * two-step temporal blocking (WAVE_KERNEL_TB2 with aux buffers bound on a
 * plan whose geometry supports it), else 1; -1 on NULL. */
WAVE_API int32_t wave_steps_per_launch(const wave_plan *plan);

/* ---- measurement --------------------------------------------------------- */

/* Kernel kinds of one time step (index into the arrays below). */
enum { WAVE_KK_INTERIOR = 0, WAVE_KK_XWALLS = 1, WAVE_KK_YWALLS = 2, WAVE_KK_SOURCE = 3,
       WAVE_KK_N = 4 };

/* Points each kernel kind computes per step (interior column incl. z caps,
 * x walls, y walls, source = 1 if owned), for algorithmic-byte accounting
 * (16 B per point-step).  With two-step blocking the interior
 * entry is the points of the two-step launch (it advances them two steps per
 * launch: 20 B per point per launch) and the wall entries are the points of
 * the two single-step wall phases of a pair divided by 2.  out[WAVE_KK_N]. */
WAVE_API wave_status wave_kernel_points(const wave_plan *plan, int64_t *out);

/* Like wave_step (same kernels and launch configurations, direct launches
 * instead of the CUDA graph) but serialized on `stream` with a CUDA event pair
 * around every kernel launch, so each pair times one kernel alone.  With
 * two-step blocking nsteps must be even; the interior kind then counts one
 * launch per two steps.
 * Synchronises `stream` at the end and returns
 * the summed device time of each kernel kind over the nsteps in
 * kernel_ms[WAVE_KK_N] and the number of launches of each kind in
 * launches[WAVE_KK_N] (either may be NULL).  Single-slab plans only. */
WAVE_API wave_status wave_step_profiled(wave_plan *plan, int64_t nsteps, void *stream,
                                        double *kernel_ms, int64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* WAVE25_WAVE_H */
