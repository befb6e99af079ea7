/*
 * rk_b200.h — C-ABI of librkb200.so: B200-native explicit Runge–Kutta time stepping of a
 * block-distributed fp64 state (the data-parallel hot path of arxiv 2309.05331,
 * "OpenFPM + Boost.Odeint distributed algebra").
 *
 * Citations: P:Lnn = PAPER.md line nn; S:Lnn = SPEC.md line nn; DESIGN.md R-n = a
 * recorded reading of the paper where it is silent, garbled or self-contradictory.
 *
 * Conventions (all entry points):
 *   - Return an rk_status; never abort or throw across the ABI.  On failure the message
 *     is available from rk_last_error() (thread-local).  CUDA/NCCL errors poison the ctx:
 *     every later call on it returns RK_ERR_CUDA / RK_ERR_NCCL.
 *   - Handles are opaque, created and destroyed by the caller.  The library owns all
 *     device buffers it allocates; pointers passed in are borrowed for the call only.
 *   - All device work is ordered on the ctx compute stream (the stream given to
 *     rk_ctx_create, normally torch's current stream).  Calls that return host values
 *     (step counts, norms, error ratios) synchronise that stream.
 *   - "Collective" calls must be made by every rank of the ctx, in the same order and
 *     with identical scalar arguments (MPI style), because they exchange halos (NCCL
 *     send/recv over NVLink) or reduce (NCCL allreduce max).
 *   - Floating point: fp64 throughout, IEEE division, no FMA contraction, no flush to
 *     zero.  Sums run left to right in increasing stage index and skip zero Butcher
 *     coefficients (R-17), so results are bitwise identical for any number of
 *     GPUs ("the same, regardless of the degree of parallelism").
 *
 * Data layout of a state's local block (host or device arrays in rk_state_set/get):
 *   grid state   (Gray–Scott):   [z][c][y][x], x fastest; the rank owns global planes
 *                                z in [begin, begin+count) of a z-slab partition.
 *   vector state (exp/logistic): [c][i]; the rank owns elements [begin, begin+count) of
 *                                every component.
 *   Partition rule: Nz (or N) split into world contiguous blocks; the remainder goes one
 *   each to the lowest ranks.  Every rank must own >= 1 plane / element.
 */
#ifndef RK_B200_H
#define RK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RK_ABI_VERSION 5
#define RK_UNIQUE_ID_BYTES 128

typedef struct rk_ctx_s* rk_ctx;     /* one per rank: device, streams, NCCL communicator */
typedef struct rk_state_s* rk_state; /* a distributed state plus its stage workspace      */

typedef enum {
    RK_OK = 0,
    RK_ERR_ARG = 1,          /* invalid argument (dt <= 0, t1 <= t0, atol <= 0, rtol < 0,
                                ncomp not in [1,6], dims <= 0, a rank owning no plane ...) */
    RK_ERR_CONTRACT = 2,     /* shape mismatch (lincomb), arity k not in [1,14]   */
    RK_ERR_UNSUPPORTED = 3,  /* adaptive stepping with a scheme without error estimate   */
    RK_ERR_STATE = 4,        /* RHS unset; Gray–Scott on a vector state or ncomp != 2     */
    RK_ERR_DIVERGED = 5,     /* non-finite error ratio (NaN) during adaptive stepping, or a
                                non-finite state found by RK_OPT_CHECK_FINITE (the
                                time is in the message and in rk_stats.diverged_t)       */
    RK_ERR_DT_UNDERFLOW = 6, /* adaptive dt fell below 16*eps*max(|t|,1)                  */
    RK_ERR_STALL = 7,        /* more than 500 tries for one step (Odeint default)         */
    RK_ERR_CUDA = 8,         /* CUDA error; the ctx is poisoned                           */
    RK_ERR_NCCL = 9,         /* NCCL error; the ctx is poisoned                           */
    RK_ERR_OOM = 10          /* device allocation failed                                  */
} rk_status;

/* Table 1, the explicit one-step rows on the hot path.  CK54 and DOPRI5 are
 * used fixed-step (do_step / integrate_const) or error-controlled (integrate_adaptive),
 * reproducing both the "fixed" and "dynamic step size" rows of Table 1. */
typedef enum {
    RK_EULER = 0,        /* explicit Euler, order 1                               */
    RK_RK4 = 1,          /* classic Runge–Kutta 4                                 */
    RK_CASH_KARP54 = 2,  /* Cash–Karp 5(4), fixed or error-controlled      */
    RK_DOPRI5 = 3,       /* Dormand–Prince 5(4), FSAL, fixed or error-controlled  */
    RK_FEHLBERG78 = 4,   /* Runge–Kutta–Fehlberg 7(8), fixed or error-controlled  */
    RK_EXPLICIT_MIDPOINT = 5, /* explicit midpoint rule, order 2: Euler half step, then the
                                 full step with the midpoint slope (R-22)  */
    RK_MIDPOINT = RK_EXPLICIT_MIDPOINT, /* (ABI v2 name of the same scheme)                   */
    RK_MODIFIED_MIDPOINT = 6, /* modified midpoint, order 2 (Table 1) = Odeint's
                                 modified_midpoint: Gragg's scheme with 2 substeps h = dt/2,
                                 3 RHS evaluations; computed in its Butcher form c = (0,1/2,1),
                                 a21 = 1/2, a32 = 1, b = (1/4,1/2,1/4) (R-22, R-17) */
    /* Adams–Bashforth k-step, order k, fixed dt only (Table 1 multi-step row).
     * The state keeps the last k-1 slopes F(u_{n-j}); the first k-1 steps after any other
     * change of u (set, another scheme, a new dt) are RKF78 bootstrap steps (R-23).
     * u_{n+1} = u_n + dt*sum_{j<k} beta_j F(u_{n-j}), summed newest first (R-24).          */
    RK_ADAMS_BASHFORTH1 = 11, RK_ADAMS_BASHFORTH2 = 12, RK_ADAMS_BASHFORTH3 = 13,
    RK_ADAMS_BASHFORTH4 = 14, RK_ADAMS_BASHFORTH5 = 15, RK_ADAMS_BASHFORTH6 = 16,
    RK_ADAMS_BASHFORTH7 = 17, RK_ADAMS_BASHFORTH8 = 18,
    /* Adams–Bashforth–Moulton k, PECE, order k, fixed dt only (Table 1; DESIGN.md
     * R-26): the AB_k history and start-up above, then per step f_n = F(u_n),
     * u_p = u_n + dt*sum_j beta_j f_{n-j}, u_{n+1} = u_n + dt*(m_0 F(u_p) + sum_{j>=1} m_j
     * f_{n-j+1}) with the k-term Adams–Moulton weights m (newest first); 2 RHS per step.     */
    RK_ADAMS_BASHFORTH_MOULTON1 = 21, RK_ADAMS_BASHFORTH_MOULTON2 = 22,
    RK_ADAMS_BASHFORTH_MOULTON3 = 23, RK_ADAMS_BASHFORTH_MOULTON4 = 24,
    RK_ADAMS_BASHFORTH_MOULTON5 = 25, RK_ADAMS_BASHFORTH_MOULTON6 = 26,
    RK_ADAMS_BASHFORTH_MOULTON7 = 27, RK_ADAMS_BASHFORTH_MOULTON8 = 28
} rk_scheme;

/* Options for rk_set_option. */
typedef enum {
    RK_OPT_HALO_OVERLAP = 1, /* 1 (default): interior stencil overlaps the halo exchange;
                                0: exchange first, then one full-slab launch              */
    RK_OPT_HALO_LOOPBACK = 2,/* world==1 only: 1 runs the multi-GPU halo path (pack, ghost
                                planes, interior+boundary launches) with a device-to-device
                                self-exchange instead of in-kernel periodic wrap (testing) */
    RK_OPT_MAX_TRIES = 3,    /* adaptive: tries per step before RK_ERR_STALL (default 500) */
    RK_OPT_TIMING = 4,       /* 1: time every stage-kernel launch with CUDA events (stats) */
    RK_OPT_USE_GRAPH = 5,    /* 1: rk_integrate_const of a grid (world == 1, no loopback, >= 5
                                steps) replays pairs of steps from one captured CUDA graph
                                (SURVEY f3): identical results, no per-launch host cost   */
    RK_OPT_DEVICE_LOOP = 6,  /* 1: rk_integrate_adaptive without a host round trip per try
                                (R-27): a vector state, or a grid within
                                RK_OPT_COOP_MAX_CELLS (one GPU, no halo path), runs as one
                                cooperative kernel; any other Gray–Scott grid -- one GPU, or the
                                P2P transport at any world -- as ONE CUDA-graph launch (a
                                conditional WHILE node over the try's stage launches and a
                                controller kernel; RK_OPT_TIMING and RK_OPT_CHECK_FINITE off).
                                Same results bit for bit; otherwise (NCCL transport) the host
                                loop is used.                                               */
    RK_OPT_HALO_P2P = 7,     /* halo path (world > 1 or HALO_LOOPBACK): 1 replaces NCCL by
                                peer-to-peer stores and atomics -- the pack kernel writes Y_i's
                                boundary planes straight into the neighbours' (double-buffered)
                                ghost planes through CUDA IPC mappings over NVLink and raises
                                their ready flags; the boundary launch waits on them and hands
                                the buffers back; the error-ratio / norm allreduce(max) is
                                atomicMax into every rank's mapped flag block plus an arrival
                                barrier.  The stage sequence numbers live on the
                                device, so RK_OPT_DEVICE_LOOP also runs on this transport.
                                Collective: set it on every rank; with NCCL the first use maps
                                the peers (NCCL all-gather of IPC handles), without NCCL see
                                rk_p2p_export.  Same results bit for bit.                   */
    RK_OPT_CONTROLLER = 8,   /* error-control reading (P:L42 fixes the semantics only):
                                0 (default) Odeint's (R-12): r = |e|/(atol + rtol*
                                (|u| + dt*|k1|)), reject if E > 1 with dt *= max(0.9E^(-1/(q-1)),
                                0.2), grow only below E = 0.5;  1 SPEC's elementary controller
                                (R-28): r = |e|/(atol + rtol*max(|u|,
                                |u_new|)), accept iff E <= 1, dt *= min(5, max(0.2, 0.9E^(-1/p)))
                                on accept, max(0.2, 0.9E^(-1/(p-1))) on reject, p = the scheme's
                                order.  Applies to rk_try_step and rk_integrate_adaptive.    */
    RK_OPT_CHECK_FINITE = 9, /* n >= 1: after every n-th completed step (and at the end of an
                                integrate call) check the state with the max-norm reduction;
                                a NaN/Inf gives RK_ERR_DIVERGED at that t.  Costs one
                                state read per check (vector integrate_const: the n steps run
                                in one launch).  0 (default): no check.                   */
    RK_OPT_COOP_MAX_CELLS = 10,/* fixed RK steps (do_step / integrate_const) of a Gray–Scott grid
                                with at most this many cells, one GPU, no halo path, run as one
                                persistent cooperative launch (all stages of all steps, grid-
                                wide barrier between stages): same results bit for
                                bit, no per-stage launch cost.  Default 2^18 (64^3); 0 = off. */
    RK_OPT_FUSED_STEP = 11,    /* temporal blocking of fixed RK4 / explicit- / modified-midpoint steps
                                of a Gray–Scott grid (above RK_OPT_COOP_MAX_CELLS), same
                                results bit for bit:
                                3 (default): K8 stage pairs -- two chained stages per launch,
                                the first on the tile grown by one cell and never stored (RK4:
                                two launches, 112 B/cell instead of 208; explicit midpoint: one,
                                32 B instead of 80); needs nx % 32 == 0 and
                                ny % 16 == 0, other grids run the stage-by-stage kernels;
                                Gragg's modified midpoint is pair (1, 2) + its last stage; on the NCCL multi-GPU slab the pairs'
                                2-deep ghost planes are exchanged before each pair (the P2P
                                transport keeps the stage-by-stage kernels); with 3 stages 2 + 3
                                and the last two stages of every error-controlled DOPRI5 try
                                are one K8 launch each (the head and the tail pair: a try is
                                4 launches, 384 B/cell instead of 432).  1 (one GPU, no halo path): K6, the whole step in ONE launch
                                with every stage value on chip (32 B/cell).  2: K7, K6 with
                                warp-specialised stage groups.  K6 and K7 are ablations, slower
                                than K8 and K3 on the B200.  0: stage-by-stage launches (K3). */
    RK_OPT_COMM_TIMEOUT_MS = 12,/* multi-GPU failure detection, applies to the state's context:
                                host waits on a stream with NCCL work poll the stream and
                                ncclCommGetAsyncError; an asynchronous NCCL error, or no
                                collective completing for this many ms (> 0; the clock restarts
                                whenever a collective issued by the ctx completes, and it is
                                off while no collective is outstanding, so it must exceed the
                                longest stretch of compute between two collectives, not the
                                whole queued backlog), aborts the communicator and
                                returns RK_ERR_NCCL (context poisoned).  0 (default): no
                                deadline (asynchronous errors are still detected).  >= 0.   */
    RK_OPT_ERROR_SPIKE = 13,  /* fault injection: n >= 1 -- the n-th error-controlled try
                                of this rank from now (host try loop) has its local error ratio
                                raised to at least 1e6 before the allreduce, forcing a rejection
                                on every rank (u unchanged, dt shrunk by the controller's floor).
                                Counted per rank; 0 (default): off.                          */
    RK_OPT_CHECK_ARGS = 14,   /* debug (SURVEY §8b "Collectives"): 1 -- every collective call
                                (do_step, try_step, integrate_*, norm_inf, eval_rhs) first
                                all-reduces a hash of its call kind and scalar arguments and
                                returns RK_ERR_CONTRACT on every rank when the ranks disagree
                                (a mismatched MPI-style call sequence).  Costs one host sync per
                                call.  0 (default): off.                                       */
    RK_OPT_FUSED_KERNELS = 15 /* 1 (default): the fused stage kernels (stage values formed inside
                                the RHS kernel, final combination and error ratio in the last
                                stage's epilogue).  0: the unfused, Odeint-like dataflow (SURVEY
                                §8b; the f4 ablation): per stage one lincomb launch
                                writes Y_i and one RHS launch k_i = F(Y_i), then lincomb
                                launches for u_new and the error estimate and a ratio-max
                                launch -- every intermediate through HBM, the same sums in the
                                same order, so bitwise the same results.  Runge–Kutta schemes,
                                fixed and error-controlled (host loop); Adams steps unaffected.*/
} rk_option;

/* Counters since creation or the last rk_reset_stats. */
typedef struct {
    int64_t rhs_evals;        /* stage RHS evaluations (per rank)                         */
    int64_t steps;            /* completed fixed steps                                    */
    int64_t tries;            /* adaptive tries                                           */
    int64_t accepted;         /* adaptive accepted tries                                  */
    int64_t rejected;         /* adaptive rejected tries                                  */
    int64_t kernel_launches;  /* kernels launched by this library                         */
    int64_t halo_exchanges;   /* halo exchanges (one per stage that needs ghost planes)   */
    int64_t halo_bytes;       /* bytes sent by this rank in halo exchanges                */
    int64_t stage_launches;   /* Gray–Scott stage-kernel launches                         */
    double stage_kernel_ms;   /* sum of their durations (RK_OPT_TIMING=1, else 0)         */
    double halo_ms;           /* time of the halo exchanges on the comm stream (TIMING=1) */
    double last_err_ratio;    /* E of the last adaptive try                               */
    double last_dt;           /* dt proposed after the last adaptive try                  */
    int64_t stage_bytes;      /* algorithmic HBM bytes of the stage-kernel launches: per
                                 launch (1 + #k_j read) arrays read + arrays written, over
                                 the launch's cells; halo re-reads,
                                 ghost planes and reductions are not counted              */
    double diverged_t;        /* t at which RK_OPT_CHECK_FINITE found a non-finite state  */
    int64_t pair_launches;    /* of the stage launches: K8 stage-pair launches (ABI 4)    */
    double pair_kernel_ms;    /* ... their share of stage_kernel_ms (RK_OPT_TIMING=1)     */
    int64_t pair_bytes;       /* ... their share of stage_bytes                           */
    int64_t head_launches;    /* of the pair launches: DOPRI5 head pairs, stages 2 + 3 (ABI 5) */
    double head_kernel_ms;    /* ... their share of pair_kernel_ms (RK_OPT_TIMING=1)      */
    int64_t head_bytes;       /* ... their share of pair_bytes                            */
} rk_stats;

/* ---- library ------------------------------------------------------------------------ */
int rk_abi_version(void);
const char* rk_last_error(void);
/* Host-only helpers (no GPU needed). */
/* Partition rule above: rank's [begin, begin+count) of n_global items. */
rk_status rk_partition(int64_t n_global, int world, int rank, int64_t* begin, int64_t* count);
/* Library's Butcher tableau as doubles a[s*s], b[s], e[s] = b - bhat (exact rational rounded
 * once, R-11), c[s]; *s <= 13; *order, *err_order (0 if none). */
rk_status rk_tableau(rk_scheme scheme, double* a, double* b, double* e, double* c, int* s,
                     int* order, int* err_order);
/* Odeint default step adjuster (R-12/R-14) applied to E and *dt: returns 1 in
 * *accepted if E <= 1 (then dt grows when E < 0.5), 0 if rejected (dt shrinks). */
rk_status rk_controller(rk_scheme scheme, double E, double* dt, int* accepted);
/* The same for either reading of RK_OPT_CONTROLLER (0 Odeint R-12, 1 SPEC R-28). */
rk_status rk_step_adjust(rk_scheme scheme, int controller, double E, double* dt, int* accepted);

/* Per-stage halo exchange of a z-slab grid (P:L168, P:L176 ghost_get), as
 * executed by every stage on the comm stream.  Buffers hold padded planes of Y_i:
 *   send  = [plane 0 | plane nzl-1] (this rank's lowest and highest owned planes),
 *   ghost = [plane nzl (from up) | plane -1 (from down)].
 * Each message moves `nplanes` planes between plane slots of those buffers.  world == 1
 * (loopback) is one self-message; world == 2 one message each way (the only peer is both
 * neighbours); world >= 3 two sends and two receives.  Host-only (no GPU needed). */
typedef struct {
    int recv;        /* 0: send from the send buffer, 1: receive into the ghost buffer */
    int peer;        /* rank (== own rank for the world == 1 self-exchange)           */
    int slot;        /* first plane slot (0 or 1) in the buffer                        */
    int nplanes;     /* 1 or 2                                                          */
} rk_halo_msg;
typedef struct {
    int up, down;    /* periodic z-neighbours: (rank+1) % world, (rank-1+world) % world */
    int nmsg;
    rk_halo_msg msg[4]; /* in posting order (sends, then receives) */
} rk_halo_plan;
rk_status rk_halo_plan_get(int world, int rank, rk_halo_plan* out);

/* The ghost exchange of a K8 stage pair on the multi-GPU slab (RK_OPT_FUSED_STEP = 3, DESIGN.md
 * §7): the pair's source needs its 2 boundary planes from each neighbour, its base (if any) 1.
 * Messages in posting order -- all sends (to up before to down), then all receives (from down
 * before from up) -- so that world 2 (one peer is both neighbours) and world 1 (self) pair each
 * send with the right receive under in-order matching per peer. */
typedef struct {
    int recv;        /* 0: send slab planes, 1: receive into a ghost array              */
    int peer;        /* rank                                                          */
    int array;       /* 0: the source (2-deep ghosts), 1: the base (1-deep ghosts)    */
    int side;        /* send: 0 the slab's bottom planes, 1 its top planes; receive: 0 the
                        ghosts below the slab (planes -n..-1), 1 above (nzl..nzl+n-1) */
    int nplanes;     /* 2 (source) or 1 (base)                                        */
} rk_pair_msg;
typedef struct {
    int up, down, nmsg;
    rk_pair_msg msg[8];
} rk_pair_plan;
rk_status rk_pair_ghost_plan(int world, int rank, int with_base, rk_pair_plan* out);

/* ---- context ------------------------------------------------------------------------ */
/* Rank 0 creates the NCCL unique id (RK_UNIQUE_ID_BYTES bytes); the caller broadcasts it
 * (torch.distributed) to all ranks before rk_ctx_create.  Not needed when world == 1. */
rk_status rk_nccl_unique_id(void* out);
/* Collective when world > 1.  device: CUDA ordinal; cuda_stream: cudaStream_t to order
 * work on (NULL = a new non-blocking stream owned by the ctx); uid: NULL if world == 1.
 * world > 1 with uid == NULL creates a context WITHOUT NCCL: its states use the P2P transport
 * only (RK_OPT_HALO_P2P forced on: halos and the error / norm allreduce run in this library's
 * kernels over CUDA IPC mappings), and the caller exchanges the IPC handles of each state with
 * rk_p2p_export / rk_p2p_import before its first collective call -- e.g. several processes
 * sharing one GPU (NCCL refuses two ranks on one device), or a launcher with its own
 * out-of-band channel. */
rk_status rk_ctx_create(int rank, int world, int device, const void* uid, void* cuda_stream,
                        rk_ctx* out);
rk_status rk_ctx_destroy(rk_ctx ctx);
/* Optional device allocator for the state arrays (u, u_new, the k_j / history / stage buffers,
 * halo send and ghost buffers), e.g. to route them through torch's caching allocator (SURVEY
 * §8b "allocator hook").  alloc(bytes, stream, user) returns device memory on the ctx device,
 * usable on `stream` (the ctx stream), or NULL (-> RK_ERR_OOM); free(ptr, stream, user) releases
 * it.  Both or neither (NULL, NULL: cudaMalloc / cudaFree, the default).  Must be set before the
 * first state is created (RK_ERR_STATE otherwise); the functions must stay valid until every
 * state is destroyed.  Buffers shared through CUDA IPC (P2P transport) always use cudaMalloc. */
typedef void* (*rk_alloc_fn)(size_t bytes, void* stream, void* user);
typedef void (*rk_free_fn)(void* ptr, void* stream, void* user);
rk_status rk_ctx_set_allocator(rk_ctx ctx, rk_alloc_fn alloc, rk_free_fn free_fn, void* user);

/* ---- state --------------------------------------------------------------------------- */
/* Distributed Nx x Ny x Nz periodic grid of ncomp fp64 components, z-slab partitioned
 * (R-20).  Collective. */
rk_status rk_state_create_grid(rk_ctx ctx, int64_t nx, int64_t ny, int64_t nz, int ncomp,
                               rk_state* out);
/* Distributed vector of n elements x ncomp components (block partition).  Collective. */
rk_status rk_state_create_vector(rk_ctx ctx, int64_t n, int ncomp, rk_state* out);
rk_status rk_state_destroy(rk_state st);
/* This rank's owned planes (grid) or elements (vector). */
rk_status rk_state_local_range(rk_state st, int64_t* begin, int64_t* count);
/* Number of fp64 values in this rank's block (count * ncomp * Nx * Ny for a grid). */
rk_status rk_state_local_size(rk_state st, int64_t* n_values);
/* Copy this rank's block in (set) or out (get), layout above.  on_device != 0: the pointer
 * is device memory on the ctx device (copied on the ctx stream); else host memory (pinned
 * or pageable).  Returns after the copy completes. */
rk_status rk_state_set(rk_state st, const double* src, int src_on_device);
rk_status rk_state_get(rk_state st, double* dst, int dst_on_device);

/* ---- right-hand sides --------------------------------------------------------------- */
/* du/dt = lambda*u, elementwise (Eq. 1a; R-9). */
rk_status rk_set_rhs_exponential(rk_state st, double lambda);
/* du/dt = u*(1-u), elementwise (Eq. 1b). */
rk_status rk_set_rhs_logistic(rk_state st);
/* 3D Gray–Scott, Listing 2 (R-1..R-3): grid state, ncomp==2.
 *   f0 = d1*Lap(C0) - C0*C1*C1 + F - F*C0,  f1 = d2*Lap(C1) + C0*C1*C1 - (F+K)*C1,
 * Lap = 7-point periodic central difference with spacing h (difference form). */
rk_status rk_set_rhs_gray_scott(rk_state st, double d1, double d2, double F, double K, double h);
rk_status rk_set_option(rk_state st, int key, int64_t value);

/* ---- stepping (all collective) ------------------------------------------------------ */
/* One explicit step u <- u + dt*sum_j b_j k_j in place ("do_step()"). */
rk_status rk_do_step(rk_state st, rk_scheme scheme, double t, double dt);
/* One error-controlled try: computes the embedded error ratio
 * E = max_i |e_i| / (atol + rtol*(|u_i| + dt*|k1_i|)) (R-12/R-13; or SPEC's ratio
 * under RK_OPT_CONTROLLER = 1), accepts (u <- u_new) iff E <= 1, and proposes the next dt.
 * CK54 / DOPRI5 / RKF78 only. */
rk_status rk_try_step(rk_state st, rk_scheme scheme, double t, double dt, double atol,
                      double rtol, int* accepted, double* err_ratio, double* dt_next);
/* Fixed-step loop of Odeint's integrate_const (R-15): steps while
 * (t_n + dt) - t1 <= eps, t_n = t0 + n*dt; *steps = n. */
rk_status rk_integrate_const(rk_state st, rk_scheme scheme, double t0, double t1, double dt,
                             int64_t* steps);
/* Error-controlled loop of Odeint's integrate_adaptive (R-16): advances
 * u from t0 to exactly t1; *accepted / *rejected count tries.  DOPRI5 reuses k7 as the next
 * k1 (FSAL); CK54 reuses k1 across retries. */
rk_status rk_integrate_adaptive(rk_state st, rk_scheme scheme, double t0, double t1, double dt0,
                                double atol, double rtol, int64_t* accepted, int64_t* rejected);

/* ---- algebra ops (P:L133-135 for_each# / for_each_norm) ------------------- */
/* out = sum_{j<k} coef[j]*in[j] elementwise, left to right, 1 <= k <= 14 (the paper's 15
 * participating states).  out may alias an input.  coef: host array. */
rk_status rk_lincomb(rk_state out, int k, const double* coef, const rk_state* in);
/* Global max |u| over all ranks (collective); NaN if any element is NaN. */
rk_status rk_norm_inf(rk_state st, double* out);
/* The right-hand side on its own: out.u = F(in.u) with in's RHS (Eq. 1a/1b, P:L208-209;
 * Listing 2), the same arithmetic as a fused stage (R-17); a grid
 * exchanges in's boundary planes first (collective when world > 1).  out: a state of the same
 * kind and shape (its own RHS is ignored), distinct from in.  Together with rk_lincomb it is the
 * unfused "native" stepping of the ablation.  Errors: RK_ERR_CONTRACT
 * on a shape mismatch, RK_ERR_ARG if out == in, RK_ERR_STATE if in has no RHS. */
rk_status rk_eval_rhs(rk_state in, rk_state out);

/* P2P transport (RK_OPT_HALO_P2P) without NCCL.  rk_p2p_export writes this rank's
 * CUDA IPC handles for the state (its double-buffered ghost planes and its flag block, both
 * allocated and zeroed here) into out (capacity bytes) and their size into *nbytes (out == NULL:
 * size query only).  The caller all-gathers them (any channel, e.g. torch.distributed over
 * gloo) and passes every rank's bytes, concatenated in rank order, to rk_p2p_import, which maps
 * the z-neighbours' ghost planes and every rank's flag block (the fused allreduce(max) writes
 * into all of them).  Collective; once per state, before its first step.  With NCCL the library
 * does this exchange itself on the first P2P stage.  Errors: RK_ERR_STATE if the state does not
 * use the P2P transport or is already connected, RK_ERR_ARG on a size mismatch, RK_ERR_CUDA if
 * a handle cannot be mapped. */
rk_status rk_p2p_export(rk_state st, void* out, int64_t capacity, int64_t* nbytes);
rk_status rk_p2p_import(rk_state st, const void* all, int64_t nbytes_per_rank);

rk_status rk_get_stats(rk_state st, rk_stats* out);
rk_status rk_reset_stats(rk_state st);

#ifdef __cplusplus
}
#endif
#endif /* RK_B200_H */
