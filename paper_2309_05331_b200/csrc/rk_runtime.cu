// rk_runtime.cu — host runtime behind the C-ABI (include/rk_b200.h).
//
// Context (device, compute + comm streams, NCCL communicator), distributed states
// (z-slab grid / block vector, ping-pong u/u_new, lazily sized k_j workspace, ghost
// planes), the stage scheduler (per stage: pack -> NCCL send/recv on the comm stream,
// overlapped with the interior stencil launch; boundary launch after the halo event),
// the drivers do_step / try_step / integrate_const / integrate_adaptive (Odeint loops,
// P:L198) and the host step-size controller (R-12).
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cfloat>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <initializer_list>
#include <string>
#include <utility>
#include <vector>

#include "rk_b200.h"
#include "rk_ddmath.cuh"
#include "rk_kernels.cuh"
#include "rk_tableau.h"

using namespace rkb;

// ------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------
static thread_local std::string g_err;

static rk_status fail(rk_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

struct rk_ctx_s {
    int rank = 0, world = 1, device = 0;
    cudaStream_t stream = nullptr, comm = nullptr;
    cudaStream_t bnd = nullptr;  // halo path: pack + boundary-plane launches, beside the interior
    bool own_stream = false;
    cudaStream_t capture = nullptr;  // private stream for CUDA-graph capture (RK_OPT_USE_GRAPH)
    ncclComm_t nccl = nullptr;
    int64_t comm_timeout_ms = 0;  // RK_OPT_COMM_TIMEOUT_MS: abort a collective wait after this
    int num_sms = 148;
    rk_status poisoned = RK_OK;
    unsigned long long* d_scratch = nullptr;  // 8 B reduction word (norm_inf)
    unsigned long long* h_scratch = nullptr;  // pinned
    std::vector<rk_state_s*> states;          // live states (destroyed with the ctx)
    // progress marks: an event recorded behind every collective; a host wait restarts its
    // RK_OPT_COMM_TIMEOUT_MS clock whenever one of them completes (ctx_wait)
    std::deque<cudaEvent_t> marks;
    std::vector<cudaEvent_t> mark_pool;
    // rk_ctx_set_allocator: the caller's device allocator for state arrays (e.g. torch's caching
    // allocator); null: cudaMalloc / cudaFree
    rk_alloc_fn alloc_fn = nullptr;
    rk_free_fn free_fn = nullptr;
    void* alloc_user = nullptr;
};

#define CK_CTX(ctx, call)                                                                     \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            (ctx)->poisoned = RK_ERR_CUDA;                                                    \
            return fail(RK_ERR_CUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_),   \
                        __FILE__, __LINE__, #call);                                           \
        }                                                                                     \
    } while (0)

#define NK_CTX(ctx, call)                                                                     \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess) {                                                              \
            (ctx)->poisoned = RK_ERR_NCCL;                                                    \
            return fail(RK_ERR_NCCL, "NCCL error %s at %s:%d", ncclGetErrorString(r_),        \
                        __FILE__, __LINE__);                                                  \
        }                                                                                     \
    } while (0)

#define TRY(call)                          \
    do {                                   \
        rk_status s_ = (call);             \
        if (s_ != RK_OK) return s_;        \
    } while (0)

// NVTX ranges (SURVEY §5 tracing): a try, a stage, a halo exchange, a whole-step launch and the
// integrate drivers show up by name in Nsight Systems / ncu --nvtx; header-only NVTX3, inert
// when no tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Record a progress mark behind a collective just enqueued on stream s (ctx_wait).
static void mark_progress(rk_ctx ctx, cudaStream_t s) {
    if (!ctx->nccl || ctx->comm_timeout_ms <= 0 || ctx->marks.size() >= 512) return;
    cudaEvent_t e = nullptr;
    if (!ctx->mark_pool.empty()) {
        e = ctx->mark_pool.back();
        ctx->mark_pool.pop_back();
    } else if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    if (cudaEventRecord(e, s) != cudaSuccess) {
        cudaGetLastError();
        ctx->mark_pool.push_back(e);
        return;
    }
    ctx->marks.push_back(e);
}

// Wait for stream s.  With a NCCL communicator the host polls instead of blocking, so an
// asynchronous NCCL error (a peer died, a link failed) or the RK_OPT_COMM_TIMEOUT_MS deadline
// aborts the communicator and returns RK_ERR_NCCL (the context is poisoned) instead of hanging
// in a collective forever (SURVEY §5 failure detection).  The deadline runs from the last
// PROGRESS: the start of the wait or the completion of the latest collective mark
// (mark_progress), so queued compute behind many collectives does not count against it -- only
// the longest stretch without a completed collective does -- and it is off once every
// collective issued so far has completed.
static rk_status ctx_wait(rk_ctx ctx, cudaStream_t s) {
    if (!ctx->nccl) {
        CK_CTX(ctx, cudaStreamSynchronize(s));
        return RK_OK;
    }
    auto t0 = std::chrono::steady_clock::now();
    for (unsigned spin = 0;; ++spin) {
        const cudaError_t q = cudaStreamQuery(s);
        while (!ctx->marks.empty() && cudaEventQuery(ctx->marks.front()) == cudaSuccess) {
            ctx->mark_pool.push_back(ctx->marks.front());
            ctx->marks.pop_front();
            t0 = std::chrono::steady_clock::now();
        }
        if (q == cudaSuccess) return RK_OK;
        if (q != cudaErrorNotReady) CK_CTX(ctx, q);
        ncclResult_t ar = ncclSuccess;
        NK_CTX(ctx, ncclCommGetAsyncError(ctx->nccl, &ar));
        // the deadline only applies while a collective is outstanding (a mark not yet reached):
        // plain compute queued behind the last completed collective cannot hang on a peer
        const bool late = ctx->comm_timeout_ms > 0 && !ctx->marks.empty() &&
                          std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(ctx->comm_timeout_ms);
        if ((ar != ncclSuccess && ar != ncclInProgress) || late) {
            ncclCommAbort(ctx->nccl);
            ctx->nccl = nullptr;
            ctx->poisoned = RK_ERR_NCCL;
            if (late)
                return fail(RK_ERR_NCCL, "no collective progress for %lld ms on rank %d: communicator aborted",
                            (long long)ctx->comm_timeout_ms, ctx->rank);
            return fail(RK_ERR_NCCL, "asynchronous NCCL error %s on rank %d: communicator aborted",
                        ncclGetErrorString(ar), ctx->rank);
        }
        if (spin >= 256) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

// Teardown wait: a context poisoned by a NCCL failure may have kernels spinning on peer flags
// (P2P halos) that the abort does not release, so its streams are drained for a bounded time
// only (then the buffers are leaked rather than freed under a running kernel).
static bool drain_stream(rk_ctx ctx, cudaStream_t s) {
    if (!s) return true;
    if (ctx->poisoned != RK_ERR_NCCL) return cudaStreamSynchronize(s) == cudaSuccess;
    const auto t0 = std::chrono::steady_clock::now();
    const auto lim = std::chrono::milliseconds(std::max<int64_t>(ctx->comm_timeout_ms, 2000));
    while (cudaStreamQuery(s) == cudaErrorNotReady) {
        if (std::chrono::steady_clock::now() - t0 > lim) return false;
        std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
    cudaGetLastError();
    return true;
}

// Every API call runs on its context's device, from any host thread: cudaSetDevice also binds the
// device's primary context to a thread that has made no CUDA call yet, which the driver-API calls
// (cuTensorMapEncodeTiled) need -- cudaGetDevice alone reports device 0 there without binding it.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// ------------------------------------------------------------------------------------
// state
// ------------------------------------------------------------------------------------
struct TimedPair {
    cudaEvent_t a, b;
    int kind;  // 0 stage kernel, 1 halo, 2 K8 pair, 3 K8 DOPRI5 head pair
};

// the four TMA maps of one padded grid array: [0]/[1] ring / interior box of 32x8 tiles,
// [2]/[3] of 32x16 tiles (rk_kernels.cuh encode_grid_maps)
struct Maps {
    CUtensorMap m[4];
};

struct rk_state_s {
    rk_ctx ctx = nullptr;
    bool grid = false;
    int ncomp = 1;
    int64_t nx = 1, ny = 1, nz = 1;  // grid (global dims)
    int64_t n = 0;                   // vector: global elements
    int64_t begin = 0, local = 0;    // owned planes (grid) or elements (vector)
    int64_t count = 0;               // fp64 values in the local block (user layout)
    int64_t alloc = 0;               // fp64 values per device array (padded layout for grids)
    GridGeom geo{};                  // padded periodic layout (grid states, rk_kernels.cuh)
    double* u = nullptr;
    double* u_new = nullptr;
    double* k[13] = {nullptr};
    Maps tm_u{}, tm_unew{}, tm_k[13]{};  // TMA maps per array (encode_grid_maps)
    Maps tm_glo{}, tm_ghi{};
    int nk = 0;
    bool k1_valid = false;           // k[0] == F(u) for the current u
    // Adams–Bashforth history: hist[0..ab_count) = f_{n-1}, f_{n-2}, ... (newest first),
    // hist[ab_k-1] is the scratch slot that receives f_n; valid for (ab_k, ab_dt) only
    int ab_k = 0, ab_count = 0, nhist = 0;
    double ab_dt = 0.0;
    double* hist[8] = {nullptr};
    double* ybuf[2] = {nullptr};     // K5 stage values (RK_OPT_COOP_MAX_CELLS)
    unsigned int* k5bar = nullptr;   // K5 grid-barrier words (arrivals, generation), zeroed once
    Maps tm_hist[8]{};
    // halo (grid, world > 1 or loopback)
    double* sendbuf = nullptr;       // [lo plane | hi plane]
    double* ghostbuf = nullptr;      // [ghost_hi | ghost_lo] (so one message serves world==2)
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_bnd = nullptr;  // stage start on the compute stream / boundary done
    // peer-to-peer halo (RK_OPT_HALO_P2P): the pack kernel stores Y_i's boundary planes straight
    // into the neighbours' ghost planes (CUDA IPC over NVLink) with a flag handshake
    bool p2p = false, p2p_ready = false;
    double* pghost = nullptr;               // [parity][ghost_hi, ghost_lo][plane], written by peers
    unsigned long long* pflags = nullptr;   // this rank's flag block (rk_kernels.cuh P2pFlag)
    double* peer_ghost[2] = {};             // [0] lower neighbour's pghost, [1] upper's
    unsigned long long* peer_flags[2] = {};
    unsigned long long* rank_flags[P2P_MAX_WORLD] = {};  // every rank's flag block (allreduce)
    std::vector<void*> ipc_mapped;          // IPC mappings to close on destroy
    Maps tm_pg[2][2]{};                     // [parity][0 ghost_hi, 1 ghost_lo]
    unsigned long long* d_err = nullptr;
    unsigned long long* h_err = nullptr;
    // K8 DOPRI5 tail pair on the multi-GPU / loopback slab: 2-deep ghost planes of Y_6, 1-deep of W
    double* pg_y = nullptr;  // [-2, -1 | nzl, nzl+1]
    double* pg_w = nullptr;  // [-1 | nzl]
    CUtensorMap tm_pgy_lo{}, tm_pgy_hi{};
    Maps tm_pgw_lo{}, tm_pgw_hi{};
    // K8 RK4 pairs on the slab: u's ghosts (pg_y, also viewed 1-deep for pair (3,4)'s base) and Y_3's
    double* pg_y2 = nullptr;
    CUtensorMap tm_pgy2_lo{}, tm_pgy2_hi{};
    Maps tm_pgu_lo{}, tm_pgu_hi{};
    // rhs
    int rhs = RHS_NONE;
    double lambda = 0.0, d1 = 0.0, d2 = 0.0, F = 0.0, K = 0.0, h = 1.0;
    // options
    bool overlap = true, loopback = false, timing = false, use_graph = false, device_loop = false;
    unsigned long long* d_loop = nullptr;  // device loop: [3] error-max slots + PwLoopResult
    int max_tries = 500;
    int controller = 0;          // RK_OPT_CONTROLLER: 0 Odeint (R-12), 1 SPEC (R-28)
    int64_t check_finite = 0;    // RK_OPT_CHECK_FINITE: check u every n steps (0: never)
    int64_t since_check = 0;     // steps since the last finiteness check
    int64_t coop_max_cells = 1 << 18;  // RK_OPT_COOP_MAX_CELLS: persistent-step path up to here
    int fused = 3;               // RK_OPT_FUSED_STEP: 3 K8 stage pairs (default), 1 K6 / 2 K7 whole steps, 0 stage by stage
    int64_t spike_at = 0, spike_seen = 0;  // RK_OPT_ERROR_SPIKE: inject at try number spike_at
    bool fused_kernels = true;   // RK_OPT_FUSED_KERNELS = 0: Odeint-like unfused stages (ablation)
    double* uf_y = nullptr;      // unfused: the stage value Y_i and the error estimate e
    double* uf_e = nullptr;
    Maps tm_uf_y{};
    bool check_args = false;     // RK_OPT_CHECK_ARGS: hash-compare collective call arguments
    const double* gl_dtp = nullptr;  // set while capturing the device-resident try loop (GLoop)
    struct GraphLoop* gloop = nullptr;
    // stats
    rk_stats stats{};
    std::vector<TimedPair> pending;
    std::vector<cudaEvent_t> event_pool;
};

static rk_status check_state(rk_state st) {
    if (!st || !st->ctx) return fail(RK_ERR_ARG, "null state");
    if (st->ctx->poisoned != RK_OK) return fail(st->ctx->poisoned, "context poisoned by an earlier CUDA/NCCL error");
    return RK_OK;
}

// State arrays: through the caller's allocator when one is set (rk_ctx_set_allocator), else
// cudaMalloc.  Buffers shared with other processes (P2P ghost planes, flags) always use cudaMalloc
// (CUDA IPC needs whole allocations).
static rk_status dev_alloc(rk_ctx ctx, double** p, int64_t count) {
    const size_t bytes = sizeof(double) * (size_t)std::max<int64_t>(count, 1);
    if (ctx->alloc_fn) {
        *p = static_cast<double*>(ctx->alloc_fn(bytes, (void*)ctx->stream, ctx->alloc_user));
        if (!*p) return fail(RK_ERR_OOM, "the caller's allocator returned NULL for %zu bytes", bytes);
        return RK_OK;
    }
    cudaError_t e = cudaMalloc((void**)p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(RK_ERR_OOM, "cudaMalloc of %lld doubles failed: %s", (long long)count,
                    cudaGetErrorString(e));
    }
    return RK_OK;
}

static void dev_free(rk_ctx ctx, void* p) {
    if (!p) return;
    if (ctx->free_fn) ctx->free_fn(p, (void*)ctx->stream, ctx->alloc_user);
    else cudaFree(p);
}

// zero-filled array (pads and ring corners stay 0) with its TMA tensor maps (grids)
static rk_status alloc_array(rk_state st, double** p, Maps* tm) {
    TRY(dev_alloc(st->ctx, p, st->alloc));
    CK_CTX(st->ctx, cudaMemsetAsync(*p, 0, sizeof(double) * (size_t)st->alloc, st->ctx->stream));
    if (st->grid && st->ncomp == 2 && tm)
        CK_CTX(st->ctx, encode_grid_maps(tm->m, *p, st->geo, (int)st->local));
    return RK_OK;
}

static rk_status ensure_k(rk_state st, int nk) {
    for (int j = st->nk; j < nk; ++j) {
        TRY(alloc_array(st, &st->k[j], &st->tm_k[j]));
        st->nk = j + 1;
    }
    return RK_OK;
}

// u changes: whatever k1 held is F(old u) now (an accepted FSAL try re-validates it after)
static void swap_u(rk_state st) {
    std::swap(st->u, st->u_new);
    std::swap(st->tm_u, st->tm_unew);
    st->k1_valid = false;
}

static void swap_k(rk_state st, int i, int j) {
    std::swap(st->k[i], st->k[j]);
    std::swap(st->tm_k[i], st->tm_k[j]);
}

static int64_t plane_values(rk_state st) { return st->geo.ps; }  // one padded plane, 2 comps

static cudaEvent_t pool_event(rk_state st) {
    if (!st->event_pool.empty()) {
        cudaEvent_t e = st->event_pool.back();
        st->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

static rk_status resolve_timing(rk_state st) {
    if (st->pending.empty()) return RK_OK;
    rk_ctx ctx = st->ctx;
    TRY(ctx_wait(ctx, ctx->stream));
    if (ctx->comm) TRY(ctx_wait(ctx, ctx->comm));
    if (ctx->bnd) TRY(ctx_wait(ctx, ctx->bnd));
    for (auto& p : st->pending) {
        float ms = 0.f;
        CK_CTX(ctx, cudaEventElapsedTime(&ms, p.a, p.b));
        if (p.kind == 1) st->stats.halo_ms += ms;
        else st->stats.stage_kernel_ms += ms;
        if (p.kind >= 2) st->stats.pair_kernel_ms += ms;  // K8 stage-pair launches
        if (p.kind == 3) st->stats.head_kernel_ms += ms;  // ... the DOPRI5 head pairs
        st->event_pool.push_back(p.a);
        st->event_pool.push_back(p.b);
    }
    st->pending.clear();
    return RK_OK;
}

// ------------------------------------------------------------------------------------
// stage plans: the compile-time StageSpec table (rk_stage_spec.h) + this step's values
// ------------------------------------------------------------------------------------
struct Coeffs {
    int s = 0, order = 0, err_order = 0;
    double a[13][13] = {{0}}, b[13] = {0}, e[13] = {0}, c[13] = {0};
};

static Coeffs coeffs_of(int scheme) {
    Coeffs C;
    const Tableau T = tableau_of(scheme);
    C.s = T.s;
    C.order = T.order;
    C.err_order = T.err_order;
    for (int i = 0; i < T.s; ++i) {
        for (int j = 0; j < i; ++j) C.a[i][j] = rat_double(T.a[i][j]);
        C.b[i] = rat_double(T.b[i]);
        C.e[i] = rat_double(err_weight(T, i));
        C.c[i] = rat_double(T.c[i]);
    }
    return C;
}

static bool valid_scheme(int s) { return (s >= RK_EULER && s <= RK_MODIFIED_MIDPOINT) || is_multistep(s); }

struct StagePlan {
    int scheme = 0, adaptive = 0, stage = 0;
    StageSpec sp{};
    double g[kMaxSlots] = {0}, beta[kMaxSlots] = {0}, delta[kMaxSlots] = {0};
    double beta_new = 0.0, delta_new = 0.0;
    double g2[kMaxSlots] = {0}, g2_new = 0.0;  // EPI_AHEAD: the final stage's a_Fj (x dt)
    double g3[kMaxSlots] = {0}, g3_new = 0.0;  // EPI_AHEAD with out_z: the last stage's a_Lj (x dt)
    int out_hist = -1;  // >= 0: the stage writes its k into Adams–Bashforth history slot
    double* out_ptr = nullptr;  // non-null: the stage's k goes here (rk_eval_rhs)
};

// adaptive: 0 fixed step, 1 error-controlled (Odeint ratio, R-12), 2 error-controlled (SPEC
// ratio, R-28)
// adaptive == 5: a fixed step whose last two stages run as one K8 pair (fixed_tail_pair): the
// plan holds stages 0 .. L-2, the last of them the write-ahead stage with Z_L (stage_spec ad 5)
static std::vector<StagePlan> build_plan(int scheme, int adaptive, double dt) {
    const Coeffs C = coeffs_of(scheme);
    std::vector<StagePlan> plan;
    const int n = adaptive == 5 ? last_stage(tableau_of(scheme), false) - 1 : num_stages(scheme, adaptive);
    for (int i = 0; i < n; ++i) {
        StagePlan p;
        p.scheme = scheme;
        p.adaptive = adaptive == 5 && i < n - 1 ? 0 : adaptive;
        p.stage = i;
        p.sp = stage_spec(scheme, p.adaptive, i);
        for (int s = 0; s < p.sp.nslots; ++s) {
            const int j = p.sp.j[s];
            p.g[s] = p.sp.gnz[s] ? dt * C.a[i][j] : 0.0;
            p.beta[s] = p.sp.bnz[s] ? dt * C.b[j] : 0.0;
            p.delta[s] = p.sp.dnz[s] ? dt * C.e[j] : 0.0;
        }
        p.beta_new = p.sp.bnew ? dt * C.b[i] : 0.0;
        p.delta_new = p.sp.dnew ? dt * C.e[i] : 0.0;
        if (p.sp.epi == EPI_AHEAD) {
            for (int s = 0; s < p.sp.nslots; ++s) p.g2[s] = p.sp.anz2[s] ? dt * C.a[i + 1][p.sp.j[s]] : 0.0;
            p.g2_new = p.sp.a2new ? dt * C.a[i + 1][i] : 0.0;
            if (p.sp.out_z >= 0) {
                for (int s = 0; s < p.sp.nslots; ++s) p.g3[s] = p.sp.anz3[s] ? dt * C.a[i + 2][p.sp.j[s]] : 0.0;
                p.g3_new = p.sp.a3new ? dt * C.a[i + 2][i] : 0.0;
            }
        }
        plan.push_back(p);
    }
    return plan;
}

static int plan_num_k(const std::vector<StagePlan>& plan) {
    int nk = 0;
    for (auto& p : plan) {
        if (p.sp.out_k >= 0) nk = std::max(nk, p.sp.out_k + 1);
        nk = std::max(nk, std::max(std::max(p.sp.out_w, p.sp.out_z), std::max(p.sp.out_e, p.sp.base_src)) + 1);
        for (int s = 0; s < p.sp.nslots; ++s)
            if (p.sp.src[s] >= 0) nk = std::max(nk, p.sp.src[s] + 1);
    }
    return nk;
}

static bool is_ratio_stage(const StagePlan& p) {
    return p.sp.epi == EPI_FINAL_ERR || p.sp.epi == EPI_TAIL_ERR;
}

// ------------------------------------------------------------------------------------
// Gray–Scott stage execution
// ------------------------------------------------------------------------------------
static bool halo_path(rk_state st) { return st->ctx->world > 1 || st->loopback; }

// The collectives of a state run through NCCL on the multi-GPU path and on the one-GPU
// loopback path; the latter uses a 1-rank communicator (ncclSend / ncclRecv to self, a 1-rank
// allreduce), so it executes exactly the NCCL calls of the multi-GPU run.
static bool use_nccl(rk_state st) { return st->ctx->nccl && halo_path(st); }

static rk_status ensure_self_comm(rk_ctx ctx) {
    if (ctx->nccl || ctx->world != 1) return RK_OK;
    ncclUniqueId id;
    NK_CTX(ctx, ncclGetUniqueId(&id));
    NK_CTX(ctx, ncclCommInitRank(&ctx->nccl, 1, id, 0));
    return RK_OK;
}

static rk_status ensure_halo(rk_state st) {
    if (st->loopback && !st->p2p) TRY(ensure_self_comm(st->ctx));  // the P2P transport needs no NCCL
    if (!halo_path(st) || st->sendbuf) return RK_OK;
    TRY(dev_alloc(st->ctx, &st->sendbuf, 2 * plane_values(st)));
    TRY(dev_alloc(st->ctx, &st->ghostbuf, 2 * plane_values(st)));
    CK_CTX(st->ctx, cudaMemsetAsync(st->ghostbuf, 0, sizeof(double) * 2 * plane_values(st), st->ctx->stream));
    CK_CTX(st->ctx, encode_grid_maps(st->tm_ghi.m, st->ghostbuf, st->geo, 1));
    CK_CTX(st->ctx, encode_grid_maps(st->tm_glo.m, st->ghostbuf + plane_values(st), st->geo, 1));
    CK_CTX(st->ctx, cudaEventCreateWithFlags(&st->ev_pack, cudaEventDisableTiming));
    CK_CTX(st->ctx, cudaEventCreateWithFlags(&st->ev_halo, cudaEventDisableTiming));
    CK_CTX(st->ctx, cudaEventCreateWithFlags(&st->ev_ready, cudaEventDisableTiming));
    CK_CTX(st->ctx, cudaEventCreateWithFlags(&st->ev_bnd, cudaEventDisableTiming));
    return RK_OK;
}

static GsStageArgs stage_args(rk_state st, const StagePlan& p, double dt, double atol, double rtol) {
    GsStageArgs a{};
    a.geo = st->geo;
    const int hb = 2 * (stage_rows(p.sp) - 1);  // map pair of this stage's tile height
    a.base = p.sp.base_src >= 0 ? st->k[p.sp.base_src] : (p.sp.base_unew ? st->u_new : st->u);
    a.tm_base = (p.sp.base_src >= 0 ? st->tm_k[p.sp.base_src] : (p.sp.base_unew ? st->tm_unew : st->tm_u)).m[hb];
    int ny = 0;
    const bool ab = is_multistep(p.scheme);  // slots are history entries, newest first
    for (int s = 0; s < p.sp.nslots; ++s) {
        const int src = p.sp.src[s];
        const int box = hb + (p.sp.halo[s] ? 0 : 1);
        a.slot[s] = ab ? st->hist[src] : (src >= 0 ? st->k[src] : st->u);
        a.tm_slot[s] = ab ? st->tm_hist[src].m[box] : (src >= 0 ? st->tm_k[src].m[box] : st->tm_u.m[box]);
        a.g[s] = p.g[s];
        a.beta[s] = p.beta[s];
        a.delta[s] = p.delta[s];
        a.g2[s] = p.g2[s];
        a.g3[s] = p.g3[s];
        if (p.sp.gnz[s]) ++ny;
    }
    a.nyslots = ny;
    a.beta_new = p.beta_new;
    a.delta_new = p.delta_new;
    a.out_k = p.out_ptr ? p.out_ptr
                        : (p.out_hist >= 0 ? st->hist[p.out_hist]
                                           : (p.sp.out_k >= 0 ? st->k[p.sp.out_k] : nullptr));
    a.out_u = p.sp.writes_u ? st->u_new : nullptr;
    a.g2_new = p.g2_new;
    a.out_w = p.sp.out_w >= 0 ? st->k[p.sp.out_w] : nullptr;
    a.out_e = p.sp.out_e >= 0 ? st->k[p.sp.out_e] : nullptr;
    a.g3_new = p.g3_new;
    a.out_z = p.sp.out_z >= 0 ? st->k[p.sp.out_z] : nullptr;
    a.errmax = st->d_err;
    a.dt = dt;
    a.dtp = st->gl_dtp;
    a.atol = atol;
    a.rtol = rtol;
    a.d1 = st->d1;
    a.d2 = st->d2;
    a.F = st->F;
    a.FK = st->F + st->K;
    a.inv_h2 = 1.0 / (st->h * st->h);
    a.z_lo = 0;
    a.z_hi = (int)st->local;
    a.zmode = 0;
    a.zpair = 0;  // set with the z chunk (pick_zchunk)
    return a;
}

// pack arguments: the Y terms only, compacted in stage order (left-to-right sum preserved)
static GsStageArgs pack_args(const GsStageArgs& a, const StagePlan& p) {
    GsStageArgs q = a;
    int n = 0;
    for (int s = 0; s < p.sp.nslots; ++s) {
        if (!p.sp.gnz[s] || p.sp.base_unew || p.sp.base_src >= 0) continue;
        q.slot[n] = a.slot[s];
        q.g[n] = a.g[s];
        ++n;
    }
    q.nyslots = n;
    return q;
}

// Planes per CTA.  Short z chunks keep y-neighbouring tiles (which re-read each other's
// ring rows through L2) progressing together; measured at 512^2 planes (profiles/r1_*tune*):
// 8 for Y-direct stages, 16 for other two-row stages and for the multi-output write-ahead
// stage (2.88 ms at 16 vs 3.26 at 32, 3.67 at 48 for DOPRI5's, gpurun_out tune_zc*), 48
// otherwise.  Small grids: shorten further so every SM gets work.
// Stage classes for the z-chunk policy: 0 Y-direct (no slot enters Y), 1 other two-row stages,
// 2 AHEAD / EPART, 3 the rest, 4 Adams–Bashforth with one or two history slots (Y-direct too;
// measured at 512^3: AB2 1.59 -> 1.48 ms, AB3 1.72 -> 1.68 ms at 4 planes instead of 8, while
// AB4 is flat and AB8 loses, gpurun_out zab2*)
static int stage_class(const StagePlan& p) {
    bool yd = true;
    for (int s = 0; s < p.sp.nslots; ++s) yd = yd && !p.sp.gnz[s];
    return yd ? (p.sp.epi == EPI_AB && p.sp.nslots > 0 && p.sp.nslots <= 2 ? 4 : 0)
              : (stage_rows(p.sp) == 2 ? 1 : (p.sp.epi == EPI_FINAL_EPART || p.sp.epi == EPI_AHEAD ? 2 : 3));
}

// Paired opposite-direction chunk sweeps (GsStageArgs::zpair, rk_stencil.cu) per stage class:
// measured per stage at 512^3 (ncu, profiles/r2_zpair_ab.txt) they cut the DRAM reads of the
// 16-plane classes 1 and 2 (write-ahead stage 12.18 -> 11.51 GB, 2.466 -> 2.424 ms; light
// k-stages 4.83 -> 4.61 GB) but add reads to the short Y-direct chunks and slow the 48-plane
// stages, so classes 1 and 2 only.  RKB_ZPAIR = class bitmask (developer knob).
static int stage_zpair(const StagePlan& p) {
    static int g[5] = {0, 0, 0, 0, 0};
    if (!g[0]) {  // developer knob RKB_ZPAIR="g0,g1,g2,g3,g4": chunk group size per stage class
        const int def[5] = {1, 2, 2, 1, 1};
        for (int c = 0; c < 5; ++c) g[c] = def[c];
        if (const char* e = getenv("RKB_ZPAIR")) {
            int v[5], n = sscanf(e, "%d,%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3], &v[4]);
            for (int c = 0; c < n; ++c) g[c] = v[c] > 0 ? v[c] : 1;
        }
    }
    return g[stage_class(p)];
}

static int pick_zchunk(rk_state st, const StagePlan& p, int range) {
    if (range <= 0) return 1;
    if (const char* e = getenv("RKB_ZCHUNK")) {  // developer tuning knob
        const int v = atoi(e);
        if (v > 0) return std::min(v, range);
    }
    const int cls = stage_class(p);
    static int tab[5] = {0, 0, 0, 0, 0};
    static bool parsed = false;
    if (!parsed) {  // developer tuning knob RKB_ZC="yd,light,epart,heavy,ab"
        const int def[5] = {8, 16, 16, 48, 4};
        for (int c = 0; c < 5; ++c) tab[c] = def[c];
        if (const char* e = getenv("RKB_ZC")) {
            int v[5], n = sscanf(e, "%d,%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3], &v[4]);
            for (int c = 0; c < n; ++c)
                if (v[c] > 0) tab[c] = v[c];
        }
        parsed = true;
    }
    int zc = tab[cls];
    const int th = 8 * stage_rows(p.sp);
    const int tiles = (int)(((st->nx + 31) / 32) * ((st->ny + th - 1) / th));
    const int want = st->ctx->num_sms * 4;  // >= 2 waves of 2 CTAs per SM
    while (zc > 4 && (int64_t)tiles * ((range + zc - 1) / zc) < want) zc /= 2;
    return std::min(zc, range);
}

static rk_status launch_stage_timed(rk_state st, const StagePlan& p, GsStageArgs& a, cudaStream_t sm = nullptr) {
    rk_ctx ctx = st->ctx;
    if (!sm) sm = ctx->stream;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (st->timing) {
        e0 = pool_event(st);
        e1 = pool_event(st);
        CK_CTX(ctx, cudaEventRecord(e0, sm));
    }
    int nl = 0;
    CK_CTX(ctx, launch_gs_stage(p.scheme, p.adaptive, p.stage, a, sm, &nl));
    st->stats.kernel_launches += nl;
    st->stats.stage_launches += nl;
    if (nl) {
        const int64_t planes = a.zmode == 1 ? (a.geo.nzl > 1 ? 2 : 1) : (int64_t)(a.z_hi - a.z_lo);
        const int64_t arrays = 1 + p.sp.nslots + (a.out_k ? 1 : 0) + (a.out_u ? 1 : 0) + (a.out_w ? 1 : 0) +
                               (a.out_e ? 1 : 0) + (a.out_z ? 1 : 0);
        st->stats.stage_bytes += planes * st->nx * st->ny * 2 * (int64_t)sizeof(double) * arrays;
    }
    if (st->timing) {
        CK_CTX(ctx, cudaEventRecord(e1, sm));
        st->pending.push_back({e0, e1, 0});
        if (st->pending.size() > 4096) TRY(resolve_timing(st));
    }
    return RK_OK;
}

// exchange the planes packed on stream `src` (comm stream; ev_halo marks completion)
static rk_status halo_exchange(rk_state st, cudaStream_t src) {
    NvtxRange nv("rk halo exchange");
    rk_ctx ctx = st->ctx;
    const int64_t pv = plane_values(st);
    CK_CTX(ctx, cudaEventRecord(st->ev_pack, src));
    CK_CTX(ctx, cudaStreamWaitEvent(ctx->comm, st->ev_pack, 0));
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (st->timing) {
        e0 = pool_event(st);
        e1 = pool_event(st);
        CK_CTX(ctx, cudaEventRecord(e0, ctx->comm));
    }
    rk_halo_plan plan;
    TRY(rk_halo_plan_get(ctx->world, ctx->rank, &plan));
    if (!ctx->nccl) return fail(RK_ERR_STATE, "halo exchange without a NCCL communicator");
    {  // world == 1 (loopback): one 2-plane message to self, [lo|hi] -> [ghost_hi|ghost_lo]
        NK_CTX(ctx, ncclGroupStart());
        for (int i = 0; i < plan.nmsg; ++i) {
            const rk_halo_msg& m = plan.msg[i];
            const size_t cnt = (size_t)(m.nplanes * pv);
            if (m.recv)
                NK_CTX(ctx, ncclRecv(st->ghostbuf + m.slot * pv, cnt, ncclDouble, m.peer, ctx->nccl, ctx->comm));
            else
                NK_CTX(ctx, ncclSend(st->sendbuf + m.slot * pv, cnt, ncclDouble, m.peer, ctx->nccl, ctx->comm));
        }
        NK_CTX(ctx, ncclGroupEnd());
        mark_progress(ctx, ctx->comm);
    }
    if (st->timing) {
        CK_CTX(ctx, cudaEventRecord(e1, ctx->comm));
        st->pending.push_back({e0, e1, 1});
    }
    CK_CTX(ctx, cudaEventRecord(st->ev_halo, ctx->comm));
    st->stats.halo_exchanges += 1;
    st->stats.halo_bytes += (int64_t)sizeof(double) * 2 * pv;
    return RK_OK;
}

// ---- peer-to-peer halo path (RK_OPT_HALO_P2P) --------------------------------
// A rank's exported CUDA IPC handles: its ghost planes (grid states) and its flag block.
struct P2pHandles {
    cudaIpcMemHandle_t ghost, flags;
    int has_ghost;
};

static bool p2p_needed(rk_state st) { return st->p2p && (st->ctx->world > 1 || st->loopback); }

// this rank's double-buffered ghost planes (grids) and flag block, zeroed
static rk_status p2p_alloc(rk_state st) {
    if (st->pflags) return RK_OK;
    rk_ctx ctx = st->ctx;
    if (st->grid) {
        const int64_t pv = plane_values(st);
        CK_CTX(ctx, cudaMalloc((void**)&st->pghost, sizeof(double) * 4 * pv));  // IPC-exported
        CK_CTX(ctx, cudaMemsetAsync(st->pghost, 0, sizeof(double) * 4 * pv, ctx->stream));
        for (int b = 0; b < 2; ++b)
            for (int g = 0; g < 2; ++g)
                CK_CTX(ctx, encode_grid_maps(st->tm_pg[b][g].m, st->pghost + (2 * b + g) * pv, st->geo, 1));
    }
    void* f = nullptr;
    CK_CTX(ctx, cudaMalloc(&f, P2P_FLAGS * sizeof(unsigned long long)));
    st->pflags = static_cast<unsigned long long*>(f);
    CK_CTX(ctx, cudaMemsetAsync(st->pflags, 0, P2P_FLAGS * sizeof(unsigned long long), ctx->stream));
    CK_CTX(ctx, cudaStreamSynchronize(ctx->stream));  // zeroed before any peer can map and write
    return RK_OK;
}

static rk_status p2p_export(rk_state st, P2pHandles* h) {
    TRY(p2p_alloc(st));
    *h = P2pHandles{};
    h->has_ghost = st->pghost ? 1 : 0;
    if (st->pghost) CK_CTX(st->ctx, cudaIpcGetMemHandle(&h->ghost, st->pghost));
    CK_CTX(st->ctx, cudaIpcGetMemHandle(&h->flags, st->pflags));
    return RK_OK;
}

// map the neighbours' ghost planes and every rank's flag block from all ranks' handles
static rk_status p2p_map(rk_state st, const P2pHandles* all) {
    rk_ctx ctx = st->ctx;
    const int world = ctx->world, rank = ctx->rank;
    if (world > P2P_MAX_WORLD) return fail(RK_ERR_UNSUPPORTED, "P2P transport: world %d > %d", world, P2P_MAX_WORLD);
    std::vector<unsigned long long*> fl(world, nullptr);
    fl[rank] = st->pflags;
    for (int q = 0; q < world; ++q) {
        if (q == rank) continue;
        void* pf = nullptr;
        CK_CTX(ctx, cudaIpcOpenMemHandle(&pf, all[q].flags, cudaIpcMemLazyEnablePeerAccess));
        st->ipc_mapped.push_back(pf);
        fl[q] = static_cast<unsigned long long*>(pf);
    }
    for (int q = 0; q < world; ++q) st->rank_flags[q] = fl[q];
    const int lower = (rank + world - 1) % world, upper = (rank + 1) % world;
    st->peer_flags[0] = fl[lower];
    st->peer_flags[1] = fl[upper];
    if (st->grid) {
        double* pg[2] = {st->pghost, st->pghost};
        for (int dir = 0; dir < 2; ++dir) {
            const int q = dir == 0 ? lower : upper;
            if (q == rank) continue;
            if (dir == 1 && upper == lower) {  // world == 2: one peer on both sides
                pg[1] = pg[0];
                break;
            }
            if (!all[q].has_ghost) return fail(RK_ERR_CONTRACT, "P2P: rank %d exported no ghost planes", q);
            void* g = nullptr;
            CK_CTX(ctx, cudaIpcOpenMemHandle(&g, all[q].ghost, cudaIpcMemLazyEnablePeerAccess));
            st->ipc_mapped.push_back(g);
            pg[dir] = static_cast<double*>(g);
        }
        st->peer_ghost[0] = pg[0];
        st->peer_ghost[1] = pg[1];
    }
    st->p2p_ready = true;
    return RK_OK;
}

// Collective (first P2P use on every rank): double-buffered ghost planes + flags; with NCCL the
// handles are all-gathered here, without NCCL (rk_p2p_import) the caller has exchanged them.
static rk_status ensure_p2p(rk_state st) {
    if (st->p2p_ready) return RK_OK;
    rk_ctx ctx = st->ctx;
    P2pHandles mine{};
    TRY(p2p_export(st, &mine));
    if (ctx->world == 1) {  // loopback: both neighbours are this rank
        return p2p_map(st, &mine);
    }
    if (!ctx->nccl)
        return fail(RK_ERR_STATE, "P2P transport without NCCL: exchange the handles with rk_p2p_export / rk_p2p_import first");
    const size_t hb = sizeof mine;
    unsigned char* d = nullptr;
    CK_CTX(ctx, cudaMalloc((void**)&d, hb * (ctx->world + 1)));
    CK_CTX(ctx, cudaMemcpyAsync(d, &mine, hb, cudaMemcpyHostToDevice, ctx->stream));
    NK_CTX(ctx, ncclAllGather(d, d + hb, hb, ncclUint8, ctx->nccl, ctx->stream));
    std::vector<P2pHandles> all(ctx->world);
    CK_CTX(ctx, cudaMemcpyAsync(all.data(), d + hb, hb * ctx->world, cudaMemcpyDeviceToHost, ctx->stream));
    TRY(ctx_wait(ctx, ctx->stream));
    cudaFree(d);
    return p2p_map(st, all.data());
}

// One stage with P2P halos: pack (waits until the neighbours released this parity's ghost
// planes, stores Y_i's boundary planes into them, raises their ready flags) -> interior planes
// -> boundary planes (wait for this rank's ready flags, then release the ghosts to the
// neighbours and advance the device-resident stage counter).  Ghost planes alternate between
// two parities so a stage's stores never wait for the previous stage's reads.  Nothing here
// depends on host-side state, so the same launches replay from a CUDA graph.
static rk_status run_gs_stage_p2p(rk_state st, const StagePlan& p, GsStageArgs& a) {
    rk_ctx ctx = st->ctx;
    TRY(ensure_p2p(st));
    const int nzl = (int)st->local;
    const int64_t pv = plane_values(st);
    P2pSync ps{};
    ps.on = 1;
    ps.role = 0;
    ps.wait[0] = st->pflags + P2P_ACK_LO;
    ps.wait[1] = st->pflags + P2P_ACK_HI;
    ps.notify[0] = st->peer_flags[0] + P2P_READY_HI;  // my plane 0 is the lower neighbour's ghost_hi
    ps.notify[1] = st->peer_flags[1] + P2P_READY_LO;  // my plane nzl-1 is the upper's ghost_lo
    ps.count = st->pflags + P2P_COUNT;
    ps.seqp = st->pflags + P2P_SEQ;
    // the boundary stream starts from everything the compute stream has issued so far
    CK_CTX(ctx, cudaEventRecord(st->ev_ready, ctx->stream));
    CK_CTX(ctx, cudaStreamWaitEvent(ctx->bnd, st->ev_ready, 0));
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (st->timing) {  // the exchange: the pack kernel's stores into the neighbours' ghost planes
        e0 = pool_event(st);
        e1 = pool_event(st);
        CK_CTX(ctx, cudaEventRecord(e0, ctx->bnd));
    }
    CK_CTX(ctx, launch_gs_pack(pack_args(a, p), st->peer_ghost[0] + 0 * pv, st->peer_ghost[1] + 1 * pv, ps, ctx->bnd));
    if (st->timing) {
        CK_CTX(ctx, cudaEventRecord(e1, ctx->bnd));
        st->pending.push_back({e0, e1, 1});
    }
    st->stats.kernel_launches += 1;
    st->stats.halo_exchanges += 1;
    st->stats.halo_bytes += (int64_t)sizeof(double) * 2 * pv;
    const int hb = 2 * (stage_rows(p.sp) - 1);
    a.has_ghi = 1;
    a.has_glo = 1;
    a.tm_ghi = st->tm_pg[0][0].m[hb];
    a.tm_glo = st->tm_pg[0][1].m[hb];
    a.tm_ghi1 = st->tm_pg[1][0].m[hb];
    a.tm_glo1 = st->tm_pg[1][1].m[hb];
    if (nzl > 2) {
        GsStageArgs in = a;  // interior planes [1, nzl-1) never touch ghost planes
        in.z_lo = 1;
        in.z_hi = nzl - 1;
        in.zchunk = pick_zchunk(st, p, nzl - 2);
        in.zpair = stage_zpair(p);
        TRY(launch_stage_timed(st, p, in));
    }
    GsStageArgs bd = a;
    bd.zmode = 1;
    P2pSync& bs = bd.sync;
    bs.on = 1;
    bs.role = 1;
    bs.wait[0] = st->pflags + P2P_READY_LO;
    bs.wait[1] = st->pflags + P2P_READY_HI;
    bs.notify[0] = st->peer_flags[0] + P2P_ACK_HI;  // my ghost_lo came from the lower neighbour
    bs.notify[1] = st->peer_flags[1] + P2P_ACK_LO;  // my ghost_hi came from the upper neighbour
    bs.count = st->pflags + P2P_COUNT;
    bs.seqp = st->pflags + P2P_SEQ;
    TRY(launch_stage_timed(st, p, bd, ctx->bnd));  // beside the interior launch
    CK_CTX(ctx, cudaEventRecord(st->ev_bnd, ctx->bnd));
    CK_CTX(ctx, cudaStreamWaitEvent(ctx->stream, st->ev_bnd, 0));  // stage complete on the compute stream
    return RK_OK;
}

// Global max of one uint64 word on the stream (collective): P2P atomics over NVLink when the
// state uses the P2P transport (no NCCL on the data path; graph-capturable), else NCCL's
// allreduce (world > 1 or the loopback's 1-rank communicator), else nothing to do.
static rk_status allreduce_max_word(rk_state st, unsigned long long* word) {
    rk_ctx ctx = st->ctx;
    if (p2p_needed(st)) {
        TRY(ensure_p2p(st));
        CK_CTX(ctx, launch_p2p_allreduce_max(word, st->rank_flags, ctx->world, ctx->rank, ctx->stream));
        st->stats.kernel_launches += 1;
        return RK_OK;
    }
    if (ctx->nccl && halo_path(st)) {
        NK_CTX(ctx, ncclAllReduce(word, word, 1, ncclUint64, ncclMax, ctx->nccl, ctx->stream));
        mark_progress(ctx, ctx->stream);
        return RK_OK;
    }
    if (ctx->world > 1) return fail(RK_ERR_STATE, "no transport for the allreduce (no NCCL, no P2P)");
    return RK_OK;
}

static rk_status run_gs_stage(rk_state st, const StagePlan& p, double dt, double atol, double rtol) {
    NvtxRange nv("rk stage");
    rk_ctx ctx = st->ctx;
    TRY(ensure_halo(st));  // every entry path (RK plans, Adams steps, eval_rhs) lands here
    GsStageArgs a = stage_args(st, p, dt, atol, rtol);
    const int nzl = (int)st->local;
    st->stats.rhs_evals += 1;
    if (!halo_path(st)) {
        a.zchunk = pick_zchunk(st, p, nzl);
        a.zpair = stage_zpair(p);
        return launch_stage_timed(st, p, a);
    }
    if (st->p2p) return run_gs_stage_p2p(st, p, a);
    // multi-GPU path: Y_i on the two boundary planes -> neighbours' ghost planes
    a.has_ghi = 1;
    a.has_glo = 1;
    a.tm_ghi = st->tm_ghi.m[2 * (stage_rows(p.sp) - 1)];
    a.tm_glo = st->tm_glo.m[2 * (stage_rows(p.sp) - 1)];
    if (st->overlap && nzl > 2) {
        // boundary stream: pack -> (comm stream: exchange) -> boundary planes, all beside the
        // interior launch on the compute stream; the two join at the end of the stage (the
        // next stage's interior reads the boundary planes as z neighbours)
        CK_CTX(ctx, cudaEventRecord(st->ev_ready, ctx->stream));
        CK_CTX(ctx, cudaStreamWaitEvent(ctx->bnd, st->ev_ready, 0));
        CK_CTX(ctx, launch_gs_pack(pack_args(a, p), st->sendbuf, st->sendbuf + plane_values(st), P2pSync{}, ctx->bnd));
        st->stats.kernel_launches += 1;
        TRY(halo_exchange(st, ctx->bnd));
        GsStageArgs in = a;  // interior planes [1, nzl-1) never touch ghost planes
        in.z_lo = 1;
        in.z_hi = nzl - 1;
        in.zchunk = pick_zchunk(st, p, nzl - 2);
        in.zpair = stage_zpair(p);
        TRY(launch_stage_timed(st, p, in));
        CK_CTX(ctx, cudaStreamWaitEvent(ctx->bnd, st->ev_halo, 0));
        GsStageArgs bd = a;
        bd.zmode = 1;
        TRY(launch_stage_timed(st, p, bd, ctx->bnd));
        CK_CTX(ctx, cudaEventRecord(st->ev_bnd, ctx->bnd));
        CK_CTX(ctx, cudaStreamWaitEvent(ctx->stream, st->ev_bnd, 0));
        return RK_OK;
    }
    CK_CTX(ctx, launch_gs_pack(pack_args(a, p), st->sendbuf, st->sendbuf + plane_values(st), P2pSync{}, ctx->stream));
    st->stats.kernel_launches += 1;
    TRY(halo_exchange(st, ctx->stream));
    CK_CTX(ctx, cudaStreamWaitEvent(ctx->stream, st->ev_halo, 0));
    a.zchunk = pick_zchunk(st, p, nzl);
    a.zpair = stage_zpair(p);
    return launch_stage_timed(st, p, a);
}

static int pick_pair_zchunk(rk_state st, int zc);

// K8 DOPRI5 tail pair (rk_pair.cu PAIR_DP_TAIL): stages 6 and 7 of an error-controlled try
// (Odeint ratio) in one launch on one GPU -- reads Y_6, W, E (written ahead by stage 5) and u,
// k_1; writes u_new, k_7 (into stage 7's buffer) and the ratio max: 7 arrays instead of 10.
// On the multi-GPU slab (and its one-GPU loopback) the pair runs over NCCL ghost planes: Y_6's two
// boundary planes and W's one are exchanged after stage 5, then one launch covers the slab.
static bool dp_tail_pair_ok(rk_state st, const std::vector<StagePlan>& plan) {
    if (st->fused != 3 || !st->grid || st->ncomp != 2 || st->rhs != RHS_GRAY_SCOTT || st->p2p ||
        !pair_shape_ok(st->geo) || plan.size() != 7)
        return false;
    if (halo_path(st) && (!st->ctx->nccl || st->local < 2)) return false;
    const StagePlan& f = plan[5];
    const StagePlan& t = plan[6];
    return f.scheme == RK_DOPRI5 && f.adaptive == 1 && f.sp.epi == EPI_FINAL_EPART && f.sp.base_src >= 0 &&
           f.sp.wslot == 0 && f.sp.eslot == 1 && t.sp.epi == EPI_TAIL_ERR && t.sp.den_k1 >= 0;
}

// Ghost planes of a K8 launch on the multi-GPU slab (and its one-GPU loopback): one NCCL group on
// the compute stream -- src's two boundary planes each side into g2 ([-2, -1 | nzl, nzl+1]) and,
// if given, base's one plane each side into pg_w ([-1 | nzl]).  To the upper neighbour go the
// top planes (its -2, -1 / -1), to the lower one the bottom planes (its nzl, nzl+1 / nzl).
// Sends to up precede sends to down and receives from down precede receives from up, so with
// world 2 (both neighbours the same peer) and world 1 (self) the messages still pair correctly.
static rk_status pair_ghost_buffers(rk_state st) {
    if (st->pg_y) return RK_OK;
    rk_ctx ctx = st->ctx;
    const int64_t pv = plane_values(st);
    TRY(dev_alloc(ctx, &st->pg_y, 4 * pv));
    TRY(dev_alloc(ctx, &st->pg_y2, 4 * pv));
    TRY(dev_alloc(ctx, &st->pg_w, 2 * pv));
    CK_CTX(ctx, encode_pair_map(&st->tm_pgy_lo, st->pg_y, st->geo, 2));
    CK_CTX(ctx, encode_pair_map(&st->tm_pgy_hi, st->pg_y + 2 * pv, st->geo, 2));
    CK_CTX(ctx, encode_pair_map(&st->tm_pgy2_lo, st->pg_y2, st->geo, 2));
    CK_CTX(ctx, encode_pair_map(&st->tm_pgy2_hi, st->pg_y2 + 2 * pv, st->geo, 2));
    CK_CTX(ctx, encode_grid_maps(st->tm_pgw_lo.m, st->pg_w, st->geo, 1));
    CK_CTX(ctx, encode_grid_maps(st->tm_pgw_hi.m, st->pg_w + pv, st->geo, 1));
    CK_CTX(ctx, encode_grid_maps(st->tm_pgu_lo.m, st->pg_y + pv, st->geo, 1));      // plane -1
    CK_CTX(ctx, encode_grid_maps(st->tm_pgu_hi.m, st->pg_y + 2 * pv, st->geo, 1));  // plane nzl
    return RK_OK;
}

static rk_status pair_ghost_exchange(rk_state st, const double* src, double* g2, const double* base) {
    NvtxRange nv("rk halo exchange (K8 pair)");
    rk_ctx ctx = st->ctx;
    const int64_t pv = plane_values(st), nzl = st->local;
    TRY(pair_ghost_buffers(st));
    const int up = (ctx->rank + 1) % ctx->world, down = (ctx->rank - 1 + ctx->world) % ctx->world;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (st->timing) {
        e0 = pool_event(st);
        e1 = pool_event(st);
        CK_CTX(ctx, cudaEventRecord(e0, ctx->stream));
    }
    rk_pair_plan plan;
    TRY(rk_pair_ghost_plan(ctx->world, ctx->rank, base ? 1 : 0, &plan));
    NK_CTX(ctx, ncclGroupStart());
    for (int i = 0; i < plan.nmsg; ++i) {
        const rk_pair_msg& m = plan.msg[i];
        const size_t cnt = (size_t)(m.nplanes * pv);
        if (m.recv) {  // ghosts below the slab at the ghost array's start, above after them
            double* g = m.array == 0 ? g2 : st->pg_w;
            NK_CTX(ctx, ncclRecv(g + (m.side ? m.nplanes * pv : 0), cnt, ncclDouble, m.peer, ctx->nccl, ctx->stream));
        } else {       // the slab's bottom planes, or its top ones
            const double* a = m.array == 0 ? src : base;
            NK_CTX(ctx, ncclSend(a + (m.side ? (nzl - m.nplanes) * pv : 0), cnt, ncclDouble, m.peer, ctx->nccl,
                                 ctx->stream));
        }
    }
    NK_CTX(ctx, ncclGroupEnd());
    mark_progress(ctx, ctx->stream);
    if (st->timing) {
        CK_CTX(ctx, cudaEventRecord(e1, ctx->stream));
        st->pending.push_back({e0, e1, 1});
    }
    st->stats.halo_exchanges += 1;
    st->stats.halo_bytes += (int64_t)sizeof(double) * (base ? 6 : 4) * pv;
    return RK_OK;
}

static rk_status dp_tail_pair(rk_state st, const std::vector<StagePlan>& plan, double dt, double atol, double rtol) {
    NvtxRange nv("rk stage pair (K8 DOPRI5 tail)");
    rk_ctx ctx = st->ctx;
    const StagePlan& f = plan[5];
    const StagePlan& t = plan[6];
    PairArgs a{};
    if (halo_path(st)) {
        TRY(pair_ghost_buffers(st));
        TRY(pair_ghost_exchange(st, st->k[f.sp.base_src], st->pg_y, st->k[f.sp.src[0]]));
        a.ghosts = 1;
        a.tm_glo = st->tm_pgy_lo;
        a.tm_ghi = st->tm_pgy_hi;
        a.tm_ulo = st->tm_pgw_lo.m[2];
        a.tm_uhi = st->tm_pgw_hi.m[2];
        a.src_lo = st->pg_y;
        a.src_hi = st->pg_y + 2 * plane_values(st);
    }
    a.geo = st->geo;
    a.d1 = st->d1;
    a.d2 = st->d2;
    a.F = st->F;
    a.FK = st->F + st->K;
    a.inv_h2 = 1.0 / (st->h * st->h);
    a.zchunk = pick_pair_zchunk(st, 16);
    double* y6 = st->k[f.sp.base_src];
    CK_CTX(ctx, encode_pair_map(&a.tm_src, y6, st->geo, (int)st->local));
    a.src = y6;
    a.tm_u = st->tm_k[f.sp.src[0]].m[2];  // W: tile + 1 ring (stored with its ring by stage 5)
    a.w_in = st->k[f.sp.src[1]];          // E
    a.u_in = st->u;
    a.k1_in = st->k[0];
    a.tm_e = st->tm_k[f.sp.src[1]].m[3];  // 34 x 16 interior boxes: L2 prefetch of the own inputs
    a.tm_uo = st->tm_u.m[3];
    a.tm_k1 = st->tm_k[0].m[3];
    a.out = st->u_new;
    a.out_y = st->k[t.sp.out_k];
    a.errmax = st->d_err;
    a.gB = f.beta_new;
    a.betaA = f.delta_new;
    a.betaB = t.delta_new;
    a.dt = dt;
    a.atol = atol;
    a.rtol = rtol;
    a.dtp = st->gl_dtp;  // device-resident try loop (captured): raw plan coefficients, dt on the device
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (st->timing) {
        e0 = pool_event(st);
        e1 = pool_event(st);
        CK_CTX(ctx, cudaEventRecord(e0, ctx->stream));
    }
    CK_CTX(ctx, launch_gs_pair(PAIR_DP_TAIL, a, ctx->stream));
    if (st->timing) {
        CK_CTX(ctx, cudaEventRecord(e1, ctx->stream));
        st->pending.push_back({e0, e1, 2});
        if (st->pending.size() > 4096) TRY(resolve_timing(st));
    }
    const int64_t pb = 7 * st->local * st->nx * st->ny * 2 * (int64_t)sizeof(double);
    st->stats.kernel_launches += 1;
    st->stats.stage_launches += 1;
    st->stats.pair_launches += 1;
    st->stats.rhs_evals += 2;
    st->stats.stage_bytes += pb;
    st->stats.pair_bytes += pb;
    return RK_OK;
}

// K8 head pair (PAIR_DP_HEAD): stages 2 and 3 of a step or try in one launch -- u and k1 (both
// with 2-cell margins; Y2 = u + (dt a21) k1 and Z3 = u + (dt a31) k1 formed in shared memory as
// they land) -> k2, k3 with their rings: 4 arrays instead of stages 2 + 3's 7.  Built for the
// DOPRI5 try; it serves every tableau whose stages 2 and 3 are plain slope stages with a21, a31,
// a32 != 0 (head_pair_ok: Cash–Karp 5(4), Dormand–Prince fixed and error-controlled, RKF 7(8)).
static rk_status dp_head_pair(rk_state st, int scheme, double dt) {
    NvtxRange nv("rk stage pair (K8 head: stages 2-3)");
    rk_ctx ctx = st->ctx;
    const Coeffs C = coeffs_of(scheme);
    PairArgs a{};
    if (halo_path(st)) {  // u's and k1's two boundary planes each side
        TRY(pair_ghost_buffers(st));
        TRY(pair_ghost_exchange(st, st->u, st->pg_y, nullptr));
        TRY(pair_ghost_exchange(st, st->k[0], st->pg_y2, nullptr));
        a.ghosts = 1;
        a.tm_glo = st->tm_pgy_lo;
        a.tm_ghi = st->tm_pgy_hi;
        a.tm_glo2 = st->tm_pgy2_lo;
        a.tm_ghi2 = st->tm_pgy2_hi;
        a.src_lo = st->pg_y;
        a.src_hi = st->pg_y + 2 * plane_values(st);
        a.src2_lo = st->pg_y2;
        a.src2_hi = st->pg_y2 + 2 * plane_values(st);
    }
    a.geo = st->geo;
    a.d1 = st->d1;
    a.d2 = st->d2;
    a.F = st->F;
    a.FK = st->F + st->K;
    a.inv_h2 = 1.0 / (st->h * st->h);
    a.zchunk = pick_pair_zchunk(st, 32);  // measured: 16 / 24 / 32 -> 2.24 / 2.16 / 2.14 ms
    CK_CTX(ctx, encode_pair_map(&a.tm_src, st->u, st->geo, (int)st->local));
    CK_CTX(ctx, encode_pair_map(&a.tm_u, st->k[0], st->geo, (int)st->local));  // k1, the same box
    a.src = st->u;
    a.src2 = st->k[0];
    a.gA = dt * C.a[1][0];
    a.gB1 = dt * C.a[2][0];
    a.gB = dt * C.a[2][1];
    a.out_y = st->k[1];  // k2
    a.out = st->k[2];    // k3
    a.dtp = st->gl_dtp;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (st->timing) {
        e0 = pool_event(st);
        e1 = pool_event(st);
        CK_CTX(ctx, cudaEventRecord(e0, ctx->stream));
    }
    CK_CTX(ctx, launch_gs_pair(PAIR_DP_HEAD, a, ctx->stream));
    if (st->timing) {
        CK_CTX(ctx, cudaEventRecord(e1, ctx->stream));
        st->pending.push_back({e0, e1, 3});
        if (st->pending.size() > 4096) TRY(resolve_timing(st));
    }
    const int64_t pb = 4 * st->local * st->nx * st->ny * 2 * (int64_t)sizeof(double);
    st->stats.kernel_launches += 1;
    st->stats.stage_launches += 1;
    st->stats.pair_launches += 1;
    st->stats.rhs_evals += 2;
    st->stats.stage_bytes += pb;
    st->stats.pair_bytes += pb;
    st->stats.head_launches += 1;
    st->stats.head_bytes += pb;
    return RK_OK;
}

static bool dp_head_pair_on() {  // developer A/B knob RKB_DP_HEAD=0 (default on)
    static int v = -1;
    if (v < 0) v = getenv("RKB_DP_HEAD") ? atoi(getenv("RKB_DP_HEAD")) : 1;
    return v != 0;
}

// Whether the head pair can take stages 2 and 3 (indices 1, 2) of this plan: one GPU or the NCCL
// slab path (as the tail pair), and plan stages 0..2 the plain slope stages k1 -> k[0],
// Y2 = u + a21 k1 -> k[1], Y3 = (u + a31 k1) + a32 k2 -> k[2] with nonzero a21, a31, a32 (the
// kernel's expressions), followed by at least one more stage.
static bool head_pair_ok(rk_state st, const std::vector<StagePlan>& plan) {
    if (!dp_head_pair_on() || st->fused != 3 || !st->grid || st->ncomp != 2 || st->rhs != RHS_GRAY_SCOTT ||
        st->p2p || !pair_shape_ok(st->geo) || plan.size() < 4 || is_multistep(plan[0].scheme))
        return false;
    if (halo_path(st) && (!st->ctx->nccl || st->local < 2)) return false;
    const StageSpec& s0 = plan[0].sp;
    const StageSpec& s1 = plan[1].sp;
    const StageSpec& s2 = plan[2].sp;
    auto plain = [](const StagePlan& p) {
        return p.sp.epi == EPI_K && p.sp.base_src < 0 && !p.sp.base_unew && p.out_hist < 0 && !p.out_ptr;
    };
    return plain(plan[0]) && plain(plan[1]) && plain(plan[2]) && s0.out_k == 0 && s0.nslots == 0 &&
           s1.out_k == 1 && s1.nslots == 1 && s1.src[0] == 0 && s1.gnz[0] && s2.out_k == 2 && s2.nslots == 2 &&
           s2.src[0] == 0 && s2.src[1] == 1 && s2.gnz[0] && s2.gnz[1];
}

// Run the stages of one step / try.  Stage 0 (k1 = F(u)) is skipped when k1 is valid.  A DOPRI5
// try on the K8 schedule: k1 if needed, the head pair (2, 3), stage 4, the write-ahead stage 5,
// the tail pair (6, 7) -- 23 arrays instead of 30.
static rk_status run_grid_plan(rk_state st, const std::vector<StagePlan>& plan, double dt,
                               double atol, double rtol) {
    TRY(ensure_k(st, plan_num_k(plan)));
    TRY(ensure_halo(st));
    const bool dp_pair = dp_tail_pair_ok(st, plan);
    const bool dp_head = head_pair_ok(st, plan);
    for (const StagePlan& p : plan) {
        if (dp_head && p.stage == 1) {
            TRY(dp_head_pair(st, p.scheme, dt));
            continue;
        }
        if (dp_head && p.stage == 2) continue;  // in the head pair
        if (dp_pair && p.stage == 5) {  // stages 6 + 7 as one K8 launch
            CK_CTX(st->ctx, cudaMemsetAsync(st->d_err, 0, sizeof(unsigned long long), st->ctx->stream));
            return dp_tail_pair(st, plan, dt, atol, rtol);
        }
        if (p.stage == 0 && p.sp.epi == EPI_K && st->k1_valid) continue;
        if (is_ratio_stage(p))
            CK_CTX(st->ctx, cudaMemsetAsync(st->d_err, 0, sizeof(unsigned long long), st->ctx->stream));
        TRY(run_gs_stage(st, p, dt, atol, rtol));
        if (p.stage == 0 && p.sp.epi == EPI_K) st->k1_valid = true;
    }
    return RK_OK;
}

// ------------------------------------------------------------------------------------
// pointwise (vector) execution
// ------------------------------------------------------------------------------------
static PwCoef pw_coef(int scheme, double dt) {
    const Coeffs C = coeffs_of(scheme);
    PwCoef cf{};
    for (int i = 0; i < C.s; ++i) {
        for (int j = 0; j < i; ++j) cf.g[i][j] = dt * C.a[i][j];
        cf.beta[i] = dt * C.b[i];
        cf.delta[i] = dt * C.e[i];
    }
    return cf;
}

static rk_status run_pointwise(rk_state st, int scheme, double dt, int nsteps, bool err,
                               double atol, double rtol) {
    rk_ctx ctx = st->ctx;
    PwArgs a{};
    a.u = st->u;
    a.u_out = st->u_new;
    a.count = st->count;
    a.rhs = st->rhs;
    a.lambda = st->lambda;
    a.nsteps = nsteps;
    a.dt = dt;
    a.atol = atol;
    a.rtol = rtol;
    a.errmax = err ? st->d_err : nullptr;
    a.ctrl = st->controller;
    a.cf = pw_coef(scheme, dt);
    if (err) CK_CTX(ctx, cudaMemsetAsync(st->d_err, 0, sizeof(unsigned long long), ctx->stream));
    CK_CTX(ctx, launch_pointwise(scheme, a, ctx->stream, ctx->num_sms));
    st->stats.kernel_launches += 1;
    st->stats.rhs_evals += (int64_t)num_stages(scheme, err) * (err ? 1 : nsteps);
    return RK_OK;
}

// ------------------------------------------------------------------------------------
// controller (host, Odeint default_step_adjuster; R-12, R-14; SPEC's R-28), with
// the correctly rounded pow of rk_ddmath.cuh (R-27) -- the same function the device-resident
// loops run, so host and device decisions agree bit for bit
// ------------------------------------------------------------------------------------
struct CtrlExp {
    double e_rej, e_acc, emin;
};
static CtrlExp ctrl_exponents(int controller, int p, int q) {
    return {controller == 1 ? -1.0 / (double)(p - 1) : -1.0 / (double)(q - 1), -1.0 / (double)p,
            pow_dd(5.0, -(double)p)};
}

static bool adjust(int controller, double E, int p, int q, double* dt) {
    const CtrlExp x = ctrl_exponents(controller, p, q);
    int ok = 0;
    *dt = step_adjust_dev(E, x.e_rej, x.e_acc, x.emin, controller, *dt, &ok);
    return ok != 0;
}

static bool step_adjust(double E, int p, int q, double* dt) { return adjust(0, E, p, q, dt); }

// RK_OPT_CHECK_ARGS (SURVEY §8b "Collectives"): every rank hashes (call kind, scalar args)
// and the ranks all-reduce max(h) and max(~h) = ~min(h); equal max and min <=> identical calls.
static rk_status check_collective_args(rk_state st, int kind, std::initializer_list<double> args) {
    if (!st->check_args || st->ctx->world == 1) return RK_OK;
    rk_ctx ctx = st->ctx;
    uint64_t h = 1469598103934665603ull ^ (uint64_t)kind;  // FNV-1a over the argument bytes
    for (double v : args) {
        unsigned char b[8];
        std::memcpy(b, &v, 8);
        for (unsigned char c : b) h = (h ^ c) * 1099511628211ull;
    }
    unsigned long long hv[2] = {h, ~h};
    for (int j = 0; j < 2; ++j) {
        CK_CTX(ctx, cudaMemcpyAsync(ctx->d_scratch, &hv[j], 8, cudaMemcpyHostToDevice, ctx->stream));
        TRY(allreduce_max_word(st, ctx->d_scratch));
        CK_CTX(ctx, cudaMemcpyAsync(ctx->h_scratch, ctx->d_scratch, 8, cudaMemcpyDeviceToHost, ctx->stream));
        TRY(ctx_wait(ctx, ctx->stream));
        hv[j] = *ctx->h_scratch;
    }
    if (hv[0] != ~hv[1])
        return fail(RK_ERR_CONTRACT, "collective call %d: the ranks' arguments differ (RK_OPT_CHECK_ARGS)", kind);
    return RK_OK;
}

// Global max |u| (collective), NaN if any element is NaN: the norm_inf reduction (K4).
static rk_status global_norm_inf(rk_state st, double* out) {
    rk_ctx ctx = st->ctx;
    CK_CTX(ctx, cudaMemsetAsync(ctx->d_scratch, 0, 8, ctx->stream));
    CK_CTX(ctx, launch_norm_inf(st->u, st->alloc, ctx->d_scratch, ctx->stream, ctx->num_sms));
    st->stats.kernel_launches += 1;
    TRY(allreduce_max_word(st, ctx->d_scratch));
    CK_CTX(ctx, launch_publish_word(ctx->d_scratch, ctx->h_scratch, ctx->stream));
    st->stats.kernel_launches += 1;
    TRY(ctx_wait(ctx, ctx->stream));
    std::memcpy(out, ctx->h_scratch, 8);
    return RK_OK;
}

// RK_OPT_CHECK_FINITE: after every n-th completed step (force: now), a non-finite state is
// RK_ERR_DIVERGED carrying the time t it was found at (stats.diverged_t).
static rk_status finite_check(rk_state st, int64_t steps_done, double t, bool force) {
    if (st->check_finite <= 0) return RK_OK;
    st->since_check += steps_done;
    if (!force && st->since_check < st->check_finite) return RK_OK;
    st->since_check = 0;
    double m = 0.0;
    TRY(global_norm_inf(st, &m));
    if (!std::isfinite(m)) {
        st->stats.diverged_t = t;
        return fail(RK_ERR_DIVERGED, "non-finite state at t=%.17g", t);
    }
    return RK_OK;
}

static rk_status check_rhs(rk_state st) {
    if (st->rhs == RHS_NONE) return fail(RK_ERR_STATE, "RHS not set");
    if (st->rhs == RHS_GRAY_SCOTT && (!st->grid || st->ncomp != 2))
        return fail(RK_ERR_STATE, "Gray-Scott RHS needs a grid state with ncomp == 2");
    if (st->rhs != RHS_GRAY_SCOTT && st->grid)
        return fail(RK_ERR_STATE, "pointwise RHS on grid state: use a vector state");
    return RK_OK;
}

// K5 (rk_smallgrid.cu): fixed RK steps of a small single-GPU grid in one cooperative launch
static bool coop_path(rk_state st, int scheme) {
    return st->grid && st->rhs == RHS_GRAY_SCOTT && st->ctx->world == 1 && !st->loopback && !st->p2p &&
           scheme >= RK_EULER && scheme <= RK_MODIFIED_MIDPOINT && st->local * st->nx * st->ny <= st->coop_max_cells;
}

static rk_status ensure_k5bar(rk_state st) {
    if (st->k5bar) return RK_OK;
    CK_CTX(st->ctx, cudaMalloc((void**)&st->k5bar, 2 * sizeof(unsigned int)));
    CK_CTX(st->ctx, cudaMemsetAsync(st->k5bar, 0, 2 * sizeof(unsigned int), st->ctx->stream));
    return RK_OK;
}

static rk_status coop_steps(rk_state st, int scheme, double dt, int64_t n) {
    NvtxRange nv("rk persistent steps (K5)");
    rk_ctx ctx = st->ctx;
    const int last = coop_last_stage(scheme);
    TRY(ensure_k(st, std::max(last, 1)));
    for (int b = 0; b < 2; ++b)
        if (!st->ybuf[b]) TRY(alloc_array(st, &st->ybuf[b], nullptr));
    const Coeffs C = coeffs_of(scheme);
    TRY(ensure_k5bar(st));
    GsCoopArgs a{};
    a.geo = st->geo;
    for (int j = 0; j < 13; ++j) a.k[j] = j < st->nk ? st->k[j] : nullptr;
    a.ybuf[0] = st->ybuf[0];
    a.ybuf[1] = st->ybuf[1];
    a.bar = st->k5bar;
    for (int i = 0; i < C.s; ++i) {
        for (int j = 0; j < i; ++j) a.cf.g[i][j] = dt * C.a[i][j];
        a.cf.beta[i] = dt * C.b[i];
    }
    a.d1 = st->d1;
    a.d2 = st->d2;
    a.F = st->F;
    a.FK = st->F + st->K;
    a.inv_h2 = 1.0 / (st->h * st->h);
    // algorithmic bytes: the stage-by-stage schedule's, per step
    int64_t arrays = 0;
    for (const StagePlan& p : build_plan(scheme, 0, dt))
        arrays += 1 + p.sp.nslots + (p.sp.out_k >= 0 ? 1 : 0) + (p.sp.writes_u ? 1 : 0) + (p.sp.out_w >= 0 ? 1 : 0) +
                  (p.sp.out_e >= 0 ? 1 : 0) + (p.sp.out_z >= 0 ? 1 : 0);
    const int64_t cells = st->local * st->nx * st->ny;
    while (n > 0) {
        const int chunk = (int)std::min<int64_t>(n, 1 << 20);
        a.nsteps = chunk;
        a.buf[0] = st->u;
        a.buf[1] = st->u_new;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (st->timing) {
            e0 = pool_event(st);
            e1 = pool_event(st);
            CK_CTX(ctx, cudaEventRecord(e0, ctx->stream));
        }
        CK_CTX(ctx, launch_gs_coop(scheme, a, ctx->stream, ctx->device));
        if (st->timing) {
            CK_CTX(ctx, cudaEventRecord(e1, ctx->stream));
            st->pending.push_back({e0, e1, 0});
        }
        if (chunk & 1) swap_u(st);
        st->stats.kernel_launches += 1;
        st->stats.stage_launches += 1;
        st->stats.rhs_evals += (int64_t)(last + 1) * chunk;
        st->stats.stage_bytes += arrays * cells * 2 * (int64_t)sizeof(double) * chunk;
        st->stats.steps += chunk;
        n -= chunk;
    }
    st->k1_valid = false;
    return RK_OK;
}

// K6 (rk_fused.cu): a whole fixed step of RK4 / explicit midpoint in one launch, temporal
// blocking across the stages (one GPU, no halo path)
static bool fused_path(rk_state st, int scheme) {
    return (st->fused == 1 || st->fused == 2) && st->grid && st->ncomp == 2 && st->rhs == RHS_GRAY_SCOTT && st->ctx->world == 1 &&
           !st->loopback && !st->p2p && fused_scheme(scheme);
}

static int pick_fused_zchunk(rk_state st) {
    const int nz = (int)st->local;
    int zc = 64;  // measured at 512^3: 8 / 16 / 32 / 64 / 128 -> 7.10 / 5.74 / 5.08 / 4.79 / ~4.8 ms (RK4)
    if (const char* e = getenv("RKB_FZ")) {  // developer tuning knob
        const int v = atoi(e);
        if (v > 0) zc = v;
    }
    const int64_t tiles = ((st->nx + 31) / 32) * ((st->ny + 15) / 16);
    while (zc > 2 && tiles * ((nz + zc - 1) / zc) < 2 * st->ctx->num_sms) zc /= 2;
    return std::max(1, std::min(zc, nz));
}

// K8 (rk_pair.cu): RK4 as two stage-pair launches (u -> k2, W; u, k2, W -> u_new), the
// explicit midpoint rule as one (u -> u_new); RK_OPT_FUSED_STEP = 3
static bool pair_path(rk_state st, int scheme) {
    if (!(st->fused == 3 && st->grid && st->ncomp == 2 && st->rhs == RHS_GRAY_SCOTT && !st->p2p &&
          (scheme == RK_RK4 || scheme == RK_EXPLICIT_MIDPOINT || scheme == RK_MODIFIED_MIDPOINT) &&
          pair_shape_ok(st->geo)))
        return false;
    // the multi-GPU slab (or its loopback): NCCL ghost planes before each launch (2 deep)
    return !halo_path(st) || (st->ctx->nccl && st->local >= 2);
}

// z chunk of a K8 launch (measured at 512^3, tools/fused_time.py / ncu: the DOPRI5 tail pair
// 16 planes (2.76 ms; 32: 3.03, 64: 3.72 -- longer chunks lose the y-neighbour rows from L2),
// RK4 pairs 24 (3.15 ms per step; 16: 3.19, 32: 3.16), explicit midpoint 32 (1.14 ms))
static int pick_pair_zchunk(rk_state st, int zc) {
    if (const char* e = getenv("RKB_PZ")) {  // developer tuning knob
        const int v = atoi(e);
        if (v > 0) zc = v;
    }
    const int64_t tiles = (int64_t)(st->nx / 32) * (st->ny / 16);
    while (zc > 2 && tiles * ((st->local + zc - 1) / zc) < 2 * st->ctx->num_sms) zc /= 2;
    return (int)std::max<int64_t>(1, std::min<int64_t>(zc, st->local));
}

static rk_status pair_steps(rk_state st, int scheme, double dt, int64_t n) {
    NvtxRange nv("rk pair steps (K8)");
    rk_ctx ctx = st->ctx;
    const Coeffs C = coeffs_of(scheme);
    const bool rk4 = scheme == RK_RK4;
    const bool gragg = scheme == RK_MODIFIED_MIDPOINT;  // pair (1, 2) + the K3 last stage
    if (rk4 || gragg) TRY(ensure_k(st, 2));  // k[0] <- Y3, k[1] <- W
    PairArgs a{};
    a.geo = st->geo;
    a.d1 = st->d1;
    a.d2 = st->d2;
    a.F = st->F;
    a.FK = st->F + st->K;
    a.inv_h2 = 1.0 / (st->h * st->h);
    a.zchunk = pick_pair_zchunk(st, rk4 ? 24 : 32);
    const int64_t cells = st->local * st->nx * st->ny;
    const bool slab = halo_path(st);  // multi-GPU slab / loopback: ghost planes, no z wrap
    a.ghosts = slab ? 1 : 0;
    auto launch = [&](int kind) -> rk_status {  // one pair launch, timed like a stage launch
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (st->timing) {
            e0 = pool_event(st);
            e1 = pool_event(st);
            CK_CTX(ctx, cudaEventRecord(e0, ctx->stream));
        }
        CK_CTX(ctx, launch_gs_pair(kind, a, ctx->stream));
        if (st->timing) {
            CK_CTX(ctx, cudaEventRecord(e1, ctx->stream));
            st->pending.push_back({e0, e1, 2});
            if (st->pending.size() > 4096) TRY(resolve_timing(st));
        }
        return RK_OK;
    };
    for (int64_t i = 0; i < n; ++i) {
        if (slab) {  // u's two boundary planes each side (also pair (3,4)'s 1-deep base ghosts)
            TRY(pair_ghost_buffers(st));
            TRY(pair_ghost_exchange(st, st->u, st->pg_y, nullptr));
            a.tm_glo = st->tm_pgy_lo;
            a.tm_ghi = st->tm_pgy_hi;
            a.src_lo = st->pg_y;
            a.src_hi = st->pg_y + 2 * plane_values(st);
        }
        CK_CTX(ctx, encode_pair_map(&a.tm_src, st->u, st->geo, (int)st->local));
        a.src = st->u;
        a.gB = dt * C.a[1][0];
        a.betaA = dt * C.b[0];
        a.betaB = dt * C.b[1];
        if (rk4) {  // (u -> Y3 = u + g3 k2, W) then (Y3, u, W -> u_new)
            a.gN = dt * C.a[2][1];
            a.out = st->k[1];
            a.out_y = st->k[0];
            TRY(launch(PAIR_FIRST));
            if (slab) {  // Y3's ghosts; u's 1-deep ghosts are the inner planes of the first exchange
                TRY(pair_ghost_exchange(st, st->k[0], st->pg_y2, nullptr));
                a.tm_glo = st->tm_pgy2_lo;
                a.tm_ghi = st->tm_pgy2_hi;
                a.src_lo = st->pg_y2;
                a.src_hi = st->pg_y2 + 2 * plane_values(st);
                a.tm_ulo = st->tm_pgu_lo.m[2];
                a.tm_uhi = st->tm_pgu_hi.m[2];
            }
            CK_CTX(ctx, encode_pair_map(&a.tm_src, st->k[0], st->geo, (int)st->local));
            a.tm_u = st->tm_u.m[2];
            a.src = st->k[0];
            a.w_in = st->k[1];
            a.gB = dt * C.a[3][2];
            a.betaA = dt * C.b[2];
            a.betaB = dt * C.b[3];
            a.out = st->u_new;
            a.out_y = nullptr;
            TRY(launch(PAIR_LAST));
        } else if (gragg) {  // (u -> Y3 = u + dt k2, W) then the K3 last stage (Y3, W -> u_new)
            a.gN = dt * C.a[2][1];
            a.out = st->k[1];
            a.out_y = st->k[0];
            TRY(launch(PAIR_FIRST));
            StagePlan q;
            q.scheme = scheme;
            q.adaptive = 4;
            q.stage = 2;
            q.sp = stage_spec(scheme, 4, 2);
            q.beta_new = dt * C.b[2];
            TRY(run_gs_stage(st, q, dt, 0.0, 0.0));  // counts its own launch, RHS and bytes
            st->stats.rhs_evals -= 1;
        } else {  // explicit midpoint: u -> u_new (b_1 = 0)
            a.out = st->u_new;
            TRY(launch(PAIR_ONLY));
        }
        swap_u(st);
        const int nl = rk4 ? 2 : 1;
        st->stats.kernel_launches += nl;
        st->stats.stage_launches += nl;
        st->stats.pair_launches += nl;
        st->stats.rhs_evals += C.s;
        // RK4: (u -> Y3, W) + (Y3, u, W -> u_new) = 7 arrays; midpoint: u -> u_new; Gragg's pair: 3
        const int64_t pb = (rk4 ? 7 : gragg ? 3 : 2) * cells * 2 * (int64_t)sizeof(double);
        st->stats.stage_bytes += pb;
        st->stats.pair_bytes += pb;
        st->stats.steps += 1;
    }
    st->k1_valid = false;
    return RK_OK;
}

static rk_status fused_steps(rk_state st, int scheme, double dt, int64_t n) {
    NvtxRange nv("rk fused steps (K6)");
    rk_ctx ctx = st->ctx;
    const Coeffs C = coeffs_of(scheme);
    GsFusedArgs a{};
    a.geo = st->geo;
    for (int s = 1; s < C.s; ++s) a.g[s] = dt * C.a[s][s - 1];
    for (int j = 0; j < C.s; ++j) a.beta[j] = dt * C.b[j];
    a.d1 = st->d1;
    a.d2 = st->d2;
    a.F = st->F;
    a.FK = st->F + st->K;
    a.inv_h2 = 1.0 / (st->h * st->h);
    a.zchunk = pick_fused_zchunk(st);
    const int64_t cells = st->local * st->nx * st->ny;
    for (int64_t i = 0; i < n; ++i) {
        CK_CTX(ctx, encode_fused_map(&a.tm_u, st->u, st->geo, (int)st->local, fused_halo(scheme)));
        a.u = st->u;
        a.out = st->u_new;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (st->timing) {
            e0 = pool_event(st);
            e1 = pool_event(st);
            CK_CTX(ctx, cudaEventRecord(e0, ctx->stream));
        }
        CK_CTX(ctx, st->fused == 2 ? launch_gs_fused_ws(scheme, a, ctx->stream) : launch_gs_fused(scheme, a, ctx->stream));
        if (st->timing) {
            CK_CTX(ctx, cudaEventRecord(e1, ctx->stream));
            st->pending.push_back({e0, e1, 0});
            if (st->pending.size() > 4096) TRY(resolve_timing(st));
        }
        swap_u(st);
        st->stats.kernel_launches += 1;
        st->stats.stage_launches += 1;
        st->stats.rhs_evals += C.s;
        st->stats.stage_bytes += 2 * cells * 2 * (int64_t)sizeof(double);  // u in, u_new out
        st->stats.steps += 1;
    }
    st->k1_valid = false;
    return RK_OK;
}

// ---- RK_OPT_FUSED_KERNELS = 0: the unfused, Odeint-like dataflow (f4 ablation) ----
// Every stage value Y_i = u + sum_j (dt a_ij) k_j goes through HBM (one lincomb launch), every
// k_i = F(Y_i) is one RHS launch (the k1-type stage kernel reading Y_i, halo path included),
// then u_new = u + sum_j (dt b_j) k_j and, under error control, e = sum_j (dt e_j) k_j (lincomb)
// and the ratio max (ratio_max_kernel).  The same left-to-right sums over the nonzero
// coefficients as the fused kernels and the oracle (R-17): bitwise the same results, only the
// traffic differs (SURVEY §8d "arrays (unfused Odeint-like dataflow)").
static rk_status uf_lincomb(rk_state st, double* out, int k, const double* coef, double* const* in) {
    LincombArgs a{};
    a.out = out;
    a.k = k;
    a.count = st->alloc;  // padded grids: ring copies combine linearly, pads stay 0
    for (int j = 0; j < k; ++j) {
        a.in[j] = in[j];
        a.coef[j] = coef[j];
    }
    CK_CTX(st->ctx, launch_lincomb(a, st->ctx->stream, st->ctx->num_sms));
    st->stats.kernel_launches += 1;
    st->stats.stage_bytes += (int64_t)(k + 1) * st->count * (int64_t)sizeof(double);
    return RK_OK;
}

// k = F(y): the k1-type stage (grids: K3 with y as its base array, exchanging y's boundary
// planes on the halo path; vectors: the pointwise RHS kernel)
static rk_status uf_eval(rk_state st, double* y, const Maps& ym, double* out) {
    if (!st->grid) {
        CK_CTX(st->ctx, launch_rhs_pointwise(y, out, st->count, st->rhs, st->lambda, st->ctx->stream, st->ctx->num_sms));
        st->stats.kernel_launches += 1;
        st->stats.rhs_evals += 1;
        st->stats.stage_bytes += 2 * st->count * (int64_t)sizeof(double);
        return RK_OK;
    }
    double* const u = st->u;
    const Maps mu = st->tm_u;
    st->u = y;
    st->tm_u = ym;
    StagePlan p = build_plan(RK_RK4, 0, 0.0)[0];
    p.out_ptr = out;
    const rk_status rc = run_gs_stage(st, p, 0.0, 0.0, 0.0);
    st->u = u;
    st->tm_u = mu;
    return rc;
}

// the stages of one step (err = false) or one try (err = true) into st->u_new (and st->d_err)
static rk_status unfused_stages(rk_state st, int scheme, double dt, bool err, double atol, double rtol) {
    rk_ctx ctx = st->ctx;
    const Coeffs C = coeffs_of(scheme);
    const int s = num_stages(scheme, err);
    TRY(ensure_k(st, s));
    if (!st->uf_y) {
        TRY(alloc_array(st, &st->uf_y, &st->tm_uf_y));
        TRY(alloc_array(st, &st->uf_e, nullptr));
    }
    double coef[14];
    double* in[14];
    for (int i = 0; i < s; ++i) {
        if (i == 0) {
            if (st->k1_valid) continue;
            TRY(uf_eval(st, st->u, st->tm_u, st->k[0]));
            st->k1_valid = true;
            continue;
        }
        int n = 0;
        coef[n] = 1.0;
        in[n++] = st->u;
        for (int j = 0; j < i; ++j)
            if (C.a[i][j] != 0.0) {
                coef[n] = dt * C.a[i][j];
                in[n++] = st->k[j];
            }
        TRY(uf_lincomb(st, st->uf_y, n, coef, in));  // Y_i
        TRY(uf_eval(st, st->uf_y, st->tm_uf_y, st->k[i]));
    }
    int n = 0;
    coef[n] = 1.0;
    in[n++] = st->u;
    for (int j = 0; j < s; ++j)
        if (C.b[j] != 0.0) {
            coef[n] = dt * C.b[j];
            in[n++] = st->k[j];
        }
    TRY(uf_lincomb(st, st->u_new, n, coef, in));  // u_new
    if (!err) return RK_OK;
    n = 0;
    for (int j = 0; j < s; ++j)
        if (C.e[j] != 0.0) {
            coef[n] = dt * C.e[j];
            in[n++] = st->k[j];
        }
    TRY(uf_lincomb(st, st->uf_e, n, coef, in));  // e
    CK_CTX(ctx, cudaMemsetAsync(st->d_err, 0, sizeof(unsigned long long), ctx->stream));
    const bool spec = st->controller == 1;
    CK_CTX(ctx, launch_ratio_max(st->uf_e, st->u, spec ? st->u_new : st->k[0], st->alloc, dt, atol, rtol,
                                 spec ? 1 : 0, st->d_err, ctx->stream, ctx->num_sms));
    st->stats.kernel_launches += 1;
    st->stats.stage_bytes += 3 * st->count * (int64_t)sizeof(double);
    return RK_OK;
}

// K8 fixed-step tail pair: the last two stages (L-1, L) of a fixed step in one launch -- the
// write-ahead stage L-2 (stage_spec ad 5) stored Y_{L-1} (the pair's source), Z_L = u + sum_{j<=L-2}
// a_Lj k_j (its base: Y_L = Z_L + (dt a_{L,L-1}) k_{L-1}) and W = u + sum_{j<=L-2} b_j k_j; the pair
// (PAIR_LAST's kernel) writes u_new = (W + b_{L-1} k_{L-1}) + b_L k_L.  Cash–Karp 5(4), Dormand–Prince
// fixed step, RKF 7(8): stages L-2 .. L move 7 + 4 arrays instead of 5 + 7 + 3 (CK54 / DOPRI5).
static bool fixed_tail_ok(rk_state st, int scheme) {
    static int knob = -1;  // developer A/B knob RKB_FIXED_TAIL=0 (default on)
    if (knob < 0) knob = getenv("RKB_FIXED_TAIL") ? atoi(getenv("RKB_FIXED_TAIL")) : 1;
    if (!knob || st->fused != 3 || !st->grid || st->ncomp != 2 || st->rhs != RHS_GRAY_SCOTT || st->p2p ||
        !pair_shape_ok(st->geo))
        return false;
    if (scheme != RK_CASH_KARP54 && scheme != RK_DOPRI5 && scheme != RK_FEHLBERG78) return false;  // instantiated
    if (halo_path(st) && (!st->ctx->nccl || st->local < 2)) return false;
    const Tableau T = tableau_of(scheme);
    const int L = last_stage(T, false);
    return stage_spec(scheme, 5, L - 2).valid && t_bnz(T, L) && t_anz(T, L, L - 1);
}

static rk_status fixed_tail_pair(rk_state st, int scheme, double dt) {
    NvtxRange nv("rk stage pair (K8 fixed-step tail)");
    rk_ctx ctx = st->ctx;
    const Coeffs C = coeffs_of(scheme);
    const Tableau T = tableau_of(scheme);
    const int L = last_stage(T, false);
    double* y = st->k[L - 2];  // Y_{L-1}
    double* z = st->k[L - 1];  // Z_L
    PairArgs a{};
    if (halo_path(st)) {  // Y_{L-1}'s two boundary planes and Z_L's one, each side
        TRY(pair_ghost_buffers(st));
        TRY(pair_ghost_exchange(st, y, st->pg_y, z));
        a.ghosts = 1;
        a.tm_glo = st->tm_pgy_lo;
        a.tm_ghi = st->tm_pgy_hi;
        a.tm_ulo = st->tm_pgw_lo.m[2];
        a.tm_uhi = st->tm_pgw_hi.m[2];
        a.src_lo = st->pg_y;
        a.src_hi = st->pg_y + 2 * plane_values(st);
    }
    a.geo = st->geo;
    a.d1 = st->d1;
    a.d2 = st->d2;
    a.F = st->F;
    a.FK = st->F + st->K;
    a.inv_h2 = 1.0 / (st->h * st->h);
    a.zchunk = pick_pair_zchunk(st, 24);
    CK_CTX(ctx, encode_pair_map(&a.tm_src, y, st->geo, (int)st->local));
    a.src = y;
    a.tm_u = st->tm_k[L - 1].m[2];  // Z_L: tile + 1 ring
    a.w_in = st->k[L];              // W
    a.gB = dt * C.a[L][L - 1];
    a.betaA = dt * C.b[L - 1];
    a.betaB = dt * C.b[L];
    a.out = st->u_new;
    a.dt = dt;
    const bool ba = t_bnz(T, L - 1);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (st->timing) {
        e0 = pool_event(st);
        e1 = pool_event(st);
        CK_CTX(ctx, cudaEventRecord(e0, ctx->stream));
    }
    CK_CTX(ctx, launch_gs_pair(ba ? PAIR_LAST : PAIR_LAST_NOA, a, ctx->stream));
    if (st->timing) {
        CK_CTX(ctx, cudaEventRecord(e1, ctx->stream));
        st->pending.push_back({e0, e1, 2});
        if (st->pending.size() > 4096) TRY(resolve_timing(st));
    }
    const int64_t pb = 4 * st->local * st->nx * st->ny * 2 * (int64_t)sizeof(double);
    st->stats.kernel_launches += 1;
    st->stats.stage_launches += 1;
    st->stats.pair_launches += 1;
    st->stats.rhs_evals += 2;
    st->stats.stage_bytes += pb;
    st->stats.pair_bytes += pb;
    return RK_OK;
}

// one fixed Runge–Kutta step, u <- u_new (does not touch the Adams–Bashforth history)
static rk_status rk_fixed_step(rk_state st, int scheme, double dt) {
    if (!st->fused_kernels) {
        TRY(unfused_stages(st, scheme, dt, false, 0.0, 0.0));
        swap_u(st);
        st->stats.steps += 1;
        return RK_OK;
    }
    if (coop_path(st, scheme)) return coop_steps(st, scheme, dt, 1);
    if (st->grid && halo_path(st)) TRY(ensure_halo(st));  // the loopback's 1-rank communicator
    if (pair_path(st, scheme)) return pair_steps(st, scheme, dt, 1);
    if (fused_path(st, scheme)) return fused_steps(st, scheme, dt, 1);
    if (st->grid && fixed_tail_ok(st, scheme)) {
        auto plan = build_plan(scheme, 5, dt);
        TRY(run_grid_plan(st, plan, dt, 0.0, 0.0));
        TRY(fixed_tail_pair(st, scheme, dt));
    } else if (st->grid) {
        auto plan = build_plan(scheme, 0, dt);
        TRY(run_grid_plan(st, plan, dt, 0.0, 0.0));
    } else {
        TRY(run_pointwise(st, scheme, dt, 1, false, 0.0, 0.0));
    }
    swap_u(st);
    st->k1_valid = false;
    st->stats.steps += 1;
    return RK_OK;
}

// ---- Adams–Bashforth k-step (Table 1 multi-step row; R-23, R-24) ---------
static void ab_invalidate(rk_state st) {
    st->ab_k = 0;
    st->ab_count = 0;
}

static rk_status ab_prepare(rk_state st, int k, double dt) {
    if (st->ab_k != k || st->ab_dt != dt) {  // new method or step size: restart the history
        st->ab_k = k;
        st->ab_dt = dt;
        st->ab_count = 0;
    }
    for (int j = st->nhist; j < k; ++j) {
        TRY(alloc_array(st, &st->hist[j], &st->tm_hist[j]));
        st->nhist = j + 1;
    }
    return RK_OK;
}

// the scratch slot hist[k-1] (just written with f_n) becomes the newest entry
static void ab_rotate(rk_state st) {
    const int k = st->ab_k;
    double* p = st->hist[k - 1];
    const Maps m = st->tm_hist[k - 1];
    for (int j = k - 1; j > 0; --j) {
        st->hist[j] = st->hist[j - 1];
        st->tm_hist[j] = st->tm_hist[j - 1];
    }
    st->hist[0] = p;
    st->tm_hist[0] = m;
    st->ab_count = std::min(st->ab_count + 1, k - 1);
}

static rk_status run_gs_stage(rk_state st, const StagePlan& p, double dt, double atol, double rtol);

// Bootstrap step (R-23): f_n = F(u_n) into the history, then one RKF78 step.
static rk_status ab_bootstrap_step(rk_state st, double dt) {
    const int k = st->ab_k;
    if (st->grid) {
        StagePlan p;  // k1-type stage (no inputs but u) writing into the scratch slot
        p.scheme = RK_RK4;
        p.stage = 0;
        p.sp = stage_spec(RK_RK4, false, 0);
        p.out_hist = k - 1;
        TRY(run_gs_stage(st, p, dt, 0.0, 0.0));
    } else {
        CK_CTX(st->ctx, launch_rhs_pointwise(st->u, st->hist[k - 1], st->count, st->rhs, st->lambda,
                                             st->ctx->stream, st->ctx->num_sms));
        st->stats.kernel_launches += 1;
        st->stats.rhs_evals += 1;
    }
    ab_rotate(st);
    return rk_fixed_step(st, RK_FEHLBERG78, dt);
}

// nsteps Adams–Bashforth (abm = false) or Adams–Bashforth–Moulton PECE (abm = true) steps,
// bootstrapping first while the history is short (R-23); the history ring is shared: it holds
// F at the past points of the trajectory whichever Adams method produced them.
static rk_status ab_steps(rk_state st, int k, double dt, int64_t nsteps, bool abm = false) {
    TRY(ab_prepare(st, k, dt));
    st->k1_valid = false;  // u moves (vectors: in place); k[0] no longer holds F(u)
    while (nsteps > 0 && st->ab_count < k - 1) {
        TRY(ab_bootstrap_step(st, dt));
        --nsteps;
    }
    if (nsteps <= 0) return RK_OK;
    double g[8], m[8];
    for (int j = 0; j < k; ++j) {
        g[j] = dt * rat_double(ab_beta(k, j));
        m[j] = dt * rat_double(am_beta(k, j));
    }
    if (!st->grid) {  // all remaining steps in one launch, history in registers
        AbPwArgs a{};
        a.u = st->u;
        for (int j = 0; j < k - 1; ++j) a.hist[j] = st->hist[j];
        a.count = st->count;
        a.rhs = st->rhs;
        a.lambda = st->lambda;
        for (int j = 0; j < k; ++j) {
            a.g[j] = g[j];
            a.m[j] = m[j];
        }
        while (nsteps > 0) {
            a.nsteps = (int)std::min<int64_t>(nsteps, 1 << 20);
            if (abm) CK_CTX(st->ctx, launch_abm_pointwise(k, a, st->ctx->stream, st->ctx->num_sms));
            else CK_CTX(st->ctx, launch_ab_pointwise(k, a, st->ctx->stream, st->ctx->num_sms));
            st->stats.kernel_launches += 1;
            st->stats.rhs_evals += (abm ? 2 : 1) * (int64_t)a.nsteps;
            st->stats.steps += a.nsteps;
            nsteps -= a.nsteps;
        }
        return RK_OK;
    }
    if (abm) {
        for (; nsteps > 0; --nsteps) {
            StagePlan e;  // E: f_n = F(u_n) into the scratch slot
            e.scheme = RK_RK4;
            e.stage = 0;
            e.sp = stage_spec(RK_RK4, false, 0);
            e.out_hist = k - 1;
            TRY(run_gs_stage(st, e, dt, 0.0, 0.0));
            StagePlan p;  // PEC: Y = u_p from f_n .. f_{n-k+1}; corrector into u_new
            p.scheme = kSchemeABM0 + k;
            p.stage = 0;
            p.sp = stage_spec(p.scheme, false, 0);
            for (int s = 0; s < k; ++s) p.g[s] = g[s];
            for (int s = 0; s < k - 1; ++s) p.beta[s] = m[s + 1];
            p.beta_new = m[0];
            TRY(run_gs_stage(st, p, dt, 0.0, 0.0));
            swap_u(st);
            ab_rotate(st);
            st->stats.steps += 1;
        }
        return RK_OK;
    }
    for (; nsteps > 0; --nsteps) {
        StagePlan p;
        p.scheme = kSchemeAB0 + k;
        p.stage = 0;
        p.sp = stage_spec(p.scheme, false, 0);
        for (int s = 0; s < k - 1; ++s) p.beta[s] = g[s + 1];
        p.beta_new = g[0];
        p.out_hist = k > 1 ? k - 1 : -1;  // AB1 keeps no history (rk_stage_spec.h)
        TRY(run_gs_stage(st, p, dt, 0.0, 0.0));
        swap_u(st);
        ab_rotate(st);
        st->stats.steps += 1;
    }
    return RK_OK;
}

// one fixed step of any scheme (public do_step / integrate_const path)
static rk_status fixed_step(rk_state st, int scheme, double dt) {
    if (is_ab_scheme(scheme)) return ab_steps(st, scheme - kSchemeAB0, dt, 1);
    if (is_abm_scheme(scheme)) return ab_steps(st, scheme - kSchemeABM0, dt, 1, true);
    ab_invalidate(st);
    return rk_fixed_step(st, scheme, dt);
}

// one try: E (global), accept -> swap
static rk_status one_try(rk_state st, int scheme, double t, double dt, double atol, double rtol,
                         int* accepted, double* E_out, double* dt_next) {
    NvtxRange nv("rk try");
    rk_ctx ctx = st->ctx;
    const Coeffs C = coeffs_of(scheme);
    ab_invalidate(st);
    int fsal_k = -1;  // FSAL: buffer holding k_s = F(u_new), the next step's k1
    if (!st->fused_kernels) {
        TRY(unfused_stages(st, scheme, dt, true, atol, rtol));
        const Tableau T = tableau_of(scheme);
        if (is_fsal(T, true)) fsal_k = last_stage(T, true);
    } else if (st->grid) {
        auto plan = build_plan(scheme, st->controller == 1 ? 2 : 1, dt);
        if (plan.back().sp.epi == EPI_TAIL_ERR) fsal_k = plan.back().sp.out_k;
        TRY(run_grid_plan(st, plan, dt, atol, rtol));
    } else {
        TRY(run_pointwise(st, scheme, dt, 1, true, atol, rtol));
    }
    if (st->spike_at > 0 && ++st->spike_seen == st->spike_at) {  // RK_OPT_ERROR_SPIKE
        CK_CTX(ctx, launch_inject_max(st->d_err, 1e6, ctx->stream));
        st->stats.kernel_launches += 1;
    }
    TRY(allreduce_max_word(st, st->d_err));  // global max of E's bit pattern
    CK_CTX(ctx, launch_publish_word(st->d_err, st->h_err, ctx->stream));  // no copy engine
    st->stats.kernel_launches += 1;
    TRY(ctx_wait(ctx, ctx->stream));
    double E;
    std::memcpy(&E, st->h_err, sizeof E);
    st->stats.tries += 1;
    st->stats.last_err_ratio = E;
    if (std::isnan(E)) return fail(RK_ERR_DIVERGED, "non-finite error ratio at t=%.17g dt=%.17g", t, dt);
    double dtn = dt;
    const bool acc = adjust(st->controller, E, C.order, C.err_order, &dtn);
    st->stats.last_dt = dtn;
    if (acc) {
        swap_u(st);
        if (fsal_k > 0) {
            swap_k(st, 0, fsal_k);
            st->k1_valid = true;
        } else {
            st->k1_valid = false;
        }
        st->stats.accepted += 1;
    } else {
        st->stats.rejected += 1;
    }
    *accepted = acc ? 1 : 0;
    *E_out = E;
    *dt_next = dtn;
    return RK_OK;
}

// RK_OPT_USE_GRAPH: fixed grid steps replayed from one CUDA graph.  The stage
// launches of two consecutive steps (u/u_new ping-pong back to the starting buffers) are
// captured once and replayed, removing the per-launch host cost that bounds small grids
// (configs[2], 64^3).  Single GPU without the halo path; the launches are the same kernels
// with the same arguments, so results are identical.
static rk_status graph_steps(rk_state st, int scheme, double dt, int64_t n) {
    rk_ctx ctx = st->ctx;
    TRY(fixed_step(st, scheme, dt));  // allocates the k buffers, configures the kernels
    --n;
    const rk_stats before = st->stats;
    // capture on a private stream (the ctx stream may be the legacy default stream, which
    // cannot be captured); the graph is then launched on the ctx stream
    if (!ctx->capture) CK_CTX(ctx, cudaStreamCreateWithFlags(&ctx->capture, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    const cudaStream_t work = ctx->stream;
    CK_CTX(ctx, cudaStreamBeginCapture(ctx->capture, cudaStreamCaptureModeThreadLocal));
    ctx->stream = ctx->capture;
    rk_status rc = fixed_step(st, scheme, dt);
    if (rc == RK_OK) rc = fixed_step(st, scheme, dt);
    ctx->stream = work;
    const cudaError_t ce = cudaStreamEndCapture(ctx->capture, &graph);
    TRY(rc);
    CK_CTX(ctx, ce);
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CK_CTX(ctx, ie);
    // the capture ran the host bookkeeping of 2 steps (stats, pointer swaps) but no kernels
    const int64_t dl = st->stats.kernel_launches - before.kernel_launches;
    const int64_t ds = st->stats.stage_launches - before.stage_launches;
    const int64_t dr = st->stats.rhs_evals - before.rhs_evals;
    const int64_t db = st->stats.stage_bytes - before.stage_bytes;
    const int64_t pairs = n / 2;
    for (int64_t i = 0; i < pairs; ++i) CK_CTX(ctx, cudaGraphLaunch(exec, ctx->stream));
    cudaGraphExecDestroy(exec);
    st->stats.kernel_launches += dl * (pairs - 1);
    st->stats.stage_launches += ds * (pairs - 1);
    st->stats.rhs_evals += dr * (pairs - 1);
    st->stats.stage_bytes += db * (pairs - 1);
    st->stats.steps += 2 * (pairs - 1);
    if (n % 2) TRY(fixed_step(st, scheme, dt));
    return RK_OK;
}

// The whole adaptive integration of a vector state in one cooperative launch (RK_OPT_DEVICE_LOOP).
static rk_status device_adaptive_loop(rk_state st, int scheme, double t0, double t1, double dt0,
                                      double atol, double rtol, int64_t* accepted, int64_t* rejected) {
    rk_ctx ctx = st->ctx;
    const Coeffs C = coeffs_of(scheme);
    ab_invalidate(st);
    st->k1_valid = false;
    if (!st->d_loop) {
        void* p = nullptr;
        CK_CTX(ctx, cudaMalloc(&p, 3 * sizeof(unsigned long long) + sizeof(PwLoopResult)));
        st->d_loop = static_cast<unsigned long long*>(p);
    }
    PwLoopArgs a{};
    a.buf[0] = st->u;
    a.buf[1] = st->u_new;
    a.count = st->count;
    a.rhs = st->rhs;
    a.lambda = st->lambda;
    a.t0 = t0;
    a.t1 = t1;
    a.dt0 = dt0;
    a.atol = atol;
    a.rtol = rtol;
    for (int i = 0; i < 13; ++i) {
        for (int j = 0; j < 13; ++j) a.a[i][j] = C.a[i][j];
        a.b[i] = C.b[i];
        a.e[i] = C.e[i];
    }
    a.ctrl = st->controller;  // the host controller's exponents (adjust)
    const CtrlExp cx = ctrl_exponents(st->controller, C.order, C.err_order);
    a.e_rej = cx.e_rej;
    a.e_acc = cx.e_acc;
    a.emin = cx.emin;
    a.max_tries = st->max_tries;
    a.red = st->d_loop;
    a.res = reinterpret_cast<PwLoopResult*>(st->d_loop + 3);
    CK_CTX(ctx, cudaMemsetAsync(st->d_loop, 0, 3 * sizeof(unsigned long long) + sizeof(PwLoopResult), ctx->stream));
    if (st->grid) {  // K5: the stencil stages, error max and controller in one cooperative launch
        GsCoopLoopArgs g{};
        TRY(ensure_k(st, std::max(coop_last_stage_adaptive(scheme), 1)));
        for (int b = 0; b < 2; ++b)
            if (!st->ybuf[b]) TRY(alloc_array(st, &st->ybuf[b], nullptr));
        g.c.buf[0] = st->u;
        g.c.buf[1] = st->u_new;
        for (int j = 0; j < 13; ++j) g.c.k[j] = j < st->nk ? st->k[j] : nullptr;
        g.c.ybuf[0] = st->ybuf[0];
        g.c.ybuf[1] = st->ybuf[1];
        TRY(ensure_k5bar(st));
        g.c.bar = st->k5bar;
        g.c.geo = st->geo;
        g.c.d1 = st->d1;
        g.c.d2 = st->d2;
        g.c.F = st->F;
        g.c.FK = st->F + st->K;
        g.c.inv_h2 = 1.0 / (st->h * st->h);
        for (int i = 0; i < 13; ++i) {
            for (int j = 0; j < 13; ++j) g.A[i][j] = a.a[i][j];
            g.B[i] = a.b[i];
            g.Ew[i] = a.e[i];
        }
        g.t0 = t0;
        g.t1 = t1;
        g.dt0 = dt0;
        g.atol = atol;
        g.rtol = rtol;
        g.e_rej = a.e_rej;
        g.e_acc = a.e_acc;
        g.emin = a.emin;
        g.ctrl = a.ctrl;
        g.max_tries = a.max_tries;
        g.red = a.red;
        g.res = a.res;
        CK_CTX(ctx, launch_gs_coop_adaptive(scheme, g, ctx->stream, ctx->device));
    } else {
        CK_CTX(ctx, launch_pointwise_loop(scheme, a, ctx->stream, ctx->device));
    }
    PwLoopResult r{};
    CK_CTX(ctx, cudaMemcpyAsync(&r, a.res, sizeof r, cudaMemcpyDeviceToHost, ctx->stream));
    TRY(ctx_wait(ctx, ctx->stream));
    if (r.which) swap_u(st);
    const int64_t tries = r.accepted + r.rejected;
    st->stats.kernel_launches += 1;
    st->stats.tries += tries;
    st->stats.accepted += r.accepted;
    st->stats.rejected += r.rejected;
    st->stats.rhs_evals += tries * (int64_t)(st->grid ? coop_last_stage_adaptive(scheme) + 1 : num_stages(scheme, true));
    st->stats.last_err_ratio = r.last_E;
    st->stats.last_dt = r.dt;
    if (accepted) *accepted = r.accepted;
    if (rejected) *rejected = r.rejected;
    switch (r.status) {
    case 0: return RK_OK;
    case 5: return fail(RK_ERR_DIVERGED, "non-finite error ratio at t=%.17g dt=%.17g", r.t, r.dt);
    case 6: return fail(RK_ERR_DT_UNDERFLOW, "dt underflow at t=%.17g", r.t);
    case 7: return fail(RK_ERR_STALL, "more than %d tries at t=%.17g", st->max_tries, r.t);
    default: return fail(RK_ERR_CUDA, "device loop status %d", r.status);
    }
}

// ------------------------------------------------------------------------------------
// Device-resident adaptive loop for grids beyond the K5 size (RK_OPT_DEVICE_LOOP):
// the whole integrate_adaptive as ONE CUDA-graph launch with a conditional WHILE node.  Body:
//   select kernel (sets the SWITCH value: buffer parity x whether k1 must be evaluated)
//   -> SWITCH over 4 captured try bodies (the stage launches of one try for each u/u_new (and
//      FSAL k1/k7) buffer assignment, with and without stage 1), dt read on the device (dtp)
//   -> controller kernel (R-12 / R-28 with the correctly rounded pow, R-16 truncation, stall /
//      underflow / NaN rules, accept = flip the parity) which sets the WHILE condition.
// No host round trip per try; results equal the host loop bit for bit (same kernels, the same
// fl(dt*a_ij), the same controller function).
// ------------------------------------------------------------------------------------
struct GLoopDev {  // device-resident loop state
    double t, dt, t1, dt_try, last_E, last_dt;
    long long acc, rej, k1_evals;
    int tries, status, parity, need_k1;
};
struct GLoopParams {
    double e_rej, e_acc, emin;
    int ctrl, max_tries, fsal;
};

__global__ void gloop_select_kernel(const GLoopDev* s, cudaGraphConditionalHandle hs) {
    cudaGraphSetConditional(hs, (unsigned)(s->parity * 2 + s->need_k1));
}

__global__ void gloop_ctrl_kernel(GLoopDev* s, const unsigned long long* err, GLoopParams p,
                                  cudaGraphConditionalHandle hw) {
    const double E = __longlong_as_double((long long)*err);
    if (s->need_k1) s->k1_evals += 1;
    s->last_E = E;
    if (isnan(E)) {  // R-14: NaN -> RK_ERR_DIVERGED
        s->status = RK_ERR_DIVERGED;
        cudaGraphSetConditional(hw, 0);
        return;
    }
    int ok = 0;
    double dt = step_adjust_dev(E, p.e_rej, p.e_acc, p.emin, p.ctrl, s->dt_try, &ok);
    s->last_dt = dt;
    double t = s->t;
    if (ok) {
        t = t + s->dt_try;
        s->t = t;
        s->acc += 1;
        s->parity ^= 1;
        s->need_k1 = p.fsal ? 0 : 1;
        s->tries = 0;
        if (!(s->t1 - t > DBL_EPSILON)) {  // R-16: t1 reached
            s->dt = dt;
            cudaGraphSetConditional(hw, 0);
            return;
        }
        if ((t + dt) - s->t1 > DBL_EPSILON) dt = s->t1 - t;
    } else {
        s->rej += 1;
        s->need_k1 = 0;  // k1 = F(u) of this u is valid (FSAL or evaluated by this try)
        if (++s->tries >= p.max_tries) {
            s->dt = dt;
            s->status = RK_ERR_STALL;
            cudaGraphSetConditional(hw, 0);
            return;
        }
    }
    s->dt = dt;
    if (dt < 16.0 * DBL_EPSILON * fmax(fabs(t), 1.0)) {
        s->status = RK_ERR_DT_UNDERFLOW;
        cudaGraphSetConditional(hw, 0);
        return;
    }
    s->dt_try = dt;
    cudaGraphSetConditional(hw, 1);
}

struct GraphLoop {
    cudaGraphExec_t exec = nullptr;
    GLoopDev* dev = nullptr;
    // what the captured launches baked in
    int scheme = -1, ctrl = -1, fsal_k = -1, max_tries = 0;
    double atol = 0, rtol = 0, d1 = 0, d2 = 0, F = 0, K = 0, h = 0;
    double* bu[2] = {};   // parity p: u = bu[p], u_new = bu[1-p]
    Maps mu[2]{};
    double* bk[2] = {};   // FSAL, parity p: k1 = bk[p], k7 = bk[1-p]
    Maps mk[2]{};
    double* k[13] = {};   // every k buffer pointer at capture
    int nk = 0;
    int64_t try_bytes = 0, k1_bytes = 0;  // algorithmic bytes of stages 2..s / of stage 1
    int nstages = 0;
};

static void gloop_destroy(rk_state st) {
    GraphLoop* g = st->gloop;
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    cudaFree(g->dev);
    delete g;
    st->gloop = nullptr;
}

// one GPU without exchange, or the P2P transport (halos and the E allreduce in this library's
// kernels); the NCCL transport keeps the host loop (NCCL calls inside conditional graph bodies
// are not relied on)
static bool gloop_path(rk_state st) {
    return st->device_loop && st->fused_kernels && st->grid && st->rhs == RHS_GRAY_SCOTT &&
           (!halo_path(st) || p2p_needed(st)) &&
           st->check_finite == 0 && !st->timing;
}

static int64_t plan_stage_bytes(rk_state st, const StagePlan& p) {
    const int64_t arrays = 1 + p.sp.nslots + (p.sp.out_k >= 0 ? 1 : 0) + (p.sp.writes_u ? 1 : 0) +
                           (p.sp.out_w >= 0 ? 1 : 0) + (p.sp.out_e >= 0 ? 1 : 0) + (p.sp.out_z >= 0 ? 1 : 0);
    return st->local * st->nx * st->ny * 2 * (int64_t)sizeof(double) * arrays;
}

static void gloop_assign(rk_state st, GraphLoop* g, int parity) {
    st->u = g->bu[parity];
    st->u_new = g->bu[1 - parity];
    st->tm_u = g->mu[parity];
    st->tm_unew = g->mu[1 - parity];
    if (g->fsal_k > 0) {
        st->k[0] = g->bk[parity];
        st->k[g->fsal_k] = g->bk[1 - parity];
        st->tm_k[0] = g->mk[parity];
        st->tm_k[g->fsal_k] = g->mk[1 - parity];
    }
}

static bool gloop_matches(rk_state st, const GraphLoop* g, int scheme, double atol, double rtol) {
    if (!g || !g->exec || g->scheme != scheme || g->ctrl != st->controller || g->max_tries != st->max_tries ||
        g->atol != atol || g->rtol != rtol ||
        g->d1 != st->d1 || g->d2 != st->d2 || g->F != st->F || g->K != st->K || g->h != st->h || g->nk != st->nk)
        return false;
    if (!((st->u == g->bu[0] && st->u_new == g->bu[1]) || (st->u == g->bu[1] && st->u_new == g->bu[0]))) return false;
    for (int j = 0; j < st->nk; ++j) {
        if (g->fsal_k > 0 && (j == 0 || j == g->fsal_k)) {
            if (st->k[j] != g->bk[0] && st->k[j] != g->bk[1]) return false;
        } else if (st->k[j] != g->k[j]) {
            return false;
        }
    }
    return true;
}

static rk_status gloop_build(rk_state st, int scheme, double atol, double rtol) {
    rk_ctx ctx = st->ctx;
    gloop_destroy(st);
    const int adaptive = st->controller == 1 ? 2 : 1;
    const std::vector<StagePlan> plan = build_plan(scheme, adaptive, 1.0);  // raw coefficients
    TRY(ensure_k(st, plan_num_k(plan)));
    GraphLoop* g = new GraphLoop();
    st->gloop = g;
    g->scheme = scheme;
    g->ctrl = st->controller;
    g->max_tries = st->max_tries;
    g->atol = atol;
    g->rtol = rtol;
    g->d1 = st->d1;
    g->d2 = st->d2;
    g->F = st->F;
    g->K = st->K;
    g->h = st->h;
    g->nk = st->nk;
    g->nstages = (int)plan.size();
    g->fsal_k = plan.back().sp.epi == EPI_TAIL_ERR ? plan.back().sp.out_k : -1;
    g->bu[0] = st->u;
    g->bu[1] = st->u_new;
    g->mu[0] = st->tm_u;
    g->mu[1] = st->tm_unew;
    if (g->fsal_k > 0) {
        g->bk[0] = st->k[0];
        g->bk[1] = st->k[g->fsal_k];
        g->mk[0] = st->tm_k[0];
        g->mk[1] = st->tm_k[g->fsal_k];
    }
    for (int j = 0; j < st->nk; ++j) g->k[j] = st->k[j];
    for (const StagePlan& p : plan) (p.stage == 0 ? g->k1_bytes : g->try_bytes) += plan_stage_bytes(st, p);
    if (dp_tail_pair_ok(st, plan))  // stages 6 + 7 as the K8 tail pair: 7 arrays instead of their 10
        g->try_bytes += 7 * st->local * st->nx * st->ny * 2 * (int64_t)sizeof(double) -
                        plan_stage_bytes(st, plan[5]) - plan_stage_bytes(st, plan[6]);
    if (head_pair_ok(st, plan))  // 2 + 3 as the head pair: 4 arrays instead of 7
        g->try_bytes += 4 * st->local * st->nx * st->ny * 2 * (int64_t)sizeof(double) -
                        plan_stage_bytes(st, plan[1]) - plan_stage_bytes(st, plan[2]);
    CK_CTX(ctx, cudaMalloc((void**)&g->dev, sizeof(GLoopDev)));
    if (!ctx->capture) CK_CTX(ctx, cudaStreamCreateWithFlags(&ctx->capture, cudaStreamNonBlocking));
    TRY(ensure_halo(st));                    // ghost buffers / events exist before the capture
    if (p2p_needed(st)) TRY(ensure_p2p(st));  // ... and the P2P mappings (collective)

    cudaGraph_t graph = nullptr;
    CK_CTX(ctx, cudaGraphCreate(&graph, 0));
    struct GraphGuard {
        cudaGraph_t g;
        ~GraphGuard() { if (g) cudaGraphDestroy(g); }
    } guard{graph};
    cudaGraphConditionalHandle hw, hs;
    CK_CTX(ctx, cudaGraphConditionalHandleCreate(&hw, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp{};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CK_CTX(ctx, cudaGraphAddNode(&wnode, graph, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    CK_CTX(ctx, cudaGraphConditionalHandleCreate(&hs, body, 0, 0));
    // select -> switch -> controller
    cudaGraphNode_t sel, sw, ctl;
    {
        GLoopDev* dv = g->dev;
        void* args[] = {&dv, &hs};
        cudaKernelNodeParams kp{};
        kp.func = (void*)gloop_select_kernel;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = args;
        CK_CTX(ctx, cudaGraphAddKernelNode(&sel, body, nullptr, 0, &kp));
    }
    cudaGraphNodeParams sp{};
    sp.type = cudaGraphNodeTypeConditional;
    sp.conditional.handle = hs;
    sp.conditional.type = cudaGraphCondTypeSwitch;
    sp.conditional.size = 4;
    CK_CTX(ctx, cudaGraphAddNode(&sw, body, &sel, 1, &sp));
    // the four try bodies, captured with this state's launch code
    const bool k1_save = st->k1_valid;
    const rk_stats stats_save = st->stats;
    const cudaStream_t work = ctx->stream;
    const double* dtp = &g->dev->dt_try;
    rk_status rc = RK_OK;
    for (int j = 0; j < 4 && rc == RK_OK; ++j) {
        const int parity = j / 2, need_k1 = j % 2;
        gloop_assign(st, g, parity);
        cudaError_t ce = cudaStreamBeginCaptureToGraph(ctx->capture, sp.conditional.phGraph_out[j], nullptr, nullptr, 0,
                                                       cudaStreamCaptureModeThreadLocal);
        if (ce != cudaSuccess) {
            ctx->poisoned = RK_ERR_CUDA;
            rc = fail(RK_ERR_CUDA, "capture of the try body: %s", cudaGetErrorString(ce));
            break;
        }
        ctx->stream = ctx->capture;
        st->gl_dtp = dtp;
        st->k1_valid = need_k1 == 0;
        rc = run_grid_plan(st, plan, 1.0, atol, rtol);
        if (rc == RK_OK) rc = allreduce_max_word(st, st->d_err);  // P2P transport: NVLink atomics
        st->gl_dtp = nullptr;
        ctx->stream = work;
        cudaGraph_t out = nullptr;
        ce = cudaStreamEndCapture(ctx->capture, &out);
        if (rc == RK_OK && ce != cudaSuccess) {
            ctx->poisoned = RK_ERR_CUDA;
            rc = fail(RK_ERR_CUDA, "capture of the try body: %s", cudaGetErrorString(ce));
        }
    }
    gloop_assign(st, g, 0);  // bu[0] / bk[0] are the assignment found at the start of the build
    st->stats = stats_save;
    st->k1_valid = k1_save;
    TRY(rc);
    {
        GLoopDev* dv = g->dev;
        unsigned long long* err = st->d_err;
        GLoopParams prm{};
        const Coeffs C = coeffs_of(scheme);
        const CtrlExp cx = ctrl_exponents(st->controller, C.order, C.err_order);
        prm.e_rej = cx.e_rej;
        prm.e_acc = cx.e_acc;
        prm.emin = cx.emin;
        prm.ctrl = st->controller;
        prm.max_tries = st->max_tries;
        prm.fsal = g->fsal_k > 0 ? 1 : 0;
        void* args[] = {&dv, &err, &prm, &hw};
        cudaKernelNodeParams kp{};
        kp.func = (void*)gloop_ctrl_kernel;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = args;
        CK_CTX(ctx, cudaGraphAddKernelNode(&ctl, body, &sw, 1, &kp));
    }
    CK_CTX(ctx, cudaGraphInstantiate(&g->exec, graph, 0));
    return RK_OK;
}

static rk_status graph_adaptive_loop(rk_state st, int scheme, double t0, double t1, double dt0, double atol,
                                     double rtol, int64_t* accepted, int64_t* rejected) {
    NvtxRange nv("rk device-resident try loop (graph)");
    rk_ctx ctx = st->ctx;
    ab_invalidate(st);
    if (accepted) *accepted = 0;
    if (rejected) *rejected = 0;
    double t = t0, dt = dt0;
    if (!(t1 - t > DBL_EPSILON)) return RK_OK;
    if ((t + dt) - t1 > DBL_EPSILON) dt = t1 - t;
    if (dt < 16.0 * DBL_EPSILON * std::max(std::fabs(t), 1.0)) return fail(RK_ERR_DT_UNDERFLOW, "dt underflow at t=%.17g", t);
    if (!gloop_matches(st, st->gloop, scheme, atol, rtol)) TRY(gloop_build(st, scheme, atol, rtol));
    GraphLoop* g = st->gloop;
    const int p0 = st->u == g->bu[0] ? 0 : 1;
    bool need_k1 = !st->k1_valid;
    if (g->fsal_k > 0 && st->k[0] != g->bk[p0]) need_k1 = true;  // a valid k1 sits in the other buffer
    gloop_assign(st, g, p0);
    GLoopDev h{};
    h.t = t;
    h.dt = dt;
    h.t1 = t1;
    h.dt_try = dt;
    h.parity = p0;
    h.need_k1 = need_k1 ? 1 : 0;
    CK_CTX(ctx, cudaMemcpyAsync(g->dev, &h, sizeof h, cudaMemcpyHostToDevice, ctx->stream));
    CK_CTX(ctx, cudaGraphLaunch(g->exec, ctx->stream));
    CK_CTX(ctx, cudaMemcpyAsync(&h, g->dev, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    TRY(ctx_wait(ctx, ctx->stream));
    gloop_assign(st, g, h.parity);
    st->k1_valid = h.need_k1 == 0;
    const int64_t tries = h.acc + h.rej;
    st->stats.tries += tries;
    st->stats.accepted += h.acc;
    st->stats.rejected += h.rej;
    const int64_t launches = tries * (g->nstages - 1) + h.k1_evals;
    st->stats.stage_launches += launches;
    st->stats.rhs_evals += launches;
    st->stats.kernel_launches += launches + 2 * tries;
    st->stats.stage_bytes += tries * g->try_bytes + h.k1_evals * g->k1_bytes;
    st->stats.last_err_ratio = h.last_E;
    st->stats.last_dt = h.last_dt;
    if (accepted) *accepted = h.acc;
    if (rejected) *rejected = h.rej;
    switch (h.status) {
    case 0: return RK_OK;
    case RK_ERR_DIVERGED: return fail(RK_ERR_DIVERGED, "non-finite error ratio at t=%.17g dt=%.17g", h.t, h.dt_try);
    case RK_ERR_DT_UNDERFLOW: return fail(RK_ERR_DT_UNDERFLOW, "dt underflow at t=%.17g", h.t);
    case RK_ERR_STALL: return fail(RK_ERR_STALL, "more than %d tries at t=%.17g", st->max_tries, h.t);
    default: return fail(RK_ERR_CUDA, "device loop status %d", h.status);
    }
}

// ====================================================================================
// C-ABI
// ====================================================================================
extern "C" {

int rk_abi_version(void) { return RK_ABI_VERSION; }

const char* rk_last_error(void) { return g_err.c_str(); }

rk_status rk_partition(int64_t n_global, int world, int rank, int64_t* begin, int64_t* count) {
    if (!begin || !count || world < 1 || rank < 0 || rank >= world || n_global < 1)
        return fail(RK_ERR_ARG, "rk_partition: bad arguments");
    const int64_t base = n_global / world, rem = n_global % world;
    *count = base + (rank < rem ? 1 : 0);
    *begin = rank * base + std::min<int64_t>(rank, rem);
    if (*count < 1) return fail(RK_ERR_ARG, "rank %d would own no plane/element", rank);
    return RK_OK;
}

rk_status rk_tableau(rk_scheme scheme, double* a, double* b, double* e, double* c, int* s,
                     int* order, int* err_order) {
    if (!valid_scheme(scheme)) return fail(RK_ERR_ARG, "bad scheme %d", (int)scheme);
    const Coeffs C = coeffs_of(scheme);
    for (int i = 0; i < C.s; ++i) {
        for (int j = 0; j < C.s; ++j)
            if (a) a[i * C.s + j] = j < i ? C.a[i][j] : 0.0;
        if (b) b[i] = C.b[i];
        if (e) e[i] = C.e[i];
        if (c) c[i] = C.c[i];
    }
    if (s) *s = C.s;
    if (order) *order = C.order;
    if (err_order) *err_order = C.err_order;
    return RK_OK;
}

rk_status rk_controller(rk_scheme scheme, double E, double* dt, int* accepted) {
    if (!valid_scheme(scheme) || !dt || !accepted) return fail(RK_ERR_ARG, "bad arguments");
    const Coeffs C = coeffs_of(scheme);
    if (C.err_order == 0) return fail(RK_ERR_UNSUPPORTED, "scheme has no error estimate");
    if (std::isnan(E)) return fail(RK_ERR_DIVERGED, "NaN error ratio");
    *accepted = step_adjust(E, C.order, C.err_order, dt) ? 1 : 0;
    return RK_OK;
}

rk_status rk_step_adjust(rk_scheme scheme, int controller, double E, double* dt, int* accepted) {
    if (!valid_scheme(scheme) || !dt || !accepted || (controller != 0 && controller != 1))
        return fail(RK_ERR_ARG, "bad arguments");
    const Coeffs C = coeffs_of(scheme);
    if (C.err_order == 0) return fail(RK_ERR_UNSUPPORTED, "scheme has no error estimate");
    if (std::isnan(E)) return fail(RK_ERR_DIVERGED, "NaN error ratio");
    *accepted = adjust(controller, E, C.order, C.err_order, dt) ? 1 : 0;
    return RK_OK;
}

rk_status rk_halo_plan_get(int world, int rank, rk_halo_plan* out) {
    if (!out || world < 1 || rank < 0 || rank >= world) return fail(RK_ERR_ARG, "rk_halo_plan_get: bad arguments");
    rk_halo_plan p{};
    p.up = (rank + 1) % world;
    p.down = (rank - 1 + world) % world;
    if (world <= 2) {
        // one peer is both neighbours: [lo|hi] lands in its [ghost_hi|ghost_lo]
        // (its plane above my top is my lowest plane, its plane below its bottom my top one)
        p.nmsg = 2;
        p.msg[0] = {0, p.up, 0, 2};
        p.msg[1] = {1, p.up, 0, 2};
    } else {
        p.nmsg = 4;
        p.msg[0] = {0, p.up, 1, 1};    // my top plane      -> up's ghost_lo
        p.msg[1] = {0, p.down, 0, 1};  // my bottom plane   -> down's ghost_hi
        p.msg[2] = {1, p.down, 1, 1};  // ghost_lo (z = -1) <- down's top plane
        p.msg[3] = {1, p.up, 0, 1};    // ghost_hi (z=nzl)  <- up's bottom plane
    }
    *out = p;
    return RK_OK;
}

rk_status rk_pair_ghost_plan(int world, int rank, int with_base, rk_pair_plan* out) {
    if (!out || world < 1 || rank < 0 || rank >= world) return fail(RK_ERR_ARG, "rk_pair_ghost_plan: bad arguments");
    rk_pair_plan p{};
    p.up = (rank + 1) % world;
    p.down = (rank - 1 + world) % world;
    const int na = with_base ? 2 : 1;
    for (int ar = 0; ar < na; ++ar) {  // sends: top planes to up, bottom planes to down
        const int np = ar == 0 ? 2 : 1;
        p.msg[p.nmsg++] = {0, p.up, ar, 1, np};
        p.msg[p.nmsg++] = {0, p.down, ar, 0, np};
    }
    for (int ar = 0; ar < na; ++ar) {  // receives: ghosts below from down, above from up
        const int np = ar == 0 ? 2 : 1;
        p.msg[p.nmsg++] = {1, p.down, ar, 0, np};
        p.msg[p.nmsg++] = {1, p.up, ar, 1, np};
    }
    *out = p;
    return RK_OK;
}

rk_status rk_nccl_unique_id(void* out) {
    if (!out) return fail(RK_ERR_ARG, "null output");
    static_assert(sizeof(ncclUniqueId) == RK_UNIQUE_ID_BYTES, "unique id size");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(RK_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
    std::memcpy(out, &id, sizeof id);
    return RK_OK;
}

rk_status rk_ctx_create(int rank, int world, int device, const void* uid, void* cuda_stream,
                        rk_ctx* out) {
    if (!out || world < 1 || rank < 0 || rank >= world || device < 0)
        return fail(RK_ERR_ARG, "rk_ctx_create: bad arguments");
    // world > 1 without a NCCL unique id: a context whose states use the P2P transport only
    // (halos and reductions in this library's kernels over CUDA IPC mappings that the caller
    // exchanges with rk_p2p_export / rk_p2p_import), e.g. several processes sharing one GPU
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(RK_ERR_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
    }
    if (device >= ndev) return fail(RK_ERR_ARG, "device %d >= device count %d", device, ndev);
    rk_ctx ctx = new rk_ctx_s();
    ctx->rank = rank;
    ctx->world = world;
    ctx->device = device;
    DeviceGuard g(device);
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    auto bail = [&](rk_status s) {
        if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
        if (ctx->comm) cudaStreamDestroy(ctx->comm);
        if (ctx->bnd) cudaStreamDestroy(ctx->bnd);
        delete ctx;
        return s;
    };
    if (cuda_stream) {
        ctx->stream = (cudaStream_t)cuda_stream;
    } else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(RK_ERR_CUDA, "cudaStreamCreate failed"));
        ctx->own_stream = true;
    }
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&ctx->comm, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&ctx->bnd, cudaStreamNonBlocking, hi) != cudaSuccess)
        return bail(fail(RK_ERR_CUDA, "comm / boundary stream create failed"));
    if (cudaMalloc((void**)&ctx->d_scratch, 8) != cudaSuccess ||
        cudaMallocHost((void**)&ctx->h_scratch, 8) != cudaSuccess)
        return bail(fail(RK_ERR_OOM, "scratch allocation failed"));
    if (world > 1 && uid) {
        ncclUniqueId id;
        std::memcpy(&id, uid, sizeof id);
        ncclResult_t r = ncclCommInitRank(&ctx->nccl, world, id, rank);
        if (r != ncclSuccess) return bail(fail(RK_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)));
    }
    *out = ctx;
    return RK_OK;
}

rk_status rk_ctx_set_allocator(rk_ctx ctx, rk_alloc_fn alloc, rk_free_fn free_fn, void* user) {
    if (!ctx) return fail(RK_ERR_ARG, "null ctx");
    if ((alloc == nullptr) != (free_fn == nullptr)) return fail(RK_ERR_ARG, "set both allocator functions or neither");
    if (!ctx->states.empty()) return fail(RK_ERR_STATE, "set the allocator before creating states");
    ctx->alloc_fn = alloc;
    ctx->free_fn = free_fn;
    ctx->alloc_user = user;
    return RK_OK;
}

rk_status rk_ctx_destroy(rk_ctx ctx) {
    if (!ctx) return RK_OK;
    DeviceGuard g(ctx->device);
    while (!ctx->states.empty()) rk_state_destroy(ctx->states.back());
    drain_stream(ctx, ctx->stream);
    if (ctx->nccl) ncclCommDestroy(ctx->nccl);
    for (auto e : ctx->marks) cudaEventDestroy(e);
    for (auto e : ctx->mark_pool) cudaEventDestroy(e);
    if (ctx->comm) cudaStreamDestroy(ctx->comm);
    if (ctx->bnd) cudaStreamDestroy(ctx->bnd);
    if (ctx->capture) cudaStreamDestroy(ctx->capture);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    cudaFree(ctx->d_scratch);
    cudaFreeHost(ctx->h_scratch);
    delete ctx;
    return RK_OK;
}

static rk_status state_common(rk_ctx ctx, rk_state st) {
    DeviceGuard g(ctx->device);
    st->p2p = ctx->world > 1 && !ctx->nccl;  // no NCCL: the P2P transport is the only one
    TRY(alloc_array(st, &st->u, &st->tm_u));
    TRY(alloc_array(st, &st->u_new, &st->tm_unew));
    CK_CTX(ctx, cudaMalloc((void**)&st->d_err, sizeof(unsigned long long)));
    CK_CTX(ctx, cudaMallocHost((void**)&st->h_err, sizeof(unsigned long long)));
    TRY(ctx_wait(ctx, ctx->stream));
    return RK_OK;
}

rk_status rk_state_create_grid(rk_ctx ctx, int64_t nx, int64_t ny, int64_t nz, int ncomp,
                               rk_state* out) {
    if (!ctx || !out) return fail(RK_ERR_ARG, "null argument");
    if (ctx->poisoned) return fail(ctx->poisoned, "context poisoned");
    if (nx < 1 || ny < 1 || nz < 1 || ncomp < 1 || ncomp > 6)
        return fail(RK_ERR_ARG, "bad grid dims / ncomp");
    if (nx * ny > (int64_t)1 << 30) return fail(RK_ERR_ARG, "plane too large");
    rk_state st = new rk_state_s();
    st->ctx = ctx;
    st->grid = true;
    st->ncomp = ncomp;
    st->nx = nx;
    st->ny = ny;
    st->nz = nz;
    rk_status s = rk_partition(nz, ctx->world, ctx->rank, &st->begin, &st->local);
    if (s != RK_OK) {
        delete st;
        return s;
    }
    st->count = st->local * nx * ny * ncomp;
    st->geo.nx = (int)nx;
    st->geo.ny = (int)ny;
    st->geo.nzl = (int)st->local;
    // row pitch: even (16-byte rows for TMA); RKB_PITCH_ALIGN (developer tuning knob) rounds
    // it up to a larger multiple of elements
    int palign = 2;
    if (const char* e = getenv("RKB_PITCH_ALIGN")) palign = std::max(2, atoi(e) / 2 * 2);
    st->geo.P = (int)((nx + 2 + palign - 1) / palign * palign);
    st->geo.cs = (ny + 2) * (int64_t)st->geo.P;
    st->geo.ps = ncomp * st->geo.cs;
    st->alloc = st->local * st->geo.ps;
    s = state_common(ctx, st);
    if (s != RK_OK) {
        rk_state_destroy(st);
        return s;
    }
    ctx->states.push_back(st);
    *out = st;
    return RK_OK;
}

rk_status rk_state_create_vector(rk_ctx ctx, int64_t n, int ncomp, rk_state* out) {
    if (!ctx || !out) return fail(RK_ERR_ARG, "null argument");
    if (ctx->poisoned) return fail(ctx->poisoned, "context poisoned");
    if (n < 1 || ncomp < 1 || ncomp > 6) return fail(RK_ERR_ARG, "bad vector size / ncomp");
    rk_state st = new rk_state_s();
    st->ctx = ctx;
    st->grid = false;
    st->ncomp = ncomp;
    st->n = n;
    rk_status s = rk_partition(n, ctx->world, ctx->rank, &st->begin, &st->local);
    if (s != RK_OK) {
        delete st;
        return s;
    }
    st->count = st->local * ncomp;
    st->alloc = st->count;
    s = state_common(ctx, st);
    if (s != RK_OK) {
        rk_state_destroy(st);
        return s;
    }
    ctx->states.push_back(st);
    *out = st;
    return RK_OK;
}

rk_status rk_state_destroy(rk_state st) {
    if (!st) return RK_OK;
    DeviceGuard g(st->ctx->device);
    bool idle = drain_stream(st->ctx, st->ctx->stream);
    idle = drain_stream(st->ctx, st->ctx->comm) && idle;
    idle = drain_stream(st->ctx, st->ctx->bnd) && idle;
    if (!idle) {  // kernels still spinning after a NCCL failure: leak the device buffers
        auto& v = st->ctx->states;
        v.erase(std::remove(v.begin(), v.end(), st), v.end());
        delete st;
        return RK_OK;
    }
    gloop_destroy(st);
    rk_ctx cx = st->ctx;
    dev_free(cx, st->uf_y);
    dev_free(cx, st->uf_e);
    dev_free(cx, st->u);
    dev_free(cx, st->u_new);
    for (int j = 0; j < st->nk; ++j) dev_free(cx, st->k[j]);
    for (int j = 0; j < st->nhist; ++j) dev_free(cx, st->hist[j]);
    dev_free(cx, st->ybuf[0]);
    cudaFree(st->k5bar);
    dev_free(cx, st->ybuf[1]);
    dev_free(cx, st->sendbuf);
    dev_free(cx, st->ghostbuf);
    for (void* m : st->ipc_mapped)
        if (m) cudaIpcCloseMemHandle(m);
    cudaFree(st->pghost);
    cudaFree(st->pflags);
    cudaFree(st->d_err);
    cudaFreeHost(st->h_err);
    dev_free(cx, st->pg_y);
    dev_free(cx, st->pg_w);
    dev_free(cx, st->pg_y2);
    cudaFree(st->d_loop);
    if (st->ev_pack) cudaEventDestroy(st->ev_pack);
    if (st->ev_halo) cudaEventDestroy(st->ev_halo);
    if (st->ev_ready) cudaEventDestroy(st->ev_ready);
    if (st->ev_bnd) cudaEventDestroy(st->ev_bnd);
    for (auto& p : st->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : st->event_pool) cudaEventDestroy(e);
    auto& v = st->ctx->states;
    v.erase(std::remove(v.begin(), v.end(), st), v.end());
    delete st;
    return RK_OK;
}

rk_status rk_state_local_range(rk_state st, int64_t* begin, int64_t* count) {
    TRY(check_state(st));
    if (begin) *begin = st->begin;
    if (count) *count = st->local;
    return RK_OK;
}

rk_status rk_state_local_size(rk_state st, int64_t* n_values) {
    TRY(check_state(st));
    if (n_values) *n_values = st->count;
    return RK_OK;
}

// dense user layout [z][c][y][x] <-> padded device layout [z][c][ny+2][P] (one 3D copy)
static cudaMemcpy3DParms pad_copy(rk_state st, const double* dense, double* padded, bool to_padded,
                                  cudaMemcpyKind kind) {
    cudaMemcpy3DParms p{};
    const size_t nx = (size_t)st->nx, ny = (size_t)st->ny;
    cudaPitchedPtr d = make_cudaPitchedPtr((void*)dense, nx * sizeof(double), nx, ny);
    cudaPitchedPtr q = make_cudaPitchedPtr((void*)padded, (size_t)st->geo.P * sizeof(double),
                                           (size_t)st->geo.P, ny + 2);
    if (to_padded) {
        p.srcPtr = d;
        p.dstPtr = q;
        p.dstPos = make_cudaPos(sizeof(double), 1, 0);
    } else {
        p.srcPtr = q;
        p.srcPos = make_cudaPos(sizeof(double), 1, 0);
        p.dstPtr = d;
    }
    p.extent = make_cudaExtent(nx * sizeof(double), ny, (size_t)(st->local * st->ncomp));
    p.kind = kind;
    return p;
}

rk_status rk_state_set(rk_state st, const double* src, int src_on_device) {
    TRY(check_state(st));
    if (!src) return fail(RK_ERR_ARG, "null src");
    rk_ctx ctx = st->ctx;
    DeviceGuard g(ctx->device);
    const cudaMemcpyKind kind = src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (st->grid) {
        cudaMemcpy3DParms p = pad_copy(st, src, st->u, true, kind);
        CK_CTX(ctx, cudaMemcpy3DAsync(&p, ctx->stream));
        CK_CTX(ctx, launch_fill_ring(st->u, st->geo, (int)(st->local * st->ncomp), ctx->stream));
        st->stats.kernel_launches += 1;
    } else {
        CK_CTX(ctx, cudaMemcpyAsync(st->u, src, sizeof(double) * (size_t)st->count, kind, ctx->stream));
    }
    TRY(ctx_wait(ctx, ctx->stream));
    st->k1_valid = false;
    ab_invalidate(st);
    return RK_OK;
}

rk_status rk_state_get(rk_state st, double* dst, int dst_on_device) {
    TRY(check_state(st));
    if (!dst) return fail(RK_ERR_ARG, "null dst");
    rk_ctx ctx = st->ctx;
    DeviceGuard g(ctx->device);
    const cudaMemcpyKind kind = dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (st->grid) {
        cudaMemcpy3DParms p = pad_copy(st, dst, st->u, false, kind);
        CK_CTX(ctx, cudaMemcpy3DAsync(&p, ctx->stream));
    } else {
        CK_CTX(ctx, cudaMemcpyAsync(dst, st->u, sizeof(double) * (size_t)st->count, kind, ctx->stream));
    }
    TRY(ctx_wait(ctx, ctx->stream));
    return RK_OK;
}

rk_status rk_set_rhs_exponential(rk_state st, double lambda) {
    TRY(check_state(st));
    st->rhs = RHS_EXP;
    st->lambda = lambda;
    st->k1_valid = false;
    ab_invalidate(st);
    return RK_OK;
}

rk_status rk_set_rhs_logistic(rk_state st) {
    TRY(check_state(st));
    st->rhs = RHS_LOGISTIC;
    st->k1_valid = false;
    ab_invalidate(st);
    return RK_OK;
}

rk_status rk_set_rhs_gray_scott(rk_state st, double d1, double d2, double F, double K, double h) {
    TRY(check_state(st));
    if (!st->grid || st->ncomp != 2)
        return fail(RK_ERR_STATE, "Gray-Scott RHS needs a grid state with ncomp == 2");
    if (!(h > 0.0) || !std::isfinite(d1) || !std::isfinite(d2) || !std::isfinite(F) || !std::isfinite(K))
        return fail(RK_ERR_ARG, "bad Gray-Scott parameters");
    st->rhs = RHS_GRAY_SCOTT;
    st->d1 = d1;
    st->d2 = d2;
    st->F = F;
    st->K = K;
    st->h = h;
    st->k1_valid = false;
    ab_invalidate(st);
    return RK_OK;
}

rk_status rk_set_option(rk_state st, int key, int64_t value) {
    TRY(check_state(st));
    switch (key) {
    case RK_OPT_HALO_OVERLAP: st->overlap = value != 0; break;
    case RK_OPT_HALO_LOOPBACK:
        if (value && st->ctx->world != 1) return fail(RK_ERR_ARG, "loopback needs world == 1");
        st->loopback = value != 0;
        break;
    case RK_OPT_MAX_TRIES:
        if (value < 1) return fail(RK_ERR_ARG, "max tries must be >= 1");
        st->max_tries = (int)value;
        break;
    case RK_OPT_TIMING: st->timing = value != 0; break;
    case RK_OPT_USE_GRAPH: st->use_graph = value != 0; break;
    case RK_OPT_DEVICE_LOOP: st->device_loop = value != 0; break;
    case RK_OPT_CONTROLLER:
        if (value != 0 && value != 1) return fail(RK_ERR_ARG, "controller must be 0 (Odeint) or 1 (SPEC)");
        st->controller = (int)value;
        break;
    case RK_OPT_CHECK_FINITE:
        if (value < 0) return fail(RK_ERR_ARG, "check interval must be >= 0");
        st->check_finite = value;
        st->since_check = 0;
        break;
    case RK_OPT_COOP_MAX_CELLS:
        if (value < 0) return fail(RK_ERR_ARG, "cell limit must be >= 0");
        st->coop_max_cells = value;
        break;
    case RK_OPT_FUSED_STEP:
        if (value < 0 || value > 3) return fail(RK_ERR_ARG, "RK_OPT_FUSED_STEP: 0, 1 (K6), 2 (K7) or 3 (K8)");
        st->fused = (int)value;
        break;
    case RK_OPT_COMM_TIMEOUT_MS:
        if (value < 0) return fail(RK_ERR_ARG, "RK_OPT_COMM_TIMEOUT_MS must be >= 0");
        st->ctx->comm_timeout_ms = value;
        break;
    case RK_OPT_ERROR_SPIKE:
        if (value < 0) return fail(RK_ERR_ARG, "RK_OPT_ERROR_SPIKE must be >= 0");
        st->spike_at = value;
        st->spike_seen = 0;
        break;
    case RK_OPT_CHECK_ARGS: st->check_args = value != 0; break;
    case RK_OPT_FUSED_KERNELS:
        if (st->fused_kernels != (value != 0)) st->k1_valid = false;  // k buffers are laid out differently
        st->fused_kernels = value != 0;
        break;
    case RK_OPT_HALO_P2P:
        if (value == 0 && st->ctx->world > 1 && !st->ctx->nccl)
            return fail(RK_ERR_ARG, "a context without NCCL has only the P2P transport");
        st->p2p = value != 0;
        break;
    default: return fail(RK_ERR_ARG, "unknown option %d", key);
    }
    return RK_OK;
}

rk_status rk_do_step(rk_state st, rk_scheme scheme, double t, double dt) {
    NvtxRange nv("rk_do_step");
    TRY(check_state(st));
    if (!valid_scheme(scheme)) return fail(RK_ERR_ARG, "bad scheme %d", (int)scheme);
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(RK_ERR_ARG, "dt must be finite and > 0");
    TRY(check_rhs(st));
    DeviceGuard g(st->ctx->device);
    TRY(check_collective_args(st, 1, {(double)scheme, t, dt}));
    TRY(fixed_step(st, scheme, dt));
    return finite_check(st, 1, t + dt, false);
}

rk_status rk_try_step(rk_state st, rk_scheme scheme, double t, double dt, double atol, double rtol,
                      int* accepted, double* err_ratio, double* dt_next) {
    TRY(check_state(st));
    if (!valid_scheme(scheme)) return fail(RK_ERR_ARG, "bad scheme %d", (int)scheme);
    if (!accepted || !err_ratio || !dt_next) return fail(RK_ERR_ARG, "null output");
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(RK_ERR_ARG, "dt must be finite and > 0");
    if (!(atol > 0.0) || !(rtol >= 0.0)) return fail(RK_ERR_ARG, "need atol > 0, rtol >= 0");
    if (coeffs_of(scheme).err_order == 0)
        return fail(RK_ERR_UNSUPPORTED, "scheme %d has no embedded error estimate", (int)scheme);
    TRY(check_rhs(st));
    DeviceGuard g(st->ctx->device);
    TRY(check_collective_args(st, 2, {(double)scheme, t, dt, atol, rtol}));
    return one_try(st, scheme, t, dt, atol, rtol, accepted, err_ratio, dt_next);
}

rk_status rk_integrate_const(rk_state st, rk_scheme scheme, double t0, double t1, double dt,
                             int64_t* steps) {
    NvtxRange nv("rk_integrate_const");
    TRY(check_state(st));
    if (!valid_scheme(scheme)) return fail(RK_ERR_ARG, "bad scheme %d", (int)scheme);
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(RK_ERR_ARG, "dt must be finite and > 0");
    if (!(t1 > t0)) return fail(RK_ERR_ARG, "need t1 > t0");
    TRY(check_rhs(st));
    DeviceGuard g(st->ctx->device);
    TRY(check_collective_args(st, 3, {(double)scheme, t0, t1, dt}));
    // Odeint integrate_const: while (t_n + dt) - t1 <= eps, t_n = t0 + n*dt
    int64_t n = 0;
    double t = t0;
    while ((t + dt) - t1 <= DBL_EPSILON) {
        ++n;
        t = t0 + (double)n * dt;
    }
    if (st->check_finite > 0 && (st->grid || is_multistep(scheme))) {
        // step by step, so a non-finite state is caught within check_finite steps
        for (int64_t i = 0; i < n; ++i) {
            TRY(fixed_step(st, scheme, dt));
            TRY(finite_check(st, 1, t0 + (double)(i + 1) * dt, false));
        }
    } else if (is_ab_scheme(scheme)) {
        TRY(ab_steps(st, scheme - kSchemeAB0, dt, n));
    } else if (is_abm_scheme(scheme)) {
        TRY(ab_steps(st, scheme - kSchemeABM0, dt, n, true));
    } else if (!st->fused_kernels) {
        for (int64_t i = 0; i < n; ++i) TRY(fixed_step(st, scheme, dt));
    } else if (!st->grid) {
        // pointwise RHS: all n steps of every element in registers, chunked launches
        ab_invalidate(st);
        int64_t left = n;
        const int64_t cap = st->check_finite > 0 ? std::min<int64_t>(st->check_finite, 1 << 20) : (1 << 20);
        while (left > 0) {
            const int chunk = (int)std::min<int64_t>(left, cap);
            TRY(run_pointwise(st, scheme, dt, chunk, false, 0.0, 0.0));
            swap_u(st);
            left -= chunk;
            TRY(finite_check(st, chunk, t0 + (double)(n - left) * dt, false));
        }
        st->k1_valid = false;
        st->stats.steps += n;
    } else if (coop_path(st, scheme)) {
        ab_invalidate(st);
        TRY(coop_steps(st, scheme, dt, n));
    } else if (st->use_graph && !halo_path(st) && !st->timing && n >= 5) {
        TRY(graph_steps(st, scheme, dt, n));
    } else {
        for (int64_t i = 0; i < n; ++i) TRY(fixed_step(st, scheme, dt));
    }
    TRY(finite_check(st, 0, t0 + (double)n * dt, true));
    TRY(ctx_wait(st->ctx, st->ctx->stream));
    if (steps) *steps = n;
    return RK_OK;
}

rk_status rk_integrate_adaptive(rk_state st, rk_scheme scheme, double t0, double t1, double dt0,
                                double atol, double rtol, int64_t* accepted, int64_t* rejected) {
    NvtxRange nv("rk_integrate_adaptive");
    TRY(check_state(st));
    if (!valid_scheme(scheme)) return fail(RK_ERR_ARG, "bad scheme %d", (int)scheme);
    if (!(dt0 > 0.0) || !std::isfinite(dt0)) return fail(RK_ERR_ARG, "dt0 must be finite and > 0");
    if (!(t1 > t0)) return fail(RK_ERR_ARG, "need t1 > t0");
    if (!(atol > 0.0) || !(rtol >= 0.0)) return fail(RK_ERR_ARG, "need atol > 0, rtol >= 0");
    if (coeffs_of(scheme).err_order == 0)
        return fail(RK_ERR_UNSUPPORTED, "scheme %d has no embedded error estimate", (int)scheme);
    TRY(check_rhs(st));
    DeviceGuard g(st->ctx->device);
    TRY(check_collective_args(st, 4, {(double)scheme, t0, t1, dt0, atol, rtol}));
    if (st->device_loop && st->fused_kernels && st->ctx->world == 1 &&
        (!st->grid || (!st->loopback && !st->p2p && st->local * st->nx * st->ny <= st->coop_max_cells))) {
        TRY(device_adaptive_loop(st, scheme, t0, t1, dt0, atol, rtol, accepted, rejected));
        return finite_check(st, 0, t1, true);
    }
    if (gloop_path(st)) return graph_adaptive_loop(st, scheme, t0, t1, dt0, atol, rtol, accepted, rejected);
    int64_t acc = 0, rej = 0;
    double t = t0, dt = dt0;
    rk_status rc = RK_OK;
    while (t1 - t > DBL_EPSILON) {
        if ((t + dt) - t1 > DBL_EPSILON) dt = t1 - t;
        int tries = 0;
        for (;;) {
            if (dt < 16.0 * DBL_EPSILON * std::max(std::fabs(t), 1.0)) {
                rc = fail(RK_ERR_DT_UNDERFLOW, "dt underflow at t=%.17g", t);
                goto done;
            }
            int ok = 0;
            double E = 0.0, dtn = dt;
            rc = one_try(st, scheme, t, dt, atol, rtol, &ok, &E, &dtn);
            if (rc != RK_OK) goto done;
            if (ok) {
                t = t + dt;
                dt = dtn;
                ++acc;
                rc = finite_check(st, 1, t, false);
                if (rc != RK_OK) goto done;
                break;
            }
            dt = dtn;
            ++rej;
            if (++tries >= st->max_tries) {
                rc = fail(RK_ERR_STALL, "more than %d tries at t=%.17g", st->max_tries, t);
                goto done;
            }
        }
    }
    rc = finite_check(st, 0, t, true);
done:
    if (accepted) *accepted = acc;
    if (rejected) *rejected = rej;
    return rc;
}

rk_status rk_lincomb(rk_state out, int k, const double* coef, const rk_state* in) {
    TRY(check_state(out));
    if (k < 1 || k > 14) return fail(RK_ERR_CONTRACT, "lincomb arity %d not in [1,14]", k);
    if (!coef || !in) return fail(RK_ERR_ARG, "null argument");
    LincombArgs a{};
    a.out = out->u;
    a.k = k;
    a.count = out->alloc;  // padded grids: ring copies combine linearly, pads stay 0
    for (int j = 0; j < k; ++j) {
        rk_state s = in[j];
        TRY(check_state(s));
        if (s->ctx != out->ctx || s->count != out->count || s->grid != out->grid ||
            s->ncomp != out->ncomp || s->nx != out->nx || s->ny != out->ny || s->nz != out->nz ||
            s->n != out->n)
            return fail(RK_ERR_CONTRACT, "lincomb input %d does not conform to the output", j);
        a.in[j] = s->u;
        a.coef[j] = coef[j];
    }
    DeviceGuard g(out->ctx->device);
    CK_CTX(out->ctx, launch_lincomb(a, out->ctx->stream, out->ctx->num_sms));
    out->stats.kernel_launches += 1;
    out->k1_valid = false;
    ab_invalidate(out);
    TRY(ctx_wait(out->ctx, out->ctx->stream));
    return RK_OK;
}

rk_status rk_norm_inf(rk_state st, double* out) {
    TRY(check_state(st));
    if (!out) return fail(RK_ERR_ARG, "null output");
    DeviceGuard g(st->ctx->device);
    TRY(check_collective_args(st, 5, {}));
    return global_norm_inf(st, out);
}

rk_status rk_eval_rhs(rk_state in, rk_state out) {
    TRY(check_state(in));
    TRY(check_state(out));
    if (in == out) return fail(RK_ERR_ARG, "eval_rhs: out must differ from in");
    if (in->ctx != out->ctx || in->count != out->count || in->grid != out->grid || in->ncomp != out->ncomp ||
        in->nx != out->nx || in->ny != out->ny || in->nz != out->nz || in->n != out->n)
        return fail(RK_ERR_CONTRACT, "eval_rhs: out does not conform to in");
    TRY(check_rhs(in));
    rk_ctx ctx = in->ctx;
    DeviceGuard g(ctx->device);
    TRY(check_collective_args(in, 6, {}));
    if (in->grid) {
        // the k1 = F(u) stage kernel of every scheme, its output redirected to out.u
        StagePlan p = build_plan(RK_RK4, 0, 0.0)[0];
        p.out_ptr = out->u;
        TRY(ensure_halo(in));
        TRY(run_gs_stage(in, p, 0.0, 0.0, 0.0));
    } else {
        CK_CTX(ctx, launch_rhs_pointwise(in->u, out->u, in->count, in->rhs, in->lambda, ctx->stream, ctx->num_sms));
        in->stats.kernel_launches += 1;
        in->stats.rhs_evals += 1;
    }
    out->k1_valid = false;
    ab_invalidate(out);
    return RK_OK;
}

rk_status rk_p2p_export(rk_state st, void* out, int64_t capacity, int64_t* nbytes) {
    TRY(check_state(st));
    if (!nbytes) return fail(RK_ERR_ARG, "null nbytes");
    *nbytes = (int64_t)sizeof(P2pHandles);
    if (!out) return RK_OK;  // size query
    if (capacity < (int64_t)sizeof(P2pHandles)) return fail(RK_ERR_ARG, "buffer too small (%lld < %lld)",
                                                           (long long)capacity, (long long)sizeof(P2pHandles));
    if (!st->p2p) return fail(RK_ERR_STATE, "the state does not use the P2P transport (RK_OPT_HALO_P2P)");
    DeviceGuard g(st->ctx->device);
    P2pHandles h{};
    TRY(p2p_export(st, &h));
    std::memcpy(out, &h, sizeof h);
    return RK_OK;
}

rk_status rk_p2p_import(rk_state st, const void* all, int64_t nbytes_per_rank) {
    TRY(check_state(st));
    if (!all || nbytes_per_rank != (int64_t)sizeof(P2pHandles))
        return fail(RK_ERR_ARG, "expected world x %lld bytes from rk_p2p_export", (long long)sizeof(P2pHandles));
    if (!st->p2p) return fail(RK_ERR_STATE, "the state does not use the P2P transport (RK_OPT_HALO_P2P)");
    if (st->p2p_ready) return fail(RK_ERR_STATE, "P2P transport already connected");
    DeviceGuard g(st->ctx->device);
    TRY(p2p_alloc(st));
    std::vector<P2pHandles> v((size_t)st->ctx->world);
    std::memcpy(v.data(), all, sizeof(P2pHandles) * v.size());
    return p2p_map(st, v.data());
}

rk_status rk_get_stats(rk_state st, rk_stats* out) {
    TRY(check_state(st));
    if (!out) return fail(RK_ERR_ARG, "null output");
    DeviceGuard g(st->ctx->device);
    TRY(resolve_timing(st));
    *out = st->stats;
    return RK_OK;
}

rk_status rk_reset_stats(rk_state st) {
    TRY(check_state(st));
    DeviceGuard g(st->ctx->device);
    TRY(resolve_timing(st));
    st->stats = rk_stats{};
    return RK_OK;
}

}  // extern "C"
