// rk_kernels.cuh — device kernels of librkb200 and their host launchers.
//
// K1 pointwise fused step (exp / logistic), K2 lincomb + halo-plane pack, K3 fused
// Gray–Scott stage kernel (TMA-fed), K4 max-norm reductions.  DESIGN.md §Kernels gives the
// roofline and the algorithmic bytes of each.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "rk_stage_spec.h"

namespace rkb {

// cudaFuncAttributeMaxDynamicSharedMemorySize once per kernel instance AND device: function
// attributes live in the device's context, so a process driving a second device sets them again.
template <typename K>
inline cudaError_t smem_attr_once(std::atomic<unsigned long long>& done, K* kernel, int bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_relaxed) & bit) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit);
    return e;
}

enum RhsKind { RHS_NONE = -1, RHS_EXP = 0, RHS_LOGISTIC = 1, RHS_GRAY_SCOTT = 2 };

// ---------------------------------------------------------------------------------------
// K1: pointwise step of a whole RK scheme in registers (vector states).
struct PwCoef {
    double g[13][13];  // dt * a_ij
    double beta[13];   // dt * b_j
    double delta[13];  // dt * (b_j - bhat_j)
};
struct PwArgs {
    const double* u;
    double* u_out;
    int64_t count;     // fp64 values (ncomp * local elements)
    int rhs;           // RHS_EXP / RHS_LOGISTIC
    double lambda;
    int nsteps;        // >= 1 fixed steps in registers (ignored with error ratio)
    double dt, atol, rtol;
    unsigned long long* errmax;  // error-ratio max (uint64 bits), non-null => error mode
    int ctrl;          // error ratio reading: 0 Odeint (R-12), 1 SPEC (R-28)
    PwCoef cf;
};
cudaError_t launch_pointwise(int scheme, const PwArgs& a, cudaStream_t st, int num_sms);

// K1 device-resident adaptive loop: the whole integrate_adaptive of a pointwise
// RHS in one cooperative launch -- tries, grid-wide error max, controller (double-double pow,
// rk_ddmath.cuh) and accept/reject all on the device, no host round trip per try.
struct PwLoopResult {
    int status;            // 0 ok, 5 diverged (NaN), 6 dt underflow, 7 stall (rk_status codes)
    int which;             // buffer holding the final u (0: buf[0], 1: buf[1])
    long long accepted, rejected;
    double t, dt, last_E, last_dt;
};
struct PwLoopArgs {
    double* buf[2];        // buf[0] = u on entry; ping-pong
    int64_t count;
    int rhs;
    double lambda;
    double t0, t1, dt0, atol, rtol;
    double a[13][13], b[13], e[13];  // the scheme's coefficients as doubles (rat_double)
    double e_rej, e_acc, emin;       // controller exponents / floor (host-computed, as the host
                                     // controller): Odeint -1/(q-1), -1/p, 5^-p; SPEC -1/(p-1), -1/p
    int ctrl;                        // 0 Odeint (R-12), 1 SPEC (R-28)
    int max_tries;
    unsigned long long* red;         // [3] zeroed: per-try error-max slots (rotating)
    PwLoopResult* res;
};
cudaError_t launch_pointwise_loop(int scheme, const PwLoopArgs& a, cudaStream_t st, int device);

// K1 (Adams–Bashforth): nsteps k-step updates with the history in registers.
struct AbPwArgs {
    double* u;         // in/out
    double* hist[7];   // f_{n-1} .. f_{n-k+1}, newest first (in/out)
    int64_t count;
    int rhs;
    double lambda;
    int nsteps;
    double g[8];       // dt*beta_j, newest first
    double m[8];       // Adams–Bashforth–Moulton: dt*m_j corrector weights (m_0: F(u_p))
};
cudaError_t launch_ab_pointwise(int k, const AbPwArgs& a, cudaStream_t st, int num_sms);
// K1 (Adams–Bashforth–Moulton, PECE): nsteps steps, history in registers, 2 RHS per step.
cudaError_t launch_abm_pointwise(int k, const AbPwArgs& a, cudaStream_t st, int num_sms);
// f = F(u) for a pointwise RHS (history bootstrap).
cudaError_t launch_rhs_pointwise(const double* u, double* f, int64_t count, int rhs, double lambda,
                                 cudaStream_t st, int num_sms);

// ---------------------------------------------------------------------------------------
// Grid arrays in HBM use a PADDED periodic layout: [z][c][ny+2][P] fp64 with P >= nx+2 even
// (16-byte rows for TMA); logical cell (x, y) sits at padded (x+1, y+1), and the producer
// of every array also writes the periodic copies x=-1 -> nx-1, x=nx -> 0 (and y alike) into
// the 1-cell ring, so a TMA box of (TX+2) x (TY+2) cells around any tile is exactly the
// periodic neighbourhood, with no wrap logic in the consumer.
struct GridGeom {
    int nx, ny, nzl;
    int P;          // padded row pitch (elements)
    int64_t cs;     // component stride = (ny+2)*P
    int64_t ps;     // plane stride = 2*cs
};

// Device-side handshake of the peer-to-peer halo path (RK_OPT_HALO_P2P).  The
// stage sequence number lives on the device (*seqp + 1 = this stage; the boundary launch's last
// CTA advances *seqp), so the same launches can be replayed from a CUDA graph.  A launch first
// waits until both wait flags reach its minimum (acquire, system scope): the pack launch (role
// 0) until both neighbours acknowledged stage seq-2 on this parity, the boundary launch (role 1)
// until both ghost planes of stage seq have landed.  Its last CTA to finish stores seq into
// both notify flags (release, system scope) -- flags that may live in a neighbour GPU's memory
// (CUDA IPC over NVLink).  count: a CTA completion counter, reset by the last CTA.  Ghost
// planes alternate between two parities, seq & 1.  on == 0: no handshake.
// Word layout of a rank's P2P flag block (IPC-exported; neighbours and, for the reduction, every
// rank write into it).
enum P2pFlag {
    P2P_READY_LO = 0, P2P_READY_HI = 1,  // ghost planes of stage seq landed (written by neighbours)
    P2P_ACK_LO = 2, P2P_ACK_HI = 3,      // neighbours consumed the planes this rank sent them
    P2P_COUNT = 4,                       // CTA completion counter of the current launch
    P2P_SEQ = 5,                         // stages completed (device-resident sequence number)
    P2P_RED0 = 6, P2P_RED1 = 7,          // allreduce(max) slots, double-buffered by round
    P2P_ARRIVE = 8,                      // allreduce arrivals (world per round, monotonic)
    P2P_ROUND = 9,                       // allreduce rounds completed by this rank
    P2P_FLAGS = 16
};
struct P2pSync {
    const unsigned long long* wait[2];
    unsigned long long* notify[2];
    unsigned long long* count;
    unsigned long long* seqp;
    int role;
    int on;
};

// K3: fused Gray–Scott stage kernel.  Which terms exist is compile-time (StageSpec of
// (scheme, adaptive, stage)); the runtime arguments are pointers, TMA maps and values.
struct GsStageArgs {
    CUtensorMap tm_base;             // Y source: u (or u_new for EPI_TAIL_ERR), tile+ring box
    CUtensorMap tm_slot[kMaxSlots];  // slot s: tile+ring box if it enters Y, else interior box
    CUtensorMap tm_glo, tm_ghi;      // ghost planes z=-1, z=nzl (multi-GPU); else periodic wrap
    CUtensorMap tm_glo1, tm_ghi1;    // P2P: the ghost planes of parity 1 (tm_glo/tm_ghi: parity 0)
    GridGeom geo;
    const double* base;              // raw pointers (pack kernel)
    const double* slot[kMaxSlots];
    double g[kMaxSlots];             // dt*a_ij per slot
    double beta[kMaxSlots];          // dt*b_j per slot
    double delta[kMaxSlots];         // dt*e_j per slot
    double beta_new, delta_new;      // weights of the k_i computed by this stage
    double g2[kMaxSlots], g2_new;    // EPI_AHEAD: dt*a_Fj per slot and dt*a_Fi (final stage F)
    double g3[kMaxSlots], g3_new;    // EPI_AHEAD with out_z (fixed-step tail pair): dt*a_Lj, dt*a_Li
    double* out_w;                   // EPI_AHEAD: partial final combination W
    double* out_z;                   // EPI_AHEAD with out_z: the last stage's base Z_L (ring)
    double* out_e;                   // EPI_AHEAD (error control): partial error sum E
    double* out_k;
    double* out_u;
    unsigned long long* errmax;
    double dt, atol, rtol;
    const double* dtp;               // non-null (device-resident try loop): this try's dt on the
                                     // device; g/beta/delta/g2 then hold the raw coefficients
    double d1, d2, F, FK, inv_h2;
    int has_glo, has_ghi;
    int z_lo, z_hi;                  // output planes [z_lo, z_hi) (zmode 0)
    int zchunk;                      // output planes per CTA
    int zmode;                       // 0: contiguous chunks; 1: chunk 0 = plane 0, chunk 1 = nzl-1
    int zpair;                       // zmode 0: chunk group size G (> 1: G consecutive chunks of a
                                     // tile launched together, alternating sweep directions; K3)
    int nyslots;                     // pack kernel: slots [0, nyslots) with g != 0 (Y terms)
    P2pSync sync;                    // boundary launch of the P2P halo path (else on = 0)
};
// (scheme, adaptive, stage) selects the compile-time StageSpec instance; adaptive: 0 fixed step,
// 1 error-controlled with Odeint's ratio (R-12), 2 with SPEC's ratio (R-28).
cudaError_t launch_gs_stage(int scheme, int adaptive, int stage, const GsStageArgs& a,
                            cudaStream_t st, int* nlaunch);
// 4D tensor maps over a padded array of `nplanes` planes, maps[4]: for 32x8 tiles the
// tile + ring box [0] and the interior box [1]; for 32x16 tiles [2] and [3]
// (stage_rows(spec) selects the pair).
cudaError_t encode_grid_maps(CUtensorMap* maps, const double* base, const GridGeom& g, int nplanes);

// Y_i on own planes 0 and nzl-1 (whole padded planes) -> dst[0] (plane 0), dst[1] (plane
// nzl-1): the NCCL send buffer, or the neighbours' ghost planes (P2P, with the handshake; dst
// then points at parity 0 and parity 1 lies 2 planes further).
cudaError_t launch_gs_pack(const GsStageArgs& a, double* dst0, double* dst1, const P2pSync& sync,
                           cudaStream_t st);
// Refresh the periodic ring of every (plane, component) slice of a padded array (after a
// user copy into the interior); nslices = planes * components.
cudaError_t launch_fill_ring(double* a, const GridGeom& g, int nslices, cudaStream_t st);

// Fused allreduce(max) of one uint64 word over the ranks' mapped P2P flag blocks (SURVEY f3:
// the NCCL allreduce replaced by NVLink atomics): every rank atomicMax-es its word into slot
// (round & 1) of every rank's block, raises every rank's arrival counter, waits for all world
// arrivals of this round, and reads the result back into *word.  flags[q]: rank q's block
// (flags[rank] = this rank's own); one thread; round counter on the device.
cudaError_t launch_p2p_allreduce_max(unsigned long long* word, unsigned long long* const* flags, int world,
                                     int rank, cudaStream_t st);
constexpr int P2P_MAX_WORLD = 16;

// ---------------------------------------------------------------------------------------
// K5: whole RK integrations of Gray–Scott on a small single-GPU grid in one persistent
// cooperative launch (rk_smallgrid.cu; grid-wide barrier between stages, u/u_new ping-pong).
struct CoopCoef {          // dt-scaled coefficients of a step / try
    double g[13][13];      // dt * a_ij
    double beta[13];       // dt * b_j
    double delta[13];      // dt * (b_j - bhat_j)
};
struct GsCoopArgs {
    double* buf[2];        // buf[0] = u on entry, buf[1] = u_new; after nsteps u is buf[nsteps & 1]
    double* k[13];         // k_j buffers (padded layout); k_last is not stored
    double* ybuf[2];       // stage values Y_i (padded layout), alternating between stages
    GridGeom geo;          // nzl = nz: one GPU, z wraps by index
    CoopCoef cf;           // fixed steps: the step's coefficients
    double d1, d2, F, FK, inv_h2;
    int nsteps;            // fixed steps
    unsigned int* bar;     // the grid barrier's two words (arrivals, generation), zeroed once per state
};
cudaError_t launch_gs_coop(int scheme, const GsCoopArgs& a, cudaStream_t st, int device);
int coop_last_stage(int scheme);           // last stage index (b_j != 0) = number of stored k_j
int coop_last_stage_adaptive(int scheme);  // last stage with b_j or e_j != 0 (CK54/DOPRI5/RKF78)
// The whole integrate_adaptive (RK_OPT_DEVICE_LOOP on a small grid): tries, error max and
// the controller on the device; results in *res (as the vector loop's PwLoopResult).
struct GsCoopLoopArgs {
    GsCoopArgs c;          // buffers, geometry, RHS parameters (c.cf, c.nsteps unused)
    double A[13][13], B[13], Ew[13];  // the scheme's a_ij, b_j, e_j as doubles (rat_double)
    double t0, t1, dt0, atol, rtol;
    double e_rej, e_acc, emin;        // the host controller's exponents / clamp
    int ctrl;                         // 0 Odeint (R-12), 1 SPEC (R-28)
    int max_tries;
    unsigned long long* red;          // [3] zeroed: per-try error-max slots (rotating)
    PwLoopResult* res;
};
cudaError_t launch_gs_coop_adaptive(int scheme, const GsCoopLoopArgs& a, cudaStream_t st, int device);

// ---------------------------------------------------------------------------------------
// K6: one whole fixed step of a chained-stage scheme (Y_s = u + g_s k_{s-1}: RK4, explicit
// midpoint) of Gray–Scott in ONE launch, temporal blocking across the stages (rk_fused.cu).
struct GsFusedArgs {
    CUtensorMap tm_u;      // u: box of a 32x16 tile + L-cell margin (encode_fused_map)
    const double* u;       // u (periodic margin patches on the domain edge)
    double* out;           // u_new (padded layout, ring copies written)
    GridGeom geo;          // nzl = nz: one GPU, z wraps by index
    double g[4];           // g[s] = dt*a_{s+1,s}: Y_{s+1} = u (+) g[s] (x) k_s (1-based stages)
    double beta[4];        // beta[j] = dt*b_{j+1}
    double d1, d2, F, FK, inv_h2;
    int zchunk;            // output planes per CTA
};
bool fused_scheme(int scheme);  // RK4 and explicit midpoint
int fused_halo(int scheme);     // L = stages = margin cells
cudaError_t encode_fused_map(CUtensorMap* map, const double* base, const GridGeom& g, int nplanes, int L);
cudaError_t launch_gs_fused(int scheme, const GsFusedArgs& a, cudaStream_t st);
// K8 (rk_pair.cu): two chained stages per launch (stage-pair temporal blocking, one GPU):
// k_A = F(src) on the tile + 1 ring; Y_B = u (+) gB k_A; k_B = F(Y_B); W = Wb (+) betaA k_A
// (+) betaB k_B with Wb = W_in or u; out = W (and out_y = u (+) gN k_B when a pair follows).
struct PairArgs {
    CUtensorMap tm_src;    // Y_A as stored (u, or the written-ahead Y): 38 x 20 box (encode_pair_map)
    CUtensorMap tm_u;      // u: K3's 34 x 18 tile + ring box (PAIR_LAST); PAIR_DP_TAIL: W
    CUtensorMap tm_e, tm_uo, tm_k1;  // PAIR_DP_TAIL: E, u, k_1 interior boxes (L2 prefetch)
    CUtensorMap tm_glo, tm_ghi;      // ghosts: the source's planes -2, -1 / nzl, nzl+1 (2-plane arrays)
    CUtensorMap tm_ulo, tm_uhi;      // ghosts: the base's planes -1 / nzl (1-plane arrays)
    const double* src_lo;            // ghosts: raw pointers of the source's ghost arrays (patches)
    const double* src_hi;
    CUtensorMap tm_glo2, tm_ghi2;    // PAIR_DP_HEAD ghosts of k_1 (2-plane arrays)
    const double* src2;              // PAIR_DP_HEAD: k_1 (patches), and its ghost arrays
    const double* src2_lo;
    const double* src2_hi;
    double gA, gB1;                  // PAIR_DP_HEAD: Y_2 = u + gA k_1, Y_3 = (u + gB1 k_1) + gB k_2
    int ghosts;                      // multi-GPU slab (or its one-GPU loopback): z does not wrap
    const double* src;     // raw pointer of the source (periodic cells beyond the padded ring)
    const double* w_in;    // PAIR_LAST: the partial sum W of the first pair; PAIR_DP_TAIL: E
    const double* u_in;    // PAIR_DP_TAIL: u and k_1 (the ratio's denominator, own cells)
    const double* k1_in;
    unsigned long long* errmax;  // PAIR_DP_TAIL: block max of the error ratio's bits
    double* out;           // W (PAIR_FIRST) or u_new (ring copies written)
    double* out_y;         // PAIR_FIRST: the next pair's stage value (ring copies written)
    GridGeom geo;          // nzl = nz: one GPU, z wraps by index
    double gB, gN, betaA, betaB;  // PAIR_DP_TAIL: gB = dt b_6, betaA / betaB = dt e_6 / dt e_7
    double dt, atol, rtol;
    const double* dtp;     // non-null (device-resident try loop): this try's dt; the coefficients are raw
    double d1, d2, F, FK, inv_h2;
    int zchunk;
};
// PAIR_LAST_NOA: PAIR_LAST without the beta_A term (b_A = 0: Cash–Karp's b_5)
enum { PAIR_FIRST = 0, PAIR_LAST = 1, PAIR_ONLY = 2, PAIR_DP_TAIL = 3, PAIR_DP_HEAD = 4, PAIR_LAST_NOA = 5 };
bool pair_shape_ok(const GridGeom& g);  // nx % 32 == 0, ny % 16 == 0
cudaError_t encode_pair_map(CUtensorMap* map, const double* base, const GridGeom& g, int nplanes);
cudaError_t launch_gs_pair(int kind, const PairArgs& a, cudaStream_t st);
// K7 (rk_fused2.cu): the same step with warp-specialised stage groups handing planes over
// through mbarriers instead of CTA-wide barriers (RK_OPT_FUSED_STEP = 2)
cudaError_t launch_gs_fused_ws(int scheme, const GsFusedArgs& a, cudaStream_t st);

// ---------------------------------------------------------------------------------------
// K2 / K4: algebra.
struct LincombArgs {
    double* out;
    const double* in[14];
    double coef[14];
    int k;
    int64_t count;
};
cudaError_t launch_lincomb(const LincombArgs& a, cudaStream_t st, int num_sms);
cudaError_t launch_norm_inf(const double* x, int64_t count, unsigned long long* out,
                            cudaStream_t st, int num_sms);
// K4 (unfused error control): max over elements of the error ratio (spec = 0: w = k1, Odeint's
// denominator; spec = 1: w = u_new, SPEC's) into *out as uint64 bits (atomicMax)
cudaError_t launch_ratio_max(const double* e, const double* u, const double* w, int64_t count, double dt,
                             double atol, double rtol, int spec, unsigned long long* out, cudaStream_t st,
                             int num_sms);
// atomicMax(word, bits of v) (v >= 0): fault injection into an error-ratio max
cudaError_t launch_inject_max(unsigned long long* word, double v, cudaStream_t st);
// *host_dst = *src by a 1-thread kernel (host_dst: cudaMallocHost memory, read after a stream wait)
cudaError_t launch_publish_word(const unsigned long long* src, unsigned long long* host_dst, cudaStream_t st);

}  // namespace rkb
