// rk_pair.cu — K8: two consecutive Runge–Kutta stages of Gray–Scott per launch (stage-pair
// temporal blocking, "fused" variants).
//
// For tableaux whose stage values chain through one slope (Y_s = u (+) g_s k_{s-1}: classic RK4
// P:L59, the explicit midpoint rule P:L58), a pair of stages (A, B = A+1) is one launch:
//   k_A = F(Y_A)                  Y_A read as stored (u, or the Y written ahead by the previous
//                                 pair), evaluated on the tile grown by one cell (the ring k_B's
//                                 stencil needs) and never stored
//   Y_B = u (+) g_B k_A           formed where k_A was computed
//   k_B = F(Y_B)                  on the tile
//   epilogue at the own cells:    W = Wb (+) beta_A k_A (+) beta_B k_B   (Wb = u, or the partial
//                                 sum W of the previous pair; this is u_new after the last pair)
//                                 and, when another pair follows, its stage value written ahead:
//                                 Y_next = u (+) g_next k_B  (with the periodic ring copies)
// RK4 is two launches -- (u -> Y_3, W) and (Y_3, u, W -> u_new), 48 + 64 = 112 B/cell/step
// instead of 208 stage by stage -- and the explicit midpoint rule one launch (u -> u_new, 32 B
// instead of 80), for 1.19x the stencil work of stage A (32x16 tile: 96 ring cells on 512).
//
// Kernel organisation (sm_100a, K3's recipe): a CTA of 256 threads owns a 32x16 xy tile (each
// thread two ADJACENT rows of one column, so one y neighbour of each own cell is the other own
// cell, in registers) and sweeps a chunk of z planes.  One elected thread streams, per plane, one
// 4D TMA box per input into an R-deep mbarrier ring: Y_A's source with a 2-cell margin (38x20
// box from the 16-byte aligned column x0-2; CTAs on the domain edge patch the periodic cells
// beyond the padded layout's 1-cell ring in place) and u with a 1-cell margin when it is not
// Y_A's source; W (own cells only) comes by plain loads issued before stage A.  Iteration t (stage A at plane t, stage B at plane t-1) has ONE
// __syncthreads: [patch plane t+1]; barrier; k_A at plane t (own cells: xy neighbours from the
// ring, z column in registers; ring cells: all from the ring) -> Y_B(t) into a 2-slot buffer
// (own cells also in registers); k_B at plane t-1 (xy from the Y_B buffer, z from registers) ->
// epilogue.  A thread's stage A and stage B chains are independent: 4-5 chains in flight.
// Arithmetic is K3's expression for expression (R-17): difference-form Laplacian
// (x, then y, then z; lower neighbour first), the same reaction trees, stage values and partial
// sums left to right, no FMA -- bitwise equal to the oracle and to the stage-by-stage kernels for
// any tile / chunk decomposition.  nx % 32 == 0, ny % 16 == 0 (else the library runs the
// stage-by-stage kernels).  One GPU: z wraps by index; on the multi-GPU slab (a.ghosts) the
// planes beyond the slab come from ghost arrays exchanged by the host before the launch.
#include <cudaTypedefs.h>

#include <type_traits>

#include "rk_device.cuh"
#include "rk_kernels.cuh"

namespace rkb {

namespace {

#define PINLINE __attribute__((always_inline))

constexpr int PX = 32;    // tile width (one warp per row pair)
constexpr int PTH = 16;   // tile height: 8 warps x 2 adjacent rows
constexpr int PNT = 256;  // threads
constexpr int BW = PX + 6;   // source box: cells x0-3 .. x0+34 (padded column x0-2: 16-byte start;
                             // a 36-wide box at x0-2 (8-byte start) faults: illegal instruction)
constexpr int BH = PTH + 4;  // rows y0-2 .. y0+17
constexpr int BOX = BW * BH;
constexpr int HSLOT = (2 * BOX * 8 + 127) / 128 * 128;  // 12160 B
constexpr int UW = PX + 2, UH = PTH + 2, UBOX = UW * UH;  // u box: tile + 1 ring (K3's 34x18 box)
constexpr int USLOT = (2 * UBOX * 8 + 127) / 128 * 128;   // 9856 B
constexpr int YBW = UW, YBH = UH, YBOX = UBOX;            // Y_B buffer: tile + 1 ring
constexpr int YBSLOT = USLOT;
constexpr int NRING = 2 * PX + 2 * PTH;                   // tile+1 ring without its corners: 96
#ifndef RKB_RING_WARPS
#define RKB_RING_WARPS 3
#endif
constexpr int RING_WARPS = RKB_RING_WARPS;                // 3 (32 lanes; measured) or 4 (24 lanes each)
static_assert(NRING % RING_WARPS == 0 && NRING / RING_WARPS <= 32, "ring split");
constexpr int NPATCH = 36 * BH;                           // source positions used (box cols 1..36)
constexpr int SMEM_BUDGET = 113 * 1024;                   // 2 CTAs per SM
#ifndef RKB_PAIR_RU
#define RKB_PAIR_RU 3  // u ring slots of the u-fed pairs
#endif
#ifndef RKB_PAIR_RMAX
#define RKB_PAIR_RMAX 5  // ring depth cap (6 measured slower: RK4 3.33 vs 3.16 ms)
#endif
constexpr int SMEM_BUDGET3 = 72 * 1024;                   // 3 CTAs per SM (u-fed pairs)

// U1: u comes in its own 1-ring box (Y_A's source is a written-ahead Y).  The ring holds the
// planes t-1, t, t+1 stage A reads and at least one plane in flight.
// The single-pair kind (u -> u_new: explicit midpoint) runs 3 CTAs per SM (<= 85 registers: Y_A
// own values from the ring, 24 warps; 1.14 -> 1.12 ms); the others 2 (their register queues
// at 80 registers spill: RK4 3.15 -> 3.28 ms).
// HD (the DOPRI5 head pair): u and k_1 both in 2-margin boxes, formed in place after they land
// into Y_A = u + (dt a_21) k_1 and the base Z = u + (dt a_31) k_1; one Y_B slot (+ a second
// barrier) so the two boxes fit two CTAs per SM.
template <bool U1, bool YOUT, bool HD = false>
struct PLayout {
    static constexpr int minb = (!U1 && !YOUT && !HD) ? 3 : 2;
    // U1: u has a ring of its own, RU slots (u(t) is read in one iteration only, so 3 slots
    // give it two planes of lead while the source ring deepens from 4 to 5 planes)
    static constexpr int RU = U1 ? RKB_PAIR_RU : 0;
    static constexpr int stage = HSLOT + (HD ? HSLOT : 0);
    static constexpr int fixed = (HD ? 1 : 2) * YBSLOT + RU * (USLOT + 8);
    static constexpr int Rb = ((minb == 3 ? SMEM_BUDGET3 : SMEM_BUDGET) - fixed - 64) / stage;
    static constexpr int R = Rb > RKB_PAIR_RMAX ? RKB_PAIR_RMAX : Rb;
    static_assert(R >= 4, "ring too shallow");
    static constexpr int off_u = HSLOT;            // HD: k_1's box in the same ring stage
    static constexpr int ur = R * stage;           // U1: the u ring (RU slots)
    static constexpr int yb = ur + RU * USLOT;     // Y_B buffer (2 slots; HD: 1)
    static constexpr int bar = yb + (HD ? 1 : 2) * YBSLOT;  // R mbarriers, then RU (U1)
    static constexpr int smem = bar + (R + RU) * 8;
};

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int pmod(int a, int n) {
    const int m = a % n;
    return m < 0 ? m + n : m;
}

// reaction and scaling of one cell (K3's trees) from the Laplacian sums s[c]
__device__ __forceinline__ void react(const double (&s)[2], const double (&ctr)[2], const PairArgs& a, double (&f)[2]) {
    const double L0 = mul(s[0], a.inv_h2), L1 = mul(s[1], a.inv_h2);
    const double C0 = ctr[0], C1 = ctr[1];
    const double rc = mul(mul(C0, C1), C1);
    f[0] = sub(add(sub(mul(a.d1, L0), rc), a.F), mul(a.F, C0));
    f[1] = sub(add(mul(a.d2, L1), rc), mul(a.FK, C1));
}

// k = F(Y) at the thread's two own cells (rows r0 = 2w, r1 = 2w+1 of one column): v0 -> cell r0's
// component 0 in a box of pitch `pitch` and component stride `cs`; c0 / c1 their values, zm / zp
// their z neighbours.  Cell r0's upper y neighbour is c1 and cell r1's lower one is c0.
__device__ __forceinline__ void rhs_two(const double* v0, int cs, int pitch, const double (&c0)[2],
                                        const double (&c1)[2], const double (&zm0)[2], const double (&zp0)[2],
                                        const double (&zm1)[2], const double (&zp1)[2], const PairArgs& a,
                                        double (&f0)[2], double (&f1)[2]) {
    double s0[2], s1[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const double* w = v0 + c * cs;
        const double a0 = c0[c], a1 = c1[c];
        double s = add(sub(w[-1], a0), sub(w[1], a0));
        s = add(s, add(sub(w[-pitch], a0), sub(a1, a0)));
        s0[c] = add(s, add(sub(zm0[c], a0), sub(zp0[c], a0)));
        const double* w1 = w + pitch;
        double t = add(sub(w1[-1], a1), sub(w1[1], a1));
        t = add(t, add(sub(a0, a1), sub(w1[pitch], a1)));
        s1[c] = add(t, add(sub(zm1[c], a1), sub(zp1[c], a1)));
    }
    react(s0, c0, a, f0);
    react(s1, c1, a, f1);
}

// The same in two parts, so a thread can start k_B's xy sums before k_A (which yields k_B's
// upper z neighbour) is done: sxy = the x and y terms, then the z pair and the reaction -- the
// identical expression tree.
__device__ __forceinline__ void lap_xy_two(const double* v0, int cs, int pitch, const double (&c0)[2],
                                           const double (&c1)[2], double (&sx0)[2], double (&sx1)[2]) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const double* w = v0 + c * cs;
        const double a0 = c0[c], a1 = c1[c];
        const double s = add(sub(w[-1], a0), sub(w[1], a0));
        sx0[c] = add(s, add(sub(w[-pitch], a0), sub(a1, a0)));
        const double* w1 = w + pitch;
        const double t = add(sub(w1[-1], a1), sub(w1[1], a1));
        sx1[c] = add(t, add(sub(a0, a1), sub(w1[pitch], a1)));
    }
}
__device__ __forceinline__ void finish_one(const double (&sx)[2], const double (&ctr)[2], const double (&zm)[2],
                                           const double (&zp)[2], const PairArgs& a, double (&f)[2]) {
    double s[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) s[c] = add(sx[c], add(sub(zm[c], ctr[c]), sub(zp[c], ctr[c])));
    react(s, ctr, a, f);
}

// k = F(Y) at one cell with every value from boxes (ring cells)
__device__ __forceinline__ void rhs_box(const double* v, const double* vm, const double* vp, int cs, int pitch,
                                        const PairArgs& a, double (&f)[2]) {
    double s[2], ctr[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const double* w = v + c * cs;
        const double cc = w[0];
        ctr[c] = cc;
        double q = add(sub(w[-1], cc), sub(w[1], cc));
        q = add(q, add(sub(w[-pitch], cc), sub(w[pitch], cc)));
        s[c] = add(q, add(sub(vm[c * cs], cc), sub(vp[c * cs], cc)));
    }
    react(s, ctr, a, f);
}
// ... the same with the lower z neighbour from registers (the ring cell's carried values)
__device__ __forceinline__ void rhs_box_r(const double* v, const double (&vm)[2], const double* vp, int cs, int pitch,
                                          const PairArgs& a, double (&f)[2]) {
    double s[2], ctr[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const double* w = v + c * cs;
        const double cc = w[0];
        ctr[c] = cc;
        double q = add(sub(w[-1], cc), sub(w[1], cc));
        q = add(q, add(sub(w[-pitch], cc), sub(w[pitch], cc)));
        s[c] = add(q, add(sub(vm[c], cc), sub(vp[c * cs], cc)));
    }
    react(s, ctr, a, f);
}

__device__ __forceinline__ void store_ring(double* p, const GridGeom& G, bool ex0, bool ex1, bool ey0, bool ey1,
                                           double v) {
    p[0] = v;
    if (ex0) p[G.nx] = v;
    if (ex1) p[-G.nx] = v;
    if (ey0) p[(int64_t)G.ny * G.P] = v;
    if (ey1) p[-(int64_t)G.ny * G.P] = v;
}

// DP: the Dormand–Prince error-controlled tail pair (stages 6 and 7 of a try): the source is
// Y_6 (written ahead), Y_B = W (+) (dt b_6) k_6 = u_new (a_7j = b_j, FSAL), k_B = k_7 = F(u_new);
// the epilogue stores u_new and k_7, forms e = (E (+) (dt e_6) k_6) (+) (dt e_7) k_7 and the
// Odeint ratio |e| / (atol (+) rtol (x) (|u| (+) dt (x) |k_1|)) with a block max.
// KK: store k_A and k_B with their rings (HD: k_2, k_3 of a DOPRI5 try).
template <bool U1, bool WIN, bool BA, bool YOUT, bool DP = false, bool DTP = false, bool KK = false, bool HD = false>
__global__ void __launch_bounds__(PNT, PLayout<U1, YOUT, HD>::minb) gs_pair_kernel(const __grid_constant__ PairArgs a) {
    using LY = PLayout<U1, YOUT, HD>;
    constexpr bool BASE = U1 || HD;  // Y_B's base comes from its own box (else it is Y_A's source)
    constexpr int R = LY::R;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + LY::bar);
    const GridGeom& G = a.geo;
    const int tid = threadIdx.x;
    const int ntx = G.nx / PX;
    const int tile = (int)blockIdx.x;
    const int x0 = (tile % ntx) * PX, y0 = (tile / ntx) * PTH;
    const int zb = (int)blockIdx.y * a.zchunk;
    const int ze = min(zb + a.zchunk, G.nzl);
    if (zb >= ze) return;
    const int nout = ze - zb;
    const int nr = nout + 4;  // raw planes zb-2 .. ze+1; index i <-> plane zb-2+i
    // Coefficients: dt-scaled by the host, or (device-resident try loop, a.dtp) raw and scaled
    // here by this try's dt -- fl(dt * c) either way, the same single rounding (K3's rule)
    // (a template flag: the host-scaled path keeps them as constant-bank operands, no registers)
    const double dsc = DTP ? *a.dtp : 1.0;
    const double cgB = DTP ? mul(dsc, a.gB) : a.gB, cgN = DTP ? mul(dsc, a.gN) : a.gN;
    const double cbA = DTP ? mul(dsc, a.betaA) : a.betaA, cbB = DTP ? mul(dsc, a.betaB) : a.betaB;
    const double cdt = DTP ? dsc : a.dt;
    const double cgA = DTP ? mul(dsc, a.gA) : a.gA, cgB1 = DTP ? mul(dsc, a.gB1) : a.gB1;  // HD
    auto plane = [&](int i) PINLINE -> int { return pmod(zb - 2 + i, G.nzl); };
    const bool edge = x0 == 0 || x0 + PX == G.nx || y0 == 0 || y0 + PTH == G.ny;  // CTA-uniform

    // own cells: column lx, rows r0 = 2w, r1 = 2w+1
    const int lx = tid % PX, w = tid / PX;
    const int pb = (2 * w + 2) * BW + (lx + 3);   // row r0 in the source box
    const int pu = (2 * w + 1) * UW + (lx + 1);   // row r0 in the u box / Y_B buffer
    const int64_t coff = (int64_t)(y0 + 2 * w + 1) * G.P + (x0 + lx + 1);  // row r0, padded
    const bool ex0 = x0 + lx == 0, ex1 = x0 + lx == G.nx - 1;
    const bool ey0 = y0 + 2 * w == 0, ey1 = y0 + 2 * w + 1 == G.ny - 1;
    const bool ering = ex0 || ex1 || ey0 || ey1;
    // ring cell of the tile grown by one (no corners): top row, bottom row, left col, right col
    // (RING_WARPS warps share the 96 ring cells, one warp per SM sub-partition when 4)
    constexpr int RPW = NRING / RING_WARPS;  // ring cells per ring warp
    const int rj = (tid / 32) * RPW + (tid % 32);
    const bool hr = tid / 32 < RING_WARPS && tid % 32 < RPW;
    int rb = 0, ru = 0;
    if (hr) {
        int rx, ry;
        if (rj < PX) { rx = rj; ry = -1; }
        else if (rj < 2 * PX) { rx = rj - PX; ry = PTH; }
        else if (rj < 2 * PX + PTH) { rx = -1; ry = rj - 2 * PX; }
        else { rx = PX; ry = rj - 2 * PX - PTH; }
        rb = (ry + 2) * BW + (rx + 3);
        ru = (ry + 1) * UW + (rx + 1);
    }

    auto raw = [&](int i) PINLINE -> unsigned char* { return smem + (size_t)(i % R) * LY::stage; };
    auto ybs = [&](int i) PINLINE -> double* {
        return reinterpret_cast<double*>(smem + LY::yb + (HD ? (size_t)0 : (size_t)(i & 1) * YBSLOT));
    };
    // base box geometry: U1 the 34x18 u box, HD the 38x20 box of the formed Z
    const int pbase = HD ? pb : pu, rbase = HD ? rb : ru;
    constexpr int BPITCH = HD ? BW : UW, BCS = HD ? BOX : UBOX;
    auto tma = [&](void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1, int q) PINLINE {
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(s32(dst)),
            "l"(reinterpret_cast<uint64_t>(m)), "r"(s32(b)), "r"(c0), "r"(c1), "r"(0), "r"(q)
            : "memory");
    };
    // multi-GPU slab (a.ghosts): planes beyond the slab come from the ghost arrays the host
    // filled before the launch (source: 2 planes each side, base: 1), not by wrapping
    auto issue = [&](int i) PINLINE {  // thread 0
        uint64_t* b = &bar[i % R];
        const int p = zb - 2 + i;
        const int q = plane(i);
        const uint32_t bytes = 2 * BOX * 8 + (HD ? 2 * BOX * 8 : 0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
        unsigned char* st = raw(i);
        if (a.ghosts && p < 0) tma(st, &a.tm_glo, b, x0 - 2, y0 - 1, p + 2);
        else if (a.ghosts && p >= G.nzl) tma(st, &a.tm_ghi, b, x0 - 2, y0 - 1, p - G.nzl);
        else tma(st, &a.tm_src, b, x0 - 2, y0 - 1, q);
        if constexpr (HD) {  // k_1: the same 2-margin box, every plane
            if (a.ghosts && p < 0) tma(st + LY::off_u, &a.tm_glo2, b, x0 - 2, y0 - 1, p + 2);
            else if (a.ghosts && p >= G.nzl) tma(st + LY::off_u, &a.tm_ghi2, b, x0 - 2, y0 - 1, p - G.nzl);
            else tma(st + LY::off_u, &a.tm_u, b, x0 - 2, y0 - 1, q);
        }
    };
    // U1: u(i) (raw index i, the stage-A planes zb-1 .. ze: 1 <= i <= nr-2) into its own ring
    constexpr int RU = LY::RU > 0 ? LY::RU : 1;
    auto ubox = [&](int i) PINLINE -> unsigned char* {
        return U1 ? smem + LY::ur + (size_t)((i - 1) % RU) * USLOT : raw(i) + LY::off_u;  // u(1) -> slot 0
    };
    auto issue_u = [&](int i) PINLINE {  // thread 0
        if constexpr (U1) {
            uint64_t* b = &bar[R + (i - 1) % RU];
            const int p = zb - 2 + i;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(2 * UBOX * 8)
                         : "memory");
            unsigned char* st = ubox(i);
            if (a.ghosts && p < 0) tma(st, &a.tm_ulo, b, x0, y0, 0);
            else if (a.ghosts && p >= G.nzl) tma(st, &a.tm_uhi, b, x0, y0, 0);
            else tma(st, &a.tm_u, b, x0, y0, plane(i));
        }
    };
    auto wait_u = [&](int i) PINLINE {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WAITU_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WAITU_%=;\n}" ::"r"(s32(&bar[R + (i - 1) % RU])),
            "r"((uint32_t)(((i - 1) / RU) & 1))
            : "memory");
    };
    auto wait = [&](int i) PINLINE {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WAITP_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WAITP_%=;\n}" ::"r"(s32(&bar[i % R])),
            "r"((uint32_t)((i / R) & 1))
            : "memory");
    };
    // Edge CTAs: the source box cells the padded layout does not hold (the 2nd margin cell, the
    // ring corners) are overwritten with their periodic images.  The list of such cells is built
    // once (one per thread, at most 2*20 + 2*36 + corners < 256), and every thread holding one
    // loads its values a plane ahead into registers, so the patch after a plane lands costs two
    // shared stores, not a global-memory round trip.
    __shared__ int s_np;
    __shared__ int s_pos[PNT], s_src[PNT];
    int my_pos = -1, my_src = 0;
    if (edge) {
        if (tid == 0) s_np = 0;
        __syncthreads();
        for (int q = tid; q < NPATCH; q += PNT) {
            const int col = 1 + q % 36, row = q / 36;
            const int x = x0 - 3 + col, yy = y0 - 2 + row;
            const bool held = (x >= 0 && x < G.nx && yy >= -1 && yy <= G.ny) || (yy >= 0 && yy < G.ny && x >= -1 && x <= G.nx);
            if (held) continue;
            const int k = atomicAdd(&s_np, 1);
            s_pos[k] = row * BW + col;
            s_src[k] = (pmod(yy, G.ny) + 1) * G.P + (pmod(x, G.nx) + 1);
        }
        __syncthreads();
        if (tid < s_np) {
            my_pos = s_pos[tid];
            my_src = s_src[tid];
        }
    }
    double pv0 = 0.0, pv1 = 0.0, pv2 = 0.0, pv3 = 0.0;  // this thread's patch values of the next plane
    auto patch_load = [&](int i) PINLINE {
        if (my_pos >= 0 && i < nr) {
            const int pz = zb - 2 + i;
            const int64_t o = a.ghosts && pz < 0 ? (int64_t)(pz + 2) * G.ps + my_src
                            : a.ghosts && pz >= G.nzl ? (int64_t)(pz - G.nzl) * G.ps + my_src
                                                      : (int64_t)plane(i) * G.ps + my_src;
            const double* p = (a.ghosts && pz < 0 ? a.src_lo : a.ghosts && pz >= G.nzl ? a.src_hi : a.src) + o;
            pv0 = p[0];
            pv1 = p[G.cs];
            if constexpr (HD) {
                const double* p2 = (a.ghosts && pz < 0 ? a.src2_lo : a.ghosts && pz >= G.nzl ? a.src2_hi : a.src2) + o;
                pv2 = p2[0];
                pv3 = p2[G.cs];
            }
        }
    };
    // HD: after the patches, Y_A = u + (dt a_21) k_1 in place of u and Z = u + (dt a_31) k_1 in
    // place of k_1, at every box position stage A or Y_B reads
    auto form = [&](int i) PINLINE {
        if constexpr (HD) {
            if (edge) __syncthreads();  // patched cells (written by other threads) visible
            // 16-byte pairs over the whole box (columns 0 and 37 are formed too and never read)
            double2* y = reinterpret_cast<double2*>(raw(i));
            double2* k = reinterpret_cast<double2*>(raw(i) + LY::off_u);
            static_assert(BW % 2 == 0 && (BOX * 8) % 16 == 0 && LY::off_u % 16 == 0, "16-byte pairs");
            for (int q = tid; q < BOX / 2; q += PNT) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const double2 uu = y[c * (BOX / 2) + q], kk = k[c * (BOX / 2) + q];
                    y[c * (BOX / 2) + q] = make_double2(add(uu.x, mul(cgA, kk.x)), add(uu.y, mul(cgA, kk.y)));
                    k[c * (BOX / 2) + q] = make_double2(add(uu.x, mul(cgB1, kk.x)), add(uu.y, mul(cgB1, kk.y)));
                }
            }
        }
    };
    auto patch = [&](int i) PINLINE {  // after wait(i); then load the values of plane i+1
        if (my_pos >= 0) {
            double* y = reinterpret_cast<double*>(raw(i));
            y[my_pos] = pv0;
            y[BOX + my_pos] = pv1;
            if constexpr (HD) {
                double* k = reinterpret_cast<double*>(raw(i) + LY::off_u);
                k[my_pos] = pv2;
                k[BOX + my_pos] = pv3;
            }
        }
        patch_load(i + 1);
        form(i);
    };

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < R + LY::RU; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(&bar[s])), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int i = 0; i < (nr < R ? nr : R); ++i) issue(i);
    if (U1 && tid == 0)
        for (int i = 1; i <= RU && i <= nr - 2; ++i) issue_u(i);

    // own-cell registers ([q][r][c]: slot q = plane mod 3 within the unrolled loop, row r0 / r1,
    // component): Y_A at planes t-1, t, t+1; Y_B at t-2, t-1, t; k_A at t-1 (for the epilogue)
    // and t; u at t-1 and t (U1).  The loop is unrolled by three so these queues rotate by
    // renaming, not by register moves.
    // own-cell Y_A: a register queue where registers allow (the u-fed pairs); the pair that also
    // streams u and W (at the 128-register cap) reads it from the ring instead
    constexpr bool YREG = LY::minb == 2 && !U1;
    double ya_q[YREG ? 3 : 1][2][2];
    // EARLY (= YREG): the ring cells carry their Y_A(t-1) in registers too, so no thread reads
    // raw plane t-1 in iteration t: its slot is refilled one iteration earlier -- two planes of
    // TMA lead instead of one (the head pair waited on its ring ~19 % of the time with one:
    // 2.15 -> 1.98 ms, the DOPRI5 try 9.63 -> 9.46 ms).  The u-fed pairs cannot also carry their own cells' Y_A(t-1): 56-120 B
    // of spills at the 128-register cap.
#ifndef RKB_PAIR_EARLY
#define RKB_PAIR_EARLY 1  // developer A/B (tools/ab_early.sh): 0 off, 1 the head pair only, 2 every
                          // YREG pair (RK4's first pair: 3.27 -> 3.34 ms, so only the head pair)
#endif
    constexpr bool EARLY = YREG && (RKB_PAIR_EARLY == 2 || (RKB_PAIR_EARLY == 1 && HD));
    double rc_q[EARLY ? 3 : 1][2] = {};
    double yb_q[3][2][2] = {}, ka_q[3][2][2] = {}, u_q[3][2][2] = {};
    double w_q[3][2][2] = {};  // WIN: W at t-1 (stage B's epilogue) and t (loaded one plane ahead)
    auto own_src = [&](int i, double (&v)[2][2]) PINLINE {
        const double* s = reinterpret_cast<const double*>(raw(i));
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            v[r][0] = s[pb + r * BW];
            v[r][1] = s[BOX + pb + r * BW];
        }
    };
    patch_load(0);
    wait(0);
    patch(0);
    wait(1);
    patch(1);
    __syncthreads();  // patched cells visible
    if constexpr (YREG) {
        own_src(0, ya_q[2]);  // plane zb-2 = "t-1" of iteration 0
        own_src(1, ya_q[0]);  // plane zb-1 = "t"
    }

    double rmax = 0.0;                // DP: running max of the ratio (exact) and its bits
    unsigned long long rbits = 0ull;

    // iteration it (J = it mod 3): stage A at plane t = zb-1+it (raw index it+1), stage B at t-1
    auto step = [&](int it, auto Jc) PINLINE {
        constexpr int J = decltype(Jc)::value;
        constexpr int Q0 = J, QP = (J + 1) % 3, QM = (J + 2) % 3;  // planes t, t+1 / t-2, t-1
        const int ic = it + 1;
        wait(it + 2);
        patch(it + 2);
        __syncthreads();  // plane t+1 (patched) visible; Y_B(t-1) stored; raw plane t-2 free
        if (tid == 0 && (EARLY ? it + R < nr : it - 1 >= 0 && it - 1 + R < nr)) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the patches
            issue(EARLY ? it + R : it - 1 + R);  // raw plane t-1 (EARLY) / t-2 is free
        }
        if (U1 && tid == 0 && it >= 1 && it + RU <= nr - 2) issue_u(it + RU);  // u(t-1)'s slot is free
        // own-cell Y_A at t-1, t, t+1 straight from the ring (registers are the scarcer resource)
        double yam[2][2], yac[2][2], yap[2][2];
        if constexpr (YREG) {
            own_src(ic + 1, ya_q[QP]);  // Y_A(t+1) (slot of Y_A(t-2))
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {  // renaming only: no moves survive unrolling
                    yam[r][c] = ya_q[QM][r][c];
                    yac[r][c] = ya_q[Q0][r][c];
                    yap[r][c] = ya_q[QP][r][c];
                }
        } else {
            own_src(ic - 1, yam);
            own_src(ic, yac);
            own_src(ic + 1, yap);
        }
        const bool doB = it >= 2;  // stage B at plane t-1: output planes zb .. ze-1
        if constexpr (WIN && !DP) {  // W of plane t (stage B's epilogue in the next iteration): plain loads
            if (it >= 1 && it <= nout) {
                const double* W = a.w_in + (int64_t)(zb + it - 1) * G.ps + coff;
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    w_q[Q0][r][0] = W[(int64_t)r * G.P];
                    w_q[Q0][r][1] = W[G.cs + (int64_t)r * G.P];
                }
            }
        }
        const double (&wbp)[2][2] = w_q[QM];
        double eo[2][2] = {}, uo[2][2] = {}, k1o[2][2] = {};  // DP: E, u, k_1 at plane t-1
        if constexpr (DP) {
            if (doB) {  // plain loads (in L2: prefetched two planes ahead), consumed after stage A
                const int64_t o = (int64_t)(zb + it - 2) * G.ps + coff;
#pragma unroll
                for (int r = 0; r < 2; ++r)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int64_t q = o + c * G.cs + (int64_t)r * G.P;
                        eo[r][c] = a.w_in[q];
                        uo[r][c] = a.u_in[q];
                        k1o[r][c] = a.k1_in[q];
                    }
            }
            if (tid == 0 && it + 2 >= 2 && it + 2 < nout + 2) {  // own inputs two planes ahead into L2
                const int q = zb + it;
#pragma unroll
                for (int m = 0; m < 3; ++m)
                    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                                     reinterpret_cast<uint64_t>(m == 0 ? &a.tm_e : m == 1 ? &a.tm_uo : &a.tm_k1)),
                                 "r"(x0), "r"(y0 + 1), "r"(0), "r"(q)
                                 : "memory");
            }
        }
        const unsigned char* st = raw(ic);
        const double* ya = reinterpret_cast<const double*>(st);
        const bool ring_plane = it >= 1 && it <= nout;  // Y_B(t) is read by stage B's xy stencil
        // Y_B: (t-2) in slot QP, (t-1) in slot QM = stage B's centres, Y_B(t) -> slot Q0
        double (&ybm)[2][2] = yb_q[QP];
        double (&ybc)[2][2] = yb_q[QM];
        double (&ybp)[2][2] = yb_q[Q0];
        // ---- stage B at plane t-1, xy part (its smem reads precede this iteration's stores) ----
        double sb0[2] = {0.0, 0.0}, sb1[2] = {0.0, 0.0};
        if (doB) lap_xy_two(ybs(ic - 1) + pu, YBOX, YBW, ybc[0], ybc[1], sb0, sb1);
        // ---- stage A at plane t ----
        double (&kac)[2][2] = ka_q[Q0];
        const double (&kap)[2][2] = ka_q[QM];
        rhs_two(ya + pb, BOX, BW, yac[0], yac[1], yam[0], yap[0], yam[1], yap[1], a, kac[0], kac[1]);
        double (&uc)[2][2] = u_q[Q0];
        const double (&up)[2][2] = u_q[QM];
        if constexpr (BASE) {
            if constexpr (U1) wait_u(ic);
            const double* U = reinterpret_cast<const double*>(ubox(ic));
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                uc[r][0] = U[pbase + r * BPITCH];
                uc[r][1] = U[BCS + pbase + r * BPITCH];
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) ybp[r][c] = add(BASE ? uc[r][c] : yac[r][c], mul(cgB, kac[r][c]));
        double yr[2] = {0.0, 0.0};  // Y_B at this thread's ring cell
        if constexpr (EARLY) {
            if (hr) {
                rc_q[Q0][0] = ya[rb];
                rc_q[Q0][1] = ya[BOX + rb];
            }
        }
        if (ring_plane && hr) {
            const double* yp = reinterpret_cast<const double*>(raw(ic + 1));
            double kr[2];
            if constexpr (EARLY) {
                rhs_box_r(ya + rb, rc_q[QM], yp + rb, BOX, BW, a, kr);
            } else {
                const double* ym = reinterpret_cast<const double*>(raw(ic - 1));
                rhs_box(ya + rb, ym + rb, yp + rb, BOX, BW, a, kr);
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const double ur = BASE ? reinterpret_cast<const double*>(ubox(ic))[c * BCS + rbase] : ya[c * BOX + rb];
                yr[c] = add(ur, mul(cgB, kr[c]));
            }
        }
        if constexpr (HD) __syncthreads();  // one Y_B slot: every stage-B read of Y_B(t-1) is done
        if (ring_plane) {
            double* yb = ybs(ic);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                yb[pu + r * UW] = ybp[r][0];
                yb[YBOX + pu + r * UW] = ybp[r][1];
            }
            if (hr) {
                yb[ru] = yr[0];
                yb[YBOX + ru] = yr[1];
            }
        }
        // ---- stage B at plane t-1 (output planes zb .. ze-1) ----
        if (doB) {
            double kb[2][2];
            finish_one(sb0, ybc[0], ybm[0], ybp[0], a, kb[0]);
            finish_one(sb1, ybc[1], ybm[1], ybp[1], a, kb[1]);
            const int64_t qo = (int64_t)(zb + it - 2) * G.ps;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const bool rx0 = ex0, rx1 = ex1, ry0 = r == 0 && ey0, ry1 = r == 1 && ey1;
                const int64_t ro = qo + coff + (int64_t)r * G.P;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if constexpr (KK) {  // k_A (plane t-1) and k_B, both with their rings
                        double* pa = a.out_y + ro + c * G.cs;
                        double* pk = a.out + ro + c * G.cs;
                        if (ering) {
                            store_ring(pa, G, rx0, rx1, ry0, ry1, kap[r][c]);
                            store_ring(pk, G, rx0, rx1, ry0, ry1, kb[r][c]);
                        } else {
                            pa[0] = kap[r][c];
                            pk[0] = kb[r][c];
                        }
                        continue;
                    }
                    if constexpr (DP) {
                        const double un = ybc[r][c];  // Y_7 = u_new
                        double* pu_ = a.out + ro + c * G.cs;
                        double* pk = a.out_y + ro + c * G.cs;
                        if (ering) {
                            store_ring(pu_, G, rx0, rx1, ry0, ry1, un);
                            store_ring(pk, G, rx0, rx1, ry0, ry1, kb[r][c]);
                        } else {
                            pu_[0] = un;
                            pk[0] = kb[r][c];
                        }
                        // e' = E (+) (dt e_6) k_6 (stage 6's epilogue), e = e' (+) (dt e_7) k_7
                        const double e = add(add(eo[r][c], mul(cbA, kap[r][c])), mul(cbB, kb[r][c]));
                        const double dd = add(a.atol, mul(a.rtol, add(fabs(uo[r][c]), mul(cdt, fabs(k1o[r][c])))));
                        // r = |e| / dd exactly; the division is skipped when e == 0 or when
                        // |e| <= rmax*dd*(1-2^-52) proves r <= rmax (K3's filter; NaN never skips)
                        const double ae = fabs(e);
                        const double th = mul(mul(rmax, dd), 0.99999999999999978);
                        if (!(ae == 0.0 || (ae <= th && th >= 2.2250738585072014e-308))) {
                            const double rr = ae / dd;
                            const unsigned long long rbv = ratio_bits(rr);
                            if (rbv > rbits) {
                                rbits = rbv;
                                rmax = rr;
                            }
                        }
                        continue;
                    }
                    // Wb: W of the previous pair, else u (= Y_A for a pair fed by u)
                    double wv = WIN ? wbp[r][c] : (U1 ? up[r][c] : yam[r][c]);
                    if constexpr (BA) wv = add(wv, mul(cbA, kap[r][c]));
                    wv = add(wv, mul(cbB, kb[r][c]));
                    double* p = a.out + ro + c * G.cs;
                    if constexpr (YOUT) {
                        p[0] = wv;  // W: read at own cells only, no ring copies
                        const double yn = add(U1 ? up[r][c] : yam[r][c], mul(cgN, kb[r][c]));
                        double* py = a.out_y + ro + c * G.cs;
                        if (ering) store_ring(py, G, rx0, rx1, ry0, ry1, yn);
                        else py[0] = yn;
                    } else {
                        if (ering) store_ring(p, G, rx0, rx1, ry0, ry1, wv);
                        else p[0] = wv;
                    }
                }
            }
        }
    };
    const int niter = nout + 2;
    int it = 0;
#ifndef RKB_PAIR_UNR1
#define RKB_PAIR_UNR1 2  // the plane loop not unrolled (queues rotate by moves): 2 = the DOPRI5 tail
                         // pair only (default: its 6.2 k-instruction unrolled body, the largest, stalled
                         // on instruction fetch; one copy is 2.1 k: 2.80 -> 2.77 ms), 1 = every pair
                         // kind (measured: RK4 -0.3 %, head pair +0.5 %, midpoint / CK54 tail +0.3 %), 0 = none
#endif
    constexpr bool UNR1 = RKB_PAIR_UNR1 == 1 || (RKB_PAIR_UNR1 == 2 && DP);
    if constexpr (UNR1) {
        // one copy of the body (a third of the instruction footprint); slot J = 0 every iteration,
        // and the queues move one plane: Y_A (t-1 <- t <- t+1), ring Y_A (t-1 <- t), Y_B (t-2 <- t-1
        // <- t), k_A, u, W (t-1 <- t)
#pragma unroll 1
        for (; it < niter; ++it) {
            step(it, std::integral_constant<int, 0>{});
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if constexpr (YREG) {
                        ya_q[2][r][c] = ya_q[0][r][c];
                        ya_q[0][r][c] = ya_q[1][r][c];
                    }
                    yb_q[1][r][c] = yb_q[2][r][c];
                    yb_q[2][r][c] = yb_q[0][r][c];
                    ka_q[2][r][c] = ka_q[0][r][c];
                    u_q[2][r][c] = u_q[0][r][c];
                    w_q[2][r][c] = w_q[0][r][c];
                }
            if constexpr (EARLY) {
                rc_q[2][0] = rc_q[0][0];
                rc_q[2][1] = rc_q[0][1];
            }
        }
    } else {
        for (; it + 2 < niter; it += 3) {
            step(it, std::integral_constant<int, 0>{});
            step(it + 1, std::integral_constant<int, 1>{});
            step(it + 2, std::integral_constant<int, 2>{});
        }
        if (it < niter) step(it, std::integral_constant<int, 0>{});
        if (it + 1 < niter) step(it + 1, std::integral_constant<int, 1>{});
    }
    if constexpr (DP) block_max_to_global(rbits, a.errmax);
}

template <bool U1, bool WIN, bool BA, bool YOUT, bool DP = false, bool DTP = false, bool KK = false, bool HD = false>
cudaError_t launch_pair_t(const PairArgs& a, cudaStream_t st) {
    using LY = PLayout<U1, YOUT, HD>;
    static std::atomic<unsigned long long> configured{0};
    if (cudaError_t e = smem_attr_once(configured, gs_pair_kernel<U1, WIN, BA, YOUT, DP, DTP, KK, HD>, LY::smem);
        e != cudaSuccess)
        return e;
    const int tiles = (a.geo.nx / PX) * (a.geo.ny / PTH);
    const int nch = (a.geo.nzl + a.zchunk - 1) / a.zchunk;
    gs_pair_kernel<U1, WIN, BA, YOUT, DP, DTP, KK, HD><<<dim3((unsigned)tiles, (unsigned)nch), PNT, LY::smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

bool pair_shape_ok(const GridGeom& g) { return g.nx % PX == 0 && g.ny % PTH == 0 && g.nx >= PX && g.ny >= PTH; }

cudaError_t encode_pair_map(CUtensorMap* map, const double* base, const GridGeom& g, int nplanes) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[4] = {(cuuint64_t)g.P, (cuuint64_t)(g.ny + 2), 2, (cuuint64_t)nplanes};
    const cuuint64_t strides[3] = {(cuuint64_t)g.P * 8, (cuuint64_t)g.cs * 8, (cuuint64_t)g.ps * 8};
    const cuuint32_t box[4] = {(cuuint32_t)BW, (cuuint32_t)BH, 2, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_gs_pair(int kind, const PairArgs& a, cudaStream_t st) {
    if (a.zchunk <= 0 || !pair_shape_ok(a.geo)) return cudaErrorInvalidValue;
    switch (kind) {
    case PAIR_FIRST: return launch_pair_t<false, false, true, true>(a, st);  // RK4 1-2: u -> Y3, W
    case PAIR_LAST: return launch_pair_t<true, true, true, false>(a, st);    // RK4 3-4: Y3, u, W -> u_new
    case PAIR_ONLY: return launch_pair_t<false, false, false, false>(a, st); // midpoint: u -> u_new
    case PAIR_LAST_NOA: return launch_pair_t<true, true, false, false>(a, st);  // b_A = 0 (CK54's tail)
    case PAIR_DP_HEAD:  // DOPRI5 stages 2-3: u, k1 -> k2, k3
        return a.dtp ? launch_pair_t<false, false, false, false, false, true, true, true>(a, st)
                     : launch_pair_t<false, false, false, false, false, false, true, true>(a, st);
    case PAIR_DP_TAIL:  // DOPRI5 stages 6-7 (dt on the device inside the graph try loop)
        return a.dtp ? launch_pair_t<true, true, true, false, true, true>(a, st)
                     : launch_pair_t<true, true, true, false, true, false>(a, st);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace rkb
