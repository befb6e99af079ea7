// rk_stencil.cu — K3: fused Gray–Scott stage kernel (TMA-fed), halo-plane pack, ring fill.
//
// One launch evaluates one Runge–Kutta stage i of the 3D Gray–Scott system (Listing 2,
// P:L169-170; R-1..R-3) over a z-slab:
//   Y_i = u + sum_{j<i} (dt a_ij) k_j      computed on the fly for every loaded cell
//                                          (Odeint's scale_sum algebra, fused
//                                          into the stencil: Y_i never goes to HBM)
//   k_i = d*Lap(Y_i) + reaction(Y_i)       7-point periodic stencil + reaction terms
//   epilogue: store k_i, or u_new = u + sum_j (dt b_j) k_j, and/or the embedded error
//             ratio with a warp-shuffle / block max (P:L42, P:L135 for_each_norm).
// Which terms exist is the compile-time StageSpec of (scheme, adaptive, stage): zero Butcher
// coefficients are skipped by the compiler, exactly where the oracle skips them.
//
// Data movement (sm_100a): a CTA owns a 32x8 tile of the xy plane and sweeps a chunk of z
// planes.  For every plane, one elected thread issues one 4D TMA box load per input array
// into an R-deep shared-memory ring guarded by mbarriers, R-1 planes ahead of the plane being
// computed: a deep, register-free HBM stream.  Arrays that enter Y_i are loaded as the tile
// plus its periodic ring (34x10 cells x 2 components, exact thanks to the padded layout);
// arrays only needed at the tile's own cells (final-combination / error terms) as the bare
// 32x8 tile.  Each plane's Y is formed once into a double-buffered smem tile; the own column
// keeps Y(z-1), Y(z), Y(z+1) in registers.  One __syncthreads per plane.  z neighbours at the
// slab ends come from ghost planes (multi-GPU, filled by NCCL) or by wrapping (one GPU).
//
// Arithmetic follows DESIGN.md R-17 bit for bit (no FMA: __dadd_rn / __dmul_rn), so the
// results equal the oracle's for any tile/chunk/GPU decomposition.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "rk_device.cuh"
#include "rk_kernels.cuh"

namespace rkb {

namespace {

// The kernel's helper lambdas capture its per-thread state by reference: keep them inlined.
#define INLINE __attribute__((always_inline))

constexpr int TX = 32;  // tile width (one warp per row)
constexpr int NT = 256;  // threads per CTA (8 warps); a thread owns ROWS cells of a column
constexpr int BW = TX + 2;
constexpr int SMEM_BUDGET = 110 * 1024;    // 2 CTAs per SM
constexpr int SMEM_BUDGET_1 = 226 * 1024;  // 1 CTA per SM (wide RKF78 stages)

// Tile geometry for ROWS tile rows per thread: a 32 x (8*ROWS) tile.
template <int ROWS>
struct Tile {
    static constexpr int TH = 8 * ROWS;                             // tile height
    static constexpr int BH = TH + 2;
    static constexpr int BOX = BW * BH;                             // ring box cells / component
    static constexpr int BOX_BYTES = 2 * BOX * 8;                   // 5440 | 9792 B
    static constexpr int HALO_SLOT = (BOX_BYTES + 127) / 128 * 128;
    // interior box: the tile's own rows, 34 wide from the 16-byte aligned column x0 (TMA
    // needs a 16-byte aligned inner start)
    static constexpr int OWN_BOX = TH * BW;
    static constexpr int OWN_BYTES = 2 * OWN_BOX * 8;               // 4352 | 8704 B
    static constexpr int NHALO = BOX - TX * TH;                     // ring positions (84 | 100)
    static_assert(NHALO <= NT, "one ring position per thread");
    static_assert(OWN_BYTES % 128 == 0, "TMA destinations stay 128-byte aligned");
};

struct Layout {
    int off[kMaxSlots] = {};  // byte offset of slot s inside a ring stage
    int stage_bytes = 0;      // one ring stage (base + slots)
    int tx_bytes = 0;         // TMA bytes landing per non-ghost output plane
    int tx_edge = 0;          // ... per z-halo plane (zb-1, ze): Y arrays only
    int R = 2;                // ring depth
    int minb = 2;             // CTAs per SM the layout is sized for (__launch_bounds__)
    bool ydirect = false;     // Y_i == base array: stencil reads the ring stage directly
    int smem = 0;
};

// Y-direct stages (no slot enters Y: every first stage, Euler, Adams–Bashforth, the FSAL
// tail) read their x/y neighbours straight from the TMA ring stage of the centre plane and
// need no Y tile in shared memory; the others form Y once per plane into a double buffer.
template <int ROWS>
__host__ __device__ constexpr Layout layout_of(const StageSpec& P) {
    using T = Tile<ROWS>;
    Layout L{};
    bool yd = true;
    for (int s = 0; s < P.nslots; ++s) yd = yd && !P.gnz[s];
    L.ydirect = yd;
    const int ybuf = yd ? 0 : 2 * T::HALO_SLOT;
    int o = T::HALO_SLOT, tx = T::BOX_BYTES, te = T::BOX_BYTES;
    for (int s = 0; s < P.nslots; ++s) {
        L.off[s] = o;
        o += P.halo[s] ? T::HALO_SLOT : T::OWN_BYTES;
        tx += P.halo[s] ? T::BOX_BYTES : T::OWN_BYTES;
        te += P.halo[s] ? T::BOX_BYTES : 0;
    }
    L.stage_bytes = o;
    L.tx_bytes = tx;
    L.tx_edge = te;
    const int rmax = yd ? 6 : 4;  // a Y-direct ring also holds the centre plane
    int R = (SMEM_BUDGET - ybuf - 64) / o;
    if (R < (yd ? 3 : 2)) {  // too wide for 2 CTAs per SM: one CTA with a deeper ring
        L.minb = 1;
        R = (SMEM_BUDGET_1 - ybuf - 64) / o;
    }
    R = R > rmax ? rmax : (R < 2 ? 2 : R);
    L.R = R;
    L.smem = R * o + ybuf + R * 8;
    return L;
}

template <int S, int AD, int I>
constexpr int kRows = stage_rows(stage_spec(S, AD, I));
template <int S, int AD, int I>
constexpr int kMinBlocks = layout_of<kRows<S, AD, I>>(stage_spec(S, AD, I)).minb;

// ---- PTX wrappers -------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

// P2P halo handshake (P2pSync, rk_kernels.cuh): every CTA reads this stage's sequence number
// (*seqp + 1: the counter only advances at the end of the stage's boundary launch, after every
// CTA of it has started) and waits for the flags on entry; the last CTA to finish publishes
// seq (and, for the boundary launch, advances the counter).  Every thread fences its own
// stores before the count.  Returns seq (0 without handshake).
__device__ __forceinline__ unsigned long long p2p_wait(const P2pSync& s) {
    if (!s.on) return 0ull;
    __shared__ unsigned long long s_seq;
    if (threadIdx.x == 0) {
        const unsigned long long seq = *(volatile const unsigned long long*)s.seqp + 1;
        const unsigned long long wmin = s.role == 0 ? (seq >= 2 ? seq - 2 : 0ull) : seq;
#pragma unroll
        for (int d = 0; d < 2; ++d)
            while (ld_acquire_sys(s.wait[d]) < wmin) __nanosleep(64);
        s_seq = seq;
    }
    __syncthreads();
    return s_seq;
}
// The pack launch (role 0) stores into the neighbours' memory, so every CTA fences those
// stores at system scope before it is counted.  The boundary launch (role 1) only READ ghost
// planes (through TMA, completed before the CTA's epilogue): its acknowledgement orders no
// remote writes, so a device-scope fence per CTA suffices and the last CTA alone issues the
// system-scope fence and the release stores.
__device__ __forceinline__ void p2p_notify(const P2pSync& s, unsigned long long seq) {
    if (!s.on) return;
    if (s.role == 0) __threadfence_system();
    else __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long nb = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
        if (atomicAdd(s.count, 1ull) + 1 == nb) {
            *s.count = 0ull;  // the next launch on this stream starts after this one ends
            __threadfence_system();
            st_release_sys(s.notify[0], seq);
            st_release_sys(s.notify[1], seq);
            if (s.role == 1) *s.seqp = seq;  // stage complete on this rank
        }
    }
}

__device__ __forceinline__ bool plane_is_ghost(const GsStageArgs& a, int p) {
    return (p < 0 && a.has_glo) || (p >= a.geo.nzl && a.has_ghi);
}

// One own cell of a padded array: its offset inside a (plane, component) slice and the
// periodic ring copies it must also write (corners are never read).
struct Cell {
    int64_t off;      // (y+1)*P + (x+1)
    bool ring;        // on the domain edge: some ring copy below applies
    bool x0, x1, y0, y1;
};
__device__ __forceinline__ void store_cell(double* out, const GridGeom& g, int64_t slice, const Cell& e,
                                           double v) {
    double* p = out + slice + e.off;
    p[0] = v;
    if (e.ring) {  // warp-uniformly false away from the domain edges
        if (e.x0) p[g.nx] = v;                    // x = 0     -> ring column nx+1
        if (e.x1) p[-g.nx] = v;                   // x = nx-1  -> ring column 0
        if (e.y0) p[(int64_t)g.ny * g.P] = v;     // y = 0     -> ring row ny+1
        if (e.y1) p[-(int64_t)g.ny * g.P] = v;    // y = ny-1  -> ring row 0
    }
}

// Per-cell partial sums completed by the epilogue with the new k_i (bitwise identical to the
// full left-to-right sums: j = i is always the last term).
template <int NH>
struct EState {
    double w[2];  // u (+) sum beta_j k_j  (Adams–Bashforth: u)
    double e[2];  // sum delta_j k_j (first term not added to 0), or e' (TAIL)
    double d[2];  // atol (+) rtol (x) (|u| (+) dt (x) |k1|)
    double h[NH > 0 ? NH : 1][2];  // Adams–Bashforth: f_{n-1} .. f_{n-k+1} at the own cell
    double y2[2];  // AHEAD: u (+) sum a_Fj k_j (the final stage's value, without k_i)
    double y3[2];  // AHEAD with out_z: u (+) sum a_Lj k_j (the last stage's base, without k_i)
};

// the error sum already holds a term before delta_i k_i is added
__host__ __device__ constexpr bool has_prev_e(const StageSpec& P) {
    bool h = P.epi == EPI_TAIL_ERR || P.eslot >= 0;
    for (int s = 0; s < P.nslots; ++s) h = h || P.dnz[s];
    return h;
}

template <int S, int AD, int I>
__global__ void __launch_bounds__(NT, kMinBlocks<S, AD, I>) gs_stage_kernel(const __grid_constant__ GsStageArgs a) {
    constexpr StageSpec P = stage_spec(S, AD, I);
    constexpr int ROWS = stage_rows(P);
    using T = Tile<ROWS>;
    constexpr int TH = T::TH, BH = T::BH, BOX = T::BOX, OWN_BOX = T::OWN_BOX, NHALO = T::NHALO;
    constexpr Layout LY = layout_of<ROWS>(P);
    constexpr int NS = P.nslots, EPI = P.epi, R = LY.R;
    constexpr bool FIN = EPI == EPI_FINAL || EPI == EPI_FINAL_ERR || EPI == EPI_FINAL_EPART;
    constexpr bool ESUM = EPI == EPI_FINAL_ERR || EPI == EPI_FINAL_EPART;  // e from slots
    constexpr bool RATIO = EPI == EPI_FINAL_ERR || EPI == EPI_TAIL_ERR;
    constexpr bool STORE_K = EPI == EPI_K || EPI == EPI_TAIL_ERR || (EPI == EPI_AB && P.out_k >= 0);
    constexpr bool AB = EPI == EPI_AB || EPI == EPI_ABM;  // Adams epilogue (raw own-cell terms)
    constexpr bool SPECR = AD == 2;  // SPEC's ratio denominator max(|u|, |u_new|) (R-28)
    constexpr bool AHEAD = EPI == EPI_AHEAD;         // write-ahead stage (rk_stage_spec.h)
    constexpr bool AHEAD_E = AHEAD && P.out_e >= 0;  // ... with the partial error sum
    constexpr bool ZOUT = AHEAD && P.out_z >= 0;     // ... with the last stage's base Z_L (ad 5)
    constexpr bool WSLOT = P.wslot >= 0, ESLOT = P.eslot >= 0;  // final stage fed by AHEAD
    using ES = EState<AB ? NS : 0>;
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr bool YD = LY.ydirect;
    double* sY = reinterpret_cast<double*>(smem + R * LY.stage_bytes);  // [2][2][BH][BW] (!YD)
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + R * LY.stage_bytes + (YD ? 0 : 2 * T::HALO_SLOT));

    const GridGeom& G = a.geo;
    const int tid = threadIdx.x;
    // Coefficients: the host passes dt*a_ij (etc.) pre-scaled and dtp == null (scale 1.0: x*1 is
    // exact), or -- in the device-resident try loop, where dt changes on the device -- the raw
    // Butcher coefficients and dtp -> this try's dt: fl(dt*a_ij) is the same single rounding the
    // host would do, so both give the same bits.
    const double dsc = a.dtp ? *a.dtp : 1.0;
    const double dtv = a.dtp ? *a.dtp : a.dt;
    const int ntx = (G.nx + TX - 1) / TX;
    // Chunk groups (a.zpair = G > 1, zmode 0): CTAs G*t .. G*t+G-1 of a grid row own the same xy
    // tile t in G consecutive z chunks and are launched together, sweeping in alternating
    // directions (even members down, odd members up): two neighbouring chunks then either both
    // START at their shared boundary or both END there, so the two planes around every boundary
    // inside the group are read by both CTAs at the same moment (the second read hits L2)
    // instead of a chunk-wave apart.
    const int zg = a.zmode == 0 && a.zpair > 1 ? a.zpair : 1;
    const int tile = (int)blockIdx.x / zg;
    const int x0 = (tile % ntx) * TX, y0 = (tile / ntx) * TH;
    const int w = min(TX, G.nx - x0), hg = min(TH, G.ny - y0);

    int zb, ze;
    bool desc = false;  // sweep z downwards (from ze-1 to zb)
    if (a.zmode == 0) {
        const int member = (int)blockIdx.x % zg;
        const int chunk = zg * (int)blockIdx.y + member;
        desc = zg > 1 && (member & 1) == 0;
        zb = a.z_lo + chunk * a.zchunk;
        ze = min(zb + a.zchunk, a.z_hi);
    } else {
        zb = blockIdx.y == 0 ? 0 : G.nzl - 1;
        ze = zb + 1;
    }
    const int dz = desc ? -1 : 1;
    const int zfirst = desc ? ze - 1 : zb;  // first output plane of the sweep
    const int nout = ze - zb;
    // sweep plane index i (0 = the z-halo plane before the first output plane) -> global plane
    auto pidx = [&](int i) INLINE -> int { return desc ? ze - i : zb - 1 + i; };
    const unsigned long long seq = p2p_wait(a.sync);  // P2P boundary launch: ghost planes landed
    const bool gpar = (seq & 1ull) != 0;                // P2P: ghost-plane parity of this stage
    if (zb >= ze) {    // CTA-uniform, before any other barrier
        p2p_notify(a.sync, seq);
        return;
    }
    const int nplanes = ze - zb + 2;  // planes zb-1 .. ze in sweep order (pidx)

    // own cells: column lx, rows ly0 + 8r (r < ROWS)
    const int lx = tid % TX, ly0 = tid / TX;
    const int x = x0 + lx;
    bool own[ROWS];
    int pos[ROWS], poi[ROWS];  // position in a ring box / in an interior box
    Cell cell[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        const int ly = ly0 + 8 * r, y = y0 + ly;
        own[r] = (lx < w) && (ly < hg);
        pos[r] = (ly + 1) * BW + (lx + 1);
        poi[r] = ly * BW + lx + 1;
        const bool ex0 = x == 0, ex1 = x == G.nx - 1, ey0 = y == 0, ey1 = y == G.ny - 1;
        cell[r] = Cell{(int64_t)(y + 1) * G.P + (x + 1), ex0 || ex1 || ey0 || ey1, ex0, ex1, ey0, ey1};
    }
    const bool hal = tid < NHALO;  // one ring position per thread
    int pos_h = 0;
    if (tid < BW) pos_h = tid;
    else if (tid < 2 * BW) pos_h = (BH - 1) * BW + (tid - BW);
    else if (tid < 2 * BW + TH) pos_h = (tid - 2 * BW + 1) * BW;
    else if (tid < NHALO) pos_h = (tid - 2 * BW - TH + 1) * BW + (BW - 1);

    auto stage_of = [&](int i) INLINE -> unsigned char* { return smem + (size_t)(i % R) * LY.stage_bytes; };
    auto issue = [&](int i) INLINE {  // thread 0 only
        const int p = pidx(i);
        unsigned char* st = stage_of(i);
        uint64_t* b = &bar[i % R];
        if (plane_is_ghost(a, p)) {
            mbar_expect_tx(b, T::BOX_BYTES);
            tma_load_4d(st, p < 0 ? (gpar ? &a.tm_glo1 : &a.tm_glo) : (gpar ? &a.tm_ghi1 : &a.tm_ghi), b, x0, y0, 0, 0);
        } else {
            const int q = p < 0 ? p + G.nzl : (p >= G.nzl ? p - G.nzl : p);
            // z-halo planes feed only Y: own-cell slots are not loaded there
            const bool edge = i == 0 || i == nplanes - 1;
            mbar_expect_tx(b, edge ? LY.tx_edge : LY.tx_bytes);
            tma_load_4d(st, &a.tm_base, b, x0, y0, 0, q);
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                if (P.halo[s]) tma_load_4d(st + LY.off[s], &a.tm_slot[s], b, x0, y0, 0, q);
                else if (!edge) tma_load_4d(st + LY.off[s], &a.tm_slot[s], b, x0, y0 + 1, 0, q);
            }
        }
    };
    auto wait_plane = [&](int i) INLINE { mbar_wait(&bar[i % R], (uint32_t)((i / R) & 1)); };

    // Y at ring-box position hp, component c (base + Y slots; a ghost plane is Y itself)
    auto y_at = [&](const unsigned char* st, int c, int hp, bool ghost) INLINE -> double {
        double v = reinterpret_cast<const double*>(st)[c * BOX + hp];
        if (!ghost && !P.base_unew && P.base_src < 0) {
#pragma unroll
            for (int s = 0; s < NS; ++s)
                if (P.gnz[s])
                    v = add(v, mul(mul(dsc, a.g[s]), reinterpret_cast<const double*>(st + LY.off[s])[c * BOX + hp]));
        }
        return v;
    };
    // own-cell value of slot s (ring box or interior box), component c, tile row r
    auto sval = [&](const unsigned char* st, int s, int c, int r) INLINE -> double {
        const double* p = reinterpret_cast<const double*>(st + LY.off[s]);
        return P.halo[s] ? p[c * BOX + pos[r]] : p[c * OWN_BOX + poi[r]];
    };
    auto make_estate = [&](const unsigned char* st, int r, ES& es) INLINE {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const double ub = reinterpret_cast<const double*>(st)[c * BOX + pos[r]];
            if constexpr (AB) {  // newest-first sum needs f_n first: keep the raw terms
                es.w[c] = ub;
#pragma unroll
                for (int s = 0; s < NS; ++s) es.h[s][c] = sval(st, s, c, r);
            }
            if constexpr (FIN && WSLOT) {
                es.w[c] = sval(st, P.wslot, c, r);  // W from the write-ahead stage
            } else if constexpr (FIN || AHEAD) {
                double wv = ub;
#pragma unroll
                for (int s = 0; s < NS; ++s)
                    if (P.bnz[s]) wv = add(wv, mul(mul(dsc, a.beta[s]), sval(st, s, c, r)));
                es.w[c] = wv;
            }
            if constexpr (AHEAD) {
                double yv = ub;
#pragma unroll
                for (int s = 0; s < NS; ++s)
                    if (P.anz2[s]) yv = add(yv, mul(mul(dsc, a.g2[s]), sval(st, s, c, r)));
                es.y2[c] = yv;
                if constexpr (ZOUT) {
                    double zv = ub;
#pragma unroll
                    for (int s = 0; s < NS; ++s)
                        if (P.anz3[s]) zv = add(zv, mul(mul(dsc, a.g3[s]), sval(st, s, c, r)));
                    es.y3[c] = zv;
                }
            }
            if constexpr (ESUM && ESLOT) {
                es.e[c] = sval(st, P.eslot, c, r);  // E from the write-ahead stage
            } else if constexpr (ESUM || AHEAD_E) {
                double e = 0.0;
                bool first = true;
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    if (!P.dnz[s]) continue;
                    const double t = mul(mul(dsc, a.delta[s]), sval(st, s, c, r));
                    e = first ? t : add(e, t);
                    first = false;
                }
                es.e[c] = e;
            }
            if constexpr (EPI == EPI_TAIL_ERR) es.e[c] = sval(st, P.epart, c, r);
            if constexpr (RATIO) {
                const double uu = P.den_u >= 0 ? sval(st, P.den_u, c, r) : ub;
                if constexpr (SPECR) {
                    es.d[c] = fabs(uu);  // completed with |u_new| in the epilogue
                } else {
                    const double k1 = sval(st, P.den_k1, c, r);
                    es.d[c] = add(a.atol, mul(a.rtol, add(fabs(uu), mul(dtv, fabs(k1)))));
                }
            }
        }
    };
    constexpr bool HAS_PREV_E = has_prev_e(P);
    constexpr bool DNEW = P.dnew;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < R; ++s) mbar_init(&bar[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0) {
        const int n0 = nplanes < R ? nplanes : R;
        for (int i = 0; i < n0; ++i) issue(i);
    }

    double Y0[ROWS][2], Y1[ROWS][2], Y2[ROWS][2];  // Y at planes z-1, z, z+1 (rotating)
    ES Ec[ROWS] = {}, En[ROWS] = {};               // !YD: epilogue state of planes z, z+1
    double rmax = 0.0;               // running max of the ratio (exact)
    unsigned long long rbits = 0ull;  // its bit pattern (NaN-propagating)

    // ---- prologue: plane zb-1 (own column only), plane zb (tile + ring) -----------------
    // Every thread forms Y at its tile positions, valid or not: for a partial tile (w < TX or
    // hg < TH) the periodic ring sits inside the box at column w+1 / row hg+1.
    {
        wait_plane(0);
        const unsigned char* s0 = stage_of(0);
        const bool gh = plane_is_ghost(a, pidx(0));
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            Y0[r][0] = y_at(s0, 0, pos[r], gh);
            Y0[r][1] = y_at(s0, 1, pos[r], gh);
        }
        wait_plane(1);
        const unsigned char* s1 = stage_of(1);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            Y1[r][0] = y_at(s1, 0, pos[r], false);
            Y1[r][1] = y_at(s1, 1, pos[r], false);
            if constexpr (!YD) {
                sY[pos[r]] = Y1[r][0];
                sY[BOX + pos[r]] = Y1[r][1];
                if (own[r]) make_estate(s1, r, Ec[r]);
            }
        }
        if constexpr (!YD) {
            if (hal) {
                sY[pos_h] = y_at(s1, 0, pos_h, false);
                sY[BOX + pos_h] = y_at(s1, 1, pos_h, false);
            }
        }
        __syncthreads();  // ring stage 0 free (YD: stage 1 stays, it is the centre plane)
        if (tid == 0) {
            if (R < nplanes) issue(R);
            if constexpr (!YD)
                if (R + 1 < nplanes) issue(R + 1);
        }
    }

    // Output step k (plane z = zfirst + k*dz): Ym, Yc hold Y(z-dz), Y(z); Yp receives Y(z+dz).
    auto step = [&](int k, double (&Ym)[ROWS][2], double (&Yc)[ROWS][2], double (&Yp)[ROWS][2]) INLINE {
        const int z = zfirst + k * dz;
        const int i = k + 2;         // plane z+dz
        const bool more = k + 1 < nout;  // plane z+dz is an output plane of this CTA
        // [A] plane z+dz from the ring
        wait_plane(i);
        const unsigned char* si = stage_of(i);
        const bool gh = plane_is_ghost(a, z + dz);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            Yp[r][0] = y_at(si, 0, pos[r], gh);
            Yp[r][1] = y_at(si, 1, pos[r], gh);
        }
        const unsigned char* sc = stage_of(i - 1);  // YD: the centre plane's ring stage
        const double* yc;                            // Y(z) tile + ring, [c][BH][BW]
        if constexpr (YD) {
            yc = reinterpret_cast<const double*>(sc);
        } else {
            const int b = k & 1;
            yc = sY + b * 2 * BOX;
            double* yn = sY + (b ^ 1) * 2 * BOX;
            if (more) {
#pragma unroll
                for (int r = 0; r < ROWS; ++r) {
                    yn[pos[r]] = Yp[r][0];
                    yn[BOX + pos[r]] = Yp[r][1];
                    if (own[r]) make_estate(si, r, En[r]);
                }
                if (hal) {
                    yn[pos_h] = y_at(si, 0, pos_h, false);
                    yn[BOX + pos_h] = y_at(si, 1, pos_h, false);
                }
            }
        }
        // [C] stencil + reaction + epilogue at plane z
        const int64_t qo = (int64_t)z * G.ps;
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            if (!own[r]) continue;
            ES el;
            if constexpr (YD) make_estate(sc, r, el);
            const ES& ec = YD ? el : Ec[r];
            double L[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const double* v = yc + c * BOX + pos[r];
                const double ctr = Yc[r][c];
                double s = add(sub(v[-1], ctr), sub(v[1], ctr));
                s = add(s, add(sub(v[-BW], ctr), sub(v[BW], ctr)));
                const double zlo = desc ? Yp[r][c] : Ym[r][c], zhi = desc ? Ym[r][c] : Yp[r][c];
                s = add(s, add(sub(zlo, ctr), sub(zhi, ctr)));  // Y(z-1), then Y(z+1) (R-17)
                L[c] = mul(s, a.inv_h2);
            }
            const double C0 = Yc[r][0], C1 = Yc[r][1];
            const double rc = mul(mul(C0, C1), C1);
            double f[2];
            f[0] = sub(add(sub(mul(a.d1, L[0]), rc), a.F), mul(a.F, C0));
            f[1] = sub(add(mul(a.d2, L[1]), rc), mul(a.FK, C1));
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int64_t slice = qo + c * G.cs;
                if constexpr (STORE_K) store_cell(a.out_k, G, slice, cell[r], f[c]);
                if constexpr (AB) {
                    // u_{n+1} = u_n (+) g_0 f (+) g_1 h_0 (+) ... newest first (R-24, R-26);
                    // AB: f = f_n, h = f_{n-1}...; ABM: f = F(u_p), h = f_n, f_{n-1}...
                    double wv = add(ec.w[c], mul(mul(dsc, a.beta_new), f[c]));
#pragma unroll
                    for (int s = 0; s < NS; ++s)
                        if (P.bnz[s]) wv = add(wv, mul(mul(dsc, a.beta[s]), ec.h[s][c]));
                    store_cell(a.out_u, G, slice, cell[r], wv);
                }
                double unew = 0.0;
                if constexpr (FIN) {
                    unew = P.bnew ? add(ec.w[c], mul(mul(dsc, a.beta_new), f[c])) : ec.w[c];
                    store_cell(a.out_u, G, slice, cell[r], unew);
                }
                if constexpr (AHEAD) {  // Y_F (read with its ring by stage F), W, E
                    store_cell(a.out_k, G, slice, cell[r], P.a2new ? add(ec.y2[c], mul(mul(dsc, a.g2_new), f[c])) : ec.y2[c]);
                    store_cell(a.out_w, G, slice, cell[r], P.bnew ? add(ec.w[c], mul(mul(dsc, a.beta_new), f[c])) : ec.w[c]);
                    if constexpr (ZOUT)
                        store_cell(a.out_z, G, slice, cell[r], P.a3new ? add(ec.y3[c], mul(mul(dsc, a.g3_new), f[c])) : ec.y3[c]);
                }
                double e = ec.e[c];
                if constexpr (ESUM || EPI == EPI_TAIL_ERR || AHEAD_E) {
                    if constexpr (DNEW) {
                        const double t = mul(mul(dsc, a.delta_new), f[c]);
                        e = HAS_PREV_E ? add(e, t) : t;
                    }
                }
                if constexpr (EPI == EPI_FINAL_EPART) store_cell(a.out_k, G, slice, cell[r], e);
                if constexpr (AHEAD_E) store_cell(a.out_e, G, slice, cell[r], e);
                if constexpr (RATIO) {
                    // r = |e| / d exactly; skip the division when e == 0 (r = +0) or when
                    // |e| <= rmax*d*(1-2^-52) (a normal number) proves r <= rmax by
                    // monotone rounding; NaN never skips.
                    double dd = ec.d[c];
                    if constexpr (SPECR) {  // TAIL: the stage's Y is u_new itself
                        const double m = fabs(FIN ? unew : Yc[r][c]);
                        dd = add(a.atol, mul(a.rtol, dd >= m ? dd : m));
                    }
                    const double ae = fabs(e);
                    const double th = mul(mul(rmax, dd), 0.99999999999999978);
                    if (!(ae == 0.0 || (ae <= th && th >= 2.2250738585072014e-308))) {
                        const double rr = ae / dd;
                        const unsigned long long rb = ratio_bits(rr);
                        if (rb > rbits) {
                            rbits = rb;
                            rmax = rr;
                        }
                    }
                }
            }
        }
        if constexpr (!YD) {
#pragma unroll
            for (int r = 0; r < ROWS; ++r) Ec[r] = En[r];
        }
        __syncthreads();  // !YD: Y(z+1) tile complete, stage of plane z+1 free; YD: plane z free
        if (tid == 0) {
            const int nx_issue = YD ? i - 1 + R : i + R;
            if (nx_issue < nplanes) issue(nx_issue);
        }
    };

    int k = 0;
    if constexpr (ROWS == 2 || YD) {  // rotate the z queue by renaming: no register moves
        for (; k + 2 < nout; k += 3) {
            step(k, Y0, Y1, Y2);
            step(k + 1, Y1, Y2, Y0);
            step(k + 2, Y2, Y0, Y1);
        }
    }
    for (; k < nout; ++k) {
        step(k, Y0, Y1, Y2);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            Y0[r][0] = Y1[r][0]; Y0[r][1] = Y1[r][1];
            Y1[r][0] = Y2[r][0]; Y1[r][1] = Y2[r][1];
        }
    }
    if constexpr (RATIO) block_max_to_global(rbits, a.errmax);
    p2p_notify(a.sync, seq);  // P2P: ghost planes consumed -> the neighbours may overwrite them
}

// ---- halo-plane pack and ring fill -------------------------------------------------------
template <int NY>
__global__ void __launch_bounds__(256) gs_pack_kernel(const GsStageArgs a, double* __restrict__ dst0,
                                                      double* __restrict__ dst1, const P2pSync sync) {
    const unsigned long long seq = p2p_wait(sync);  // P2P: the previous use of dst was consumed
    const double dsc = a.dtp ? *a.dtp : 1.0;         // as in gs_stage_kernel
    const int64_t ps = a.geo.ps, total = 2 * ps;
    if (seq & 1ull) {  // P2P: ghost planes of parity 1
        dst0 += 2 * ps;
        dst1 += 2 * ps;
    }
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sel = e / ps, rest = e - sel * ps;
        const int64_t base = (sel ? (int64_t)(a.geo.nzl - 1) : 0) * ps + rest;
        double v = __ldg(a.base + base);
#pragma unroll
        for (int s = 0; s < NY; ++s) v = add(v, mul(mul(dsc, a.g[s]), __ldg(a.slot[s] + base)));
        (sel ? dst1 : dst0)[rest] = v;
    }
    p2p_notify(sync, seq);  // P2P: ghost planes stored -> neighbours may read them
}

__global__ void fill_ring_kernel(double* __restrict__ p, GridGeom g, int nslices) {
    const int64_t zc = blockIdx.y;  // (plane, component) slice of (ny+2) x P values
    if (zc >= nslices) return;
    double* b = p + zc * g.cs;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < max(g.nx, g.ny); t += gridDim.x * blockDim.x) {
        if (t < g.ny) {
            double* row = b + (int64_t)(t + 1) * g.P;
            row[0] = row[g.nx];
            row[g.nx + 1] = row[1];
        }
        if (t < g.nx) {
            b[t + 1] = b[(int64_t)g.ny * g.P + t + 1];
            b[(int64_t)(g.ny + 1) * g.P + t + 1] = b[(int64_t)g.P + t + 1];
        }
    }
}

// Fused allreduce(max) over the ranks' P2P flag blocks (launch_p2p_allreduce_max).  Round r uses
// slot r & 1 of every block; this rank zeroes its own other slot before arriving (nobody writes
// it again before every rank has arrived in this round, and it was last read in round r-1).
struct FlagPtrs {
    unsigned long long* f[P2P_MAX_WORLD];
};
__global__ void p2p_allreduce_max_kernel(unsigned long long* word, FlagPtrs fl, int world, int rank) {
    unsigned long long* mine = fl.f[rank];
    const unsigned long long r = mine[P2P_ROUND];
    const int slot = P2P_RED0 + (int)(r & 1ull);
    const unsigned long long v = *word;
    mine[P2P_RED0 + (int)((r + 1) & 1ull)] = 0ull;
    for (int q = 0; q < world; ++q) atomicMax_system(fl.f[q] + slot, v);
    __threadfence_system();
    for (int q = 0; q < world; ++q) atomicAdd_system(fl.f[q] + P2P_ARRIVE, 1ull);
    const unsigned long long need = (unsigned long long)world * (r + 1);
    while (ld_acquire_sys(mine + P2P_ARRIVE) < need) __nanosleep(32);
    *word = ld_acquire_sys(mine + slot);
    mine[P2P_ROUND] = r + 1;
}

template <int S, int AD, int I>
cudaError_t launch_one(const GsStageArgs& a, dim3 grid, cudaStream_t st) {
    constexpr StageSpec P = stage_spec(S, AD, I);
    static_assert(P.valid, "invalid stage");
    constexpr int bytes = layout_of<kRows<S, AD, I>>(P).smem;
    static std::atomic<unsigned long long> configured{0};
    if (cudaError_t e = smem_attr_once(configured, gs_stage_kernel<S, AD, I>, bytes); e != cudaSuccess) return e;
    gs_stage_kernel<S, AD, I><<<grid, NT, bytes, st>>>(a);
    return cudaGetLastError();
}

// Stages whose spec does not depend on the adaptive flag share one instantiation.
template <int S, int AD, int I>
cudaError_t launch_norm(const GsStageArgs& a, dim3 grid, cudaStream_t st) {
    constexpr StageSpec P = stage_spec(S, AD, I);
    if constexpr (!P.valid) {
        return cudaErrorInvalidValue;
    } else if constexpr (P.epi == EPI_K && I == 0) {
        return launch_one<1, 0, 0>(a, grid, st);  // k1 = F(u): identical for every scheme
    } else if constexpr (P.epi == EPI_K && AD != 0 && stage_spec(S, 0, I).epi == EPI_K) {
        return launch_one<S, 0, I>(a, grid, st);  // same k-only stage (not AHEAD when fixed)
    } else if constexpr (AD == 2 && P.epi != EPI_FINAL_ERR && P.epi != EPI_TAIL_ERR) {
        return launch_one<S, 1, I>(a, grid, st);  // only the ratio stages differ (R-28)
    } else {
        return launch_one<S, AD, I>(a, grid, st);
    }
}

template <int S, int AD>
cudaError_t launch_stage_i(int i, const GsStageArgs& a, dim3 grid, cudaStream_t st) {
    switch (i) {
    case 0: return launch_norm<S, AD, 0>(a, grid, st);
    case 1: return launch_norm<S, AD, 1>(a, grid, st);
    case 2: return launch_norm<S, AD, 2>(a, grid, st);
    case 3: return launch_norm<S, AD, 3>(a, grid, st);
    case 4: return launch_norm<S, AD, 4>(a, grid, st);
    case 5: return launch_norm<S, AD, 5>(a, grid, st);
    case 6: return launch_norm<S, AD, 6>(a, grid, st);
    case 7: return launch_norm<S, AD, 7>(a, grid, st);
    case 8: return launch_norm<S, AD, 8>(a, grid, st);
    case 9: return launch_norm<S, AD, 9>(a, grid, st);
    case 10: return launch_norm<S, AD, 10>(a, grid, st);
    case 11: return launch_norm<S, AD, 11>(a, grid, st);
    case 12: return launch_norm<S, AD, 12>(a, grid, st);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace

// Developer tuning knob (not part of the ABI): RKB_L2PROMO = 0 none, 1 64B, 2 128B, 3 256B.
static CUtensorMapL2promotion l2_promotion() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("RKB_L2PROMO");
        v = e ? atoi(e) : 3;
        if (v < 0 || v > 3) v = 3;
    }
    const CUtensorMapL2promotion tab[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    return tab[v];
}

cudaError_t encode_grid_maps(CUtensorMap* maps, const double* base, const GridGeom& g, int nplanes) {
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
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    // maps[2*(ROWS-1) + 0]: tile + ring box, maps[2*(ROWS-1) + 1]: interior box (own rows)
    const cuuint32_t boxes[4][4] = {{BW, Tile<1>::BH, 2, 1}, {BW, Tile<1>::TH, 2, 1},
                                    {BW, Tile<2>::BH, 2, 1}, {BW, Tile<2>::TH, 2, 1}};
    for (int m = 0; m < 4; ++m) {
        CUresult r = encode(&maps[m], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims,
                            strides, boxes[m], estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    return cudaSuccess;
}

cudaError_t launch_gs_stage(int scheme, int adaptive, int stage, const GsStageArgs& a,
                            cudaStream_t st, int* nlaunch) {
    const int th = 8 * stage_rows(stage_spec(scheme, adaptive, stage));
    const int ntx = (a.geo.nx + TX - 1) / TX, nty = (a.geo.ny + th - 1) / th;
    const int tiles = ntx * nty;
    int nchunks;
    if (a.zmode == 1) {
        nchunks = a.geo.nzl > 1 ? 2 : 1;
    } else {
        const int range = a.z_hi - a.z_lo;
        if (range <= 0) return cudaSuccess;
        nchunks = (range + a.zchunk - 1) / a.zchunk;
    }
    dim3 grid((unsigned)tiles, (unsigned)nchunks);
    if (a.zpair > 1 && a.zmode == 0) grid = dim3((unsigned)(a.zpair * tiles), (unsigned)((nchunks + a.zpair - 1) / a.zpair));
    if (nlaunch) ++*nlaunch;
    if (adaptive == 4) {  // the last stage after a K8 pair (Gragg's modified midpoint, stage 3)
        if (scheme == 6 && stage == 2) return launch_one<6, 4, 2>(a, grid, st);
        return cudaErrorInvalidValue;
    }
    if (adaptive == 5) {  // the write-ahead stage before a K8 fixed-step tail pair (stage L-2)
        if (scheme == 2 && stage == 3) return launch_one<2, 5, 3>(a, grid, st);   // Cash–Karp 5(4)
        if (scheme == 3 && stage == 3) return launch_one<3, 5, 3>(a, grid, st);   // Dormand–Prince fixed
        if (scheme == 4 && stage == 10) return launch_one<4, 5, 10>(a, grid, st); // RKF 7(8)
        return cudaErrorInvalidValue;
    }
    if (adaptive == 2) {  // SPEC's error ratio (R-28)
        switch (scheme) {
        case 2: return launch_stage_i<2, 2>(stage, a, grid, st);
        case 3: return launch_stage_i<3, 2>(stage, a, grid, st);
        case 4: return launch_stage_i<4, 2>(stage, a, grid, st);
        default: return cudaErrorInvalidValue;
        }
    }
    const int ad = adaptive ? 1 : 0;
    switch (scheme * 2 + ad) {
    case 0: return launch_stage_i<0, 0>(stage, a, grid, st);
    case 2: return launch_stage_i<1, 0>(stage, a, grid, st);
    case 4: return launch_stage_i<2, 0>(stage, a, grid, st);
    case 5: return launch_stage_i<2, 1>(stage, a, grid, st);
    case 6: return launch_stage_i<3, 0>(stage, a, grid, st);
    case 7: return launch_stage_i<3, 1>(stage, a, grid, st);
    case 8: return launch_stage_i<4, 0>(stage, a, grid, st);
    case 9: return launch_stage_i<4, 1>(stage, a, grid, st);
    case 10: return launch_stage_i<5, 0>(stage, a, grid, st);
    case 12: return launch_stage_i<6, 0>(stage, a, grid, st);
    case 22: return launch_one<11, 0, 0>(a, grid, st);  // Adams–Bashforth 1..8: one launch/step
    case 24: return launch_one<12, 0, 0>(a, grid, st);
    case 26: return launch_one<13, 0, 0>(a, grid, st);
    case 28: return launch_one<14, 0, 0>(a, grid, st);
    case 30: return launch_one<15, 0, 0>(a, grid, st);
    case 32: return launch_one<16, 0, 0>(a, grid, st);
    case 34: return launch_one<17, 0, 0>(a, grid, st);
    case 36: return launch_one<18, 0, 0>(a, grid, st);
    case 42: return launch_one<21, 0, 0>(a, grid, st);  // Adams–Bashforth–Moulton 1..8: PEC launch
    case 44: return launch_one<22, 0, 0>(a, grid, st);
    case 46: return launch_one<23, 0, 0>(a, grid, st);
    case 48: return launch_one<24, 0, 0>(a, grid, st);
    case 50: return launch_one<25, 0, 0>(a, grid, st);
    case 52: return launch_one<26, 0, 0>(a, grid, st);
    case 54: return launch_one<27, 0, 0>(a, grid, st);
    case 56: return launch_one<28, 0, 0>(a, grid, st);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_gs_pack(const GsStageArgs& a, double* dst0, double* dst1, const P2pSync& sync,
                           cudaStream_t st) {
    const int64_t total = 2 * a.geo.ps;
    int64_t blocks = (total + 255) / 256;
    // P2P: every CTA fences its remote stores at system scope, so fewer, longer CTAs (2 per SM)
    if (blocks > (sync.on ? 148 * 2 : 148 * 8)) blocks = sync.on ? 148 * 2 : 148 * 8;
    switch (a.nyslots) {
    case 0: gs_pack_kernel<0><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    case 1: gs_pack_kernel<1><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    case 2: gs_pack_kernel<2><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    case 3: gs_pack_kernel<3><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    case 4: gs_pack_kernel<4><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    case 5: gs_pack_kernel<5><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    case 6: gs_pack_kernel<6><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    case 7: gs_pack_kernel<7><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    case 8: gs_pack_kernel<8><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    case 9: gs_pack_kernel<9><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    case 10: gs_pack_kernel<10><<<(unsigned)blocks, 256, 0, st>>>(a, dst0, dst1, sync); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_p2p_allreduce_max(unsigned long long* word, unsigned long long* const* flags, int world,
                                     int rank, cudaStream_t st) {
    if (world < 1 || world > P2P_MAX_WORLD || rank < 0 || rank >= world) return cudaErrorInvalidValue;
    FlagPtrs fl{};
    for (int q = 0; q < world; ++q) fl.f[q] = flags[q];
    p2p_allreduce_max_kernel<<<1, 1, 0, st>>>(word, fl, world, rank);
    return cudaGetLastError();
}

cudaError_t launch_fill_ring(double* p, const GridGeom& g, int nslices, cudaStream_t st) {
    const int n = g.nx > g.ny ? g.nx : g.ny;
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)nslices);
    fill_ring_kernel<<<grid, 256, 0, st>>>(p, g, nslices);
    return cudaGetLastError();
}

}  // namespace rkb
