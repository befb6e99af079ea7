// rk_fused.cu — K6: one whole fixed Runge–Kutta step of Gray–Scott per launch (temporal
// blocking across the stages of the step, "fused" variants).
//
// For the tableaux whose stage values chain through ONE slope -- Y_1 = u and
// Y_s = u (+) g_s k_{s-1} (a_ij != 0 only for j = i-1): classic RK4 and the explicit
// midpoint rule (R-22) -- the step u -> u_new = u (+) beta_1 k_1 (+) ...
// (+) beta_L k_L at a cell depends only on u within L cells of it (7-point stencil per stage,
// Listing 2).  A CTA owns a 32x16 xy tile and sweeps a chunk of z planes:
//   * u is loaded ONCE per plane by TMA: the tile plus an L-cell margin (periodic margin
//     cells beyond the padded layout's 1-cell ring are patched from global memory by the
//     CTAs on the domain edge);
//   * stage s runs one plane behind stage s-1, on the tile grown by L-s cells (k_s there
//     needs Y_s on L-s+1 cells); Y_2 .. Y_L live in 3-plane shared-memory windows, the
//     partial final sums W = u (+) beta_1 k_1 (+) ... in registers (one own cell per thread);
//   * the last stage stores u_new (with its periodic ring copies).
// HBM traffic per step is u once (+ the margins re-read by neighbouring CTAs through L2) and
// u_new once: 32 B/cell instead of the stage-by-stage 208 (RK4) / 80 (midpoint), for
// (38*22 + 36*20 + 34*18 + 32*16) / (4*32*16) = 1.31x the RK4 stencil work (margins).
// Measured on the B200 this is SLOWER than the stage-by-stage kernels (RK4 4.65-4.69 vs 4.42
// ms at 512^3): 196 KB of shared memory allow one 16-warp CTA per SM and every stage phase
// ends in a CTA barrier, so the kernel is latency-bound at ~36 % FP64-pipe use (DESIGN.md §7,
// profiles/r1_k6_fused_rk4_ncu.txt).  It is therefore opt-in (RK_OPT_FUSED_STEP), an ablation
// that locates the stage-by-stage roofline against on-chip fusion on this part.
//
// Arithmetic is the stage kernel's (K3, rk_stencil.cu) expression for expression (DESIGN.md
// R-17): the Laplacian in difference form (x, then y, then z), the same reaction trees,
// Y_s = u (+) g_s (x) k_{s-1}, W = u (+) beta_1 (x) k_1 (+) ... left to right, no FMA.  So the
// result equals K3's and the oracle's bit for bit for any tile / chunk decomposition.
// One GPU only (z wraps by index); the multi-GPU halo paths keep the stage-by-stage kernels.
#include <cudaTypedefs.h>

#include <type_traits>

#include "rk_device.cuh"
#include "rk_kernels.cuh"
#include "rk_tableau.h"

namespace rkb {

namespace {

#define FINLINE __attribute__((always_inline))

constexpr int FX = 32;   // tile width (one warp per row)
constexpr int FY = 16;   // tile height
constexpr int FNT = 512; // threads per CTA: one own cell each

// stage values chain through one slope: a_ij != 0 iff j == i-1
__host__ __device__ constexpr bool chained(int S) {
    const Tableau T = tableau_of(S);
    if (T.s < 2 || T.s > 4 || T.err_order != 0) return false;
    for (int i = 0; i < T.s; ++i)
        for (int j = 0; j < i; ++j)
            if (rat_nz(T.a[i][j]) != (j == i - 1)) return false;
    return true;
}

__host__ __device__ constexpr bool b_nz(int S, int j) { return rat_nz(tableau_of(S).b[j]); }

template <int S>
struct FCfg {
    static constexpr int L = tableau_of(S).s;
    static constexpr int XL = (L + 1) / 2 * 2;  // left margin rounded up to even (16-byte TMA start)
    static constexpr int UW = FX + 2 * XL + 2;  // u box: padded columns x0-XL .. (even start, 16 B)
    static constexpr int UH = FY + 2 * L;
    static constexpr int UBOX = UW * UH;       // cells per component
    static constexpr int UBYTES = 2 * UBOX * 8;
    static constexpr int USLOT = (UBYTES + 127) / 128 * 128;
    static constexpr int NEED = L > 3 ? L : 3;  // u planes in use at once
    static constexpr int R = NEED + 2;          // ring depth (2 planes of prefetch)
    static constexpr int NFIX = (UBOX + FNT - 1) / FNT;  // box positions scanned per thread
    // window of Y_s (s = 2..L): the tile plus hw(s) = L-s+1 cells, 3 planes
    static constexpr int hw(int s) { return L - s + 1; }
    static constexpr int ww(int s) { return FX + 2 * hw(s); }
    static constexpr int wbox(int s) { return ww(s) * (FY + 2 * hw(s)); }
    static constexpr int wslot(int s) { return (2 * wbox(s) * 8 + 127) / 128 * 128; }
    static constexpr int woff(int s) {
        int o = R * USLOT;
        for (int q = 2; q < s; ++q) o += 3 * wslot(q);
        return o;
    }
    static constexpr int smem = woff(L + 1) + R * 8;
    static constexpr int nring(int r) { return (FX + 2 * r) * (FY + 2 * r) - FX * FY; }
    static_assert(nring(L - 1) <= FNT, "one ring cell per thread and stage");
};

// region coordinates of ring cell j of the tile grown by r cells: top band, bottom band,
// then the side columns row by row
__device__ __forceinline__ void ring_coord(int j, int r, int& rx, int& ry) {
    const int wr = FX + 2 * r;
    if (j < r * wr) {
        ry = -r + j / wr;
        rx = -r + j % wr;
        return;
    }
    j -= r * wr;
    if (j < r * wr) {
        ry = FY + j / wr;
        rx = -r + j % wr;
        return;
    }
    j -= r * wr;
    ry = j / (2 * r);
    const int k = j % (2 * r);
    rx = k < r ? -r + k : FX + (k - r);
}

struct FCell {
    int64_t off;  // (y+1)*P + (x+1)
    bool ring;    // on the domain edge: some periodic ring copy applies
    bool x0, x1, y0, y1;
};

__device__ __forceinline__ int imod(int a, int n) {
    const int m = a % n;
    return m < 0 ? m + n : m;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// k = F(Y) at one cell: zc / zm / zp point at the cell's component 0 in the centre / lower /
// upper plane, cs = component stride, pitch = row pitch (K3's expression trees, R-17)
__device__ __forceinline__ void gs_rhs(const double* zc, const double* zm, const double* zp, int cs, int pitch,
                                       const GsFusedArgs& a, double f[2]) {
    double Lp[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const double* v = zc + c * cs;
        const double ctr = v[0];
        double s = add(sub(v[-1], ctr), sub(v[1], ctr));
        s = add(s, add(sub(v[-pitch], ctr), sub(v[pitch], ctr)));
        s = add(s, add(sub(zm[c * cs], ctr), sub(zp[c * cs], ctr)));
        Lp[c] = mul(s, a.inv_h2);
    }
    const double C0 = zc[0], C1 = zc[cs];
    const double rc = mul(mul(C0, C1), C1);
    f[0] = sub(add(sub(mul(a.d1, Lp[0]), rc), a.F), mul(a.F, C0));
    f[1] = sub(add(mul(a.d2, Lp[1]), rc), mul(a.FK, C1));
}

// the same with the cell's centre value and z neighbours in registers (bitwise the same value)
__device__ __forceinline__ void gs_rhs_q(const double* v0, int cs, int pitch, const double (&ctr)[2],
                                         const double (&zm)[2], const double (&zp)[2], const GsFusedArgs& a,
                                         double f[2]) {
    double Lp[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const double* v = v0 + c * cs;
        const double cc = ctr[c];
        double s = add(sub(v[-1], cc), sub(v[1], cc));
        s = add(s, add(sub(v[-pitch], cc), sub(v[pitch], cc)));
        s = add(s, add(sub(zm[c], cc), sub(zp[c], cc)));
        Lp[c] = mul(s, a.inv_h2);
    }
    const double C0 = ctr[0], C1 = ctr[1];
    const double rc = mul(mul(C0, C1), C1);
    f[0] = sub(add(sub(mul(a.d1, Lp[0]), rc), a.F), mul(a.F, C0));
    f[1] = sub(add(mul(a.d2, Lp[1]), rc), mul(a.FK, C1));
}

template <int S>
__global__ void __launch_bounds__(FNT, 1) gs_fused_kernel(const __grid_constant__ GsFusedArgs a) {
    using C = FCfg<S>;
    constexpr int L = C::L, XL = C::XL, UW = C::UW, UBOX = C::UBOX, R = C::R, NEED = C::NEED, UQ = NEED;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::woff(L + 1));

    const GridGeom& G = a.geo;
    const int tid = threadIdx.x;
    const int ntx = (G.nx + FX - 1) / FX;
    const int x0 = (int)(blockIdx.x % ntx) * FX, y0 = (int)(blockIdx.x / ntx) * FY;
    const int zb = (int)blockIdx.y * a.zchunk;
    const int ze = min(zb + a.zchunk, G.nzl);
    if (zb >= ze) return;
    const int nU = ze - zb + 2 * L;  // u planes zb-L .. ze+L-1; index i is plane zb-L+i

    // own cell
    const int lx = tid % FX, ly = tid / FX;
    const bool own = x0 + lx < G.nx && y0 + ly < G.ny;
    const int o_ub = (lx + XL + 1) + (ly + L) * UW;
    int o_w[L + 1];  // window position of the own cell in Y_s's window (s >= 2)
#pragma unroll
    for (int s = 2; s <= L; ++s) o_w[s] = (lx + C::hw(s)) + (ly + C::hw(s)) * C::ww(s);
    FCell cell;
    {
        const int x = x0 + lx, y = y0 + ly;
        const bool ex0 = x == 0, ex1 = x == G.nx - 1, ey0 = y == 0, ey1 = y == G.ny - 1;
        cell = FCell{(int64_t)(y + 1) * G.P + (x + 1), ex0 || ex1 || ey0 || ey1, ex0, ex1, ey0, ey1};
    }
    // ring cell of stage s (s < L, tile grown by r = L-s): u box pos, Y_s window pos (s >= 2),
    // Y_{s+1} window pos
    bool rg_on[L];
    int rg_ub[L], rg_wc[L], rg_wn[L];
#pragma unroll
    for (int s = 1; s < L; ++s) {
        const int r = L - s;
        rg_on[s] = tid < C::nring(r);
        int rx = 0, ry = 0;
        if (rg_on[s]) ring_coord(tid, r, rx, ry);
        rg_ub[s] = (rx + XL + 1) + (ry + L) * UW;
        rg_wc[s] = s >= 2 ? (rx + C::hw(s)) + (ry + C::hw(s)) * C::ww(s) : 0;
        rg_wn[s] = (rx + C::hw(s + 1)) + (ry + C::hw(s + 1)) * C::ww(s + 1);
    }
    // periodic margin cells beyond the padded ring: patched from global memory
    int fx_pos[C::NFIX];
    int64_t fx_src[C::NFIX];
    bool anyfix = false;
#pragma unroll
    for (int k = 0; k < C::NFIX; ++k) {
        const int p = tid + k * FNT;
        const int x = x0 - XL - 1 + p % UW, y = y0 - L + p / UW;
        // the padded layout holds cells x in [0, nx), y in [-1, ny] and y in [0, ny), x in
        // [-1, nx] (not the ring corners); everything else wraps
        const bool held = (x >= 0 && x < G.nx && y >= -1 && y <= G.ny) || (y >= 0 && y < G.ny && x >= -1 && x <= G.nx);
        const bool need = p < UBOX && !held;
        fx_pos[k] = need ? p : -1;
        fx_src[k] = (int64_t)(imod(y, G.ny) + 1) * G.P + (imod(x, G.nx) + 1);
        anyfix = anyfix || need;
    }
    const bool edge = __syncthreads_or(anyfix);

    auto uslot = [&](int i) FINLINE -> double* { return reinterpret_cast<double*>(smem + (size_t)(i % R) * C::USLOT); };
    auto wslot = [&](int s, int i) FINLINE -> double* {
        return reinterpret_cast<double*>(smem + C::woff(s) + (size_t)(i % 3) * C::wslot(s));
    };
    auto plane_of = [&](int i) FINLINE -> int { return imod(zb - L + i, G.nzl); };
    auto issue = [&](int i) FINLINE {  // thread 0
        uint64_t* b = &bar[i % R];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
                     "r"((uint32_t)C::UBYTES)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_addr(uslot(i))),
            "l"(reinterpret_cast<uint64_t>(&a.tm_u)), "r"(smem_addr(b)), "r"(x0 - XL), "r"(y0 - L + 1), "r"(0),
            "r"(plane_of(i))
            : "memory");
    };
    auto wait = [&](int i) FINLINE {
        const uint32_t ad = smem_addr(&bar[i % R]), par = (uint32_t)((i / R) & 1);
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WAITF_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WAITF_%=;\n}" ::"r"(ad),
            "r"(par)
            : "memory");
    };

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < R; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&bar[s])), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int i = 0; i < (nU < R ? nU : R); ++i) issue(i);

    // own-cell registers: partial final sums W of the planes in flight (slot = plane index
    // % L), u at plane indices t, t-1, ... (newest first), and Y_s (s >= 2) at the centre
    // plane c = t-s and its two z neighbours ([0] c-1, [1] c, [2] c+1): the z column of the
    // stencil never comes from shared memory
    double W[L][2], uq[UQ][2], yq[L + 1][3][2];
#pragma unroll
    for (int q = 0; q < L; ++q) W[q][0] = W[q][1] = 0.0;
#pragma unroll
    for (int q = 0; q < UQ; ++q) uq[q][0] = uq[q][1] = 0.0;
#pragma unroll
    for (int q = 0; q <= L; ++q)
#pragma unroll
        for (int k = 0; k < 3; ++k) yq[q][k][0] = yq[q][k][1] = 0.0;

    // stage s at iteration t: k_s on plane index t-s over the tile grown by L-s cells
    auto stage = [&](auto sc, auto qc, int t) FINLINE {
        constexpr int s = decltype(sc)::value;
        constexpr int q = decltype(qc)::value;     // t % L
        constexpr int wq = ((q - s) % L + L) % L;  // W slot of plane index t-s
        const bool act = t >= 2 * s;               // CTA-uniform
        const int ic = t - s;                      // centre plane index
        double yo[2] = {0.0, 0.0};                 // Y_{s+1} at the own cell
        if (act) {
            const double *pc, *pm, *pp;
            int cs, pitch;
            if constexpr (s == 1) {
                pc = uslot(ic);
                pm = uslot(ic - 1);
                pp = uslot(ic + 1);
                cs = UBOX;
                pitch = UW;
            } else {
                pc = wslot(s, ic);
                pm = wslot(s, ic - 1);
                pp = wslot(s, ic + 1);
                cs = C::wbox(s);
                pitch = C::ww(s);
            }
            double f[2];
            // own cell: xy neighbours from shared memory, the z column from registers
            if constexpr (s == 1) gs_rhs_q(pc + o_ub, cs, pitch, uq[1], uq[2], uq[0], a, f);
            else gs_rhs_q(pc + o_w[s], cs, pitch, yq[s][1], yq[s][0], yq[s][2], a, f);
            if constexpr (s < L) {
                double* yn = wslot(s + 1, ic);
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    yo[c] = add(uq[s][c], mul(a.g[s], f[c]));
                    yn[c * C::wbox(s + 1) + o_w[s + 1]] = yo[c];
                }
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                double w = s == 1 ? uq[1][c] : W[wq][c];
                if constexpr (b_nz(S, s - 1)) w = add(w, mul(a.beta[s - 1], f[c]));
                W[wq][c] = w;
            }
            if constexpr (s == L) {
                if (own) {
                    const int z = zb - 2 * L + t;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        double* p = a.out + (int64_t)z * G.ps + c * G.cs + cell.off;
                        const double v = W[wq][c];
                        p[0] = v;
                        if (cell.ring) {
                            if (cell.x0) p[G.nx] = v;
                            if (cell.x1) p[-G.nx] = v;
                            if (cell.y0) p[(int64_t)G.ny * G.P] = v;
                            if (cell.y1) p[-(int64_t)G.ny * G.P] = v;
                        }
                    }
                }
            }
            // ring cell of the grown tile (shared memory only)
            if constexpr (s < L) {
                if (rg_on[s]) {
                    const int pos = s == 1 ? rg_ub[s] : rg_wc[s];
                    gs_rhs(pc + pos, pm + pos, pp + pos, cs, pitch, a, f);
                    double* yn = wslot(s + 1, ic);
                    const double* U = uslot(ic);
#pragma unroll
                    for (int c = 0; c < 2; ++c)
                        yn[c * C::wbox(s + 1) + rg_wn[s]] = add(U[c * UBOX + rg_ub[s]], mul(a.g[s], f[c]));
                }
            }
        }
        if constexpr (s < L) {  // every iteration, active or not: the queue stays aligned
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                yq[s + 1][0][c] = yq[s + 1][1][c];
                yq[s + 1][1][c] = yq[s + 1][2][c];
                yq[s + 1][2][c] = yo[c];
            }
        }
    };

    auto iteration = [&](auto qc, int t) FINLINE {
        wait(t);
        if (edge) {
            double* U = uslot(t);
            const int64_t zo = (int64_t)plane_of(t) * G.ps;
#pragma unroll
            for (int k = 0; k < C::NFIX; ++k) {
                if (fx_pos[k] >= 0) {
                    U[fx_pos[k]] = a.u[zo + fx_src[k]];
                    U[UBOX + fx_pos[k]] = a.u[zo + G.cs + fx_src[k]];
                }
            }
        }
        // Barriers: the patched margin must be visible (edge CTAs only: elsewhere every thread
        // waited on the plane itself); one between consecutive stages (stage s+1 reads the Y
        // plane stage s just wrote).  The u plane t-NEED+1 is last read by stage L-1 (its Y_L),
        // so it is refilled right after the barrier before stage L.  A window slot that stage s
        // rewrites in the next iteration was last read by stage s+1 of this one, at least one
        // barrier earlier -- except for L = 2 (stage 1 rewrites what stage 2 just read).
        if (edge) __syncthreads();
        {
            const double* U = uslot(t);
#pragma unroll
            for (int k = UQ - 1; k > 0; --k) {
                uq[k][0] = uq[k - 1][0];
                uq[k][1] = uq[k - 1][1];
            }
            uq[0][0] = U[o_ub];
            uq[0][1] = U[UBOX + o_ub];
        }
        auto refill = [&]() FINLINE {
            if (tid == 0) {
                const int nxt = t - NEED + 1 + R;
                if (t >= NEED - 1 && nxt < nU) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the patches
                    issue(nxt);
                }
            }
        };
        stage(std::integral_constant<int, 1>{}, qc, t);
        if constexpr (L >= 2) {
            __syncthreads();
            if constexpr (L == 2) refill();
            stage(std::integral_constant<int, 2>{}, qc, t);
        }
        if constexpr (L >= 3) {
            __syncthreads();
            if constexpr (L == 3) refill();
            stage(std::integral_constant<int, 3>{}, qc, t);
        }
        if constexpr (L >= 4) {
            __syncthreads();
            refill();
            stage(std::integral_constant<int, 4>{}, qc, t);
        }
        if constexpr (L <= 2) __syncthreads();
    };

    for (int t0 = 0; t0 < nU; t0 += L) {
        iteration(std::integral_constant<int, 0>{}, t0);
        if (t0 + 1 < nU) iteration(std::integral_constant<int, 1 % L>{}, t0 + 1);
        if constexpr (L >= 3)
            if (t0 + 2 < nU) iteration(std::integral_constant<int, 2 % L>{}, t0 + 2);
        if constexpr (L >= 4)
            if (t0 + 3 < nU) iteration(std::integral_constant<int, 3 % L>{}, t0 + 3);
    }
}

template <int S>
cudaError_t launch_fused_t(const GsFusedArgs& a, cudaStream_t st) {
    static_assert(chained(S), "K6 needs a chained-stage tableau");
    constexpr int bytes = FCfg<S>::smem;
    static std::atomic<unsigned long long> configured{0};
    if (cudaError_t e = smem_attr_once(configured, gs_fused_kernel<S>, bytes); e != cudaSuccess) return e;
    const int ntx = (a.geo.nx + FX - 1) / FX, nty = (a.geo.ny + FY - 1) / FY;
    const int nch = (a.geo.nzl + a.zchunk - 1) / a.zchunk;
    gs_fused_kernel<S><<<dim3((unsigned)(ntx * nty), (unsigned)nch), FNT, bytes, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

bool fused_scheme(int scheme) { return scheme == 1 || scheme == 5 || scheme == 6; }

int fused_halo(int scheme) { return fused_scheme(scheme) ? tableau_of(scheme).s : 0; }

cudaError_t encode_fused_map(CUtensorMap* map, const double* base, const GridGeom& g, int nplanes, int L) {
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
    const int XL = (L + 1) / 2 * 2;  // FCfg<S>::XL
    const cuuint32_t box[4] = {(cuuint32_t)(FX + 2 * XL + 2), (cuuint32_t)(FY + 2 * L), 2, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_gs_fused(int scheme, const GsFusedArgs& a, cudaStream_t st) {
    if (a.zchunk <= 0) return cudaErrorInvalidValue;
    switch (scheme) {
    case 1: return launch_fused_t<1>(a, st);  // RK4
    case 5: return launch_fused_t<5>(a, st);  // explicit midpoint
    case 6: return launch_fused_t<6>(a, st);  // modified midpoint (Gragg, 2 substeps)
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace rkb
