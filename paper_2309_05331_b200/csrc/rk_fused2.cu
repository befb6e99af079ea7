// rk_fused2.cu — K7: one whole fixed Runge–Kutta step of Gray–Scott per launch, temporal
// blocking across the stages with WARP-SPECIALISED stage groups (RK_OPT_FUSED_STEP = 2).
//
// Same method and arithmetic as K6 (rk_fused.cu; chained tableaux Y_1 = u, Y_s = u (+) g_s k_{s-1}:
// RK4, the explicit and the modified midpoint), same tile (32x16 own cells, 1 CTA per SM),
// same u box (TMA, L-cell margin, periodic patches on edge CTAs), same 3-plane windows of the
// stage values -- but instead of all 16 warps running stage 1, barrier, stage 2, barrier, ...
// every plane, the warps are split into L groups, group s evaluating k_s for the cells of the
// tile grown by L-s (836 / 720 / 612 / 512 cells for RK4: the groups get 5 / 4 / 4 / 3 warps so
// the per-thread work is balanced, ~5-6 cells each).  Group s runs its own loop over the z
// planes one plane behind group s-1; the groups hand planes over through mbarriers in shared
// memory (full / empty per window slot, per u-ring slot, per partial-sum slot), so no CTA-wide
// barrier remains and the uneven stage sizes no longer serialise (K6: 7 evaluation passes per
// plane for 5.2 passes of work).
//
//   u ring (R slots, TMA)  --group 1-->  Y_2 window (3 slots)  --group 2-->  Y_3 ... --group L-->
//   u_new (global).  Each thread keeps its cells' z columns (previous and current plane) in
//   registers; the own cells' partial final sums W = u (+) beta_1 k_1 (+) ... travel through a
//   ring of NW shared-memory planes, updated by each group in stage order (R-17).
//
// Arithmetic: the stencil, reaction, stage values and partial sums are K6's expression trees
// (gs_rhs_q, add/mul without FMA), so the result equals K6's, K3's and the oracle's bit for bit.
#include <cudaTypedefs.h>

#include <type_traits>

#include "rk_device.cuh"
#include "rk_kernels.cuh"
#include "rk_tableau.h"

namespace rkb {

namespace {

#define K7INLINE __attribute__((always_inline))

constexpr int KX = 32;    // tile width
constexpr int KY = 16;    // tile height
constexpr int KNT = 512;  // threads (16 warps)

__host__ __device__ constexpr bool k7_chained(int S) {
    const Tableau T = tableau_of(S);
    if (T.s < 2 || T.s > 4 || T.err_order != 0) return false;
    for (int i = 0; i < T.s; ++i)
        for (int j = 0; j < i; ++j)
            if (rat_nz(T.a[i][j]) != (j == i - 1)) return false;
    return true;
}
__host__ __device__ constexpr bool k7_bnz(int S, int j) { return rat_nz(tableau_of(S).b[j]); }

template <int S>
struct KCfg {
    static constexpr int L = tableau_of(S).s;
    static constexpr int XL = (L + 1) / 2 * 2;  // left margin rounded up to even (16-byte TMA start)
    static constexpr int UW = KX + 2 * XL + 2;
    static constexpr int UH = KY + 2 * L;
    static constexpr int UBOX = UW * UH;
    static constexpr int UBYTES = 2 * UBOX * 8;
    static constexpr int USLOT = (UBYTES + 127) / 128 * 128;
    static constexpr int R = L + 1;             // u ring: planes in use (L) + 1 of prefetch
    static constexpr int NW = L + 1;            // partial-sum planes in flight
    // group s (1..L) evaluates k_s on the tile grown by r(s) = L-s cells
    static constexpr int r(int s) { return L - s; }
    static constexpr int gw(int s) { return KX + 2 * r(s); }
    static constexpr int gh(int s) { return KY + 2 * r(s); }
    static constexpr int ncell(int s) { return gw(s) * gh(s); }
    static constexpr int total() {
        int t = 0;
        for (int s = 1; s <= L; ++s) t += ncell(s);
        return t;
    }
    // warps per group: proportional to the cells, at least 1, 16 in total (largest remainder)
    static constexpr int warps(int s) {
        int w[5] = {0, 0, 0, 0, 0}, used = 0;
        for (int q = 1; q <= L; ++q) {
            w[q] = 16 * ncell(q) / total();
            if (w[q] < 1) w[q] = 1;
            used += w[q];
        }
        while (used < 16) {  // give the spare warps to the groups with the most cells per warp
            int best = 1;
            for (int q = 2; q <= L; ++q)
                if (ncell(q) * w[best] > ncell(best) * w[q]) best = q;
            ++w[best];
            ++used;
        }
        return w[s];
    }
    static constexpr int wfirst(int s) {
        int o = 0;
        for (int q = 1; q < s; ++q) o += warps(q);
        return o;
    }
    static constexpr int T(int s) { return 32 * warps(s); }
    static constexpr int M(int s) { return (ncell(s) + T(s) - 1) / T(s); }  // cells per thread
    // window of Y_s (s >= 2): the tile grown by hw(s) = L-s+1 cells, 3 planes
    static constexpr int hw(int s) { return L - s + 1; }
    static constexpr int ww(int s) { return KX + 2 * hw(s); }
    static constexpr int wbox(int s) { return ww(s) * (KY + 2 * hw(s)); }
    static constexpr int wslot(int s) { return (2 * wbox(s) * 8 + 127) / 128 * 128; }
    static constexpr int woff(int s) {  // s = 2..L
        int o = R * USLOT;
        for (int q = 2; q < s; ++q) o += 3 * wslot(q);
        return o;
    }
    static constexpr int WPLANE = 2 * KX * KY * 8;  // own-cell partial sums, one plane
    static constexpr int wsum_off = woff(L + 1);
    static constexpr int bar_off = wsum_off + NW * WPLANE;
    // barriers: u full[R], u empty[R], y full[L+1][3], y empty[L+1][3], w empty[NW]
    static constexpr int NBAR = 2 * R + 2 * 3 * (L + 1) + NW;
    static constexpr int smem = bar_off + NBAR * 8;
    static_assert(smem <= 227 * 1024, "K7 shared memory");
};

__device__ __forceinline__ uint32_t k7_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void k7_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(k7_smem(b)) : "memory");
}
__device__ __forceinline__ void k7_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "K7W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra K7W_%=;\n}" ::"r"(k7_smem(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ int k7_mod(int a, int n) {
    const int m = a % n;
    return m < 0 ? m + n : m;
}

// k = F(Y) at one cell with the centre value and the z neighbours in registers (K6's gs_rhs_q)
__device__ __forceinline__ void k7_rhs(const double* v0, int cs, int pitch, const double (&ctr)[2],
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
__global__ void __launch_bounds__(KNT, 1) gs_ws_kernel(const __grid_constant__ GsFusedArgs a) {
    using C = KCfg<S>;
    constexpr int L = C::L, XL = C::XL, UW = C::UW, UBOX = C::UBOX, R = C::R, NW = C::NW;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::bar_off);
    uint64_t* uFull = bars;
    uint64_t* uEmpty = bars + R;
    uint64_t* yFull = bars + 2 * R;               // [s][3], s = 2..L (index s)
    uint64_t* yEmpty = bars + 2 * R + 3 * (L + 1);
    uint64_t* wEmpty = bars + 2 * R + 6 * (L + 1);

    const GridGeom& G = a.geo;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int ntx = (G.nx + KX - 1) / KX;
    const int x0 = (int)(blockIdx.x % ntx) * KX, y0 = (int)(blockIdx.x / ntx) * KY;
    const int zb = (int)blockIdx.y * a.zchunk;
    const int ze = min(zb + a.zchunk, G.nzl);
    if (zb >= ze) return;
    const int nU = ze - zb + 2 * L;  // u planes zb-L .. ze+L-1 (sweep index i)

    auto uslot = [&](int i) K7INLINE -> double* { return reinterpret_cast<double*>(smem + (size_t)(i % R) * C::USLOT); };
    auto plane_of = [&](int i) K7INLINE -> int { return k7_mod(zb - L + i, G.nzl); };
    auto issue = [&](int i) K7INLINE {  // one thread
        uint64_t* b = &uFull[i % R];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(k7_smem(b)),
                     "r"((uint32_t)C::UBYTES)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(k7_smem(uslot(i))),
            "l"(reinterpret_cast<uint64_t>(&a.tm_u)), "r"(k7_smem(b)), "r"(x0 - XL), "r"(y0 - L + 1), "r"(0),
            "r"(plane_of(i))
            : "memory");
    };

    if (tid == 0) {
        for (int k = 0; k < R; ++k) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(k7_smem(&uFull[k])), "r"(1) : "memory");
            int cnt = 0;
            for (int s = 1; s < L; ++s) cnt += C::warps(s);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(k7_smem(&uEmpty[k])), "r"(cnt) : "memory");
        }
        for (int s = 2; s <= L; ++s)
            for (int k = 0; k < 3; ++k) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(k7_smem(&yFull[3 * s + k])),
                             "r"(C::warps(s - 1))
                             : "memory");
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(k7_smem(&yEmpty[3 * s + k])),
                             "r"(C::warps(s))
                             : "memory");
            }
        for (int k = 0; k < NW; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(k7_smem(&wEmpty[k])), "r"(C::warps(L))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // edge CTAs patch the periodic margin beyond the padded layout's 1-cell ring (group 1)
    bool anyfix = false;
    for (int p = tid; p < UBOX; p += KNT) {
        const int x = x0 - XL - 1 + p % UW, y = y0 - L + p / UW;
        const bool held = (x >= 0 && x < G.nx && y >= -1 && y <= G.ny) || (y >= 0 && y < G.ny && x >= -1 && x <= G.nx);
        anyfix = anyfix || !held;
    }
    const bool edge = __syncthreads_or(anyfix);
    if (tid == 0)
        for (int i = 0; i < (nU < R ? nU : R); ++i) issue(i);

    // ---- group s: k_s on its cells, one plane at a time ------------------------------------
    auto run = [&](auto sc) K7INLINE {
        constexpr int s = decltype(sc)::value;
        constexpr int TS = C::T(s), MS = C::M(s), GW = C::gw(s), NC = C::ncell(s), RS = C::r(s);
        const int j = tid - 32 * C::wfirst(s);  // thread index within the group
        const bool lane0 = (tid & 31) == 0;
        // the group's cells m = j + k*TS of the grown tile (gx, gy relative to the tile origin)
        auto cell_xy = [&](int k, int& gx, int& gy) K7INLINE {
            const int m = j + k * TS;
            gx = m % GW - RS;
            gy = m / GW - RS;
        };
        // centre-value offset of a cell in the source plane (u box for s = 1, window s else)
        auto src_off = [&](int gx, int gy) K7INLINE -> int {
            if constexpr (s == 1) return (gx + XL + 1) + (gy + L) * UW;
            else return (gx + C::hw(s)) + (gy + C::hw(s)) * C::ww(s);
        };
        // Window s holds the planes group s-1 produces, from plane s-1 on: plane i is its
        // (i-s+1)-th, in slot (i-s+1) % 3, completing phase (i-s+1) / 3 of that slot's barriers.
        auto src_plane = [&](int i) K7INLINE -> const double* {
            if constexpr (s == 1) return uslot(i);
            else return reinterpret_cast<const double*>(smem + C::woff(s) + (size_t)((i - s + 1) % 3) * C::wslot(s));
        };
        constexpr int CS = s == 1 ? UBOX : C::wbox(s);
        constexpr int PITCH = s == 1 ? UW : C::ww(s);
        auto wait_src = [&](int i) K7INLINE {  // plane i of Y_s is ready
            if constexpr (s == 1) {
                k7_wait(&uFull[i % R], (uint32_t)((i / R) & 1));
            } else {
                const int q = i - s + 1;
                k7_wait(&yFull[3 * s + q % 3], (uint32_t)((q / 3) & 1));
            }
        };
        auto release_src = [&](int i) K7INLINE {  // this warp no longer reads plane i of Y_s
            __syncwarp();
            if (lane0) {
                if constexpr (s == 1) k7_arrive(&uEmpty[i % R]);
                else k7_arrive(&yEmpty[3 * s + (i - s + 1) % 3]);
            }
        };
        auto patch = [&](int i) K7INLINE {  // group 1, edge CTAs: periodic margin of u plane i
            double* U = uslot(i);
            const int64_t zo = (int64_t)plane_of(i) * G.ps;
            for (int p = j; p < UBOX; p += TS) {
                const int x = x0 - XL - 1 + p % UW, y = y0 - L + p / UW;
                const bool held = (x >= 0 && x < G.nx && y >= -1 && y <= G.ny) ||
                                  (y >= 0 && y < G.ny && x >= -1 && x <= G.nx);
                if (!held) {
                    const int64_t o = (int64_t)(k7_mod(y, G.ny) + 1) * G.P + (k7_mod(x, G.nx) + 1);
                    U[p] = a.u[zo + o];
                    U[UBOX + p] = a.u[zo + G.cs + o];
                }
            }
            asm volatile("bar.sync 1, %0;" ::"r"(TS) : "memory");  // group 1 only
        };

        const int first = s, last = nU - s;  // centre planes [first, last)
        // non-read u planes of groups 2..L-1 (never reused beyond nU - R: no arrival needed)
        if constexpr (s >= 2 && s < L) {
            for (int i = 0; i < s; ++i) {
                __syncwarp();
                if (lane0) k7_arrive(&uEmpty[i % R]);
            }
        }
        // prologue: planes first-1 and first into the z queue
        double zq0[MS][2], zq1[MS][2];  // Y_s at planes ic-1, ic (own cells of this thread)
        wait_src(first - 1);
        if constexpr (s == 1) {
            if (edge) patch(first - 1);
        }
        {
            const double* P0 = src_plane(first - 1);
#pragma unroll
            for (int k = 0; k < MS; ++k) {
                int gx, gy;
                cell_xy(k, gx, gy);
                const bool on = j + k * TS < NC;
                const int o = on ? src_off(gx, gy) : 0;
                zq0[k][0] = P0[o];
                zq0[k][1] = P0[CS + o];
            }
        }
        wait_src(first);
        if constexpr (s == 1) {
            if (edge) patch(first);
        }
        {
            const double* P1 = src_plane(first);
#pragma unroll
            for (int k = 0; k < MS; ++k) {
                int gx, gy;
                cell_xy(k, gx, gy);
                const bool on = j + k * TS < NC;
                const int o = on ? src_off(gx, gy) : 0;
                zq1[k][0] = P1[o];
                zq1[k][1] = P1[CS + o];
            }
        }
        release_src(first - 1);

        for (int ic = first; ic < last; ++ic) {
            if constexpr (s == 1) {
                // producer: u plane ic+2 (needed at iteration ic+1) into the slot of plane
                // ic+2-R = ic-L+1, which every reader has released by now or soon: group 1 at
                // plane ic-L+1 < ic, group s >= 2 there needs only group 1's planes <= ic-1
                const int q = ic + 2;
                if (tid == 0 && q >= R && q < nU) {
                    k7_wait(&uEmpty[(q - R) % R], (uint32_t)(((q - R) / R) & 1));
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(q);
                }
            }
            wait_src(ic + 1);
            if constexpr (s == 1) {
                if (edge) patch(ic + 1);
            }
            if constexpr (s >= 2 && s < L) k7_wait(&uFull[ic % R], (uint32_t)((ic / R) & 1));
            const bool outp = ic >= L && ic < nU - L;  // an output plane: partial sums kept
            const int qy = ic - s;                      // plane ic's index in window s+1
            const int qw = ic - L;                      // ... in the partial-sum ring
            if constexpr (s < L) {  // the Y_{s+1} slot was released by group s+1 (plane ic-3)
                if (qy >= 3) k7_wait(&yEmpty[3 * (s + 1) + qy % 3], (uint32_t)(((qy - 3) / 3) & 1));
            }
            if constexpr (s == 1) {  // the partial-sum slot was stored by group L (plane ic-NW)
                if (outp && qw >= NW) k7_wait(&wEmpty[qw % NW], (uint32_t)(((qw - NW) / NW) & 1));
            }
            const double* Pc = src_plane(ic);
            const double* Pn = src_plane(ic + 1);
            const double* U = uslot(ic);
            double* Yn = nullptr;
            if constexpr (s < L)
                Yn = reinterpret_cast<double*>(smem + C::woff(s + 1) + (size_t)(qy % 3) * C::wslot(s + 1));
            double* Wp = reinterpret_cast<double*>(smem + C::wsum_off + (size_t)((qw + NW) % NW) * C::WPLANE);
#pragma unroll
            for (int k = 0; k < MS; ++k) {
                int gx, gy;
                cell_xy(k, gx, gy);
                const bool on = j + k * TS < NC;
                const int o = on ? src_off(gx, gy) : 0;
                double zn[2];
                zn[0] = Pn[o];
                zn[1] = Pn[CS + o];
                if (on) {
                    double f[2];
                    k7_rhs(Pc + o, CS, PITCH, zq1[k], zq0[k], zn, a, f);
                    if constexpr (s < L) {  // Y_{s+1} = u (+) g_s k_s on the tile grown by L-s
                        const int uo = (gx + XL + 1) + (gy + L) * UW;
                        const int yo = (gx + C::hw(s + 1)) + (gy + C::hw(s + 1)) * C::ww(s + 1);
#pragma unroll
                        for (int c = 0; c < 2; ++c)
                            Yn[c * C::wbox(s + 1) + yo] = add(s == 1 ? zq1[k][c] : U[c * UBOX + uo], mul(a.g[s], f[c]));
                    }
                    if (outp && gx >= 0 && gx < KX && gy >= 0 && gy < KY) {  // own cell: W
                        const int wo = gx + gy * KX;
#pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            double w = s == 1 ? zq1[k][c] : Wp[c * KX * KY + wo];
                            if constexpr (k7_bnz(S, s - 1)) w = add(w, mul(a.beta[s - 1], f[c]));
                            if constexpr (s < L) {
                                Wp[c * KX * KY + wo] = w;
                            } else if (x0 + gx < G.nx && y0 + gy < G.ny) {
                                const int x = x0 + gx, y = y0 + gy;
                                const int z = zb - L + ic;
                                double* p = a.out + (int64_t)z * G.ps + c * G.cs + (int64_t)(y + 1) * G.P + (x + 1);
                                p[0] = w;
                                if (x == 0) p[G.nx] = w;
                                if (x == G.nx - 1) p[-G.nx] = w;
                                if (y == 0) p[(int64_t)G.ny * G.P] = w;
                                if (y == G.ny - 1) p[-(int64_t)G.ny * G.P] = w;
                            }
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    zq0[k][c] = zq1[k][c];
                    zq1[k][c] = zn[c];
                }
            }
            __syncwarp();
            if (lane0) {
                if constexpr (s < L) k7_arrive(&yFull[3 * (s + 1) + qy % 3]);  // Y_{s+1} plane ic
                if constexpr (s == L) {
                    if (outp) k7_arrive(&wEmpty[qw % NW]);
                }
                if constexpr (s >= 2 && s < L) k7_arrive(&uEmpty[ic % R]);
            }
            release_src(ic);
        }
        (void)XL;
    };

    // dispatch the warps to their groups (warp-uniform)
    if (warp < C::wfirst(2)) run(std::integral_constant<int, 1>{});
    else if constexpr (L >= 3) {
        if (warp < C::wfirst(3)) run(std::integral_constant<int, 2>{});
        else if constexpr (L >= 4) {
            if (warp < C::wfirst(4)) run(std::integral_constant<int, 3>{});
            else run(std::integral_constant<int, 4>{});
        } else {
            run(std::integral_constant<int, 3>{});
        }
    } else {
        run(std::integral_constant<int, 2>{});
    }
}

template <int S>
cudaError_t launch_ws_t(const GsFusedArgs& a, cudaStream_t st) {
    static_assert(k7_chained(S), "K7 needs a chained-stage tableau");
    constexpr int bytes = KCfg<S>::smem;
    static std::atomic<unsigned long long> configured{0};
    if (cudaError_t e = smem_attr_once(configured, gs_ws_kernel<S>, bytes); e != cudaSuccess) return e;
    const int ntx = (a.geo.nx + KX - 1) / KX, nty = (a.geo.ny + KY - 1) / KY;
    const int nch = (a.geo.nzl + a.zchunk - 1) / a.zchunk;
    gs_ws_kernel<S><<<dim3((unsigned)(ntx * nty), (unsigned)nch), KNT, bytes, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gs_fused_ws(int scheme, const GsFusedArgs& a, cudaStream_t st) {
    if (a.zchunk <= 0) return cudaErrorInvalidValue;
    switch (scheme) {
    case 1: return launch_ws_t<1>(a, st);  // RK4
    case 5: return launch_ws_t<5>(a, st);  // explicit midpoint
    case 6: return launch_ws_t<6>(a, st);  // modified midpoint (Gragg)
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace rkb
