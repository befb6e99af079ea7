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
//
// Data movement (sm_100a): a CTA owns a 32x8 tile of the xy plane and sweeps a chunk of z
// planes.  For every plane, one elected thread issues one 4D TMA box load per input array
// (u and each k_j: 34x10 cells x 2 components, the tile plus its periodic ring thanks to
// the padded layout) into an R-deep shared-memory ring guarded by mbarriers, R-1 planes
// ahead of the plane being computed, so HBM sees a deep, register-free stream of loads.
// Each plane's Y is formed once from the staged raw tiles into a double-buffered Y tile;
// the own column keeps Y(z-1), Y(z), Y(z+1) in registers (register queue along z).  One
// __syncthreads per plane.  Periodic x/y wrap is in the padded layout; z neighbours come
// from ghost planes (multi-GPU, filled by NCCL) or by wrapping inside the slab (one GPU).
//
// Arithmetic follows DESIGN.md R-17 bit for bit (no FMA: __dadd_rn / __dmul_rn), so the
// results equal the oracle's for any tile/chunk/GPU decomposition.
#include <cudaTypedefs.h>

#include "rk_device.cuh"
#include "rk_kernels.cuh"

namespace rkb {

namespace {

constexpr int TX = 32;            // tile width  (one warp per row)
constexpr int TY = 8;             // tile height (8 warps)
constexpr int NT = TX * TY;
constexpr int BW = TX + 2, BH = TY + 2;
constexpr int BOX = BW * BH;                  // cells per component in one TMA box
constexpr int BOX_BYTES = 2 * BOX * 8;        // one array, both components (5440 B)
constexpr int ARR_BYTES = (BOX_BYTES + 127) / 128 * 128;  // 128-B aligned slot stride
constexpr int ARR_DBL = ARR_BYTES / 8;
constexpr int NHALO = BOX - NT;               // ring positions of the box (84)
static_assert(NHALO <= NT, "one ring position per thread");

__host__ __device__ constexpr int ring_depth(int ns) { return ns <= 3 ? 4 : 3; }
__host__ __device__ constexpr int smem_bytes(int ns) {
    return ring_depth(ns) * (ns + 1) * ARR_BYTES + 2 * ARR_BYTES + ring_depth(ns) * 8;
}

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

__device__ __forceinline__ bool plane_is_ghost(const GsStageArgs& a, int p) {
    return (p < 0 && a.has_glo) || (p >= a.geo.nzl && a.has_ghi);
}

// Y = u (+) g_s (x) k_s over slots with g_s != 0, left to right (R-17); a ghost plane holds
// Y itself.  r points at component c, box position pos, of array 0 of a ring slot.
template <int NS>
__device__ __forceinline__ double y_at(const GsStageArgs& a, const double* r, bool ghost) {
    double v = r[0];
    if (!ghost) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
            if (a.g[s] != 0.0) v = add(v, mul(a.g[s], r[(s + 1) * ARR_DBL]));
    }
    return v;
}

// Per-cell partial sums the epilogue completes with the new k_i (bitwise identical to the
// full left-to-right sums because j = i is always the last term).
struct EState {
    double w[2];  // u (+) sum beta_j k_j
    double e[2];  // sum delta_j k_j (first term not added to 0)
    double d[2];  // atol (+) rtol (x) (|u| (+) dt (x) |k1|)
};

template <int NS, int EPI>
__device__ __forceinline__ void make_estate(const GsStageArgs& a, const double* slot, int pos,
                                            EState& es) {
    constexpr bool FIN = (EPI == EPI_FINAL || EPI == EPI_FINAL_ERR);
    constexpr bool ERR = (EPI == EPI_FINAL_ERR || EPI == EPI_FSAL_ERR);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const double* r = slot + c * BOX + pos;
        const double u = r[0];
        if constexpr (FIN) {
            double w = u;
#pragma unroll
            for (int s = 0; s < NS; ++s)
                if (a.beta[s] != 0.0) w = add(w, mul(a.beta[s], r[(s + 1) * ARR_DBL]));
            es.w[c] = w;
        }
        if constexpr (ERR) {
            double e = 0.0;
            bool first = true;
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                if (a.delta[s] == 0.0) continue;
                const double t = mul(a.delta[s], r[(s + 1) * ARR_DBL]);
                e = first ? t : add(e, t);
                first = false;
            }
            es.e[c] = e;
            const double k1 = NS > 0 ? r[ARR_DBL] : 0.0;  // slot 0 holds k1 in error stages
            es.d[c] = add(a.atol, mul(a.rtol, add(fabs(u), mul(a.dt, fabs(k1)))));
        }
    }
}

// Store one cell of a padded array and its periodic ring copies (corners are never read).
__device__ __forceinline__ void store_cell(double* out, const GridGeom& g, int64_t off, int x, int y,
                                           double v) {
    out[off + (int64_t)(y + 1) * g.P + (x + 1)] = v;
    if (x == 0) out[off + (int64_t)(y + 1) * g.P + (g.nx + 1)] = v;
    if (x == g.nx - 1) out[off + (int64_t)(y + 1) * g.P] = v;
    if (y == 0) out[off + (int64_t)(g.ny + 1) * g.P + (x + 1)] = v;
    if (y == g.ny - 1) out[off + (x + 1)] = v;
}

template <int NS, int EPI>
__global__ void __launch_bounds__(NT, 2) gs_stage_kernel(const __grid_constant__ GsStageArgs a) {
    constexpr int R = ring_depth(NS);
    constexpr int NA = NS + 1;
    constexpr bool FIN = (EPI == EPI_FINAL || EPI == EPI_FINAL_ERR);
    constexpr bool ERR = (EPI == EPI_FINAL_ERR || EPI == EPI_FSAL_ERR);
    extern __shared__ __align__(128) unsigned char smem[];
    double* raw = reinterpret_cast<double*>(smem);                          // [R][NA][2][BH][BW]
    double* sY = reinterpret_cast<double*>(smem + R * NA * ARR_BYTES);      // [2][2][BH][BW]
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + R * NA * ARR_BYTES + 2 * ARR_BYTES);

    const GridGeom& G = a.geo;
    const int tid = threadIdx.x;
    const int ntx = (G.nx + TX - 1) / TX;
    const int x0 = (int)(blockIdx.x % ntx) * TX, y0 = (int)(blockIdx.x / ntx) * TY;
    const int w = min(TX, G.nx - x0), hg = min(TY, G.ny - y0);

    int zb, ze;
    if (a.zmode == 0) {
        zb = a.z_lo + (int)blockIdx.y * a.zchunk;
        ze = min(zb + a.zchunk, a.z_hi);
    } else {
        zb = blockIdx.y == 0 ? 0 : G.nzl - 1;
        ze = zb + 1;
    }
    if (zb >= ze) return;  // CTA-uniform, before any barrier
    const int nplanes = ze - zb + 2;  // planes zb-1 .. ze, plane i is global zb-1+i

    const int lx = tid % TX, ly = tid / TX;
    const bool own = (lx < w) && (ly < hg);
    const int pos_own = (ly + 1) * BW + (lx + 1);
    // ring position handled by this thread (all 84 box positions outside the tile)
    const bool hal = tid < NHALO;
    int pos_h = 0;
    if (tid < BW) pos_h = tid;                                  // row 0
    else if (tid < 2 * BW) pos_h = (BH - 1) * BW + (tid - BW);  // row BH-1
    else if (tid < 2 * BW + TY) pos_h = (tid - 2 * BW + 1) * BW;             // col 0
    else if (tid < NHALO) pos_h = (tid - 2 * BW - TY + 1) * BW + (BW - 1);  // col BW-1

    auto issue = [&](int i) {  // thread 0 only
        const int p = zb - 1 + i, s = i % R;
        double* dst = raw + (size_t)s * NA * ARR_DBL;
        if (plane_is_ghost(a, p)) {
            mbar_expect_tx(&bar[s], BOX_BYTES);
            tma_load_4d(dst, p < 0 ? &a.tm_glo : &a.tm_ghi, &bar[s], x0, y0, 0, 0);
        } else {
            const int q = p < 0 ? p + G.nzl : (p >= G.nzl ? p - G.nzl : p);
            mbar_expect_tx(&bar[s], NA * BOX_BYTES);
            tma_load_4d(dst, &a.tm_u, &bar[s], x0, y0, 0, q);
#pragma unroll
            for (int k = 0; k < NS; ++k)
                tma_load_4d(dst + (k + 1) * ARR_DBL, &a.tm_k[k], &bar[s], x0, y0, 0, q);
        }
    };
    auto slot_of = [&](int i) -> const double* { return raw + (size_t)(i % R) * NA * ARR_DBL; };
    auto wait_plane = [&](int i) { mbar_wait(&bar[i % R], (uint32_t)((i / R) & 1)); };

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

    double Ym[2] = {0.0, 0.0}, Yc[2] = {0.0, 0.0}, Yp[2] = {0.0, 0.0};
    EState Ec{}, En{};
    unsigned long long rmax = 0ull;

    // ---- prologue: plane zb-1 (own column only), plane zb (tile + ring) -----------------
    {
        wait_plane(0);
        const double* s0 = slot_of(0);
        const bool gh = plane_is_ghost(a, zb - 1);
        // every thread forms Y at its tile position, valid or not: for a partial tile
        // (w < TX or hg < TY) the periodic ring sits inside the box at column w+1 / row hg+1
        Ym[0] = y_at<NS>(a, s0 + pos_own, gh);
        Ym[1] = y_at<NS>(a, s0 + BOX + pos_own, gh);
        wait_plane(1);
        const double* s1 = slot_of(1);
        Yc[0] = y_at<NS>(a, s1 + pos_own, false);
        Yc[1] = y_at<NS>(a, s1 + BOX + pos_own, false);
        sY[pos_own] = Yc[0];
        sY[BOX + pos_own] = Yc[1];
        if (own) make_estate<NS, EPI>(a, s1, pos_own, Ec);
        if (hal) {
            sY[pos_h] = y_at<NS>(a, s1 + pos_h, false);
            sY[BOX + pos_h] = y_at<NS>(a, s1 + BOX + pos_h, false);
        }
        __syncthreads();
        if (tid == 0) {
            if (R < nplanes) issue(R);
            if (R + 1 < nplanes) issue(R + 1);
        }
    }

    for (int z = zb; z < ze; ++z) {
        const int i = z - zb + 2;  // plane z+1
        const int b = (z - zb) & 1;
        const bool more = z + 1 < ze;  // plane z+1 is an output plane of this CTA
        double* yc = sY + b * 2 * BOX;
        double* yn = sY + (b ^ 1) * 2 * BOX;
        // [A] plane z+1 from the ring
        wait_plane(i);
        const double* si = slot_of(i);
        const bool gh = plane_is_ghost(a, z + 1);
        Yp[0] = y_at<NS>(a, si + pos_own, gh);
        Yp[1] = y_at<NS>(a, si + BOX + pos_own, gh);
        if (more) {
            yn[pos_own] = Yp[0];
            yn[BOX + pos_own] = Yp[1];
            if (own) make_estate<NS, EPI>(a, si, pos_own, En);
        }
        if (hal && more) {
            yn[pos_h] = y_at<NS>(a, si + pos_h, false);
            yn[BOX + pos_h] = y_at<NS>(a, si + BOX + pos_h, false);
        }
        // [C] stencil + reaction + epilogue at plane z
        if (own) {
            double L[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const double* v = yc + c * BOX + pos_own;
                const double ctr = Yc[c];
                double s = add(sub(v[-1], ctr), sub(v[1], ctr));
                s = add(s, add(sub(v[-BW], ctr), sub(v[BW], ctr)));
                s = add(s, add(sub(Ym[c], ctr), sub(Yp[c], ctr)));
                L[c] = mul(s, a.inv_h2);
            }
            const double C0 = Yc[0], C1 = Yc[1];
            const double r = mul(mul(C0, C1), C1);
            double f[2];
            f[0] = sub(add(sub(mul(a.d1, L[0]), r), a.F), mul(a.F, C0));
            f[1] = sub(add(mul(a.d2, L[1]), r), mul(a.FK, C1));
            const int x = x0 + lx, y = y0 + ly;
            const int64_t qo = (int64_t)z * G.ps;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int64_t off = qo + c * G.cs;
                if constexpr (EPI == EPI_K || EPI == EPI_FSAL_ERR) store_cell(a.out_k, G, off, x, y, f[c]);
                if constexpr (FIN) {
                    const double wv = a.beta_new != 0.0 ? add(Ec.w[c], mul(a.beta_new, f[c])) : Ec.w[c];
                    store_cell(a.out_u, G, off, x, y, wv);
                }
                if constexpr (EPI == EPI_FSAL_ERR) store_cell(a.out_u, G, off, x, y, Yc[c]);
                if constexpr (ERR) {
                    bool has_prev = false;
#pragma unroll
                    for (int s2 = 0; s2 < NS; ++s2) has_prev |= (a.delta[s2] != 0.0);
                    double e = Ec.e[c];
                    if (a.delta_new != 0.0) {
                        const double t = mul(a.delta_new, f[c]);
                        e = has_prev ? add(e, t) : t;
                    }
                    const unsigned long long rb = ratio_bits(fabs(e) / Ec.d[c]);
                    rmax = rb > rmax ? rb : rmax;
                }
            }
        }
        Ym[0] = Yc[0]; Ym[1] = Yc[1];
        Yc[0] = Yp[0]; Yc[1] = Yp[1];
        Ec = En;
        __syncthreads();  // Y(z+1) tile complete; ring slot of plane z+1 free
        if (tid == 0 && i + R < nplanes) issue(i + R);
    }
    if constexpr (ERR) block_max_to_global(rmax, a.errmax);
}

// ---- halo-plane pack and ring fill -------------------------------------------------------
template <int NS>
__global__ void __launch_bounds__(256) gs_pack_kernel(const GsStageArgs a, double* __restrict__ send) {
    const int64_t ps = a.geo.ps, total = 2 * ps;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sel = e / ps, rest = e - sel * ps;
        const int64_t base = (sel ? (int64_t)(a.geo.nzl - 1) : 0) * ps + rest;
        double v = __ldg(a.u + base);
#pragma unroll
        for (int s = 0; s < NS; ++s)
            if (a.g[s] != 0.0) v = add(v, mul(a.g[s], __ldg(a.k[s] + base)));
        send[e] = v;
    }
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

template <int NS, int EPI>
cudaError_t launch_one(const GsStageArgs& a, dim3 grid, cudaStream_t st) {
    static bool configured = false;
    constexpr int bytes = smem_bytes(NS);
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(gs_stage_kernel<NS, EPI>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    gs_stage_kernel<NS, EPI><<<grid, NT, bytes, st>>>(a);
    return cudaGetLastError();
}

template <int NS>
cudaError_t launch_ns(int epi, const GsStageArgs& a, dim3 grid, cudaStream_t st) {
    switch (epi) {
    case EPI_K: return launch_one<NS, EPI_K>(a, grid, st);
    case EPI_FINAL: return launch_one<NS, EPI_FINAL>(a, grid, st);
    case EPI_FINAL_ERR: return launch_one<NS, EPI_FINAL_ERR>(a, grid, st);
    case EPI_FSAL_ERR: return launch_one<NS, EPI_FSAL_ERR>(a, grid, st);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace

void gs_tile_dims(int* tx, int* ty) {
    *tx = TX;
    *ty = TY;
}

cudaError_t encode_grid_map(CUtensorMap* m, const double* base, const GridGeom& g, int nplanes) {
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
    const cuuint32_t box[4] = {BW, BH, 2, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_gs_stage(int epi, const GsStageArgs& a, cudaStream_t st, int* nlaunch) {
    const int ntx = (a.geo.nx + TX - 1) / TX, nty = (a.geo.ny + TY - 1) / TY;
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
    if (nlaunch) ++*nlaunch;
    switch (a.nslots) {
    case 0: return launch_ns<0>(epi, a, grid, st);
    case 1: return launch_ns<1>(epi, a, grid, st);
    case 2: return launch_ns<2>(epi, a, grid, st);
    case 3: return launch_ns<3>(epi, a, grid, st);
    case 4: return launch_ns<4>(epi, a, grid, st);
    case 5: return launch_ns<5>(epi, a, grid, st);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_gs_pack(const GsStageArgs& a, double* send, cudaStream_t st) {
    const int64_t total = 2 * a.geo.ps;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    switch (a.nslots) {
    case 0: gs_pack_kernel<0><<<(unsigned)blocks, 256, 0, st>>>(a, send); break;
    case 1: gs_pack_kernel<1><<<(unsigned)blocks, 256, 0, st>>>(a, send); break;
    case 2: gs_pack_kernel<2><<<(unsigned)blocks, 256, 0, st>>>(a, send); break;
    case 3: gs_pack_kernel<3><<<(unsigned)blocks, 256, 0, st>>>(a, send); break;
    case 4: gs_pack_kernel<4><<<(unsigned)blocks, 256, 0, st>>>(a, send); break;
    case 5: gs_pack_kernel<5><<<(unsigned)blocks, 256, 0, st>>>(a, send); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_fill_ring(double* p, const GridGeom& g, int nslices, cudaStream_t st) {
    const int n = g.nx > g.ny ? g.nx : g.ny;
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)nslices);
    fill_ring_kernel<<<grid, 256, 0, st>>>(p, g, nslices);
    return cudaGetLastError();
}

}  // namespace rkb
