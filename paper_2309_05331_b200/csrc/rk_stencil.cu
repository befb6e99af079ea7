// rk_stencil.cu — K3: fused Gray–Scott stage kernel, and the halo-plane pack.
//
// One launch evaluates one Runge–Kutta stage i of the 3D Gray–Scott system (Listing 2,
// P:L169-170; R-1..R-3) over a z-slab:
//   Y_i = u + sum_{j<i} (dt a_ij) k_j      computed on the fly for every loaded cell
//                                          (Odeint's scale_sum algebra, fused
//                                          into the stencil's loads: Y_i never hits HBM)
//   k_i = d*Lap(Y_i) + reaction(Y_i)       7-point periodic stencil + reaction terms
//   epilogue: store k_i, or u_new = u + sum_j (dt b_j) k_j, and/or the embedded error
//             ratio with a warp-shuffle / block max (P:L42, P:L135 for_each_norm).
//
// Decomposition: a CTA owns a TX x TY tile of the xy plane and sweeps a chunk of z planes.
// Per plane it stages Y on the tile plus its 1-cell xy halo in shared memory (double
// buffered, one __syncthreads per plane) and keeps the own column's Y(z-1), Y(z), Y(z+1)
// in registers (register queue along the sweep axis).  Raw inputs (u, k_j) of plane z+2
// are loaded into registers while plane z is being computed (one-plane software
// pipeline), so each HBM byte is read once; halo cells are re-read from L2.
// Periodic x/y wrap is by index arithmetic; the z neighbours of the slab come from ghost
// planes (multi-GPU, filled by NCCL) or by wrapping inside the slab (one GPU).
//
// Every arithmetic expression follows DESIGN.md R-17 bit for bit (no FMA: __dadd_rn /
// __dmul_rn), so results equal the oracle's for any tile/chunk/GPU decomposition.
#include "rk_device.cuh"
#include "rk_kernels.cuh"

namespace rkb {

namespace {

constexpr int TX = 32;  // tile width  (one warp per row, 8 B per lane: 256 B coalesced)
constexpr int TY = 8;   // tile height (8 warps)
constexpr int NT = TX * TY;
static_assert(NT >= 2 * TX + 2 * TY, "halo items need one thread each");

template <int NS>
struct Raw {
    double u[2];
    double k[NS > 0 ? NS : 1][2];
};

// Load the raw inputs of one cell (offset o inside a plane) of plane p in [-1, nzl].
// ghost: the plane is a received Y plane, stored in r.u directly.
template <int NS, bool HALO>
__device__ __forceinline__ void load_cell(const GsStageArgs& a, int p, int64_t o, int64_t cs,
                                          int64_t ps, Raw<NS>& r) {
    const double* gh = nullptr;
    if (p < 0 && a.ghost_lo) gh = a.ghost_lo;
    if (p >= a.nzl && a.ghost_hi) gh = a.ghost_hi;
    if (gh) {
        r.u[0] = __ldg(gh + o);
        r.u[1] = __ldg(gh + cs + o);
        return;
    }
    const int q = p < 0 ? p + a.nzl : (p >= a.nzl ? p - a.nzl : p);
    const int64_t base = (int64_t)q * ps + o;
    r.u[0] = __ldg(a.u + base);
    r.u[1] = __ldg(a.u + base + cs);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        if (HALO && a.g[s] == 0.0) continue;  // uniform: slot not part of Y
        r.k[s][0] = __ldg(a.k[s] + base);
        r.k[s][1] = __ldg(a.k[s] + base + cs);
    }
}

__device__ __forceinline__ bool is_ghost(const GsStageArgs& a, int p) {
    return (p < 0 && a.ghost_lo) || (p >= a.nzl && a.ghost_hi);
}

// Y = u (+) g_s (x) k_s over slots with g_s != 0, left to right (R-17).
template <int NS>
__device__ __forceinline__ void combine_y(const GsStageArgs& a, bool ghost, const Raw<NS>& r,
                                          double (&y)[2]) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        double v = r.u[c];
        if (!ghost) {
#pragma unroll
            for (int s = 0; s < NS; ++s)
                if (a.g[s] != 0.0) v = add(v, mul(a.g[s], r.k[s][c]));
        }
        y[c] = v;
    }
}

// Per-cell partial sums that the epilogue completes with the new k_i (bitwise identical to
// the full left-to-right sums because j = i is always the last term).
struct EState {
    double w[2];  // u (+) sum beta_j k_j
    double e[2];  // sum delta_j k_j (first term not added to 0)
    double d[2];  // atol (+) rtol (x) (|u| (+) dt (x) |k1|)
};

template <int NS, int EPI>
__device__ __forceinline__ void make_estate(const GsStageArgs& a, const Raw<NS>& r, EState& es) {
    constexpr bool FIN = (EPI == EPI_FINAL || EPI == EPI_FINAL_ERR);
    constexpr bool ERR = (EPI == EPI_FINAL_ERR || EPI == EPI_FSAL_ERR);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        if constexpr (FIN) {
            double w = r.u[c];
#pragma unroll
            for (int s = 0; s < NS; ++s)
                if (a.beta[s] != 0.0) w = add(w, mul(a.beta[s], r.k[s][c]));
            es.w[c] = w;
        }
        if constexpr (ERR) {
            double e = 0.0;
            bool first = true;
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                if (a.delta[s] == 0.0) continue;
                const double t = mul(a.delta[s], r.k[s][c]);
                e = first ? t : add(e, t);
                first = false;
            }
            es.e[c] = e;
            const double k1 = NS > 0 ? r.k[0][c] : 0.0;  // slot 0 holds k1 in error stages
            es.d[c] = add(a.atol, mul(a.rtol, add(fabs(r.u[c]), mul(a.dt, fabs(k1)))));
        }
    }
}

template <int NS, int EPI>
__global__ void __launch_bounds__(NT, 2) gs_stage_kernel(const GsStageArgs a) {
    constexpr int SW = TX + 2, SH = TY + 2;
    constexpr bool FIN = (EPI == EPI_FINAL || EPI == EPI_FINAL_ERR);
    constexpr bool ERR = (EPI == EPI_FINAL_ERR || EPI == EPI_FSAL_ERR);
    __shared__ double sY[2][2][SH][SW];

    const int tid = threadIdx.x;
    const int ntx = (a.nx + TX - 1) / TX;
    const int x0 = (int)(blockIdx.x % ntx) * TX, y0 = (int)(blockIdx.x / ntx) * TY;
    const int w = min(TX, a.nx - x0), hg = min(TY, a.ny - y0);

    int zb, ze;
    if (a.zmode == 0) {
        zb = a.z_lo + (int)blockIdx.y * a.zchunk;
        ze = min(zb + a.zchunk, a.z_hi);
    } else {
        zb = blockIdx.y == 0 ? 0 : a.nzl - 1;
        ze = zb + 1;
    }
    if (zb >= ze) return;  // CTA-uniform, before any barrier

    const int64_t cs = (int64_t)a.nx * a.ny;  // component stride
    const int64_t ps = 2 * cs;                // plane stride

    // own cell
    const int lx = tid % TX, ly = tid / TX;
    const bool own = (lx < w) && (ly < hg);
    const int64_t o_own = (int64_t)(y0 + ly) * a.nx + (x0 + lx);

    // halo item: rows y0-1 / y0+hg, columns x0-1 / x0+w (corners are not needed)
    bool hal = false;
    int hr = 0, hc = 0;
    int64_t o_hal = 0;
    if (tid < TX) {
        hal = tid < w;
        o_hal = (int64_t)((y0 - 1 + a.ny) % a.ny) * a.nx + (x0 + tid);
        hr = 0; hc = tid + 1;
    } else if (tid < 2 * TX) {
        const int t = tid - TX;
        hal = t < w;
        o_hal = (int64_t)((y0 + hg) % a.ny) * a.nx + (x0 + t);
        hr = hg + 1; hc = t + 1;
    } else if (tid < 2 * TX + TY) {
        const int t = tid - 2 * TX;
        hal = t < hg;
        o_hal = (int64_t)(y0 + t) * a.nx + ((x0 - 1 + a.nx) % a.nx);
        hr = t + 1; hc = 0;
    } else if (tid < 2 * TX + 2 * TY) {
        const int t = tid - 2 * TX - TY;
        hal = t < hg;
        o_hal = (int64_t)(y0 + t) * a.nx + ((x0 + w) % a.nx);
        hr = t + 1; hc = w + 1;
    }

    Raw<NS> P, H;  // raw inputs in flight: own cell, halo cell
    double Ym[2] = {0.0, 0.0}, Yc[2] = {0.0, 0.0}, Yp[2] = {0.0, 0.0};
    EState Ec{}, En{};
    unsigned long long rmax = 0ull;

    // ---- prologue: Y(zb-1) own column; Y(zb) tile + halo; issue plane zb+1 -------------
    if (own) {
        load_cell<NS, false>(a, zb - 1, o_own, cs, ps, P);
        combine_y<NS>(a, is_ghost(a, zb - 1), P, Ym);
        load_cell<NS, false>(a, zb, o_own, cs, ps, P);
    }
    if (hal) load_cell<NS, true>(a, zb, o_hal, cs, ps, H);
    if (own) {
        combine_y<NS>(a, false, P, Yc);
        sY[0][0][ly + 1][lx + 1] = Yc[0];
        sY[0][1][ly + 1][lx + 1] = Yc[1];
        make_estate<NS, EPI>(a, P, Ec);
    }
    if (hal) {
        double y[2];
        combine_y<NS>(a, false, H, y);
        sY[0][0][hr][hc] = y[0];
        sY[0][1][hr][hc] = y[1];
    }
    if (own) load_cell<NS, false>(a, zb + 1, o_own, cs, ps, P);
    if (hal && zb + 1 < ze) load_cell<NS, true>(a, zb + 1, o_hal, cs, ps, H);
    __syncthreads();

    for (int z = zb; z < ze; ++z) {
        const int b = (z - zb) & 1;
        const bool more = z + 1 < ze;  // plane z+1 is an output plane of this CTA
        const bool gz1 = is_ghost(a, z + 1);
        // [A] consume plane z+1
        if (own) {
            combine_y<NS>(a, gz1, P, Yp);
            if (more) {
                sY[b ^ 1][0][ly + 1][lx + 1] = Yp[0];
                sY[b ^ 1][1][ly + 1][lx + 1] = Yp[1];
                make_estate<NS, EPI>(a, P, En);
            }
        }
        if (hal && more) {
            double y[2];
            combine_y<NS>(a, gz1, H, y);
            sY[b ^ 1][0][hr][hc] = y[0];
            sY[b ^ 1][1][hr][hc] = y[1];
        }
        // [A'] issue loads of plane z+2 (own: needed as the z+1 neighbour; halo: if output)
        if (more) {
            if (own) load_cell<NS, false>(a, z + 2, o_own, cs, ps, P);
            if (hal && z + 2 < ze) load_cell<NS, true>(a, z + 2, o_hal, cs, ps, H);
        }
        // [C] stencil + reaction + epilogue at plane z
        if (own) {
            double L[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const double ctr = Yc[c];
                double s = add(sub(sY[b][c][ly + 1][lx], ctr), sub(sY[b][c][ly + 1][lx + 2], ctr));
                s = add(s, add(sub(sY[b][c][ly][lx + 1], ctr), sub(sY[b][c][ly + 2][lx + 1], ctr)));
                s = add(s, add(sub(Ym[c], ctr), sub(Yp[c], ctr)));
                L[c] = mul(s, a.inv_h2);
            }
            const double C0 = Yc[0], C1 = Yc[1];
            const double r = mul(mul(C0, C1), C1);
            double f[2];
            f[0] = sub(add(sub(mul(a.d1, L[0]), r), a.F), mul(a.F, C0));
            f[1] = sub(add(mul(a.d2, L[1]), r), mul(a.FK, C1));
            const int64_t oz = (int64_t)z * ps + o_own;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                if constexpr (EPI == EPI_K || EPI == EPI_FSAL_ERR) a.out_k[oz + c * cs] = f[c];
                if constexpr (FIN) {
                    const double wv = a.beta_new != 0.0 ? add(Ec.w[c], mul(a.beta_new, f[c])) : Ec.w[c];
                    a.out_u[oz + c * cs] = wv;
                }
                if constexpr (EPI == EPI_FSAL_ERR) a.out_u[oz + c * cs] = Yc[c];
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
        __syncthreads();
    }
    if constexpr (ERR) block_max_to_global(rmax, a.errmax);
}

template <int NS>
__global__ void __launch_bounds__(256) gs_pack_kernel(const GsStageArgs a, double* __restrict__ send) {
    const int64_t cs = (int64_t)a.nx * a.ny, ps = 2 * cs;
    const int64_t total = 2 * ps;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sel = e / ps, rest = e - sel * ps;
        const int64_t base = (sel ? (int64_t)(a.nzl - 1) : 0) * ps + rest;
        double v = __ldg(a.u + base);
#pragma unroll
        for (int s = 0; s < NS; ++s)
            if (a.g[s] != 0.0) v = add(v, mul(a.g[s], __ldg(a.k[s] + base)));
        send[e] = v;
    }
}

template <int NS>
cudaError_t launch_ns(int epi, const GsStageArgs& a, dim3 grid, cudaStream_t st) {
    switch (epi) {
    case EPI_K: gs_stage_kernel<NS, EPI_K><<<grid, NT, 0, st>>>(a); break;
    case EPI_FINAL: gs_stage_kernel<NS, EPI_FINAL><<<grid, NT, 0, st>>>(a); break;
    case EPI_FINAL_ERR: gs_stage_kernel<NS, EPI_FINAL_ERR><<<grid, NT, 0, st>>>(a); break;
    case EPI_FSAL_ERR: gs_stage_kernel<NS, EPI_FSAL_ERR><<<grid, NT, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gs_stage(int epi, const GsStageArgs& a, cudaStream_t st, int* nlaunch) {
    const int ntx = (a.nx + TX - 1) / TX, nty = (a.ny + TY - 1) / TY;
    const int tiles = ntx * nty;
    int nchunks;
    if (a.zmode == 1) {
        nchunks = a.nzl > 1 ? 2 : 1;
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
    const int64_t total = 4 * (int64_t)a.nx * a.ny;
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

}  // namespace rkb
