// rk_smallgrid.cu — K5: whole fixed-step Runge–Kutta steps of Gray–Scott on a small grid in ONE
// persistent cooperative launch ("launch-bound small configs"; configs[2], 64^3).
//
// At 64^3 every array is 4 MiB and a whole step lives in the 126 MB L2, so the TMA stencil
// kernel (K3, rk_stencil.cu) is bound by fixed per-launch costs -- launch, CTA start-up, the
// first TMA round trip, too few CTAs -- at ~9 us per stage whatever the z-chunk
// (DESIGN.md §9).  Here one cooperative grid runs all stages of all steps: per stage every
// thread takes cells in a grid-stride loop, reads Y_i at the cell and its six neighbours
// (L1/L2 hits), evaluates the 7-point Laplacian and the reaction
// (Listing 2), stores k_i (or, at the last stage, u_new = u + sum_j beta_j k_j)
// with its periodic ring copies, and a grid-wide barrier separates the stages.  u / u_new
// ping-pong inside the kernel.  Each stage also writes the NEXT stage value Y_{i+1} at its
// own cells (it holds u, the k_j and the new k_i there), so a stage's stencil reads a single
// array, Y_i, at seven points; two Y buffers alternate.
//
// Arithmetic is the stencil kernel's expression for expression (R-17, SURVEY
// App. C): Y = u (+) g_ij (x) k_j over a_ij != 0 in increasing j; the Laplacian in difference
// form x, then y, then z; the same reaction trees; u_new = u (+) beta_j (x) k_j in increasing j.
// Results therefore equal the oracle's and the stage-by-stage path's bit for bit.
#include <cooperative_groups.h>

#include "rk_device.cuh"
#include "rk_kernels.cuh"
#include "rk_tableau.h"

namespace rkb {

namespace {

struct CoopMask {
    bool a[13][13];
    bool b[13];
    int last;  // last stage with b_j != 0 (fused with u_new)
};

template <int S>
__host__ __device__ constexpr CoopMask coop_mask() {
    const Tableau T = tableau_of(S);
    CoopMask m{};
    m.last = 0;
    for (int i = 0; i < 13; ++i) {
        for (int j = 0; j < 13; ++j) m.a[i][j] = i < T.s && j < i && rat_nz(T.a[i][j]);
        m.b[i] = i < T.s && rat_nz(T.b[i]);
        if (m.b[i]) m.last = i;
    }
    return m;
}

// k_I must be stored if a stage after I+1 or the final combination reads it (stage I+1's Y
// takes it from the register that computed it)
template <int S, int I>
__host__ __device__ constexpr bool keep_k() {
    constexpr CoopMask M = coop_mask<S>();
    bool k = M.b[I];
    for (int m = I + 2; m <= M.last; ++m) k = k || M.a[m][I];
    return k;
}

__device__ __forceinline__ void store_ring(double* out, const GridGeom& G, int64_t o, bool ex0, bool ex1,
                                           bool ey0, bool ey1, double v) {
    double* p = out + o;
    p[0] = v;  // plus the periodic ring copies of an edge cell (corners are never read)
    if (ex0) p[G.nx] = v;
    if (ex1) p[-G.nx] = v;
    if (ey0) p[(int64_t)G.ny * G.P] = v;
    if (ey1) p[-(int64_t)G.ny * G.P] = v;
}

// Stage I: k_I = F(Y_I) from the 7-point neighbourhood of Y_I (u for I = 0, else the Y buffer
// written by stage I-1); then either u_new (last stage) or k_I and Y_{I+1} at the own cell
// ("write Y ahead": the next stage's stencil reads one array).
template <int S, int I>
__device__ __forceinline__ void coop_stage(const GsCoopArgs& a, const double* u, double* un) {
    constexpr CoopMask M = coop_mask<S>();
    constexpr bool FIN = I == M.last;
    const double* Y = I == 0 ? u : a.ybuf[(I - 1) & 1];
    double* Ynext = a.ybuf[I & 1];
    const GridGeom& G = a.geo;
    const int64_t ncell = (int64_t)G.nzl * G.ny * G.nx;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < ncell; q += stride) {
        const int x = (int)(q % G.nx);
        const int64_t r = q / G.nx;
        const int y = (int)(r % G.ny), z = (int)(r / G.ny);
        const int zm = z == 0 ? G.nzl - 1 : z - 1, zp = z == G.nzl - 1 ? 0 : z + 1;
        const int64_t own = (int64_t)(y + 1) * G.P + (x + 1);
        double C[2], L[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int64_t o = (int64_t)z * G.ps + c * G.cs + own;
            const double ctr = Y[o];
            double s = add(sub(Y[o - 1], ctr), sub(Y[o + 1], ctr));
            s = add(s, add(sub(Y[o - G.P], ctr), sub(Y[o + G.P], ctr)));
            const double ym = Y[(int64_t)zm * G.ps + c * G.cs + own];
            const double yp = Y[(int64_t)zp * G.ps + c * G.cs + own];
            s = add(s, add(sub(ym, ctr), sub(yp, ctr)));
            L[c] = mul(s, a.inv_h2);
            C[c] = ctr;
        }
        const double rc = mul(mul(C[0], C[1]), C[1]);
        double f[2];
        f[0] = sub(add(sub(mul(a.d1, L[0]), rc), a.F), mul(a.F, C[0]));
        f[1] = sub(add(mul(a.d2, L[1]), rc), mul(a.FK, C[1]));
        const bool ex0 = x == 0, ex1 = x == G.nx - 1, ey0 = y == 0, ey1 = y == G.ny - 1;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int64_t o = (int64_t)z * G.ps + c * G.cs + own;
            const double uo = u[o];
            if constexpr (FIN) {
                double w = uo;
#pragma unroll
                for (int j = 0; j < I; ++j)
                    if (M.b[j]) w = add(w, mul(a.beta[j], a.k[j][o]));
                store_ring(un, G, o, ex0, ex1, ey0, ey1, add(w, mul(a.beta[I], f[c])));
            } else {
                if constexpr (keep_k<S, I>()) store_ring(a.k[I], G, o, ex0, ex1, ey0, ey1, f[c]);
                double v = uo;  // Y_{I+1} = u (+) g_{I+1,j} k_j over a != 0, increasing j
#pragma unroll
                for (int j = 0; j <= I; ++j)
                    if (M.a[I + 1][j]) v = add(v, mul(a.g[I + 1][j], j == I ? f[c] : a.k[j][o]));
                store_ring(Ynext, G, o, ex0, ex1, ey0, ey1, v);
            }
        }
    }
}

template <int S, int I>
__device__ __forceinline__ void coop_stages(const GsCoopArgs& a, const double* u, double* un,
                                            cooperative_groups::grid_group& grid) {
    constexpr CoopMask M = coop_mask<S>();
    if constexpr (I <= M.last) {
        coop_stage<S, I>(a, u, un);
        grid.sync();  // k_I, Y_{I+1} (or u_new) complete everywhere before the next stage
        coop_stages<S, I + 1>(a, u, un, grid);
    }
}

template <int S, int MINB>
__global__ void __launch_bounds__(256, MINB) gs_coop_kernel(const __grid_constant__ GsCoopArgs a) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    double* u = a.buf[0];
    double* un = a.buf[1];
    for (int n = 0; n < a.nsteps; ++n) {
        coop_stages<S, 0>(a, u, un, grid);
        double* t = u;
        u = un;
        un = t;
    }
}

template <int S, int MINB>
cudaError_t launch_coop_m(const GsCoopArgs& a, cudaStream_t st, int device) {
    static int per_sm = -1;
    if (per_sm < 0) {
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gs_coop_kernel<S, MINB>, 256, 0);
        if (e != cudaSuccess) return e;
    }
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    const int64_t ncell = (int64_t)a.geo.nzl * a.geo.ny * a.geo.nx;
    int64_t blocks = (ncell + 255) / 256;
    const int64_t cap = (int64_t)sms * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    void* args[] = {const_cast<GsCoopArgs*>(&a)};
    return cudaLaunchCooperativeKernel((void*)gs_coop_kernel<S, MINB>, dim3((unsigned)blocks), dim3(256), args, 0,
                                       st);
}

// 4 CTAs of 256 threads per SM (64 registers): measured best at 16^3..64^3 against 6 and 8
// (more CTAs make every grid-wide barrier slower; tools/prof_small.py)
template <int S>
cudaError_t launch_coop_s(const GsCoopArgs& a, cudaStream_t st, int device) {
    return launch_coop_m<S, 4>(a, st, device);
}

}  // namespace

int coop_last_stage(int scheme) {
    switch (scheme) {
    case 0: return coop_mask<0>().last;
    case 1: return coop_mask<1>().last;
    case 2: return coop_mask<2>().last;
    case 3: return coop_mask<3>().last;
    case 4: return coop_mask<4>().last;
    case 5: return coop_mask<5>().last;
    default: return -1;
    }
}

cudaError_t launch_gs_coop(int scheme, const GsCoopArgs& a, cudaStream_t st, int device) {
    switch (scheme) {
    case 0: return launch_coop_s<0>(a, st, device);
    case 1: return launch_coop_s<1>(a, st, device);
    case 2: return launch_coop_s<2>(a, st, device);
    case 3: return launch_coop_s<3>(a, st, device);
    case 4: return launch_coop_s<4>(a, st, device);
    case 5: return launch_coop_s<5>(a, st, device);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace rkb
