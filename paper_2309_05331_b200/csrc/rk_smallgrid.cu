// rk_smallgrid.cu — K5: whole Runge–Kutta integrations of Gray–Scott on a small grid in ONE
// persistent cooperative launch ("launch-bound small configs" and "device-resident
// controller"; configs[2], 64^3).
//
// At 64^3 every array is 4 MiB and a whole step lives in the 126 MB L2, so the TMA stencil
// kernel (K3, rk_stencil.cu) is bound by fixed per-launch costs -- launch, CTA start-up, the
// first TMA round trip, too few CTAs -- at ~9 us per stage whatever the z-chunk
// (DESIGN.md §9).  Here one cooperative grid runs all stages of all steps: per stage every
// thread takes cells in a grid-stride loop, reads Y_i at the cell and its six neighbours
// (L1/L2 hits), evaluates the 7-point Laplacian and the reaction (Listing 2),
// stores k_i (or, at the last stage, u_new = u + sum_j beta_j k_j) with its periodic ring
// copies, and a grid-wide barrier separates the stages.  u / u_new ping-pong inside the
// kernel.  Each stage also writes the NEXT stage value Y_{i+1} at its own cells (it holds u,
// the k_j and the new k_i there), so a stage's stencil reads a single array, Y_i, at seven
// points; two Y buffers alternate.
//
// Two drivers share the stage code:
//   gs_coop_kernel           fixed steps (do_step / integrate_const), coefficients from the host;
//   gs_coop_adaptive_kernel  the whole integrate_adaptive (Odeint loop R-16): per try
//                            the stages, the embedded error ratio and its grid-wide max
//                            (P:L42), then the controller of R-12 or R-28 evaluated on
//                            the device by every thread on the same E (double-double pow,
//                            R-27), the stage coefficients dt*a_ij recomputed per try.  No
//                            host round trip per try.  k1 is re-evaluated every try (no FSAL
//                            buffer swap): F(u_new) is the same value either way.
//
// Arithmetic is the stencil kernel's expression for expression (R-17, SURVEY
// App. C): Y = u (+) g_ij (x) k_j over a_ij != 0 in increasing j; the Laplacian in difference
// form x, then y, then z; the same reaction trees; u_new = u (+) beta_j (x) k_j and
// e = delta_j (x) k_j (+) ... in increasing j; r = |e| / d with d as in R-12 / R-28.
// Results therefore equal the oracle's and the stage-by-stage path's bit for bit.
#include <cooperative_groups.h>

#include <cfloat>

#include "rk_ddmath.cuh"
#include "rk_device.cuh"
#include "rk_kernels.cuh"
#include "rk_tableau.h"

namespace rkb {

namespace {

#ifndef RKB_COOP_NT
#define RKB_COOP_NT 1024
#endif
constexpr int kCoopThreads = RKB_COOP_NT;  // threads per CTA of the persistent kernels

struct CoopMask {
    bool a[13][13];
    bool b[13];
    bool e[13];
    int last;   // fixed step: last stage with b_j != 0 (fused with u_new)
    int lasta;  // error control: last stage with b_j or e_j != 0
};

template <int S>
__host__ __device__ constexpr CoopMask coop_mask() {
    const Tableau T = tableau_of(S);
    CoopMask m{};
    m.last = 0;
    m.lasta = 0;
    for (int i = 0; i < 13; ++i) {
        for (int j = 0; j < 13; ++j) m.a[i][j] = i < T.s && j < i && rat_nz(T.a[i][j]);
        m.b[i] = i < T.s && rat_nz(T.b[i]);
        m.e[i] = i < T.s && T.err_order > 0 && rat_nz(err_weight(T, i));
        if (m.b[i]) m.last = i;
        if (m.b[i] || m.e[i]) m.lasta = i;
    }
    return m;
}

// MODE: 0 fixed step; 1 error control with Odeint's ratio (R-12); 2 with SPEC's (R-28)
template <int S, int MODE>
__host__ __device__ constexpr int last_of() {
    return MODE == 0 ? coop_mask<S>().last : coop_mask<S>().lasta;
}

// k_I must be stored if a stage after I+1, the final combination, the error sum or (Odeint's
// ratio) the denominator reads it; stage I+1's Y takes it from the register that computed it
template <int S, int MODE, int I>
__host__ __device__ constexpr bool keep_k() {
    constexpr CoopMask M = coop_mask<S>();
    constexpr int L = last_of<S, MODE>();
    bool k = M.b[I] || (MODE != 0 && M.e[I]) || (MODE == 1 && I == 0);
    for (int m = I + 2; m <= L; ++m) k = k || M.a[m][I];
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

// Per-launch constants of the stage code.
struct StageEnv {
    GridGeom geo;
    double* const* k;   // k_j buffers
    double* const* yb;  // Y buffers
    double d1, d2, F, FK, inv_h2;
    double dt, atol, rtol;  // error control
};

// Stage I: k_I = F(Y_I) from the 7-point neighbourhood of Y_I (u for I = 0, else the Y buffer
// written by stage I-1); then either the last stage's epilogue (u_new; with error control also
// e and the ratio max) or k_I and Y_{I+1} at the own cell ("write Y ahead").
template <int S, int MODE, int I>
__device__ __forceinline__ void coop_stage(const StageEnv& v, const CoopCoef& cf, const double* u, double* un,
                                           unsigned long long& rbits) {
    constexpr CoopMask M = coop_mask<S>();
    constexpr int L = last_of<S, MODE>();
    constexpr bool LAST = I == L;
    const double* Y = I == 0 ? u : v.yb[(I - 1) & 1];
    double* Ynext = v.yb[I & 1];
    const GridGeom& G = v.geo;
    const int64_t ncell = (int64_t)G.nzl * G.ny * G.nx;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < ncell; q += stride) {
        const int x = (int)(q % G.nx);
        const int64_t r = q / G.nx;
        const int y = (int)(r % G.ny), z = (int)(r / G.ny);
        const int zm = z == 0 ? G.nzl - 1 : z - 1, zp = z == G.nzl - 1 ? 0 : z + 1;
        const int64_t own = (int64_t)(y + 1) * G.P + (x + 1);
        double C[2], Lp[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int64_t o = (int64_t)z * G.ps + c * G.cs + own;
            const double ctr = Y[o];
            double s = add(sub(Y[o - 1], ctr), sub(Y[o + 1], ctr));
            s = add(s, add(sub(Y[o - G.P], ctr), sub(Y[o + G.P], ctr)));
            const double ym = Y[(int64_t)zm * G.ps + c * G.cs + own];
            const double yp = Y[(int64_t)zp * G.ps + c * G.cs + own];
            s = add(s, add(sub(ym, ctr), sub(yp, ctr)));
            Lp[c] = mul(s, v.inv_h2);
            C[c] = ctr;
        }
        const double rc = mul(mul(C[0], C[1]), C[1]);
        double f[2];
        f[0] = sub(add(sub(mul(v.d1, Lp[0]), rc), v.F), mul(v.F, C[0]));
        f[1] = sub(add(mul(v.d2, Lp[1]), rc), mul(v.FK, C[1]));
        const bool ex0 = x == 0, ex1 = x == G.nx - 1, ey0 = y == 0, ey1 = y == G.ny - 1;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int64_t o = (int64_t)z * G.ps + c * G.cs + own;
            const double uo = u[o];
            if constexpr (LAST) {
                double w = uo;
#pragma unroll
                for (int j = 0; j < I; ++j)
                    if (M.b[j]) w = add(w, mul(cf.beta[j], v.k[j][o]));
                if (M.b[I]) w = add(w, mul(cf.beta[I], f[c]));
                store_ring(un, G, o, ex0, ex1, ey0, ey1, w);
                if constexpr (MODE != 0) {
                    double e = 0.0;
                    bool first = true;
#pragma unroll
                    for (int j = 0; j <= I; ++j) {
                        if (!M.e[j]) continue;
                        const double t = mul(cf.delta[j], j == I ? f[c] : v.k[j][o]);
                        e = first ? t : add(e, t);
                        first = false;
                    }
                    double d;
                    if constexpr (MODE == 2) {
                        const double au = fabs(uo), aw = fabs(w);
                        d = add(v.atol, mul(v.rtol, au >= aw ? au : aw));
                    } else {
                        d = add(v.atol, mul(v.rtol, add(fabs(uo), mul(v.dt, fabs(v.k[0][o])))));
                    }
                    const unsigned long long rb = ratio_bits(fabs(e) / d);
                    rbits = rb > rbits ? rb : rbits;
                }
            } else {
                if constexpr (keep_k<S, MODE, I>()) store_ring(v.k[I], G, o, ex0, ex1, ey0, ey1, f[c]);
                double yv = uo;  // Y_{I+1} = u (+) g_{I+1,j} k_j over a != 0, increasing j
#pragma unroll
                for (int j = 0; j <= I; ++j)
                    if (M.a[I + 1][j]) yv = add(yv, mul(cf.g[I + 1][j], j == I ? f[c] : v.k[j][o]));
                store_ring(Ynext, G, o, ex0, ex1, ey0, ey1, yv);
            }
        }
    }
}

#ifndef RKB_K5_BAR
#define RKB_K5_BAR 1  // 1: GBar (rk_device.cuh), 0: cooperative_groups' grid_group::sync
#endif
// stages I..L with a grid-wide barrier between them (the caller synchronises after the last:
// before the next step, or through the error-max reduction)
template <int S, int MODE, int I, class GB>
__device__ __forceinline__ void coop_stages(const StageEnv& v, const CoopCoef& cf, const double* u, double* un,
                                            unsigned long long& rbits, GB& grid) {
    constexpr int L = last_of<S, MODE>();
    coop_stage<S, MODE, I>(v, cf, u, un, rbits);
    if constexpr (I < L) {
        grid.sync();  // k_I, Y_{I+1} complete everywhere before the next stage
        coop_stages<S, MODE, I + 1, GB>(v, cf, u, un, rbits, grid);
    }
}

__device__ __forceinline__ StageEnv env_of(const GsCoopArgs& a) {
    StageEnv v;
    v.geo = a.geo;
    v.k = a.k;
    v.yb = a.ybuf;
    v.d1 = a.d1;
    v.d2 = a.d2;
    v.F = a.F;
    v.FK = a.FK;
    v.inv_h2 = a.inv_h2;
    v.dt = v.atol = v.rtol = 0.0;
    return v;
}

// ---- fixed steps -------------------------------------------------------------------------
template <int S, int MINB>
__global__ void __launch_bounds__(kCoopThreads, MINB) gs_coop_kernel(const __grid_constant__ GsCoopArgs a) {
#if RKB_K5_BAR
    GBar grid{a.bar};
#else
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
#endif
    const StageEnv v = env_of(a);
    double* u = a.buf[0];
    double* un = a.buf[1];
    unsigned long long rb = 0ull;
    for (int n = 0; n < a.nsteps; ++n) {
        coop_stages<S, 0, 0>(v, a.cf, u, un, rb, grid);
        grid.sync();  // u_new complete before the next step reads it
        double* t = u;
        u = un;
        un = t;
    }
}

// ---- the whole integrate_adaptive --------------------------------------------------------
template <int S, int MODE, int MINB>
__global__ void __launch_bounds__(kCoopThreads, MINB) gs_coop_adaptive_kernel(const __grid_constant__ GsCoopLoopArgs a) {
#if RKB_K5_BAR
    GBar grid{a.c.bar};
#else
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
#endif
    __shared__ CoopCoef cf;   // this try's dt-scaled coefficients
    __shared__ double s_dtn;  // controller result, computed once per CTA
    __shared__ int s_ok;
    constexpr int L = last_of<S, MODE>();
    StageEnv v = env_of(a.c);
    v.atol = a.atol;
    v.rtol = a.rtol;
    double* u = a.c.buf[0];
    double* un = a.c.buf[1];
    int which = 0;
    double t = a.t0, dt = a.dt0, E = 0.0;
    long long acc = 0, rej = 0;
    unsigned tri = 0;
    int status = 0;
    while (__dsub_rn(a.t1, t) > DBL_EPSILON) {
        if (__dsub_rn(__dadd_rn(t, dt), a.t1) > DBL_EPSILON) dt = __dsub_rn(a.t1, t);
        int tries = 0;
        for (;;) {
            if (dt < __dmul_rn(16.0 * DBL_EPSILON, fmax(fabs(t), 1.0))) {
                status = 6;
                goto done;
            }
            for (int q = threadIdx.x; q < (L + 1) * (L + 1); q += blockDim.x) {
                const int i = q / (L + 1), j = q % (L + 1);
                cf.g[i][j] = __dmul_rn(dt, a.A[i][j]);
            }
            if (threadIdx.x <= L) {
                cf.beta[threadIdx.x] = __dmul_rn(dt, a.B[threadIdx.x]);
                cf.delta[threadIdx.x] = __dmul_rn(dt, a.Ew[threadIdx.x]);
            }
            v.dt = dt;
            __syncthreads();
            unsigned long long rbits = 0ull;
            coop_stages<S, MODE, 0>(v, cf, u, un, rbits, grid);
            block_max_to_global(rbits, a.red + tri % 3);
            grid.sync();
            // slot (tri+2)%3 was last read before this barrier (try tri-1): clear it for try tri+2
            if (blockIdx.x == 0 && threadIdx.x == 0) a.red[(tri + 2) % 3] = 0ull;
            E = __longlong_as_double((long long)__ldcg(a.red + tri % 3));
            ++tri;
            if (isnan(E)) {
                status = 5;
                goto done;
            }
            if (threadIdx.x == 0) {  // same inputs in every CTA -> the same decision everywhere
                int ok = 0;
                s_dtn = step_adjust_dev(E, a.e_rej, a.e_acc, a.emin, MODE == 2 ? 1 : 0, dt, &ok);
                s_ok = ok;
            }
            __syncthreads();
            const double dtn = s_dtn;
            const bool ok = s_ok != 0;
            if (ok) {
                double* tmp = u;
                u = un;
                un = tmp;
                which ^= 1;
                t = __dadd_rn(t, dt);
                dt = dtn;
                ++acc;
                break;
            }
            dt = dtn;
            ++rej;
            if (++tries >= a.max_tries) {
                status = 7;
                goto done;
            }
        }
    }
done:
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.res->status = status;
        a.res->which = which;
        a.res->accepted = acc;
        a.res->rejected = rej;
        a.res->t = t;
        a.res->dt = dt;
        a.res->last_E = E;
    }
}

template <typename K>
cudaError_t coop_launch(K kernel, void* arg, const GridGeom& g, cudaStream_t st, int device) {
    int per_sm = 0, sms = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kCoopThreads, 0);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    const int64_t ncell = (int64_t)g.nzl * g.ny * g.nx;
    int64_t blocks = (ncell + kCoopThreads - 1) / kCoopThreads;
    const int64_t cap = (int64_t)sms * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    void* args[] = {arg};
    return cudaLaunchCooperativeKernel((void*)kernel, dim3((unsigned)blocks), dim3(kCoopThreads), args, 0, st);
}

// One CTA of 1024 threads per SM (64 registers): the grid-wide barrier then counts 148
// arrivals instead of 592.  configs[2] (64^3 RK4, 20 steps, one launch): 31.9 us/step with
// 4 x 256 threads per SM, 31.4 with 2 x 512, 27.6 with 1 x 1024 (measured on the B200; 6 and
// 8 CTAs of 256 were slower still, tools/prof_small.py).
constexpr int kCoopMinBlocks = 1024 / kCoopThreads;

template <int S>
cudaError_t launch_coop_s(const GsCoopArgs& a, cudaStream_t st, int device) {
    return coop_launch(gs_coop_kernel<S, kCoopMinBlocks>, const_cast<GsCoopArgs*>(&a), a.geo, st, device);
}

template <int S>
cudaError_t launch_coop_adaptive_s(const GsCoopLoopArgs& a, cudaStream_t st, int device) {
    void* p = const_cast<GsCoopLoopArgs*>(&a);
    if (a.ctrl == 1) return coop_launch(gs_coop_adaptive_kernel<S, 2, kCoopMinBlocks>, p, a.c.geo, st, device);
    return coop_launch(gs_coop_adaptive_kernel<S, 1, kCoopMinBlocks>, p, a.c.geo, st, device);
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
    case 6: return coop_mask<6>().last;
    default: return -1;
    }
}

int coop_last_stage_adaptive(int scheme) {
    switch (scheme) {
    case 2: return coop_mask<2>().lasta;
    case 3: return coop_mask<3>().lasta;
    case 4: return coop_mask<4>().lasta;
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
    case 6: return launch_coop_s<6>(a, st, device);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_gs_coop_adaptive(int scheme, const GsCoopLoopArgs& a, cudaStream_t st, int device) {
    switch (scheme) {
    case 2: return launch_coop_adaptive_s<2>(a, st, device);
    case 3: return launch_coop_adaptive_s<3>(a, st, device);
    case 4: return launch_coop_adaptive_s<4>(a, st, device);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace rkb
