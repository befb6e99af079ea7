// rk_pointwise.cu — K1: the whole explicit RK step of a pointwise RHS in registers.
//
// For du/dt = lambda*u (Eq. 1a) and du/dt = u(1-u) (Eq. 1b) every element
// is an independent ODE, so all stages Y_i, k_i, the final combination u_new and the
// embedded error live in registers: one 16 B/element HBM round trip per launch however
// many stages or fixed steps it covers (the "on-the-fly computation of stages" the paper
// credits for Odeint's speed).  Expression trees follow DESIGN.md R-17 exactly:
//   Y_i = u (+) (g_ij (x) k_j) over a_ij != 0, left to right;  u_new likewise with beta_j;
//   e = (delta_j (x) k_j) (+) ... over e_j != 0;  r = |e| / (atol (+) rtol (x) (|u| (+) dt (x) |k1|))
//   (Odeint, R-12) or r = |e| / (atol (+) rtol (x) max(|u|, |u_new|)) (SPEC, R-28).
#include <cooperative_groups.h>

#include <cfloat>

#include "rk_ddmath.cuh"
#include "rk_device.cuh"
#include "rk_kernels.cuh"
#include "rk_tableau.h"

namespace rkb {

__host__ __device__ constexpr bool a_nz(int S, int i, int j) { return rat_nz(tableau_of(S).a[i][j]); }
__host__ __device__ constexpr bool b_nz(int S, int j) { return rat_nz(tableau_of(S).b[j]); }
__host__ __device__ constexpr bool e_nz(int S, int j) { return rat_nz(err_weight(tableau_of(S), j)); }
// stages actually evaluated: up to the last j with b_j != 0 (or e_j != 0 with error)
__host__ __device__ constexpr int s_eff(int S, bool err) {
    int n = 0;
    for (int j = 0; j < tableau_of(S).s; ++j)
        if (b_nz(S, j) || (err && e_nz(S, j))) n = j + 1;
    return n;
}

// Nonzero pattern of a tableau, evaluated at compile time: used through a constexpr object so
// the rational arithmetic (err_weight's b - bhat with gcd reduction) can never be left to run
// time inside the kernel.
struct PwMask {
    bool a[13][13];
    bool b[13];
    bool e[13];
};
template <int S>
__host__ __device__ constexpr PwMask pw_mask() {
    PwMask m{};
    for (int i = 0; i < 13; ++i) {
        for (int j = 0; j < 13; ++j) m.a[i][j] = a_nz(S, i, j);
        m.b[i] = b_nz(S, i);
        m.e[i] = e_nz(S, i);
    }
    return m;
}

template <int RHS>
__device__ __forceinline__ double f_pointwise(double y, double lambda) {
    if constexpr (RHS == RHS_EXP) return mul(lambda, y);
    else return mul(y, sub(1.0, y));
}

// ERR: 0 no error estimate, 1 Odeint's ratio (R-12), 2 SPEC's ratio (R-28)
template <int S, int RHS, int ERR>
__device__ __forceinline__ double pw_steps(double x, const PwArgs& a, unsigned long long& rmax) {
    constexpr int SE = s_eff(S, ERR != 0);
    constexpr PwMask M = pw_mask<S>();
    const int nsteps = ERR ? 1 : a.nsteps;
    for (int n = 0; n < nsteps; ++n) {
        double k[13];
#pragma unroll
        for (int i = 0; i < SE; ++i) {
            double y = x;
#pragma unroll
            for (int j = 0; j < i; ++j)
                if (M.a[i][j]) y = add(y, mul(a.cf.g[i][j], k[j]));
            k[i] = f_pointwise<RHS>(y, a.lambda);
        }
        double w = x;
#pragma unroll
        for (int j = 0; j < SE; ++j)
            if (M.b[j]) w = add(w, mul(a.cf.beta[j], k[j]));
        if constexpr (ERR != 0) {
            double e = 0.0;
            bool first = true;
#pragma unroll
            for (int j = 0; j < SE; ++j) {
                if (!M.e[j]) continue;
                const double t = mul(a.cf.delta[j], k[j]);
                e = first ? t : add(e, t);
                first = false;
            }
            double den;
            if constexpr (ERR == 2) {
                const double au = fabs(x), aw = fabs(w);
                den = add(a.atol, mul(a.rtol, au >= aw ? au : aw));
            } else {
                den = add(a.atol, mul(a.rtol, add(fabs(x), mul(a.dt, fabs(k[0])))));
            }
            const unsigned long long rb = ratio_bits(fabs(e) / den);
            rmax = rb > rmax ? rb : rmax;
        }
        x = w;
    }
    return x;
}

template <int S, int RHS, int ERR>
__global__ void __launch_bounds__(256) pointwise_kernel(const PwArgs a) {
    unsigned long long rmax = 0ull;
    const int64_t n2 = a.count >> 1;
    const double2* __restrict__ u2 = reinterpret_cast<const double2*>(a.u);
    double2* __restrict__ o2 = reinterpret_cast<double2*>(a.u_out);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
        double2 v = __ldg(u2 + i);
        v.x = pw_steps<S, RHS, ERR>(v.x, a, rmax);
        v.y = pw_steps<S, RHS, ERR>(v.y, a, rmax);
        o2[i] = v;
    }
    if ((a.count & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = a.count - 1;
        a.u_out[i] = pw_steps<S, RHS, ERR>(a.u[i], a, rmax);
    }
    if constexpr (ERR != 0) block_max_to_global(rmax, a.errmax);
}

template <int S, int RHS>
static cudaError_t launch_s_rhs(const PwArgs& a, cudaStream_t st, int num_sms) {
    const int64_t n2 = (a.count + 1) / 2;
    int64_t blocks = (n2 + 255) / 256;
    const int64_t cap = (int64_t)num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (a.errmax && a.ctrl == 1)
        pointwise_kernel<S, RHS, 2><<<(unsigned)blocks, 256, 0, st>>>(a);
    else if (a.errmax)
        pointwise_kernel<S, RHS, 1><<<(unsigned)blocks, 256, 0, st>>>(a);
    else
        pointwise_kernel<S, RHS, 0><<<(unsigned)blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

template <int S>
static cudaError_t launch_s(const PwArgs& a, cudaStream_t st, int num_sms) {
    if (a.rhs == RHS_EXP) return launch_s_rhs<S, RHS_EXP>(a, st, num_sms);
    return launch_s_rhs<S, RHS_LOGISTIC>(a, st, num_sms);
}

// ---- device-resident adaptive loop (R-27) ------------------------
// The host loop of rk_integrate_adaptive (Odeint integrate_adaptive; R-16) and its
// controller (R-12), replayed on the device by every thread in lock step: each try runs the
// K1 step of every element (pw_steps, the same arithmetic as the host-driven launch), the
// error-ratio max is combined with one atomicMax per CTA and a grid-wide barrier, and all
// threads then take the same accept/reject decision from the same E.  Only the final state
// and the counters return to the host.
template <int S, int RHS, int ERR>
__global__ void __launch_bounds__(256) pointwise_loop_kernel(const PwLoopArgs a) {
    // (cooperative_groups' barrier: GBar measured slower here -- 296 CTAs of 256 threads, 11.5 ->
    // 13.2 us per try of configs[1] -- while it helps K5's 148 CTAs of 1024)
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ PwArgs sa;        // this try's coefficients (dt * tableau)
    __shared__ double s_dtn;     // controller result, computed once per CTA
    __shared__ int s_ok;
    constexpr int SE = s_eff(S, true);
    const double* u = a.buf[0];
    double* un = a.buf[1];
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
            for (int q = threadIdx.x; q < SE * SE; q += blockDim.x) {
                const int i = q / SE, j = q % SE;
                sa.cf.g[i][j] = __dmul_rn(dt, a.a[i][j]);
            }
            if (threadIdx.x < SE) {
                sa.cf.beta[threadIdx.x] = __dmul_rn(dt, a.b[threadIdx.x]);
                sa.cf.delta[threadIdx.x] = __dmul_rn(dt, a.e[threadIdx.x]);
            }
            if (threadIdx.x == 0) {
                sa.lambda = a.lambda;
                sa.dt = dt;
                sa.atol = a.atol;
                sa.rtol = a.rtol;
            }
            __syncthreads();
            unsigned long long rmax = 0ull;
            {
                const int64_t n2 = a.count >> 1;
                const double2* u2 = reinterpret_cast<const double2*>(u);
                double2* o2 = reinterpret_cast<double2*>(un);
                const int64_t stride = (int64_t)gridDim.x * blockDim.x;
                for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
                    double2 v = u2[i];
                    v.x = pw_steps<S, RHS, ERR>(v.x, sa, rmax);
                    v.y = pw_steps<S, RHS, ERR>(v.y, sa, rmax);
                    o2[i] = v;
                }
                if ((a.count & 1) && blockIdx.x == 0 && threadIdx.x == 0)
                    un[a.count - 1] = pw_steps<S, RHS, ERR>(u[a.count - 1], sa, rmax);
            }
            block_max_to_global(rmax, a.red + tri % 3);
            grid.sync();
            // slot (tri+2)%3 was last read before this barrier (try tri-1): clear it for try tri+2
            if (blockIdx.x == 0 && threadIdx.x == 0) a.red[(tri + 2) % 3] = 0ull;
            const unsigned long long eb = __ldcg(a.red + tri % 3);
            ++tri;
            E = __longlong_as_double((long long)eb);
            if (isnan(E)) {
                status = 5;
                goto done;
            }
            if (threadIdx.x == 0) {  // same inputs in every CTA -> the same decision everywhere
                int ok = 0;
                s_dtn = step_adjust_dev(E, a.e_rej, a.e_acc, a.emin, a.ctrl, dt, &ok);
                s_ok = ok;
            }
            __syncthreads();
            const double dtn = s_dtn;
            const bool ok = s_ok != 0;
            if (ok) {
                const double* tmp = u;
                u = un;
                un = const_cast<double*>(tmp);
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

template <int S, int RHS, int ERR>
static cudaError_t launch_loop_err(const PwLoopArgs& a, cudaStream_t st, int device) {
    int per_sm = 0, sms = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pointwise_loop_kernel<S, RHS, ERR>, 256, 0);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    int64_t blocks = ((a.count + 1) / 2 + 255) / 256;
    const int64_t cap = (int64_t)sms * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    void* args[] = {const_cast<PwLoopArgs*>(&a)};
    return cudaLaunchCooperativeKernel((void*)pointwise_loop_kernel<S, RHS, ERR>, dim3((unsigned)blocks),
                                       dim3(256), args, 0, st);
}

template <int S, int RHS>
static cudaError_t launch_loop_s_rhs(const PwLoopArgs& a, cudaStream_t st, int device) {
    return a.ctrl == 1 ? launch_loop_err<S, RHS, 2>(a, st, device) : launch_loop_err<S, RHS, 1>(a, st, device);
}

cudaError_t launch_pointwise_loop(int scheme, const PwLoopArgs& a, cudaStream_t st, int device) {
    const bool ex = a.rhs == RHS_EXP;
    switch (scheme) {
    case 2: return ex ? launch_loop_s_rhs<2, RHS_EXP>(a, st, device) : launch_loop_s_rhs<2, RHS_LOGISTIC>(a, st, device);
    case 3: return ex ? launch_loop_s_rhs<3, RHS_EXP>(a, st, device) : launch_loop_s_rhs<3, RHS_LOGISTIC>(a, st, device);
    case 4: return ex ? launch_loop_s_rhs<4, RHS_EXP>(a, st, device) : launch_loop_s_rhs<4, RHS_LOGISTIC>(a, st, device);
    default: return cudaErrorInvalidValue;
    }
}

// ---- Adams–Bashforth (Table 1 multi-step row): f_n = F(u_n),
// u_{n+1} = u_n (+) g_0 f_n (+) g_1 f_{n-1} (+) ... newest first (R-24).  The k-1
// past slopes stay in registers across all nsteps; each element is read and written once.
template <int K, int RHS>
__global__ void __launch_bounds__(256) ab_pointwise_kernel(const AbPwArgs a) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.count; i += stride) {
        double x = a.u[i];
        double h[K > 1 ? K - 1 : 1];
#pragma unroll
        for (int j = 0; j < K - 1; ++j) h[j] = a.hist[j][i];
        for (int n = 0; n < a.nsteps; ++n) {
            const double f = f_pointwise<RHS>(x, a.lambda);
            double w = add(x, mul(a.g[0], f));
#pragma unroll
            for (int j = 0; j < K - 1; ++j) w = add(w, mul(a.g[j + 1], h[j]));
#pragma unroll
            for (int j = K - 2; j > 0; --j) h[j] = h[j - 1];
            if (K > 1) h[0] = f;
            x = w;
        }
        a.u[i] = x;
#pragma unroll
        for (int j = 0; j < K - 1; ++j) a.hist[j][i] = h[j];
    }
}

template <int K>
static cudaError_t launch_ab_k(const AbPwArgs& a, unsigned blocks, cudaStream_t st) {
    if (a.rhs == RHS_EXP) ab_pointwise_kernel<K, RHS_EXP><<<blocks, 256, 0, st>>>(a);
    else ab_pointwise_kernel<K, RHS_LOGISTIC><<<blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_ab_pointwise(int k, const AbPwArgs& a, cudaStream_t st, int num_sms) {
    int64_t blocks = (a.count + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    const unsigned b = (unsigned)blocks;
    switch (k) {
    case 1: return launch_ab_k<1>(a, b, st);
    case 2: return launch_ab_k<2>(a, b, st);
    case 3: return launch_ab_k<3>(a, b, st);
    case 4: return launch_ab_k<4>(a, b, st);
    case 5: return launch_ab_k<5>(a, b, st);
    case 6: return launch_ab_k<6>(a, b, st);
    case 7: return launch_ab_k<7>(a, b, st);
    case 8: return launch_ab_k<8>(a, b, st);
    default: return cudaErrorInvalidValue;
    }
}

// Adams–Bashforth–Moulton k, PECE (R-26), nsteps steps per launch:
//   f = F(u_n); p = u_n (+) g_0 f (+) g_1 f_{n-1} ...; fp = F(p);
//   u_{n+1} = u_n (+) m_0 fp (+) m_1 f (+) m_2 f_{n-1} ...   (newest first)
template <int K, int RHS>
__global__ void __launch_bounds__(256) abm_pointwise_kernel(const AbPwArgs a) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.count; i += stride) {
        double x = a.u[i];
        double h[K > 1 ? K - 1 : 1];
#pragma unroll
        for (int j = 0; j < K - 1; ++j) h[j] = a.hist[j][i];
        for (int n = 0; n < a.nsteps; ++n) {
            const double f = f_pointwise<RHS>(x, a.lambda);
            double p = add(x, mul(a.g[0], f));
#pragma unroll
            for (int j = 0; j < K - 1; ++j) p = add(p, mul(a.g[j + 1], h[j]));
            const double fp = f_pointwise<RHS>(p, a.lambda);
            double w = add(x, mul(a.m[0], fp));
            if (K > 1) w = add(w, mul(a.m[1], f));
#pragma unroll
            for (int j = 0; j + 2 < K; ++j) w = add(w, mul(a.m[j + 2], h[j]));
#pragma unroll
            for (int j = K - 2; j > 0; --j) h[j] = h[j - 1];
            if (K > 1) h[0] = f;
            x = w;
        }
        a.u[i] = x;
#pragma unroll
        for (int j = 0; j < K - 1; ++j) a.hist[j][i] = h[j];
    }
}

template <int K>
static cudaError_t launch_abm_k(const AbPwArgs& a, unsigned blocks, cudaStream_t st) {
    if (a.rhs == RHS_EXP) abm_pointwise_kernel<K, RHS_EXP><<<blocks, 256, 0, st>>>(a);
    else abm_pointwise_kernel<K, RHS_LOGISTIC><<<blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_abm_pointwise(int k, const AbPwArgs& a, cudaStream_t st, int num_sms) {
    int64_t blocks = (a.count + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    const unsigned b = (unsigned)blocks;
    switch (k) {
    case 1: return launch_abm_k<1>(a, b, st);
    case 2: return launch_abm_k<2>(a, b, st);
    case 3: return launch_abm_k<3>(a, b, st);
    case 4: return launch_abm_k<4>(a, b, st);
    case 5: return launch_abm_k<5>(a, b, st);
    case 6: return launch_abm_k<6>(a, b, st);
    case 7: return launch_abm_k<7>(a, b, st);
    case 8: return launch_abm_k<8>(a, b, st);
    default: return cudaErrorInvalidValue;
    }
}

template <int RHS>
__global__ void __launch_bounds__(256) rhs_pointwise_kernel(const double* __restrict__ u,
                                                            double* __restrict__ f, int64_t n,
                                                            double lambda) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        f[i] = f_pointwise<RHS>(__ldg(u + i), lambda);
}

cudaError_t launch_rhs_pointwise(const double* u, double* f, int64_t count, int rhs, double lambda,
                                 cudaStream_t st, int num_sms) {
    int64_t blocks = (count + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    if (rhs == RHS_EXP) rhs_pointwise_kernel<RHS_EXP><<<(unsigned)blocks, 256, 0, st>>>(u, f, count, lambda);
    else rhs_pointwise_kernel<RHS_LOGISTIC><<<(unsigned)blocks, 256, 0, st>>>(u, f, count, lambda);
    return cudaGetLastError();
}

cudaError_t launch_pointwise(int scheme, const PwArgs& a, cudaStream_t st, int num_sms) {
    switch (scheme) {
    case 0: return launch_s<0>(a, st, num_sms);
    case 1: return launch_s<1>(a, st, num_sms);
    case 2: return launch_s<2>(a, st, num_sms);
    case 3: return launch_s<3>(a, st, num_sms);
    case 4: return launch_s<4>(a, st, num_sms);
    case 5: return launch_s<5>(a, st, num_sms);
    case 6: return launch_s<6>(a, st, num_sms);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace rkb
