// rk_algebra.cu — K2 lincomb and K4 max-norm: the paper's distributed algebra ops
// ("for_each#() ... a total of #=15 inline methods", "for_each_norm()").
//
// lincomb: out = coef_0*in_0 (+) coef_1*in_1 (+) ... left to right, k <= 14 inputs,
// out may alias an input (every input element is read before the output is written).
// norm_inf: max |x| as uint64 bit patterns (exact, NaN-propagating), warp shuffle + one
// atomicMax per CTA; multi-GPU ranks then allreduce(max) the 8-byte result.
#include "rk_device.cuh"
#include "rk_kernels.cuh"

namespace rkb {

template <int K>
__global__ void __launch_bounds__(256) lincomb_kernel(const LincombArgs a) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.count; i += stride) {
        double acc = mul(a.coef[0], a.in[0][i]);
#pragma unroll
        for (int j = 1; j < K; ++j) acc = add(acc, mul(a.coef[j], a.in[j][i]));
        a.out[i] = acc;
    }
}

template <int K>
static void launch_k(const LincombArgs& a, unsigned blocks, cudaStream_t st) {
    lincomb_kernel<K><<<blocks, 256, 0, st>>>(a);
}

cudaError_t launch_lincomb(const LincombArgs& a, cudaStream_t st, int num_sms) {
    int64_t blocks = (a.count + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    const unsigned b = (unsigned)blocks;
    switch (a.k) {
    case 1: launch_k<1>(a, b, st); break;
    case 2: launch_k<2>(a, b, st); break;
    case 3: launch_k<3>(a, b, st); break;
    case 4: launch_k<4>(a, b, st); break;
    case 5: launch_k<5>(a, b, st); break;
    case 6: launch_k<6>(a, b, st); break;
    case 7: launch_k<7>(a, b, st); break;
    case 8: launch_k<8>(a, b, st); break;
    case 9: launch_k<9>(a, b, st); break;
    case 10: launch_k<10>(a, b, st); break;
    case 11: launch_k<11>(a, b, st); break;
    case 12: launch_k<12>(a, b, st); break;
    case 13: launch_k<13>(a, b, st); break;
    case 14: launch_k<14>(a, b, st); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

__global__ void __launch_bounds__(256) norm_inf_kernel(const double* __restrict__ x, int64_t n,
                                                       unsigned long long* out) {
    unsigned long long m = 0ull;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const unsigned long long b = ratio_bits(fabs(__ldg(x + i)));
        m = b > m ? b : m;
    }
    block_max_to_global(m, out);
}

// Unfused error control (RK_OPT_FUSED_KERNELS = 0): r = |e| / (atol + rtol*(|u| + dt*|k1|))
// (Odeint, R-12; w = k1) or |e| / (atol + rtol*max(|u|, |u_new|)) (SPEC, R-28; w = u_new) per
// element, the max over their bit patterns -- the fused epilogue's expression trees (R-17).
__global__ void __launch_bounds__(256) ratio_max_kernel(const double* __restrict__ e, const double* __restrict__ u,
                                                        const double* __restrict__ w, int64_t n, double dt,
                                                        double atol, double rtol, int spec,
                                                        unsigned long long* out) {
    unsigned long long m = 0ull;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double d;
        if (spec) {
            const double a = fabs(__ldg(u + i)), b = fabs(__ldg(w + i));
            d = add(atol, mul(rtol, a >= b ? a : b));
        } else {
            d = add(atol, mul(rtol, add(fabs(__ldg(u + i)), mul(dt, fabs(__ldg(w + i))))));
        }
        const unsigned long long bits = ratio_bits(fabs(__ldg(e + i)) / d);
        m = bits > m ? bits : m;
    }
    block_max_to_global(m, out);
}

cudaError_t launch_ratio_max(const double* e, const double* u, const double* w, int64_t count, double dt,
                             double atol, double rtol, int spec, unsigned long long* out, cudaStream_t st,
                             int num_sms) {
    int64_t blocks = (count + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    ratio_max_kernel<<<(unsigned)blocks, 256, 0, st>>>(e, u, w, count, dt, atol, rtol, spec, out);
    return cudaGetLastError();
}

// RK_OPT_ERROR_SPIKE: raise a try's local error-ratio max to at least v (fault injection)
__global__ void inject_max_kernel(unsigned long long* word, double v) { atomicMax(word, ratio_bits(v)); }

cudaError_t launch_inject_max(unsigned long long* word, double v, cudaStream_t st) {
    inject_max_kernel<<<1, 1, 0, st>>>(word, v);
    return cudaGetLastError();
}

// One 8-byte result (the try's error-ratio max, a norm) stored by a kernel straight into
// page-locked host memory (mapped under unified addressing), so the host's per-try read never
// queues on a copy engine behind a large transfer another stream has in flight.
__global__ void publish_word_kernel(const unsigned long long* src, unsigned long long* host_dst) {
    *reinterpret_cast<volatile unsigned long long*>(host_dst) = *reinterpret_cast<const volatile unsigned long long*>(src);
}

cudaError_t launch_publish_word(const unsigned long long* src, unsigned long long* host_dst, cudaStream_t st) {
    publish_word_kernel<<<1, 1, 0, st>>>(src, host_dst);
    return cudaGetLastError();
}

cudaError_t launch_norm_inf(const double* x, int64_t count, unsigned long long* out,
                            cudaStream_t st, int num_sms) {
    int64_t blocks = (count + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    norm_inf_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, count, out);
    return cudaGetLastError();
}

}  // namespace rkb
