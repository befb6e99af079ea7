// rk_device.cuh — device helpers: correctly rounded fp64 ops that are never contracted
// into FMA (R-17), and the uint64-bit-pattern max reduction (J subsystem 3).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace rkb {

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }

// Error ratios are >= +0 or NaN, so their IEEE bit patterns order like the values as
// unsigned integers, and every NaN pattern compares above +inf: max over bits is an exact,
// order-independent, NaN-propagating max (P:L46, P:L135 for_each_norm).
__device__ __forceinline__ unsigned long long ratio_bits(double r) {
    return (unsigned long long)__double_as_longlong(r);
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        unsigned long long o = __shfl_xor_sync(0xffffffffu, v, off);
        v = o > v ? o : v;
    }
    return v;
}

// System-scope acquire load / release store (flags written by another GPU over NVLink).
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block-wide max then one atomicMax per CTA.  Must be called by every thread of the CTA.
__device__ __forceinline__ void block_max_to_global(unsigned long long v, unsigned long long* out) {
    __shared__ unsigned long long s_red[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    v = warp_max_u64(v);
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < nwarps ? s_red[lane] : 0ull;
        v = warp_max_u64(v);
        if (lane == 0 && v != 0ull) atomicMax(out, v);
    }
}

// Grid-wide barrier of the cooperative K5 kernels (one 1024-thread CTA per SM) on the state's own
// two words (arrivals, generation; zeroed once; concurrent launches of other states use their
// own): thread 0 of each CTA arrives after a fence, the last arrival resets the counter and
// releases the next generation, the others poll it with acquire loads.  Replaces
// cooperative_groups' grid_group::sync there (configs[2]: 27.2 -> 26.4-26.7 us per 64^3 RK4 step;
// the vector device loop's 296 CTAs of 256 threads measured slower with it and keep grid_group).
struct GBar {
    unsigned int* w;
    __device__ __forceinline__ void sync() {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned int g;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(w + 1) : "memory");
            __threadfence();
            if (atomicAdd(w, 1u) == gridDim.x - 1) {
                atomicExch(w, 0u);
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(w + 1), "r"(g + 1) : "memory");
            } else {
                unsigned int c;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(w + 1) : "memory");
                } while (c == g);
            }
        }
        __syncthreads();
    }
};

}  // namespace rkb
