// bw_mix.cu — HBM bandwidth of streaming kernels with NR read and NW write arrays (fp64,
// 16-byte vector accesses, grid-stride, 1 GiB per array), to calibrate what a read/write mix
// like the stage kernels' can reach on this B200.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bw_mix tools/bw_mix.cu && /tmp/bw_mix
#include <cuda_runtime.h>

#include <cstdio>

template <int NR, int NW>
__global__ void __launch_bounds__(256) mix(const double2* __restrict__ const* in, double2* __restrict__ const* out,
                                           long n) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        double2 s = make_double2(1.0, 2.0);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const double2 v = __ldcs(in[r] + i);
            s.x += v.x;
            s.y += v.y;
        }
#pragma unroll
        for (int w = 0; w < NW; ++w) __stcs(out[w] + i, make_double2(s.x + w, s.y));
    }
}

template <int NR, int NW>
void run(double2** din, double2** dout, long n, int blocks) {
    const double2** ri;
    double2** wo;
    cudaMalloc(&ri, sizeof(void*) * 8);
    cudaMalloc(&wo, sizeof(void*) * 8);
    cudaMemcpy(ri, din, sizeof(void*) * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(wo, dout, sizeof(void*) * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int it = 0; it < 8; ++it) {
        cudaEventRecord(a);
        mix<NR, NW><<<blocks, 256>>>(ri, wo, n);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it > 0 && ms < best) best = ms;
    }
    const double bytes = (double)(NR + NW) * n * 16;
    printf("reads %d writes %d : %.3f ms  %.0f GB/s\n", NR, NW, best, bytes / (best * 1e-3) / 1e9);
    cudaFree(ri);
    cudaFree(wo);
}

int main() {
    const long n = (1l << 30) / 16;  // 1 GiB per array
    double2 *din[8], *dout[8];
    for (int i = 0; i < 8; ++i) {
        cudaMalloc(&din[i], n * 16);
        cudaMalloc(&dout[i], n * 16);
        cudaMemset(din[i], 0, n * 16);
    }
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8;
    run<1, 0>(din, dout, n, blocks);
    run<0, 1>(din, dout, n, blocks);
    run<1, 1>(din, dout, n, blocks);
    run<1, 2>(din, dout, n, blocks);
    run<2, 1>(din, dout, n, blocks);
    run<3, 1>(din, dout, n, blocks);
    run<4, 1>(din, dout, n, blocks);
    run<6, 1>(din, dout, n, blocks);
    run<2, 2>(din, dout, n, blocks);
    run<4, 2>(din, dout, n, blocks);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
