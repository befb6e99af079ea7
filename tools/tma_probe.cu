// Standalone probe: 4D TMA box load of a small padded array; dumps smem box to global.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
constexpr int BW = 34, BH = 10;
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void probe(const __grid_constant__ CUtensorMap m, double* out, int x0, int y0, int q) {
  __shared__ __align__(128) double box[2 * BW * BH];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(2*BW*BH*8));
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
      ::"r"(su(box)), "l"((uint64_t)&m), "r"(su(&bar)), "r"(x0), "r"(y0), "r"(0), "r"(q) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W%=;\n}" ::"r"(su(&bar)));
  for (int i = threadIdx.x; i < 2 * BW * BH; i += blockDim.x) out[i] = box[i];
}
int main() {
  int nx = 4, ny = 4, nz = 4, P = 6;
  long cs = (long)(ny + 2) * P, ps = 2 * cs;
  std::vector<double> h(nz * ps);
  for (long i = 0; i < (long)h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 2 * BW * BH * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)P, (cuuint64_t)ny + 2, 2, (cuuint64_t)nz};
  cuuint64_t str[3] = {(cuuint64_t)P * 8, (cuuint64_t)cs * 8, (cuuint64_t)ps * 8};
  cuuint32_t box[4] = {BW, BH, 2, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  probe<<<1, 128>>>(m, o, 0, 0, 1);
  printf("kernel %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<double> b(2 * BW * BH);
  cudaMemcpy(b.data(), o, b.size() * 8, cudaMemcpyDeviceToHost);
  for (int c = 0; c < 2; ++c) for (int y = 0; y < 7; ++y) {
    printf("c%d y%d:", c, y);
    for (int x = 0; x < 8; ++x) printf(" %5.0f", b[c * BW * BH + y * BW + x]);
    printf("\n");
  }
  // expected: plane 1 base = ps = 72; element (c,y,x) = 72 + c*36 + y*6 + x for x<6,y<6
}
