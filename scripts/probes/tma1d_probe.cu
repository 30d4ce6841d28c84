// Probe: 1-D FLOAT64 tensor-map TMA load at arbitrary element coordinates.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap map, double* out, int c, int variant) {
  extern __shared__ __align__(128) double buf[];
  __shared__ __align__(8) uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  uint32_t d = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(512) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];\n" ::"r"(d),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(c), "r"(b)
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(b) : "memory");
  for (int i = threadIdx.x; i < 64; i += 32) out[i] = buf[i];
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int n = 1000;
  std::vector<double> h(n);
  for (int i = 0; i < n; ++i) h[i] = i;
  double *x, *o;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&o, 64 * 8);
  cudaMemcpy(x, h.data(), n * 8, cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dim[1] = {(cuuint64_t)n}, str[1] = {8};
  cuuint32_t box[1] = {64}, es[1] = {1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, x, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int c : {0, 3, -5, 990}) {
    cudaMemset(o, 0xff, 512);
    k<<<1, 32, 512>>>(m, o, c, 0);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> g(64);
    cudaMemcpy(g.data(), o, 512, cudaMemcpyDeviceToHost);
    printf("c=%d err=%s first=%g %g last=%g\n", c, cudaGetErrorString(e), g[0], g[1], g[63]);
    if (e) return 1;
  }
  return 0;
}
