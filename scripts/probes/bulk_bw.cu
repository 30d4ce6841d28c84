// Probe: streaming bandwidth of cp.async.bulk (global -> shared, mbarrier
// complete_tx) as a function of copy size, copies per stage, ring depth and
// CTAs per SM; against a plain LDG streaming read. Each CTA streams its own
// contiguous slice of a 2 GiB buffer; one producer warp issues the copies of a
// stage (lanes 0..M-1, one copy each), one consumer warp waits on the stage's
// full barrier, touches one double per copy and releases the stage.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_bw bulk_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t a, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t p) {
  asm volatile("{\n .reg .pred q;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W;\n}\n" ::"r"(a),
               "r"(p)
               : "memory");
}

__global__ void k_bulk(const char* __restrict__ src, size_t slice, int B, int M, int S, int skew, double* out) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)S * M * (B + 128));
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(sa(full + s), 1);
      mbar_init(sa(empty + s), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const char* base = src + (size_t)blockIdx.x * slice;
  const size_t per_stage = (size_t)M * (B + skew);
  const int nst = (int)(slice / per_stage);
  double acc = 0;
  if (warp == 0) {
    for (int st = 0; st < nst; ++st) {
      const int slot = st % S;
      const uint32_t ph = (st / S) & 1;
      mbar_wait(sa(empty + slot), ph ^ 1);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(full + slot)), "r"(M * B)
                     : "memory");
      __syncwarp();
      for (int c = lane; c < M; c += 32) {
        const char* g = base + (size_t)st * per_stage + (size_t)c * (B + skew) + (skew ? 16 : 0);
        const uint32_t d = sa(sm + ((size_t)slot * M + c) * (B + 128));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
                     "l"(g), "r"(B), "r"(sa(full + slot))
                     : "memory");
      }
    }
  } else if (warp == 1) {
    for (int st = 0; st < nst; ++st) {
      const int slot = st % S;
      const uint32_t ph = (st / S) & 1;
      mbar_wait(sa(full + slot), ph);
      for (int c = lane; c < M; c += 32) acc += *reinterpret_cast<const double*>(sm + ((size_t)slot * M + c) * (B + 128));
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sa(empty + slot)) : "memory");
    }
    if (acc == 12345.678) out[0] = acc;
  }
}

__global__ void k_ldg(const double2* __restrict__ src, size_t n, double* out) {
  double2 acc = make_double2(0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = __ldg(src + i);
    acc.x += v.x;
    acc.y += v.y;
  }
  if (acc.x == 12345.678) out[0] = acc.y;
}

int main() {
  const size_t bytes = size_t(2) << 30;
  char* buf;
  double* out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(buf, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  {
    k_ldg<<<sms * 8, 256>>>((const double2*)buf, bytes / 16, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_ldg<<<sms * 8, 256>>>((const double2*)buf, bytes / 16, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG.128 stream: %.0f GB/s\n", 5.0 * bytes / (ms * 1e-3) / 1e9);
  }
  struct Cfg {
    int B, M, S, per_sm, skew;
  } cfgs[] = {
      {1024, 18, 6, 2, 0},   {1024, 18, 6, 2, 16},  {1024, 18, 12, 1, 16}, {1024, 32, 6, 1, 16},
      {512, 32, 6, 2, 16},   {2048, 16, 6, 2, 16},  {4096, 4, 6, 2, 16},   {4096, 8, 6, 2, 0},
      {16384, 1, 6, 2, 0},   {16384, 1, 12, 1, 0},  {32768, 1, 6, 1, 0},   {1024, 4, 24, 2, 16},
      {1024, 1, 32, 4, 16},  {8192, 2, 6, 2, 16},   {1024, 18, 3, 4, 16},  {256, 32, 8, 4, 16},
  };
  for (const Cfg& c : cfgs) {
    const size_t smem = (size_t)c.S * c.M * (c.B + 128) + 2 * c.S * 8;
    if (smem > 220 * 1024) continue;
    const int grid = sms * c.per_sm;
    const size_t slice = bytes / grid / 4096 * 4096 - 4096;
    k_bulk<<<grid, 64, smem>>>(buf, slice, c.B, c.M, c.S, c.skew, out);
    cudaEventRecord(a);
    const int reps = 3;
    for (int r = 0; r < reps; ++r) k_bulk<<<grid, 64, smem>>>(buf, slice, c.B, c.M, c.S, c.skew, out);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const size_t per_stage = (size_t)c.M * (c.B + c.skew);
    const double moved = (double)reps * grid * (double)(slice / per_stage) * c.M * c.B;
    printf("bulk B=%5d M=%2d S=%2d cta/sm=%d skew=%2d inflight/SM=%6zu B: %.0f GB/s %s\n", c.B, c.M, c.S, c.per_sm,
           c.skew, (size_t)c.per_sm * (c.S) * c.M * c.B, moved / (ms * 1e-3) / 1e9,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
