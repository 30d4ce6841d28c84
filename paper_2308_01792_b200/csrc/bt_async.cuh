// cp.async helpers shared by the staged kernels (k_stencil_fast, k_n1e1_fast)
#pragma once
#include <cstdint>

namespace bt {
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// 8-byte global -> shared copy (per lane; lands at a fixed place whatever the
// source's 16-byte alignment)
__device__ __forceinline__ void cp8(uint32_t dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
// ... or 8 zero bytes when !valid (src is not read)
__device__ __forceinline__ void cp8z(uint32_t dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
}  // namespace bt
