// P1 constant-coefficient 15-point stencil apply (apply_stencil,
// operators.hpp:247-271), per-cell phase. The interface phase (replica sums
// and Dirichlet rows) is bt_interface.cu.
//
// Data path. A warp owns 30 consecutive columns i of one layer k of one
// macro-cell (lanes 0 and 31 are halo columns) and marches up to kMarchRows
// rows j. Each step needs three new rows at its columns — A(j+1) of layer k,
// B(j) of layer k+1 and C(j+1) of layer k-1, each one coalesced 256 B
// segment — which are staged by cp.async into a per-warp shared-memory ring
// kStages-1 steps ahead (zero-filled outside the lattice, so lattice-boundary
// vertices need no special loads). Neighbours i-1 / i+1 come from the staged
// rows; values reused by the next steps stay in registers. Every x value is
// fetched from L2 once per layer that needs it (3x) and from HBM once.
//
// Rows: interior vertices use the merged row (compute_stencil
// operators.hpp:204-221) held in registers; lattice-boundary vertices use
// their zero-set-typed partial row (per-cell part of partial_row_apply,
// operators.hpp:78-96) from shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "bt_internal.hpp"

namespace bt {

namespace {
constexpr int kT = 256;
constexpr int kW = kT / 32;
constexpr int kMarchRows = 32;
constexpr int kMarchCols = 30;
constexpr int kStages = 4;
constexpr int kRowPad = 34;                 // staged row: 32 lanes + slack, keeps rows 16 B aligned
constexpr int kStageD = 3 * kRowPad;        // doubles per stage
constexpr int kRingD = kStages * kStageD;   // doubles per warp

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(kT, 2) k_stencil(const double* __restrict__ x, double* __restrict__ y,
                                                   const StencilCell* __restrict__ cells,
                                                   const int4* __restrict__ tasks, int ntasks, int w,
                                                   int64_t cell_slots) {
  __shared__ double sw[16][15];
  extern __shared__ __align__(16) double ring_all[];
  const int cell = blockIdx.y;
  {
    const double* src = cells[cell].w[0];
    for (int q = threadIdx.x; q < 16 * 15; q += blockDim.x) sw[q / 15][q % 15] = src[q];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int task = blockIdx.x * kW + warp;
  if (task >= ntasks) return;
  double w0[15];
#pragma unroll
  for (int d = 0; d < 15; ++d) w0[d] = sw[0][d];
  const int4 tk = tasks[task];
  const int k = tk.x, j0 = tk.z, nsteps = tk.w - tk.z;
  const int n = w - 1;
  const int i = kMarchCols * tk.y + lane - 1;
  const bool out_lane = lane >= 1 && lane <= kMarchCols;
  const double* __restrict__ xc = x + (int64_t)cell * cell_slots;
  double* __restrict__ yc = y + (int64_t)cell * cell_slots;
  double* ring = ring_all + warp * kRingD;
  const bool up = k + 1 <= n, dn = k >= 1;

  // issue cursors: rows staged for step q are A(j+1), B(j), C(j+1), j = j0 + q
  int iA = row_start(w, j0 + 1, k), iLA = w - k - j0 - 1;
  int iB = up ? row_start(w, j0, k + 1) : 0, iLB = w - k - 1 - j0;
  int iC = dn ? row_start(w, j0 + 1, k - 1) : 0, iLC = w - k - j0;
  auto issue = [&](int stage) {
    double* st = ring + stage * kStageD + 1;  // +1: st[lane - 1] stays in-bounds
    const bool vA = i >= 0 && i < iLA, vB = up && i >= 0 && i < iLB, vC = dn && i >= 0 && i < iLC;
    cp_async8(st + lane, vA ? xc + iA + i : xc, vA);
    cp_async8(st + kRowPad + lane, vB ? xc + iB + i : xc, vB);
    cp_async8(st + 2 * kRowPad + lane, vC ? xc + iC + i : xc, vC);
    cp_commit();
    iA += iLA;
    --iLA;
    iB += iLB;
    --iLB;
    iC += iLC;
    --iLC;
  };
#pragma unroll
  for (int q = 0; q < kStages - 1; ++q) {
    if (q < nsteps) issue(q);
    else cp_commit();
  }

  // register window at step j0: A(j0-1), A(j0), B(j0-1), C(j0) and shifts
  auto ld = [&](bool ok, int rs, int len) -> double { return (ok && i >= 0 && i < len) ? __ldg(xc + rs + i) : 0.0; };
  double Am1 = j0 >= 1 ? ld(true, row_start(w, j0 - 1, k), w - k - j0 + 1) : 0.0;
  double A0 = ld(true, row_start(w, j0, k), w - k - j0);
  double Bm1 = (j0 >= 1 && up) ? ld(true, row_start(w, j0 - 1, k + 1), w - k - j0) : 0.0;
  double C0 = dn ? ld(true, row_start(w, j0, k - 1), w - k - j0 + 1) : 0.0;
  double Am1p = __shfl_down_sync(0xffffffffu, Am1, 1);
  double A0p = __shfl_down_sync(0xffffffffu, A0, 1);
  double A0m = __shfl_up_sync(0xffffffffu, A0, 1);
  double Bm1p = __shfl_down_sync(0xffffffffu, Bm1, 1);
  double C0p = __shfl_down_sync(0xffffffffu, C0, 1);

  int sY = row_start(w, j0, k), LY = w - k - j0;
  const bool kin = k >= 1;
#pragma unroll 2
  for (int q = 0; q < nsteps; ++q) {
    const int j = j0 + q;
    cp_wait<kStages - 2>();
    __syncwarp();
    if (q + kStages - 1 < nsteps) issue((q + kStages - 1) % kStages);
    else cp_commit();
    const double* st = ring + (q % kStages) * kStageD + 1 + lane;
    const double A1m = st[-1], A1 = st[0], A1p = st[1];
    const double B0m = st[kRowPad - 1], B0 = st[kRowPad], B0p = st[kRowPad + 1];
    const double C1m = st[2 * kRowPad - 1], C1 = st[2 * kRowPad], C1p = st[2 * kRowPad + 1];
    if (out_lane && i < LY) {
      // kStencilDirs order (operators.hpp:22-26)
      const double v[15] = {A0, A0p, A1, B0, Am1p, C0p, C1, Bm1p, A0m, Am1, C0, A1m, B0m, Bm1, C1m};
      double acc;
      if (i >= 1 && i <= LY - 2 && j >= 1 && kin) {
        acc = w0[0] * v[0];
#pragma unroll
        for (int d = 1; d < 15; ++d) acc = fma(w0[d], v[d], acc);
      } else {
        const int z = (i == LY - 1 ? 1 : 0) | (i == 0 ? 2 : 0) | (j == 0 ? 4 : 0) | (kin ? 0 : 8);
        acc = sw[z][0] * v[0];
#pragma unroll
        for (int d = 1; d < 15; ++d) acc = fma(sw[z][d], v[d], acc);
      }
      yc[sY + i] = acc;
    }
    sY += LY;
    --LY;
    Am1 = A0;
    Am1p = A0p;
    A0 = A1;
    A0p = A1p;
    A0m = A1m;
    Bm1 = B0;
    Bm1p = B0p;
    C0 = C1;
    C0p = C1p;
  }
  cp_wait<0>();
}

}  // namespace

void init_stencil_tasks(bt_stencil& st) {
  const int w = (1 << st.level) + 1;
  std::vector<int4> t;
  for (int k = 0; k < w; ++k)
    for (int b = 0; kMarchCols * b < w - k; ++b) {
      const int jmax = w - k - kMarchCols * b;
      for (int j0 = 0; j0 < jmax; j0 += kMarchRows) t.push_back(make_int4(k, b, j0, std::min(j0 + kMarchRows, jmax)));
    }
  st.ntasks = (int)t.size();
  st.d_tasks.upload(t);
}

void launch_stencil(const bt_stencil& st, const double* x, double* y, cudaStream_t s) {
  const int w = (1 << st.level) + 1;
  const size_t smem = sizeof(double) * (kW * kRingD + 2);
  static bool attr = false;
  if (!attr) {
    BT_CUDA(cudaFuncSetAttribute(k_stencil, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  dim3 grid((st.ntasks + kW - 1) / kW, st.grid->mesh.n_cells());
  k_stencil<<<grid, kT, smem, s>>>(x, y, st.d_cells.p, st.d_tasks.p, st.ntasks, w, n_tet(w));
  count_launch();
  check_launch("k_stencil");
}

}  // namespace bt
