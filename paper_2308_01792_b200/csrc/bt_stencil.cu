// P1 constant-coefficient 15-point stencil apply (apply_stencil,
// operators.hpp:247-271), per-cell phase. The interface phase (replica sums
// and Dirichlet rows) is bt_interface.cu.
//
// Data path. A warp owns 30 consecutive columns i of one layer k of one
// macro-cell (lanes 0 and 31 are halo columns) and marches up to kMarchRows
// rows j. Each step needs three new rows at its columns — A(j+1) of layer k,
// B(j) of layer k+1 and C(j+1) of layer k-1, each one coalesced 256 B
// segment — loaded kAhead steps early into rotating registers (predicated
// to 0 outside the lattice, so lattice-boundary vertices need no special
// loads); neighbours i-1 / i+1 come from warp shuffles, and values reused by
// later steps stay in registers. Every x value is read from L2 once per layer
// that needs it (3x) and from HBM once.
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
constexpr int kMarchRows = 48;
constexpr int kMarchCols = 30;

__global__ void __launch_bounds__(kT, 2) k_stencil(const double* __restrict__ x, double* __restrict__ y,
                                                   const StencilCell* __restrict__ cells,
                                                   const int4* __restrict__ tasks, int ntasks, int w,
                                                   int64_t cell_slots) {
  __shared__ double sw[16][15];
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
  const bool out_lane = lane >= 1 && lane <= kMarchCols && i >= 0;
  const double* __restrict__ xc = x + (int64_t)cell * cell_slots + i;  // column i of every row
  double* __restrict__ yc = y + (int64_t)cell * cell_slots + i;
  const bool up = k + 1 <= n, dn = k >= 1;

  // row cursors of the loads for step s (j = j0 + s): A(j+1), B(j), C(j+1)
  int oA = row_start(w, j0 + 1, k), LA = w - k - j0 - 1;
  int oB = up ? row_start(w, j0, k + 1) : 0, LB = up ? w - k - 1 - j0 : 0;
  int oC = dn ? row_start(w, j0 + 1, k - 1) : 0, LC = dn ? w - k - j0 : 0;
  const bool col_ok = i >= 0;
#define BT_LOAD(dstA, dstB, dstC)                                  \
  do {                                                             \
    dstA = (col_ok && i < LA) ? __ldg(xc + oA) : 0.0;              \
    dstB = (col_ok && i < LB) ? __ldg(xc + oB) : 0.0;              \
    dstC = (col_ok && i < LC) ? __ldg(xc + oC) : 0.0;              \
    oA += LA;                                                      \
    --LA;                                                          \
    oB += LB;                                                      \
    LB = LB > 0 ? LB - 1 : 0;                                      \
    oC += LC;                                                      \
    LC = LC > 0 ? LC - 1 : 0;                                      \
  } while (0)
  double pA0, pB0, pC0, pA1, pB1, pC1, pA2, pB2, pC2;
  BT_LOAD(pA0, pB0, pC0);
  BT_LOAD(pA1, pB1, pC1);
  BT_LOAD(pA2, pB2, pC2);

  // register window at step j0: A(j0-1), A(j0), B(j0-1), C(j0)
  double Am1 = 0.0, A0 = 0.0, Bm1 = 0.0, C0 = 0.0;
  if (col_ok) {
    if (j0 >= 1 && i < w - k - j0 + 1) Am1 = __ldg(xc + row_start(w, j0 - 1, k));
    if (i < w - k - j0) A0 = __ldg(xc + row_start(w, j0, k));
    if (j0 >= 1 && up && i < w - k - j0) Bm1 = __ldg(xc + row_start(w, j0 - 1, k + 1));
    if (dn && i < w - k - j0 + 1) C0 = __ldg(xc + row_start(w, j0, k - 1));
  }
  double Am1p = __shfl_down_sync(0xffffffffu, Am1, 1);
  double A0p = __shfl_down_sync(0xffffffffu, A0, 1);
  double A0m = __shfl_up_sync(0xffffffffu, A0, 1);
  double Bm1p = __shfl_down_sync(0xffffffffu, Bm1, 1);
  double C0p = __shfl_down_sync(0xffffffffu, C0, 1);

  int oY = row_start(w, j0, k), LY = w - k - j0;
  const bool kin = k >= 1;
  int j = j0;
  // one march step consuming prefetched (a, b, c) and refilling them 3 steps ahead
#define BT_STEP(a, b, c, s)                                                                      \
  {                                                                                              \
    const double A1 = a, B0 = b, C1 = c;                                                         \
    if ((s) + 3 < nsteps) BT_LOAD(a, b, c);                                                      \
    const double A1m = __shfl_up_sync(0xffffffffu, A1, 1);                                       \
    const double A1p = __shfl_down_sync(0xffffffffu, A1, 1);                                     \
    const double B0m = __shfl_up_sync(0xffffffffu, B0, 1);                                       \
    const double B0p = __shfl_down_sync(0xffffffffu, B0, 1);                                     \
    const double C1m = __shfl_up_sync(0xffffffffu, C1, 1);                                       \
    const double C1p = __shfl_down_sync(0xffffffffu, C1, 1);                                     \
    if (out_lane && i < LY) {                                                                    \
      const double v[15] = {A0, A0p, A1, B0, Am1p, C0p, C1, Bm1p, A0m, Am1, C0, A1m, B0m, Bm1, C1m}; \
      double acc;                                                                                \
      if (i >= 1 && i <= LY - 2 && j >= 1 && kin) {                                              \
        acc = w0[0] * v[0];                                                                      \
        _Pragma("unroll") for (int d = 1; d < 15; ++d) acc = fma(w0[d], v[d], acc);              \
      } else {                                                                                   \
        const int z = (i == LY - 1 ? 1 : 0) | (i == 0 ? 2 : 0) | (j == 0 ? 4 : 0) | (kin ? 0 : 8); \
        acc = sw[z][0] * v[0];                                                                   \
        _Pragma("unroll") for (int d = 1; d < 15; ++d) acc = fma(sw[z][d], v[d], acc);           \
      }                                                                                          \
      yc[oY] = acc;                                                                              \
    }                                                                                            \
    oY += LY;                                                                                    \
    --LY;                                                                                        \
    ++j;                                                                                         \
    Am1 = A0;                                                                                    \
    Am1p = A0p;                                                                                  \
    A0 = A1;                                                                                     \
    A0p = A1p;                                                                                   \
    A0m = A1m;                                                                                   \
    Bm1 = B0;                                                                                    \
    Bm1p = B0p;                                                                                  \
    C0 = C1;                                                                                     \
    C0p = C1p;                                                                                   \
  }
  for (int s = 0; s < nsteps; s += 3) {
    BT_STEP(pA0, pB0, pC0, s)
    if (s + 1 >= nsteps) break;
    BT_STEP(pA1, pB1, pC1, s + 1)
    if (s + 2 >= nsteps) break;
    BT_STEP(pA2, pB2, pC2, s + 2)
  }
#undef BT_STEP
#undef BT_LOAD
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
  dim3 grid((st.ntasks + kW - 1) / kW, st.grid->mesh.n_cells());
  k_stencil<<<grid, kT, 0, s>>>(x, y, st.d_cells.p, st.d_tasks.p, st.ntasks, w, n_tet(w));
  count_launch();
  check_launch("k_stencil");
}

}  // namespace bt
