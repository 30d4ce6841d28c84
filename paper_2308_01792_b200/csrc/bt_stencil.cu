// P1 constant-coefficient 15-point stencil apply (apply_stencil,
// operators.hpp:247-271), per-cell phase. The interface phase (replica sums
// and Dirichlet rows) is bt_interface.cu.
//
// Data path. A warp owns 30 consecutive columns i of one layer k of one
// macro-cell (lanes 0 and 31 are halo columns) and marches up to kMarchRows
// rows j. Each step needs three new rows at its columns — A(j+1) of layer k,
// B(j) of layer k+1 and C(j+1) of layer k-1, each one coalesced 256 B
// segment — loaded two steps early into registers (predicated to 0 outside
// the lattice, so lattice-boundary vertices need no special loads);
// neighbours i-1 / i+1 come from warp shuffles. The march is unrolled by two
// over two alternating window sets, so the sliding window costs no moves.
// Every x value is read from L2 once per layer that needs it (3x) and from
// HBM once.
//
// Rows. The host splits every (layer, column block) march into fast rows and
// a few general rows. Fast rows (k >= 1, j >= 1, and row length >= 3 in
// column block 0) contain interior vertices plus at most the diagonal-face
// vertex (i = row end) and the i = 0 vertex; k_stencil_fast evaluates the
// merged row (compute_stencil operators.hpp:204-221) in its symmetric
// 8-weight form (W[d] == W[-d] bitwise, checked on the host) and switches the
// two face vertices to their zero-set-typed partial rows (per-cell part of
// partial_row_apply, operators.hpp:78-96) by 7-term corrections selected per
// lane — no per-lane branches. All weights are kernel parameters, so they
// reach the DFMAs as uniform-register operands. General rows (layer 0, row
// 0, the last two rows of column block 0) go through k_stencil_general, which
// reads the typed rows from shared memory; it is also the fallback for
// tables that fail the fast-path checks.
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

// directions whose weight differs between the interior row and the typed row
// of the diagonal face (zero set {0}) / the face i = 0 (zero set {1});
// structural (which micro-cells are missing), verified on the host.
constexpr int kDiagDirs[7] = {0, 4, 5, 6, 11, 12, 13};
constexpr int kI0Dirs[7] = {0, 2, 3, 6, 9, 10, 13};

template <int kMaxC>
struct FastParams {
  double w[kMaxC][8];   // symmetric interior row: centre + 7 direction pairs
  double dd[kMaxC][7];  // diagonal-face correction on kDiagDirs
  double di[kMaxC][7];  // i = 0 face correction on kI0Dirs
};
constexpr int kMaxCells = 176;  // 176 * 22 * 8 B = 30 KB of kernel parameters

struct Win {  // row j of layer k (a), row j-1 of layer k+1 (b), row j of layer k-1 (c)
  double a, ap, am, b, bp, c, cp;
};

template <int kMaxC>
__global__ void __launch_bounds__(kT, 3) k_stencil_fast(const double* __restrict__ x, double* __restrict__ y,
                                                        const int4* __restrict__ tasks, int ntasks, int w,
                                                        int64_t cell_slots, int cell0,
                                                        const __grid_constant__ FastParams<kMaxC> fp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int task = blockIdx.x * kW + warp;
  if (task >= ntasks) return;
  const int cell = cell0 + blockIdx.y;
  const double* W = fp.w[blockIdx.y];
  const double* DD = fp.dd[blockIdx.y];
  const double* DI = fp.di[blockIdx.y];
  const int4 tk = tasks[task];
  const int k = tk.x, blk = tk.y, j0 = tk.z, j1 = tk.w;  // k >= 1, j0 >= 1 by construction
  const int n = w - 1;
  const int i = kMarchCols * blk + lane - 1;
  const bool out_lane = lane >= 1 && lane <= kMarchCols && i >= 0;
  const bool col_ok = i >= 0;
  const double* __restrict__ xc = x + (int64_t)cell * cell_slots + i;  // column i of every row
  const bool up = k + 1 <= n;

  // load cursors (lane's column) for the rows consumed at row j: A(j+1),
  // B(j), C(j+1); remaining lengths <= 0 (or an absent layer k+1) load 0.
  const double* __restrict__ qA = xc + row_start(w, j0 + 1, k);
  const double* __restrict__ qB = xc + (up ? row_start(w, j0, k + 1) : 0);
  const double* __restrict__ qC = xc + row_start(w, j0 + 1, k - 1);
  int rA = w - k - j0 - 1, rB = w - k - 1 - j0, rC = w - k - j0;  // row lengths
  int LA = col_ok ? rA - i : -1;
  int LB = (col_ok && up) ? rB - i : -1;
  int LC = col_ok ? rC - i : -1;
  auto load3 = [&](double& pa, double& pb, double& pc, bool live) {
    pa = (live && LA > 0) ? __ldg(qA) : 0.0;
    pb = (live && LB > 0) ? __ldg(qB) : 0.0;
    pc = (live && LC > 0) ? __ldg(qC) : 0.0;
    qA += rA;
    qB += rB;
    qC += rC;
    --rA;
    --rB;
    --rC;
    --LA;
    --LB;
    --LC;
  };
  double pa0, pb0, pc0, pa1, pb1, pc1;
  load3(pa0, pb0, pc0, true);
  load3(pa1, pb1, pc1, j0 + 1 < j1);

  // window sets: X = row j0 (current), Y = row j0 - 1 (previous)
  Win X, Y;
  {
    double am1 = 0.0, a0 = 0.0, bm1 = 0.0, c0 = 0.0;
    if (col_ok) {
      if (i < w - k - j0 + 1) am1 = __ldg(xc + row_start(w, j0 - 1, k));
      if (i < w - k - j0) a0 = __ldg(xc + row_start(w, j0, k));
      if (up && i < w - k - j0) bm1 = __ldg(xc + row_start(w, j0 - 1, k + 1));
      if (i < w - k - j0 + 1) c0 = __ldg(xc + row_start(w, j0, k - 1));
    }
    X.a = a0;
    X.ap = __shfl_down_sync(0xffffffffu, a0, 1);
    X.am = __shfl_up_sync(0xffffffffu, a0, 1);
    X.b = bm1;
    X.bp = __shfl_down_sync(0xffffffffu, bm1, 1);
    X.c = c0;
    X.cp = __shfl_down_sync(0xffffffffu, c0, 1);
    Y.a = am1;
    Y.ap = __shfl_down_sync(0xffffffffu, am1, 1);
  }

  int LY = w - k - j0;  // length of the output row
  double* __restrict__ py = y + (int64_t)cell * cell_slots + i + row_start(w, j0, k);
  const bool blk0 = blk == 0;
  const int colend = kMarchCols * blk + kMarchCols;  // LY <= colend: the row ends inside this warp
  int j = j0;
#define BT_STEP(cur, prv, pa, pb, pc)                                                               \
  {                                                                                                 \
    const double A1 = pa, B0 = pb, C1 = pc;                                                         \
    const double A1m = __shfl_up_sync(0xffffffffu, A1, 1);                                          \
    const double A1p = __shfl_down_sync(0xffffffffu, A1, 1);                                        \
    const double B0m = __shfl_up_sync(0xffffffffu, B0, 1);                                          \
    const double B0p = __shfl_down_sync(0xffffffffu, B0, 1);                                        \
    const double C1m = __shfl_up_sync(0xffffffffu, C1, 1);                                          \
    const double C1p = __shfl_down_sync(0xffffffffu, C1, 1);                                        \
    if (out_lane && i < LY) {                                                                       \
      double acc = W[0] * cur.a;                                                                    \
      acc = fma(W[1], cur.ap + cur.am, acc);                                                        \
      acc = fma(W[2], A1 + prv.a, acc);                                                             \
      acc = fma(W[3], B0 + cur.c, acc);                                                             \
      acc = fma(W[4], prv.ap + A1m, acc);                                                           \
      acc = fma(W[5], cur.cp + B0m, acc);                                                           \
      acc = fma(W[6], C1 + cur.b, acc);                                                             \
      acc = fma(W[7], cur.bp + C1m, acc);                                                           \
      if (LY <= colend) { /* row end in this warp: diagonal face, dirs 0, 4, 5, 6, 11, 12, 13 */     \
        double dg = fma(DD[0], cur.a, acc);                                                         \
        dg = fma(DD[1], prv.ap, dg);                                                                \
        dg = fma(DD[2], cur.cp, dg);                                                                \
        dg = fma(DD[3], C1, dg);                                                                    \
        dg = fma(DD[4], A1m, dg);                                                                   \
        dg = fma(DD[5], B0m, dg);                                                                   \
        dg = fma(DD[6], cur.b, dg);                                                                 \
        acc = (i == LY - 1) ? dg : acc;                                                             \
      }                                                                                             \
      if (blk0) { /* face i = 0 (zero set {1}): dirs 0, 2, 3, 6, 9, 10, 13 */                       \
        double f0 = fma(DI[0], cur.a, acc);                                                         \
        f0 = fma(DI[1], A1, f0);                                                                    \
        f0 = fma(DI[2], B0, f0);                                                                    \
        f0 = fma(DI[3], C1, f0);                                                                    \
        f0 = fma(DI[4], prv.a, f0);                                                                 \
        f0 = fma(DI[5], cur.c, f0);                                                                 \
        f0 = fma(DI[6], cur.b, f0);                                                                 \
        acc = (i == 0) ? f0 : acc;                                                                  \
      }                                                                                             \
      *py = acc;                                                                                    \
    }                                                                                               \
    py += LY;                                                                                       \
    --LY;                                                                                           \
    ++j;                                                                                            \
    prv.a = A1;                                                                                     \
    prv.ap = A1p;                                                                                   \
    prv.am = A1m;                                                                                   \
    prv.b = B0;                                                                                     \
    prv.bp = B0p;                                                                                   \
    prv.c = C1;                                                                                     \
    prv.cp = C1p;                                                                                   \
    load3(pa, pb, pc, j + 1 < j1); /* refill for row j + 2 once A1/B0/C1 are dead */                \
  }
  while (true) {
    BT_STEP(X, Y, pa0, pb0, pc0)
    if (j >= j1) break;
    BT_STEP(Y, X, pa1, pb1, pc1)
    if (j >= j1) break;
  }
#undef BT_STEP
}

// Any rows of the march schedule, every row read from the zero-set-typed
// table in shared memory (interior vertices use type 0 = the merged row).
__global__ void __launch_bounds__(kT) k_stencil_general(const double* __restrict__ x, double* __restrict__ y,
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
  const int4 tk = tasks[task];
  const int k = tk.x, j0 = tk.z, j1 = tk.w, n = w - 1;
  const int i = kMarchCols * tk.y + lane - 1;
  const bool out_lane = lane >= 1 && lane <= kMarchCols && i >= 0;
  const double* __restrict__ xc = x + (int64_t)cell * cell_slots;
  double* __restrict__ yc = y + (int64_t)cell * cell_slots;
  auto at = [&](int jj, int kk) -> double {  // x at column i of row (jj, kk), 0 outside
    if (i < 0 || jj < 0 || kk < 0 || kk > n || i >= w - kk - jj) return 0.0;
    return __ldg(xc + row_start(w, jj, kk) + i);
  };
  for (int j = j0; j < j1; ++j) {
    const double A0 = at(j, k), Am1 = at(j - 1, k), A1 = at(j + 1, k), B0 = at(j, k + 1), Bm1 = at(j - 1, k + 1);
    const double C0 = at(j, k - 1), C1 = at(j + 1, k - 1);
    const double A0p = __shfl_down_sync(0xffffffffu, A0, 1), A0m = __shfl_up_sync(0xffffffffu, A0, 1);
    const double Am1p = __shfl_down_sync(0xffffffffu, Am1, 1), A1m = __shfl_up_sync(0xffffffffu, A1, 1);
    const double B0m = __shfl_up_sync(0xffffffffu, B0, 1), Bm1p = __shfl_down_sync(0xffffffffu, Bm1, 1);
    const double C0p = __shfl_down_sync(0xffffffffu, C0, 1), C1m = __shfl_up_sync(0xffffffffu, C1, 1);
    const int LY = w - k - j;
    if (out_lane && i < LY) {
      const double v[15] = {A0, A0p, A1, B0, Am1p, C0p, C1, Bm1p, A0m, Am1, C0, A1m, B0m, Bm1, C1m};
      const bool interior = i >= 1 && i <= LY - 2 && j >= 1 && k >= 1;
      const int z = interior ? 0 : ((i == LY - 1 ? 1 : 0) | (i == 0 ? 2 : 0) | (j == 0 ? 4 : 0) | (k == 0 ? 8 : 0));
      double acc = sw[z][0] * v[0];
#pragma unroll
      for (int d = 1; d < 15; ++d) acc = fma(sw[z][d], v[d], acc);
      yc[row_start(w, j, k) + i] = acc;
    }
  }
}

}  // namespace

void init_stencil_tasks(bt_stencil& st) {
  const int w = (1 << st.level) + 1;
  std::vector<int4> fast, gen, all;
  auto push = [](std::vector<int4>& v, int k, int b, int a, int e) {
    for (int j0 = a; j0 < e; j0 += kMarchRows) v.push_back(make_int4(k, b, j0, std::min(j0 + kMarchRows, e)));
  };
  for (int k = 0; k < w; ++k)
    for (int b = 0; kMarchCols * b < w - k; ++b) {
      const int jmax = w - k - kMarchCols * b;  // rows of this column block
      push(all, k, b, 0, jmax);
      if (k == 0) {
        push(gen, k, b, 0, jmax);
        continue;
      }
      push(gen, k, b, 0, 1);                                        // row 0
      const int fe = b == 0 ? std::max(1, std::min(jmax, w - k - 2)) : jmax;  // block 0: row length >= 3
      push(fast, k, b, 1, fe);
      push(gen, k, b, fe, jmax);
    }
  st.ntasks = (int)fast.size();
  st.d_tasks.upload(fast);
  st.ngtasks = (int)gen.size();
  st.d_gtasks.upload(gen);
  st.natasks = (int)all.size();
  st.d_atasks.upload(all);
  // Fast path preconditions: bitwise-symmetric merged rows, and face rows
  // that differ from them only on the structural correction directions
  // (neighbours outside the lattice load as 0 and are exempt).
  st.symmetric = true;
  const int nc = st.grid->mesh.n_cells();
  std::vector<StencilCell> cells(nc);
  BT_CUDA(cudaMemcpy(cells.data(), st.d_cells.p, sizeof(StencilCell) * nc, cudaMemcpyDeviceToHost));
  static const int kOutside[3][4] = {{0, 0, 0, 0}, {1, 2, 3, 7}, {8, 11, 12, 14}};
  st.fast.assign(22 * (size_t)nc, 0.0);
  for (int c = 0; c < nc; ++c) {
    const auto& r = st.rows[c];
    for (int d = 1; d <= 7; ++d) st.symmetric = st.symmetric && r[d] == r[d + 7];
    for (int z : {1, 2}) {
      const int* dirs = z == 1 ? kDiagDirs : kI0Dirs;
      for (int d = 0; d < 15; ++d) {
        bool exempt = false;
        for (int q = 0; q < 7; ++q) exempt = exempt || dirs[q] == d;
        for (int q = 0; q < 4; ++q) exempt = exempt || kOutside[z][q] == d;
        if (!exempt && cells[c].w[z][d] != r[d]) st.symmetric = false;
      }
    }
    double* f = &st.fast[22 * (size_t)c];
    for (int d = 0; d < 8; ++d) f[d] = r[d];
    for (int q = 0; q < 7; ++q) {
      f[8 + q] = cells[c].w[1][kDiagDirs[q]] - r[kDiagDirs[q]];
      f[15 + q] = cells[c].w[2][kI0Dirs[q]] - r[kI0Dirs[q]];
    }
  }
}

void launch_stencil(const bt_stencil& st, const double* x, double* y, cudaStream_t s) {
  const int w = (1 << st.level) + 1;
  const int nc = st.grid->mesh.n_cells();
  const int64_t cs = n_tet(w);
  if (!st.symmetric) {
    k_stencil_general<<<dim3((st.natasks + kW - 1) / kW, nc), kT, 0, s>>>(x, y, st.d_cells.p, st.d_atasks.p,
                                                                          st.natasks, w, cs);
    count_launch();
    check_launch("k_stencil_general");
    return;
  }
  if (st.ngtasks) {
    k_stencil_general<<<dim3((st.ngtasks + kW - 1) / kW, nc), kT, 0, s>>>(x, y, st.d_cells.p, st.d_gtasks.p,
                                                                          st.ngtasks, w, cs);
    count_launch();
  }
  static FastParams<kMaxCells> fp;
  for (int c0 = 0; c0 < nc && st.ntasks; c0 += kMaxCells) {
    const int cnt = std::min(kMaxCells, nc - c0);
    for (int c = 0; c < cnt; ++c) {
      const double* f = &st.fast[22 * (size_t)(c0 + c)];
      for (int d = 0; d < 8; ++d) fp.w[c][d] = f[d];
      for (int q = 0; q < 7; ++q) {
        fp.dd[c][q] = f[8 + q];
        fp.di[c][q] = f[15 + q];
      }
    }
    k_stencil_fast<kMaxCells><<<dim3((st.ntasks + kW - 1) / kW, cnt), kT, 0, s>>>(x, y, st.d_tasks.p, st.ntasks, w,
                                                                                 cs, c0, fp);
    count_launch();
  }
  check_launch("k_stencil");
}

}  // namespace bt
