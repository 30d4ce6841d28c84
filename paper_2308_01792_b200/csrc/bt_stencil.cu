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
// Rows: interior vertices use the merged row (compute_stencil
// operators.hpp:204-221) from registers — as 8 symmetric weights when the
// row is symmetric (W[d] == W[-d] bitwise, checked on the host; true for
// every mesh tested) — and lattice-boundary vertices use their
// zero-set-typed partial row (per-cell part of partial_row_apply,
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

struct Win {  // row j of layer k (a), row j-1 of layer k+1 (b), row j of layer k-1 (c)
  double a, ap, am, b, bp, c, cp;
};

// Merged interior rows of up to kMaxC cells, passed by value so they live in
// the launch's constant bank and reach the DFMAs as uniform-register operands
// (no vector registers, no shared-memory traffic).
template <int NW, int kMaxC>
struct RowParams {
  double w[kMaxC][NW];
};
constexpr int kMaxCellsSym = 480;   // 480 * 8 * 8 B = 30 KB of kernel parameters
constexpr int kMaxCellsFull = 256;  // 256 * 15 * 8 B

template <bool kSym, int kMaxC>
__global__ void __launch_bounds__(kT, 3) k_stencil(const double* __restrict__ x, double* __restrict__ y,
                                                   const StencilCell* __restrict__ cells,
                                                   const int4* __restrict__ tasks, int ntasks, int w,
                                                   int64_t cell_slots, int cell0,
                                                   const __grid_constant__ RowParams<kSym ? 8 : 15, kMaxC> rp) {
  __shared__ double sw[16][15];
  const int cell = cell0 + blockIdx.y;
  {
    const double* src = cells[cell].w[0];
    for (int q = threadIdx.x; q < 16 * 15; q += blockDim.x) sw[q / 15][q % 15] = src[q];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int task = blockIdx.x * kW + warp;
  if (task >= ntasks) return;
  constexpr int kNW = kSym ? 8 : 15;
  const double* w0 = rp.w[blockIdx.y];
  const int4 tk = tasks[task];
  const int k = tk.x, j0 = tk.z, nsteps = tk.w - tk.z;
  const int n = w - 1;
  const int i = kMarchCols * tk.y + lane - 1;
  const bool out_lane = lane >= 1 && lane <= kMarchCols && i >= 0;
  const bool col_ok = i >= 0;
  const double* __restrict__ xc = x + (int64_t)cell * cell_slots + i;  // column i of every row
  double* __restrict__ yc = y + (int64_t)cell * cell_slots + i;
  const bool up = k + 1 <= n, dn = k >= 1;

  // cursors (lane's column) of the rows loaded for step s (j = j0 + s):
  // A(j+1), B(j), C(j+1); a row with length <= i (or absent: -1) loads 0.
  const double* __restrict__ qA = xc + row_start(w, j0 + 1, k);
  const double* __restrict__ qB = xc + (up ? row_start(w, j0, k + 1) : 0);
  const double* __restrict__ qC = xc + (dn ? row_start(w, j0 + 1, k - 1) : 0);
  int LA = col_ok ? w - k - j0 - 1 - i : -1;  // remaining length beyond column i
  int LB = (col_ok && up) ? w - k - 1 - j0 - i : -1;
  int LC = (col_ok && dn) ? w - k - j0 - i : -1;
  int rA = w - k - j0 - 1, rB = w - k - 1 - j0, rC = w - k - j0;  // row lengths
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
  load3(pa1, pb1, pc1, nsteps > 1);

  // window sets: X = row j0 (current), Y = row j0 - 1 (previous)
  Win X, Y;
  {
    double am1 = 0.0, a0 = 0.0, bm1 = 0.0, c0 = 0.0;
    if (col_ok) {
      if (j0 >= 1 && i < w - k - j0 + 1) am1 = __ldg(xc + row_start(w, j0 - 1, k));
      if (i < w - k - j0) a0 = __ldg(xc + row_start(w, j0, k));
      if (j0 >= 1 && up && i < w - k - j0) bm1 = __ldg(xc + row_start(w, j0 - 1, k + 1));
      if (dn && i < w - k - j0 + 1) c0 = __ldg(xc + row_start(w, j0, k - 1));
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

  int oY = row_start(w, j0, k), LY = w - k - j0;
  const bool kin = k >= 1;
  int j = j0;
  // one step: output row j from (cur, prv.a/ap) and the prefetched rows;
  // prv is overwritten with row j+1 and becomes the next step's current set.
#define BT_STEP(cur, prv, pa, pb, pc, s)                                                            \
  {                                                                                                 \
    const double A1 = pa, B0 = pb, C1 = pc;                                                         \
    const double A1m = __shfl_up_sync(0xffffffffu, A1, 1);                                          \
    const double A1p = __shfl_down_sync(0xffffffffu, A1, 1);                                        \
    const double B0m = __shfl_up_sync(0xffffffffu, B0, 1);                                          \
    const double B0p = __shfl_down_sync(0xffffffffu, B0, 1);                                        \
    const double C1m = __shfl_up_sync(0xffffffffu, C1, 1);                                          \
    const double C1p = __shfl_down_sync(0xffffffffu, C1, 1);                                        \
    if (out_lane && i < LY) {                                                                       \
      double acc;                                                                                   \
      if (i >= 1 && i <= LY - 2 && j >= 1 && kin) {                                                 \
        if (kSym) {                                                                                 \
          /* pairs (d, d+7) of kStencilDirs share one weight */                                     \
          acc = w0[0] * cur.a;                                                                      \
          acc = fma(w0[1], cur.ap + cur.am, acc);                                                   \
          acc = fma(w0[2], A1 + prv.a, acc);                                                        \
          acc = fma(w0[3], B0 + cur.c, acc);                                                        \
          acc = fma(w0[4], prv.ap + A1m, acc);                                                      \
          acc = fma(w0[5], cur.cp + B0m, acc);                                                      \
          acc = fma(w0[6], C1 + cur.b, acc);                                                        \
          acc = fma(w0[7], cur.bp + C1m, acc);                                                      \
        } else {                                                                                    \
          const double v[15] = {cur.a, cur.ap, A1,    B0,  prv.ap, cur.cp, C1, cur.bp,              \
                                cur.am, prv.a, cur.c, A1m, B0m,    cur.b,  C1m};                    \
          acc = w0[0] * v[0];                                                                       \
          _Pragma("unroll") for (int d = 1; d < kNW; ++d) acc = fma(w0[d], v[d], acc);              \
        }                                                                                           \
      } else {                                                                                      \
        const double v[15] = {cur.a, cur.ap, A1,    B0,  prv.ap, cur.cp, C1, cur.bp,                \
                              cur.am, prv.a, cur.c, A1m, B0m,    cur.b,  C1m};                      \
        const int z = (i == LY - 1 ? 1 : 0) | (i == 0 ? 2 : 0) | (j == 0 ? 4 : 0) | (kin ? 0 : 8);  \
        acc = sw[z][0] * v[0];                                                                      \
        _Pragma("unroll") for (int d = 1; d < 15; ++d) acc = fma(sw[z][d], v[d], acc);              \
      }                                                                                             \
      yc[oY] = acc;                                                                                 \
    }                                                                                               \
    oY += LY;                                                                                       \
    --LY;                                                                                           \
    ++j;                                                                                            \
    prv.a = A1;                                                                                     \
    prv.ap = A1p;                                                                                   \
    prv.am = A1m;                                                                                   \
    prv.b = B0;                                                                                     \
    prv.bp = B0p;                                                                                   \
    prv.c = C1;                                                                                     \
    prv.cp = C1p;                                                                                   \
    load3(pa, pb, pc, (s) + 2 < nsteps); /* refill for step s + 2 once A1/B0/C1 are dead */         \
  }
  for (int s = 0; s < nsteps; s += 2) {
    BT_STEP(X, Y, pa0, pb0, pc0, s)
    if (s + 1 >= nsteps) break;
    BT_STEP(Y, X, pa1, pb1, pc1, s + 1)
  }
#undef BT_STEP
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
  // merged rows symmetric in every cell? (pairs d, d + 7 of kStencilDirs)
  st.symmetric = true;
  for (const auto& r : st.rows)
    for (int d = 1; d <= 7; ++d) st.symmetric = st.symmetric && r[d] == r[d + 7];
}

void launch_stencil(const bt_stencil& st, const double* x, double* y, cudaStream_t s) {
  const int w = (1 << st.level) + 1;
  const int nc = st.grid->mesh.n_cells();
  const int per = st.symmetric ? kMaxCellsSym : kMaxCellsFull;
  for (int c0 = 0; c0 < nc; c0 += per) {
    const int cnt = std::min(per, nc - c0);
    dim3 grid((st.ntasks + kW - 1) / kW, cnt);
    if (st.symmetric) {
      static RowParams<8, kMaxCellsSym> rp;
      for (int c = 0; c < cnt; ++c)
        for (int d = 0; d < 8; ++d) rp.w[c][d] = st.rows[c0 + c][d];
      k_stencil<true, kMaxCellsSym><<<grid, kT, 0, s>>>(x, y, st.d_cells.p, st.d_tasks.p, st.ntasks, w, n_tet(w), c0, rp);
    } else {
      static RowParams<15, kMaxCellsFull> rp;
      for (int c = 0; c < cnt; ++c)
        for (int d = 0; d < 15; ++d) rp.w[c][d] = st.rows[c0 + c][d];
      k_stencil<false, kMaxCellsFull><<<grid, kT, 0, s>>>(x, y, st.d_cells.p, st.d_tasks.p, st.ntasks, w, n_tet(w), c0, rp);
    }
    count_launch();
    check_launch("k_stencil");
  }
}

}  // namespace bt
