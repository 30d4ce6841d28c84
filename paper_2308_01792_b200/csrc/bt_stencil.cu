// P1 constant-coefficient 15-point stencil apply (apply_stencil,
// operators.hpp:247-271), per-cell phase. The interface phase (replica sums
// and Dirichlet rows) is bt_interface.cu.
//
// Data path (k_stencil_fast). A warp owns 60 consecutive columns i of one
// layer k of one macro-cell — two adjacent columns per lane, lanes 0 and 31
// carry halo columns — and marches up to kMarchRows rows j. Each step needs
// three new rows at its columns — A(j+1) of layer k, B(j) of layer k+1 and
// C(j+1) of layer k-1, each one coalesced 512 B segment — loaded one step
// early into registers (predicated to 0 outside the lattice, so
// lattice-boundary vertices need no special loads); the i-1 / i+2 columns
// of a lane come from two warp shuffles per row. The march is unrolled by
// two over alternating window sets, so the sliding window costs no moves.
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
// lane; the corrections only run in warps that contain such a vertex. All
// weights are kernel parameters, so they reach the DFMAs as uniform-register
// operands. General rows (layer 0, row 0, the last two rows of column 0) go
// through k_stencil_general, which reads the typed rows from shared memory;
// it is also the fallback for tables that fail the fast-path checks.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "bt_internal.hpp"

namespace bt {

namespace {
constexpr int kT = 256;
constexpr int kW = kT / 32;
constexpr int kMarchRows = 48;
constexpr int kFastCols = 60;  // output columns per warp in k_stencil_fast
constexpr int kGenCols = 30;   // output columns per warp in k_stencil_general

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

// One row at a lane's two columns (c0 = v0, c1 = v1) with the neighbours
// l = column c0 - 1 and r = column c1 + 1.
struct Row4 {
  double l, v0, v1, r;
};
struct Win {  // A(j) of layer k, B(j-1) of layer k+1, C(j) of layer k-1
  Row4 a, b, c;
};

// per-warp cp.async ring: kStages stages x 3 staged rows; a row holds the
// warp's 64 columns at offset kRowOff (slack on both sides for the l / r reads)
constexpr int kStages = 4;
constexpr int kRowOff = 2;
constexpr int kRowD = 68;                  // doubles per staged row (16 B multiple)
constexpr int kStageD = 3 * kRowD;
constexpr int kRingD = kStages * kStageD;  // doubles per warp

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ double shup(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shdn(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

template <int kMaxC>
__global__ void __launch_bounds__(kT, 2) k_stencil_fast(const double* __restrict__ x, double* __restrict__ y,
                                                        const int4* __restrict__ tasks, int ntasks, int w,
                                                        int64_t cell_slots, int cell0,
                                                        const __grid_constant__ FastParams<kMaxC> fp) {
  extern __shared__ __align__(16) double ring_all[];
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
  const int c0 = kFastCols * blk + 2 * lane - 2;  // this lane's columns c0, c0 + 1
  const bool out_lane = lane >= 1 && lane <= kFastCols / 2;
  const bool up = k + 1 <= n;
  const double* __restrict__ xc = x + (int64_t)cell * cell_slots + c0;  // column c0 of every row
  double* ring = ring_all + warp * kRingD;
  const int me = kRowOff + 2 * lane;  // this lane's pair inside a staged row

  // ---- producer: stage rows A(j+1), B(j), C(j+1) of step j into the ring.
  // len(A(j+1)) = len(B(j)) = r, len(C(j+1)) = r + 1 with r = w - k - j - 1.
  int r = w - k - j0 - 1;
  const double* __restrict__ qA = xc + row_start(w, j0 + 1, k);
  const double* __restrict__ qB = xc + (up ? row_start(w, j0, k + 1) : 0);
  const double* __restrict__ qC = xc + row_start(w, j0 + 1, k - 1);
  auto stage_rows = [&](int stage, bool live) {
    double* st = ring + stage * kStageD + me;
    const bool a0 = live && c0 >= 0 && c0 < r, a1 = live && c0 + 1 >= 0 && c0 + 1 < r;
    const bool b0 = a0 && up, b1 = a1 && up;
    const bool e0 = live && c0 >= 0 && c0 <= r, e1 = live && c0 + 1 >= 0 && c0 + 1 <= r;
    cp_async8(st, a0 ? qA : x, a0);
    cp_async8(st + 1, a1 ? qA + 1 : x, a1);
    cp_async8(st + kRowD, b0 ? qB : x, b0);
    cp_async8(st + kRowD + 1, b1 ? qB + 1 : x, b1);
    cp_async8(st + 2 * kRowD, e0 ? qC : x, e0);
    cp_async8(st + 2 * kRowD + 1, e1 ? qC + 1 : x, e1);
    cp_commit();
    qA += r;
    qB += r;
    qC += r + 1;
    --r;
  };
  const int nsteps = j1 - j0;
#pragma unroll
  for (int q = 0; q < kStages - 1; ++q) stage_rows(q, q < nsteps);

  // window at row j0: A(j0), B(j0 - 1), C(j0) and A(j0 - 1), loaded directly
  auto ld2 = [&](const double* p, int len, double& v0, double& v1) {
    v0 = (c0 >= 0 && c0 < len) ? __ldg(p) : 0.0;
    v1 = (c0 + 1 >= 0 && c0 + 1 < len) ? __ldg(p + 1) : 0.0;
  };
  auto make_row = [&](double v0, double v1) {
    Row4 q;
    q.v0 = v0;
    q.v1 = v1;
    q.l = shup(v1);
    q.r = shdn(v0);
    return q;
  };
  Win X, Y;
  Row4 Am1, Am1y;
  {
    double a0, a1, b0, b1, e0, e1, m0, m1;
    ld2(xc + row_start(w, j0, k), w - k - j0, a0, a1);
    ld2(xc + (up ? row_start(w, j0 - 1, k + 1) : 0), up ? w - k - j0 : 0, b0, b1);
    ld2(xc + row_start(w, j0, k - 1), w - k - j0 + 1, e0, e1);
    ld2(xc + row_start(w, j0 - 1, k), w - k - j0 + 1, m0, m1);
    X.a = make_row(a0, a1);
    X.b = make_row(b0, b1);
    X.c = make_row(e0, e1);
    Am1 = make_row(m0, m1);
  }

  int LY = w - k - j0;  // length of the output row
  double* __restrict__ py = y + (int64_t)cell * cell_slots + c0 + row_start(w, j0, k);
  const int colend = kFastCols * blk + kFastCols;  // LY <= colend: the row ends in this warp
  const bool blk0 = blk == 0;
  int j = j0, q = 0;

  // One step: output row j at columns c0 (s0) and c0 + 1 (s1).
  // cur: A(j), B(j-1), C(j); am1: A(j-1); staged rows A1 = A(j+1), B0 = B(j),
  // C1 = C(j+1). kStencilDirs pairs (d, d + 7):
  //   (1,0,0)/(-1,0,0)  A(j) at i+1 / i-1      (0,1,0)/(0,-1,0)  A(j+1) / A(j-1)
  //   (0,0,1)/(0,0,-1)  B(j) / C(j)            (1,-1,0)/(-1,1,0) A(j-1) i+1 / A(j+1) i-1
  //   (1,0,-1)/(-1,0,1) C(j) i+1 / B(j) i-1    (0,1,-1)/(0,-1,1) C(j+1) / B(j-1)
  //   (1,-1,1)/(-1,1,-1) B(j-1) i+1 / C(j+1) i-1
#define BT_STEP(cur, nxt, am1, am1n)                                                                \
  {                                                                                                 \
    cp_wait<kStages - 2>();                                                                         \
    __syncwarp();                                                                                   \
    const double* sg = ring + (q % kStages) * kStageD + me;                                         \
    Row4 A1, B0, C1;                                                                                \
    A1.l = sg[-1];                                                                                  \
    A1.v0 = sg[0];                                                                                  \
    A1.v1 = sg[1];                                                                                  \
    A1.r = sg[2];                                                                                   \
    B0.l = sg[kRowD - 1];                                                                           \
    B0.v0 = sg[kRowD];                                                                              \
    B0.v1 = sg[kRowD + 1];                                                                          \
    B0.r = sg[kRowD + 2];                                                                           \
    C1.l = sg[2 * kRowD - 1];                                                                       \
    C1.v0 = sg[2 * kRowD];                                                                          \
    C1.v1 = sg[2 * kRowD + 1];                                                                      \
    C1.r = sg[2 * kRowD + 2];                                                                       \
    stage_rows((q + kStages - 1) % kStages, q + kStages - 1 < nsteps);                              \
    if (out_lane) {                                                                                 \
      double s0 = W[0] * cur.a.v0;                                                                  \
      s0 = fma(W[1], cur.a.v1 + cur.a.l, s0);                                                       \
      s0 = fma(W[2], A1.v0 + am1.v0, s0);                                                           \
      s0 = fma(W[3], B0.v0 + cur.c.v0, s0);                                                         \
      s0 = fma(W[4], am1.v1 + A1.l, s0);                                                            \
      s0 = fma(W[5], cur.c.v1 + B0.l, s0);                                                          \
      s0 = fma(W[6], C1.v0 + cur.b.v0, s0);                                                         \
      s0 = fma(W[7], cur.b.v1 + C1.l, s0);                                                          \
      double s1 = W[0] * cur.a.v1;                                                                  \
      s1 = fma(W[1], cur.a.r + cur.a.v0, s1);                                                       \
      s1 = fma(W[2], A1.v1 + am1.v1, s1);                                                           \
      s1 = fma(W[3], B0.v1 + cur.c.v1, s1);                                                         \
      s1 = fma(W[4], am1.r + A1.v0, s1);                                                            \
      s1 = fma(W[5], cur.c.r + B0.v0, s1);                                                          \
      s1 = fma(W[6], C1.v1 + cur.b.v1, s1);                                                         \
      s1 = fma(W[7], cur.b.r + C1.v0, s1);                                                          \
      if (LY <= colend) { /* row end in this warp: diagonal face, dirs 0, 4, 5, 6, 11, 12, 13 */     \
        double d0 = fma(DD[0], cur.a.v0, s0);                                                       \
        d0 = fma(DD[1], am1.v1, d0);                                                                \
        d0 = fma(DD[2], cur.c.v1, d0);                                                              \
        d0 = fma(DD[3], C1.v0, d0);                                                                 \
        d0 = fma(DD[4], A1.l, d0);                                                                  \
        d0 = fma(DD[5], B0.l, d0);                                                                  \
        d0 = fma(DD[6], cur.b.v0, d0);                                                              \
        double d1 = fma(DD[0], cur.a.v1, s1);                                                       \
        d1 = fma(DD[1], am1.r, d1);                                                                 \
        d1 = fma(DD[2], cur.c.r, d1);                                                               \
        d1 = fma(DD[3], C1.v1, d1);                                                                 \
        d1 = fma(DD[4], A1.v0, d1);                                                                 \
        d1 = fma(DD[5], B0.v0, d1);                                                                 \
        d1 = fma(DD[6], cur.b.v1, d1);                                                              \
        s0 = (c0 == LY - 1) ? d0 : s0;                                                              \
        s1 = (c0 + 1 == LY - 1) ? d1 : s1;                                                          \
      }                                                                                             \
      if (blk0) { /* face i = 0 at column c0 of lane 1: dirs 0, 2, 3, 6, 9, 10, 13 */                \
        double f0 = fma(DI[0], cur.a.v0, s0);                                                       \
        f0 = fma(DI[1], A1.v0, f0);                                                                 \
        f0 = fma(DI[2], B0.v0, f0);                                                                 \
        f0 = fma(DI[3], C1.v0, f0);                                                                 \
        f0 = fma(DI[4], am1.v0, f0);                                                                \
        f0 = fma(DI[5], cur.c.v0, f0);                                                              \
        f0 = fma(DI[6], cur.b.v0, f0);                                                              \
        s0 = (c0 == 0) ? f0 : s0;                                                                   \
      }                                                                                             \
      if (c0 < LY) py[0] = s0;                                                                      \
      if (c0 + 1 < LY) py[1] = s1;                                                                  \
    }                                                                                               \
    py += LY;                                                                                       \
    --LY;                                                                                           \
    ++j;                                                                                            \
    ++q;                                                                                            \
    am1n = cur.a;                                                                                   \
    nxt.a = A1;                                                                                     \
    nxt.b = B0;                                                                                     \
    nxt.c = C1;                                                                                     \
  }
  while (true) {
    BT_STEP(X, Y, Am1, Am1y)
    if (j >= j1) break;
    BT_STEP(Y, X, Am1y, Am1)
    if (j >= j1) break;
  }
#undef BT_STEP
  cp_wait<0>();
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
  const int i = kGenCols * tk.y + lane - 1;
  const bool out_lane = lane >= 1 && lane <= kGenCols && i >= 0;
  const double* __restrict__ xc = x + (int64_t)cell * cell_slots;
  double* __restrict__ yc = y + (int64_t)cell * cell_slots;
  auto at = [&](int jj, int kk) -> double {  // x at column i of row (jj, kk), 0 outside
    if (i < 0 || jj < 0 || kk < 0 || kk > n || i >= w - kk - jj) return 0.0;
    return __ldg(xc + row_start(w, jj, kk) + i);
  };
  for (int j = j0; j < j1; ++j) {
    const double A0 = at(j, k), Am1 = at(j - 1, k), A1 = at(j + 1, k), B0 = at(j, k + 1), Bm1 = at(j - 1, k + 1);
    const double C0 = at(j, k - 1), C1 = at(j + 1, k - 1);
    const double A0p = shdn(A0), A0m = shup(A0), Am1p = shdn(Am1), A1m = shup(A1);
    const double B0m = shup(B0), Bm1p = shdn(Bm1), C0p = shdn(C0), C1m = shup(C1);
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
  // general rows are unprefetched: one row per task keeps them parallel
  auto push1 = [](std::vector<int4>& v, int k, int b, int a, int e) {
    for (int j = a; j < e; ++j) v.push_back(make_int4(k, b, j, j + 1));
  };
  for (int k = 0; k < w; ++k) {
    // general-kernel column blocks (30 wide): layer 0, row 0, and rows of
    // length <= 2 (columns 0, 1: block 0)
    for (int b = 0; kGenCols * b < w - k; ++b) {
      const int jmax = w - k - kGenCols * b;
      push1(all, k, b, 0, jmax);
      if (k == 0) {
        push1(gen, k, b, 0, jmax);
      } else {
        push1(gen, k, b, 0, 1);
        if (b == 0) push1(gen, k, b, std::max(1, w - k - 2), jmax);
      }
    }
    if (k == 0) continue;
    // fast column blocks (60 wide): rows 1 .. (block 0: row length >= 3)
    for (int b = 0; kFastCols * b < w - k; ++b) {
      const int jmax = w - k - kFastCols * b;
      const int fe = b == 0 ? std::min(jmax, w - k - 2) : jmax;
      for (int j0 = 1; j0 < fe; j0 += kMarchRows) fast.push_back(make_int4(k, b, j0, std::min(j0 + kMarchRows, fe)));
    }
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
    const auto& rw = st.rows[c];
    for (int d = 1; d <= 7; ++d) st.symmetric = st.symmetric && rw[d] == rw[d + 7];
    for (int z : {1, 2}) {
      const int* dirs = z == 1 ? kDiagDirs : kI0Dirs;
      for (int d = 0; d < 15; ++d) {
        bool exempt = false;
        for (int q = 0; q < 7; ++q) exempt = exempt || dirs[q] == d;
        for (int q = 0; q < 4; ++q) exempt = exempt || kOutside[z][q] == d;
        if (!exempt && cells[c].w[z][d] != rw[d]) st.symmetric = false;
      }
    }
    double* f = &st.fast[22 * (size_t)c];
    for (int d = 0; d < 8; ++d) f[d] = rw[d];
    for (int q = 0; q < 7; ++q) {
      f[8 + q] = cells[c].w[1][kDiagDirs[q]] - rw[kDiagDirs[q]];
      f[15 + q] = cells[c].w[2][kI0Dirs[q]] - rw[kI0Dirs[q]];
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
    const size_t smem = sizeof(double) * kW * kRingD;
    static bool attr = false;
    if (!attr) {
      BT_CUDA(cudaFuncSetAttribute(k_stencil_fast<kMaxCells>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    k_stencil_fast<kMaxCells><<<dim3((st.ntasks + kW - 1) / kW, cnt), kT, smem, s>>>(x, y, st.d_tasks.p, st.ntasks,
                                                                                    w, cs, c0, fp);
    count_launch();
  }
  check_launch("k_stencil");
}

}  // namespace bt
