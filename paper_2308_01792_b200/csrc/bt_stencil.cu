// P1 constant-coefficient 15-point stencil apply (apply_stencil,
// operators.hpp:247-271), per-cell phase. The interface phase (replica sums
// and Dirichlet rows) is bt_interface.cu.
//
// Data path (k_stencil_fast). A warp owns 62 consecutive output columns i of
// one layer k of one macro-cell and marches up to kMarchRows rows j. Each
// step needs three new rows — A(j+1) of layer k, B(j) of layer k+1 and C(j+1)
// of layer k-1 — over the warp's 64 staged columns [base - 1, base + 63).
// Lane 0 stages them with TMA bulk copies (cp.async.bulk, 528 B each, 16 B
// aligned with a per-row shift) into a per-warp kStages-deep shared-memory
// ring completed on mbarriers, so the copies cost no LSU wavefronts and no
// registers. Lanes read two contiguous 32-column halves (columns base-1+l and
// base+31+l) plus their i-1 / i+1 neighbours from the ring; values reused by
// later rows stay in registers (window sets alternate, no moves). Every x
// value is read from L2 once per layer that needs it (3x) and from HBM once.
//
// Rows. The host splits every (layer, column block) march into fast rows and
// a few general rows. Fast rows (1 <= k <= n-2, j >= 1, row length >= 3 in
// column block 0) hold interior vertices, evaluated with the merged row
// (compute_stencil operators.hpp:204-221) in its symmetric 8-weight form
// (W[d] == W[-d] bitwise, checked on the host), plus at most the
// diagonal-face vertex (i = row end) and the i = 0 vertex, evaluated with
// their zero-set-typed partial rows (per-cell part of partial_row_apply,
// operators.hpp:78-96) over their 11 present neighbours only — so nothing
// outside the lattice is ever used and the staged rows need no masking. All
// weights are kernel parameters: they reach the DFMAs as uniform-register
// operands. General rows (layers 0, n-1, n, row 0, the last two rows of
// column 0) go through k_stencil_general, which reads the typed rows from
// shared memory; it is also the fallback for tables that fail the fast-path
// checks.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "bt_internal.hpp"

namespace bt {

namespace {
constexpr int kT = 256;
constexpr int kW = kT / 32;
constexpr int kMarchRows = 48;
constexpr int kFastCols = 62;  // output columns per warp in k_stencil_fast
constexpr int kGenCols = 30;   // output columns per warp in k_stencil_general

// present neighbour directions (kStencilDirs indices) of a diagonal-face
// vertex (zero set {0}) and of an i = 0 vertex (zero set {1})
constexpr int kDiagPresent[11] = {0, 4, 5, 6, 8, 9, 10, 11, 12, 13, 14};
constexpr int kI0Present[11] = {0, 1, 2, 3, 4, 5, 6, 7, 9, 10, 13};

template <int kMaxC>
struct FastParams {
  double w[kMaxC][8];    // symmetric interior row: centre + 7 direction pairs
  double dg[kMaxC][11];  // diagonal-face typed row on kDiagPresent
  double f0[kMaxC][11];  // i = 0 face typed row on kI0Present
};
constexpr int kMaxCells = 128;  // 128 * 30 * 8 B = 30 KB of kernel parameters

// per-warp TMA ring: kStages stages x 3 staged rows of kRowD doubles
constexpr int kStages = 4;
constexpr int kRowD = 72;                  // >= 66 doubles (528 B copy), 16 B multiple
constexpr int kStageD = 3 * kRowD;
constexpr int kRingD = kStages * kStageD;  // doubles per warp
constexpr int kCopyBytes = 528;            // 64 columns + one 16 B alignment chunk

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_row(double* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct Row3 {  // one row at a lane's two columns: v = value, l = column - 1, r = column + 1
  double l0, v0, r0, l1, v1, r1;
};
struct Win {  // A(j) of layer k, B(j-1) of layer k+1, C(j) of layer k-1
  Row3 a, b, c;
};

template <int kMaxC>
__global__ void __launch_bounds__(kT, 2) k_stencil_fast(const double* __restrict__ x, double* __restrict__ y,
                                                        const int4* __restrict__ tasks, int ntasks, int w,
                                                        int64_t cell_slots, int cell0, const double* x_end,
                                                        const __grid_constant__ FastParams<kMaxC> fp) {
  extern __shared__ __align__(128) double ring_all[];
  __shared__ __align__(8) uint64_t bars[kW][kStages];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int task = blockIdx.x * kW + warp;
  if (task >= ntasks) return;
  const int cell = cell0 + blockIdx.y;
  const double* W = fp.w[blockIdx.y];
  const double* DG = fp.dg[blockIdx.y];
  const double* F0 = fp.f0[blockIdx.y];
  const int4 tk = tasks[task];
  const int k = tk.x, blk = tk.y, j0 = tk.z, j1 = tk.w;  // k in [1, n-2], j0 >= 1 by construction
  const int base = kFastCols * blk;
  const int c0 = base - 1 + lane, c1 = base + 31 + lane;  // this lane's two columns
  const bool out0 = lane >= 1, out1 = lane <= 30;
  const double* __restrict__ xcell = x + (int64_t)cell * cell_slots;
  double* ring = ring_all + warp * kRingD;
  uint64_t* bar = bars[warp];
  const uint64_t end16 = ((uint64_t)x_end + 15) & ~(uint64_t)15;

  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();

  // producer cursors: rows A(j+1), B(j), C(j+1) of step j; offsets of column
  // base - 1 in each row. len(A(j+1)) = len(B(j)) = r, len(C(j+1)) = r + 1.
  int r = w - k - j0 - 1;
  int oA = row_start(w, j0 + 1, k) + base - 1;
  int oB = row_start(w, j0, k + 1) + base - 1;
  int oC = row_start(w, j0 + 1, k - 1) + base - 1;
  auto produce = [&](int stage) {  // lane 0 only
    double* st = ring + stage * kStageD;
    const double* srcs[3] = {xcell + oA, xcell + oB, xcell + oC};
    uint32_t total = 0, bytes[3];
    uint64_t al[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      al[q] = (uint64_t)srcs[q] & ~(uint64_t)15;
      const uint64_t lim = end16 - al[q];
      bytes[q] = lim < (uint64_t)kCopyBytes ? (uint32_t)lim : (uint32_t)kCopyBytes;
      total += bytes[q];
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(&bar[stage], total);
#pragma unroll
    for (int q = 0; q < 3; ++q) tma_row(st + q * kRowD, (const void*)al[q], bytes[q], &bar[stage]);
  };
  auto advance = [&]() {
    oA += r;
    oB += r;
    oC += r + 1;
    --r;
  };
  // shift (in doubles) of column base - 1 inside a staged row
  auto shift_of = [&](int o) -> int { return (int)(((uint64_t)(xcell + o) >> 3) & 1); };
  const int nsteps = j1 - j0;
  // per-stage shifts of the three rows (3 bits per stage), tracked
  // identically by every lane
  uint32_t shbits = 0;
  auto note_shifts = [&](int stage) {
    const uint32_t b = (uint32_t)(shift_of(oA) | (shift_of(oB) << 1) | (shift_of(oC) << 2));
    shbits = (shbits & ~(7u << (3 * stage))) | (b << (3 * stage));
  };
#pragma unroll
  for (int q = 0; q < kStages - 1; ++q) {
    note_shifts(q);
    if (q < nsteps && lane == 0) produce(q);
    advance();
  }

  // window at row j0: A(j0), B(j0 - 1), C(j0) and A(j0 - 1), loaded directly
  auto at = [&](int rs, int len, int c) -> double { return (c >= 0 && c < len) ? __ldg(xcell + rs + c) : 0.0; };
  auto load_row = [&](int rs, int len) {
    Row3 q;
    q.l0 = at(rs, len, c0 - 1);
    q.v0 = at(rs, len, c0);
    q.r0 = at(rs, len, c0 + 1);
    q.l1 = at(rs, len, c1 - 1);
    q.v1 = at(rs, len, c1);
    q.r1 = at(rs, len, c1 + 1);
    return q;
  };
  Win X, Y;
  Row3 Am1, Am1y;
  X.a = load_row(row_start(w, j0, k), w - k - j0);
  X.b = load_row(row_start(w, j0 - 1, k + 1), w - k - j0);
  X.c = load_row(row_start(w, j0, k - 1), w - k - j0 + 1);
  Am1 = load_row(row_start(w, j0 - 1, k), w - k - j0 + 1);

  int LY = w - k - j0;  // length of the output row
  double* __restrict__ py = y + (int64_t)cell * cell_slots + row_start(w, j0, k);
  const int colend = base + kFastCols;  // LY <= colend: the row ends inside this warp
  const bool blk0 = blk == 0;
  int j = j0, q = 0;

  auto read_row = [&](const double* row, int sh) {
    Row3 o;
    const double* p = row + sh + lane;  // column base - 1 + lane
    o.l0 = p[-1];
    o.v0 = p[0];
    o.r0 = p[1];
    o.l1 = p[31];
    o.v1 = p[32];
    o.r1 = p[33];
    return o;
  };

  // One step: output row j at columns c0 (s0) and c1 (s1).
  // cur: A(j), B(j-1), C(j); am1: A(j-1); staged rows A1 = A(j+1), B0 = B(j),
  // C1 = C(j+1). kStencilDirs pairs (d, d + 7):
  //   (1,0,0)/(-1,0,0)  A(j) i+1 / i-1         (0,1,0)/(0,-1,0)  A(j+1) / A(j-1)
  //   (0,0,1)/(0,0,-1)  B(j) / C(j)            (1,-1,0)/(-1,1,0) A(j-1) i+1 / A(j+1) i-1
  //   (1,0,-1)/(-1,0,1) C(j) i+1 / B(j) i-1    (0,1,-1)/(0,-1,1) C(j+1) / B(j-1)
  //   (1,-1,1)/(-1,1,-1) B(j-1) i+1 / C(j+1) i-1
#define BT_INTERIOR(cur, am1, s, v, l, r)                                                                     \
  double s = W[0] * cur.a.v;                                                                        \
  s = fma(W[1], cur.a.r + cur.a.l, s);                                                              \
  s = fma(W[2], A1.v + am1.v, s);                                                                   \
  s = fma(W[3], B0.v + cur.c.v, s);                                                                 \
  s = fma(W[4], am1.r + A1.l, s);                                                                   \
  s = fma(W[5], cur.c.r + B0.l, s);                                                                 \
  s = fma(W[6], C1.v + cur.b.v, s);                                                                 \
  s = fma(W[7], cur.b.r + C1.l, s);
  // typed rows over present neighbours (kDiagPresent / kI0Present order)
#define BT_DIAG(cur, am1, v, l, r)                                                                            \
  (DG[0] * cur.a.v + DG[1] * am1.r + DG[2] * cur.c.r + DG[3] * C1.v + DG[4] * cur.a.l +             \
   DG[5] * am1.v + DG[6] * cur.c.v + DG[7] * A1.l + DG[8] * B0.l + DG[9] * cur.b.v + DG[10] * C1.l)
#define BT_FACE0(cur, am1, v, l, r)                                                                           \
  (F0[0] * cur.a.v + F0[1] * cur.a.r + F0[2] * A1.v + F0[3] * B0.v + F0[4] * am1.r +                \
   F0[5] * cur.c.r + F0[6] * C1.v + F0[7] * cur.b.r + F0[8] * am1.v + F0[9] * cur.c.v +             \
   F0[10] * cur.b.v)
#define BT_STEP(cur, nxt, am1, am1n)                                                                \
  {                                                                                                 \
    const int sg = q % kStages;                                                                     \
    mbar_wait(&bar[sg], (uint32_t)((q / kStages) & 1));                                             \
    const double* st = ring + sg * kStageD;                                                         \
    const uint32_t sb = shbits >> (3 * sg);                                                         \
    const Row3 A1 = read_row(st, sb & 1);                                                           \
    const Row3 B0 = read_row(st + kRowD, (sb >> 1) & 1);                                            \
    const Row3 C1 = read_row(st + 2 * kRowD, (sb >> 2) & 1);                                        \
    __syncwarp();                                                                                   \
    {                                                                                               \
      const int ps = (q + kStages - 1) % kStages;                                                   \
      note_shifts(ps);                                                                              \
      if (q + kStages - 1 < nsteps && lane == 0) produce(ps);                                       \
      advance();                                                                                    \
    }                                                                                               \
    BT_INTERIOR(cur, am1, s0, v0, l0, r0)                                                                     \
    BT_INTERIOR(cur, am1, s1, v1, l1, r1)                                                                     \
    if (LY <= colend) { /* the diagonal-face vertex is in this warp */                              \
      if (c0 == LY - 1) s0 = BT_DIAG(cur, am1, v0, l0, r0);                                                   \
      if (c1 == LY - 1) s1 = BT_DIAG(cur, am1, v1, l1, r1);                                                   \
    }                                                                                               \
    if (blk0 && c0 == 0) s0 = BT_FACE0(cur, am1, v0, l0, r0); /* lane 1 of block 0 */                         \
    if (out0 && c0 < LY) py[c0] = s0;                                                               \
    if (out1 && c1 < LY) py[c1] = s1;                                                               \
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
#undef BT_FACE0
#undef BT_DIAG
#undef BT_INTERIOR
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
  auto shup = [](double v) { return __shfl_up_sync(0xffffffffu, v, 1); };
  auto shdn = [](double v) { return __shfl_down_sync(0xffffffffu, v, 1); };
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
  const int n = w - 1;
  std::vector<int4> fast, gen, all;
  // general rows are unprefetched: one row per task keeps them parallel
  auto push1 = [](std::vector<int4>& v, int k, int b, int a, int e) {
    for (int j = a; j < e; ++j) v.push_back(make_int4(k, b, j, j + 1));
  };
  for (int k = 0; k < w; ++k) {
    // fast rows: 1 <= k <= n - 2, 1 <= j, and in column block 0 row length >= 3
    const bool fast_layer = k >= 1 && k <= n - 2;
    for (int b = 0; kGenCols * b < w - k; ++b) {  // general-kernel blocks (30 wide)
      const int jmax = w - k - kGenCols * b;
      push1(all, k, b, 0, jmax);
      if (!fast_layer) {
        push1(gen, k, b, 0, jmax);
      } else {
        push1(gen, k, b, 0, 1);
        if (b == 0) push1(gen, k, b, std::max(1, w - k - 2), jmax);
      }
    }
    if (!fast_layer) continue;
    for (int b = 0; kFastCols * b < w - k; ++b) {  // fast blocks (62 wide)
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
  // Fast path preconditions: bitwise-symmetric merged rows, and typed face
  // rows that vanish off their present directions.
  st.symmetric = true;
  const int nc = st.grid->mesh.n_cells();
  std::vector<StencilCell> cells(nc);
  BT_CUDA(cudaMemcpy(cells.data(), st.d_cells.p, sizeof(StencilCell) * nc, cudaMemcpyDeviceToHost));
  st.fast.assign(30 * (size_t)nc, 0.0);
  for (int c = 0; c < nc; ++c) {
    const auto& rw = st.rows[c];
    for (int d = 1; d <= 7; ++d) st.symmetric = st.symmetric && rw[d] == rw[d + 7];
    for (int d = 0; d < 15; ++d) {
      bool pd = false, pi = false;
      for (int q = 0; q < 11; ++q) {
        pd = pd || kDiagPresent[q] == d;
        pi = pi || kI0Present[q] == d;
      }
      if ((!pd && cells[c].w[1][d] != 0.0) || (!pi && cells[c].w[2][d] != 0.0)) st.symmetric = false;
    }
    double* f = &st.fast[30 * (size_t)c];
    for (int d = 0; d < 8; ++d) f[d] = rw[d];
    for (int q = 0; q < 11; ++q) {
      f[8 + q] = cells[c].w[1][kDiagPresent[q]];
      f[19 + q] = cells[c].w[2][kI0Present[q]];
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
  const size_t smem = sizeof(double) * kW * kRingD;
  static bool attr = false;
  if (!attr) {
    BT_CUDA(cudaFuncSetAttribute(k_stencil_fast<kMaxCells>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const double* x_end = x + cs * nc;
  for (int c0 = 0; c0 < nc && st.ntasks; c0 += kMaxCells) {
    const int cnt = std::min(kMaxCells, nc - c0);
    for (int c = 0; c < cnt; ++c) {
      const double* f = &st.fast[30 * (size_t)(c0 + c)];
      for (int d = 0; d < 8; ++d) fp.w[c][d] = f[d];
      for (int q = 0; q < 11; ++q) {
        fp.dg[c][q] = f[8 + q];
        fp.f0[c][q] = f[19 + q];
      }
    }
    k_stencil_fast<kMaxCells><<<dim3((st.ntasks + kW - 1) / kW, cnt), kT, smem, s>>>(x, y, st.d_tasks.p, st.ntasks,
                                                                                    w, cs, c0, x_end, fp);
    count_launch();
  }
  check_launch("k_stencil");
}

}  // namespace bt
