// P1 constant-coefficient 15-point stencil apply (apply_stencil,
// operators.hpp:247-271), per-cell phase. The interface phase (replica sums
// and Dirichlet rows) is bt_interface.cu.
//
// Data path (k_stencil_fast). A warp owns 62 consecutive output columns i of
// one layer k of one macro-cell (lane l: the pair c0 = base - 1 + 2l, c0 + 1)
// and marches up to kMarchRows rows j. Each step needs three new rows — A(j+1)
// of layer k, B(j) of layer k+1 and C(j+1) of layer k-1 — over the warp's 64
// staged columns [base - 1, base + 63). Every lane stages its two columns of
// each row with 8-byte cp.async into a per-warp kStages-deep shared ring (so a
// row lands at a fixed place whatever its alignment), then reads its pair
// with one 16-byte shared load and the i-1 / i+1 neighbours by shuffle.
// Values reused by later rows stay in registers (window sets alternate). The
// grid is persistent: warps stride over a task list sorted longest first, and
// the staging stream runs ahead across task boundaries (two phantom steps per
// march fill the register window). Every x value is read from L2 once per
// layer that needs it (3x) and from HBM about once.
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
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <cstdlib>
#include <string>
#include <vector>

#include "bt_async.cuh"
#include "bt_internal.hpp"

namespace bt {

#ifndef BT_ST16
#define BT_ST16 0  // 1: 16-byte stores of address-aligned pairs
#endif
#ifndef BT_STQ
#define BT_STQ ""  // cache qualifier of the march's stores (profiling: ".cg", ".cs", ".wt")
#endif

namespace {
constexpr int kMarchRows = 64;  // measured at config 2 (r2_notes section 7): 32 -> 84.1, 64 -> 81.5, 72 -> 81.1, 128 -> 91.7 us per apply
// small problems (all slots of the handle <= kSmallSlots): one launch for the
// whole apply (k_stencil_small) and short marches, whose serial step chains
// set the latency there
constexpr int64_t kSmallSlots = int64_t(1) << 21;
constexpr int kSmallMarch = 4;
constexpr int kGroup = 4;  // layers per fast march (plus one 2-layer group); 6 measured slower (2 blocks/SM)
constexpr int kFastCols = 62;  // output columns per warp in k_stencil_fast (of 64 staged: one halo column each side)
constexpr int kGenCols = 30;   // output columns per warp in k_stencil_general
// k_stencil_general / k_stencil_ends blocks are small and register-light so
// that one fits on an SM beside three k_stencil_fast blocks: they run on a
// side stream concurrently with the fast kernel (launch_stencil).
constexpr int kGT = 128;
constexpr int kGW = kGT / 32;

// present neighbour directions (kStencilDirs indices) of a diagonal-face
// vertex (zero set {0}) and of an i = 0 vertex (zero set {1})
constexpr int kDiagPresent[11] = {0, 4, 5, 6, 8, 9, 10, 11, 12, 13, 14};
constexpr int kI0Present[11] = {0, 1, 2, 3, 4, 5, 6, 7, 9, 10, 13};

template <int kMaxC>
struct FastParams {
  double w[kMaxC][8];  // symmetric interior row: centre + 7 direction pairs
};
constexpr int kMaxCells = 256;  // 256 * 8 * 8 B = 16 KB of kernel parameters

// per-warp staging ring: kStages stages x (N + 2) staged rows of kRowD doubles
#ifndef BT_STAGES
#define BT_STAGES 3  // measured: 3 beats 4 (more L1 beside the rings) and 2
#endif
constexpr int kStages = BT_STAGES;
constexpr int kRowD = 64;  // staged columns [base - 1, base + 63)
#ifndef BT_FT
#define BT_FT 128
#endif
constexpr int kFT = BT_FT;  // k_stencil_fast block (warps of a block are independent: the size only sets how early a
                            // finished block's registers return to the SM)
constexpr int kFW = kFT / 32;
template <int N>
__host__ __device__ constexpr int ring_doubles() {  // per warp
  return kStages * (N + 2) * kRowD;
}


struct Row2 {  // one row at a lane's columns c0, c1 = c0 + 1
  double v0, v1;
};
// Register window of an N-layer march at row j: layers k .. k+N-1 (rows j-1
// and j), layer k-1 (row j) below, layer k+N (row j-1) above.
template <int N>
struct Win {
  Row2 am1[N], a[N];
  Row2 c, qm1;
};

// Task word: x = k (first layer of the march's N layers), y = column block |
// (cell - cell0) << 16, z = j0, w = j1.
//
// A warp owns 62 output columns of N adjacent layers k .. k+N-1 of one cell
// and marches rows j0..j1-1 of all of them (each layer's rows end one row
// before the one below; rows that are not interior rows are masked). Per
// step it stages N + 2 rows — row j+1 of layers k-1 .. k+N-1 and row j of
// layer k+N — which serve all N layers: N + 2 staged rows per N output rows.
//
// Persistent warps: warp g runs tasks g, g + G, g + 2G, ... (the host sorts
// tasks by length, longest first). Each march is preceded by two phantom
// steps (j0 - 2, j0 - 1) whose staged rows fill the register window, so the
// staging stream runs through the ring across task boundaries without
// draining. Lane l stages columns base - 1 + l and base + 31 + l of each row
// (two 8-byte cp.async, each warp-contiguous; none past the row's end), so
// every row lands at the same place whatever its alignment and lane l reads
// its pair (c0, c1) with one 16-byte shared load. Column -1 (lane 0 of
// column block 0) is not staged: it feeds only column 0's output, which is
// never stored. So every copy stays inside its row:
// any march of any cell runs here, whatever the vector's extent.
// (body shared by k_stencil_fast and the single-launch k_stencil_small: block
// vblock of a vgrid-block persistent grid)
// predicated stores of the fast march (one SETP + one predicated STG each, no branches)
__device__ __forceinline__ void st_if(double* p, double v, int ly, int thr) {  // *p = v if ly > thr
  asm volatile("{ .reg .pred q; setp.gt.s32 q, %2, %3; @q st.global" BT_STQ ".f64 [%0], %1; }" ::"l"(p), "d"(v), "r"(ly), "r"(thr)
               : "memory");
}
// (p[0], p[1]) = (a, b), p 16-byte aligned: one 16-byte store if ly > ta and ly > tb, else the valid half
__device__ __forceinline__ void st_pair(double* p, double a, double b, int ly, int ta, int tb) {
  asm volatile(
      "{ .reg .pred qa, qb, qab, qa1, qb1;\n"
      "setp.gt.s32 qa, %3, %4; setp.gt.s32 qb, %3, %5;\n"
      "and.pred qab, qa, qb; and.pred qa1, qa, !qb; and.pred qb1, qb, !qa;\n"
      "@qab st.global.v2.f64 [%0], {%1, %2};\n"
      "@qa1 st.global.f64 [%0], %1;\n"
      "@qb1 st.global.f64 [%0+8], %2; }" ::"l"(p),
      "d"(a), "d"(b), "r"(ly), "r"(ta), "r"(tb)
      : "memory");
}

template <int N, int kMaxC>
__device__ __forceinline__ void stencil_fast_body(const double* __restrict__ x, double* __restrict__ y,
                                                  const int4* __restrict__ tasks, int ntasks, int w,
                                                  int64_t cell_slots, const FastParams<kMaxC>& fp, int vblock,
                                                  int vgrid, double* ring_all, int* __restrict__ ctr = nullptr) {
  constexpr int NS = N + 2;  // staged rows per step: C (layer k-1), layers k..k+N-1, Q (layer k+N)
  constexpr int kStageD = NS * kRowD;
  // warp index and task words broadcast by shuffles: provably warp-uniform, so
  // the march loop's shuffles need no divergence handling (WARPSYNC)
  const int lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int G = vgrid * kFW;
  const int t0 = vblock * kFW + warp;
  // ctr != nullptr: dynamic schedule. Warps draw tasks (sorted longest first)
  // from the queue ctr[0] as they finish, so SMs that run slower (the two
  // dies' different distances to a cell's memory) take fewer tasks; the
  // producer, which runs ahead of the consumer, hands each task word over
  // through a four-deep per-warp ring in shared memory. ctr[1] counts
  // finished warps; the last one resets both for the next launch.
  const bool dyn = ctr != nullptr;
  if (!dyn && t0 >= ntasks) return;
  const double* ring = ring_all + warp * ring_doubles<N>();
  int4* fifo = reinterpret_cast<int4*>(ring_all + kFW * ring_doubles<N>()) + 4 * warp;
  const int4 kNull = make_int4(1, 0, 1, -1);  // no steps (w - z + 2 == 0)
  auto draw = [&]() -> int4 {  // the next task of the queue (dynamic schedule)
    int i = 0;
    if (lane == 0) i = atomicAdd(ctr, 1);
    i = __shfl_sync(0xffffffffu, i, 0);
    return i < ntasks ? tasks[i] : kNull;
  };
  int pn = 0, cn = 0;  // task words pushed / popped
  const uint32_t my_s = smem_u32(ring) + 8u * lane;

  // ---- producer (every lane copies its two columns of each staged row) ----
  // po[s]: element offset (within the cell) of column base - 1 + lane in the
  // producer's next step j of stream s: 0 = C(j+1) (layer k-1), 1 + q = row
  // j+1 of layer k+q, N+1 = Q(j) (layer k+N); pr = len(row j+1 of layer k)
  int pt = t0, pr = 0, pleft = 0, pcol = 0;
  int po[NS];
  const double* pcell = x;
  int4 pnext = dyn ? draw() : tasks[t0];
  auto p_start = [&]() {
    const int4 tk = pnext;
    if (dyn) {
      if (lane == 0) fifo[pn & 3] = tk;
      ++pn;
    }
    const int k = tk.x, base = kFastCols * (tk.y & 0xffff), cl = tk.y >> 16;
    const int j = tk.z - 2, cb = base - 1 + lane;
    pcol = cb;  // this lane's first staged column (the second is pcol + 32)
    pcell = x + (int64_t)cl * cell_slots;
    po[0] = cb + row_start(w, j + 1, k - 1);
#pragma unroll
    for (int q = 0; q < N; ++q) po[1 + q] = cb + row_start(w, j + 1, k + q);
    po[N + 1] = cb + row_start(w, j, k + N);
    pr = w - k - j - 1;
    pleft = tk.w - tk.z + 2;
    if (dyn) {
      if (pleft > 0) pnext = draw();
    } else if (pt + G < ntasks) {
      pnext = tasks[pt + G];
    }
  };
  p_start();
  int ps = 0;  // producer stage
  auto produce = [&]() {  // one (possibly empty) group of copies
    if (pleft > 0) {
      const uint32_t d = my_s + (uint32_t)(ps * kStageD * 8);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        // length of stream s's current row; columns past it are never used
        const int len = s == 0 ? pr + 1 : (s <= N ? pr - (s - 1) : pr + 1 - N);
        const double* src = pcell + po[s];
        if ((unsigned)pcol < (unsigned)len) cp8(d + s * kRowD * 8, src);
        if (pcol + 32 < len) cp8(d + s * kRowD * 8 + 256, src + 32);
        po[s] += len;  // next row of the stream
      }
      ps = ps == kStages - 1 ? 0 : ps + 1;
      --pr;
      if (--pleft == 0) {
        pt += G;
        if (dyn || pt < ntasks) p_start();
      }
    }
    cp_commit();
  };
#pragma unroll 1
  for (int q = 0; q < kStages - 1; ++q) produce();

  // ---- consumer ----
  int cs = 0;
  auto read_row = [&](const double* row, Row2& o) {
    const double2 v = reinterpret_cast<const double2*>(row)[lane];
    o.v0 = v.x;
    o.v1 = v.y;
  };
  // staged rows of one step: C1 = C(j+1), A1[q] = row j+1 of layer k+q, Q0 = Q(j)
  auto consume = [&](Row2& C1, Row2* A1, Row2& Q0) {
    cp_wait<kStages - 2>();
    __syncwarp();
    const double* st = ring + cs * kStageD;
    read_row(st, C1);
#pragma unroll
    for (int q = 0; q < N; ++q) read_row(st + (1 + q) * kRowD, A1[q]);
    read_row(st + (N + 1) * kRowD, Q0);
    cs = cs == kStages - 1 ? 0 : cs + 1;
    // the stage refilled next is the one every lane read in the previous
    // step, which the __syncwarp above orders before this refill
    produce();
  };

  // Window rows rotate through three register sets (phase p: row j-1 in set
  // p, row j in set p+1, the step's new row j+1 into set p+2, all mod 3), so
  // the march loop, unrolled over the three phases, moves no registers.
  Row2 R[3][N], Cc[3], Qq[3];
  const unsigned ybits = (unsigned)(reinterpret_cast<uintptr_t>(y) >> 3);
#pragma unroll 1
  for (int t = t0; dyn || t < ntasks; t += G) {
    int4 tk;
    if (dyn) {
      __syncwarp();
      tk = fifo[cn & 3];
      ++cn;
    } else {
      tk = tasks[t];
    }
    tk.x = __shfl_sync(0xffffffffu, tk.x, 0);
    tk.y = __shfl_sync(0xffffffffu, tk.y, 0);
    tk.z = __shfl_sync(0xffffffffu, tk.z, 0);
    tk.w = __shfl_sync(0xffffffffu, tk.w, 0);
    const int k = tk.x, blk = tk.y & 0xffff, cl = tk.y >> 16, j0 = tk.z, j1 = tk.w;
    if (j1 < j0) break;  // null task: the end of this warp's list in a balanced schedule (build_sched)
    double W[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) W[d] = fp.w[cl][d];
    const int base = kFastCols * blk;
    // this lane's two columns: c0, c0 + 1. Lane 0's c0 (base - 1) and lane 31's c0 + 1 (base + 62) are halo
    // columns: they only feed their neighbours' +-i partial sums.
    const int c0 = base - 1 + 2 * lane;
    const int pmin = blk == 0 ? 3 : 0;  // shorter rows of column block 0 are not interior rows
    // Store thresholds: column c of a row of length LY is an interior output
    // iff 0 < c < LY - 1 (row ends are the boundary kernel's) and LY >= pmin,
    // i.e. LY > max(c + 1, pmin - 1). T0 / T1: this lane's c0 / c0 + 1; T2:
    // the next lane's c0 (= c0 + 2), stored by this lane when the row's
    // address parity pairs it with this lane's c0 + 1.
    constexpr int kNever = 1 << 30;
    const int T0 = lane >= 1 && c0 > 0 ? max(c0 + 1, pmin - 1) : kNever;
    const int T1 = lane <= 30 && c0 + 1 > 0 ? max(c0 + 2, pmin - 1) : kNever;
    const int T2 = lane <= 30 && c0 + 2 > 0 ? max(c0 + 3, pmin - 1) : kNever;
    {
      Row2 cj, qj;
      consume(cj, R[0], qj);         // phantom step j0 - 2: rows j0 - 1
      consume(Cc[0], R[1], Qq[0]);   // phantom step j0 - 1: rows j0, C(j0), Q(j0 - 1)
    }
    int LA = w - k - j0;  // length of row j of layer k; layer k+q's is LA - q
    const int64_t celloff = (int64_t)cl * cell_slots;
    double* __restrict__ yl = y + celloff + c0;  // + a row's start: this lane's c0 in that row
    const unsigned ypar = ybits + (unsigned)celloff + (unsigned)(c0 & 1);  // parity of (yl + oy): that of ypar + oy
    int oy[N];
#pragma unroll
    for (int q = 0; q < N; ++q) oy[q] = row_start(w, j0, k + q);
    int j = j0;

    // One layer's output row at columns c0 (s0) and c0 + 1 (s1): see the
    // formula at the other body. Stored as one 16-byte store per lane: of
    // (c0, c0 + 1) when that pair is 16-byte aligned in y, else of (c0 + 1,
    // next lane's c0); pairs broken by a row end fall back to 8-byte stores.
    auto layer = [&](const Row2& a, const Row2& b, const Row2& c, const Row2& am1, const Row2& A1, const Row2& B0,
                     const Row2& C1, int LY, int o) {
      const double upv = fma(W[7], C1.v1, fma(W[5], B0.v1, fma(W[4], A1.v1, W[1] * a.v1)));  // to column c1 + 1
      const double dnv = fma(W[7], b.v0, fma(W[5], c.v0, fma(W[4], am1.v0, W[1] * a.v0)));   // to column c0 - 1
      const double lft = __shfl_up_sync(0xffffffffu, upv, 1);    // column c0 - 1's, for c0
      const double rgt = __shfl_down_sync(0xffffffffu, dnv, 1);  // column c1 + 1's, for c1
      double s0 = fma(W[6], C1.v0 + b.v0, fma(W[3], B0.v0 + c.v0, fma(W[2], A1.v0 + am1.v0, W[0] * a.v0)));
      double s1 = fma(W[6], C1.v1 + b.v1, fma(W[3], B0.v1 + c.v1, fma(W[2], A1.v1 + am1.v1, W[0] * a.v1)));
      s0 += lft;
      s0 += fma(W[7], b.v1, fma(W[5], c.v1, fma(W[4], am1.v1, W[1] * a.v1)));  // i+1 of c0 = own c1
      s1 += fma(W[7], C1.v0, fma(W[5], B0.v0, fma(W[4], A1.v0, W[1] * a.v0)));  // i-1 of c1 = own c0
      s1 += rgt;
#if BT_ST16
      double* p = yl + o;
      if ((ypar + (unsigned)o) & 1u) {  // warp-uniform
        const double nx = __shfl_down_sync(0xffffffffu, s0, 1);  // the next lane's c0
        st_pair(p + 1, s1, nx, LY, T1, T2);
      } else {
        st_pair(p, s0, s1, LY, T0, T1);
      }
#else
      double* p;
      asm("mad.wide.s32 %0, %1, 8, %2;" : "=l"(p) : "r"(o), "l"(yl));
      st_if(p, s0, LY, T0);
      st_if(p + 1, s1, LY, T1);
#endif
    };
    // phase P: am1 = R[P], a = R[P+1], new rows into R[P+2] (mod 3); c / C1 and qm1 / Q0 likewise in Cc, Qq
#define BT_STEP(P)                                                                                       \
  {                                                                                                      \
    constexpr int im = (P) % 3, ia = ((P) + 1) % 3, in = ((P) + 2) % 3;                                  \
    consume(Cc[ia], R[in], Qq[ia]);                                                                      \
    _Pragma("unroll") for (int q = 0; q < N; ++q) {                                                      \
      const int qu = q < N - 1 ? q + 1 : q, ql = q > 0 ? q - 1 : q; /* in-range indices */               \
      const Row2& b = q < N - 1 ? R[im][qu] : Qq[im];                                                    \
      const Row2& B0 = q < N - 1 ? R[ia][qu] : Qq[ia];                                                   \
      const Row2& c = q > 0 ? R[ia][ql] : Cc[im];                                                        \
      const Row2& Cn = q > 0 ? R[in][ql] : Cc[ia];                                                       \
      layer(R[ia][q], b, c, R[im][q], R[in][q], B0, Cn, LA - q, oy[q]);                                  \
      oy[q] += LA - q;                                                                                   \
    }                                                                                                    \
    --LA;                                                                                                \
    ++j;                                                                                                 \
  }
    while (true) {
      BT_STEP(0)
      if (j >= j1) break;
      BT_STEP(1)
      if (j >= j1) break;
      BT_STEP(2)
      if (j >= j1) break;
    }
#undef BT_STEP
  }
  cp_wait<0>();
  if (dyn && lane == 0) {
    const int total = G;
    if (atomicAdd(ctr + 1, 1) == total - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
}

template <int N, int kMaxC>
__global__ void __launch_bounds__(kFT, (N <= 2 ? 16 : (N <= 4 ? 12 : 8)) / kFW)
    k_stencil_fast(const double* __restrict__ x, double* __restrict__ y, const int4* __restrict__ tasks, int ntasks,
                   int w, int64_t cell_slots, const __grid_constant__ FastParams<kMaxC> fp, int* __restrict__ ctr) {
  extern __shared__ __align__(128) double ring_all[];
  stencil_fast_body<N, kMaxC>(x, y, tasks, ntasks, w, cell_slots, fp, blockIdx.x, gridDim.x, ring_all, ctr);
}

// Both ends of every fast row (1 <= k <= n-2, j >= 1, length L >= 3): the
// i = 0 vertex (zero set {i = 0}) and the diagonal-face vertex i = L - 1
// (zero set {S = n}), each from its typed partial row over its 11 present
// neighbours (per-cell part of partial_row_apply, operators.hpp:78-96). One
// thread per row; rows of a layer are consecutive threads, whose end vertices
// are each other's neighbours, so most loads hit L1.
__global__ void __launch_bounds__(128) k_stencil_ends(const double* __restrict__ x, double* __restrict__ y,
                                                      const double* __restrict__ ends, int w, int64_t cell_slots,
                                                      int cell0) {
  const int n = w - 1;
  const int k = blockIdx.y + 1, j = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (j > n - 2 - k) return;  // L = w - k - j >= 3
  const int cell = cell0 + blockIdx.z;
  const double* __restrict__ e = ends + 22 * (size_t)cell;  // [0, 11): diagonal face, [11, 22): i = 0
  const double* __restrict__ xc = x + (int64_t)cell * cell_slots;
  double* __restrict__ yc = y + (int64_t)cell * cell_slots;
  int off[15];
  row_offsets(w, j, k, off);
  const int t0 = row_start(w, j, k), tL = t0 + (w - k - j) - 1;
  constexpr int dp[11] = {0, 4, 5, 6, 8, 9, 10, 11, 12, 13, 14};  // kDiagPresent
  constexpr int ip[11] = {0, 1, 2, 3, 4, 5, 6, 7, 9, 10, 13};     // kI0Present
  double sd = 0.0, s0 = 0.0;
#pragma unroll
  for (int q = 0; q < 11; ++q) {
    sd = fma(__ldg(e + q), __ldg(xc + tL + off[dp[q]]), sd);
    s0 = fma(__ldg(e + 11 + q), __ldg(xc + t0 + off[ip[q]]), s0);
  }
  yc[tL] = sd;
  yc[t0] = s0;
}

// Fused boundary pass of apply_stencil (operators.hpp:247-271 with
// sync_additive fe_function.hpp:400-423 and the Dirichlet identity rows):
// every lattice point on a macro face, edge or vertex is computed once per
// interface group. For each member cell (ascending cell order) the point's
// per-cell partial row — the zero-set-typed row over the cell's micro-tets
// containing it (partial_row_apply, operators.hpp:78-96) — is evaluated from
// that cell's x; the partials are summed from 0.0 in member order, exactly
// the replica sum sync_additive forms from per-cell results, and the sum (or
// x on Dirichlet groups under BC::DirichletIdentity) is written to every
// replica. No dependency on the interior kernel: the two run concurrently.
struct BndArgs {
  const DevFace* faces;
  const DevPrimHdr* eh;
  const DevPrimMem* em;
  const DevPrimHdr* vh;
  const DevPrimMem* vm;
  const StencilCell* cells;
  int nf, ne, nv, n;
  int64_t cs;
  int cb, ce;  // this handle's cells: groups with a member outside are skipped (exchanged instead)
  // the groups this handle computes (every member local): indices into
  // faces / eh / vh; nf, ne, nv count these lists
  const int* lf;
  const int* le;
  const int* lv;
  // per-cell partial rows of the i = 0 and diagonal face-interior points,
  // precomputed by k_face_march (nullptr: gathered here like the other faces)
  const double* fpart = nullptr;
};
// slot of point (j, k) of local cell c, face f (0: i = 0, 1: diagonal) in fpart
__device__ __forceinline__ int64_t fpart_slot(int w, int c, int f, int j, int k) {
  return (int64_t)(2 * c + f) * tri32(w) + (k * w - k * (k - 1) / 2) + j;
}

// decode_tri (bt_index.cuh) with a single-precision first guess: the two
// correction loops make the result exact whatever the guess's rounding
__device__ __forceinline__ void decode_tri_f(int m, int q, int& a, int& b) {
  const float c = 2.0f * m + 1.0f;
  int bb = (int)((c - sqrtf(fmaxf(c * c - 8.0f * (float)q, 0.0f))) * 0.5f);
  bb = max(0, min(bb, m - 1));
  while (bb > 0 && bb * m - bb * (bb - 1) / 2 > q) --bb;
  while ((bb + 1) * m - (bb + 1) * bb / 2 <= q) ++bb;
  b = bb;
  a = q - (bb * m - bb * (bb - 1) / 2);
}

__device__ __forceinline__ void bary_ijk(const int8_t* lv, int nl, const int* wt, int& i, int& j, int& k) {
  i = j = k = 0;
  for (int q = 0; q < nl; ++q) {
    if (lv[q] == 1) i += wt[q];
    if (lv[q] == 2) j += wt[q];
    if (lv[q] == 3) k += wt[q];
  }
}

// The 15 neighbour values of lattice point (i, j, k) of `cell` — all loads
// issued at once (an absent direction, whose typed weight is 0, reads the
// point itself) — and its slot.
struct Gather15 {
  double v[15];
  const double* wz;  // the zero-set-typed row
};
__device__ __forceinline__ int64_t gather15(const double* __restrict__ x, const BndArgs& a, int cell, int i, int j,
                                            int k, Gather15& gt) {
  const int w = a.n + 1;
  const int z = zero_set(a.n, i, j, k);
  const StencilCell& sc = a.cells[cell];
  const uint32_t mask = __ldg(&sc.mask[z]);
  const int64_t slot = (int64_t)cell * a.cs + row_start(w, j, k) + i;
  const double* __restrict__ xc = x + slot;
  int off[15];
  row_offsets(w, j, k, off);
#pragma unroll
  for (int d = 0; d < 15; ++d) gt.v[d] = __ldg(xc + ((mask >> d) & 1 ? off[d] : 0));
  gt.wz = sc.w[z];
  return slot;
}
// Face-interior points: the zero set is one bit and the typed row has 11
// present directions (those not leaving the face's half-space).
template <int Z>
__device__ __forceinline__ constexpr int face_dir(int q) {
  constexpr int dg[11] = {0, 4, 5, 6, 8, 9, 10, 11, 12, 13, 14};  // diagonal face S = n: no dx + dy + dz = +1
  constexpr int di[11] = {0, 1, 2, 3, 4, 5, 6, 7, 9, 10, 13};     // i = 0: no dx = -1
  constexpr int dj[11] = {0, 1, 2, 3, 5, 6, 8, 10, 11, 12, 14};    // j = 0: no dy = -1
  constexpr int dk[11] = {0, 1, 2, 3, 4, 7, 8, 9, 11, 12, 13};     // k = 0: no dz = -1
  return Z == 1 ? dg[q] : (Z == 2 ? di[q] : (Z == 4 ? dj[q] : dk[q]));
}
struct Gather11 {
  double v[11];
  const double* wz;
  int z;
};
template <int Z>
__device__ __forceinline__ void gather11_z(const double* __restrict__ xc, int w, int j, int k, double* v) {
  int off[15];
  row_offsets(w, j, k, off);
#pragma unroll
  for (int q = 0; q < 11; ++q) v[q] = __ldg(xc + off[face_dir<Z>(q)]);
}
__device__ __forceinline__ void gather11(const double* __restrict__ x, const BndArgs& a, int cell, int i, int j, int k,
                                         Gather11& gt) {
  const int w = a.n + 1;
  gt.z = zero_set(a.n, i, j, k);  // one bit
  gt.wz = a.cells[cell].w[gt.z];
  const double* __restrict__ xc = x + (int64_t)cell * a.cs + row_start(w, j, k) + i;
  switch (gt.z) {
    case 1: gather11_z<1>(xc, w, j, k, gt.v); break;
    case 2: gather11_z<2>(xc, w, j, k, gt.v); break;
    case 4: gather11_z<4>(xc, w, j, k, gt.v); break;
    default: gather11_z<8>(xc, w, j, k, gt.v); break;
  }
}
template <int Z>
__device__ __forceinline__ double face_row_z(const double* __restrict__ wz, const double* v) {
  double acc = __ldg(wz) * v[0];  // direction 0 first, then ascending: the typed row's order
#pragma unroll
  for (int q = 1; q < 11; ++q) acc = fma(__ldg(wz + face_dir<Z>(q)), v[q], acc);
  return acc;
}
__device__ __forceinline__ double face_row(const Gather11& gt) {
  switch (gt.z) {
    case 1: return face_row_z<1>(gt.wz, gt.v);
    case 2: return face_row_z<2>(gt.wz, gt.v);
    case 4: return face_row_z<4>(gt.wz, gt.v);
    default: return face_row_z<8>(gt.wz, gt.v);
  }
}

// per-cell partial row (partial_row_apply, operators.hpp:78-96) from a gather
__device__ __forceinline__ double partial_row(const Gather15& gt) {
  double acc = __ldg(gt.wz) * gt.v[0];
#pragma unroll
  for (int d = 1; d < 15; ++d) acc = fma(__ldg(gt.wz + d), gt.v[d], acc);
  return acc;
}
__device__ __forceinline__ double typed_partial(const double* __restrict__ x, const BndArgs& a, int cell, int i,
                                                int j, int k, int64_t& slot) {
  Gather15 gt;
  slot = gather15(x, a, cell, i, j, k, gt);
  return partial_row(gt);
}

template <bool kDir>
__device__ __forceinline__ void boundary_body(const double* __restrict__ x, double* __restrict__ y, const BndArgs& a,
                                              int vblock) {
  const int n = a.n, w = n + 1;
  const int fpts = tri32(n - 2);
  int64_t q = (int64_t)vblock * blockDim.x + threadIdx.x;
  // the group: members as (cell, local-vertex map), barycentric weights
  int count, dir, nl;
  int wt[3];
  const DevFace* F = nullptr;
  const DevPrimMem* mem = nullptr;
  if (q < (int64_t)a.nf * fpts) {  // face-interior point (a, b), weights (n - a - b, a, b)
    // 32-bit index arithmetic where the point count allows (a 64-bit division is a subroutine)
    int fi, fr;
    if ((int64_t)a.nf * fpts < (int64_t(1) << 31)) {
      fi = (int)((uint32_t)q / (uint32_t)fpts);
      fr = (int)((uint32_t)q - (uint32_t)fi * (uint32_t)fpts);
    } else {
      fi = (int)(q / fpts);
      fr = (int)(q % fpts);
    }
    F = a.faces + __ldg(a.lf + fi);
    int ap, bp;
    decode_tri_f(n - 2, fr, ap, bp);
    wt[0] = n - (ap + 1) - (bp + 1);
    wt[1] = ap + 1;
    wt[2] = bp + 1;
    count = F->ncell;
    dir = F->dir;
    nl = 3;
  } else {
    q -= (int64_t)a.nf * fpts;
    DevPrimHdr h;
    if (q < (int64_t)a.ne * (n - 1)) {  // macro-edge point a = 1..n-1, weights (n - a, a)
      h = a.eh[__ldg(a.le + q / (n - 1))];
      mem = a.em + h.first;
      wt[1] = (int)(q % (n - 1)) + 1;
      wt[0] = n - wt[1];
      nl = 2;
    } else {  // macro vertex
      q -= (int64_t)a.ne * (n - 1);
      if (q >= a.nv) return;
      h = a.vh[__ldg(a.lv + q)];
      mem = a.vm + h.first;
      wt[0] = n;
      nl = 1;
    }
    count = h.count;
    dir = h.dir;
  }
  auto member = [&](int m, int& cell, int& i, int& j, int& k) {
    if (F) {
      cell = F->cell[m];
      bary_ijk(F->lv[m], 3, wt, i, j, k);
    } else {
      const DevPrimMem pm = mem[m];
      cell = pm.cell;
      bary_ijk(pm.lv, nl, wt, i, j, k);
    }
  };
  // partitioned grid: only groups whose members are all this handle's cells
  // (the rank-spanning ones go through the exchange, k_xpartials)
  for (int m = 0; m < count; ++m) {
    const int c = F ? F->cell[m] : mem[m].cell;
    if (c < a.cb || c >= a.ce) return;
  }
  double sum = 0.0, single = 0.0;
  if (F) {  // face point: one or two members, all their loads in flight together
    Gather11 g0, g1;
    int cell, i, j, k;
    double pre[2] = {0.0, 0.0};
    bool has[2] = {false, false};
    auto fetch = [&](int m, Gather11& g) {
      member(m, cell, i, j, k);
      const int z = zero_set(n, i, j, k);
      if (a.fpart && (z == 1 || z == 2)) {  // strided faces: the march kernel's partial row
        has[m] = true;
        pre[m] = __ldg(a.fpart + fpart_slot(w, cell - a.cb, z == 2 ? 0 : 1, j, k));
      } else {
        gather11(x, a, cell, i, j, k, g);
      }
    };
    fetch(0, g0);
    if (count == 2) fetch(1, g1);
    single = has[0] ? pre[0] : face_row(g0);
    sum += single;
    if (count == 2) {
      single = has[1] ? pre[1] : face_row(g1);
      sum += single;
    }
  } else {
    for (int m = 0; m < count; ++m) {
      int cell, i, j, k;
      member(m, cell, i, j, k);
      int64_t slot;
      single = typed_partial(x, a, cell, i, j, k, slot);
      sum += single;
    }
  }
  if (count < 2) sum = single;  // no replicas: sync_additive leaves the value alone
  for (int m = 0; m < count; ++m) {
    int cell, i, j, k;
    member(m, cell, i, j, k);
    const int64_t slot = (int64_t)cell * a.cs + row_start(w, j, k) + i;
    y[slot] = (kDir && dir) ? __ldg(x + slot) : sum;
  }
}

template <bool kDir>
__global__ void __launch_bounds__(128) k_boundary(const double* __restrict__ x, double* __restrict__ y, BndArgs a) {
  boundary_body<kDir>(x, y, a, blockIdx.x);
}

// Per-cell partial rows of the two strided faces of every local cell: the
// i = 0 face (F = 0) and the diagonal face i + j + k = n (F = 1). Their
// face-interior points (j, k >= 1, j + k <= n - 1) sit at one end of row
// (j, k), a row length apart in memory, so a gather per point (k_boundary)
// costs 11 single-lane L1 wavefronts. Here a warp owns 30 consecutive j and
// marches k: each lane loads only the two end values of its row (j, k + 1) per
// step, keeps the pairs of layers k - 1, k, k + 1 in registers, and gets rows
// j - 1, j + 1 from the neighbour lanes by shuffle: 2 loads per point. The
// partial row is evaluated in k_boundary's order (direction 0, then the
// present directions ascending), so the values are bitwise the gathered ones.
// Task: x = local cell | face << 16, y = j block, z = k0, w = k1.
constexpr int kFaceCols = 30;
constexpr int kFaceChunk = 8;  // layers per task (plus two phantom steps)
template <int F>
__device__ __forceinline__ double2 face_pair(const double* __restrict__ xc, int w, int j, int k) {
  // F = 0: (x[0], x[1]) of row (j, k); F = 1: (x[L - 2], x[L - 1]); 0.0 where the row has no such entry
  const int L = w - j - k;
  if (j < 0 || k < 0 || L < 1) return make_double2(0.0, 0.0);
  const double* r = xc + row_start(w, j, k);
  if (F == 0) return make_double2(__ldg(r), L >= 2 ? __ldg(r + 1) : 0.0);
  return make_double2(L >= 2 ? __ldg(r + L - 2) : 0.0, __ldg(r + L - 1));
}
struct FacePair {  // a row's end pair and its copies from the rows j - 1 (up) and j + 1 (dn)
  double v0, v1, u0, u1, d0, d1;
};
__device__ __forceinline__ FacePair face_spread(double2 p) {
  FacePair q;
  q.v0 = p.x;
  q.v1 = p.y;
  q.u0 = __shfl_up_sync(0xffffffffu, p.x, 1);
  q.u1 = __shfl_up_sync(0xffffffffu, p.y, 1);
  q.d0 = __shfl_down_sync(0xffffffffu, p.x, 1);
  q.d1 = __shfl_down_sync(0xffffffffu, p.y, 1);
  return q;
}
template <int F>
__device__ __forceinline__ void face_march_body(const double* __restrict__ x, double* __restrict__ fpart,
                                                const StencilCell* __restrict__ cells, int4 T, int n, int64_t cs,
                                                int cb) {
  const int w = n + 1, lane = threadIdx.x & 31;
  const int lc = T.x & 0xffff, cell = cb + lc;
  const int j = kFaceCols * T.y + lane;  // lanes 1..30 hold outputs, 0 and 31 their neighbours
  const double* __restrict__ xc = x + (int64_t)cell * cs;
  const double* __restrict__ wz = cells[cell].w[F == 0 ? 2 : 1];
  constexpr int dirs0[11] = {0, 1, 2, 3, 4, 5, 6, 7, 9, 10, 13};
  constexpr int dirs1[11] = {0, 4, 5, 6, 8, 9, 10, 11, 12, 13, 14};
  double W[11];
#pragma unroll
  for (int q = 0; q < 11; ++q) W[q] = __ldg(wz + (F == 0 ? dirs0[q] : dirs1[q]));
  const int k0 = T.z, k1 = T.w;
  FacePair C = face_spread(face_pair<F>(xc, w, j, k0 - 1));  // layer k - 1
  FacePair A = face_spread(face_pair<F>(xc, w, j, k0));      // layer k
  double2 nx = face_pair<F>(xc, w, j, k0 + 1);
  for (int k = k0; k < k1; ++k) {
    const FacePair B = face_spread(nx);  // layer k + 1
    nx = face_pair<F>(xc, w, j, k + 2);  // in flight during this step
    double acc;
    if (F == 0) {
      acc = W[0] * A.v0;
      acc = fma(W[1], A.v1, acc);   // (1, 0, 0)
      acc = fma(W[2], A.d0, acc);   // (0, 1, 0)
      acc = fma(W[3], B.v0, acc);   // (0, 0, 1)
      acc = fma(W[4], A.u1, acc);   // (1, -1, 0)
      acc = fma(W[5], C.v1, acc);   // (1, 0, -1)
      acc = fma(W[6], C.d0, acc);   // (0, 1, -1)
      acc = fma(W[7], B.u1, acc);   // (1, -1, 1)
      acc = fma(W[8], A.u0, acc);   // (0, -1, 0)
      acc = fma(W[9], C.v0, acc);   // (0, 0, -1)
      acc = fma(W[10], B.u0, acc);  // (0, -1, 1)
    } else {
      acc = W[0] * A.v1;
      acc = fma(W[1], A.u1, acc);   // (1, -1, 0): row j - 1's last
      acc = fma(W[2], C.v1, acc);   // (1, 0, -1): layer k - 1's last
      acc = fma(W[3], C.d1, acc);   // (0, 1, -1)
      acc = fma(W[4], A.v0, acc);   // (-1, 0, 0)
      acc = fma(W[5], A.u0, acc);   // (0, -1, 0)
      acc = fma(W[6], C.v0, acc);   // (0, 0, -1)
      acc = fma(W[7], A.d1, acc);   // (-1, 1, 0): row j + 1's last
      acc = fma(W[8], B.v1, acc);   // (-1, 0, 1)
      acc = fma(W[9], B.u1, acc);   // (0, -1, 1)
      acc = fma(W[10], C.d0, acc);  // (-1, 1, -1)
    }
    if (lane >= 1 && lane <= kFaceCols && j + k <= n - 1) fpart[fpart_slot(w, lc, F, j, k)] = acc;
    C = A;
    A = B;
  }
}
__global__ void __launch_bounds__(128) k_face_march(const double* __restrict__ x, double* __restrict__ fpart,
                                                    const StencilCell* __restrict__ cells,
                                                    const int4* __restrict__ tasks, int ntasks, int n, int64_t cs,
                                                    int cb) {
  const int t = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (t >= ntasks) return;
  const int4 T = tasks[t];
  if (T.x >> 16)
    face_march_body<1>(x, fpart, cells, T, n, cs, cb);
  else
    face_march_body<0>(x, fpart, cells, T, n, cs, cb);
}

// Rank-spanning interface groups of a partitioned fused apply: this rank's
// members' per-cell partial rows (the same typed rows, in the same operation
// order, as k_boundary forms them) straight into the exchange buffer; after
// the ranks' allreduce, k_xcombine sums every group in member order from 0.0,
// which is k_boundary's replica sum bit for bit.
__global__ void __launch_bounds__(128) k_xpartials(const double* __restrict__ x, double* __restrict__ buf,
                                                   const XEntry* __restrict__ e, const int4* __restrict__ pts,
                                                   int nent, BndArgs a) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nent) return;
  const int4 P = pts[q];
  const int z = zero_set(a.n, P.y, P.z, P.w);
  double v;
  if (__popc(z) == 1) {  // face point: its 11 present directions
    Gather11 gt;
    gather11(x, a, P.x, P.y, P.z, P.w, gt);
    v = face_row(gt);
  } else {
    int64_t slot;
    v = typed_partial(x, a, P.x, P.y, P.z, P.w, slot);
  }
  buf[e[q].buf] = v;
}

// Small problems (one launch is latency, not bandwidth): the whole fused
// apply in one kernel — blocks [0, b4) run the 4-layer marches, [b4, b4 + b2)
// the 2-layer group, the rest the boundary points. The three sets of points
// are disjoint, so the roles need no ordering.
template <bool kDir>
__global__ void __launch_bounds__(kFT, 12 / kFW)
    k_stencil_small(const double* __restrict__ x, double* __restrict__ y, const int4* __restrict__ t4, int n4,
                    const int4* __restrict__ t2, int n2, int w, int64_t cell_slots, int b4, int b2, BndArgs a,
                    const __grid_constant__ FastParams<kMaxCells> fp) {
  extern __shared__ __align__(128) double ring_all[];
  const int b = blockIdx.x;
  if (b < b4)
    stencil_fast_body<kGroup, kMaxCells>(x, y, t4, n4, w, cell_slots, fp, b, b4, ring_all);
  else if (b < b4 + b2)
    stencil_fast_body<2, kMaxCells>(x, y, t2, n2, w, cell_slots, fp, b - b4, b2, ring_all);
  else
    boundary_body<kDir>(x, y, a, b - b4 - b2);
}

// Any rows of the march schedule, every row read from the zero-set-typed
// table in shared memory (interior vertices use type 0 = the merged row).
// Block row y works on cell cell0 + y; every cell runs all ntasks.
__global__ void __launch_bounds__(kGT, 9) k_stencil_general(const double* __restrict__ x, double* __restrict__ y,
                                                        const StencilCell* __restrict__ cells,
                                                        const int4* __restrict__ tasks, int ntasks, int w,
                                                        int64_t cell_slots, int cell0) {
  __shared__ double sw[16][15];
  const int cell = cell0 + blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int task = blockIdx.x * kGW + warp;
  {
    const double* src = cells[cell].w[0];
    for (int q = threadIdx.x; q < 16 * 15; q += blockDim.x) sw[q / 15][q % 15] = src[q];
  }
  __syncthreads();
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
  static const int env_march = std::getenv("BT_STENCIL_MARCH") ? std::atoi(std::getenv("BT_STENCIL_MARCH")) : 0;
  std::vector<int4> fast, fast2, gen, all;  // fast: groups of kGroup layers; fast2: the 2-layer group
  {  // k_face_march tasks: (local cell, face) x j block x k chunk, longest first
    std::vector<int4> ft;
    const int ncl = st.grid->part_end - st.grid->part_begin;
    for (int kc = 1; kc <= n - 2; kc += kFaceChunk)
      for (int b = 0; kFaceCols * b + 1 <= n - 1 - kc; ++b)
        for (int f = 0; f < 2; ++f)
          for (int c = 0; c < ncl; ++c)
            ft.push_back(make_int4(c | (f << 16), b, kc, std::min(kc + kFaceChunk, n - 1 - (kFaceCols * b + 1) + 1)));
    st.nftasks = (int)ft.size();
    st.d_ftasks.upload(ft);
    if (std::getenv("BT_STENCIL_FACEMARCH") && std::atoi(std::getenv("BT_STENCIL_FACEMARCH")))
      st.d_fpart.alloc((size_t)2 * std::max(1, ncl) * tri32(w));
  }
  for (FastTasks* ft : {&st.fast4, &st.fast2}) {
    ft->segs.clear();
    ft->sched.clear();
    ft->d_ctr.alloc(2);
    BT_CUDA(cudaMemset(ft->d_ctr.p, 0, 2 * sizeof(int)));
  }
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
    // fast marches: groups of kGroup layers k .. k+kGroup-1 starting at
    // k = 1, then one group of 2 (n - 2 fast layers, n - 2 = 2 mod 4)
    const int ng = (n - 2) / kGroup;
    const bool start4 = fast_layer && (k - 1) % kGroup == 0 && (k - 1) / kGroup < ng;
    const bool start2 = fast_layer && k == 1 + ng * kGroup && k + 1 <= n - 2;
    if (!start4 && !start2) continue;
    for (int b = 0; kFastCols * b < w - k; ++b) {  // fast blocks (62 wide)
      const int jmax = w - k - kFastCols * b;
      // layer k's fast rows: in block b >= 1 the row whose only column here is its diagonal end (L = 62 b + 1)
      // has no interior output
      const int fe = b == 0 ? std::min(jmax, w - k - 2) : jmax - 1;
      if (fe > 1) (start4 ? st.fast4 : st.fast2).segs.push_back(make_int4(k, b, 1, fe));
    }
  }
  // March length. Every march costs two phantom steps, so long marches mean
  // less work, and the idle tail their coarser balance leaves is where the
  // boundary kernel runs (config 2: 32 rows 84.1, 64 rows 81.5, 128 rows 91.7
  // us per apply). With little work per warp (level 7 on one GPU: 64 rows
  // 27.9 us against 18.9) the marches stay short, and the single-launch
  // path's are shorter still.
  int march = kSmallMarch;
  if ((int64_t)(st.grid->part_end - st.grid->part_begin) * n_tet(w) > kSmallSlots) {
    int64_t rows = 0;
    for (const int4& sg : st.fast4.segs) rows += sg.w - sg.z;
    rows *= st.grid->part_end - st.grid->part_begin;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, st.grid->device);
    march = rows / (12 * (int64_t)sms) >= 40 ? kMarchRows : kMarchRows / 2;
    if (env_march > 0) march = env_march;
  }
  for (int pass = 0; pass < 2; ++pass)
    for (const int4& sg : (pass == 0 ? st.fast4 : st.fast2).segs)
      for (int j0 = sg.z; j0 < sg.w; j0 += march)
        (pass == 0 ? fast : fast2).push_back(make_int4(sg.x, sg.y, j0, std::min(j0 + march, sg.w)));
  if ((n - 2) % kGroup != 0 && (n - 2) % kGroup != 2)
    raise(BT_LOGIC_ERROR, "stencil: fast layer count must be 0 or 2 mod the group size");
  // Fast tasks of every cell of this handle, in chunks of kMaxCells cells
  // (the kernel's parameter table); longest marches first.
  // Task order (BT_STENCIL_ORDER, profiling): 1 = longest march first, cells
  // interleaved (default: best balance); 0 = spatial, cells outermost (better
  // L2 reuse of staged rows, but a longer tail: measured slower).
  static const int order = [] {
    const char* e = std::getenv("BT_STENCIL_ORDER");
    return e ? std::atoi(e) : 1;
  }();
  st.part_begin = st.grid->part_begin;
  st.part_end = st.grid->part_end;
  auto build = [&](std::vector<int4>& list, FastTasks& out) {
    if (order == 1)
      std::stable_sort(list.begin(), list.end(), [](const int4& a, const int4& b) { return a.w - a.z > b.w - b.z; });
    std::vector<int4> all_fast;
    out.chunk_first.clear();
    for (int c0 = st.part_begin; c0 < st.part_end; c0 += kMaxCells) {
      out.chunk_first.push_back((int)all_fast.size());
      const int cnt = std::min(kMaxCells, st.part_end - c0);
      const int64_t ntc = (int64_t)list.size() * cnt;
      for (int64_t q = 0; q < ntc; ++q) {
        const int c = order == 1 ? (int)(q % cnt) : (int)(q / (int64_t)list.size());
        const int4& t = list[order == 1 ? (size_t)(q / cnt) : (size_t)(q % (int64_t)list.size())];
        all_fast.push_back(make_int4(t.x, t.y | (c << 16), t.z, t.w));
      }
    }
    out.chunk_first.push_back((int)all_fast.size());
    out.ntasks = (int)all_fast.size();
    out.d_tasks.upload(all_fast);
  };
  build(fast, st.fast4);
  build(fast2, st.fast2);
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
  st.fast.assign(8 * (size_t)nc, 0.0);
  std::vector<double> ends(22 * (size_t)nc, 0.0);
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
      // the boundary kernel's face rows use 11 fixed directions per face zero set
      static const int fdirs[4][11] = {{0, 4, 5, 6, 8, 9, 10, 11, 12, 13, 14}, {0, 1, 2, 3, 4, 5, 6, 7, 9, 10, 13},
                                       {0, 1, 2, 3, 5, 6, 8, 10, 11, 12, 14}, {0, 1, 2, 3, 4, 7, 8, 9, 11, 12, 13}};
      for (int f = 0; f < 4; ++f) {
        bool in = false;
        for (int q = 0; q < 11; ++q) in = in || fdirs[f][q] == d;
        if (!in && cells[c].w[1 << f][d] != 0.0) st.symmetric = false;
      }
    }
    double* f = &st.fast[8 * (size_t)c];
    for (int d = 0; d < 8; ++d) f[d] = rw[d];
    for (int q = 0; q < 11; ++q) {
      ends[22 * (size_t)c + q] = cells[c].w[1][kDiagPresent[q]];
      ends[22 * (size_t)c + 11 + q] = cells[c].w[2][kI0Present[q]];
    }
  }
  st.d_ends.upload(ends);
  // the interface groups whose members are all this handle's cells (k_boundary)
  {
    const Topology& t = st.grid->topo;
    auto local = [&](int c) { return c >= st.part_begin && c < st.part_end; };
    std::vector<int> lf, le, lv;
    for (int f = 0; f < (int)t.faces.size(); ++f) {
      bool ok = true;
      for (int m = 0; m < t.faces[f].ncell; ++m) ok = ok && local(t.faces[f].cell[m]);
      if (ok) lf.push_back(f);
    }
    auto prims = [&](const std::vector<DevPrimHdr>& hs, const std::vector<DevPrimMem>& mem, std::vector<int>& out) {
      for (int e = 0; e < (int)hs.size(); ++e) {
        bool ok = true;
        for (int m = 0; m < hs[e].count; ++m) ok = ok && local(mem[hs[e].first + m].cell);
        if (ok) out.push_back(e);
      }
    };
    prims(t.ehdr, t.emem, le);
    prims(t.vhdr, t.vmem, lv);
    st.bnd_f.upload(lf);
    st.bnd_e.upload(le);
    st.bnd_v.upload(lv);
  }
  init_prism_tasks(st);
}

namespace {
// side stream (per device) and fork/join events for the small kernels
}  // namespace

// per host thread and device, so concurrent host threads never share the
// fork/join events
SideStream& side_stream() {
  static thread_local SideStream ss[16];
  int dev = 0;
  BT_CUDA(cudaGetDevice(&dev));
  SideStream& r = ss[dev & 15];
  if (!r.s) {
    BT_CUDA(cudaStreamCreateWithFlags(&r.s, cudaStreamNonBlocking));
    BT_CUDA(cudaStreamCreateWithFlags(&r.s2, cudaStreamNonBlocking));
    BT_CUDA(cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming));
    BT_CUDA(cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming));
    BT_CUDA(cudaEventCreateWithFlags(&r.join2, cudaEventDisableTiming));
  }
  return r;
}

// BT_STENCIL_PARTS (profiling only) drops parts of an apply: bit 0 interior
// kernel, 1 row ends, 2 general rows, 3 fused boundary kernel; bit 4 set
// selects k_stencil_prism (bt_prism.cu) for the interior instead of the
// k_stencil_fast marches.
static int stencil_parts() {
  static const int parts = [] {
    const char* e = std::getenv("BT_STENCIL_PARTS");
    return e ? std::atoi(e) : 15;
  }();
  return parts;
}

// fast kernel launches (interior rows of the N-layer marches in ft) for this
// handle's cells, on stream s

// Balanced schedule of one chunk's fast marches over G persistent warps. The
// column segments (cell, layer group, column block; rows j0..j1) are cut so
// that every warp's list costs the same number of march steps (a piece of r
// rows costs r + 2: two phantom steps fill the register window): segments are
// dealt in order, a warp taking rows until its list reaches the target, so
// consecutive warps work on consecutive pieces of the same segment. (The
// round-1 schedule of fixed 32-row marches dealt round-robin left 1,776 warps
// with 58.4 steps on average and 68 at most at level 8.)
static const FastSched& build_sched(const FastTasks& ft, int chunk, int cnt, int G) {
  auto& slot = ft.sched[{chunk, G}];
  if (slot) return *slot;
  constexpr int kMinPiece = 6;  // rows; shorter pieces only where a segment ends
  int64_t rows = 0;
  for (const int4& sg : ft.segs) rows += sg.w - sg.z;
  rows *= cnt;
  const int64_t nseg = (int64_t)ft.segs.size() * cnt;
  std::vector<std::vector<int4>> lists;
  for (int64_t T = (rows + 2 * (nseg + G) + G - 1) / G;; ++T) {
    lists.assign(G, {});
    int g = 0, load = 0;
    bool fits = true;
    for (size_t si = 0; si < ft.segs.size() && fits; ++si) {
      for (int c = 0; c < cnt && fits; ++c) {
        const int4 sg = ft.segs[si];
        int j = sg.z;
        while (j < sg.w) {
          const int rem = sg.w - j, room = (int)T - load - 2;
          if (room >= std::min(rem, kMinPiece)) {
            int take = std::min(rem, room);
            if (rem - take > 0 && rem - take < kMinPiece && take - (kMinPiece - (rem - take)) >= kMinPiece)
              take -= kMinPiece - (rem - take);  // leave a remainder worth its two phantom steps
            lists[g].push_back(make_int4(sg.x, sg.y | (c << 16), j, j + take));
            load += take + 2;
            j += take;
          } else if (++g < G) {
            load = 0;
          } else {
            fits = false;
            break;
          }
        }
      }
    }
    if (fits) break;
  }
  size_t slots = 1;
  for (const auto& l : lists) slots = std::max(slots, l.size());
  std::vector<int4> flat(slots * (size_t)G, make_int4(1, 0, 1, -1));  // null task: no steps (w - z + 2 == 0)
  for (int g = 0; g < G; ++g)
    for (size_t q = 0; q < lists[g].size(); ++q) flat[q * G + g] = lists[g][q];
  slot = std::make_unique<FastSched>();
  slot->ntasks = (int)flat.size();
  slot->d_tasks.upload(flat);
  return *slot;
}

template <int N>
static void launch_fast(const bt_stencil& st, const FastTasks& ft, const double* x, double* y, cudaStream_t s,
                        int reserve_sms = 0) {
  if (!ft.ntasks) return;
  const int w = (1 << st.level) + 1;
  const int64_t cs = n_tet(w);
  // BT_STENCIL_PAD (profiling): extra dynamic shared memory per block, to lower the resident blocks per SM
  static const size_t pad = std::getenv("BT_STENCIL_PAD") ? (size_t)std::atoi(std::getenv("BT_STENCIL_PAD")) : 0;
  const size_t smem = sizeof(double) * kFW * ring_doubles<N>() + sizeof(int4) * 4 * kFW + (N == kGroup ? pad : 0);
  auto kern = k_stencil_fast<N, kMaxCells>;
  // persistent grid: SMs x resident blocks, per device (set up once)
  static std::mutex mu;
  static int grids[64] = {0}, persm[64] = {0};
  int dev = 0;
  BT_CUDA(cudaGetDevice(&dev));
  int grid, per_sm;
  {
    std::lock_guard<std::mutex> lock(mu);
    int& gr = grids[dev & 63];
    if (!gr) {
      BT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int sms = 0, ps = 0;
      BT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      BT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, kFT, smem));
      persm[dev & 63] = std::max(1, ps);
      gr = sms * persm[dev & 63];
    }
    grid = gr;
    per_sm = persm[dev & 63];
  }
  // BT_STENCIL_SCHED (profiling): 0 = the round-1 schedule (fixed 32-row marches dealt round-robin, longest first)
  // 1 = balanced static lists (build_sched), 2 = dynamic queue
  static const int sched = [] {
    const char* e = std::getenv("BT_STENCIL_SCHED");
    return e ? std::atoi(e) : 0;
  }();
  const bool balanced = sched == 1;
  FastParams<kMaxCells> fp;  // copied into the launch's parameter buffer
  for (int ch = 0; ch + 1 < (int)ft.chunk_first.size(); ++ch) {
    const int cc0 = st.part_begin + ch * kMaxCells, cnt = std::min(kMaxCells, st.part_end - cc0);
    const int t0 = ft.chunk_first[ch], nt = ft.chunk_first[ch + 1] - t0;
    if (!nt) continue;
    for (int c = 0; c < cnt; ++c) {
      const double* f = &st.fast[8 * (size_t)(cc0 + c)];
      for (int d = 0; d < 8; ++d) fp.w[c][d] = f[d];
    }
    const int64_t e0 = (int64_t)cc0 * cs;
    // reserve_sms: leave SMs free for concurrent kernels (exchange, boundary)
    const int avail = std::max(per_sm, grid - reserve_sms * per_sm);
    // one warp per ~40 march steps at least, else the whole persistent grid;
    // little work (under half the grid at that rate) keeps the short marches
    int64_t cost = 0;
    for (const int4& sg : ft.segs) cost += sg.w - sg.z + 2;
    cost *= cnt;
    if (balanced && cost / (40 * kFW) >= avail / 2) {
      const int blocks = (int)std::min<int64_t>(avail, std::max<int64_t>(1, cost / (40 * kFW)));
      std::lock_guard<std::mutex> lock(mu);
      const FastSched& sc = build_sched(ft, ch, cnt, blocks * kFW);
      kern<<<blocks, kFT, smem, s>>>(x + e0, y + e0, sc.d_tasks.p, sc.ntasks, w, cs, fp, nullptr);
    } else {
      const int blocks = std::min(avail, (nt + kFW - 1) / kFW);
      // enough tasks per warp: dynamic queue (the list is sorted longest first)
      int* ctr = nullptr;
      if (sched == 2 && nt > blocks * kFW) ctr = ft.d_ctr.p;
      kern<<<blocks, kFT, smem, s>>>(x + e0, y + e0, ft.d_tasks.p + t0, nt, w, cs, fp, ctr);
    }
    count_launch();
  }
}

void launch_stencil(const bt_stencil& st, const double* x, double* y, cudaStream_t s, int xmode) {
  const int w = (1 << st.level) + 1;
  const int64_t cs = n_tet(w);
  if (st.part_begin != st.grid->part_begin || st.part_end != st.grid->part_end)
    raise(BT_LOGIC_ERROR, "apply_stencil: the grid was repartitioned after compute_stencil");
  const int c0 = st.part_begin, nc = st.part_end - st.part_begin;  // this handle's cells
  const double* xl = x;  // local pointers (for the interface pass)
  double* yl = y;
  x = shifted(x, *st.grid, BT_SPACE_P1, st.level);  // local -> global-cell indexing
  y = shifted(y, *st.grid, BT_SPACE_P1, st.level);
  if (!st.symmetric || !nc) {
    if (nc) {
      k_stencil_general<<<dim3((st.natasks + kGW - 1) / kGW, nc), kGT, 0, s>>>(x, y, st.d_cells.p, st.d_atasks.p,
                                                                              st.natasks, w, cs, c0);
      count_launch();
      check_launch("k_stencil_general");
    }
    if (xmode >= 0) sync(*st.grid, st.level, (IfaceMode)xmode, yl, xl, s);
    return;
  }
  // The rows that hold the lattice-boundary (interface) points — row ends and
  // general rows — go first, on the side stream, followed there by the
  // interface pass (xmode >= 0: including the rank exchange), so the
  // exchange overlaps the interior marches on s. The two sets of points are
  // disjoint: the interior kernels write interior points only.
  const int parts = stencil_parts();
  SideStream& ss = side_stream();
  BT_CUDA(cudaEventRecord(ss.fork, s));
  BT_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
  if ((parts & 2) && w - 1 >= 4) {
    const int n = w - 1;
    k_stencil_ends<<<dim3((n - 3 + 127) / 128, n - 3, nc), 128, 0, ss.s>>>(x, y, st.d_ends.p, w, cs, c0);
    count_launch();
  }
  if ((parts & 4) && st.ngtasks) {
    k_stencil_general<<<dim3((st.ngtasks + kGW - 1) / kGW, nc), kGT, 0, ss.s>>>(x, y, st.d_cells.p, st.d_gtasks.p,
                                                                               st.ngtasks, w, cs, c0);
    count_launch();
  }
  if (parts & 1) launch_fast<kGroup>(st, st.fast4, x, y, s);
  if (parts & 1) launch_fast<2>(st, st.fast2, x, y, s);  // the 2-layer group
  if (xmode >= 0) sync(*st.grid, st.level, (IfaceMode)xmode, yl, xl, ss.s);
  BT_CUDA(cudaEventRecord(ss.join, ss.s));
  BT_CUDA(cudaStreamWaitEvent(s, ss.join, 0));
  check_launch("k_stencil");
}

bool stencil_fused(const bt_stencil& st) {
  return st.symmetric;
}

static void launch_stencil_small(const bt_stencil& st, const double* x, double* y, int bc, cudaStream_t s) {
  const bt_grid& g = *st.grid;
  const int n = 1 << st.level, w = n + 1;
  const int64_t cs = n_tet(w);
  BndArgs a{g.d_faces.p, g.d_ehdr.p, g.d_emem.p, g.d_vhdr.p, g.d_vmem.p, st.d_cells.p,
            (int)st.bnd_f.n, (int)st.bnd_e.n, (int)st.bnd_v.n, n, cs, 0, g.mesh.n_cells(),
            st.bnd_f.p, st.bnd_e.p, st.bnd_v.p};
  const int64_t pts = (int64_t)a.nf * tri32(n - 2) + (int64_t)a.ne * (n - 1) + a.nv;
  const int n4 = st.fast4.ntasks, n2 = st.fast2.ntasks;
  const int b4 = (n4 + kFW - 1) / kFW, b2 = (n2 + kFW - 1) / kFW;
  const int bb = (int)((pts + kFT - 1) / kFT);
  const size_t smem = sizeof(double) * kFW * ring_doubles<kGroup>();
  static std::once_flag once[2];
  auto kern = bc ? k_stencil_small<true> : k_stencil_small<false>;
  std::call_once(once[bc ? 1 : 0], [&] {
    BT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  FastParams<kMaxCells> fp;
  for (int c = 0; c < g.mesh.n_cells(); ++c)
    for (int d = 0; d < 8; ++d) fp.w[c][d] = st.fast[8 * (size_t)c + d];
  kern<<<b4 + b2 + bb, kFT, smem, s>>>(x, y, st.fast4.d_tasks.p, n4, st.fast2.d_tasks.p, n2, w, cs, b4, b2, a, fp);
  count_launch();
  check_launch("k_stencil_small");
}

void launch_stencil_fused(const bt_stencil& st, const double* x, double* y, int bc, cudaStream_t s) {
  const bt_grid& g = *st.grid;
  const int n = 1 << st.level;
  const int parts = stencil_parts();
  const bool part = g.part_nranks > 1;
  if (st.part_begin != g.part_begin || st.part_end != g.part_end)
    raise(BT_LOGIC_ERROR, "apply_stencil: the grid was repartitioned after compute_stencil");
  if (!part && parts == 15 && g.mesh.n_cells() <= kMaxCells &&
      (int64_t)g.mesh.n_cells() * n_tet(n + 1) <= kSmallSlots) {
    launch_stencil_small(st, x, y, bc, s);
    return;
  }
  const double* xl = x;  // local pointers (the exchange's combine shifts them itself)
  double* yl = y;
  x = shifted(x, g, BT_SPACE_P1, st.level);  // local -> global-cell indexing
  y = shifted(y, g, BT_SPACE_P1, st.level);
  BndArgs a{g.d_faces.p, g.d_ehdr.p, g.d_emem.p, g.d_vhdr.p, g.d_vmem.p, st.d_cells.p,
            (int)st.bnd_f.n, (int)st.bnd_e.n, (int)st.bnd_v.n, n, n_tet(n + 1),
            g.part_begin, g.part_end, st.bnd_f.p, st.bnd_e.p, st.bnd_v.p};
  SideStream& ss = side_stream();
  BT_CUDA(cudaEventRecord(ss.fork, s));
  // partitioned: the rank-spanning groups' partial rows go first, on the side
  // stream, so the exchange overlaps the interior marches; SMs are reserved
  // beside the persistent interior grid for it and the boundary kernel
  static const int env_reserve = getenv("BT_STENCIL_RESERVE") ? atoi(getenv("BT_STENCIL_RESERVE")) : -1;
  const int reserve = env_reserve >= 0 ? env_reserve : (part ? 12 : 0);
  if (part && (parts & 8)) {
    const XPlan& p = xchg_plan(g, st.level);
    if (p.buf_size) {
      BT_CUDA(cudaStreamWaitEvent(ss.s2, ss.fork, 0));
      if (g.xbuf.n < (size_t)p.buf_size) g.xbuf.alloc((size_t)p.buf_size);
      BT_CUDA(cudaMemsetAsync(g.xbuf.p, 0, sizeof(double) * (size_t)p.buf_size, ss.s2));
      const int ne = (int)p.entries.size();
      if (ne) {
        k_xpartials<<<(ne + 127) / 128, 128, 0, ss.s2>>>(x, g.xbuf.p, p.d_entries.p, p.d_pts.p, ne, a);
        count_launch();
      }
      exchange_buffer(g, p, g.xbuf.p, ss.s2);
      launch_xchg_combine(g, st.level, bc ? IF_SYNC_DIR : IF_SYNC, yl, xl, g.xbuf.p, ss.s2);
      BT_CUDA(cudaEventRecord(ss.join2, ss.s2));
    } else {
      BT_CUDA(cudaEventRecord(ss.join2, s));  // nothing to exchange
    }
  }
  const bool prism = !part && prism_ok(st, x) && (parts & 16);
  if (prism) {
    if (parts & 1) launch_prism(st, x, y, s);  // every interior point (bt_prism.cu)
    BT_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
  } else {
    if (parts & 1) launch_fast<kGroup>(st, st.fast4, x, y, s, reserve);  // first: its blocks resident first
    BT_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
    if (parts & 1) launch_fast<2>(st, st.fast2, x, y, ss.s, reserve);  // the 2-layer group, beside the main launch
  }
  // BT_STENCIL_FACEMARCH=1 (opt-in): the strided faces' partial rows by warp marches (k_face_march) instead of
  // k_boundary's gathers. Bitwise the same values; measured slower in the whole apply (92.5 vs 85.1 us at config 2:
  // k_boundary stays instruction-bound, 8.3 M instead of 9.6 M warp instructions, and the march adds a 13 us
  // latency-bound pass), profiles/r2_notes.md section 7.
  static const bool facemarch = std::getenv("BT_STENCIL_FACEMARCH") && std::atoi(std::getenv("BT_STENCIL_FACEMARCH"));
  if ((parts & 8) && facemarch && st.nftasks && a.nf && st.d_fpart.n) {
    k_face_march<<<(st.nftasks + 3) / 4, 128, 0, ss.s>>>(x, st.d_fpart.p, st.d_cells.p, st.d_ftasks.p, st.nftasks, n,
                                                        n_tet(n + 1), g.part_begin);
    count_launch();
    a.fpart = st.d_fpart.p;
  }
  if ((parts & 8) && (int64_t)a.nf * tri32(n - 2) + (int64_t)a.ne * (n - 1) + a.nv > 0) {
    const int64_t pts = (int64_t)a.nf * tri32(n - 2) + (int64_t)a.ne * (n - 1) + a.nv;
    // 64-thread blocks pack the registers a finished march block returns better than 128-thread ones
    // (config 2: 80.7 -> 80.2 us per apply; BT_BND_THREADS for profiling)
    static const int bt_ = std::getenv("BT_BND_THREADS") ? std::atoi(std::getenv("BT_BND_THREADS")) : 64;
    const unsigned blocks = (unsigned)((pts + bt_ - 1) / bt_);
    if (bc)
      k_boundary<true><<<blocks, bt_, 0, ss.s>>>(x, y, a);
    else
      k_boundary<false><<<blocks, bt_, 0, ss.s>>>(x, y, a);
    count_launch();
  }
  BT_CUDA(cudaEventRecord(ss.join, ss.s));
  BT_CUDA(cudaStreamWaitEvent(s, ss.join, 0));
  if (part && (parts & 8)) BT_CUDA(cudaStreamWaitEvent(s, ss.join2, 0));
  check_launch("k_stencil_fused");
}

// ---------------------------------------------------------------------------
// Hybrid Gauss-Seidel sweep (gauss_seidel_sweep, operators.hpp:327-387).
//
// Interior: in-place lexicographic Gauss-Seidel per cell. With f(d) =
// dx + 2 dy + 3 dz, every stencil direction that is lexicographically earlier
// (k, then j, then i) has f(d) < 0 and every later one f(d) > 0, so the
// points of one hyperplane i + 2j + 3k = f are independent and hyperplanes in
// increasing f (forward; decreasing for backward) reproduce the sequential
// order exactly: every update sees the same neighbour values and evaluates
// acc = rhs - sum_d row[d] x[p + d] (d = 1..14, unfused), x = acc / row[0]
// bit for bit. One cooperative launch per sweep, a grid barrier between
// hyperplanes. Then the Jacobi step on the non-interior points: scratch =
// apply_stencil(x) (partial rows + replica sums), x = rhs on Dirichlet
// points, else x + (rhs - scratch) / assembled diagonal.
// ---------------------------------------------------------------------------
constexpr int kGsT = 256;

__global__ void __launch_bounds__(kGsT) k_gs_interior(double* __restrict__ x, const double* __restrict__ rhs,
                                                       const StencilCell* __restrict__ cells, int n, int64_t cs,
                                                       int cell0, int ncells, int backward) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int w = n + 1;
  const int npairs = tri32(n - 3);  // rows (j, k) with j, k >= 1, j + k <= n - 2
  const int64_t items = (int64_t)ncells * npairs;
  const int fmin = 6, fmax = 3 * n - 6;  // i + 2j + 3k over the interior
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int q = 0; q <= fmax - fmin; ++q) {
    const int f = backward ? fmax - q : fmin + q;
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items; it += stride) {
      const int cl = (int)(it / npairs);
      int a, b;
      decode_tri(n - 3, (int)(it % npairs), a, b);
      const int j = a + 1, k = b + 1, i = f - 2 * j - 3 * k;
      if (i < 1 || i > n - 1 - j - k) continue;
      const int cell = cell0 + cl;
      const double* __restrict__ row = cells[cell].w[0];
      int off[15];
      row_offsets(w, j, k, off);
      const int64_t t = (int64_t)cell * cs + row_start(w, j, k) + i;
      double acc = rhs[t];
#pragma unroll
      for (int d = 1; d < 15; ++d) acc = __dsub_rn(acc, __dmul_rn(row[d], x[t + off[d]]));
      x[t] = __ddiv_rn(acc, row[0]);
    }
    grid.sync();
  }
}

// grid (row chunks of 64 rows, cells): warps over rows, lanes over i
__global__ void __launch_bounds__(256) k_gs_boundary(double* __restrict__ x, const double* __restrict__ rhs,
                                                     const double* __restrict__ scratch,
                                                     const double* __restrict__ diag,
                                                     const DevCellInfo* __restrict__ info, int n, int64_t cs,
                                                     int cell0) {
  const int cell = cell0 + blockIdx.y, w = n + 1;
  const uint16_t dir = info[cell].dir_by_z;
  const int64_t base = (int64_t)cell * cs;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rend = min(tri32(w), (int)(blockIdx.x + 1) * 64);
  for (int r = blockIdx.x * 64 + warp; r < rend; r += 8) {
    int j, k;
    decode_row(w, r, j, k);
    const int L = w - j - k;
    const int64_t t0 = base + row_start(w, j, k);
    const bool edge_row = j == 0 || k == 0;  // whole row on the lattice boundary
    for (int i = lane; i < L; i += 32) {
      if (!edge_row && i != 0 && i != L - 1) continue;  // interior: done by the sweep
      const int z = zero_set(n, i, j, k);
      const int64_t u = t0 + i;
      x[u] = (dir >> z & 1) ? rhs[u] : __dadd_rn(x[u], __ddiv_rn(__dsub_rn(rhs[u], scratch[u]), diag[u]));
    }
  }
}

void launch_gs_sweep(const bt_stencil& st, const double* rhs, double* x, double* scratch, bool backward,
                     cudaStream_t s) {
  const bt_grid& g = *st.grid;
  for (int c = 0; c < g.mesh.n_cells(); ++c)
    if (st.rows[c][0] == 0.0) raise(BT_INVALID_ARGUMENT, "gauss_seidel_sweep: zero center weight");
  const int n = 1 << st.level;
  const int64_t cs = n_tet(n + 1);
  const int nc = g.part_end - g.part_begin;
  if (nc && n >= 4) {
    static std::mutex mu;
    static int slots[64] = {0};
    int dev = 0;
    BT_CUDA(cudaGetDevice(&dev));
    int grid;
    {
      std::lock_guard<std::mutex> lock(mu);
      if (!slots[dev & 63]) {
        int per_sm = 0, sms = 0;
        BT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gs_interior, kGsT, 0));
        BT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        slots[dev & 63] = std::max(1, per_sm) * sms;
      }
      grid = slots[dev & 63];
    }
    const int64_t items = (int64_t)nc * tri32(n - 3);
    grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, (items + kGsT - 1) / kGsT));
    double* xs = shifted(x, g, BT_SPACE_P1, st.level);
    const double* rs = shifted(rhs, g, BT_SPACE_P1, st.level);
    const StencilCell* cells = st.d_cells.p;
    int cell0 = g.part_begin, bw = backward ? 1 : 0, nn = n;
    int64_t css = cs;
    void* args[] = {&xs, &rs, &cells, &nn, &css, &cell0, (void*)&nc, &bw};
    BT_CUDA(cudaLaunchCooperativeKernel((const void*)k_gs_interior, dim3(grid), dim3(kGsT), args, 0, s));
    count_launch();
    check_launch("k_gs_interior");
  }
  // non-interior points: Jacobi with the assembled diagonal on the synced residual
  if (stencil_fused(st)) {
    launch_stencil_fused(st, x, scratch, 0, s);
  } else {
    launch_stencil(st, x, scratch, s);
    sync(g, st.level, IF_SYNC, scratch, nullptr, s);
  }
  const double* diag = stencil_diag(st, s);
  if (nc) {
    const dim3 grid((unsigned)((tri32(n + 1) + 63) / 64), nc);
    k_gs_boundary<<<grid, 256, 0, s>>>(shifted(x, g, BT_SPACE_P1, st.level), shifted(rhs, g, BT_SPACE_P1, st.level),
                                       shifted(scratch, g, BT_SPACE_P1, st.level),
                                       shifted(diag, g, BT_SPACE_P1, st.level), g.d_info.p, n, cs, g.part_begin);
    count_launch();
    check_launch("k_gs_boundary");
  }
}

}  // namespace bt
