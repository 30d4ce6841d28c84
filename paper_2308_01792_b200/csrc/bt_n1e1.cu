// Nédélec N1E1 (lowest-order Whitney edge element) curl-curl + mass
// operator, alpha curl curl u + beta u, applied matrix-free over the seven
// micro-edge orientations (x, y, z, xy, xz, yz, xyz) of the reference's edge
// storage (micro_index.hpp:220-228). The reference has no N1E1 operator
// (SPEC.md:8); conventions are documented in oracle/bt_oracle_n1e1.c and
// DESIGN.md, and the oracle there is the checker.
//
// Layout: the edge space of one level is cells outer, then the 7 edge
// subgroups (widths 2^l, ..., 2^l - 1), then lattice slots (Code-1 order).
// Kernels walk the rows of each subgroup lattice; an interior edge uses the
// merged per-(cell, orientation) stencil of 19 or 13 coupled edges, a
// lattice-boundary edge sums the element rows of its present micro-tets.
// Replicated edges on macro faces/edges are summed with orientation signs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <random>
#include <vector>

#include <type_traits>

#include "bt_async.cuh"
#include "bt_internal.hpp"
#include "bt_n1e1_tables.cuh"

namespace bt {

namespace {

constexpr int kT = 256;
constexpr int kW = kT / 32;
constexpr int kRows = 256;  // rows per block (per warp: kRows / kW consecutive rows)

static const int hOffEdge[7][2][3] = BT_EDGE_OFFSETS;
static const int hOffCell[6][4][3] = BT_CELL_OFFSETS;
static const int hLoc[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

// coupled edges / incident micro-tets of orientation g (checked against the
// tables in build_static): x, z, xy, yz edges have 6 incident micro-tets and
// couple to 19 edges; y, xz, xyz edges 4 and 13
__host__ __device__ constexpr int n1e1_nnb(int g) { return g == 2 || g == 5 || g == 7 ? 13 : 19; }
__host__ __device__ constexpr int n1e1_ninc(int g) { return g == 2 || g == 5 || g == 7 ? 4 : 6; }

struct IncTet {  // a micro-tet containing an edge of subgroup g
  int s, le, sigma;
  int dq[3];     // tet anchor - edge anchor
  int nb[6];     // neighbour index of the tet's local edge j
};
struct Nb {      // coupled edge: subgroup and anchor offset
  int g, d[3];
};
struct N1e1Static {
  int ninc[8];
  IncTet inc[8][6];
  int nnb[8];
  Nb nb[8][19];
  int emap_g[6][6], emap_sigma[6][6];
  int dir_g[27], dir_sigma[27];  // lattice direction code -> (subgroup, sign)
  int nbmask[8][19];  // incident tets (bits q) containing coupled edge m
  int mask_off[8];    // first row of orientation g in a cell's masked-row table
  int mask_rows;      // rows per cell: sum over g of 2^ninc[g]
};
__constant__ N1e1Static cS;
static N1e1Static hS;
static bool hS_ready = false;

int dcode(int dx, int dy, int dz) { return (dx + 1) * 9 + (dy + 1) * 3 + (dz + 1); }

void build_static() {
  if (hS_ready) return;
  std::memset(&hS, 0, sizeof hS);
  for (int c = 0; c < 27; ++c) hS.dir_g[c] = -1;
  for (int g = 1; g <= 7; ++g) {
    int e[3];
    for (int a = 0; a < 3; ++a) e[a] = hOffEdge[g - 1][1][a] - hOffEdge[g - 1][0][a];
    hS.dir_g[dcode(e[0], e[1], e[2])] = g;
    hS.dir_sigma[dcode(e[0], e[1], e[2])] = 1;
    hS.dir_g[dcode(-e[0], -e[1], -e[2])] = g;
    hS.dir_sigma[dcode(-e[0], -e[1], -e[2])] = -1;
  }
  int emap_d[6][6][3];
  for (int s = 0; s < 6; ++s)
    for (int le = 0; le < 6; ++le) {
      const int* oa = hOffCell[s][hLoc[le][0]];
      const int* ob = hOffCell[s][hLoc[le][1]];
      const int c = dcode(ob[0] - oa[0], ob[1] - oa[1], ob[2] - oa[2]);
      const int g = hS.dir_g[c], sg = hS.dir_sigma[c];
      hS.emap_g[s][le] = g;
      hS.emap_sigma[s][le] = sg;
      const int* from = sg > 0 ? oa : ob;
      for (int a = 0; a < 3; ++a) emap_d[s][le][a] = from[a] - hOffEdge[g - 1][0][a];
    }
  for (int s = 0; s < 6; ++s)
    for (int le = 0; le < 6; ++le) {
      const int g = hS.emap_g[s][le];
      IncTet& it = hS.inc[g][hS.ninc[g]++];
      it.s = s;
      it.le = le;
      it.sigma = hS.emap_sigma[s][le];
      for (int a = 0; a < 3; ++a) it.dq[a] = -emap_d[s][le][a];
      for (int j = 0; j < 6; ++j) {
        Nb nb{hS.emap_g[s][j], {it.dq[0] + emap_d[s][j][0], it.dq[1] + emap_d[s][j][1], it.dq[2] + emap_d[s][j][2]}};
        int m = 0;
        for (; m < hS.nnb[g]; ++m)
          if (hS.nb[g][m].g == nb.g && hS.nb[g][m].d[0] == nb.d[0] && hS.nb[g][m].d[1] == nb.d[1] &&
              hS.nb[g][m].d[2] == nb.d[2])
            break;
        if (m == hS.nnb[g]) hS.nb[g][hS.nnb[g]++] = nb;
        it.nb[j] = m;
        hS.nbmask[g][m] |= 1 << (hS.ninc[g] - 1);
      }
    }
  for (int g = 1; g <= 7; ++g)
    if (hS.nnb[g] != n1e1_nnb(g) || hS.ninc[g] != n1e1_ninc(g))
      raise(BT_LOGIC_ERROR, "n1e1: coupling table does not match the per-orientation counts");
  int rows = 0;
  for (int g = 1; g <= 7; ++g) {
    hS.mask_off[g] = rows;
    rows += 1 << hS.ninc[g];
  }
  hS.mask_rows = rows;
  BT_CUDA(cudaMemcpyToSymbol(cS, &hS, sizeof hS));
  hS_ready = true;
}


// presence mask of the incident micro-tets of edge (i, j, k) of orientation g
// (the face kernel's per-row intervals)
unsigned host_mask(int g, int i, int j, int k, int n) {
  unsigned mask = 0;
  for (int q = 0; q < hS.ninc[g]; ++q) {
    const IncTet& it = hS.inc[g][q];
    const int ws = it.s == 0 ? n : (it.s == 1 ? n - 2 : n - 1);
    const int lo = std::max(0, -it.dq[0]);
    const int hi = (j + it.dq[1] < 0 || k + it.dq[2] < 0) ? -1 : ws - 1 - it.dq[0] - (j + it.dq[1]) - (k + it.dq[2]);
    if (i >= lo && i <= hi) mask |= 1u << q;
  }
  return mask;
}
// the mask cases of an edge: row case rc (bit 0: k == 0, bit 1: j == 0) x
// lane case wsel (0 full, 1 i == 0, 2 diagonal i + j + k == n - 1, 3 both)
unsigned case_mask(int g, int wsel, int n, int rc) {
  if (wsel == 0 && rc == 0) return (1u << hS.ninc[g]) - 1;  // all incident micro-tets (no such edge at n = 4)
  static const int rep[4][4][3] = {  // representative (i, j, k); negative: n + value
      {{1, 1, 1}, {0, 1, 1}, {-3, 1, 1}, {0, 1, -2}},    // j, k >= 1
      {{1, 1, 0}, {0, 1, 0}, {-2, 1, 0}, {0, -1, 0}},    // k == 0, j >= 1
      {{1, 0, 1}, {0, 0, 1}, {-2, 0, 1}, {0, 0, -1}},    // j == 0, k >= 1
      {{1, 0, 0}, {0, 0, 0}, {-1, 0, 0}, {0, 0, 0}}};    // j == k == 0 (no "both" edge for n > 1)
  const int* r = rep[rc][wsel];
  auto v = [&](int a) { return a < 0 ? n + a : a; };
  return host_mask(g, v(r[0]), v(r[1]), v(r[2]), n);
}
// k_n1e1_fast relies on: an edge's mask depends only on (j == 0, k == 0,
// i == 0, i + j + k == n - 1). Checked exhaustively at width nchk.
void check_mask_cases(int nchk) {
  for (int g = 1; g <= 7; ++g) {
    const int w = g == 7 ? nchk - 1 : nchk;
    for (int k = 0; k < w; ++k)
      for (int j = 0; j < w - k; ++j)
        for (int i = 0; i < w - k - j; ++i) {
          const int wsel = (i == 0 ? 1 : 0) | (i + j + k == nchk - 1 ? 2 : 0);
          if (wsel == 3) continue;  // rows of length 1: the face kernel's
          const int rc = (k == 0 ? 1 : 0) | (j == 0 ? 2 : 0);
          if (host_mask(g, i, j, k, nchk) != case_mask(g, wsel, nchk, rc))
            raise(BT_LOGIC_ERROR, "n1e1: mask cases do not hold");
        }
  }
}
// the generated coupling table (bt_n1e1_tables.cuh) must match build_static's
void check_generated_tables() {
  for (int g = 1; g <= 7; ++g)
    for (int m = 0; m < hS.nnb[g]; ++m) {
      const int s = n1_nb(g, m, 0);
      const Nb& nb = hS.nb[g][m];
      const int q = n1_nb(g, m, 3);
      if (n1_stream(s, 0) != nb.g || n1_stream(s, 1) != nb.d[2] || n1_nb(g, m, 1) != nb.d[1] ||
          n1_nb(g, m, 2) != nb.d[0] || nb.d[1] > n1_stream(s, 2) || nb.d[1] < n1_stream(s, 3) ||
          (nb.d[0] == 0) != (q < 0) ||
          (q >= 0 && (n1_shuf(q, 0) != s || n1_shuf(q, 1) != nb.d[1] || n1_shuf(q, 2) != nb.d[0])))
        raise(BT_LOGIC_ERROR, "n1e1: generated coupling table differs from build_static");
    }
}

// alpha K + beta M on the tet with corners X (same formulas as the oracle)
void local_n1e1(const double X[4][3], double alpha, double beta, double out[36]) {
  double a[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a[3 * r + c] = X[c + 1][r] - X[0][r];
  const double det = a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
                     a[2] * (a[3] * a[7] - a[4] * a[6]);
  if (det == 0.0 || !std::isfinite(det)) raise(BT_INVALID_ARGUMENT, "n1e1: degenerate element");
  const double vol = std::abs(det) / 6.0, d = det;
  const double inv[9] = {(a[4] * a[8] - a[5] * a[7]) / d, (a[2] * a[7] - a[1] * a[8]) / d,
                         (a[1] * a[5] - a[2] * a[4]) / d, (a[5] * a[6] - a[3] * a[8]) / d,
                         (a[0] * a[8] - a[2] * a[6]) / d, (a[2] * a[3] - a[0] * a[5]) / d,
                         (a[3] * a[7] - a[4] * a[6]) / d, (a[1] * a[6] - a[0] * a[7]) / d,
                         (a[0] * a[4] - a[1] * a[3]) / d};
  double gr[4][3], G[4][4], C[6][3];
  for (int c = 0; c < 3; ++c) {
    gr[1][c] = inv[c];
    gr[2][c] = inv[3 + c];
    gr[3][c] = inv[6 + c];
    gr[0][c] = -gr[1][c] - gr[2][c] - gr[3][c];
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) G[i][j] = gr[i][0] * gr[j][0] + gr[i][1] * gr[j][1] + gr[i][2] * gr[j][2];
  for (int e = 0; e < 6; ++e) {
    const double* u = gr[hLoc[e][0]];
    const double* v = gr[hLoc[e][1]];
    C[e][0] = u[1] * v[2] - u[2] * v[1];
    C[e][1] = u[2] * v[0] - u[0] * v[2];
    C[e][2] = u[0] * v[1] - u[1] * v[0];
  }
  auto mm = [&](int i, int j) { return vol * (i == j ? 2.0 : 1.0) / 20.0; };
  for (int e = 0; e < 6; ++e)
    for (int f = 0; f < 6; ++f) {
      const int ea = hLoc[e][0], eb = hLoc[e][1], fc = hLoc[f][0], fd = hLoc[f][1];
      const double K = 4.0 * vol * (C[e][0] * C[f][0] + C[e][1] * C[f][1] + C[e][2] * C[f][2]);
      const double M = mm(ea, fc) * G[eb][fd] - mm(ea, fd) * G[eb][fc] - mm(eb, fc) * G[ea][fd] + mm(eb, fd) * G[ea][fc];
      out[6 * e + f] = alpha * K + beta * M;
    }
}

}  // namespace

struct N1e1Cell {    // host-side setup of one cell
  double A[6][36];  // class element matrices
};

}  // namespace bt

struct bt_n1e1 {
  const bt_grid* grid = nullptr;
  int level = 0;
  double alpha = 1, beta = 1;
  // per cell, per orientation g, per presence mask of the incident micro-tets:
  // the merged 19-weight row of the present ones (cS.mask_off / mask_rows)
  bt::DevBuf<double> d_masked;
  // k_n1e1_fast: per cell and row case (j == 0, k == 0), the base merged rows
  // and the lane-case corrections; one cell's march list
  bt::DevBuf<double> d_cellw;  // per cell: 4 x (base rows 7 x kN1Wt, corrections kN1Corr), padded
  bt::DevBuf<int4> d_marches;  // one cell's marches {k | block << 16, j0, j1}, spatial order
  int nmarch = 0;
  bt::DevBuf<int> d_next;      // per cell: march queue counter
  int part_epoch = 0;          // the grid's partition at creation
};

namespace bt {
namespace {

// ---------------------------------------------------------------------------
// Per-edge path (k_n1e1_face): rows of length 1, whose single edge is both
// at i == 0 and on the diagonal face. Every edge applies one merged row — the
// row of its present incident micro-tets (presence mask from per-row
// intervals), from the block's shared table — with straight-line loads: a
// coupled edge that does not exist reads slot 0 with weight 0. Every longer
// row is k_n1e1_fast's.
// ---------------------------------------------------------------------------
// edges i = ifirst, ifirst + istep, ... of row (j, k): a warp per row
// (lane, 32), or a thread per row of length 1 (0, 1)
template <int G>
__device__ __forceinline__ void n1e1_row(const double* __restrict__ x, double* __restrict__ y, const double* sM,
                                         int cell, int j, int k, int n, int64_t cs, int ifirst, int istep) {
  constexpr int NNB = n1e1_nnb(G), NINC = n1e1_ninc(G);
  const int wg = G == 7 ? n - 1 : n;  // subgroup width: 2^l, xyz 2^l - 1
  const int tn = tet32(n);  // entry offsets: subgroups 1..6 have width n, xyz (7) n - 1
  auto eoff = [&](int q) { return (q - 1) * tn; };
  const double* __restrict__ xc = x + (int64_t)cell * cs;
  double* __restrict__ yc = y + (int64_t)cell * cs + eoff(G);
  int base[NNB];
#pragma unroll
  for (int m = 0; m < NNB; ++m) {
    const Nb nb = cS.nb[G][m];
    const int w2 = nb.g == 7 ? n - 1 : n;
    base[m] = eoff(nb.g) + row_start(w2, j + nb.d[1], k + nb.d[2]) + nb.d[0];
  }
  const int L = wg - j - k, t0 = row_start(wg, j, k);
  // incident micro-tet q exists (anchor in I_tet(w_s)) for i in [lo_q, hi_q]
  int lo[NINC], hi[NINC];
#pragma unroll
  for (int q = 0; q < NINC; ++q) {
    const IncTet& it = cS.inc[G][q];
    const int ws = it.s == 0 ? n : (it.s == 1 ? n - 2 : n - 1);
    lo[q] = max(0, -it.dq[0]);
    hi[q] = (j + it.dq[1] < 0 || k + it.dq[2] < 0) ? -1 : ws - 1 - it.dq[0] - (j + it.dq[1]) - (k + it.dq[2]);
  }
  for (int i = ifirst; i < L; i += istep) {
    unsigned mask = 0;
#pragma unroll
    for (int q = 0; q < NINC; ++q)
      if (i >= lo[q] && i <= hi[q]) mask |= 1u << q;
    const double* wrow = sM + NNB * mask;
    double v[NNB];
#pragma unroll
    for (int m = 0; m < NNB; ++m) v[m] = __ldg(xc + ((cS.nbmask[G][m] & mask) ? base[m] + i : 0));
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < NNB; ++m) acc = fma(wrow[m], v[m], acc);
    yc[t0 + i] = acc;
  }
}

// grid (row chunk x 7 orientations, cells): orientation G's rows of length 1
// (G != 7: k = q, j = n - 1 - k). The warp-per-row mode (long rows) is kept for
// any other row set but unused: k_n1e1_fast takes every longer row.
__host__ __device__ inline int n1e1_long_rows(int g, int n) { return 0; }
__host__ __device__ inline int n1e1_short_rows(int g, int n) { return g == 7 ? 0 : n; }
// block x = chunk * 7 + (g - 1): chunks [0, kLong) hold kW long rows each (a
// warp per row), the rest kT rows of length 1 each (a thread per row)
__global__ void __launch_bounds__(kT) k_n1e1_face(const double* __restrict__ x, double* __restrict__ y,
                                                  const double* __restrict__ masked, int n, int64_t cs,
                                                  int long_chunks) {
  __shared__ double sM[64 * 19];
  const int g = blockIdx.x % 7 + 1;
  const int chunk = blockIdx.x / 7;
  const int cell = blockIdx.y;
  const int nnb = n1e1_nnb(g);
  const int wg = g == 7 ? n - 1 : n;
  {
    const double* __restrict__ src = masked + (size_t)cell * cS.mask_rows * 19 + (size_t)cS.mask_off[g] * 19;
    const int nw = (1 << n1e1_ninc(g)) * 19;
    for (int e = threadIdx.x; e < nw; e += kT) {
      const int row = e / 19, m = e % 19;  // repack rows to nnb weights
      if (m < nnb) sM[row * nnb + m] = src[e];
    }
  }
  __syncthreads();
  int j, k, ifirst, istep;
  if (chunk < long_chunks) {  // rows j = 0 of every layer: (0, k = q)
    const int q = chunk * kW + (threadIdx.x >> 5);
    if (q >= n1e1_long_rows(g, n)) return;
    j = 0;
    k = q;
    ifirst = threadIdx.x & 31;
    istep = 32;
  } else {  // rows of length 1 (orientations 1..6): k = q, j = n - 1 - k
    const int q = (chunk - long_chunks) * kT + threadIdx.x;
    if (q >= n1e1_short_rows(g, n)) return;
    k = q;
    j = n - 1 - k;
    ifirst = 0;
    istep = 1;
  }
  switch (g) {
    case 1: n1e1_row<1>(x, y, sM, cell, j, k, n, cs, ifirst, istep); break;
    case 2: n1e1_row<2>(x, y, sM, cell, j, k, n, cs, ifirst, istep); break;
    case 3: n1e1_row<3>(x, y, sM, cell, j, k, n, cs, ifirst, istep); break;
    case 4: n1e1_row<4>(x, y, sM, cell, j, k, n, cs, ifirst, istep); break;
    case 5: n1e1_row<5>(x, y, sM, cell, j, k, n, cs, ifirst, istep); break;
    case 6: n1e1_row<6>(x, y, sM, cell, j, k, n, cs, ifirst, istep); break;
    default: n1e1_row<7>(x, y, sM, cell, j, k, n, cs, ifirst, istep); break;
  }
}

// ---------------------------------------------------------------------------
// k_n1e1_fast: every row of length >= 2 of all 7 orientations, staged
// like the P1 interior kernel. A warp owns 30 output columns i = 30b ..
// 30b + 29 of layer k of one cell (lane l: column 30b - 1 + l; lanes 1..30
// store) and marches rows j0 .. j1 - 1 of all 7 orientations at once. The 19
// (13) coupled edges of an edge of orientation G lie in 31 x rows (subgroup
// g, row j + dy, layer k + dz), dy, dz in {-1, 0, 1}, which form 16 streams
// (g, dz) (bt_n1e1_tables.cuh). Each step stages one new row per stream —
// row j + max dy — with one 8-byte cp.async per lane into a per-warp ring
// (zero-filled outside the lattice), so 16 staged rows serve 7 output rows.
// Each lane keeps its column of the last <= 3 rows of every stream in
// registers (slot = row mod 3, compile-time per unrolled phase); the 23
// distinct column i +- 1 values come from the neighbour lanes by shuffle.
//
// Block row y works on cell y; its blocks take the cell's marches from a
// queue. The cell's weights sit in shared memory and every lane reads the
// same address (broadcast). The presence mask of an edge's incident
// micro-tets depends on a row case (j == 0, k == 0: uniform over a step, each
// with its own merged rows) and a lane case (i == 0, diagonal face i + j + k ==
// n - 1), for which a correction (partial - base weight) over the 33 affected
// couplings is added (rows of length 1, which are both, are the face
// kernel's). Coupled edges outside the lattice read the zero fill.
// ---------------------------------------------------------------------------
constexpr int kN1FT = 128;
constexpr int kN1FW = kN1FT / 32;
constexpr int kN1Stages = 3;   // ring stages per warp (prefetch distance 2 steps)
constexpr int kN1Cols = 30;    // output columns per warp
constexpr int kN1March = 64;   // rows per march
constexpr int kN1Wt = 20;      // padded weight row (19 coupled edges)
constexpr int kN1Corr = kN1Corr0 + kN1Corr1;
constexpr int kN1RingD = kN1Stages * kN1Streams * 32;  // doubles per warp
// per cell and row case (bit 0: layer k == 0, bit 1: row j == 0): the base
// rows, then the corrections of lane cases 0 (i == 0) and 1 (diagonal)
constexpr int kN1CaseW = 7 * kN1Wt + kN1Corr;
constexpr int kN1CaseWP = (kN1CaseW + 1) / 2 * 2;      // padded to 16 bytes
constexpr int kN1CellWP = 4 * kN1CaseWP;
constexpr int kN1BlocksPerCell = 16;

template <int G, int PH>
__device__ __forceinline__ double n1_val(const double (&win)[kN1Streams][3], const double (&sh)[kN1Shuf], int m) {
  const int q = n1_nb(G, m, 3);
  return q >= 0 ? sh[q] : win[n1_nb(G, m, 0)][(PH + n1_nb(G, m, 1) + 3) % 3];
}

template <int G, int PH>
__device__ __forceinline__ double n1_edge(const double (&win)[kN1Streams][3], const double (&sh)[kN1Shuf],
                                          const double (&w)[kN1Wt]) {
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < n1e1_nnb(G); ++m) acc = fma(w[m], n1_val<G, PH>(win, sh, m), acc);
  return acc;
}

template <int C, int PH>
__device__ __forceinline__ void n1_correct(const double (&win)[kN1Streams][3], const double (&sh)[kN1Shuf],
                                           const double* __restrict__ cw, double (&e)[8]) {
  constexpr int NQ = C == 0 ? kN1Corr0 : kN1Corr1;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int G = n1_corr(C, q, 0), m = n1_corr(C, q, 1);
    double v;
    switch (G) {  // compile-time after unrolling
      case 1: v = n1_val<1, PH>(win, sh, m); break;
      case 2: v = n1_val<2, PH>(win, sh, m); break;
      case 3: v = n1_val<3, PH>(win, sh, m); break;
      case 4: v = n1_val<4, PH>(win, sh, m); break;
      case 5: v = n1_val<5, PH>(win, sh, m); break;
      case 6: v = n1_val<6, PH>(win, sh, m); break;
      default: v = n1_val<7, PH>(win, sh, m); break;
    }
    e[G] = fma(cw[(C == 0 ? 0 : kN1Corr0) + q], v, e[G]);
  }
}

__global__ void __launch_bounds__(kN1FT, 2) k_n1e1_fast(const double* __restrict__ x, double* __restrict__ y,
                                                        const int4* __restrict__ marches, int nmarch, int n,
                                                        int64_t cs, const double* __restrict__ cellw,
                                                        int* __restrict__ next_march) {
  extern __shared__ __align__(16) double n1_smem[];
  // warp index and march words broadcast by shuffles: provably warp-uniform,
  // so the march's shuffles need no divergence handling (WARPSYNC)
  const int lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int cl = blockIdx.y;  // this block's cell
  double* sw = n1_smem;       // the cell's weights (kN1CellWP)
  for (int q = threadIdx.x; q < kN1CellWP; q += kN1FT) sw[q] = __ldg(cellw + (size_t)cl * kN1CellWP + q);
  __syncthreads();
  const int GB = gridDim.x * kN1FW;
  const int t0 = blockIdx.x * kN1FW + warp;
  if (t0 >= nmarch) return;
  double* ring = n1_smem + kN1CellWP + warp * kN1RingD;
  const uint32_t my_s = smem_u32(ring) + 8u * lane;
  const int tn = tet32(n);
  const double* __restrict__ xc = x + (int64_t)cl * cs;
  double* __restrict__ yc = y + (int64_t)cl * cs;


  // ---- producer: lane copies its column of one row per stream per step ----
  int pt = t0, pnext_t = t0, pleft = 0, pj = 0, pk = 0, pcol = 0;
  int po[kN1Streams];
  int4 pnext = marches[t0];
  auto p_start = [&]() {
    const int4 tk = pnext;
    pk = tk.x & 0xffff;
    pcol = kN1Cols * (tk.x >> 16) - 1 + lane;
    pj = tk.y - 2;  // two phantom steps fill the register window
#pragma unroll
    for (int s = 0; s < kN1Streams; ++s) {
      const int g = n1_stream(s, 0), w = g == 7 ? n - 1 : n;
      po[s] = (g - 1) * tn + row_start(w, pj + n1_stream(s, 2), pk + n1_stream(s, 1)) + pcol;
    }
    pleft = tk.z - tk.y + 2;
    // the warp's next march: first come, first served, so the warps of a
    // cell stay on a compact range of its spatially ordered march list
    int nt = 0;
    if (lane == 0) nt = GB + atomicAdd(next_march + cl, 1);
    pnext_t = __shfl_sync(0xffffffffu, nt, 0);
    if (pnext_t < nmarch) pnext = marches[pnext_t];
  };
  p_start();
  int ps = 0;
  auto produce = [&]() {
    if (pleft > 0) {
      const uint32_t d = my_s + (uint32_t)(ps * kN1Streams * 32 * 8);
#pragma unroll
      for (int s = 0; s < kN1Streams; ++s) {
        const int g = n1_stream(s, 0), w = g == 7 ? n - 1 : n;
        const int jr = pj + n1_stream(s, 2);
        const int kr = pk + n1_stream(s, 1);
        const int len = w - jr - kr;  // staged row's length
        const bool ok = jr >= 0 && kr >= 0 && (unsigned)pcol < (unsigned)len;
        cp8z(d + s * 256, ok ? xc + po[s] : xc, ok);
        po[s] += len;
      }
      ++pj;
      ps = ps == kN1Stages - 1 ? 0 : ps + 1;
      if (--pleft == 0) {
        pt = pnext_t;
        if (pt < nmarch) p_start();
      }
    }
    cp_commit();
  };
#pragma unroll 1
  for (int q = 0; q < kN1Stages - 1; ++q) produce();

  // ---- consumer ----
  int cst = 0;
  auto consume = [&](double (&v)[kN1Streams]) {
    cp_wait<kN1Stages - 2>();
    __syncwarp();
    const double* st = ring + cst * kN1Streams * 32;
#pragma unroll
    for (int s = 0; s < kN1Streams; ++s) v[s] = st[s * 32 + lane];
    cst = cst == kN1Stages - 1 ? 0 : cst + 1;
    // the stage refilled next is the one read in the previous step, ordered
    // by the __syncwarp above
    produce();
  };

  int t = t0;
#pragma unroll 1
  while (t < nmarch) {
    int4 tk = marches[t];
    tk.x = __shfl_sync(0xffffffffu, tk.x, 0);
    tk.y = __shfl_sync(0xffffffffu, tk.y, 0);
    tk.z = __shfl_sync(0xffffffffu, tk.z, 0);
    const int k = tk.x & 0xffff, b = tk.x >> 16, j0 = tk.y, j1 = tk.z;
    const int i = kN1Cols * b - 1 + lane;
    const bool out = lane >= 1 && lane <= kN1Cols;
    int yo[7];  // this lane's output slot in orientation G's row j
#pragma unroll
    for (int G = 1; G <= 7; ++G) yo[G - 1] = (G - 1) * tn + row_start(G == 7 ? n - 1 : n, j0, k) + i;
    double win[kN1Streams][3];
    auto place = [&](auto phc, const double (&v)[kN1Streams]) {
      constexpr int PH = decltype(phc)::value;
#pragma unroll
      for (int s = 0; s < kN1Streams; ++s) win[s][(PH + n1_stream(s, 2) + 3) % 3] = v[s];
    };
    {
      double v[kN1Streams];
      consume(v);
      place(std::integral_constant<int, 0>{}, v);  // phantom step j0 - 2
      consume(v);
      place(std::integral_constant<int, 1>{}, v);  // phantom step j0 - 1
    }
    int j = j0;
    auto step = [&](auto phc) {
      constexpr int PH = decltype(phc)::value;
      double v[kN1Streams];
      consume(v);
      place(phc, v);
      const int L = n - j - k;  // row length of orientations 1..6 (xyz: L - 1)
      // this row's case: layer 0 and row 0 have their own base rows and corrections
      const double* wcase = sw + ((k == 0 ? 1 : 0) | (j == 0 ? 2 : 0)) * kN1CaseWP;
      const double (&W)[7][kN1Wt] = *reinterpret_cast<const double(*)[7][kN1Wt]>(wcase);
      double sh[kN1Shuf];       // column i +- 1 values, each distinct one shuffled once
#pragma unroll
      for (int q = 0; q < kN1Shuf; ++q) {
        const double u = win[n1_shuf(q, 0)][(PH + n1_shuf(q, 1) + 3) % 3];
        sh[q] = n1_shuf(q, 2) > 0 ? __shfl_down_sync(0xffffffffu, u, 1) : __shfl_up_sync(0xffffffffu, u, 1);
      }
      double e[8];
      e[1] = n1_edge<1, PH>(win, sh, W[0]);
      e[2] = n1_edge<2, PH>(win, sh, W[1]);
      e[3] = n1_edge<3, PH>(win, sh, W[2]);
      e[4] = n1_edge<4, PH>(win, sh, W[3]);
      e[5] = n1_edge<5, PH>(win, sh, W[4]);
      e[6] = n1_edge<6, PH>(win, sh, W[5]);
      e[7] = n1_edge<7, PH>(win, sh, W[6]);
      if (b == 0) {  // lane 1 holds i == 0
        double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        n1_correct<0, PH>(win, sh, wcase + 7 * kN1Wt, c);
        if (i == 0)
#pragma unroll
          for (int G = 1; G <= 7; ++G) e[G] += c[G];
      }
      const int dl = L - kN1Cols * b;  // the lane holding the diagonal edge i == L - 1
      if (dl >= 1 && dl <= kN1Cols) {
        double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        n1_correct<1, PH>(win, sh, wcase + 7 * kN1Wt, c);
        if (i == L - 1)
#pragma unroll
          for (int G = 1; G <= 7; ++G) e[G] += c[G];
      }
      if (out && i < L) {
#pragma unroll
        for (int G = 1; G <= 6; ++G) yc[yo[G - 1]] = e[G];
        if (i < L - 1) yc[yo[6]] = e[7];
      }
#pragma unroll
      for (int G = 0; G < 6; ++G) yo[G] += L;
      yo[6] += L - 1;
      ++j;
    };
    while (true) {
      step(std::integral_constant<int, 2>{});
      if (j >= j1) break;
      step(std::integral_constant<int, 0>{});
      if (j >= j1) break;
      step(std::integral_constant<int, 1>{});
      if (j >= j1) break;
    }
    // the producer, 2 steps ahead and every march >= 3 steps long, is already
    // on this warp's next march
    t = pt;
  }
  cp_wait<0>();
}

// ---------------------------------------------------------------------------
// signed edge-interface pass
// ---------------------------------------------------------------------------
struct EdgeIfaceArgs {
  const DevFace* faces;
  const int* flist;
  const DevPrimHdr* eh;
  const DevPrimMem* em;
  const int* elist;
  int ne;
  int n;
  int64_t cs;
};

// slot and sign of the micro-edge P0 -> P1 (cell lattice coordinates)
__device__ __forceinline__ int64_t edge_slot(int n, int64_t cs, int cell, int i0, int j0, int k0, int i1, int j1,
                                             int k1, int& sigma) {
  const int c = (i1 - i0 + 1) * 9 + (j1 - j0 + 1) * 3 + (k1 - k0 + 1);
  const int g = cS.dir_g[c];
  sigma = cS.dir_sigma[c];
  int ai = sigma > 0 ? i0 : i1, aj = sigma > 0 ? j0 : j1, ak = sigma > 0 ? k0 : k1;
  // anchor = first canonical endpoint - offs[g][0]
  const int o0 = g == 4 || g == 7 ? 1 : 0;  // y-offset of offs[g][0] for xy, xyz
  const int o2 = g == 5 || g == 6 ? 1 : 0;  // z-offset for xz, yz
  aj -= o0;
  ak -= o2;
  const int eoff = (g - 1) * tet32(n);  // subgroups 1..6 have width n; xyz (7) comes last
  const int wg = g == 7 ? n - 1 : n;
  return (int64_t)cell * cs + eoff + row_start(wg, aj, ak) + ai;
}

__device__ __forceinline__ void ijk3(const int8_t* lv, int w0, int w1, int w2, int& i, int& j, int& k) {
  i = (lv[0] == 1 ? w0 : 0) + (lv[1] == 1 ? w1 : 0) + (lv[2] == 1 ? w2 : 0);
  j = (lv[0] == 2 ? w0 : 0) + (lv[1] == 2 ? w1 : 0) + (lv[2] == 2 ? w2 : 0);
  k = (lv[0] == 3 ? w0 : 0) + (lv[1] == 3 ? w1 : 0) + (lv[2] == 3 ? w2 : 0);
}

// faces (at most 2 members): slots and signs computed once, then the same
// member-order operations as signed_group
template <int MODE, class S>
__device__ __forceinline__ void signed_group2(double* __restrict__ v, const double* __restrict__ src, int count,
                                              bool dir, S slot) {
  int sg[2] = {1, 1};
  int64_t t[2] = {0, 0};
#pragma unroll
  for (int m = 0; m < 2; ++m)
    if (m < count) t[m] = slot(m, sg[m]);
  if (MODE == IF_SYNC || (MODE == IF_SYNC_DIR && !dir)) {
    if (count < 2) return;
    const double a = v[t[0]], b = v[t[1]];
    double sum = 0;
    sum += sg[0] > 0 ? a : -a;
    sum += sg[1] > 0 ? b : -b;
    v[t[0]] = sg[0] > 0 ? sum : -sum;
    v[t[1]] = sg[1] > 0 ? sum : -sum;
  } else if (MODE == IF_SYNC_DIR || MODE == IF_IMPOSE) {
    if (!dir) return;
    for (int m = 0; m < count; ++m) v[t[m]] = src[t[m]];
  } else if (MODE == IF_ZERO_DIR) {
    if (!dir) return;
    for (int m = 0; m < count; ++m) v[t[m]] = 0.0;
  } else if (MODE == IF_BCAST) {
    if (count < 2) return;
    const double u = sg[0] > 0 ? v[t[0]] : -v[t[0]];
    v[t[1]] = sg[1] > 0 ? u : -u;
  }
}

template <int MODE, class S>
__device__ __forceinline__ void signed_group(double* __restrict__ v, const double* __restrict__ src, int count,
                                             bool dir, S slot) {
  int sg;
  if (MODE == IF_SYNC || (MODE == IF_SYNC_DIR && !dir)) {
    if (count < 2) return;
    double sum = 0;
    for (int m = 0; m < count; ++m) {
      const int64_t t = slot(m, sg);
      sum += sg > 0 ? v[t] : -v[t];
    }
    for (int m = 0; m < count; ++m) {
      const int64_t t = slot(m, sg);
      v[t] = sg > 0 ? sum : -sum;
    }
  } else if (MODE == IF_SYNC_DIR || MODE == IF_IMPOSE) {
    if (!dir) return;
    for (int m = 0; m < count; ++m) {
      const int64_t t = slot(m, sg);
      v[t] = src[t];
    }
  } else if (MODE == IF_ZERO_DIR) {
    if (!dir) return;
    for (int m = 0; m < count; ++m) v[slot(m, sg)] = 0.0;
  } else if (MODE == IF_BCAST) {
    if (count < 2) return;
    int64_t t = slot(0, sg);
    const double u = sg > 0 ? v[t] : -v[t];
    for (int m = 1; m < count; ++m) {
      t = slot(m, sg);
      v[t] = sg > 0 ? u : -u;
    }
  }
}

// face-interior micro-edges: tau in {0,1,2} x (a, b) with a + b <= n - 1
template <int MODE>
__global__ void __launch_bounds__(kT) k_edge_faces(double* __restrict__ v, const double* __restrict__ src,
                                                   EdgeIfaceArgs a) {
  const int n = a.n;
  const int per = tri32(n);
  const int q = blockIdx.x * kT + threadIdx.x;
  if (q >= 3 * per) return;
  const int tau = q / per;
  int aa, bb;
  decode_tri(n, q - tau * per, aa, bb);
  if ((tau == 0 && bb == 0) || (tau == 1 && aa == 0) || (tau == 2 && aa + bb + 1 == n)) return;  // on a macro edge
  int a0 = aa, b0 = bb, a1 = aa, b1 = bb;
  if (tau == 0) a1 = aa + 1;
  else if (tau == 1) b1 = bb + 1;
  else { a0 = aa + 1; b1 = bb + 1; }
  const DevFace f = a.faces[a.flist[blockIdx.y]];
  signed_group2<MODE>(v, src, f.ncell, f.dir != 0, [&](int m, int& sg) {
    int i0, j0, k0, i1, j1, k1;
    ijk3(f.lv[m], n - a0 - b0, a0, b0, i0, j0, k0);
    ijk3(f.lv[m], n - a1 - b1, a1, b1, i1, j1, k1);
    return edge_slot(n, a.cs, f.cell[m], i0, j0, k0, i1, j1, k1, sg);
  });
}

// micro-edges along macro edges: a = 0..n-1, (n - a, a) -> (n - a - 1, a + 1)
template <int MODE>
__global__ void __launch_bounds__(kT) k_edge_edges(double* __restrict__ v, const double* __restrict__ src,
                                                   EdgeIfaceArgs a) {
  const int n = a.n;
  const int aa = blockIdx.x * kT + threadIdx.x;
  if (aa >= n) return;
  const DevPrimHdr h = a.eh[a.elist[blockIdx.y]];
  const DevPrimMem* mem = a.em + h.first;
  signed_group<MODE>(v, src, h.count, h.dir != 0, [&](int m, int& sg) {
    const DevPrimMem pm = mem[m];
    const int8_t lv[3] = {pm.lv[0], pm.lv[1], -1};
    int i0, j0, k0, i1, j1, k1;
    ijk3(lv, n - aa, aa, 0, i0, j0, k0);
    ijk3(lv, n - aa - 1, aa + 1, 0, i1, j1, k1);
    return edge_slot(n, a.cs, pm.cell, i0, j0, k0, i1, j1, k1, sg);
  });
}

// the groups local to this handle's partition (g.loc; all groups when
// unpartitioned); local pointers
template <int MODE>
void edge_iface(const bt_grid& g, int level, double* v, const double* src, cudaStream_t s) {
  build_static();
  const int n = 1 << level;
  const IfaceLists& Lg = g.loc;
  v = shifted(v, g, BT_SPACE_EDGES, level);
  src = shifted(src, g, BT_SPACE_EDGES, level);
  EdgeIfaceArgs a{g.d_faces.p, nullptr, g.d_ehdr.p, g.d_emem.p, Lg.d_edge_act.p, (int)Lg.edge_act.size(), n,
                  level_slots(BT_SPACE_EDGES, level)};
  const int per = 3 * tri32(n);
  const bool sync_like = MODE == IF_SYNC || MODE == IF_BCAST || MODE == IF_SYNC_DIR;
  const bool dir_like = MODE == IF_SYNC_DIR || MODE == IF_IMPOSE || MODE == IF_ZERO_DIR;
  if (sync_like && !Lg.face_shared.empty()) {
    a.flist = Lg.d_face_shared.p;
    k_edge_faces<MODE><<<dim3((per + kT - 1) / kT, (unsigned)Lg.face_shared.size()), kT, 0, s>>>(v, src, a);
    count_launch();
  }
  if (dir_like && !Lg.face_bdir.empty()) {
    a.flist = Lg.d_face_bdir.p;
    k_edge_faces<MODE><<<dim3((per + kT - 1) / kT, (unsigned)Lg.face_bdir.size()), kT, 0, s>>>(v, src, a);
    count_launch();
  }
  if (a.ne) {
    k_edge_edges<MODE><<<dim3((n + kT - 1) / kT, (unsigned)a.ne), kT, 0, s>>>(v, src, a);
    count_launch();
  }
  check_launch("k_edge_iface");
}

// owned-DoF dot over the edge space: deterministic (cell, orientation, row block) partials
__global__ void __launch_bounds__(kT) k_edge_dot(const double* __restrict__ x, const double* __restrict__ y,
                                                 const DevCellInfo* __restrict__ info, int n, int64_t cs,
                                                 double* __restrict__ partials) {
  __shared__ double red[kW];
  const int g = blockIdx.z + 1, cell = blockIdx.y;
  const int wg = g == 7 ? n - 1 : n;
  int eoff = 0;
  for (int q = 1; q < g; ++q) eoff += tet32(q == 7 ? n - 1 : n);
  const uint16_t own = info[cell].owned_by_z;
  const double* xc = x + (int64_t)cell * cs + eoff;
  const double* yc = y + (int64_t)cell * cs + eoff;
  const int o[7][2][3] = BT_EDGE_OFFSETS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nrows = tri32(wg);
  const int rend = min(nrows, (int)(blockIdx.x + 1) * kRows);
  double acc = 0.0;
  for (int r = blockIdx.x * kRows + warp; r < rend; r += kW) {
    int j, k;
    decode_row(wg, r, j, k);
    const int L = wg - j - k, t0 = row_start(wg, j, k);
    for (int i = lane; i < L; i += 32) {
      const int z = zero_set(n, i + o[g - 1][0][0], j + o[g - 1][0][1], k + o[g - 1][0][2]) &
                    zero_set(n, i + o[g - 1][1][0], j + o[g - 1][1][1], k + o[g - 1][1][2]);
      if (own >> z & 1) acc = fma(__ldg(xc + t0 + i), __ldg(yc + t0 + i), acc);
    }
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int q = 0; q < kW; ++q) s += red[q];
    partials[((int64_t)blockIdx.z * gridDim.y + cell) * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(1024) k_edge_sum(const double* __restrict__ p, int64_t n, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < n; q += blockDim.x) acc += p[q];
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int q = 0; q < 32; ++q) s += red[q];
    *out = s;
  }
}

}  // namespace

void launch_edge_interface(const bt_grid& g, int level, IfaceMode mode, double* v, const double* src,
                           cudaStream_t s) {
  switch (mode) {
    case IF_SYNC: edge_iface<IF_SYNC>(g, level, v, src, s); break;
    case IF_SYNC_DIR: edge_iface<IF_SYNC_DIR>(g, level, v, src, s); break;
    case IF_BCAST: edge_iface<IF_BCAST>(g, level, v, src, s); break;
    case IF_IMPOSE: edge_iface<IF_IMPOSE>(g, level, v, src, s); break;
    case IF_ZERO_DIR: edge_iface<IF_ZERO_DIR>(g, level, v, src, s); break;
    default: raise(BT_INVALID_ARGUMENT, "edge interface: unsupported mode");
  }
}

// owned-DoF dot over the edge space: per-cell sums (orientation, then row
// block, in order), then the cells in order — the same association on any
// number of GPUs
double dot_edges(const bt_grid& g, int level, const double* x, const double* y, cudaStream_t s) {
  const int n = 1 << level, nc = g.mesh.n_cells(), nl = g.part_end - g.part_begin;
  const int bx = (tri32(n) + kRows - 1) / kRows;
  std::vector<double> cells(nc, 0.0);
  if (nl) {
    DevBuf<double> part((size_t)bx * nl * 7);
    k_edge_dot<<<dim3(bx, nl, 7), kT, 0, s>>>(x, y, g.d_info.p + g.part_begin, n,
                                              level_slots(BT_SPACE_EDGES, level), part.p);
    count_launch();
    check_launch("k_edge_dot");
    std::vector<double> h(part.n);
    BT_CUDA(cudaMemcpyAsync(h.data(), part.p, sizeof(double) * part.n, cudaMemcpyDeviceToHost, s));
    BT_CUDA(cudaStreamSynchronize(s));
    for (int c = 0; c < nl; ++c) {  // partials[(g, cell, block)]
      double t = 0.0;
      for (int gg = 0; gg < 7; ++gg)
        for (int b = 0; b < bx; ++b) t += h[((size_t)gg * nl + c) * bx + b];
      cells[g.part_begin + c] = t;
    }
  }
  if (g.part_nranks > 1) {
    if (g.dot_cells.n < (size_t)nc + 1) g.dot_cells.alloc((size_t)nc + 1);
    BT_CUDA(cudaMemcpyAsync(g.dot_cells.p, cells.data(), sizeof(double) * nc, cudaMemcpyHostToDevice, s));
    allreduce(g, g.dot_cells.p, nc, s);
    BT_CUDA(cudaMemcpyAsync(cells.data(), g.dot_cells.p, sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
    BT_CUDA(cudaStreamSynchronize(s));
  }
  double acc = 0.0;
  for (int c = 0; c < nc; ++c) acc += cells[c];
  return acc;
}

bool n1e1_fast_available(int level) { return (1 << level) >= 4; }

constexpr size_t kN1Smem = (kN1CellWP + kN1FW * kN1RingD) * sizeof(double);
// opt-in shared memory of k_n1e1_fast (once per device)
void n1e1_fast_setup(int device) {
  static std::mutex mu;
  static bool done[64] = {false};
  std::lock_guard<std::mutex> lock(mu);
  if (!done[device]) {
    BT_CUDA(cudaFuncSetAttribute(k_n1e1_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kN1Smem));
    done[device] = true;
  }
}

// mt19937_64 over owned edge slots in canonical (cell, orientation, t) order,
// then a signed broadcast so replicas carry the same oriented field. A
// partitioned grid draws its cells' part of the single-GPU stream (after
// discarding the draws of the cells before its block) and broadcasts through
// the exchange (collective).
void random_fill_edges(const bt_grid& g, int level, uint64_t seed, double* x, cudaStream_t s) {
  const int n = 1 << level;
  const int64_t cs = level_slots(BT_SPACE_EDGES, level);
  const int cb = g.part_begin, ce = g.part_end;
  std::vector<double> h((size_t)(cs * (ce - cb)), 0.0);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  auto zset = [&](int e, int i, int j, int k) {
    const int* a = hOffEdge[e - 1][0];
    const int* b = hOffEdge[e - 1][1];
    return zero_set(n, i + a[0], j + a[1], k + a[2]) & zero_set(n, i + b[0], j + b[1], k + b[2]);
  };
  if (cb > 0) {  // edges per zero set (the same for every cell), then the owned ones of cells < cb
    std::vector<int64_t> per_z(16, 0);
    for (int e = 1; e <= 7; ++e) {
      const int w = width_formula(e, level);
      for (int k = 0; k < w; ++k)
        for (int j = 0; j < w - k; ++j)
          for (int i = 0; i < w - k - j; ++i) ++per_z[zset(e, i, j, k)];
    }
    unsigned long long skip = 0;
    for (int c = 0; c < cb; ++c)
      for (int z = 0; z < 16; ++z)
        if (g.topo.info[c].owned_by_z >> z & 1) skip += (unsigned long long)per_z[z];
    rng.discard(skip);  // one engine call per value
  }
  for (int c = cb; c < ce; ++c) {
    const uint16_t own = g.topo.info[c].owned_by_z;
    int64_t t = cs * (c - cb);
    for (int e = 1; e <= 7; ++e) {
      const int w = width_formula(e, level);
      for (int k = 0; k < w; ++k)
        for (int j = 0; j < w - k; ++j)
          for (int i = 0; i < w - k - j; ++i, ++t)
            if (own >> zset(e, i, j, k) & 1) h[t] = dist(rng);
    }
  }
  BT_CUDA(cudaMemcpyAsync(x, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, s));
  sync_edges(g, level, IF_BCAST, x, nullptr, s);
  BT_CUDA(cudaStreamSynchronize(s));
}

// host twin of edge_slot: element index and sign of the micro-edge P0 -> P1
static int64_t edge_slot_host(int n, int64_t cs, int cell, int i0, int j0, int k0, int i1, int j1, int k1,
                              int& sigma) {
  const int c = (i1 - i0 + 1) * 9 + (j1 - j0 + 1) * 3 + (k1 - k0 + 1);
  const int g = hS.dir_g[c];
  sigma = hS.dir_sigma[c];
  int ai = sigma > 0 ? i0 : i1, aj = sigma > 0 ? j0 : j1, ak = sigma > 0 ? k0 : k1;
  aj -= (g == 4 || g == 7) ? 1 : 0;
  ak -= (g == 5 || g == 6) ? 1 : 0;
  int64_t eoff = 0;
  for (int q = 1; q < g; ++q) eoff += tet32(q == 7 ? n - 1 : n);
  return (int64_t)cell * cs + eoff + row_start(g == 7 ? n - 1 : n, aj, ak) + ai;
}

static void ijk3_host(const int8_t* lv, int w0, int w1, int w2, int& i, int& j, int& k) {
  i = (lv[0] == 1 ? w0 : 0) + (lv[1] == 1 ? w1 : 0) + (lv[2] == 1 ? w2 : 0);
  j = (lv[0] == 2 ? w0 : 0) + (lv[1] == 2 ? w1 : 0) + (lv[2] == 2 ? w2 : 0);
  k = (lv[0] == 3 ? w0 : 0) + (lv[1] == 3 ? w1 : 0) + (lv[2] == 3 ? w2 : 0);
}

// exchange plan of the rank-spanning signed edge groups: shared faces'
// interior micro-edges (k_edge_faces' enumeration), then macro edges'
// micro-edges (k_edge_edges'); members in ascending cell order
static void build_xplan_edges(const bt_grid& g, int level, XPlan& out) {
  build_static();
  const int nc = g.mesh.n_cells(), n = 1 << level;
  const int64_t cs = level_slots(BT_SPACE_EDGES, level);
  std::vector<int> owner(nc);
  for (int r = 0; r < g.part_nranks; ++r) {
    int b, e;
    partition_range(nc, r, g.part_nranks, b, e);
    for (int c = b; c < e; ++c) owner[c] = r;
  }
  const Topology& t = g.topo;
  out.reset();
  int64_t off = 0;
  std::vector<int> own;
  auto add = [&](int count, int dir, auto&& member) {  // member(m, cell&, slot&, sign&)
    own.resize(count);
    for (int m = 0; m < count; ++m) {
      int cell, sg;
      int64_t slot;
      member(m, cell, slot, sg);
      own[m] = owner[cell];
      if (owner[cell] == g.part_rank) {
        XEntry e{slot, (int32_t)(off + m), (int32_t)off, count, dir};
        e.sign = sg;
        out.entries.push_back(e);
      }
    }
    xplan_group_peers(out, g.part_rank, own.data(), count, off);
    off += count;
  };
  for (const DevFace& F : t.faces) {
    if (F.ncell != 2 || owner[F.cell[0]] == owner[F.cell[1]]) continue;
    for (int tau = 0; tau < 3; ++tau)
      for (int q = 0; q < tri32(n); ++q) {
        int aa, bb;
        decode_tri(n, q, aa, bb);
        if ((tau == 0 && bb == 0) || (tau == 1 && aa == 0) || (tau == 2 && aa + bb + 1 == n)) continue;
        int a0 = aa, b0 = bb, a1 = aa, b1 = bb;
        if (tau == 0) a1 = aa + 1;
        else if (tau == 1) b1 = bb + 1;
        else { a0 = aa + 1; b1 = bb + 1; }
        add(2, F.dir, [&](int m, int& cell, int64_t& slot, int& sg) {
          int i0, j0, k0, i1, j1, k1;
          ijk3_host(F.lv[m], n - a0 - b0, a0, b0, i0, j0, k0);
          ijk3_host(F.lv[m], n - a1 - b1, a1, b1, i1, j1, k1);
          cell = F.cell[m];
          slot = edge_slot_host(n, cs, cell, i0, j0, k0, i1, j1, k1, sg);
        });
      }
  }
  for (const DevPrimHdr& h : t.ehdr) {
    if (h.count < 2) continue;
    bool spans = false;
    for (int m = 1; m < h.count; ++m) spans = spans || owner[t.emem[h.first + m].cell] != owner[t.emem[h.first].cell];
    if (!spans) continue;
    for (int aa = 0; aa < n; ++aa)
      add(h.count, h.dir, [&](int m, int& cell, int64_t& slot, int& sg) {
        const DevPrimMem& pm = t.emem[h.first + m];
        const int8_t lv[3] = {pm.lv[0], pm.lv[1], -1};
        int i0, j0, k0, i1, j1, k1;
        ijk3_host(lv, n - aa, aa, 0, i0, j0, k0);
        ijk3_host(lv, n - aa - 1, aa + 1, 0, i1, j1, k1);
        cell = pm.cell;
        slot = edge_slot_host(n, cs, cell, i0, j0, k0, i1, j1, k1, sg);
      });
  }
  if (off > INT32_MAX) raise(BT_OUT_OF_RANGE, "exchange buffer exceeds 2^31 entries");
  out.buf_size = off;
  out.built = true;
}

const XPlan& xchg_plan_edges(const bt_grid& g, int level) {
  XPlan& p = g.xplan_edges.at(level);
  if (!p.built) {
    build_xplan_edges(g, level, p);
    p.d_entries.upload(p.entries);
  }
  return p;
}

void sync_edges(const bt_grid& g, int level, IfaceMode mode, double* v, const double* src, cudaStream_t s) {
  if (g.part_nranks > 1) {
    const XPlan& p = xchg_plan_edges(g, level);
    const int64_t shift = part_shift(g, BT_SPACE_EDGES, level);
    const bool needs_buf = mode == IF_SYNC || mode == IF_SYNC_DIR || mode == IF_BCAST;
    const double* buf = nullptr;
    if (needs_buf && p.buf_size) {
      if (g.xbuf.n < (size_t)p.buf_size) g.xbuf.alloc((size_t)p.buf_size);
      launch_xchg_pack_plan(p, shift, v, g.xbuf.p, s);
      exchange_buffer(g, p, g.xbuf.p, s);
      buf = g.xbuf.p;
    }
    launch_edge_interface(g, level, mode, v, src, s);
    launch_xchg_combine_plan(p, shift, mode, v, src, buf, s);
  } else {
    launch_edge_interface(g, level, mode, v, src, s);
  }
}

}  // namespace bt

using namespace bt;


extern "C" {

bt_status bt_n1e1_create(const bt_grid* g, int level, double alpha, double beta, bt_n1e1** out) {
  BT_TRY
  check_level(g, level);
  BT_CUDA(cudaSetDevice(g->device));
  build_static();
  auto op = std::make_unique<bt_n1e1>();
  op->grid = g;
  op->part_epoch = g->part_epoch;
  op->level = level;
  op->alpha = alpha;
  op->beta = beta;
  const int nc = g->mesh.n_cells();
  std::vector<N1e1Cell> cells(nc);
  std::vector<double> masked((size_t)nc * hS.mask_rows * 19, 0.0);
  const double h = 1.0 / (double)(1 << level);
  for (int c = 0; c < nc; ++c) {
    N1e1Cell& cc = cells[c];
    std::memset(&cc, 0, sizeof cc);
    const CellMap& mp = g->topo.maps[c];
    for (int s = 0; s < 6; ++s) {
      double X[4][3];
      for (int v = 0; v < 4; ++v) {
        const double r[3] = {h * hOffCell[s][v][0], h * hOffCell[s][v][1], h * hOffCell[s][v][2]};
        for (int d = 0; d < 3; ++d) X[v][d] = (mp.a[3 * d] * r[0] + mp.a[3 * d + 1] * r[1] + mp.a[3 * d + 2] * r[2]) + mp.b[d];
      }
      local_n1e1(X, alpha, beta, cc.A[s]);
    }
    double* mt = &masked[(size_t)c * hS.mask_rows * 19];
    for (int gg = 1; gg <= 7; ++gg)
      for (int mask = 0; mask < (1 << hS.ninc[gg]); ++mask) {
        double* row = mt + 19 * (size_t)(hS.mask_off[gg] + mask);
        for (int q = 0; q < hS.ninc[gg]; ++q) {
          if (!(mask >> q & 1)) continue;
          const IncTet& it = hS.inc[gg][q];
          for (int j = 0; j < 6; ++j) row[it.nb[j]] += it.sigma * hS.emap_sigma[it.s][j] * cc.A[it.s][6 * it.le + j];
        }
      }
  }
  op->d_masked.upload(masked);
  // k_n1e1_fast: every row of length >= 2 of every cell (n >= 4)
  if (n1e1_fast_available(level)) {  // (n >= 4)
    const int n = 1 << level;
    check_generated_tables();
    check_mask_cases(std::min(n, 64));
    std::vector<double> cw((size_t)nc * kN1CellWP, 0.0);
    for (int c = 0; c < nc; ++c) {
      auto mrow = [&](int gg, unsigned mask) {
        return &masked[((size_t)c * hS.mask_rows + hS.mask_off[gg] + mask) * 19];
      };
      for (int k0 = 0; k0 < 4; ++k0) {  // row case
        double* cc_w = &cw[(size_t)c * kN1CellWP + (size_t)k0 * kN1CaseWP];
        for (int gg = 1; gg <= 7; ++gg) {
          const double* base = mrow(gg, case_mask(gg, 0, n, k0));
          for (int m = 0; m < hS.nnb[gg]; ++m) cc_w[(gg - 1) * kN1Wt + m] = base[m];
          // corrections: every coupling outside the generated lists must keep its base weight
          for (int cc = 0; cc < 2; ++cc) {
            if (cc == 1 && gg == 7) continue;
            const double* part = mrow(gg, case_mask(gg, cc == 0 ? 1 : 2, n, k0));
            for (int m = 0; m < hS.nnb[gg]; ++m) {
              int q = -1;
              const int nq = cc == 0 ? kN1Corr0 : kN1Corr1;
              for (int e = 0; e < nq; ++e)
                if (n1_corr(cc, e, 0) == gg && n1_corr(cc, e, 1) == m) q = e;
              if (q < 0) {
                if (part[m] != base[m])
                  raise(BT_LOGIC_ERROR, "n1e1: correction table misses coupling " + std::to_string(m) +
                                            " of orientation " + std::to_string(gg) + ", case " + std::to_string(cc));
              } else {
                cc_w[7 * kN1Wt + (cc == 0 ? 0 : kN1Corr0) + q] = part[m] - base[m];
              }
            }
          }
        }
      }
    }
    // One cell's marches in spatial order — column block, row block, layer
    // k innermost — so the warps working on a cell at any time cover a
    // compact region whose x rows the neighbouring layers re-read from L2.
    // Every row of length >= 2 (orientations 1..6; xyz rows are one shorter
    // and all covered).
    std::vector<int4> marches;
    for (int b = 0; kN1Cols * b <= n - 2; ++b)
      for (int j0 = 0; j0 <= n - 1 - kN1Cols * b; j0 += kN1March)
        for (int k = 0; k <= n - 2; ++k) {
          const int jmax = b == 0 ? n - k - 2 : n - k - 1 - kN1Cols * b;  // last row with an output in block b
          if (j0 > jmax) continue;
          marches.push_back(make_int4(k | (b << 16), j0, std::min(j0 + kN1March, jmax + 1), 0));
        }
    op->d_cellw.upload(cw);
    op->d_marches.upload(marches);
    op->nmarch = (int)marches.size();
    op->d_next.alloc((size_t)std::max(1, g->part_end - g->part_begin));
  }
  *out = op.release();
  BT_CATCH
}

void bt_n1e1_destroy(bt_n1e1* op) { delete op; }

bt_status bt_apply_n1e1(const bt_n1e1* op, const double* x, double* y, int bc, void* stream) {
  BT_TRY
  if (!op) raise(BT_INVALID_ARGUMENT, "apply_n1e1: operator required");
  if (op->part_epoch != op->grid->part_epoch)
    raise(BT_LOGIC_ERROR, "apply_n1e1: the grid was repartitioned after the operator was built");
  if (x == y && bt_space_size(op->grid, BT_SPACE_EDGES, op->level) > 0)
    raise(BT_INVALID_ARGUMENT, "source and destination must be distinct");
  const bt_grid& g = *op->grid;
  const int n = 1 << op->level;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t cs = level_slots(BT_SPACE_EDGES, op->level);
  // this handle's cells: x, y hold them (block row y = local cell); the
  // per-cell tables are indexed from the first of them
  const int nc = g.part_end - g.part_begin, c0 = g.part_begin;
  if (!nc) {
    sync_edges(g, op->level, bc ? IF_SYNC_DIR : IF_SYNC, y, x, s);
    return BT_OK;
  }
  // face rows (j = 0 or k = 0) and rows of length 1 of every orientation, on
  // the side stream beside the staged kernel
  SideStream& ss = side_stream();
  BT_CUDA(cudaEventRecord(ss.fork, s));
  BT_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
  const int long_chunks = (n1e1_long_rows(1, n) + kW - 1) / kW;
  const int short_chunks = (n1e1_short_rows(1, n) + kT - 1) / kT;
  const dim3 fgrid(7 * (long_chunks + short_chunks), nc);
  k_n1e1_face<<<fgrid, kT, 0, ss.s>>>(x, y, op->d_masked.p + (size_t)c0 * hS.mask_rows * 19, n, cs, long_chunks);
  count_launch();
  // the other rows: staged marches over all 7 orientations, kN1BlocksPerCell
  // blocks per cell sharing the cell's march queue
  if (op->nmarch) {
    BT_CUDA(cudaMemsetAsync(op->d_next.p, 0, sizeof(int) * (size_t)nc, s));
    n1e1_fast_setup(g.device);
    const int per_cell = std::min(kN1BlocksPerCell, (op->nmarch + kN1FW - 1) / kN1FW);
    k_n1e1_fast<<<dim3(per_cell, nc), kN1FT, kN1Smem, s>>>(x, y, op->d_marches.p, op->nmarch, n, cs,
                                                          op->d_cellw.p + (size_t)c0 * kN1CellWP, op->d_next.p);
    count_launch();
  }
  BT_CUDA(cudaEventRecord(ss.join, ss.s));
  BT_CUDA(cudaStreamWaitEvent(s, ss.join, 0));
  check_launch("k_n1e1");
  sync_edges(g, op->level, bc ? IF_SYNC_DIR : IF_SYNC, y, x, s);
  BT_CATCH
}

bt_status bt_n1e1_sync(const bt_grid* g, int level, double* x, void* stream) {
  BT_TRY
  check_level(g, level);
  sync_edges(*g, level, IF_SYNC, x, nullptr, (cudaStream_t)stream);
  BT_CATCH
}

}  // extern "C"
