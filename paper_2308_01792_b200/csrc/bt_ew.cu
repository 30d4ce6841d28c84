// Elementwise P1 apply with an on-the-fly coefficient (apply_elementwise
// operators.hpp:115-164, local_matrix forms.hpp:75-120), and the assembled
// diagonal (extract_diagonal operators.hpp:277-316).
//
// y_v = sum over the micro-cells T of v (class s, v = vertex `slot` of T):
// kbar_T * (G_s row slot) . x_T, with G_s the cell's class matrix
// (class_matrices operators.hpp:54-69; diffusion for div_k_grad, since the
// affine map makes grad phi constant per class) and kbar_T = 1/4 sum_q k(x_q)
// the reference's 4-point rule (forms.hpp:107-116). kbar depends on the
// micro-cell only, so each one is evaluated ONCE, into shared memory, and the
// vertices then pull it (the sum over (s, slot) in the fixed order of the
// reference's per-vertex contributions; no atomics, no cache in HBM).
//
// Work unit: a tile of one macro-cell — rows j0 .. j0+7, columns i0 .. i0+63
// — marched bottom-up over the layers k. Step k first evaluates kbar for every
// micro-cell anchored in layer k at rows j0-1 .. j0+7 and columns i0-1 ..
// i0+63 (all 6 classes; a vertex's micro-cells are anchored at v - o with o
// in {0,1}^3) into a two-layer ring, then computes the tile's vertices of
// layer k (warp = row, lanes = columns i0 + lane and i0 + lane + 32).
//
// kbar of the sin-product coefficient k = c0 + c1 sin(f x) sin(f y) sin(f z):
// the phase of quadrature point q of class s at anchor p is beta_d . p +
// gamma_{s,q,d} (affine map), so with S_d, C_d = sin, cos(beta_d . p) and the
// 8 monomials M_m = prod_d (bit d of m ? C_d : S_d),
//   kbar = c0 + sum_m coefh[s][m] M_m,
//   coefh[s][m] = c1/4 sum_q prod_d (bit d ? sin gamma_{s,q,d} : cos gamma_{s,q,d})
// (host tables): 3 sincos per anchor (by angle addition of a column table and
// a row table), 12 products and 8 FMAs per micro-cell instead of 12 sin.
// Affine k: kbar = k(centroid) = lin0[s] + lin . p exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "bt_internal.hpp"

namespace bt {

namespace {
constexpr int kER = 8;          // rows per tile
constexpr int kEC = 64;         // columns per tile (two per lane)
constexpr int kEA = kEC + 1;    // anchor columns i0-1 .. i0+63
constexpr int kERA = kER + 1;   // anchor rows j0-1 .. j0+kER-1
constexpr int kET = 256;        // threads

// present micro-cells (bit 4 s + slot) and needed stencil directions per zero
// set (as bt_kernels.cu); stencil direction of (o_j - o_slot) for class s
__constant__ uint32_t kEwPresent[16] = {0xffffff, 0xe8cc8e, 0x962b4d, 0x80080c, 0x4d962b, 0x48840a,
                                        0x40209,  0x8,      0x337117, 0x204006, 0x122105, 0x4,
                                        0x11003,  0x2,      0x1,      0x0};
__constant__ uint32_t kEwDirMask[16] = {0x7fff, 0x7f71, 0x26ff, 0x2671, 0x5d6f, 0x5d61, 0x46f, 0x461,
                                        0x3b9f, 0x3b11, 0x229f, 0x2211, 0x190f, 0x1901, 0xf,   0x0};

// a 16-byte shared load the compiler may not hoist out of the layer loop
__device__ __forceinline__ double2 lds2_v(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}
// a 16-byte read-only load the compiler may not hoist out of a loop: the
// per-cell class rows and kbar coefficients are re-read (L1 broadcast) each
// layer instead of pinning 144 registers
__device__ __forceinline__ double2 ldg2_nohoist(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__host__ __device__ inline int ew_class_width(int s, int n) { return s == 0 ? n : (s == 1 ? n - 2 : n - 1); }

struct EwShared {
  double kb[2][6][kERA][kEA];  // kbar ring: [layer & 1][class][anchor row][anchor column]
  double colT[3][2][kEA];      // sin, cos of beta_d[0] * p_i
  double rowT[2][3][2][kERA];  // [layer & 1]: sin, cos of beta_d[1] * p_j + beta_d[2] * p_k
  EwCell cell;
};

template <int CK, bool DIAG>
__global__ void __launch_bounds__(kET) k_ew(const double* __restrict__ x, double* __restrict__ y,
                                            const EwCell* __restrict__ cells, const int4* __restrict__ units, double c0,
                                            int n, int64_t cs) {
  extern __shared__ __align__(16) double ew_smem[];
  EwShared& S = *reinterpret_cast<EwShared*>(ew_smem);
  const int4 U = units[blockIdx.x];
  const int cell = U.x, j0 = U.y, i0 = U.z, kmax = U.w;
  const int w = n + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    const double* src = reinterpret_cast<const double*>(cells + cell);
    double* dst = reinterpret_cast<double*>(&S.cell);
    for (int q = tid; q < (int)(sizeof(EwCell) / 8); q += kET) dst[q] = src[q];
  }
  __syncthreads();
  const EwCell& E = S.cell;
  // row table of layer k (sincos of the row phase per anchor row), into buffer b
  auto row_table = [&](int k, int b) {
    if (CK == 1 && tid < 3 * kERA) {
      const int d = tid / kERA, r = tid % kERA;
      double sv, cv;
      sincos(E.beta[d][1] * (j0 - 1 + r) + E.beta[d][2] * k, &sv, &cv);
      S.rowT[b][d][0][r] = sv;
      S.rowT[b][d][1][r] = cv;
    }
  };
  if (CK == 1) {
    for (int q = tid; q < 3 * kEA; q += kET) {
      const int d = q / kEA, c = q % kEA;
      double sv, cv;
      sincos(E.beta[d][0] * (i0 - 1 + c), &sv, &cv);
      S.colT[d][0][c] = sv;
      S.colT[d][1][c] = cv;
    }
    row_table(0, 0);
  }
  __syncthreads();
  constexpr int kOff[6][4][3] = BT_CELL_OFFSETS;
  constexpr int kTetDir[6][4][4] = {{{0, 1, 2, 3}, {8, 0, 11, 12}, {9, 4, 0, 13}, {10, 5, 6, 0}},
                                    {{0, 13, 12, 3}, {6, 0, 11, 2}, {5, 4, 0, 1}, {10, 9, 8, 0}},
                                    {{0, 13, 7, 3}, {6, 0, 1, 2}, {14, 8, 0, 11}, {10, 9, 4, 0}},
                                    {{0, 11, 2, 3}, {4, 0, 1, 7}, {9, 8, 0, 13}, {10, 14, 6, 0}},
                                    {{0, 11, 12, 3}, {4, 0, 13, 7}, {5, 6, 0, 1}, {10, 14, 8, 0}},
                                    {{0, 1, 7, 3}, {8, 0, 13, 12}, {14, 6, 0, 11}, {10, 5, 4, 0}}};
  const double* __restrict__ xc = x + (int64_t)cell * cs;
  double* __restrict__ yc = y + (int64_t)cell * cs;

  for (int k = 0; k <= kmax; ++k) {
    const int b = k & 1;
    // ---- kbar of the micro-cells anchored in layer k (rows j0-1 .. j0+7,
    // columns i0-1 .. i0+63 with pi + pj + k <= n - 1), enumerated densely ----
    {
      int acount[kERA + 1];
      acount[0] = 0;
      const int ca = max(i0 - 1, 0);
#pragma unroll
      for (int r = 0; r < kERA; ++r) {
        const int pj = j0 - 1 + r;
        const int hi = min(i0 + kEC, n - k - pj);  // exclusive column bound
        acount[r + 1] = acount[r] + (pj >= 0 && hi > ca ? hi - ca : 0);
      }
      for (int q = tid; q < acount[kERA]; q += kET) {
        int r = 0, base = 0;  // (no dynamic indexing: acount stays in registers)
#pragma unroll
        for (int t = 1; t < kERA; ++t)
          if (q >= acount[t]) {
            r = t;
            base = acount[t];
          }
        const int pi = ca + q - base, pj = j0 - 1 + r;
        const int c = pi - (i0 - 1);
        if (CK == 0) {
#pragma unroll
          for (int s = 0; s < 6; ++s) S.kb[b][s][r][c] = c0;
        } else if (CK == 2) {
          const double lp = E.lin[0] * pi + E.lin[1] * pj + E.lin[2] * k;
#pragma unroll
          for (int s = 0; s < 6; ++s) S.kb[b][s][r][c] = E.lin0[s] + lp;
        } else {
          double Sd[3], Cd[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {  // sin, cos of (column phase + row phase)
            const double sa = S.colT[d][0][c], ca_ = S.colT[d][1][c];
            const double sb = S.rowT[b][d][0][r], cb = S.rowT[b][d][1][r];
            Sd[d] = fma(sa, cb, ca_ * sb);
            Cd[d] = fma(ca_, cb, -(sa * sb));
          }
          const double m2[4] = {Sd[0] * Sd[1], Cd[0] * Sd[1], Sd[0] * Cd[1], Cd[0] * Cd[1]};
          double M[8];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            M[m] = m2[m] * Sd[2];
            M[m + 4] = m2[m] * Cd[2];
          }
#pragma unroll
          for (int s = 0; s < 6; ++s) {
            double kb = c0;
#pragma unroll
            for (int m = 0; m < 8; ++m) kb = fma(E.coefh[s][m], M[m], kb);
            S.kb[b][s][r][c] = kb;
          }
        }
      }
    }
    if (CK == 1 && k < kmax) row_table(k + 1, b ^ 1);
    __syncthreads();
    // ---- vertices of layer k (rows j0 .. j0+7, columns i0 .. i0+63 inside
    // the layer), enumerated densely; a thread takes two at a time so each
    // class row G_s[slot] is loaded once for both.
    // Branch-free over the 24 (class, slot) pairs: an absent micro-cell gets
    // kbar 0 (selected, so stale ring values never enter) and absent
    // directions read 0, which adds +0.0 to the sum: the present terms are
    // summed in the reference's order, bit for bit as a skip would.
    int vcount[kER + 1];
    vcount[0] = 0;
#pragma unroll
    for (int r = 0; r < kER; ++r) {
      const int hi = min(i0 + kEC, w - k - (j0 + r));  // row length L = w - k - j
      vcount[r + 1] = vcount[r] + (hi > i0 ? hi - i0 : 0);
    }
    for (int q0 = tid; q0 < vcount[kER]; q0 += 2 * kET) {
      uint32_t present[2];
      double xv[2][15];
      int tt[2], rr[2], cc[2];
      bool live[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = q0 + h * kET;
        live[h] = q < vcount[kER];
        int r = 0, base = 0;
#pragma unroll
        for (int t = 1; t < kER; ++t)
          if (q >= vcount[t]) {
            r = t;
            base = vcount[t];
          }
        const int j = j0 + r, i = i0 + (live[h] ? q - base : 0);
        rr[h] = r;
        cc[h] = i - i0;
        const int z = live[h] ? zero_set(n, i, j, k) : 15;
        present[h] = kEwPresent[z];
        tt[h] = row_start(w, j, k) + i;
        if (!DIAG) {
          int off[15];
          row_offsets(w, j, k, off);
          const uint32_t dm = kEwDirMask[z];
#pragma unroll
          for (int d = 0; d < 15; ++d) xv[h][d] = (dm >> d & 1) ? __ldg(xc + tt[h] + off[d]) : 0.0;
        }
      }
      double acc[2] = {0.0, 0.0};
#pragma unroll
      for (int s = 0; s < 6; ++s) {
#pragma unroll
        for (int slot = 0; slot < 4; ++slot) {
          double g[4];
          if (DIAG) {
            g[0] = E.G[s][5 * slot];
          } else {
            const double2 g01 = *reinterpret_cast<const double2*>(&E.G[s][4 * slot]);
            const double2 g23 = *reinterpret_cast<const double2*>(&E.G[s][4 * slot + 2]);
            g[0] = g01.x;
            g[1] = g01.y;
            g[2] = g23.x;
            g[3] = g23.y;
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            // anchor v - o: ring layer k - o_k, row j - o_j, column i - o_i
            const double kr = S.kb[(k - kOff[s][slot][2]) & 1][s][rr[h] + 1 - kOff[s][slot][1]]
                                  [cc[h] + 1 - kOff[s][slot][0]];
            const double kb = (present[h] >> (4 * s + slot) & 1) ? kr : 0.0;
            if (DIAG) {
              acc[h] = fma(kb, g[0], acc[h]);
            } else {
              double row = 0.0;
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) row = fma(g[jj], xv[h][kTetDir[s][slot][jj]], row);
              acc[h] = fma(kb, row, acc[h]);
            }
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (live[h]) yc[tt[h]] = acc[h];
    }
    __syncthreads();  // the ring slot of layer k - 1 is rewritten next step
  }
}

// ---------------------------------------------------------------------------
// Warp-autonomous variant (k_ew_row, the default): a warp owns one row j of
// one macro-cell, lanes = columns 31q - 1 + lane (lane 0 only supplies the
// i - 1 anchors of lane 1), and marches the layers k. Per step each lane
// evaluates kbar of the 6 classes at its two anchors (c, j - 1, k) and
// (c, j, k) — the micro-cells anchored in layer k that its vertex column
// touches — keeps the previous layer's, and takes the column c - 1 ones from
// lane - 1 by shuffle. No barriers and no shared memory: every anchor row is
// evaluated by the two warps of the rows it touches (each bitwise alike: same
// column table, same row/layer recurrence from k = 0), which costs less than
// the synchronisation of a shared ring. The sin/cos of the row/layer phase
// beta_d1 (j - o_j) + beta_d2 k advance by rotation, the column phase
// beta_d0 c is one sincos per lane per row.
// ---------------------------------------------------------------------------
// The march of one warp (row j of one cell, lanes = columns c): GA(i) / CA(i)
// return 2 consecutive class-row / kbar-coefficient values of the cell
// (shared-memory copies, or kernel parameters that reach the FMAs as uniform
// registers).
template <int CK, bool DIAG, class GAcc, class CAcc>
__device__ __forceinline__ void ew_row_march(const double* __restrict__ x, double* __restrict__ y,
                                             const EwCell* __restrict__ E, int cell, int j, int c, int kmax,
                                             double c0, int n, int64_t cs, const double* __restrict__ phase,
                                             int cell0, double (*kb)[12][32], int lane, GAcc GA, CAcc CA) {
  const int w = n + 1;
  constexpr int kOff[6][4][3] = BT_CELL_OFFSETS;
  constexpr int kTetDir[6][4][4] = {{{0, 1, 2, 3}, {8, 0, 11, 12}, {9, 4, 0, 13}, {10, 5, 6, 0}},
                                    {{0, 13, 12, 3}, {6, 0, 11, 2}, {5, 4, 0, 1}, {10, 9, 8, 0}},
                                    {{0, 13, 7, 3}, {6, 0, 1, 2}, {14, 8, 0, 11}, {10, 9, 4, 0}},
                                    {{0, 11, 2, 3}, {4, 0, 1, 7}, {9, 8, 0, 13}, {10, 14, 6, 0}},
                                    {{0, 11, 12, 3}, {4, 0, 13, 7}, {5, 6, 0, 1}, {10, 14, 8, 0}},
                                    {{0, 1, 7, 3}, {8, 0, 13, 12}, {14, 6, 0, 11}, {10, 5, 4, 0}}};
  const double* __restrict__ xc = x + (int64_t)cell * cs;
  double* __restrict__ yc = y + (int64_t)cell * cs;
  // column phase (per lane), one-layer rotation, row/layer phases of anchor
  // rows j, j - 1: from the per-cell phase tables (ew_phase_tables)
  double sa[3], ca[3], sr[3], cr[3], sb[2][3], cb[2][3];
  if (CK == 1) {
    const int np = n + 2;  // table entries for -1 .. n
    const double* __restrict__ P = phase + (int64_t)(cell - cell0) * (12 * np + 6);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      sa[d] = __ldg(P + (0 * 3 + d) * np + c + 1);
      ca[d] = __ldg(P + (1 * 3 + d) * np + c + 1);
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        sb[o][d] = __ldg(P + (2 * 3 + d) * np + j - o + 1);
        cb[o][d] = __ldg(P + (3 * 3 + d) * np + j - o + 1);
      }
      sr[d] = __ldg(P + 12 * np + d);
      cr[d] = __ldg(P + 12 * np + 3 + d);
    }
  }
  const int cl = lane > 0 ? lane - 1 : 0;  // lane of column c - 1 (lane 0's vertex is never live)
  int t0 = row_start(w, j, 0);
#pragma unroll 1
  for (int k = 0; k <= kmax; ++k) {
    const int b = k & 1;
    // ---- kbar of the 6 classes at anchors (c, j - o, k) ----
    if (CK == 0) {
#pragma unroll
      for (int q = 0; q < 12; ++q) kb[b][q][lane] = c0;
    } else if (CK == 2) {
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        const double lp = __ldg(&E->lin[0]) * c + __ldg(&E->lin[1]) * (j - o) + __ldg(&E->lin[2]) * k;
#pragma unroll
        for (int s = 0; s < 6; ++s) kb[b][o * 6 + s][lane] = __ldg(&E->lin0[s]) + lp;
      }
    } else {
      double M[2][8];
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        double S[3], C[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          S[d] = fma(sa[d], cb[o][d], ca[d] * sb[o][d]);
          C[d] = fma(ca[d], cb[o][d], -(sa[d] * sb[o][d]));
        }
        const double m2[4] = {S[0] * S[1], C[0] * S[1], S[0] * C[1], C[0] * C[1]};
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          M[o][m] = m2[m] * S[2];
          M[o][m + 4] = m2[m] * C[2];
        }
      }
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        double k0v = c0, k1v = c0;
#pragma unroll
        for (int m = 0; m < 8; m += 2) {
          const double2 cv = CA(8 * s + m);
          const double cx = cv.x, cy = cv.y;
          k0v = fma(cx, M[0][m], k0v);
          k0v = fma(cy, M[0][m + 1], k0v);
          k1v = fma(cx, M[1][m], k1v);
          k1v = fma(cy, M[1][m + 1], k1v);
        }
        kb[b][s][lane] = k0v;
        kb[b][6 + s][lane] = k1v;
      }
    }
    if (CK == 1) {
#pragma unroll
      for (int o = 0; o < 2; ++o)
#pragma unroll
        for (int d = 0; d < 3; ++d) {  // rotate the row/layer phase by one layer
          const double sn = fma(sb[o][d], cr[d], cb[o][d] * sr[d]);
          cb[o][d] = fma(cb[o][d], cr[d], -(sb[o][d] * sr[d]));
          sb[o][d] = sn;
        }
    }
    __syncwarp();
    // ---- the vertex (c, j, k) ----
    const bool live = lane > 0 && c >= 0 && c + j + k <= n;
    const int z = live ? zero_set(n, c, j, k) : 15;
    const uint32_t present = kEwPresent[z];
    double xv[15];
    if (!DIAG) {
      int off[15];
      row_offsets(w, j, k, off);
      const uint32_t dm = kEwDirMask[z];
#pragma unroll
      for (int d = 0; d < 15; ++d) xv[d] = (dm >> d & 1) ? __ldg(xc + t0 + c + off[d]) : 0.0;
    }
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
#pragma unroll
      for (int slot = 0; slot < 4; ++slot) {
        const int oi = kOff[s][slot][0], oj = kOff[s][slot][1], ok = kOff[s][slot][2];
        const double kr = kb[(k - ok) & 1][oj * 6 + s][oi ? cl : lane];
        const double kv = (present >> (4 * s + slot) & 1) ? kr : 0.0;
        if (DIAG) {
          const double2 gd = GA(16 * s + 4 * slot + (slot & ~1));  // holds G_s[slot][slot]
          acc = fma(kv, (slot & 1) ? gd.y : gd.x, acc);
        } else {
          const double2 g01 = GA(16 * s + 4 * slot), g23 = GA(16 * s + 4 * slot + 2);
          double row = g01.x * xv[kTetDir[s][slot][0]];
          row = fma(g01.y, xv[kTetDir[s][slot][1]], row);
          row = fma(g23.x, xv[kTetDir[s][slot][2]], row);
          row = fma(g23.y, xv[kTetDir[s][slot][3]], row);
          acc = fma(kv, row, acc);
        }
      }
    }
    if (live) yc[t0 + c] = acc;
    t0 += tri32(w - k) - j;  // row j of layer k + 1
    __syncwarp();            // every lane has read the ring slot rewritten next step
  }
}

template <int CK, bool DIAG>
__global__ void __launch_bounds__(128) k_ew_row(const double* __restrict__ x, double* __restrict__ y,
                                                const EwCell* __restrict__ cells, const int4* __restrict__ tasks,
                                                int ntasks, double c0, int n, int64_t cs,
                                                const double* __restrict__ phase, int cell0) {
  // per warp: kbar of the lanes' anchors, [layer parity][o * 6 + class][lane]
  // (o = 0: anchor row j, o = 1: row j - 1); lane - 1's entries are the
  // column c - 1 anchors, so no shuffles and nothing held in registers
  __shared__ double kbs[4][2][12][32];
  // the warp's cell: class rows G_s and kbar coefficients, read with
  // non-hoisted loads each layer (held in registers they would take 144)
  __shared__ __align__(16) double egs[4][96 + 48];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int task = blockIdx.x * 4 + wib;
  if (task >= ntasks) return;
  const int4 T = tasks[task];
  const int cell = T.x;
  const EwCell* __restrict__ E = cells + cell;
  for (int q = lane; q < 96; q += 32) egs[wib][q] = __ldg(&E->G[0][0] + q);
  for (int q = lane; q < 48; q += 32) egs[wib][96 + q] = __ldg(&E->coefh[0][0] + q);
  __syncwarp();
  const double* EG = egs[wib];
  const double* EC = egs[wib] + 96;
  ew_row_march<CK, DIAG>(x, y, E, cell, T.y, 31 * T.z - 1 + lane, T.w, c0, n, cs, phase, cell0, kbs[wib], lane,
                         [&](int i) { return lds2_v(EG + i); }, [&](int i) { return lds2_v(EC + i); });
}

// Per-cell weights as kernel parameters: a block is 4 warps of one cell
// (blockIdx.y), so every weight is read at a block-uniform address and
// reaches the FMAs through the uniform datapath (LDCU -> DFMA R, R, UR):
// no shared-memory traffic for the 144 weights of a step.
constexpr int kEwPC = 27;  // cells per launch (27 x 1152 B of parameters)
struct EwParams {
  double G[kEwPC][96];
  double coefh[kEwPC][48];
};
template <int CK, bool DIAG>
__global__ void __launch_bounds__(128) k_ew_rowp(const double* __restrict__ x, double* __restrict__ y,
                                                 const EwCell* __restrict__ cells, const int4* __restrict__ rows,
                                                 int nrows, double c0, int n, int64_t cs,
                                                 const double* __restrict__ phase, int cell0, int chunk0,
                                                 const __grid_constant__ EwParams p) {
  __shared__ double kbs[4][2][12][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int task = blockIdx.y * 4 + wib;
  if (task >= nrows) return;
  const int4 T = rows[task];  // (j, q, kmax)
  const int cell = chunk0 + blockIdx.x;
  const int pc = blockIdx.x;
  ew_row_march<CK, DIAG>(x, y, cells + cell, cell, T.x, 31 * T.y - 1 + lane, T.z, c0, n, cs, phase, cell0,
                         kbs[wib], lane, [&](int i) { return make_double2(p.G[pc][i], p.G[pc][i + 1]); },
                         [&](int i) { return make_double2(p.coefh[pc][i], p.coefh[pc][i + 1]); });
}

// Per-cell sin/cos tables of the sin-product phases for k_ew_row, cells
// [cell0, cell0 + ncells): [sin, cos] x [d] of beta_d0 i and of beta_d1 j for
// i, j = -1 .. n, then sin, cos of beta_d2 (one layer step).
__global__ void __launch_bounds__(256) k_ew_phase(const EwCell* __restrict__ cells, int n, int cell0,
                                                  double* __restrict__ out) {
  const int cell = cell0 + blockIdx.y, np = n + 2;
  const EwCell* E = cells + cell;
  double* P = out + (int64_t)blockIdx.y * (12 * np + 6);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 3 * np; q += gridDim.x * blockDim.x) {
    const int d = q / np, t = q % np - 1;
    double sv, cv;
    sincos(E->beta[d][0] * t, &sv, &cv);
    P[(0 * 3 + d) * np + t + 1] = sv;
    P[(1 * 3 + d) * np + t + 1] = cv;
    sincos(E->beta[d][1] * t, &sv, &cv);
    P[(2 * 3 + d) * np + t + 1] = sv;
    P[(3 * 3 + d) * np + t + 1] = cv;
  }
  if (blockIdx.x == 0 && threadIdx.x < 3) {
    double sv, cv;
    sincos(E->beta[threadIdx.x][2], &sv, &cv);
    P[12 * np + threadIdx.x] = sv;
    P[12 * np + 3 + threadIdx.x] = cv;
  }
}

// Exact positivity check of k at every quadrature point of every micro-cell
// (local_matrix's "div_k_grad coefficient must be positive", forms.hpp:114),
// for coefficients whose sign is not settled on the host. Sets *bad.
__global__ void __launch_bounds__(256) k_kpos(const double* __restrict__ maps, bt_form f, int n, int cell0,
                                              int* __restrict__ bad) {
  constexpr int kOff[6][4][3] = BT_CELL_OFFSETS;
  const int cell = cell0 + blockIdx.y, s = blockIdx.z;
  const int ws = ew_class_width(s, n);
  const double* A = maps + 12 * cell;  // row-major 3x3, then b
  const double h = 1.0 / n;
  const double qa = (5.0 + 3.0 * sqrt(5.0)) / 20.0, qb = (5.0 - sqrt(5.0)) / 20.0;
  const int64_t cnt = (int64_t)ws * (ws + 1) * (ws + 2) / 6;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < cnt; p += (int64_t)gridDim.x * blockDim.x) {
    // delinearize p in I_tet(ws)
    int64_t t = p;
    int kk = 0;
    while (t >= (int64_t)(ws - kk) * (ws - kk + 1) / 2) t -= (int64_t)(ws - kk) * (ws - kk + 1) / 2, ++kk;
    int jj = 0;
    while (t >= ws - kk - jj) t -= ws - kk - jj, ++jj;
    const int ii = (int)t;
    for (int q = 0; q < 4; ++q) {
      double r[3];
      for (int a = 0; a < 3; ++a) {
        double dl = 0;
        for (int v = 0; v < 4; ++v) dl += (v == q ? qa : qb) * kOff[s][v][a];
        r[a] = h * ((a == 0 ? ii : (a == 1 ? jj : kk)) + dl);
      }
      double xq[3];
      for (int d = 0; d < 3; ++d) xq[d] = A[3 * d] * r[0] + A[3 * d + 1] * r[1] + A[3 * d + 2] * r[2] + A[9 + d];
      const double kv = f.coeff_kind == 1
                            ? f.c[0] + f.c[1] * sin(f.c[2] * xq[0]) * sin(f.c[2] * xq[1]) * sin(f.c[2] * xq[2])
                            : f.c[0] + f.c[1] * xq[0] + f.c[2] * xq[1] + f.c[3] * xq[2];
      if (!(kv > 0.0)) atomicExch(bad, 1);
    }
  }
}
}  // namespace

void build_ew_phase(const bt_grid& g, int level, const EwCell* d_cells, DevBuf<double>& out) {
  const int n = 1 << level, nl = g.part_end - g.part_begin;
  out.alloc((size_t)std::max(nl, 1) * (12 * (n + 2) + 6));
  if (!nl) return;
  k_ew_phase<<<dim3((3 * (n + 2) + 255) / 256, nl), 256>>>(d_cells, n, g.part_begin, out.p);
  count_launch();
  check_launch("k_ew_phase");
  BT_CUDA(cudaDeviceSynchronize());
}

// tiles of this handle's cells: (cell, j0, i0, top layer)
static const DevBuf<int4>& ew_units(const bt_grid& g, int level, int& count) {
  if (g.ew_tiles[level].p || g.ew_ntiles[level] == -1) {
    count = std::max(0, g.ew_ntiles[level]);
    return g.ew_tiles[level];
  }
  const int n = 1 << level;
  std::vector<int4> u;
  for (int cell = g.part_begin; cell < g.part_end; ++cell)
    for (int j0 = 0; j0 <= n; j0 += kER)
      for (int i0 = 0; i0 + j0 <= n; i0 += kEC) u.push_back(make_int4(cell, j0, i0, n - j0 - i0));
  g.ew_tiles[level].upload(u);
  g.ew_ntiles[level] = u.empty() ? -1 : (int)u.size();
  count = (int)u.size();
  return g.ew_tiles[level];
}

// row tasks of this handle's cells for k_ew_row: (cell, j, column chunk q, top layer)
static const DevBuf<int4>& ew_row_tasks(const bt_grid& g, int level, int& count) {
  if (g.ew_rows[level].p || g.ew_nrows[level] == -1) {
    count = std::max(0, g.ew_nrows[level]);
    return g.ew_rows[level];
  }
  const int n = 1 << level;
  std::vector<int4> u;
  // longest marches first (rows near j = 0, chunks near i = 0), cells interleaved
  for (int j = 0; j <= n; ++j)
    for (int q = 0; 31 * q + j <= n; ++q)
      for (int cell = g.part_begin; cell < g.part_end; ++cell) u.push_back(make_int4(cell, j, q, n - j - 31 * q));
  std::stable_sort(u.begin(), u.end(), [](const int4& a, const int4& b) { return a.w > b.w; });
  g.ew_rows[level].upload(u);
  g.ew_nrows[level] = u.empty() ? -1 : (int)u.size();
  count = (int)u.size();
  return g.ew_rows[level];
}

// the (j, q, top layer) row marches of one cell (the same for every cell of a
// level), longest first, for k_ew_rowp
static const DevBuf<int4>& ew_row_table(const bt_grid& g, int level, int& count) {
  if (!g.ew_rowtab[level].p) {
    const int n = 1 << level;
    std::vector<int4> u;
    for (int j = 0; j <= n; ++j)
      for (int q = 0; 31 * q + j <= n; ++q) u.push_back(make_int4(j, q, n - j - 31 * q, 0));
    std::stable_sort(u.begin(), u.end(), [](const int4& a, const int4& b) { return a.z > b.z; });
    g.ew_rowtab[level].upload(u);
  }
  count = (int)g.ew_rowtab[level].n;
  return g.ew_rowtab[level];
}

void launch_elementwise(const bt_grid& g, int level, int ck, const double* c, const EwCell* d_cells, const double* x,
                        double* y, bool diag_only, cudaStream_t s, const double* phase, const EwCell* h_cells) {
  const int n = 1 << level, w = n + 1;
  if (g.part_end == g.part_begin) return;
  // levels >= 5 with host copies of the cells: weights as kernel parameters
  // (k_ew_rowp, one launch per kEwPC cells); coarser levels: k_ew_row
  static const int noparam = [] {
    const char* e = std::getenv("BT_EW_NOPARAM");
    return e ? std::atoi(e) : 0;
  }();
  if (h_cells && n >= 32 && !noparam && (ck != 1 || phase)) {
    int nr = 0;
    const DevBuf<int4>& rows = ew_row_table(g, level, nr);
    const double* xs = shifted(x, g, BT_SPACE_P1, level);
    double* ys = shifted(y, g, BT_SPACE_P1, level);
    EwParams prm;
    // chunks round-robin over the main and two side streams, so one launch's
    // tail overlaps the next launch's blocks
    SideStream& ss = side_stream();
    BT_CUDA(cudaEventRecord(ss.fork, s));
    BT_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
    BT_CUDA(cudaStreamWaitEvent(ss.s2, ss.fork, 0));
    int chunk = 0;
    for (int c0 = g.part_begin; c0 < g.part_end; c0 += kEwPC, ++chunk) {
      cudaStream_t st = chunk % 3 == 0 ? s : (chunk % 3 == 1 ? ss.s : ss.s2);
      const int cnt = std::min(kEwPC, g.part_end - c0);
      for (int q = 0; q < cnt; ++q) {
        std::memcpy(prm.G[q], &h_cells[c0 + q].G[0][0], sizeof(double) * 96);
        std::memcpy(prm.coefh[q], &h_cells[c0 + q].coefh[0][0], sizeof(double) * 48);
      }
      const dim3 grid((unsigned)cnt, (unsigned)((nr + 3) / 4));  // cells fastest: every cell's longest rows first
#define BT_EWP(CK_, D_) \
  k_ew_rowp<CK_, D_><<<grid, 128, 0, st>>>(xs, ys, d_cells, rows.p, nr, c[0], n, n_tet(w), phase, g.part_begin, c0, prm)
      if (ck == 0) { if (diag_only) BT_EWP(0, true); else BT_EWP(0, false); }
      else if (ck == 1) { if (diag_only) BT_EWP(1, true); else BT_EWP(1, false); }
      else { if (diag_only) BT_EWP(2, true); else BT_EWP(2, false); }
#undef BT_EWP
      count_launch();
    }
    BT_CUDA(cudaEventRecord(ss.join, ss.s));
    BT_CUDA(cudaStreamWaitEvent(s, ss.join, 0));
    BT_CUDA(cudaEventRecord(ss.join2, ss.s2));
    BT_CUDA(cudaStreamWaitEvent(s, ss.join2, 0));
    check_launch("k_ew_rowp");
    return;
  }
  // BT_EW_KERNEL=1 (profiling): the shared-ring tile kernel k_ew instead of k_ew_row
  static const int tile = [] {
    const char* e = std::getenv("BT_EW_KERNEL");
    return e ? std::atoi(e) : 0;
  }();
  if (!tile && (ck != 1 || phase)) {
    int nt = 0;
    const DevBuf<int4>& tasks = ew_row_tasks(g, level, nt);
    const double* xs = shifted(x, g, BT_SPACE_P1, level);
    double* ys = shifted(y, g, BT_SPACE_P1, level);
    const unsigned blocks = (unsigned)((nt + 3) / 4);  // 4 warps (rows) per block
    const double c0r = c[0];
#define BT_EWR(CK_, D_) \
  k_ew_row<CK_, D_><<<blocks, 128, 0, s>>>(xs, ys, d_cells, tasks.p, nt, c0r, n, n_tet(w), phase, g.part_begin)
    if (ck == 0) { if (diag_only) BT_EWR(0, true); else BT_EWR(0, false); }
    else if (ck == 1) { if (diag_only) BT_EWR(1, true); else BT_EWR(1, false); }
    else { if (diag_only) BT_EWR(2, true); else BT_EWR(2, false); }
#undef BT_EWR
    count_launch();
    check_launch("k_ew_row");
    return;
  }
  int nu = 0;
  const DevBuf<int4>& units = ew_units(g, level, nu);
  x = shifted(x, g, BT_SPACE_P1, level);  // global-cell indexing
  y = shifted(y, g, BT_SPACE_P1, level);
  const size_t smem = sizeof(EwShared);
  const double c0 = c[0];
#define BT_EW(CK_, D_)                                                                                   \
  {                                                                                                      \
    static bool attr = false;                                                                            \
    if (!attr) {                                                                                         \
      BT_CUDA(cudaFuncSetAttribute(k_ew<CK_, D_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
      attr = true;                                                                                       \
    }                                                                                                    \
    k_ew<CK_, D_><<<nu, kET, smem, s>>>(x, y, d_cells, units.p, c0, n, n_tet(w));                        \
  }
  if (ck == 0) { if (diag_only) BT_EW(0, true) else BT_EW(0, false) }
  else if (ck == 1) { if (diag_only) BT_EW(1, true) else BT_EW(1, false) }
  else { if (diag_only) BT_EW(2, true) else BT_EW(2, false) }
#undef BT_EW
  count_launch();
  check_launch("k_ew");
}

// local_matrix's positivity check of a div_k_grad coefficient (forms.hpp:114):
// settled on the host when the coefficient's range is (sin product: c0 > |c1|;
// affine: positive at every macro-cell vertex, hence on the cells), else
// evaluated at every quadrature point on the device
void check_coefficient(const bt_grid& g, const bt_form& f, int level, const double* d_maps, cudaStream_t s) {
  if (f.kind != BT_FORM_DIV_K_GRAD) return;
  if (f.coeff_kind == 0) {
    if (!(f.c[0] > 0)) raise(BT_INVALID_ARGUMENT, "div_k_grad coefficient must be positive");
    return;
  }
  if (f.coeff_kind == 1 && f.c[0] > std::fabs(f.c[1])) return;
  if (f.coeff_kind == 2) {
    bool ok = true;
    for (int c = g.part_begin; c < g.part_end && ok; ++c)
      for (int v = 0; v < 4 && ok; ++v) {
        const auto& p = g.mesh.coords[g.mesh.cells[c][v]];
        ok = f.c[0] + f.c[1] * p[0] + f.c[2] * p[1] + f.c[3] * p[2] > 0;
      }
    if (ok) return;
  }
  const int n = 1 << level, nl = g.part_end - g.part_begin;
  if (!nl) return;
  DevBuf<int> bad(1);
  BT_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
  k_kpos<<<dim3(64, nl, 6), 256, 0, s>>>(d_maps, f, n, g.part_begin, bad.p);
  count_launch();
  check_launch("k_kpos");
  int h = 0;
  BT_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  BT_CUDA(cudaStreamSynchronize(s));
  if (h) raise(BT_INVALID_ARGUMENT, "div_k_grad coefficient must be positive");
}

}  // namespace bt
