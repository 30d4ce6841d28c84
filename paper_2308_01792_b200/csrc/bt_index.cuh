// Analytic micro-primitive index algebra, usable from host and device.
// Restates micro_index.hpp (n_tri :85, n_tet :89, width_formula :97-121,
// linearize :145, offset tables :218-252) plus the row/layer bookkeeping of
// the tetrahedral row layout that the kernels walk.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define BT_HD __host__ __device__ __forceinline__
#else
#define BT_HD inline
#endif

namespace bt {

BT_HD int64_t n_tri(int64_t w) { return w > 0 ? w * (w + 1) / 2 : 0; }
BT_HD int64_t n_tet(int64_t w) { return w > 0 ? w * (w + 1) * (w + 2) / 6 : 0; }
// 32-bit variants for in-cell offsets (level <= 10 keeps n_tet(1025) < 2^31)
BT_HD int tri32(int w) { return w > 0 ? w * (w + 1) / 2 : 0; }
// w (w + 1) (w + 2) < 2^31 for w <= 1025 (level 10)
BT_HD int tet32(int w) { return w > 0 ? w * (w + 1) * (w + 2) / 6 : 0; }

// Subgroup ids follow enum Subgroup (micro_index.hpp:22-28).
BT_HD int width_formula(int g, int level) {
  const int n = 1 << level;
  switch (g) {
    case 0: return n + 1;
    case 7: case 9: case 11: case 13: case 15: case 16: case 17: case 18: case 19:
    case 22: case 23: case 24: case 25:
      return n - 1;
    case 21: return n - 2;
    default: return n;
  }
}

BT_HD bool in_i_tet(int w, int i, int j, int k) {
  return i >= 0 && j >= 0 && k >= 0 && i + j + k < w;
}

// Eq. (8): k-outer, j-middle, i-inner enumeration (micro_index.hpp:145).
BT_HD int64_t linearize(int w, int i, int j, int k) {
  return n_tet(w) - n_tet(w - k) + n_tri(w - k) - n_tri(w - k - j) + i;
}
// In-cell offset of the first slot of row (j, k).
BT_HD int row_start(int w, int j, int k) {
  return tet32(w) - tet32(w - k) + tri32(w - k) - tri32(w - k - j);
}

// Row r (rows enumerated k outer, j inner; layer k holds w-k rows) -> (j, k).
BT_HD void decode_row(int w, int r, int& j, int& k) {
  const double b = 2.0 * w + 1.0;
  int kk = (int)((b - sqrt(b * b - 8.0 * (double)r)) * 0.5);
  if (kk < 0) kk = 0;
  // row_start of layer k is k*w - k(k-1)/2
  while (kk > 0 && kk * w - kk * (kk - 1) / 2 > r) --kk;
  while ((kk + 1) * w - (kk + 1) * kk / 2 <= r) ++kk;
  k = kk;
  j = r - (kk * w - kk * (kk - 1) / 2);
}

// Point q of the triangle {(a, b): a, b >= 0, a + b < m} enumerated b outer.
BT_HD void decode_tri(int m, int q, int& a, int& b) {
  const double c = 2.0 * m + 1.0;
  int bb = (int)((c - sqrt(c * c - 8.0 * (double)q)) * 0.5);
  if (bb < 0) bb = 0;
  while (bb > 0 && bb * m - bb * (bb - 1) / 2 > q) --bb;
  while ((bb + 1) * m - (bb + 1) * bb / 2 <= q) ++bb;
  b = bb;
  a = q - (bb * m - bb * (bb - 1) / 2);
}

// Zero set of a lattice point: bit v set iff the barycentric weight of local
// macro vertex v vanishes (weights (n - i - j - k, i, j, k)). 0 = interior of
// the macro-cell; one bit = macro face opposite v; two bits = macro edge;
// three bits = macro vertex.
BT_HD int zero_set(int n, int i, int j, int k) {
  return (i + j + k == n ? 1 : 0) | (i == 0 ? 2 : 0) | (j == 0 ? 4 : 0) | (k == 0 ? 8 : 0);
}

// kStencilDirs (operators.hpp:22-26)
#define BT_STENCIL_DIRS                                                              \
  {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, -1, 0}, {1, 0, -1}, {0, 1, -1},     \
   {1, -1, 1}, {-1, 0, 0}, {0, -1, 0}, {0, 0, -1}, {-1, 1, 0}, {-1, 0, 1}, {0, -1, 1}, \
   {-1, 1, -1}}

// Cell-class vertex offsets (micro_index.hpp:245-252), generation order.
#define BT_CELL_OFFSETS                                                              \
  {{{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, {{1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}}, \
   {{0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {0, 1, 1}}, {{1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {1, 0, 1}}, \
   {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}}, {{0, 1, 0}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}}}

// Edge-class vertex offsets (micro_index.hpp:220-228).
#define BT_EDGE_OFFSETS                                                              \
  {{{0, 0, 0}, {1, 0, 0}}, {{0, 0, 0}, {0, 1, 0}}, {{0, 0, 0}, {0, 0, 1}},             \
   {{0, 1, 0}, {1, 0, 0}}, {{0, 0, 1}, {1, 0, 0}}, {{0, 0, 1}, {0, 1, 0}},             \
   {{0, 1, 0}, {1, 0, 1}}}

// Neighbour-slot offsets of the 15 stencil directions for every i of row
// (j, k) at width w: t(i + dx, j + dy, k + dz) - t(i, j, k), which does not
// depend on i. Only meaningful where the neighbour
// exists.
BT_HD void row_offsets(int w, int j, int k, int off[15]) {
  const int L = w - j - k;           // length of row (j, k)
  const int m = w - k;               // width of layer k
  const int U = tri32(m) - j;        // to row (j, k+1)
  const int D = -(tri32(m + 1) - j); // to row (j, k-1)
  off[0] = 0;
  off[1] = 1;
  off[2] = L;
  off[3] = U;
  off[4] = -L;
  off[5] = D + 1;
  off[6] = D + L + 1;
  off[7] = U - L + 1;
  off[8] = -1;
  off[9] = -(L + 1);
  off[10] = D;
  off[11] = L - 1;
  off[12] = U - 1;
  off[13] = U - L;
  off[14] = D + L;
}

}  // namespace bt
