/* TEST INFRASTRUCTURE — CPU restatement of the Nédélec N1E1 (lowest-order
 * Whitney edge element) curl-curl + mass operator on the reference's edge
 * storage. PARITY UNPINNED: the reference has no N1E1 implementation
 * (SPEC.md:8 lists it out of scope; the paper describes it only in prose,
 * PAPER.md:1656-1760). This restatement is built on the reference's edge
 * subgroups (micro_index.hpp:220-228) and interface groups
 * (fe_function.hpp:162-220), and self-pinned by algebraic identities in
 * tests/test_n1e1_oracle.py: K grad = 0, symmetry, u^T M u = |c|^2 |Omega|
 * for constant fields, element matrices vs closed forms.
 *
 * Conventions (builder decisions, shared with the CUDA path):
 *  - The DoF of an edge micro-primitive of subgroup g is the tangential
 *    integral along its canonical direction offs[g][0] -> offs[g][1].
 *  - Local tet edges (0,1)(0,2)(0,3)(1,2)(1,3)(2,3) in the class's vertex
 *    generation order; basis w_ab = l_a grad l_b - l_b grad l_a.
 *  - Replicas on macro faces/edges may be stored with opposite canonical
 *    orientation; the additive sync sums sigma_m v_m over the group in member
 *    order, sigma relative to member 0's orientation, and writes sigma_m S.
 *  - Tangential Dirichlet: identity rows on the edge Dirichlet masks. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "bt_oracle.h"

int bo_width_formula(int g, int level);
int64_t bo_n_tet(int64_t w);
int64_t bo_linearize(int w, int i, int j, int k);
int bo_delinearize(int w, int64_t t, int* ijk);

static const int kOffEdge[7][2][3] = {
    {{0, 0, 0}, {1, 0, 0}}, {{0, 0, 0}, {0, 1, 0}}, {{0, 0, 0}, {0, 0, 1}},
    {{0, 1, 0}, {1, 0, 0}}, {{0, 0, 1}, {1, 0, 0}}, {{0, 0, 1}, {0, 1, 0}},
    {{0, 1, 0}, {1, 0, 1}}};
static const int kOffCell[6][4][3] = {
    {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
    {{1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}},
    {{0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {0, 1, 1}},
    {{1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {1, 0, 1}},
    {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}},
    {{0, 1, 0}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}}};
static const int kLocEdge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

/* subgroup and orientation of lattice direction d (+1 canonical, -1 reversed) */
static int edge_dir(const int* d, int* sigma) {
  for (int g = 0; g < 7; ++g) {
    int e[3], same = 1, opp = 1;
    for (int a = 0; a < 3; ++a) {
      e[a] = kOffEdge[g][1][a] - kOffEdge[g][0][a];
      same &= d[a] == e[a];
      opp &= d[a] == -e[a];
    }
    if (same) { *sigma = 1; return g + 1; }
    if (opp) { *sigma = -1; return g + 1; }
  }
  return -1;
}

/* flat offset of edge entry g (1..7) within one cell of the edge space */
static int64_t entry_off(int g, int l) {
  int64_t o = 0;
  for (int q = 1; q < g; ++q) o += bo_n_tet(bo_width_formula(q, l));
  return o;
}
static int64_t cell_size(int l) { return entry_off(8, l); }

/* element matrix: alpha K + beta M on the tet with corners X (12) */
int bo_n1e1_local(const double* X, double alpha, double beta, double* out) {
  double a[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a[3 * r + c] = X[3 * (c + 1) + r] - X[r];
  const double det = a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
                     a[2] * (a[3] * a[7] - a[4] * a[6]);
  if (det == 0.0 || !isfinite(det)) return 1;
  const double vol = fabs(det) / 6.0;
  const double d = det;
  const double inv[9] = {(a[4] * a[8] - a[5] * a[7]) / d, (a[2] * a[7] - a[1] * a[8]) / d,
                         (a[1] * a[5] - a[2] * a[4]) / d, (a[5] * a[6] - a[3] * a[8]) / d,
                         (a[0] * a[8] - a[2] * a[6]) / d, (a[2] * a[3] - a[0] * a[5]) / d,
                         (a[3] * a[7] - a[4] * a[6]) / d, (a[1] * a[6] - a[0] * a[7]) / d,
                         (a[0] * a[4] - a[1] * a[3]) / d};
  double gr[4][3];
  for (int c = 0; c < 3; ++c) {
    gr[1][c] = inv[c];
    gr[2][c] = inv[3 + c];
    gr[3][c] = inv[6 + c];
    gr[0][c] = -gr[1][c] - gr[2][c] - gr[3][c];
  }
  double G[4][4], C[6][3];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) G[i][j] = gr[i][0] * gr[j][0] + gr[i][1] * gr[j][1] + gr[i][2] * gr[j][2];
  for (int e = 0; e < 6; ++e) {
    const double* u = gr[kLocEdge[e][0]];
    const double* v = gr[kLocEdge[e][1]];
    C[e][0] = u[1] * v[2] - u[2] * v[1];
    C[e][1] = u[2] * v[0] - u[0] * v[2];
    C[e][2] = u[0] * v[1] - u[1] * v[0];
  }
  for (int e = 0; e < 6; ++e)
    for (int f = 0; f < 6; ++f) {
      const int ea = kLocEdge[e][0], eb = kLocEdge[e][1], fc = kLocEdge[f][0], fd = kLocEdge[f][1];
      const double K = 4.0 * vol * (C[e][0] * C[f][0] + C[e][1] * C[f][1] + C[e][2] * C[f][2]);
#define MM(i, j) (vol * ((i) == (j) ? 2.0 : 1.0) / 20.0)
      const double M = MM(ea, fc) * G[eb][fd] - MM(ea, fd) * G[eb][fc] - MM(eb, fc) * G[ea][fd] +
                       MM(eb, fd) * G[ea][fc];
#undef MM
      out[6 * e + f] = alpha * K + beta * M;
    }
  return 0;
}

static void map_point(const bo_mesh* m, int cell, int l, int i, int j, int k, double* out) {
  const double h = 1.0 / (double)(1 << l);
  const double r[3] = {h * i, h * j, h * k};
  const double* A = m->maps + 12 * cell;
  for (int d = 0; d < 3; ++d) out[d] = (A[3 * d] * r[0] + A[3 * d + 1] * r[1] + A[3 * d + 2] * r[2]) + A[9 + d];
}

/* Signs of group members relative to member 0 (edge members only; vertex
 * members get 0). Orientation compared through the doubled-barycentric
 * position keys of the canonical first endpoint (fe_function.hpp:147-160). */
static void endpoint_key(const bo_grid* G, int l, int cell, int g, int64_t t, int which, int64_t key[8]) {
  const int w = bo_width_formula(g, l);
  int p[3];
  bo_delinearize(w, t, p);
  const int* o = kOffEdge[g - 1][which];
  const int q[3] = {p[0] + o[0], p[1] + o[1], p[2] + o[2]};
  const int64_t n = (int64_t)1 << l;
  const int64_t wt[4] = {n - (q[0] + q[1] + q[2]), q[0], q[1], q[2]};
  int64_t pairs[4][2];
  int np = 0;
  for (int a = 0; a < 4; ++a)
    if (wt[a] > 0) {
      pairs[np][0] = G->mesh.cells[4 * cell + a];
      pairs[np][1] = wt[a];
      ++np;
    }
  for (int x = 1; x < np; ++x)
    for (int y = x; y > 0 && pairs[y][0] < pairs[y - 1][0]; --y) {
      int64_t t0 = pairs[y][0], t1 = pairs[y][1];
      pairs[y][0] = pairs[y - 1][0]; pairs[y][1] = pairs[y - 1][1];
      pairs[y - 1][0] = t0; pairs[y - 1][1] = t1;
    }
  for (int x = 0; x < 8; ++x) key[x] = -1;
  for (int x = 0; x < np; ++x) { key[2 * x] = pairs[x][0]; key[2 * x + 1] = pairs[x][1]; }
}

void bo_n1e1_signs(const bo_grid* G, int l, int8_t* sign) {
  const bo_level* L = bo_grid_level(G, l);
  for (int64_t gi = 0; gi < L->ngroups; ++gi) {
    int64_t first = -1;
    int64_t k0[8];
    for (int64_t k = L->goff[gi]; k < L->goff[gi + 1]; ++k) {
      if (L->mg[k] == 0) { sign[k] = 0; continue; }
      int64_t kk[8];
      endpoint_key(G, l, L->mcell[k], L->mg[k], L->mt[k], 0, kk);
      if (first < 0) {
        first = k;
        memcpy(k0, kk, sizeof k0);
        sign[k] = 1;
      } else {
        sign[k] = memcmp(kk, k0, sizeof kk) == 0 ? 1 : -1;
      }
    }
  }
}

/* signed additive sync over edge groups (broadcast = 0) or signed owner
 * broadcast (broadcast = 1), on the edge space (space 2) */
static void n1e1_sync(const bo_grid* G, int l, double* v, int broadcast) {
  const bo_level* L = bo_grid_level(G, l);
  int8_t* sign = malloc((size_t)L->nmembers + 1);
  bo_n1e1_signs(G, l, sign);
  const int64_t cs = cell_size(l);
  for (int64_t gi = 0; gi < L->ngroups; ++gi) {
    int present = 0;
    for (int64_t k = L->goff[gi]; k < L->goff[gi + 1]; ++k) present += L->mg[k] != 0;
    if (present < 2) continue;
    double s = 0;
    int have = 0;
    for (int64_t k = L->goff[gi]; k < L->goff[gi + 1]; ++k) {
      if (!L->mg[k]) continue;
      const double val = v[cs * L->mcell[k] + entry_off(L->mg[k], l) + L->mt[k]];
      if (broadcast) {
        if (!have) { s = sign[k] * val; have = 1; }
      } else {
        s += sign[k] * val;
      }
    }
    for (int64_t k = L->goff[gi]; k < L->goff[gi + 1]; ++k)
      if (L->mg[k]) v[cs * L->mcell[k] + entry_off(L->mg[k], l) + L->mt[k]] = sign[k] * s;
  }
  free(sign);
}

void bo_n1e1_sync(const bo_grid* G, int l, double* v) { n1e1_sync(G, l, v, 0); }

void bo_n1e1_random_fill(const bo_grid* G, int l, uint64_t seed, double* out) {
  bo_mt64 rng;
  bo_mt64_seed(&rng, seed);
  const int64_t cs = cell_size(l);
  memset(out, 0, sizeof(double) * (size_t)(cs * G->mesh.nc));
  const bo_level* L = bo_grid_level(G, l);
  for (int c = 0; c < G->mesh.nc; ++c)
    for (int g = 1; g <= 7; ++g) {
      const int64_t n = bo_n_tet(bo_width_formula(g, l));
      const uint8_t* owned = L->owned[g] + n * c;
      double* a = out + cs * c + entry_off(g, l);
      for (int64_t t = 0; t < n; ++t)
        if (owned[t]) a[t] = bo_uniform(&rng, -1.0, 1.0);
    }
  n1e1_sync(G, l, out, 1);
}

int bo_n1e1_apply(const bo_grid* G, int l, double alpha, double beta, int bc, const double* x, double* y) {
  if (!G->with_edges) return 1;
  const int64_t cs = cell_size(l);
  const int nc = G->mesh.nc;
  memset(y, 0, sizeof(double) * (size_t)(cs * nc));
  for (int c = 0; c < nc; ++c) {
    for (int s = 0; s < 6; ++s) {
      const int w = bo_width_formula(20 + s, l);
      if (w <= 0) continue;
      double X[12], A[36];
      for (int v = 0; v < 4; ++v) map_point(&G->mesh, c, l, kOffCell[s][v][0], kOffCell[s][v][1], kOffCell[s][v][2], X + 3 * v);
      if (bo_n1e1_local(X, alpha, beta, A)) return 1;
      /* static edge map of this class: subgroup, sign, anchor shift */
      int eg[6], es[6], esh[6][3];
      for (int e = 0; e < 6; ++e) {
        const int* oa = kOffCell[s][kLocEdge[e][0]];
        const int* ob = kOffCell[s][kLocEdge[e][1]];
        const int d[3] = {ob[0] - oa[0], ob[1] - oa[1], ob[2] - oa[2]};
        eg[e] = edge_dir(d, &es[e]);
        const int* from = es[e] > 0 ? oa : ob;
        for (int a = 0; a < 3; ++a) esh[e][a] = from[a] - kOffEdge[eg[e] - 1][0][a];
      }
      for (int k = 0; k < w; ++k)
        for (int j = 0; j < w - k; ++j)
          for (int i = 0; i < w - k - j; ++i) {
            int64_t idx[6];
            double u[6];
            for (int e = 0; e < 6; ++e) {
              const int we = bo_width_formula(eg[e], l);
              idx[e] = cs * c + entry_off(eg[e], l) + bo_linearize(we, i + esh[e][0], j + esh[e][1], k + esh[e][2]);
              u[e] = es[e] * x[idx[e]];
            }
            for (int e = 0; e < 6; ++e) {
              double acc = 0;
              for (int f = 0; f < 6; ++f) acc += A[6 * e + f] * u[f];
              y[idx[e]] += es[e] * acc;
            }
          }
    }
  }
  n1e1_sync(G, l, y, 0);
  if (bc) {
    const bo_level* L = bo_grid_level(G, l);
    for (int c = 0; c < nc; ++c)
      for (int g = 1; g <= 7; ++g) {
        const int64_t n = bo_n_tet(bo_width_formula(g, l));
        const uint8_t* dm = L->dir[g] + n * c;
        const int64_t o = cs * c + entry_off(g, l);
        for (int64_t t = 0; t < n; ++t)
          if (dm[t]) y[o + t] = x[o + t];
      }
  }
  return 0;
}

/* u_e = phi(Q1) - phi(Q0) for a P1 vector phi (discrete gradient, edge
 * canonical direction) and u_e = c . (X(Q1) - X(Q0)) for a constant field. */
void bo_n1e1_gradient(const bo_grid* G, int l, const double* phi, double* u) {
  const int64_t cs = cell_size(l);
  const int wv = bo_width_formula(0, l);
  const int64_t nv = bo_n_tet(wv);
  for (int c = 0; c < G->mesh.nc; ++c)
    for (int g = 1; g <= 7; ++g) {
      const int w = bo_width_formula(g, l);
      const int* o0 = kOffEdge[g - 1][0];
      const int* o1 = kOffEdge[g - 1][1];
      int64_t t = 0;
      for (int k = 0; k < w; ++k)
        for (int j = 0; j < w - k; ++j)
          for (int i = 0; i < w - k - j; ++i, ++t)
            u[cs * c + entry_off(g, l) + t] =
                phi[nv * c + bo_linearize(wv, i + o1[0], j + o1[1], k + o1[2])] -
                phi[nv * c + bo_linearize(wv, i + o0[0], j + o0[1], k + o0[2])];
    }
}

void bo_n1e1_constant_field(const bo_grid* G, int l, const double* cvec, double* u) {
  const int64_t cs = cell_size(l);
  for (int c = 0; c < G->mesh.nc; ++c)
    for (int g = 1; g <= 7; ++g) {
      const int w = bo_width_formula(g, l);
      const int* o0 = kOffEdge[g - 1][0];
      const int* o1 = kOffEdge[g - 1][1];
      int64_t t = 0;
      for (int k = 0; k < w; ++k)
        for (int j = 0; j < w - k; ++j)
          for (int i = 0; i < w - k - j; ++i, ++t) {
            double a[3], b[3];
            map_point(&G->mesh, c, l, i + o0[0], j + o0[1], k + o0[2], a);
            map_point(&G->mesh, c, l, i + o1[0], j + o1[1], k + o1[2], b);
            u[cs * c + entry_off(g, l) + t] = cvec[0] * (b[0] - a[0]) + cvec[1] * (b[1] - a[1]) + cvec[2] * (b[2] - a[2]);
          }
    }
  n1e1_sync(G, l, u, 1);
}
