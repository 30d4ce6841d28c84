/* TEST INFRASTRUCTURE — C restatement of the reference hot path (see
 * bt_oracle.h for the contract). Each function cites the reference
 * file:line it restates (paths relative to
 * /root/reference/proj/include/blocktet/). Compiled with -ffp-contract=off so
 * the floating-point operation sequence equals the reference's FMA-free
 * build; tests/test_oracle_vs_ref.py checks bit equality. */
#define _POSIX_C_SOURCE 200809L
#include "bt_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
const char* bo_last_error(void) { return g_err; }
static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return 1;
}

/* ======================================================================
 * Index algebra — micro_index.hpp
 * ====================================================================== */

int64_t bo_n_tri(int64_t w) { return w > 0 ? w * (w + 1) / 2 : 0; }         /* :85 */
int64_t bo_n_tet(int64_t w) { return w > 0 ? w * (w + 1) * (w + 2) / 6 : 0; } /* :89 */

/* :97-121 — subgroup ids follow enum Subgroup (:22-28). */
int bo_width_formula(int g, int level) {
  const int n = 1 << level;
  switch (g) {
    case 0: return n + 1;                           /* V */
    case 7: case 9: case 11: case 13: case 15:      /* xyz, z/y/x/xyz-down */
    case 16: case 17: case 18: case 19:             /* xy/yz faces */
    case 22: case 23: case 24: case 25:             /* II/III cells */
      return n - 1;
    case 21: return n - 2;                          /* I-down */
    default: return n;
  }
}

static int in_i_tet(int w, int i, int j, int k) {                          /* :140 */
  return i >= 0 && j >= 0 && k >= 0 && i + j + k < w;
}

int64_t bo_linearize(int w, int i, int j, int k) {                         /* :145 */
  return bo_n_tet(w) - bo_n_tet(w - k) + bo_n_tri(w - k) - bo_n_tri(w - k - j) + i;
}

int bo_delinearize(int w, int64_t t, int* ijk) {                           /* :157 */
  if (t < 0 || t >= bo_n_tet(w)) return fail("delinearize: offset out of range");
  int k = 0, j = 0;
  while (t >= bo_n_tri(w - k)) t -= bo_n_tri(w - k), ++k;
  while (t >= w - k - j) t -= w - k - j, ++j;
  ijk[0] = (int)t;
  ijk[1] = j;
  ijk[2] = k;
  return 0;
}

/* Frozen offset tables, micro_index.hpp:218-252 (values restated). */
static const int kOffV[1][3] = {{0, 0, 0}};
static const int kOffEdge[7][2][3] = {
    {{0, 0, 0}, {1, 0, 0}}, {{0, 0, 0}, {0, 1, 0}}, {{0, 0, 0}, {0, 0, 1}},
    {{0, 1, 0}, {1, 0, 0}}, {{0, 0, 1}, {1, 0, 0}}, {{0, 0, 1}, {0, 1, 0}},
    {{0, 1, 0}, {1, 0, 1}}};
static const int kOffFace[12][3][3] = {
    {{0, 0, 0}, {0, 1, 0}, {1, 0, 0}}, {{0, 1, 0}, {1, 0, 0}, {1, 1, 0}},
    {{0, 0, 0}, {0, 0, 1}, {1, 0, 0}}, {{0, 0, 1}, {1, 0, 0}, {1, 0, 1}},
    {{0, 0, 0}, {0, 0, 1}, {0, 1, 0}}, {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}},
    {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}}, {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
    {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}}, {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}},
    {{0, 0, 1}, {0, 1, 0}, {1, 0, 1}}, {{0, 1, 0}, {1, 0, 1}, {1, 1, 0}}};
static const int kOffCell[6][4][3] = {
    {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
    {{1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}},
    {{0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {0, 1, 1}},
    {{1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {1, 0, 1}},
    {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}},
    {{0, 1, 0}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}}};

/* :257-263 */
static const int* offsets_of(int g, int* count) {
  if (g == 0) { *count = 1; return &kOffV[0][0]; }
  if (g <= 7) { *count = 2; return &kOffEdge[g - 1][0][0]; }
  if (g <= 19) { *count = 3; return &kOffFace[g - 8][0][0]; }
  *count = 4;
  return &kOffCell[g - 20][0][0];
}

int bo_subgroup_offsets(int g, int* out) {
  int n;
  const int* o = offsets_of(g, &n);
  memcpy(out, o, sizeof(int) * 3 * n);
  return n;
}

/* kStencilDirs, operators.hpp:22-26 */
static const int kDirs[15][3] = {{0, 0, 0},  {1, 0, 0},  {0, 1, 0},  {0, 0, 1},  {1, -1, 0},
                                 {1, 0, -1}, {0, 1, -1}, {1, -1, 1}, {-1, 0, 0}, {0, -1, 0},
                                 {0, 0, -1}, {-1, 1, 0}, {-1, 0, 1}, {0, -1, 1}, {-1, 1, -1}};

static int dir_index(int dx, int dy, int dz) {                    /* operators.hpp:28-32 */
  for (int i = 0; i < 15; ++i)
    if (kDirs[i][0] == dx && kDirs[i][1] == dy && kDirs[i][2] == dz) return i;
  return -1;
}

/* ======================================================================
 * libstdc++ std::mt19937_64 and uniform_real_distribution<double>
 * (fe_function.hpp:481-482 draw through these; restated from the
 * published MT19937-64 algorithm and libstdc++'s generate_canonical).
 * ====================================================================== */

void bo_mt64_seed(bo_mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = 312;
}

uint64_t bo_mt64_next(bo_mt64* r) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  static const uint64_t MA = 0xB5026F5AA96619E9ULL;
  if (r->mti >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? MA : 0ULL);
    }
    for (; i < 311; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1ULL) ? MA : 0ULL);
    }
    uint64_t x = (r->mt[311] & UM) | (r->mt[0] & LM);
    r->mt[311] = r->mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? MA : 0ULL);
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

double bo_uniform(bo_mt64* r, double a, double b) {
  /* generate_canonical<double,53>: one 64-bit draw, sum/2^64, clamp < 1 */
  double c = (double)bo_mt64_next(r) / 18446744073709551616.0;
  if (c >= 1.0) c = nextafter(1.0, 0.0);
  return c * (b - a) + a;
}

/* ======================================================================
 * Mesh — coarse_mesh.hpp
 * ====================================================================== */

typedef struct { int v[3]; int cell; } face_use;
typedef struct { int v[2]; } edge_use;

static int cmp_face_use(const void* a, const void* b) {
  const face_use* x = a;
  const face_use* y = b;
  for (int i = 0; i < 3; ++i)
    if (x->v[i] != y->v[i]) return x->v[i] < y->v[i] ? -1 : 1;
  return (x->cell > y->cell) - (x->cell < y->cell);
}
static int cmp_edge_use(const void* a, const void* b) {
  const edge_use* x = a;
  const edge_use* y = b;
  for (int i = 0; i < 2; ++i)
    if (x->v[i] != y->v[i]) return x->v[i] < y->v[i] ? -1 : 1;
  return 0;
}
static int cmp_int(const void* a, const void* b) {
  return (*(const int*)a > *(const int*)b) - (*(const int*)a < *(const int*)b);
}

static double signed_volume6(const double* c, const int* cell) {          /* :109 */
  const double* v0 = c + 3 * cell[0];
  double u[3], w[3], z[3];
  for (int i = 0; i < 3; ++i) {
    u[i] = c[3 * cell[1] + i] - v0[i];
    w[i] = c[3 * cell[2] + i] - v0[i];
    z[i] = c[3 * cell[3] + i] - v0[i];
  }
  /* dot(u, cross(w, z)) */
  const double cx = w[1] * z[2] - w[2] * z[1];
  const double cy = w[2] * z[0] - w[0] * z[2];
  const double cz = w[0] * z[1] - w[1] * z[0];
  return u[0] * cx + u[1] * cy + u[2] * cz;
}

static int face_index(const bo_mesh* m, int a, int b, int c) {            /* :49 */
  int f[3] = {a, b, c};
  qsort(f, 3, sizeof(int), cmp_int);
  int lo = 0, hi = m->nf;
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    const int* g = m->faces + 3 * mid;
    int cmp = 0;
    for (int i = 0; i < 3 && !cmp; ++i) cmp = (g[i] > f[i]) - (g[i] < f[i]);
    if (cmp < 0) lo = mid + 1; else hi = mid;
  }
  if (lo < m->nf && !memcmp(m->faces + 3 * lo, f, sizeof f)) return lo;
  return -1;
}

/* Line reader with '#' comments and blank lines skipped (:230-240). */
typedef struct { const char* p; int lineno; char buf[512]; } line_rd;
static int next_line(line_rd* r) {
  while (*r->p) {
    const char* e = strchr(r->p, '\n');
    size_t n = e ? (size_t)(e - r->p) : strlen(r->p);
    if (n >= sizeof r->buf) n = sizeof r->buf - 1;
    memcpy(r->buf, r->p, n);
    r->buf[n] = 0;
    r->p = e ? e + 1 : r->p + strlen(r->p);
    ++r->lineno;
    char* h = strchr(r->buf, '#');
    if (h) *h = 0;
    if (strspn(r->buf, " \t\r\n") == strlen(r->buf)) continue;
    return 1;
  }
  return 0;
}

void bo_mesh_free(bo_mesh* m) {
  free(m->coords); free(m->cells); free(m->faces); free(m->face_cells);
  free(m->bflags); free(m->edges); free(m->cell_faces); free(m->maps);
  memset(m, 0, sizeof *m);
}

/* parse_mesh :225-308 (+ validate_and_finalize :195-209, derive_topology
 * :165-193). The hanging-node scan (:117-163) is validation only and is not
 * restated. */
int bo_mesh_parse(const char* text, bo_mesh* m, char* err, int errlen) {
  memset(m, 0, sizeof *m);
  line_rd r = {text, 0, {0}};
  char word[64];
  long long cnt;
  if (!next_line(&r) || sscanf(r.buf, "%63s %lld", word, &cnt) != 2 || strcmp(word, "vertices"))
    return snprintf(err, errlen, "line %d: expected 'vertices <count>'", r.lineno), 1;
  m->nv = (int)cnt;
  m->coords = malloc(sizeof(double) * 3 * (m->nv ? m->nv : 1));
  for (int i = 0; i < m->nv; ++i) {
    if (!next_line(&r) ||
        sscanf(r.buf, "%lf %lf %lf", &m->coords[3 * i], &m->coords[3 * i + 1], &m->coords[3 * i + 2]) != 3)
      return snprintf(err, errlen, "line %d: expected three vertex coordinates", r.lineno), 1;
  }
  if (!next_line(&r) || sscanf(r.buf, "%63s %lld", word, &cnt) != 2 || strcmp(word, "cells"))
    return snprintf(err, errlen, "line %d: expected 'cells <count>'", r.lineno), 1;
  m->nc = (int)cnt;
  if (m->nc <= 0) return snprintf(err, errlen, "mesh has no cells"), 1;
  m->cells = malloc(sizeof(int) * 4 * m->nc);
  for (int i = 0; i < m->nc; ++i) {
    int* c = m->cells + 4 * i;
    if (!next_line(&r) || sscanf(r.buf, "%d %d %d %d", c, c + 1, c + 2, c + 3) != 4)
      return snprintf(err, errlen, "line %d: expected four vertex ids", r.lineno), 1;
    for (int k = 0; k < 4; ++k)
      if (c[k] < 0 || c[k] >= m->nv)
        return snprintf(err, errlen, "line %d: vertex id out of range", r.lineno), 1;
  }
  /* orientation repair :196-206 */
  for (int i = 0; i < m->nc; ++i) {
    int* c = m->cells + 4 * i;
    double vol = signed_volume6(m->coords, c);
    if (vol < 0) {
      int t = c[2]; c[2] = c[3]; c[3] = t;
      vol = -vol;
      ++m->nwarn;
    }
    if (vol == 0.0 || !isfinite(vol))
      return snprintf(err, errlen, "cell %d is degenerate", i), 1;
  }
  /* derive_topology :165-193 */
  face_use* fu = malloc(sizeof(face_use) * 4 * m->nc);
  edge_use* eu = malloc(sizeof(edge_use) * 6 * m->nc);
  int nfu = 0, neu = 0;
  for (int ci = 0; ci < m->nc; ++ci) {
    int v[4];
    memcpy(v, m->cells + 4 * ci, sizeof v);
    qsort(v, 4, sizeof(int), cmp_int);
    for (int a = 0; a < 3; ++a)
      if (v[a] == v[a + 1]) { free(fu); free(eu); return snprintf(err, errlen, "cell %d repeats a vertex", ci), 1; }
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) {
        eu[neu].v[0] = v[a]; eu[neu].v[1] = v[b]; ++neu;
        for (int c = b + 1; c < 4; ++c) {
          fu[nfu].v[0] = v[a]; fu[nfu].v[1] = v[b]; fu[nfu].v[2] = v[c]; fu[nfu].cell = ci; ++nfu;
        }
      }
  }
  qsort(fu, nfu, sizeof(face_use), cmp_face_use);
  qsort(eu, neu, sizeof(edge_use), cmp_edge_use);
  m->faces = malloc(sizeof(int) * 3 * nfu);
  m->face_cells = malloc(sizeof(int) * 2 * nfu);
  m->bflags = malloc(nfu);
  m->nf = 0;
  for (int i = 0; i < nfu;) {
    int j = i;
    while (j < nfu && !memcmp(fu[j].v, fu[i].v, sizeof fu[i].v)) ++j;
    if (j - i > 2) { free(fu); free(eu); return snprintf(err, errlen, "non-conforming mesh: face shared by %d cells", j - i), 1; }
    memcpy(m->faces + 3 * m->nf, fu[i].v, sizeof fu[i].v);
    m->face_cells[2 * m->nf] = fu[i].cell;
    m->face_cells[2 * m->nf + 1] = j - i == 2 ? fu[i + 1].cell : -1;
    m->bflags[m->nf] = j - i == 1 ? 1 : 0;
    ++m->nf;
    i = j;
  }
  m->edges = malloc(sizeof(int) * 2 * neu);
  m->ne = 0;
  for (int i = 0; i < neu;) {
    int j = i;
    while (j < neu && !cmp_edge_use(&eu[j], &eu[i])) ++j;
    memcpy(m->edges + 2 * m->ne, eu[i].v, sizeof eu[i].v);
    ++m->ne;
    i = j;
  }
  free(fu);
  free(eu);
  /* optional boundary section :281-305 */
  if (next_line(&r)) {
    if (sscanf(r.buf, "%63s %lld", word, &cnt) != 2 || strcmp(word, "boundary"))
      return snprintf(err, errlen, "line %d: trailing content after mesh data", r.lineno), 1;
    for (long long i = 0; i < cnt; ++i) {
      int f0, f1, f2, flag;
      if (!next_line(&r) || sscanf(r.buf, "%d %d %d %d", &f0, &f1, &f2, &flag) != 4)
        return snprintf(err, errlen, "line %d: expected three vertex ids and a flag", r.lineno), 1;
      int fi = face_index(m, f0, f1, f2);
      if (fi < 0) return snprintf(err, errlen, "line %d: boundary line names a non-existent face", r.lineno), 1;
      if (m->face_cells[2 * fi + 1] >= 0)
        return snprintf(err, errlen, "line %d: boundary line names an interior face", r.lineno), 1;
      m->bflags[fi] = flag != 0 ? 1 : 0;
    }
    if (next_line(&r)) return snprintf(err, errlen, "line %d: trailing content after mesh data", r.lineno), 1;
  }
  /* cell_face_indices :66-70 and macro_cell_map :92-105 */
  m->cell_faces = malloc(sizeof(int) * 4 * m->nc);
  m->maps = malloc(sizeof(double) * 12 * m->nc);
  for (int c = 0; c < m->nc; ++c) {
    const int* v = m->cells + 4 * c;
    m->cell_faces[4 * c + 0] = face_index(m, v[1], v[2], v[3]);
    m->cell_faces[4 * c + 1] = face_index(m, v[0], v[2], v[3]);
    m->cell_faces[4 * c + 2] = face_index(m, v[0], v[1], v[3]);
    m->cell_faces[4 * c + 3] = face_index(m, v[0], v[1], v[2]);
    const double* v0 = m->coords + 3 * v[0];
    double* A = m->maps + 12 * c;
    for (int row = 0; row < 3; ++row)
      for (int col = 0; col < 3; ++col) A[3 * row + col] = m->coords[3 * v[col + 1] + row] - v0[row];
    A[9] = v0[0]; A[10] = v0[1]; A[11] = v0[2];
  }
  return 0;
}

/* Builder-decided mesh generator for configs 3-5: cubes
 * i-fastest, six Kuhn tets per cube in cube_kuhn_text order and orientation
 * (coarse_mesh.hpp:344-368), vertex ids a + (n+1)(b + (n+1)c). */
int64_t bo_cubes_mesh_text(int n, double perturb, uint64_t seed, char* buf, int64_t buflen) {
  const int nv1 = n + 1;
  const int nverts = nv1 * nv1 * nv1;
  const double h = 1.0 / n;
  double* xyz = malloc(sizeof(double) * 3 * nverts);
  bo_mt64 rng;
  bo_mt64_seed(&rng, seed);
  for (int c = 0; c <= n; ++c)
    for (int b = 0; b <= n; ++b)
      for (int a = 0; a <= n; ++a) {
        const int id = a + nv1 * (b + nv1 * c);
        const int idx[3] = {a, b, c};
        for (int d = 0; d < 3; ++d) {
          const double off = bo_uniform(&rng, -perturb * h, perturb * h);
          const int on_bdry = idx[d] == 0 || idx[d] == n;
          xyz[3 * id + d] = idx[d] * h + (perturb > 0 && !on_bdry ? off : 0.0);
        }
      }
  /* cube_kuhn_text cell recipe */
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  int64_t len = 0;
  char tmp[256];
#define EMIT(...)                                                        \
  do {                                                                   \
    int k_ = snprintf(tmp, sizeof tmp, __VA_ARGS__);                     \
    if (buf && len + k_ < buflen) memcpy(buf + len, tmp, (size_t)k_ + 1); \
    len += k_;                                                           \
  } while (0)
  EMIT("# %d^3 unit cubes x 6 Kuhn tets, perturb %.17g, seed %llu\n", n, perturb,
       (unsigned long long)seed);
  EMIT("vertices %d\n", nverts);
  for (int i = 0; i < nverts; ++i) EMIT("%.17g %.17g %.17g\n", xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
  EMIT("cells %d\n", 6 * n * n * n);
  for (int c = 0; c < n; ++c)
    for (int b = 0; b < n; ++b)
      for (int a = 0; a < n; ++a)
        for (int p = 0; p < 6; ++p) {
          int loc[4] = {0, 0, 0, 7};
          loc[1] = 1 << perms[p][0];
          loc[2] = loc[1] | (1 << perms[p][1]);
          /* orientation of the unit-cube Kuhn tet (unperturbed corners) */
          double cc[4][3];
          for (int k = 0; k < 4; ++k)
            for (int d = 0; d < 3; ++d) cc[k][d] = (double)((loc[k] >> d) & 1);
          double u[3], w[3], z[3];
          for (int d = 0; d < 3; ++d) {
            u[d] = cc[1][d] - cc[0][d]; w[d] = cc[2][d] - cc[0][d]; z[d] = cc[3][d] - cc[0][d];
          }
          const double vol = u[0] * (w[1] * z[2] - w[2] * z[1]) + u[1] * (w[2] * z[0] - w[0] * z[2]) +
                             u[2] * (w[0] * z[1] - w[1] * z[0]);
          if (vol < 0) { int t = loc[2]; loc[2] = loc[3]; loc[3] = t; }
          int id[4];
          for (int k = 0; k < 4; ++k)
            id[k] = (a + (loc[k] & 1)) + nv1 * ((b + ((loc[k] >> 1) & 1)) + nv1 * (c + ((loc[k] >> 2) & 1)));
          EMIT("%d %d %d %d\n", id[0], id[1], id[2], id[3]);
        }
#undef EMIT
  free(xyz);
  return len;
}

/* ======================================================================
 * Grid — fe_function.hpp:92-226
 * ====================================================================== */

typedef struct {
  int nkey;
  int64_t key[6];
  int32_t cell, g;
  int64_t t;
} shared_entry;

static int cmp_shared(const void* a, const void* b) {
  const shared_entry* x = a;
  const shared_entry* y = b;
  /* lexicographic over the (id, weight) pair vector; shorter prefix first */
  const int n = x->nkey < y->nkey ? x->nkey : y->nkey;
  for (int i = 0; i < 2 * n; ++i)
    if (x->key[i] != y->key[i]) return x->key[i] < y->key[i] ? -1 : 1;
  if (x->nkey != y->nkey) return x->nkey < y->nkey ? -1 : 1;
  if (x->cell != y->cell) return x->cell < y->cell ? -1 : 1;  /* Member <=> */
  if (x->g != y->g) return x->g < y->g ? -1 : 1;
  return (x->t > y->t) - (x->t < y->t);
}

static int build_level(bo_grid* G, int l, bo_level* L) {                 /* :162-220 */
  const bo_mesh* m = &G->mesh;
  const int64_t n = (int64_t)1 << l;
  const int nslots = G->with_edges ? 8 : 1;
  L->level = l;
  size_t cap = 1 << 16, cnt = 0;
  shared_entry* sh = malloc(sizeof(shared_entry) * cap);
  for (int slot = 0; slot < nslots; ++slot) {
    const int w = bo_width_formula(slot, l);
    const int64_t count = w > 0 ? bo_n_tet(w) : 0;
    L->owned[slot] = malloc((size_t)(count * m->nc) + 1);
    L->dir[slot] = malloc((size_t)(count * m->nc) + 1);
    memset(L->owned[slot], 1, (size_t)(count * m->nc));
    memset(L->dir[slot], 0, (size_t)(count * m->nc));
  }
  for (int c = 0; c < m->nc; ++c) {
    const int* cf = m->cell_faces + 4 * c;
    for (int slot = 0; slot < nslots; ++slot) {
      const int w = bo_width_formula(slot, l);
      const int64_t count = w > 0 ? bo_n_tet(w) : 0;
      uint8_t* dir = L->dir[slot] + count * c;
      int no;
      const int* offs = offsets_of(slot, &no);
      int64_t t = 0;
      for (int k = 0; k < w; ++k)
        for (int j = 0; j < w - k; ++j)
          for (int i = 0; i < w - k - j; ++i, ++t) {
            int64_t wsum[4] = {0, 0, 0, 0}, wmax[4] = {0, 0, 0, 0};
            for (int o = 0; o < no; ++o) {
              const int q0 = i + offs[3 * o], q1 = j + offs[3 * o + 1], q2 = k + offs[3 * o + 2];
              const int64_t b[4] = {2 * (n - (q0 + q1 + q2)), 2 * (int64_t)q0, 2 * (int64_t)q1,
                                    2 * (int64_t)q2};
              for (int a = 0; a < 4; ++a) {
                wsum[a] += b[a];
                if (b[a] > wmax[a]) wmax[a] = b[a];
              }
            }
            for (int local = 0; local < 4; ++local)
              if (wmax[local] == 0 && m->bflags[cf[local]] != 0) dir[t] = 1;
            int support = 0;
            for (int a = 0; a < 4; ++a) {
              wsum[a] /= no;
              support += wsum[a] > 0;
            }
            if (support < 4) {
              if (cnt == cap) sh = realloc(sh, sizeof(shared_entry) * (cap *= 2));
              shared_entry* e = &sh[cnt++];
              e->nkey = 0;
              int64_t pairs[4][2];
              for (int a = 0; a < 4; ++a)
                if (wsum[a] > 0) {
                  pairs[e->nkey][0] = m->cells[4 * c + a];
                  pairs[e->nkey][1] = wsum[a];
                  ++e->nkey;
                }
              /* std::sort of the pair vector (position_key :154-160) */
              for (int x = 1; x < e->nkey; ++x)
                for (int y = x; y > 0 && (pairs[y][0] < pairs[y - 1][0] ||
                                          (pairs[y][0] == pairs[y - 1][0] && pairs[y][1] < pairs[y - 1][1]));
                     --y) {
                  int64_t t0 = pairs[y][0], t1 = pairs[y][1];
                  pairs[y][0] = pairs[y - 1][0]; pairs[y][1] = pairs[y - 1][1];
                  pairs[y - 1][0] = t0; pairs[y - 1][1] = t1;
                }
              memset(e->key, 0, sizeof e->key);
              for (int x = 0; x < e->nkey; ++x) {
                e->key[2 * x] = pairs[x][0];
                e->key[2 * x + 1] = pairs[x][1];
              }
              e->cell = c;
              e->g = slot;
              e->t = t;
            }
          }
    }
  }
  qsort(sh, cnt, sizeof(shared_entry), cmp_shared);
  /* groups with >= 2 members, :207-219 */
  L->goff = malloc(sizeof(int64_t) * (cnt + 1));
  L->mcell = malloc(sizeof(int32_t) * (cnt + 1));
  L->mg = malloc(sizeof(int32_t) * (cnt + 1));
  L->mt = malloc(sizeof(int64_t) * (cnt + 1));
  L->ngroups = 0;
  L->nmembers = 0;
  L->goff[0] = 0;
  for (size_t i = 0; i < cnt;) {
    size_t j = i + 1;
    while (j < cnt && sh[j].nkey == sh[i].nkey && !memcmp(sh[j].key, sh[i].key, sizeof(int64_t) * 2 * sh[i].nkey)) ++j;
    if (j - i >= 2) {
      uint8_t d = 0;
      for (size_t k = i; k < j; ++k) {
        const int64_t cnt_g = bo_n_tet(bo_width_formula(sh[k].g, l));
        d |= L->dir[sh[k].g][cnt_g * sh[k].cell + sh[k].t];
      }
      for (size_t k = i; k < j; ++k) {
        const int64_t cnt_g = bo_n_tet(bo_width_formula(sh[k].g, l));
        L->dir[sh[k].g][cnt_g * sh[k].cell + sh[k].t] = d;
        if (k > i) L->owned[sh[k].g][cnt_g * sh[k].cell + sh[k].t] = 0;
        L->mcell[L->nmembers] = sh[k].cell;
        L->mg[L->nmembers] = sh[k].g;
        L->mt[L->nmembers] = sh[k].t;
        ++L->nmembers;
      }
      L->goff[++L->ngroups] = L->nmembers;
    }
    i = j;
  }
  free(sh);
  return 0;
}

bo_grid* bo_grid_new(const char* text, int lo, int hi, int with_edges, char* err, int errlen) {
  if (lo < 2 || hi > 10 || lo > hi) {
    snprintf(err, errlen, "grid levels must satisfy 2 <= min <= max <= 10");
    return NULL;
  }
  bo_grid* G = calloc(1, sizeof *G);
  if (bo_mesh_parse(text, &G->mesh, err, errlen)) {
    bo_mesh_free(&G->mesh);
    free(G);
    return NULL;
  }
  G->lo = lo;
  G->hi = hi;
  G->with_edges = with_edges;
  G->levels = calloc((size_t)(hi - lo + 1), sizeof(bo_level));
  for (int l = lo; l <= hi; ++l) build_level(G, l, &G->levels[l - lo]);
  return G;
}

void bo_grid_free(bo_grid* G) {
  if (!G) return;
  for (int l = G->lo; l <= G->hi; ++l) {
    bo_level* L = &G->levels[l - G->lo];
    free(L->goff); free(L->mcell); free(L->mg); free(L->mt);
    for (int s = 0; s < 8; ++s) { free(L->owned[s]); free(L->dir[s]); }
  }
  free(G->levels);
  bo_mesh_free(&G->mesh);
  free(G);
}

const bo_level* bo_grid_level(const bo_grid* G, int l) {
  if (l < G->lo || l > G->hi) return NULL;
  return &G->levels[l - G->lo];
}

/* ======================================================================
 * FE vectors — fe_function.hpp:232-497
 * ====================================================================== */

static int space_entries(int space, int* gs) {
  if (space == 0) { gs[0] = 0; return 1; }
  if (space == 1) { for (int g = 0; g < 8; ++g) gs[g] = g; return 8; }
  for (int g = 1; g <= 7; ++g) gs[g - 1] = g;
  return 7;
}

static int64_t slots_of(int g, int l) {
  const int w = bo_width_formula(g, l);
  return w > 0 ? bo_n_tet(w) : 0;
}

static int64_t per_cell(int space, int l) {
  int gs[8];
  const int ne = space_entries(space, gs);
  int64_t s = 0;
  for (int e = 0; e < ne; ++e) s += slots_of(gs[e], l);
  return s;
}

/* offset of (cell, subgroup g) block in the flat array, -1 if absent */
static int64_t block_off(int space, int l, int cell, int g) {
  int gs[8];
  const int ne = space_entries(space, gs);
  int64_t o = per_cell(space, l) * cell;
  for (int e = 0; e < ne; ++e) {
    if (gs[e] == g) return o;
    o += slots_of(gs[e], l);
  }
  return -1;
}

int64_t bo_space_size(const bo_grid* G, int space, int l) {
  return per_cell(space, l) * G->mesh.nc;
}

static const uint8_t* owned_mask(const bo_grid* G, int l, int cell, int g) {
  const bo_level* L = bo_grid_level(G, l);
  return L->owned[g] + slots_of(g, l) * cell;
}
static const uint8_t* dir_mask(const bo_grid* G, int l, int cell, int g) {
  const bo_level* L = bo_grid_level(G, l);
  return L->dir[g] + slots_of(g, l) * cell;
}

/* sync_broadcast :425-446 */
static void sync_broadcast(const bo_grid* G, int space, int l, double* v) {
  const bo_level* L = bo_grid_level(G, l);
  for (int64_t gi = 0; gi < L->ngroups; ++gi) {
    int64_t owner = -1;
    for (int64_t k = L->goff[gi]; k < L->goff[gi + 1]; ++k)
      if (block_off(space, l, L->mcell[k], L->mg[k]) >= 0) { owner = k; break; }
    if (owner < 0) continue;
    const double val = v[block_off(space, l, L->mcell[owner], L->mg[owner]) + L->mt[owner]];
    for (int64_t k = L->goff[gi]; k < L->goff[gi + 1]; ++k) {
      if (k == owner) continue;
      const int64_t o = block_off(space, l, L->mcell[k], L->mg[k]);
      if (o >= 0) v[o + L->mt[k]] = val;
    }
  }
}

/* sync_additive :400-423 */
static void sync_additive(const bo_grid* G, int space, int l, double* v) {
  const bo_level* L = bo_grid_level(G, l);
  for (int64_t gi = 0; gi < L->ngroups; ++gi) {
    int present = 0;
    for (int64_t k = L->goff[gi]; k < L->goff[gi + 1]; ++k)
      present += block_off(space, l, L->mcell[k], L->mg[k]) >= 0;
    if (present < 2) continue;
    double sum = 0;
    for (int64_t k = L->goff[gi]; k < L->goff[gi + 1]; ++k) {
      const int64_t o = block_off(space, l, L->mcell[k], L->mg[k]);
      if (o >= 0) sum += v[o + L->mt[k]];
    }
    for (int64_t k = L->goff[gi]; k < L->goff[gi + 1]; ++k) {
      const int64_t o = block_off(space, l, L->mcell[k], L->mg[k]);
      if (o >= 0) v[o + L->mt[k]] = sum;
    }
  }
}

void bo_sync(const bo_grid* G, int space, int l, int broadcast, double* v) {
  if (broadcast) sync_broadcast(G, space, l, v);
  else sync_additive(G, space, l, v);
}

/* random_fill :479-497 */
void bo_random_fill(const bo_grid* G, int space, int l, uint64_t seed, double* out) {
  bo_mt64 rng;
  bo_mt64_seed(&rng, seed);
  int gs[8];
  const int ne = space_entries(space, gs);
  memset(out, 0, sizeof(double) * (size_t)bo_space_size(G, space, l));
  for (int c = 0; c < G->mesh.nc; ++c)
    for (int e = 0; e < ne; ++e) {
      const int64_t n = slots_of(gs[e], l);
      const uint8_t* owned = owned_mask(G, l, c, gs[e]);
      double* a = out + block_off(space, l, c, gs[e]);
      for (int64_t t = 0; t < n; ++t)
        if (owned[t]) a[t] = bo_uniform(&rng, -1.0, 1.0);
    }
  sync_broadcast(G, space, l, out);
}

/* dot :376-394 */
double bo_dot(const bo_grid* G, int space, int l, const double* x, const double* y) {
  int gs[8];
  const int ne = space_entries(space, gs);
  double acc = 0;
  for (int c = 0; c < G->mesh.nc; ++c)
    for (int e = 0; e < ne; ++e) {
      const int64_t n = slots_of(gs[e], l);
      const uint8_t* owned = owned_mask(G, l, c, gs[e]);
      const int64_t o = block_off(space, l, c, gs[e]);
      for (int64_t t = 0; t < n; ++t)
        if (owned[t]) acc += x[o + t] * y[o + t];
    }
  return acc;
}

int64_t bo_owned_count(const bo_grid* G, int space, int l) {               /* :550-566 */
  int gs[8];
  const int ne = space_entries(space, gs);
  int64_t cnt = 0;
  for (int c = 0; c < G->mesh.nc; ++c)
    for (int e = 0; e < ne; ++e) {
      const int64_t n = slots_of(gs[e], l);
      const uint8_t* owned = owned_mask(G, l, c, gs[e]);
      for (int64_t t = 0; t < n; ++t) cnt += owned[t];
    }
  return cnt;
}

/* P1 algebra on the flat level array (fe_function.hpp:324-371,
 * solvers.hpp:53-72) */
static void vassign(double* v, int64_t n, double a) { for (int64_t i = 0; i < n; ++i) v[i] = a; }
static void vscale(double* v, int64_t n, double s) { for (int64_t i = 0; i < n; ++i) v[i] *= s; }
static void vcopy(const double* s, double* d, int64_t n) { memcpy(d, s, sizeof(double) * (size_t)n); }
static void vaxpy(double* y, double a, const double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] += a * x[i];
}
static void vhadamard(double* v, const double* d, int64_t n, int divide) {
  for (int64_t i = 0; i < n; ++i) v[i] = divide ? v[i] / d[i] : v[i] * d[i];
}

void bo_impose_dirichlet(const bo_grid* G, int l, const double* src, double* dst) { /* operators.hpp:98 */
  const int64_t n = slots_of(0, l);
  for (int c = 0; c < G->mesh.nc; ++c) {
    const uint8_t* d = dir_mask(G, l, c, 0);
    for (int64_t t = 0; t < n; ++t)
      if (d[t]) dst[n * c + t] = src[n * c + t];
  }
}

void bo_zero_dirichlet(const bo_grid* G, int l, double* x) {              /* solvers.hpp:66 */
  const int64_t n = slots_of(0, l);
  for (int c = 0; c < G->mesh.nc; ++c) {
    const uint8_t* d = dir_mask(G, l, c, 0);
    for (int64_t t = 0; t < n; ++t)
      if (d[t]) x[n * c + t] = 0.0;
  }
}

/* ======================================================================
 * Forms — forms.hpp:29-120
 * ====================================================================== */

static double kval(const double* kp, const double* x) {
  const int kind = (int)kp[0];
  if (kind == 0) return kp[1];
  if (kind == 1) return kp[1] + kp[2] * sin(kp[3] * x[0]) * sin(kp[3] * x[1]) * sin(kp[3] * x[2]);
  return kp[1] + kp[2] * x[0] + kp[3] * x[1] + kp[4] * x[2];
}

/* local_matrix :75-120 (Mat3 det/inverse geometry.hpp:43-58) */
int bo_local_matrix(int form, const double* kp, const double* x, double* out) {
  double a[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a[3 * r + c] = x[3 * (c + 1) + r] - x[r];
  const double det = a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
                     a[2] * (a[3] * a[7] - a[4] * a[6]);
  if (det == 0.0 || !isfinite(det)) return fail("local_matrix: degenerate element");
  const double vol = fabs(det) / 6.0;
  if (form == 1) {
    for (int k = 0; k < 4; ++k)
      for (int l = 0; l < 4; ++l) out[4 * k + l] = vol / 20.0 * (k == l ? 2.0 : 1.0);
    return 0;
  }
  const double d = det;
  const double inv[9] = {(a[4] * a[8] - a[5] * a[7]) / d, (a[2] * a[7] - a[1] * a[8]) / d,
                         (a[1] * a[5] - a[2] * a[4]) / d, (a[5] * a[6] - a[3] * a[8]) / d,
                         (a[0] * a[8] - a[2] * a[6]) / d, (a[2] * a[3] - a[0] * a[5]) / d,
                         (a[3] * a[7] - a[4] * a[6]) / d, (a[1] * a[6] - a[0] * a[7]) / d,
                         (a[0] * a[4] - a[1] * a[3]) / d};
  static const double rg[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  double grad[4][3];
  for (int i = 0; i < 4; ++i) {
    const double gx = rg[i][0], gy = rg[i][1], gz = rg[i][2];
    grad[i][0] = inv[0] * gx + inv[3] * gy + inv[6] * gz;
    grad[i][1] = inv[1] * gx + inv[4] * gy + inv[7] * gz;
    grad[i][2] = inv[2] * gx + inv[5] * gy + inv[8] * gz;
  }
#define DOT3(p, q) ((p)[0] * (q)[0] + (p)[1] * (q)[1] + (p)[2] * (q)[2])
  if (form == 0) {
    for (int k = 0; k < 4; ++k)
      for (int l = 0; l < 4; ++l) out[4 * k + l] = vol * DOT3(grad[k], grad[l]);
    return 0;
  }
  const double qa = (5.0 + 3.0 * sqrt(5.0)) / 20.0;                       /* :56-61 */
  const double qb = (5.0 - sqrt(5.0)) / 20.0;
  double weight = 0;
  for (int q = 0; q < 4; ++q) {
    double p[3] = {0, 0, 0};
    for (int i = 0; i < 4; ++i) {
      const double bary = i == q ? qa : qb;
      for (int dd = 0; dd < 3; ++dd) p[dd] = p[dd] + x[3 * i + dd] * bary;
    }
    const double kq = kval(kp, p);
    if (!(kq > 0)) return fail("div_k_grad coefficient must be positive");
    weight += 0.25 * kq;
  }
  for (int k = 0; k < 4; ++k)
    for (int l = 0; l < 4; ++l) out[4 * k + l] = vol * weight * DOT3(grad[k], grad[l]);
#undef DOT3
  return 0;
}

/* MacroCellMap::map ∘ micro_vertex_coord (coarse_mesh.hpp:89,
 * micro_index.hpp:266-271) */
static void map_point(const bo_mesh* m, int cell, int l, int i, int j, int k, double* out) {
  const double h = 1.0 / (double)(1 << l);
  const double r[3] = {h * i, h * j, h * k};
  const double* A = m->maps + 12 * cell;
  for (int d = 0; d < 3; ++d) out[d] = (A[3 * d] * r[0] + A[3 * d + 1] * r[1] + A[3 * d + 2] * r[2]) + A[9 + d];
}

/* class_matrices operators.hpp:54-69 */
int bo_class_matrices(const bo_grid* G, int form, int l, int cell, double* out96) {
  for (int s = 0; s < 6; ++s) {
    const int g = 20 + s;
    if (bo_width_formula(g, l) <= 0) { memset(out96 + 16 * s, 0, sizeof(double) * 16); continue; }
    double corners[12];
    for (int i = 0; i < 4; ++i)
      map_point(&G->mesh, cell, l, kOffCell[s][i][0], kOffCell[s][i][1], kOffCell[s][i][2], corners + 3 * i);
    if (bo_local_matrix(form, NULL, corners, out96 + 16 * s)) return 1;
  }
  return 0;
}

/* compute_stencil operators.hpp:183-242 (probe (1,1,1)) */
int bo_compute_stencil(const bo_grid* G, int form, int l, double* rows, double* diag) {
  if (form == 2) return fail("compute_stencil: variable-coefficient forms are unsupported");
  const int wv = bo_width_formula(0, l);
  const int64_t nv = bo_n_tet(wv);
  double cls[96];
  for (int c = 0; c < G->mesh.nc; ++c) {
    if (bo_class_matrices(G, form, l, c, cls)) return 1;
    double* row = rows + 15 * c;
    for (int d = 0; d < 15; ++d) row[d] = 0.0;
    int combos = 0;
    for (int s = 0; s < 6; ++s) {
      const int w = bo_width_formula(20 + s, l);
      if (w <= 0) continue;
      for (int slot = 0; slot < 4; ++slot) {
        const int* o = kOffCell[s][slot];
        if (!in_i_tet(w, 1 - o[0], 1 - o[1], 1 - o[2])) continue;
        ++combos;
        for (int j = 0; j < 4; ++j) {
          const int* oj = kOffCell[s][j];
          row[dir_index(oj[0] - o[0], oj[1] - o[1], oj[2] - o[2])] += cls[16 * s + 4 * slot + j];
        }
      }
    }
    if (combos != 24) return fail("interior probe must touch 24 micro-cells");
    if (diag) {
      int64_t t = 0;
      for (int k = 0; k < wv; ++k)
        for (int j = 0; j < wv - k; ++j)
          for (int i = 0; i < wv - k - j; ++i, ++t) {
            double dg = 0;
            for (int s = 0; s < 6; ++s) {
              const int w = bo_width_formula(20 + s, l);
              if (w <= 0) continue;
              for (int slot = 0; slot < 4; ++slot) {
                const int* o = kOffCell[s][slot];
                if (in_i_tet(w, i - o[0], j - o[1], k - o[2])) dg += cls[16 * s + 5 * slot];
              }
            }
            diag[nv * c + t] = dg;
          }
    }
  }
  if (diag) sync_additive(G, 0, l, diag);
  return 0;
}

static int p1_interior(int i, int j, int k, int64_t n) {                /* operators.hpp:71 */
  return i >= 1 && j >= 1 && k >= 1 && i + j + k <= n - 1;
}

/* partial_row_apply operators.hpp:78-96 */
static double partial_row(const double* cls, const double* x, int l, int wv, int i, int j, int k) {
  double acc = 0;
  for (int s = 0; s < 6; ++s) {
    const int w = bo_width_formula(20 + s, l);
    if (w <= 0) continue;
    for (int slot = 0; slot < 4; ++slot) {
      const int* o = kOffCell[s][slot];
      const int ai = i - o[0], aj = j - o[1], ak = k - o[2];
      if (!in_i_tet(w, ai, aj, ak)) continue;
      for (int jj = 0; jj < 4; ++jj) {
        const int* oj = kOffCell[s][jj];
        acc += cls[16 * s + 4 * slot + jj] * x[bo_linearize(wv, ai + oj[0], aj + oj[1], ak + oj[2])];
      }
    }
  }
  return acc;
}

/* apply_stencil operators.hpp:247-271 */
int bo_apply_stencil(const bo_grid* G, int form, int l, int bc, const double* x, double* y) {
  const int nc = G->mesh.nc;
  double* rows = malloc(sizeof(double) * 15 * nc);
  double* clsall = malloc(sizeof(double) * 96 * nc);
  if (bo_compute_stencil(G, form, l, rows, NULL)) { free(rows); free(clsall); return 1; }
  for (int c = 0; c < nc; ++c) bo_class_matrices(G, form, l, c, clsall + 96 * c);
  const int64_t n = (int64_t)1 << l;
  const int wv = bo_width_formula(0, l);
  const int64_t nv = bo_n_tet(wv);
  for (int c = 0; c < nc; ++c) {
    const double* row = rows + 15 * c;
    const double* xc = x + nv * c;
    double* yc = y + nv * c;
    int64_t t = 0;
    for (int k = 0; k < wv; ++k)
      for (int j = 0; j < wv - k; ++j)
        for (int i = 0; i < wv - k - j; ++i, ++t) {
          double acc;
          if (p1_interior(i, j, k, n)) {
            acc = row[0] * xc[bo_linearize(wv, i, j, k)];
            for (int d = 1; d < 15; ++d)
              acc += row[d] * xc[bo_linearize(wv, i + kDirs[d][0], j + kDirs[d][1], k + kDirs[d][2])];
          } else {
            acc = partial_row(clsall + 96 * c, xc, l, wv, i, j, k);
          }
          yc[t] = acc;
        }
  }
  free(rows);
  free(clsall);
  sync_additive(G, 0, l, y);
  if (bc) bo_impose_dirichlet(G, l, x, y);
  return 0;
}

/* apply_elementwise operators.hpp:115-164 */
int bo_apply_elementwise(const bo_grid* G, int form, const double* kp, int l, int add, int bc,
                         const double* x, double* y) {
  const int64_t total = bo_space_size(G, 0, l);
  if (add) {
    double* scratch = malloc(sizeof(double) * (size_t)total);
    int rc = bo_apply_elementwise(G, form, kp, l, 0, bc, x, scratch);
    if (!rc) vaxpy(y, 1.0, scratch, total);
    free(scratch);
    return rc;
  }
  vassign(y, total, 0.0);
  const int wv = bo_width_formula(0, l);
  const int64_t nv = bo_n_tet(wv);
  double cls[96], em[16], corners[12];
  for (int c = 0; c < G->mesh.nc; ++c) {
    if (form != 2 && bo_class_matrices(G, form, l, c, cls)) return 1;
    const double* xc = x + nv * c;
    double* yc = y + nv * c;
    for (int s = 0; s < 6; ++s) {
      const int w = bo_width_formula(20 + s, l);
      if (w <= 0) continue;
      for (int k = 0; k < w; ++k)
        for (int j = 0; j < w - k; ++j)
          for (int i = 0; i < w - k - j; ++i) {
            int64_t idx[4];
            double xv[4];
            for (int v = 0; v < 4; ++v) {
              const int* o = kOffCell[s][v];
              idx[v] = bo_linearize(wv, i + o[0], j + o[1], k + o[2]);
              xv[v] = xc[idx[v]];
            }
            const double* m;
            if (form != 2) {
              m = cls + 16 * s;
            } else {
              for (int v = 0; v < 4; ++v) {
                const int* o = kOffCell[s][v];
                map_point(&G->mesh, c, l, i + o[0], j + o[1], k + o[2], corners + 3 * v);
              }
              if (bo_local_matrix(form, kp, corners, em)) return 1;
              m = em;
            }
            for (int a = 0; a < 4; ++a) {
              double acc = 0;
              for (int b = 0; b < 4; ++b) acc += m[4 * a + b] * xv[b];
              yc[idx[a]] += acc;
            }
          }
    }
  }
  sync_additive(G, 0, l, y);
  if (bc) bo_impose_dirichlet(G, l, x, y);
  return 0;
}

/* extract_diagonal operators.hpp:277-308 */
int bo_extract_diagonal(const bo_grid* G, int form, const double* kp, int l, double* d) {
  vassign(d, bo_space_size(G, 0, l), 0.0);
  const int wv = bo_width_formula(0, l);
  const int64_t nv = bo_n_tet(wv);
  double cls[96], em[16], corners[12];
  for (int c = 0; c < G->mesh.nc; ++c) {
    if (form != 2 && bo_class_matrices(G, form, l, c, cls)) return 1;
    for (int s = 0; s < 6; ++s) {
      const int w = bo_width_formula(20 + s, l);
      if (w <= 0) continue;
      for (int k = 0; k < w; ++k)
        for (int j = 0; j < w - k; ++j)
          for (int i = 0; i < w - k - j; ++i) {
            const double* m;
            if (form != 2) {
              m = cls + 16 * s;
            } else {
              for (int v = 0; v < 4; ++v) {
                const int* o = kOffCell[s][v];
                map_point(&G->mesh, c, l, i + o[0], j + o[1], k + o[2], corners + 3 * v);
              }
              if (bo_local_matrix(form, kp, corners, em)) return 1;
              m = em;
            }
            for (int v = 0; v < 4; ++v) {
              const int* o = kOffCell[s][v];
              d[nv * c + bo_linearize(wv, i + o[0], j + o[1], k + o[2])] += m[5 * v];
            }
          }
    }
  }
  sync_additive(G, 0, l, d);
  return 0;
}

/* ======================================================================
 * Transfers — solvers.hpp:183-293
 * ====================================================================== */

static int coarse_endpoints(int i, int j, int k, int e[2][3]) {           /* :183-211 */
  const int code = (i & 1) | ((j & 1) << 1) | ((k & 1) << 2);
  static const int d[8][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {1, -1, 0},
                              {0, 0, 1}, {1, 0, -1}, {0, 1, -1}, {-1, 1, -1}};
  if (code == 0) {
    e[0][0] = i; e[0][1] = j; e[0][2] = k;
    return 1;
  }
  /* first endpoint p - d for codes 1,2,4 and p + d for 3,5,6; code 7 is
   * (p - (1,-1,1), p + (1,-1,1)) — all expressed as p + s*d below */
  const int s0 = (code == 1 || code == 2 || code == 4 || code == 7) ? -1 : 1;
  if (code == 7) {
    e[0][0] = i - 1; e[0][1] = j + 1; e[0][2] = k - 1;
    e[1][0] = i + 1; e[1][1] = j - 1; e[1][2] = k + 1;
    return 2;
  }
  for (int a = 0; a < 3; ++a) {
    e[0][a] = (a == 0 ? i : a == 1 ? j : k) + s0 * d[code][a];
    e[1][a] = (a == 0 ? i : a == 1 ? j : k) - s0 * d[code][a];
  }
  return 2;
}

void bo_prolongate(const bo_grid* G, int fine_l, const double* coarse, double* fine) { /* :227-253 */
  const int wf = bo_width_formula(0, fine_l), wc = bo_width_formula(0, fine_l - 1);
  const int64_t nf = bo_n_tet(wf), ncs = bo_n_tet(wc);
  for (int c = 0; c < G->mesh.nc; ++c) {
    int64_t t = 0;
    for (int k = 0; k < wf; ++k)
      for (int j = 0; j < wf - k; ++j)
        for (int i = 0; i < wf - k - j; ++i, ++t) {
          int e[2][3];
          const int ne = coarse_endpoints(i, j, k, e);
          double value;
          if (ne == 1) {
            value = coarse[ncs * c + bo_linearize(wc, i / 2, j / 2, k / 2)];
          } else {
            double sum = 0;
            for (int q = 0; q < 2; ++q) sum += coarse[ncs * c + bo_linearize(wc, e[q][0] / 2, e[q][1] / 2, e[q][2] / 2)];
            value = 0.5 * sum;
          }
          fine[nf * c + t] = value;
        }
  }
}

void bo_restrict(const bo_grid* G, int fine_l, const double* fine, double* coarse) { /* :259-293 */
  const int wf = bo_width_formula(0, fine_l), wc = bo_width_formula(0, fine_l - 1);
  const int64_t nf = bo_n_tet(wf), ncs = bo_n_tet(wc);
  const int nc = G->mesh.nc;
  double* tmp = malloc(sizeof(double) * (size_t)(nf * nc));
  vcopy(fine, tmp, nf * nc);
  for (int c = 0; c < nc; ++c) {
    const uint8_t* owned = owned_mask(G, fine_l, c, 0);
    for (int64_t t = 0; t < nf; ++t)
      if (!owned[t]) tmp[nf * c + t] = 0.0;
  }
  vassign(coarse, ncs * nc, 0.0);
  for (int c = 0; c < nc; ++c) {
    int64_t t = 0;
    for (int k = 0; k < wf; ++k)
      for (int j = 0; j < wf - k; ++j)
        for (int i = 0; i < wf - k - j; ++i, ++t) {
          const double v = tmp[nf * c + t];
          int e[2][3];
          const int ne = coarse_endpoints(i, j, k, e);
          if (ne == 1) {
            coarse[ncs * c + bo_linearize(wc, i / 2, j / 2, k / 2)] += v;
          } else {
            for (int q = 0; q < 2; ++q)
              coarse[ncs * c + bo_linearize(wc, e[q][0] / 2, e[q][1] / 2, e[q][2] / 2)] += 0.5 * v;
          }
        }
  }
  free(tmp);
  sync_additive(G, 0, fine_l - 1, coarse);
}

/* ======================================================================
 * Hierarchy, smoothers, CG, V-cycle — solvers.hpp:84-541
 * ====================================================================== */

struct bo_hier {
  const bo_grid* G;
  int form, kernel;
  double kp[5];
  double** diag;     /* per level */
  double* lambda;    /* per level, 0 = not yet estimated */
};

bo_hier* bo_hier_new(const bo_grid* G, int form, const double* kp, int kernel) { /* :323-350 */
  if (kernel == 1 && form == 2) {
    fail("stencil kernel requires a constant-coefficient form");
    return NULL;
  }
  bo_hier* h = calloc(1, sizeof *h);
  h->G = G;
  h->form = form;
  h->kernel = kernel;
  if (kp) memcpy(h->kp, kp, sizeof h->kp);
  const int nl = G->hi - G->lo + 1;
  h->diag = calloc((size_t)nl, sizeof(double*));
  h->lambda = calloc((size_t)nl, sizeof(double));
  for (int l = G->lo; l <= G->hi; ++l) {
    double* d = malloc(sizeof(double) * (size_t)bo_space_size(G, 0, l));
    int rc;
    if (form != 2) {
      double* rows = malloc(sizeof(double) * 15 * G->mesh.nc);
      rc = bo_compute_stencil(G, form, l, rows, d);
      free(rows);
    } else {
      rc = bo_extract_diagonal(G, form, h->kp, l, d);
    }
    if (rc) { free(d); bo_hier_free(h); return NULL; }
    h->diag[l - G->lo] = d;
  }
  return h;
}

void bo_hier_free(bo_hier* h) {
  if (!h) return;
  for (int l = h->G->lo; l <= h->G->hi; ++l) free(h->diag[l - h->G->lo]);
  free(h->diag);
  free(h->lambda);
  free(h);
}

const double* bo_hier_diag(bo_hier* h, int l) { return h->diag[l - h->G->lo]; }

int bo_hier_apply(bo_hier* h, int l, int bc, const double* x, double* y) {   /* :352-360 */
  if (h->kernel == 1) return bo_apply_stencil(h->G, h->form, l, bc, x, y);
  return bo_apply_elementwise(h->G, h->form, h->kp, l, 0, bc, x, y);
}

static double norm2(const bo_grid* G, int l, const double* x) { return sqrt(bo_dot(G, 0, l, x, x)); }

/* estimate_lambda_max :140-172 via spectral_estimate :362-371 */
double bo_hier_lambda(bo_hier* h, int l) {
  double* lam = &h->lambda[l - h->G->lo];
  if (*lam != 0.0) return *lam;
  const bo_grid* G = h->G;
  const int64_t n = bo_space_size(G, 0, l);
  const double* diag = bo_hier_diag(h, l);
  for (int64_t i = 0; i < n; ++i)
    if (diag[i] == 0.0) { fail("estimate_lambda_max: zero diagonal entry"); return -1; }
  double* v = malloc(sizeof(double) * (size_t)n);
  double* w = malloc(sizeof(double) * (size_t)n);
  double* z = malloc(sizeof(double) * (size_t)n);
  bo_random_fill(G, 0, l, 0x51cbu, v);
  bo_zero_dirichlet(G, l, v);
  const double nv = norm2(G, l, v);
  vscale(v, n, 1.0 / nv);
  double rho = 0;
  for (int k = 0; k < 25; ++k) {
    bo_hier_apply(h, l, 1, v, w);
    vcopy(v, z, n);
    vhadamard(z, diag, n, 0);
    rho = bo_dot(G, 0, l, v, w) / bo_dot(G, 0, l, v, z);
    vcopy(w, v, n);
    vhadamard(v, diag, n, 1);
    const double nn = norm2(G, l, v);
    if (nn == 0) break;
    vscale(v, n, 1.0 / nn);
  }
  free(v); free(w); free(z);
  *lam = 1.1 * rho;
  return *lam;
}

/* chebyshev_apply :425-456 */
static void chebyshev(bo_hier* h, const double* rhs, double* x, int l, int order, double a, double b) {
  const bo_grid* G = h->G;
  const int64_t n = bo_space_size(G, 0, l);
  const double* diag = bo_hier_diag(h, l);
  const double theta = 0.5 * (b + a);
  const double delta = 0.5 * (b - a);
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  double* r = calloc((size_t)n, sizeof(double));
  double* d = calloc((size_t)n, sizeof(double));
  bo_hier_apply(h, l, 1, x, r);
  vscale(r, n, -1.0);
  vaxpy(r, 1.0, rhs, n);
  vhadamard(r, diag, n, 1);
  vcopy(r, d, n);
  vscale(d, n, 1.0 / theta);
  vaxpy(x, 1.0, d, n);
  bo_impose_dirichlet(G, l, rhs, x);
  for (int k = 1; k < order; ++k) {
    bo_hier_apply(h, l, 1, x, r);
    vscale(r, n, -1.0);
    vaxpy(r, 1.0, rhs, n);
    vhadamard(r, diag, n, 1);
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    vscale(d, n, rho_new * rho);
    vaxpy(d, 2.0 * rho_new / delta, r, n);
    vaxpy(x, 1.0, d, n);
    bo_impose_dirichlet(G, l, rhs, x);
    rho = rho_new;
  }
  free(r);
  free(d);
}

/* gauss_seidel_sweep operators.hpp:327-387 (stencil hierarchies only) */
static int gauss_seidel(bo_hier* h, const double* rhs, double* x, int l, int backward) {
  const bo_grid* G = h->G;
  const int nc = G->mesh.nc;
  const int64_t n = (int64_t)1 << l;
  const int wv = bo_width_formula(0, l);
  const int64_t nv = bo_n_tet(wv);
  double* rows = malloc(sizeof(double) * 15 * nc);
  double* cls = malloc(sizeof(double) * 96 * nc);
  bo_compute_stencil(G, h->form, l, rows, NULL);
  for (int c = 0; c < nc; ++c) bo_class_matrices(G, h->form, l, c, cls + 96 * c);
  for (int c = 0; c < nc; ++c)
    if (rows[15 * c] == 0.0) { free(rows); free(cls); return fail("gauss_seidel_sweep: zero center weight"); }
  const int ni = (int)n;
  for (int c = 0; c < nc; ++c) {
    const double* row = rows + 15 * c;
    double* xc = x + nv * c;
    const double* bc = rhs + nv * c;
#define GS_UPDATE(I, J, K)                                                                  \
  do {                                                                                      \
    const int64_t t_ = bo_linearize(wv, I, J, K);                                           \
    double acc_ = bc[t_];                                                                   \
    for (int d_ = 1; d_ < 15; ++d_)                                                         \
      acc_ -= row[d_] * xc[bo_linearize(wv, (I) + kDirs[d_][0], (J) + kDirs[d_][1], (K) + kDirs[d_][2])]; \
    xc[t_] = acc_ / row[0];                                                                 \
  } while (0)
    if (!backward) {
      for (int k = 1; k < ni; ++k)
        for (int j = 1; j < ni - k; ++j)
          for (int i = 1; i <= ni - 1 - k - j; ++i) GS_UPDATE(i, j, k);
    } else {
      for (int k = ni - 1; k >= 1; --k)
        for (int j = ni - k - 1; j >= 1; --j)
          for (int i = ni - 1 - k - j; i >= 1; --i) GS_UPDATE(i, j, k);
    }
#undef GS_UPDATE
  }
  double* scratch = calloc((size_t)(nv * nc), sizeof(double));
  for (int c = 0; c < nc; ++c) {
    int64_t t = 0;
    for (int k = 0; k < wv; ++k)
      for (int j = 0; j < wv - k; ++j)
        for (int i = 0; i < wv - k - j; ++i, ++t)
          if (!p1_interior(i, j, k, n)) scratch[nv * c + t] = partial_row(cls + 96 * c, x + nv * c, l, wv, i, j, k);
  }
  sync_additive(G, 0, l, scratch);
  const double* diag = bo_hier_diag(h, l);
  for (int c = 0; c < nc; ++c) {
    const uint8_t* dm = dir_mask(G, l, c, 0);
    int64_t t = 0;
    for (int k = 0; k < wv; ++k)
      for (int j = 0; j < wv - k; ++j)
        for (int i = 0; i < wv - k - j; ++i, ++t) {
          if (p1_interior(i, j, k, n)) continue;
          const int64_t o = nv * c + t;
          if (dm[t]) x[o] = rhs[o];
          else x[o] += (rhs[o] - scratch[o]) / diag[o];
        }
  }
  free(scratch);
  free(rows);
  free(cls);
  return 0;
}

/* smooth :460-492 */
int bo_smooth(bo_hier* h, const double* sm, int l, int sweeps, int backward, const double* rhs, double* x) {
  const int kind = (int)sm[0];
  const double omega = sm[1], lo = sm[3], hi = sm[4];
  const int order = (int)sm[2];
  if (!(omega > 0) || omega > 1) return fail("smoother: omega must lie in (0, 1]");
  if (order < 1) return fail("smoother: order must be >= 1");
  if (!(lo > 0) || !(hi > lo)) return fail("smoother: need 0 < lo < hi");
  const bo_grid* G = h->G;
  const int64_t n = bo_space_size(G, 0, l);
  for (int s = 0; s < sweeps; ++s) {
    if (kind == 1) {
      if (h->form == 2) return fail("gauss-seidel smoothing requires a stencil table");
      if (gauss_seidel(h, rhs, x, l, backward)) return 1;
    } else if (kind == 0) {
      double* r = calloc((size_t)n, sizeof(double));
      bo_hier_apply(h, l, 1, x, r);
      vscale(r, n, -1.0);
      vaxpy(r, 1.0, rhs, n);
      vhadamard(r, bo_hier_diag(h, l), n, 1);
      vaxpy(x, omega, r, n);
      bo_impose_dirichlet(G, l, rhs, x);
      free(r);
    } else {
      const double lam = bo_hier_lambda(h, l);
      chebyshev(h, rhs, x, l, order, lo * lam, hi * lam);
    }
  }
  return 0;
}

/* cg :84-131 */
int bo_cg(bo_hier* h, int l, double tol, int maxit, const double* rhs, double* x, double* hist, int* iters) {
  const bo_grid* G = h->G;
  const int64_t n = bo_space_size(G, 0, l);
  double* r = calloc((size_t)n, sizeof(double));
  double* p = calloc((size_t)n, sizeof(double));
  double* ap = calloc((size_t)n, sizeof(double));
  int rc = 0;
  bo_hier_apply(h, l, 1, x, r);
  vscale(r, n, -1.0);
  vaxpy(r, 1.0, rhs, n);
  vcopy(r, p, n);
  const double nb = norm2(G, l, rhs);
  const double denom = nb > 0 ? nb : 1.0;
  double rs = bo_dot(G, 0, l, r, r);
  *iters = 0;
  if (sqrt(rs) / denom <= tol) goto done;
  for (int it = 1; it <= maxit; ++it) {
    bo_hier_apply(h, l, 1, p, ap);
    const double pap = bo_dot(G, 0, l, p, ap);
    if (!(pap > 0)) { rc = fail("cg breakdown: operator is not positive definite"); goto done; }
    const double alpha = rs / pap;
    vaxpy(x, alpha, p, n);
    vaxpy(r, -alpha, ap, n);
    const double rs_new = bo_dot(G, 0, l, r, r);
    *iters = it;
    if (hist) hist[it - 1] = sqrt(rs_new) / denom;
    if (sqrt(rs_new) / denom <= tol) break;
    vscale(p, n, rs_new / rs);
    vaxpy(p, 1.0, r, n);
    rs = rs_new;
  }
done:
  free(r); free(p); free(ap);
  return rc;
}

/* v_cycle :509-541 */
static int v_cycle(bo_hier* h, int l, const double* rhs, double* x, const double* sm, int coarse_level,
                   double coarse_tol, int coarse_maxit) {
  const bo_grid* G = h->G;
  if (coarse_level < G->lo || l < coarse_level) return fail("v_cycle: level range invalid");
  if (l == coarse_level) {
    int it;
    return bo_cg(h, l, coarse_tol, coarse_maxit, rhs, x, NULL, &it);
  }
  const int64_t n = bo_space_size(G, 0, l), nc = bo_space_size(G, 0, l - 1);
  if (bo_smooth(h, sm, l, (int)sm[5], 0, rhs, x)) return 1;
  double* r = calloc((size_t)n, sizeof(double));
  bo_hier_apply(h, l, 1, x, r);
  vscale(r, n, -1.0);
  vaxpy(r, 1.0, rhs, n);
  double* rc = calloc((size_t)nc, sizeof(double));
  bo_restrict(G, l, r, rc);
  bo_zero_dirichlet(G, l - 1, rc);
  double* ec = calloc((size_t)nc, sizeof(double));
  int err = v_cycle(h, l - 1, rc, ec, sm, coarse_level, coarse_tol, coarse_maxit);
  if (!err) {
    double* ef = calloc((size_t)n, sizeof(double));
    bo_prolongate(G, l, ec, ef);
    vaxpy(x, 1.0, ef, n);
    free(ef);
    err = bo_smooth(h, sm, l, (int)sm[6], 1, rhs, x);
  }
  free(r); free(rc); free(ec);
  return err;
}

int bo_vcycles(bo_hier* h, int l, const double* sm, int coarse_level, double coarse_tol, int coarse_maxit,
               int cycles, const double* rhs, double* x, double* hist) {
  const bo_grid* G = h->G;
  const int64_t n = bo_space_size(G, 0, l);
  double* r = calloc((size_t)n, sizeof(double));
  const double nb = norm2(G, l, rhs);
  const double den = nb > 0 ? nb : 1.0;
#define RESID()                        \
  (bo_hier_apply(h, l, 1, x, r), vscale(r, n, -1.0), vaxpy(r, 1.0, rhs, n), norm2(G, l, r) / den)
  hist[0] = RESID();
  for (int c = 1; c <= cycles; ++c) {
    if (v_cycle(h, l, rhs, x, sm, coarse_level, coarse_tol, coarse_maxit)) { free(r); return 1; }
    hist[c] = RESID();
  }
#undef RESID
  free(r);
  return 0;
}

/* ---- flat exports for the python test harness ------------------------- */
int64_t bo_group_count(const bo_grid* G, int l, int64_t* members) {
  const bo_level* L = bo_grid_level(G, l);
  *members = L->nmembers;
  return L->ngroups;
}

void bo_groups(const bo_grid* G, int l, int64_t* off, int32_t* cell, int32_t* g, int64_t* t) {
  const bo_level* L = bo_grid_level(G, l);
  memcpy(off, L->goff, sizeof(int64_t) * (size_t)(L->ngroups + 1));
  memcpy(cell, L->mcell, sizeof(int32_t) * (size_t)L->nmembers);
  memcpy(g, L->mg, sizeof(int32_t) * (size_t)L->nmembers);
  memcpy(t, L->mt, sizeof(int64_t) * (size_t)L->nmembers);
}

int bo_masks(const bo_grid* G, int l, int cell, int g, uint8_t* owned, uint8_t* dir) {
  if (g > 7 || (g > 0 && !G->with_edges)) return fail("masks: subgroup not built");
  const int64_t n = slots_of(g, l);
  memcpy(owned, owned_mask(G, l, cell, g), (size_t)n);
  memcpy(dir, dir_mask(G, l, cell, g), (size_t)n);
  return 0;
}

int bo_mesh_cells(const bo_grid* G, int* cells, double* maps, char* bflags) {
  memcpy(cells, G->mesh.cells, sizeof(int) * 4 * (size_t)G->mesh.nc);
  if (maps) memcpy(maps, G->mesh.maps, sizeof(double) * 12 * (size_t)G->mesh.nc);
  if (bflags) memcpy(bflags, G->mesh.bflags, (size_t)G->mesh.nf);
  return G->mesh.nc;
}
int bo_grid_ncells(const bo_grid* G) { return G->mesh.nc; }
