// Host side of blocktet_b200: mesh ingestion, the implicit macro-interface
// tables, element matrices and stencil setup, and the host-only C ABI entry
// points. Setup work only; every per-apply operation runs on the device
// (bt_kernels.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <random>
#include <sstream>

#include "bt_internal.hpp"

#include <nvtx3/nvToolsExt.h>

namespace bt {

bool nvtx_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("BT_NVTX");
    return e && std::atoi(e) != 0;
  }();
  return on;
}
void nvtx_push(const char* name) { nvtxRangePushA(name); }
void nvtx_pop() { nvtxRangePop(); }


static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
std::atomic<uint64_t> g_launches{0};

void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) raise(BT_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// Mesh text format (coarse_mesh.hpp:217-308)
// ---------------------------------------------------------------------------
namespace {

struct LineReader {
  std::istringstream in;
  int lineno = 0;
  std::string raw;
  explicit LineReader(const std::string& t) : in(t) {}
  bool next(std::istringstream& out) {
    while (std::getline(in, raw)) {
      ++lineno;
      const auto h = raw.find('#');
      if (h != std::string::npos) raw.erase(h);
      if (raw.find_first_not_of(" \t\r\n") == std::string::npos) continue;
      out = std::istringstream(raw);
      return true;
    }
    return false;
  }
  [[noreturn]] void fail(const std::string& m) const {
    raise(BT_INVALID_ARGUMENT, "line " + std::to_string(lineno) + ": " + m);
  }
};

double signed_volume6(const Mesh& m, const std::array<int, 4>& c) {
  const auto& v0 = m.coords[c[0]];
  double u[3], w[3], z[3];
  for (int i = 0; i < 3; ++i) {
    u[i] = m.coords[c[1]][i] - v0[i];
    w[i] = m.coords[c[2]][i] - v0[i];
    z[i] = m.coords[c[3]][i] - v0[i];
  }
  const double cx = w[1] * z[2] - w[2] * z[1];
  const double cy = w[2] * z[0] - w[0] * z[2];
  const double cz = w[0] * z[1] - w[1] * z[0];
  return u[0] * cx + u[1] * cy + u[2] * cz;
}

}  // namespace

Mesh parse_mesh(const std::string& text) {
  LineReader rd(text);
  std::istringstream line;
  auto section = [&](const char* name, bool required) -> long long {
    if (!rd.next(line)) {
      if (required) rd.fail(std::string("expected '") + name + "' section");
      return -1;
    }
    std::string word;
    long long count = -1;
    const bool ok = static_cast<bool>(line >> word >> count);
    if (!required && (!ok || word != name)) rd.fail("trailing content after mesh data");
    if (!ok || word != name || count < 0) rd.fail(std::string("expected '") + name + " <count>'");
    return count;
  };
  Mesh m;
  const long long nv = section("vertices", true);
  for (long long i = 0; i < nv; ++i) {
    if (!rd.next(line)) rd.fail("unexpected end of vertex list");
    std::array<double, 3> v{};
    if (!(line >> v[0] >> v[1] >> v[2])) rd.fail("expected three vertex coordinates");
    m.coords.push_back(v);
  }
  const long long nc = section("cells", true);
  for (long long i = 0; i < nc; ++i) {
    if (!rd.next(line)) rd.fail("unexpected end of cell list");
    std::array<int, 4> c{};
    if (!(line >> c[0] >> c[1] >> c[2] >> c[3])) rd.fail("expected four vertex ids");
    for (int id : c)
      if (id < 0 || id >= (int)m.coords.size()) rd.fail("vertex id " + std::to_string(id) + " out of range");
    m.cells.push_back(c);
  }
  if (m.cells.empty()) rd.fail("mesh has no cells");
  const long long nb = section("boundary", false);

  // orientation repair (coarse_mesh.hpp:196-206)
  for (size_t ci = 0; ci < m.cells.size(); ++ci) {
    double vol = signed_volume6(m, m.cells[ci]);
    if (vol < 0) {
      std::swap(m.cells[ci][2], m.cells[ci][3]);
      vol = -vol;
      ++m.warnings;
    }
    if (vol == 0.0 || !std::isfinite(vol))
      raise(BT_INVALID_ARGUMENT, "cell " + std::to_string(ci) + " is degenerate");
  }
  // derived faces / edges, sorted (coarse_mesh.hpp:165-193)
  std::map<std::array<int, 3>, std::vector<int>> face_use;
  std::map<std::array<int, 2>, int> edge_use;
  for (int ci = 0; ci < (int)m.cells.size(); ++ci) {
    std::array<int, 4> v = m.cells[ci];
    std::sort(v.begin(), v.end());
    if (std::unique(v.begin(), v.end()) != v.end())
      raise(BT_INVALID_ARGUMENT, "cell " + std::to_string(ci) + " repeats a vertex");
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) {
        ++edge_use[{v[a], v[b]}];
        for (int c = b + 1; c < 4; ++c) {
          auto& use = face_use[{v[a], v[b], v[c]}];
          use.push_back(ci);
          if (use.size() > 2) raise(BT_INVALID_ARGUMENT, "non-conforming mesh: face shared by >2 cells");
        }
      }
  }
  for (const auto& [e, n] : edge_use) m.edges.push_back(e);
  for (const auto& [f, use] : face_use) {
    m.faces.push_back(f);
    m.face_cells.push_back({use[0], use.size() == 2 ? use[1] : -1});
    m.bflags.push_back(use.size() == 1 ? 1 : 0);
  }
  for (long long i = 0; i < nb; ++i) {
    if (!rd.next(line)) rd.fail("unexpected end of boundary list");
    std::array<int, 3> f{};
    int flag = 0;
    if (!(line >> f[0] >> f[1] >> f[2] >> flag)) rd.fail("expected three vertex ids and a flag");
    std::sort(f.begin(), f.end());
    auto it = std::lower_bound(m.faces.begin(), m.faces.end(), f);
    if (it == m.faces.end() || *it != f) rd.fail("boundary line names a non-existent face");
    const size_t fi = it - m.faces.begin();
    if (m.face_cells[fi][1] >= 0) rd.fail("boundary line names an interior face");
    m.bflags[fi] = flag != 0 ? 1 : 0;
  }
  if (rd.next(line)) rd.fail("trailing content after mesh data");
  return m;
}

// ---------------------------------------------------------------------------
// Implicit interface tables
// ---------------------------------------------------------------------------
static int face_of(const Mesh& m, std::array<int, 3> f) {
  std::sort(f.begin(), f.end());
  auto it = std::lower_bound(m.faces.begin(), m.faces.end(), f);
  return (int)(it - m.faces.begin());
}
static int edge_of(const Mesh& m, std::array<int, 2> e) {
  if (e[0] > e[1]) std::swap(e[0], e[1]);
  auto it = std::lower_bound(m.edges.begin(), m.edges.end(), e);
  return (int)(it - m.edges.begin());
}

void build_topology(const Mesh& m, Topology& t) {
  const int nc = m.n_cells(), nv = (int)m.coords.size();
  const int ne = (int)m.edges.size(), nf = (int)m.faces.size();
  t.edge_cells.assign(ne, {});
  t.vert_cells.assign(nv, {});
  t.cell_faces.resize(nc);
  t.cell_edges.resize(nc);
  t.maps.resize(nc);
  for (int c = 0; c < nc; ++c) {
    const auto& v = m.cells[c];
    for (int a = 0; a < 4; ++a) t.vert_cells[v[a]].push_back(c);
    t.cell_faces[c] = {face_of(m, {v[1], v[2], v[3]}), face_of(m, {v[0], v[2], v[3]}),
                       face_of(m, {v[0], v[1], v[3]}), face_of(m, {v[0], v[1], v[2]})};
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) {
        const int e = edge_of(m, {v[a], v[b]});
        t.cell_edges[c][local_edge(a, b)] = e;
        t.edge_cells[e].push_back(c);
      }
    // macro_cell_map (coarse_mesh.hpp:92-105)
    CellMap& mp = t.maps[c];
    for (int r = 0; r < 3; ++r)
      for (int col = 0; col < 3; ++col) mp.a[3 * r + col] = m.coords[v[col + 1]][r] - m.coords[v[0]][r];
    for (int r = 0; r < 3; ++r) mp.b[r] = m.coords[v[0]][r];
  }
  // Dirichlet flags of edges / vertices: any constrained face contains them
  // (the OR over group members of fe_function.hpp:209-216).
  t.edge_dir.assign(ne, 0);
  t.vert_dir.assign(nv, 0);
  for (int f = 0; f < nf; ++f) {
    if (!m.bflags[f]) continue;
    const auto& fv = m.faces[f];
    for (int q = 0; q < 3; ++q) t.vert_dir[fv[q]] = 1;
    t.edge_dir[edge_of(m, {fv[0], fv[1]})] = 1;
    t.edge_dir[edge_of(m, {fv[0], fv[2]})] = 1;
    t.edge_dir[edge_of(m, {fv[1], fv[2]})] = 1;
  }
  // per-cell owned / Dirichlet bits by zero set
  t.info.resize(nc);
  for (int c = 0; c < nc; ++c) {
    uint16_t own = 1, dir = 0;  // Z = 0: cell interior
    for (int z = 1; z < 15; ++z) {
      const int pc = __builtin_popcount(z);
      bool o = false, d = false;
      if (pc == 1) {
        const int v = __builtin_ctz(z);
        const int f = t.cell_faces[c][v];
        o = m.face_cells[f][0] == c;
        d = m.bflags[f] != 0;
      } else if (pc == 2) {
        const int nz = ~z & 15;
        const int a = __builtin_ctz(nz), b = 31 - __builtin_clz(nz);
        const int e = t.cell_edges[c][local_edge(a, b)];
        o = t.edge_cells[e][0] == c;
        d = t.edge_dir[e] != 0;
      } else {
        const int u = __builtin_ctz(~z & 15);
        const int gv = m.cells[c][u];
        o = t.vert_cells[gv][0] == c;
        d = t.vert_dir[gv] != 0;
      }
      if (o) own |= (uint16_t)(1u << z);
      if (d) dir |= (uint16_t)(1u << z);
    }
    t.info[c] = {own, dir};
  }
  auto local_of = [&](int c, int gv) -> int8_t {
    for (int a = 0; a < 4; ++a)
      if (m.cells[c][a] == gv) return (int8_t)a;
    raise(BT_LOGIC_ERROR, "interface table: vertex not in cell");
  };
  t.faces.resize(nf);
  for (int f = 0; f < nf; ++f) {
    DevFace& r = t.faces[f];
    r.ncell = m.face_cells[f][1] >= 0 ? 2 : 1;
    r.dir = (uint8_t)m.bflags[f];
    for (int s = 0; s < 2; ++s) {
      r.cell[s] = m.face_cells[f][s];
      for (int q = 0; q < 3; ++q) r.lv[s][q] = s < r.ncell ? local_of(r.cell[s], m.faces[f][q]) : (int8_t)-1;
    }
  }
  t.ehdr.resize(ne);
  t.emem.clear();
  for (int e = 0; e < ne; ++e) {
    t.ehdr[e] = {(int)t.emem.size(), (int)t.edge_cells[e].size(), (uint8_t)t.edge_dir[e]};
    for (int c : t.edge_cells[e]) t.emem.push_back({c, {local_of(c, m.edges[e][0]), local_of(c, m.edges[e][1])}});
  }
  t.vhdr.resize(nv);
  t.vmem.clear();
  for (int v = 0; v < nv; ++v) {
    t.vhdr[v] = {(int)t.vmem.size(), (int)t.vert_cells[v].size(), (uint8_t)t.vert_dir[v]};
    for (int c : t.vert_cells[v]) t.vmem.push_back({c, {local_of(c, v), -1}});
  }
}

int64_t part_shift(const bt_grid& g, int space, int level) {
  return g.part_nranks > 1 ? level_slots(space, level) * g.part_begin : 0;
}

int64_t level_slots(int space, int level) {
  int64_t s = 0;
  if (space == BT_SPACE_P1 || space == BT_SPACE_P2) s += n_tet(width_formula(0, level));
  if (space == BT_SPACE_P2 || space == BT_SPACE_EDGES)
    for (int g = 1; g <= 7; ++g) s += n_tet(width_formula(g, level));
  return s;
}

void check_level(const bt_grid* g, int level) {
  if (!g) raise(BT_INVALID_ARGUMENT, "grid required");
  if (level < g->lo || level > g->hi) raise(BT_OUT_OF_RANGE, "level not covered by grid");
}

void validate_form(const bt_form* f) {
  if (!f) raise(BT_INVALID_ARGUMENT, "form required");
  if (f->kind < 0 || f->kind > 2) raise(BT_INVALID_ARGUMENT, "unknown form kind");
  if (f->kind == BT_FORM_DIV_K_GRAD && (f->coeff_kind < 0 || f->coeff_kind > 2))
    raise(BT_INVALID_ARGUMENT, "div_k_grad needs a coefficient");
}

// ---------------------------------------------------------------------------
// Element matrices (forms.hpp:75-120), class matrices (operators.hpp:54-69)
// ---------------------------------------------------------------------------
static const int kOffCell[6][4][3] = BT_CELL_OFFSETS;
static const int kDirs[15][3] = BT_STENCIL_DIRS;

static void local_matrix_const(int form_kind, const double x[4][3], double out[16]) {
  double a[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a[3 * r + c] = x[c + 1][r] - x[0][r];
  const double det = a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
                     a[2] * (a[3] * a[7] - a[4] * a[6]);
  if (det == 0.0 || !std::isfinite(det)) raise(BT_INVALID_ARGUMENT, "local_matrix: degenerate element");
  const double vol = std::abs(det) / 6.0;
  if (form_kind == BT_FORM_MASS) {
    for (int k = 0; k < 4; ++k)
      for (int l = 0; l < 4; ++l) out[4 * k + l] = vol / 20.0 * (k == l ? 2.0 : 1.0);
    return;
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
    grad[i][0] = inv[0] * rg[i][0] + inv[3] * rg[i][1] + inv[6] * rg[i][2];
    grad[i][1] = inv[1] * rg[i][0] + inv[4] * rg[i][1] + inv[7] * rg[i][2];
    grad[i][2] = inv[2] * rg[i][0] + inv[5] * rg[i][1] + inv[8] * rg[i][2];
  }
  for (int k = 0; k < 4; ++k)
    for (int l = 0; l < 4; ++l)
      out[4 * k + l] = vol * (grad[k][0] * grad[l][0] + grad[k][1] * grad[l][1] + grad[k][2] * grad[l][2]);
}

static void map_point(const CellMap& mp, int level, int i, int j, int k, double out[3]) {
  const double h = 1.0 / (double)(1 << level);
  const double r[3] = {h * i, h * j, h * k};
  for (int d = 0; d < 3; ++d) out[d] = (mp.a[3 * d] * r[0] + mp.a[3 * d + 1] * r[1] + mp.a[3 * d + 2] * r[2]) + mp.b[d];
}

void class_matrices(const bt_grid& g, int form_kind, int level, int cell, double out[6][16]) {
  for (int s = 0; s < 6; ++s) {
    double x[4][3];
    for (int i = 0; i < 4; ++i)
      map_point(g.topo.maps[cell], level, kOffCell[s][i][0], kOffCell[s][i][1], kOffCell[s][i][2], x[i]);
    local_matrix_const(form_kind, x, out[s]);
  }
}

static int dir_index(int dx, int dy, int dz) {
  for (int i = 0; i < 15; ++i)
    if (kDirs[i][0] == dx && kDirs[i][1] == dy && kDirs[i][2] == dz) return i;
  raise(BT_LOGIC_ERROR, "not a stencil direction");
}

// Is micro-cell (class s) with vertex `slot` at a lattice point of zero set z
// present? Anchor p - o must lie in I_tet(w_s): components need p_e >= o_e
// and the sum condition fails exactly when the point is on the diagonal face
// (weight 0 == 0) and |o| <= n - w_s (verified in tests).
static bool tet_present(int s, int slot, int z) {
  static const int deficit[6] = {0, 2, 1, 1, 1, 1};  // n - w_s
  const int* o = kOffCell[s][slot];
  for (int e = 0; e < 3; ++e)
    if (o[e] == 1 && (z >> (e + 1) & 1)) return false;
  if ((z & 1) && o[0] + o[1] + o[2] < deficit[s] + 1) return false;
  return true;
}

void build_stencil_cells(const bt_grid& g, const bt_form& f, int level, std::vector<StencilCell>& cells,
                         std::vector<std::array<double, 15>>& rows) {
  const int nc = g.mesh.n_cells();
  cells.assign(nc, StencilCell{});
  rows.assign(nc, {});
  for (int c = 0; c < nc; ++c) {
    double cls[6][16];
    class_matrices(g, f.kind, level, c, cls);
    StencilCell& sc = cells[c];
    std::memset(&sc, 0, sizeof sc);
    for (int z = 0; z < 16; ++z) {
      if (z == 15) continue;
      int combos = 0;
      for (int s = 0; s < 6; ++s)
        for (int slot = 0; slot < 4; ++slot) {
          if (!tet_present(s, slot, z)) continue;
          ++combos;
          for (int j = 0; j < 4; ++j) {
            const int d = dir_index(kOffCell[s][j][0] - kOffCell[s][slot][0], kOffCell[s][j][1] - kOffCell[s][slot][1],
                                    kOffCell[s][j][2] - kOffCell[s][slot][2]);
            sc.w[z][d] += cls[s][4 * slot + j];
            sc.mask[z] |= 1u << d;
          }
        }
      if (z == 0 && combos != 24) raise(BT_LOGIC_ERROR, "interior probe must touch 24 micro-cells");
    }
    for (int d = 0; d < 15; ++d) rows[c][d] = sc.w[0][d];
  }
}

// Zero-set-typed partial diagonal (compute_stencil operators.hpp:224-238).
static void typed_diag(const double cls[6][16], double out[16]) {
  for (int z = 0; z < 16; ++z) {
    double d = 0;
    if (z != 15)
      for (int s = 0; s < 6; ++s)
        for (int slot = 0; slot < 4; ++slot)
          if (tet_present(s, slot, z)) d += cls[s][5 * slot];
    out[z] = d;
  }
}

void build_ew_cells(const bt_grid& g, const bt_form& f, int level, std::vector<EwCell>& cells) {
  const int nc = g.mesh.n_cells();
  cells.assign(nc, EwCell{});
  const bool var = f.kind == BT_FORM_DIV_K_GRAD;
  const int ck = var ? f.coeff_kind : 0;
  const double h = 1.0 / (double)(1 << level);
  const double qa = (5.0 + 3.0 * std::sqrt(5.0)) / 20.0;  // forms.hpp:56-61
  const double qb = (5.0 - std::sqrt(5.0)) / 20.0;
  for (int c = 0; c < nc; ++c) {
    EwCell& e = cells[c];
    class_matrices(g, var ? BT_FORM_DIFFUSION : f.kind, level, c, e.G);
    const CellMap& mp = g.topo.maps[c];
    for (int d = 0; d < 3; ++d)
      for (int q = 0; q < 3; ++q) e.beta[d][q] = (ck == 1 ? f.c[2] : 0.0) * mp.a[3 * d + q] * h;
    if (ck == 2) {
      // k affine: kbar = k(centroid) = c0 + c . (A h (p + centroid_s) + b)
      for (int q = 0; q < 3; ++q) {
        e.lin[q] = 0;
        for (int d = 0; d < 3; ++d) e.lin[q] += f.c[1 + d] * mp.a[3 * d + q] * h;
      }
      for (int s = 0; s < 6; ++s) {
        double r[3];
        for (int q = 0; q < 3; ++q) {
          double mean = 0;
          for (int i = 0; i < 4; ++i) mean += kOffCell[s][i][q];
          r[q] = 0.25 * mean;
        }
        double v = f.c[0];
        for (int d = 0; d < 3; ++d) {
          double x = mp.b[d];
          for (int q = 0; q < 3; ++q) x += mp.a[3 * d + q] * h * r[q];
          v += f.c[1 + d] * x;
        }
        e.lin0[s] = v;
      }
    }
    if (ck == 1) {
      // phase of quadrature point q of class s relative to its anchor p:
      // gamma_{s,q,d} = f (A h delta_{s,q} + b)_d; the monomial coefficients
      // coefh[s][m] = c1/4 sum_q prod_d (bit d of m ? sin : cos)(gamma_{s,q,d})
      const double fr = f.c[2];
      for (int s = 0; s < 6; ++s) {
        double sg[4][3], cg[4][3];
        for (int q = 0; q < 4; ++q) {
          double r[3];
          for (int a = 0; a < 3; ++a) {
            double dl = 0;
            for (int i = 0; i < 4; ++i) dl += (i == q ? qa : qb) * kOffCell[s][i][a];
            r[a] = dl;
          }
          for (int d = 0; d < 3; ++d) {
            double x = mp.b[d];
            for (int a = 0; a < 3; ++a) x += mp.a[3 * d + a] * h * r[a];
            sg[q][d] = std::sin(fr * x);
            cg[q][d] = std::cos(fr * x);
          }
        }
        for (int m = 0; m < 8; ++m) {
          double acc = 0;
          for (int q = 0; q < 4; ++q) {
            double p = 1;
            for (int d = 0; d < 3; ++d) p *= (m >> d & 1) ? sg[q][d] : cg[q][d];
            acc += p;
          }
          e.coefh[s][m] = 0.25 * f.c[1] * acc;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Builder mesh generator, shared with oracle/bt_oracle.c
// ---------------------------------------------------------------------------
// nx x ny x nz cubes of side h, each split into 6 Kuhn tets (positive
// orientation); vertices not on the box boundary perturbed per component by
// U(-perturb h, perturb h) from mt19937_64(seed) in vertex order.
static std::string box_text(int nx, int ny, int nz, double h, double perturb, uint64_t seed, const char* header,
                            int bx = 0, int by = 0, int bz = 0) {
  const int vx = nx + 1, vy = ny + 1, vz = nz + 1, nverts = vx * vy * vz;
  const int dims[3] = {nx, ny, nz};
  std::vector<double> xyz(3 * (size_t)nverts);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-perturb * h, perturb * h);
  for (int c = 0; c <= nz; ++c)
    for (int b = 0; b <= ny; ++b)
      for (int a = 0; a <= nx; ++a) {
        const int id = a + vx * (b + vy * c);
        const int idx[3] = {a, b, c};
        for (int d = 0; d < 3; ++d) {
          const double off = dist(rng);
          const bool on_bdry = idx[d] == 0 || idx[d] == dims[d];
          xyz[3 * id + d] = idx[d] * h + (perturb > 0 && !on_bdry ? off : 0.0);
        }
      }
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  std::string out = header;
  char tmp[256];
  snprintf(tmp, sizeof tmp, "vertices %d\n", nverts);
  out += tmp;
  for (int i = 0; i < nverts; ++i) {
    snprintf(tmp, sizeof tmp, "%.17g %.17g %.17g\n", xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    out += tmp;
  }
  snprintf(tmp, sizeof tmp, "cells %d\n", 6 * nx * ny * nz);
  out += tmp;
  auto vid = [&](int a, int b, int c, int bits) {
    return (a + (bits & 1)) + vx * ((b + ((bits >> 1) & 1)) + vy * (c + ((bits >> 2) & 1)));
  };
  // cubes in cube order (a fastest), or block-major with blocks of bx x by x bz
  // cubes (blocks in block order, cubes inside a block in cube order), so that
  // contiguous cell ranges (bt_grid_set_partition) are compact blocks
  if (bx <= 0) bx = nx;
  if (by <= 0) by = ny;
  if (bz <= 0) bz = nz;
  std::vector<std::array<int, 3>> order;
  for (int BZ = 0; BZ < nz; BZ += bz)
    for (int BY = 0; BY < ny; BY += by)
      for (int BX = 0; BX < nx; BX += bx)
        for (int c = BZ; c < std::min(nz, BZ + bz); ++c)
          for (int b = BY; b < std::min(ny, BY + by); ++b)
            for (int a = BX; a < std::min(nx, BX + bx); ++a) order.push_back({a, b, c});
  for (const auto& abc : order)
    for (const auto& pm : perms) {
      const int a = abc[0], b = abc[1], c = abc[2];
      {
          int loc[4] = {0, 0, 0, 7};
          loc[1] = 1 << pm[0];
          loc[2] = loc[1] | (1 << pm[1]);
          double cc[4][3];
          for (int k = 0; k < 4; ++k)
            for (int d = 0; d < 3; ++d) cc[k][d] = (double)((loc[k] >> d) & 1);
          double u[3], w[3], z[3];
          for (int d = 0; d < 3; ++d) {
            u[d] = cc[1][d] - cc[0][d];
            w[d] = cc[2][d] - cc[0][d];
            z[d] = cc[3][d] - cc[0][d];
          }
          const double vol = u[0] * (w[1] * z[2] - w[2] * z[1]) + u[1] * (w[2] * z[0] - w[0] * z[2]) +
                             u[2] * (w[0] * z[1] - w[1] * z[0]);
          if (vol < 0) std::swap(loc[2], loc[3]);
          snprintf(tmp, sizeof tmp, "%d %d %d %d\n", vid(a, b, c, loc[0]), vid(a, b, c, loc[1]), vid(a, b, c, loc[2]),
                   vid(a, b, c, loc[3]));
          out += tmp;
        }
    }
  return out;
}

std::string cubes_mesh_text(int n, double perturb, uint64_t seed) {
  char header[256];
  snprintf(header, sizeof header, "# %d^3 unit cubes x 6 Kuhn tets, perturb %.17g, seed %llu\n", n, perturb,
           (unsigned long long)seed);
  return box_text(n, n, n, 1.0 / n, perturb, seed, header);
}

std::string box_mesh_text(int nx, int ny, int nz, double perturb, uint64_t seed) {
  char header[256];
  snprintf(header, sizeof header, "# %dx%dx%d unit cubes x 6 Kuhn tets, perturb %.17g, seed %llu\n", nx, ny, nz,
           perturb, (unsigned long long)seed);
  return box_text(nx, ny, nz, 1.0, perturb, seed, header);
}

// nx x ny x nz cubes of side h, cubes numbered block-major (blocks of
// bx x by x bz cubes): the multi-GPU workloads, whose contiguous cell ranges
// are then compact blocks
std::string blocked_mesh_text(int nx, int ny, int nz, int bx, int by, int bz, double h, double perturb,
                              uint64_t seed) {
  char header[256];
  snprintf(header, sizeof header,
           "# %dx%dx%d cubes of side %.17g x 6 Kuhn tets, blocks %dx%dx%d, perturb %.17g, seed %llu\n", nx, ny, nz, h,
           bx, by, bz, perturb, (unsigned long long)seed);
  return box_text(nx, ny, nz, h, perturb, seed, header, bx, by, bz);
}

// Elementwise tables are cached on the grid per (form, level): a repeated
// apply_elementwise launches kernels only.
const EwTables& ew_tables(const bt_grid& g, const bt_form& f, int level) {
  auto same = [&](const EwTables& t) {
    if (t.level != level || t.form.kind != f.kind) return false;
    if (f.kind != BT_FORM_DIV_K_GRAD) return true;
    if (t.form.coeff_kind != f.coeff_kind) return false;
    for (int q = 0; q < 4; ++q)
      if (t.form.c[q] != f.c[q]) return false;
    return true;
  };
  for (const auto& t : g.ew_cache)
    if (same(*t)) return *t;
  auto t = std::make_unique<EwTables>();
  t->form = f;
  t->level = level;
  check_coefficient(g, f, level, cell_maps(g), 0);
  std::vector<EwCell> cells;
  build_ew_cells(g, f, level, cells);
  t->cells.upload(cells);
  t->host = cells;
  if (f.kind == BT_FORM_DIV_K_GRAD && f.coeff_kind == 1) build_ew_phase(g, level, t->cells.p, t->phase);
  if (g.ew_cache.size() >= 16) g.ew_cache.erase(g.ew_cache.begin());
  g.ew_cache.push_back(std::move(t));
  return *g.ew_cache.back();
}

// Zero set of an edge micro-primitive = intersection of its endpoints' sets.
static int prim_zero_set(int g, int n, int i, int j, int k) {
  static const int kOffEdge[7][2][3] = BT_EDGE_OFFSETS;
  if (g == 0) return zero_set(n, i, j, k);
  const int* a = kOffEdge[g - 1][0];
  const int* b = kOffEdge[g - 1][1];
  return zero_set(n, i + a[0], j + a[1], k + a[2]) & zero_set(n, i + b[0], j + b[1], k + b[2]);
}

}  // namespace bt

// ===========================================================================
// C ABI (host-side entry points)
// ===========================================================================
using namespace bt;


bt_grid::~bt_grid() {
  if (h_pinned) cudaFreeHost(h_pinned);
}

// Interface work lists of the groups whose members all lie in cells
// [begin, end) (every group when the range covers the mesh).
static void interface_lists(const bt_grid& g, int begin, int end, IfaceLists& L) {
  auto in = [&](int c) { return c >= begin && c < end; };
  L.face_shared.clear();
  L.face_bdir.clear();
  L.edge_act.clear();
  L.vert_act.clear();
  for (int f = 0; f < (int)g.topo.faces.size(); ++f) {
    const DevFace& F = g.topo.faces[f];
    if (F.ncell == 2) {
      if (in(F.cell[0]) && in(F.cell[1])) L.face_shared.push_back(f);
    } else if (F.dir && in(F.cell[0])) {
      L.face_bdir.push_back(f);
    }
  }
  auto all_in = [&](const DevPrimHdr& h, const std::vector<DevPrimMem>& mem) {
    for (int m = 0; m < h.count; ++m)
      if (!in(mem[h.first + m].cell)) return false;
    return true;
  };
  for (int e = 0; e < (int)g.topo.ehdr.size(); ++e) {
    const DevPrimHdr& h = g.topo.ehdr[e];
    if ((h.count >= 2 || h.dir) && all_in(h, g.topo.emem)) L.edge_act.push_back(e);
  }
  for (int v = 0; v < (int)g.topo.vhdr.size(); ++v) {
    const DevPrimHdr& h = g.topo.vhdr[v];
    if ((h.count >= 2 || h.dir) && all_in(h, g.topo.vmem)) L.vert_act.push_back(v);
  }
  L.upload();
}

void bt::require_unpartitioned(const bt_grid* g, const char* what) {
  if (g && g->part_nranks > 1)
    raise(BT_LOGIC_ERROR, std::string(what) +
                              ": not available on a partitioned grid (rank-spanning groups need the exchange; see "
                              "bt_xchg_pack / bt_xchg_finish)");
}

void bt::partition_range(int nc, int rank, int nranks, int& begin, int& end) {
  begin = (int)((int64_t)nc * rank / nranks);
  end = (int)((int64_t)nc * (rank + 1) / nranks);
}

extern "C" {

const char* bt_last_error(void) { return bt::g_err.c_str(); }
const char* bt_version(void) { return "blocktet_b200 0.1 (sm_100a)"; }
uint64_t bt_launch_count(void) { return bt::g_launches; }

int64_t bt_n_tri(int64_t w) { return n_tri(w); }
int64_t bt_n_tet(int64_t w) { return n_tet(w); }
int bt_width_formula(int g, int level) { return width_formula(g, level); }
bt_status bt_width(int g, int level, int* out) {
  BT_TRY
  if (level < 0) raise(BT_INVALID_ARGUMENT, "width: negative level");
  if (g < 0 || g > 25) raise(BT_INVALID_ARGUMENT, "width: unknown subgroup");
  const int w = width_formula(g, level);
  if (w <= 0)
    raise(BT_DOMAIN_ERROR, "width: subgroup " + std::to_string(g) + " has no instances on level " +
                               std::to_string(level));
  *out = w;
  BT_CATCH
}
int64_t bt_linearize(int w, int i, int j, int k) { return linearize(w, i, j, k); }
bt_status bt_linearize_checked(int w, int i, int j, int k, int64_t* out) {
  BT_TRY
  if (!out) raise(BT_INVALID_ARGUMENT, "linearize: output required");
  if (!in_i_tet(w, i, j, k)) raise(BT_OUT_OF_RANGE, "linearize: index outside I_tet(w)");
  *out = linearize(w, i, j, k);
  BT_CATCH
}
bt_status bt_linearize_aos(int w, int m, int i, int j, int k, int d, int64_t* out) {
  BT_TRY
  if (!out) raise(BT_INVALID_ARGUMENT, "linearize_aos: output required");
  if (d < 0 || d >= m) raise(BT_OUT_OF_RANGE, "linearize_aos: bad DoF index");
  if (!in_i_tet(w, i, j, k)) raise(BT_OUT_OF_RANGE, "linearize: index outside I_tet(w)");
  *out = (int64_t)m * linearize(w, i, j, k) + d;
  BT_CATCH
}
bt_status bt_linearize_soa(int w, int m, int i, int j, int k, int d, int64_t* out) {
  BT_TRY
  if (!out) raise(BT_INVALID_ARGUMENT, "linearize_soa: output required");
  if (d < 0 || d >= m) raise(BT_OUT_OF_RANGE, "linearize_soa: bad DoF index");
  if (!in_i_tet(w, i, j, k)) raise(BT_OUT_OF_RANGE, "linearize: index outside I_tet(w)");
  *out = (int64_t)d * n_tet(w) + linearize(w, i, j, k);
  BT_CATCH
}
bt_status bt_mesh_parse(const char* text, int* n_vertices, int* n_cells, double* coords, int* cells,
                        int* n_warnings) {
  BT_TRY
  if (!text) raise(BT_INVALID_ARGUMENT, "parse_mesh: text required");
  const Mesh m = parse_mesh(text);
  if (n_vertices) *n_vertices = (int)m.coords.size();
  if (n_cells) *n_cells = m.n_cells();
  if (n_warnings) *n_warnings = m.warnings;
  if (coords)
    for (size_t v = 0; v < m.coords.size(); ++v)
      for (int d = 0; d < 3; ++d) coords[3 * v + d] = m.coords[v][d];
  if (cells)
    for (int c = 0; c < m.n_cells(); ++c)
      for (int q = 0; q < 4; ++q) cells[4 * c + q] = m.cells[c][q];
  BT_CATCH
}
bt_status bt_delinearize(int w, int64_t t, int* ijk) {
  BT_TRY
  if (t < 0 || t >= n_tet(w)) raise(BT_OUT_OF_RANGE, "delinearize: offset out of range");
  // closed-form layer/row search instead of the reference's subtraction loop
  int k = 0;
  {
    int lo = 0, hi = w;  // largest k with n_tet(w) - n_tet(w - k) <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (n_tet(w) - n_tet(w - mid) <= t) lo = mid; else hi = mid - 1;
    }
    k = lo;
  }
  int64_t r = t - (n_tet(w) - n_tet(w - k));
  int j = 0;
  {
    const int m = w - k;
    int lo = 0, hi = m;
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (n_tri(m) - n_tri(m - mid) <= r) lo = mid; else hi = mid - 1;
    }
    j = lo;
    r -= n_tri(m) - n_tri(m - j);
  }
  ijk[0] = (int)r;
  ijk[1] = j;
  ijk[2] = k;
  BT_CATCH
}
int bt_subgroup_offsets(int g, int* out) {
  static const int kOffFace[12][3][3] = {
      {{0, 0, 0}, {0, 1, 0}, {1, 0, 0}}, {{0, 1, 0}, {1, 0, 0}, {1, 1, 0}},
      {{0, 0, 0}, {0, 0, 1}, {1, 0, 0}}, {{0, 0, 1}, {1, 0, 0}, {1, 0, 1}},
      {{0, 0, 0}, {0, 0, 1}, {0, 1, 0}}, {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}},
      {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}}, {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
      {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}}, {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}},
      {{0, 0, 1}, {0, 1, 0}, {1, 0, 1}}, {{0, 1, 0}, {1, 0, 1}, {1, 1, 0}}};
  static const int kOffEdge[7][2][3] = BT_EDGE_OFFSETS;
  if (g < 0 || g > 25) return 0;
  int n;
  const int* src;
  if (g == 0) { static const int z[3] = {0, 0, 0}; src = z; n = 1; }
  else if (g <= 7) { src = &kOffEdge[g - 1][0][0]; n = 2; }
  else if (g <= 19) { src = &kOffFace[g - 8][0][0]; n = 3; }
  else { src = &kOffCell[g - 20][0][0]; n = 4; }
  std::memcpy(out, src, sizeof(int) * 3 * n);
  return n;
}

bt_status bt_grid_create(const char* text, int lo, int hi, int device, bt_grid** out) {
  BT_TRY
  if (!text || !out) raise(BT_INVALID_ARGUMENT, "bt_grid_create: null argument");
  if (lo < 2 || hi > 10 || lo > hi) raise(BT_INVALID_ARGUMENT, "grid levels must satisfy 2 <= min <= max <= 10");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    raise(BT_CUDA_ERROR, "no CUDA device: blocktet_b200 has no CPU path");
  if (device < 0 || device >= ndev) raise(BT_INVALID_ARGUMENT, "bad device ordinal");
  BT_CUDA(cudaSetDevice(device));
  auto g = std::make_unique<bt_grid>();
  g->device = device;
  g->lo = lo;
  g->hi = hi;
  g->mesh = parse_mesh(text);
  build_topology(g->mesh, g->topo);
  g->d_faces.upload(g->topo.faces);
  g->d_ehdr.upload(g->topo.ehdr);
  g->d_emem.upload(g->topo.emem);
  g->d_vhdr.upload(g->topo.vhdr);
  g->d_vmem.upload(g->topo.vmem);
  g->d_info.upload(g->topo.info);
  g->part_end = g->mesh.n_cells();
  interface_lists(*g, 0, g->mesh.n_cells(), g->full);
  interface_lists(*g, 0, g->mesh.n_cells(), g->loc);
  BT_CUDA(cudaMallocHost(&g->h_pinned, sizeof(double) * 8));
  *out = g.release();
  BT_CATCH
}

void bt_grid_destroy(bt_grid* g) { delete g; }

bt_status bt_grid_set_partition(bt_grid* g, int rank, int nranks) {
  BT_TRY
  if (!g) raise(BT_INVALID_ARGUMENT, "bt_grid_set_partition: grid required");
  if (nranks < 1 || rank < 0 || rank >= nranks) raise(BT_INVALID_ARGUMENT, "bt_grid_set_partition: bad rank");
  BT_CUDA(cudaSetDevice(g->device));
  g->part_rank = rank;
  g->part_nranks = nranks;
  partition_range(g->mesh.n_cells(), rank, nranks, g->part_begin, g->part_end);
  interface_lists(*g, g->part_begin, g->part_end, g->loc);
  // everything derived from the previous partition: exchange plans (P1 and
  // N1E1 edges), elementwise tables, reduction and exchange scratch
  BT_CUDA(cudaDeviceSynchronize());
  for (auto& p : g->xplan) p.reset();
  for (auto& p : g->xplan_edges) p.reset();
  g->ew_cache.clear();
  g->ew_scratch.release();
  for (auto& b : g->ew_rows) b.release();
  for (auto& b : g->ew_tiles) b.release();
  for (auto& b : g->ew_rowtab) b.release();
  g->ew_nrows.fill(0);
  g->ew_ntiles.fill(0);
  g->d_partials.release();
  g->dot_cells.release();
  g->xbuf.release();
  ++g->part_epoch;
  BT_CATCH
}
int bt_num_cells(const bt_grid* g) { return g ? g->mesh.n_cells() : 0; }
int bt_grid_min_level(const bt_grid* g) { return g->lo; }
int bt_grid_max_level(const bt_grid* g) { return g->hi; }
int64_t bt_space_size(const bt_grid* g, int space, int level) {
  // a partitioned grid's vectors hold its cell block only
  return level_slots(space, level) * (g->part_end - g->part_begin);
}

int64_t bt_owned_dof_count(const bt_grid* g, int space, int level) {
  const int n = 1 << level;
  int64_t cnt = 0;
  for (int c = 0; c < g->mesh.n_cells(); ++c) {
    const uint16_t own = g->topo.info[c].owned_by_z;
    for (int gg = (space == BT_SPACE_EDGES ? 1 : 0); gg <= (space == BT_SPACE_P1 ? 0 : 7); ++gg) {
      const int w = width_formula(gg, level);
      for (int k = 0; k < w; ++k)
        for (int j = 0; j < w - k; ++j)
          for (int i = 0; i < w - k - j; ++i) cnt += (own >> prim_zero_set(gg, n, i, j, k)) & 1;
    }
  }
  return cnt;
}

bt_status bt_grid_masks(const bt_grid* g, int level, int cell, int subgroup, uint8_t* owned, uint8_t* dir) {
  BT_TRY
  check_level(g, level);
  if (subgroup < 0 || subgroup > 7) raise(BT_INVALID_ARGUMENT, "masks: vertex or edge subgroup expected");
  if (cell < 0 || cell >= g->mesh.n_cells()) raise(BT_OUT_OF_RANGE, "masks: no such cell");
  const int n = 1 << level, w = width_formula(subgroup, level);
  const DevCellInfo inf = g->topo.info[cell];
  int64_t t = 0;
  for (int k = 0; k < w; ++k)
    for (int j = 0; j < w - k; ++j)
      for (int i = 0; i < w - k - j; ++i, ++t) {
        const int z = prim_zero_set(subgroup, n, i, j, k);
        if (owned) owned[t] = (inf.owned_by_z >> z) & 1;
        if (dir) dir[t] = (inf.dir_by_z >> z) & 1;
      }
  BT_CATCH
}

// Groups of the vertex space, expanded from the implicit tables.
bt_status bt_grid_groups(const bt_grid* g, int level, int space, int64_t* n_groups, int64_t* n_members,
                         int64_t* offsets, int32_t* cell, int32_t* subgroup, int64_t* t) {
  BT_TRY
  check_level(g, level);
  if (space != BT_SPACE_P1) raise(BT_INVALID_ARGUMENT, "bt_grid_groups: P1 space only");
  const int n = 1 << level, w = n + 1;
  std::vector<std::vector<std::pair<int, int64_t>>> groups;
  auto emit = [&](const std::vector<std::pair<int, int64_t>>& mem) {
    if (mem.size() >= 2) groups.push_back(mem);
  };
  const Topology& tp = g->topo;
  for (const DevFace& f : tp.faces) {
    if (f.ncell < 2) continue;
    for (int b = 1; b <= n - 2; ++b)
      for (int a = 1; a + b <= n - 1; ++a) {
        std::vector<std::pair<int, int64_t>> mem;
        for (int s = 0; s < 2; ++s) {
          int wt[4] = {0, 0, 0, 0};
          wt[f.lv[s][0]] = n - a - b;
          wt[f.lv[s][1]] = a;
          wt[f.lv[s][2]] = b;
          mem.push_back({f.cell[s], linearize(w, wt[1], wt[2], wt[3])});
        }
        emit(mem);
      }
  }
  for (const DevPrimHdr& e : tp.ehdr) {
    if (e.count < 2) continue;
    for (int a = 1; a <= n - 1; ++a) {
      std::vector<std::pair<int, int64_t>> mem;
      for (int m = 0; m < e.count; ++m) {
        const DevPrimMem& pm = tp.emem[e.first + m];
        int wt[4] = {0, 0, 0, 0};
        wt[pm.lv[0]] = n - a;
        wt[pm.lv[1]] = a;
        mem.push_back({pm.cell, linearize(w, wt[1], wt[2], wt[3])});
      }
      emit(mem);
    }
  }
  for (const DevPrimHdr& v : tp.vhdr) {
    if (v.count < 2) continue;
    std::vector<std::pair<int, int64_t>> mem;
    for (int m = 0; m < v.count; ++m) {
      const DevPrimMem& pm = tp.vmem[v.first + m];
      int wt[4] = {0, 0, 0, 0};
      wt[pm.lv[0]] = n;
      mem.push_back({pm.cell, linearize(w, wt[1], wt[2], wt[3])});
    }
    emit(mem);
  }
  int64_t nm = 0;
  for (const auto& gr : groups) nm += (int64_t)gr.size();
  *n_groups = (int64_t)groups.size();
  *n_members = nm;
  if (offsets) {
    int64_t o = 0, k = 0;
    offsets[0] = 0;
    for (const auto& gr : groups) {
      for (const auto& [c, tt] : gr) {
        cell[o] = c;
        subgroup[o] = 0;
        t[o] = tt;
        ++o;
      }
      offsets[++k] = o;
    }
  }
  BT_CATCH
}

int64_t bt_box_mesh_text(int nx, int ny, int nz, double perturb, uint64_t seed, char* buf, int64_t buflen) {
  if (nx < 1 || ny < 1 || nz < 1) return -1;
  const std::string s = box_mesh_text(nx, ny, nz, perturb, seed);
  if (buf && buflen > 0) {
    const int64_t k = std::min<int64_t>((int64_t)s.size(), buflen - 1);
    std::memcpy(buf, s.data(), (size_t)k);
    buf[k] = 0;
  }
  return (int64_t)s.size();
}

int64_t bt_blocked_mesh_text(int nx, int ny, int nz, int bx, int by, int bz, double h, double perturb, uint64_t seed,
                             char* buf, int64_t buflen) {
  if (nx < 1 || ny < 1 || nz < 1 || bx < 1 || by < 1 || bz < 1 || !(h > 0)) return -1;
  const std::string s = blocked_mesh_text(nx, ny, nz, bx, by, bz, h, perturb, seed);
  if (buf && buflen > 0) {
    const int64_t k = std::min<int64_t>((int64_t)s.size(), buflen - 1);
    std::memcpy(buf, s.data(), (size_t)k);
    buf[k] = 0;
  }
  return (int64_t)s.size();
}

int64_t bt_cubes_mesh_text(int n, double perturb, uint64_t seed, char* buf, int64_t buflen) {
  const std::string s = cubes_mesh_text(n, perturb, seed);
  if (buf && buflen > 0) {
    const int64_t k = std::min<int64_t>((int64_t)s.size(), buflen - 1);
    std::memcpy(buf, s.data(), (size_t)k);
    buf[k] = 0;
  }
  return (int64_t)s.size();
}

bt_status bt_random_fill(const bt_grid* g, int space, int level, uint64_t seed, double* x, void* stream) {
  BT_TRY
  check_level(g, level);
  if (space == BT_SPACE_EDGES) {
    random_fill_edges(*g, level, seed, x, (cudaStream_t)stream);
    return BT_OK;
  }
  if (space != BT_SPACE_P1) raise(BT_INVALID_ARGUMENT, "bt_random_fill: P1 or edge space expected");
  // fe_function.hpp:479-497: owned slots in canonical (cell, entry, t) order.
  // A partitioned grid generates its own cells' values, after discarding the
  // draws of the owned slots of the cells before its block.
  const int n = 1 << level, w = n + 1;
  const int64_t per = n_tet(w);
  const int cb = g->part_begin, ce = g->part_end;
  std::vector<double> h((size_t)(per * (ce - cb)), 0.0);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  {
    // lattice points per zero set: interior n_tet(n-3), face tri(n-2), edge n-1, vertex 1
    auto points = [&](int z) -> int64_t {
      const int bits = __builtin_popcount((unsigned)z);
      return bits == 0 ? n_tet(n - 3) : bits == 1 ? n_tri(n - 2) : bits == 2 ? n - 1 : 1;
    };
    unsigned long long skip = 0;
    for (int c = 0; c < cb; ++c)
      for (int z = 0; z < 15; ++z)
        if ((g->topo.info[c].owned_by_z >> z) & 1) skip += (unsigned long long)points(z);
    rng.discard(skip);  // one engine call per value (64-bit engine, generate_canonical<double>)
  }
  for (int c = cb; c < ce; ++c) {
    const uint16_t own = g->topo.info[c].owned_by_z;
    int64_t t = per * (c - cb);
    for (int k = 0; k < w; ++k)
      for (int j = 0; j < w - k; ++j)
        for (int i = 0; i < w - k - j; ++i, ++t)
          if ((own >> zero_set(n, i, j, k)) & 1) h[t] = dist(rng);
  }
  cudaStream_t s = (cudaStream_t)stream;
  BT_CUDA(cudaMemcpyAsync(x, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, s));
  // replicas: every group on one handle; on a partitioned grid the groups
  // local to the rank (the caller completes rank-spanning ones with
  // bt_xchg_pack / allreduce / bt_xchg_finish(mode 2))
  launch_interface(*g, level, IF_BCAST, x, nullptr, s);
  BT_CUDA(cudaStreamSynchronize(s));
  BT_CATCH
}

bt_status bt_stencil_create(const bt_grid* g, const bt_form* form, int level, bt_stencil** out) {
  BT_TRY
  check_level(g, level);
  validate_form(form);
  if (form->kind == BT_FORM_DIV_K_GRAD)
    raise(BT_INVALID_ARGUMENT, "compute_stencil: variable-coefficient forms are unsupported");
  BT_CUDA(cudaSetDevice(g->device));
  auto st = std::make_unique<bt_stencil>();
  st->grid = g;
  st->level = level;
  st->form = *form;
  std::vector<StencilCell> cells;
  build_stencil_cells(*g, *form, level, cells, st->rows);
  st->d_cells.upload(cells);
  init_stencil_tasks(*st);
  BT_CUDA(cudaStreamSynchronize(0));
  *out = st.release();
  BT_CATCH
}

}  // extern "C"

// assembled diagonal (operators.hpp:277-316 for stencil tables): zero-set-typed
// partial diagonals, then additive sync. Built on first use, because on a
// partitioned grid the sync is a collective.
const double* bt::stencil_diag(const bt_stencil& st, cudaStream_t s) {
  if (st.d_diag.p) return st.d_diag.p;
  const bt_grid& g = *st.grid;
  const int nc = g.mesh.n_cells();
  std::vector<double> tbl(16 * (size_t)nc);
  for (int c = 0; c < nc; ++c) {
    double cls[6][16];
    class_matrices(g, st.form.kind, st.level, c, cls);
    typed_diag(cls, &tbl[16 * (size_t)c]);
  }
  DevBuf<double> d_tbl;
  d_tbl.upload(tbl);
  DevBuf<double> diag;
  diag.alloc((size_t)bt_space_size(&g, BT_SPACE_P1, st.level));
  launch_fill_by_z(g, st.level, d_tbl.p, diag.p, s);
  sync(g, st.level, IF_SYNC, diag.p, nullptr, s);
  BT_CUDA(cudaStreamSynchronize(s));
  std::swap(st.d_diag.p, diag.p);
  std::swap(st.d_diag.n, diag.n);
  return st.d_diag.p;
}

extern "C" {

void bt_stencil_destroy(bt_stencil* s) { delete s; }

bt_status bt_stencil_rows(const bt_stencil* s, double* rows) {
  BT_TRY
  for (size_t c = 0; c < s->rows.size(); ++c)
    for (int d = 0; d < 15; ++d) rows[15 * c + d] = s->rows[c][d];
  BT_CATCH
}

bt_status bt_stencil_diagonal(const bt_stencil* s, double* diag, void* stream) {
  BT_TRY
  const double* d = stencil_diag(*s, (cudaStream_t)stream);
  BT_CUDA(cudaMemcpyAsync(diag, d, sizeof(double) * s->d_diag.n, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  BT_CATCH
}

}  // extern "C"
