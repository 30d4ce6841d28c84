// blocktet_b200.hpp — C++ facade over the C ABI (blocktet_b200.h) with the
// reference library's API for the hot path: same function names, argument
// order and meaning, and the same std exception types, so a reference call
// site compiles against this header with the namespace changed
// (`namespace blocktet = blocktet_b200;` via BLOCKTET_B200_ALIAS).
//
// Reference interfaces mirrored (paths relative to
// /root/reference/proj/include/blocktet/):
//   allocate / assign / scale / copy / axpy / dot / norm2   fe_function.hpp:277-396
//   sync_additive / sync_broadcast / random_fill            fe_function.hpp:400-497
//   owned_dof_count                                         fe_function.hpp:550
//   FormId (coefficient as a device-evaluable descriptor)   forms.hpp:29-41
//   compute_stencil / apply_stencil / apply_elementwise     operators.hpp:115-271
//   impose_dirichlet / extract_diagonal                     operators.hpp:98, 277
//   hadamard / zero_dirichlet / cg                          solvers.hpp:53-131
//   prolongate_p1 / restrict_p1                             solvers.hpp:227-293
//   make_hierarchy / hierarchy_apply / spectral_estimate    solvers.hpp:323-371
//   SmootherConfig / smooth / MultigridConfig / v_cycle     solvers.hpp:379-541
//
//   parse_mesh / CoarseMesh / Grid(CoarseMesh, lo, hi)     coarse_mesh.hpp:37,225; fe_function.hpp:105
//   Subgroup, linearize(_checked/_aos/_soa), delinearize   micro_index.hpp:22-175
//   FEFunction::values[l][cell][entry], array, at, offset  fe_function.hpp:232-275
//   cg(std::function op, ...), estimate_lambda_max(op,...) solvers.hpp:84-172
//
// Differences:
//   - FEFunction levels live in device memory. `values` is a host mirror with
//     the reference's shape values[level - min][cell][entry]: it is
//     downloaded when read after a device operation wrote the function, and
//     uploaded before the next device operation after it was written through
//     a non-const access. Keep no reference into it across device calls.
//     Copies of an FEFunction are deep, as the reference's.
//   - FormId::div_k_grad takes a Coefficient descriptor, not std::function.
//   - Device storage exists for P1 and the seven edge subgroups (N1E1); P2
//     allocates (sizes as the reference) but its syncs/dots are not on the
//     device path.
//   - Grid levels 2..10 (the reference caps at 6, fe_function.hpp:108).
//   - threads arguments are accepted and ignored (work is stream-ordered).
#ifndef BLOCKTET_B200_HPP
#define BLOCKTET_B200_HPP

#include <cuda_runtime.h>

#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "blocktet_b200.h"

namespace blocktet_b200 {

using Level = int;

// ---- errors: bt_status -> the reference's exception types ----------------
inline void check(bt_status s) {
  if (s == BT_OK) return;
  const std::string m = bt_last_error();
  switch (s) {
    case BT_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case BT_OUT_OF_RANGE: throw std::out_of_range(m);
    case BT_DOMAIN_ERROR: throw std::domain_error(m);
    case BT_LOGIC_ERROR: throw std::logic_error(m);
    default: throw std::runtime_error(m);
  }
}

// ---- index algebra (micro_index.hpp:22-175) -----------------------------------
enum class Subgroup : std::uint8_t {
  V = 0,
  EdgeX, EdgeY, EdgeZ, EdgeXY, EdgeXZ, EdgeYZ, EdgeXYZ,
  FaceZUp, FaceZDown, FaceYUp, FaceYDown, FaceXUp, FaceXDown,
  FaceXYZUp, FaceXYZDown, FaceXYUp, FaceXYDown, FaceYZUp, FaceYZDown,
  CellIUp, CellIDown, CellIIUp, CellIIDown, CellIIIUp, CellIIIDown,
};
enum class MicroKind : std::uint8_t { Vertex, Edge, Face, Cell };
constexpr MicroKind subgroup_kind(Subgroup g) {
  return (int)g == 0 ? MicroKind::Vertex : ((int)g <= 7 ? MicroKind::Edge : ((int)g <= 19 ? MicroKind::Face : MicroKind::Cell));
}
using Idx3 = std::array<int, 3>;
inline std::int64_t n_tri(std::int64_t w) { return bt_n_tri(w); }
inline std::int64_t n_tet(std::int64_t w) { return bt_n_tet(w); }
inline int width_formula(int subgroup, Level l) { return bt_width_formula(subgroup, l); }
inline int width_formula(Subgroup g, Level l) { return bt_width_formula((int)g, l); }
inline int width(int subgroup, Level l) {
  int w = 0;
  check(bt_width(subgroup, l, &w));
  return w;
}
inline int width(Subgroup g, Level l) { return width((int)g, l); }
inline std::int64_t linearize(int w, int i, int j, int k) { return bt_linearize(w, i, j, k); }
inline std::int64_t linearize(int w, Idx3 p) { return bt_linearize(w, p[0], p[1], p[2]); }
inline std::int64_t linearize_checked(int w, Idx3 p) {
  std::int64_t t = 0;
  check(bt_linearize_checked(w, p[0], p[1], p[2], &t));
  return t;
}
inline std::int64_t linearize_aos(int w, int m, Idx3 p, int d) {
  std::int64_t t = 0;
  check(bt_linearize_aos(w, m, p[0], p[1], p[2], d, &t));
  return t;
}
inline std::int64_t linearize_soa(int w, int m, Idx3 p, int d) {
  std::int64_t t = 0;
  check(bt_linearize_soa(w, m, p[0], p[1], p[2], d, &t));
  return t;
}
inline Idx3 delinearize(int w, std::int64_t t) {
  Idx3 p{};
  check(bt_delinearize(w, t, p.data()));
  return p;
}

// ---- coarse mesh (coarse_mesh.hpp:37-47, 225-368) ----------------------------
struct Vec3 {
  double x = 0, y = 0, z = 0;
};
struct CoarseMesh {
  std::vector<Vec3> vertex_coords;
  std::vector<std::array<int, 4>> cells;  // after the orientation repair
  int n_warnings = 0;
  int n_vertices() const { return (int)vertex_coords.size(); }
  int n_cells() const { return (int)cells.size(); }
  std::string text() const {  // the mesh text format (write_mesh), round-trip exact
    std::string out = "vertices " + std::to_string(n_vertices()) + "\n";
    char buf[96];
    for (const Vec3& v : vertex_coords) {
      std::snprintf(buf, sizeof buf, "%.17g %.17g %.17g\n", v.x, v.y, v.z);
      out += buf;
    }
    out += "cells " + std::to_string(n_cells()) + "\n";
    for (const auto& c : cells)
      out += std::to_string(c[0]) + " " + std::to_string(c[1]) + " " + std::to_string(c[2]) + " " +
             std::to_string(c[3]) + "\n";
    return out;
  }
};
inline CoarseMesh parse_mesh(const std::string& text) {
  int nv = 0, nc = 0, nw = 0;
  check(bt_mesh_parse(text.c_str(), &nv, &nc, nullptr, nullptr, &nw));
  std::vector<double> xyz(3 * (size_t)nv);
  std::vector<int> cells(4 * (size_t)nc);
  check(bt_mesh_parse(text.c_str(), &nv, &nc, xyz.data(), cells.data(), &nw));
  CoarseMesh m;
  m.n_warnings = nw;
  for (int v = 0; v < nv; ++v) m.vertex_coords.push_back({xyz[3 * v], xyz[3 * v + 1], xyz[3 * v + 2]});
  for (int c = 0; c < nc; ++c) m.cells.push_back({cells[4 * c], cells[4 * c + 1], cells[4 * c + 2], cells[4 * c + 3]});
  return m;
}
inline std::string ref_tet_text() {  // coarse_mesh.hpp:335-341
  return "# reference tetrahedron\nvertices 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ncells 1\n0 1 2 3\n";
}
inline std::string cube_kuhn_text() {  // coarse_mesh.hpp:344-368: six tets around the (0,0,0)-(1,1,1) diagonal
  std::string out = "# unit cube, six tetrahedra around the main diagonal\nvertices 8\n";
  for (int v = 0; v < 8; ++v)
    out += std::to_string(v & 1) + " " + std::to_string((v >> 1) & 1) + " " + std::to_string((v >> 2) & 1) + "\n";
  out += "cells 6\n";
  const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  for (const auto& a : perms) {
    int c[4] = {0, 1 << a[0], (1 << a[0]) | (1 << a[1]), 7};
    double e[3][3];
    for (int q = 0; q < 3; ++q)
      for (int d = 0; d < 3; ++d) e[q][d] = (double)((c[q + 1] >> d) & 1);
    const double vol = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                       e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                       e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
    if (vol < 0) std::swap(c[2], c[3]);
    out += std::to_string(c[0]) + " " + std::to_string(c[1]) + " " + std::to_string(c[2]) + " " +
           std::to_string(c[3]) + "\n";
  }
  return out;
}

// ---- grid (fe_function.hpp:92) ---------------------------------------------
class Grid {
 public:
  struct Member {  // fe_function.hpp:94-99
    int cell;
    Subgroup g;
    std::int64_t t;
  };
  Grid(const std::string& mesh_text, Level min_level, Level max_level, int device = 0)
      : Grid(parse_mesh(mesh_text), min_level, max_level, device) {}
  Grid(CoarseMesh mesh, Level min_level, Level max_level, int device = 0) : mesh_(std::move(mesh)) {
    check(bt_grid_create(mesh_.text().c_str(), min_level, max_level, device, &g_));
  }
  const CoarseMesh& mesh() const { return mesh_; }
  // the interface groups of a level (P1; members sorted (cell, g, t), first = owner)
  std::vector<std::vector<Member>> groups(Level l) const {
    std::int64_t ng = 0, nm = 0;
    check(bt_grid_groups(g_, l, BT_SPACE_P1, &ng, &nm, nullptr, nullptr, nullptr, nullptr));
    std::vector<std::int64_t> off((size_t)ng + 1), t((size_t)nm);
    std::vector<std::int32_t> cell((size_t)nm), sg((size_t)nm);
    check(bt_grid_groups(g_, l, BT_SPACE_P1, &ng, &nm, off.data(), cell.data(), sg.data(), t.data()));
    std::vector<std::vector<Member>> out((size_t)ng);
    for (std::int64_t q = 0; q < ng; ++q)
      for (std::int64_t m = off[q]; m < off[q + 1]; ++m) out[q].push_back({cell[m], (Subgroup)sg[m], t[m]});
    return out;
  }
  ~Grid() { bt_grid_destroy(g_); }
  Grid(const Grid&) = delete;
  Grid& operator=(const Grid&) = delete;
  int n_cells() const { return bt_num_cells(g_); }
  Level min_level() const { return bt_grid_min_level(g_); }
  Level max_level() const { return bt_grid_max_level(g_); }
  bool has_level(Level l) const { return l >= min_level() && l <= max_level(); }
  const bt_grid* handle() const { return g_; }
  // multi-GPU (one process per GPU): this handle computes and stores the cell
  // block of `rank`; `allreduce` sums device doubles over the ranks in stream
  // order (e.g. ncclAllReduce on the stream). Call before allocating.
  void set_partition(int rank, int nranks, bt_allreduce_fn allreduce, void* user) {
    check(bt_grid_set_partition(g_, rank, nranks));
    check(bt_grid_set_allreduce(g_, allreduce, user));
  }

 private:
  CoarseMesh mesh_;
  bt_grid* g_ = nullptr;
};
inline std::shared_ptr<const Grid> make_grid(const std::string& mesh_text, Level min_level, Level max_level,
                                             int device = 0) {
  return std::make_shared<const Grid>(mesh_text, min_level, max_level, device);
}
// make_grid for one rank of a partitioned run
inline std::shared_ptr<const Grid> make_partitioned_grid(const std::string& mesh_text, Level min_level,
                                                         Level max_level, int device, int rank, int nranks,
                                                         bt_allreduce_fn allreduce, void* user) {
  auto g = std::make_shared<Grid>(mesh_text, min_level, max_level, device);
  g->set_partition(rank, nranks, allreduce, user);
  return g;
}
inline std::string cubes_mesh_text(int n, double perturb = 0.1, std::uint64_t seed = 0) {
  std::string s((size_t)bt_cubes_mesh_text(n, perturb, seed, nullptr, 0), '\0');
  bt_cubes_mesh_text(n, perturb, seed, s.data(), (std::int64_t)s.size());
  while (!s.empty() && s.back() == '\0') s.pop_back();
  return s;
}

// ---- spaces and functions (fe_function.hpp:21-307) -------------------------
enum class LayoutKind : std::uint8_t { AoS, SoA };
enum class Space : int { P1 = BT_SPACE_P1, P2 = BT_SPACE_P2, Edges = BT_SPACE_EDGES };
struct SpaceDescriptor {
  std::string name;
  std::vector<std::pair<Subgroup, int>> entries;  // (subgroup, DoFs per instance); m = 1 here
  LayoutKind layout = LayoutKind::AoS;
  int entry_of(Subgroup g) const {
    for (std::size_t e = 0; e < entries.size(); ++e)
      if (entries[e].first == g) return (int)e;
    return -1;
  }
  bool same_space(const SpaceDescriptor& o) const { return entries == o.entries; }
  Space space() const {
    if (entries.size() == 1 && entries[0].first == Subgroup::V) return Space::P1;
    if (entries.size() == 8 && entries[0].first == Subgroup::V) return Space::P2;
    if (entries.size() == 7 && entries[0].first == Subgroup::EdgeX) return Space::Edges;
    throw std::invalid_argument("space descriptor: P1, P2 or the seven edge subgroups expected");
  }
};
inline SpaceDescriptor p1_space(LayoutKind layout = LayoutKind::AoS) { return {"p1", {{Subgroup::V, 1}}, layout}; }
inline SpaceDescriptor p2_space(LayoutKind layout = LayoutKind::AoS) {
  SpaceDescriptor d{"p2", {{Subgroup::V, 1}}, layout};
  for (int g = 1; g <= 7; ++g) d.entries.emplace_back((Subgroup)g, 1);
  return d;
}
inline SpaceDescriptor edge_space(LayoutKind layout = LayoutKind::AoS) {  // N1E1 storage
  SpaceDescriptor d{"n1e1", {}, layout};
  for (int g = 1; g <= 7; ++g) d.entries.emplace_back((Subgroup)g, 1);
  return d;
}

class FEFunction {
 public:
  // Host mirror with the reference's shape: values[level - min][cell][entry].
  class Values {
   public:
    using Level3 = std::vector<std::vector<std::vector<double>>>;
    Level3& operator[](std::size_t i) {
      owner_->pull();
      owner_->host_dirty_ = true;
      return v_.at(i);
    }
    const Level3& operator[](std::size_t i) const {
      owner_->pull();
      return v_.at(i);
    }
    std::size_t size() const { return (std::size_t)(owner_->hi_ - owner_->lo_ + 1); }

   private:
    friend class FEFunction;
    FEFunction* owner_ = nullptr;
    std::vector<Level3> v_;
  };

  FEFunction() { values.owner_ = this; }
  FEFunction(SpaceDescriptor d, std::shared_ptr<const Grid> g, Level lo, Level hi)
      : descriptor(std::move(d)), grid(std::move(g)), lo_(lo), hi_(hi) {
    values.owner_ = this;
    space_ = (int)descriptor.space();
    for (Level l = lo; l <= hi; ++l) {
      const size_t n = (size_t)bt_space_size(grid->handle(), space_, l);
      levels_.push_back(device_alloc(n));
      sizes_.push_back(n);
    }
  }
  FEFunction(const FEFunction& o) : descriptor(o.descriptor), grid(o.grid), lo_(o.lo_), hi_(o.hi_), space_(o.space_) {
    values.owner_ = this;  // deep copy, as the reference's std::vector storage
    o.push();
    for (std::size_t q = 0; q < o.levels_.size(); ++q) {
      levels_.push_back(device_alloc(o.sizes_[q]));
      sizes_.push_back(o.sizes_[q]);
      if (cudaMemcpy(levels_.back().get(), o.levels_[q].get(), o.sizes_[q] * sizeof(double),
                     cudaMemcpyDeviceToDevice) != cudaSuccess)
        throw std::runtime_error("FEFunction: copy failed");
    }
  }
  FEFunction(FEFunction&& o) noexcept { *this = std::move(o); }
  FEFunction& operator=(FEFunction&& o) noexcept {
    descriptor = std::move(o.descriptor);
    grid = std::move(o.grid);
    lo_ = o.lo_;
    hi_ = o.hi_;
    space_ = o.space_;
    levels_ = std::move(o.levels_);
    sizes_ = std::move(o.sizes_);
    values.v_ = std::move(o.values.v_);
    values.owner_ = this;
    host_valid_ = o.host_valid_;
    host_dirty_ = o.host_dirty_;
    return *this;
  }
  FEFunction& operator=(const FEFunction& o) {
    if (this != &o) *this = FEFunction(o);
    return *this;
  }

  Level min_level() const { return lo_; }
  Level max_level() const { return hi_; }
  bool has_level(Level l) const { return l >= lo_ && l <= hi_; }
  int check_level(Level l) const {  // fe_function.hpp:268-272
    if (!has_level(l)) throw std::out_of_range("level not allocated");
    return l - lo_;
  }
  int space() const { return space_; }
  int width_of(int entry, Level l) const { return width_formula(descriptor.entries.at((size_t)entry).first, l); }
  std::int64_t slots_of(int entry, Level l) const {
    const int w = width_of(entry, l);
    return w > 0 ? n_tet(w) : 0;
  }
  // layout-aware slot offset of (t, d) (fe_function.hpp:257-261)
  std::int64_t offset(Level l, int entry, std::int64_t t, int d) const {
    const int m = descriptor.entries.at((size_t)entry).second;
    return descriptor.layout == LayoutKind::AoS ? m * t + d : d * slots_of(entry, l) + t;
  }
  std::vector<double>& array(Level l, int cell, int entry) { return values[(size_t)check_level(l)][cell][entry]; }
  const std::vector<double>& array(Level l, int cell, int entry) const {
    return values[(size_t)check_level(l)][cell][entry];
  }
  double& at(Level l, int cell, int entry, std::int64_t t, int d) {
    return array(l, cell, entry).at((size_t)offset(l, entry, t, d));
  }
  double at(Level l, int cell, int entry, std::int64_t t, int d) const {
    return array(l, cell, entry).at((size_t)offset(l, entry, t, d));
  }

  // device array of one level (all cells of this handle, reference layout).
  // The non-const form assumes the caller writes it (the host mirror goes stale).
  double* device(Level l) {
    push();
    host_valid_ = false;
    return levels_.at((size_t)check_level(l)).get();
  }
  const double* device(Level l) const {
    push();
    return levels_.at((size_t)check_level(l)).get();
  }
  std::size_t size(Level l) const { return sizes_.at((size_t)check_level(l)); }
  // one level as a flat host array (cells in order, entries in order)
  std::vector<double> level_values(Level l) const {
    std::vector<double> h(size(l));
    if (cudaMemcpy(h.data(), device(l), h.size() * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      throw std::runtime_error("FEFunction: download failed");
    return h;
  }
  void upload(Level l, const std::vector<double>& h) {
    if (h.size() != size(l)) throw std::invalid_argument("FEFunction::upload: size mismatch");
    if (cudaMemcpy(device(l), h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      throw std::runtime_error("FEFunction::upload: copy failed");
  }

  SpaceDescriptor descriptor;
  std::shared_ptr<const Grid> grid;
  Values values;

 private:
  static std::shared_ptr<double> device_alloc(std::size_t n) {
    double* p = nullptr;
    if (n && cudaMalloc(&p, n * sizeof(double)) != cudaSuccess) throw std::runtime_error("FEFunction: cudaMalloc failed");
    if (n) cudaMemset(p, 0, n * sizeof(double));
    return std::shared_ptr<double>(p, [](double* q) {
      if (q) cudaFree(q);
    });
  }
  // per cell of this handle's block: the entries' slot counts (m = 1)
  std::vector<std::int64_t> entry_slots(Level l) const {
    std::vector<std::int64_t> e;
    for (std::size_t q = 0; q < descriptor.entries.size(); ++q) e.push_back(slots_of((int)q, l));
    return e;
  }
  int cells_here() const {
    int r = 0, n = 0, b = 0, e = 0;
    check(bt_grid_partition(grid->handle(), &r, &n, &b, &e));
    return e - b;
  }
  // device -> host mirror (when a device operation wrote the function since)
  void pull() const {
    if (host_valid_) return;
    auto& self = const_cast<FEFunction&>(*this);
    self.values.v_.assign(levels_.size(), {});
    const int nc = cells_here();
    for (std::size_t q = 0; q < levels_.size(); ++q) {
      std::vector<double> flat(sizes_[q]);
      if (sizes_[q] && cudaMemcpy(flat.data(), levels_[q].get(), sizes_[q] * sizeof(double),
                                  cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("FEFunction: download failed");
      const auto es = entry_slots(lo_ + (Level)q);
      std::size_t pos = 0;
      auto& lv = self.values.v_[q];
      lv.assign((size_t)nc, {});
      for (int c = 0; c < nc; ++c)
        for (std::int64_t n : es) {
          lv[c].emplace_back(flat.begin() + (std::ptrdiff_t)pos, flat.begin() + (std::ptrdiff_t)(pos + n));
          pos += (std::size_t)n;
        }
    }
    self.host_valid_ = true;
    self.host_dirty_ = false;
  }
  // host mirror -> device (when it was written through a non-const access)
  void push() const {
    if (!host_dirty_) return;
    auto& self = const_cast<FEFunction&>(*this);
    for (std::size_t q = 0; q < levels_.size(); ++q) {
      std::vector<double> flat;
      flat.reserve(sizes_[q]);
      for (const auto& cell : values.v_[q])
        for (const auto& e : cell) flat.insert(flat.end(), e.begin(), e.end());
      if (flat.size() != sizes_[q]) throw std::logic_error("FEFunction: host mirror reshaped");
      if (sizes_[q] && cudaMemcpy(levels_[q].get(), flat.data(), sizes_[q] * sizeof(double),
                                  cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("FEFunction: upload failed");
    }
    self.host_dirty_ = false;
  }
  Level lo_ = 0, hi_ = -1;
  int space_ = BT_SPACE_P1;
  std::vector<std::shared_ptr<double>> levels_;
  std::vector<std::size_t> sizes_;
  bool host_valid_ = false, host_dirty_ = false;
};

inline FEFunction allocate(const SpaceDescriptor& descriptor, std::shared_ptr<const Grid> grid, int min_level = -1,
                           int max_level = -1) {
  if (!grid) throw std::invalid_argument("allocate: grid required");
  if (min_level < 0) min_level = grid->min_level();
  if (max_level < 0) max_level = grid->max_level();
  if (min_level > max_level || !grid->has_level(min_level) || !grid->has_level(max_level))
    throw std::out_of_range("allocate: levels outside the grid");
  return FEFunction(descriptor, std::move(grid), min_level, max_level);
}

namespace detail {
inline void require_pair(const FEFunction& a, const FEFunction& b, Level l) {
  if (a.grid != b.grid) throw std::invalid_argument("functions live on different grids");
  if (a.space() != b.space()) throw std::invalid_argument("functions have different spaces");
  if (!a.has_level(l) || !b.has_level(l)) throw std::out_of_range("level not allocated");
}
inline const bt_grid* G(const FEFunction& f) { return f.grid->handle(); }
}  // namespace detail

inline void assign(FEFunction& fn, Level l, double value) {
  check(bt_assign(detail::G(fn), fn.space(), l, fn.device(l), value, nullptr));
}
inline void scale(FEFunction& fn, Level l, double s) {
  check(bt_scale(detail::G(fn), fn.space(), l, fn.device(l), s, nullptr));
}
inline void copy(const FEFunction& src, FEFunction& dst, Level l) {
  detail::require_pair(src, dst, l);
  check(bt_copy(detail::G(src), src.space(), l, src.device(l), dst.device(l), nullptr));
}
inline void axpy(FEFunction& y, double a, const FEFunction& x, Level l) {
  detail::require_pair(x, y, l);
  check(bt_axpy(detail::G(x), x.space(), l, y.device(l), a, x.device(l), nullptr));
}
inline double dot(const FEFunction& x, const FEFunction& y, Level l) {
  detail::require_pair(x, y, l);
  double r = 0;
  check(bt_dot(detail::G(x), x.space(), l, x.device(l), y.device(l), &r, nullptr));
  return r;
}
inline double norm2(const FEFunction& x, Level l) { return std::sqrt(dot(x, x, l)); }
inline void sync_additive(FEFunction& fn, Level l) {
  check(bt_sync_additive(detail::G(fn), fn.space(), l, fn.device(l), nullptr));
}
inline void sync_broadcast(FEFunction& fn, Level l) {
  check(bt_sync_broadcast(detail::G(fn), fn.space(), l, fn.device(l), nullptr));
}
inline void random_fill(FEFunction& fn, Level l, std::uint64_t seed) {
  check(bt_random_fill(detail::G(fn), fn.space(), l, seed, fn.device(l), nullptr));
}
inline std::int64_t owned_dof_count(const FEFunction& fn, Level l) {
  return bt_owned_dof_count(detail::G(fn), fn.space(), l);
}
inline void impose_dirichlet(const FEFunction& src, FEFunction& dst, Level l) {
  detail::require_pair(src, dst, l);
  check(bt_impose_dirichlet(detail::G(src), l, src.device(l), dst.device(l), nullptr));
}
inline void zero_dirichlet(FEFunction& fn, Level l) {
  check(bt_zero_dirichlet(detail::G(fn), l, fn.device(l), nullptr));
}
inline void hadamard(FEFunction& fn, const FEFunction& diag, Level l, bool divide) {
  detail::require_pair(fn, diag, l);
  check(bt_hadamard(detail::G(fn), l, fn.device(l), diag.device(l), divide ? 1 : 0, nullptr));
}

// ---- forms (forms.hpp:29-41) -------------------------------------------------
enum class FormKind : int { Diffusion = BT_FORM_DIFFUSION, Mass = BT_FORM_MASS, DivKGrad = BT_FORM_DIV_K_GRAD };
struct Coefficient {  // device-evaluable stand-in for std::function<double(Vec3)>
  int kind = 0;
  std::array<double, 4> c{1.0, 0.0, 0.0, 0.0};
  static Coefficient constant(double c0) { return {0, {c0, 0, 0, 0}}; }
  static Coefficient sin_product(double c0 = 1.0, double c1 = 0.5, double freq = 2.0 * M_PI) {
    return {1, {c0, c1, freq, 0}};
  }
  static Coefficient affine(double c0, double cx, double cy, double cz) { return {2, {c0, cx, cy, cz}}; }
};
struct FormId {
  FormKind kind = FormKind::Diffusion;
  Coefficient k;
  static FormId diffusion() { return {FormKind::Diffusion, {}}; }
  static FormId mass() { return {FormKind::Mass, {}}; }
  static FormId div_k_grad(Coefficient k) { return {FormKind::DivKGrad, k}; }
  bool constant_coefficient() const { return kind != FormKind::DivKGrad; }
  bt_form c_form() const {
    bt_form f{};
    f.kind = (int)kind;
    f.coeff_kind = k.kind;
    for (int i = 0; i < 4; ++i) f.c[i] = k.c[i];
    return f;
  }
};

enum class ApplyMode : int { Replace = BT_MODE_REPLACE, Add = BT_MODE_ADD };
enum class BC : int { None = BT_BC_NONE, DirichletIdentity = BT_BC_DIRICHLET_IDENTITY };
enum class SweepDirection : int { Forward = 0, Backward = 1 };

// ---- P1 operators (operators.hpp) ------------------------------------------
struct StencilTable {
  std::shared_ptr<const Grid> grid;
  FormKind form = FormKind::Diffusion;
  Level level = 0;
  std::shared_ptr<bt_stencil> handle;
  std::vector<std::array<double, 15>> rows() const {
    std::vector<std::array<double, 15>> r((size_t)grid->n_cells());
    check(bt_stencil_rows(handle.get(), r.data()->data()));
    return r;
  }
};
inline StencilTable compute_stencil(const FormId& form, std::shared_ptr<const Grid> grid, Level l) {
  if (!form.constant_coefficient())
    throw std::invalid_argument("compute_stencil: variable-coefficient forms are unsupported");
  const bt_form f = form.c_form();
  bt_stencil* s = nullptr;
  check(bt_stencil_create(grid->handle(), &f, l, &s));
  return StencilTable{std::move(grid), form.kind, l, std::shared_ptr<bt_stencil>(s, bt_stencil_destroy)};
}
inline void apply_stencil(const StencilTable& table, const FEFunction& src, FEFunction& dst, Level l,
                          BC bc = BC::None, int /*threads*/ = 1) {
  detail::require_pair(src, dst, l);
  if (src.grid != table.grid) throw std::invalid_argument("apply_stencil: table built for another grid");
  if (l != table.level) throw std::invalid_argument("apply_stencil: table built for another level");
  check(bt_apply_stencil(table.handle.get(), src.device(l), dst.device(l), (int)bc, nullptr));
}
inline void apply_elementwise(const FormId& form, const FEFunction& src, FEFunction& dst, Level l,
                              ApplyMode mode = ApplyMode::Replace, BC bc = BC::None, int /*threads*/ = 1) {
  detail::require_pair(src, dst, l);
  const bt_form f = form.c_form();
  check(bt_apply_elementwise(detail::G(src), &f, l, src.device(l), dst.device(l), (int)mode, (int)bc, nullptr,
                             nullptr));
}
inline void extract_diagonal(const FormId& form, FEFunction& diag, Level l, int /*threads*/ = 1) {
  const bt_form f = form.c_form();
  check(bt_extract_diagonal(detail::G(diag), &f, l, diag.device(l), nullptr));
}

// ---- transfers (solvers.hpp:227-293) ---------------------------------------
inline void prolongate_p1(const FEFunction& coarse, FEFunction& fine, Level fine_l) {
  if (coarse.grid != fine.grid) throw std::invalid_argument("transfer between different grids");
  if (!coarse.has_level(fine_l - 1) || !fine.has_level(fine_l)) throw std::out_of_range("transfer levels");
  check(bt_prolongate(detail::G(fine), fine_l, coarse.device(fine_l - 1), fine.device(fine_l), 0, nullptr));
}
inline void restrict_p1(const FEFunction& fine, FEFunction& coarse, Level fine_l) {
  if (coarse.grid != fine.grid) throw std::invalid_argument("transfer between different grids");
  if (!coarse.has_level(fine_l - 1) || !fine.has_level(fine_l)) throw std::out_of_range("transfer levels");
  check(bt_restrict(detail::G(fine), fine_l, fine.device(fine_l), coarse.device(fine_l - 1), nullptr));
}

// ---- hierarchy, smoothers, multigrid (solvers.hpp:296-541) -----------------
enum class KernelKind : int { Elementwise = 0, Stencil = 1 };
struct GridHierarchy {
  std::shared_ptr<const Grid> grid;
  FormId form;
  KernelKind kernel = KernelKind::Stencil;
  std::shared_ptr<bt_hierarchy> handle;
};
inline GridHierarchy make_hierarchy(std::shared_ptr<const Grid> grid, FormId form,
                                    KernelKind kernel = KernelKind::Stencil, int /*threads*/ = 1) {
  if (!grid) throw std::invalid_argument("make_hierarchy: grid required");
  if (kernel == KernelKind::Stencil && !form.constant_coefficient())
    throw std::invalid_argument("stencil kernel requires a constant-coefficient form");
  const bt_form f = form.c_form();
  bt_hierarchy* h = nullptr;
  check(bt_hierarchy_create(grid->handle(), &f, (int)kernel, &h));
  return GridHierarchy{std::move(grid), form, kernel, std::shared_ptr<bt_hierarchy>(h, bt_hierarchy_destroy)};
}
inline void hierarchy_apply(const GridHierarchy& h, const FEFunction& x, FEFunction& y, Level l,
                            BC bc = BC::DirichletIdentity) {
  detail::require_pair(x, y, l);
  check(bt_hierarchy_apply(h.handle.get(), l, x.device(l), y.device(l), (int)bc, nullptr));
}
inline double spectral_estimate(GridHierarchy& h, Level l) {
  double r = 0;
  check(bt_estimate_lambda_max(h.handle.get(), l, &r, nullptr));
  return r;
}

enum class SmootherKind : int { Jacobi = 0, GaussSeidel = 1, Chebyshev = 2 };
struct SmootherConfig {
  SmootherKind kind = SmootherKind::GaussSeidel;
  double omega = 0.8;
  int order = 2;
  double lo = 0.25;
  double hi = 1.1;
  int nu1 = 1;
  int nu2 = 1;
  static SmootherConfig gauss_seidel() { return {}; }
  static SmootherConfig jacobi(double omega = 0.8) {
    SmootherConfig c;
    c.kind = SmootherKind::Jacobi;
    c.omega = omega;
    return c;
  }
  static SmootherConfig chebyshev(int order = 2) {
    SmootherConfig c;
    c.kind = SmootherKind::Chebyshev;
    c.order = order;
    return c;
  }
  bt_smoother_config c_config() const { return {(int)kind, omega, order, lo, hi, nu1, nu2}; }
};
struct MultigridConfig {
  int coarse_level = 2;
  int cycles = 5;
  double coarse_tol = 1e-12;
  int coarse_maxit = 4000;
  bt_multigrid_config c_config() const { return {coarse_level, cycles, coarse_tol, coarse_maxit}; }
};
inline void smooth(GridHierarchy& h, const SmootherConfig& cfg, const FEFunction& rhs, FEFunction& x, Level l,
                   int sweeps, SweepDirection direction = SweepDirection::Forward) {
  detail::require_pair(rhs, x, l);
  const bt_smoother_config c = cfg.c_config();
  check(bt_smooth(h.handle.get(), &c, rhs.device(l), x.device(l), l, sweeps, (int)direction, nullptr));
}

struct IterationRow {
  int level = 0;
  int cycle = 0;
  double residual = 0;
  double error = 0;
  double seconds = 0;
};
struct IterationReport {
  std::vector<IterationRow> rows;
  int iterations = 0;
  double residual = 0;
  bool converged = false;
};
inline IterationReport cg(GridHierarchy& h, const FEFunction& rhs, FEFunction& x, Level l, double tol, int maxit) {
  detail::require_pair(rhs, x, l);
  std::vector<double> hist((size_t)std::max(maxit, 1));
  int it = 0;
  check(bt_cg(h.handle.get(), l, tol, maxit, rhs.device(l), x.device(l), hist.data(), &it, nullptr));
  IterationReport rep;
  for (int i = 0; i < it; ++i) rep.rows.push_back({l, i + 1, hist[(size_t)i], 0.0, 0.0});
  rep.iterations = it;
  rep.residual = it ? hist[(size_t)it - 1] : 0.0;
  rep.converged = rep.residual <= tol;
  return rep;
}
// cg over any operator callable (solvers.hpp:84-131), the reference's
// algorithm step for step on device vectors; scalars on the host. (The
// hierarchy overload above keeps the scalars on the device.)
inline IterationReport cg(const std::function<void(const FEFunction&, FEFunction&)>& apply_op, const FEFunction& rhs,
                          FEFunction& x, Level l, double tol, int maxit) {
  detail::require_pair(rhs, x, l);
  if (!apply_op) throw std::invalid_argument("cg: operator required");
  FEFunction r = allocate(x.descriptor, x.grid, l, l);
  FEFunction p = allocate(x.descriptor, x.grid, l, l);
  FEFunction ap = allocate(x.descriptor, x.grid, l, l);
  apply_op(x, r);
  scale(r, l, -1.0);
  axpy(r, 1.0, rhs, l);
  copy(r, p, l);
  const double nb = norm2(rhs, l);
  const double denom = nb > 0 ? nb : 1.0;
  double rs = dot(r, r, l);
  IterationReport report;
  report.residual = std::sqrt(rs) / denom;
  if (report.residual <= tol) {
    report.converged = true;
    return report;
  }
  for (int it = 1; it <= maxit; ++it) {
    apply_op(p, ap);
    const double pap = dot(p, ap, l);
    if (!(pap > 0)) throw std::runtime_error("cg breakdown: operator is not positive definite");
    const double alpha = rs / pap;
    axpy(x, alpha, p, l);
    axpy(r, -alpha, ap, l);
    const double rs_new = dot(r, r, l);
    report.iterations = it;
    report.residual = std::sqrt(rs_new) / denom;
    report.rows.push_back({l, it, report.residual, 0.0, 0.0});
    if (report.residual <= tol) {
      report.converged = true;
      break;
    }
    scale(p, l, rs_new / rs);
    axpy(p, 1.0, r, l);
    rs = rs_new;
  }
  return report;
}

// estimate_lambda_max over any operator callable (solvers.hpp:140-172)
inline double estimate_lambda_max(const std::function<void(const FEFunction&, FEFunction&)>& apply_op,
                                  const FEFunction& diag, Level l, int iterations = 25) {
  if (diag.space() != BT_SPACE_P1) throw std::invalid_argument("P1 function required");
  for (double v : diag.level_values(l))
    if (v == 0.0) throw std::invalid_argument("estimate_lambda_max: zero diagonal entry");
  FEFunction v = allocate(diag.descriptor, diag.grid, l, l);
  FEFunction w = allocate(diag.descriptor, diag.grid, l, l);
  FEFunction z = allocate(diag.descriptor, diag.grid, l, l);
  random_fill(v, l, 0x51cbu);
  zero_dirichlet(v, l);
  const double nv = norm2(v, l);
  if (nv == 0) throw std::runtime_error("estimate_lambda_max: empty free space");
  scale(v, l, 1.0 / nv);
  double rho = 0;
  for (int k = 0; k < iterations; ++k) {
    apply_op(v, w);
    copy(v, z, l);
    hadamard(z, diag, l, false);
    rho = dot(v, w, l) / dot(v, z, l);
    copy(w, v, l);
    hadamard(v, diag, l, true);
    const double nn = norm2(v, l);
    if (nn == 0) break;
    scale(v, l, 1.0 / nn);
  }
  return 1.1 * rho;
}

inline void v_cycle(GridHierarchy& h, Level l, const FEFunction& rhs, FEFunction& x, const SmootherConfig& sm,
                    const MultigridConfig& mg) {
  detail::require_pair(rhs, x, l);
  const bt_smoother_config s = sm.c_config();
  const bt_multigrid_config m = mg.c_config();
  check(bt_v_cycle(h.handle.get(), l, rhs.device(l), x.device(l), &s, &m, nullptr));
}

// ---- model-problem tools: interpolate, l2_error, fmg ------------------------
// The std::function arguments become device-evaluable Coefficient fields.
namespace detail {
inline bt_field c_field(const Coefficient& f) { return bt_field{f.kind, {f.c[0], f.c[1], f.c[2], f.c[3]}}; }
}  // namespace detail
inline void interpolate(FEFunction& fn, Level l, const Coefficient& f) {  // fe_function.hpp:454 (P1)
  const bt_field c = detail::c_field(f);
  check(bt_interpolate(fn.grid->handle(), l, &c, fn.device(l), nullptr));
}
inline double l2_error(const FEFunction& fn, Level l, const Coefficient& exact) {  // solvers.hpp:613
  const bt_field c = detail::c_field(exact);
  double out = 0;
  check(bt_l2_error(fn.grid->handle(), l, fn.device(l), &c, &out, nullptr));
  return out;
}
// fmg (solvers.hpp:547); `exact` replaces the error callback (nullptr: no errors)
inline IterationReport fmg(GridHierarchy& h, Level finest, const std::vector<FEFunction>& rhs_levels, FEFunction& x,
                           const SmootherConfig& sm, const MultigridConfig& mg,
                           const Coefficient* exact = nullptr) {
  if (finest < mg.coarse_level) throw std::invalid_argument("fmg: finest below coarse level");
  if ((int)rhs_levels.size() != finest - mg.coarse_level + 1)
    throw std::invalid_argument("fmg: one rhs per level expected");
  std::vector<const double*> ptrs;
  for (size_t i = 0; i < rhs_levels.size(); ++i) ptrs.push_back(rhs_levels[i].device(mg.coarse_level + (int)i));
  std::vector<bt_fmg_row> rows((size_t)(1 + mg.cycles * (finest - mg.coarse_level)));
  int n = 0;
  const bt_smoother_config s = sm.c_config();
  const bt_multigrid_config m = mg.c_config();
  bt_field ex{};
  if (exact) ex = detail::c_field(*exact);
  check(bt_fmg(h.handle.get(), finest, ptrs.data(), x.device(finest), &s, &m, exact ? &ex : nullptr, rows.data(),
               (int)rows.size(), &n, nullptr));
  IterationReport rep;
  for (int i = 0; i < n; ++i) rep.rows.push_back({rows[i].level, rows[i].cycle, rows[i].residual, rows[i].error, 0.0});
  rep.iterations = mg.cycles * (finest - mg.coarse_level);
  rep.residual = n ? rows[n - 1].residual : 0.0;
  rep.converged = true;
  return rep;
}

// ---- N1E1 curl-curl + mass (no reference implementation) -------------------
struct N1E1Operator {
  std::shared_ptr<const Grid> grid;
  Level level = 0;
  std::shared_ptr<bt_n1e1> handle;
};
inline N1E1Operator make_n1e1(std::shared_ptr<const Grid> grid, Level l, double alpha = 1.0, double beta = 1.0) {
  bt_n1e1* op = nullptr;
  check(bt_n1e1_create(grid->handle(), l, alpha, beta, &op));
  return N1E1Operator{std::move(grid), l, std::shared_ptr<bt_n1e1>(op, bt_n1e1_destroy)};
}
inline void apply_n1e1(const N1E1Operator& op, const FEFunction& src, FEFunction& dst,
                       BC bc = BC::DirichletIdentity) {
  detail::require_pair(src, dst, op.level);
  check(bt_apply_n1e1(op.handle.get(), src.device(op.level), dst.device(op.level), (int)bc, nullptr));
}

}  // namespace blocktet_b200

#ifdef BLOCKTET_B200_ALIAS
namespace blocktet = blocktet_b200;
#endif

#endif
