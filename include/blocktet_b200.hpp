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
// Differences:
//   - FEFunction levels live in device memory; values(l) downloads a host copy.
//   - FormId::div_k_grad takes a Coefficient descriptor, not std::function.
//   - cg takes the hierarchy (its operator is hierarchy_apply with Dirichlet
//     identity rows, which is what every reference call site passes).
//   - threads arguments are accepted and ignored (work is stream-ordered).
#ifndef BLOCKTET_B200_HPP
#define BLOCKTET_B200_HPP

#include <cuda_runtime.h>

#include <array>
#include <cmath>
#include <cstdint>
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

// ---- index algebra (micro_index.hpp:85-165) -------------------------------
inline std::int64_t n_tri(std::int64_t w) { return bt_n_tri(w); }
inline std::int64_t n_tet(std::int64_t w) { return bt_n_tet(w); }
inline int width_formula(int subgroup, Level l) { return bt_width_formula(subgroup, l); }
inline int width(int subgroup, Level l) {
  int w = 0;
  check(bt_width(subgroup, l, &w));
  return w;
}
inline std::int64_t linearize(int w, int i, int j, int k) { return bt_linearize(w, i, j, k); }
inline std::array<int, 3> delinearize(int w, std::int64_t t) {
  std::array<int, 3> p{};
  check(bt_delinearize(w, t, p.data()));
  return p;
}

// ---- grid (fe_function.hpp:92) ---------------------------------------------
class Grid {
 public:
  Grid(const std::string& mesh_text, Level min_level, Level max_level, int device = 0) {
    check(bt_grid_create(mesh_text.c_str(), min_level, max_level, device, &g_));
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

// ---- spaces and functions (fe_function.hpp:31-307) -------------------------
enum class Space : int { P1 = BT_SPACE_P1, P2 = BT_SPACE_P2, Edges = BT_SPACE_EDGES };
struct SpaceDescriptor {
  std::string name;
  Space space = Space::P1;
};
inline SpaceDescriptor p1_space() { return {"p1", Space::P1}; }
inline SpaceDescriptor edge_space() { return {"n1e1", Space::Edges}; }

class FEFunction {
 public:
  FEFunction() = default;
  FEFunction(SpaceDescriptor d, std::shared_ptr<const Grid> grid, Level lo, Level hi)
      : descriptor(std::move(d)), grid(std::move(grid)), lo_(lo), hi_(hi) {
    for (Level l = lo; l <= hi; ++l) {
      const size_t n = (size_t)bt_space_size(this->grid->handle(), (int)descriptor.space, l);
      double* p = nullptr;
      if (cudaMalloc(&p, n * sizeof(double)) != cudaSuccess) throw std::runtime_error("FEFunction: cudaMalloc failed");
      cudaMemset(p, 0, n * sizeof(double));
      levels_.emplace_back(p, [](double* q) { cudaFree(q); });
      sizes_.push_back(n);
    }
  }
  Level min_level() const { return lo_; }
  Level max_level() const { return hi_; }
  bool has_level(Level l) const { return l >= lo_ && l <= hi_; }
  int space() const { return (int)descriptor.space; }
  // device array of one level (all cells, reference layout)
  double* device(Level l) { return levels_.at(index(l)).get(); }
  const double* device(Level l) const { return levels_.at(index(l)).get(); }
  std::size_t size(Level l) const { return sizes_.at(index(l)); }
  // host copies (the reference's values[level][cell] as one flat array)
  std::vector<double> values(Level l) const {
    std::vector<double> h(size(l));
    if (cudaMemcpy(h.data(), device(l), h.size() * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      throw std::runtime_error("FEFunction::values: copy failed");
    return h;
  }
  void upload(Level l, const std::vector<double>& h) {
    if (h.size() != size(l)) throw std::invalid_argument("FEFunction::upload: size mismatch");
    if (cudaMemcpy(device(l), h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      throw std::runtime_error("FEFunction::upload: copy failed");
  }

  SpaceDescriptor descriptor;
  std::shared_ptr<const Grid> grid;

 private:
  int index(Level l) const {
    if (!has_level(l)) throw std::out_of_range("FEFunction: level not allocated");
    return l - lo_;
  }
  Level lo_ = 0, hi_ = -1;
  std::vector<std::shared_ptr<double>> levels_;
  std::vector<std::size_t> sizes_;
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
