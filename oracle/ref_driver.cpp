// Test infrastructure only: an extern "C" shim over the UNMODIFIED reference
// headers (/root/reference/proj/include/blocktet, compiled from a temporary
// copy whose level guard fe_function.hpp:108 is lifted from 6 to 10 by
// oracle/Makefile). It exists to pin the C restatement (oracle/bt_oracle.c),
// to generate tests/golden fixtures, and to time the reference CPU path for
// bench.py's `cpu_baseline` / `--impl reference`. Nothing in the product
// links or loads it.
//
// Flat array convention (matches FEFunction::values[level][cell][entry],
// fe_function.hpp:237-238): one level, cells outer, entries next, slots inner.
#include <cstdint>
#include <functional>
#include <cstring>
#include <chrono>
#include <cmath>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "blocktet/reference_assembly.hpp"
#include "blocktet/solvers.hpp"

using namespace blocktet;

namespace {

thread_local std::string g_err;

struct Ctx {
  std::shared_ptr<const Grid> grid;
  std::map<std::pair<int, int>, StencilTable> tables;  // (form, level)
  std::unique_ptr<GridHierarchy> hier;
};

SpaceDescriptor space_of(int space) {
  if (space == 0) return p1_space();
  if (space == 1) return p2_space();
  // 2: the seven edge subgroups only (N1E1 storage).
  SpaceDescriptor d{"edges", {}, LayoutKind::AoS};
  for (int g = 1; g <= 7; ++g) d.entries.emplace_back(static_cast<Subgroup>(g), 1);
  return d;
}

std::int64_t level_size(const FEFunction& fn, int l) {
  std::int64_t n = 0;
  for (std::size_t e = 0; e < fn.descriptor.entries.size(); ++e)
    n += fn.slots_of(static_cast<int>(e), l);
  return n * fn.grid->mesh().n_cells();
}

void load(FEFunction& fn, int l, const double* src) {
  std::int64_t o = 0;
  for (auto& per_entry : fn.values[fn.check_level(l)])
    for (auto& arr : per_entry) {
      std::memcpy(arr.data(), src + o, arr.size() * sizeof(double));
      o += static_cast<std::int64_t>(arr.size());
    }
}

void store(const FEFunction& fn, int l, double* dst) {
  std::int64_t o = 0;
  for (const auto& per_entry : fn.values[fn.check_level(l)])
    for (const auto& arr : per_entry) {
      std::memcpy(dst + o, arr.data(), arr.size() * sizeof(double));
      o += static_cast<std::int64_t>(arr.size());
    }
}

// Coefficient kinds shared with the product's bt_coeff descriptor:
// 0 constant c0; 1 c0 + c1 sin(f x) sin(f y) sin(f z) with f = p[2];
// 2 affine c0 + c1 x + c2 y + c3 z.
FormId make_form(int form, const double* p) {
  if (form == 0) return FormId::diffusion();
  if (form == 1) return FormId::mass();
  const int kind = static_cast<int>(p[0]);
  const double c0 = p[1], c1 = p[2], c2 = p[3], c3 = p[4];
  if (kind == 0) return FormId::div_k_grad([c0](Vec3) { return c0; });
  if (kind == 1)
    return FormId::div_k_grad([c0, c1, c2](Vec3 x) {
      return c0 + c1 * std::sin(c2 * x.x) * std::sin(c2 * x.y) * std::sin(c2 * x.z);
    });
  return FormId::div_k_grad(
      [c0, c1, c2, c3](Vec3 x) { return c0 + c1 * x.x + c2 * x.y + c3 * x.z; });
}

const StencilTable& table_of(Ctx& c, int form, int l) {
  auto key = std::make_pair(form, l);
  auto it = c.tables.find(key);
  if (it == c.tables.end())
    it = c.tables.emplace(key, compute_stencil(make_form(form, nullptr), c.grid, l)).first;
  return it->second;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_new(const char* text, int lo, int hi) {
  Ctx* c = nullptr;
  if (guarded([&] {
        auto ctx = std::make_unique<Ctx>();
        ctx->grid = std::make_shared<const Grid>(parse_mesh(text), lo, hi);
        c = ctx.release();
      }))
    return nullptr;
  return c;
}

void ref_free(void* h) { delete static_cast<Ctx*>(h); }

int ref_ncells(void* h) { return static_cast<Ctx*>(h)->grid->mesh().n_cells(); }

std::int64_t ref_space_size(void* h, int space, int l) {
  Ctx& c = *static_cast<Ctx*>(h);
  const FEFunction fn = allocate(space_of(space), c.grid, l, l);
  return level_size(fn, l);
}

int ref_masks(void* h, int l, int cell, int g, std::uint8_t* owned, std::uint8_t* dir) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    const auto& m = c.grid->masks(l, cell, static_cast<Subgroup>(g));
    std::memcpy(owned, m.owned.data(), m.owned.size());
    std::memcpy(dir, m.dirichlet.data(), m.dirichlet.size());
  });
}

// Groups flattened: offsets[ngroups+1] into member arrays (cell, g, t).
std::int64_t ref_group_count(void* h, int l, std::int64_t* members) {
  Ctx& c = *static_cast<Ctx*>(h);
  const auto& gs = c.grid->groups(l);
  std::int64_t m = 0;
  for (const auto& g : gs) m += static_cast<std::int64_t>(g.size());
  *members = m;
  return static_cast<std::int64_t>(gs.size());
}

void ref_groups(void* h, int l, std::int64_t* offsets, std::int32_t* cell,
                std::int32_t* g, std::int64_t* t) {
  Ctx& c = *static_cast<Ctx*>(h);
  std::int64_t o = 0, k = 0;
  offsets[0] = 0;
  for (const auto& grp : c.grid->groups(l)) {
    for (const auto& m : grp) {
      cell[o] = m.cell;
      g[o] = static_cast<int>(m.g);
      t[o] = m.t;
      ++o;
    }
    offsets[++k] = o;
  }
}

std::int64_t ref_owned_dof_count(void* h, int space, int l) {
  Ctx& c = *static_cast<Ctx*>(h);
  const FEFunction fn = allocate(space_of(space), c.grid, l, l);
  return owned_dof_count(fn, l);
}

int ref_random_fill(void* h, int space, int l, std::uint64_t seed, double* out) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction fn = allocate(space_of(space), c.grid, l, l);
    random_fill(fn, l, seed);
    store(fn, l, out);
  });
}

int ref_sync(void* h, int space, int l, int broadcast, double* inout) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction fn = allocate(space_of(space), c.grid, l, l);
    load(fn, l, inout);
    if (broadcast)
      sync_broadcast(fn, l);
    else
      sync_additive(fn, l);
    store(fn, l, inout);
  });
}

double ref_dot(void* h, int space, int l, const double* x, const double* y) {
  Ctx& c = *static_cast<Ctx*>(h);
  FEFunction a = allocate(space_of(space), c.grid, l, l);
  FEFunction b = allocate(space_of(space), c.grid, l, l);
  load(a, l, x);
  load(b, l, y);
  return dot(a, b, l);
}

// Stencil rows (15 per cell, kStencilDirs order) and the assembled diagonal.
int ref_stencil_rows(void* h, int form, int l, double* rows, double* diag) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    const StencilTable& t = table_of(c, form, l);
    for (std::size_t cell = 0; cell < t.rows.size(); ++cell)
      for (int d = 0; d < 15; ++d) rows[15 * cell + d] = t.rows[cell][d];
    if (diag) store(t.diagonal, l, diag);
  });
}

int ref_class_matrices(void* h, int form, int l, int cell, double* out96) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    const auto cls = detail::class_matrices(make_form(form, nullptr), *c.grid, cell, l);
    for (int s = 0; s < 6; ++s)
      for (int i = 0; i < 16; ++i) out96[16 * s + i] = cls[s].a[i];
  });
}

int ref_apply_stencil(void* h, int form, int l, int bc, const double* x, double* y,
                      int threads) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    const StencilTable& t = table_of(c, form, l);
    FEFunction a = allocate(p1_space(), c.grid, l, l);
    FEFunction b = allocate(p1_space(), c.grid, l, l);
    load(a, l, x);
    apply_stencil(t, a, b, l, bc ? BC::DirichletIdentity : BC::None, threads);
    store(b, l, y);
  });
}

int ref_apply_elementwise(void* h, int form, const double* kp, int l, int add, int bc,
                          const double* x, double* y, int threads) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction a = allocate(p1_space(), c.grid, l, l);
    FEFunction b = allocate(p1_space(), c.grid, l, l);
    load(a, l, x);
    load(b, l, y);
    apply_elementwise(make_form(form, kp), a, b, l, add ? ApplyMode::Add : ApplyMode::Replace,
                      bc ? BC::DirichletIdentity : BC::None, threads);
    store(b, l, y);
  });
}

int ref_extract_diagonal(void* h, int form, const double* kp, int l, double* d) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction a = allocate(p1_space(), c.grid, l, l);
    extract_diagonal(make_form(form, kp), a, l, 1);
    store(a, l, d);
  });
}

int ref_prolongate(void* h, int fine_l, const double* coarse, double* fine) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction a = allocate(p1_space(), c.grid, fine_l - 1, fine_l);
    FEFunction b = allocate(p1_space(), c.grid, fine_l - 1, fine_l);
    load(a, fine_l - 1, coarse);
    prolongate_p1(a, b, fine_l);
    store(b, fine_l, fine);
  });
}

int ref_restrict(void* h, int fine_l, const double* fine, double* coarse) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction a = allocate(p1_space(), c.grid, fine_l - 1, fine_l);
    FEFunction b = allocate(p1_space(), c.grid, fine_l - 1, fine_l);
    load(a, fine_l, fine);
    restrict_p1(a, b, fine_l);
    store(b, fine_l - 1, coarse);
  });
}

// Hierarchy for smoothers / V-cycles. kernel: 0 elementwise, 1 stencil.
int ref_hierarchy(void* h, int form, const double* kp, int kernel, int threads) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    c.hier = std::make_unique<GridHierarchy>(make_hierarchy(
        c.grid, make_form(form, kp), kernel ? KernelKind::Stencil : KernelKind::Elementwise,
        threads));
  });
}

int ref_hierarchy_diag(void* h, int l, double* d) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] { store(c.hier->diagonals[c.hier->index(l)], l, d); });
}

int ref_hierarchy_apply(void* h, int l, int bc, const double* x, double* y) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction a = allocate(p1_space(), c.grid, l, l);
    FEFunction b = allocate(p1_space(), c.grid, l, l);
    load(a, l, x);
    hierarchy_apply(*c.hier, a, b, l, bc ? BC::DirichletIdentity : BC::None);
    store(b, l, y);
  });
}

double ref_lambda_max(void* h, int l) {
  Ctx& c = *static_cast<Ctx*>(h);
  double v = -1;
  guarded([&] { v = spectral_estimate(*c.hier, l); });
  return v;
}

// sm: [kind(0 jacobi,1 gs,2 cheb), omega, order, lo, hi, nu1, nu2]
SmootherConfig make_smoother(const double* sm) {
  SmootherConfig s;
  s.kind = static_cast<SmootherKind>(static_cast<int>(sm[0]) == 0   ? 0
                                     : static_cast<int>(sm[0]) == 1 ? 1
                                                                     : 2);
  s.omega = sm[1];
  s.order = static_cast<int>(sm[2]);
  s.lo = sm[3];
  s.hi = sm[4];
  s.nu1 = static_cast<int>(sm[5]);
  s.nu2 = static_cast<int>(sm[6]);
  return s;
}

int ref_smooth(void* h, const double* sm, int l, int sweeps, int backward,
               const double* rhs, double* x) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction b = allocate(p1_space(), c.grid, l, l);
    FEFunction u = allocate(p1_space(), c.grid, l, l);
    load(b, l, rhs);
    load(u, l, x);
    smooth(*c.hier, make_smoother(sm), b, u, l, sweeps,
           backward ? SweepDirection::Backward : SweepDirection::Forward);
    store(u, l, x);
  });
}

// Coarse CG through hierarchy_apply with Dirichlet identity rows. Returns
// iterations; residual history (relative) in hist[0..maxit].
int ref_cg(void* h, int l, double tol, int maxit, const double* rhs, double* x,
           double* hist, int* iters) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction b = allocate(p1_space(), c.grid, l, l);
    FEFunction u = allocate(p1_space(), c.grid, l, l);
    load(b, l, rhs);
    load(u, l, x);
    const IterationReport rep = cg(
        [&](const FEFunction& a, FEFunction& y) {
          hierarchy_apply(*c.hier, a, y, l, BC::DirichletIdentity);
        },
        b, u, l, tol, maxit);
    for (std::size_t i = 0; i < rep.rows.size(); ++i) hist[i] = rep.rows[i].residual;
    *iters = rep.iterations;
    store(u, l, x);
  });
}

// Runs `cycles` V-cycles on level l from x (in/out); hist[c] = ||b - A x||/||b||
// after cycle c (owned norms), hist[0] before the first cycle.
int ref_vcycles(void* h, int l, const double* sm, int coarse_level, double coarse_tol,
                int coarse_maxit, int cycles, const double* rhs, double* x, double* hist,
                double* seconds) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    MultigridConfig mg;
    mg.coarse_level = coarse_level;
    mg.coarse_tol = coarse_tol;
    mg.coarse_maxit = coarse_maxit;
    const SmootherConfig s = make_smoother(sm);
    FEFunction b = allocate(p1_space(), c.grid, l, l);
    FEFunction u = allocate(p1_space(), c.grid, l, l);
    FEFunction r = allocate(p1_space(), c.grid, l, l);
    load(b, l, rhs);
    load(u, l, x);
    const double nb = norm2(b, l);
    const auto resid = [&] {
      hierarchy_apply(*c.hier, u, r, l, BC::DirichletIdentity);
      scale(r, l, -1.0);
      axpy(r, 1.0, b, l);
      return norm2(r, l) / (nb > 0 ? nb : 1.0);
    };
    hist[0] = resid();
    for (int cyc = 1; cyc <= cycles; ++cyc) {
      const auto t0 = std::chrono::steady_clock::now();
      v_cycle(*c.hier, l, b, u, s, mg);
      if (seconds)
        seconds[cyc - 1] =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      hist[cyc] = resid();
    }
    store(u, l, x);
  });
}

// Model-problem fields, same kinds as make_form's coefficient: p = {kind, c0, c1, c2, c3}.
std::function<double(Vec3)> make_field(const double* p) {
  const int kind = static_cast<int>(p[0]);
  const double c0 = p[1], c1 = p[2], c2 = p[3], c3 = p[4];
  if (kind == 0) return [c0](Vec3) { return c0; };
  if (kind == 1)
    return [c0, c1, c2](Vec3 x) { return c0 + c1 * std::sin(c2 * x.x) * std::sin(c2 * x.y) * std::sin(c2 * x.z); };
  return [c0, c1, c2, c3](Vec3 x) { return c0 + c1 * x.x + c2 * x.y + c3 * x.z; };
}

int ref_interpolate(void* h, int l, const double* fp, double* out) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction u = allocate(p1_space(), c.grid, l, l);
    interpolate(u, l, make_field(fp));
    store(u, l, out);
  });
}

int ref_l2_error(void* h, int l, const double* x, const double* fp, double* out) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction u = allocate(p1_space(), c.grid, l, l);
    load(u, l, x);
    *out = l2_error(u, l, make_field(fp));
  });
}

// Full multigrid from the given per-level right-hand sides (rhs_all: levels
// coarse_level..finest concatenated); x receives the finest solution; rows:
// 4 doubles (level, cycle, residual, error) each, error against fp (NULL: none).
int ref_fmg(void* h, int finest, const double* sm, int coarse_level, double coarse_tol, int coarse_maxit,
            int cycles, const double* rhs_all, double* x, const double* fp, double* rows, int* nrows) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    MultigridConfig mg;
    mg.coarse_level = coarse_level;
    mg.coarse_tol = coarse_tol;
    mg.coarse_maxit = coarse_maxit;
    mg.cycles = cycles;
    std::vector<FEFunction> rhs;
    std::int64_t off = 0;
    for (int l = coarse_level; l <= finest; ++l) {
      rhs.push_back(allocate(p1_space(), c.grid, l, l));
      load(rhs.back(), l, rhs_all + off);
      off += level_size(rhs.back(), l);
    }
    FEFunction u = allocate(p1_space(), c.grid, finest, finest);
    std::function<double(const FEFunction&, Level)> err;
    if (fp) {
      const auto f = make_field(fp);
      err = [f](const FEFunction& v, Level l) { return l2_error(v, l, f); };
    }
    const IterationReport rep = fmg(*c.hier, finest, rhs, u, make_smoother(sm), mg, err);
    for (std::size_t i = 0; i < rep.rows.size(); ++i) {
      rows[4 * i] = rep.rows[i].level;
      rows[4 * i + 1] = rep.rows[i].cycle;
      rows[4 * i + 2] = rep.rows[i].residual;
      rows[4 * i + 3] = rep.rows[i].error;
    }
    *nrows = static_cast<int>(rep.rows.size());
    store(u, finest, x);
  });
}

int ref_zero_dirichlet(void* h, int l, double* x) {
  Ctx& c = *static_cast<Ctx*>(h);
  return guarded([&] {
    FEFunction u = allocate(p1_space(), c.grid, l, l);
    load(u, l, x);
    detail::zero_dirichlet(u, l);
    store(u, l, x);
  });
}

// Timed reference applies (CPU baseline): kind 0 stencil(diffusion),
// 1 elementwise(form/kp). Returns seconds per apply (median of reps).
double ref_time_apply(void* h, int kind, int form, const double* kp, int l, int bc,
                      int reps, int threads, const double* x) {
  Ctx& c = *static_cast<Ctx*>(h);
  double med = -1;
  guarded([&] {
    FEFunction a = allocate(p1_space(), c.grid, l, l);
    FEFunction b = allocate(p1_space(), c.grid, l, l);
    load(a, l, x);
    const FormId f = make_form(form, kp);
    const StencilTable* t = kind == 0 ? &table_of(c, form, l) : nullptr;
    std::vector<double> ts;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      if (kind == 0)
        apply_stencil(*t, a, b, l, bc ? BC::DirichletIdentity : BC::None, threads);
      else
        apply_elementwise(f, a, b, l, ApplyMode::Replace,
                          bc ? BC::DirichletIdentity : BC::None, threads);
      ts.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(ts.begin(), ts.end());
    med = ts[ts.size() / 2];
  });
  return med;
}

// Frozen subgroup offsets (micro_index.hpp:218-263) for the index pins.
int ref_subgroup_offsets(int g, int* out) {
  const auto offs = subgroup_offsets(static_cast<Subgroup>(g));
  int k = 0;
  for (const Idx3& o : offs) {
    out[k++] = o[0];
    out[k++] = o[1];
    out[k++] = o[2];
  }
  return static_cast<int>(offs.size());
}

int ref_width_formula(int g, int l) { return width_formula(static_cast<Subgroup>(g), l); }
std::int64_t ref_linearize(int w, int i, int j, int k) { return linearize(w, {i, j, k}); }

// Serialized mesh after parse/validate (orientation repair visible).
int ref_mesh_info(void* h, int* nv, int* nc, int* nf, int* ne, int* cells, double* coords,
                  char* bflags) {
  Ctx& c = *static_cast<Ctx*>(h);
  const CoarseMesh& m = c.grid->mesh();
  *nv = m.n_vertices();
  *nc = m.n_cells();
  *nf = static_cast<int>(m.faces.size());
  *ne = static_cast<int>(m.edges.size());
  if (cells)
    for (int i = 0; i < m.n_cells(); ++i)
      for (int k = 0; k < 4; ++k) cells[4 * i + k] = m.cells[i][k];
  if (coords)
    for (int i = 0; i < m.n_vertices(); ++i) {
      coords[3 * i] = m.vertex_coords[i].x;
      coords[3 * i + 1] = m.vertex_coords[i].y;
      coords[3 * i + 2] = m.vertex_coords[i].z;
    }
  if (bflags)
    for (std::size_t f = 0; f < m.faces.size(); ++f) bflags[f] = m.boundary_flags[f];
  return 0;
}

}  // extern "C"
