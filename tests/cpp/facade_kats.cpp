// Reference-style call sites compiled against the C++ facade
// (include/blocktet_b200.hpp) with `namespace blocktet` aliased: the grid is
// built as the reference's tests build it (std::make_shared<Grid>(parse_mesh
// (text), lo, hi)), functions are read and written through the host mirror
// values[level - min][cell][entry] / at(l, cell, entry, t, d), and the
// known answers are the reference tests' (proj/tests/test_fe_function.cpp:
// allocation sizes 35 / 125 / 729, owned dots 35 / 125 / 55, sync 2.0 on the
// shared face and 6.0 on the Kuhn diagonal, single-cell sync is a no-op;
// solvers.hpp:84 cg over a callable). Driven by tests/test_facade.py.
#include <cstdio>
#include <memory>
#include <set>
#include <string>

#define BLOCKTET_B200_ALIAS
#include "blocktet_b200.hpp"

using namespace blocktet;

#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAILED: %s (line %d)\n", #c, __LINE__); \
      return 1;                                                    \
    }                                                              \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
  }
  return false;
}

static const char* kGlued =  // two positive tets sharing the face (1, 2, 3)
    "vertices 5\n0 0 0\n1 0 0\n0 1 0\n0 0 1\n1 1 1\ncells 2\n0 1 2 3\n1 2 3 4\n";

static std::shared_ptr<const Grid> grid_of(const std::string& text, int lo, int hi) {
  return std::make_shared<Grid>(parse_mesh(text), lo, hi);
}

int main() {
  // ---- sizes and level guards
  {
    auto g = grid_of(ref_tet_text(), 2, 2);
    const FEFunction f = allocate(p1_space(), g);
    EXPECT(f.values[0][0].size() == 1 && f.values[0][0][0].size() == 35);
    auto k = grid_of(cube_kuhn_text(), 2, 3);
    const FEFunction q = allocate(p1_space(), k);
    EXPECT(q.values.size() == 2 && q.values[0].size() == 6 && q.values[1].size() == 6);
    EXPECT(owned_dof_count(q, 2) == 125 && owned_dof_count(q, 3) == 729);
    const CoarseMesh mesh = parse_mesh(ref_tet_text());
    EXPECT(throws<std::invalid_argument>([&] { Grid(mesh, 1, 3); }));
    EXPECT(throws<std::invalid_argument>([&] { Grid(mesh, 4, 3); }));
    EXPECT(throws<std::out_of_range>([&] { allocate(p1_space(), grid_of(ref_tet_text(), 2, 3), 2, 4); }));
    EXPECT(throws<std::out_of_range>([&] { linearize_checked(5, {3, 1, 1}); }));
    EXPECT(throws<std::out_of_range>([&] { linearize_aos(5, 1, {0, 0, 0}, 1); }));
    EXPECT(linearize_soa(5, 2, {1, 0, 0}, 1) == 35 + 1 && linearize_aos(5, 2, {1, 0, 0}, 1) == 3);
  }
  // ---- owned dots count every physical DoF once
  {
    auto g = grid_of(ref_tet_text(), 2, 2);
    FEFunction ones = allocate(p1_space(), g), zeros = allocate(p1_space(), g);
    assign(ones, 2, 1.0);
    EXPECT(dot(ones, ones, 2) == 35.0 && dot(ones, zeros, 2) == 0.0);
    auto k = grid_of(cube_kuhn_text(), 2, 2);
    FEFunction o = allocate(p1_space(), k);
    assign(o, 2, 1.0);
    EXPECT(dot(o, o, 2) == 125.0);
    auto t = grid_of(kGlued, 2, 2);
    FEFunction p = allocate(p1_space(), t);
    assign(p, 2, 1.0);
    EXPECT(dot(p, p, 2) == 55.0);  // 2 * 35 - 15 shared face vertices
  }
  // ---- additive sync
  {
    auto g = grid_of(ref_tet_text(), 2, 2);
    FEFunction f = allocate(p1_space(), g);
    random_fill(f, 2, 7);
    FEFunction before = f;  // deep copy
    sync_additive(f, 2);
    EXPECT(f.values[0][0][0] == before.values[0][0][0]);
    auto t = grid_of(kGlued, 2, 2);
    FEFunction s = allocate(p1_space(), t);
    assign(s, 2, 1.0);
    sync_additive(s, 2);
    EXPECT(s.at(2, 0, 0, linearize(5, {2, 1, 1}), 0) == 2.0);  // on the shared face (cell 0's diagonal plane)
    EXPECT(s.at(2, 0, 0, linearize(5, {1, 1, 1}), 0) == 1.0);  // cell interior
    auto k = grid_of(cube_kuhn_text(), 2, 2);
    FEFunction d = allocate(p1_space(), k);
    assign(d, 2, 1.0);
    sync_additive(d, 2);
    std::multiset<double> seen(d.values[0][0][0].begin(), d.values[0][0][0].end());
    EXPECT(seen.count(6.0) >= 3 && seen.count(1.0) > 0);  // diagonal vertices shared by all six cells
    int sixes = 0;
    for (const auto& group : k->groups(2))
      if (group.size() == 6) {
        ++sixes;
        for (const Grid::Member& m : group) EXPECT(d.at(2, m.cell, d.descriptor.entry_of(m.g), m.t, 0) == 6.0);
      }
    EXPECT(sixes == 5);  // the 5 lattice points of the Kuhn diagonal at level 2
  }
  // ---- host writes reach the device, device writes reach the host
  {
    auto k = grid_of(cube_kuhn_text(), 2, 2);
    FEFunction a = allocate(p1_space(), k), b = allocate(p1_space(), k);
    a.at(2, 3, 0, linearize(5, {1, 1, 1}), 0) = 4.0;  // an interior vertex of cell 3
    EXPECT(dot(a, a, 2) == 16.0);
    copy(a, b, 2);
    EXPECT(b.at(2, 3, 0, linearize(5, {1, 1, 1}), 0) == 4.0);
    scale(b, 2, 0.5);
    EXPECT(b.array(2, 3, 0)[(size_t)linearize(5, {1, 1, 1})] == 2.0);
  }
  // ---- cg over a callable operator (solvers.hpp:84): the stencil with Dirichlet rows
  {
    auto k = grid_of(cube_kuhn_text(), 2, 3);
    const StencilTable tbl = compute_stencil(FormId::diffusion(), k, 3);
    FEFunction rhs = allocate(p1_space(), k, 3, 3), x = allocate(p1_space(), k, 3, 3);
    random_fill(rhs, 3, 1);
    zero_dirichlet(rhs, 3);
    const IterationReport rep = cg([&](const FEFunction& in, FEFunction& out) {
      apply_stencil(tbl, in, out, 3, BC::DirichletIdentity);
    }, rhs, x, 3, 1e-10, 200);
    EXPECT(rep.converged && rep.iterations > 5);
    GridHierarchy h = make_hierarchy(k, FormId::diffusion(), KernelKind::Stencil);
    FEFunction x2 = allocate(p1_space(), k, 3, 3);
    const IterationReport rep2 = cg(h, rhs, x2, 3, 1e-10, 200);
    EXPECT(rep2.iterations == rep.iterations);
    FEFunction diag = allocate(p1_space(), k, 3, 3);
    extract_diagonal(FormId::diffusion(), diag, 3);
    const double lam = estimate_lambda_max([&](const FEFunction& in, FEFunction& out) {
      apply_stencil(tbl, in, out, 3, BC::DirichletIdentity);
    }, diag, 3);
    EXPECT(std::fabs(lam - spectral_estimate(h, 3)) <= 1e-12 * lam);
    std::printf("cg %d its, lambda %.17g\n", rep.iterations, lam);
  }
  std::puts("ok");
  return 0;
}
