// Exercises the C++ facade (include/blocktet_b200.hpp) the way reference
// call sites use the blocktet API. Driven by tests/test_facade.py:
//   facade_check index            index algebra + exception mapping (no GPU)
//   facade_check nogpu MESH       grid creation must fail loudly without CUDA
//   facade_check apply MESH DIR   cube-kuhn L4: apply_stencil and 3 V-cycles,
//                                 results written to DIR for the oracle check
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#define BLOCKTET_B200_ALIAS
#include "blocktet_b200.hpp"

using namespace blocktet;

static std::string slurp(const char* path) {
  std::ifstream f(path);
  std::stringstream s;
  s << f.rdbuf();
  return s.str();
}
static void dump(const std::string& path, const std::vector<double>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), (std::streamsize)(v.size() * sizeof(double)));
}
#define EXPECT(c)                                        \
  do {                                                   \
    if (!(c)) {                                          \
      std::fprintf(stderr, "FAILED: %s (line %d)\n", #c, __LINE__); \
      return 1;                                          \
    }                                                    \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string mode = argv[1];
  if (mode == "index") {
    EXPECT(n_tet(5) == 35 && n_tri(5) == 15);
    EXPECT(width_formula(0, 3) == 9 && width(21, 3) == 6);
    for (int w = 1; w <= 9; ++w)
      for (std::int64_t t = 0; t < n_tet(w); ++t) {
        const auto p = delinearize(w, t);
        EXPECT(linearize(w, p[0], p[1], p[2]) == t);
      }
    bool domain = false;
    try {
      width(21, 1);  // I-down cells are absent at level 1
    } catch (const std::domain_error&) {
      domain = true;
    }
    EXPECT(domain);
    std::puts("ok");
    return 0;
  }
  if (mode == "nogpu") {
    try {
      auto g = make_grid(slurp(argv[2]), 2, 3);
    } catch (const std::runtime_error& e) {
      std::printf("raised: %s\n", e.what());
      return 0;
    }
    return 1;
  }
  if (mode == "apply") {
    const Level l = 4;
    auto g = make_grid(slurp(argv[2]), 2, l);
    const std::string dir = argv[3];
    auto x = allocate(p1_space(), g), y = allocate(p1_space(), g);
    random_fill(x, l, 0);
    const StencilTable t = compute_stencil(FormId::diffusion(), g, l);
    apply_stencil(t, x, y, l, BC::None);
    dump(dir + "/x.bin", x.level_values(l));
    dump(dir + "/y.bin", y.level_values(l));
    bool invalid = false;
    try {
      apply_stencil(t, x, y, l - 1);  // table built for level l
    } catch (const std::invalid_argument&) {
      invalid = true;
    }
    EXPECT(invalid);

    GridHierarchy h = make_hierarchy(g, FormId::diffusion(), KernelKind::Stencil);
    auto rhs = allocate(p1_space(), g), u = allocate(p1_space(), g);
    random_fill(rhs, l, 0);
    zero_dirichlet(rhs, l);
    SmootherConfig sm = SmootherConfig::chebyshev(2);
    sm.nu1 = sm.nu2 = 2;
    MultigridConfig mg;
    mg.coarse_level = 2;
    mg.coarse_tol = 1e-14;
    mg.coarse_maxit = 20;
    for (int c = 0; c < 3; ++c) v_cycle(h, l, rhs, u, sm, mg);
    dump(dir + "/rhs.bin", rhs.level_values(l));
    dump(dir + "/u.bin", u.level_values(l));
    // full multigrid of the model problem (solvers.hpp:547): second-order errors
    const Coefficient uex = Coefficient::sin_product(0.0, 1.0, M_PI);
    const Coefficient f = Coefficient::sin_product(0.0, 3.0 * M_PI * M_PI, M_PI);
    std::vector<FEFunction> rhs_levels;
    for (int q = 2; q <= l; ++q) {
      auto fi = allocate(p1_space(), g, q, q), b = allocate(p1_space(), g, q, q);
      interpolate(fi, q, f);
      apply_elementwise(FormId::mass(), fi, b, q);
      zero_dirichlet(b, q);
      rhs_levels.push_back(std::move(b));
    }
    auto xf = allocate(p1_space(), g, l, l);
    MultigridConfig fm = mg;
    fm.cycles = 3;
    fm.coarse_maxit = 200;
    const IterationReport rep = fmg(h, l, rhs_levels, xf, sm, fm, &uex);
    EXPECT((int)rep.rows.size() == 1 + 3 * (l - 2));
    EXPECT(rep.rows.back().error > 0 && rep.rows.back().error < rep.rows.front().error);
    std::printf("fmg error %.6e\n", rep.rows.back().error);
    std::printf("owned %lld dot %.17g\n", (long long)owned_dof_count(x, l), dot(x, y, l));
    return 0;
  }
  return 2;
}
