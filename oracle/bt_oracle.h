/* TEST INFRASTRUCTURE — CPU restatement ("oracle") of the reference
 * algorithms on the matrix-free hot path of arXiv 2308.01792's `blocktet`
 * library (/root/reference/proj/include/blocktet). It is the checker for the
 * CUDA product, never the product: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it.
 *
 * Parity pinned: every function is checked bit-for-bit against the compiled
 * reference (oracle/_ref/libbtref.so, built by oracle/Makefile) in
 * tests/test_oracle_vs_ref.py, and against the committed fixtures in
 * tests/golden/ (generated from the reference by tests/golden/make_golden.py).
 * The N1E1 restatement (bt_oracle_n1e1.c) has no reference implementation
 * (SPEC.md:8 lists it out of scope): "parity unpinned", self-pinned by
 * algebraic identities only.
 *
 * Flat vector layout = FEFunction::values[level][cell][entry] flattened with
 * cells outer, entries next, lattice slots inner (fe_function.hpp:237-261,
 * m = 1 for every entry used here, so AoS == SoA). */
#ifndef BT_ORACLE_H
#define BT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- index algebra (micro_index.hpp) ---------------------------------- */
int64_t bo_n_tri(int64_t w);                           /* micro_index.hpp:85 */
int64_t bo_n_tet(int64_t w);                           /* micro_index.hpp:89 */
int bo_width_formula(int g, int level);                /* micro_index.hpp:97 */
int64_t bo_linearize(int w, int i, int j, int k);      /* micro_index.hpp:145 */
int bo_delinearize(int w, int64_t t, int* ijk);        /* micro_index.hpp:157 */
int bo_subgroup_offsets(int g, int* out);              /* micro_index.hpp:218-263 */

/* ---- RNG (libstdc++ mt19937_64 + uniform_real_distribution<double>) --- */
typedef struct { uint64_t mt[312]; int mti; } bo_mt64;
void bo_mt64_seed(bo_mt64* r, uint64_t seed);
uint64_t bo_mt64_next(bo_mt64* r);
double bo_uniform(bo_mt64* r, double a, double b);

/* ---- mesh (coarse_mesh.hpp) ------------------------------------------- */
typedef struct {
  int nv, nc, nf, ne;
  double* coords;      /* 3*nv */
  int* cells;          /* 4*nc, after orientation repair */
  int* faces;          /* 3*nf sorted triples, lexicographic */
  int* face_cells;     /* 2*nf, -1 if none */
  char* bflags;        /* nf */
  int* edges;          /* 2*ne */
  int* cell_faces;     /* 4*nc, slot t = face opposite local vertex t */
  double* maps;        /* 12*nc: A (row-major 3x3) then b */
  int nwarn;
} bo_mesh;

int bo_mesh_parse(const char* text, bo_mesh* m, char* err, int errlen);
void bo_mesh_free(bo_mesh* m);
/* n x n x n unit-cube Kuhn mesh, vertex perturbation `perturb` * h
 * (interior vertices in all components, boundary vertices tangentially),
 * mt19937_64(seed). Returns bytes written (excluding NUL) or needed size. */
int64_t bo_cubes_mesh_text(int n, double perturb, uint64_t seed, char* buf, int64_t buflen);

/* ---- grid (fe_function.hpp:92-226) ------------------------------------ */
typedef struct {
  int level;
  int64_t ngroups, nmembers;
  int64_t* goff;       /* ngroups+1 */
  int32_t* mcell;
  int32_t* mg;
  int64_t* mt;
  uint8_t* owned[8];   /* per slot: ncells * n_tet(w_slot) */
  uint8_t* dir[8];
} bo_level;

typedef struct {
  bo_mesh mesh;
  int lo, hi, with_edges;
  bo_level* levels;
} bo_grid;

bo_grid* bo_grid_new(const char* text, int lo, int hi, int with_edges, char* err, int errlen);
void bo_grid_free(bo_grid* g);
const bo_level* bo_grid_level(const bo_grid* g, int l);

/* spaces: 0 = P1 {V}; 1 = P2 {V, 7 edges}; 2 = edges {7 edges} */
int64_t bo_space_size(const bo_grid* g, int space, int l);
void bo_random_fill(const bo_grid* g, int space, int l, uint64_t seed, double* out);
void bo_sync(const bo_grid* g, int space, int l, int broadcast, double* v);
double bo_dot(const bo_grid* g, int space, int l, const double* x, const double* y);
int64_t bo_owned_count(const bo_grid* g, int space, int l);

/* ---- forms / operators (forms.hpp, operators.hpp) ---------------------- */
/* form: 0 diffusion, 1 mass, 2 div_k_grad with kp = {kind, c0, c1, c2, c3}
 * kind 0: c0; kind 1: c0 + c1 sin(c2 x) sin(c2 y) sin(c2 z);
 * kind 2: c0 + c1 x + c2 y + c3 z */
int bo_local_matrix(int form, const double* kp, const double* corners12, double* out16);
int bo_class_matrices(const bo_grid* g, int form, int l, int cell, double* out96);
int bo_compute_stencil(const bo_grid* g, int form, int l, double* rows, double* diag);
int bo_apply_stencil(const bo_grid* g, int form, int l, int bc, const double* x, double* y);
int bo_apply_elementwise(const bo_grid* g, int form, const double* kp, int l, int add, int bc,
                         const double* x, double* y);
int bo_extract_diagonal(const bo_grid* g, int form, const double* kp, int l, double* d);
void bo_impose_dirichlet(const bo_grid* g, int l, const double* src, double* dst);
void bo_zero_dirichlet(const bo_grid* g, int l, double* x);

/* ---- transfers / solvers (solvers.hpp) -------------------------------- */
void bo_prolongate(const bo_grid* g, int fine_l, const double* coarse, double* fine);
void bo_restrict(const bo_grid* g, int fine_l, const double* fine, double* coarse);

typedef struct bo_hier bo_hier;
/* kernel: 0 elementwise, 1 stencil */
bo_hier* bo_hier_new(const bo_grid* g, int form, const double* kp, int kernel);
void bo_hier_free(bo_hier* h);
int bo_hier_apply(bo_hier* h, int l, int bc, const double* x, double* y);
const double* bo_hier_diag(bo_hier* h, int l);
double bo_hier_lambda(bo_hier* h, int l);
/* sm = {kind(0 jacobi,1 gs,2 cheb), omega, order, lo, hi, nu1, nu2} */
int bo_smooth(bo_hier* h, const double* sm, int l, int sweeps, int backward,
              const double* rhs, double* x);
int bo_cg(bo_hier* h, int l, double tol, int maxit, const double* rhs, double* x,
          double* hist, int* iters);
int bo_vcycles(bo_hier* h, int l, const double* sm, int coarse_level, double coarse_tol,
               int coarse_maxit, int cycles, const double* rhs, double* x, double* hist);

/* ---- N1E1 curl-curl + mass (no reference implementation) --------------- */
int bo_n1e1_local(const double* corners12, double alpha, double beta, double* out36);
int bo_n1e1_apply(const bo_grid* g, int l, double alpha, double beta, int bc,
                  const double* x, double* y);
void bo_n1e1_sync(const bo_grid* g, int l, double* v);
void bo_n1e1_signs(const bo_grid* g, int l, int8_t* sign_of_member);
void bo_n1e1_random_fill(const bo_grid* g, int l, uint64_t seed, double* out);
void bo_n1e1_gradient(const bo_grid* g, int l, const double* phi, double* u);
void bo_n1e1_constant_field(const bo_grid* g, int l, const double* c3, double* u);

const char* bo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
