/* blocktet_b200 — C ABI of the B200-native matrix-free operator path.
 *
 * This is the drop-in boundary for the hot path of arXiv 2308.01792's
 * reference library `blocktet` (header-only C++20, /root/reference/proj).
 * Every entry point below names the reference interface it replaces
 * (file:line relative to proj/include/blocktet/). The C++ facade
 * (include/blocktet_b200.hpp) and the Python mirror
 * (paper_2308_01792_b200/api.py) both sit on top of exactly these symbols.
 *
 * Conventions
 *  - No C++ or torch types cross the boundary: opaque handles, plain
 *    pointers, sizes, and a cudaStream_t passed as `void*` (NULL = default
 *    stream of the handle's device).
 *  - Vectors are caller-owned DEVICE arrays of double, one array per
 *    (function, level): cells outer, entries next, lattice slots inner —
 *    byte-for-byte the layout of FEFunction::values[level][cell][entry]
 *    (fe_function.hpp:237-261). A P1 vector at level l has
 *    bt_num_cells(grid) * n_tet(2^l + 1) doubles.
 *  - Calls are stream-ordered and asynchronous unless they return a host
 *    scalar (dot, norm2, solver reports), which synchronise the stream.
 *  - Nothing throws. Failures return a bt_status; bt_last_error() holds the
 *    message (thread-local). The facades map statuses back to the
 *    reference's exception types (std::invalid_argument, std::out_of_range,
 *    std::domain_error, std::logic_error, std::runtime_error).
 *  - There is no CPU fallback: without a CUDA device every compute entry
 *    point returns BT_CUDA_ERROR.
 */
#ifndef BLOCKTET_B200_H
#define BLOCKTET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BT_OK = 0,
  BT_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  BT_OUT_OF_RANGE = 2,     /* std::out_of_range */
  BT_DOMAIN_ERROR = 3,     /* std::domain_error */
  BT_LOGIC_ERROR = 4,      /* std::logic_error */
  BT_RUNTIME_ERROR = 5,    /* std::runtime_error (e.g. CG breakdown) */
  BT_CUDA_ERROR = 6,
  BT_NCCL_ERROR = 7
} bt_status;

typedef struct bt_grid bt_grid;           /* Grid (fe_function.hpp:92) */
typedef struct bt_stencil bt_stencil;     /* StencilTable (operators.hpp:174) */
typedef struct bt_hierarchy bt_hierarchy; /* GridHierarchy (solvers.hpp:308) */
typedef struct bt_n1e1 bt_n1e1;           /* N1E1 curl-curl + mass operator (no ref) */
typedef struct bt_comm bt_comm;           /* the ranks' NCCL communicator (multi-GPU data plane) */

/* Bilinear form descriptor — FormId (forms.hpp:29-41). The reference's
 * std::function coefficient cannot cross to the device; div_k_grad takes an
 * analytic coefficient instead (documented API deviation):
 *   coeff_kind 0: k = c[0]
 *   coeff_kind 1: k = c[0] + c[1] sin(c[2] x) sin(c[2] y) sin(c[2] z)
 *   coeff_kind 2: k = c[0] + c[1] x + c[2] y + c[3] z                      */
typedef enum { BT_FORM_DIFFUSION = 0, BT_FORM_MASS = 1, BT_FORM_DIV_K_GRAD = 2 } bt_form_kind;
typedef struct {
  int kind;       /* bt_form_kind */
  int coeff_kind; /* see above; ignored unless kind == BT_FORM_DIV_K_GRAD */
  double c[4];
} bt_form;

typedef enum { BT_BC_NONE = 0, BT_BC_DIRICHLET_IDENTITY = 1 } bt_bc;  /* operators.hpp:17 */
typedef enum { BT_MODE_REPLACE = 0, BT_MODE_ADD = 1 } bt_apply_mode;  /* operators.hpp:16 */
typedef enum { BT_SPACE_P1 = 0, BT_SPACE_P2 = 1, BT_SPACE_EDGES = 2 } bt_space;

/* ---- errors / library --------------------------------------------------- */
const char* bt_last_error(void);
const char* bt_version(void);
/* Number of kernel launches issued by this process so far (instrumentation
 * for bench.py's gpu_launches claim). */
uint64_t bt_launch_count(void);
/* Measurement utility (not a reference interface): `blocks` x 256 threads each
 * issue 16 independent fp64 FMA chains of `iters` steps (16 * iters DFMA per
 * thread) on `stream`; *sink receives a data-dependent sum so nothing is
 * eliminated. bench.py times it with CUDA events to measure the FP64 peak that
 * the FP64-bound rooflines (configs 3 and 5) are quoted against. */
bt_status bt_dfma_probe(int blocks, int iters, double* sink, void* stream);

/* ---- index algebra (micro_index.hpp:85-165, host side) ------------------ */
int64_t bt_n_tri(int64_t w);                                /* :85 */
int64_t bt_n_tet(int64_t w);                                /* :89 */
int bt_width_formula(int subgroup, int level);              /* :97 */
bt_status bt_width(int subgroup, int level, int* out);      /* :125 (domain_error if absent) */
int64_t bt_linearize(int w, int i, int j, int k);           /* :145 */
bt_status bt_delinearize(int w, int64_t t, int* ijk3);      /* :157 */
/* linearize_checked (:150-154): BT_OUT_OF_RANGE outside I_tet(w) */
bt_status bt_linearize_checked(int w, int i, int j, int k, int64_t* out);
/* linearize_aos / linearize_soa (:167-175): m * t + d / d * n_tet(w) + t;
 * BT_OUT_OF_RANGE for d outside [0, m) or p outside I_tet(w) */
bt_status bt_linearize_aos(int w, int m, int i, int j, int k, int d, int64_t* out);
bt_status bt_linearize_soa(int w, int m, int i, int j, int k, int d, int64_t* out);
int bt_subgroup_offsets(int subgroup, int* out_xyz);        /* :257, returns arity */

/* ---- grid (Grid ctor fe_function.hpp:106-115 over parse_mesh
 *      coarse_mesh.hpp:225) ------------------------------------------------ */
/* parse_mesh (coarse_mesh.hpp:225-308) with validate_and_finalize's
 * orientation repair: vertex coordinates (3 per vertex) and cell vertex ids
 * (4 per cell, after repair). Pass NULL arrays to query the counts. */
bt_status bt_mesh_parse(const char* mesh_text, int* n_vertices, int* n_cells, double* coords, int* cells,
                        int* n_warnings);
/* Parses the reference mesh text format, builds the implicit interface
 * tables for levels [min_level, max_level] on CUDA device `device`.
 * Levels 2..10 (the reference caps at 6, fe_function.hpp:108). */
bt_status bt_grid_create(const char* mesh_text, int min_level, int max_level, int device,
                         bt_grid** out);
void bt_grid_destroy(bt_grid* g);
int bt_num_cells(const bt_grid* g);
int bt_grid_min_level(const bt_grid* g);
int bt_grid_max_level(const bt_grid* g);
/* doubles in one level of a function of `space` (all cells) */
int64_t bt_space_size(const bt_grid* g, int space, int level);
/* owned_dof_count (fe_function.hpp:550) */
int64_t bt_owned_dof_count(const bt_grid* g, int space, int level);
/* Grid::masks (fe_function.hpp:128): host copies, n_tet(width) bytes each */
bt_status bt_grid_masks(const bt_grid* g, int level, int cell, int subgroup, uint8_t* owned,
                        uint8_t* dirichlet);
/* Grid::groups (fe_function.hpp:123) expanded from the implicit tables, for
 * tests: pass NULL arrays to query sizes. Members are sorted (cell, g, t). */
bt_status bt_grid_groups(const bt_grid* g, int level, int space, int64_t* n_groups,
                         int64_t* n_members, int64_t* offsets, int32_t* cell, int32_t* subgroup,
                         int64_t* t);
/* builder mesh generator for configs 2-5: n^3 unit cubes x 6 Kuhn tets,
 * interior vertices perturbed by U(-perturb h, perturb h) per component from
 * mt19937_64(seed). Writes at most buflen bytes; returns bytes needed. */
int64_t bt_cubes_mesh_text(int n, double perturb, uint64_t seed, char* buf, int64_t buflen);
/* nx x ny x nz unit cubes (side 1) x 6 Kuhn tets, same perturbation rule:
 * the weak-scaling workload of bench.py (6 cells per GPU at N = nx ny nz) */
int64_t bt_box_mesh_text(int nx, int ny, int nz, double perturb, uint64_t seed, char* buf, int64_t buflen);
/* nx x ny x nz cubes of side h (6 Kuhn tets each, same perturbation rule),
 * cubes numbered block-major with blocks of bx x by x bz cubes, so the
 * contiguous cell ranges of bt_grid_set_partition are compact blocks (SURVEY
 * §8(e)); returns -1 on bad arguments */
int64_t bt_blocked_mesh_text(int nx, int ny, int nz, int bx, int by, int bz, double h, double perturb, uint64_t seed,
                             char* buf, int64_t buflen);

/* ---- vectors (fe_function.hpp:324-497, solvers.hpp:53-72) ---------------- */
/* random_fill (fe_function.hpp:479): mt19937_64 on the host in canonical
 * owned order, uploaded, replicas broadcast on the device. */
bt_status bt_random_fill(const bt_grid* g, int space, int level, uint64_t seed, double* x,
                         void* stream);
bt_status bt_assign(const bt_grid* g, int space, int level, double* x, double value, void* stream);
bt_status bt_scale(const bt_grid* g, int space, int level, double* x, double s, void* stream);
bt_status bt_copy(const bt_grid* g, int space, int level, const double* src, double* dst,
                  void* stream);
bt_status bt_axpy(const bt_grid* g, int space, int level, double* y, double a, const double* x,
                  void* stream);
/* owned-DoF dot (fe_function.hpp:376): fixed-order, GPU-count invariant */
bt_status bt_dot(const bt_grid* g, int space, int level, const double* x, const double* y,
                 double* out, void* stream);
bt_status bt_hadamard(const bt_grid* g, int level, double* x, const double* d, int divide,
                      void* stream);
bt_status bt_sync_additive(const bt_grid* g, int space, int level, double* x, void* stream);  /* :400 */
bt_status bt_sync_broadcast(const bt_grid* g, int space, int level, double* x, void* stream); /* :425 */
bt_status bt_impose_dirichlet(const bt_grid* g, int level, const double* src, double* dst,
                              void* stream);                          /* operators.hpp:98 */
bt_status bt_zero_dirichlet(const bt_grid* g, int level, double* x, void* stream); /* solvers.hpp:66 */

/* ---- P1 operators (operators.hpp) -------------------------------------- */
/* compute_stencil (operators.hpp:183): merged 15-point row, class matrices,
 * typed lattice-boundary rows and the assembled diagonal (device). */
bt_status bt_stencil_create(const bt_grid* g, const bt_form* form, int level, bt_stencil** out);
void bt_stencil_destroy(bt_stencil* s);
/* StencilTable::rows / diagonal (host copies) */
bt_status bt_stencil_rows(const bt_stencil* s, double* rows15xcells);
bt_status bt_stencil_diagonal(const bt_stencil* s, double* diag, void* stream);
/* apply_stencil (operators.hpp:247): y = A x, interface sync, Dirichlet rows */
bt_status bt_apply_stencil(const bt_stencil* s, const double* x, double* y, int bc, void* stream);
/* The two phases of bt_apply_stencil, exposed for overlap and measurement:
 * (1) per-cell rows — merged 15-point rows on interior vertices, per-cell
 *     partial rows on lattice-boundary vertices (operators.hpp:255-268);
 * (2) the interface pass — replica sums over macro faces/edges/vertices
 *     (sync_additive fe_function.hpp:400) and Dirichlet identity rows. */
bt_status bt_apply_stencil_cells(const bt_stencil* s, const double* x, double* y, void* stream);
bt_status bt_apply_stencil_interface(const bt_stencil* s, const double* x, double* y, int bc,
                                     void* stream);
/* apply_elementwise (operators.hpp:115): on-the-fly element integration
 * (4-point rule for k, forms.hpp:107-118), sync, Dirichlet rows.
 * ADD mode needs a scratch level array (NULL: allocated internally). */
bt_status bt_apply_elementwise(const bt_grid* g, const bt_form* form, int level, const double* x,
                               double* y, int mode, int bc, double* scratch, void* stream);
/* extract_diagonal (operators.hpp:277) */
bt_status bt_extract_diagonal(const bt_grid* g, const bt_form* form, int level, double* diag,
                              void* stream);

/* ---- transfers (solvers.hpp:227-293) ------------------------------------ */
/* prolongate_p1; add != 0 fuses v_cycle's axpy(x, 1, ef) (solvers.hpp:536-538) */
bt_status bt_prolongate(const bt_grid* g, int fine_level, const double* coarse, double* fine,
                        int add, void* stream);
/* restrict_p1 (includes the coarse sync_additive) */
bt_status bt_restrict(const bt_grid* g, int fine_level, const double* fine, double* coarse,
                      void* stream);

/* ---- hierarchy / smoothers / multigrid (solvers.hpp:308-541) ------------ */
typedef struct {     /* SmootherConfig (solvers.hpp:379) */
  int kind;          /* 0 jacobi, 1 gauss-seidel, 2 chebyshev */
  double omega;
  int order;
  double lo, hi;
  int nu1, nu2;
} bt_smoother_config;
typedef struct {     /* MultigridConfig (solvers.hpp:498) */
  int coarse_level;
  int cycles;
  double coarse_tol;
  int coarse_maxit;
} bt_multigrid_config;
/* make_hierarchy (solvers.hpp:323); kernel: 0 elementwise, 1 stencil */
bt_status bt_hierarchy_create(const bt_grid* g, const bt_form* form, int kernel,
                              bt_hierarchy** out);
void bt_hierarchy_destroy(bt_hierarchy* h);
bt_status bt_hierarchy_apply(bt_hierarchy* h, int level, const double* x, double* y, int bc,
                             void* stream);                            /* :352 */
bt_status bt_hierarchy_diagonal(bt_hierarchy* h, int level, const double** diag);
bt_status bt_estimate_lambda_max(bt_hierarchy* h, int level, double* out, void* stream); /* :362 */
bt_status bt_smooth(bt_hierarchy* h, const bt_smoother_config* cfg, const double* rhs, double* x,
                    int level, int sweeps, int backward, void* stream);  /* :460 */
/* cg (solvers.hpp:84) through hierarchy_apply with Dirichlet rows;
 * hist[0..maxit-1] receives relative residuals (may be NULL). */
bt_status bt_cg(bt_hierarchy* h, int level, double tol, int maxit, const double* rhs, double* x,
                double* hist, int* iterations, void* stream);
bt_status bt_v_cycle(bt_hierarchy* h, int level, const double* rhs, double* x,
                     const bt_smoother_config* sm, const bt_multigrid_config* mg,
                     void* stream);                                     /* :509 */

/* gauss_seidel_sweep (operators.hpp:327-387): in-place lexicographic
 * Gauss-Seidel on every cell's interior (bitwise the sequential order, by
 * hyperplane wavefronts), then Jacobi with the assembled diagonal on the
 * synced residual at the other vertices; Dirichlet rows pinned to rhs.
 * scratch: a P1 vector of the table's level (NULL: allocated per call). */
bt_status bt_gauss_seidel_sweep(const bt_stencil* table, const double* rhs, double* x, int backward,
                                double* scratch, void* stream);

/* ---- model-problem tools: interpolation, L2 error, full multigrid ---------
 * A device-evaluable scalar field replaces the reference's std::function
 * (same kinds as the div_k_grad coefficient): 0 c0; 1 c0 + c1 sin(c2 x)
 * sin(c2 y) sin(c2 z); 2 c0 + c1 x + c2 y + c3 z. */
typedef struct {
  int kind;
  double c[4];
} bt_field;
/* interpolate (fe_function.hpp:454-477), P1: x = f at every vertex, then
 * sync_broadcast (collective on a partitioned grid) */
bt_status bt_interpolate(const bt_grid* g, int level, const bt_field* f, double* x, void* stream);
/* l2_error (solvers.hpp:613-648): || u_h - exact ||_L2 by the 4-point rule per
 * micro-cell */
bt_status bt_l2_error(const bt_grid* g, int level, const double* x, const bt_field* exact, double* out,
                      void* stream);
typedef struct {      /* IterationRow (solvers.hpp:21) */
  int level, cycle;
  double residual;    /* relative to the level's rhs norm */
  double error;       /* l2_error against `exact`, 0 without one */
} bt_fmg_row;
/* fmg (solvers.hpp:547-604): CG on the coarse level, then per finer level
 * prolongate, impose the level's Dirichlet values and run mg->cycles
 * V-cycles. rhs_levels[i] belongs to level coarse_level + i; x (level
 * finest) receives the solution. rows: 1 + cycles * (finest - coarse_level)
 * entries (max_rows checked). exact may be NULL. */
bt_status bt_fmg(bt_hierarchy* h, int finest, const double* const* rhs_levels, double* x,
                 const bt_smoother_config* sm, const bt_multigrid_config* mg, const bt_field* exact,
                 bt_fmg_row* rows, int max_rows, int* nrows, void* stream);

/* ---- multi-GPU: cell partition --------------------------
 * One process per GPU, each with its own bt_grid. bt_grid_set_partition
 * gives a handle the contiguous cell block [rank*nc/nranks,
 * (rank+1)*nc/nranks). Vectors are memory-sharded: on a partitioned grid
 * every vector argument holds that block only (bt_space_size is the local
 * size, same layout). Set the partition before allocating vectors and before
 * bt_stencil_create. Interface groups with members on several ranks go
 * through an exchange buffer of bt_xchg_size doubles:
 *   bt_apply_stencil_cells(s, x, y)     per-cell rows of this rank's cells
 *   bt_xchg_pack(g, l, y, buf)          this rank's replica values, zeros elsewhere
 *   allreduce(buf, sum) over ranks      the ranks' collective (NCCL / gloo)
 *   bt_xchg_finish(g, l, mode, y, x, buf)  local groups + member-order sums
 * mode: 0 sync_additive, 1 sync with Dirichlet identity rows (src = x),
 * 2 sync_broadcast, 3 impose_dirichlet, 4 zero_dirichlet. Replica sums run
 * in ascending cell order, so results are bitwise independent of nranks.
 *
 * With an allreduce hook (bt_grid_set_allreduce) the library runs that
 * protocol itself, and every P1 entry point works on a partitioned grid as a
 * collective (all ranks call it in the same order): bt_apply_stencil,
 * bt_apply_elementwise, bt_extract_diagonal, bt_sync_*, bt_dot, transfers,
 * hierarchies, smoothers, CG and the V-cycle. Without a hook they return
 * BT_LOGIC_ERROR on a partitioned grid. bt_random_fill never calls the hook:
 * on a partitioned grid it fills the block (its part of the single-GPU
 * stream) and broadcasts the rank-local groups; finish with
 * bt_exchange(mode 2). The edge space (N1E1 operator, edge syncs, dots,
 * random_fill) runs partitioned through its own signed exchange, as a
 * collective (random_fill included).
 *
 * The hook sums n doubles at buf (device memory) over the ranks in place
 * and returns 0 on success. It is stream-ordered: buf is complete once the
 * work queued on `stream` before the call has run, and the sum must be in
 * buf for the work queued on `stream` after it (e.g. ncclAllReduce on
 * `stream`; a hook may also synchronize and block). Every entry a rank
 * contributes is either its own value or 0, so the sum is exact in any
 * order. */
typedef int (*bt_allreduce_fn)(double* buf, int64_t n, void* stream, void* user);
bt_status bt_grid_set_allreduce(bt_grid* g, bt_allreduce_fn fn, void* user);
/* Native data plane (no hook, no Python): an NCCL communicator over the
 * ranks, created by every rank from one unique id (rank 0 draws it with
 * bt_comm_unique_id and the ranks share its 128 bytes out of band). With a
 * communicator set (bt_grid_set_comm; it takes precedence over the hook):
 *   - the interface exchange is neighbour-only: each rank sends to each peer
 *     only its members of the rank-spanning groups it shares with that peer
 *     and receives the peer's (grouped ncclSend / ncclRecv on the call's
 *     stream), instead of an allreduce of the whole exchange buffer;
 *   - dot partials are summed by ncclAllReduce.
 * The communicator's (rank, nranks) must be the grid's partition. NCCL is
 * loaded at bt_comm_create (libnccl.so.2, the one already in the process if
 * any). The caller owns the communicator and destroys it after the grids
 * that use it. */
bt_status bt_comm_unique_id(uint8_t id[128]);
bt_status bt_comm_create(const uint8_t id[128], int rank, int nranks, int device, bt_comm** out);
void bt_comm_destroy(bt_comm* c);
bt_status bt_grid_set_comm(bt_grid* g, bt_comm* c); /* NULL detaches */
/* host-only neighbour plan of the P1 exchange of `rank`: which = 0 the
 * (peer, buffer position) pairs it sends, 1 those it receives, in the order
 * the messages carry them; NULL arrays query the count. -1 on error. */
int64_t bt_xchg_peers_host(const char* mesh_text, int level, int rank, int nranks, int which, int32_t* peer,
                           int32_t* pos);
/* The same neighbour exchange over a caller transport (e.g. MPI, gloo): fn
 * sends peer i the doubles sendbuf[send_off[i], send_off[i+1]) and receives
 * recvbuf[recv_off[i], recv_off[i+1]) from it, for the npeers peers (ranks,
 * ascending), stream-ordered like the allreduce hook; returns 0 on success.
 * Used when no communicator is set; it takes precedence over the hook. */
typedef int (*bt_sendrecv_fn)(int npeers, const int* peers, const int64_t* send_off, const int64_t* recv_off,
                              const double* sendbuf, double* recvbuf, void* stream, void* user);
bt_status bt_grid_set_sendrecv(bt_grid* g, bt_sendrecv_fn fn, void* user);
/* pack + hook + finish in one call (mode as bt_xchg_finish) */
bt_status bt_exchange(const bt_grid* g, int level, int mode, double* x, const double* src, void* stream);
bt_status bt_grid_set_partition(bt_grid* g, int rank, int nranks);
bt_status bt_grid_partition(const bt_grid* g, int* rank, int* nranks, int* cell_begin, int* cell_end);
int64_t bt_xchg_size(const bt_grid* g, int level); /* -1 on error */
bt_status bt_xchg_pack(const bt_grid* g, int level, const double* x, double* buf, void* stream);
bt_status bt_xchg_finish(const bt_grid* g, int level, int mode, double* x, const double* src, const double* buf,
                         void* stream);
/* owned-DoF dot partials per cell (host array of bt_num_cells doubles; cells
 * of other ranks are 0): sum them in cell order after an allreduce */
bt_status bt_dot_cells(const bt_grid* g, int space, int level, const double* x, const double* y, double* per_cell,
                       void* stream);
/* host-only exchange plan (no CUDA needed): entries of `rank`; NULL arrays
 * query the count. Returns the entry count, -1 on error. */
int64_t bt_xchg_plan_host(const char* mesh_text, int level, int rank, int nranks, int64_t* buf_size,
                          int64_t* slot, int32_t* buf, int32_t* base, int32_t* count, uint8_t* dir);

/* ---- N1E1 curl-curl + mass (no reference implementation) ----- */
bt_status bt_n1e1_create(const bt_grid* g, int level, double alpha, double beta, bt_n1e1** out);
void bt_n1e1_destroy(bt_n1e1* op);
bt_status bt_apply_n1e1(const bt_n1e1* op, const double* x, double* y, int bc, void* stream);
bt_status bt_n1e1_sync(const bt_grid* g, int level, double* x, void* stream);

#ifdef __cplusplus
}
#endif
#endif
