// Internal structures of the blocktet_b200 library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <map>
#include <memory>
#include <vector>

#include "../../include/blocktet_b200.h"
#include "bt_index.cuh"

namespace bt {

// ---------------------------------------------------------------------------
// errors: exceptions inside, statuses at the C boundary
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
  bt_status status;
  Error(bt_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] inline void raise(bt_status s, const std::string& m) { throw Error(s, m); }
void set_error(const std::string& m);

#define BT_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      ::bt::raise(BT_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_));  \
  } while (0)

// C-ABI entry point bodies: exceptions inside, statuses at the boundary.
bool nvtx_enabled();  // BT_NVTX=1 (bt_host.cpp)
void nvtx_push(const char* name);
void nvtx_pop();
struct NvtxRange {
  bool on;
  explicit NvtxRange(const char* name) : on(nvtx_enabled()) {
    if (on) nvtx_push(name);
  }
  ~NvtxRange() {
    if (on) nvtx_pop();
  }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
// Every C-ABI entry point opens an NVTX range named after itself when BT_NVTX=1 (nsys / ncu --nvtx timelines of
// the applies, cycles and transfers; off by default: one predictable branch per call).
#define BT_TRY                            \
  ::bt::NvtxRange bt_nvtx_range_(__func__); \
  try {
#define BT_CATCH                                     \
  }                                                  \
  catch (const ::bt::Error& e) {                     \
    ::bt::set_error(e.what());                       \
    return e.status;                                 \
  }                                                  \
  catch (const std::bad_alloc&) {                    \
    ::bt::set_error("out of host memory");           \
    return BT_RUNTIME_ERROR;                         \
  }                                                  \
  catch (const std::exception& e) {                  \
    ::bt::set_error(e.what());                       \
    return BT_LOGIC_ERROR;                           \
  }                                                  \
  return BT_OK;

extern std::atomic<uint64_t> g_launches;
inline void count_launch(int n = 1) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
void check_launch(const char* what);

// Device buffer owned by the library.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) BT_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  void upload(const std::vector<T>& h) {
    alloc(h.size());
    if (n) BT_CUDA(cudaMemcpy(p, h.data(), sizeof(T) * n, cudaMemcpyHostToDevice));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// ---------------------------------------------------------------------------
// macro mesh (coarse_mesh.hpp) and implicit interface tables
// ---------------------------------------------------------------------------
struct Mesh {
  std::vector<std::array<double, 3>> coords;
  std::vector<std::array<int, 4>> cells;        // after orientation repair
  std::vector<std::array<int, 3>> faces;        // sorted triples, lexicographic
  std::vector<std::array<int, 2>> face_cells;   // ascending, -1 if none
  std::vector<char> bflags;
  std::vector<std::array<int, 2>> edges;        // sorted pairs, lexicographic
  int warnings = 0;
  int n_cells() const { return (int)cells.size(); }
};
Mesh parse_mesh(const std::string& text);
struct Topology;
void build_topology(const Mesh& m, Topology& t);

// Affine map x = A r + b of a macro-cell (coarse_mesh.hpp:84-105).
struct CellMap {
  double a[9];  // row-major
  double b[3];
};

// Device-side interface records. Global face vertices / edge endpoints are
// sorted ascending; lv maps them to the local vertex index in each cell.
struct DevFace {
  int ncell;
  int cell[2];
  int8_t lv[2][3];
  uint8_t dir;
};
struct DevPrimHdr {  // macro edge or vertex
  int first, count;
  uint8_t dir;
};
struct DevPrimMem {
  int cell;
  int8_t lv[2];  // edge: local indices of (e0, e1); vertex: lv[0]
};
// Per-cell bits indexed by the zero set Z (bt::zero_set).
struct DevCellInfo {
  uint16_t owned_by_z;
  uint16_t dir_by_z;
};

// Interface work lists (indices into Topology::faces / ehdr / vhdr).
struct IfaceLists {
  std::vector<int> face_shared, face_bdir, edge_act, vert_act;
  DevBuf<int> d_face_shared, d_face_bdir, d_edge_act, d_vert_act;
  void upload() {
    d_face_shared.upload(face_shared);
    d_face_bdir.upload(face_bdir);
    d_edge_act.upload(edge_act);
    d_vert_act.upload(vert_act);
  }
};

// Exchange plan for interface groups whose members lie on several ranks.
// The exchange buffer holds, for every such group (faces, then macro edges,
// then macro vertices in topology order; points in the interface kernel's
// order), one double per member in ascending cell order. Each rank writes its
// members' values (bt_xchg_pack), the caller sums the buffers over ranks, and
// each rank then reduces every group in member order (bt_xchg_combine) — the
// same order as a single-handle sync, so results do not depend on the rank
// count. One entry per member on this rank:
struct XEntry {
  int64_t slot;   // element index in the full-size vector
  int32_t buf;    // this member's value in the buffer
  int32_t base;   // first member of the group
  int32_t count;  // members in the group
  int32_t dir;    // group is Dirichlet-constrained
  int32_t sign = 1;  // replica orientation (N1E1 edges: -1 when the cell's edge runs the other way)
};
struct XPlan {
  bool built = false;
  int64_t buf_size = 0;
  std::vector<XEntry> entries;
  DevBuf<XEntry> d_entries;
  // P1 plans: each entry's lattice point (cell, i, j, k), for the fused
  // stencil apply, which computes this rank's members' partial rows straight
  // into the exchange buffer (k_xpartials, bt_stencil.cu)
  DevBuf<int4> d_pts;
  // neighbour-only exchange (bt_comm): (peer, buffer position) of this
  // rank's members of groups shared with the peer (sends), and of the peer's
  // members of groups with a member here (recvs), in group order on every
  // rank, so rank r's sends to p are p's recvs from r, entry for entry
  std::vector<std::pair<int, int32_t>> sends, recvs;
  // built on first exchange (exchange_buffer)
  mutable bool nbr_built = false;
  mutable std::vector<int> peers;                  // ascending
  mutable std::vector<int64_t> send_off, recv_off;  // per peer, CSR (peers + 1)
  mutable DevBuf<int32_t> d_send_pos, d_recv_pos;
  mutable DevBuf<double> d_sendbuf, d_recvbuf;
  void reset() {
    built = false;
    buf_size = 0;
    entries.clear();
    d_entries.release();
    d_pts.release();
    sends.clear();
    recvs.clear();
    nbr_built = false;
    peers.clear();
    send_off.clear();
    recv_off.clear();
    d_send_pos.release();
    d_recv_pos.release();
    d_sendbuf.release();
    d_recvbuf.release();
  }
};
// record the neighbour traffic of one rank-spanning group: owner[m] is the
// rank of member m, positions off .. off + count - 1
void xplan_group_peers(XPlan& p, int rank, const int* owner, int count, int64_t off);

// fast-kernel march schedule of one layer-group size (see bt_stencil.cu)
// A balanced per-warp schedule of the fast marches of one chunk of cells for
// a grid of G persistent warps (bt_stencil.cu: build_sched)
struct FastSched {
  DevBuf<int4> d_tasks;  // slot s of warp g at s * G + g; empty slots are null tasks (w < z)
  int ntasks = 0;        // slots * G
};
struct FastTasks {
  DevBuf<int4> d_tasks;
  int ntasks = 0;
  std::vector<int> chunk_first;  // first task of each kMaxCells-cell chunk (+ end)
  // whole column segments (k, column block, j0, j1) of one cell, unsplit: the
  // source of the balanced schedules, built per (chunk, G) on first use
  std::vector<int4> segs;
  mutable std::map<std::pair<int, int>, std::unique_ptr<FastSched>> sched;
  mutable DevBuf<int> d_ctr;  // dynamic schedule: task queue head + finished-warp count (self-resetting)
};
struct EwCell;
struct EwTables;

struct Topology {
  // incidence (cells ascending)
  std::vector<std::vector<int>> edge_cells, vert_cells;
  std::vector<std::array<int, 4>> cell_faces;  // local face v -> global face
  std::vector<std::array<int, 6>> cell_edges;  // local edge (a<b) -> global edge
  std::vector<char> edge_dir, vert_dir;
  std::vector<DevCellInfo> info;               // per cell
  std::vector<CellMap> maps;
  // flattened device tables
  std::vector<DevFace> faces;
  std::vector<DevPrimHdr> ehdr, vhdr;
  std::vector<DevPrimMem> emem, vmem;
};

// local edge index of local vertices (a, b), a < b: (0,1)(0,2)(0,3)(1,2)(1,3)(2,3)
inline int local_edge(int a, int b) {
  if (a > b) std::swap(a, b);
  static const int tbl[4][4] = {{-1, 0, 1, 2}, {0, -1, 3, 4}, {1, 3, -1, 5}, {2, 4, 5, -1}};
  return tbl[a][b];
}

}  // namespace bt

// Opaque ABI handles --------------------------------------------------------
struct bt_grid {
  int device = 0;
  int lo = 2, hi = 2;
  bt::Mesh mesh;
  bt::Topology topo;
  bt::DevBuf<bt::DevFace> d_faces;
  bt::DevBuf<bt::DevPrimHdr> d_ehdr, d_vhdr;
  bt::DevBuf<bt::DevPrimMem> d_emem, d_vmem;
  bt::DevBuf<bt::DevCellInfo> d_info;
  // interface work lists: shared faces (2 cells), constrained boundary faces,
  // edges / vertices that are shared or constrained. `full` covers every
  // cell; `loc` only the groups whose members all lie in this handle's cell
  // partition (== full when unpartitioned).
  bt::IfaceLists full, loc;
  // cell partition (bt_grid_set_partition): this handle computes cells
  // [part_begin, part_end) of rank part_rank out of part_nranks
  int part_rank = 0, part_nranks = 1, part_begin = 0, part_end = 0;
  // bumped by every bt_grid_set_partition: objects built for one partition
  // (stencil tables, hierarchies, N1E1 operators) refuse to run on another
  int part_epoch = 0;
  mutable std::array<bt::XPlan, 11> xplan;  // per level, built on first use
  mutable std::array<bt::XPlan, 11> xplan_edges;  // the same for N1E1 edge replicas
  // the ranks' sum-allreduce (bt_grid_set_allreduce): lets the library run
  // the exchange itself inside syncs, dots and solvers
  bt_allreduce_fn allreduce = nullptr;
  void* allreduce_user = nullptr;
  bt_comm* comm = nullptr;  // native data plane (bt_grid_set_comm), takes precedence over the hook
  bt_sendrecv_fn sendrecv = nullptr;  // neighbour exchange over a caller transport (bt_grid_set_sendrecv)
  void* sendrecv_user = nullptr;
  mutable bt::DevBuf<double> xbuf;       // exchange buffer of the library's own syncs
  mutable bt::DevBuf<double> dot_cells;  // per-cell dot partials of every cell (partitioned dots)
  // elementwise-kernel tables per (form, level), built on first use
  mutable std::vector<std::unique_ptr<bt::EwTables>> ew_cache;
  mutable bt::DevBuf<double> ew_scratch;  // ApplyMode::Add without a caller scratch
  // elementwise work lists per level (bt_ew.cu: row tasks, tile units), built on first use
  mutable std::array<bt::DevBuf<int4>, 11> ew_rows, ew_tiles, ew_rowtab;
  mutable std::array<int, 11> ew_nrows{}, ew_ntiles{};
  // reduction scratch for dot products
  mutable bt::DevBuf<double> d_partials;
  mutable bt::DevBuf<double> d_maps;  // per cell: the affine map (a row-major, b), built on first use
  mutable double* h_pinned = nullptr;
  ~bt_grid();
};

namespace bt {
// Per-cell stencil data: zero-set-typed rows (type 0 = merged interior row,
// compute_stencil operators.hpp:204-221), and a bitmask of present
// directions per type.
struct StencilCell {
  double w[16][15];
  uint32_t mask[16];
};
// Per-cell data for the elementwise kernel (bt_ew.cu).
struct EwCell {
  double G[6][16];      // class matrices (diffusion for div_k_grad; else the form)
  double beta[3][3];    // coeff kind 1: phase slope f * A[d][e] * h per lattice direction e
  double coefh[6][8];   // coeff kind 1: c1/4 sum_q prod_d (bit d of m ? sin : cos)(gamma_{s,q,d})
  double lin[3];        // coeff kind 2: c . (A h) per lattice direction
  double lin0[6];       // coeff kind 2: c0 + c . (A h centroid_s + b)
};
struct EwTables {  // device tables of one (form, level) for the elementwise kernel
  bt_form form{};
  int level = 0;
  DevBuf<EwCell> cells;
  std::vector<EwCell> host;  // the same on the host (kernel-parameter weights)
  DevBuf<double> phase;  // sin-product phase tables of this handle's cells (build_ew_phase)
};
// per-cell sin/cos tables of the sin-product phases (k_ew_row), this handle's cells
void build_ew_phase(const bt_grid& g, int level, const EwCell* d_cells, DevBuf<double>& out);
const EwTables& ew_tables(const bt_grid& g, const bt_form& f, int level);
}  // namespace bt

struct bt_stencil {
  const bt_grid* grid = nullptr;
  int level = 0;
  bt_form form{};
  std::vector<std::array<double, 15>> rows;  // host copy of StencilTable::rows
  bt::DevBuf<bt::StencilCell> d_cells;
  mutable bt::DevBuf<double> d_diag;         // assembled diagonal (this handle's cells), built on first use
  bt::FastTasks fast4, fast2;                // fast-kernel marches: 4-layer groups, the 2-layer group
  int part_begin = 0, part_end = 0;          // the grid's cell partition when the tasks were built
  bt::DevBuf<int4> d_gtasks;                 // general rows (layer 0, row 0, corner rows)
  int ngtasks = 0;
  bt::DevBuf<int4> d_atasks;                 // all rows (general-kernel fallback)
  int natasks = 0;
  bool symmetric = false;                    // fast-path preconditions hold (see bt_stencil.cu)
  std::vector<double> fast;                  // per cell: the 8 symmetric interior weights
  bt::DevBuf<double> d_ends;                 // per cell: typed rows of the two row ends (11 + 11)
  bt::DevBuf<int> bnd_f, bnd_e, bnd_v;       // k_boundary: faces / macro edges / vertices with every member local
  bt::DevBuf<int4> d_ftasks;                 // k_face_march tasks (strided faces' partial rows)
  int nftasks = 0;
  mutable bt::DevBuf<double> d_fpart;        // ... their output, read by k_boundary (allocated on first use)
  bt::DevBuf<int4> d_prism;                  // k_stencil_prism units (bt_prism.cu), longest first
  int nprism = 0;
  bt::DevBuf<double> d_w8;                   // per cell (global index): the 8 symmetric weights
  bt::DevBuf<int> d_prism_ctr;               // unit queue + finished-CTA counter (self-resetting)
};

namespace bt {
// host helpers shared between translation units
void class_matrices(const bt_grid& g, int form_kind, int level, int cell, double out[6][16]);
void build_stencil_cells(const bt_grid& g, const bt_form& f, int level,
                         std::vector<StencilCell>& cells, std::vector<std::array<double, 15>>& rows);
void build_ew_cells(const bt_grid& g, const bt_form& f, int level, std::vector<EwCell>& cells);
int64_t level_slots(int space, int level);  // per cell
// Vectors of a partitioned grid hold the rank's cells [part_begin, part_end)
// only; every pointer inside the library is such a local pointer. Kernels
// index by global cell, so the launchers shift the pointer back by
// part_begin cells (only local cells are ever touched).
int64_t part_shift(const bt_grid& g, int space, int level);
template <class T>
T* shifted(T* p, const bt_grid& g, int space, int level) {
  return p ? p - part_shift(g, space, level) : p;
}
void validate_form(const bt_form* f);
// entry points that need every group local (no exchange step) refuse a
// partitioned grid
void require_unpartitioned(const bt_grid* g, const char* what);
void check_level(const bt_grid* g, int level);

// kernel launchers (bt_kernels.cu)
enum IfaceMode { IF_SYNC = 0, IF_SYNC_DIR = 1, IF_BCAST = 2, IF_IMPOSE = 3, IF_ZERO_DIR = 4, IF_ZERO_NONOWNED = 5 };
// The groups local to this handle's partition (g.loc; every group when
// unpartitioned). Local pointers.
void launch_interface(const bt_grid& g, int level, IfaceMode mode, double* v, const double* src,
                      cudaStream_t s);
// Every interface group of a P1 vector, whatever the partition: the local
// pass plus, on a partitioned grid, pack -> allreduce hook -> member-order
// combine for rank-spanning groups (collective: every rank calls it).
void sync(const bt_grid& g, int level, IfaceMode mode, double* v, const double* src, cudaStream_t s);
// the grid's allreduce hook on n doubles (raises if none is set)
void allreduce(const bt_grid& g, double* buf, int64_t n, cudaStream_t s);
// the exchange step of a rank-spanning sync: buf holds this rank's members
// (zeros elsewhere); afterwards every position of every group with a member
// here holds its member's value. Neighbour-only send/recv over the grid's
// communicator, else the allreduce hook.
void exchange_buffer(const bt_grid& g, const XPlan& p, double* buf, cudaStream_t s);
// NCCL (bt_comm.cpp): grouped send/recv with each peer, stream-ordered
void comm_check(const bt_comm* c, int rank, int nranks);
void comm_sendrecv(bt_comm* c, const std::vector<int>& peers, const std::vector<int64_t>& send_off,
                   const std::vector<int64_t>& recv_off, const double* sendbuf, double* recvbuf, cudaStream_t s);
void comm_allreduce(bt_comm* c, double* buf, int64_t n, cudaStream_t s);
// assembled diagonal of a stencil table (collective on a partitioned grid)
const double* stencil_diag(const bt_stencil& st, cudaStream_t s);
// exchange for rank-spanning groups (bt_xchg.cu)
const XPlan& xchg_plan(const bt_grid& g, int level);
void build_xplan(const Mesh& m, const Topology& t, int level, int rank, int nranks, XPlan& out);
void launch_xchg_pack(const bt_grid& g, int level, const double* x, double* buf, cudaStream_t s);
void launch_xchg_combine(const bt_grid& g, int level, IfaceMode mode, double* x, const double* src,
                         const double* buf, cudaStream_t s);
void partition_range(int nc, int rank, int nranks, int& begin, int& end);
// edge space (N1E1): the exchange of rank-spanning signed edge replicas (bt_n1e1.cu)
const XPlan& xchg_plan_edges(const bt_grid& g, int level);
void launch_xchg_pack_plan(const XPlan& p, int64_t shift, const double* x, double* buf, cudaStream_t s);
void launch_xchg_combine_plan(const XPlan& p, int64_t shift, IfaceMode mode, double* x, const double* src,
                              const double* buf, cudaStream_t s);
// every signed edge-interface group of an edge-space vector (collective when partitioned)
void sync_edges(const bt_grid& g, int level, IfaceMode mode, double* v, const double* src, cudaStream_t s);
// per-cell rows (interior + row ends + general rows); xmode >= 0 also runs
// the interface pass in that mode (IfaceMode, src = x) — with the rank
// exchange on a partitioned grid — overlapped with the interior marches
void launch_stencil(const bt_stencil& st, const double* x, double* y, cudaStream_t s, int xmode = -1);
// the whole apply_stencil (replica sums and, bc != 0, Dirichlet identity rows
// included): interior kernel and fused boundary kernel run concurrently.
// Available when stencil_fused(st): symmetric tables on an unpartitioned grid.
bool stencil_fused(const bt_stencil& st);
void launch_stencil_fused(const bt_stencil& st, const double* x, double* y, int bc, cudaStream_t s);
void init_stencil_tasks(bt_stencil& st);
// interior points of a symmetric table as prism k-marches (bt_prism.cu)
void init_prism_tasks(bt_stencil& st);
bool prism_ok(const bt_stencil& st, const double* x);
void launch_prism(const bt_stencil& st, const double* x, double* y, cudaStream_t s);
// one hybrid Gauss-Seidel sweep (operators.hpp:327-387); scratch: a P1 vector
void launch_gs_sweep(const bt_stencil& st, const double* rhs, double* x, double* scratch, bool backward,
                     cudaStream_t s);
// a second stream (per host thread and device) for kernels that run beside
// the main launch, with fork / join events
struct SideStream {
  cudaStream_t s = nullptr, s2 = nullptr;  // s2: a second side stream (partitioned fused apply)
  cudaEvent_t fork = nullptr, join = nullptr, join2 = nullptr;
};
SideStream& side_stream();
void launch_elementwise(const bt_grid& g, int level, int coeff_kind, const double* c, const EwCell* d_cells,
                        const double* x, double* y, bool diag_only, cudaStream_t s, const double* phase = nullptr,
                        const EwCell* h_cells = nullptr);
// local_matrix's positivity check of a div_k_grad coefficient (bt_ew.cu)
void check_coefficient(const bt_grid& g, const bt_form& f, int level, const double* d_maps, cudaStream_t s);
// per cell: the affine map (a row-major, b), built on first use (bt_kernels.cu)
const double* cell_maps(const bt_grid& g);
void launch_vec(int op, double* y, const double* x, double a, int64_t n, cudaStream_t s);
void launch_fill_by_z(const bt_grid& g, int level, const double* tbl, double* out, cudaStream_t s);
double dot_p1(const bt_grid& g, int level, const double* x, const double* y, cudaStream_t s);
// the owned dot left on the device at *dst (stream-ordered; collective when partitioned)
void dot_p1_device(const bt_grid& g, int level, const double* x, const double* y, double* dst, cudaStream_t s);
// device-resident CG scalars (bt_solvers.cpp cg)
struct CgState {
  double nb2, rs, pap, rs_new, denom, alpha, malpha, beta, one;
  int it, done, breakdown;
};
void launch_cg_init(CgState* st, double tol, cudaStream_t s);
// fused smoother update (kind 0: first Chebyshev step, 1: later steps, 2: Jacobi)
void launch_smooth_update(int kind, double* x, double* d, const double* ax, const double* rhs, const double* diag,
                          double c1, double c2, int64_t n, cudaStream_t s);
// device-resident estimate_lambda_max scalars
struct LamState {
  double num, den, nn2, rho, inv;
  int done, empty, zero_diag;
};
void launch_lam_step(LamState* st, bool first, cudaStream_t s);
// zero_diag = 1 if any entry of diag[0, n) is 0.0 (estimate_lambda_max's precondition, solvers.hpp:143-147)
void launch_lam_check_diag(LamState* st, const double* diag, int64_t n, cudaStream_t s);
void launch_cg_alpha(CgState* st, cudaStream_t s);
void launch_cg_update(CgState* st, double tol, double* hist, cudaStream_t s);
void launch_vec_dev(int op, double* y, const double* x, const double* a, const int* done, int64_t n, cudaStream_t s);
// l2_error (solvers.hpp:613-648) of a P1 function against a field (collective when partitioned)
double l2_error_p1(const bt_grid& g, int level, const double* x, const bt_field& f, cudaStream_t s);
// edge space (N1E1, bt_n1e1.cu): signed replica sync / broadcast, Dirichlet rows
void launch_edge_interface(const bt_grid& g, int level, IfaceMode mode, double* v, const double* src,
                           cudaStream_t s);
double dot_edges(const bt_grid& g, int level, const double* x, const double* y, cudaStream_t s);
void random_fill_edges(const bt_grid& g, int level, uint64_t seed, double* x, cudaStream_t s);
void launch_prolongate(const bt_grid& g, int fine_level, const double* coarse, double* fine, bool add,
                       cudaStream_t s);
void launch_restrict(const bt_grid& g, int fine_level, const double* fine, double* coarse,
                     cudaStream_t s);
enum VecOp { V_ASSIGN = 0, V_SCALE = 1, V_COPY = 2, V_AXPY = 3, V_MUL = 4, V_DIV = 5 };
}  // namespace bt
