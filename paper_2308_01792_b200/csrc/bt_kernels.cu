// Device kernels of blocktet_b200 (sm_100a) and the device-side C ABI.
//
// All kernels address the tetrahedral row layout implicitly: no per-DoF
// index arrays. A warp owns one lattice row (j, k) of one macro-cell at a
// time, its lanes walk i, and the 15 stencil neighbours are fixed offsets of
// the row (bt::row_offsets). Macro-cell interfaces ("ghost layers" of the
// reference: replicated DoFs summed by sync_additive, fe_function.hpp:400)
// are handled by one kernel over macro faces, edges and vertices whose
// member slots are computed from barycentric weights.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "bt_internal.hpp"

namespace bt {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRowsPerCta = 64;

static inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ---------------------------------------------------------------------------
// Row-walk helpers: fill-by-zero-set, owned dot products, transfers
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_fill_by_z(const double* __restrict__ tbl, double* __restrict__ out,
                                                        int w, int64_t cell_slots, int cell0) {
  const int cell = cell0 + blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = w - 1, nrows = tri32(w);
  const int rend = min(nrows, (int)(blockIdx.x + 1) * kRowsPerCta);
  for (int r = blockIdx.x * kRowsPerCta + warp; r < rend; r += kWarps) {
    int j, k;
    decode_row(w, r, j, k);
    const int L = w - j - k, t0 = row_start(w, j, k);
    for (int i = lane; i < L; i += 32) out[(int64_t)cell * cell_slots + t0 + i] = tbl[16 * cell + zero_set(n, i, j, k)];
  }
}

void launch_fill_by_z(const bt_grid& g, int level, const double* tbl, double* out, cudaStream_t s) {
  const int w = (1 << level) + 1;
  const int nc = g.part_end - g.part_begin;
  if (!nc) return;
  dim3 grid(ceil_div(tri32(w), kRowsPerCta), nc);
  k_fill_by_z<<<grid, kThreads, 0, s>>>(tbl, shifted(out, g, BT_SPACE_P1, level), w, n_tet(w), g.part_begin);
  count_launch();
  check_launch("k_fill_by_z");
}

// Deterministic owned-DoF dot: fixed (cell, row block) partials, fixed
// shuffle tree, fixed final order. Independent of the GPU count because
// partials never straddle cells (fe_function.hpp:373-394 order up to
// reassociation).
__global__ void __launch_bounds__(kThreads) k_dot_partial(const double* __restrict__ x, const double* __restrict__ y,
                                                          const DevCellInfo* __restrict__ info, int w,
                                                          int64_t cell_slots, int cell0,
                                                          double* __restrict__ partials) {
  __shared__ double red[kWarps];
  const int cell = cell0 + blockIdx.y;
  const uint16_t own = info[cell].owned_by_z;
  const double* xc = x + (int64_t)cell * cell_slots;
  const double* yc = y + (int64_t)cell * cell_slots;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = w - 1, nrows = tri32(w);
  const int rend = min(nrows, (int)(blockIdx.x + 1) * kRowsPerCta);
  double acc = 0.0;
  for (int r = blockIdx.x * kRowsPerCta + warp; r < rend; r += kWarps) {
    int j, k;
    decode_row(w, r, j, k);
    const int L = w - j - k, t0 = row_start(w, j, k);
    for (int i = lane; i < L; i += 32)
      if (own >> zero_set(n, i, j, k) & 1) acc = fma(__ldg(xc + t0 + i), __ldg(yc + t0 + i), acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < kWarps; ++q) s += red[q];
    partials[(int64_t)cell * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(1024) k_sum(const double* __restrict__ partials, int64_t n, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < n; q += blockDim.x) acc += partials[q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += red[q];
    *out = s;
  }
}

// Per-cell sums of the row-block partials (fixed order), then the cells in
// order: the same association on any number of GPUs (bt_dot_cells).
__global__ void k_cell_sums(const double* __restrict__ partials, int per_cell, int cell0, int ncells,
                            double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const double* p = partials + (int64_t)(cell0 + c) * per_cell;
  double s = 0.0;
  for (int q = 0; q < per_cell; ++q) s += p[q];
  out[c] = s;
}
__global__ void k_ordered_sum(const double* __restrict__ v, int n, double* out) {
  double s = 0.0;
  for (int q = 0; q < n; ++q) s += v[q];
  *out = s;
}

// owned dot over this handle's cells: per-cell sums into host[cell_begin..
// cell_end) and/or into dev_cells[0 .. cells of the handle) (device); total !=
// nullptr: also their ordered sum
static void dot_p1_cells(const bt_grid& g, int level, const double* x, const double* y, cudaStream_t s,
                         double* host_cells, double* total, double* dev_cells = nullptr) {
  const int w = (1 << level) + 1;
  const int bx = ceil_div(tri32(w), kRowsPerCta);
  const int nc = g.mesh.n_cells(), c0 = g.part_begin, nl = g.part_end - g.part_begin;
  const int64_t np = (int64_t)bx * nc;
  if (g.d_partials.n < (size_t)(np + nc + 1)) g.d_partials.alloc((size_t)(np + nc + 1));
  double* cells = dev_cells ? dev_cells : g.d_partials.p + np;
  x = shifted(x, g, BT_SPACE_P1, level);
  y = shifted(y, g, BT_SPACE_P1, level);
  if (nl) {
    k_dot_partial<<<dim3(bx, nl), kThreads, 0, s>>>(x, y, g.d_info.p, w, n_tet(w), c0, g.d_partials.p);
    k_cell_sums<<<ceil_div(nl, 128), 128, 0, s>>>(g.d_partials.p, bx, c0, nl, cells);
    count_launch(2);
  }
  if (total) {
    k_ordered_sum<<<1, 1, 0, s>>>(cells, nl, g.d_partials.p + np + nc);
    count_launch();
  }
  check_launch("k_dot");
  if (host_cells && nl)
    BT_CUDA(cudaMemcpyAsync(host_cells + c0, cells, sizeof(double) * nl, cudaMemcpyDeviceToHost, s));
  if (total) BT_CUDA(cudaMemcpyAsync(g.h_pinned, g.d_partials.p + np + nc, sizeof(double), cudaMemcpyDeviceToHost, s));
  if (host_cells || total) BT_CUDA(cudaStreamSynchronize(s));
  if (total) *total = g.h_pinned[0];
}

double dot_p1(const bt_grid& g, int level, const double* x, const double* y, cudaStream_t s) {
  double t = 0.0;
  if (g.part_nranks == 1) {
    dot_p1_cells(g, level, x, y, s, nullptr, &t);
    return t;
  }
  // partitioned: this rank's per-cell partials into an every-cell array
  // (zeros elsewhere), allreduce, then the cells in order as on one GPU
  const int nc = g.mesh.n_cells();
  if (g.dot_cells.n < (size_t)nc + 1) g.dot_cells.alloc((size_t)nc + 1);
  BT_CUDA(cudaMemsetAsync(g.dot_cells.p, 0, sizeof(double) * (size_t)nc, s));
  dot_p1_cells(g, level, x, y, s, nullptr, nullptr, g.dot_cells.p + g.part_begin);
  allreduce(g, g.dot_cells.p, nc, s);
  k_ordered_sum<<<1, 1, 0, s>>>(g.dot_cells.p, nc, g.dot_cells.p + nc);
  count_launch();
  check_launch("k_ordered_sum");
  BT_CUDA(cudaMemcpyAsync(g.h_pinned, g.dot_cells.p + nc, sizeof(double), cudaMemcpyDeviceToHost, s));
  BT_CUDA(cudaStreamSynchronize(s));
  return g.h_pinned[0];
}

// the same owned dot, left on the device at *dst (stream-ordered, no host sync)
void dot_p1_device(const bt_grid& g, int level, const double* x, const double* y, double* dst, cudaStream_t s) {
  const int nc = g.mesh.n_cells();
  if (g.part_nranks == 1) {
    const int w = (1 << level) + 1;
    const int bx = ceil_div(tri32(w), kRowsPerCta);
    const int64_t np = (int64_t)bx * nc;
    if (g.d_partials.n < (size_t)(np + nc + 1)) g.d_partials.alloc((size_t)(np + nc + 1));
    dot_p1_cells(g, level, x, y, s, nullptr, nullptr, g.d_partials.p + np);
    k_ordered_sum<<<1, 1, 0, s>>>(g.d_partials.p + np, nc, dst);
  } else {
    if (g.dot_cells.n < (size_t)nc + 1) g.dot_cells.alloc((size_t)nc + 1);
    BT_CUDA(cudaMemsetAsync(g.dot_cells.p, 0, sizeof(double) * (size_t)nc, s));
    dot_p1_cells(g, level, x, y, s, nullptr, nullptr, g.dot_cells.p + g.part_begin);
    allreduce(g, g.dot_cells.p, nc, s);
    k_ordered_sum<<<1, 1, 0, s>>>(g.dot_cells.p, nc, dst);
  }
  count_launch();
  check_launch("k_ordered_sum");
}

// ---------------------------------------------------------------------------
// Device-resident CG scalars (cg, solvers.hpp:84-131): the scalar recurrences
// run in one-thread kernels in the reference's operation order, so no host
// round trip per iteration; `done` stops every later update (convergence or
// breakdown), exactly where the reference returns or throws.
// ---------------------------------------------------------------------------
__global__ void k_cg_init(CgState* st, double tol) {
  const double nb = sqrt(st->nb2);
  st->denom = nb > 0 ? nb : 1.0;
  st->one = 1.0;
  st->it = 0;
  st->breakdown = 0;
  st->done = sqrt(st->rs) / st->denom <= tol ? 1 : 0;
}
__global__ void k_cg_alpha(CgState* st) {
  if (st->done) return;
  if (!(st->pap > 0)) {
    st->breakdown = 1;
    st->done = 1;
    return;
  }
  st->alpha = st->rs / st->pap;
  st->malpha = -st->alpha;
}
__global__ void k_cg_update(CgState* st, double tol, double* hist) {
  if (st->done) return;
  st->it += 1;
  const double r = sqrt(st->rs_new) / st->denom;
  if (hist) hist[st->it - 1] = r;
  if (r <= tol) {
    st->done = 1;
    return;
  }
  st->beta = st->rs_new / st->rs;
  st->rs = st->rs_new;
}
// y = y + a x / y = a y with a read from the device, skipped once done
template <int OP>
__global__ void __launch_bounds__(kThreads) k_vec_dev(double* __restrict__ y, const double* __restrict__ x,
                                                      const double* __restrict__ a, const int* __restrict__ done,
                                                      int64_t n) {
  if (*done) return;
  const double av = *a;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    if (OP == V_SCALE) y[q] = __dmul_rn(y[q], av);
    else y[q] = __dadd_rn(y[q], __dmul_rn(av, x[q]));
  }
}
// Fused Chebyshev / Jacobi update (chebyshev_apply solvers.hpp:425-456,
// smooth 460-492): from ax = A x (Dirichlet identity rows, synced),
//   r = D^-1 (rhs - A x)          (scale(r, -1); axpy(r, 1, rhs); hadamard /)
//   KIND 0 (Chebyshev, first):  d = r * c1                (copy; scale 1/theta)
//   KIND 1 (Chebyshev, later):  d = d * c1 + c2 * r       (scale rho' rho; axpy 2 rho'/delta)
//   KIND 2 (Jacobi):            d = c2 * r (not stored)   (axpy omega)
//   x = x + d
// one pass instead of 6 to 7 streaming passes, every step rounded as the
// reference's separate vector operations round it (bitwise the unfused path)
template <int KIND>
__global__ void __launch_bounds__(kThreads) k_smooth_update(double* __restrict__ x, double* __restrict__ d,
                                                            const double* __restrict__ ax,
                                                            const double* __restrict__ rhs,
                                                            const double* __restrict__ diag, double c1, double c2,
                                                            int64_t n) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const double r = __ddiv_rn(__dadd_rn(__dmul_rn(ax[q], -1.0), __dmul_rn(1.0, rhs[q])), diag[q]);
    double dn;
    if (KIND == 0) dn = __dmul_rn(r, c1);
    else if (KIND == 1) dn = __dadd_rn(__dmul_rn(d[q], c1), __dmul_rn(c2, r));
    else dn = __dmul_rn(c2, r);
    if (KIND != 2) d[q] = dn;
    x[q] = __dadd_rn(x[q], KIND == 2 ? dn : __dmul_rn(1.0, dn));
  }
}

void launch_smooth_update(int kind, double* x, double* d, const double* ax, const double* rhs, const double* diag,
                          double c1, double c2, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  const int blocks = (int)std::min<int64_t>(ceil_div(n, kThreads), (int64_t)148 * 8);
  if (kind == 0) k_smooth_update<0><<<blocks, kThreads, 0, s>>>(x, d, ax, rhs, diag, c1, c2, n);
  else if (kind == 1) k_smooth_update<1><<<blocks, kThreads, 0, s>>>(x, d, ax, rhs, diag, c1, c2, n);
  else k_smooth_update<2><<<blocks, kThreads, 0, s>>>(x, d, ax, rhs, diag, c1, c2, n);
  count_launch();
  check_launch("k_smooth_update");
}

// estimate_lambda_max scalars on the device (solvers.hpp:140-172): after the
// dots num = v.w, den = v.z, nn2 = v.v: rho = num / den, and the scale 1/||v||
// (or stop once ||v|| == 0, where the reference breaks out of its loop)
__global__ void k_lam_step(LamState* st) {
  if (st->done) return;
  st->rho = st->num / st->den;
  const double nn = sqrt(st->nn2);
  if (nn == 0) {
    st->done = 1;
    return;
  }
  st->inv = 1.0 / nn;
}
__global__ void k_lam_norm(LamState* st) {  // the start vector's normalisation
  const double nv = sqrt(st->nn2);
  st->empty = nv == 0 ? 1 : 0;
  st->inv = nv == 0 ? 0.0 : 1.0 / nv;
  st->done = 0;
  st->rho = 0.0;
}
__global__ void k_lam_check_diag(LamState* st, const double* __restrict__ diag, int64_t n) {
  bool zero = false;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    zero = zero || diag[t] == 0.0;
  if (__syncthreads_or(zero) && threadIdx.x == 0) st->zero_diag = 1;
}
void launch_lam_check_diag(LamState* st, const double* diag, int64_t n, cudaStream_t s) {
  BT_CUDA(cudaMemsetAsync(&st->zero_diag, 0, sizeof(int), s));
  if (n > 0) {
    const int blocks = (int)std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 8);
    k_lam_check_diag<<<blocks, kThreads, 0, s>>>(st, diag, n);
    count_launch();
  }
}
void launch_lam_step(LamState* st, bool first, cudaStream_t s) {
  if (first) k_lam_norm<<<1, 1, 0, s>>>(st);
  else k_lam_step<<<1, 1, 0, s>>>(st);
  count_launch();
}

void launch_cg_init(CgState* st, double tol, cudaStream_t s) {
  k_cg_init<<<1, 1, 0, s>>>(st, tol);
  count_launch();
}
void launch_cg_alpha(CgState* st, cudaStream_t s) {
  k_cg_alpha<<<1, 1, 0, s>>>(st);
  count_launch();
}
void launch_cg_update(CgState* st, double tol, double* hist, cudaStream_t s) {
  k_cg_update<<<1, 1, 0, s>>>(st, tol, hist);
  count_launch();
}
void launch_vec_dev(int op, double* y, const double* x, const double* a, const int* done, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  const int blocks = (int)std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 8);
  if (op == V_SCALE) k_vec_dev<V_SCALE><<<blocks, kThreads, 0, s>>>(y, x, a, done, n);
  else k_vec_dev<V_AXPY><<<blocks, kThreads, 0, s>>>(y, x, a, done, n);
  count_launch();
  check_launch("k_vec_dev");
}

// prolongate_p1 (solvers.hpp:227-253), optionally fused with axpy(x, 1, ef)
__global__ void __launch_bounds__(kThreads) k_prolongate(const double* __restrict__ coarse, double* __restrict__ fine,
                                                         int wf, int add, int cell0) {
  const int cell = cell0 + blockIdx.y;
  const int wc = (wf - 1) / 2 + 1;
  const double* cc = coarse + (int64_t)cell * tet32(wc);
  double* fc = fine + (int64_t)cell * tet32(wf);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nrows = tri32(wf);
  const int rend = min(nrows, (int)(blockIdx.x + 1) * kRowsPerCta);
  for (int r = blockIdx.x * kRowsPerCta + warp; r < rend; r += kWarps) {
    int j, k;
    decode_row(wf, r, j, k);
    const int L = wf - j - k, t0 = row_start(wf, j, k);
    for (int i = lane; i < L; i += 32) {
      const int code = (i & 1) | ((j & 1) << 1) | ((k & 1) << 2);
      double value;
      if (code == 0) {
        value = __ldg(cc + row_start(wc, j >> 1, k >> 1) + (i >> 1));
      } else {
        // coarse_endpoints (solvers.hpp:183-211): first / second endpoint
        int a0, b0, c0, a1, b1, c1;
        switch (code) {
          case 1: a0 = i - 1; b0 = j; c0 = k; a1 = i + 1; b1 = j; c1 = k; break;
          case 2: a0 = i; b0 = j - 1; c0 = k; a1 = i; b1 = j + 1; c1 = k; break;
          case 4: a0 = i; b0 = j; c0 = k - 1; a1 = i; b1 = j; c1 = k + 1; break;
          case 3: a0 = i + 1; b0 = j - 1; c0 = k; a1 = i - 1; b1 = j + 1; c1 = k; break;
          case 5: a0 = i + 1; b0 = j; c0 = k - 1; a1 = i - 1; b1 = j; c1 = k + 1; break;
          case 6: a0 = i; b0 = j + 1; c0 = k - 1; a1 = i; b1 = j - 1; c1 = k + 1; break;
          default: a0 = i - 1; b0 = j + 1; c0 = k - 1; a1 = i + 1; b1 = j - 1; c1 = k + 1; break;
        }
        const double v0 = __ldg(cc + row_start(wc, b0 >> 1, c0 >> 1) + (a0 >> 1));
        const double v1 = __ldg(cc + row_start(wc, b1 >> 1, c1 >> 1) + (a1 >> 1));
        value = 0.5 * __dadd_rn(v0, v1);
      }
      if (add) fc[t0 + i] = __dadd_rn(fc[t0 + i], value);
      else fc[t0 + i] = value;
    }
  }
}

void launch_prolongate(const bt_grid& g, int fine_level, const double* coarse, double* fine, bool add, cudaStream_t s) {
  const int wf = (1 << fine_level) + 1;
  const int nc = g.part_end - g.part_begin;
  if (!nc) return;
  dim3 grid(ceil_div(tri32(wf), kRowsPerCta), nc);
  k_prolongate<<<grid, kThreads, 0, s>>>(shifted(coarse, g, BT_SPACE_P1, fine_level - 1),
                                         shifted(fine, g, BT_SPACE_P1, fine_level), wf, add ? 1 : 0, g.part_begin);
  count_launch();
  check_launch("k_prolongate");
}

// restrict_p1 (solvers.hpp:259-293) as a pull over coarse vertices: the fine
// points 2P + d (d a stencil direction) contribute in ascending fine-slot
// order, exactly the reference's scatter order; non-owned fine replicas
// contribute 0.
__global__ void __launch_bounds__(kThreads) k_restrict(const double* __restrict__ fine, double* __restrict__ coarse,
                                                       const DevCellInfo* __restrict__ info, int wc, int cell0) {
  // directions sorted by (dz, dy, dx)
  constexpr int kOrd[15][3] = {{0, 0, -1}, {1, 0, -1}, {-1, 1, -1}, {0, 1, -1}, {0, -1, 0},
                               {1, -1, 0}, {-1, 0, 0}, {0, 0, 0},   {1, 0, 0},  {-1, 1, 0},
                               {0, 1, 0},  {0, -1, 1}, {1, -1, 1},  {-1, 0, 1}, {0, 0, 1}};
  const int cell = cell0 + blockIdx.y;
  const int wf = 2 * (wc - 1) + 1, nf = wf - 1;
  const uint16_t own = info[cell].owned_by_z;
  const double* fc = fine + (int64_t)cell * tet32(wf);
  double* cc = coarse + (int64_t)cell * tet32(wc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nrows = tri32(wc);
  const int rend = min(nrows, (int)(blockIdx.x + 1) * kRowsPerCta);
  for (int r = blockIdx.x * kRowsPerCta + warp; r < rend; r += kWarps) {
    int J, K;
    decode_row(wc, r, J, K);
    const int L = wc - J - K, t0 = row_start(wc, J, K);
    for (int I = lane; I < L; I += 32) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < 15; ++q) {
        const int fi = 2 * I + kOrd[q][0], fj = 2 * J + kOrd[q][1], fk = 2 * K + kOrd[q][2];
        if (!in_i_tet(wf, fi, fj, fk)) continue;
        const double v = (own >> zero_set(nf, fi, fj, fk) & 1) ? __ldg(fc + row_start(wf, fj, fk) + fi) : 0.0;
        if (q == 7) acc = __dadd_rn(acc, v);
        else acc = __dadd_rn(acc, 0.5 * v);
      }
      cc[t0 + I] = acc;
    }
  }
}

void launch_restrict(const bt_grid& g, int fine_level, const double* fine, double* coarse, cudaStream_t s) {
  const int wc = (1 << (fine_level - 1)) + 1;
  const int nc = g.part_end - g.part_begin;
  if (nc) {
    dim3 grid(ceil_div(tri32(wc), kRowsPerCta), nc);
    k_restrict<<<grid, kThreads, 0, s>>>(shifted(fine, g, BT_SPACE_P1, fine_level),
                                         shifted(coarse, g, BT_SPACE_P1, fine_level - 1), g.d_info.p, wc, g.part_begin);
    count_launch();
    check_launch("k_restrict");
  }
  sync(g, fine_level - 1, IF_SYNC, coarse, nullptr, s);
}

// ---------------------------------------------------------------------------
// interpolate (fe_function.hpp:454-477, P1) and l2_error (solvers.hpp:613-648).
// Coordinates follow micro_vertex_coord (micro_index.hpp:266-271) and
// MacroCellMap::map (coarse_mesh.hpp:87) in the reference's operation order,
// unfused (_rn intrinsics).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double eval_field(const bt_field& f, double x, double y, double z) {
  if (f.kind == 0) return f.c[0];
  if (f.kind == 1) {
    const double s = __dmul_rn(__dmul_rn(__dmul_rn(f.c[1], sin(__dmul_rn(f.c[2], x))), sin(__dmul_rn(f.c[2], y))),
                               sin(__dmul_rn(f.c[2], z)));
    return __dadd_rn(f.c[0], s);
  }
  return __dadd_rn(__dadd_rn(__dadd_rn(f.c[0], __dmul_rn(f.c[1], x)), __dmul_rn(f.c[2], y)), __dmul_rn(f.c[3], z));
}
__device__ __forceinline__ void map_vertex(const double* __restrict__ m, double h, int i, int j, int k,
                                           double out[3]) {
  const double r0 = __dmul_rn(h, (double)i), r1 = __dmul_rn(h, (double)j), r2 = __dmul_rn(h, (double)k);
#pragma unroll
  for (int d = 0; d < 3; ++d)
    out[d] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[3 * d], r0), __dmul_rn(m[3 * d + 1], r1)),
                                 __dmul_rn(m[3 * d + 2], r2)),
                       m[9 + d]);
}

__global__ void __launch_bounds__(kThreads) k_interpolate(double* __restrict__ out, const double* __restrict__ maps,
                                                          bt_field f, int w, int64_t cell_slots, int cell0) {
  const int cell = cell0 + blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nrows = tri32(w);
  const double h = 1.0 / (double)(w - 1);
  const double* m = maps + 12 * (size_t)cell;
  const int rend = min(nrows, (int)(blockIdx.x + 1) * kRowsPerCta);
  for (int r = blockIdx.x * kRowsPerCta + warp; r < rend; r += kWarps) {
    int j, k;
    decode_row(w, r, j, k);
    const int L = w - j - k, t0 = row_start(w, j, k);
    for (int i = lane; i < L; i += 32) {
      double p[3];
      map_vertex(m, h, i, j, k, p);
      out[(int64_t)cell * cell_slots + t0 + i] = eval_field(f, p[0], p[1], p[2]);
    }
  }
}

// one block per (row chunk, cell, class s): sum over the class's micro-cells
// anchored in the chunk's rows; partial[(cell * 6 + s) * gridDim.x + chunk]
__global__ void __launch_bounds__(kThreads) k_l2_error(const double* __restrict__ x, const double* __restrict__ maps,
                                                       bt_field f, int n, int64_t cell_slots, int cell0,
                                                       double* __restrict__ partial) {
  __shared__ double red[kWarps];
  constexpr int kOff[6][4][3] = BT_CELL_OFFSETS;
  const int cell = cell0 + blockIdx.y, s = blockIdx.z;
  const int ws = s == 0 ? n : (s == 1 ? n - 2 : n - 1);  // class widths (micro_index.hpp:97-121)
  const int wv = n + 1;
  const double h = 1.0 / (double)n;
  const double* m = maps + 12 * (size_t)cell;
  const double* __restrict__ xc = x + (int64_t)cell * cell_slots;
  const double qa = (5.0 + 3.0 * sqrt(5.0)) / 20.0, qb = (5.0 - sqrt(5.0)) / 20.0;  // forms.hpp:56-66
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0.0;
  if (ws > 0) {
    const int nrows = tri32(ws);
    const int rend = min(nrows, (int)(blockIdx.x + 1) * kRowsPerCta);
    for (int r = blockIdx.x * kRowsPerCta + warp; r < rend; r += kWarps) {
      int j, k;
      decode_row(ws, r, j, k);
      const int L = ws - j - k;
      for (int i = lane; i < L; i += 32) {
        double c[4][3], v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int a = i + kOff[s][q][0], b = j + kOff[s][q][1], e = k + kOff[s][q][2];
          map_vertex(m, h, a, b, e, c[q]);
          v[q] = __ldg(xc + row_start(wv, b, e) + a);
        }
        double u[3], w2[3], z[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          u[d] = __dsub_rn(c[1][d], c[0][d]);
          w2[d] = __dsub_rn(c[2][d], c[0][d]);
          z[d] = __dsub_rn(c[3][d], c[0][d]);
        }
        const double cx = __dsub_rn(__dmul_rn(w2[1], z[2]), __dmul_rn(w2[2], z[1]));
        const double cy = __dsub_rn(__dmul_rn(w2[2], z[0]), __dmul_rn(w2[0], z[2]));
        const double cz = __dsub_rn(__dmul_rn(w2[0], z[1]), __dmul_rn(w2[1], z[0]));
        const double vol =
            fabs(__dadd_rn(__dadd_rn(__dmul_rn(u[0], cx), __dmul_rn(u[1], cy)), __dmul_rn(u[2], cz))) / 6.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double xq[3] = {0.0, 0.0, 0.0}, uh = 0.0;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const double bw = t == q ? qa : qb;
#pragma unroll
            for (int d = 0; d < 3; ++d) xq[d] = __dadd_rn(xq[d], __dmul_rn(c[t][d], bw));
            uh = __dadd_rn(uh, __dmul_rn(v[t], bw));
          }
          const double diff = __dsub_rn(uh, eval_field(f, xq[0], xq[1], xq[2]));
          acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(vol, 0.25), diff), diff));
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < kWarps; ++q) t += red[q];
    partial[((int64_t)blockIdx.y * 6 + s) * gridDim.x + blockIdx.x] = t;
  }
}

const double* cell_maps(const bt_grid& g) {
  if (!g.d_maps.p) {
    std::vector<double> m(12 * (size_t)g.mesh.n_cells());
    for (int c = 0; c < g.mesh.n_cells(); ++c) {
      for (int q = 0; q < 9; ++q) m[12 * (size_t)c + q] = g.topo.maps[c].a[q];
      for (int d = 0; d < 3; ++d) m[12 * (size_t)c + 9 + d] = g.topo.maps[c].b[d];
    }
    g.d_maps.upload(m);
  }
  return g.d_maps.p;
}

static void launch_interpolate(const bt_grid& g, int level, const bt_field& f, double* x, cudaStream_t s) {
  const int w = (1 << level) + 1, nc = g.part_end - g.part_begin;
  if (nc) {
    dim3 grid(ceil_div(tri32(w), kRowsPerCta), nc);
    k_interpolate<<<grid, kThreads, 0, s>>>(shifted(x, g, BT_SPACE_P1, level), cell_maps(g), f, w, n_tet(w),
                                            g.part_begin);
    count_launch();
    check_launch("k_interpolate");
  }
  sync(g, level, IF_BCAST, x, nullptr, s);  // replicas bitwise identical (fe_function.hpp:476)
}

double l2_error_p1(const bt_grid& g, int level, const double* x, const bt_field& f, cudaStream_t s) {
  const int n = 1 << level, nc = g.mesh.n_cells(), nl = g.part_end - g.part_begin;
  const int bx = std::max(1, ceil_div(tri32(n), kRowsPerCta));
  std::vector<double> per_cell(nc, 0.0);
  if (nl) {
    DevBuf<double> part((size_t)nl * 6 * bx);
    k_l2_error<<<dim3(bx, nl, 6), kThreads, 0, s>>>(shifted(x, g, BT_SPACE_P1, level), cell_maps(g), f, n,
                                                    n_tet(n + 1), g.part_begin, part.p);
    count_launch();
    check_launch("k_l2_error");
    std::vector<double> h(part.n);
    BT_CUDA(cudaMemcpyAsync(h.data(), part.p, sizeof(double) * part.n, cudaMemcpyDeviceToHost, s));
    BT_CUDA(cudaStreamSynchronize(s));
    for (int c = 0; c < nl; ++c) {
      double t = 0.0;
      for (size_t q = 0; q < (size_t)6 * bx; ++q) t += h[(size_t)c * 6 * bx + q];
      per_cell[g.part_begin + c] = t;
    }
  }
  if (g.part_nranks > 1) {  // every cell's sum, then the cells in order as on one GPU
    if (g.dot_cells.n < (size_t)nc + 1) g.dot_cells.alloc((size_t)nc + 1);
    BT_CUDA(cudaMemcpyAsync(g.dot_cells.p, per_cell.data(), sizeof(double) * nc, cudaMemcpyHostToDevice, s));
    allreduce(g, g.dot_cells.p, nc, s);
    BT_CUDA(cudaMemcpyAsync(per_cell.data(), g.dot_cells.p, sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
    BT_CUDA(cudaStreamSynchronize(s));
  }
  double acc = 0.0;
  for (int c = 0; c < nc; ++c) acc += per_cell[c];
  return std::sqrt(acc);
}

// FP64 FMA throughput probe (bt_dfma_probe): 16 independent chains per thread
__global__ void __launch_bounds__(256) k_dfma_probe(int iters, double* sink) {
  double a[16];
  const double m = 1.0 - 1e-9 * (threadIdx.x & 7), c = 1e-12 * (blockIdx.x & 3);
#pragma unroll
  for (int q = 0; q < 16; ++q) a[q] = 1.0 + q * 1e-3 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 16; ++q) a[q] = fma(a[q], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 16; ++q) s += a[q];
  if (s == 12345.678) sink[0] = s;  // never true; keeps the chains alive
}

static void validate_field(const bt_field* f) {
  if (!f) raise(BT_INVALID_ARGUMENT, "a field is required");
  if (f->kind < 0 || f->kind > 2) raise(BT_INVALID_ARGUMENT, "field kind must be 0, 1 or 2");
}

// ---------------------------------------------------------------------------
// Streaming vector kernels (fe_function.hpp:324-371, solvers.hpp:53-64).
// Explicit _rn intrinsics keep the reference's unfused rounding.
// ---------------------------------------------------------------------------
template <int OP>
__global__ void __launch_bounds__(kThreads) k_vec(double* __restrict__ y, const double* __restrict__ x, double a,
                                                  int64_t n) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    if (OP == V_ASSIGN) y[q] = a;
    else if (OP == V_SCALE) y[q] = __dmul_rn(y[q], a);
    else if (OP == V_COPY) y[q] = x[q];
    else if (OP == V_AXPY) y[q] = __dadd_rn(y[q], __dmul_rn(a, x[q]));
    else if (OP == V_MUL) y[q] = __dmul_rn(y[q], x[q]);
    else if (OP == V_DIV) y[q] = __ddiv_rn(y[q], x[q]);
  }
}

void launch_vec(int op, double* y, const double* x, double a, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  int sms = 148;
  const int blocks = (int)std::min<int64_t>(ceil_div(n, kThreads), (int64_t)sms * 8);
  switch (op) {
    case V_ASSIGN: k_vec<V_ASSIGN><<<blocks, kThreads, 0, s>>>(y, x, a, n); break;
    case V_SCALE: k_vec<V_SCALE><<<blocks, kThreads, 0, s>>>(y, x, a, n); break;
    case V_COPY: k_vec<V_COPY><<<blocks, kThreads, 0, s>>>(y, x, a, n); break;
    case V_AXPY: k_vec<V_AXPY><<<blocks, kThreads, 0, s>>>(y, x, a, n); break;
    case V_MUL: k_vec<V_MUL><<<blocks, kThreads, 0, s>>>(y, x, a, n); break;
    case V_DIV: k_vec<V_DIV><<<blocks, kThreads, 0, s>>>(y, x, a, n); break;
  }
  count_launch();
  check_launch("k_vec");
}

}  // namespace bt

// ===========================================================================
// C ABI (device-side entry points)
// ===========================================================================
using namespace bt;


static void require_p1(int space) {
  if (space != BT_SPACE_P1) raise(BT_INVALID_ARGUMENT, "operator kernels require a P1 function");
}

extern "C" {

bt_status bt_assign(const bt_grid* g, int space, int level, double* x, double value, void* stream) {
  BT_TRY
  check_level(g, level);
  launch_vec(V_ASSIGN, x, nullptr, value, bt_space_size(g, space, level), (cudaStream_t)stream);
  BT_CATCH
}
bt_status bt_scale(const bt_grid* g, int space, int level, double* x, double s, void* stream) {
  BT_TRY
  check_level(g, level);
  launch_vec(V_SCALE, x, nullptr, s, bt_space_size(g, space, level), (cudaStream_t)stream);
  BT_CATCH
}
bt_status bt_copy(const bt_grid* g, int space, int level, const double* src, double* dst, void* stream) {
  BT_TRY
  check_level(g, level);
  launch_vec(V_COPY, dst, src, 0.0, bt_space_size(g, space, level), (cudaStream_t)stream);
  BT_CATCH
}
bt_status bt_axpy(const bt_grid* g, int space, int level, double* y, double a, const double* x, void* stream) {
  BT_TRY
  check_level(g, level);
  launch_vec(V_AXPY, y, x, a, bt_space_size(g, space, level), (cudaStream_t)stream);
  BT_CATCH
}
bt_status bt_hadamard(const bt_grid* g, int level, double* x, const double* d, int divide, void* stream) {
  BT_TRY
  check_level(g, level);
  launch_vec(divide ? V_DIV : V_MUL, x, d, 0.0, bt_space_size(g, BT_SPACE_P1, level), (cudaStream_t)stream);
  BT_CATCH
}
bt_status bt_dot(const bt_grid* g, int space, int level, const double* x, const double* y, double* out,
                 void* stream) {
  BT_TRY
  check_level(g, level);
  if (space == BT_SPACE_EDGES) {
    *out = dot_edges(*g, level, x, y, (cudaStream_t)stream);
    return BT_OK;
  }
  require_p1(space);
  *out = dot_p1(*g, level, x, y, (cudaStream_t)stream);
  BT_CATCH
}
bt_status bt_dot_cells(const bt_grid* g, int space, int level, const double* x, const double* y, double* per_cell,
                       void* stream) {
  BT_TRY
  check_level(g, level);
  require_p1(space);
  if (!per_cell) raise(BT_INVALID_ARGUMENT, "bt_dot_cells: output required");
  for (int c = 0; c < g->mesh.n_cells(); ++c) per_cell[c] = 0.0;
  dot_p1_cells(*g, level, x, y, (cudaStream_t)stream, per_cell, nullptr);
  BT_CATCH
}
bt_status bt_sync_additive(const bt_grid* g, int space, int level, double* x, void* stream) {
  BT_TRY
  check_level(g, level);
  if (space == BT_SPACE_EDGES) {
    sync_edges(*g, level, IF_SYNC, x, nullptr, (cudaStream_t)stream);
    return BT_OK;
  }
  require_p1(space);
  sync(*g, level, IF_SYNC, x, nullptr, (cudaStream_t)stream);
  BT_CATCH
}
bt_status bt_sync_broadcast(const bt_grid* g, int space, int level, double* x, void* stream) {
  BT_TRY
  check_level(g, level);
  if (space == BT_SPACE_EDGES) {
    sync_edges(*g, level, IF_BCAST, x, nullptr, (cudaStream_t)stream);
    return BT_OK;
  }
  require_p1(space);
  sync(*g, level, IF_BCAST, x, nullptr, (cudaStream_t)stream);
  BT_CATCH
}
bt_status bt_impose_dirichlet(const bt_grid* g, int level, const double* src, double* dst, void* stream) {
  BT_TRY
  check_level(g, level);
  sync(*g, level, IF_IMPOSE, dst, src, (cudaStream_t)stream);  // no exchange: masks are per cell
  BT_CATCH
}
bt_status bt_zero_dirichlet(const bt_grid* g, int level, double* x, void* stream) {
  BT_TRY
  check_level(g, level);
  sync(*g, level, IF_ZERO_DIR, x, nullptr, (cudaStream_t)stream);  // no exchange: masks are per cell
  BT_CATCH
}

bt_status bt_apply_stencil(const bt_stencil* st, const double* x, double* y, int bc, void* stream) {
  BT_TRY
  if (!st) raise(BT_INVALID_ARGUMENT, "apply_stencil: table required");
  if (x == y && bt_space_size(st->grid, BT_SPACE_P1, st->level) > 0)  // (empty cell blocks pass nulls)
    raise(BT_INVALID_ARGUMENT, "source and destination must be distinct");
  cudaStream_t s = (cudaStream_t)stream;
  if (stencil_fused(*st)) {
    launch_stencil_fused(*st, x, y, bc, s);
    return BT_OK;
  }
  launch_stencil(*st, x, y, s, bc ? IF_SYNC_DIR : IF_SYNC);  // interface pass overlapped with the interior
  BT_CATCH
}

bt_status bt_apply_stencil_cells(const bt_stencil* st, const double* x, double* y, void* stream) {
  BT_TRY
  if (!st) raise(BT_INVALID_ARGUMENT, "apply_stencil: table required");
  if (x == y && bt_space_size(st->grid, BT_SPACE_P1, st->level) > 0)  // (empty cell blocks pass nulls)
    raise(BT_INVALID_ARGUMENT, "source and destination must be distinct");
  launch_stencil(*st, x, y, (cudaStream_t)stream);
  BT_CATCH
}

bt_status bt_apply_stencil_interface(const bt_stencil* st, const double* x, double* y, int bc, void* stream) {
  BT_TRY
  if (!st) raise(BT_INVALID_ARGUMENT, "apply_stencil: table required");
  sync(*st->grid, st->level, bc ? IF_SYNC_DIR : IF_SYNC, y, x, (cudaStream_t)stream);
  BT_CATCH
}

bt_status bt_apply_elementwise(const bt_grid* g, const bt_form* form, int level, const double* x, double* y,
                               int mode, int bc, double* scratch, void* stream) {
  BT_TRY
  check_level(g, level);
  validate_form(form);
  if (x == y && bt_space_size(g, BT_SPACE_P1, level) > 0)  // (empty cell blocks pass nulls)
    raise(BT_INVALID_ARGUMENT, "source and destination must be distinct");
  cudaStream_t s = (cudaStream_t)stream;
  const EwTables& t = ew_tables(*g, *form, level);
  const int ck = form->kind == BT_FORM_DIV_K_GRAD ? form->coeff_kind : 0;
  const double one[4] = {1.0, 0.0, 0.0, 0.0};
  const double* c = form->kind == BT_FORM_DIV_K_GRAD ? form->c : one;
  double* out = y;
  if (mode == BT_MODE_ADD) {
    if (!scratch) {
      const size_t n = (size_t)bt_space_size(g, BT_SPACE_P1, level);
      if (g->ew_scratch.n < n) g->ew_scratch.alloc(n);
      scratch = g->ew_scratch.p;
    }
    out = scratch;
  }
  launch_elementwise(*g, level, ck, c, t.cells.p, x, out, false, s, t.phase.p, t.host.data());
  sync(*g, level, bc ? IF_SYNC_DIR : IF_SYNC, out, x, s);
  if (mode == BT_MODE_ADD) launch_vec(V_AXPY, y, out, 1.0, bt_space_size(g, BT_SPACE_P1, level), s);
  BT_CATCH
}

bt_status bt_extract_diagonal(const bt_grid* g, const bt_form* form, int level, double* diag, void* stream) {
  BT_TRY
  check_level(g, level);
  validate_form(form);
  cudaStream_t s = (cudaStream_t)stream;
  const EwTables& t = ew_tables(*g, *form, level);
  const int ck = form->kind == BT_FORM_DIV_K_GRAD ? form->coeff_kind : 0;
  const double one[4] = {1.0, 0.0, 0.0, 0.0};
  const double* c = form->kind == BT_FORM_DIV_K_GRAD ? form->c : one;
  launch_elementwise(*g, level, ck, c, t.cells.p, nullptr, diag, true, s, t.phase.p, t.host.data());
  sync(*g, level, IF_SYNC, diag, nullptr, s);
  BT_CATCH
}

bt_status bt_gauss_seidel_sweep(const bt_stencil* table, const double* rhs, double* x, int backward,
                                double* scratch, void* stream) {
  BT_TRY
  if (!table) raise(BT_INVALID_ARGUMENT, "gauss_seidel_sweep: table required");
  if (rhs == x && bt_space_size(table->grid, BT_SPACE_P1, table->level) > 0)
    raise(BT_INVALID_ARGUMENT, "gauss_seidel_sweep: distinct rhs and x required");
  DevBuf<double> own;
  if (!scratch) {
    own.alloc((size_t)bt_space_size(table->grid, BT_SPACE_P1, table->level));
    scratch = own.p;
  }
  cudaStream_t s = (cudaStream_t)stream;
  launch_gs_sweep(*table, rhs, x, scratch, backward != 0, s);
  if (own.p) BT_CUDA(cudaStreamSynchronize(s));  // before the scratch is freed
  BT_CATCH
}

bt_status bt_interpolate(const bt_grid* g, int level, const bt_field* f, double* x, void* stream) {
  BT_TRY
  check_level(g, level);
  validate_field(f);
  launch_interpolate(*g, level, *f, x, (cudaStream_t)stream);
  BT_CATCH
}

bt_status bt_l2_error(const bt_grid* g, int level, const double* x, const bt_field* exact, double* out,
                      void* stream) {
  BT_TRY
  check_level(g, level);
  validate_field(exact);
  if (!out) raise(BT_INVALID_ARGUMENT, "l2_error: output required");
  *out = l2_error_p1(*g, level, x, *exact, (cudaStream_t)stream);
  BT_CATCH
}

bt_status bt_prolongate(const bt_grid* g, int fine_level, const double* coarse, double* fine, int add,
                        void* stream) {
  BT_TRY
  check_level(g, fine_level);
  check_level(g, fine_level - 1);
  launch_prolongate(*g, fine_level, coarse, fine, add != 0, (cudaStream_t)stream);
  BT_CATCH
}

bt_status bt_restrict(const bt_grid* g, int fine_level, const double* fine, double* coarse, void* stream) {
  BT_TRY
  check_level(g, fine_level);
  check_level(g, fine_level - 1);
  launch_restrict(*g, fine_level, fine, coarse, (cudaStream_t)stream);
  BT_CATCH
}

}  // extern "C"

extern "C" bt_status bt_dfma_probe(int blocks, int iters, double* sink, void* stream) {
  BT_TRY
  if (blocks < 1 || iters < 1 || !sink) bt::raise(BT_INVALID_ARGUMENT, "dfma_probe: blocks, iters >= 1 and a sink");
  bt::k_dfma_probe<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, sink);
  bt::count_launch();
  bt::check_launch("k_dfma_probe");
  BT_CATCH
}
