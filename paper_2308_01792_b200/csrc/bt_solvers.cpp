// Multigrid hierarchy, smoothers, CG and the V-cycle (solvers.hpp:84-541),
// orchestrated on the host over device kernels. Every vector operation keeps
// the reference's operation order (and its unfused rounding, see k_vec), so
// residual histories track the CPU reference to round-off.
#include <cuda_runtime.h>

#include <cmath>
#include <random>
#include <vector>

#include "bt_internal.hpp"

namespace bt {

struct LevelData {
  int level = 0;
  int64_t n = 0;
  std::unique_ptr<bt_stencil> stencil;  // stencil kernel
  DevBuf<EwCell> ew;                    // elementwise kernel tables
  DevBuf<double> phase;                 // sin-product phase tables (k_ew_row)
  std::vector<EwCell> ew_host;          // host copy of ew (kernel-parameter weights)
  DevBuf<double> diag;
  double lambda = 0.0;
  // work vectors, allocated on first use (need()): the finest level of a
  // V-cycle holds only r (the smoother's A x), d (the Chebyshev direction)
  // and tmp (the residual); b, x serve as the coarse problem of the level
  // above; p, ap, z as CG and spectral-estimate vectors
  DevBuf<double> r, d, p, ap, z, b, x, tmp;
  DevBuf<CgState> cg;                   // CG scalars (device-resident)
  DevBuf<LamState> lam;                 // estimate_lambda_max scalars (device-resident)
  DevBuf<double> cg_hist;               // CG residual history (grown on demand)
};

}  // namespace bt

struct bt_hierarchy {
  const bt_grid* grid = nullptr;
  bt_form form{};
  int kernel = 1;
  std::vector<std::unique_ptr<bt::LevelData>> levels;
  int part_epoch = 0;  // the grid's partition when the levels were built
  bt::LevelData& at(int l) {
    if (part_epoch != grid->part_epoch)
      bt::raise(BT_LOGIC_ERROR, "hierarchy: the grid was repartitioned after the hierarchy was built");
    if (l < grid->lo || l > grid->hi) bt::raise(BT_OUT_OF_RANGE, "level not in hierarchy");
    return *levels[l - grid->lo];
  }
};

namespace bt {

// a level's work vector, allocated (zeroed) on first use
static double* need(DevBuf<double>& b, int64_t n) {
  if (!b.p && n > 0) {
    b.alloc((size_t)n);  // (inside a graph capture this fails: run once before capturing)
    BT_CUDA(cudaMemset(b.p, 0, sizeof(double) * (size_t)n));
  }
  return b.p;
}

static void hier_apply(bt_hierarchy& h, int l, const double* x, double* y, int bc, cudaStream_t s) {
  LevelData& L = h.at(l);
  if (h.kernel == 1) {
    if (stencil_fused(*L.stencil)) {
      launch_stencil_fused(*L.stencil, x, y, bc, s);  // interior and boundary (incl. sync, Dirichlet rows)
      return;
    }
    launch_stencil(*L.stencil, x, y, s, bc ? IF_SYNC_DIR : IF_SYNC);
    return;
  } else {
    const int ck = h.form.kind == BT_FORM_DIV_K_GRAD ? h.form.coeff_kind : 0;
    static const double one[4] = {1.0, 0.0, 0.0, 0.0};
    launch_elementwise(*h.grid, l, ck, h.form.kind == BT_FORM_DIV_K_GRAD ? h.form.c : one, L.ew.p, x, y, false, s,
                       L.phase.p, L.ew_host.data());
  }
  sync(*h.grid, l, bc ? IF_SYNC_DIR : IF_SYNC, y, x, s);
}

static double dot(bt_hierarchy& h, int l, const double* x, const double* y, cudaStream_t s) {
  return dot_p1(*h.grid, l, x, y, s);
}

// estimate_lambda_max (solvers.hpp:140-172) through spectral_estimate (:362).
// The scalars stay on the device (LamState; one host read at the end), the
// iterate in the level's p / ap / z vectors.
static double lambda_max(bt_hierarchy& h, int l, cudaStream_t s) {
  LevelData& L = h.at(l);
  if (L.lambda != 0.0) return L.lambda;
  const int64_t n = L.n;
  double* v = need(L.p, n);
  double* w = need(L.ap, n);
  double* z = need(L.z, n);
  if (!L.lam.p) L.lam.alloc(1);
  LamState* S = L.lam.p;
  BT_CUDA(cudaStreamSynchronize(s));
  launch_lam_check_diag(S, L.diag.p, n, s);  // read back with the start vector's norm below
  if (bt_random_fill(h.grid, BT_SPACE_P1, l, 0x51cbu, v, s) != BT_OK) raise(BT_CUDA_ERROR, bt_last_error());
  if (h.grid->part_nranks > 1) sync(*h.grid, l, IF_BCAST, v, nullptr, s);  // rank-spanning groups
  sync(*h.grid, l, IF_ZERO_DIR, v, nullptr, s);
  dot_p1_device(*h.grid, l, v, v, &S->nn2, s);
  launch_lam_step(S, true, s);
  LamState hs{};
  BT_CUDA(cudaMemcpyAsync(&hs, S, sizeof(LamState), cudaMemcpyDeviceToHost, s));
  BT_CUDA(cudaStreamSynchronize(s));
  if (hs.zero_diag) raise(BT_INVALID_ARGUMENT, "estimate_lambda_max: zero diagonal entry");
  if (hs.empty) raise(BT_RUNTIME_ERROR, "estimate_lambda_max: empty free space");
  launch_vec_dev(V_SCALE, v, nullptr, &S->inv, &S->done, n, s);
  for (int k = 0; k < 25; ++k) {
    hier_apply(h, l, v, w, 1, s);
    launch_vec(V_COPY, z, v, 0.0, n, s);
    launch_vec(V_MUL, z, L.diag.p, 0.0, n, s);
    dot_p1_device(*h.grid, l, v, w, &S->num, s);
    dot_p1_device(*h.grid, l, v, z, &S->den, s);
    launch_vec(V_COPY, v, w, 0.0, n, s);
    launch_vec(V_DIV, v, L.diag.p, 0.0, n, s);
    dot_p1_device(*h.grid, l, v, v, &S->nn2, s);
    launch_lam_step(S, false, s);  // rho = num / den; 1 / ||v|| (or stop at ||v|| == 0)
    launch_vec_dev(V_SCALE, v, nullptr, &S->inv, &S->done, n, s);
  }
  BT_CUDA(cudaMemcpyAsync(&hs, S, sizeof(LamState), cudaMemcpyDeviceToHost, s));
  BT_CUDA(cudaStreamSynchronize(s));
  L.lambda = 1.1 * hs.rho;
  // the iterate vectors are dead now (a coarse-level CG reallocates its own)
  L.p.release();
  L.ap.release();
  L.z.release();
  return L.lambda;
}

// chebyshev_apply (solvers.hpp:425-456): per step one apply (A x into r), one
// fused update pass (residual, D^-1, direction, x += d) and the Dirichlet pin
static void chebyshev(bt_hierarchy& h, const double* rhs, double* x, int l, int order, double a, double b,
                      cudaStream_t s) {
  LevelData& L = h.at(l);
  const double theta = 0.5 * (b + a);
  const double delta = 0.5 * (b - a);
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  double* r = need(L.r, L.n);
  double* d = need(L.d, L.n);
  hier_apply(h, l, x, r, 1, s);
  launch_smooth_update(0, x, d, r, rhs, L.diag.p, 1.0 / theta, 0.0, L.n, s);
  sync(*h.grid, l, IF_IMPOSE, x, rhs, s);
  for (int k = 1; k < order; ++k) {
    hier_apply(h, l, x, r, 1, s);
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    launch_smooth_update(1, x, d, r, rhs, L.diag.p, rho_new * rho, 2.0 * rho_new / delta, L.n, s);
    sync(*h.grid, l, IF_IMPOSE, x, rhs, s);
    rho = rho_new;
  }
}

static void validate(const bt_smoother_config& c) {                    // solvers.hpp:413-421
  if (!(c.omega > 0) || c.omega > 1) raise(BT_INVALID_ARGUMENT, "smoother: omega must lie in (0, 1]");
  if (c.order < 1) raise(BT_INVALID_ARGUMENT, "smoother: order must be >= 1");
  if (!(c.lo > 0) || !(c.hi > c.lo)) raise(BT_INVALID_ARGUMENT, "smoother: need 0 < lo < hi");
  if (c.nu1 < 0 || c.nu2 < 0) raise(BT_INVALID_ARGUMENT, "smoother: sweep counts must be >= 0");
}

static void smooth(bt_hierarchy& h, const bt_smoother_config& c, const double* rhs, double* x, int l, int sweeps,
                   int backward, cudaStream_t s) {
  validate(c);
  LevelData& L = h.at(l);
  for (int q = 0; q < sweeps; ++q) {
    if (c.kind == 1) {
      if (h.kernel != 1 || !L.stencil) raise(BT_INVALID_ARGUMENT, "gauss-seidel smoothing requires a stencil table");
      launch_gs_sweep(*L.stencil, rhs, x, need(L.r, L.n), backward != 0, s);
    } else if (c.kind == 0) {  // damped Jacobi: x += omega D^-1 (rhs - A x), fused
      double* r = need(L.r, L.n);
      hier_apply(h, l, x, r, 1, s);
      launch_smooth_update(2, x, nullptr, r, rhs, L.diag.p, 0.0, c.omega, L.n, s);
      sync(*h.grid, l, IF_IMPOSE, x, rhs, s);
    } else {
      const double lam = lambda_max(h, l, s);
      chebyshev(h, rhs, x, l, c.order, c.lo * lam, c.hi * lam, s);
    }
  }
}

// cg (solvers.hpp:84-131) with the scalar recurrences on the device (no host
// round trip per iteration; the host polls the done flag every kPoll
// iterations). Operation order as the reference: r = -(A x) + rhs, p = r,
// alpha = rs / pap, x += alpha p, r += (-alpha) ap, p = (rs_new / rs) p + r.
static int cg(bt_hierarchy& h, int l, double tol, int maxit, const double* rhs, double* x, double* hist,
              cudaStream_t s) {
  constexpr int kPoll = 8;
  LevelData& L = h.at(l);
  const int64_t n = L.n;
  double* r = need(L.r, n);
  double* p = need(L.p, n);
  double* ap = need(L.ap, n);
  // Inside a CUDA-graph capture the host cannot poll: every iteration is
  // recorded and the done flag turns the ones after convergence into no-ops
  // (a breakdown then stops the updates instead of raising).
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  BT_CUDA(cudaStreamIsCapturing(s, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (!L.cg.p) {
    if (capturing) raise(BT_LOGIC_ERROR, "cg: run once before capturing a graph (buffers)");
    L.cg.alloc(1);
  }
  if (hist && L.cg_hist.n < (size_t)std::max(maxit, 1)) {
    if (capturing) raise(BT_LOGIC_ERROR, "cg: no residual history inside a graph capture");
    L.cg_hist.alloc((size_t)std::max(maxit, 1));
  }
  double* dh = hist ? L.cg_hist.p : nullptr;
  CgState* S = L.cg.p;
  hier_apply(h, l, x, r, 1, s);
  launch_vec(V_SCALE, r, nullptr, -1.0, n, s);
  launch_vec(V_AXPY, r, rhs, 1.0, n, s);
  launch_vec(V_COPY, p, r, 0.0, n, s);
  dot_p1_device(*h.grid, l, rhs, rhs, &S->nb2, s);
  dot_p1_device(*h.grid, l, r, r, &S->rs, s);
  launch_cg_init(S, tol, s);
  CgState hs{};
  auto poll = [&] {
    if (capturing) return;
    BT_CUDA(cudaMemcpyAsync(&hs, S, sizeof(CgState), cudaMemcpyDeviceToHost, s));
    BT_CUDA(cudaStreamSynchronize(s));
  };
  poll();
  if (hs.done) return 0;
  for (int it = 1; it <= maxit; ++it) {
    hier_apply(h, l, p, ap, 1, s);
    dot_p1_device(*h.grid, l, p, ap, &S->pap, s);
    launch_cg_alpha(S, s);
    launch_vec_dev(V_AXPY, x, p, &S->alpha, &S->done, n, s);
    launch_vec_dev(V_AXPY, r, ap, &S->malpha, &S->done, n, s);
    dot_p1_device(*h.grid, l, r, r, &S->rs_new, s);
    launch_cg_update(S, tol, dh, s);
    launch_vec_dev(V_SCALE, p, nullptr, &S->beta, &S->done, n, s);
    launch_vec_dev(V_AXPY, p, r, &S->one, &S->done, n, s);  // p += 1.0 r
    if (it % kPoll == 0 || it == maxit) {
      poll();
      if (hs.done) break;
    }
  }
  if (capturing) return 0;
  if (hs.breakdown) raise(BT_RUNTIME_ERROR, "cg breakdown: operator is not positive definite");
  if (hist && hs.it) BT_CUDA(cudaMemcpy(hist, dh, sizeof(double) * (size_t)hs.it, cudaMemcpyDeviceToHost));
  return hs.it;
}

// v_cycle (solvers.hpp:509-541). Level-l temporaries: r (residual), and the
// coarse problem (b = restricted residual, x = correction) lives in level
// l-1's b/x buffers.
static void v_cycle(bt_hierarchy& h, int l, const double* rhs, double* x, const bt_smoother_config& sm,
                    const bt_multigrid_config& mg, cudaStream_t s) {
  if (mg.coarse_level < h.grid->lo || l < mg.coarse_level) raise(BT_INVALID_ARGUMENT, "v_cycle: level range invalid");
  if (l == mg.coarse_level) {
    cg(h, l, mg.coarse_tol, mg.coarse_maxit, rhs, x, nullptr, s);
    return;
  }
  LevelData& L = h.at(l);
  LevelData& C = h.at(l - 1);
  smooth(h, sm, rhs, x, l, sm.nu1, 0, s);
  double* r = need(L.tmp, L.n);
  double* cb = need(C.b, C.n);
  double* cx = need(C.x, C.n);
  hier_apply(h, l, x, r, 1, s);
  launch_vec(V_SCALE, r, nullptr, -1.0, L.n, s);
  launch_vec(V_AXPY, r, rhs, 1.0, L.n, s);
  launch_restrict(*h.grid, l, r, cb, s);
  sync(*h.grid, l - 1, IF_ZERO_DIR, cb, nullptr, s);
  launch_vec(V_ASSIGN, cx, nullptr, 0.0, C.n, s);
  v_cycle(h, l - 1, cb, cx, sm, mg, s);
  launch_prolongate(*h.grid, l, cx, x, true, s);
  smooth(h, sm, rhs, x, l, sm.nu2, 1, s);
}

// relative residual ||b - A v|| / ||b|| with Dirichlet identity rows (fmg's
// relative_residual, solvers.hpp:558-566)
static double relative_residual(bt_hierarchy& h, int l, const double* b, const double* v, double* r,
                                cudaStream_t s) {
  const int64_t n = h.at(l).n;
  hier_apply(h, l, v, r, 1, s);
  launch_vec(V_SCALE, r, nullptr, -1.0, n, s);
  launch_vec(V_AXPY, r, b, 1.0, n, s);
  const double nb = std::sqrt(dot(h, l, b, b, s));
  return std::sqrt(dot(h, l, r, r, s)) / (nb > 0 ? nb : 1.0);
}

// fmg (solvers.hpp:547-604)
static int fmg(bt_hierarchy& h, int finest, const double* const* rhs, double* x, const bt_smoother_config& sm,
               const bt_multigrid_config& mg, const bt_field* exact, bt_fmg_row* rows, int max_rows,
               cudaStream_t s) {
  const int cl = mg.coarse_level;
  if (finest < cl) raise(BT_INVALID_ARGUMENT, "fmg: finest below coarse level");
  if (cl < h.grid->lo || finest > h.grid->hi) raise(BT_OUT_OF_RANGE, "fmg: levels outside the hierarchy");
  if (!rhs) raise(BT_INVALID_ARGUMENT, "fmg: one rhs per level expected");
  for (int l = cl; l <= finest; ++l)  // (an empty cell block passes nulls)
    if (!rhs[l - cl] && h.at(l).n > 0) raise(BT_INVALID_ARGUMENT, "fmg: one rhs per level expected");
  const int need = 1 + mg.cycles * (finest - cl);
  if (!rows || max_rows < need) raise(BT_INVALID_ARGUMENT, "fmg: row buffer too small");
  int nrows = 0;
  auto row = [&](int l, int cyc, const double* b, const double* v, double* r) {
    const double res = relative_residual(h, l, b, v, r, s);
    rows[nrows++] = bt_fmg_row{l, cyc, res, exact ? l2_error_p1(*h.grid, l, v, *exact, s) : 0.0};
  };
  DevBuf<double> cur(h.at(cl).n), tmp(h.at(cl).n);
  if (cur.n) BT_CUDA(cudaMemsetAsync(cur.p, 0, sizeof(double) * cur.n, s));
  sync(*h.grid, cl, IF_IMPOSE, cur.p, rhs[0], s);
  cg(h, cl, mg.coarse_tol, mg.coarse_maxit, rhs[0], cur.p, nullptr, s);
  row(cl, 0, rhs[0], cur.p, tmp.p);
  for (int l = cl + 1; l <= finest; ++l) {
    const double* b = rhs[l - cl];
    DevBuf<double> next(h.at(l).n), r(h.at(l).n);
    launch_prolongate(*h.grid, l, cur.p, next.p, false, s);
    sync(*h.grid, l, IF_IMPOSE, next.p, b, s);
    for (int cyc = 1; cyc <= mg.cycles; ++cyc) {
      v_cycle(h, l, b, next.p, sm, mg, s);
      row(l, cyc, b, next.p, r.p);
    }
    std::swap(cur.p, next.p);
    std::swap(cur.n, next.n);
  }
  if (cur.n) BT_CUDA(cudaMemcpyAsync(x, cur.p, sizeof(double) * cur.n, cudaMemcpyDeviceToDevice, s));
  BT_CUDA(cudaStreamSynchronize(s));
  return nrows;
}

}  // namespace bt

using namespace bt;


extern "C" {

bt_status bt_hierarchy_create(const bt_grid* g, const bt_form* form, int kernel, bt_hierarchy** out) {
  BT_TRY
  if (!g) raise(BT_INVALID_ARGUMENT, "make_hierarchy: grid required");
  validate_form(form);
  if (kernel == 1 && form->kind == BT_FORM_DIV_K_GRAD)
    raise(BT_INVALID_ARGUMENT, "stencil kernel requires a constant-coefficient form");
  BT_CUDA(cudaSetDevice(g->device));
  auto h = std::make_unique<bt_hierarchy>();
  h->grid = g;
  h->part_epoch = g->part_epoch;
  h->form = *form;
  h->kernel = kernel;
  for (int l = g->lo; l <= g->hi; ++l) {
    auto L = std::make_unique<LevelData>();
    L->level = l;
    L->n = bt_space_size(g, BT_SPACE_P1, l);
    const size_t n = (size_t)L->n;
    need(L->diag, (int64_t)n);  // the work vectors are allocated on first use
    if (kernel == 1) {
      bt_stencil* st = nullptr;
      if (bt_stencil_create(g, form, l, &st) != BT_OK) raise(BT_INVALID_ARGUMENT, bt_last_error());
      L->stencil.reset(st);
      BT_CUDA(cudaMemcpy(L->diag.p, stencil_diag(*st, 0), sizeof(double) * n, cudaMemcpyDeviceToDevice));
    } else {
      check_coefficient(*g, *form, l, cell_maps(*g), 0);
      std::vector<EwCell> cells;
      build_ew_cells(*g, *form, l, cells);
      L->ew.upload(cells);
      L->ew_host = cells;
      const int ck = form->kind == BT_FORM_DIV_K_GRAD ? form->coeff_kind : 0;
      static const double one[4] = {1.0, 0.0, 0.0, 0.0};
      const double* c = form->kind == BT_FORM_DIV_K_GRAD ? form->c : one;
      if (ck == 1) build_ew_phase(*g, l, L->ew.p, L->phase);
      launch_elementwise(*g, l, ck, c, L->ew.p, nullptr, L->diag.p, true, 0, L->phase.p, L->ew_host.data());
      sync(*g, l, IF_SYNC, L->diag.p, nullptr, 0);
    }
    h->levels.push_back(std::move(L));
  }
  BT_CUDA(cudaDeviceSynchronize());
  *out = h.release();
  BT_CATCH
}

void bt_hierarchy_destroy(bt_hierarchy* h) { delete h; }

bt_status bt_hierarchy_apply(bt_hierarchy* h, int level, const double* x, double* y, int bc, void* stream) {
  BT_TRY
  if (x == y && h && bt_space_size(h->grid, BT_SPACE_P1, level) > 0)
    raise(BT_INVALID_ARGUMENT, "source and destination must be distinct");
  hier_apply(*h, level, x, y, bc, (cudaStream_t)stream);
  BT_CATCH
}

bt_status bt_hierarchy_diagonal(bt_hierarchy* h, int level, const double** diag) {
  BT_TRY
  *diag = h->at(level).diag.p;
  BT_CATCH
}

bt_status bt_estimate_lambda_max(bt_hierarchy* h, int level, double* out, void* stream) {
  BT_TRY
  *out = lambda_max(*h, level, (cudaStream_t)stream);
  BT_CATCH
}

bt_status bt_smooth(bt_hierarchy* h, const bt_smoother_config* cfg, const double* rhs, double* x, int level,
                    int sweeps, int backward, void* stream) {
  BT_TRY
  smooth(*h, *cfg, rhs, x, level, sweeps, backward, (cudaStream_t)stream);
  BT_CATCH
}

bt_status bt_cg(bt_hierarchy* h, int level, double tol, int maxit, const double* rhs, double* x, double* hist,
                int* iterations, void* stream) {
  BT_TRY
  const int it = cg(*h, level, tol, maxit, rhs, x, hist, (cudaStream_t)stream);
  if (iterations) *iterations = it;
  BT_CATCH
}

bt_status bt_fmg(bt_hierarchy* h, int finest, const double* const* rhs_levels, double* x,
                 const bt_smoother_config* sm, const bt_multigrid_config* mg, const bt_field* exact,
                 bt_fmg_row* rows, int max_rows, int* nrows, void* stream) {
  BT_TRY
  if (!h || !sm || !mg) raise(BT_INVALID_ARGUMENT, "fmg: hierarchy and configs required");
  if (!x && bt_space_size(h->grid, BT_SPACE_P1, finest) > 0) raise(BT_INVALID_ARGUMENT, "fmg: x required");
  if (exact && (exact->kind < 0 || exact->kind > 2)) raise(BT_INVALID_ARGUMENT, "field kind must be 0, 1 or 2");
  const int nr = fmg(*h, finest, rhs_levels, x, *sm, *mg, exact, rows, max_rows, (cudaStream_t)stream);
  if (nrows) *nrows = nr;
  BT_CATCH
}

bt_status bt_v_cycle(bt_hierarchy* h, int level, const double* rhs, double* x, const bt_smoother_config* sm,
                     const bt_multigrid_config* mg, void* stream) {
  BT_TRY
  v_cycle(*h, level, rhs, x, *sm, *mg, (cudaStream_t)stream);
  BT_CATCH
}

}  // extern "C"
