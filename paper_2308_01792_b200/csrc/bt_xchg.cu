// Cell partition across ranks: the interface groups whose
// members live on several ranks. The per-cell phase of an apply and the
// groups local to a rank run as on one GPU; a rank-spanning group goes
// through an exchange buffer (XPlan, bt_internal.hpp):
//   bt_xchg_pack     this rank's member values -> buffer (zeros elsewhere)
//   (caller)         allreduce(sum) of the buffer over ranks (NCCL / gloo)
//   bt_xchg_finish   local groups + member-order reduction of each spanning
//                    group from the buffer (sync_additive fe_function.hpp:
//                    400-423 order, starting from 0.0), so replicas are
//                    bitwise those of a single-GPU sync for any rank count.
// Adding the other ranks' zeros is exact, so the allreduce is an allgather.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "bt_internal.hpp"

namespace bt {

namespace {
constexpr int kT = 256;

// lattice slot of the point with barycentric weights (w0, w1, w2) on the
// local vertices (l0, l1, l2) of a cell (the interface kernel's slot_of)
int64_t slot_of(int64_t cs, int w, int cell, int l0, int w0, int l1, int w1, int l2, int w2) {
  const int i = (l0 == 1 ? w0 : 0) + (l1 == 1 ? w1 : 0) + (l2 == 1 ? w2 : 0);
  const int j = (l0 == 2 ? w0 : 0) + (l1 == 2 ? w1 : 0) + (l2 == 2 ? w2 : 0);
  const int k = (l0 == 3 ? w0 : 0) + (l1 == 3 ? w1 : 0) + (l2 == 3 ? w2 : 0);
  return (int64_t)cell * cs + row_start(w, j, k) + i;
}

__global__ void __launch_bounds__(kT) k_xpack(const XEntry* __restrict__ e, int n, const double* __restrict__ x,
                                              double* __restrict__ buf) {
  const int q = blockIdx.x * kT + threadIdx.x;
  if (q < n) {
    const double v = x[e[q].slot];
    buf[e[q].buf] = e[q].sign > 0 ? v : -v;  // signed replica (N1E1 edges); P1: sign 1
  }
}

template <int MODE>
__global__ void __launch_bounds__(kT) k_xcombine(const XEntry* __restrict__ e, int n, double* __restrict__ x,
                                                 const double* __restrict__ src, const double* __restrict__ buf) {
  const int q = blockIdx.x * kT + threadIdx.x;
  if (q >= n) return;
  const XEntry E = e[q];
  if (MODE == IF_SYNC || (MODE == IF_SYNC_DIR && !E.dir)) {
    double sum = 0.0;
    for (int m = 0; m < E.count; ++m) sum += buf[E.base + m];
    x[E.slot] = E.sign > 0 ? sum : -sum;
  } else if (MODE == IF_SYNC_DIR || MODE == IF_IMPOSE) {
    if (E.dir) x[E.slot] = src[E.slot];
  } else if (MODE == IF_ZERO_DIR) {
    if (E.dir) x[E.slot] = 0.0;
  } else if (MODE == IF_BCAST) {
    const double u = buf[E.base];
    x[E.slot] = E.sign > 0 ? u : -u;
  } else if (MODE == IF_ZERO_NONOWNED) {
    if (E.buf != E.base) x[E.slot] = 0.0;
  }
}

bool needs_buffer(IfaceMode m) { return m == IF_SYNC || m == IF_SYNC_DIR || m == IF_BCAST; }

void check_partitioned_level(const bt_grid* g, int level) {
  check_level(g, level);
}
}  // namespace

void build_xplan(const Mesh& m, const Topology& t, int level, int rank, int nranks, XPlan& out) {
  const int nc = m.n_cells();
  const int n = 1 << level, w = n + 1;
  const int64_t cs = n_tet(w);
  std::vector<int> owner(nc);
  for (int r = 0; r < nranks; ++r) {
    int b, e;
    partition_range(nc, r, nranks, b, e);
    for (int c = b; c < e; ++c) owner[c] = r;
  }
  out.reset();
  int64_t off = 0;
  std::vector<int> own;
  auto add_group = [&](int count, int dir, auto&& slot_of_member, auto&& cell_of_member) {
    own.resize(count);
    for (int mm = 0; mm < count; ++mm) {
      own[mm] = owner[cell_of_member(mm)];
      if (own[mm] == rank)
        out.entries.push_back(XEntry{slot_of_member(mm), (int32_t)(off + mm), (int32_t)off, count, dir});
    }
    xplan_group_peers(out, rank, own.data(), count, off);
    off += count;
  };
  // shared macro faces: interior points (a, b), weights (n - a - b, a, b)
  for (const DevFace& F : t.faces) {
    if (F.ncell != 2 || owner[F.cell[0]] == owner[F.cell[1]]) continue;
    for (int q = 0; q < tri32(n - 2); ++q) {
      int ap, bp;
      decode_tri(n - 2, q, ap, bp);
      const int aa = ap + 1, bb = bp + 1, cc = n - aa - bb;
      add_group(
          2, F.dir,
          [&](int mm) {
            return slot_of(cs, w, F.cell[mm], F.lv[mm][0], cc, F.lv[mm][1], aa, F.lv[mm][2], bb);
          },
          [&](int mm) { return F.cell[mm]; });
    }
  }
  auto spans = [&](const DevPrimHdr& h, const std::vector<DevPrimMem>& mem) {
    for (int mm = 1; mm < h.count; ++mm)
      if (owner[mem[h.first + mm].cell] != owner[mem[h.first].cell]) return true;
    return false;
  };
  // macro edges: points a = 1..n-1, weights (n - a, a)
  for (const DevPrimHdr& h : t.ehdr) {
    if (h.count < 2 || !spans(h, t.emem)) continue;
    for (int aa = 1; aa <= n - 1; ++aa)
      add_group(
          h.count, h.dir,
          [&](int mm) {
            const DevPrimMem& pm = t.emem[h.first + mm];
            return slot_of(cs, w, pm.cell, pm.lv[0], n - aa, pm.lv[1], aa, -1, 0);
          },
          [&](int mm) { return t.emem[h.first + mm].cell; });
  }
  // macro vertices
  for (const DevPrimHdr& h : t.vhdr) {
    if (h.count < 2 || !spans(h, t.vmem)) continue;
    add_group(
        h.count, h.dir,
        [&](int mm) {
          const DevPrimMem& pm = t.vmem[h.first + mm];
          return slot_of(cs, w, pm.cell, pm.lv[0], n, -1, 0, -1, 0);
        },
        [&](int mm) { return t.vmem[h.first + mm].cell; });
  }
  if (off > INT32_MAX) raise(BT_OUT_OF_RANGE, "exchange buffer exceeds 2^31 entries");
  out.buf_size = off;
  out.built = true;
}

void xplan_group_peers(XPlan& p, int rank, const int* owner, int count, int64_t off) {
  bool here = false;
  for (int m = 0; m < count; ++m) here = here || owner[m] == rank;
  if (!here) return;
  for (int m = 0; m < count; ++m) {
    if (owner[m] != rank) {
      p.recvs.emplace_back(owner[m], (int32_t)(off + m));
      continue;
    }
    // this member goes once to every other rank of the group
    for (int q = 0; q < count; ++q) {
      bool first = owner[q] != rank;
      for (int r = 0; r < q && first; ++r) first = owner[r] != owner[q];
      if (first) p.sends.emplace_back(owner[q], (int32_t)(off + m));
    }
  }
}

const XPlan& xchg_plan(const bt_grid& g, int level) {
  XPlan& p = g.xplan.at(level);
  if (!p.built) {
    build_xplan(g.mesh, g.topo, level, g.part_rank, g.part_nranks, p);
    p.d_entries.upload(p.entries);
    const int w = (1 << level) + 1;
    const int64_t cs = n_tet(w);
    std::vector<int4> pts;
    pts.reserve(p.entries.size());
    for (const XEntry& e : p.entries) {
      int64_t t = e.slot % cs;
      const int cell = (int)(e.slot / cs);
      int k = 0;
      while (t >= n_tri(w - k)) t -= n_tri(w - k), ++k;
      int j = 0;
      while (t >= w - k - j) t -= w - k - j, ++j;
      pts.push_back(make_int4(cell, (int)t, j, k));
    }
    p.d_pts.upload(pts);
  }
  return p;
}

void launch_xchg_pack(const bt_grid& g, int level, const double* x, double* buf, cudaStream_t s) {
  launch_xchg_pack_plan(xchg_plan(g, level), part_shift(g, BT_SPACE_P1, level), x, buf, s);
}

void launch_xchg_pack_plan(const XPlan& p, int64_t shift, const double* x, double* buf, cudaStream_t s) {
  if (x) x -= shift;
  if (!p.buf_size) return;
  BT_CUDA(cudaMemsetAsync(buf, 0, sizeof(double) * (size_t)p.buf_size, s));
  const int n = (int)p.entries.size();
  if (!n) return;
  k_xpack<<<(n + kT - 1) / kT, kT, 0, s>>>(p.d_entries.p, n, x, buf);
  count_launch();
  check_launch("k_xpack");
}

void launch_xchg_combine(const bt_grid& g, int level, IfaceMode mode, double* x, const double* src,
                         const double* buf, cudaStream_t s) {
  launch_xchg_combine_plan(xchg_plan(g, level), part_shift(g, BT_SPACE_P1, level), mode, x, src, buf, s);
}

void launch_xchg_combine_plan(const XPlan& p, int64_t shift, IfaceMode mode, double* x, const double* src,
                              const double* buf, cudaStream_t s) {
  const int n = (int)p.entries.size();
  if (!n) return;
  if (x) x -= shift;
  if (src) src -= shift;
  const dim3 grid((n + kT - 1) / kT);
  const XEntry* e = p.d_entries.p;
  switch (mode) {
    case IF_SYNC: k_xcombine<IF_SYNC><<<grid, kT, 0, s>>>(e, n, x, src, buf); break;
    case IF_SYNC_DIR: k_xcombine<IF_SYNC_DIR><<<grid, kT, 0, s>>>(e, n, x, src, buf); break;
    case IF_BCAST: k_xcombine<IF_BCAST><<<grid, kT, 0, s>>>(e, n, x, src, buf); break;
    case IF_IMPOSE: k_xcombine<IF_IMPOSE><<<grid, kT, 0, s>>>(e, n, x, src, buf); break;
    case IF_ZERO_DIR: k_xcombine<IF_ZERO_DIR><<<grid, kT, 0, s>>>(e, n, x, src, buf); break;
    case IF_ZERO_NONOWNED: k_xcombine<IF_ZERO_NONOWNED><<<grid, kT, 0, s>>>(e, n, x, src, buf); break;
  }
  count_launch();
  check_launch("k_xcombine");
}

void allreduce(const bt_grid& g, double* buf, int64_t n, cudaStream_t s) {
  if (g.comm) {
    comm_check(g.comm, g.part_rank, g.part_nranks);
    comm_allreduce(g.comm, buf, n, s);
    return;
  }
  if (!g.allreduce)
    raise(BT_LOGIC_ERROR, "partitioned grid: this call needs the ranks' allreduce (bt_grid_set_allreduce)");
  // stream-ordered: the hook enqueues the collective on s (or blocks until done)
  if (g.allreduce(buf, n, (void*)s, g.allreduce_user) != 0) raise(BT_RUNTIME_ERROR, "allreduce hook failed");
}

namespace {
__global__ void __launch_bounds__(kT) k_xgather(const int32_t* __restrict__ pos, int64_t n,
                                                const double* __restrict__ buf, double* __restrict__ out) {
  const int64_t q = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (q < n) out[q] = buf[pos[q]];
}
__global__ void __launch_bounds__(kT) k_xscatter(const int32_t* __restrict__ pos, int64_t n,
                                                 const double* __restrict__ in, double* __restrict__ buf) {
  const int64_t q = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (q < n) buf[pos[q]] = in[q];
}

// per-peer CSR of the plan's (peer, position) lists; messages keep the
// build (group) order, which every rank shares
void build_neighbours(const XPlan& p) {
  if (p.nbr_built) return;
  std::vector<int> peers;
  for (const auto& e : p.sends) peers.push_back(e.first);
  for (const auto& e : p.recvs) peers.push_back(e.first);
  std::sort(peers.begin(), peers.end());
  peers.erase(std::unique(peers.begin(), peers.end()), peers.end());
  auto csr = [&](const std::vector<std::pair<int, int32_t>>& v, std::vector<int64_t>& off, DevBuf<int32_t>& d) {
    off.assign(peers.size() + 1, 0);
    std::vector<int32_t> pos;
    pos.reserve(v.size());
    for (size_t i = 0; i < peers.size(); ++i) {
      for (const auto& e : v)
        if (e.first == peers[i]) pos.push_back(e.second);
      off[i + 1] = (int64_t)pos.size();
    }
    d.upload(pos);
  };
  csr(p.sends, p.send_off, p.d_send_pos);
  csr(p.recvs, p.recv_off, p.d_recv_pos);
  p.d_sendbuf.alloc(p.send_off.back());
  p.d_recvbuf.alloc(p.recv_off.back());
  p.peers = std::move(peers);
  p.nbr_built = true;
}
}  // namespace

void exchange_buffer(const bt_grid& g, const XPlan& p, double* buf, cudaStream_t s) {
  if (!g.comm && !g.sendrecv) {
    allreduce(g, buf, p.buf_size, s);
    return;
  }
  if (g.comm) comm_check(g.comm, g.part_rank, g.part_nranks);
  build_neighbours(p);
  if (p.peers.empty()) return;
  const int64_t ns = p.send_off.back(), nr = p.recv_off.back();
  if (ns) {
    k_xgather<<<(unsigned)((ns + kT - 1) / kT), kT, 0, s>>>(p.d_send_pos.p, ns, buf, p.d_sendbuf.p);
    count_launch();
  }
  if (g.comm) {
    comm_sendrecv(g.comm, p.peers, p.send_off, p.recv_off, p.d_sendbuf.p, p.d_recvbuf.p, s);
  } else if (g.sendrecv((int)p.peers.size(), p.peers.data(), p.send_off.data(), p.recv_off.data(), p.d_sendbuf.p,
                        p.d_recvbuf.p, (void*)s, g.sendrecv_user) != 0) {
    raise(BT_RUNTIME_ERROR, "sendrecv hook failed");
  }
  if (nr) {
    k_xscatter<<<(unsigned)((nr + kT - 1) / kT), kT, 0, s>>>(p.d_recv_pos.p, nr, p.d_recvbuf.p, buf);
    count_launch();
  }
  check_launch("exchange_buffer");
}

void sync(const bt_grid& g, int level, IfaceMode mode, double* v, const double* src, cudaStream_t s) {
  if (g.part_nranks > 1) {
    const XPlan& p = xchg_plan(g, level);
    const double* buf = nullptr;
    if (needs_buffer(mode) && p.buf_size) {
      if (g.xbuf.n < (size_t)p.buf_size) g.xbuf.alloc((size_t)p.buf_size);
      launch_xchg_pack(g, level, v, g.xbuf.p, s);
      exchange_buffer(g, p, g.xbuf.p, s);
      buf = g.xbuf.p;
    }
    launch_interface(g, level, mode, v, src, s);
    launch_xchg_combine(g, level, mode, v, src, buf, s);
  } else {
    launch_interface(g, level, mode, v, src, s);
  }
}

}  // namespace bt

using namespace bt;

extern "C" {

bt_status bt_grid_partition(const bt_grid* g, int* rank, int* nranks, int* cell_begin, int* cell_end) {
  BT_TRY
  if (!g) raise(BT_INVALID_ARGUMENT, "bt_grid_partition: grid required");
  if (rank) *rank = g->part_rank;
  if (nranks) *nranks = g->part_nranks;
  if (cell_begin) *cell_begin = g->part_begin;
  if (cell_end) *cell_end = g->part_end;
  BT_CATCH
}

int64_t bt_xchg_size(const bt_grid* g, int level) {
  try {
    check_level(g, level);
    BT_CUDA(cudaSetDevice(g->device));
    return xchg_plan(*g, level).buf_size;
  } catch (const Error& e) {
    set_error(e.what());
    return -1;
  } catch (const std::exception& e) {
    set_error(e.what());
    return -1;
  }
}

bt_status bt_xchg_pack(const bt_grid* g, int level, const double* x, double* buf, void* stream) {
  BT_TRY
  check_partitioned_level(g, level);
  launch_xchg_pack(*g, level, x, buf, (cudaStream_t)stream);
  BT_CATCH
}

bt_status bt_xchg_finish(const bt_grid* g, int level, int mode, double* x, const double* src, const double* buf,
                         void* stream) {
  BT_TRY
  check_partitioned_level(g, level);
  if (mode < IF_SYNC || mode > IF_ZERO_NONOWNED) raise(BT_INVALID_ARGUMENT, "bt_xchg_finish: bad mode");
  const IfaceMode m = (IfaceMode)mode;
  if ((m == IF_SYNC_DIR || m == IF_IMPOSE) && !src) raise(BT_INVALID_ARGUMENT, "bt_xchg_finish: src required");
  if (needs_buffer(m) && !buf && xchg_plan(*g, level).buf_size)
    raise(BT_INVALID_ARGUMENT, "bt_xchg_finish: exchange buffer required");
  cudaStream_t s = (cudaStream_t)stream;
  launch_interface(*g, level, m, x, src, s);
  launch_xchg_combine(*g, level, m, x, src, buf, s);
  BT_CATCH
}

bt_status bt_grid_set_allreduce(bt_grid* g, bt_allreduce_fn fn, void* user) {
  BT_TRY
  if (!g) raise(BT_INVALID_ARGUMENT, "bt_grid_set_allreduce: grid required");
  g->allreduce = fn;
  g->allreduce_user = user;
  BT_CATCH
}

bt_status bt_grid_set_comm(bt_grid* g, bt_comm* c) {
  BT_TRY
  if (!g) raise(BT_INVALID_ARGUMENT, "bt_grid_set_comm: grid required");
  if (c) comm_check(c, g->part_rank, g->part_nranks);
  g->comm = c;
  BT_CATCH
}

bt_status bt_grid_set_sendrecv(bt_grid* g, bt_sendrecv_fn fn, void* user) {
  BT_TRY
  if (!g) raise(BT_INVALID_ARGUMENT, "bt_grid_set_sendrecv: grid required");
  g->sendrecv = fn;
  g->sendrecv_user = user;
  BT_CATCH
}

int64_t bt_xchg_peers_host(const char* mesh_text, int level, int rank, int nranks, int which, int32_t* peer,
                           int32_t* pos) {
  try {
    if (!mesh_text || level < 1 || level > 10 || nranks < 1 || rank < 0 || rank >= nranks || which < 0 || which > 1)
      raise(BT_INVALID_ARGUMENT, "bt_xchg_peers_host: bad arguments");
    const Mesh m = parse_mesh(mesh_text);
    Topology t;
    build_topology(m, t);
    XPlan p;
    build_xplan(m, t, level, rank, nranks, p);
    const auto& v = which ? p.recvs : p.sends;
    for (size_t q = 0; q < v.size(); ++q) {
      if (peer) peer[q] = v[q].first;
      if (pos) pos[q] = v[q].second;
    }
    return (int64_t)v.size();
  } catch (const std::exception& e) {
    set_error(e.what());
    return -1;
  }
}

bt_status bt_exchange(const bt_grid* g, int level, int mode, double* x, const double* src, void* stream) {
  BT_TRY
  check_partitioned_level(g, level);
  if (mode < IF_SYNC || mode > IF_ZERO_NONOWNED) raise(BT_INVALID_ARGUMENT, "bt_exchange: bad mode");
  const IfaceMode m = (IfaceMode)mode;
  if ((m == IF_SYNC_DIR || m == IF_IMPOSE) && !src) raise(BT_INVALID_ARGUMENT, "bt_exchange: src required");
  BT_CUDA(cudaSetDevice(g->device));
  sync(*g, level, m, x, src, (cudaStream_t)stream);
  BT_CATCH
}

int64_t bt_xchg_plan_host(const char* mesh_text, int level, int rank, int nranks, int64_t* buf_size,
                          int64_t* slot, int32_t* buf, int32_t* base, int32_t* count, uint8_t* dir) {
  try {
    if (!mesh_text || level < 1 || level > 10 || nranks < 1 || rank < 0 || rank >= nranks)
      raise(BT_INVALID_ARGUMENT, "bt_xchg_plan_host: bad arguments");
    const Mesh m = parse_mesh(mesh_text);
    Topology t;
    build_topology(m, t);
    XPlan p;
    build_xplan(m, t, level, rank, nranks, p);
    if (buf_size) *buf_size = p.buf_size;
    for (size_t q = 0; q < p.entries.size(); ++q) {
      if (slot) slot[q] = p.entries[q].slot;
      if (buf) buf[q] = p.entries[q].buf;
      if (base) base[q] = p.entries[q].base;
      if (count) count[q] = p.entries[q].count;
      if (dir) dir[q] = (uint8_t)p.entries[q].dir;
    }
    return (int64_t)p.entries.size();
  } catch (const std::exception& e) {
    set_error(e.what());
    return -1;
  }
}

}  // extern "C"
