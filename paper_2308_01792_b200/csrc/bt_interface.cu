// Interface pass: the reference's replica synchronisation
// (sync_additive fe_function.hpp:400-423, sync_broadcast :425-446) and
// Dirichlet rows (impose_dirichlet operators.hpp:98-104, zero_dirichlet
// solvers.hpp:66-72) for P1 vertex DoFs, organised by macro primitive.
//
// Every lattice point on a macro face / edge / vertex is parametrised by its
// barycentric weights on the primitive's sorted global vertices; each member
// cell maps them to its own (i, j, k) through the local-vertex table lv, so
// replica slots are computed, never stored. Members are visited in ascending
// cell order — the reference's group order — so replica sums are bitwise
// those of the reference.
#include <cuda_runtime.h>

#include "bt_internal.hpp"

namespace bt {

namespace {
constexpr int kT = 256;

struct FaceArgs {
  const DevFace* faces;
  const int* list;
  int n;
  int64_t cs;
};
struct PrimArgs {
  const DevPrimHdr* eh;
  const DevPrimMem* em;
  const int* elist;
  int ne;
  const DevPrimHdr* vh;
  const DevPrimMem* vm;
  const int* vlist;
  int nv;
  int n;
  int64_t cs;
};

__device__ __forceinline__ int64_t slot_of(int64_t cs, int w, int cell, int l0, int w0, int l1, int w1, int l2,
                                           int w2) {
  const int i = (l0 == 1 ? w0 : 0) + (l1 == 1 ? w1 : 0) + (l2 == 1 ? w2 : 0);
  const int j = (l0 == 2 ? w0 : 0) + (l1 == 2 ? w1 : 0) + (l2 == 2 ? w2 : 0);
  const int k = (l0 == 3 ? w0 : 0) + (l1 == 3 ? w1 : 0) + (l2 == 3 ? w2 : 0);
  return (int64_t)cell * cs + row_start(w, j, k) + i;
}

// mode semantics for one replica group with slot function S(m), m < count
template <int MODE, class S>
__device__ __forceinline__ void apply_group(double* __restrict__ v, const double* __restrict__ src, int count,
                                            bool dir, S slot) {
  if (MODE == IF_SYNC || (MODE == IF_SYNC_DIR && !dir)) {
    if (count < 2) return;
    double sum = 0;
    for (int m = 0; m < count; ++m) sum += v[slot(m)];
    for (int m = 0; m < count; ++m) v[slot(m)] = sum;
  } else if (MODE == IF_SYNC_DIR || MODE == IF_IMPOSE) {
    if (!dir) return;
    for (int m = 0; m < count; ++m) {
      const int64_t t = slot(m);
      v[t] = src[t];
    }
  } else if (MODE == IF_ZERO_DIR) {
    if (!dir) return;
    for (int m = 0; m < count; ++m) v[slot(m)] = 0.0;
  } else if (MODE == IF_BCAST) {
    if (count < 2) return;
    const double val = v[slot(0)];
    for (int m = 1; m < count; ++m) v[slot(m)] = val;
  } else if (MODE == IF_ZERO_NONOWNED) {
    for (int m = 1; m < count; ++m) v[slot(m)] = 0.0;
  }
}

// All primitives of one mode in a single launch: a 1-D grid whose leading
// blocks cover up to two face lists (xb blocks per face) and whose trailing
// blocks cover macro edges (eb blocks per edge) and vertices.
struct AllArgs {
  FaceArgs f1, f2;
  int nf1, nf2, xb;
  PrimArgs p;
  int eb;
};

template <int MODE>
__global__ void __launch_bounds__(kT) k_interface(double* __restrict__ v, const double* __restrict__ src, AllArgs a) {
  const int n = a.p.n, w = n + 1;
  int b = blockIdx.x;
  const int nfb1 = a.nf1 * a.xb, nfb2 = a.nf2 * a.xb;
  if (b < nfb1 + nfb2) {
    const FaceArgs& fa = b < nfb1 ? a.f1 : a.f2;
    if (b >= nfb1) b -= nfb1;
    const int q = (b % a.xb) * kT + threadIdx.x;
    if (q >= tri32(n - 2)) return;
    const DevFace f = fa.faces[fa.list[b / a.xb]];
    int ap, bp;
    decode_tri(n - 2, q, ap, bp);
    const int aa = ap + 1, bb = bp + 1, cc = n - aa - bb;
    const int64_t s0 = slot_of(fa.cs, w, f.cell[0], f.lv[0][0], cc, f.lv[0][1], aa, f.lv[0][2], bb);
    const int64_t s1 = f.ncell == 2 ? slot_of(fa.cs, w, f.cell[1], f.lv[1][0], cc, f.lv[1][1], aa, f.lv[1][2], bb) : 0;
    apply_group<MODE>(v, src, f.ncell, f.dir != 0, [&](int m) { return m == 0 ? s0 : s1; });
    return;
  }
  b -= nfb1 + nfb2;
  const PrimArgs& pa = a.p;
  if (b < pa.ne * a.eb) {
    const int aa = (b % a.eb) * kT + threadIdx.x + 1;
    if (aa > n - 1) return;
    const DevPrimHdr h = pa.eh[pa.elist[b / a.eb]];
    const DevPrimMem* mem = pa.em + h.first;
    apply_group<MODE>(v, src, h.count, h.dir != 0, [&](int m) {
      const DevPrimMem pm = mem[m];
      return slot_of(pa.cs, w, pm.cell, pm.lv[0], n - aa, pm.lv[1], aa, -1, 0);
    });
    return;
  }
  b -= pa.ne * a.eb;
  const int vi = b * kT + threadIdx.x;
  if (vi >= pa.nv) return;
  const DevPrimHdr h = pa.vh[pa.vlist[vi]];
  const DevPrimMem* mem = pa.vm + h.first;
  apply_group<MODE>(v, src, h.count, h.dir != 0, [&](int m) {
    const DevPrimMem pm = mem[m];
    return slot_of(pa.cs, w, pm.cell, pm.lv[0], n, -1, 0, -1, 0);
  });
}

template <int MODE>
void launch_mode(const bt_grid& g, int level, double* v, const double* src, cudaStream_t s) {
  const IfaceLists& L = g.loc;
  const int n = 1 << level;
  const int64_t cs = n_tet(n + 1);
  const int fp = tri32(n - 2);
  const bool sync_like = MODE == IF_SYNC || MODE == IF_BCAST || MODE == IF_ZERO_NONOWNED || MODE == IF_SYNC_DIR;
  const bool dir_like = MODE == IF_SYNC_DIR || MODE == IF_IMPOSE || MODE == IF_ZERO_DIR;
  AllArgs a{};
  a.xb = (fp + kT - 1) / kT;
  if (sync_like && fp) {
    a.f1 = FaceArgs{g.d_faces.p, L.d_face_shared.p, n, cs};
    a.nf1 = (int)L.face_shared.size();
  }
  if (dir_like && fp) {
    a.f2 = FaceArgs{g.d_faces.p, L.d_face_bdir.p, n, cs};
    a.nf2 = (int)L.face_bdir.size();
  }
  const int ne = (int)L.edge_act.size(), nv = (int)L.vert_act.size();
  a.p = PrimArgs{g.d_ehdr.p, g.d_emem.p, L.d_edge_act.p, ne, g.d_vhdr.p, g.d_vmem.p, L.d_vert_act.p, nv, n, cs};
  a.eb = (n - 1 + kT - 1) / kT;
  const int64_t blocks = (int64_t)(a.nf1 + a.nf2) * a.xb + (int64_t)ne * a.eb + (nv + kT - 1) / kT;
  if (!blocks) return;
  k_interface<MODE><<<(unsigned)blocks, kT, 0, s>>>(v, src, a);
  count_launch();
  check_launch("k_interface");
}

}  // namespace

void launch_interface(const bt_grid& g, int level, IfaceMode mode, double* v, const double* src, cudaStream_t s) {
  v = shifted(v, g, BT_SPACE_P1, level);  // local -> global-cell indexing
  src = shifted(src, g, BT_SPACE_P1, level);
  switch (mode) {
    case IF_SYNC: launch_mode<IF_SYNC>(g, level, v, src, s); break;
    case IF_SYNC_DIR: launch_mode<IF_SYNC_DIR>(g, level, v, src, s); break;
    case IF_BCAST: launch_mode<IF_BCAST>(g, level, v, src, s); break;
    case IF_IMPOSE: launch_mode<IF_IMPOSE>(g, level, v, src, s); break;
    case IF_ZERO_DIR: launch_mode<IF_ZERO_DIR>(g, level, v, src, s); break;
    case IF_ZERO_NONOWNED: launch_mode<IF_ZERO_NONOWNED>(g, level, v, src, s); break;
  }
}

}  // namespace bt
