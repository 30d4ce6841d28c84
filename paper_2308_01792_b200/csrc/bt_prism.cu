// Interior rows of apply_stencil (operators.hpp:247-271, merged row of
// compute_stencil operators.hpp:204-221) as a warp-specialised k-march over
// prisms, the headline kernel of the fused apply (launch_stencil_fused).
//
// Work unit: a prism of one macro-cell — rows j0 .. j0+15 (a j-band) and
// columns i0 .. i0+119 of layers k0 .. k1-1. Every layer k of the prism needs
// rows j0-1 .. j0+16 of layers k-1, k, k+1 at columns i0-1 .. i0+120, and in
// the tetrahedral row layout (micro_index.hpp:145) each of those row segments
// is contiguous. So one producer warp per CTA streams the prism's layers
// k0-1 .. k1 bottom-up, one layer-band per ring stage: lane r copies row
// segment r with one cp.async.bulk (its 16-byte-aligned enclosing range,
// landing so that smem and global addresses agree mod 16 bytes) and the stage's
// mbarrier counts the bytes. Eight consumer warps hold three stages (k-1, k,
// k+1) and write layer k: warp (q, h) owns output columns i0 + 30q .. +29 (lane
// l: column i0 + 30q + l - 1; lanes 0 and 31 only feed their neighbours) and
// marches rows j0 + 8h .. +7 with a register window along j: per row it reads
// three new values from shared memory (rows j+1 of layers k and k-1, row j of
// layer k+1). The merged row is bitwise symmetric (checked on the host), so
// the +-i terms are formed by the neighbouring lanes as partial sums and
// shuffled, exactly as in k_stencil_fast (bt_stencil.cu) and with the same
// operation order, so the two kernels agree bit for bit.
//
// Scheduling: persistent CTAs (two per SM) take units from a global queue,
// longest first; the last CTA to finish resets the queue for the next launch
// (graph-replay safe). Only interior points (i, j, k >= 1, i + j + k <= n - 1)
// are written: macro face / edge / vertex points are k_boundary's.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <mutex>
#include <vector>

#include "bt_async.cuh"
#include "bt_internal.hpp"

namespace bt {

namespace {
constexpr int kPSlotD = 4224;            // doubles per ring stage (one layer-band, 33 KB)
constexpr int kPS = 6;                   // ring stages
constexpr int kPFront = 2;               // pad before the ring (column -1 of the first stage)
constexpr int kPBack = 1024;             // pad after it (over-reads past the last stage's band)
constexpr int kPCols = 62;               // output columns per item (lanes hold columns c and c + 32)
constexpr int kPNR = 4;                  // output rows per item
constexpr int kPCons = 15;               // consumer warps (+ the producer: 4 warps per SM sub-partition)
constexpr int kPThreads = (kPCons + 1) * 32;
constexpr int kPMaxReg = 96;             // leaves registers for a k_boundary block beside each CTA
constexpr int kPK = 12;                  // output layers per unit (k-chunk)

struct StageMeta {
  long long ga;  // x index of the stage's first double (16-byte aligned)
  int cell, kl, k0, k1, j0, R, nch, pad;
};
constexpr size_t kPRingD = kPFront + (size_t)kPS * kPSlotD + kPBack;
constexpr size_t kPSmem = sizeof(double) * kPRingD + 2 * kPS * sizeof(uint64_t) + kPS * sizeof(StageMeta);

__device__ __forceinline__ void mbar_init(uint32_t a, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ double lds64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

// first and one-past-last x index of rows j0-1 .. j0+R of layer kl (the rows that exist)
__host__ __device__ __forceinline__ void band_range(int w, int64_t cb, int j0, int R, int kl, int64_t& g0,
                                                    int64_t& g1) {
  const int ja = j0 > 0 ? j0 - 1 : 0, jb = j0 + R < w - 1 - kl ? j0 + R : w - 1 - kl;  // rows 0 .. w-1-kl
  g0 = cb + row_start(w, ja, kl);
  g1 = cb + row_start(w, jb + 1, kl);
}

// One item's rows of one layer: set row t (0 .. 5) = lattice row ja - 1 + t
// (row -1 reads row 0: it feeds only row 0, which is never stored), columns
// cA and cA + 32.
struct Rows6 {
  double A[6], B[6];
};

__global__ void __maxnreg__(kPMaxReg)
    k_stencil_prism(const double* __restrict__ x, double* __restrict__ y, const int4* __restrict__ units, int nunits,
                    const double* __restrict__ wts, int w, int64_t cs, int* __restrict__ ctr, int mode) {
  extern __shared__ __align__(128) double psm[];
  double* ring = psm + kPFront;
  uint64_t* full = reinterpret_cast<uint64_t*>(psm + kPRingD);
  uint64_t* empty = full + kPS;
  StageMeta* meta = reinterpret_cast<StageMeta*>(empty + kPS);
  // warp index through a shuffle: provably warp-uniform, so branches on it
  // (and on values broadcast the same way) need no divergence handling
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPS; ++s) {
      mbar_init(smem_u32(full + s), 1);
      mbar_init(smem_u32(empty + s), kPCons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int n = w - 1;
  const uint32_t ring_s = smem_u32(ring), full_s = smem_u32(full), empty_s = smem_u32(empty);

  if (warp == kPCons) {
    // ---------------- producer (lane 0): one contiguous layer-band per stage ----------------
    if (lane == 0) {
      uint32_t sc = 0;
      while (true) {
        const int u = atomicAdd(ctr, 1);
        const int4 U = u < nunits ? units[u] : make_int4(-1, 0, 1, 0);
        const int cell = U.x, j0 = U.y & 0x7ff, R = (U.y >> 11) & 0x7f, nch = U.y >> 18, k0 = U.z, k1 = U.w;
        const int klo = k0 - 1, khi = cell < 0 ? klo : k1;
        const int64_t cb = (int64_t)max(cell, 0) * cs;
        for (int kl = klo; kl <= khi; ++kl, ++sc) {
          const int slot = (int)(sc % kPS);
          mbar_wait(empty_s + 8u * slot, ((sc / kPS) & 1u) ^ 1u);
          const uint32_t fb = full_s + 8u * slot;
          StageMeta& m = meta[slot];
          m.cell = cell;
          if (cell < 0) {  // end of the queue
            mbar_arrive(fb);
            break;
          }
          int64_t g0, g1;
          band_range(w, cb, j0, R, kl, g0, g1);
          const int64_t ga = g0 & ~int64_t(1);
          const uint32_t bytes = (uint32_t)(((g1 + 1) & ~int64_t(1)) - ga) * 8u;
          m.ga = ga;
          m.kl = kl;
          m.k0 = k0;
          m.k1 = k1;
          m.j0 = j0;
          m.R = R;
          m.nch = nch;
          if (mode & 2) {  // profiling: no copies
            mbar_arrive(fb);
          } else {
            mbar_expect_tx(fb, bytes);  // release: orders the meta writes
            bulk_g2s(ring_s + 8u * (uint32_t)(slot * kPSlotD), x + ga, bytes, fb);
          }
        }
        if (cell < 0) break;
      }
    }
  } else {
    // ---------------- consumers: one item (chunk q, rows ja .. ja+3) per unit ----------------
    uint32_t sc = 0;
    int cell = 0, kl = 0, ja = 0, cA = 0;
    bool active = false;
    int64_t cb = 0;
    double W[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // wait for the next stage, read it into X (if this warp has an item), release it
    auto next = [&](Rows6& X) {
      const int slot = (int)(sc % kPS);
      mbar_wait(full_s + 8u * slot, (sc / kPS) & 1u);
      ++sc;
      kl = meta[slot].kl;
      if (active) {
        // offsets of rows ja - 1 + t (t = 0 .. 5) in layer kl; row -1 reads
        // row 0 (it feeds only row 0, never stored) and rows past the layer's
        // top stay at its end (lengths clamped at 0)
        const int jr = ja - 1, j0r = jr < 0 ? 0 : jr;
        int off = row_start(w, j0r, kl), Lr = w - kl - j0r;
        const uint32_t base = ring_s + 8u * (uint32_t)(slot * kPSlotD + (int)(cb - meta[slot].ga) + cA);
#pragma unroll
        for (int t = 0; t < 6; ++t) {
          X.A[t] = lds64(base + 8u * (uint32_t)off);
          X.B[t] = lds64(base + 8u * (uint32_t)off + 256u);
          if (t > 0 || jr >= 0) {
            off += max(Lr, 0);
            --Lr;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_s + 8u * slot);  // release: the reads above are done
    };
    // output layer k from layers k-1 (M), k (C), k+1 (P)
    // output layer k from layers k-1 (M), k (C), k+1 (P); both column halves
    // (cA and cA + 32) or, when the second half holds no interior point, the
    // first only
    auto rows = [&](const Rows6& M, const Rows6& C, const Rows6& P, int k, auto both) {
      constexpr bool kBoth = decltype(both)::value;
      int L = w - k - ja;  // length of row ja of layer k
      double* yA = y + cb + row_start(w, ja, k) + cA;
#pragma unroll
      for (int t = 1; t <= kPNR; ++t) {  // row j = ja - 1 + t
        const double aA = C.A[t], amA = C.A[t - 1], A1A = C.A[t + 1];
        const double bA = P.A[t - 1], B0A = P.A[t];
        const double cAv = M.A[t], C1A = M.A[t + 1];
        // partial sums for the lanes of columns i + 1 (up) and i - 1 (dn)
        const double upA = fma(W[7], C1A, fma(W[5], B0A, fma(W[4], A1A, W[1] * aA)));
        const double dnA = fma(W[7], bA, fma(W[5], cAv, fma(W[4], amA, W[1] * aA)));
        double sA = fma(W[6], C1A + bA, fma(W[3], B0A + cAv, fma(W[2], A1A + amA, W[0] * aA)));
        const int j = ja - 1 + t;
        const bool row = j >= 1 && j <= n - 2 - k;
        // column cA - 1: lane - 1's cA
        const double lA = __shfl_up_sync(0xffffffffu, upA, 1);
        if (kBoth) {
          const double aB = C.B[t], amB = C.B[t - 1], A1B = C.B[t + 1];
          const double bB = P.B[t - 1], B0B = P.B[t];
          const double cBv = M.B[t], C1B = M.B[t + 1];
          const double upB = fma(W[7], C1B, fma(W[5], B0B, fma(W[4], A1B, W[1] * aB)));
          const double dnB = fma(W[7], bB, fma(W[5], cBv, fma(W[4], amB, W[1] * aB)));
          // cA + 31: lane - 1's cB (lane 0: lane 31's cA); cA + 1: lane + 1's cA
          // (lane 31: lane 0's cB); cA + 33: lane + 1's cB
          const double lB = __shfl_sync(0xffffffffu, lane == 31 ? upA : upB, (lane + 31) & 31);
          const double rA = __shfl_sync(0xffffffffu, lane == 0 ? dnB : dnA, (lane + 1) & 31);
          const double rB = __shfl_down_sync(0xffffffffu, dnB, 1);
          double sB = fma(W[6], C1B + bB, fma(W[3], B0B + cBv, fma(W[2], A1B + amB, W[0] * aB)));
          sA += lA;  // (centre + its i-1 partial) + its i+1 partial, as k_stencil_fast
          sA += rA;
          sB += lB;
          sB += rB;
          if (row && lane > 0 && cA >= 1 && cA <= L - 2) yA[0] = sA;
          if (row && lane < 31 && cA + 32 <= L - 2) yA[32] = sB;
        } else {
          const double rA = __shfl_down_sync(0xffffffffu, dnA, 1);  // lane 31's column is no output
          sA += lA;
          sA += rA;
          if (row && lane > 0 && lane < 31 && cA >= 1 && cA <= L - 2) yA[0] = sA;
        }
        yA += L;
        --L;
      }
    };
    auto compute = [&](const Rows6& M, const Rows6& C, const Rows6& P, int k) {
      if (!active || (mode & 1)) return;
      // the item's widest output row: interior columns 1 .. n-1-k-jf
      const int jf = max(ja, 1), last = n - 1 - k - jf, c0 = cA - lane + 1;  // c0: the chunk's first column
      if (jf > n - 2 - k || c0 > last) {  // no interior point left in this item (nor above it)
        active = false;
        return;
      }
      if (c0 + 30 > last)
        rows(M, C, P, k, std::false_type());
      else
        rows(M, C, P, k, std::true_type());
    };
    Rows6 X0, X1, X2;
    while (true) {
      // first stage of a unit: its item
      {
        const int slot = (int)(sc % kPS);
        mbar_wait(full_s + 8u * slot, (sc / kPS) & 1u);
        const StageMeta& m = meta[slot];
        cell = __shfl_sync(0xffffffffu, m.cell, 0);
        if (cell < 0) break;
        const int nch = __shfl_sync(0xffffffffu, m.nch, 0), P = kPCons / nch;
        active = warp < nch * P;
        const int q = warp % nch, part = warp / nch;
        const int j0 = __shfl_sync(0xffffffffu, m.j0, 0), R = __shfl_sync(0xffffffffu, m.R, 0);
        ja = j0 + kPNR * part;
        active = active && ja < j0 + R;
        cA = kPCols * q - 1 + lane;
        cb = (int64_t)cell * cs;
#pragma unroll
        for (int d = 0; d < 8; ++d) W[d] = __ldg(wts + 8 * cell + d);
      }
      const int k1 = __shfl_sync(0xffffffffu, meta[(int)(sc % kPS)].k1, 0);
      next(X0);  // layer k0 - 1
      next(X1);  // layer k0
      int k = __shfl_sync(0xffffffffu, kl, 0);
      while (true) {
        next(X2);
        compute(X0, X1, X2, k);
        if (++k == k1) break;
        next(X0);
        compute(X1, X2, X0, k);
        if (++k == k1) break;
        next(X1);
        compute(X2, X0, X1, k);
        if (++k == k1) break;
      }
    }
  }
  // the last CTA out resets the queue (every producer has seen the end)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
}
}  // namespace

// Units of this handle's cells: k-chunks of kPK output layers; within a
// chunk, bands of R = 4 P rows, P = the row parts that fit beside the nch
// column chunks of the band's widest row (nch * P <= 15 consumer warps).
// Ordered by k-chunk, so all CTAs stream the same height of every cell at
// about the same time (a unit's two warm-up layers are the lower chunk's last
// two, read at about the same time, from L2).
void init_prism_tasks(bt_stencil& st) {
  const int n = 1 << st.level, w = n + 1;
  st.nprism = 0;
  if (!st.symmetric || n < 8 || (n + kPCols - 1) / kPCols > kPCons) return;
  std::vector<int4> units;
  for (int k0 = 1; k0 <= n - 3; k0 += kPK) {
    const int k1 = std::min(k0 + kPK, n - 2);  // interior layers 1 .. n-3
    for (int cell = st.part_begin; cell < st.part_end; ++cell) {
      for (int j0 = 0; j0 <= n - 2 - k0;) {
        const int jl = std::max(j0, 1);
        const int nch = (n - k0 - jl + kPCols - 1) / kPCols;  // chunks over columns 0 .. n-1-k0-jl
        const int R = kPNR * (kPCons / nch);
        units.push_back(make_int4(cell, j0 | (R << 11) | (nch << 18), k0, k1));
        j0 += R;
      }
    }
  }
  // every stage fits a slot: the unit's first (largest) one, checked on the host
  for (const int4& u : units) {
    int64_t g0, g1;
    band_range(w, 0, u.y & 0x7ff, (u.y >> 11) & 0x7f, u.z - 1, g0, g1);
    if (g1 - g0 + 2 > kPSlotD) raise(BT_LOGIC_ERROR, "prism: band larger than a ring slot");
  }
  st.d_prism.upload(units);
  st.nprism = (int)units.size();
  std::vector<double> w8(8 * (size_t)st.grid->mesh.n_cells(), 0.0);
  for (size_t q = 0; q < st.fast.size() && q < w8.size(); ++q) w8[q] = st.fast[q];
  st.d_w8.upload(w8);
  std::vector<int> z(2, 0);
  st.d_prism_ctr.upload(z);
}

bool prism_ok(const bt_stencil& st, const double* x) {
  return st.nprism > 0 && ((uintptr_t)x & 15) == 0;
}

void launch_prism(const bt_stencil& st, const double* x, double* y, cudaStream_t s) {
  const int w = (1 << st.level) + 1;
  static std::mutex mu;
  static int grids[64] = {0};
  int dev = 0;
  BT_CUDA(cudaGetDevice(&dev));
  int grid;
  {
    std::lock_guard<std::mutex> lock(mu);
    int& gr = grids[dev & 63];
    if (!gr) {
      BT_CUDA(cudaFuncSetAttribute(k_stencil_prism, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPSmem));
      int sms = 0, per_sm = 0;
      BT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      BT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stencil_prism, kPThreads, kPSmem));
      gr = sms * std::max(1, per_sm);
    }
    grid = gr;
  }
  grid = std::min(grid, st.nprism);
  // x, y are global-cell indexed (unpartitioned handle: the caller's pointers)
  // BT_PRISM_MODE (profiling only): bit 0 skips the compute, bit 1 the copies
  static const int mode = [] {
    const char* e = std::getenv("BT_PRISM_MODE");
    return e ? std::atoi(e) : 0;
  }();
  k_stencil_prism<<<grid, kPThreads, kPSmem, s>>>(x, y, st.d_prism.p, st.nprism, st.d_w8.p, w, n_tet(w),
                                                  st.d_prism_ctr.p, mode);
  count_launch();
}

}  // namespace bt
