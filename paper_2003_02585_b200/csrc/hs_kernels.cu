// sm_100a kernels of the helmsweep hot path. complex128 = double2 (re, im).
//
//   (the multifrontal solve kernels live in hs_solve.cu)
//   factor_level_kernel     assembly + extend-add + panel LDL^T of one tree height
//                           (src/direct.cpp:55-87, 181-281)
//   rhs/inject/nonzero      split source, trace injection, exact-zero test
//                           (src/sweeper.cpp:189-251, src/transfer.cpp:68-89)
//   extract_deposit         trace extraction, routing, mailbox accumulation
//                           (src/transfer.cpp:13-66, src/sweeper.cpp:295-307)
//   accumulate              weighted partition-of-unity gather (src/transfer.cpp:91-102)
//   residual / spmv / dots  global operator and Krylov vector kernels
#include "hs_kernels.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#include <algorithm>
#include <climits>
#include <type_traits>
#include <atomic>
#include <cstdio>

#include "hs_common.hpp"

namespace hsb {

std::atomic<long long> g_kernel_launches{0};

namespace {

inline void after_launch() {
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  HS_CUDA(cudaGetLastError());
}

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kNB = 16;  // factorization panel width

__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ unsigned long long reduce_or64(unsigned long long v) {  // warp OR of a 64-bit mask
  const unsigned lo = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(v));
  const unsigned hi = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(v >> 32));
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ void cfms(double2& acc, double2 a, double2 b) {
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
// 1/d (Smith's algorithm, avoids overflow in |d|^2)
__device__ __forceinline__ double2 crecip(double2 d) {
  if (fabs(d.x) >= fabs(d.y)) {
    const double r = d.y / d.x, den = d.x + d.y * r;
    return make_double2(1.0 / den, -r / den);
  }
  const double r = d.x / d.y, den = d.x * r + d.y;
  return make_double2(r / den, -1.0 / den);
}
__device__ __forceinline__ void cacc(double2* p, double2 v) {
  p->x += v.x;
  p->y += v.y;
}


// ----------------------------------------------------------------------------
// factorization

__device__ __forceinline__ long long band_base_dev(int t, int kb) {  // hs_symbolic.hpp band_base
  const int j0 = kb >> 2;
  const long long s = t <= j0 ? 2LL * t * (t + 1) : 2LL * j0 * (j0 + 1) + static_cast<long long>(t - j0) * kb;
  return s * 256;
}

// One front per CTA (NC = 1), or per thread-block cluster of NC CTAs for large fronts (m up to
// several thousand in 3D): element loops, trailing-update tiles, the rows of M and W are split
// over the cluster; the panel LDL^T of each block column runs on rank 0 into its scratch, which
// the other CTAs read after a cluster barrier. Every phase boundary is a cluster barrier
// (release/acquire at cluster scope, which also orders the global-memory front).
template <int NC>
__global__ void __launch_bounds__(kThreads) factor_level_kernel(FactorArgs a, int use_smem,
                                                              long long scratch_stride) {
  extern __shared__ double2 sm[];
  const int tid = threadIdx.x;
  const int rank = NC == 1 ? 0 : static_cast<int>(blockIdx.x % NC);
  const int gtid = rank * kThreads + tid;   // thread index within the front's CTAs
  constexpr int GT = NC * kThreads;        // threads per front
  auto sync_front = [&]() {
    if constexpr (NC == 1)
      __syncthreads();
    else
      cg::this_cluster().sync();
  };
  const FactorTask task = a.tasks[blockIdx.x / NC];
  const DevSub& S = a.subs[task.sub];
  const DevClass& C = a.cls[S.cls];
  const DevFront f = C.fronts[task.front];
  const int m = f.m, k = f.k;
  double2* F = a.work + task.fbase + f.f_off;
  const long long mm = static_cast<long long>(m) * m;
  for (long long idx = gtid; idx < mm; idx += GT) F[idx] = czero();
  sync_front();
  // original entries of the separator rows, lower triangle (src/direct.cpp:219-237)
  for (int q = gtid; q < f.orig_cnt; q += GT) cacc(&F[C.orig_fpos[f.orig_off + q]], S.val[C.orig_eidx[f.orig_off + q]]);
  sync_front();
  // extend-add of the children's Schur complements (src/direct.cpp:239-265)
#pragma unroll 1
  for (int q = 0; q < 2; ++q) {
    const int ch = q ? f.child1 : f.child0;
    if (ch < 0) continue;
    const DevFront cf = C.fronts[ch];
    const double2* Fc = a.work + task.fbase + cf.f_off;
    const int cb = cf.m - cf.k;
    const int* cmap = C.child_map + (q ? f.cmap1 : f.cmap0);
    for (int idx = gtid; idx < cb * cb; idx += GT) {
      const int i = idx % cb, j = idx / cb;
      if (i >= j)
        cacc(&F[static_cast<long long>(cmap[j]) * m + cmap[i]],
             Fc[static_cast<long long>(cf.k + j) * cf.m + cf.k + i]);
    }
    sync_front();  // child by child: two children may add into the same entry
  }
  // panel buffers: rank 0's (shared by the cluster through global memory); own scratch for rows
  double2* Ps = use_smem ? sm : a.scratch + (blockIdx.x - rank) * scratch_stride;
  double2* Ws = Ps + static_cast<long long>(m) * kNB;
  double2* own = use_smem ? sm : a.scratch + blockIdx.x * scratch_stride;
#pragma unroll 1
  for (int p0 = 0; p0 < k; p0 += kNB) {
    const int p1 = min(p0 + kNB, k), nbw = p1 - p0, rows = m - p0, rows2 = m - p1;
    if (rank == 0) {  // panel LDL^T on rank 0 (CTA-local barriers)
    for (int idx = tid; idx < nbw * rows; idx += kThreads) {
      const int c = idx / rows, i = idx % rows;
      Ps[idx] = F[static_cast<long long>(p0 + c) * m + p0 + i];
    }
    __syncthreads();
    // unblocked right-looking LDL^T of the panel, full column height (src/direct.cpp:62-74)
#pragma unroll 1
    for (int jj = 0; jj < nbw; ++jj) {
      const double2 d = Ps[jj * rows + jj];
      if (tid == 0 && hypot(d.x, d.y) < S.tol)
        atomicMin(a.err_key, (static_cast<unsigned long long>(task.sub) << 32) |
                                 static_cast<unsigned>(f.sep_off + p0 + jj));
      const double2 inv = crecip(d);
      for (int i = jj + 1 + tid; i < rows; i += kThreads) Ps[jj * rows + i] = cmul(Ps[jj * rows + i], inv);
      __syncthreads();
      const int ncols = nbw - jj - 1;
      for (int idx = tid; idx < ncols * rows; idx += kThreads) {
        const int c = jj + 1 + idx / rows, i = idx % rows;
        if (i >= c) {
          const double2 s = cmul(d, Ps[jj * rows + c]);
          cfms(Ps[c * rows + i], Ps[jj * rows + i], s);
        }
      }
      __syncthreads();
    }
    for (int idx = tid; idx < nbw * rows2; idx += kThreads) {
      const int c = idx / rows2, i = idx % rows2;
      Ws[idx] = cmul(Ps[c * rows + (p1 - p0) + i], Ps[c * rows + c]);
    }
    for (int idx = tid; idx < nbw * rows; idx += kThreads) {
      const int c = idx / rows, i = idx % rows;
      F[static_cast<long long>(p0 + c) * m + p0 + i] = Ps[idx];
    }
    }  // rank 0
    sync_front();
    // trailing lower update F[p1:, p1:] -= L W^T in 64x64 tiles (split over the cluster), 4x4 per thread
    if (rows2 > 0) {
      const int nt = (rows2 + 63) / 64;
      const int ty = tid / 16, tx = tid % 16;
#pragma unroll 1
      for (int tp = rank; tp < nt * (nt + 1) / 2; tp += NC) {
        int ti = 0;
        while ((ti + 1) * (ti + 2) / 2 <= tp) ++ti;
        const int tc = tp - ti * (ti + 1) / 2;
        double2 acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = czero();
        int ir[4], ic[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ir[u] = ti * 64 + ty + 16 * u;  // offset from p1
          ic[u] = tc * 64 + tx + 16 * u;
        }
#pragma unroll 1
        for (int cc = 0; cc < nbw; ++cc) {
          double2 lr[4], wc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            lr[u] = ir[u] < rows2 ? Ps[cc * rows + (p1 - p0) + ir[u]] : czero();
            wc[u] = ic[u] < rows2 ? Ws[cc * rows2 + ic[u]] : czero();
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) cfma(acc[u][v], lr[u], wc[v]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v)
            if (ir[u] < rows2 && ic[v] < rows2 && ir[u] >= ic[v]) {
              double2& y = F[static_cast<long long>(p1 + ic[v]) * m + p1 + ir[u]];
              y = csub(y, acc[u][v]);
            }
      }
    }
    sync_front();
  }
  // D^-1, then the partitioned inverse of the eliminated columns: M = L11^-1 (unit lower)
  // and W = L21 M replace L11 / L21, so each front's solve is a dense product (hs_solve.cu).
  for (int j = gtid; j < k; j += GT) S.dinv[f.sep_off + j] = crecip(F[static_cast<long long>(j) * m + j]);
  double2* rowbuf = own;  // >= 32 m entries of this CTA's scratch (smem or global)
  sync_front();
#pragma unroll 1
  for (int i = 1; i < k; ++i) {  // M row i: M[i][j] = -sum_{l=j}^{i-1} L[i][l] M[l][j]
    for (int l = tid; l < i; l += kThreads) rowbuf[l] = F[static_cast<long long>(l) * m + i];
    sync_front();  // every CTA holds row i of L before any CTA overwrites it with row i of M
    for (int j = gtid; j < i; j += GT) {
      double2 acc = rowbuf[j];
      for (int l = j + 1; l < i; ++l) cfma(acc, rowbuf[l], F[static_cast<long long>(j) * m + l]);
      F[static_cast<long long>(j) * m + i] = make_double2(-acc.x, -acc.y);
    }
    sync_front();
  }
  {  // W rows: one warp per row, the row of L21 staged in a per-warp buffer
    const int warp = tid >> 5, lane = tid & 31;
    double2* wb = rowbuf + static_cast<long long>(warp) * k;
    for (int r = k + rank * kWarps + warp; r < m; r += NC * kWarps) {
      for (int l = lane; l < k; l += 32) wb[l] = F[static_cast<long long>(l) * m + r];
      __syncwarp();
      for (int j = lane; j < k; j += 32) {
        double2 acc = wb[j];
        for (int l = j + 1; l < k; ++l) cfma(acc, wb[l], F[static_cast<long long>(j) * m + l]);
        F[static_cast<long long>(j) * m + r] = acc;
      }
      __syncwarp();
    }
  }
  sync_front();
  // [M; W] in the solve layout (hs_symbolic.hpp front_block_elems): padded rows [sep | bnd],
  // 8x8 complex blocks row-major, bands of 4 block rows holding column blocks [0, min(kb, 4t+4)).
  {
    const int kp = (k + 7) & ~7, kb = kp >> 3, nrb = kb + ((m - k + 7) >> 3), nband = (nrb + 3) >> 2;
    auto val = [&](int pr, int pc) {
      if (pc >= k) return czero();
      if (pr < k) {
        if (pr > pc) return F[static_cast<long long>(pc) * m + pr];
        return pr == pc ? make_double2(1.0, 0.0) : czero();
      }
      const int row = k + pr - kp;  // boundary row of the front
      if (pr < kp || row >= m) return czero();
      return F[static_cast<long long>(pc) * m + row];
    };
    double2* P = S.factor + f.fac_off;
    for (int t = 0; t < nband; ++t) {
      const int rbs = min(4, nrb - 4 * t), ncb = min(kb, 4 * t + 4);
      double2* B = P + band_base_dev(t, kb);
      const int tot = ncb * rbs * 64;
      for (int idx = gtid; idx < tot; idx += GT) {
        const int blk = idx >> 6, e = idx & 63, cb = blk / rbs, i = blk % rbs;
        B[idx] = val(8 * (4 * t + i) + (e >> 3), 8 * cb + (e & 7));
      }
    }
  }
}

// ----------------------------------------------------------------------------
// sweep kernels

__device__ __forceinline__ int weight2(const DevGeom& g, int axis, int cell, int index) {
  const int w = g.cut_w[axis];
  const int lo = cell * w, hi = (cell + 1) * w;
  const int lo_ext = cell == 0 ? lo - g.pad : lo;
  const int hi_ext = cell == g.counts[axis] - 1 ? hi + g.pad : hi;
  if (index < lo_ext || index > hi_ext) return 0;
  if (index == lo && cell > 0) return 1;
  if (index == hi && cell < g.counts[axis] - 1) return 1;
  return 2;
}

constexpr int HS_SLOTS_PER_DIR = 16;  // generating sweeps that can route into one sweep and face

__device__ __forceinline__ double2* task_x(const SweepArgs& a, const DevSub& S, int l) {
  return S.x + static_cast<long long>((l - 1) % a.nbuf) * a.xstride;
}
// the right-hand side of the macro-step's task t lives in slot t
__device__ __forceinline__ double2* task_b(const SweepArgs& a, int t) {
  return a.rbs + static_cast<long long>(t) * a.slot_stride;
}

// RHS of a task before injection (src/sweeper.cpp:189-239). Sweep 1: the split source
// w(sub, p) * b[p] off the local shell (src/sweeper.cpp:189-202), written over the whole buffer.
// Later sweeps: zero, which the buffer already is except on the injection lines of its previous
// use; those are cleared (the whole buffer when that use was a sweep-1 task).
__global__ void rhs_init_kernel(SweepArgs a) {
  const int sub = a.tasks[blockIdx.y].x, l = a.tasks[blockIdx.y].y;
  const DevSub& S = a.subs[sub];
  double2* B = task_b(a, blockIdx.y);
  const DevClass& C = a.cls[S.cls];
  const int dim = a.g.dim;
  const int2 prev = a.prev[blockIdx.y];
  if (l > 1 && prev.y == 0) {  // the slot is zero off its previous occupant's injection lines: clear those
    if (prev.x < 0) return;
    const DevClass& P = a.cls[prev.x];
    for (int d = 0; d < a.dirs; ++d) {
      const int len = P.line_len[d];
      for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < len * a.R;
           idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx / a.R), r = static_cast<int>(idx % a.R);
        const int p0 = P.inj_p0[d][i], pm = P.inj_pm[d][i];
        if (p0 >= 0) B[static_cast<long long>(p0) * a.R + r] = czero();
        if (pm >= 0) B[static_cast<long long>(pm) * a.R + r] = czero();
      }
    }
    return;
  }
  // sweep 1 (or a slot whose previous occupant wrote all of it): split source / zero over the
  // whole buffer (the larger of this class's and the previous occupant's extent); nonzero bits of
  // positions off the injection lines are final here (lines: nonzero_kernel)
  const long long total = a.slot_stride;  // the whole slot: every occupant then keeps it zero off its lines
  const double inv = 1.0 / static_cast<double>(1 << dim);
  rmask bits = 0, anyb = 0;
  // Four elements per thread and iteration, their loads issued in two waves (weight / global node /
  // on-line flag, then b): one element at a time the weight -> node -> b chain left a thread with
  // 16 bytes in flight per three memory round trips (ncu: 43% of HBM bandwidth on sweep-1 steps).
  constexpr int U = 4;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long nloc = l == 1 ? static_cast<long long>(C.n) * a.R : 0;
  const unsigned R = static_cast<unsigned>(a.R);
  for (long long base = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; base < total; base += U * stride) {
    int wn[U], gp[U];
    unsigned rr[U];
    bool line[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const long long idx = base + q * stride;
      const bool in = idx < nloc;
      // (element indices fit 32 bits: a slot holds n_max * R < 2^31 values)
      const unsigned e = static_cast<unsigned>(idx) / R;
      rr[q] = static_cast<unsigned>(idx) - e * R;
      wn[q] = in ? S.split_w[e] : 0;
      gp[q] = in ? S.split_gp[e] : 0;
      line[q] = in ? C.on_line[e] != 0 : true;
    }
    double2 bv[U];
#pragma unroll
    for (int q = 0; q < U; ++q) bv[q] = wn[q] ? a.b[static_cast<long long>(gp[q]) * a.R + rr[q]] : czero();
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const long long idx = base + q * stride;
      if (idx >= total) break;
      double2 v = czero();
      if (wn[q]) {
        const double w = wn[q] * inv;
        v = make_double2(w * bv[q].x, w * bv[q].y);
        if (v.x != 0.0 || v.y != 0.0) {
          anyb |= 1ull << rr[q];
          if (!line[q]) bits |= 1ull << rr[q];
        }
      }
      B[idx] = v;
    }
  }
  if (l == 1) {
    bits = reduce_or64(bits);
    if ((threadIdx.x & 31) == 0 && bits) atomicOr(&a.nzmask[static_cast<long long>(l - 1) * a.g.nsub + sub], bits);
    // 8-column groups in which the split source is nonzero somewhere in this subdomain (on or off
    // the lines): every front is live for them (bits 16 + group of the task's face word). The other
    // columns of a sweep-1 task only carry injected traces, like the tasks of later sweeps: their
    // live fronts follow from the receiving faces (nonzero_kernel)
    anyb = reduce_or64(anyb);
    unsigned gb = 0;
    for (int g8 = 0; g8 < 8; ++g8)
      if ((anyb >> (8 * g8)) & 0xFFull) gb |= 1u << g8;
    if (gb && (threadIdx.x & 31) == 0) atomicOr(&a.tface[static_cast<long long>(l - 1) * a.g.nsub + sub], gb << 16);
  }
}

// trace_to_source of the mailbox slots of sweep l (src/transfer.cpp:68-89) for the two faces of
// one axis. The faces' lines are disjoint, so every (task, line chunk) is its own block; the axes
// are separate launches in the reference's (axis, sign) order, which fixes the order at the nodes
// where lines of different axes cross. Deposits are kept per generating sweep (one writer per
// slot) and summed here in generating-sweep order: the reference mailbox's "first deposit copies,
// later deposits add" (src/transfer.cpp:30-35).
constexpr int kInjectChunk = 1024;  // line x RHS elements per block
__global__ void inject_kernel(SweepArgs a, int axis) {
  const int sub = a.tasks[blockIdx.y].x, l = a.tasks[blockIdx.y].y;
  const DevSub& S = a.subs[sub];
  const DevClass& C = a.cls[S.cls];
  double2* B = task_b(a, blockIdx.y);  // the task's right-hand side
  const int R = a.R;
  __shared__ long long s_slot[2][HS_SLOTS_PER_DIR];
  __shared__ rmask s_pres[2][HS_SLOTS_PER_DIR];
  __shared__ int s_n[2];
  if (threadIdx.x < 64) {
    // warp q lists face q's generating sweeps with a deposit, in ascending order: a lane per
    // candidate sweep, compacted by ballot (one thread walking route -> presence word sweep by
    // sweep was a chain of up to 2 * l dependent loads ahead of every block's work)
    const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int d = 2 * axis + q;
    int n = 0;
    for (int lg0 = 1; lg0 <= l && n < HS_SLOTS_PER_DIR; lg0 += 32) {
      const int lg = lg0 + lane;
      long long slot = 0;
      rmask pres = 0;
      if (lg <= l && a.route[(lg - 1) * a.dirs + d] == l) {
        slot = (static_cast<long long>(sub) * a.nsweeps + (lg - 1)) * a.dirs + d;
        pres = a.mpres[slot];
      }
      const unsigned have = __ballot_sync(kFull, pres != 0);
      const int at = n + __popc(have & ((1u << lane) - 1u));
      if (pres != 0 && at < HS_SLOTS_PER_DIR) {
        s_slot[q][at] = slot;
        s_pres[q][at] = pres;
      }
      n = min(n + __popc(have), HS_SLOTS_PER_DIR);
    }
    if (lane == 0) s_n[q] = n;
  }
  __syncthreads();
#pragma unroll 1
  for (int q = 0; q < 2; ++q) {
    const int d = 2 * axis + q, n = s_n[q];
    if (n == 0) continue;
    const int len = C.line_len[d];
    const int idx = blockIdx.x * kInjectChunk + threadIdx.x;
    if (idx >= len * R) continue;
    const int i = idx / R, r = idx % R;
    double2 u0 = czero(), um1 = czero();
    bool first = true;
    for (int k = 0; k < n; ++k) {
      if (!((s_pres[q][k] >> r) & 1ull)) continue;
      const double2* s0 = a.mbox + s_slot[q][k] * a.mbox_dir_stride;
      const double2 v0 = s0[idx], v1 = s0[static_cast<long long>(len) * R + idx];
      u0 = first ? v0 : cadd(u0, v0);
      um1 = first ? v1 : cadd(um1, v1);
      first = false;
    }
    if (first) continue;
    const double2 c = S.coef[d][i];
    const int p0 = C.inj_p0[d][i], pm = C.inj_pm[d][i];
    if (p0 >= 0) cfms(B[static_cast<long long>(p0) * R + r], c, um1);
    if (pm >= 0) cfma(B[static_cast<long long>(pm) * R + r], c, u0);
  }
}

// Exact-zero test of a task's RHS (src/sweeper.cpp:240-251) on the injection lines; positions off
// the lines were tested by rhs_init (sweep 1) or are zero (later sweeps).
__global__ void nonzero_kernel(SweepArgs a) {
  const int sub = a.tasks[blockIdx.y].x, l = a.tasks[blockIdx.y].y;
  const DevSub& S = a.subs[sub];
  const DevClass& C = a.cls[S.cls];
  const double2* B = task_b(a, blockIdx.y);
  const int R = a.R;
  rmask bits = 0;
  unsigned faces = 0;
  {
    for (int d = 0; d < a.dirs; ++d) {
      const int len = C.line_len[d];
      const rmask b0 = bits;
      bits = 0;
      for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < len * R;
           idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx / R), r = static_cast<int>(idx % R);
        const int p0 = C.inj_p0[d][i], pm = C.inj_pm[d][i];
        if (p0 >= 0) {
          const double2 v = B[static_cast<long long>(p0) * R + r];
          if (v.x != 0.0 || v.y != 0.0) bits |= 1ull << r;
        }
        if (pm >= 0) {
          const double2 v = B[static_cast<long long>(pm) * R + r];
          if (v.x != 0.0 || v.y != 0.0) bits |= 1ull << r;
        }
      }
      if (bits) faces |= 1u << d;
      bits |= b0;
    }
  }
  bits = reduce_or64(bits);
  faces = __reduce_or_sync(kFull, faces);
  // Only faces whose mailbox slots some generating sweep fills for this sweep carry injected data;
  // lines of other faces can hold a nonzero value only where they cross a receiving face's line,
  // at nodes whose fronts are live through that face. The host prunes the forward item lists with
  // the same static face set (DdmHandle::build_items), so the run-time set must stay inside it: a
  // front listed as dead must never be waited for.
  unsigned recv = 0;
  for (int d = 0; d < a.dirs; ++d) {
    const int ax = d >> 1, nb = S.sub[ax] - ((d & 1) ? 1 : -1);
    if (nb < 0 || nb >= a.g.counts[ax]) continue;
    for (int lg = 1; lg <= l; ++lg)
      if (a.route[(lg - 1) * a.dirs + d] == l) {
        recv |= 1u << d;
        break;
      }
  }
  faces &= recv;
  const long long ti = static_cast<long long>(l - 1) * a.g.nsub + sub;
  if ((threadIdx.x & 31) == 0 && bits) atomicOr(&a.nzmask[ti], bits);
  // (the column groups of a sweep-1 task that hold part of the split source were marked all-live by rhs_init)
  if ((threadIdx.x & 31) == 0 && faces) atomicOr(&a.tface[ti], faces);
}

// extract_trace (src/transfer.cpp:47-66) + route_trace (src/sweeper.cpp:58-73) + deposit into the
// target's slot of this generating sweep (unique writer: plain stores, presence = RHS columns).
constexpr int kExtractPer = 4;  // line x RHS elements per thread
__global__ void extract_deposit_kernel(SweepArgs a) {
  const int task = blockIdx.y / a.dirs, d = blockIdx.y % a.dirs;
  const int sub = a.tasks[task].x, l = a.tasks[task].y;
  const int axis = d >> 1, sign = (d & 1) ? 1 : -1;
  const DevSub& S = a.subs[sub];
  const int t = S.sub[axis] + sign;
  if (t < 0 || t >= a.g.counts[axis]) return;
  if (a.route[(l - 1) * a.dirs + d] == 0) return;
  const rmask nz = a.nzmask[static_cast<long long>(l - 1) * a.g.nsub + sub];
  if (nz == 0) return;
  int stride = 1;
  for (int ax = 0; ax < axis; ++ax) stride *= a.g.counts[ax];
  const int target = sub + sign * stride;
  const DevClass& C = a.cls[S.cls];
  const double2* X = task_x(a, S, l);
  const int R = a.R, len = C.line_len[d];
  const long long slot = (static_cast<long long>(target) * a.nsweeps + (l - 1)) * a.dirs + d;
  double2* u0 = a.mbox + slot * a.mbox_dir_stride;
  double2* um1 = u0 + static_cast<long long>(len) * R;
  // kExtractPer elements per thread, all of a thread's index loads, then all of its x loads in
  // flight together (one element per thread made 8000 blocks of one index -> x -> store chain
  // each: 7 block waves per launch, 17 us for 70 MB)
  int e0[kExtractPer], e1[kExtractPer];
#pragma unroll
  for (int q = 0; q < kExtractPer; ++q) {
    const int idx = (blockIdx.x * kExtractPer + q) * blockDim.x + threadIdx.x;
    const bool on = idx < len * R && ((nz >> (idx % R)) & 1ull);
    e0[q] = on ? C.ext_u0[d][idx / R] : -1;
    e1[q] = on ? C.ext_um1[d][idx / R] : -1;
  }
  double2 v0[kExtractPer], v1[kExtractPer];
#pragma unroll
  for (int q = 0; q < kExtractPer; ++q) {
    const int idx = (blockIdx.x * kExtractPer + q) * blockDim.x + threadIdx.x;
    const int r = idx % R;
    v0[q] = e0[q] >= 0 ? X[static_cast<long long>(e0[q]) * R + r] : czero();
    v1[q] = e1[q] >= 0 ? X[static_cast<long long>(e1[q]) * R + r] : czero();
  }
#pragma unroll
  for (int q = 0; q < kExtractPer; ++q) {
    const int idx = (blockIdx.x * kExtractPer + q) * blockDim.x + threadIdx.x;
    if (e0[q] >= 0) {
      u0[idx] = v0[q];
      um1[idx] = v1[q];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.mpres[slot] = nz;
}

// u += sum over the subdomains whose support holds the node of w * u_local, in the reference's
// order (step of the sweep, then ascending id: src/sweeper.cpp:285-309, src/transfer.cpp:91-102).
// The host precomputes, per sweep direction, each node's entries already in that order.
template <int E>
__global__ void __launch_bounds__(kThreads) accumulate_kernel(AccumArgs a) {
  __shared__ double red[kThreads];
  const int dim = a.g.dim, R = a.R;
  const int npb = kThreads / R;  // whole nodes per block so thread t always owns column t % R
  const long long node = a.n0 + static_cast<long long>(blockIdx.x) * npb + threadIdx.x / R;
  const int r = threadIdx.x % R;
  double nrm = 0.0;
  if (threadIdx.x < npb * R && node < a.n1) {
    int2 ent[E];
#pragma unroll
    for (int e = 0; e < E; ++e) ent[e] = __ldg(a.acc_ent + node * E + e);
    // every load of the node is issued before the sum; tasks skipped for an exactly-zero RHS
    // column (nzmask) contribute nothing, as in the reference, and their x buffer is not read
    const double2 uv = a.u[node * R + r];
    double2 xv[E];
    bool on[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      on[i] = ent[i].x >= 0 && ((a.nzmask[ent[i].y >> 4] >> r) & 1ull);
      xv[i] = on[i] ? a.x[a.xoff + static_cast<long long>(ent[i].x) * R + r] : czero();
    }
    double2 acc = czero();
    const double inv = 1.0 / static_cast<double>(1 << dim);
#pragma unroll
    for (int i = 0; i < E; ++i) {
      if (!on[i]) continue;
      const double w = (ent[i].y & 15) * inv;
      acc.x += w * xv[i].x;
      acc.y += w * xv[i].y;
    }
    a.u[node * R + r] = cadd(uv, acc);
    nrm = acc.x * acc.x + acc.y * acc.y;
  }
  red[threadIdx.x] = nrm;
  __syncthreads();
  if (threadIdx.x < R) {
    double s = 0.0;
    for (int q = threadIdx.x; q < kThreads; q += R) s += red[q];
    a.partial[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = s;
  }
}

// Deterministic two-stage reduction of per-block partials out[r] = sum_b partial[b][r]: stage 1
// sums a fixed contiguous range of rows per block (coalesced rows, fixed tree), stage 2 sums the
// stage-1 results in block order.
constexpr int kReduceBlocks = kReducePad;
__global__ void reduce_partials_stage1(const double* partial, int nblocks, int R, double* mid) {
  __shared__ double red[kThreads];
  const int rows_per_iter = kThreads / R, row = threadIdx.x / R, r = threadIdx.x % R;
  const int per = (nblocks + gridDim.x - 1) / gridDim.x, b0 = blockIdx.x * per, b1 = min(nblocks, b0 + per);
  double s = 0.0;
  if (row < rows_per_iter)
    for (int b = b0 + row; b < b1; b += rows_per_iter) s += partial[static_cast<long long>(b) * R + r];
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < R) {
    double t = 0.0;
    for (int q = 0; q < rows_per_iter; ++q) t += red[q * R + threadIdx.x];
    mid[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = t;
  }
}
__global__ void reduce_partials_stage2(const double* mid, int nmid, int R, double* out) {
  const int r = blockIdx.x, lane = threadIdx.x;  // one warp (block) per column, fixed tree
  if (r >= R) return;
  double s = 0.0;
  for (int b = lane; b < nmid; b += 32) s += mid[static_cast<long long>(b) * R + r];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) out[r] = s;
}

__global__ void reduce_cpartials_kernel(const double2* partial, int nblocks, int R, double2* out) {
  __shared__ double2 red[kThreads];
  const int r = blockIdx.x;
  double2 s = czero();
  for (int b = threadIdx.x; b < nblocks; b += kThreads) s = cadd(s, partial[static_cast<long long>(b) * R + r]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = cadd(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[r] = red[0];
}

constexpr int kResThreads = 512;  // rows x RHS per block (64-RHS batches still get 8 rows per block)
constexpr int kResRows = 8;       // grid rows a block walks: a row's x is the next row's lower neighbour (L1 hit)
// Rows are taken in tiles of (kResThreads / R nodes along x) x kResRows grid rows: the operator is a
// 5 / 7-point stencil, so a block walking up its columns re-reads each x row from L1 instead of
// three times from L2 (ncu: the one-row blocks ran at 38% of HBM bandwidth with L2 as the bound).
// gx = 0: rows in plain order (any CSR matrix; the column indices are used either way).
__global__ void __launch_bounds__(kResThreads) residual_kernel(long long n, const std::int64_t* row_ptr, const int* col,
                                                                const double2* val, const double2* x, const double2* b,
                                                                int R, double* pnum, double* pden, int gx, int tiles_x) {
  __shared__ double rn[kResThreads], rd[kResThreads];
  const int npb = kResThreads / R;
  const int tn = threadIdx.x / R, r = threadIdx.x % R;
  double num = 0.0, den = 0.0;
  const int iters = gx > 0 ? kResRows : 1;
  const long long bx = gx > 0 ? blockIdx.x % tiles_x : 0, by = gx > 0 ? blockIdx.x / tiles_x : 0;
  for (int j = 0; j < iters; ++j) {
    long long row;
    bool ok = tn < npb;
    if (gx > 0) {
      const long long xi = bx * npb + tn;
      row = (by * kResRows + j) * gx + xi;
      ok = ok && xi < gx;
    } else {
      row = static_cast<long long>(blockIdx.x) * npb + tn;
    }
    if (!ok || row >= n) continue;
    // all of the row's loads in flight before the sum (rows hold <= 7 entries: 2D 5, 3D 7)
    const long long e0 = row_ptr[row], e1 = row_ptr[row + 1];
    double2 s = czero();
    // Interior rows of the 5 / 7-point operator: exactly N entries, every load unconditional and
    // issued before the sums (with predicated loads the compiler chained column index -> x ->
    // multiply-add one entry at a time: 70% long-scoreboard stalls, 36% of HBM bandwidth).
    auto fixed = [&](auto nn) {
      constexpr int N = decltype(nn)::value;
      int c[N];
      double2 v[N], xv[N];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        c[q] = col[e0 + q];
        v[q] = val[e0 + q];
      }
#pragma unroll
      for (int q = 0; q < N; ++q) xv[q] = x[static_cast<long long>(c[q]) * R + r];
#pragma unroll
      for (int q = 0; q < N; ++q) cfma(s, v[q], xv[q]);
    };
    if (e1 - e0 == 5) {
      fixed(std::integral_constant<int, 5>{});
    } else if (e1 - e0 == 7) {
      fixed(std::integral_constant<int, 7>{});
    } else
    for (long long eb = e0; eb < e1; eb += 8) {
      double2 v[8], xv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const bool in = eb + q < e1;
        v[q] = in ? val[eb + q] : czero();
        xv[q] = in ? x[static_cast<long long>(col[eb + q]) * R + r] : czero();
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (eb + q < e1) cfma(s, v[q], xv[q]);
    }
    const double2 bv = b[row * R + r];
    const double2 dv = csub(bv, s);
    num += dv.x * dv.x + dv.y * dv.y;
    den += bv.x * bv.x + bv.y * bv.y;
  }
  rn[threadIdx.x] = num;
  rd[threadIdx.x] = den;
  __syncthreads();
  if (threadIdx.x < R) {
    double s1 = 0.0, s2 = 0.0;
    for (int q = threadIdx.x; q < npb * R; q += R) {
      s1 += rn[q];
      s2 += rd[q];
    }
    pnum[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = s1;
    pden[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = s2;
  }
}

// Residual partials with the operator in stencil form (StencilOp): the coefficients (broadcast) and
// the x values of a row are all independent loads. The CSR form walks row pointer -> column index
// -> x (ncu: 70% long-scoreboard stalls, 36% of HBM bandwidth). Same tiles and the same per-row
// sums in CSR column order as residual_kernel.
template <int S>
__global__ void __launch_bounds__(kResThreads) residual_stencil_kernel(long long n, StencilOp op, const double2* x,
                                                                        const double2* b, int R, double* pnum,
                                                                        double* pden, int gx, int tiles_x) {
  __shared__ double rn[kResThreads], rd[kResThreads];
  const int npb = kResThreads / R;
  const int tn = threadIdx.x / R, r = threadIdx.x % R;
  double num = 0.0, den = 0.0;
  const long long bx = blockIdx.x % tiles_x, by = blockIdx.x / tiles_x;
  const long long xi = bx * npb + tn;
#pragma unroll 2
  for (int j = 0; j < kResRows; ++j) {
    const long long row = (by * kResRows + j) * gx + xi;
    if (tn >= npb || xi >= gx || row >= n) continue;
    double2 v[S], xv[S];
#pragma unroll
    for (int q = 0; q < S; ++q) {
      v[q] = __ldg(op.val + row * S + q);
      const long long c = min(max(row + op.off[q], 0LL), n - 1);  // (an absent entry's coefficient is zero)
      xv[q] = x[c * R + r];
    }
    const double2 bv = b[row * R + r];
    double2 s = czero();
#pragma unroll
    for (int q = 0; q < S; ++q)
      if (v[q].x != 0.0 || v[q].y != 0.0) cfma(s, v[q], xv[q]);
    const double2 dv = csub(bv, s);
    num += dv.x * dv.x + dv.y * dv.y;
    den += bv.x * bv.x + bv.y * bv.y;
  }
  rn[threadIdx.x] = num;
  rd[threadIdx.x] = den;
  __syncthreads();
  if (threadIdx.x < R) {
    double s1 = 0.0, s2 = 0.0;
    for (int q = threadIdx.x; q < npb * R; q += R) {
      s1 += rn[q];
      s2 += rd[q];
    }
    pnum[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = s1;
    pden[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = s2;
  }
}

__global__ void stencil_build_kernel(long long n, const std::int64_t* row_ptr, const int* col, const double2* val,
                                     StencilOp op, double2* out, unsigned* bad) {
  const long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (row >= n) return;
  for (int q = 0; q < op.S; ++q) out[row * op.S + q] = czero();
  for (std::int64_t e = row_ptr[row]; e < row_ptr[row + 1]; ++e) {
    const long long d = static_cast<long long>(col[e]) - row;
    int q = 0;
    while (q < op.S && op.off[q] != d) ++q;
    if (q < op.S)
      out[row * op.S + q] = val[e];
    else
      *bad = 1u;
  }
}

__global__ void spmv_kernel(long long n, const std::int64_t* row_ptr, const int* col, const double2* val,
                            const double2* x, double2* y, int R) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= n * R) return;
  const long long row = idx / R;
  const int r = static_cast<int>(idx % R);
  double2 s = czero();
  for (long long e = row_ptr[row]; e < row_ptr[row + 1]; ++e) cfma(s, val[e], x[static_cast<long long>(col[e]) * R + r]);
  y[idx] = s;
}

__global__ void dot_partials_kernel(const double2* a, const double2* b, long long n, int R, double2* partial) {
  __shared__ double2 red[kThreads];
  const int npb = kThreads / R;
  const long long node = static_cast<long long>(blockIdx.x) * npb + threadIdx.x / R;
  const long long idx = node * R + threadIdx.x % R;
  double2 s = czero();
  if (threadIdx.x < npb * R && node < n) {  // conj(a) * b (src/krylov.cpp:9-13)
    const double2 x = a[idx], y = b[idx];
    s = make_double2(x.x * y.x + x.y * y.y, x.x * y.y - x.y * y.x);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < R) {
    double2 t = czero();
    for (int q = threadIdx.x; q < kThreads; q += R) t = cadd(t, red[q]);
    partial[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = t;
  }
}

__global__ void axpy_cols_kernel(double2* y, const double2* x, const double2* alpha, int neg, long long n, int R) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= n * R) return;
  double2 al = alpha[idx % R];
  if (neg) al = make_double2(-al.x, -al.y);
  cfma(y[idx], al, x[idx]);
}

__global__ void scale_cols_kernel(double2* y, const double* inv, long long n, int R) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= n * R) return;
  const double s = inv[idx % R];
  y[idx] = make_double2(y[idx].x * s, y[idx].y * s);
}

// RHS-major [R][N] <-> node-major [N][R] for nodes [n0, n1): 32 nodes x R per block through
// shared memory, so both sides are coalesced.
constexpr int kTransNodes = 32;
__global__ void transpose_in_kernel(const double2* src, double2* dst, long long n, int R, long long n0, long long n1,
                                    const int* perm) {
  __shared__ double2 tile[kTransNodes][kMaxRhs + 1];
  const long long base = n0 + static_cast<long long>(blockIdx.x) * kTransNodes;
  for (int e = threadIdx.x; e < kTransNodes * R; e += blockDim.x) {  // read rows of src: r, then node
    const int r = e / kTransNodes, i = e % kTransNodes;
    if (base + i < n1) tile[i][r] = src[static_cast<long long>(perm ? perm[r] : r) * n + base + i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kTransNodes * R; e += blockDim.x) {  // write node-major
    const int i = e / R, r = e % R;
    if (base + i < n1) dst[(base + i) * R + r] = tile[i][r];
  }
}
__global__ void transpose_out_kernel(const double2* src, double2* dst, long long n, int R, long long n0, long long n1,
                                    const int* perm) {
  __shared__ double2 tile[kTransNodes][kMaxRhs + 1];
  const long long base = n0 + static_cast<long long>(blockIdx.x) * kTransNodes;
  for (int e = threadIdx.x; e < kTransNodes * R; e += blockDim.x) {  // read node-major
    const int i = e / R, r = e % R;
    if (base + i < n1) tile[i][r] = src[(base + i) * R + r];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kTransNodes * R; e += blockDim.x) {  // write rows of dst
    const int r = e / kTransNodes, i = e % kTransNodes;
    if (base + i < n1) dst[static_cast<long long>(perm ? perm[r] : r) * n + base + i] = tile[i][r];
  }
}

// The same for a tile of rows [row0, row0 + gridDim.y) x columns [x0, x1) of the fastest axis
// (gx nodes per row): block (i, y) transposes 32 nodes of row row0 + y.
__global__ void transpose_in_tile_kernel(const double2* src, double2* dst, long long n, int R, int gx, int x0, int x1,
                                         long long row0, const int* perm) {
  __shared__ double2 tile[kTransNodes][kMaxRhs + 1];
  const long long rowb = (row0 + blockIdx.y) * gx;
  const long long base = rowb + x0 + static_cast<long long>(blockIdx.x) * kTransNodes, end = rowb + x1;
  for (int e = threadIdx.x; e < kTransNodes * R; e += blockDim.x) {
    const int r = e / kTransNodes, i = e % kTransNodes;
    if (base + i < end) tile[i][r] = src[static_cast<long long>(perm ? perm[r] : r) * n + base + i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kTransNodes * R; e += blockDim.x) {
    const int i = e / R, r = e % R;
    if (base + i < end) dst[(base + i) * R + r] = tile[i][r];
  }
}

__global__ void transpose_out_tile_kernel(const double2* src, double2* dst, long long n, int R, int gx, int x0, int x1,
                                          long long row0, const int* perm) {
  __shared__ double2 tile[kTransNodes][kMaxRhs + 1];
  const long long rowb = (row0 + blockIdx.y) * gx;
  const long long base = rowb + x0 + static_cast<long long>(blockIdx.x) * kTransNodes, end = rowb + x1;
  for (int e = threadIdx.x; e < kTransNodes * R; e += blockDim.x) {
    const int i = e / R, r = e % R;
    if (base + i < end) tile[i][r] = src[(base + i) * R + r];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kTransNodes * R; e += blockDim.x) {
    const int r = e / kTransNodes, i = e % kTransNodes;
    if (base + i < end) dst[static_cast<long long>(perm ? perm[r] : r) * n + base + i] = tile[i][r];
  }
}

__global__ void bump_epoch_kernel(unsigned* e, unsigned by) { *e += by; }

int blocks_for(long long n, int t = kThreads) { return static_cast<int>((n + t - 1) / t); }

}  // namespace

size_t factor_smem_bytes(int max_m) { return static_cast<size_t>(2) * max_m * kNB * sizeof(double2); }

void launch_factor_level(const FactorArgs& a, int max_m, cudaStream_t s) {
  static PerDevice configured;
  configured.get([](int) {
    HS_CUDA(cudaFuncSetAttribute(factor_level_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    return 1;
  });
  const size_t need = factor_smem_bytes(max_m);
  const bool use_smem = need <= 200 * 1024;
  factor_level_kernel<1><<<a.ntasks, kThreads, use_smem ? need : 0, s>>>(
      a, use_smem ? 1 : 0, static_cast<long long>(2) * max_m * kNB);
  after_launch();
}

// Large fronts: one thread-block cluster of kFactorCluster CTAs per front, scratch (global) per CTA.
void launch_factor_level_cluster(const FactorArgs& a, int max_m, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(a.ntasks) * kFactorCluster);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kFactorCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HS_CUDA(cudaLaunchKernelEx(&cfg, factor_level_kernel<kFactorCluster>, a, 0, static_cast<long long>(2) * max_m * kNB));
  after_launch();
}

// Pack (arrays -> message) or unpack (message -> arrays) of one exchange, a block per segment.
__global__ void __launch_bounds__(kThreads) xpack_kernel(const XSeg* segs, bool pack, double* buf, double2* mbox,
                                                         rmask* mpres, double2* x, rmask* nz,
                                                         const long long* gpos, int R) {
  const XSeg sg = segs[blockIdx.x];
  double* B = buf + sg.b;
  if (sg.kind == 1 || sg.kind == 3) {
    rmask* w = sg.kind == 1 ? mpres + sg.a : nz + sg.a;
    if (threadIdx.x == 0) {  // a 64-bit mask travels as the bit pattern of one double (no arithmetic)
      if (pack)
        B[0] = __longlong_as_double(static_cast<long long>(*w));
      else
        *w = static_cast<rmask>(__double_as_longlong(B[0]));
    }
    return;
  }
  for (int i = threadIdx.x; i < sg.count; i += blockDim.x) {
    double2* p;
    if (sg.kind == 0) {
      p = mbox + sg.a + i;
    } else {
      const long long pos = gpos[sg.a + i / R];
      p = x + sg.c + pos * R + i % R;
    }
    if (pack) {
      const double2 v = *p;
      B[2 * i] = v.x;
      B[2 * i + 1] = v.y;
    } else {
      *p = make_double2(B[2 * i], B[2 * i + 1]);
    }
  }
}

// Owner-slab gather of u (partitioned solves): each rank packs the values of its home nodes, an
// all-gather moves the slabs, and every rank scatters all slabs into u. Every node is nonzero on
// its home rank only, so this equals the sum over ranks bit for bit, at half an all-reduce's traffic.
__global__ void pack_home_kernel(const double2* u, const int* list, long long count, int R, double2* out) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= count * R) return;
  out[i] = u[static_cast<long long>(list[i / R]) * R + i % R];
}
__global__ void unpack_home_kernel(const double2* in, const int* lists, long long max_home, int R, double2* u) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long slab = static_cast<long long>(blockIdx.y) * max_home;
  if (i >= max_home * R) return;
  const int node = lists[slab + i / R];
  if (node >= 0) u[static_cast<long long>(node) * R + i % R] = in[slab * R + i];
}
void launch_pack_home(const double2* u, const int* list, long long count, int R, double2* out, cudaStream_t s) {
  if (count <= 0) return;
  pack_home_kernel<<<blocks_for(count * R), kThreads, 0, s>>>(u, list, count, R, out);
  after_launch();
}
void launch_unpack_home(const double2* in, const int* lists, long long max_home, int world, int R, double2* u,
                        cudaStream_t s) {
  if (max_home <= 0) return;
  unpack_home_kernel<<<dim3(blocks_for(max_home * R), world), kThreads, 0, s>>>(in, lists, max_home, R, u);
  after_launch();
}

void launch_xpack(const XSeg* segs, int nseg, bool pack, double* buf, double2* mbox, rmask* mpres, double2* x,
                  rmask* nzmask, const long long* gpos, int R, cudaStream_t s) {
  if (nseg <= 0) return;
  xpack_kernel<<<nseg, kThreads, 0, s>>>(segs, pack, buf, mbox, mpres, x, nzmask, gpos, R);
  after_launch();
}

// max_n = 0: no task of the launch rewrites its whole buffer (lines only)
void launch_build_rhs(const SweepArgs& a, long long max_n, int max_line, cudaStream_t s) {
  const int bx = std::max(1, std::min(blocks_for(std::max<long long>(max_n, max_line) * a.R), 512));
  rhs_init_kernel<<<dim3(bx, a.ntasks), kThreads, 0, s>>>(a);
  after_launch();
  const int nchunk = std::max(1, (max_line * a.R + kInjectChunk - 1) / kInjectChunk);
  for (int axis = 0; axis < a.dirs / 2; ++axis) {
    inject_kernel<<<dim3(nchunk, a.ntasks), kInjectChunk, 0, s>>>(a, axis);
    after_launch();
  }
  // a block per kThreads line elements of the longest face (each element is an index -> value chain)
  nonzero_kernel<<<dim3(std::max(1, std::min(blocks_for(static_cast<long long>(max_line) * a.R), 128)), a.ntasks),
                   kThreads, 0, s>>>(a);
  after_launch();
}

void launch_extract_deposit(const SweepArgs& a, int max_line, cudaStream_t s) {
  const int nchunk = std::max(1, (max_line * a.R + kThreads * kExtractPer - 1) / (kThreads * kExtractPer));
  extract_deposit_kernel<<<dim3(nchunk, a.ntasks * a.dirs), kThreads, 0, s>>>(a);
  after_launch();
}

constexpr int kAccThreads = 256;
#ifndef HS_ACC_MINB
#define HS_ACC_MINB 4
#endif
// LT: the number of sweeps when it is 4 or 8 (one straight-line body the compiler can schedule
// across sweeps), 0: any number up to HS_MAX_ACC_SWEEPS (early exit per sweep).
template <int E, int LT>
__global__ void __launch_bounds__(kAccThreads, HS_ACC_MINB) accumulate_all_kernel(AccumAllArgs a) {
  // One thread per (node, RHS pair): its two x values are independent 16-byte loads, so a thread
  // keeps twice the bytes in flight of the one-RHS form (ncu: 37% of HBM bandwidth, bound by the
  // bytes in flight per SM). Per-sweep |c_l|^2 terms go straight to shared memory (no registers
  // held across the sweeps) and are reduced once at the end (one barrier).
  constexpr int LM = LT ? LT : HS_MAX_ACC_SWEEPS;
  __shared__ double red[LM][2][kAccThreads];
  const int dim = a.g.dim, R = a.R, RP = (R + 1) >> 1;
  const int L = LT ? LT : a.L;
  const int npb = kAccThreads / RP;
  const int tn = threadIdx.x / RP;
  const long long li = static_cast<long long>(blockIdx.x) * npb + tn;  // index in the region
  const long long node = (a.row0 + li / a.w) * a.gx + a.x0 + li % a.w;
  const int r = 2 * (threadIdx.x % RP);
  const bool two = r + 1 < R;
  const bool live = tn < npb && li < a.cnt;
  const double inv = 1.0 / static_cast<double>(1 << dim);
  const double2* __restrict__ xs = a.x;
#pragma unroll
  for (int l = 0; l < LM; ++l) red[l][0][threadIdx.x] = red[l][1][threadIdx.x] = 0.0;
  if (live) {
    double2 u0 = czero(), u1 = czero();
    // A thread's loads are issued in three waves -- the plan entries of every sweep, their nonzero
    // words, then the x values of four sweeps at a time -- instead of a dependent entry -> nonzero
    // word -> x chain per sweep (24 memory round trips for 8 sweeps, now 4). Only a node's first
    // entry is on this path: interior nodes of a support have exactly one, the nodes of shared
    // faces (2 to 2^dim entries, compacted to the front of the node's E slots) take the loop below.
    int pos[LM];              // first entry's position in x
    unsigned long long meta = 0;  // per sweep one byte: weight numerator (4 bits), more-entries flag, RHS pair's nonzero bits
    {
      int4 e01[LM];  // entries 0 and 1 of the node for sweep l's direction: (pos, id << 4 | w) x 2
      rmask nzw[LM];
#pragma unroll
      for (int l = 0; l < LM; ++l)
        e01[l] = l < L ? __ldg(reinterpret_cast<const int4*>(a.acc_ent[l] + node * E)) : make_int4(-1, 0, -1, 0);
#pragma unroll
      for (int l = 0; l < LM; ++l) nzw[l] = e01[l].x >= 0 ? __ldg(a.nzmask[l] + (e01[l].y >> 4)) : 0ull;
#pragma unroll
      for (int l = 0; l < LM; ++l) {
        pos[l] = e01[l].x;
        const unsigned on = static_cast<unsigned>((nzw[l] >> r) & (two ? 3ull : 1ull));
        const unsigned byte = (e01[l].y & 15u) | (e01[l].z >= 0 ? 16u : 0u) | (on << 5);
        meta |= static_cast<unsigned long long>(byte) << (8 * l);
      }
    }
#ifndef HS_ACC_G
#define HS_ACC_G 4
#endif
    constexpr int G = HS_ACC_G;  // sweeps whose x values are in flight together
#pragma unroll
    for (int l0 = 0; l0 < LM; l0 += G) {
      if (!LT && l0 >= L) break;
      double2 x0[G], x1[G];
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const int l = l0 + k < LM ? l0 + k : 0;
        const unsigned on = l0 + k < LM ? static_cast<unsigned>(meta >> (8 * l + 5)) & 3u : 0u;
        const double2* px = xs + a.xoff[l] + static_cast<long long>(pos[l]) * R + r;
        x0[k] = (on & 1u) ? __ldcs(px) : czero();
        x1[k] = (on & 2u) ? __ldcs(px + 1) : czero();
      }
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const int l = l0 + k;
        if (l >= LM || (!LT && l >= L)) break;
        const unsigned mb = static_cast<unsigned>(meta >> (8 * l)) & 255u;
        const double w = (mb & 15u) * inv;
        double2 c0 = czero(), c1 = czero();
        if (mb & 32u) {
          c0.x += w * x0[k].x;
          c0.y += w * x0[k].y;
        }
        if (mb & 64u) {
          c1.x += w * x1[k].x;
          c1.y += w * x1[k].y;
        }
        if (mb & 16u) {  // a shared face: the node's other entries, in plan order
          const int2* __restrict__ pe = a.acc_ent[l] + node * E;
#pragma unroll 1
          for (int i = 1; i < E; ++i) {
            const int2 en = __ldg(pe + i);
            if (en.x < 0) break;
            const unsigned o = static_cast<unsigned>((__ldg(a.nzmask[l] + (en.y >> 4)) >> r) & (two ? 3ull : 1ull));
            const double2* px = xs + a.xoff[l] + static_cast<long long>(en.x) * R + r;
            const double wi = (en.y & 15) * inv;
            if (o & 1u) {
              const double2 xv = __ldcs(px);
              c0.x += wi * xv.x;
              c0.y += wi * xv.y;
            }
            if (o & 2u) {
              const double2 xv = __ldcs(px + 1);
              c1.x += wi * xv.x;
              c1.y += wi * xv.y;
            }
          }
        }
        u0 = cadd(u0, c0);
        u1 = cadd(u1, c1);
        red[l][0][threadIdx.x] = c0.x * c0.x + c0.y * c0.y;
        red[l][1][threadIdx.x] = c1.x * c1.x + c1.y * c1.y;
        if (a.uround && (l + 1) % a.rlen == 0 && l + 1 < L) {  // u after this round
          double2* ur = a.uround + static_cast<long long>((l + 1) / a.rlen - 1) * a.rstride + node * R + r;
          ur[0] = u0;
          if (two) ur[1] = u1;
        }
      }
    }
    __stcs(a.u + node * R + r, u0);
    if (two) __stcs(a.u + node * R + r + 1, u1);
  }
  __syncthreads();
  // partial of sweep l, column c: the block's nodes in order (fixed order)
  for (int q = threadIdx.x; q < L * R; q += kAccThreads) {
    const int l = q / R, c = q % R;
    double sm = 0.0;
    for (int t = 0; t < npb; ++t) sm += red[l][c & 1][t * RP + (c >> 1)];
    a.partial[l * a.pstride + static_cast<long long>(blockIdx.x) * R + c] = sm;
  }
}

int launch_accumulate_all(const AccumAllArgs& a, cudaStream_t s) {
  const int nb = blocks_for(a.cnt, kAccThreads / ((a.R + 1) / 2));
  if (nb == 0) return 0;
  if (a.g.dim == 3)
    accumulate_all_kernel<8, 0><<<nb, kAccThreads, 0, s>>>(a);
  else if (a.L == 8)
    accumulate_all_kernel<4, 8><<<nb, kAccThreads, 0, s>>>(a);
  else if (a.L == 4)
    accumulate_all_kernel<4, 4><<<nb, kAccThreads, 0, s>>>(a);
  else
    accumulate_all_kernel<4, 0><<<nb, kAccThreads, 0, s>>>(a);
  after_launch();
  return nb;
}

int launch_accumulate(const AccumArgs& a, cudaStream_t s) {
  const int nb = blocks_for(a.n1 - a.n0, kThreads / a.R);
  if (nb == 0) return 0;
  if (a.g.dim == 3)
    accumulate_kernel<8><<<nb, kThreads, 0, s>>>(a);
  else
    accumulate_kernel<4><<<nb, kThreads, 0, s>>>(a);
  after_launch();
  return nb;
}

// The stage-1 scratch lives right after the used partials: the caller's buffer holds at least
// (nblocks + kReducePad) * R doubles.
void launch_reduce_partials(double* partial, int nblocks, int R, double* out, cudaStream_t s) {
  double* mid = partial + static_cast<long long>(nblocks) * R;
  const int g = std::max(1, std::min(kReduceBlocks, nblocks));
  reduce_partials_stage1<<<g, kThreads, 0, s>>>(partial, nblocks, R, mid);
  after_launch();
  reduce_partials_stage2<<<R, 32, 0, s>>>(mid, g, R, out);
  after_launch();
}

void launch_reduce_cpartials(const double2* partial, int nblocks, int R, double2* out, cudaStream_t s) {
  reduce_cpartials_kernel<<<R, kThreads, 0, s>>>(partial, nblocks, R, out);
  after_launch();
}

void launch_stencil_build(long long n, const std::int64_t* row_ptr, const int* col, const double2* val, StencilOp op,
                          double2* out, unsigned* bad, cudaStream_t s) {
  stencil_build_kernel<<<blocks_for(n), kThreads, 0, s>>>(n, row_ptr, col, val, op, out, bad);
  after_launch();
}

int launch_residual(long long n, const std::int64_t* row_ptr, const int* col, const double2* val, const double2* x,
                    const double2* b, int R, double* pnum, double* pden, cudaStream_t s, int gx, StencilOp sop) {
  const int npb = kResThreads / R;
  int nb, tiles_x = 0;
  if (gx > 0 && n % gx == 0) {  // grid operator: tiles of npb nodes x kResRows grid rows
    tiles_x = (gx + npb - 1) / npb;
    nb = tiles_x * static_cast<int>((n / gx + kResRows - 1) / kResRows);
  } else {
    gx = 0;
    nb = blocks_for(n, npb);
  }
  if (gx > 0 && sop.val && (sop.S == 5 || sop.S == 7)) {
    if (sop.S == 5)
      residual_stencil_kernel<5><<<nb, kResThreads, 0, s>>>(n, sop, x, b, R, pnum, pden, gx, tiles_x);
    else
      residual_stencil_kernel<7><<<nb, kResThreads, 0, s>>>(n, sop, x, b, R, pnum, pden, gx, tiles_x);
  } else {
    residual_kernel<<<nb, kResThreads, 0, s>>>(n, row_ptr, col, val, x, b, R, pnum, pden, gx, tiles_x);
  }
  after_launch();
  return nb;
}

void launch_spmv(long long n, const std::int64_t* row_ptr, const int* col, const double2* val, const double2* x,
                 double2* y, int R, cudaStream_t s) {
  spmv_kernel<<<blocks_for(n * R), kThreads, 0, s>>>(n, row_ptr, col, val, x, y, R);
  after_launch();
}

int launch_dot_partials(const double2* a, const double2* b, long long n, int R, double2* partial, cudaStream_t s) {
  const int nb = blocks_for(n, kThreads / R);
  dot_partials_kernel<<<nb, kThreads, 0, s>>>(a, b, n, R, partial);
  after_launch();
  return nb;
}

void launch_axpy_cols(double2* y, const double2* x, const double2* alpha, int neg, long long n, int R,
                      cudaStream_t s) {
  axpy_cols_kernel<<<blocks_for(n * R), kThreads, 0, s>>>(y, x, alpha, neg, n, R);
  after_launch();
}

void launch_scale_cols(double2* y, const double* inv, long long n, int R, cudaStream_t s) {
  scale_cols_kernel<<<blocks_for(n * R), kThreads, 0, s>>>(y, inv, n, R);
  after_launch();
}

void launch_transpose_in(const double2* src, double2* dst, long long n, int R, cudaStream_t s, const int* perm) {
  transpose_in_kernel<<<static_cast<int>((n + kTransNodes - 1) / kTransNodes), kThreads, 0, s>>>(src, dst, n, R, 0, n, perm);
  after_launch();
}

void launch_transpose_out(const double2* src, double2* dst, long long n, int R, cudaStream_t s, const int* perm) {
  transpose_out_kernel<<<static_cast<int>((n + kTransNodes - 1) / kTransNodes), kThreads, 0, s>>>(src, dst, n, R, 0, n, perm);
  after_launch();
}

void launch_transpose_in_range(const double2* src, double2* dst, long long n, int R, long long n0, long long n1,
                               cudaStream_t s) {
  if (n1 <= n0) return;
  transpose_in_kernel<<<static_cast<int>((n1 - n0 + kTransNodes - 1) / kTransNodes), kThreads, 0, s>>>(src, dst, n, R,
                                                                                                     n0, n1, nullptr);
  after_launch();
}
void launch_transpose_in_tile(const double2* src, double2* dst, long long n, int R, int gx, int x0, int x1,
                              long long row0, long long row1, cudaStream_t s, const int* perm) {
  if (x1 <= x0 || row1 <= row0) return;
  const dim3 grid((x1 - x0 + kTransNodes - 1) / kTransNodes, static_cast<unsigned>(row1 - row0));
  transpose_in_tile_kernel<<<grid, kThreads, 0, s>>>(src, dst, n, R, gx, x0, x1, row0, perm);
  after_launch();
}
void launch_transpose_out_tile(const double2* src, double2* dst, long long n, int R, int gx, int x0, int x1,
                               long long row0, long long row1, cudaStream_t s, const int* perm) {
  if (x1 <= x0 || row1 <= row0) return;
  const dim3 grid((x1 - x0 + kTransNodes - 1) / kTransNodes, static_cast<unsigned>(row1 - row0));
  transpose_out_tile_kernel<<<grid, kThreads, 0, s>>>(src, dst, n, R, gx, x0, x1, row0, perm);
  after_launch();
}
void launch_transpose_out_range(const double2* src, double2* dst, long long n, int R, long long n0, long long n1,
                                cudaStream_t s) {
  if (n1 <= n0) return;
  transpose_out_kernel<<<static_cast<int>((n1 - n0 + kTransNodes - 1) / kTransNodes), kThreads, 0, s>>>(src, dst, n, R,
                                                                                                      n0, n1, nullptr);
  after_launch();
}

// ---- RHS ordering -------------------------------------------------------------------------------
// A batch's columns are independent, so the library may hold them in any order. Tasks skip RHS
// groups that are exactly zero for them (hs_solve.cu), which pays when the columns of a group
// have their sources close together: the columns are ordered along a Morton curve over the
// subdomain cells that hold the centres of their nonzeros' bounding boxes.
// bbox[r] = {min x, min y, min z, max x, max y, max z} over the sampled grid rows (row % rstep == 0).
__global__ void rhs_bbox_kernel(const double2* b, long long n, int gx, int gy, int rstep, long long srows, int* bbox) {
  const int r = blockIdx.y;
  int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {-1, -1, -1};
  const double2* br = b + static_cast<long long>(r) * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < srows * gx;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long row = (e / gx) * rstep;
    const int x = static_cast<int>(e % gx);
    const double2 v = br[row * gx + x];
    if (v.x != 0.0 || v.y != 0.0) {
      const int c[3] = {x, static_cast<int>(row % gy), static_cast<int>(row / gy)};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        lo[a] = min(lo[a], c[a]);
        hi[a] = max(hi[a], c[a]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = __reduce_min_sync(kFull, lo[a]);
    hi[a] = __reduce_max_sync(kFull, hi[a]);
  }
  if ((threadIdx.x & 31) == 0 && hi[0] >= 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(bbox + 6 * r + a, lo[a]);
      atomicMax(bbox + 6 * r + 3 + a, hi[a]);
    }
  }
}

__global__ void rhs_bbox_init_kernel(int R, int* bbox) {
  if (static_cast<int>(threadIdx.x) < 6 * R) bbox[threadIdx.x] = threadIdx.x % 6 < 3 ? INT_MAX : -1;
}

__host__ __device__ inline unsigned rhs_morton_key(const DevGeom& g, const int* bb) {
  if (bb[3] < 0) return 0xFFFFFFFFu;  // no nonzero seen: last
  unsigned cell[3] = {0, 0, 0};
  for (int a = 0; a < g.dim; ++a) {
    const int c = ((bb[a] + bb[3 + a]) / 2 + g.glo[a]) / g.cut_w[a];
    cell[a] = static_cast<unsigned>(c < 0 ? 0 : c >= g.counts[a] ? g.counts[a] - 1 : c);
  }
  unsigned key = 0;
  for (int bit = 9; bit >= 0; --bit)
    for (int a = g.dim - 1; a >= 0; --a) key = (key << 1) | ((cell[a] >> bit) & 1u);
  return key;
}

// perm[j] = the caller's column held at internal position j: ascending key, ties by column
__global__ void rhs_order_kernel(DevGeom g, int R, const int* bbox, int* perm) {
  __shared__ unsigned key[kMaxRhs];
  const int r = threadIdx.x;
  if (r < R) key[r] = rhs_morton_key(g, bbox + 6 * r);
  __syncthreads();
  if (r >= R) return;
  int rank = 0;
  for (int q = 0; q < R; ++q) rank += key[q] < key[r] || (key[q] == key[r] && q < r);
  perm[rank] = r;
}

void launch_rhs_order(const double2* b, long long n, int R, const DevGeom& g, int* bbox, int* perm, cudaStream_t s) {
  rhs_bbox_init_kernel<<<1, 6 * kMaxRhs, 0, s>>>(R, bbox);
  after_launch();
  const int gx = g.gsize[0], gy = g.dim > 1 ? g.gsize[1] : 1;
  const long long rows = n / gx;
  const int rstep = 4;  // every fourth grid row: a quarter of b's bytes
  const long long srows = (rows + rstep - 1) / rstep;
  const int bx = std::max(1, std::min(blocks_for(srows * gx), 1184));
  rhs_bbox_kernel<<<dim3(bx, R), kThreads, 0, s>>>(b, n, gx, gy, rstep, srows, bbox);
  after_launch();
  rhs_order_kernel<<<1, kMaxRhs, 0, s>>>(g, R, bbox, perm);
  after_launch();
}

unsigned rhs_order_key(const DevGeom& g, const int* bbox6) { return rhs_morton_key(g, bbox6); }


void launch_bump_epoch(unsigned* e, unsigned by, cudaStream_t s) {
  bump_epoch_kernel<<<1, 1, 0, s>>>(e, by);
  after_launch();
}

}  // namespace hsb
