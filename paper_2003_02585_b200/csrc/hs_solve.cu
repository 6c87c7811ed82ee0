// Multifrontal forward / backward solves of the helmsweep hot path on sm_100a
// (Factorization::solve_inplace, /root/reference/proj/src/direct.cpp:290-325), batched over
// every subdomain of a sweep step group and the RHS of the batch.
//
// Partitioned inverse: the factorization stores, per front, M = L11^-1 (unit lower) and
// W = L21 M instead of L11 / L21 (hs_kernels.cu). The reference's per-front operations
//   forward   t = L11^-1 x[sep]; x[bnd] -= L21 t          (direct.cpp:296-307)
//   backward  x[sep] = L11^-T (x[sep] - L21^T x[bnd])     (direct.cpp:311-324)
// become dense products without any serial dependency inside a front:
//   forward   [z_sep; u] = [M; W] x_sep,  z = D^-1 z_sep (direct.cpp:309),  V = bnd updates - u
//   backward  x_sep = [M; W]^T [z_sep; -x_bnd]
// Work items (one warp each, no CTA barriers):
//   kind 0  forward gather of 32 front positions: T = [rhs_sep; 0] + child0 V + child1 V
//           (the extend-add, in the reference's child order, src/direct.cpp:239-265);
//   kind 1  forward 32-row block of [M; W] x T_sep for rw RHS (lane = row);
//   kind 2  backward 32-column panel of [M; W]^T y for rw RHS (lane = column).
// Fronts with k >= big_k use 4-RHS items (4x more warps on the long upper-tree critical
// path), the others 16-RHS items (each factor byte read once for 16 RHS). Items are listed in
// topological order and dequeued greedily; dependencies are per-front completion counters
// (relaxed spin, one acquire, release increments). A warp dequeues only while running and
// every dependency sits earlier in the list, so the launch cannot deadlock; every reduction
// has a fixed order, so results are bitwise reproducible.
//
// Factor streams: copy F (forward, column-major 32-row chunks) and copy B (backward, row-major
// 32-column panels), coalesced 512-byte warp loads that bypass L1 (ld.global.nc.L1::no_allocate).
// Vector operands are staged 32 rows at a time into a per-warp shared tile with cp.async.cg
// (L2, coherent with the producers' release); 4-RHS items double-buffer the tile.
#include <algorithm>
#include <atomic>
#include <cstdint>

#include "hs_common.hpp"
#include "hs_kernels.cuh"

namespace hsb {

extern std::atomic<long long> g_kernel_launches;

namespace {

constexpr int kThreads = 256;
constexpr int kTile = 32 * 16;  // double2 per warp tile (8 KB)

__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_count(const int* p, int target, int lane) {
  if (lane == 0) {
    while (ld_relaxed(p) < target) __nanosleep(32);
    (void)ld_acquire(p);
  }
  __syncwarp();
}
__device__ __forceinline__ void signal(int* p, int lane) {
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    red_release_add(p, 1);
  }
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ int nrb_of(const DevFront& f) { return (f.m + 31) >> 5; }
__device__ __forceinline__ int np_of(const DevFront& f) { return (f.k + 31) >> 5; }
__device__ __forceinline__ int rw_of(const DevFront& f, int R, int big_k) { return f.k >= big_k ? min(4, R) : min(16, R); }
__device__ __forceinline__ int ngroups(const DevFront& f, int R, int big_k) {
  const int w = rw_of(f, R, big_k);
  return (R + w - 1) / w;
}
// element offset of row block rb in copy F (all earlier row blocks are full)
__device__ __forceinline__ long long rb_base(int rb, int np) {
  const long long pre = rb <= np ? static_cast<long long>(rb) * (rb + 1) / 2
                                 : static_cast<long long>(np) * (np + 1) / 2 + static_cast<long long>(rb - np) * np;
  return pre * 1024;
}
__device__ __forceinline__ long long copy_elems(int m, int k) {
  const int np = (k + 31) >> 5;
  return 32LL * (static_cast<long long>(np) * m - 16LL * np * (np - 1));
}

// kind 0: T[p] = (p < k ? rhs[sep + p] : 0) + child0 V + child1 V for 32 positions, all RHS.
__device__ void fwd_gather(const SolveArgs& a, const DevClass& C, const DevSub& S, const DevFront& fr, int pb, double2* T,
                           const double2* V, int lane) {
  const int R = a.R, p = 32 * pb + lane;
  if (p >= fr.m) return;
  const int2 pm = C.pmap[fr.t_off + p];
  const double2* g0 = p < fr.k ? S.x + static_cast<long long>(fr.sep_off + p) * R : nullptr;
  const double2* g1 = pm.x >= 0 ? V + (C.fronts[fr.child0].v_off + pm.x) * R : nullptr;
  const double2* g2 = pm.y >= 0 ? V + (C.fronts[fr.child1].v_off + pm.y) * R : nullptr;
  double2* t = T + static_cast<long long>(p) * R;
#pragma unroll 4
  for (int r = 0; r < R; ++r) {
    double2 v = g0 ? __ldcg(g0 + r) : czero();
    if (g1) {
      const double2 w = __ldcg(g1 + r);
      v = make_double2(v.x + w.x, v.y + w.y);
    }
    if (g2) {
      const double2 w = __ldcg(g2 + r);
      v = make_double2(v.x + w.x, v.y + w.y);
    }
    __stcg(t + r, v);
  }
}

// Stage rows [0, nrows) (row l at src(l) .. + RW) into tile[32][RW]; rows >= nrows zero.
template <int RW, class Src>
__device__ __forceinline__ void stage(double2* tile, int nrows, int nr, int lane, Src&& src) {
  double2* dst = tile + lane * RW;
  if (lane < nrows) {
    const double2* g = src(lane);
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      if (r < nr)
        cp_async16(dst + r, g + r);
      else
        dst[r] = czero();
    }
  } else {
#pragma unroll
    for (int r = 0; r < RW; ++r) dst[r] = czero();
  }
  cp_commit();
}

// kind 1: out[row] = sum_j [M; W][row, j] T_sep[j] for RHS [r0, r0 + RW)
template <int RW>
__device__ void fwd_block(const SolveArgs& a, const DevSub& S, const DevFront& fr, int rb, const double2* T, double2* V,
                          int r0, int nr, int lane, double2* tiles) {
  constexpr int NB = kTile / (32 * RW) >= 2 ? 2 : 1;  // double buffer when the tile allows
  const int R = a.R, m = fr.m, k = fr.k, np = np_of(fr);
  const int rc = min(32, m - 32 * rb), nj = min(rb, np - 1) + 1;
  const double2* P = S.factor + fr.fac_off + rb_base(rb, np);
  double2 acc[RW];
#pragma unroll
  for (int r = 0; r < RW; ++r) acc[r] = czero();
  const bool active = lane < rc;
  auto src_of = [&](int J) {
    return [=](int l) { return T + static_cast<long long>(32 * J + l) * R + r0; };
  };
  stage<RW>(tiles, min(32, k), nr, lane, src_of(0));
  for (int J = 0; J < nj; ++J) {
    double2* tile = tiles + (J % NB) * 32 * RW;
    if (NB == 2 && J + 1 < nj) {
      stage<RW>(tiles + ((J + 1) % NB) * 32 * RW, min(32, k - 32 * (J + 1)), nr, lane, src_of(J + 1));
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncwarp();
    const double2* ch = P + static_cast<long long>(J) * rc * 32;
    const int jmax = min(32, k - 32 * J);
    int j = 0;
    for (; j + 8 <= jmax; j += 8) {
      double2 L[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) L[u] = active ? ld_stream(ch + (j + u) * rc + lane) : czero();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double2* xr = tile + (j + u) * RW;
#pragma unroll
        for (int r = 0; r < RW; ++r) cfma(acc[r], L[u], xr[r]);
      }
    }
    for (; j < jmax; ++j) {
      const double2 L = active ? ld_stream(ch + j * rc + lane) : czero();
      const double2* xr = tile + j * RW;
#pragma unroll
      for (int r = 0; r < RW; ++r) cfma(acc[r], L, xr[r]);
    }
    __syncwarp();
    if (NB == 1 && J + 1 < nj) stage<RW>(tiles, min(32, k - 32 * (J + 1)), nr, lane, src_of(J + 1));
  }
  if (!active) return;
  const int row = 32 * rb + lane;
  if (row < k) {  // z_sep = D^-1 M x_sep
    const long long pos = fr.sep_off + row;
    const double2 d = S.dinv[pos];
#pragma unroll
    for (int r = 0; r < RW; ++r)
      if (r < nr) __stcg(&S.x1[pos * R + r0 + r], cmul(acc[r], d));
  } else {        // V = (children's bnd updates) - W x_sep
    const double2* t = T + static_cast<long long>(row) * R + r0;
#pragma unroll
    for (int r = 0; r < RW; ++r)
      if (r < nr) {
        const double2 w = __ldcg(t + r);
        __stcg(&V[(fr.v_off + row - k) * R + r0 + r], make_double2(w.x - acc[r].x, w.y - acc[r].y));
      }
  }
}

// kind 2: x_sep[col] = sum_i [M; W][i, col] [z_sep; -x_bnd][i] for RHS [r0, r0 + RW)
template <int RW>
__device__ void bwd_panel(const SolveArgs& a, const DevClass& C, const DevSub& S, const DevFront& fr, int J, int r0,
                          int nr, int lane, double2* tiles) {
  constexpr int NB = kTile / (32 * RW) >= 2 ? 2 : 1;
  const int R = a.R, m = fr.m, k = fr.k;
  const double2* P = S.factor + fr.fac_off + copy_elems(m, k) + 32LL * (static_cast<long long>(J) * m - 16LL * J * (J - 1));
  double2 acc[RW];
#pragma unroll
  for (int r = 0; r < RW; ++r) acc[r] = czero();
  auto src_of = [&](int i0) {
    return [=](int l) {
      const int ii = i0 + l;
      const long long pos = ii < k ? static_cast<long long>(fr.sep_off + ii)
                                   : static_cast<long long>(C.bnd_elim[fr.bnd_off + ii - k]);
      return (ii < k ? S.x1 : S.x) + pos * R + r0;
    };
  };
  const int nbt = (m - 32 * J + 31) / 32;
  stage<RW>(tiles, min(32, m - 32 * J), nr, lane, src_of(32 * J));
  for (int b = 0; b < nbt; ++b) {
    const int i0 = 32 * J + 32 * b;
    const int nrow = min(32, m - i0);
    double2* tile = tiles + (b % NB) * 32 * RW;
    if (NB == 2 && b + 1 < nbt) {
      stage<RW>(tiles + ((b + 1) % NB) * 32 * RW, min(32, m - i0 - 32), nr, lane, src_of(i0 + 32));
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    if (i0 + lane >= k && lane < nrow) {  // bnd rows enter as -x_bnd
#pragma unroll
      for (int r = 0; r < RW; ++r) tile[lane * RW + r] = make_double2(-tile[lane * RW + r].x, -tile[lane * RW + r].y);
    }
    __syncwarp();
    const double2* Pb = P + static_cast<long long>(i0 - 32 * J) * 32;
    int u0 = 0;
    for (; u0 + 8 <= nrow; u0 += 8) {
      double2 L[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) L[u] = ld_stream(Pb + (u0 + u) * 32 + lane);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double2* y = tile + (u0 + u) * RW;
#pragma unroll
        for (int r = 0; r < RW; ++r) cfma(acc[r], L[u], y[r]);
      }
    }
    for (; u0 < nrow; ++u0) {
      const double2 L = ld_stream(Pb + u0 * 32 + lane);
      const double2* y = tile + u0 * RW;
#pragma unroll
      for (int r = 0; r < RW; ++r) cfma(acc[r], L, y[r]);
    }
    __syncwarp();
    if (NB == 1 && b + 1 < nbt) stage<RW>(tiles, min(32, m - i0 - 32), nr, lane, src_of(i0 + 32));
  }
  const int col = 32 * J + lane;
  if (col < k) {
#pragma unroll
    for (int r = 0; r < RW; ++r)
      if (r < nr) __stcg(&S.x[static_cast<long long>(fr.sep_off + col) * R + r0 + r], acc[r]);
  }
}

template <bool FWD>
__global__ void __launch_bounds__(kThreads, 2) solve5_kernel(SolveArgs a) {
  extern __shared__ __align__(16) double2 smem_tiles[];
  const int lane = threadIdx.x & 31;
  double2* tiles = smem_tiles + (threadIdx.x >> 5) * kTile;
  const int R = a.R;
  for (;;) {
    int it = 0;
    if (lane == 0) it = static_cast<int>(atomicAdd(a.queue, 1u));
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= a.nitems) break;
    const SolveItem item = a.items[it];
    if (a.nzmask[item.sub] == 0) continue;  // skipped subdomain: nothing depends on it
    unsigned long long* tr = a.trace ? a.trace + 4LL * it : nullptr;
    if (tr && lane == 0) tr[0] = gtime();
    const DevSub& S = a.subs[item.sub];
    const DevClass& C = a.cls[S.cls];
    const DevFront fr = C.fronts[item.front];
    const long long cbase = static_cast<long long>(item.slot) * a.nf_max;
    int* cnt0 = a.cnt + cbase;                 // forward gathers / backward panels
    int* cnt1 = a.cnt + a.cnt_stride + cbase;  // forward row blocks
    double2* V = a.vbuf + item.slot * a.vslot_stride;
    double2* T = a.tbuf + item.slot * a.tslot_stride + fr.t_off * R;
    const int nr = min(item.rw, R - item.r0);
    if (FWD) {
      if (item.kind == 0) {  // children complete = all their row-block items
#pragma unroll 1
        for (int q = 0; q < 2; ++q) {
          const int ch = q ? fr.child1 : fr.child0;
          if (ch < 0) continue;
          const DevFront cf = C.fronts[ch];
          wait_count(cnt1 + ch, nrb_of(cf) * ngroups(cf, R, a.big_k), lane);
        }
        if (tr && lane == 0) tr[1] = gtime();
        fwd_gather(a, C, S, fr, item.idx, T, V, lane);
        signal(cnt0 + item.front, lane);
      } else {
        wait_count(cnt0 + item.front, nrb_of(fr), lane);
        if (tr && lane == 0) tr[1] = gtime();
        if (item.rw <= 4)
          fwd_block<4>(a, S, fr, item.idx, T, V, item.r0, nr, lane, tiles);
        else
          fwd_block<16>(a, S, fr, item.idx, T, V, item.r0, nr, lane, tiles);
        signal(cnt1 + item.front, lane);
      }
    } else {
      if (fr.parent >= 0) {
        const DevFront pf = C.fronts[fr.parent];
        wait_count(cnt0 + fr.parent, np_of(pf) * ngroups(pf, R, a.big_k), lane);
      }
      if (tr && lane == 0) tr[1] = gtime();
      if (item.rw <= 4)
        bwd_panel<4>(a, C, S, fr, item.idx, item.r0, nr, lane, tiles);
      else
        bwd_panel<16>(a, C, S, fr, item.idx, item.r0, nr, lane, tiles);
      signal(cnt0 + item.front, lane);
    }
    if (tr && lane == 0) {
      tr[2] = gtime();
      tr[3] = smid();
    }
  }
}

constexpr size_t kSmem = static_cast<size_t>(kThreads / 32) * kTile * sizeof(double2);
int g_grid[2] = {0, 0};

}  // namespace

int solve_rhs_width(int k, int R, int big_k) { return k >= big_k ? std::min(4, R) : std::min(16, R); }

void launch_solve(const SolveArgs& a, bool fwd, cudaStream_t s) {
  int& grid = g_grid[fwd ? 1 : 0];
  if (!grid) {
    int dev = 0, sms = 0, per = 0;
    HS_CUDA(cudaGetDevice(&dev));
    HS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    HS_CUDA(cudaFuncSetAttribute(solve5_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    HS_CUDA(cudaFuncSetAttribute(solve5_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    if (fwd)
      HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, solve5_kernel<true>, kThreads, kSmem));
    else
      HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, solve5_kernel<false>, kThreads, kSmem));
    grid = sms * std::max(per, 1);
  }
  const int g = std::max(1, std::min(grid, (a.nitems + kThreads / 32 - 1) / (kThreads / 32)));
  if (fwd)
    solve5_kernel<true><<<g, kThreads, kSmem, s>>>(a);
  else
    solve5_kernel<false><<<g, kThreads, kSmem, s>>>(a);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  HS_CUDA(cudaGetLastError());
}

}  // namespace hsb
