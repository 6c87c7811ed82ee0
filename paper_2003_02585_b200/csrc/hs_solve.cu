// Multifrontal forward / backward solves of the helmsweep hot path on sm_100a
// (Factorization::solve_inplace, /root/reference/proj/src/direct.cpp:290-325), batched over
// every subdomain of a sweep step group and the RHS of the batch.
//
// Partitioned inverse: the factorization stores, per front, M = L11^-1 (unit lower) and
// W = L21 M instead of L11 / L21 (hs_kernels.cu). The reference's per-front operations
//   forward   t = L11^-1 x[sep]; x[bnd] -= L21 t          (direct.cpp:296-307)
//   backward  x[sep] = L11^-T (x[sep] - L21^T x[bnd])     (direct.cpp:311-324)
// become one dense product per front without any serial dependency inside it:
//   forward   [z_sep; u] = [M; W] T_sep,  z = D^-1 z_sep (direct.cpp:309),  V = T_bnd - u
//   backward  x_sep = [M; W]^T [z_sep; -x_bnd]
// where T = rhs + the children's update vectors V (the extend-add, in the reference's child
// order, src/direct.cpp:239-265), gathered on the fly through the front's source map.
//
// Tensor cores: the products run on FP64 DMMA (mma.sync m8n8k4 f64) with complex
// arithmetic as four real products (re*re - im*im, re*im + im*re). The factor is stored once
// in 8x8 complex blocks (hs_symbolic.hpp front_block_elems): the forward reads them as A
// fragments (lane = row 8i + lane/4, column lane%4), the backward as transposed A fragments
// of [M; W]^T (lane = row lane%4, column lane/4); both loads use whole 32-byte sectors. B
// fragments (4 rows x 8 RHS) come straight from L2 (rhs / update vectors / z / x).
//
// Work items (one warp each, no shared memory):
//   kind 1  forward band t (32 padded rows) x column-block chunk c x 16-RHS group;
//   kind 2  backward column band u (32 separator columns) x block-row chunk c x RHS group.
// Bands longer than one chunk are split-K: each chunk stores its partial tile and the last
// arriving chunk sums all partials in chunk order (bitwise reproducible) and finalizes. Items
// are listed in topological order and dequeued greedily; dependencies are per-front counters of
// finalized bands (relaxed spin, one acquire, release increments); a warp dequeues only while
// running and every dependency sits earlier in the list, so the launch cannot deadlock. The
// factor range of an item is bulk-prefetched into L2 before its dependency wait.
#include <algorithm>
#include <atomic>
#include <cstdint>

#include "hs_common.hpp"
#include "hs_kernels.cuh"

namespace hsb {

extern std::atomic<long long> g_kernel_launches;

namespace {

constexpr int kThreads = 128;

__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
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
#ifndef HS_POLL_ACQUIRE
#define HS_POLL_ACQUIRE 0
#endif
#ifndef HS_SPIN_MAX_NS
#define HS_SPIN_MAX_NS 256
#endif
__device__ __forceinline__ void wait_count(const int* p, int target, int lane) {
  if (lane == 0) {
    unsigned ns = 32;  // short backoff: waiters on the critical path must react quickly
#if HS_POLL_ACQUIRE
    // every poll is an acquire load: the one that sees the target already orders the reads that
    // follow, saving the extra L2 round trip of a relaxed poll plus a separate acquire
    while (ld_acquire(p) < target) {
      __nanosleep(ns);
      ns = min(ns * 2, static_cast<unsigned>(HS_SPIN_MAX_NS));
    }
#else
    while (ld_relaxed(p) < target) {
      __nanosleep(ns);
      ns = min(ns * 2, static_cast<unsigned>(HS_SPIN_MAX_NS));
    }
    (void)ld_acquire(p);
#endif
  }
  __syncwarp();
}
// Release: the warp's stores are ordered before lane 0's release by the warp barrier (the
// CUTLASS-semaphore pattern); no full fence.
__device__ __forceinline__ void signal(int* p, int lane, int count = 1) {
  __syncwarp();
  if (lane == 0) red_release_add(p, count);
}
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
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
// D[8x8] += A[8x4] B[4x8], FP64 tensor core
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Solve-layout geometry of a front (hs_symbolic.hpp)
struct Geo {
  int kp, kb, nrb, nband, ncband;
};
__device__ __forceinline__ long long band_base(int t, int kb) {
  const int j0 = kb >> 2;
  const long long s = t <= j0 ? 2LL * t * (t + 1) : 2LL * j0 * (j0 + 1) + static_cast<long long>(t - j0) * kb;
  return s * 256;
}
__device__ __forceinline__ int nch_fwd(const Geo& g, int t, int kc) { return (min(g.kb, 4 * t + 4) + kc - 1) / kc; }
__device__ __forceinline__ int nch_bwd(const Geo& g, int u, int kr) { return (g.nrb - 4 * u + kr - 1) / kr; }

constexpr unsigned kAllLive = 0x100u;  // task face mask bit: every front is live

// Complex products as three real products (HS_3M): with P1 = Ar Br, P2 = Ai Bi and
// P3 = (Ar + Ai)(Br + Bi), Re = P1 - P2 and Im = P3 - P1 - P2, so a complex k-step costs 3 DMMAs
// per tile instead of 4 (the FP64 tensor pipe is the bound when many items run at once). The
// k-loop accumulates P1, P2, P3 in planes 0, 1, 2; acc_finish turns them into re / im (planes
// 0, 1), which is all the split-K reduction and the finalize see.
// Both forms are compiled (template M3): 3M needs 162-168 registers and so runs 3 CTAs per SM,
// the four-product form 4 (SolveArgs::m3 selects; 3M measured faster on C2 and C5).
template <int NT, bool M3>
struct Acc {
  static constexpr int P = M3 ? 3 : 2;
  double v[4][NT][P][2];  // m-tile i, n-tile q, re/im (3M: P1 / P2 / P3), fragment element e
};
constexpr int kTileDoubles = 1024;  // partial tile: 32 lanes x up to 32 accumulator doubles

template <int NT, bool M3>
__device__ __forceinline__ void acc_zero(Acc<NT, M3>& c) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < NT; ++q)
#pragma unroll
      for (int p = 0; p < Acc<NT, M3>::P; ++p) c.v[i][q][p][0] = c.v[i][q][p][1] = 0.0;
}
// start value x + iy of one accumulator element (before the k-loop)
template <int NT, bool M3>
__device__ __forceinline__ void acc_set(Acc<NT, M3>& c, int i, int q, int e, double x, double y) {
  c.v[i][q][0][e] = x;
  if (M3) {  // Re = P1 - P2 = x, Im = P3 - P1 - P2 = y
    c.v[i][q][1][e] = 0.0;
    c.v[i][q][Acc<NT, M3>::P - 1][e] = x + y;
  } else {
    c.v[i][q][1][e] = y;
  }
}
// after the k-loop: planes 0 / 1 = re / im
template <int NT, bool M3>
__device__ __forceinline__ void acc_finish(Acc<NT, M3>& c) {
  if constexpr (M3) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < NT; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double p1 = c.v[i][q][0][e], p2 = c.v[i][q][1][e], p3 = c.v[i][q][Acc<NT, M3>::P - 1][e];
          c.v[i][q][0][e] = p1 - p2;
          c.v[i][q][1][e] = p3 - p1 - p2;
        }
  }
}

// one k-step (4 columns of the product's inner dimension) of the complex 32 x (8 NT) tile
// Only m-tiles in `mask` (warp-uniform) are computed: the others are structural zeros (rows past
// the front, columns past k, the upper triangle of M in the diagonal band).
// NEG: the k-step's B enters negated (the backward pass's -x_bnd rows); the signs fold into the
// DMMA operand modifiers instead of costing FP64-pipe negations.
// FULL: every m-tile live (the common case) -- no per-tile predicate, so the warp-synchronous
// DMMAs issue back to back instead of each behind a WARPSYNC / NOP pair.
template <bool NEG, bool FULL, int NT, bool M3>
__device__ __forceinline__ void mma_step(Acc<NT, M3>& c, const double2 (&A)[4], const double2 (&B)[NT], unsigned mask) {
  if (FULL) mask = 0xFu;
  if constexpr (M3) {
  double bx[NT], by[NT], bs[NT], as[4];
#pragma unroll
  for (int q = 0; q < NT; ++q) {
    bx[q] = NEG ? -B[q].x : B[q].x;
    by[q] = NEG ? -B[q].y : B[q].y;
    bs[q] = bx[q] + by[q];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) as[i] = A[i].x + A[i].y;
#pragma unroll
  for (int q = 0; q < NT; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (mask & (1u << i)) {
        dmma(c.v[i][q][0][0], c.v[i][q][0][1], A[i].x, bx[q]);
        dmma(c.v[i][q][1][0], c.v[i][q][1][1], A[i].y, by[q]);
        dmma(c.v[i][q][Acc<NT, M3>::P - 1][0], c.v[i][q][Acc<NT, M3>::P - 1][1], as[i], bs[q]);
      }
  } else {
  double bx[NT], by[NT], nby[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) {
    bx[q] = NEG ? -B[q].x : B[q].x;
    by[q] = NEG ? -B[q].y : B[q].y;
    nby[q] = NEG ? B[q].y : -B[q].y;
  }
#pragma unroll
  for (int q = 0; q < NT; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (mask & (1u << i)) {
        dmma(c.v[i][q][0][0], c.v[i][q][0][1], A[i].x, bx[q]);
        dmma(c.v[i][q][1][0], c.v[i][q][1][1], A[i].x, by[q]);
      }
#pragma unroll
  for (int q = 0; q < NT; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (mask & (1u << i)) {
        dmma(c.v[i][q][0][0], c.v[i][q][0][1], A[i].y, nby[q]);
        dmma(c.v[i][q][1][0], c.v[i][q][1][1], A[i].y, bx[q]);
      }
  }
}

// One k-step over the m-tiles [LO, HI) only, unpredicated (a per-tile predicate puts a warp barrier
// and a NOP in front of every DMMA: ncu showed the masked k-steps -- 63% of the backward's on C3,
// the diagonal block rows of every chunk-0 item and the short last column bands -- dominated the
// loop's fixed-latency stalls).
template <bool NEG, int LO, int HI, int NT, bool M3>
__device__ __forceinline__ void mma_range(Acc<NT, M3>& c, const double2 (&A)[4], const double2 (&B)[NT]) {
  if constexpr (M3) {
    double bx[NT], by[NT], bs[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      bx[q] = NEG ? -B[q].x : B[q].x;
      by[q] = NEG ? -B[q].y : B[q].y;
      bs[q] = bx[q] + by[q];
    }
#pragma unroll
    for (int q = 0; q < NT; ++q)
#pragma unroll
      for (int i = LO; i < HI; ++i) {
        const double as = A[i].x + A[i].y;
        dmma(c.v[i][q][0][0], c.v[i][q][0][1], A[i].x, bx[q]);
        dmma(c.v[i][q][1][0], c.v[i][q][1][1], A[i].y, by[q]);
        dmma(c.v[i][q][Acc<NT, M3>::P - 1][0], c.v[i][q][Acc<NT, M3>::P - 1][1], as, bs[q]);
      }
  } else {
    double bx[NT], by[NT], nby[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      bx[q] = NEG ? -B[q].x : B[q].x;
      by[q] = NEG ? -B[q].y : B[q].y;
      nby[q] = NEG ? B[q].y : -B[q].y;
    }
#pragma unroll
    for (int q = 0; q < NT; ++q)
#pragma unroll
      for (int i = LO; i < HI; ++i) {
        dmma(c.v[i][q][0][0], c.v[i][q][0][1], A[i].x, bx[q]);
        dmma(c.v[i][q][1][0], c.v[i][q][1][1], A[i].x, by[q]);
        dmma(c.v[i][q][0][0], c.v[i][q][0][1], A[i].y, nby[q]);
        dmma(c.v[i][q][1][0], c.v[i][q][1][1], A[i].y, bx[q]);
      }
  }
}
// A tile mask of the lean k-loops is always a contiguous range of m-tiles (backward: a prefix,
// forward: a suffix); dispatch it to the unpredicated range step.
template <bool NEG, int NT, bool M3>
__device__ __forceinline__ void mma_masked(Acc<NT, M3>& c, const double2 (&A)[4], const double2 (&B)[NT], unsigned mk) {
  if (!mk) return;
  const int lo = __ffs(mk) - 1, hi = 32 - __clz(mk);
  switch (lo * 8 + hi) {
    case 0 * 8 + 1: mma_range<NEG, 0, 1>(c, A, B); break;
    case 0 * 8 + 2: mma_range<NEG, 0, 2>(c, A, B); break;
    case 0 * 8 + 3: mma_range<NEG, 0, 3>(c, A, B); break;
    case 0 * 8 + 4: mma_range<NEG, 0, 4>(c, A, B); break;
    case 1 * 8 + 2: mma_range<NEG, 1, 2>(c, A, B); break;
    case 1 * 8 + 3: mma_range<NEG, 1, 3>(c, A, B); break;
    case 1 * 8 + 4: mma_range<NEG, 1, 4>(c, A, B); break;
    case 2 * 8 + 3: mma_range<NEG, 2, 3>(c, A, B); break;
    case 2 * 8 + 4: mma_range<NEG, 2, 4>(c, A, B); break;
    case 3 * 8 + 4: mma_range<NEG, 3, 4>(c, A, B); break;
    default: mma_step<NEG, false>(c, A, B, mk); break;  // (never: masks are contiguous)
  }
}

// Split-K: store this chunk's partial, and if it arrived last, replace acc by the sum of all
// chunks in chunk order (read back from memory, own partial included). Returns whether this
// warp finalizes the band.
template <int NT, bool M3>
__device__ __forceinline__ bool split_reduce(Acc<NT, M3>& c, double* base, long long cstride, int nch, int chunk,
                                             int* arr, int lane) {
  double* mine = base + chunk * cstride + lane;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < NT; ++q)
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int e = 0; e < 2; ++e) __stcg(mine + ((((i * NT + q) * 2 + p) * 2 + e) << 5), c.v[i][q][p][e]);
  __syncwarp();
  int last = 0;
  if (lane == 0) last = atom_add_acq_rel(arr, 1) == nch - 1;
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return false;
  // chunk order, own partial read back like the others; CB chunks' loads in flight per round
  constexpr int CB = NT == 1 ? 2 : 1;
  acc_zero(c);
  for (int c0 = 0; c0 < nch; c0 += CB) {
    double t[CB][4][NT][2][2];
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const double* pc = base + (c0 + b) * cstride + lane;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < NT; ++q)
#pragma unroll
          for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              t[b][i][q][p][e] = c0 + b < nch ? __ldcg(pc + ((((i * NT + q) * 2 + p) * 2 + e) << 5)) : 0.0;
    }
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      if (c0 + b >= nch) break;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < NT; ++q)
#pragma unroll
          for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int e = 0; e < 2; ++e) c.v[i][q][p][e] += t[b][i][q][p][e];
    }
  }
  return true;
}


// 16-byte cp.async with zero fill: when !ok no byte is read (src-size 0), so src may be any
// address (the lean k-loops pass the computed one instead of selecting a fallback)
__device__ __forceinline__ void cp16z(double2* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
// CA: the copy allocates in L1 (factor tiles of a quad: the CTA's four warps stream the same band
// chunk for four RHS groups, so three of the four reads hit L1 instead of going to L2)
template <bool CA = false>
__device__ __forceinline__ void cp16a(double2* dst, const void* src) {
  if (CA)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
  else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp16(double2* dst, const double2* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_small(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src), "n"(BYTES)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Per-warp shared memory: a ring of NS k-steps (stage = A fragments, 4 x 32 double2, then B
// parts, NB x 2 x 32 double2: forward NB = 3 = rhs, child0 V, child1 V; backward NB = 1),
// followed by the item's index slice (kIdx entries: source-map pairs / boundary positions).
constexpr int kIdx = 128;  // >= 8 * max(kc, kr)
#ifndef HS_ST2
#define HS_ST2 256  // double2 per k-step stage of the block-granular loops (below)
#endif
#ifndef HS_NS_FWD
#define HS_NS_FWD 2
#endif
#ifndef HS_NS_FWD1
#define HS_NS_FWD1 3
#endif
#ifndef HS_NS_BWD
#define HS_NS_BWD 3
#endif
#ifndef HS_NS_BWD1
#define HS_NS_BWD1 4
#endif
// Forward items also stage, per band row, the extend-add source of boundary rows (int2) and
// 1/d of separator rows (double2), so their finalize issues no dependent loads.
#ifndef HS_KUNROLL
#define HS_KUNROLL 1
#endif
[[maybe_unused]] constexpr int kKUnroll = HS_KUNROLL;  // k-loop unroll (tuning experiments)
// When a warp takes its next ticket: 1 = after the current item's k-loop (its atomic overlaps the
// reduction / finalize, and the held ticket is blocked only for that short tail), 0 = at the
// start of the current item (the held ticket then waits behind the whole item: at the end of a
// pass, idle warps could not start critical-path items other warps held).
#ifndef HS_LATE_TICKET
#define HS_LATE_TICKET 1
#endif

// Ring depth by RHS width: a stage of an 8-RHS (NT = 1) item is smaller, so the critical-path
// items (8-RHS groups) get a deeper ring in the same shared memory; their lone warps are bound by
// the latency of each k-step's loads.
template <bool FWD, int NT>
struct Ring {
  static constexpr int NS = FWD ? (NT == 1 ? HS_NS_FWD1 : HS_NS_FWD) : (NT == 1 ? HS_NS_BWD1 : HS_NS_BWD);
  static constexpr int NB = FWD ? 3 : 1;
  static constexpr int kStage = (4 + NB * NT) * 32;  // double2: A fragments, then B parts (p, q) at 4 + p NT + q
};
template <bool FWD>
struct RingArea {
  static constexpr int a1 = Ring<FWD, 1>::NS * Ring<FWD, 1>::kStage, a2 = Ring<FWD, 2>::NS * Ring<FWD, 2>::kStage;
  static constexpr int kRing1 = a1 > a2 ? a1 : a2;
  static constexpr int kRing = kRing1 > 4 * HS_ST2 ? kRing1 : 4 * HS_ST2;  // the block-granular loops need two block stages
  static constexpr int kFin = FWD ? 32 / 2 + 32 : 0;
  static constexpr int kWarp = kRing + kIdx / 2 + kFin;
};

// The pipelined k-loop shared by both passes: issue(s, stage) stages k-step s with cp.async,
// use(s, stage, A, B) reads it back. All global loads go through the ring, so in-flight data
// costs shared memory, not registers.
template <bool FWD, int NT, bool M3, class Issue, class Use, class Mask, class Neg>
__device__ __forceinline__ void kloop(Acc<NT, M3>& acc, int ns, double2* ring, Issue&& issue, Use&& use, Mask&& mask_of,
                                      Neg&& neg_of) {
  constexpr int NS = Ring<FWD, NT>::NS, ST = Ring<FWD, NT>::kStage;
#pragma unroll
  for (int j = 0; j < NS - 1; ++j) {
    if (j < ns) issue(j, ring + j * ST, true);
    cp_commit();
  }
#pragma unroll kKUnroll
  for (int s = 0; s < ns; ++s) {
    const int si = s + NS - 1;
    if (si < ns) issue(si, ring + (si % NS) * ST, true);
    cp_commit();
    cp_wait<NS - 1>();
    __syncwarp();
    double2 A[4], B[NT];
    use(s, ring + (s % NS) * ST, A, B);
    __syncwarp();
    const unsigned mk = mask_of(s);
    if (neg_of(s)) {
      if (mk == 0xFu)
        mma_step<true, true>(acc, A, B, mk);
      else
        mma_step<true, false>(acc, A, B, mk);
    } else {
      if (mk == 0xFu)
        mma_step<false, true>(acc, A, B, mk);
      else
        mma_step<false, false>(acc, A, B, mk);
    }
  }
  cp_wait<0>();
}

// ---------------------------------------------------------------------------------------
// Lean k-loops (HS_LEAN, default). The generic kloop above recomputes every address, tile mask
// and fallback pointer of a k-step from the k-step index, which the compiler turned into ~250
// instructions per 24 DMMAs (ncu, C3 macro-step 35: 15 instructions per DMMA, DMMA pipe 24-37%
// active). Here each lane keeps running pointers that advance by constants, and every m-tile is
// computed: the factor stores M's blocks above the diagonal (within the diagonal band) as zeros
// and its padded rows / columns as zeros, so the skipped tiles only ever added 0 * finite; m-tiles
// past the stored band (the front's last band) read tile 0 again and their rows are discarded by
// the finalize. B rows past the front (columns >= k, boundary rows >= m - k) are zero-filled, so
// nothing outside the vectors is read. Each lane reads back only the ring entries it staged
// itself, so the ring needs no warp barriers.
#ifndef HS_LEAN
#define HS_LEAN 1
#endif
// 1: the forward's chunk-0 accumulators start at -T_bnd (loaded before the k-loop, round 1);
// 0: V = T_bnd - W T_sep is formed in the finalize, so no load precedes the k-loop
#ifndef HS_TB_START
#define HS_TB_START 0
#endif
// 1: the finalize's T_bnd gathers go through the ring with cp.async (all in flight at once)
#ifndef HS_STAGE_TB
#define HS_STAGE_TB 1
#endif

// Ring slot of a lane whose copy shares a 128-byte global line with the lanes of equal lane % 4
// (B rows: 8 RHS of one row; the backward's A: 8 columns of one block row). cp.async writes shared
// memory line by line as the data returns, so with slot = lane those 8 lanes (64 bytes apart) hit
// two bank groups four deep (ncu: 109 M of the backward's 208 M shared wavefronts were LDGSTS
// bank conflicts). Slot (lane % 4) * 8 + ((lane / 4 + 2 (lane % 4)) % 8) keeps a line's 8 lanes on
// 8 distinct 16-byte bank groups and so does each quarter warp of the read-back.
__device__ __forceinline__ int ring_slot(int lane) { return (lane & 3) * 8 + (((lane >> 2) + 2 * (lane & 3)) & 7); }

// Forward band item: out[32 band rows][8 NT RHS] += [M; W][rows, chunk cols] * T_sep[chunk cols],
// T = rhs + child0 V + child1 V summed at use in the reference's child order.
//   pa    this lane's A address for k-step 0, m-tile 0 (bytes)
//   toff  byte offsets of m-tiles 1..3 (tile 0's when the band has fewer row blocks)
//   xr    rhs row of this lane's column in k-step 0, RHS r0 + lane/4 (bytes)
//   vr    update-vector slot base at RHS r0 + lane/4 (bytes); rows from the staged source map
//   kcnt  k-steps whose column (col0 + 4 s) lies below k for this lane
//   okq   bit q: RHS r0 + 8q + lane/4 exists
template <int NT, bool M3, bool LEAF, bool CA>
__device__ __forceinline__ void fwd_kloop(Acc<NT, M3>& acc, int ns, double2* ring, int lane, const char* pa,
                                          unsigned astep, unsigned toff1, unsigned toff2, unsigned toff3,
                                          const char* xr, unsigned xstep, int kcnt, const char* vr, unsigned R16,
                                          const int2* sidx, bool c0, bool c1, unsigned okq, int sfull, unsigned mbase,
                                          unsigned msep, int dshift) {
  constexpr int NS = Ring<true, NT>::NS, ST = Ring<true, NT>::kStage;
  double2* const last = ring + (NS - 1) * ST;
  double2* wslot = ring;
  double2* rslot = ring;
  int si = 0;
  const int2* sx = sidx + (lane & 3);
  const int pl = ring_slot(lane);  // B parts (the A fragments of a block row are 64 contiguous bytes per lane quad)
  auto issue = [&]() {
    double2* st = wslot + lane;
    cp16a<CA>(st, pa);
    cp16a<CA>(st + 32, pa + toff1);
    cp16a<CA>(st + 64, pa + toff2);
    cp16a<CA>(st + 96, pa + toff3);
    const bool okc = si < kcnt;
    double2* sb = wslot + 4 * 32 + pl;
    if (LEAF) {
#pragma unroll
      for (int q = 0; q < NT; ++q) cp16z(sb + q * 32, xr + q * 128, okc && ((okq >> q) & 1u));
    } else {
      const int2 src = sx[4 * si];
      const char* v0 = vr + static_cast<long long>(src.x) * R16;
      const char* v1 = vr + static_cast<long long>(src.y) * R16;
      const bool o0 = okc && c0 && src.x >= 0, o1 = okc && c1 && src.y >= 0;
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const bool oq = (okq >> q) & 1u;
        cp16z(sb + q * 32, xr + q * 128, okc && oq);
        cp16z(sb + (NT + q) * 32, v0 + q * 128, o0 && oq);
        cp16z(sb + (2 * NT + q) * 32, v1 + q * 128, o1 && oq);
      }
    }
    pa += (si & 1) ? astep : 64u;
    xr += xstep;
    ++si;
    wslot = wslot == last ? ring : wslot + ST;
  };
#pragma unroll
  for (int j = 0; j < NS - 1; ++j) {
    if (j < ns) issue();
    cp_commit();
  }
  for (int s = 0; s < ns; ++s) {
    if (s + NS - 1 < ns) issue();
    cp_commit();
    cp_wait<NS - 1>();
    const double2* st = rslot + lane;
    double2 A[4], B[NT];
#pragma unroll
    for (int i = 0; i < 4; ++i) A[i] = st[i * 32];
    const double2* sb = rslot + pl;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      double2 v = sb[(4 + q) * 32];
      if (!LEAF) {
        const double2 w0 = sb[(4 + NT + q) * 32], w1 = sb[(4 + 2 * NT + q) * 32];
        v = make_double2(v.x + w0.x, v.y + w0.y);  // rhs + child0 V + child1 V, in this order
        v = make_double2(v.x + w1.x, v.y + w1.y);
      }
      B[q] = v;
    }
    rslot = rslot == last ? ring : rslot + ST;
    if (s < sfull) {
      mma_step<false, true>(acc, A, B, 0xFu);
    } else {  // diagonal column blocks (M's zero blocks above the diagonal) or a short last band
      const int d = min(max(dshift + (s >> 1), 0), 4);
      mma_masked<false>(acc, A, B, mbase & ~(msep & ((1u << d) - 1u)));
    }
  }
  cp_wait<0>();
}

// Backward column-band item: x_sep[32 band cols][8 NT RHS] = sum over the chunk's rows of
// [M; W][rows, band cols]^T y[rows], y = [z_sep; 0; -x_bnd]. Row band ta = a0/4 + s/8 holds the
// k-step's rows; its column blocks 4u..4u+3 are the m-tiles (stride rbs(ta) KB, tiles past the
// front's column blocks re-read tile 0 and are discarded).
template <int NT, bool M3, bool CA>
__device__ __forceinline__ void bwd_kloop(Acc<NT, M3>& acc, int ns, double2* ring, int lane, const double2* P,
                                          int kb, int nrb, int u, int a0, int cn, const char* zr, const char* XR,
                                          unsigned R16, int row0, int k, int kp, int nb, bool zlive, unsigned okq,
                                          const int2* sidx, int smask, unsigned mcol) {
  constexpr int NS = Ring<false, NT>::NS, ST = Ring<false, NT>::kStage;
  double2* const last = ring + (NS - 1) * ST;
  double2* wslot = ring;
  double2* rslot = ring;
  const unsigned zstep = 4u * R16;
  const int pl = ring_slot(lane);
  const int ssep = 2 * (kb - a0);  // k-steps over separator rows (z); the rest are boundary rows
  // A front the forward pass skipped (structurally zero right-hand side) has z = 0: its separator
  // rows contribute nothing, so the item starts at its first boundary row (x_sep = -W^T x_bnd).
  const int s0 = zlive ? 0 : min(max(ssep, 0), ns);
  int si = s0;
  zr += static_cast<long long>(s0) * zstep;
  const char* pa = nullptr;
  unsigned t1 = 0, t2 = 0, t3 = 0;
  auto issue = [&]() {
    if ((si & 7) == 0 || si == s0) {  // next row band (or the first k-step's)
      const int ta = (a0 >> 2) + (si >> 3);
      const int rbs = min(4, nrb - 4 * ta);
      pa = reinterpret_cast<const char*>(P + band_base(ta, kb) + 4 * u * rbs * 64);
      const unsigned ts = static_cast<unsigned>(rbs) * 1024u;
      t1 = cn > 1 ? ts : 0u;
      t2 = cn > 2 ? 2u * ts : 0u;
      t3 = cn > 3 ? 3u * ts : 0u;
    }
    double2* st = wslot + pl;
    const char* p = pa + (si & 7) * 512;
    cp16a<CA>(st, p);
    cp16a<CA>(st + 32, p + t1);
    cp16a<CA>(st + 64, p + t2);
    cp16a<CA>(st + 96, p + t3);
    const int row = row0 + 4 * si;
    const char* src;
    bool okb;
    if (si < ssep) {  // separator rows: z (a structurally zero front has z = 0)
      okb = zlive && row < k;
      src = zr;
    } else {  // boundary rows: the parent's x at the boundary positions
      okb = row - kp < nb;
      src = XR + static_cast<long long>(okb ? sidx[row - 8 * a0].x : 0) * R16;
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) cp16z(st + (4 + q) * 32, src + q * 128, okb && ((okq >> q) & 1u));
    zr += zstep;
    ++si;
    wslot = wslot == last ? ring : wslot + ST;
  };
#pragma unroll
  for (int j = 0; j < NS - 1; ++j) {
    if (s0 + j < ns) issue();
    cp_commit();
  }
  for (int s = s0; s < ns; ++s) {
    if (s + NS - 1 < ns) issue();
    cp_commit();
    cp_wait<NS - 1>();
    const double2* st = rslot + pl;
    double2 A[4], B[NT];
#pragma unroll
    for (int i = 0; i < 4; ++i) A[i] = st[i * 32];
#pragma unroll
    for (int q = 0; q < NT; ++q) B[q] = st[(4 + q) * 32];
    rslot = rslot == last ? ring : rslot + ST;
    if (s >= smask) {
      if (s >= ssep)  // boundary rows enter as -x_bnd (signs folded into the DMMA operands)
        mma_step<true, true>(acc, A, B, 0xFu);
      else
        mma_step<false, true>(acc, A, B, 0xFu);
    } else {  // M's zero blocks above the diagonal, or column blocks past the front's k
      const int ab = a0 + (s >> 1);
      unsigned mk = mcol;
      if (ab < kb) mk &= (1u << min(max(ab - 4 * u + 1, 0), 4)) - 1u;
      if (s >= ssep)
        mma_masked<true>(acc, A, B, mk);
      else
        mma_masked<false>(acc, A, B, mk);
    }
  }
  cp_wait<0>();
}


// ---------------------------------------------------------------------------------------
// Block-granular k-loops (HS_KLOOP2, default). ncu on the lean loops above (C3, 64 RHS): 263
// instructions per k-step for 24 DMMAs -- under the 168-register cap the compiler rematerialises
// the lane-derived addresses, the ring pointers and the tile masks in every k-step (S2R, BREV /
// FLO / BRX mask dispatch, 64-bit pointer selects), and a warp's k-step takes ~1900 cycles against
// 384 cycles of DMMA issue. Here the loop unit is a column block (forward) / block row (backward) =
// 2 k-steps: the ring holds two block stages (2 x 2 k-steps x 4 KB per warp), a block's copies are
// one cp.async group issued one block ahead, the tile range [lo, hi) of a block is dispatched
// once to an unpredicated body, and the loop carries only pointers that advance by constants.
// The forward's three-part stages (rhs + two child update vectors) at 16 RHS need 5 KB per k-step
// and keep the k-step-granular loop above.
#ifndef HS_KLOOP2
#define HS_KLOOP2 1
#endif
#ifndef HS_KLOOP3
#define HS_KLOOP3 1
#endif
constexpr int kSt2 = HS_ST2;       // double2 per k-step stage (4 KB): A tiles at i * 32, B parts at 128 + j * 32
                                   // (192 = one-part stages only: 13.75 KB per warp, 4 CTAs per SM)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void cpa(unsigned s, const char* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cpz(unsigned s, const char* g, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(g), "r"(ok ? 16 : 0) : "memory");
}

// one staged k-step over the m-tiles [LO, HI); NB = 3: B = rhs + child0 V + child1 V
template <bool NEG, int LO, int HI, int NT, bool M3, int NB>
__device__ __forceinline__ void kstep_mma(Acc<NT, M3>& acc, const double2* sA, const double2* sB) {
  double2 A[4], B[NT];
#pragma unroll
  for (int i = LO; i < HI; ++i) A[i] = sA[i * 32];
#pragma unroll
  for (int q = 0; q < NT; ++q) {
    double2 v = sB[q * 32];
    if (NB == 3) {
      const double2 w0 = sB[(NT + q) * 32], w1 = sB[(2 * NT + q) * 32];
      v = make_double2(v.x + w0.x, v.y + w0.y);  // rhs + child0 V + child1 V, in this order
      v = make_double2(v.x + w1.x, v.y + w1.y);
    }
    B[q] = v;
  }
  mma_range<NEG, LO, HI>(acc, A, B);
}
// both k-steps of a staged block
template <bool NEG, int LO, int HI, int NT, bool M3, int NB>
__device__ __forceinline__ void block_mma(Acc<NT, M3>& acc, const double2* sA, const double2* sB) {
#pragma unroll
  for (int h = 0; h < 2; ++h) kstep_mma<NEG, LO, HI, NT, M3, NB>(acc, sA + h * kSt2, sB + h * kSt2);
}
// one k-step, tile range [lo, hi) (the forward's cases)
template <int NT, bool M3, int NB>
__device__ __forceinline__ void kstep_dispatch(Acc<NT, M3>& acc, const double2* sA, const double2* sB, int lo, int hi) {
  if (lo == 0 && hi == 4)
    kstep_mma<false, 0, 4, NT, M3, NB>(acc, sA, sB);
  else if (hi == 4 && lo == 1)
    kstep_mma<false, 1, 4, NT, M3, NB>(acc, sA, sB);
  else if (hi == 4 && lo == 2)
    kstep_mma<false, 2, 4, NT, M3, NB>(acc, sA, sB);
  else if (hi == 4 && lo == 3)
    kstep_mma<false, 3, 4, NT, M3, NB>(acc, sA, sB);
  else if (lo == 0 && hi == 3)
    kstep_mma<false, 0, 3, NT, M3, NB>(acc, sA, sB);
  else if (lo == 0 && hi == 2)
    kstep_mma<false, 0, 2, NT, M3, NB>(acc, sA, sB);
  else if (lo == 0 && hi == 1)
    kstep_mma<false, 0, 1, NT, M3, NB>(acc, sA, sB);
  else if (lo < hi) {
    double2 A[4], B[NT];
#pragma unroll
    for (int i = 0; i < 4; ++i) A[i] = sA[i * 32];
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      double2 v = sB[q * 32];
      if (NB == 3) {
        const double2 w0 = sB[(NT + q) * 32], w1 = sB[(2 * NT + q) * 32];
        v = make_double2(v.x + w0.x, v.y + w0.y);
        v = make_double2(v.x + w1.x, v.y + w1.y);
      }
      B[q] = v;
    }
    mma_step<false, false>(acc, A, B, ((1u << hi) - 1u) & ~((1u << lo) - 1u));
  }
}
// tile ranges of the two passes: the backward's are prefixes [0, hi), the forward's suffixes
// [lo, 4) or, in a short last band, prefixes; anything else (a short last band that also crosses
// the diagonal) takes the predicated step
template <bool NEG, int NT, bool M3, int NB>
__device__ __forceinline__ void block_dispatch(Acc<NT, M3>& acc, const double2* sA, const double2* sB, int lo, int hi) {
  if (lo == 0) {
    if (hi == 4)
      block_mma<NEG, 0, 4, NT, M3, NB>(acc, sA, sB);
    else if (hi == 3)
      block_mma<NEG, 0, 3, NT, M3, NB>(acc, sA, sB);
    else if (hi == 2)
      block_mma<NEG, 0, 2, NT, M3, NB>(acc, sA, sB);
    else if (hi == 1)
      block_mma<NEG, 0, 1, NT, M3, NB>(acc, sA, sB);
  } else if (hi == 4 && !NEG) {
    if (lo == 1)
      block_mma<NEG, 1, 4, NT, M3, NB>(acc, sA, sB);
    else if (lo == 2)
      block_mma<NEG, 2, 4, NT, M3, NB>(acc, sA, sB);
    else if (lo == 3)
      block_mma<NEG, 3, 4, NT, M3, NB>(acc, sA, sB);
  } else if (lo < hi) {
    const unsigned mk = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      double2 A[4], B[NT];
#pragma unroll
      for (int i = 0; i < 4; ++i) A[i] = sA[h * kSt2 + i * 32];
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        double2 v = sB[h * kSt2 + q * 32];
        if (NB == 3) {
          const double2 w0 = sB[h * kSt2 + (NT + q) * 32], w1 = sB[h * kSt2 + (2 * NT + q) * 32];
          v = make_double2(v.x + w0.x, v.y + w0.y);
          v = make_double2(v.x + w1.x, v.y + w1.y);
        }
        B[q] = v;
      }
      mma_step<NEG, false>(acc, A, B, mk);
    }
  }
}

// Forward band item over its nblk column blocks (arguments as fwd_kloop):
//   bstep  bytes from a column block to the next (rbs KB)      bfull  leading blocks with every tile live
//   dl     first block's column block index minus 4 t          sepn   separator row blocks of the band
template <int NT, bool M3, bool LEAF>
__device__ __forceinline__ void fwd_kloop2(Acc<NT, M3>& acc, int nblk, double2* ring, int lane, const char* pa,
                                           unsigned bstep, unsigned t1, unsigned t2, unsigned t3, const char* xr,
                                           unsigned xstep, int kcnt, const char* vr, unsigned R16, const int2* sidx,
                                           bool c0, bool c1, unsigned okq, int bfull, int dl, int sepn, int rbs) {
  constexpr int NB = LEAF ? 1 : 3;
  static_assert((4 + NB * NT) * 32 <= kSt2, "stage");
  const int pl = ring_slot(lane);
  const unsigned wA = smem_u32(ring) + lane * 16, wB = smem_u32(ring) + 128 * 16 + pl * 16;
  const double2* rA = ring + lane;
  const double2* rB = ring + 128 + pl;
  unsigned woff = 0;
  int irem = kcnt;  // k-steps of this lane's column still below k
  const int2* sx = sidx + (lane & 3);
  const bool q0 = okq & 1u, q1 = (okq >> 1) & 1u;
  auto issue_block = [&]() {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const char* p = pa + h * 64;
      const unsigned sa = wA + woff + h * (kSt2 * 16);
      cpa(sa, p);
      cpa(sa + 512, p + t1);
      cpa(sa + 1024, p + t2);
      cpa(sa + 1536, p + t3);
      const bool okc = irem > h;
      const unsigned sb = wB + woff + h * (kSt2 * 16);
      if (LEAF) {
        cpz(sb, xr, okc && q0);
        if (NT > 1) cpz(sb + 512, xr + 128, okc && q1);
      } else {
        const int2 src = sx[4 * h];
        const char* v0 = vr + static_cast<long long>(src.x) * R16;
        const char* v1 = vr + static_cast<long long>(src.y) * R16;
        const bool o0 = okc && c0 && src.x >= 0, o1 = okc && c1 && src.y >= 0;
        cpz(sb, xr, okc && q0);
        cpz(sb + NT * 512, v0, o0 && q0);
        cpz(sb + 2 * NT * 512, v1, o1 && q0);
        if (NT > 1) {
          cpz(sb + 512, xr + 128, okc && q1);
          cpz(sb + (NT + 1) * 512, v0 + 128, o0 && q1);
          cpz(sb + (2 * NT + 1) * 512, v1 + 128, o1 && q1);
        }
      }
      xr += xstep;
    }
    pa += bstep;
    irem -= 2;
    sx += 8;
    woff ^= 2 * kSt2 * 16;
  };
  if (nblk > 0) issue_block();
  cp_commit();
  int roff = 0;
#pragma unroll 1
  for (int b = 0; b < nblk; ++b) {
    if (b + 1 < nblk) issue_block();
    cp_commit();
    cp_wait<1>();
    if (b < bfull) {
      block_mma<false, 0, 4, NT, M3, NB>(acc, rA + roff, rB + roff);
    } else {  // diagonal column blocks (M's zero blocks above the diagonal) or a short last band
      const int lo = min(max(dl + b, 0), sepn);
      block_dispatch<false, NT, M3, NB>(acc, rA + roff, rB + roff, lo, rbs);
    }
    roff ^= 2 * kSt2;
  }
  cp_wait<0>();
}

// The forward's three-part stages at 16 RHS (a front with children: rhs + two update vectors,
// 5 KB per k-step): a ring of three k-step stages, copies two k-steps ahead, the same constant-
// stride pointers and per-range bodies as fwd_kloop2.
template <bool M3>
__device__ __forceinline__ void fwd_kloop3(Acc<2, M3>& acc, int nblk, double2* ring, int lane, const char* pa,
                                           unsigned bstep, unsigned t1, unsigned t2, unsigned t3, const char* xr,
                                           unsigned xstep, int kcnt, const char* vr, unsigned R16, const int2* sidx,
                                           bool c0, bool c1, unsigned okq, int bfull, int dl, int sepn, int rbs) {
  constexpr int NT = 2, ST = (4 + 3 * NT) * 32;  // double2 per stage
  const int ns = 2 * nblk;
  const int pl = ring_slot(lane);
  const unsigned wA = smem_u32(ring) + lane * 16, wB = smem_u32(ring) + 128 * 16 + pl * 16;
  const double2* rA = ring + lane;
  const double2* rB = ring + 128 + pl;
  unsigned woff = 0;
  int irem = kcnt;
  const int2* sx = sidx + (lane & 3);
  const bool q0 = okq & 1u, q1 = (okq >> 1) & 1u;
  unsigned astep = 64u;  // to the block's second k-step, then on to the next block
  auto issue_step = [&]() {
    const unsigned sa = wA + woff;
    cpa(sa, pa);
    cpa(sa + 512, pa + t1);
    cpa(sa + 1024, pa + t2);
    cpa(sa + 1536, pa + t3);
    const bool okc = irem > 0;
    const unsigned sb = wB + woff;
    const int2 src = *sx;
    const char* v0 = vr + static_cast<long long>(src.x) * R16;
    const char* v1 = vr + static_cast<long long>(src.y) * R16;
    const bool o0 = okc && c0 && src.x >= 0, o1 = okc && c1 && src.y >= 0;
    cpz(sb, xr, okc && q0);
    cpz(sb + 512, xr + 128, okc && q1);
    cpz(sb + 2 * 512, v0, o0 && q0);
    cpz(sb + 3 * 512, v0 + 128, o0 && q1);
    cpz(sb + 4 * 512, v1, o1 && q0);
    cpz(sb + 5 * 512, v1 + 128, o1 && q1);
    pa += astep;
    astep = bstep - astep;  // 64, bstep - 64, 64, ...
    xr += xstep;
    --irem;
    sx += 4;
    woff = woff == 2 * ST * 16 ? 0u : woff + ST * 16;
  };
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    if (j < ns) issue_step();
    cp_commit();
  }
  int roff = 0;
#pragma unroll 1
  for (int sidx_k = 0; sidx_k < ns; ++sidx_k) {
    if (sidx_k + 2 < ns) issue_step();
    cp_commit();
    cp_wait<2>();
    const int b = sidx_k >> 1;
    if (b < bfull)
      kstep_mma<false, 0, 4, NT, M3, 3>(acc, rA + roff, rB + roff);
    else
      kstep_dispatch<NT, M3, 3>(acc, rA + roff, rB + roff, min(max(dl + b, 0), sepn), rbs);
    roff = roff == 2 * ST ? 0 : roff + ST;
  }
  cp_wait<0>();
}

// Backward column-band item over the block rows a0 + [b0, nblk) (arguments as bwd_kloop; b0 > 0
// skips the separator rows of a front whose z is structurally zero).
template <int NT, bool M3>
__device__ __forceinline__ void bwd_kloop2(Acc<NT, M3>& acc, int nblk, double2* ring, int lane, const double2* P, int kb,
                                           int nrb, int u, int a0, int cn, const char* zr, const char* XR, unsigned R16,
                                           int row0, int k, int kp, int nb, bool zlive, unsigned okq, const int2* sidx) {
  const int pl = ring_slot(lane);
  const unsigned wA = smem_u32(ring) + pl * 16;
  const double2* rA = ring + pl;
  const int bsep = max(min(kb - a0, nblk), 0);  // block rows of separator rows (z); the rest are boundary rows
  const int b0 = zlive ? 0 : bsep;
  const unsigned zstep = 4u * R16;
  const bool q0 = okq & 1u, q1 = (okq >> 1) & 1u;
  // issue side
  int ib = b0;
  unsigned woff = 0;
  const char* pa = nullptr;
  unsigned t1 = 0, t2 = 0, t3 = 0;
  int zrem = k > row0 ? ((k - row0 + 3) >> 2) - 2 * b0 : 0;  // k-steps of this lane's row still below k
  int brow = row0 + 8 * b0 - kp;                                 // this lane's boundary row index in k-step 0 of block ib
  zr += static_cast<long long>(2 * b0) * zstep;
  const int* bx = reinterpret_cast<const int*>(sidx) + 2 * (lane & 3) + 16 * b0;  // .x of entry (lane & 3) + 8 ib + 4 h
  auto issue_block = [&]() {
    if ((ib & 3) == 0 || ib == b0) {  // next row band (or the first block's)
      const int ta = (a0 >> 2) + (ib >> 2);
      const int rbs = min(4, nrb - 4 * ta);
      pa = reinterpret_cast<const char*>(P + band_base(ta, kb) + 4 * u * rbs * 64) + (ib & 3) * 1024;
      const unsigned ts = static_cast<unsigned>(rbs) * 1024u;
      t1 = cn > 1 ? ts : 0u;
      t2 = cn > 2 ? 2u * ts : 0u;
      t3 = cn > 3 ? 3u * ts : 0u;
    }
    const bool sep = ib < bsep;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const char* p = pa + h * 512;
      const unsigned sa = wA + woff + h * (kSt2 * 16);
      cpa(sa, p);
      cpa(sa + 512, p + t1);
      cpa(sa + 1024, p + t2);
      cpa(sa + 1536, p + t3);
      const char* src;
      bool okb;
      if (sep) {  // separator rows: z
        okb = zrem > h;
        src = zr + h * zstep;
      } else {  // boundary rows: the parent's x at the boundary positions
        okb = brow + 4 * h < nb;
        src = XR + static_cast<long long>(okb ? bx[8 * h] : 0) * R16;  // (int2 entries: .x at stride 2 ints)
      }
      cpz(sa + 2048, src, okb && q0);
      if (NT > 1) cpz(sa + 2048 + 512, src + 128, okb && q1);
    }
    pa += 1024;
    zr += 2 * zstep;
    zrem -= 2;
    brow += 8;
    bx += 16;
    ++ib;
    woff ^= 2 * kSt2 * 16;
  };
  if (ib < nblk) issue_block();
  cp_commit();
  int roff = 0;
  const int hz = 1 - 4 * u + a0;  // live tiles of separator block row a0 + b: min(b + hz, cn)
#pragma unroll 1
  for (int b = b0; b < nblk; ++b) {
    if (ib < nblk) issue_block();
    cp_commit();
    cp_wait<1>();
    if (b < bsep) {
      const int hi = min(b + hz, cn);
      block_dispatch<false, NT, M3, 1>(acc, rA + roff, rA + roff + 128, 0, hi);
    } else {  // boundary rows enter as -x_bnd (signs folded into the DMMA operands)
      block_dispatch<true, NT, M3, 1>(acc, rA + roff, rA + roff + 128, 0, cn);
    }
    roff ^= 2 * kSt2;
  }
  cp_wait<0>();
}

// Item ranges
struct FwdRange {
  int t, rbs, cb0, cb1;
};
__device__ __forceinline__ FwdRange fwd_range(const SolveJob& J, const Geo& g, const SolveItem& it) {
  FwdRange r;
  r.t = it.idx;
  r.rbs = min(4, g.nrb - 4 * r.t);
  r.cb0 = it.chunk * J.kc;
  r.cb1 = min(min(g.kb, 4 * r.t + 4), r.cb0 + J.kc);
  return r;
}
struct BwdRange {
  int u, a0, a1;
};
__device__ __forceinline__ BwdRange bwd_range(const SolveJob& J, const Geo& g, const SolveItem& it) {
  BwdRange r;
  r.u = it.idx;
  r.a0 = 4 * r.u + it.chunk * J.kr;
  r.a1 = min(g.nrb, r.a0 + J.kr);
  return r;
}

// Issued before the dependency wait: the item's factor range -> L2 (bulk prefetch) and its
// index slice -> shared memory (cp.async group, waited for after the dependency wait).
template <bool FWD>
__device__ __forceinline__ void item_prefetch(const SolveArgs& a, const SolveJob& J, const Geo& g, const SolveItem& it,
                                              int2* sidx, int lane, bool pf_l2 = true) {
  if (FWD) {
    const FwdRange r = fwd_range(J, g, it);
    if (lane == 0 && pf_l2)
      prefetch_l2(J.factor + band_base(r.t, g.kb) + r.cb0 * r.rbs * 64,
                  static_cast<unsigned>((r.cb1 - r.cb0) * r.rbs) * 1024u);
    const bool leaf = J.child0 < 0 && J.child1 < 0;
    if (!leaf) {
      const int n = min(8 * r.cb1, J.k) - 8 * r.cb0;
      for (int j = lane; j < n; j += 32) cp_small<8>(sidx + j, J.pm + 8 * r.cb0 + j);
    }
    // finalize data of band row `lane`: boundary rows' sources (T_bnd, also the chunk-0
    // accumulator start), separator rows' 1/d
    int2* fsrc = sidx + kIdx;
    double2* fdv = reinterpret_cast<double2*>(fsrc + 32);
    const int pr = 32 * r.t + lane;
    if (!leaf && pr >= g.kp && pr - g.kp < J.m - J.k)
      cp_small<8>(fsrc + lane, J.pm + J.k + (pr - g.kp));
    else
      fsrc[lane] = make_int2(-1, -1);
    if (pr < J.k) cp_small<16>(fdv + lane, J.dinv + pr);
  } else {
    const BwdRange r = bwd_range(J, g, it);
    if (lane == 0 && pf_l2) {
      const int ncol = min(4, g.kb - 4 * r.u);
      for (int ta = r.a0 >> 2; ta <= (r.a1 - 1) >> 2; ++ta) {
        const int rbs = min(4, g.nrb - 4 * ta);
        prefetch_l2(J.factor + band_base(ta, g.kb) + 4 * r.u * rbs * 64, static_cast<unsigned>(ncol * rbs) * 1024u);
      }
    }
    const int nb = J.m - J.k, lo = max(8 * r.a0, g.kp), hi = min(8 * r.a1, g.kp + nb);
    for (int row = lo + lane; row < hi; row += 32) cp_small<4>(sidx + (row - 8 * r.a0), J.be + (row - g.kp));
  }
  cp_commit();
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p) : "memory");
}
// the warp's next ticket (lane 0's atomic; its latency is paid only where the value is used)
__device__ __forceinline__ void take_ticket(const SolveArgs& a, unsigned& tk, bool& took, int lane) {
  if (HS_LATE_TICKET && !took) {
    if (lane == 0) tk = atomicAdd(a.queue, 1u);
    took = true;
  }
}
// HS_PREFETCH_NEXT (measured neutral on C3, off): once the ticket is back (before the split reduce / finalize), the next item's
// record is prefetched into L1, and after its load the next job record and task masks too, so the
// next item starts on L1 hits instead of two dependent L2 round trips
#ifndef HS_PREFETCH_NEXT
#define HS_PREFETCH_NEXT 0
#endif
// HS_NEXT_L2 (measured 3% slower on C3, off): the next item's first factor range prefetched to L2
// as soon as its record is known
#ifndef HS_NEXT_L2
#define HS_NEXT_L2 0
#endif
__device__ __forceinline__ void prefetch_next_record(const SolveArgs& a, unsigned tk, int lane) {
  if (HS_PREFETCH_NEXT && lane == 0) {
    const int nxt = static_cast<int>(gridDim.x * (kThreads / 32) + tk);
    if (nxt < a.nitems) prefetch_l1(a.items + nxt);
  }
}

// ---------------------------------------------------------------------------------------
// forward band item: out[32 rows][8 NT RHS] = [M; W][band rows, chunk cols] T_sep[chunk cols].
// Boundary rows produce V = T_bnd - W T_sep: their chunk-0 accumulators start at -T_bnd (the
// children's updates at the front's boundary, in the reference's child order), loaded while the
// k-loop's first stages are in flight, so the finalize only scales and stores. Returns whether
// this warp finalized the band (the caller signals it).
template <int NT, bool M3, bool CA>
__device__ bool fwd_item(const SolveArgs& a, const SolveJob& J, const Geo& g, const SolveItem& it, double2* V,
                         int lane, double2* ring, const int2* sidx, unsigned long long* tr, unsigned clive,
                         unsigned& tk, bool& took) {
  const int R = a.R, r0 = it.r0, rl = lane >> 2;
  const FwdRange rg = fwd_range(J, g, it);
  const int t = rg.t, rbs = rg.rbs, cb0 = rg.cb0, cb1 = rg.cb1;
  const double2* P = J.factor + band_base(t, g.kb) + rl * 8 + (lane & 3);
  const double2* X = a.rbs + it.slot * a.slot_stride + static_cast<long long>(J.sep_off) * R;  // right-hand side (the task's slot)
  const bool leaf = J.child0 < 0 && J.child1 < 0;
  const int2* fsrc = sidx + kIdx;
  const double2* fdv = reinterpret_cast<const double2*>(fsrc + 32);
  // live m-tiles of k-step s: row blocks of the band, minus M's zero blocks above the diagonal
  // Per-item constants of the k-loop (the loop body is what a lone critical-path warp waits on:
  // per k-step it computes a mask, one shared index load and a few wide multiply-adds).
  // live m-tiles of k-step s: row blocks of the band (base), minus M's zero blocks above the
  // diagonal: tile i is a separator row block (i < kb - 4t) whose column block cb exceeds 4t + i
  const unsigned mbase = (1u << rbs) - 1u;
  const int sepn = g.kb - 4 * t;
  const unsigned msep = sepn >= 4 ? 0xFu : sepn <= 0 ? 0u : (1u << sepn) - 1u;
  auto mask_of = [&](int s) {
    const int d = min(max(cb0 + (s >> 1) - 4 * t, 0), 4);
    return mbase & ~(msep & ((1u << d) - 1u));
  };
  const double2* PA = P + cb0 * rbs * 64;  // A of k-step 0
  const int col0 = 8 * cb0 + (lane & 3);   // inner-dimension position of this lane in k-step 0
  const unsigned R16 = static_cast<unsigned>(R) * 16u;
  const char* XR = reinterpret_cast<const char*>(X + r0 + rl) + static_cast<size_t>(static_cast<unsigned>(col0)) * R16;
  const char* VR = reinterpret_cast<const char*>(V + r0 + rl);
  bool okr[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) okr[q] = r0 + 8 * q + rl < R;
  const bool c0 = !leaf && (clive & 1u), c1 = !leaf && (clive & 2u);  // a structurally zero child's V is stale
  auto issue = [&](int s, double2* st, bool live) {  // live = false: a k-step past the end (no loads)
    const double2* p = PA + (s >> 1) * rbs * 64 + 4 * (s & 1);
    const unsigned mk = live ? mask_of(s) : 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool ok = (mk >> i) & 1u;
      cp16(st + i * 32 + lane, ok ? p + i * 64 : P, ok);
    }
    const bool okc = live && col0 + 4 * s < J.k;
    int2 src = make_int2(0, 0);
    if ((c0 || c1) && okc) src = sidx[(lane & 3) + 4 * s];
    const bool o0 = okc && c0 && src.x >= 0, o1 = okc && c1 && src.y >= 0;  // -1: not in that child
    const char* xr = XR + static_cast<size_t>(static_cast<unsigned>(4 * s)) * R16;
    const char* v0 = VR + static_cast<size_t>(static_cast<unsigned>(src.x)) * R16;
    const char* v1 = VR + static_cast<size_t>(static_cast<unsigned>(src.y)) * R16;
    double2* sb = st + 4 * 32 + lane;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const bool ok = okc && okr[q];
      cp16(sb + (0 * NT + q) * 32, ok ? reinterpret_cast<const double2*>(xr) + 8 * q : X, ok);
      cp16(sb + (1 * NT + q) * 32, ok && o0 ? reinterpret_cast<const double2*>(v0) + 8 * q : X, ok && o0);
      cp16(sb + (2 * NT + q) * 32, ok && o1 ? reinterpret_cast<const double2*>(v1) + 8 * q : X, ok && o1);
    }
  };
  auto use = [&](int, const double2* st, double2 (&A)[4], double2 (&B)[NT]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) A[i] = st[i * 32 + lane];
    const double2* sb = st + 4 * 32 + lane;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      double2 v = sb[(0 * NT + q) * 32];
      const double2 w0 = sb[(1 * NT + q) * 32], w1 = sb[(2 * NT + q) * 32];
      v = make_double2(v.x + w0.x, v.y + w0.y);  // rhs + child0 V + child1 V, in this order
      B[q] = make_double2(v.x + w1.x, v.y + w1.y);
    }
  };
  Acc<NT, M3> acc;
  acc_zero(acc);
  if (HS_TB_START && it.chunk == 0 && !leaf) {  // -T_bnd = -((0 + child0 V) + child1 V) on boundary rows
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (4 * t + i < g.kb) continue;  // separator row block
      int2 src = fsrc[8 * i + rl];
      if (!(clive & 1u)) src.x = -1;
      if (!(clive & 2u)) src.y = -1;
#pragma unroll
      for (int q = 0; q < NT; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = r0 + 8 * q + 2 * (lane & 3) + e;
          double2 tb = czero();
          if (src.x >= 0 && r < R) {
            const double2 w = __ldcg(V + static_cast<long long>(src.x) * R + r);
            tb = make_double2(tb.x + w.x, tb.y + w.y);
          }
          if (src.y >= 0 && r < R) {
            const double2 w = __ldcg(V + static_cast<long long>(src.y) * R + r);
            tb = make_double2(tb.x + w.x, tb.y + w.y);
          }
          acc_set(acc, i, q, e, -tb.x, -tb.y);
        }
    }
  }
#if HS_LEAN
  {
    const unsigned rb1 = static_cast<unsigned>(rbs);
    const unsigned t1 = rb1 > 1 ? 1024u : 0u, t2 = rb1 > 2 ? 2048u : 0u, t3 = rb1 > 3 ? 3072u : 0u;
    const char* pa = reinterpret_cast<const char*>(PA);
    const int kcnt = J.k > col0 ? (J.k - col0 + 3) >> 2 : 0;
    unsigned okq = 0;
#pragma unroll
    for (int q = 0; q < NT; ++q) okq |= okr[q] ? 1u << q : 0u;
    const int ns = 2 * (cb1 - cb0);
    // k-steps before the diagonal column blocks run every m-tile (when the band is full)
    const int sfull = mbase == 0xFu ? max(0, 2 * (4 * t - cb0)) : 0;
    const int bfull = rbs == 4 ? max(0, 4 * t - cb0) : 0, sepc = min(max(sepn, 0), 4);
    if (HS_KLOOP2 && !CA && !c0 && !c1)
      fwd_kloop2<NT, M3, true>(acc, cb1 - cb0, ring, lane, pa, rb1 * 1024u, t1, t2, t3, XR, 4u * R16, kcnt, VR, R16, sidx,
                               false, false, okq, bfull, cb0 - 4 * t, sepc, rbs);
    else if (!c0 && !c1)
      fwd_kloop<NT, M3, true, CA>(acc, ns, ring, lane, pa, rb1 * 1024u - 64u, t1, t2, t3, XR, 4u * R16, kcnt, VR, R16,
                              sidx, false, false, okq, sfull, mbase, msep, cb0 - 4 * t);
    else if (HS_KLOOP2 && !CA && NT == 1 && (4 + 3 * NT) * 32 <= kSt2) {
      if constexpr (NT == 1 && (4 + 3 * NT) * 32 <= kSt2)  // (three-part stages at 16 RHS exceed the block stage)
        fwd_kloop2<NT, M3, false>(acc, cb1 - cb0, ring, lane, pa, rb1 * 1024u, t1, t2, t3, XR, 4u * R16, kcnt, VR, R16, sidx,
                                  c0, c1, okq, bfull, cb0 - 4 * t, sepc, rbs);
    } else if (HS_KLOOP2 && HS_KLOOP3 && !CA && NT == 2 && 3 * 320 <= RingArea<true>::kRing) {
      if constexpr (NT == 2 && 3 * 320 <= RingArea<true>::kRing)
        fwd_kloop3<M3>(acc, cb1 - cb0, ring, lane, pa, rb1 * 1024u, t1, t2, t3, XR, 4u * R16, kcnt, VR, R16, sidx, c0, c1,
                       okq, bfull, cb0 - 4 * t, sepc, rbs);
    } else
      fwd_kloop<NT, M3, false, CA>(acc, ns, ring, lane, pa, rb1 * 1024u - 64u, t1, t2, t3, XR, 4u * R16, kcnt, VR, R16,
                               sidx, c0, c1, okq, sfull, mbase, msep, cb0 - 4 * t);
  }
#else
  kloop<true, NT>(acc, 2 * (cb1 - cb0), ring, issue, use, mask_of, [](int) { return false; });
#endif
  acc_finish(acc);
  take_ticket(a, tk, took, lane);
  prefetch_next_record(a, tk, lane);
  if (tr && lane == 0) {
    tr[2] = gtime();
    tr[6] += 2 * (cb1 - cb0);
  }
  const int nch = nch_fwd(g, t, J.kc);
  if (nch > 1) {
    int loc = 0;
    for (int tt = 0; tt < t; ++tt) loc += nch_fwd(g, tt, J.kc);
    const long long slot_part = static_cast<long long>(it.slot) * a.part_stride + J.part_off + loc;
    double* base = a.part + (slot_part * a.ngr + r0 / 8) * kTileDoubles;
    int* arr = a.arr + (static_cast<long long>(it.slot) * a.arr_stride + J.arr_off + t) * a.ngr + r0 / 8;
    if (!split_reduce(acc, base, static_cast<long long>(a.ngr) * kTileDoubles, nch, it.chunk, arr, lane)) return false;
  }
  if (tr && lane == 0) tr[3] = gtime();
  // T_bnd of the band's boundary rows (the children's update vectors at the front's boundary)
  // staged through the ring, which is free after the k-loop: all of a lane's up to 32 gathers are
  // in flight at once. As plain loads feeding the sums they ran nearly one at a time under the
  // register cap (trace, C3: fronts with k <= 16 spent 7.6 us per item here against 3.8 us in the
  // k-loop; ncu: long-scoreboard stalls on the finalize's DADDs led the forward kernel).
  const bool stage_tb = HS_STAGE_TB && 16 * NT * 32 <= RingArea<true>::kRing && !(HS_TB_START || leaf);
  if (stage_tb) {
    const unsigned sb = smem_u32(ring) + lane * 16;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (4 * t + i < g.kb) continue;  // separator row block
      int2 src = fsrc[8 * i + rl];     // (-1, -1) off the boundary rows
      if (!(clive & 1u)) src.x = -1;
      if (!(clive & 2u)) src.y = -1;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int sr = c ? src.y : src.x;
        const char* gp = reinterpret_cast<const char*>(V + static_cast<long long>(sr) * R + r0 + 2 * (lane & 3));
#pragma unroll
        for (int q = 0; q < NT; ++q)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            cpz(sb + (((i * 2 + c) * NT + q) * 2 + e) * 512, gp + (8 * q + e) * 16,
                sr >= 0 && r0 + 8 * q + 2 * (lane & 3) + e < R);
      }
    }
    cp_commit();
    cp_wait<0>();
  }
  // finalize: z = D^-1 (M T_sep) on separator rows, V = -(acc) = T_bnd - W T_sep on boundary rows
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int pr = 32 * t + 8 * i + rl;
    if (pr < J.k) {
      const double2 dv = fdv[8 * i + rl];
      double2* zo = a.x1s + it.slot * a.slot_stride + static_cast<long long>(J.sep_off + pr) * R;
#pragma unroll
      for (int q = 0; q < NT; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = r0 + 8 * q + 2 * (lane & 3) + e;
          if (r < R) __stcg(zo + r, cmul(make_double2(acc.v[i][q][0][e], acc.v[i][q][1][e]), dv));
        }
    } else if (pr >= g.kp && pr - g.kp < J.m - J.k) {
      double2* vo = V + static_cast<long long>(J.v_off + pr - g.kp) * R;
      if (HS_TB_START || leaf) {  // V = -acc (acc started at -T_bnd; a leaf has T_bnd = 0)
#pragma unroll
        for (int q = 0; q < NT; ++q)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = r0 + 8 * q + 2 * (lane & 3) + e;
            if (r < R) __stcg(vo + r, make_double2(-acc.v[i][q][0][e], -acc.v[i][q][1][e]));
          }
      } else if (stage_tb) {  // V = T_bnd - W T_sep from the staged T_bnd = (0 + child0 V) + child1 V (zero where absent)
#pragma unroll
        for (int q = 0; q < NT; ++q)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = r0 + 8 * q + 2 * (lane & 3) + e;
            if (r >= R) continue;
            const double2 w0 = ring[(((i * 2 + 0) * NT + q) * 2 + e) * 32 + lane];
            const double2 w1 = ring[(((i * 2 + 1) * NT + q) * 2 + e) * 32 + lane];
            double2 tb = czero();
            tb = make_double2(tb.x + w0.x, tb.y + w0.y);
            tb = make_double2(tb.x + w1.x, tb.y + w1.y);
            __stcg(vo + r, make_double2(tb.x - acc.v[i][q][0][e], tb.y - acc.v[i][q][1][e]));
          }
      } else {  // V = T_bnd - W T_sep, T_bnd = (0 + child0 V) + child1 V (reference order: product first)
        int2 src = fsrc[8 * i + rl];
        if (!(clive & 1u)) src.x = -1;
        if (!(clive & 2u)) src.y = -1;
#pragma unroll
        for (int q = 0; q < NT; ++q)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = r0 + 8 * q + 2 * (lane & 3) + e;
            if (r >= R) continue;
            double2 tb = czero();
            if (src.x >= 0) {
              const double2 w = __ldcg(V + static_cast<long long>(src.x) * R + r);
              tb = make_double2(tb.x + w.x, tb.y + w.y);
            }
            if (src.y >= 0) {
              const double2 w = __ldcg(V + static_cast<long long>(src.y) * R + r);
              tb = make_double2(tb.x + w.x, tb.y + w.y);
            }
            __stcg(vo + r, make_double2(tb.x - acc.v[i][q][0][e], tb.y - acc.v[i][q][1][e]));
          }
      }
    }
  }
  return true;
}

// ---------------------------------------------------------------------------------------
// backward column-band item: x_sep[32 cols][8 NT RHS] = sum over the chunk's rows of
// [M; W][rows, band cols]^T y[rows], y = [z_sep; 0; -x_bnd]
template <int NT, bool M3, bool CA>
__device__ bool bwd_item(const SolveArgs& a, const SolveJob& J, const Geo& g, const SolveItem& it, int lane,
                         double2* ring, const int2* sidx, unsigned long long* tr, bool zlive, unsigned& tk,
                         bool& took) {
  const int R = a.R, r0 = it.r0, rl = lane >> 2;
  const BwdRange rg = bwd_range(J, g, it);
  const int u = rg.u, a0 = rg.a0, a1 = rg.a1;
  const double2* P = J.factor + (lane & 3) * 8 + rl;
  const double2* Z = a.x1s + it.slot * a.slot_stride + static_cast<long long>(J.sep_off) * R;
  const int nb = J.m - J.k;
  // live m-tiles (column blocks 4u + i) of k-step s: columns below k (mcol), minus M's zero
  // blocks above the diagonal while the rows are separator rows (column block 4u + i > row block)
  const int cn = g.kb - 4 * u;
  const unsigned mcol = cn >= 4 ? 0xFu : (1u << cn) - 1u;
  auto mask_of = [&](int s) {
    const int ab = a0 + (s >> 1);
    if (ab >= g.kb) return mcol;
    const int d = min(max(ab - 4 * u + 1, 0), 4);
    return mcol & ((1u << d) - 1u);
  };
  // a0 is a multiple of 4 (kr is), so k-steps 8j..8j+7 read row band (a0 >> 2) + j
  const double2* PB = P;  // base of the k-step's row band + this item's column blocks
  int rbs = 4;
  const unsigned R16 = static_cast<unsigned>(R) * 16u;
  const int row0 = 8 * a0 + (lane & 3);  // row of this lane in k-step 0
  const char* ZR = reinterpret_cast<const char*>(Z + r0 + rl);
  const char* XR = reinterpret_cast<const char*>(J.x + r0 + rl);
  bool okr[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) okr[q] = r0 + 8 * q + rl < R;
  auto issue = [&](int s, double2* st, bool live) {  // live = false: a k-step past the end (no loads)
    {  // row band of k-step s (branch-free: stays in the k-step's basic block)
      const int ta = (a0 >> 2) + (s >> 3);
      rbs = min(4, g.nrb - 4 * ta);
      PB = P + band_base(ta, g.kb) + 4 * u * rbs * 64;
    }
    const double2* p = PB + ((s >> 1) & 3) * 64 + 32 * (s & 1);
    const unsigned mk = live ? mask_of(s) : 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool ok = (mk >> i) & 1u;
      cp16(st + i * 32 + lane, ok ? p + i * rbs * 64 : P, ok);
    }
    const int row = row0 + 4 * s;
    const char* src;
    bool okb;
    if (a0 + (s >> 1) < g.kb) {  // separator rows: z (a structurally zero front has z = 0)
      okb = live && zlive && row < J.k;
      src = ZR + static_cast<size_t>(static_cast<unsigned>(row)) * R16;
    } else {  // boundary rows: the parent's x at the boundary positions
      okb = live && row - g.kp < nb;
      const int pos = okb ? sidx[row - 8 * a0].x : 0;
      src = XR + static_cast<size_t>(static_cast<unsigned>(pos)) * R16;
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const bool ok = okb && okr[q];
      cp16(st + (4 + q) * 32 + lane, ok ? reinterpret_cast<const double2*>(src) + 8 * q : Z, ok);
    }
  };
  auto use = [&](int s, const double2* st, double2 (&A)[4], double2 (&B)[NT]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) A[i] = st[i * 32 + lane];
#pragma unroll
    for (int q = 0; q < NT; ++q) B[q] = st[(4 + q) * 32 + lane];
  };
  // boundary row blocks enter as -x_bnd (zeros stay zero): warp-uniform per k-step, folded into
  // the DMMA operand signs
  auto neg_of = [&](int s) { return a0 + (s >> 1) >= g.kb; };
  Acc<NT, M3> acc;
  acc_zero(acc);
#if HS_LEAN
  {
    unsigned okq = 0;
#pragma unroll
    for (int q = 0; q < NT; ++q) okq |= okr[q] ? 1u << q : 0u;
    const int cn4 = min(4, g.kb - 4 * u);
    // masked k-steps: the diagonal block rows 4u..4u+2 (M's zero blocks above the diagonal), all of
    // them when the column band is short
    const int ns = 2 * (a1 - a0);
    const int smask = mcol == 0xFu ? max(0, 2 * (4 * u + 3 - a0)) : ns;
    if (HS_KLOOP2 && !CA)
      bwd_kloop2<NT, M3>(acc, a1 - a0, ring, lane, P, g.kb, g.nrb, u, a0, cn4,
                         ZR + static_cast<size_t>(static_cast<unsigned>(row0)) * R16, XR, R16, row0, J.k, g.kp, nb, zlive,
                         okq, sidx);
    else
      bwd_kloop<NT, M3, CA>(acc, ns, ring, lane, P, g.kb, g.nrb, u, a0, cn4,
                        ZR + static_cast<size_t>(static_cast<unsigned>(row0)) * R16, XR, R16, row0, J.k, g.kp, nb, zlive,
                        okq, sidx, smask, mcol);
  }
#else
  kloop<false, NT>(acc, 2 * (a1 - a0), ring, issue, use, mask_of, neg_of);
#endif
  acc_finish(acc);
  take_ticket(a, tk, took, lane);
  prefetch_next_record(a, tk, lane);
  if (tr && lane == 0) {
    tr[2] = gtime();
    tr[6] += 2 * (a1 - a0);
  }
  const int nch = nch_bwd(g, u, J.kr);
  if (nch > 1) {
    int loc = 0;
    for (int uu = 0; uu < u; ++uu) loc += nch_bwd(g, uu, J.kr);
    const long long slot_part = static_cast<long long>(it.slot) * a.part_stride + J.part_off + loc;
    double* base = a.part + (slot_part * a.ngr + r0 / 8) * kTileDoubles;
    int* arr = a.arr + (static_cast<long long>(it.slot) * a.arr_stride + J.arr_off + u) * a.ngr + r0 / 8;
    if (!split_reduce(acc, base, static_cast<long long>(a.ngr) * kTileDoubles, nch, it.chunk, arr, lane)) return false;
  }
  if (tr && lane == 0) tr[3] = gtime();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int col = 32 * u + 8 * i + rl;
    if (col >= J.k) continue;
    double2* xo = J.x + static_cast<long long>(J.sep_off + col) * R;
#pragma unroll
    for (int q = 0; q < NT; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = r0 + 8 * q + 2 * (lane & 3) + e;
        if (r < R) __stcg(xo + r, make_double2(acc.v[i][q][0][e], acc.v[i][q][1][e]));
      }
  }
  return true;
}

__device__ __forceinline__ Geo geo_km(int k, int m) {
  Geo g;
  g.kp = (k + 7) & ~7;
  g.kb = g.kp >> 3;
  g.nrb = g.kb + ((m - k + 7) >> 3);
  g.nband = (g.nrb + 3) >> 2;
  g.ncband = (g.kb + 3) >> 2;
  return g;
}

// An item whose RHS group is exactly zero for its task: no loads, no products, no stores; only the
// arrival of a split band's chunk, so the band is still finalized (signalled) exactly once.
template <bool FWD>
__device__ __forceinline__ bool zero_item(const SolveArgs& a, const SolveJob& J, const Geo& g, const SolveItem& it, int lane) {
  int band, nch;
  if (FWD) {
    band = fwd_range(J, g, it).t;
    nch = nch_fwd(g, band, J.kc);
  } else {
    band = bwd_range(J, g, it).u;
    nch = nch_bwd(g, band, J.kr);
  }
  if (nch <= 1) return true;
  int* arr = a.arr + (static_cast<long long>(it.slot) * a.arr_stride + J.arr_off + band) * a.ngr + it.r0 / 8;
  int last = 0;
  if (lane == 0) last = atom_add_acq_rel(arr, 1) == nch - 1;
  return __shfl_sync(0xffffffffu, last, 0) != 0;
}

#ifndef HS_GROUP_SKIP
#define HS_GROUP_SKIP 1  // items of all-zero RHS groups only signal (0: every group of a nonzero task computes)
#endif
#ifndef HS_MINB_M3
#define HS_MINB_M3 3  // CTAs per SM the 3M kernels are register-budgeted for (tuning experiments)
#endif
// QUAD: the CTA dequeues four consecutive items at a time (one ticket, taken by warp 0), which the
// host lists as the RHS groups of one (band, chunk) -- padded with null items to a multiple of
// four. Its warps then stream the same factor tiles at about the same time and the A copies
// allocate in L1 (cp.async.ca), so the tiles cross the L2 -> SM path once per quad instead of once
// per RHS group (ncu, C3 64 RHS: the per-warp loads ran L2 at 74% of its throughput with DRAM at
// 22% and the DMMA pipe at 30%).
template <bool FWD, bool M3, bool QUAD>
__global__ void __launch_bounds__(kThreads, M3 ? HS_MINB_M3 : 4) solve6_kernel(SolveArgs a) {
  extern __shared__ __align__(16) double2 smem_ring[];
  __shared__ unsigned s_next[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* ring = smem_ring + warp * RingArea<FWD>::kWarp;
  int2* sidx = reinterpret_cast<int2*>(ring + RingArea<FWD>::kRing);
  // First round static: item i goes to warp i / gridDim.x of CTA i % gridDim.x, so the head
  // of the list (the critical-path fronts of the backward pass) spreads over all SMs instead
  // of packing onto the first CTAs' warps. Then dynamic tickets past the static range, each
  // taken once the current item's k-loop is done (HS_LATE_TICKET; its atomic overlaps the
  // reduction and finalize, the next item's record load overlaps the release of a finalized
  // band). A held ticket is always above its holder's current item, so the lowest current item
  // can always finish: no deadlock.
  const int nstatic = gridDim.x * (kThreads / 32);
  int cur = QUAD ? 4 * static_cast<int>(blockIdx.x) + warp : blockIdx.x + warp * gridDim.x;
  int par = 0;
  SolveItem it{};
  if (cur < a.nitems) it = a.items[cur];
  while (cur < a.nitems) {  // (QUAD: the list is a multiple of four long, so the CTA's warps leave together)
    unsigned tk = 0;
    bool took = !HS_LATE_TICKET || (QUAD && warp != 0);
    if (!HS_LATE_TICKET && (!QUAD || warp == 0) && lane == 0) tk = atomicAdd(a.queue, 1u);  // the next ticket
    bool fin = false;
    int nfin = 0;
    int* done = a.done + static_cast<long long>(it.slot) * a.nf_max;
    // the item's task and front records, loaded together (all are read-only during the launch)
    const bool null_item = QUAD && it.nzi < 0;  // padding of a quad
    const rmask nzm = null_item ? 0 : __ldg(a.nzmask + it.nzi);
    const unsigned fm = null_item ? 0u : a.tface ? __ldg(a.tface + it.nzi) : kAllLive;  // kAllLive: sweep 1 (split source)
    const SolveJob J = a.jobs[null_item ? 0 : it.job];
    if (nzm != 0) {  // else: skipped task (exactly-zero RHS), nothing depends on it
      unsigned long long* tr = a.trace ? a.trace + 8LL * cur : nullptr;
      if (tr && lane == 0) tr[0] = gtime();
      // live fronts: past sweep 1 the right-hand side is zero off the injection lines of the faces
      // that received traces; a front whose subtree holds none of them has T = z = V = 0 exactly.
      // Its forward items are skipped (nothing waits for them: a live parent ignores the child),
      // and its backward items read z = 0.
      const unsigned act = static_cast<unsigned>(J.act);
      // every front is live for the task (kAllLive) or for the 8-column groups named in bits 16-23
      // (sweep 1: the groups whose split source is nonzero in this subdomain)
      const bool all_task = (fm & kAllLive) != 0 || (fm >> 16) != 0;
      const bool live_task = all_task || (act & fm & 0xFFu) != 0;
      // backward: a front whose subtree holds no position the application reads back (PML frame
      // away from the support and the extraction lines) is skipped, and so is its subtree
      bool needed = true;
      if (!FWD && a.need) {
        const int sub = it.nzi % a.nsub;
        needed = (a.need[static_cast<long long>(sub) * a.need_words + (it.front >> 5)] >> (it.front & 31)) & 1u;
      }
      // An RHS group whose columns are all exactly zero for this task (the reference skips each of
      // those solves, src/sweeper.cpp:240-251): every reader of x masks by the task's nonzero word,
      // so the group's items neither wait nor compute, they only keep the fronts' counters whole.
      const bool gzero = HS_GROUP_SKIP && !QUAD && !a.no_group_skip &&
                         (nzm & (((it.rw >= 64 ? 0ull : 1ull << it.rw) - 1ull) << it.r0)) == 0;
      if (HS_GROUP_SKIP && !QUAD && !a.no_group_skip && !gzero && it.rw > 8) {
        // a 16-RHS item whose lower or upper 8 columns are all zero runs as an 8-RHS item on the
        // other half (every item of the task's group narrows the same way: the word is per task)
        const unsigned lo = static_cast<unsigned>(nzm >> it.r0) & 0xFFu;
        const unsigned hi = static_cast<unsigned>(nzm >> (it.r0 + 8)) & ((1u << (it.rw - 8)) - 1u);
        if (hi == 0) {
          it.rw = 8;
        } else if (lo == 0) {
          it.r0 += 8;
          it.rw -= 8;
        }
      }
      // (the item's groups after the narrowing: consistent over the items of a task's group)
      const bool all = (fm & kAllLive) != 0 ||
                       (((fm >> 16) >> (it.r0 >> 3)) & ((1u << ((it.rw + 7) >> 3)) - 1u)) != 0;
      const bool live = all || (act & fm & 0xFFu) != 0;
      // A front that is live for some group of the task but not for this item's: the item only
      // signals, like a zero group (the front's counters count the items of every group)
      if (gzero || (FWD && live_task && !live)) {  // (its own short path: the item path below stays as it is without the skip)
        if (FWD ? live_task : needed) {
          take_ticket(a, tk, took, lane);
          fin = zero_item<FWD>(a, J, geo_km(J.k, J.m), it, lane);
          nfin = fin ? 1 : 0;
        }
      } else if (FWD ? live : needed) {
        const unsigned clive = (all || ((act >> 8) & fm & 0xFFu) ? 1u : 0u) | (all || ((act >> 16) & fm & 0xFFu) ? 2u : 0u);
        const Geo g = geo_km(J.k, J.m);
        item_prefetch<FWD>(a, J, g, it, sidx, lane, !QUAD || warp == 0);  // (a quad shares the factor range)
        if (FWD) {
          if (J.child0 >= 0 && (clive & 1u)) wait_count(done + J.child0, J.tgt_c0, lane);
          if (J.child1 >= 0 && (clive & 2u)) wait_count(done + J.child1, J.tgt_c1, lane);
        } else if (J.parent >= 0) {
          wait_count(done + J.parent, J.tgt_p, lane);
        }
        cp_wait<0>();
        __syncwarp();
        if (tr && lane == 0) tr[1] = gtime();  // [0] dequeue [1] ready [2] k-loop done [3] reduced [4] done [5] sm [6] k-steps
        double2* V = a.vbuf + it.slot * a.vslot_stride;
        // the item's units: band t x RHS group r (one unit unless merged); the ticket is taken in
        // the last unit, the completed units are released together
#if HS_MERGE_UNITS
        SolveItem un = it;
        for (int t = it.idx; t < it.idx1; ++t)
          for (int r = it.r0; r < it.r1; r += J.gw) {
            const bool first = t == it.idx && r == it.r0;
            const bool lastu = t + 1 == it.idx1 && r + J.gw >= it.r1;
            un.idx = t;
            un.r0 = r;
            un.rw = min(J.gw, a.R - r);
            if (!first) {  // stage this unit's index slice / finalize data (the wait is done)
              __syncwarp();
              item_prefetch<FWD>(a, J, g, un, sidx, lane);
              cp_wait<0>();
              __syncwarp();
            }
            bool tku = lastu ? took : true;  // only the last unit takes the next ticket
            bool f;
            const SolveJob& Ju = J;
            if (FWD)
              f = un.rw > 8 ? fwd_item<2, M3, QUAD>(a, Ju, g, un, V, lane, ring, sidx, tr, clive, tk, tku)
                            : fwd_item<1, M3, QUAD>(a, Ju, g, un, V, lane, ring, sidx, tr, clive, tk, tku);
            else
              f = un.rw > 8 ? bwd_item<2, M3, QUAD>(a, Ju, g, un, lane, ring, sidx, tr, live, tk, tku)
                            : bwd_item<1, M3, QUAD>(a, Ju, g, un, lane, ring, sidx, tr, live, tk, tku);
            if (lastu) took = tku;
            nfin += f ? 1 : 0;
          }
        fin = nfin > 0;
#else
        // one unit per item (merged items measured slower; HS_MERGE_UNITS=1 compiles them in)
        if (FWD)
          fin = it.rw > 8 ? fwd_item<2, M3, QUAD>(a, J, g, it, V, lane, ring, sidx, tr, clive, tk, took)
                          : fwd_item<1, M3, QUAD>(a, J, g, it, V, lane, ring, sidx, tr, clive, tk, took);
        else
          fin = it.rw > 8 ? bwd_item<2, M3, QUAD>(a, J, g, it, lane, ring, sidx, tr, live, tk, took)
                          : bwd_item<1, M3, QUAD>(a, J, g, it, lane, ring, sidx, tr, live, tk, took);
        nfin = fin ? 1 : 0;
#endif
        if (tr && lane == 0) {
          tr[4] = gtime();
          tr[5] = smid();
        }
      }
    }
    // nothing waits for a front without dependents (forward: the root; backward: the leaves, 45% of
    // its items on C3), so its bands are not released (a release costs the warp a fence over its
    // stores); the end of the launch publishes them
    if (fin && !(FWD ? J.parent >= 0 : (J.child0 >= 0 || J.child1 >= 0))) fin = false;
    if (!took && lane == 0) tk = atomicAdd(a.queue, 1u);  // skipped item: no k-loop to overlap
    int nxt;
    if (QUAD) {  // warp 0's ticket names the CTA's next quad
      if (fin) signal(done + it.front, lane, nfin);
      fin = false;
      if (warp == 0 && lane == 0) s_next[par] = tk;
      __syncthreads();
      nxt = nstatic + 4 * static_cast<int>(s_next[par]) + warp;
      par ^= 1;
    } else {
      nxt = nstatic + static_cast<int>(__shfl_sync(0xffffffffu, tk, 0));
    }
    SolveItem nit{};
    if (nxt < a.nitems) nit = a.items[nxt];
    // the next item's first factor range toward L2 now, ahead of this item's release and the next
    // item's record loads and dependency wait (HS_NEXT_L2)
    if (HS_NEXT_L2 && lane == 0 && nxt < a.nitems && nit.pf_bytes) prefetch_l2(nit.pf, nit.pf_bytes);
    if (HS_PREFETCH_NEXT && lane == 0 && nxt < a.nitems) {  // the next item's job record and task masks
      prefetch_l1(a.jobs + nit.job);
      prefetch_l1(reinterpret_cast<const char*>(a.jobs + nit.job) + 64);
      prefetch_l1(a.nzmask + nit.nzi);
      if (a.tface) prefetch_l1(a.tface + nit.nzi);
    }
    if (fin) signal(done + it.front, lane, nfin);
    __syncwarp();  // the index slice is rewritten by the next item
    cur = nxt;
    it = nit;
  }
}


}  // namespace

int solve_fwd_chunks(int m, int k, int band, int kc) {
  const int kb = ((k + 7) & ~7) >> 3;
  return (std::min(kb, 4 * band + 4) + kc - 1) / kc;
}
int solve_bwd_chunks(int m, int k, int cband, int kr) {
  const int nrb = (((k + 7) & ~7) >> 3) + (((m - k + 7) & ~7) >> 3);
  return (nrb - 4 * cband + kr - 1) / kr;
}

template <bool FWD>
constexpr size_t ring_bytes() {
  return static_cast<size_t>(kThreads / 32) * RingArea<FWD>::kWarp * sizeof(double2);
}

template <bool FWD, bool M3, bool QUAD>
int solve_grid() {
  static PerDevice grid;  // per device: the attribute opt-in and the co-resident grid size
  return grid.get([](int dev) {
    int sms = 0, per = 0;
    HS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    HS_CUDA(cudaFuncSetAttribute(solve6_kernel<FWD, M3, QUAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, ring_bytes<FWD>()));
    HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, solve6_kernel<FWD, M3, QUAD>, kThreads, ring_bytes<FWD>()));
    return sms * std::max(per, 1);
  });
}

template <bool FWD, bool M3, bool QUAD>
void launch_solve_t(const SolveArgs& a, cudaStream_t s) {
  const int g = std::max(1, std::min(solve_grid<FWD, M3, QUAD>(), (a.nitems + kThreads / 32 - 1) / (kThreads / 32)));
  // Cooperative launch: the whole grid is co-resident, which the static first round relies on
  // (a static item of a CTA that is not yet resident could otherwise be waited for by every
  // resident warp, e.g. while another stream's kernel holds part of the GPU).
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = ring_bytes<FWD>();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HS_CUDA(cudaLaunchKernelEx(&cfg, solve6_kernel<FWD, M3, QUAD>, a));
}

void launch_solve(const SolveArgs& a, bool fwd, cudaStream_t s) {
  if (a.quad && (a.nitems & 3)) throw Error(kInternal, "quad item list not a multiple of four");
  if (a.quad) {
    if (fwd)
      a.m3 ? launch_solve_t<true, true, true>(a, s) : launch_solve_t<true, false, true>(a, s);
    else
      a.m3 ? launch_solve_t<false, true, true>(a, s) : launch_solve_t<false, false, true>(a, s);
  } else if (fwd) {
    a.m3 ? launch_solve_t<true, true, false>(a, s) : launch_solve_t<true, false, false>(a, s);
  } else {
    a.m3 ? launch_solve_t<false, true, false>(a, s) : launch_solve_t<false, false, false>(a, s);
  }
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  HS_CUDA(cudaGetLastError());
}

}  // namespace hsb
