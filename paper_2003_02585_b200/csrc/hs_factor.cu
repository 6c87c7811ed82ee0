// Blocked factorization of large fronts (m >= kFactorBigM, 3D tops of the nested-dissection
// tree) on thread-block clusters, src/direct.cpp:55-87 (eliminate_front) and :181-281
// (factor_numeric) restated as GEMM-shaped phases:
//
//   1. panels of kPB = 32 columns: every CTA factors the kPB x kPB diagonal block (redundantly,
//      in shared memory); the rows below it are solved against it, one row per thread in
//      registers, split over the cluster (L21 of the panel, and (L D) into scratch); the trailing
//      lower update F[p1:, p1:] -= L (L D)^T runs as 64x64 tiles split over the cluster.
//   2. D^-1 and unit diagonal.
//   3. M = L11^-1 by 64-row blocks I: T[I, J] = sum_{J <= K < I} L[I, K] M[K, J] (tiles split
//      over the cluster, into scratch), then M[I, J] = -L_II^-1 T[I, J]; L_II^-1 (64 x 64) is
//      formed per CTA from two 32 x 32 in-register inversions.
//   4. W = L21 M in place: row blocks of 64 rows per CTA, column tiles in increasing order (tile
//      J reads L21[R, K >= J] only, so writing W[R, J] over L21[R, J] is safe).
//   5. [M; W] into the banded 8x8-block solve layout (hs_symbolic.hpp front_block_elems).
//
// Every GEMM phase is a 64 x 64 complex tile per CTA (4 x 4 per thread, 256 threads), k-chunks
// of 32 staged in shared memory by a two-stage cp.async pipeline that also prefetches the next
// tile's first chunk. On B200 scalar DFMA and DMMA share the FP64 peak (profiles/fp64_peak.json),
// so the tile is register-blocked DFMA. Phase boundaries are cluster barriers.
#include "hs_kernels.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#include <atomic>

#include "hs_common.hpp"

namespace hsb {

extern std::atomic<long long> g_kernel_launches;

namespace {

constexpr int kT = 256;   // threads per CTA
constexpr int kPB = 32;   // panel width of the LDL^T
constexpr int kOB = 128;  // outer block: panels update only the block's columns, the rest of the
                          // front is updated once per block (a 128-deep GEMM) instead of per panel
constexpr int kTB = 64;   // GEMM tile (rows and columns)
constexpr int kKC = 32;   // GEMM k-chunk
constexpr int kSL = 65;   // shared leading dimension (double2) of staged chunks: conflict-free transposed stores
constexpr int kDL = 33;   // leading dimension of the panel diagonal block
constexpr int kStage = 2 * kKC * kSL;          // one pipeline stage: A chunk + B chunk
constexpr int kRegion0 = 2 * 64 * kSL + 32 * kDL;  // max(2 stages, L_II + X + Y of the inversion)
constexpr int kRegion1 = 2 * 32 * kDL + 2 * 32;    // panel diagonal block, e, 1/d, d
constexpr size_t kSmemBytes = static_cast<size_t>(kRegion0 + kRegion1) * sizeof(double2);
static_assert(2 * kStage <= kRegion0, "stage area");

__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }
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
__device__ __forceinline__ double2 crecip(double2 d) {  // Smith's algorithm
  if (fabs(d.x) >= fabs(d.y)) {
    const double r = d.y / d.x, den = d.x + d.y * r;
    return make_double2(1.0 / den, -r / den);
  }
  const double r = d.x / d.y, den = d.x * r + d.y;
  return make_double2(r / den, -1.0 / den);
}
__device__ __forceinline__ void cp16(double2* dst, const double2* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ long long band_base_dev(int t, int kb) {  // hs_symbolic.hpp band_base
  const int j0 = kb >> 2;
  const long long s = t <= j0 ? 2LL * t * (t + 1) : 2LL * j0 * (j0 + 1) + static_cast<long long>(t - j0) * kb;
  return s * 256;
}

// GEMM operand: element (r, kk) is p[r + kk * ld] (column-major, trans = 0) or p[r * ld + kk]
// (trans = 1); rows r >= rows read as zero.
struct Opnd {
  const double2* p;
  long long ld;
  int trans, rows;
};
struct Tile {
  Opnd a, b;
  int k0, k1;  // k range [k0, k1); an empty range is one all-zero chunk
};

__device__ __forceinline__ void stage_opnd(double2* s, const Opnd& o, int k0, int k1, int tid) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    int r, kk;
    if (!o.trans) {
      r = tid & 63;
      kk = (tid >> 6) + 4 * q;
    } else {
      kk = tid & 31;
      r = (tid >> 5) + 8 * q;
    }
    const int gk = k0 + kk;
    const bool ok = r < o.rows && gk < k1;
    const double2* src = o.p;
    if (ok) src = o.trans ? o.p + static_cast<long long>(r) * o.ld + gk : o.p + r + static_cast<long long>(gk) * o.ld;
    cp16(s + kk * kSL + r, src, ok);
  }
}

// acc[u][v] (rows tx + 16u, columns ty + 16v) += A chunk * B chunk^T (NEG: -=)
template <bool NEG = false>
__device__ __forceinline__ void mma_chunk(double2 (&acc)[4][4], const double2* sA, const double2* sB, int tx, int ty) {
#pragma unroll 4
  for (int kk = 0; kk < kKC; ++kk) {
    double2 a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = sA[kk * kSL + tx + 16 * u];
      b[u] = sB[kk * kSL + ty + 16 * u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        if (NEG)
          cfms(acc[u][v], a[u], b[v]);
        else
          cfma(acc[u][v], a[u], b[v]);
      }
  }
}

// FP64 tensor-core path of the tile GEMM (mma.sync m8n8k4 f64 = SASS DMMA): warp w owns the
// 32 x 16 complex sub-tile (rows 32 (w & 1), columns 16 (w >> 1)) as 4 x 2 blocks of 8 x 8, complex
// arithmetic as four real products (the solve kernel's mma_step); one DMMA replaces 256 DFMAs
// of issue. Accumulators cross to the (tx, ty) layout of the epilogues through shared memory.
#ifndef HS_FACTOR_DMMA
#define HS_FACTOR_DMMA 1
#endif
struct DAcc {
  double v[4][2][2][2];  // m-tile i, n-tile q, re/im, element e
};
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
template <bool NEG>
__device__ __forceinline__ void dmma_chunk(DAcc& c, const double2* sA, const double2* sB, int lane, int warp) {
  const int r0 = 32 * (warp & 1) + (lane >> 2), c0 = 16 * (warp >> 1) + (lane >> 2);
#pragma unroll 2
  for (int ks = 0; ks < kKC / 4; ++ks) {
    const int kk = 4 * ks + (lane & 3);
    double2 A[4], B[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) A[i] = sA[kk * kSL + r0 + 8 * i];
#pragma unroll
    for (int q = 0; q < 2; ++q) B[q] = sB[kk * kSL + c0 + 8 * q];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double bx = NEG ? -B[q].x : B[q].x, by = NEG ? -B[q].y : B[q].y, nby = NEG ? B[q].y : -B[q].y;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        dmma(c.v[i][q][0][0], c.v[i][q][0][1], A[i].x, bx);
        dmma(c.v[i][q][1][0], c.v[i][q][1][1], A[i].x, by);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        dmma(c.v[i][q][0][0], c.v[i][q][0][1], A[i].y, nby);
        dmma(c.v[i][q][1][0], c.v[i][q][1][1], A[i].y, bx);
      }
    }
  }
}
constexpr int kTL = 65;  // leading dimension of the 64 x 64 transposition tile (double2)
// DMMA fragments <-> the (tx, ty) layout (rows tx + 16u, columns ty + 16v) through shared memory
__device__ __forceinline__ void dacc_to_smem(const DAcc& c, double2* T, int lane, int warp) {
  const int r0 = 32 * (warp & 1) + (lane >> 2), c0 = 16 * (warp >> 1) + 2 * (lane & 3);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) T[(c0 + 8 * q + e) * kTL + r0 + 8 * i] = make_double2(c.v[i][q][0][e], c.v[i][q][1][e]);
}
__device__ __forceinline__ void smem_to_dacc(DAcc& c, const double2* T, int lane, int warp) {
  const int r0 = 32 * (warp & 1) + (lane >> 2), c0 = 16 * (warp >> 1) + 2 * (lane & 3);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double2 v = T[(c0 + 8 * q + e) * kTL + r0 + 8 * i];
        c.v[i][q][0][e] = v.x;
        c.v[i][q][1][e] = v.y;
      }
}
__device__ __forceinline__ void smem_to_acc(double2 (&acc)[4][4], const double2* T, int tx, int ty) {
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = T[(ty + 16 * v) * kTL + tx + 16 * u];
}
__device__ __forceinline__ void acc_to_smem(const double2 (&acc)[4][4], double2* T, int tx, int ty) {
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) T[(ty + 16 * v) * kTL + tx + 16 * u] = acc[u][v];
}
static_assert(64 * kTL <= kKC * kSL * 2, "transposition tile fits one stage");

// Load (STORE = false; element missing -> 0) or store the tile's elements through addr(r, c)
// (nullptr: not part of the tile) in either accumulator layout.
template <bool STORE, class Addr>
__device__ __forceinline__ void tile_rw(double2 (&acc)[4][4], int tx, int ty, Addr addr) {
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double2* p = addr(tx + 16 * u, ty + 16 * v);
      if (STORE) {
        if (p) *p = acc[u][v];
      } else {
        acc[u][v] = p ? *p : make_double2(0.0, 0.0);
      }
    }
}
template <bool STORE, class Addr>
__device__ __forceinline__ void tile_rw(DAcc& c, int r0, int c0, Addr addr) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double2* p = addr(r0 + 8 * i, c0 + 8 * q + e);
        if (STORE) {
          if (p) *p = make_double2(c.v[i][q][0][e], c.v[i][q][1][e]);
        } else {
          const double2 v = p ? *p : make_double2(0.0, 0.0);
          c.v[i][q][0][e] = v.x;
          c.v[i][q][1][e] = v.y;
        }
      }
}

struct ZeroInit {
  __device__ __forceinline__ void operator()(int, double2 (&acc)[4][4], int, int) const {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = make_double2(0.0, 0.0);
  }
};

// The CTA's sequence of cnt tiles: get(q) describes tile q, init(q, acc, tx, ty) sets its
// accumulators (zero, or C for an update C -= A B^T with NEG, so the epilogue only stores and
// C's loads overlap the tile's first chunk instead of stalling the epilogue), epi(q, acc, tx, ty)
// consumes them. Chunks stream through two cp.async stages; the next chunk (of this tile or the
// next one) is in flight while the current one is multiplied.
// FRAG (DMMA path): init / epi take the DMMA fragments directly, (q, dacc, r0, c0) with lane
// element (i, q2, e) at tile row r0 + 8 i, column c0 + 8 q2 + e -- no transposition.
template <bool NEG = false, bool FRAG = false, class Get, class Epi, class Init = ZeroInit>
__device__ __forceinline__ void gemm_tiles(int cnt, Get get, Epi epi, double2* stages, int tid, Init init = Init{}) {
  if (cnt <= 0) return;
  const int tx = tid & 15, ty = tid >> 4;
  int q = 0;
  Tile cur = get(0);
  int c = cur.k0;
  stage_opnd(stages, cur.a, c, cur.k1, tid);
  stage_opnd(stages + kKC * kSL, cur.b, c, cur.k1, tid);
  cp_commit();
#if HS_FACTOR_DMMA
  const int lane = tid & 31, warp = tid >> 5;
  const int fr0 = 32 * (warp & 1) + (lane >> 2), fc0 = 16 * (warp >> 1) + 2 * (lane & 3);
  DAcc dacc;
  double2 acc[4][4];
  if constexpr (FRAG) {
    init(0, dacc, fr0, fc0);
  } else {  // the first tile's start values through the free stage
    init(0, acc, tx, ty);
    double2* T = stages + kStage;
    acc_to_smem(acc, T, tx, ty);
    __syncthreads();
    smem_to_dacc(dacc, T, lane, warp);
    __syncthreads();
  }
#else
  double2 acc[4][4];
  init(0, acc, tx, ty);
#endif
  int sb = 0;
#pragma unroll 1
  while (true) {
    const bool last_chunk = c + kKC >= cur.k1;
    int nq = q, nc = c + kKC;
    Tile nxt = cur;
    if (last_chunk) {
      nq = q + 1;
      if (nq < cnt) {
        nxt = get(nq);
        nc = nxt.k0;
      }
    }
    const bool has_next = nq < cnt;
    if (has_next) {
      double2* s = stages + (sb ^ 1) * kStage;
      stage_opnd(s, nxt.a, nc, nxt.k1, tid);
      stage_opnd(s + kKC * kSL, nxt.b, nc, nxt.k1, tid);
    }
    cp_commit();
    cp_wait1();
    __syncthreads();
#if HS_FACTOR_DMMA
    dmma_chunk<NEG>(dacc, stages + sb * kStage, stages + sb * kStage + kKC * kSL, lane, warp);
    __syncthreads();
    if constexpr (FRAG) {
      if (last_chunk) {
        epi(q, dacc, fr0, fc0);
        if (has_next) init(nq, dacc, fr0, fc0);
      }
    } else if (last_chunk) {  // stage sb is free: the next tile's first chunk is in flight in sb ^ 1
      double2* T = stages + sb * kStage;
      dacc_to_smem(dacc, T, lane, warp);
      __syncthreads();
      smem_to_acc(acc, T, tx, ty);
      epi(q, acc, tx, ty);
      if (has_next) {
        init(nq, acc, tx, ty);
        __syncthreads();
        acc_to_smem(acc, T, tx, ty);
        __syncthreads();
        smem_to_dacc(dacc, T, lane, warp);
      }
      __syncthreads();
    }
#else
    mma_chunk<NEG>(acc, stages + sb * kStage, stages + sb * kStage + kKC * kSL, tx, ty);
    __syncthreads();
    if (last_chunk) {
      epi(q, acc, tx, ty);
      if (has_next) init(nq, acc, tx, ty);
    }
#endif
    if (!has_next) break;
    q = nq;
    c = nc;
    cur = nxt;
    sb ^= 1;
  }
}

// X = L^-1 for the unit lower 64 x 64 block L_II = F[I0 + r, I0 + c] (bs valid rows, identity
// padding), written column-major to out (64 x 64). Diagonal 32-blocks by warps 0 / 1 in registers
// (lane = column), the off-diagonal block as -B^-1 (C A^-1).
__device__ void invert_unit_lower64(const double2* F, long long m, int I0, int bs, double2* sm, double2* out, int tid) {
  double2* sL = sm;             // 64 x kSL, row-major: sL[r * kSL + c]
  double2* sX = sm + 64 * kSL;  // 64 x kSL
  double2* sY = sm + 128 * kSL; // 32 x kDL
  for (int idx = tid; idx < 64 * 64; idx += kT) {
    const int r = idx & 63, c = idx >> 6;
    double2 v = czero();
    if (r > c && r < bs) v = F[static_cast<long long>(I0 + c) * m + I0 + r];
    sL[r * kSL + c] = v;
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < 2) {
    const int o = 32 * warp;
    double2 x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      double2 acc = make_double2(i == lane ? 1.0 : 0.0, 0.0);
#pragma unroll
      for (int l = 0; l < i; ++l) cfms(acc, sL[(o + i) * kSL + o + l], x[l]);
      x[i] = acc;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) sX[(o + i) * kSL + o + lane] = x[i];
  }
  __syncthreads();
  // Y = C A^-1, C = L[32:64, 0:32]
  for (int idx = tid; idx < 32 * 32; idx += kT) {
    const int i = idx >> 5, j = idx & 31;
    double2 acc = czero();
    for (int l = j; l < 32; ++l) cfma(acc, sL[(32 + i) * kSL + l], sX[l * kSL + j]);
    sY[i * kDL + j] = acc;
  }
  __syncthreads();
  // X21 = -B^-1 Y
  for (int idx = tid; idx < 32 * 32; idx += kT) {
    const int i = idx >> 5, j = idx & 31;
    double2 acc = czero();
    for (int l = 0; l <= i; ++l) cfms(acc, sX[(32 + i) * kSL + 32 + l], sY[l * kDL + j]);
    sX[(32 + i) * kSL + j] = acc;
  }
  __syncthreads();
  for (int idx = tid; idx < 64 * 64; idx += kT) {
    const int r = idx & 63, c = idx >> 6;
    double2 v = czero();
    if (r == c)
      v = make_double2(1.0, 0.0);
    else if (r > c)
      v = sX[r * kSL + c];
    out[r + 64 * c] = v;
  }
  __syncthreads();
}

template <int NC>
__global__ void __launch_bounds__(kT, 1) factor_big_kernel(FactorArgs a, long long scratch_stride) {
  extern __shared__ double2 smem[];
  double2* region0 = smem;
  double2* sD = smem + kRegion0;  // panel diagonal block (row-major, kDL)
  double2* sE = sD + 32 * kDL;    // e[jj][c] = d_c L[jj][c]
  double2* sInv = sE + 32 * kDL;  // 1 / d_c
  double2* sDd = sInv + 32;       // d_c
  const int tid = threadIdx.x;
  const int rank = static_cast<int>(blockIdx.x % NC);
  const int gtid = rank * kT + tid;
  constexpr int GT = NC * kT;
  auto sync_front = [&]() { cg::this_cluster().sync(); };
  const FactorTask task = a.tasks[blockIdx.x / NC];
  const DevSub& S = a.subs[task.sub];
  const DevClass& C = a.cls[S.cls];
  const DevFront f = C.fronts[task.front];
  const int m = f.m, k = f.k;
  double2* F = a.work + task.fbase + f.f_off;
  const long long mm = static_cast<long long>(m) * m;
  // scratch of the cluster: (L D) of the outer block (m x kOB), T (64 x k), L_II^-1 per CTA (64 x 64)
  double2* Ws = a.scratch + (blockIdx.x / NC) * scratch_stride;
  double2* Tb = Ws + static_cast<long long>(m) * kOB;
  double2* Li = Tb + static_cast<long long>(64) * k + rank * 4096;

  // ---- assembly (src/direct.cpp:219-265)
  for (long long idx = gtid; idx < mm; idx += GT) F[idx] = czero();
  sync_front();
  for (int q = gtid; q < f.orig_cnt; q += GT) {
    double2& y = F[C.orig_fpos[f.orig_off + q]];
    const double2 v = S.val[C.orig_eidx[f.orig_off + q]];
    y.x += v.x;
    y.y += v.y;
  }
  sync_front();
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
      if (i >= j) {
        double2& y = F[static_cast<long long>(cmap[j]) * m + cmap[i]];
        const double2 v = Fc[static_cast<long long>(cf.k + j) * cf.m + cf.k + i];
        y.x += v.x;
        y.y += v.y;
      }
    }
    sync_front();
  }

  // ---- 1. panel LDL^T with GEMM updates (src/direct.cpp:55-87), outer blocks of kOB columns:
  // each panel updates the rest of its outer block, each outer block the rest of the front
#pragma unroll 1
  for (int B0 = 0; B0 < k; B0 += kOB) {
  const int B1 = min(k, B0 + kOB);
  const long long ldw = m - B0;  // Ws(r, c) = (L D)[B0 + r, B0 + c]
#pragma unroll 1
  for (int p0 = B0; p0 < B1; p0 += kPB) {
    const int nbw = min(kPB, k - p0), p1 = p0 + nbw, rows2 = m - p1;
    // (a) diagonal block, every CTA
    for (int idx = tid; idx < kPB * kPB; idx += kT) {
      const int r = idx & 31, c = idx >> 5;
      sD[r * kDL + c] = (r < nbw && c <= r) ? F[static_cast<long long>(p0 + c) * m + p0 + r] : czero();
    }
    __syncthreads();
#pragma unroll 1
    for (int jj = 0; jj < nbw; ++jj) {
      const double2 d = sD[jj * kDL + jj];
      const double2 inv = crecip(d);
      if (tid > jj && tid < nbw) sD[tid * kDL + jj] = cmul(sD[tid * kDL + jj], inv);
      __syncthreads();
      const int w = nbw - jj - 1;
      for (int idx = tid; idx < w * w; idx += kT) {
        const int r = jj + 1 + idx / w, c = jj + 1 + idx % w;
        if (c <= r) cfms(sD[r * kDL + c], sD[r * kDL + jj], cmul(d, sD[c * kDL + jj]));
      }
      __syncthreads();
    }
    for (int idx = tid; idx < kPB * kPB; idx += kT) {
      const int jj = idx >> 5, c = idx & 31;
      sE[jj * kDL + c] = (jj < nbw && c < jj) ? cmul(sD[c * kDL + c], sD[jj * kDL + c]) : czero();
    }
    if (tid < kPB) {
      const double2 d = tid < nbw ? sD[tid * kDL + tid] : czero();
      sDd[tid] = d;
      sInv[tid] = tid < nbw ? crecip(d) : czero();
      if (rank == 0 && tid < nbw && hypot(d.x, d.y) < S.tol)
        atomicMin(a.err_key, (static_cast<unsigned long long>(task.sub) << 32) | static_cast<unsigned>(f.sep_off + p0 + tid));
    }
    __syncthreads();
    // (b) rows below the block: L[i, p0:p1] and (L D)[i, :] -> scratch, one row per thread, in two
    // halves of 16 columns (the first half's multipliers wait in the idle GEMM stage area)
    double2* sl = region0 + tid;
#pragma unroll 1
    for (int i = p1 + gtid; i < m; i += GT) {
      double2 x[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) x[c] = c < nbw ? F[static_cast<long long>(p0 + c) * m + i] : czero();
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const double2 l = cmul(x[c], sInv[c]);
        x[c] = l;
        sl[c * kT] = l;
#pragma unroll
        for (int jj = c + 1; jj < 16; ++jj) cfms(x[jj], l, sE[jj * kDL + c]);
      }
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < nbw) {
          F[static_cast<long long>(p0 + c) * m + i] = x[c];
          Ws[(i - B0) + static_cast<long long>(p0 - B0 + c) * ldw] = cmul(x[c], sDd[c]);
        }
      if (nbw > 16) {
#pragma unroll
        for (int c = 0; c < 16; ++c) x[c] = 16 + c < nbw ? F[static_cast<long long>(p0 + 16 + c) * m + i] : czero();
#pragma unroll 4
        for (int c = 0; c < 16; ++c) {
          const double2 l = sl[c * kT];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) cfms(x[jj], l, sE[(16 + jj) * kDL + c]);
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const double2 l = cmul(x[c], sInv[16 + c]);
          x[c] = l;
#pragma unroll
          for (int jj = c + 1; jj < 16; ++jj) cfms(x[jj], l, sE[(16 + jj) * kDL + 16 + c]);
        }
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (16 + c < nbw) {
            F[static_cast<long long>(p0 + 16 + c) * m + i] = x[c];
            Ws[(i - B0) + static_cast<long long>(p0 - B0 + 16 + c) * ldw] = cmul(x[c], sDd[16 + c]);
          }
      }
    }
    sync_front();
    // (c) diagonal block back (rank 0); update of the rest of the outer block,
    // F[p1:, p1:B1] -= L[p1:, p0:p1] (L D)[p1:B1, p0:p1]^T (lower part)
    if (rank == 0)
      for (int idx = tid; idx < kPB * kPB; idx += kT) {
        const int r = idx & 31, c = idx >> 5;
        if (r < nbw && c <= r) F[static_cast<long long>(p0 + c) * m + p0 + r] = sD[r * kDL + c];
      }
    if (p1 < B1) {
      const int ncol = B1 - p1, nti = (rows2 + kTB - 1) / kTB, ntj = (ncol + kTB - 1) / kTB;
      const int ntiles = nti * ntj;  // tiles above the diagonal (ti < tj) hold no lower entries
      const int cnt = ntiles > rank ? (ntiles - rank + NC - 1) / NC : 0;
      auto tile_of = [&](int q, int& ti, int& tj) {
        const int tp = rank + NC * q;
        ti = tp / ntj;
        tj = tp % ntj;
      };
      gemm_tiles<true, HS_FACTOR_DMMA != 0>(
          cnt,
          [&](int q) {
            int ti, tj;
            tile_of(q, ti, tj);
            Tile t;
            t.a = Opnd{F + static_cast<long long>(p0) * m + p1 + ti * kTB, m, 0, ti < tj ? 0 : min(kTB, rows2 - ti * kTB)};
            t.b = Opnd{Ws + (p1 - B0) + tj * kTB + static_cast<long long>(p0 - B0) * ldw, ldw, 0,
                       min(kTB, ncol - tj * kTB)};
            t.k0 = 0;
            t.k1 = ti < tj ? 0 : nbw;
            return t;
          },
          [&](int q, auto& acc, int tx, int ty) {  // F = acc = F - L (L D)^T, lower part
            int ti, tj;
            tile_of(q, ti, tj);
            if (ti < tj) return;
            tile_rw<true>(acc, tx, ty, [&](int r, int c) -> double2* {
              const int gi = ti * kTB + r, gj = tj * kTB + c;
              return (gj < ncol && gi < rows2 && gi >= gj) ? F + static_cast<long long>(p1 + gj) * m + p1 + gi : nullptr;
            });
          },
          region0, tid,
          [&](int q, auto& acc, int tx, int ty) {  // start from the F tile
            int ti, tj;
            tile_of(q, ti, tj);
            tile_rw<false>(acc, tx, ty, [&](int r, int c) -> double2* {
              const int gi = ti * kTB + r, gj = tj * kTB + c;
              return (ti >= tj && gj < ncol && gi < rows2 && gi >= gj) ? F + static_cast<long long>(p1 + gj) * m + p1 + gi
                                                                       : nullptr;
            });
          });
    }
    sync_front();
  }
  // (d) the rest of the front, F[B1:, B1:] -= L[B1:, B0:B1] (L D)[B1:, B0:B1]^T (lower triangle)
  if (B1 < m) {
    const int rows2 = m - B1;
    const int nt = (rows2 + kTB - 1) / kTB, ntiles = nt * (nt + 1) / 2;
    auto tile_of = [&](int q, int& ti, int& tc) {
      const int tp = rank + NC * q;
      ti = static_cast<int>((sqrt(8.0 * tp + 1.0) - 1.0) * 0.5);
      while (ti * (ti + 1) / 2 > tp) --ti;
      while ((ti + 1) * (ti + 2) / 2 <= tp) ++ti;
      tc = tp - ti * (ti + 1) / 2;
    };
    const int cnt = ntiles > rank ? (ntiles - rank + NC - 1) / NC : 0;
    gemm_tiles<true, HS_FACTOR_DMMA != 0>(
        cnt,
        [&](int q) {
          int ti, tc;
          tile_of(q, ti, tc);
          Tile t;
          t.a = Opnd{F + static_cast<long long>(B0) * m + B1 + ti * kTB, m, 0, min(kTB, rows2 - ti * kTB)};
          t.b = Opnd{Ws + (B1 - B0) + tc * kTB, ldw, 0, min(kTB, rows2 - tc * kTB)};
          t.k0 = 0;
          t.k1 = B1 - B0;
          return t;
        },
        [&](int q, auto& acc, int tx, int ty) {  // F = acc = F - L (L D)^T, lower triangle
          int ti, tc;
          tile_of(q, ti, tc);
          tile_rw<true>(acc, tx, ty, [&](int r, int c) -> double2* {
            const int gi = ti * kTB + r, gj = tc * kTB + c;
            return (gj < rows2 && gi < rows2 && gi >= gj) ? F + static_cast<long long>(B1 + gj) * m + B1 + gi : nullptr;
          });
        },
        region0, tid,
        [&](int q, auto& acc, int tx, int ty) {  // start from the F tile
          int ti, tc;
          tile_of(q, ti, tc);
          tile_rw<false>(acc, tx, ty, [&](int r, int c) -> double2* {
            const int gi = ti * kTB + r, gj = tc * kTB + c;
            return (gj < rows2 && gi < rows2 && gi >= gj) ? F + static_cast<long long>(B1 + gj) * m + B1 + gi : nullptr;
          });
        });
  }
  sync_front();
  }

  // ---- 2. D^-1 (kept per node for the solve) and unit diagonal for the inversion
  for (int j = gtid; j < k; j += GT) {
    double2& d = F[static_cast<long long>(j) * m + j];
    S.dinv[f.sep_off + j] = crecip(d);
    d = make_double2(1.0, 0.0);
  }
  sync_front();

  // ---- 3. M = L11^-1 in place, 64-row blocks
  const int nI = (k + kTB - 1) / kTB;
#pragma unroll 1
  for (int I = 0; I < nI; ++I) {
    const int I0 = I * kTB, bs = min(kTB, k - I0);
    invert_unit_lower64(F, m, I0, bs, region0, Li, tid);
    // T[I, J] = sum_{J0 <= K < I0} L[I, K] M[K, J], J < I
    const int cnt = I > rank ? (I - rank + NC - 1) / NC : 0;
    gemm_tiles(
        cnt,
        [&](int q) {
          const int J = rank + NC * q, J0 = J * kTB;
          Tile t;
          t.a = Opnd{F + I0, m, 0, bs};
          t.b = Opnd{F + static_cast<long long>(J0) * m, m, 1, kTB};
          t.k0 = J0;
          t.k1 = I0;
          return t;
        },
        [&](int q, double2(&acc)[4][4], int tx, int ty) {
          const int J0 = (rank + NC * q) * kTB;
#pragma unroll
          for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int u = 0; u < 4; ++u) Tb[tx + 16 * u + static_cast<long long>(J0 + ty + 16 * v) * kTB] = acc[u][v];
        },
        region0, tid);
    sync_front();
    // M[I, J] = -L_II^-1 T[I, J]; M_II = L_II^-1 (rank 0)
    if (rank == 0)
      for (int idx = tid; idx < kTB * kTB; idx += kT) {
        const int r = idx & 63, c = idx >> 6;
        if (r > c && r < bs) F[static_cast<long long>(I0 + c) * m + I0 + r] = Li[r + 64 * c];
      }
    gemm_tiles(
        cnt,
        [&](int q) {
          const int J0 = (rank + NC * q) * kTB;
          Tile t;
          t.a = Opnd{Li, kTB, 0, bs};
          t.b = Opnd{Tb + static_cast<long long>(J0) * kTB, kTB, 1, kTB};
          t.k0 = 0;
          t.k1 = bs;
          return t;
        },
        [&](int q, double2(&acc)[4][4], int tx, int ty) {
          const int J0 = (rank + NC * q) * kTB;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            double2* col = F + static_cast<long long>(J0 + ty + 16 * v) * m + I0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = tx + 16 * u;
              if (i < bs) col[i] = make_double2(-acc[u][v].x, -acc[u][v].y);
            }
          }
        },
        region0, tid);
    sync_front();
  }

  // ---- 4. W = L21 M in place, row blocks of 64 per CTA, column tiles in increasing order
  if (m > k) {
    const int nR = (m - k + kTB - 1) / kTB, nJ = nI;
    const int myR = nR > rank ? (nR - rank + NC - 1) / NC : 0;
    gemm_tiles(
        myR * nJ,
        [&](int q) {
          const int r0 = k + (rank + NC * (q / nJ)) * kTB, J0 = (q % nJ) * kTB;
          Tile t;
          t.a = Opnd{F + r0, m, 0, min(kTB, m - r0)};
          t.b = Opnd{F + static_cast<long long>(J0) * m, m, 1, min(kTB, k - J0)};
          t.k0 = J0;
          t.k1 = k;
          return t;
        },
        [&](int q, double2(&acc)[4][4], int tx, int ty) {
          const int r0 = k + (rank + NC * (q / nJ)) * kTB, J0 = (q % nJ) * kTB;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int j = J0 + ty + 16 * v;
            if (j >= k) continue;
            double2* col = F + static_cast<long long>(j) * m + r0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = tx + 16 * u;
              if (r0 + i < m) col[i] = acc[u][v];
            }
          }
        },
        region0, tid);
  }
  sync_front();

  // ---- 5. [M; W] in the solve layout (as factor_level_kernel)
  {
    const int kp = (k + 7) & ~7, kb = kp >> 3, nrb = kb + ((m - k + 7) >> 3), nband = (nrb + 3) >> 2;
    auto val = [&](int pr, int pc) {
      if (pc >= k) return czero();
      if (pr < k) {
        if (pr > pc) return F[static_cast<long long>(pc) * m + pr];
        return pr == pc ? make_double2(1.0, 0.0) : czero();
      }
      const int row = k + pr - kp;
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

}  // namespace

long long factor_big_scratch(int max_m) {  // per cluster, double2 entries
  return static_cast<long long>(max_m) * kOB + static_cast<long long>(64) * max_m + static_cast<long long>(kFactorCluster) * 4096;
}

void launch_factor_big(const FactorArgs& a, int max_m, cudaStream_t s) {
  static PerDevice configured;
  configured.get([](int) {
    HS_CUDA(cudaFuncSetAttribute(factor_big_kernel<kFactorCluster>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kSmemBytes)));
    return 1;
  });
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(a.ntasks) * kFactorCluster);
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kFactorCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HS_CUDA(cudaLaunchKernelEx(&cfg, factor_big_kernel<kFactorCluster>, a, factor_big_scratch(max_m)));
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  HS_CUDA(cudaGetLastError());
}

}  // namespace hsb
