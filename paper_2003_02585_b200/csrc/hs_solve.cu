// Multifrontal forward / backward solves of the helmsweep hot path on sm_100a
// (Factorization::solve_inplace, /root/reference/proj/src/direct.cpp:290-325), batched over
// every subdomain of a sweep step group and 16 right-hand sides per task.
//
// Partitioned inverse: the factorization stores, per front, M = L11^-1 (unit lower) and
// W = L21 M instead of L11 / L21 (hs_kernels.cu). The reference's per-front operations
//   forward   t = L11^-1 x[sep]; x[bnd] -= L21 t          (direct.cpp:296-307)
//   backward  x[sep] = L11^-T (x[sep] - L21^T x[bnd])     (direct.cpp:311-324)
// become dense products with no serial dependency inside a front:
//   forward   [x_sep; u] = [M; W] x_sep,  x[sep] = D^-1 x_sep,  V = (children's bnd) - u
//   backward  x_sep = [M; W]^T [z_sep; -x_bnd]
//
// One persistent launch per pass and task class. Tasks are either a whole low subtree
// ("bundle", processed in postorder by one CTA) or one upper front; they are dequeued in
// topological order and synchronise through per-(front, RHS group) completion epochs
// (release/acquire at gpu scope): deadlock-free and deterministic (fixed reduction orders).
//
// CTA = 8 consumer warps + 1 producer warp. The producer streams the task's factor chunks
// (<= 32 rows x 32 columns, <= 16 KB) into a 4-slot shared-memory ring with cp.async.bulk
// (TMA bulk copies) completing on full/empty mbarriers; consumers never issue factor loads.
// Chunks are column-major with an XOR-8 row swizzle, so both the forward pattern (lanes =
// rows) and the backward pattern (lanes = columns) are free of bank conflicts. Consumer warp
// pairs ("groups") own disjoint outputs: row blocks in the forward, column panels in the
// backward, each with 8 RHS per thread.
#include <algorithm>
#include <atomic>
#include <cstdint>

#include "hs_common.hpp"
#include "hs_kernels.cuh"

namespace hsb {

extern std::atomic<long long> g_kernel_launches;

namespace {

constexpr int kCW = 8;              // consumer warps
constexpr int kCT = kCW * 32;       // consumer threads
constexpr int kBlock = kCT + 32;    // + producer warp
constexpr int kRG = 16;             // RHS per task
constexpr int kTP = kRG + 1;        // t row pitch
constexpr int kS = 4;               // ring slots
constexpr int kChunk = 1024;        // elements per chunk slot (32 x 32)

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
__device__ __forceinline__ int swz(int il, int j) { return (il & ~7) | ((il ^ j) & 7); }

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(kCT) : "memory"); }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct Ring {
  double2* slots;
  uint64_t* full;
  uint64_t* empty;
  volatile unsigned* issued;  // chunks issued so far (monotonic, written by the producer)
};

// Wait until chunk qq has landed. A group skips the chunks other groups own, so it may reach
// qq while its slot still holds qq-8: waiting on the full barrier's parity alone would alias
// that older phase. Observing `issued > qq` first (qq is issued only after qq-4 is released)
// keeps the waiter at most one phase ahead, which makes the parity wait exact.
__device__ __forceinline__ const double2* await_chunk(const Ring& rg, unsigned qq) {
  while (*rg.issued <= qq) {
  }
  const int s = qq % kS;
  mbar_wait(&rg.full[s], (qq / kS) & 1u);
  return rg.slots + s * kChunk;
}

// Chunk geometry of a front's [M; W] stream (hs_kernels.cu factor output): chunk (rb, J)
// for J <= min(rb, np-1), rb-major, rows padded to 8, rc(rb) rows per row block.
struct FrontGeom {
  int m_pad, nrb, np;
  __device__ explicit FrontGeom(const DevFront& f)
      : m_pad((f.m + 7) & ~7), nrb((((f.m + 7) & ~7) + 31) >> 5), np((f.k + 31) >> 5) {}
  __device__ int rc(int rb) const { return min(32, m_pad - 32 * rb); }
  __device__ int nj(int rb) const { return min(rb, np - 1) + 1; }
  // element offset of chunk (rb, J); every row block before rb is full (32 rows)
  __device__ long long off(int rb, int J) const {
    const long long pre = rb <= np ? static_cast<long long>(rb) * (rb + 1) / 2
                                   : static_cast<long long>(np) * (np + 1) / 2 + static_cast<long long>(rb - np) * np;
    return pre * 1024 + static_cast<long long>(J) * rc(rb) * 32;
  }
  __device__ int chunks() const {
    int c = 0;
    for (int rb = 0; rb < nrb; ++rb) c += nj(rb);
    return c;
  }
};

// Stream order. Forward: rb-major (storage order); group g owns row blocks rb % 4 == g.
// Backward: panel quads; inside quad p all row blocks rb >= 4p, J in the quad, J <= rb;
// group g owns panel J % 4 == g.
template <bool FWD, class Fn>
__device__ __forceinline__ void for_each_chunk(const FrontGeom& G, Fn&& fn) {
  if (FWD) {
    for (int rb = 0; rb < G.nrb; ++rb)
      for (int J = 0; J < G.nj(rb); ++J) fn(rb, J);
  } else {
    for (int p = 0; 4 * p < G.np; ++p)
      for (int rb = 4 * p; rb < G.nrb; ++rb)
        for (int J = 4 * p; J < min(4 * p + 4, G.nj(rb)); ++J) fn(rb, J);
  }
}

// Producer: stream every chunk of the task in consumption order.
template <bool FWD>
__device__ void produce(const Ring& rg, const DevClass& C, const DevSub& S, const SolveTask& task, unsigned& q) {
  const int nfr = task.f1 - task.f0 + 1;
  for (int fi = 0; fi < nfr; ++fi) {
    const int f = FWD ? task.f0 + fi : task.f1 - fi;
    const DevFront fr = C.fronts[f];
    const FrontGeom G(fr);
    const double2* base = S.factor + fr.fac_off;
    for_each_chunk<FWD>(G, [&](int rb, int J) {
      const unsigned bytes = static_cast<unsigned>(G.rc(rb)) * 32u * 16u;
      const int s = q % kS;
      const unsigned ph = (q / kS) & 1u;
      mbar_wait(&rg.empty[s], ph ^ 1u);
      mbar_expect_tx(&rg.full[s], bytes);
      bulk_g2s(rg.slots + s * kChunk, base + G.off(rb, J), bytes, &rg.full[s]);
      ++q;
      *rg.issued = q;
    });
  }
}

template <bool FWD>
__device__ void consume(const SolveArgs& a, const Ring& rg, const DevClass& C, const DevSub& S, const SolveTask& task,
                        int r0, unsigned& q, double2* t) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = warp >> 1, h = warp & 1;
  const int R = a.R;
  double2* V = a.vbuf + task.slot * a.vslot_stride;
  const int nfr = task.f1 - task.f0 + 1;
  for (int fi = 0; fi < nfr; ++fi) {
    const int f = FWD ? task.f0 + fi : task.f1 - fi;
    const DevFront fr = C.fronts[f];
    const FrontGeom G(fr);
    const int k = fr.k, m = fr.m;
    const int rows = max(G.m_pad, 32 * G.np);
    // gather: forward t = [x[sep]; 0] (+ children below); backward t = [z_sep; -x_bnd]
    for (int idx = tid; idx < rows * kRG; idx += kCT) {
      const int e = idx >> 4, r = idx & 15;
      double2 v = czero();
      if (r0 + r < R && e < m) {
        if (e < k) {
          v = __ldcg(&S.x[static_cast<long long>(fr.sep_off + e) * R + r0 + r]);
        } else if (!FWD) {
          v = __ldcg(&S.x[static_cast<long long>(C.bnd_elim[fr.bnd_off + e - k]) * R + r0 + r]);
          v.x = -v.x;
          v.y = -v.y;
        }
      }
      t[e * kTP + r] = v;
    }
    cbar();
    if (FWD) {  // extend-add of the children's update vectors, child0 then child1
#pragma unroll 1
      for (int cq = 0; cq < 2; ++cq) {
        const int ch = cq ? fr.child1 : fr.child0;
        if (ch < 0) continue;
        const DevFront cf = C.fronts[ch];
        const int cb = cf.m - cf.k;
        const int* cmap = C.child_map + (cq ? fr.cmap1 : fr.cmap0);
        for (int idx = tid; idx < cb * kRG; idx += kCT) {
          const int i = idx >> 4, r = idx & 15;
          if (r0 + r < R) {
            const double2 v = __ldcg(&V[(cf.v_off + i) * R + r0 + r]);
            double2& y = t[cmap[i] * kTP + r];
            y.x += v.x;
            y.y += v.y;
          }
        }
        cbar();
      }
    }
    double2 acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = czero();
    unsigned qq = q;  // every consumer walks the whole stream to keep the ring position
    if (FWD) {
      // out[rows of rb] = sum_J chunk(rb, J) t[J]; thread = row (lane), 8 RHS per thread
      for (int rb = 0; rb < G.nrb; ++rb) {
        const int nj = G.nj(rb), rc = G.rc(rb);
        if ((rb & 3) != g) {
          qq += nj;
          continue;
        }
        for (int J = 0; J < nj; ++J, ++qq) {
          const int s = qq % kS;
          const double2* ch = await_chunk(rg, qq);
          if (lane < rc) {
            const double2* tb = t + (32 * J) * kTP + 8 * h;
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
              const double2 L = ch[j * rc + swz(lane, j)];
              const double2* tj = tb + j * kTP;
#pragma unroll
              for (int r = 0; r < 8; ++r) cfma(acc[r], L, tj[r]);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&rg.empty[s], 4);
        }
        const int row = 32 * rb + lane;
        if (lane < rc && row < m) {
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            if (r0 + 8 * h + r >= R) continue;
            if (row < k) {  // x[sep] = D^-1 M x_sep (src/direct.cpp:303-309)
              const long long pos = fr.sep_off + row;
              __stcg(&S.x[pos * R + r0 + 8 * h + r], cmul(acc[r], S.dinv[pos]));
            } else {        // V = children's bnd updates - W x_sep (x[bnd] -= L21 t, :306)
              const double2 tin = t[row * kTP + 8 * h + r];
              __stcg(&V[(fr.v_off + row - k) * R + r0 + 8 * h + r],
                     make_double2(tin.x - acc[r].x, tin.y - acc[r].y));
            }
          }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[r] = czero();
      }
    } else {
      // x_sep[J] = sum_rb chunk(rb, J)^T [z_sep; -x_bnd][rb]; lane = column, 8 RHS per warp
      for (int p = 0; 4 * p < G.np; ++p) {
        for (int rb = 4 * p; rb < G.nrb; ++rb) {
          const int jend = min(4 * p + 4, G.nj(rb)), rc = G.rc(rb);
          for (int J = 4 * p; J < jend; ++J, ++qq) {
            if ((J & 3) != g) continue;
            const int s = qq % kS;
            const double2* ch = await_chunk(rg, qq);
            const int il_hi = min(rc, m - 32 * rb);
#pragma unroll 2
            for (int il = 0; il < il_hi; ++il) {
              const double2 L = ch[lane * rc + swz(il, lane)];
              const double2* tr = t + (32 * rb + il) * kTP + 8 * h;
#pragma unroll
              for (int r = 0; r < 8; ++r) cfma(acc[r], L, tr[r]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&rg.empty[s], 4);
          }
        }
        const int J = 4 * p + g;
        const int col = 32 * J + lane;
        if (J < G.np && col < k) {
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (r0 + 8 * h + r < R)
              __stcg(&S.x[static_cast<long long>(fr.sep_off + col) * R + r0 + 8 * h + r], acc[r]);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[r] = czero();
      }
    }
    q += G.chunks();
    cbar();
  }
}

template <bool FWD>
__global__ void __launch_bounds__(kBlock, 2) solve3_kernel(SolveArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bar_full[kS], bar_empty[kS];
  __shared__ int s_task;
  __shared__ unsigned s_issued;
  double2* ring = reinterpret_cast<double2*>(smraw);
  double2* t = ring + kS * kChunk;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_issued = 0;
    for (int s = 0; s < kS; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const Ring rg{ring, bar_full, bar_empty, &s_issued};
  const unsigned epoch = *a.epoch_base + a.epoch_off;
  const int total = a.ntasks * a.n_rg;
  unsigned q = 0;  // ring position (identical sequence in producer and consumers)
  const bool producer = tid >= kCT;
  for (;;) {
    if (tid == 0) s_task = static_cast<int>(atomicAdd(a.queue, 1u));
    __syncthreads();
    const int tk = s_task;
    __syncthreads();
    if (tk >= total) break;
    const SolveTask task = a.tasks[tk / a.n_rg];
    const int rgi = tk % a.n_rg;
    if (a.nzmask[task.sub] == 0) continue;  // skipped subdomain: nothing depends on it
    const DevSub& S = a.subs[task.sub];
    const DevClass& C = a.cls[S.cls];
    if (producer) {
      if (tid == kCT) produce<FWD>(rg, C, S, task, q);
      __syncwarp();  // reconverge the producer warp before the next CTA barrier
      continue;
    }
    unsigned* fl = a.flags + static_cast<long long>(task.sub) * a.nf_max * a.n_rg + rgi;
    if (tid == 0) {
      if (FWD) {
        for (int f = task.f0; f <= task.f1; ++f) {
          const DevFront fr = C.fronts[f];
          if (fr.child0 >= 0 && fr.child0 < task.f0)
            while (ld_acquire(fl + static_cast<long long>(fr.child0) * a.n_rg) != epoch) __nanosleep(32);
          if (fr.child1 >= 0 && fr.child1 < task.f0)
            while (ld_acquire(fl + static_cast<long long>(fr.child1) * a.n_rg) != epoch) __nanosleep(32);
        }
      } else {
        const int p = C.fronts[task.f1].parent;
        if (p >= 0)
          while (ld_acquire(fl + static_cast<long long>(p) * a.n_rg) != epoch) __nanosleep(32);
      }
      __threadfence();
    }
    __syncwarp();
    cbar();
    consume<FWD>(a, rg, C, S, task, rgi * kRG, q, t);
    if (tid == 0) {
      __threadfence();
      st_release(fl + static_cast<long long>(task.f1) * a.n_rg, epoch);
    }
  }
}

int g_sms = 0;

}  // namespace

size_t solve_smem_bytes(int max_rows, bool) {
  return (static_cast<size_t>(kS) * kChunk + static_cast<size_t>(max_rows) * kTP) * sizeof(double2);
}

int solve_grid(size_t smem) {
  if (!g_sms) {
    int dev = 0;
    HS_CUDA(cudaGetDevice(&dev));
    HS_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  // resident CTAs per SM allowed by shared memory (228 KB per SM, 1 KB reserved per CTA)
  const int per = std::max(1, std::min(2, static_cast<int>((228 * 1024) / (smem + 2048))));
  return g_sms * per;
}

int solve_rhs_group() { return kRG; }

void launch_solve(const SolveArgs& a, bool fwd, int grid, size_t smem, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    HS_CUDA(cudaFuncSetAttribute(solve3_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
    HS_CUDA(cudaFuncSetAttribute(solve3_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
    configured = true;
  }
  if (smem > 224 * 1024)
    throw Error(kInternal, "solve: front too large for the shared-memory staging (" + std::to_string(smem) + " B)");
  if (fwd)
    solve3_kernel<true><<<grid, kBlock, smem, s>>>(a);
  else
    solve3_kernel<false><<<grid, kBlock, smem, s>>>(a);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  HS_CUDA(cudaGetLastError());
}

}  // namespace hsb
