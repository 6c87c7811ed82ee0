// Host orchestration of the helmsweep B200 hot path and the C-ABI of
// include/helmsweep_b200.h.
//
//   Engine      a set of factorized subdomain operators resident on one device: symbolic
//               classes, factors, dinv, solve vectors, dataflow task lists.
//   DdmSolver   the reference's DdmSolver (src/sweeper.cpp:133-334) on top of an Engine:
//               setup on the host, factorization, then every sweep step on the device.
//   GMRES       right-preconditioned full GMRES (src/krylov.cpp:17-123), one Krylov
//               process per RHS with device-resident basis and deterministic reductions.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

#include "helmsweep_b200.h"
#include "hs_kernels.cuh"
#include "hs_assemble.cuh"
#include "hs_nccl.hpp"
#include "hs_partition.hpp"
#include "hs_symbolic.hpp"

namespace hsb {

extern std::atomic<long long> g_kernel_launches;

namespace {

thread_local std::string g_last_error;

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count == 0) return;
    HS_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    alloc(std::max<size_t>(v.size(), 1));
    if (!v.empty()) HS_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void zero(cudaStream_t s) {
    if (p) HS_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
};

// Host-side setup work split over the host cores (static partition; each index is independent).
template <class F>
void parallel_for(long long n, F&& fn) {
  const int nt = static_cast<int>(std::max(1u, std::min(std::thread::hardware_concurrency(), 64u)));
  if (n < 2 || nt == 1) {
    for (long long i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex mu;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      try {
        for (long long i = t; i < n; i += nt) fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

struct ClassDev {
  std::unique_ptr<SymbolicClass> sym;
  DBuf<DevFront> fronts;
  DBuf<int> bnd_elim, child_map, orig_fpos, orig_eidx, elim_of_local, local_of_elim;
  DBuf<int2> pmap;
  std::vector<DevFront> h_fronts;
  std::vector<int> fkc, fkr;   // per front split-K chunk (column blocks / block rows)
  std::vector<int> fgw;        // per front RHS group width (8 on the critical path, else 16)
  std::vector<unsigned> fbits; // per front: faces whose injection lines lie in its subtree
  std::vector<int> front_of_pos;  // elimination position -> front whose separator holds it
  std::vector<int> ext_pos;       // elimination positions of every trace-extraction line
  DBuf<int> ext_u0[kMaxDirs], ext_um1[kMaxDirs], inj_p0[kMaxDirs], inj_pm[kMaxDirs];
  DBuf<unsigned char> on_line;
  DBuf<std::int64_t> csr_rp, csr_col;  // CSR structure on the device (device subdomain assembly)
  std::vector<int> level_start_down;
  DevClass dev{};
};

struct Engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  int dim = 2;
  std::vector<std::unique_ptr<ClassDev>> classes;
  std::vector<int> sub_cls;
  std::vector<DevSub> h_subs;
  DBuf<DevClass> d_cls;
  DBuf<DevSub> d_subs;
  DBuf<double2> factor, dinv, val;
  std::vector<long long> fac_base, n_base;
  std::vector<double> tol;
  double factor_gpu_seconds = 0.0;
  int nf_max = 0, max_m = 0;
  long long v_total_max = 0, n_max = 0;
  // solve state
  int R = 0, nslots = 0, ngr = 1;
  int kc = 4, kr = 4;          // split-K chunks of the top-of-tree fronts (column blocks / block rows)
  int split_depth = 7;         // fronts at depth < split_depth are split; the others run whole (swept: C2 12.9 / 12.7 / 12.4 / 12.3 / 12.55 / 16.1 ms at 4 / 5 / 6 / 7 / 8 / 10)
  int crit_gw = 8;             // RHS per item of the split (critical-path) fronts
  int max_chunks = 16;         // target split-K chunks per band (HS_MAX_CHUNKS); chunks stay <= 16 blocks
  long long arr_total = 0, part_total = 0;     // per slot
  DBuf<double2> x, x1, rb, vbuf;
  DBuf<double> part;
  DBuf<int> cnt;
  std::vector<int> job_base;   // per subdomain: first (subdomain, front) job of x buffer 0
  int njobs = 0, nbuf = 1;     // jobs per x buffer; x buffers (sweeps in flight)
  long long xstride = 0;       // elements between x buffers
  long long slot_stride = 0;   // elements between per-slot right-hand side / z buffers
  DBuf<SolveJob> jobs;

  ~Engine() {
    if (stream) cudaStreamDestroy(stream);
  }

  void init(int dev, int d) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw Error(kCuda, "no CUDA device available (helmsweep_b200 has no CPU fallback)");
    if (dev < 0 || dev >= count) throw Error(kConfig, "device index out of range");
    device = dev;
    dim = d;
    HS_CUDA(cudaSetDevice(device));
    HS_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  }

  int add_class(std::unique_ptr<SymbolicClass> sc) {
    auto cd = std::make_unique<ClassDev>();
    cd->sym = std::move(sc);
    classes.push_back(std::move(cd));
    return static_cast<int>(classes.size()) - 1;
  }

  // Line tables of one class (elimination positions of trace lines), see DevClass.
  void build_lines(ClassDev& cd, int pad) {
    const SymbolicClass& c = *cd.sym;
    GridRange loc;
    loc.dim = c.dim;
    for (int a = 0; a < c.dim; ++a) {
      loc.lo[a] = 0;
      loc.hi[a] = c.size[a] - 1;
    }
    auto on_shell = [&](const Vec3i& p) {
      for (int a = 0; a < c.dim; ++a)
        if (p[a] == 0 || p[a] == c.size[a] - 1) return true;
      return false;
    };
    std::vector<unsigned char> fl(c.n, 0);
    std::vector<int>& front_of_pos = cd.front_of_pos;
    front_of_pos.clear();
    cd.ext_pos.clear();
    for (int d = 0; d < 2 * c.dim; ++d) {
      const int a = d / 2, sign = (d & 1) ? 1 : -1;
      GridRange line = loc;
      const int ext_face = sign > 0 ? c.size[a] - 1 - pad : pad;
      const int inj_face = sign > 0 ? pad : c.size[a] - 1 - pad;
      line.lo[a] = line.hi[a] = 0;
      const std::int64_t cnt = line.count();
      std::vector<int> u0(cnt), um1(cnt), p0(cnt), pm(cnt);
      for (std::int64_t i = 0; i < cnt; ++i) {
        Vec3i p = line.unlinear(i);
        p[a] = ext_face;
        u0[i] = c.elim_of_local[loc.linear(p)];
        p[a] = ext_face - sign;
        um1[i] = c.elim_of_local[loc.linear(p)];
        p[a] = inj_face;
        p0[i] = on_shell(p) ? -1 : c.elim_of_local[loc.linear(p)];
        p[a] = inj_face - sign;
        pm[i] = on_shell(p) ? -1 : c.elim_of_local[loc.linear(p)];
      }
      cd.ext_u0[d].upload(u0, stream);
      cd.ext_um1[d].upload(um1, stream);
      cd.inj_p0[d].upload(p0, stream);
      cd.inj_pm[d].upload(pm, stream);
      cd.dev.ext_u0[d] = cd.ext_u0[d].p;
      cd.dev.ext_um1[d] = cd.ext_um1[d].p;
      cd.dev.inj_p0[d] = cd.inj_p0[d].p;
      cd.dev.inj_pm[d] = cd.inj_pm[d].p;
      cd.dev.line_len[d] = static_cast<int>(cnt);
      for (std::int64_t i = 0; i < cnt; ++i) {
        if (p0[i] >= 0) fl[p0[i]] = 1;
        if (pm[i] >= 0) fl[pm[i]] = 1;
      }
      cd.ext_pos.insert(cd.ext_pos.end(), u0.begin(), u0.end());
      cd.ext_pos.insert(cd.ext_pos.end(), um1.begin(), um1.end());
      // fronts whose subtree holds an injection position of face d (the front owning the
      // position's separator slot and its ancestors)
      if (front_of_pos.empty()) {
        front_of_pos.assign(c.n, -1);
        for (size_t f = 0; f < c.fronts.size(); ++f)
          for (int q = 0; q < c.fronts[f].k; ++q) front_of_pos[c.fronts[f].sep_off + q] = static_cast<int>(f);
        cd.fbits.assign(c.fronts.size(), 0u);
      }
      for (std::int64_t i = 0; i < cnt; ++i)
        for (int pos : {p0[i], pm[i]}) {
          if (pos < 0) continue;
          for (int f = front_of_pos[pos]; f >= 0 && !(cd.fbits[f] >> d & 1u); f = c.fronts[f].parent) cd.fbits[f] |= 1u << d;
        }
    }
    cd.on_line.upload(fl, stream);
    cd.dev.on_line = cd.on_line.p;
  }

  void upload_classes(int pad) {
    std::vector<DevClass> hc;
    for (auto& cdp : classes) {
      ClassDev& cd = *cdp;
      const SymbolicClass& c = *cd.sym;
      std::vector<DevFront> fr(c.fronts.size());
      for (size_t f = 0; f < c.fronts.size(); ++f) {
        const FrontDesc& s = c.fronts[f];
        DevFront& d = fr[f];
        d.k = s.k;
        d.m = s.m;
        d.sep_off = s.sep_off;
        d.bnd_off = s.bnd_off;
        d.parent = s.parent;
        d.child0 = s.child[0];
        d.child1 = s.child[1];
        d.cmap0 = s.cmap_off[0];
        d.cmap1 = s.cmap_off[1];
        d.orig_off = s.orig_off;
        d.orig_cnt = s.orig_cnt;
        d.arr_off = 0;
        d.part_off = 0;
        d.pad_ = 0;
        d.fac_off = s.fac_off;
        d.v_off = s.v_off;
        d.f_off = s.f_off;
        d.t_off = s.t_off;
      }
      cd.fronts.upload(fr, stream);
      cd.h_fronts = fr;
      cd.bnd_elim.upload(c.bnd_elim, stream);
      cd.child_map.upload(c.child_map, stream);
      cd.orig_fpos.upload(c.orig_fpos, stream);
      cd.orig_eidx.upload(c.orig_eidx, stream);
      cd.elim_of_local.upload(c.elim_of_local, stream);
      cd.local_of_elim.upload(c.local_of_elim, stream);
      cd.dev.fronts = cd.fronts.p;
      cd.dev.bnd_elim = cd.bnd_elim.p;
      cd.dev.child_map = cd.child_map.p;
      {  // extend-add source map: parent position -> update-vector row (v_off + i) of child0 / child1
        std::vector<int2> pm(std::max<long long>(c.t_total, 1), make_int2(-1, -1));
        for (const FrontDesc& fd : c.fronts)
          for (int q = 0; q < 2; ++q) {
            const int ch = fd.child[q];
            if (ch < 0) continue;
            const int cb = c.fronts[ch].m - c.fronts[ch].k;
            for (int i = 0; i < cb; ++i) {
              int2& e = pm[fd.t_off + c.child_map[fd.cmap_off[q] + i]];
              (q ? e.y : e.x) = static_cast<int>(c.fronts[ch].v_off) + i;
            }
          }
        cd.pmap.upload(pm, stream);
        cd.dev.pmap = cd.pmap.p;
      }
      cd.dev.orig_fpos = cd.orig_fpos.p;
      cd.dev.orig_eidx = cd.orig_eidx.p;
      cd.dev.elim_of_local = cd.elim_of_local.p;
      cd.dev.local_of_elim = cd.local_of_elim.p;
      cd.dev.n = static_cast<int>(c.n);
      cd.dev.nfronts = static_cast<int>(c.fronts.size());
      for (int a = 0; a < 3; ++a) cd.dev.size[a] = c.size[a];
      if (pad >= 0) build_lines(cd, pad);
      cd.level_start_down.assign(c.max_depth + 2, 0);
      for (const auto& f : c.fronts) cd.level_start_down[f.depth + 1]++;
      for (int h = 0; h <= c.max_depth; ++h) cd.level_start_down[h + 1] += cd.level_start_down[h];
      nf_max = std::max(nf_max, static_cast<int>(c.fronts.size()));
      max_m = std::max(max_m, c.max_m);
      v_total_max = std::max(v_total_max, c.v_total);
      n_max = std::max<long long>(n_max, c.n);
      hc.push_back(cd.dev);
    }
    d_cls.upload(hc, stream);
  }

  // Factorizes every subdomain (values[sub] = CSR values in the class's CSR structure).
  // Subdomains this engine factorizes and solves (empty: all). A subdomain-partitioned solver
  // keeps only its own factors; vectors keep a slot for every subdomain.
  std::vector<char> owned;
  bool owns(int s) const { return owned.empty() || owned[s]; }

  // Factor / vector / CSR-value layout of every subdomain (values in the class's CSR structure).
  std::vector<long long> val_base;
  void layout() {
    const int nsub = static_cast<int>(sub_cls.size());
    fac_base.assign(nsub + 1, 0);
    n_base.assign(nsub + 1, 0);
    val_base.assign(nsub + 1, 0);
    for (int s = 0; s < nsub; ++s) {
      const SymbolicClass& c = *classes[sub_cls[s]]->sym;
      fac_base[s + 1] = fac_base[s] + (owns(s) ? c.fac_total : 0);
      n_base[s + 1] = n_base[s] + c.n;
      val_base[s + 1] = val_base[s] + (owns(s) ? static_cast<long long>(c.csr_col.size()) : 0);
    }
    factor.alloc(std::max<long long>(fac_base[nsub], 1));
    dinv.alloc(std::max<long long>(n_base[nsub], 1));
    val.alloc(std::max<long long>(val_base[nsub], 1));
    tol.assign(nsub, 0.0);
  }
  // Host CSR values (standalone factorization, host setup): uploaded, pivot tolerances on the host.
  void factorize(const std::vector<const CVector*>& values) {
    layout();
    const int nsub = static_cast<int>(sub_cls.size());
    parallel_for(nsub, [&](long long s) {
      if (!owns(static_cast<int>(s))) return;
      double scale = 0.0;
      for (const Complex& z : *values[s]) scale = std::max(scale, std::abs(z));
      tol[s] = 1e-14 * scale;  // src/direct.cpp:191-193
    });
    for (int s = 0; s < nsub; ++s)
      if (owns(s)) {
        if (static_cast<long long>(values[s]->size()) != val_base[s + 1] - val_base[s])
          throw Error(kInternal, "factorize: CSR values do not match the class structure");
        HS_CUDA(cudaMemcpyAsync(val.p + val_base[s], values[s]->data(), values[s]->size() * sizeof(Complex),
                                cudaMemcpyHostToDevice, stream));
      }
    factorize_numeric();
  }
  // CSR values already on the device (val, device assembly) with the pivot tolerances in tol.
  void factorize_numeric() {
    const int nsub = static_cast<int>(sub_cls.size());
    h_subs.resize(nsub);
    for (int s = 0; s < nsub; ++s) {
      DevSub& d = h_subs[s];
      d.cls = sub_cls[s];
      d.tol = tol[s];
      d.factor = factor.p + fac_base[s];
      d.dinv = dinv.p + n_base[s];
      d.val = val.p + val_base[s];
      d.x = nullptr;
    }
    d_subs.upload(h_subs, stream);

    DBuf<unsigned long long> err;
    err.alloc(1);
    HS_CUDA(cudaMemsetAsync(err.p, 0xff, sizeof(unsigned long long), stream));
    // chunk subdomains so the dense workspaces stay within a memory budget
    size_t free_b = 0, total_b = 0;
    HS_CUDA(cudaMemGetInfo(&free_b, &total_b));
    // (the dense workspaces live only during the factorization; the per-cluster scratch of the large
    // fronts and the solve buffers allocated later come out of the remainder)
    double frac = 0.6;
    if (const char* e = std::getenv("HS_FACTOR_MEM_FRAC")) frac = std::min(0.9, std::max(0.05, std::atof(e)));
    const long long budget = static_cast<long long>(free_b * frac) / sizeof(double2);
    cudaEvent_t e0, e1;
    HS_CUDA(cudaEventCreate(&e0));
    HS_CUDA(cudaEventCreate(&e1));
    HS_CUDA(cudaEventRecord(e0, stream));
    DBuf<double2> work, scratch;
    DBuf<FactorTask> d_tasks;
    int s0 = 0;
    while (s0 < nsub) {
      long long need = 0;
      int s1 = s0;
      while (s1 < nsub) {
        const long long ft = owns(s1) ? classes[sub_cls[s1]]->sym->f_total : 0;
        if (s1 > s0 && need + ft > budget) break;
        need += ft;
        ++s1;
      }
      if (static_cast<long long>(work.n) < need) work.alloc(need);
      std::vector<long long> fb(s1 - s0 + 1, 0);
      for (int s = s0; s < s1; ++s) fb[s - s0 + 1] = fb[s - s0] + (owns(s) ? classes[sub_cls[s]]->sym->f_total : 0);
      int hmax = 0;
      for (int s = s0; s < s1; ++s)
        if (owns(s)) hmax = std::max(hmax, classes[sub_cls[s]]->sym->max_height);
      // per height: small fronts (one CTA each) then large fronts (one CTA cluster each)
      std::vector<FactorTask> tasks;
      int big_m = kFactorBigM;  // HS_FACTOR_BIG_M: route smaller fronts to the cluster path (tests)
      if (const char* e = std::getenv("HS_FACTOR_BIG_M")) big_m = std::max(64, std::atoi(e));
      std::vector<int> lstart(hmax + 2, 0), lbig(hmax + 1, 0), lmaxm(hmax + 1, 0), lmaxm_big(hmax + 1, 0);
      for (int h = 0; h <= hmax; ++h) {
        lstart[h] = static_cast<int>(tasks.size());
        for (int pass = 0; pass < 2; ++pass) {
          if (pass == 1) lbig[h] = static_cast<int>(tasks.size());
          for (int s = s0; s < s1; ++s) {
            const SymbolicClass& c = *classes[sub_cls[s]]->sym;
            if (!owns(s) || h > c.max_height) continue;
            for (int q = c.level_start_up[h]; q < c.level_start_up[h + 1]; ++q) {
              const int f = c.order_up[q];
              const bool big = c.fronts[f].m >= big_m;
              if (big != (pass == 1)) continue;
              tasks.push_back(FactorTask{s, f, fb[s - s0]});
              int& mx = big ? lmaxm_big[h] : lmaxm[h];
              mx = std::max(mx, c.fronts[f].m);
            }
          }
        }
      }
      lstart[hmax + 1] = static_cast<int>(tasks.size());
      d_tasks.upload(tasks, stream);
      for (int h = 0; h <= hmax; ++h) {
        FactorArgs fa{};
        fa.cls = d_cls.p;
        fa.subs = d_subs.p;
        fa.work = work.p;
        fa.err_key = err.p;
        const int nsmall = lbig[h] - lstart[h], nbig = lstart[h + 1] - lbig[h];
        if (nsmall > 0) {
          fa.tasks = d_tasks.p + lstart[h];
          fa.ntasks = nsmall;
          if (factor_smem_bytes(lmaxm[h]) > 200 * 1024) {
            const size_t sz = static_cast<size_t>(nsmall) * 2 * lmaxm[h] * 16;
            if (scratch.n < sz) scratch.alloc(sz);
            fa.scratch = scratch.p;
          }
          launch_factor_level(fa, lmaxm[h], stream);
        }
        if (nbig > 0) {
          fa.tasks = d_tasks.p + lbig[h];
          fa.ntasks = nbig;
          static const bool old_path = std::getenv("HS_FACTOR_OLD") != nullptr;
          const size_t sz = old_path ? static_cast<size_t>(nbig) * kFactorCluster * 2 * lmaxm_big[h] * 16
                                     : static_cast<size_t>(nbig) * factor_big_scratch(lmaxm_big[h]);
          if (scratch.n < sz) scratch.alloc(sz);
          fa.scratch = scratch.p;
          if (old_path)
            launch_factor_level_cluster(fa, lmaxm_big[h], stream);
          else
            launch_factor_big(fa, lmaxm_big[h], stream);
        }
      }
      HS_CUDA(cudaStreamSynchronize(stream));
      s0 = s1;
    }
    HS_CUDA(cudaEventRecord(e1, stream));
    HS_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    HS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    factor_gpu_seconds = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    unsigned long long key = 0;
    HS_CUDA(cudaMemcpy(&key, err.p, sizeof(key), cudaMemcpyDeviceToHost));
    if (key != ~0ull) {
      const int s = static_cast<int>(key >> 32);
      const int e = static_cast<int>(key & 0xffffffffu);
      const int g = classes[sub_cls[s]]->sym->local_of_elim[e];
      Error err2(kSingular, "factorize: near-zero pivot at grid node " + std::to_string(g));
      err2.pivot_index = g;
      err2.pivot_sub = s;
      throw err2;
    }
  }

  // Solve buffers for R right-hand sides and up to `slots` concurrently solved subdomains,
  // and the split-K bookkeeping of every front (arrival counters, partial tiles).
  long long gen = 0;  // bumped whenever solve buffers are (re)allocated (captured graphs go stale)
  bool quad = false;  // item lists in null-padded quads of RHS groups (one CTA dequeue each)
  void ensure_solve(int r, int slots, int nb = 1) {
    if (r == R && slots <= nslots && nb == nbuf) return;
    ++gen;
    R = r;
    nbuf = nb;
    ngr = (R + 7) / 8;  // arrival / partial slots per (front, band): one per 8-RHS group
    // Critical-path shaping by batch width. A 32-RHS batch (C3: 31-34 tasks per macro-step) is
    // throughput-bound: fewer, wider split items win (C3 257 -> 220 ms per 64-RHS application with
    // 16-RHS groups, chunks of 8 blocks, split above depth 5). Narrower batches keep the finer split
    // of the latency-bound tree top (C2, 16 RHS: 12.2 ms with 8-RHS groups, chunks of 4, depth 7;
    // 13.0-13.3 ms with the wide settings).
    if (r >= 32) {
      kc = kr = 8;
      // (64 RHS: 128.7 ms at depth 3, 129.5 at 5, 131.2 at 7; with the zero-group skip 111.1 ms at
      // depth 1, 111.4 at 2, 112.3 at 3, 112.0 at 0; 32 RHS flat)
      split_depth = r >= 48 ? 1 : 5;
      crit_gw = 16;
    } else {
      kc = kr = 4;
      split_depth = 7;
      crit_gw = 8;
    }
    if (const char* e = std::getenv("HS_KC")) kc = std::min(16, std::max(1, std::atoi(e)));
    if (const char* e = std::getenv("HS_KR")) kr = std::min(16, std::max(4, std::atoi(e) & ~3));
    if (const char* e = std::getenv("HS_SPLIT_DEPTH")) split_depth = std::atoi(e);
    if (const char* e = std::getenv("HS_CRIT_GW")) crit_gw = std::atoi(e) <= 8 ? 8 : 16;
    int gw_bulk = 16;  // RHS per item of the unsplit fronts (HS_GW: 8 or 16)
    if (const char* e = std::getenv("HS_GW")) gw_bulk = std::atoi(e) <= 8 ? 8 : 16;
    // target chunks per band: 16 in 2D (the C2 / C3 fronts never need more), 4 in 3D, whose big
    // top fronts have bands enough (C5 application 0.456 s uncapped -> 0.399 at 16 -> 0.388 at 4);
    // chunks are never wider than 16 blocks, which bounds the 3D top fronts' count from below
    max_chunks = dim == 3 ? 4 : 16;
    if (const char* e = std::getenv("HS_MAX_CHUNKS")) max_chunks = std::max(1, std::atoi(e));
    // quads (HS_QUAD=1, off): one CTA takes the RHS groups of a band chunk together and its warps
    // share the factor tiles through L1 (hs_solve.cu QUAD). C3, 64 RHS: 198 -> 176 ms while the
    // ring's cp.async bank conflicts made L1 / L2 throughput the bound; with conflict-free ring
    // slots the per-warp dequeue runs 154 ms and quads 168 ms (CTA barrier per item)
    quad = false;
    if (const char* e = std::getenv("HS_QUAD")) quad = std::atoi(e) != 0 && r > 8;
    nslots = std::max(slots, nslots);
    arr_total = 0;
    part_total = 0;
    for (auto& cdp : classes) {
      ClassDev& cd = *cdp;
      const SymbolicClass& c = *cd.sym;
      long long arr = 0, parts = 0;
      cd.fkc.assign(c.fronts.size(), 16);
      cd.fkr.assign(c.fronts.size(), 16);
      cd.fgw.assign(c.fronts.size(), gw_bulk);
      for (size_t f = 0; f < c.fronts.size(); ++f) {
        const int m = c.fronts[f].m, k = c.fronts[f].k;
        if (c.fronts[f].depth < split_depth) {  // critical path: split long bands over many warps
          // chunk width raised so a band splits into about max_chunks chunks (the last arriver sums
          // the partials serially, and the big 3D top fronts have bands enough to fill the GPU
          // without fine splits) -- but a chunk never exceeds 16 blocks, since the solve kernel
          // stages an item's index slice in 128 entries: bands longer than 16 x max_chunks blocks
          // (C5's top fronts, k = 3249: about 26 chunks) still split into more than max_chunks
          const int kb0 = pad8(k) >> 3, nrb0 = kb0 + (pad8(m - k) >> 3);
          cd.fkc[f] = std::min(16, std::max(kc, (kb0 + max_chunks - 1) / max_chunks));
          cd.fkr[f] = std::min(16, std::max(kr, (((nrb0 + max_chunks - 1) / max_chunks) + 3) & ~3));
          cd.fgw[f] = crit_gw;
        }
        const int fkc = cd.fkc[f], fkr = cd.fkr[f];
        const int kb = pad8(k) >> 3, nrb = kb + (pad8(m - k) >> 3);
        const int nband = (nrb + 3) / 4, ncband = (kb + 3) / 4;
        cd.h_fronts[f].arr_off = static_cast<int>(arr);
        arr += std::max(nband, ncband);
        int pf = 0, pb = 0;
        bool split = false;
        for (int t = 0; t < nband; ++t) {
          const int n = solve_fwd_chunks(m, k, t, fkc);
          pf += n;
          split |= n > 1;
        }
        for (int u = 0; u < ncband; ++u) {
          const int n = solve_bwd_chunks(m, k, u, fkr);
          pb += n;
          split |= n > 1;
        }
        cd.h_fronts[f].part_off = static_cast<int>(parts);
        if (split) parts += std::max(pf, pb);
      }
      cd.fronts.upload(cd.h_fronts, stream);  // same size: device pointer unchanged
      arr_total = std::max(arr_total, arr);
      part_total = std::max(part_total, parts);
    }
    const int nsub = static_cast<int>(sub_cls.size());
    xstride = static_cast<long long>(n_base[nsub]) * R;
    x.alloc(static_cast<size_t>(xstride) * nbuf);
    // the right-hand side and z of a task live only within its macro-step: one buffer per slot
    slot_stride = n_max * R;
    if (slot_stride >= (1ll << 31)) config_error("solve: subdomain too large for a batch of this width");
    x1.alloc(static_cast<size_t>(slot_stride) * nslots);
    rb.alloc(static_cast<size_t>(slot_stride) * nslots);
    rb.zero(stream);  // right-hand sides are zero off their injection lines between uses
    vbuf.alloc(static_cast<size_t>(std::max<long long>(v_total_max, 1)) * R * nslots);
    part.alloc(static_cast<size_t>(std::max<long long>(part_total, 1)) * nslots * ngr * 1024);
    cnt.alloc(static_cast<size_t>(cnt_ints()));
    for (int s = 0; s < nsub; ++s) {
      h_subs[s].x = x.p + n_base[s] * R;
      h_subs[s].x1 = nullptr;
      h_subs[s].rb = nullptr;
    }
    d_subs.upload(h_subs, stream);
    // per (subdomain, front) job records for the solve kernels
    job_base.assign(nsub + 1, 0);
    for (int s = 0; s < nsub; ++s) job_base[s + 1] = job_base[s] + static_cast<int>(classes[sub_cls[s]]->sym->fronts.size());
    njobs = job_base[nsub];
    std::vector<SolveJob> hj(static_cast<size_t>(njobs) * nbuf);
    auto nband_of = [](const FrontDesc& d) { return ((pad8(d.k) >> 3) + (pad8(d.m - d.k) >> 3) + 3) / 4; };
    auto ncband_of = [](const FrontDesc& d) { return ((pad8(d.k) >> 3) + 3) / 4; };
    auto groups_of = [&](const ClassDev& cd, int f) { return (R + cd.fgw[f] - 1) / cd.fgw[f]; };
    for (int s = 0; s < nsub; ++s) {
      const ClassDev& cd = *classes[sub_cls[s]];
      const SymbolicClass& c = *cd.sym;
      for (size_t f = 0; f < c.fronts.size(); ++f) {
        const FrontDesc& fd = c.fronts[f];
        SolveJob& J = hj[job_base[s] + f];  // buffer 0; copies below
        J.factor = factor.p + fac_base[s] + fd.fac_off;
        J.dinv = dinv.p + n_base[s] + fd.sep_off;
        J.x = h_subs[s].x;
        J.x1 = nullptr;
        J.b = nullptr;
        J.pm = cd.pmap.p + fd.t_off;
        J.be = cd.bnd_elim.p + fd.bnd_off;
        J.k = fd.k;
        J.m = fd.m;
        J.sep_off = fd.sep_off;
        J.v_off = static_cast<int>(fd.v_off);
        J.child0 = fd.child[0];
        J.child1 = fd.child[1];
        J.tgt_c0 = fd.child[0] >= 0 ? nband_of(c.fronts[fd.child[0]]) * groups_of(cd, fd.child[0]) : 0;
        J.tgt_c1 = fd.child[1] >= 0 ? nband_of(c.fronts[fd.child[1]]) * groups_of(cd, fd.child[1]) : 0;
        J.parent = fd.parent;
        J.tgt_p = fd.parent >= 0 ? ncband_of(c.fronts[fd.parent]) * groups_of(cd, fd.parent) : 0;
        J.gw = cd.fgw[f];
        auto fb = [&](int q) { return q < 0 ? 0u : cd.fbits.empty() ? 0xFFu : cd.fbits[q]; };
        J.act = static_cast<int>(fb(static_cast<int>(f)) | fb(fd.child[0]) << 8 | fb(fd.child[1]) << 16);
        J.arr_off = cd.h_fronts[f].arr_off;
        J.part_off = cd.h_fronts[f].part_off;
        J.kc = cd.fkc[f];
        J.kr = cd.fkr[f];
      }
    }
    for (int b = 1; b < nbuf; ++b)
      for (int j = 0; j < njobs; ++j) {
        SolveJob J = hj[j];
        J.x += b * xstride;
        hj[static_cast<size_t>(b) * njobs + j] = J;
      }
    jobs.upload(hj, stream);
    jobs_h = std::move(hj);
  }
  std::vector<SolveJob> jobs_h;  // host copy of the job records (factor addresses for item prefetch)
  // counter array: [done fwd | done bwd] per slot x front, [arrivals fwd | bwd], 2 queues
  long long cnt_ints() const {
    return 2LL * nslots * nf_max + 2LL * nslots * arr_total * ngr + 2;
  }

  // Work items of the tasks of one macro-step (slot = position of the task): every front's bands
  // x split-K chunks x RHS groups (forward: row bands x column chunks; backward: column bands x
  // block-row chunks). A task is (subdomain, sweep l, x buffer).
  //
  // List order = dequeue priority. Fronts are ordered by the estimated length of the dependency
  // chain still ahead of them (forward: the front and its ancestors up to the root; backward: the
  // front and its longest descendant chain), longest first, so the fronts of the critical chain
  // are not queued behind short-chain fronts of the same level (HS_ORDER=0: the plain level order,
  // forward by height, backward by depth). A front's chain is strictly longer than that of the
  // fronts depending on it, so every dependency still sits earlier in the list (deadlock freedom
  // of the dataflow launch).
  struct TaskRef {
    int sub, l, xb;
    // static pruning of the item lists (the kernels also skip at run time, but every listed item
    // costs a ticket and its record loads): faces that can ever carry injected data in this task
    // (0x100: every front is live, sweep 1's split source) and the subdomain's bitset of fronts whose
    // x the application reads back (null: every front)
    unsigned faces = 0x100u;
    const unsigned* need = nullptr;
  };
  // estimated time of one front's items (us): wake-up + the longest item's k-loop + split-K reduce
  static double front_cost(const FrontDesc& fd, int chunk, bool fwd) {
    const int kb = pad8(fd.k) >> 3, nrb = kb + (pad8(fd.m - fd.k) >> 3);
    const int full = fwd ? kb : nrb;  // blocks of the longest band's inner dimension
    return 4.0 + 1.1 * std::min(full, chunk) + (full > chunk ? 2.5 : 0.0);
  }
  void front_priorities(const ClassDev& cd, std::vector<double>& pf, std::vector<double>& pb) const {
    const SymbolicClass& c = *cd.sym;
    const int nf = static_cast<int>(c.fronts.size());
    pf.assign(nf, 0.0);
    pb.assign(nf, 0.0);
    for (int q = nf - 1; q >= 0; --q) {  // forward: parents first (order_up reversed)
      const int f = c.order_up[q];
      const FrontDesc& fd = c.fronts[f];
      pf[f] = front_cost(fd, cd.fkc[f], true) + (fd.parent >= 0 ? pf[fd.parent] : 0.0);
    }
    for (int q = 0; q < nf; ++q) {  // backward: children first
      const int f = c.order_up[q];
      const FrontDesc& fd = c.fronts[f];
      double below = 0.0;
      for (int ch : fd.child)
        if (ch >= 0) below = std::max(below, pb[ch]);
      pb[f] = front_cost(fd, cd.fkr[f], false) + below;
    }
  }
  void build_items(const std::vector<TaskRef>& tasks, std::vector<SolveItem>& fwd, std::vector<SolveItem>& bwd) const {
    static const int mode = std::getenv("HS_ORDER") ? std::atoi(std::getenv("HS_ORDER")) : 1;
    static const bool no_prune = std::getenv("HS_NO_PRUNE") != nullptr;  // developer A/B switch
    const int nsub = static_cast<int>(sub_cls.size());
    struct Ent {
      double key;
      int g, q, f;
    };
    std::vector<Ent> ef, eb;
    std::vector<double> pf, pb;
    const ClassDev* last = nullptr;
    for (size_t g = 0; g < tasks.size(); ++g) {
      const ClassDev& cd = *classes[sub_cls[tasks[g].sub]];
      const SymbolicClass& c = *cd.sym;
      if (&cd != last) front_priorities(cd, pf, pb);
      last = &cd;
      const TaskRef& tk = tasks[g];
      const bool all_live = (tk.faces & 0x100u) != 0 || cd.fbits.empty() || no_prune;
      for (int q = 0; q < static_cast<int>(c.fronts.size()); ++q) {
        const int fu = c.order_up[q], fd = c.order_down[q];
        // level order: forward by height, backward by depth (key = -level, ties by task, order)
        // forward: a front whose subtree holds no injection line of a face that can receive data has
        // T = z = V = 0 (its live parent ignores it); backward: a front whose x is never read back
        // (nor its subtree's) is skipped -- neither is listed
        if (all_live || (cd.fbits[fu] & tk.faces & 0xFFu))
          ef.push_back(Ent{mode ? pf[fu] : -static_cast<double>(c.fronts[fu].height), static_cast<int>(g), q, fu});
        if (!tk.need || no_prune || ((tk.need[fd >> 5] >> (fd & 31)) & 1u))
          eb.push_back(Ent{mode ? pb[fd] : -static_cast<double>(c.fronts[fd].depth), static_cast<int>(g), q, fd});
      }
    }
    auto cmp = [](const Ent& x, const Ent& y) {
      if (x.key != y.key) return x.key > y.key;
      if (x.g != y.g) return x.g < y.g;
      return x.q < y.q;
    };
    std::sort(ef.begin(), ef.end(), cmp);
    std::sort(eb.begin(), eb.end(), cmp);
    // Unsplit bands of a front are merged into items of at most merge_ksteps k-steps (every RHS
    // group of a band in the same item, consecutive bands while they fit): a unit of a small front
    // is a few k-steps, so per-item costs (records, dependency wait, ticket, release) dominated.
    // (the kernel runs merged items only when built with HS_MERGE_UNITS=1)
    static const int merge_ksteps = HS_MERGE_UNITS && std::getenv("HS_MERGE") ? std::atoi(std::getenv("HS_MERGE")) : 0;
    auto emit = [&](std::vector<SolveItem>& out, int nzi, int f, int job, int slot, int gw, int nb,
                    const std::function<int(int)>& nch, const std::function<int(int)>& ksteps) {
      const int ngrp = (R + gw - 1) / gw;
      int t = 0;
      while (t < nb) {
        if (nch(t) > 1 || merge_ksteps <= 0) {  // split band (or merging off): one item per unit
          for (int ch = 0; ch < nch(t); ++ch) {
            for (int r0 = 0; r0 < R; r0 += gw)
              out.push_back(SolveItem{nzi, f, job, t, slot, r0, std::min(gw, R - r0), ch, t + 1, r0 + std::min(gw, R - r0),
                                      nullptr, 0u, 0});
            while (quad && (out.size() & 3)) {  // null items (nzi < 0) fill the chunk's last quad
              out.push_back(out.back());
              out.back().nzi = -1;
            }
          }
          ++t;
          continue;
        }
        int t1 = t, ks = 0;
        while (t1 < nb && nch(t1) == 1 && (t1 == t || ks + ksteps(t1) * ngrp <= merge_ksteps)) ks += ksteps(t1++) * ngrp;
        out.push_back(SolveItem{nzi, f, job, t, slot, 0, std::min(gw, R), 0, t1, R, nullptr, 0u, 0});
        t = t1;
      }
    };
    for (const Ent& e : ef) {
      const TaskRef& tk = tasks[e.g];
      const ClassDev& cd = *classes[sub_cls[tk.sub]];
      const FrontDesc& fd = cd.sym->fronts[e.f];
      const int f = e.f, nzi = (tk.l - 1) * nsub + tk.sub, jb = tk.xb * njobs + job_base[tk.sub];
      const int kb = pad8(fd.k) >> 3, nrb = kb + (pad8(fd.m - fd.k) >> 3), nband = (nrb + 3) / 4;
      const size_t first = fwd.size();
      emit(fwd, nzi, f, jb + f, e.g, cd.fgw[f], nband, [&](int t) { return solve_fwd_chunks(fd.m, fd.k, t, cd.fkc[f]); },
           [&](int t) { return 2 * std::min(kb, 4 * t + 4); });
      for (size_t i = first; i < fwd.size(); ++i) {  // band t, column blocks of chunk `chunk`
        SolveItem& it = fwd[i];
        const int t = it.idx, rbs = std::min(4, nrb - 4 * t), kc = cd.fkc[f];
        const int cb0 = it.chunk * kc, cb1 = std::min(std::min(kb, 4 * t + 4), cb0 + kc);
        it.pf = jobs_h[jb + f].factor + band_base(t, kb) + static_cast<long long>(cb0) * rbs * 64;
        it.pf_bytes = static_cast<unsigned>((cb1 - cb0) * rbs) * 1024u;
      }
    }
    for (const Ent& e : eb) {
      const TaskRef& tk = tasks[e.g];
      const ClassDev& cd = *classes[sub_cls[tk.sub]];
      const FrontDesc& fd = cd.sym->fronts[e.f];
      const int f = e.f, nzi = (tk.l - 1) * nsub + tk.sub, jb = tk.xb * njobs + job_base[tk.sub];
      const int kb = pad8(fd.k) >> 3, nrb = kb + (pad8(fd.m - fd.k) >> 3), ncband = (kb + 3) / 4;
      const size_t first = bwd.size();
      emit(bwd, nzi, f, jb + f, e.g, cd.fgw[f], ncband, [&](int u) { return solve_bwd_chunks(fd.m, fd.k, u, cd.fkr[f]); },
           [&](int u) { return 2 * (nrb - 4 * u); });
      for (size_t i = first; i < bwd.size(); ++i) {  // column band u: its first row band's blocks
        SolveItem& it = bwd[i];
        const int u = it.idx, a0 = 4 * u + it.chunk * cd.fkr[f], ta = a0 >> 2;
        const int rbs = std::min(4, nrb - 4 * ta), ncol = std::min(4, kb - 4 * u);
        it.pf = jobs_h[jb + f].factor + band_base(ta, kb) + static_cast<long long>(4 * u) * rbs * 64;
        it.pf_bytes = static_cast<unsigned>(ncol * rbs) * 1024u;
      }
    }
  }

  // One forward and one backward launch over the items of a step group.
  DBuf<unsigned long long> trace;
  void run_solve(const SolveItem* fwd, int nfwd, const SolveItem* bwd, int nbwd, const rmask* nzmask,
                 bool traced = false, const unsigned* tface = nullptr, const unsigned* need = nullptr,
                 int need_words = 0) {
    const long long per = static_cast<long long>(nslots) * nf_max;
    const long long arr = static_cast<long long>(nslots) * arr_total * ngr;
    HS_CUDA(cudaMemsetAsync(cnt.p, 0, cnt_ints() * sizeof(int), stream));
    SolveArgs a{};
    a.R = R;
    a.ngr = ngr;
    a.nf_max = nf_max;
    a.jobs = jobs.p;
    a.vbuf = vbuf.p;
    a.vslot_stride = v_total_max * R;
    a.part = part.p;
    a.part_stride = part_total;
    a.arr_stride = arr_total;
    a.nzmask = nzmask;
    a.tface = tface;
    // 3M products (3 CTAs per SM) unless HS_M3=0: C2 12.5 vs 12.8 ms, C5 0.384 vs 0.394 s
    static const int m3env = std::getenv("HS_M3") ? std::atoi(std::getenv("HS_M3")) : 1;
    a.m3 = m3env != 0;
    a.quad = quad ? 1 : 0;
    a.need = need;
    a.need_words = need_words;
    static const bool no_group_skip = std::getenv("HS_NO_GROUP_SKIP") != nullptr;  // developer A/B switch
    a.no_group_skip = no_group_skip ? 1 : 0;
    a.nsub = static_cast<int>(sub_cls.size());
    a.rbs = rb.p;
    a.x1s = x1.p;
    a.slot_stride = slot_stride;
    a.items = fwd;
    a.nitems = nfwd;
    a.done = cnt.p;
    a.arr = cnt.p + 2 * per;
    a.queue = reinterpret_cast<unsigned*>(cnt.p + 2 * per + 2 * arr);
    if (traced) {  // developer instrumentation (HS_TRACE): per-item timestamps of this step
      trace.alloc(static_cast<size_t>(8) * (nfwd + nbwd));
      HS_CUDA(cudaMemsetAsync(trace.p, 0, trace.n * sizeof(unsigned long long), stream));
      a.trace = trace.p;
    }
    launch_solve(a, true, stream);
    a.items = bwd;
    a.nitems = nbwd;
    a.done = cnt.p + per;
    a.arr = cnt.p + 2 * per + arr;
    a.queue = reinterpret_cast<unsigned*>(cnt.p + 2 * per + 2 * arr + 1);
    if (traced) a.trace = trace.p + 8LL * nfwd;
    launch_solve(a, false, stream);
    if (traced) {
      std::vector<unsigned long long> h(trace.n);
      std::vector<SolveItem> items(nfwd + nbwd);
      HS_CUDA(cudaMemcpyAsync(h.data(), trace.p, h.size() * 8, cudaMemcpyDeviceToHost, stream));
      HS_CUDA(cudaMemcpyAsync(items.data(), fwd, nfwd * sizeof(SolveItem), cudaMemcpyDeviceToHost, stream));
      HS_CUDA(cudaMemcpyAsync(items.data() + nfwd, bwd, nbwd * sizeof(SolveItem), cudaMemcpyDeviceToHost, stream));
      HS_CUDA(cudaStreamSynchronize(stream));
      if (FILE* fp = std::fopen(std::getenv("HS_TRACE"), "w")) {
        std::fprintf(fp, "pass,sub,front,kind,idx,chunk,r0,rw,t_deq,t_ready,t_loop,t_red,t_done,sm,nsteps,k,m\n");
        for (int i = 0; i < nfwd + nbwd; ++i) {
          const SolveItem& it = items[i];
          if (it.nzi < 0) continue;  // quad padding
          const int sub = it.nzi % static_cast<int>(sub_cls.size());
          const FrontDesc& fd = classes[sub_cls[sub]]->sym->fronts[it.front];
          const unsigned long long* q = &h[8 * i];
          std::fprintf(fp, "%d,%d,%d,%d,%d,%d,%d,%d,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%d,%d\n", i < nfwd ? 0 : 1, sub,
                       it.front, i < nfwd ? 1 : 2, it.idx, it.chunk, it.r0, it.rw, q[0], q[1], q[2], q[3], q[4], q[5],
                       q[6], fd.k, fd.m);
        }
        std::fclose(fp);
      }
    }
  }
};

// ----------------------------------------------------------------------------
// standalone factorization (hs_factor)

__global__ void gather_in_kernel(const double2* src, double2* dst, const int* local_of_elim, long long n, int R) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= n * R) return;
  const long long e = idx / R;
  const int r = static_cast<int>(idx % R);
  dst[idx] = src[static_cast<long long>(r) * n + local_of_elim[e]];
}
__global__ void scatter_out_kernel(const double2* src, double2* dst, const int* elim_of_local, long long n, int R) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= n * R) return;
  const int r = static_cast<int>(idx / n);
  const long long l = idx % n;
  dst[idx] = src[static_cast<long long>(elim_of_local[l]) * R + r];
}

}  // namespace

struct FactorHandle {
  Engine eng;
  hs_factor_stats stats{};
  std::vector<SolveItem> fwd, bwd;
  int items_R = 0;
  DBuf<SolveItem> d_fwd, d_bwd;
  DBuf<rmask> nz;
  DBuf<double2> io;
  // Factorization::solve is "reentrant; safe for concurrent calls on one factorization"
  // (include/helmsweep/direct.hpp:29). The device solve shares the engine's buffers, so
  // concurrent calls on one handle are serialised here; calls on different handles overlap.
  std::mutex mu;
};

struct DdmHandle;

}  // namespace hsb

struct hs_factor {
  hsb::FactorHandle h;
};

namespace hsb {
namespace {

template <class F>
int guarded(F&& fn, int* pivot_sub = nullptr, std::int64_t* pivot_index = nullptr) {
  try {
    fn();
    return kOk;
  } catch (const Error& e) {
    g_last_error = e.what();
    if (e.code == kSingular) {
      if (pivot_sub) *pivot_sub = e.pivot_sub;
      if (pivot_index) *pivot_index = e.pivot_index;
    }
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return kInternal;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return kInternal;
  }
}

void factor_solve_device(FactorHandle& H, int nrhs, double2* d_x, cudaStream_t user) {
  Engine& eng = H.eng;
  const SymbolicClass& c = *eng.classes[0]->sym;
  const long long n = c.n;
  for (int b0 = 0; b0 < nrhs; b0 += kMaxRhs) {
    const int R = std::min(kMaxRhs, nrhs - b0);
    eng.ensure_solve(R, 1);
    if (H.items_R != R) {  // item lists depend on the RHS grouping
      H.fwd.clear();
      H.bwd.clear();
      eng.build_items({Engine::TaskRef{0, 1, 0}}, H.fwd, H.bwd);
      H.d_fwd.upload(H.fwd, eng.stream);
      H.d_bwd.upload(H.bwd, eng.stream);
      H.items_R = R;
    }
    if (user) {
      cudaEvent_t ev;
      HS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      HS_CUDA(cudaEventRecord(ev, user));
      HS_CUDA(cudaStreamWaitEvent(eng.stream, ev, 0));
      cudaEventDestroy(ev);
    }
    double2* xb = d_x + b0 * n;
    const int threads = 256;
    const int blocks = static_cast<int>((n * R + threads - 1) / threads);
    gather_in_kernel<<<blocks, threads, 0, eng.stream>>>(xb, eng.rb.p, eng.classes[0]->local_of_elim.p, n, R);
    g_kernel_launches.fetch_add(1);
    HS_CUDA(cudaGetLastError());
    const rmask mask = R >= 64 ? ~0ull : ((1ull << R) - 1ull);
    HS_CUDA(cudaMemcpyAsync(H.nz.p, &mask, sizeof(rmask), cudaMemcpyHostToDevice, eng.stream));
    eng.run_solve(H.d_fwd.p, static_cast<int>(H.fwd.size()), H.d_bwd.p, static_cast<int>(H.bwd.size()), H.nz.p);
    scatter_out_kernel<<<blocks, threads, 0, eng.stream>>>(eng.x.p, xb, eng.classes[0]->elim_of_local.p, n, R);
    g_kernel_launches.fetch_add(1);
    HS_CUDA(cudaGetLastError());
    if (user) {
      cudaEvent_t ev;
      HS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      HS_CUDA(cudaEventRecord(ev, eng.stream));
      HS_CUDA(cudaStreamWaitEvent(user, ev, 0));
      cudaEventDestroy(ev);
    }
  }
}

}  // namespace
}  // namespace hsb

namespace hsb {
// One sparse-direct factorization on the device (the engine of factorize(), src/direct.cpp:333-348).
std::unique_ptr<hs_factor> make_factor(int dim, const GridRange& rng, std::vector<std::int64_t> rp,
                                       std::vector<std::int64_t> cl, const CVector& v, int device) {
  const auto t0 = std::chrono::steady_clock::now();
  auto f = std::make_unique<hs_factor>();
  FactorHandle& H = f->h;
  H.eng.init(device, dim);
  const std::int64_t n = rng.count(), nnz = rp[n];
  H.eng.sub_cls.push_back(H.eng.add_class(build_symbolic(dim, rng, rp, cl)));
  H.eng.upload_classes(-1);
  H.eng.factorize({&v});
  const SymbolicClass& c = *H.eng.classes[0]->sym;
  H.nz.alloc(1);
  HS_CUDA(cudaStreamSynchronize(H.eng.stream));
  H.stats.n = n;
  H.stats.matrix_nnz = nnz;
  H.stats.factor_nnz = c.factor_nnz;
  H.stats.peak_bytes = c.peak_bytes;
  H.stats.factor_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return f;
}
}  // namespace hsb

using namespace hsb;

extern "C" {

const char* hs_last_error(void) { return g_last_error.c_str(); }

int hs_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int64_t hs_kernel_launches(void) { return g_kernel_launches.load(); }

int hs_factorize(int dim, const int lo[3], const int hi[3], int64_t n, const int64_t* row_ptr,
                 const int64_t* col, const double* val, int device, hs_factor** out,
                 hs_factor_stats* stats, int64_t* pivot_index) {
  std::unique_ptr<hs_factor> f;
  int rc = guarded([&] {
    if (n <= 0) config_error("factorize: empty operator");
    if (dim != 2 && dim != 3) config_error("factorize: dim must be 2 or 3");
    GridRange rng;
    rng.dim = dim;
    for (int a = 0; a < 3; ++a) {
      rng.lo[a] = a < dim ? lo[a] : 0;
      rng.hi[a] = a < dim ? hi[a] : 0;
    }
    if (rng.count() != n) config_error("factorize: grid range does not match operator size");
    std::vector<std::int64_t> rp(row_ptr, row_ptr + n + 1), cl(col, col + row_ptr[n]);
    CVector v(reinterpret_cast<const Complex*>(val), reinterpret_cast<const Complex*>(val) + row_ptr[n]);
    f = make_factor(dim, rng, std::move(rp), std::move(cl), v, device);
    if (stats) *stats = f->h.stats;
  }, nullptr, pivot_index);
  if (rc != kOk) return rc;
  *out = f.release();
  return kOk;
}

}  // extern "C"

extern "C" int hs_factor_solve_device(hs_factor* f, int nrhs, double* d_x, void* stream) {
  return guarded([&] {
    if (!f) config_error("hs_factor_solve_device: null handle");
    if (nrhs <= 0) return;
    HS_CUDA(cudaSetDevice(f->h.eng.device));
    std::lock_guard<std::mutex> lk(f->h.mu);  // one solve at a time per factorization (shared engine buffers)
    // NULL is the legacy default stream: order the solve after the caller's work there too
    cudaStream_t user = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    factor_solve_device(f->h, nrhs, reinterpret_cast<double2*>(d_x), user);
    if (!stream) HS_CUDA(cudaStreamSynchronize(f->h.eng.stream));
  });
}

extern "C" int hs_factor_solve(hs_factor* f, int nrhs, double* x) {
  return guarded([&] {
    if (!f) config_error("hs_factor_solve: null handle");
    if (nrhs <= 0) return;
    FactorHandle& H = f->h;
    HS_CUDA(cudaSetDevice(H.eng.device));
    std::lock_guard<std::mutex> lk(H.mu);  // one solve at a time per factorization (shared engine buffers)
    const long long n = H.stats.n;
    H.io.alloc(static_cast<size_t>(n) * nrhs);
    HS_CUDA(cudaMemcpyAsync(H.io.p, x, sizeof(double2) * n * nrhs, cudaMemcpyHostToDevice, H.eng.stream));
    factor_solve_device(H, nrhs, H.io.p, nullptr);
    HS_CUDA(cudaMemcpyAsync(x, H.io.p, sizeof(double2) * n * nrhs, cudaMemcpyDeviceToHost, H.eng.stream));
    HS_CUDA(cudaStreamSynchronize(H.eng.stream));
  });
}

extern "C" int hs_factor_stats_get(const hs_factor* f, hs_factor_stats* stats) {
  if (!f || !stats) return kConfig;
  *stats = f->h.stats;
  return kOk;
}

extern "C" void hs_factor_destroy(hs_factor* f) { delete f; }

// ============================================================================
// DdmSolver

namespace hsb {
namespace {

struct SubHost {
  Vec3i sub{0, 0, 0};
  GridRange owned, range;
  Box cell;
  int cls = 0;
};


}  // namespace

struct DdmHandle {
  Engine eng;
  int dim = 2;
  PmlSpec pml;
  Medium medium;
  Box interior;
  Vec3i intervals{1, 1, 1};
  Partition part;
  Weights wts;
  LocalGrid ggrid;
  PmlCoefficients gcoeffs;
  std::vector<SubHost> subs;
  std::vector<hs_factor_stats> sub_stats;
  double factor_seconds = 0.0;
  DevGeom geom{};
  int steps = 0, ndir = 4, dirs = 4, max_group = 1;
  long long line_max = 1;
  std::vector<std::vector<int>> groups;  // [di * steps + s-1]: the reference's step groups
  std::vector<int> grp_off;
  DBuf<int> d_groups;
  // Macro-step schedule (per rounds): tasks (subdomain, sweep) levelled by their longest
  // dependency path, so sweeps overlap wherever the trace routing allows (build_schedule).
  int nbuf = 1, max_width = 1;
  std::vector<std::vector<int2>> msteps;   // per macro-step: (subdomain, sweep), ascending (sweep, id)
  std::vector<std::vector<int>> acc_after; // per macro-step: sweeps accumulated after it, ascending
  std::vector<int> mstep_of;               // [(l-1) * nsub + id] -> macro-step
  std::vector<int> sweep_first_m, mt_off, fwd_off, fwd_cnt, bwd_off, bwd_cnt;
  // streamed host transfers: stripes of the slowest axis, and per macro-step the last stripe of b
  // its sweep-1 tasks read (-1: none)
  std::vector<long long> stripe_n;  // node bounds, size nstripe + 1
  // b travels in tiles (a stripe x a segment of the fastest axis), in the order the sweep-1
  // tasks first read them: the early macro-steps wait only for their own subdomains' part of b
  struct InTile {
    long long row0, row1;  // rows of the fastest axis (gsize[0] nodes each)
    int x0, x1;            // fastest-axis columns
    int need;              // first macro-step reading it (nmacro: only the residual)
  };
  std::vector<InTile> in_tiles;  // copy order
  std::vector<int> need_tiles;   // per macro-step: leading tiles (copy order) it needs
  // the last sweep is accumulated stripe by stripe, after the macro-step that completes the
  // stripe (acc_stripe_m), so streamed transfers can copy u out while the tail still runs
  std::vector<int> acc_stripe_m;
  // final regions of u: the stripes, or (streamed, fused accumulate) the tiles of b's tiling,
  // which the last sweep's diagonal wavefront completes earlier than whole stripes, so the copy
  // of u to the host starts earlier
  struct OutRegion {
    long long row0, row1;  // rows of the fastest axis
    int x0, x1;
    int acc_m;  // macro-step after which the region is final
  };
  std::vector<OutRegion> out_stripes, out_tiles;
  const std::vector<OutRegion>& out_regions(bool streamed) const {
    static const bool stripes_only = std::getenv("HS_OUT_STRIPES") != nullptr;  // developer A/B switch
    return streamed && fuse_acc && !out_tiles.empty() && !stripes_only ? out_tiles : out_stripes;
  }
  // every sweep in its own x buffer (sweeps <= buffers): all contributions are accumulated in one
  // pass per stripe at the end (accumulate_all_kernel) instead of one pass per sweep
  bool fuse_acc = false;
  std::vector<int> sweep_end_m;  // per sweep: the macro-step its last task runs in
  static constexpr int kCopyStreams = 2;  // streamed host I/O: b in, u out
  cudaStream_t cs[kCopyStreams] = {};
  std::vector<cudaEvent_t> ev_in, ev_out;
  DBuf<int2> d_mtasks, d_prev;
  std::vector<int2> prev_h;
  DBuf<SolveItem> d_tasks;
  DBuf<int2> acc_ent;          // accumulate plan: per global node, 2^dim (position, sub, weight) entries
  // per subdomain, a bitset over fronts: the front's subtree holds a position the application
  // reads back (accumulated with a nonzero weight, or on a trace-extraction line); the backward
  // pass skips the others, whose x nobody reads (the PML frame away from the support)
  DBuf<unsigned> need;
  int need_words = 0;
  std::vector<unsigned> need_h;
  DBuf<int> split_gp;          // split-source plan per (subdomain, elimination position): global node
  DBuf<unsigned char> split_w; // and weight numerator (0: shell or outside the support)
  DBuf<double2> d_coef;
  // per (R, rounds) state
  int R = 0, nsweeps = 0, rounds = 0;
  std::vector<Vec3i> plan;
  std::vector<int> route_h;
  DBuf<double2> mbox;
  DBuf<rmask> mpres, nzmask;
  DBuf<unsigned> tface;
  DBuf<int> route;
  DBuf<double2> bN, u, io;
  DBuf<double2> uround;  // fused accumulate over several rounds: u after each round but the last
  DBuf<double> partial, norms, pnum, pden, rnum, rden;
  long long partial_stride = 0;  // elements between sweeps' partials (fused accumulate)
  std::vector<cudaEvent_t> ev;  // [0]=start, [1..nsweeps]=after sweep l's accumulate, then macro-step solve pairs
  // global operator (lazy) and its direct factorization (global_direct_solve, lazy)
  hs_factor* gfact = nullptr;
  bool gop_ready = false;
  long long g_nnz = 0;
  DBuf<std::int64_t> g_rp;
  DBuf<int> g_col;
  DBuf<double2> g_val;
  DBuf<double2> g_sten;  // the same operator in stencil form (StencilOp), for the residual kernel
  StencilOp g_sop;
  void build_stencil_op();
  // subdomain partition over ranks; world == 1: every subdomain is local
  int rank = 0, world = 1;
  std::vector<int> owner;                       // per subdomain
  hs_exchange_fn xfn = nullptr;
  hs_allreduce_fn arfn = nullptr;
  void* cuser = nullptr;
  std::vector<std::vector<int2>> msteps_own;    // per macro-step: this rank's tasks
  // ghost x positions (n_base[sub] + elimination position) per (subdomain, home rank): values of
  // the subdomain's solution that rank accumulates although another rank owns the subdomain
  std::vector<std::vector<std::vector<long long>>> ghost;
  std::vector<long long> ghost_off;             // [sub * world + rank] into d_gpos
  DBuf<long long> d_gpos;
  struct XPlan {
    std::vector<int> peers;
    std::vector<std::int64_t> soff, scnt, roff, rcnt;
    int s0 = 0, ns = 0, r0 = 0, nr = 0;         // segments in d_xseg
  };
  std::vector<XPlan> xplan;
  DBuf<XSeg> d_xseg;
  DBuf<double> xsend, xrecv, dtmp;
  DBuf<double2> ufull;
  long long x_sent = 0, x_msgs = 0;
  // the library's own NCCL communicator (hs_ddm_create_nccl): exchange and reductions issued on the
  // solver stream without caller callbacks, so partitioned applications are graph-captured too. With
  // it the partitioned machinery runs even at world 1 (every node home, no peers).
  std::unique_ptr<NcclComm> ncomm;
  bool partitioned() const { return world > 1 || ncomm != nullptr; }
  void build_xplan();
  void comm_allreduce(double* buf, long long count);
  // u summed over ranks: an owner-slab all-gather with the native NCCL transport, else an all-reduce
  void comm_gather_u(double2* buf);
  long long max_home = 0, home_cnt = 0;
  DBuf<int> d_homes;
  DBuf<double2> gsend, grecv;

  ~DdmHandle() {
    drop_graphs();
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : ev_in) cudaEventDestroy(e);
    for (auto e : ev_out) cudaEventDestroy(e);
    for (auto c : cs)
      if (c) cudaStreamDestroy(c);
    for (int q = 0; q < 2; ++q) {
      if (ev_din_free[q]) cudaEventDestroy(ev_din_free[q]);
      if (ev_dout_free[q]) cudaEventDestroy(ev_dout_free[q]);
    }
    if (gfact) hs_factor_destroy(gfact);
  }

  void build(const hs_problem& P, int device, int rank_ = 0, int world_ = 1, const int* owner_ = nullptr);
  // device subdomain setup: extended wavenumber + CSR values of every owned subdomain into eng.val,
  // pivot tolerances into eng.tol (hs_assemble.cu)
  DBuf<float> vel_dev;
  DBuf<double2> alpha_dev;
  DBuf<AsmSub> asm_subs;
  AsmMedium asm_medium();
  void assemble_device(const std::vector<PmlCoefficients>& coeffs);
  void ensure_state(int r, int nrounds);
  void ensure_state_body(int r, int nrounds);
  int nbuf_cap = HS_MAX_ACC_SWEEPS;  // x buffers at most (4 after an allocation failure)
  void build_schedule(int r);
  void build_items();
  void ensure_gop();
  // Streamed host transfers (solve_streamed): per stripe, the event of its H2D copy into the
  // RHS-major staging buffer din; run() transposes each stripe into bN on the compute stream when
  // a macro-step first needs it, and each final stripe of u out to dout. Every kernel stays on the
  // compute stream: nothing runs beside the dataflow solve kernels, whose items assume the
  // whole grid is resident.
  struct StreamIO {
    const cudaEvent_t* copied;
    const double2* din;
    double2* dout;
  };
  void run(int nrounds, bool track, bool timed, const StreamIO* io = nullptr);
  void run_body(int nrounds, bool track, bool timed, const StreamIO* io);
  // One application from device-resident b (no streamed host I/O, one process) is a fixed
  // sequence of ~8 launches per macro-step; it is captured once per (rounds, track, timed) and
  // state generation into a CUDA graph and replayed (HS_GRAPH=0 launches it stream by stream).
  struct AppGraph {
    int rounds;
    bool track, timed;
    long long gen;
    long long launches;
    cudaGraphExec_t exec;
  };
  std::vector<AppGraph> graphs;
  // graphs on unless HS_GRAPH=0; a capture this handle cannot do turns them off for this handle only
  bool use_graph = !(std::getenv("HS_GRAPH") && std::atoi(std::getenv("HS_GRAPH")) == 0);
  long long state_gen = 0;
  bool capturing = false;
  // timing events inside a captured application must be graph event-record nodes
  void record(cudaEvent_t e, cudaStream_t st) const {
    HS_CUDA(cudaEventRecordWithFlags(e, st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
  }
  void drop_graphs() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    graphs.clear();
  }
  // Column order of the current batch (launch_rhs_order): the device path orders from d_b, the
  // streamed path from samples of the host buffer; reports map back through perm_h.
  DBuf<int> rperm, rbbox;
  std::vector<int> perm_h;
  bool perm_on = false;    // rperm holds the batch's order (the transposes apply it)
  bool perm_host = false;  // perm_h already holds it (ordered on the host)
  const int* order_device(const double2* d_b, int nr);
  const int* order_host(const double* b, int nr);
  void solve_streamed(int R, const double* b, double* u, int rounds, bool track, hs_solve_report* reps, int slot = 0,
                      bool last = true, int cap = 0);
  cudaEvent_t ev_din_free[2] = {}, ev_dout_free[2] = {};
  void reports(int nrounds, bool track, hs_solve_report* out);
};

namespace {

Medium medium_from(const hs_problem& P) {
  Medium m;
  switch (P.medium_kind) {
    case 0:
      if (P.kappa <= 0.0) config_error("WaveNumberModel: kappa must be positive");
      m.kind = Medium::Constant;
      m.kappa = P.kappa;
      break;
    case 1:
      if (P.kappa_down <= 0.0 || P.kappa_up <= 0.0) config_error("WaveNumberModel: kappa must be positive");
      if (P.eps < 0.0) config_error("WaveNumberModel: blend width must be >= 0");
      m.kind = Medium::TwoLayered;
      m.kappa_down = P.kappa_down;
      m.kappa_up = P.kappa_up;
      m.axis = P.interface_axis;
      m.eta = P.eta;
      m.eps = P.eps;
      break;
    case 2: {
      m.kind = Medium::Gridded;
      VelocityGrid& g = m.velocity;
      g.dim = P.vel_dim;
      if (g.dim != 2 && g.dim != 3) data_error("VelocityGrid: dim must be 2 or 3");
      std::int64_t cnt = 1;
      for (int a = 0; a < 3; ++a) {
        g.n[a] = a < g.dim ? P.vel_n[a] : 1;
        g.origin[a] = P.vel_origin[a];
        g.spacing[a] = P.vel_spacing[a];
      }
      for (int a = 0; a < g.dim; ++a) {
        if (g.n[a] < 2) data_error("VelocityGrid: need at least 2 samples per axis");
        if (g.spacing[a] <= 0.0) data_error("VelocityGrid: spacing must be positive");
        cnt *= g.n[a];
      }
      if (!P.vel_c) data_error("VelocityGrid: missing samples");
      g.c.assign(P.vel_c, P.vel_c + cnt);
      for (float v : g.c)
        if (!(v > 0.0f)) data_error("VelocityGrid: non-positive velocity sample");
      if (P.omega <= 0.0) config_error("WaveNumberModel: omega must be positive");
      m.omega = P.omega;
      break;
    }
    default:
      config_error("unknown medium kind");
  }
  return m;
}

}  // namespace

// DdmSolver ctor + build_subdomain_states (src/sweeper.cpp:75-157).
void DdmHandle::build(const hs_problem& P, int device, int rank_, int world_, const int* owner_) {
  dim = P.dim;
  if (dim != 2 && dim != 3) config_error("Box: dim must be 2 or 3");
  interior.dim = dim;
  for (int a = 0; a < 3; ++a) {
    interior.lo[a] = a < dim ? P.interior_lo[a] : 0.0;
    interior.hi[a] = a < dim ? P.interior_hi[a] : 1.0;
    intervals[a] = a < dim ? P.intervals[a] : 1;
  }
  for (int a = 0; a < dim; ++a)
    if (!(interior.lo[a] < interior.hi[a])) config_error("Box: lo must be strictly below hi on every axis");
  pml.width = P.pml_width;
  pml.strength = P.pml_strength;
  pml.exponent = P.pml_exponent;
  if (pml.width < 1) config_error("PmlSpec: width must be >= 1 layer");
  if (pml.strength <= 0.0) config_error("PmlSpec: strength must be positive");
  if (pml.exponent < 1) config_error("PmlSpec: exponent must be >= 1");
  if (pml.width < 2) config_error("DdmSolver: pml.width must be >= 2 so trace lines stay off the shell");
  medium = medium_from(P);
  auto t0 = std::chrono::steady_clock::now();
  const bool prof = std::getenv("HS_SETUP_PROFILE") != nullptr;  // developer instrumentation
  auto tprev = t0;
  auto phase = [&](const char* name) {
    if (!prof) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[setup] %-28s %8.1f ms\n", name, std::chrono::duration<double, std::milli>(t - tprev).count());
    tprev = t;
  };
  part = make_partition(interior, intervals, Vec3i{P.counts[0], P.counts[1], P.counts[2]});
  wts.p = &part;
  wts.pad = pml.width;
  ggrid.dim = dim;
  ggrid.range.dim = dim;
  for (int a = 0; a < dim; ++a) {
    ggrid.h[a] = part.h[a];
    ggrid.origin[a] = interior.lo[a];
    ggrid.range.lo[a] = -pml.width;
    ggrid.range.hi[a] = intervals[a] + pml.width;
  }
  gcoeffs = build_coefficients(pml, interior, ggrid);

  phase("global grid + coefficients");
  eng.init(device, dim);
  HS_CUDA(cudaFree(nullptr));  // create the context here: process start-up, not factorization
  phase("device init");
  t0 = std::chrono::steady_clock::now();  // factor_seconds: subdomain setup + factorization
  const int nsub = part.cell_count();
  subs.resize(nsub);
  std::vector<CVector> vals(nsub);
  std::map<std::vector<int>, int> class_of_key;
  std::vector<PmlCoefficients> coeffs(nsub);
  std::vector<Csr> ops(nsub);
  for (int id = 0; id < nsub; ++id) {
    SubHost& st = subs[id];
    st.sub = part.unflatten(id);
    st.owned = part.owned(st.sub);
    st.cell = part.cell(st.sub);
    st.range = st.owned;
    for (int a = 0; a < dim; ++a) {
      st.range.lo[a] -= pml.width;
      st.range.hi[a] += pml.width;
    }
  }
  // Subdomain setup (src/sweeper.cpp:89-124). The 1-D PML tables are built on the host (O(n) per
  // axis); the extended wavenumber and the CSR values of every subdomain are computed on the device
  // (hs_assemble.cu, bit for bit with the host restatement). Only one representative per symbolic
  // class is assembled on the host, for the CSR structure the symbolic analysis needs.
  // HS_HOST_SETUP=1 assembles every subdomain on the host instead (A/B, tests).
  const bool host_setup = std::getenv("HS_HOST_SETUP") != nullptr;
  auto local_grid = [&](const SubHost& st) {
    LocalGrid g;
    g.dim = dim;
    g.range = st.range;
    g.h = ggrid.h;
    g.origin = ggrid.origin;
    return g;
  };
  parallel_for(nsub, [&](long long id) { coeffs[id] = build_coefficients(pml, subs[id].cell, local_grid(subs[id])); });
  // symbolic classes: key = extents and the lower index (or its parity when non-negative: C++
  // truncating mid = (lo+hi)/2 only depends on it through that); one symbolic build per class
  std::vector<int> first_of_class;
  for (int id = 0; id < nsub; ++id) {
    SubHost& st = subs[id];
    std::vector<int> key;
    for (int a = 0; a < dim; ++a) {
      key.push_back(st.range.size(a));
      key.push_back(st.range.lo[a] < 0 ? st.range.lo[a] : (1 << 30) + (st.range.lo[a] & 1));
    }
    auto it = class_of_key.find(key);
    if (it == class_of_key.end()) {
      st.cls = static_cast<int>(first_of_class.size());
      class_of_key[key] = st.cls;
      first_of_class.push_back(id);
    } else {
      st.cls = it->second;
    }
  }
  std::vector<char> assemble_host(nsub, host_setup ? 1 : 0);
  for (int id : first_of_class) assemble_host[id] = 1;
  parallel_for(nsub, [&](long long id) {
    if (!assemble_host[id]) return;
    const LocalGrid g = local_grid(subs[id]);
    ops[id] = assemble(g, coeffs[id], extend_to_subdomain(medium, subs[id].cell, g));
  });
  std::vector<std::unique_ptr<SymbolicClass>> syms(first_of_class.size());
  parallel_for(static_cast<long long>(syms.size()), [&](long long c) {
    const int id = first_of_class[c];
    syms[c] = build_symbolic(dim, subs[id].range, ops[id].row_ptr, ops[id].col);
  });
  for (auto& sc : syms) eng.add_class(std::move(sc));
  for (int id = 0; id < nsub; ++id) {
    const SubHost& st = subs[id];
    if (assemble_host[id] && eng.classes[st.cls]->sym->csr_col.size() != ops[id].col.size())
      throw Error(kInternal, "symbolic class CSR mismatch");
    eng.sub_cls.push_back(st.cls);
    if (host_setup) vals[id] = std::move(ops[id].val);
  }
  phase("assembly + symbolic");
  eng.upload_classes(pml.width);
  phase("upload classes");
  // injection couplings per subdomain and incoming direction (src/transfer.cpp:80-86)
  dirs = 2 * dim;
  for (auto& cdp : eng.classes)
    for (int d = 0; d < dirs; ++d) line_max = std::max<long long>(line_max, cdp->dev.line_len[d]);
  std::vector<Complex> coef(static_cast<size_t>(nsub) * dirs * line_max);
  for (int id = 0; id < nsub; ++id) {
    const SubHost& st = subs[id];
    const SymbolicClass& c = *eng.classes[st.cls]->sym;
    for (int d = 0; d < dirs; ++d) {
      const int a = d / 2, sign = (d & 1) ? 1 : -1;
      GridRange line = st.range;
      const int face = sign > 0 ? st.owned.lo[a] : st.owned.hi[a];
      line.lo[a] = line.hi[a] = face;
      const std::int64_t cnt = line.count();
      for (std::int64_t i = 0; i < cnt; ++i) {
        const Vec3i p0 = line.unlinear(i);
        Vec3i pm = p0;
        pm[a] = face - sign;
        const Vec3i edge = sign > 0 ? pm : p0;
        coef[(static_cast<size_t>(id) * dirs + d) * line_max + i] = coeffs[id].coupling(a, edge);
      }
      (void)c;
    }
  }
  d_coef.alloc(coef.size());
  HS_CUDA(cudaMemcpyAsync(d_coef.p, coef.data(), coef.size() * sizeof(Complex), cudaMemcpyHostToDevice, eng.stream));
  rank = rank_;
  world = world_;
  if (world < 1 || rank < 0 || rank >= world) config_error("partition: rank out of range");
  if (owner_) {
    owner.assign(owner_, owner_ + nsub);
  } else {
    owner = default_owners(dim, part.counts, world);
  }
  for (int id = 0; id < nsub; ++id)
    if (owner[id] < 0 || owner[id] >= world) config_error("partition: owner out of range");
  if (partitioned()) {
    eng.owned.assign(nsub, 0);
    for (int id = 0; id < nsub; ++id) eng.owned[id] = owner[id] == rank;
  }
  // factorize (the DevSub array is re-uploaded with the coefficient pointers below)
  phase("couplings");
  if (host_setup) {
    std::vector<const CVector*> vp(nsub);
    for (int id = 0; id < nsub; ++id) vp[id] = &vals[id];
    eng.factorize(vp);
  } else {
    eng.layout();
    assemble_device(coeffs);  // eng.val and the pivot tolerances
    phase("assembly (device)");
    eng.factorize_numeric();
  }
  phase("factorize (device)");
  for (int id = 0; id < nsub; ++id) {
    DevSub& d = eng.h_subs[id];
    for (int a = 0; a < 3; ++a) {
      d.sub[a] = subs[id].sub[a];
      d.lo[a] = a < dim ? subs[id].range.lo[a] : 0;
    }
    for (int q = 0; q < kMaxDirs; ++q)
      d.coef[q] = q < dirs ? reinterpret_cast<const double2*>(d_coef.p) + (static_cast<size_t>(id) * dirs + q) * line_max
                           : nullptr;
  }
  // geometry for the sweep kernels
  geom.dim = dim;
  geom.pad = pml.width;
  geom.nsub = nsub;
  geom.gn = ggrid.range.count();
  for (int a = 0; a < 3; ++a) {
    geom.glo[a] = a < dim ? ggrid.range.lo[a] : 0;
    geom.gsize[a] = a < dim ? ggrid.range.size(a) : 1;
    geom.counts[a] = part.counts[a];
    geom.cut_w[a] = a < dim ? intervals[a] / part.counts[a] : 1;
  }
  // The setup plans (split source, accumulate) are built by device kernels (hs_assemble.cu) from
  // the partition geometry; a partitioned solver (home nodes, ghost lists) or HS_HOST_SETUP=1 builds
  // them on the host.
  const bool host_plans = host_setup || partitioned();
  PlanGeom pg{};
  DBuf<int> d_subcls;
  DBuf<long long> d_nbase;
  if (!host_plans) {
    pg.dim = dim;
    pg.gn = geom.gn;
    pg.pad = pml.width;
    for (int a = 0; a < 3; ++a) {
      pg.glo[a] = geom.glo[a];
      pg.gsize[a] = geom.gsize[a];
      pg.counts[a] = geom.counts[a];
      pg.w[a] = geom.cut_w[a];
    }
    d_subcls.upload(eng.sub_cls, eng.stream);
    d_nbase.upload(eng.n_base, eng.stream);
    pg.cls = eng.d_cls.p;
    pg.sub_cls = d_subcls.p;
    pg.n_base = d_nbase.p;
  }
  if (!host_plans) {  // split-source plan on the device
    split_gp.alloc(std::max<long long>(eng.n_base[nsub], 1));
    split_w.alloc(std::max<long long>(eng.n_base[nsub], 1));
    long long max_n = 1;
    for (auto& cdp : eng.classes) max_n = std::max<long long>(max_n, cdp->sym->n);
    launch_split_plan(pg, nsub, max_n, split_gp.p, split_w.p, eng.stream);
    for (int id = 0; id < nsub; ++id) {
      eng.h_subs[id].split_gp = split_gp.p + eng.n_base[id];
      eng.h_subs[id].split_w = split_w.p + eng.n_base[id];
    }
  } else {  // split-source plan (src/sweeper.cpp:189-202): per elimination position, the global node and
     // the weight numerator of w(sub, p) * b[p] (0 on the local shell or outside the support)
    const long long ntot = eng.n_base[nsub];
    std::vector<int> gp(std::max<long long>(ntot, 1), 0);
    std::vector<unsigned char> wn(std::max<long long>(ntot, 1), 0);
    parallel_for(nsub, [&](long long id) {
      const SymbolicClass& c = *eng.classes[subs[id].cls]->sym;
      const GridRange& rg = subs[id].range;
      for (std::int64_t e = 0; e < c.n; ++e) {
        const Vec3i p = rg.unlinear(c.local_of_elim[e]);
        bool shell = false;
        int num = 1;
        for (int ax = 0; ax < dim; ++ax) {
          shell |= p[ax] == rg.lo[ax] || p[ax] == rg.hi[ax];
          num *= wts.weight2(ax, subs[id].sub[ax], p[ax]);
        }
        if (num == 0 || shell) continue;
        gp[eng.n_base[id] + e] = static_cast<int>(ggrid.range.linear(p));
        wn[eng.n_base[id] + e] = static_cast<unsigned char>(num);
      }
    });
    split_gp.upload(gp, eng.stream);
    split_w.upload(wn, eng.stream);
    for (int id = 0; id < nsub; ++id) {
      eng.h_subs[id].split_gp = split_gp.p + eng.n_base[id];
      eng.h_subs[id].split_w = split_w.p + eng.n_base[id];
    }
  }
  eng.d_subs.upload(eng.h_subs, eng.stream);
  HS_CUDA(cudaStreamSynchronize(eng.stream));
  factor_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  sub_stats.resize(nsub);
  for (int id = 0; id < nsub; ++id) {
    const SymbolicClass& c = *eng.classes[subs[id].cls]->sym;
    hs_factor_stats& s = sub_stats[id];
    s.n = c.n;
    s.matrix_nnz = static_cast<int64_t>(c.csr_col.size());
    s.factor_nnz = c.factor_nnz;
    s.peak_bytes = c.peak_bytes;
    s.factor_seconds = eng.factor_gpu_seconds;
  }
  phase("stats + split plan");
  if (!host_plans) {
    // accumulate plan on the device, one plan per sweep direction (entries in the reference's order)
    const int E = 1 << dim, ndirs = 1 << dim;
    if (nsub >= (1 << 27)) config_error("partition: too many subdomains");
    const std::vector<Vec3i> dplan = sweep_plan(dim, 1);
    int dv[8][3] = {};
    for (int di = 0; di < ndirs; ++di)
      for (int a = 0; a < 3; ++a) dv[di][a] = dplan[di][a];
    acc_ent.alloc(static_cast<size_t>(geom.gn) * E * ndirs);
    launch_acc_plan(pg, ndirs, dv, acc_ent.p, eng.stream);
    // fronts whose x is read back (support positions, all of nonzero weight, and the trace
    // extraction lines), per subdomain; the set depends only on the class and the support box
    // within the local grid, so it is computed once per such pair
    int nfm = 1;
    for (auto& cdp : eng.classes) nfm = std::max(nfm, static_cast<int>(cdp->sym->fronts.size()));
    need_words = (nfm + 31) / 32;
    need_h.assign(static_cast<size_t>(nsub) * need_words, 0u);
    std::map<std::vector<int>, int> memo;
    for (int id = 0; id < nsub; ++id) {
      const GridRange sup = wts.support(subs[id].sub);
      std::vector<int> key{subs[id].cls};
      for (int a = 0; a < dim; ++a) {
        key.push_back(sup.lo[a] - subs[id].range.lo[a]);
        key.push_back(sup.hi[a] - subs[id].range.lo[a]);
      }
      unsigned* w = need_h.data() + static_cast<size_t>(id) * need_words;
      auto it = memo.find(key);
      if (it != memo.end()) {
        std::copy(need_h.begin() + static_cast<size_t>(it->second) * need_words,
                  need_h.begin() + static_cast<size_t>(it->second + 1) * need_words, w);
        continue;
      }
      memo[key] = id;
      const ClassDev& cd = *eng.classes[subs[id].cls];
      const SymbolicClass& c = *cd.sym;
      auto mark = [&](int e) {
        for (int f = cd.front_of_pos.empty() ? -1 : cd.front_of_pos[e]; f >= 0 && !(w[f >> 5] >> (f & 31) & 1u);
             f = c.fronts[f].parent)
          w[f >> 5] |= 1u << (f & 31);
      };
      Vec3i p{0, 0, 0};
      for (p[2] = sup.lo[2]; p[2] <= (dim > 2 ? sup.hi[2] : sup.lo[2]); ++p[2])
        for (p[1] = sup.lo[1]; p[1] <= sup.hi[1]; ++p[1])
          for (p[0] = sup.lo[0]; p[0] <= sup.hi[0]; ++p[0]) {
            long long loc = 0, ls = 1;
            for (int a = 0; a < dim; ++a) {
              loc += static_cast<long long>(p[a] - subs[id].range.lo[a]) * ls;
              ls *= c.size[a];
            }
            mark(c.elim_of_local[loc]);
          }
      for (int e : cd.ext_pos) mark(e);
    }
    need.upload(need_h, eng.stream);
  } else {  // accumulate plan (src/transfer.cpp:91-102): per global node, every subdomain whose support
     // holds it, as (x position n_base[sub] + elim, sub << 4 | weight numerator)
    const long long gn = geom.gn;
    std::vector<int> off(gn, 0);
    std::vector<int2> ent;
    auto visit = [&](auto&& fn) {
      for (int id = 0; id < nsub; ++id) {
        const GridRange sup = wts.support(subs[id].sub);
        const SymbolicClass& c = *eng.classes[subs[id].cls]->sym;
        Vec3i p{0, 0, 0};
        for (p[2] = sup.lo[2]; p[2] <= (dim > 2 ? sup.hi[2] : sup.lo[2]); ++p[2])
          for (p[1] = sup.lo[1]; p[1] <= sup.hi[1]; ++p[1])
            for (p[0] = sup.lo[0]; p[0] <= sup.hi[0]; ++p[0]) {
              int num = 1;
              long long g = 0, gs = 1, loc = 0, ls = 1;
              for (int ax = 0; ax < dim; ++ax) {
                num *= wts.weight2(ax, subs[id].sub[ax], p[ax]);
                g += static_cast<long long>(p[ax] - geom.glo[ax]) * gs;
                gs *= geom.gsize[ax];
                loc += static_cast<long long>(p[ax] - subs[id].range.lo[ax]) * ls;
                ls *= c.size[ax];
              }
              if (num != 0) fn(g, id, num, c.elim_of_local[loc]);
            }
      }
    };
    const int E = 1 << dim, ndirs = 1 << dim;
    if (nsub >= (1 << 27)) config_error("partition: too many subdomains");
    std::vector<int2> raw(static_cast<size_t>(gn) * E, make_int2(-1, 0));
    visit([&](long long g, int id, int num, int e) {
      if (off[g] >= E) throw Error(kInternal, "accumulate plan: more than 2^dim subdomains at a node");
      raw[static_cast<size_t>(g) * E + off[g]++] = make_int2(static_cast<int>(eng.n_base[id] + e), (id << 4) | num);
    });
    {  // fronts whose x is read back: support positions with a nonzero weight and extraction lines
      int nfm = 1;
      for (auto& cdp : eng.classes) nfm = std::max(nfm, static_cast<int>(cdp->sym->fronts.size()));
      need_words = (nfm + 31) / 32;
      need_h.assign(static_cast<size_t>(nsub) * need_words, 0u);
      auto mark = [&](int id, int e) {
        const ClassDev& cd = *eng.classes[subs[id].cls];
        unsigned* w = need_h.data() + static_cast<size_t>(id) * need_words;
        for (int f = cd.front_of_pos.empty() ? -1 : cd.front_of_pos[e]; f >= 0 && !(w[f >> 5] >> (f & 31) & 1u);
             f = cd.sym->fronts[f].parent)
          w[f >> 5] |= 1u << (f & 31);
      };
      for (long long g = 0; g < gn; ++g)
        for (int i = 0; i < off[g]; ++i) {
          const int2 en = raw[static_cast<size_t>(g) * E + i];
          const int id = en.y >> 4;
          mark(id, static_cast<int>(en.x - eng.n_base[id]));
        }
      for (int id = 0; id < nsub; ++id)
        for (int e : eng.classes[subs[id].cls]->ext_pos) mark(id, e);
      need.upload(need_h, eng.stream);
    }
    // one plan per sweep direction, entries in the reference's order: step, then ascending id
    const std::vector<Vec3i> dplan = sweep_plan(dim, 1);
    std::vector<int> stab(static_cast<size_t>(ndirs) * nsub);
    for (int di = 0; di < ndirs; ++di)
      for (int id = 0; id < nsub; ++id) stab[static_cast<size_t>(di) * nsub + id] = step_of(part.counts, dim, dplan[di], subs[id].sub);
    ent.assign(static_cast<size_t>(gn) * E * ndirs, make_int2(-1, 0));
    const long long nchunk = 256;
    parallel_for(ndirs * nchunk, [&](long long job) {
      const int di = static_cast<int>(job / nchunk);
      const long long c = job % nchunk, g0 = gn * c / nchunk, g1 = gn * (c + 1) / nchunk;
      int2* dst = ent.data() + static_cast<size_t>(di) * gn * E;
      const int* st = stab.data() + static_cast<size_t>(di) * nsub;
      for (long long g = g0; g < g1; ++g) {
        int2 tmp[8];
        long long key[8];
        const int n = off[g];
        for (int i = 0; i < n; ++i) {
          tmp[i] = raw[static_cast<size_t>(g) * E + i];
          const int id = tmp[i].y >> 4;
          key[i] = (static_cast<long long>(st[id]) << 32) | id;
        }
        for (int i = 1; i < n; ++i)
          for (int j = i; j > 0 && key[j] < key[j - 1]; --j) {
            std::swap(key[j], key[j - 1]);
            std::swap(tmp[j], tmp[j - 1]);
          }
        for (int i = 0; i < n; ++i) dst[g * E + i] = tmp[i];
      }
    });
    if (partitioned()) {
      // home rank of a node: the owner of its lowest-id subdomain; only the home rank
      // accumulates the node, reading other ranks' values from ghost copies of their x
      ghost.assign(nsub, std::vector<std::vector<long long>>(world));
      std::vector<std::vector<int>> homes(world);
      for (long long g = 0; g < gn; ++g) {
        const int n = off[g];
        if (n == 0) continue;
        int lo = 1 << 30;
        for (int i = 0; i < n; ++i) lo = std::min(lo, raw[static_cast<size_t>(g) * E + i].y >> 4);
        const int home = owner[lo];
        homes[home].push_back(static_cast<int>(g));
        for (int i = 0; i < n; ++i) {
          const int2 e = raw[static_cast<size_t>(g) * E + i];
          const int id = e.y >> 4;
          if (owner[id] != home) ghost[id][home].push_back(e.x);
        }
        if (home != rank)
          for (int di = 0; di < ndirs; ++di)
            for (int i = 0; i < E; ++i) ent[(static_cast<size_t>(di) * gn + g) * E + i] = make_int2(-1, 0);
      }
      // owner slabs of u for the gather (every rank holds every rank's list, padded with -1)
      max_home = 1;
      for (const auto& h : homes) max_home = std::max<long long>(max_home, static_cast<long long>(h.size()));
      home_cnt = static_cast<long long>(homes[rank].size());
      std::vector<int> hl(static_cast<size_t>(world) * max_home, -1);
      for (int q = 0; q < world; ++q) std::copy(homes[q].begin(), homes[q].end(), hl.begin() + static_cast<size_t>(q) * max_home);
      d_homes.upload(hl, eng.stream);
      std::vector<long long> flat;
      ghost_off.assign(static_cast<size_t>(nsub) * world + 1, 0);
      for (int id = 0; id < nsub; ++id)
        for (int q = 0; q < world; ++q) {
          auto& v = ghost[id][q];
          std::sort(v.begin(), v.end());
          v.erase(std::unique(v.begin(), v.end()), v.end());
          ghost_off[static_cast<size_t>(id) * world + q] = static_cast<long long>(flat.size());
          flat.insert(flat.end(), v.begin(), v.end());
        }
      ghost_off.back() = static_cast<long long>(flat.size());
      if (flat.empty()) flat.push_back(0);
      d_gpos.upload(flat, eng.stream);
    }
    acc_ent.upload(ent, eng.stream);
  }
  phase("accumulate plan");
  // step groups and dataflow task lists per (sweep direction, step)
  steps = sweep_step_count(part.counts, dim);
  ndir = 1 << dim;
  const std::vector<Vec3i> dirs_plan = sweep_plan(dim, 1);
  std::vector<int> gflat;
  groups.assign(ndir * steps, {});
  grp_off.assign(ndir * steps, 0);
  for (int di = 0; di < ndir; ++di)
    for (int s = 1; s <= steps; ++s) {
      const int gi = di * steps + s - 1;
      for (int id = 0; id < nsub; ++id)
        if (step_of(part.counts, dim, dirs_plan[di], subs[id].sub) == s) groups[gi].push_back(id);
      max_group = std::max(max_group, static_cast<int>(groups[gi].size()));
      grp_off[gi] = static_cast<int>(gflat.size());
      gflat.insert(gflat.end(), groups[gi].begin(), groups[gi].end());
    }
  d_groups.upload(gflat, eng.stream);
  HS_CUDA(cudaStreamSynchronize(eng.stream));
  phase("step groups");
}

AsmMedium DdmHandle::asm_medium() {
  AsmMedium m{};
  m.kind = static_cast<int>(medium.kind);
  m.kappa = medium.kappa;
  m.kd = medium.kappa_down;
  m.ku = medium.kappa_up;
  m.eta = medium.eta;
  m.eps = medium.eps;
  m.omega = medium.omega;
  m.axis = medium.axis;
  if (medium.kind == Medium::Gridded) {
    const VelocityGrid& g = medium.velocity;
    m.vdim = g.dim;
    for (int a = 0; a < 3; ++a) {
      m.vn[a] = g.n[a];
      m.vorg[a] = g.origin[a];
      m.vsp[a] = g.spacing[a];
    }
    if (vel_dev.n != g.c.size()) {
      vel_dev.alloc(g.c.size());
      HS_CUDA(cudaMemcpyAsync(vel_dev.p, g.c.data(), g.c.size() * sizeof(float), cudaMemcpyHostToDevice, eng.stream));
    }
    m.vc = vel_dev.p;
  }
  return m;
}

void DdmHandle::assemble_device(const std::vector<PmlCoefficients>& coeffs) {
  const int nsub = geom.nsub > 0 ? geom.nsub : static_cast<int>(subs.size());
  // class CSR structures
  long long max_rows = 0;
  for (auto& cdp : eng.classes) {
    ClassDev& cd = *cdp;
    if (!cd.csr_rp.p) {
      cd.csr_rp.upload(cd.sym->csr_row_ptr, eng.stream);
      cd.csr_col.upload(cd.sym->csr_col, eng.stream);
    }
    max_rows = std::max<long long>(max_rows, cd.sym->n);
  }
  // 1-D PML tables of the owned subdomains, flattened
  std::vector<Complex> tab;
  std::vector<std::array<long long, 6>> off(nsub);
  for (int id = 0; id < nsub; ++id) {
    if (!eng.owns(id)) continue;
    for (int a = 0; a < dim; ++a) {
      off[id][2 * a] = static_cast<long long>(tab.size());
      tab.insert(tab.end(), coeffs[id].node[a].begin(), coeffs[id].node[a].end());
      off[id][2 * a + 1] = static_cast<long long>(tab.size());
      tab.insert(tab.end(), coeffs[id].half[a].begin(), coeffs[id].half[a].end());
    }
  }
  alpha_dev.alloc(std::max<size_t>(tab.size(), 1));
  HS_CUDA(cudaMemcpyAsync(alpha_dev.p, tab.data(), tab.size() * sizeof(Complex), cudaMemcpyHostToDevice, eng.stream));
  DBuf<unsigned long long> dmax;
  dmax.alloc(nsub + 1);  // [nsub]: the bad-sample flag
  dmax.zero(eng.stream);
  std::vector<AsmSub> hs;
  std::vector<int> ids;
  for (int id = 0; id < nsub; ++id) {
    if (!eng.owns(id)) continue;
    const SubHost& st = subs[id];
    const ClassDev& cd = *eng.classes[st.cls];
    AsmSub a{};
    for (int ax = 0; ax < 3; ++ax) {
      a.lo[ax] = ax < dim ? st.range.lo[ax] : 0;
      a.size[ax] = ax < dim ? st.range.size(ax) : 1;
      a.cell_lo[ax] = st.cell.lo[ax];
      a.cell_hi[ax] = st.cell.hi[ax];
      a.anode[ax] = ax < dim ? alpha_dev.p + off[id][2 * ax] : nullptr;
      a.ahalf[ax] = ax < dim ? alpha_dev.p + off[id][2 * ax + 1] : nullptr;
    }
    a.row_ptr = cd.csr_rp.p;
    a.col = cd.csr_col.p;
    a.val = eng.val.p + eng.val_base[id];
    a.maxabs = dmax.p + id;
    hs.push_back(a);
    ids.push_back(id);
  }
  if (hs.empty()) return;
  asm_subs.upload(hs, eng.stream);
  AsmArgs args{};
  args.dim = dim;
  for (int ax = 0; ax < 3; ++ax) {
    args.h[ax] = ggrid.h[ax];
    args.origin[ax] = ggrid.origin[ax];
  }
  args.med = asm_medium();
  args.subs = asm_subs.p;
  args.nsub = static_cast<int>(hs.size());
  args.bad = reinterpret_cast<unsigned*>(dmax.p + nsub);
  launch_assemble(args, max_rows, eng.stream);
  std::vector<unsigned long long> mx(nsub + 1);
  HS_CUDA(cudaMemcpyAsync(mx.data(), dmax.p, mx.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, eng.stream));
  HS_CUDA(cudaStreamSynchronize(eng.stream));
  if (mx[nsub]) data_error("eval_kappa: non-positive velocity sample");
  for (int id : ids) {
    double scale = 0.0;
    std::memcpy(&scale, &mx[id], sizeof(double));
    eng.tol[id] = 1e-14 * scale;  // src/direct.cpp:191-193
  }
}

// Macro-step schedule of one application: task (l, id) runs one macro-step after the latest of
//  * the tasks whose traces it consumes: (l', nb) with nb its neighbour across face (a, sign) and
//    route_trace(l', a, sign) == l (src/sweeper.cpp:58-73, 285-307) — the only data it reads;
//  * the accumulate of sweep l - nbuf, whose x buffer sweep l reuses.
// Sweep accumulates stay in sweep order (u += contribution_l, src/sweeper.cpp:311), and every
// mailbox slot has one writer, so the results equal the sequential order's: only independent
// work is reordered. C2 (8x8, 4 sweeps): 60 sequential steps -> 29 macro-steps.
void DdmHandle::build_schedule(int r) {
  const int nsub = geom.nsub;
  // x buffers in flight: one per sweep when they fit (every sweep then overlaps as the routing
  // allows and all contributions are accumulated in one fused pass per region at the end; C3's 8
  // sweeps: 267 -> 249 ms per 64-RHS application), else 4
  nbuf = 4;
  {
    const int want = std::min(std::min(nsweeps, HS_MAX_ACC_SWEEPS), nbuf_cap);
    if (want > nbuf) {
      size_t free_b = 0, total_b = 0;
      HS_CUDA(cudaMemGetInfo(&free_b, &total_b));
      const double have = static_cast<double>(free_b) +
                          static_cast<double>(eng.x.n + eng.x1.n + eng.rb.n) * sizeof(double2);
      const double per_buf = static_cast<double>(eng.n_base.back()) * r * sizeof(double2);  // x
      const double reserve = 8.0 * r * static_cast<double>(geom.gn) * sizeof(double2) + 4e9;  // io slots, bN, u, uround
      if (want * per_buf + reserve <= 0.9 * have) nbuf = want;
    }
  }
  if (const char* e = std::getenv("HS_NBUF")) nbuf = std::max(1, std::atoi(e));
  nbuf = std::min(nbuf, nsweeps);
  std::vector<int> level, accl;
  task_levels(dim, part.counts, plan, route_h, nsweeps, nbuf, level, accl);
  const int nmacro = accl[nsweeps];
  msteps.assign(nmacro, {});
  acc_after.assign(nmacro, {});
  mstep_of.assign(static_cast<size_t>(nsweeps) * nsub, 0);
  sweep_first_m.assign(nsweeps + 1, nmacro);
  for (int l = 1; l <= nsweeps; ++l) {
    for (int id = 0; id < nsub; ++id) {
      const int m = level[static_cast<size_t>(l - 1) * nsub + id] - 1;
      msteps[m].push_back(make_int2(id, l));
      mstep_of[static_cast<size_t>(l - 1) * nsub + id] = m;
      sweep_first_m[l] = std::min(sweep_first_m[l], m);
    }
    acc_after[accl[l] - 1].push_back(l);
  }
  {  // stripes of the slowest axis for streamed host transfers
    const int la = dim - 1;
    long long plane = 1;
    for (int a = 0; a < la; ++a) plane *= geom.gsize[a];
    int spr = 2;  // stripes per subdomain row (HS_STRIPES_PER_ROW: developer knob)
    if (const char* e = std::getenv("HS_STRIPES_PER_ROW")) spr = std::max(1, std::atoi(e));
    const int rows = geom.gsize[la], ns = std::max(1, std::min(rows, spr * part.counts[la]));
    stripe_n.assign(ns + 1, 0);
    for (int j = 0; j <= ns; ++j) stripe_n[j] = plane * ((static_cast<long long>(rows) * j) / ns);
    {
      // segments of the fastest axis: at most one per subdomain column, and rows of at least 4 KB
      // (narrower 3D copies lose DMA bandwidth: C2 e2e 17.9 ms at 8 segments, 16.7 at 4)
      const int gx = geom.gsize[0];
      int spx = std::max(1, std::min(part.counts[0], gx * static_cast<int>(sizeof(double2)) / 4096));
      if (const char* e = std::getenv("HS_TILE_SEGS")) spx = std::max(1, std::atoi(e));  // developer knob
      spx = std::min(spx, gx);
      in_tiles.clear();
      for (int j = 0; j < ns; ++j)
        for (int c = 0; c < spx; ++c) {
          InTile t{stripe_n[j] / gx, stripe_n[j + 1] / gx, static_cast<int>((static_cast<long long>(gx) * c) / spx),
                   static_cast<int>((static_cast<long long>(gx) * (c + 1)) / spx), nmacro};
          if (t.x1 <= t.x0 || t.row1 <= t.row0) continue;
          const long long sl0 = stripe_n[j] / plane, sl1 = (stripe_n[j + 1] + plane - 1) / plane;  // slowest-axis rows
          for (int m = 0; m < nmacro && t.need == nmacro; ++m)
            for (const int2& tk : msteps[m]) {
              if (tk.y != 1) continue;
              const GridRange sup = wts.support(subs[tk.x].sub);
              const long long a0 = sup.lo[la] - geom.glo[la], a1 = sup.hi[la] - geom.glo[la] + 1;
              const int b0 = sup.lo[0] - geom.glo[0], b1 = sup.hi[0] - geom.glo[0] + 1;
              if (a0 < sl1 && a1 > sl0 && b0 < t.x1 && b1 > t.x0) {
                t.need = m;
                break;
              }
            }
          in_tiles.push_back(t);
        }
      std::stable_sort(in_tiles.begin(), in_tiles.end(), [](const InTile& a, const InTile& b) { return a.need < b.need; });
      need_tiles.assign(nmacro, 0);
      for (int m = 0; m < nmacro; ++m) {
        int k = 0;
        while (k < static_cast<int>(in_tiles.size()) && in_tiles[k].need <= m) ++k;
        need_tiles[m] = k;
      }
    }
    // stripes of the last sweep's accumulate (of every sweep's, fused)
    fuse_acc = nsweeps <= nbuf && nsweeps <= HS_MAX_ACC_SWEEPS && !std::getenv("HS_NO_FUSED_ACC");
    sweep_end_m.assign(nsweeps + 1, 0);
    for (int l = 1; l <= nsweeps; ++l) sweep_end_m[l] = accl[l] - 1;
    // unfused, the last sweep's striped accumulate follows the whole-domain accumulate of the one
    // before it (u += in sweep order); fused, a region is final after its own tasks
    const int acc_m0 = fuse_acc || nsweeps == 1 ? 0 : accl[nsweeps - 1] - 1;
    acc_stripe_m.assign(ns, acc_m0);
    for (int l = fuse_acc ? 1 : nsweeps; l <= nsweeps; ++l)
      for (int id = 0; id < nsub; ++id) {
        const int m = mstep_of[static_cast<size_t>(l - 1) * nsub + id];
        const GridRange sup = wts.support(subs[id].sub);
        const long long lo = static_cast<long long>(sup.lo[la] - geom.glo[la]) * plane;
        const long long hi = (static_cast<long long>(sup.hi[la] - geom.glo[la]) + 1) * plane;
        for (int j = 0; j < ns; ++j)
          if (stripe_n[j] < hi && stripe_n[j + 1] > lo) acc_stripe_m[j] = std::max(acc_stripe_m[j], m);
      }
    {
      const int gx = geom.gsize[0];
      out_stripes.clear();
      for (int j = 0; j < ns; ++j) out_stripes.push_back(OutRegion{stripe_n[j] / gx, stripe_n[j + 1] / gx, 0, gx, acc_stripe_m[j]});
      out_tiles.clear();
      if (fuse_acc)
        for (const InTile& t : in_tiles) {
          OutRegion o{t.row0, t.row1, t.x0, t.x1, acc_m0};
          const long long sl0 = t.row0 * gx / plane, sl1 = (t.row1 * gx + plane - 1) / plane;
          for (int l = 1; l <= nsweeps; ++l)
            for (int id = 0; id < nsub; ++id) {
              const GridRange sup = wts.support(subs[id].sub);
              const long long a0 = sup.lo[la] - geom.glo[la], a1 = sup.hi[la] - geom.glo[la] + 1;
              const int b0 = sup.lo[0] - geom.glo[0], b1 = sup.hi[0] - geom.glo[0] + 1;
              if (a0 < sl1 && a1 > sl0 && b0 < t.x1 && b1 > t.x0)
                o.acc_m = std::max(o.acc_m, mstep_of[static_cast<size_t>(l - 1) * nsub + id]);
            }
          out_tiles.push_back(o);
        }
      std::sort(out_tiles.begin(), out_tiles.end(), [](const OutRegion& a, const OutRegion& b) {
        return a.acc_m != b.acc_m ? a.acc_m < b.acc_m : a.row0 != b.row0 ? a.row0 < b.row0 : a.x0 < b.x0;
      });
    }
    for (int l = 1; l <= nsweeps; ++l) {  // the striped accumulate replaces the whole-domain ones
      auto& v = acc_after[accl[l] - 1];
      if (l == nsweeps || fuse_acc) v.erase(std::remove(v.begin(), v.end(), l), v.end());
    }
  }
  // this rank's tasks (all of them unless partitioned)
  msteps_own.assign(nmacro, {});
  for (int m = 0; m < nmacro; ++m)
    for (const int2& t : msteps[m])
      if (owner[t.x] == rank) msteps_own[m].push_back(t);
  std::vector<int2> flat;
  mt_off.assign(nmacro, 0);
  max_width = 1;
  for (int m = 0; m < nmacro; ++m) {
    mt_off[m] = static_cast<int>(flat.size());
    flat.insert(flat.end(), msteps_own[m].begin(), msteps_own[m].end());
    max_width = std::max(max_width, static_cast<int>(msteps_own[m].size()));
  }
  // previous occupant of each task's slot within the application: (class, 1 if it was a sweep-1 task
  // that wrote its whole slot), or (-1, 0) for the slot's first use (rb is cleared per application)
  std::vector<int2> prev(std::max<size_t>(flat.size(), 1), make_int2(-1, 0));
  {
    std::vector<int2> last(static_cast<size_t>(max_width), make_int2(-1, 0));
    for (int m = 0; m < nmacro; ++m)
      for (size_t t = 0; t < msteps_own[m].size(); ++t) {
        prev[mt_off[m] + t] = last[t];
        const int2 tk = msteps_own[m][t];
        last[t] = make_int2(subs[tk.x].cls, tk.y == 1 ? 1 : 0);
      }
  }
  d_prev.upload(prev, eng.stream);
  prev_h = prev;
  if (flat.empty()) flat.push_back(make_int2(0, 1));
  d_mtasks.upload(flat, eng.stream);
}

// Work items of every macro-step for the current batch width.
void DdmHandle::build_items() {
  std::vector<SolveItem> tasks;
  const int nm = static_cast<int>(msteps.size());
  fwd_off.assign(nm, 0);
  fwd_cnt.assign(nm, 0);
  bwd_off.assign(nm, 0);
  bwd_cnt.assign(nm, 0);
  for (int m = 0; m < nm; ++m) {
    std::vector<Engine::TaskRef> refs;
    for (const int2& t : msteps_own[m]) {
      Engine::TaskRef r{t.x, t.y, (t.y - 1) % nbuf};
      if (t.y > 1) {  // faces whose mailbox slots some generating sweep can fill for sweep t.y
        r.faces = 0;
        const Vec3i sb = subs[t.x].sub;
        for (int d = 0; d < dirs; ++d) {
          const int ax = d / 2, sg = (d & 1) ? 1 : -1;
          if (!part.has_neighbor(sb, ax, -sg)) continue;  // the trace travels +sg from the neighbour at -sg
          for (int lg = 1; lg <= t.y; ++lg)
            if (route_h[(lg - 1) * dirs + d] == t.y) {
              r.faces |= 1u << d;
              break;
            }
        }
      }
      if (!need_h.empty()) r.need = need_h.data() + static_cast<size_t>(t.x) * need_words;
      refs.push_back(r);
    }
    std::vector<SolveItem> fw, bw;
    eng.build_items(refs, fw, bw);
    fwd_off[m] = static_cast<int>(tasks.size());
    fwd_cnt[m] = static_cast<int>(fw.size());
    tasks.insert(tasks.end(), fw.begin(), fw.end());
    bwd_off[m] = static_cast<int>(tasks.size());
    bwd_cnt[m] = static_cast<int>(bw.size());
    tasks.insert(tasks.end(), bw.begin(), bw.end());
  }
  if (tasks.empty()) tasks.push_back(SolveItem{});
  d_tasks.upload(tasks, eng.stream);
  if (partitioned()) build_xplan();
}

// Exchange plan of every macro-step for the current batch width: message (src -> dst) lists,
// in the global task order of the macro-step, the traces src deposited for dst's subdomains
// (mailbox slot of the generating sweep + presence word) and src's solution values on dst's
// home nodes (ghost x + the task's nonzero word). Sender and receiver enumerate the same list.
void DdmHandle::build_xplan() {
  const int nm = static_cast<int>(msteps.size()), nsub = geom.nsub;
  const long long dstride = 2 * line_max * R;
  std::vector<XSeg> segs;
  xplan.assign(nm, XPlan{});
  x_sent = x_msgs = 0;
  long long smax = 1, rmax = 1;
  auto message = [&](int m, int src, int dst, long long base, std::vector<XSeg>* out) {
    long long at = base;
    for (const int2& t : msteps[m]) {
      const int id = t.x, l = t.y;
      if (owner[id] != src) continue;
      const Vec3i sb = subs[id].sub;
      const DevClass& C = eng.classes[subs[id].cls]->dev;
      for (int d = 0; d < dirs; ++d) {
        const int ax = d / 2, sg = (d & 1) ? 1 : -1;
        if (!part.has_neighbor(sb, ax, sg) || route_h[(l - 1) * dirs + d] == 0) continue;
        Vec3i tb = sb;
        tb[ax] += sg;
        const int tid = part.flatten(tb);
        if (owner[tid] != dst) continue;
        const long long slot = (static_cast<long long>(tid) * nsweeps + (l - 1)) * dirs + d;
        if (out) out->push_back(XSeg{1, 1, slot, at, 0});
        at += 1;
        const int cnt = 2 * C.line_len[d] * R;
        if (out) out->push_back(XSeg{0, cnt, slot * dstride, at, 0});
        at += 2LL * cnt;
      }
      const long long g0 = ghost_off[static_cast<size_t>(id) * world + dst],
                      g1 = ghost_off[static_cast<size_t>(id) * world + dst + 1];
      if (g1 > g0) {
        if (out) out->push_back(XSeg{3, 1, static_cast<long long>(l - 1) * nsub + id, at, 0});
        at += 1;
        const long long xoff = static_cast<long long>((l - 1) % nbuf) * eng.xstride;
        for (long long q = g0; q < g1; q += 1024) {  // runs of <= 1024 positions per segment
          const int np = static_cast<int>(std::min<long long>(1024, g1 - q));
          if (out) out->push_back(XSeg{2, np * R, q, at, xoff});
          at += 2LL * np * R;
        }
      }
    }
    return at - base;
  };
  for (int m = 0; m < nm; ++m) {
    XPlan& xp = xplan[m];
    std::vector<XSeg> send, recv;
    long long so = 0, ro = 0;
    for (int p = 0; p < world; ++p) {
      if (p == rank) continue;
      const long long ns = message(m, rank, p, so, nullptr), nr = message(m, p, rank, ro, nullptr);
      if (ns == 0 && nr == 0) continue;
      message(m, rank, p, so, &send);
      message(m, p, rank, ro, &recv);
      xp.peers.push_back(p);
      xp.soff.push_back(so);
      xp.scnt.push_back(ns);
      xp.roff.push_back(ro);
      xp.rcnt.push_back(nr);
      so += ns;
      ro += nr;
      x_sent += ns;
      x_msgs += ns > 0;
    }
    smax = std::max(smax, so);
    rmax = std::max(rmax, ro);
    xp.s0 = static_cast<int>(segs.size());
    xp.ns = static_cast<int>(send.size());
    segs.insert(segs.end(), send.begin(), send.end());
    xp.r0 = static_cast<int>(segs.size());
    xp.nr = static_cast<int>(recv.size());
    segs.insert(segs.end(), recv.begin(), recv.end());
  }
  if (segs.empty()) segs.push_back(XSeg{});
  d_xseg.upload(segs, eng.stream);
  xsend.alloc(smax);
  xrecv.alloc(rmax);
}

void DdmHandle::comm_gather_u(double2* buf) {
  if (!ncomm || !d_homes.p) {
    comm_allreduce(reinterpret_cast<double*>(buf), 2LL * geom.gn * R);
    return;
  }
  const long long slab = max_home * R;
  gsend.alloc(static_cast<size_t>(slab));
  grecv.alloc(static_cast<size_t>(slab) * world);
  launch_pack_home(buf, d_homes.p + static_cast<size_t>(rank) * max_home, home_cnt, R, gsend.p, eng.stream);
  ncomm->allgather(reinterpret_cast<const double*>(gsend.p), reinterpret_cast<double*>(grecv.p), 2 * slab, eng.stream);
  launch_unpack_home(grecv.p, d_homes.p, max_home, world, R, buf, eng.stream);
}

void DdmHandle::comm_allreduce(double* buf, long long count) {
  if (ncomm) {
    ncomm->allreduce(buf, count, eng.stream);
    return;
  }
  if (!arfn) throw Error(kConfig, "partitioned solve: no allreduce callback");
  if (arfn(cuser, buf, count, eng.stream) != 0) throw Error(kCuda, "partitioned solve: allreduce callback failed");
}

// With one x buffer per sweep the solve state can exceed what the factors leave free (C5: 106 GB
// of factors); an allocation failure then rebuilds the state with the 4-buffer schedule.
void DdmHandle::ensure_state(int r, int nrounds) {
  try {
    ensure_state_body(r, nrounds);
  } catch (const Error& e) {
    if (e.code != kCuda || nbuf <= 4 || std::string(e.what()).find("out of memory") == std::string::npos) throw;
    (void)cudaGetLastError();
    nbuf_cap = 4;
    eng.x.release();
    eng.x1.release();
    eng.rb.release();
    eng.R = 0;  // force the solve buffers to be rebuilt
    rounds = 0;
    R = 0;
    ensure_state_body(r, nrounds);
  }
}

void DdmHandle::ensure_state_body(int r, int nrounds) {
  if (r < 1 || r > kMaxRhs) config_error("ddm_solve: batch size out of range");
  if (nrounds < 1) config_error("SweepPlan: rounds must be >= 1");
  const int ns = nrounds * ndir;
  if (ns > HS_MAX_SWEEPS || nrounds > HS_MAX_ROUNDS) config_error("ddm_solve: too many rounds");
  const bool new_rounds = nrounds != rounds, new_r = r != R;
  if (new_rounds) {
    rounds = nrounds;
    nsweeps = ns;
    plan = sweep_plan(dim, nrounds);
    route_h.assign(nsweeps * dirs, 0);
    for (int l = 1; l <= nsweeps; ++l)
      for (int d = 0; d < dirs; ++d) route_h[(l - 1) * dirs + d] = route_trace(plan, dim, l, d / 2, (d & 1) ? 1 : -1);
    route.upload(route_h, eng.stream);
    build_schedule(r);
  }
  eng.ensure_solve(r, max_width, nbuf);
  if (!new_rounds && !new_r) return;
  ++state_gen;
  R = r;
  build_items();
  const int nsub = geom.nsub;
  mbox.alloc(static_cast<size_t>(nsub) * nsweeps * dirs * 2 * line_max * R);
  mpres.alloc(static_cast<size_t>(nsub) * nsweeps * dirs);
  nzmask.alloc(static_cast<size_t>(nsweeps) * nsub);
  tface.alloc(static_cast<size_t>(nsweeps) * nsub);
  bN.alloc(static_cast<size_t>(geom.gn) * R);
  u.alloc(static_cast<size_t>(geom.gn) * R);
  // + striped rounding + reduction scratch
  const long long nb = (geom.gn * R + 255) / 256 + static_cast<long long>(std::max(stripe_n.size(), out_tiles.size() + 1)) + kReducePad;
  partial_stride = nb * R;
  partial.alloc(static_cast<size_t>(nb) * R * (fuse_acc ? nsweeps : 1));
  pnum.alloc(static_cast<size_t>(nb) * R);
  pden.alloc(static_cast<size_t>(nb) * R);
  norms.alloc(static_cast<size_t>(nsweeps) * R);
  rnum.alloc(static_cast<size_t>(nrounds) * R);
  uround.alloc(fuse_acc && nrounds > 1 ? static_cast<size_t>(nrounds - 1) * geom.gn * R : 0);
  rden.alloc(static_cast<size_t>(nrounds) * R);
  for (auto e : ev) cudaEventDestroy(e);
  ev.assign(1 + nsweeps + 2 * msteps.size(), nullptr);
  for (auto& e : ev) HS_CUDA(cudaEventCreate(&e));
  for (auto e : ev_out) cudaEventDestroy(e);
  ev_out.assign(std::max(out_stripes.size(), out_tiles.size()), nullptr);
  for (auto& e : ev_out) HS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

// The global J-scaled operator (DdmSolver::global_op, src/sweeper.cpp:159-162) on the device: its
// CSR structure is integer work on the host (the class-independent stencil pattern), its values
// come from the device assembly (hs_assemble.cu) with the interior box as the extension cell.
void DdmHandle::ensure_gop() {
  if (gop_ready) return;
  if (std::getenv("HS_HOST_SETUP")) {
    Csr op = assemble(ggrid, gcoeffs, extend_to_subdomain(medium, interior, ggrid));
    g_nnz = static_cast<long long>(op.col.size());
    std::vector<int> col32(op.col.begin(), op.col.end());
    g_rp.upload(op.row_ptr, eng.stream);
    g_col.upload(col32, eng.stream);
    g_val.alloc(op.val.size());
    HS_CUDA(cudaMemcpyAsync(g_val.p, op.val.data(), op.val.size() * sizeof(Complex), cudaMemcpyHostToDevice,
                            eng.stream));
    HS_CUDA(cudaStreamSynchronize(eng.stream));
    build_stencil_op();
    gop_ready = true;
    return;
  }
  const GridRange& rg = ggrid.range;
  const std::int64_t n = rg.count();
  std::vector<std::int64_t> rp(n + 1, 0);
  std::vector<int> col32;
  col32.reserve(static_cast<size_t>(n) * (2 * dim + 1));
  long long stride[3] = {1, 1, 1};
  for (int a = 1; a < dim; ++a) stride[a] = stride[a - 1] * rg.size(a - 1);
  for (std::int64_t r = 0; r < n; ++r) {  // src/operator.cpp:41-86: sorted columns, shell rows identity
    const Vec3i p = rg.unlinear(r);
    if (ggrid.on_shell(p)) {
      col32.push_back(static_cast<int>(r));
    } else {
      for (int a = dim - 1; a >= 0; --a)  // lower neighbours, farthest first
        if (!(p[a] - 1 == rg.lo[a])) col32.push_back(static_cast<int>(r - stride[a]));
        else (void)0;
      col32.push_back(static_cast<int>(r));
      for (int a = 0; a < dim; ++a)
        if (!(p[a] + 1 == rg.hi[a])) col32.push_back(static_cast<int>(r + stride[a]));
    }
    rp[r + 1] = static_cast<std::int64_t>(col32.size());
  }
  g_nnz = static_cast<long long>(col32.size());
  g_rp.upload(rp, eng.stream);
  g_col.upload(col32, eng.stream);
  g_val.alloc(col32.size());
  DBuf<std::int64_t> col64;
  col64.upload(std::vector<std::int64_t>(col32.begin(), col32.end()), eng.stream);
  std::vector<Complex> tab;
  std::array<long long, 6> off{};
  for (int a = 0; a < dim; ++a) {
    off[2 * a] = static_cast<long long>(tab.size());
    tab.insert(tab.end(), gcoeffs.node[a].begin(), gcoeffs.node[a].end());
    off[2 * a + 1] = static_cast<long long>(tab.size());
    tab.insert(tab.end(), gcoeffs.half[a].begin(), gcoeffs.half[a].end());
  }
  DBuf<double2> gtab;
  gtab.alloc(tab.size());
  HS_CUDA(cudaMemcpyAsync(gtab.p, tab.data(), tab.size() * sizeof(Complex), cudaMemcpyHostToDevice, eng.stream));
  DBuf<unsigned long long> flags;
  flags.alloc(2);
  flags.zero(eng.stream);
  AsmSub g{};
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = a < dim ? rg.lo[a] : 0;
    g.size[a] = a < dim ? rg.size(a) : 1;
    g.cell_lo[a] = interior.lo[a];
    g.cell_hi[a] = interior.hi[a];
    g.anode[a] = a < dim ? gtab.p + off[2 * a] : nullptr;
    g.ahalf[a] = a < dim ? gtab.p + off[2 * a + 1] : nullptr;
  }
  g.row_ptr = g_rp.p;
  g.col = col64.p;
  g.val = g_val.p;
  g.maxabs = flags.p;
  DBuf<AsmSub> dg;
  dg.upload(std::vector<AsmSub>{g}, eng.stream);
  AsmArgs args{};
  args.dim = dim;
  for (int a = 0; a < 3; ++a) {
    args.h[a] = ggrid.h[a];
    args.origin[a] = ggrid.origin[a];
  }
  args.med = asm_medium();
  args.subs = dg.p;
  args.nsub = 1;
  args.bad = reinterpret_cast<unsigned*>(flags.p + 1);
  launch_assemble(args, n, eng.stream);
  HS_CUDA(cudaStreamSynchronize(eng.stream));
  build_stencil_op();
  gop_ready = true;
}

// The global operator's values regrouped by stencil offset (column order: -stride[dim-1] ... -1, 0,
// +1 ... +stride[dim-1]), so the residual kernel's loads are independent (hs_kernels.cu). Dropped
// (the CSR kernels are used) when memory is short or an entry is off the stencil.
void DdmHandle::build_stencil_op() {
  g_sop = StencilOp();
  if (std::getenv("HS_NO_STENCIL_OP")) return;  // developer A/B switch
  const GridRange& rg = ggrid.range;
  const long long n = rg.count();
  StencilOp op;
  op.S = 2 * dim + 1;
  long long stride[3] = {1, 1, 1};
  for (int a = 1; a < dim; ++a) stride[a] = stride[a - 1] * rg.size(a - 1);
  for (int a = 0; a < dim; ++a) {
    op.off[dim - 1 - a] = -stride[a];
    op.off[dim + 1 + a] = stride[a];
  }
  op.off[dim] = 0;
  size_t free_b = 0, total_b = 0;
  HS_CUDA(cudaMemGetInfo(&free_b, &total_b));
  if (static_cast<double>(n) * op.S * sizeof(double2) > 0.05 * static_cast<double>(free_b)) return;
  g_sten.alloc(static_cast<size_t>(n) * op.S);
  DBuf<unsigned> bad;
  bad.alloc(1);
  bad.zero(eng.stream);
  launch_stencil_build(n, g_rp.p, g_col.p, g_val.p, op, g_sten.p, bad.p, eng.stream);
  unsigned hbad = 0;
  HS_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(unsigned), cudaMemcpyDeviceToHost, eng.stream));
  HS_CUDA(cudaStreamSynchronize(eng.stream));
  if (hbad) return;
  op.val = g_sten.p;
  g_sop = op;
}

// One DDM application on bN -> u (node-major), src/sweeper.cpp:176-334.
void DdmHandle::run(int nrounds, bool track, bool timed, const StreamIO* io) {
  // caller callbacks (host-side transport) cannot be captured; the native NCCL transport can
  if (io || (partitioned() && !ncomm) || !use_graph || std::getenv("HS_TRACE")) {
    run_body(nrounds, track, timed, io);
    return;
  }
  if (track) ensure_gop();  // synchronous setup stays outside the capture
  const long long gen = state_gen * 1000003LL + eng.gen;
  AppGraph* hit = nullptr;
  for (auto& g : graphs)
    if (g.rounds == nrounds && g.track == track && g.timed == timed && g.gen == gen) hit = &g;
  if (!hit) {
    for (auto& g : graphs)
      if (g.gen != gen) {  // buffers were reallocated since: every graph is stale
        drop_graphs();
        break;
      }
    cudaStream_t s = eng.stream;
    const long long l0 = g_kernel_launches.load();
    cudaGraph_t graph = nullptr;
    HS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    bool ok = true;
    capturing = true;
    std::exception_ptr err;
    try {
      run_body(nrounds, track, timed, nullptr);
    } catch (const Error&) {
      ok = false;
    } catch (...) {  // anything else (e.g. host allocation): end the capture, then rethrow
      ok = false;
      err = std::current_exception();
    }
    capturing = false;
    const cudaError_t ec = cudaStreamEndCapture(s, &graph);
    if (err) {
      if (graph) cudaGraphDestroy(graph);
      (void)cudaGetLastError();
      g_kernel_launches.fetch_sub(g_kernel_launches.load() - l0);
      std::rethrow_exception(err);
    }
    AppGraph g{nrounds, track, timed, gen, g_kernel_launches.load() - l0, nullptr};
    g_kernel_launches.fetch_sub(g.launches);  // counted when the graph runs
    if (ok && ec == cudaSuccess && graph && cudaGraphInstantiate(&g.exec, graph, 0) == cudaSuccess) {
      cudaGraphDestroy(graph);
      graphs.push_back(g);
    } else {  // capture unsupported here: launch stream by stream from now on
      if (graph) cudaGraphDestroy(graph);
      (void)cudaGetLastError();
      use_graph = false;
      run_body(nrounds, track, timed, nullptr);
      return;
    }
    hit = &graphs.back();
  }
  HS_CUDA(cudaGraphLaunch(hit->exec, eng.stream));
  g_kernel_launches.fetch_add(hit->launches);
}

void DdmHandle::run_body(int nrounds, bool track, bool timed, const StreamIO* io) {
  cudaStream_t s = eng.stream;
  const int nsub = geom.nsub;
  if (track) ensure_gop();
  // (the fused accumulate writes every node of u, region by region)
  if (!fuse_acc || partitioned()) HS_CUDA(cudaMemsetAsync(u.p, 0, u.n * sizeof(double2), s));
  HS_CUDA(cudaMemsetAsync(mpres.p, 0, mpres.n * sizeof(rmask), s));
  HS_CUDA(cudaMemsetAsync(nzmask.p, 0, nzmask.n * sizeof(rmask), s));
  HS_CUDA(cudaMemsetAsync(tface.p, 0, tface.n * sizeof(unsigned), s));
  if (timed) record(ev[0], s);
  SweepArgs sa{};
  sa.g = geom;
  sa.cls = eng.d_cls.p;
  sa.subs = eng.d_subs.p;
  sa.R = R;
  sa.nsweeps = nsweeps;
  sa.dirs = dirs;
  sa.nbuf = nbuf;
  sa.xstride = eng.xstride;
  sa.b = bN.p;
  sa.mbox = mbox.p;
  sa.mbox_dir_stride = 2 * line_max * R;
  sa.mpres = mpres.p;
  sa.nzmask = nzmask.p;
  sa.tface = tface.p;
  sa.route = route.p;
  sa.rbs = eng.rb.p;
  sa.slot_stride = eng.slot_stride;
  // slots start clean every application (their previous occupants are then within it)
  HS_CUDA(cudaMemsetAsync(eng.rb.p, 0, eng.rb.n * sizeof(double2), s));
  const int nm = static_cast<int>(msteps.size());
  int waited = 0, stripes_done = 0;  // waited: tiles of b staged (copy order)
  bool u_reduced = false;
  static const bool no_skip = std::getenv("HS_NO_FRONT_SKIP") != nullptr;  // developer A/B switch
  // the backward's unread fronts are pruned from the item lists (build_items); the run-time check
  // of the need bitset is only needed without that pruning
  static const bool no_prune = std::getenv("HS_NO_PRUNE") != nullptr;
  auto stage_in = [&](int upto) {  // tiles [waited, upto) of b: copied -> transposed into bN
    for (int k = waited; k < upto; ++k) {
      const InTile& t = in_tiles[k];
      HS_CUDA(cudaStreamWaitEvent(s, io->copied[k], 0));
      launch_transpose_in_tile(io->din, bN.p, geom.gn, R, geom.gsize[0], t.x0, t.x1, t.row0, t.row1, s,
                               perm_on ? rperm.p : nullptr);
    }
    waited = std::max(waited, upto);
  };
  const std::vector<OutRegion>& regs = out_regions(io != nullptr);
  const int gx = geom.gsize[0];
  auto reg_cnt = [&](const OutRegion& o) { return (o.row1 - o.row0) * (o.x1 - o.x0); };
  std::vector<int> stripe_blocks(regs.size(), 0);
  auto stripe_pbase = [&](int j) {  // partial blocks of the regions before j (exact: one block per npb nodes)
    const int npb = fuse_acc ? 256 / ((R + 1) / 2) : 256 / R;  // (the fused pass runs a thread per RHS pair)
    long long b = 0;
    for (int q = 0; q < j; ++q) b += (reg_cnt(regs[q]) + npb - 1) / npb;
    return b;
  };
  for (int m = 0; m < nm; ++m) {
    if (io && need_tiles[m] > waited) stage_in(need_tiles[m]);  // streamed b: the tiles this step's sources read
    sa.tasks = d_mtasks.p + mt_off[m];
    sa.prev = d_prev.p + mt_off[m];
    sa.ntasks = static_cast<int>(msteps_own[m].size());
    if (sa.ntasks > 0) {
      // tasks past sweep 1 touch only their injection lines: size the init grid for that
      bool full = false;
      // (a sweep-1 task writes its whole slot, and so does any task whose slot's previous occupant did)
      for (size_t t = 0; t < msteps_own[m].size(); ++t) full |= msteps_own[m][t].y == 1 || prev_h[mt_off[m] + t].y == 1;
      launch_build_rhs(sa, full ? eng.n_max : 0, static_cast<int>(line_max), s);
    }
    if (timed) record(ev[1 + nsweeps + 2 * m], s);
    const char* tstep = std::getenv("HS_TRACE_STEP");
    const bool traced = std::getenv("HS_TRACE") && m == (tstep ? std::atoi(tstep) : nm / 2);
    if (sa.ntasks > 0)
      eng.run_solve(d_tasks.p + fwd_off[m], fwd_cnt[m], d_tasks.p + bwd_off[m], bwd_cnt[m], nzmask.p, traced,
                    no_skip ? nullptr : tface.p, no_skip || !no_prune ? nullptr : need.p, need_words);
    if (timed) record(ev[2 + nsweeps + 2 * m], s);
    if (sa.ntasks > 0) launch_extract_deposit(sa, static_cast<int>(line_max), s);
    if (partitioned() && !xplan[m].peers.empty()) {  // traces and ghost values to / from other ranks
      const XPlan& xp = xplan[m];
      launch_xpack(d_xseg.p + xp.s0, xp.ns, true, xsend.p, mbox.p, mpres.p, eng.x.p, nzmask.p, d_gpos.p, R, s);
      if (ncomm) {
        ncomm->exchange(static_cast<int>(xp.peers.size()), xp.peers.data(), xp.soff.data(), xp.scnt.data(),
                        xp.roff.data(), xp.rcnt.data(), xsend.p, xrecv.p, s);
      } else {
        if (!xfn) throw Error(kConfig, "partitioned solve: no exchange callback");
        if (xfn(cuser, static_cast<int>(xp.peers.size()), xp.peers.data(), xp.soff.data(), xp.scnt.data(),
                xp.roff.data(), xp.rcnt.data(), xsend.p, xrecv.p, s) != 0)
          throw Error(kCuda, "partitioned solve: exchange callback failed");
      }
      launch_xpack(d_xseg.p + xp.r0, xp.nr, false, xrecv.p, mbox.p, mpres.p, eng.x.p, nzmask.p, d_gpos.p, R, s);
    }
    auto accumulate = [&](int l, long long n0, long long n1, long long pbase) {
      AccumArgs aa{};
      aa.g = geom;
      aa.x = eng.x.p;
      aa.acc_ent = acc_ent.p + static_cast<size_t>((l - 1) % ndir) * geom.gn * (1 << dim);
      aa.R = R;
      aa.l = l;
      for (int a = 0; a < 3; ++a) aa.dvec[a] = plan[l - 1][a];
      aa.xoff = static_cast<long long>((l - 1) % nbuf) * eng.xstride;
      aa.nzmask = nzmask.p + static_cast<size_t>(l - 1) * nsub;
      aa.u = u.p;
      aa.partial = partial.p + pbase * R;
      aa.n0 = n0;
      aa.n1 = n1;
      return launch_accumulate(aa, s);
    };
    auto after_sweep = [&](int l, int nb) {  // sweep l fully accumulated (nb < 0: norms reduced already)
      if (nb >= 0) launch_reduce_partials(partial.p, nb, R, norms.p + static_cast<size_t>(l - 1) * R, s);
      if (timed) record(ev[l], s);
      if (track && l % ndir == 0) {  // per-round relative residual (src/sweeper.cpp:313-325)
        const int last = static_cast<int>(in_tiles.size());
        if (io && waited < last) stage_in(last);  // the residual reads all of b
        const int rr = l / ndir - 1;
        const double2* ures = u.p;
        if (partitioned()) {  // every node is nonzero on its home rank only: the sum is exact
          double2* t = u.p;
          if (l != nsweeps) {
            ufull.alloc(u.n);
            HS_CUDA(cudaMemcpyAsync(ufull.p, u.p, u.n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
            t = ufull.p;
          } else {
            u_reduced = true;
          }
          comm_gather_u(t);
          ures = t;
        }
        const int nb2 = launch_residual(geom.gn, g_rp.p, g_col.p, g_val.p, ures, bN.p, R, pnum.p, pden.p, s, geom.gsize[0], g_sop);
        launch_reduce_partials(pnum.p, nb2, R, rnum.p + static_cast<size_t>(rr) * R, s);
        launch_reduce_partials(pden.p, nb2, R, rden.p + static_cast<size_t>(rr) * R, s);
      }
    };
    for (int l : acc_after[m]) after_sweep(l, accumulate(l, 0, geom.gn, 0));
    if (fuse_acc && timed)  // sweeps that end here (their contributions are accumulated at the end)
      for (int l = 1; l < nsweeps; ++l)
        if (sweep_end_m[l] == m) record(ev[l], s);
    // the last sweep (every sweep, fused), stripe by stripe (partials in stripe order: a fixed
    // reduction order)
    const int nst = static_cast<int>(regs.size());
    for (int j = 0; j < nst; ++j) {
      const OutRegion& rg = regs[j];
      if (rg.acc_m != m) continue;
      if (fuse_acc) {
        AccumAllArgs aa{};
        aa.g = geom;
        aa.R = R;
        aa.L = nsweeps;
        for (int l = 1; l <= nsweeps; ++l) {
          aa.acc_ent[l - 1] = acc_ent.p + static_cast<size_t>((l - 1) % ndir) * geom.gn * (1 << dim);
          aa.xoff[l - 1] = static_cast<long long>((l - 1) % nbuf) * eng.xstride;
          aa.nzmask[l - 1] = nzmask.p + static_cast<size_t>(l - 1) * nsub;
        }
        aa.x = eng.x.p;
        aa.u = u.p;
        if (track && nrounds > 1) {
          aa.uround = uround.p;
          aa.rstride = geom.gn * R;
          aa.rlen = ndir;
        }
        aa.partial = partial.p + stripe_pbase(j) * R;
        aa.pstride = partial_stride;
        aa.row0 = rg.row0;
        aa.cnt = reg_cnt(rg);
        aa.gx = gx;
        aa.x0 = rg.x0;
        aa.w = rg.x1 - rg.x0;
        stripe_blocks[j] = launch_accumulate_all(aa, s);
      } else {  // regions are the stripes here
        stripe_blocks[j] = accumulate(nsweeps, rg.row0 * gx, rg.row1 * gx, stripe_pbase(j));
      }
      if (io)
        launch_transpose_out_tile(u.p, io->dout, geom.gn, R, gx, rg.x0, rg.x1, rg.row0, rg.row1, s,
                                  perm_on ? rperm.p : nullptr);
      record(ev_out[j], s);
      if (++stripes_done == nst) {
        int nbt = 0;
        for (int q = 0; q < nst; ++q) nbt += stripe_blocks[q];
        if (fuse_acc) {
          for (int l = 1; l <= nsweeps; ++l)
            launch_reduce_partials(partial.p + (l - 1) * partial_stride, nbt, R, norms.p + static_cast<size_t>(l - 1) * R, s);
          if (track)  // residuals of the rounds before the last, on u as it stood after each of them
            for (int q = 0; q + 1 < nrounds; ++q) {
              double2* uq = uround.p + static_cast<size_t>(q) * geom.gn * R;
              if (partitioned()) comm_gather_u(uq);
              const int nb2 = launch_residual(geom.gn, g_rp.p, g_col.p, g_val.p, uq, bN.p, R, pnum.p, pden.p, s, geom.gsize[0], g_sop);
              launch_reduce_partials(pnum.p, nb2, R, rnum.p + static_cast<size_t>(q) * R, s);
              launch_reduce_partials(pden.p, nb2, R, rden.p + static_cast<size_t>(q) * R, s);
            }
          after_sweep(nsweeps, -1);
        } else {
          after_sweep(nsweeps, nbt);
        }
      }
    }
  }
  if (partitioned()) {  // home-node slices of u, and the per-sweep |contribution|^2 sums
    if (!u_reduced) comm_gather_u(u.p);
    comm_allreduce(norms.p, static_cast<long long>(nsweeps) * R);
  }
}

// SolveReport per RHS: counters replayed from the device's per-task nonzero masks in the
// reference's canonical order (src/sweeper.cpp:285-307).
void DdmHandle::reports(int nrounds, bool track, hs_solve_report* out) {
  const int nsub = geom.nsub;
  std::vector<rmask> nz(static_cast<size_t>(nsweeps) * nsub);
  std::vector<double> nrm(static_cast<size_t>(nsweeps) * R), num(static_cast<size_t>(nrounds) * R),
      den(static_cast<size_t>(nrounds) * R);
  if (perm_on && !perm_host) {  // internal column j is the caller's column perm_h[j]
    perm_h.resize(R);
    HS_CUDA(cudaMemcpyAsync(perm_h.data(), rperm.p, R * sizeof(int), cudaMemcpyDeviceToHost, eng.stream));
  }
  HS_CUDA(cudaMemcpyAsync(nz.data(), nzmask.p, nz.size() * sizeof(rmask), cudaMemcpyDeviceToHost, eng.stream));
  HS_CUDA(cudaMemcpyAsync(nrm.data(), norms.p, nrm.size() * sizeof(double), cudaMemcpyDeviceToHost, eng.stream));
  if (track) {
    HS_CUDA(cudaMemcpyAsync(num.data(), rnum.p, num.size() * sizeof(double), cudaMemcpyDeviceToHost, eng.stream));
    HS_CUDA(cudaMemcpyAsync(den.data(), rden.p, den.size() * sizeof(double), cudaMemcpyDeviceToHost, eng.stream));
  }
  HS_CUDA(cudaStreamSynchronize(eng.stream));
  if (partitioned()) {  // every task's mask from its owner (ghost copies are dropped first); the sum
                        // over ranks runs on the two 32-bit halves of each mask (exact in doubles)
    std::vector<double> w(2 * nz.size());
    for (int l = 1; l <= nsweeps; ++l)
      for (int id = 0; id < nsub; ++id) {
        const size_t i = static_cast<size_t>(l - 1) * nsub + id;
        const bool mine = owner[id] == rank;
        w[2 * i] = mine ? static_cast<double>(nz[i] & 0xffffffffull) : 0.0;
        w[2 * i + 1] = mine ? static_cast<double>(nz[i] >> 32) : 0.0;
      }
    dtmp.alloc(w.size());
    HS_CUDA(cudaMemcpyAsync(dtmp.p, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice, eng.stream));
    comm_allreduce(dtmp.p, static_cast<long long>(w.size()));
    HS_CUDA(cudaMemcpyAsync(w.data(), dtmp.p, w.size() * sizeof(double), cudaMemcpyDeviceToHost, eng.stream));
    HS_CUDA(cudaStreamSynchronize(eng.stream));
    for (size_t i = 0; i < nz.size(); ++i)
      nz[i] = static_cast<rmask>(w[2 * i]) | (static_cast<rmask>(w[2 * i + 1]) << 32);
  }
  const int nm = static_cast<int>(msteps.size());
  std::vector<double> sweep_sec(nsweeps, 0.0), step_sec(nm, 0.0);
  std::vector<int> active(nm, 0);
  float ms = 0.f;
  for (int m = 0; m < nm; ++m) {
    HS_CUDA(cudaEventElapsedTime(&ms, ev[1 + nsweeps + 2 * m], ev[2 + nsweeps + 2 * m]));
    step_sec[m] = ms * 1e-3;
    for (const int2& t : msteps_own[m]) active[m] += nz[static_cast<size_t>(t.y - 1) * nsub + t.x] != 0;
  }
  for (int l = 1; l <= nsweeps; ++l) {  // from the sweep's first macro-step to its accumulate
    HS_CUDA(cudaEventElapsedTime(&ms, ev[1 + nsweeps + 2 * sweep_first_m[l]], ev[l]));
    sweep_sec[l - 1] = ms * 1e-3;
  }
  if (const char* path = std::getenv("HS_DUMP_NZ")) {  // developer instrumentation: per-task nonzero RHS masks
    if (FILE* fp = std::fopen(path, "w")) {
      std::fprintf(fp, "sweep,sub,mask\n");
      for (int l = 1; l <= nsweeps; ++l)
        for (int id = 0; id < nsub; ++id)
          std::fprintf(fp, "%d,%d,%llx\n", l, id, static_cast<unsigned long long>(nz[static_cast<size_t>(l - 1) * nsub + id]));
      std::fclose(fp);
    }
  }
  if (const char* path = std::getenv("HS_STEP_TIMES")) {  // developer instrumentation
    if (FILE* fp = std::fopen(path, "w")) {
      std::fprintf(fp, "mstep,ntasks,active,solve_us\n");
      for (int m = 0; m < nm; ++m)
        std::fprintf(fp, "%d,%d,%d,%.2f\n", m, static_cast<int>(msteps[m].size()), active[m], 1e6 * step_sec[m]);
      std::fclose(fp);
    }
  }
  double total = 0.0;
  HS_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[nsweeps]));
  total = ms * 1e-3;
  for (int r = 0; r < R; ++r) {
    hs_solve_report& rep = out[perm_on || perm_host ? perm_h[r] : r];
    std::memset(&rep, 0, sizeof(rep));
    rep.factor_seconds = factor_seconds;
    rep.sweep_seconds_total = total;
    rep.n_sweeps = nsweeps;
    std::vector<double> task_times;
    for (int l = 1; l <= nsweeps; ++l) {
      const int di = (l - 1) % ndir;
      rep.sweep_seconds[l - 1] = sweep_sec[l - 1];
      rep.sweep_contrib_norm[l - 1] = std::sqrt(nrm[static_cast<size_t>(l - 1) * R + r]);
      for (int st = 1; st <= steps; ++st) {
        const auto& grp = groups[di * steps + st - 1];
        for (int id : grp) {
          const bool nonzero = (nz[static_cast<size_t>(l - 1) * nsub + id] >> r) & 1ull;
          if (!nonzero) {
            ++rep.skipped_zero_solves;
            continue;
          }
          ++rep.local_solves;
          const int m = mstep_of[static_cast<size_t>(l - 1) * nsub + id];
          task_times.push_back(step_sec[m] / std::max(active[m], 1));
          const Vec3i sb = subs[id].sub;
          for (int d = 0; d < dirs; ++d) {
            if (!part.has_neighbor(sb, d / 2, (d & 1) ? 1 : -1)) continue;
            ++rep.traces_generated;
            if (route_h[(l - 1) * dirs + d] == 0)
              ++rep.traces_discarded;
            else
              ++rep.traces_routed;
          }
        }
      }
    }
    if (!task_times.empty()) {
      std::sort(task_times.begin(), task_times.end());
      rep.median_subdomain_solve_seconds = task_times[task_times.size() / 2];
    }
    if (track) {
      rep.n_round_residuals = nrounds;
      for (int q = 0; q < nrounds; ++q) {
        const double dd = den[static_cast<size_t>(q) * R + r];
        rep.round_residuals[q] = dd > 0 ? std::sqrt(num[static_cast<size_t>(q) * R + r] / dd) : 0.0;
      }
    }
  }
}

// Column order of a batch. Tasks skip RHS groups that are exactly zero for them (hs_solve.cu); with
// the columns ordered by where their sources are, the columns of a group reach a subdomain together.
static bool rhs_sort_enabled() {
  static const bool off = std::getenv("HS_NO_RHS_SORT") != nullptr;  // developer A/B switch
  return !off;
}

const int* DdmHandle::order_device(const double2* d_b, int nr) {
  perm_host = false;
  perm_on = rhs_sort_enabled() && nr >= 16 && !partitioned();
  if (!perm_on) return nullptr;
  rperm.alloc(kMaxRhs);
  rbbox.alloc(6 * kMaxRhs);
  launch_rhs_order(d_b, geom.gn, nr, geom, rbbox.p, rperm.p, eng.stream);
  return rperm.p;
}

// The same order for a batch of the streamed host-buffer path, from samples of the host buffer
// (every 32nd node of every 32nd grid row: well under a millisecond on the host cores), taken
// while the batch's first tiles are already on their way to the device. Ordering across the
// batches of a call would cluster better, but then every tile is one copy per column: measured
// 403 ms against 207 ms per 64-RHS C3 call (32 K cudaMemcpy3DAsync calls).
const int* DdmHandle::order_host(const double* b, int nr) {
  perm_host = perm_on = rhs_sort_enabled() && nr >= 16 && !partitioned();
  if (!perm_on) return nullptr;
  const long long n = geom.gn;
  const int gx = geom.gsize[0], gy = dim > 1 ? geom.gsize[1] : 1;
  const long long rows = n / gx;
  std::vector<unsigned> key(nr);
  parallel_for(nr, [&](long long r) {
    int bb[6] = {INT_MAX, INT_MAX, INT_MAX, -1, -1, -1};
    const double* br = b + 2 * r * n;
    for (long long row = 0; row < rows; row += 32)
      for (int x = 0; x < gx; x += 32) {
        const double* v = br + 2 * (row * gx + x);
        if (v[0] != 0.0 || v[1] != 0.0) {
          const int c[3] = {x, static_cast<int>(row % gy), static_cast<int>(row / gy)};
          for (int a = 0; a < 3; ++a) {
            bb[a] = std::min(bb[a], c[a]);
            bb[3 + a] = std::max(bb[3 + a], c[a]);
          }
        }
      }
    key[r] = rhs_order_key(geom, bb);
  });
  perm_h.resize(nr);
  for (int r = 0; r < nr; ++r) perm_h[r] = r;
  std::stable_sort(perm_h.begin(), perm_h.end(), [&](int x, int y) { return key[x] < key[y]; });
  rperm.alloc(kMaxRhs);
  HS_CUDA(cudaMemcpyAsync(rperm.p, perm_h.data(), nr * sizeof(int), cudaMemcpyHostToDevice, eng.stream));
  return rperm.p;
}

// One batch from / to pinned host buffers with the transfers overlapped: b streams in by tiles
// (stripe of the slowest axis x segment of the fastest), in the order the sweep-1 sources first
// read them, while the first macro-steps run; u streams out by regions (tiles when the accumulate
// is fused, else stripes) as the tail of the application completes them. One copy stream per
// direction; the copy streams carry copies only, never kernels.
void DdmHandle::solve_streamed(int nr, const double* b, double* uh, int nrounds, bool track, hs_solve_report* reps,
                               int slot, bool last, int cap) {
  ensure_state(nr, nrounds);
  const long long n = geom.gn;
  const int nt = static_cast<int>(in_tiles.size());
  for (auto& c : cs)
    if (!c) HS_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
  while (static_cast<int>(ev_in.size()) < nt + 1 + kCopyStreams) {
    cudaEvent_t e;
    HS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev_in.push_back(e);
  }
  for (int q = 0; q < 2; ++q)
    for (cudaEvent_t* e : {&ev_din_free[q], &ev_dout_free[q]})
      if (!*e) {
        HS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        HS_CUDA(cudaEventRecord(*e, eng.stream));
      }
  // Two staging slots (din, dout) so consecutive batches overlap: batch k + 1's b streams in while
  // batch k computes, and batch k's u streams out while batch k + 1 computes. A slot is reused two
  // batches later, after the application that read its din and the copies that read its dout.
  cap = std::max(cap, nr);  // RHS per staging slot: the call's widest batch
  io.alloc(static_cast<size_t>(n) * cap * 4);
  double2* din = io.p + static_cast<size_t>(slot) * 2 * n * cap;
  double2* dout = din + static_cast<size_t>(n) * cap;
  HS_CUDA(cudaStreamWaitEvent(cs[0], ev_din_free[slot], 0));
  HS_CUDA(cudaStreamWaitEvent(eng.stream, ev_dout_free[slot], 0));
  const size_t gx = static_cast<size_t>(geom.gsize[0]), rows = static_cast<size_t>(n) / gx;
  auto copy3d = [&](const void* src, void* dst, int x0, int x1, long long r0, long long r1, cudaMemcpyKind kind,
                    cudaStream_t st) {  // (x, rows, RHS) box of the RHS-major grid
    cudaMemcpy3DParms c{};
    c.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), gx * sizeof(double2), gx * sizeof(double2), rows);
    c.dstPtr = make_cudaPitchedPtr(dst, gx * sizeof(double2), gx * sizeof(double2), rows);
    c.srcPos = c.dstPos = make_cudaPos(x0 * sizeof(double2), static_cast<size_t>(r0), 0);
    c.extent = make_cudaExtent(static_cast<size_t>(x1 - x0) * sizeof(double2), static_cast<size_t>(r1 - r0),
                               static_cast<size_t>(nr));
    c.kind = kind;
    HS_CUDA(cudaMemcpy3DAsync(&c, st));
  };
  auto copy_in = [&](const cudaEvent_t* evs) {  // tiles of b in need order
    for (int k = 0; k < nt; ++k) {
      const InTile& t = in_tiles[k];
      copy3d(b, din, t.x0, t.x1, t.row0, t.row1, cudaMemcpyHostToDevice, cs[0]);
      HS_CUDA(cudaEventRecord(evs[k], cs[0]));
    }
  };
  copy_in(ev_in.data());
  order_host(b, nr);  // (the tile copies are already queued: the sampling overlaps them)
  const StreamIO sio{ev_in.data(), din, dout};
  run(nrounds, track, true, &sio);
  HS_CUDA(cudaEventRecord(ev_din_free[slot], eng.stream));
  // each region of u is transposed out after its accumulate of the last sweep (ev_out); copy the
  // regions to the host in the order they complete, while the tail of the application still runs
  const std::vector<OutRegion>& regs = out_regions(true);
  const int no = static_cast<int>(regs.size());
  std::vector<int> order(no);
  for (int j = 0; j < no; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return regs[x].acc_m < regs[y].acc_m; });
  auto copy_out = [&](int q, const cudaEvent_t* fin, const cudaEvent_t* done) {
    const int j = order[q];
    const OutRegion& o = regs[j];
    cudaStream_t st = cs[1];
    HS_CUDA(cudaStreamWaitEvent(st, ev_out[j], 0));
    if (fin) HS_CUDA(cudaEventRecord(fin[j], st));
    copy3d(dout, uh, o.x0, o.x1, o.row0, o.row1, cudaMemcpyDeviceToHost, st);
    if (done) HS_CUDA(cudaEventRecord(done[j], st));
  };
  for (int q = 0; q < no; ++q) copy_out(q, nullptr, nullptr);
  HS_CUDA(cudaEventRecord(ev_dout_free[slot], cs[1]));
  if (last)
    for (int c = 0; c < kCopyStreams; ++c) {  // later work may reuse io / u
      HS_CUDA(cudaEventRecord(ev_in[nt + 1 + c], cs[c]));
      HS_CUDA(cudaStreamWaitEvent(eng.stream, ev_in[nt + 1 + c], 0));
    }
  if (const char* path = std::getenv("HS_STREAM_TRACE")) {  // developer timeline (timing events)
    // te: [0] start, [1, 1 + nt) tile copied, then per region u final / copied out, then compute end
    std::vector<cudaEvent_t> te(nt + 2 * no + 2);
    const int uf = 1 + nt, ud = 1 + nt + no, ce = 1 + nt + 2 * no;
    // re-run the same schedule with timing events
    for (auto c : cs) HS_CUDA(cudaStreamSynchronize(c));
    HS_CUDA(cudaStreamSynchronize(eng.stream));
    for (auto& e : te) HS_CUDA(cudaEventCreate(&e));
    HS_CUDA(cudaEventRecord(te[0], eng.stream));
    for (auto c : cs) HS_CUDA(cudaStreamWaitEvent(c, te[0], 0));
    copy_in(te.data() + 1);
    const StreamIO tio{te.data() + 1, din, dout};
    run(nrounds, track, true, &tio);
    for (int q = 0; q < no; ++q) copy_out(q, te.data() + uf, te.data() + ud);
    HS_CUDA(cudaEventRecord(te[ce], eng.stream));
    for (auto c : cs) HS_CUDA(cudaStreamSynchronize(c));
    HS_CUDA(cudaStreamSynchronize(eng.stream));
    if (FILE* fp = std::fopen(path, "w")) {
      float t = 0.f;
      std::fprintf(fp, "what,index,ms\n");
      for (int k = 0; k < nt; ++k) {
        cudaEventElapsedTime(&t, te[0], te[1 + k]);
        std::fprintf(fp, "h2d_done,%d,%.3f\n", k, t);
      }
      for (int j = 0; j < no; ++j) {
        cudaEventElapsedTime(&t, te[0], te[uf + j]);
        std::fprintf(fp, "u_final,%d,%.3f\n", j, t);
        cudaEventElapsedTime(&t, te[0], te[ud + j]);
        std::fprintf(fp, "d2h_done,%d,%.3f\n", j, t);
      }
      for (size_t m = 0; m < msteps.size(); ++m) {
        cudaEventElapsedTime(&t, te[0], ev[1 + nsweeps + 2 * m]);
        std::fprintf(fp, "mstep_solve_start,%zu,%.3f\n", m, t);
      }
      cudaEventElapsedTime(&t, te[0], te[ce]);
      std::fprintf(fp, "compute_end,0,%.3f\n", t);
      std::fclose(fp);
    }
    for (auto e : te) cudaEventDestroy(e);
  }
  if (reps) reports(nrounds, track, reps);
  if (last) {
    for (auto c : cs) HS_CUDA(cudaStreamSynchronize(c));
    HS_CUDA(cudaStreamSynchronize(eng.stream));
  }
}

}  // namespace hsb

struct hs_ddm {
  hsb::DdmHandle h;
};

namespace {

constexpr int kStreamBatch = 32;  // RHS per batch of the streamed host-buffer path

void ddm_solve_batch(DdmHandle& H, int R, const double2* d_b, double2* d_u, int rounds, bool track,
                     hs_solve_report* reps) {
  H.ensure_state(R, rounds);
  const int* perm = H.order_device(d_b, R);
  launch_transpose_in(d_b, H.bN.p, H.geom.gn, R, H.eng.stream, perm);
  H.run(rounds, track, true);
  launch_transpose_out(H.u.p, d_u, H.geom.gn, R, H.eng.stream, perm);
  if (reps) H.reports(rounds, track, reps);
}

}  // namespace

extern "C" int hs_ddm_create(const hs_problem* setup, int device, hs_ddm** out, int* pivot_sub,
                             int64_t* pivot_index) {
  std::unique_ptr<hs_ddm> s;
  const int rc = guarded(
      [&] {
        if (!setup || !out) config_error("hs_ddm_create: null argument");
        s = std::make_unique<hs_ddm>();
        s->h.build(*setup, device);
      },
      pivot_sub, pivot_index);
  if (rc != kOk) return rc;
  *out = s.release();
  return kOk;
}

extern "C" void hs_ddm_destroy(hs_ddm* s) { delete s; }

extern "C" int hs_ddm_create_partitioned(const hs_problem* setup, int device, int rank, int world, const int* owner,
                                         hs_exchange_fn exchange, hs_allreduce_fn allreduce, void* user, hs_ddm** out,
                                         int* pivot_sub, int64_t* pivot_index) {
  std::unique_ptr<hs_ddm> s;
  const int rc = guarded(
      [&] {
        if (!setup || !out) config_error("hs_ddm_create_partitioned: null argument");
        if (world > 1 && (!exchange || !allreduce)) config_error("hs_ddm_create_partitioned: missing callbacks");
        s = std::make_unique<hs_ddm>();
        s->h.xfn = exchange;
        s->h.arfn = allreduce;
        s->h.cuser = user;
        s->h.build(*setup, device, rank, world, owner);
      },
      pivot_sub, pivot_index);
  if (rc != kOk) return rc;
  *out = s.release();
  return kOk;
}

extern "C" int hs_ddm_sub_csr(const hs_ddm* s, int sub, int64_t* row_ptr, int64_t* col, double* val, int64_t* n,
                              int64_t* nnz) {
  return guarded([&] {
    if (!s) config_error("hs_ddm_sub_csr: null handle");
    const DdmHandle& H = s->h;
    if (sub < 0 || sub >= static_cast<int>(H.subs.size())) config_error("hs_ddm_sub_csr: subdomain out of range");
    if (!H.eng.owns(sub)) config_error("hs_ddm_sub_csr: subdomain owned by another rank");
    const SymbolicClass& c = *H.eng.classes[H.subs[sub].cls]->sym;
    if (n) *n = c.n;
    if (nnz) *nnz = static_cast<int64_t>(c.csr_col.size());
    if (row_ptr) std::copy(c.csr_row_ptr.begin(), c.csr_row_ptr.end(), row_ptr);
    if (col) std::copy(c.csr_col.begin(), c.csr_col.end(), col);
    if (val) {
      HS_CUDA(cudaSetDevice(H.eng.device));
      HS_CUDA(cudaMemcpy(val, H.eng.val.p + H.eng.val_base[sub], c.csr_col.size() * sizeof(double2),
                         cudaMemcpyDeviceToHost));
    }
  });
}

extern "C" int hs_nccl_unique_id(unsigned char id[128]) {
  return guarded([&] {
    if (!id) config_error("hs_nccl_unique_id: null argument");
    nccl_unique_id(id);
  });
}

extern "C" int hs_nccl_version(int* version) {
  return guarded([&] {
    if (!version) config_error("hs_nccl_version: null argument");
    *version = nccl_version();
  });
}

extern "C" int hs_ddm_create_nccl(const hs_problem* setup, int device, int rank, int world, const int* owner,
                                  const unsigned char id[128], hs_ddm** out, int* pivot_sub, int64_t* pivot_index) {
  std::unique_ptr<hs_ddm> s;
  const int rc = guarded(
      [&] {
        if (!setup || !out || !id) config_error("hs_ddm_create_nccl: null argument");
        if (world < 1 || rank < 0 || rank >= world) config_error("partition: rank out of range");
        s = std::make_unique<hs_ddm>();
        HS_CUDA(cudaSetDevice(device));
        s->h.ncomm = std::make_unique<NcclComm>(id, rank, world);  // collective over the ranks
        s->h.build(*setup, device, rank, world, owner);
      },
      pivot_sub, pivot_index);
  if (rc != kOk) return rc;
  *out = s.release();
  return kOk;
}

extern "C" int hs_ddm_partition_info(const hs_ddm* s, int* rank, int* world, int* owned, int64_t* sent_doubles,
                                     int64_t* messages) {
  if (!s) return kConfig;
  const DdmHandle& H = s->h;
  if (rank) *rank = H.rank;
  if (world) *world = H.world;
  if (owned) *owned = static_cast<int>(std::count(H.owner.begin(), H.owner.end(), H.rank));
  if (sent_doubles) *sent_doubles = H.x_sent;
  if (messages) *messages = H.x_msgs;
  return kOk;
}

namespace {
Vec3i counts_of(int dim, const int counts[3]) {
  if (dim != 2 && dim != 3) config_error("Box: dim must be 2 or 3");
  Vec3i c{1, 1, 1};
  for (int a = 0; a < dim; ++a) {
    if (counts[a] < 1) config_error("partition: counts must be >= 1");
    c[a] = counts[a];
  }
  return c;
}
}  // namespace

extern "C" int hs_partition_owners(int dim, const int counts[3], int world, int* owner) {
  return guarded([&] {
    if (!counts || !owner || world < 1) config_error("hs_partition_owners: bad argument");
    const std::vector<int> o = default_owners(dim, counts_of(dim, counts), world);
    std::copy(o.begin(), o.end(), owner);
  });
}

extern "C" int hs_partition_traffic(int dim, const int counts[3], int rounds, int world, const int* owner,
                                    int* macro_steps, int64_t* makespan_tasks, int64_t* cross_faces,
                                    int64_t* traces) {
  return guarded([&] {
    if (!counts || !owner || world < 1 || rounds < 1) config_error("hs_partition_traffic: bad argument");
    const Vec3i c = counts_of(dim, counts);
    const int nsub = c[0] * c[1] * (dim == 3 ? c[2] : 1);
    std::vector<int> o(owner, owner + nsub);
    for (int v : o)
      if (v < 0 || v >= world) config_error("hs_partition_traffic: owner out of range");
    const PartitionCost pc = partition_cost(dim, c, rounds, world, o);
    if (macro_steps) *macro_steps = pc.macro_steps;
    if (makespan_tasks) *makespan_tasks = pc.makespan_tasks;
    if (cross_faces) *cross_faces = pc.cross_faces;
    if (traces) std::copy(pc.traces.begin(), pc.traces.end(), traces);
  });
}

extern "C" int hs_ddm_info(const hs_ddm* s, int* dim, int64_t* global_n, int* nsub, double* factor_seconds,
                           int lo[3], int hi[3]) {
  if (!s) return kConfig;
  const DdmHandle& H = s->h;
  if (dim) *dim = H.dim;
  if (global_n) *global_n = H.ggrid.range.count();
  if (nsub) *nsub = H.geom.nsub;
  if (factor_seconds) *factor_seconds = H.factor_seconds;
  for (int a = 0; a < 3; ++a) {
    if (lo) lo[a] = a < H.dim ? H.ggrid.range.lo[a] : 0;
    if (hi) hi[a] = a < H.dim ? H.ggrid.range.hi[a] : 0;
  }
  return kOk;
}

extern "C" int hs_ddm_sub_stats(const hs_ddm* s, int sub, hs_factor_stats* stats) {
  if (!s || !stats || sub < 0 || sub >= s->h.geom.nsub) return kConfig;
  *stats = s->h.sub_stats[sub];
  return kOk;
}

// DdmSolver::scale_source (src/sweeper.cpp:164-174): input marshaling on the host.
extern "C" int hs_ddm_scale_source(const hs_ddm* s, int nrhs, const double* f, double* b) {
  return guarded([&] {
    if (!s) config_error("scale_source: null handle");
    const DdmHandle& H = s->h;
    const std::int64_t n = H.ggrid.range.count();
    const Complex* fi = reinterpret_cast<const Complex*>(f);
    Complex* bo = reinterpret_cast<Complex*>(b);
    for (int r = 0; r < nrhs; ++r)
      for (std::int64_t i = 0; i < n; ++i) {
        const Vec3i p = H.ggrid.range.unlinear(i);
        bo[r * n + i] = H.ggrid.on_shell(p) ? Complex(0.0) : H.gcoeffs.jacobian(p) * fi[r * n + i];
      }
  });
}

extern "C" int hs_ddm_solve_device(hs_ddm* s, int nrhs, const double* d_b, double* d_u, int rounds,
                                   int track_residuals, hs_solve_report* reports, void* stream) {
  return guarded([&] {
    if (!s) config_error("ddm_solve: null handle");
    DdmHandle& H = s->h;
    HS_CUDA(cudaSetDevice(H.eng.device));
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    cudaEvent_t evw;
    HS_CUDA(cudaEventCreateWithFlags(&evw, cudaEventDisableTiming));
    // NULL is the legacy default stream: the solver stream is non-blocking, so order the
    // application after the caller's work there explicitly (b may be written by it)
    HS_CUDA(cudaEventRecord(evw, user ? user : cudaStreamLegacy));
    HS_CUDA(cudaStreamWaitEvent(H.eng.stream, evw, 0));
    const long long n = H.geom.gn;
    for (int b0 = 0; b0 < nrhs; b0 += kMaxRhs) {
      const int R = std::min(kMaxRhs, nrhs - b0);
      ddm_solve_batch(H, R, reinterpret_cast<const double2*>(d_b) + b0 * n, reinterpret_cast<double2*>(d_u) + b0 * n,
                      rounds, track_residuals != 0, reports ? reports + b0 : nullptr);
    }
    if (user) {
      HS_CUDA(cudaEventRecord(evw, H.eng.stream));
      HS_CUDA(cudaStreamWaitEvent(user, evw, 0));
    } else {
      HS_CUDA(cudaStreamSynchronize(H.eng.stream));
    }
    cudaEventDestroy(evw);
  });
}

extern "C" int hs_ddm_solve(hs_ddm* s, int nrhs, const double* b, double* u, int rounds, int track_residuals,
                            hs_solve_report* reports) {
  return guarded([&] {
    if (!s) config_error("ddm_solve: null handle");
    DdmHandle& H = s->h;
    HS_CUDA(cudaSetDevice(H.eng.device));
    const long long n = H.geom.gn;
    cudaPointerAttributes pa{}, pu{};
    const bool pinned = cudaPointerGetAttributes(&pa, b) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                        cudaPointerGetAttributes(&pu, u) == cudaSuccess && pu.type == cudaMemoryTypeHost;
    (void)cudaGetLastError();  // pageable pointers may leave an error on older runtimes
    if (pinned && !H.partitioned()) {  // (a partitioned u is final only after its reduction)
      // Host buffers: batches of at most kStreamBatch RHS, so that consecutive batches overlap (two
      // slots: batch k + 1's b streams in while batch k computes, batch k's u streams out while
      // batch k + 1 computes). One 64-RHS batch computes faster on the device (C3: 216 vs 228 ms)
      // but leaves its 4.6 GB of b and u each way to PCIe with nothing to overlap (e2e 345 vs 272 ms).
      int sb = kStreamBatch;
      if (const char* e = std::getenv("HS_STREAM_BATCH")) sb = std::min(kMaxRhs, std::max(1, std::atoi(e)));
      const int bw = nrhs > sb ? sb : nrhs;
      for (int b0 = 0, k = 0; b0 < nrhs; b0 += bw, ++k) {
        const int R = std::min(bw, nrhs - b0);
        H.solve_streamed(R, b + 2 * b0 * n, u + 2 * b0 * n, rounds, track_residuals != 0,
                         reports ? reports + b0 : nullptr, k & 1, b0 + bw >= nrhs, bw);
      }
      return;
    }
    for (int b0 = 0; b0 < nrhs; b0 += kMaxRhs) {
      const int R = std::min(kMaxRhs, nrhs - b0);
      const int cap = std::min(nrhs, kMaxRhs);
      H.io.alloc(static_cast<size_t>(n) * cap * 2);
      double2* din = H.io.p;
      double2* dout = H.io.p + static_cast<size_t>(n) * cap;
      HS_CUDA(cudaMemcpyAsync(din, b + 2 * b0 * n, sizeof(double2) * n * R, cudaMemcpyHostToDevice, H.eng.stream));
      ddm_solve_batch(H, R, din, dout, rounds, track_residuals != 0, reports ? reports + b0 : nullptr);
      HS_CUDA(cudaMemcpyAsync(u + 2 * b0 * n, dout, sizeof(double2) * n * R, cudaMemcpyDeviceToHost, H.eng.stream));
      HS_CUDA(cudaStreamSynchronize(H.eng.stream));
    }
  });
}

extern "C" int hs_ddm_apply_op(hs_ddm* s, int nrhs, const double* x, double* y) {
  return guarded([&] {
    if (!s) config_error("apply: null handle");
    DdmHandle& H = s->h;
    HS_CUDA(cudaSetDevice(H.eng.device));
    H.ensure_gop();
    const long long n = H.geom.gn;
    DBuf<double2> a, b2, c, d;
    a.alloc(static_cast<size_t>(n) * nrhs);
    b2.alloc(static_cast<size_t>(n) * nrhs);
    c.alloc(static_cast<size_t>(n) * nrhs);
    d.alloc(static_cast<size_t>(n) * nrhs);
    HS_CUDA(cudaMemcpyAsync(a.p, x, sizeof(double2) * n * nrhs, cudaMemcpyHostToDevice, H.eng.stream));
    launch_transpose_in(a.p, b2.p, n, nrhs, H.eng.stream);
    launch_spmv(n, H.g_rp.p, H.g_col.p, H.g_val.p, b2.p, c.p, nrhs, H.eng.stream);
    launch_transpose_out(c.p, d.p, n, nrhs, H.eng.stream);
    HS_CUDA(cudaMemcpyAsync(y, d.p, sizeof(double2) * n * nrhs, cudaMemcpyDeviceToHost, H.eng.stream));
    HS_CUDA(cudaStreamSynchronize(H.eng.stream));
  });
}

// Right-preconditioned full GMRES with MGS and complex Givens (src/krylov.cpp:17-123), the
// DDM application as preconditioner and the global operator as A (src/harness.cpp:285-305).
// One Krylov process per RHS column; the preconditioner and operator are batched.
namespace {

// Right-preconditioned GMRES with MGS and complex Givens (src/krylov.cpp:17-123), the DDM
// application as preconditioner and the global operator as A (src/harness.cpp:285-305). One
// Krylov process per RHS column; the preconditioner and operator are batched. restart >= maxit
// is the reference's full GMRES; a smaller restart runs GMRES(restart) cycles from the current
// iterate (r = b - A x recomputed, the convergence test stays |g_{j+1}| / ||b|| <= tol) until
// tol or maxit total iterations. When no restart happens the result is the full GMRES's.
// The operator / preconditioner seam of gmres(op, pc, b, cfg) (include/helmsweep/krylov.hpp:30-36):
// everything the Krylov loop needs from its two LinearOperators, on device node-major n x R arrays.
struct KrylovOps {
  int device = 0;
  cudaStream_t st = nullptr;
  long long n = 0;
  std::function<int(int)> batch;                                   // RHS per batch for an nrhs-wide call
  std::function<void(int)> prepare;                                // before a batch of R columns
  std::function<double2*(int)> pc_in;                              // a buffer the update's V y may be built in
  std::function<const double2*(const double2*, int)> pc;           // z = M^-1 v; returns z
  std::function<void(const double2*, double2*, int)> op;           // w = A z
  std::function<void(const double2*, const double2*, int, double*)> true_res;  // |b - A x|^2 per column
};

void gmres_loop(const KrylovOps& K, int nrhs, const double* b, double* x, double tol, int maxit, int restart,
                hs_gmres_report* reports) {
  if (!(tol > 0.0)) config_error("GmresConfig: tol must be positive");
  if (maxit < 1) config_error("GmresConfig: max_iterations must be >= 1");
  if (maxit + 1 > HS_MAX_GMRES_HISTORY) config_error("gmres: maxit too large for the report");
  if (restart < 1) config_error("gmres: restart must be >= 1");
  const int mk = std::min(restart, maxit);  // Krylov basis per cycle
  HS_CUDA(cudaSetDevice(K.device));
  cudaStream_t st = K.st;
  const long long n = K.n;
  const int rmax = std::max(1, K.batch(nrhs));
  for (int b0 = 0; b0 < nrhs; b0 += rmax) {
    const int R = std::min(rmax, nrhs - b0);
    K.prepare(R);
    const size_t nr = static_cast<size_t>(n) * R;
    DBuf<double2> Bv, V, W, X, io, part, hcol, ones;
    DBuf<double> inv;
    Bv.alloc(nr);
    V.alloc(nr * (mk + 1));
    W.alloc(nr);
    X.alloc(nr);
    io.alloc(nr);
    const int nb = static_cast<int>((nr + 255) / 256);
    part.alloc(static_cast<size_t>(nb) * R);
    hcol.alloc(static_cast<size_t>(mk + 2) * R);
    inv.alloc(R);
    ones.alloc(R);
    {
      const std::vector<double2> o(R, make_double2(1.0, 0.0));
      HS_CUDA(cudaMemcpyAsync(ones.p, o.data(), sizeof(double2) * R, cudaMemcpyHostToDevice, st));
    }
    HS_CUDA(cudaMemcpyAsync(io.p, b + 2 * b0 * n, sizeof(double2) * nr, cudaMemcpyHostToDevice, st));
    launch_transpose_in(io.p, Bv.p, n, R, st);
    HS_CUDA(cudaMemsetAsync(X.p, 0, sizeof(double2) * nr, st));
    auto dot = [&](const double2* a, const double2* c, double2* out) {
      const int blocks = launch_dot_partials(a, c, n, R, part.p, st);
      launch_reduce_cpartials(part.p, blocks, R, out, st);
    };
    std::vector<double2> hh(static_cast<size_t>(mk + 2) * R);
    std::vector<double> bnorm(R), invh(R), fin(R, 1.0);
    std::vector<int> iters(R, 0), active(R, 1), breakdown(R, 0);
    std::vector<std::vector<double>> hist(R);
    for (int cycle = 0;; ++cycle) {
      // r0 = b (first cycle, x = 0) or b - A x; its norm starts the Givens right-hand side
      const double2* r0 = Bv.p;
      if (cycle > 0) {
        K.op(X.p, W.p, R);
        HS_CUDA(cudaMemcpyAsync(V.p, Bv.p, sizeof(double2) * nr, cudaMemcpyDeviceToDevice, st));
        launch_axpy_cols(V.p, W.p, ones.p, 1, n, R, st);
        r0 = V.p;
      }
      dot(r0, r0, hcol.p);
      HS_CUDA(cudaMemcpyAsync(hh.data(), hcol.p, sizeof(double2) * R, cudaMemcpyDeviceToHost, st));
      HS_CUDA(cudaStreamSynchronize(st));
      std::vector<int> cyc_it(R, 0), live(R, 0);
      std::vector<std::vector<std::vector<Complex>>> hess(R);
      std::vector<std::vector<Complex>> cs(R, std::vector<Complex>(mk)), sn(R, std::vector<Complex>(mk)),
          g(R, std::vector<Complex>(mk + 1, Complex(0.0)));
      for (int r = 0; r < R; ++r) {
        const double beta = std::sqrt(hh[r].x);
        if (cycle == 0) {
          bnorm[r] = beta;
          hist[r].push_back(beta == 0.0 ? 0.0 : 1.0);
          if (beta == 0.0) active[r] = 0;
        }
        invh[r] = 0.0;
        if (!active[r] || beta == 0.0) continue;
        live[r] = 1;
        invh[r] = 1.0 / beta;
        g[r][0] = beta;
      }
      bool any = false;
      for (int r = 0; r < R; ++r) any |= live[r] != 0;
      if (!any) break;
      // v0 = r0 / ||r0|| (columns not iterating this cycle are zero)
      if (r0 != V.p) HS_CUDA(cudaMemcpyAsync(V.p, r0, sizeof(double2) * nr, cudaMemcpyDeviceToDevice, st));
      HS_CUDA(cudaMemcpyAsync(inv.p, invh.data(), sizeof(double) * R, cudaMemcpyHostToDevice, st));
      launch_scale_cols(V.p, inv.p, n, R, st);
      int j = 0;
      auto any_live = [&] {
        for (int r = 0; r < R; ++r)
          if (live[r]) return true;
        return false;
      };
      while (j < mk && any_live()) {
        double2* vj = V.p + static_cast<size_t>(j) * nr;
        K.op(K.pc(vj, R), W.p, R);  // w = A M^-1 v_j
        for (int i = 0; i <= j; ++i) {                                         // modified Gram-Schmidt
          const double2* vi = V.p + static_cast<size_t>(i) * nr;
          dot(vi, W.p, hcol.p + static_cast<size_t>(i) * R);
          launch_axpy_cols(W.p, vi, hcol.p + static_cast<size_t>(i) * R, 1, n, R, st);
        }
        dot(W.p, W.p, hcol.p + static_cast<size_t>(j + 1) * R);
        HS_CUDA(cudaMemcpyAsync(hh.data(), hcol.p, sizeof(double2) * (j + 2) * R, cudaMemcpyDeviceToHost, st));
        HS_CUDA(cudaStreamSynchronize(st));
        for (int r = 0; r < R; ++r) {
          invh[r] = 0.0;
          if (!live[r]) continue;
          std::vector<Complex> h(j + 2);
          for (int i = 0; i <= j; ++i) h[i] = Complex(hh[static_cast<size_t>(i) * R + r].x, hh[static_cast<size_t>(i) * R + r].y);
          const double wnorm = std::sqrt(hh[static_cast<size_t>(j + 1) * R + r].x);
          h[j + 1] = wnorm;
          for (int i = 0; i < j; ++i) {
            const Complex t = cs[r][i] * h[i] + sn[r][i] * h[i + 1];
            h[i + 1] = -std::conj(sn[r][i]) * h[i] + std::conj(cs[r][i]) * h[i + 1];
            h[i] = t;
          }
          {
            const Complex a = h[j], bb = h[j + 1];
            const double rr = std::sqrt(std::norm(a) + std::norm(bb));
            if (rr == 0.0) {
              cs[r][j] = 1.0;
              sn[r][j] = 0.0;
            } else {
              cs[r][j] = std::conj(a) / rr;
              sn[r][j] = std::conj(bb) / rr;
            }
            h[j] = cs[r][j] * a + sn[r][j] * bb;
            h[j + 1] = 0.0;
          }
          hess[r].push_back(h);
          g[r][j + 1] = -std::conj(sn[r][j]) * g[r][j];
          g[r][j] = cs[r][j] * g[r][j];
          const double rel = std::abs(g[r][j + 1]) / bnorm[r];
          hist[r].push_back(rel);
          fin[r] = rel;
          ++iters[r];
          cyc_it[r] = j + 1;
          if (wnorm <= 1e-14 * bnorm[r]) {
            breakdown[r] = 1;
            live[r] = active[r] = 0;
            continue;
          }
          if (rel <= tol) {
            live[r] = active[r] = 0;
            continue;
          }
          if (iters[r] >= maxit) {
            live[r] = active[r] = 0;
            continue;
          }
          invh[r] = 1.0 / wnorm;
        }
        double2* vn = V.p + static_cast<size_t>(j + 1) * nr;
        HS_CUDA(cudaMemcpyAsync(vn, W.p, sizeof(double2) * nr, cudaMemcpyDeviceToDevice, st));
        HS_CUDA(cudaMemcpyAsync(inv.p, invh.data(), sizeof(double) * R, cudaMemcpyHostToDevice, st));
        launch_scale_cols(vn, inv.p, n, R, st);  // columns that stopped get a zero vector
        ++j;
      }
      // y by back substitution, then x += M^-1 (V y) (columns that did not iterate add M^-1 0 = 0)
      std::vector<std::vector<Complex>> y(R);
      int jmax = 0;
      for (int r = 0; r < R; ++r) {
        const int jr = cyc_it[r];
        jmax = std::max(jmax, jr);
        y[r].assign(jr, Complex(0.0));
        for (int i = jr - 1; i >= 0; --i) {
          Complex sacc = g[r][i];
          for (int k2 = i + 1; k2 < jr; ++k2) sacc -= hess[r][k2][i] * y[r][k2];
          y[r][i] = sacc / hess[r][i][i];
        }
      }
      double2* vy = K.pc_in(R);
      HS_CUDA(cudaMemsetAsync(vy, 0, sizeof(double2) * nr, st));
      std::vector<double2> alpha(R);
      for (int k2 = 0; k2 < jmax; ++k2) {
        for (int r = 0; r < R; ++r)
          alpha[r] = k2 < cyc_it[r] ? make_double2(y[r][k2].real(), y[r][k2].imag()) : make_double2(0.0, 0.0);
        HS_CUDA(cudaMemcpyAsync(hcol.p, alpha.data(), sizeof(double2) * R, cudaMemcpyHostToDevice, st));
        launch_axpy_cols(vy, V.p + static_cast<size_t>(k2) * nr, hcol.p, 0, n, R, st);
      }
      launch_axpy_cols(X.p, K.pc(vy, R), ones.p, 0, n, R, st);
      HS_CUDA(cudaStreamSynchronize(st));  // alpha / hcol host buffers are reused
    }
    // true residual ||b - A x|| / ||b||
    DBuf<double> tn;
    tn.alloc(R);
    K.true_res(X.p, Bv.p, R, tn.p);
    std::vector<double> tnh(R);
    HS_CUDA(cudaMemcpyAsync(tnh.data(), tn.p, sizeof(double) * R, cudaMemcpyDeviceToHost, st));
    launch_transpose_out(X.p, io.p, n, R, st);
    HS_CUDA(cudaMemcpyAsync(x + 2 * b0 * n, io.p, sizeof(double2) * nr, cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
    if (reports)
      for (int r = 0; r < R; ++r) {
        hs_gmres_report& rep = reports[b0 + r];
        std::memset(&rep, 0, sizeof(rep));
        rep.iterations = iters[r];
        const double f = iters[r] > 0 ? fin[r] : 1.0;
        rep.final_residual = bnorm[r] == 0.0 ? 0.0 : f;
        rep.converged = bnorm[r] == 0.0 || breakdown[r] || f <= tol;
        rep.true_residual = bnorm[r] == 0.0 ? 0.0 : std::sqrt(tnh[r]) / bnorm[r];
        rep.n_history = static_cast<int>(hist[r].size());
        for (int q = 0; q < rep.n_history; ++q) rep.history[q] = hist[r][q];
      }
  }
}


// gmres(global_op, DdmPreconditioner, b, cfg) as run_precond wires it (src/harness.cpp:285-305)
void gmres_impl(hs_ddm* s, int nrhs, const double* b, double* x, double tol, int maxit, int restart, int rounds,
                hs_gmres_report* reports) {
  if (!s) config_error("gmres: null handle");
  DdmHandle& H = s->h;
  HS_CUDA(cudaSetDevice(H.eng.device));
  H.ensure_gop();
  KrylovOps K;
  K.device = H.eng.device;
  K.st = H.eng.stream;
  K.n = H.geom.gn;
  const long long n = K.n;
  cudaStream_t st = K.st;
  K.batch = [&](int) {
    if (!(tol > 0.0) || maxit < 1 || restart < 1) return 1;  // (reported by the loop's checks)
    const int mk = std::min(restart, maxit);
    size_t free_b = 0, total_b = 0;
    HS_CUDA(cudaMemGetInfo(&free_b, &total_b));
    // per RHS column: the Krylov basis and work vectors, plus the DDM application's per-RHS
    // buffers (x / z / rhs per subdomain and x buffer, b / u / staging on the global grid)
    const int nbuf_max = std::max(4, std::min(rounds * H.ndir, HS_MAX_ACC_SWEEPS));  // x buffers (build_schedule)
    const double ddm_col = (static_cast<double>(nbuf_max) * H.eng.n_base.back() + 2.0 * H.geom.nsub * H.eng.n_max +
                            6.0 * n) * sizeof(double2);
    const double per_col = static_cast<double>(mk + 5) * n * sizeof(double2) + ddm_col;
    int rmax = std::max(1, std::min(kMaxRhs, static_cast<int>(0.6 * free_b / per_col)));
    if (H.partitioned()) rmax = kMaxRhs;  // every rank must batch identically
    return rmax;
  };
  K.prepare = [&](int R) { H.ensure_state(R, rounds); };
  K.pc_in = [&](int) { return H.bN.p; };
  K.pc = [&](const double2* v, int R) -> const double2* {  // one DDM application: z = M^-1 v
    if (v != H.bN.p)
      HS_CUDA(cudaMemcpyAsync(H.bN.p, v, sizeof(double2) * static_cast<size_t>(n) * R, cudaMemcpyDeviceToDevice, st));
    H.run(rounds, false, false);
    return H.u.p;
  };
  K.op = [&](const double2* z, double2* w, int R) { launch_spmv(n, H.g_rp.p, H.g_col.p, H.g_val.p, z, w, R, st); };
  K.true_res = [&](const double2* xx, const double2* bb, int R, double* out) {
    const int nb2 = launch_residual(n, H.g_rp.p, H.g_col.p, H.g_val.p, xx, bb, R, H.pnum.p, H.pden.p, st, H.geom.gsize[0], H.g_sop);
    launch_reduce_partials(H.pnum.p, nb2, R, out, st);
  };
  gmres_loop(K, nrhs, b, x, tol, maxit, restart, reports);
}

}  // namespace

extern "C" int hs_gmres(hs_ddm* s, int nrhs, const double* b, double* x, double tol, int maxit, int rounds,
                        hs_gmres_report* reports) {
  return guarded([&] { gmres_impl(s, nrhs, b, x, tol, maxit, maxit, rounds, reports); });
}

extern "C" int hs_gmres_restarted(hs_ddm* s, int nrhs, const double* b, double* x, double tol, int maxit, int restart,
                                  int rounds, hs_gmres_report* reports) {
  return guarded([&] { gmres_impl(s, nrhs, b, x, tol, maxit, restart, rounds, reports); });
}

// gmres(apply_op, apply_precond, rhs, cfg) for any pair of LinearMaps (include/helmsweep/krylov.hpp:30-36;
// pc = NULL is identity_preconditioner(), :38-40): the Krylov loop of hs_gmres with the caller's apply
// callbacks in place of the global operator and the DDM preconditioner. The vectors stay on the
// device; a host callback sees them staged through pinned buffers as RHS-major CVectors.
extern "C" int hs_gmres_general(int device, int64_t n64, int nrhs, hs_linop_fn op, hs_linop_fn pc, void* user,
                                int on_device, const double* b, double* x, double tol, int maxit, int restart,
                                hs_gmres_report* reports) {
  return guarded([&] {
    if (!op || !b || !x) config_error("gmres: null argument");
    if (n64 < 1 || nrhs < 1) config_error("gmres: empty system");
    if (!(tol > 0.0)) config_error("GmresConfig: tol must be positive");  // (config errors before device work)
    if (maxit < 1) config_error("GmresConfig: max_iterations must be >= 1");
    if (maxit + 1 > HS_MAX_GMRES_HISTORY) config_error("gmres: maxit too large for the report");
    if (restart < 1) config_error("gmres: restart must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
      throw Error(kCuda, "gmres: no usable CUDA device");
    HS_CUDA(cudaSetDevice(device));
    const long long n = n64;
    cudaStream_t st = nullptr;
    HS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct Guard {
      cudaStream_t s;
      double *hx = nullptr, *hy = nullptr;
      ~Guard() {
        cudaStreamSynchronize(s);
        if (hx) cudaFreeHost(hx);
        if (hy) cudaFreeHost(hy);
        cudaStreamDestroy(s);
      }
    } guard{st};
    DBuf<double2> T, Z, W2, cin, cout, dtmp;
    int cap = 0;
    KrylovOps K;
    K.device = device;
    K.st = st;
    K.n = n;
    K.batch = [&](int want) {
      if (!(tol > 0.0) || maxit < 1 || restart < 1) return 1;
      size_t free_b = 0, total_b = 0;
      HS_CUDA(cudaMemGetInfo(&free_b, &total_b));
      const double per_col = static_cast<double>(std::min(restart, maxit) + 12) * n * sizeof(double2);
      return std::max(1, std::min(std::min(want, kMaxRhs), static_cast<int>(0.6 * free_b / per_col)));
    };
    K.prepare = [&](int R) {
      if (R <= cap) return;
      cap = R;
      const size_t nr = static_cast<size_t>(n) * R;
      for (DBuf<double2>* d : {&T, &Z, &W2, &cin, &cout}) d->alloc(nr);
      dtmp.alloc(static_cast<size_t>(R) + (nr + 255) / 256 * R);
      if (!on_device) {
        if (guard.hx) cudaFreeHost(guard.hx);
        if (guard.hy) cudaFreeHost(guard.hy);
        HS_CUDA(cudaMallocHost(&guard.hx, nr * sizeof(double2)));
        HS_CUDA(cudaMallocHost(&guard.hy, nr * sizeof(double2)));
      }
    };
    // y = F v through the caller's callback: node-major -> RHS-major CVectors -> callback -> back
    auto apply = [&](hs_linop_fn f, const double2* v, double2* y, int R) {
      const size_t bytes = static_cast<size_t>(n) * R * sizeof(double2);
      launch_transpose_out(v, cin.p, n, R, st);
      int rc;
      if (on_device) {
        rc = f(user, R, reinterpret_cast<const double*>(cin.p), reinterpret_cast<double*>(cout.p), st);
      } else {
        HS_CUDA(cudaMemcpyAsync(guard.hx, cin.p, bytes, cudaMemcpyDeviceToHost, st));
        HS_CUDA(cudaStreamSynchronize(st));
        rc = f(user, R, guard.hx, guard.hy, nullptr);
        HS_CUDA(cudaMemcpyAsync(cout.p, guard.hy, bytes, cudaMemcpyHostToDevice, st));
      }
      if (rc != 0) data_error("gmres: operator callback failed");
      launch_transpose_in(cout.p, y, n, R, st);
    };
    K.pc_in = [&](int) { return T.p; };
    K.pc = [&](const double2* v, int R) -> const double2* {
      if (!pc) return v;  // identity preconditioner
      apply(pc, v, Z.p, R);
      return Z.p;
    };
    K.op = [&](const double2* z, double2* w, int R) { apply(op, z, w, R); };
    K.true_res = [&](const double2* xx, const double2* bb, int R, double* out) {  // |b - A x|^2 per column
      apply(op, xx, W2.p, R);
      std::vector<double2> one(R, make_double2(1.0, 0.0)), h(R);
      HS_CUDA(cudaMemcpyAsync(dtmp.p, one.data(), sizeof(double2) * R, cudaMemcpyHostToDevice, st));
      launch_axpy_cols(W2.p, bb, dtmp.p, 1, n, R, st);  // A x - b
      const int blocks = launch_dot_partials(W2.p, W2.p, n, R, dtmp.p + R, st);
      launch_reduce_cpartials(dtmp.p + R, blocks, R, dtmp.p, st);
      HS_CUDA(cudaMemcpyAsync(h.data(), dtmp.p, sizeof(double2) * R, cudaMemcpyDeviceToHost, st));
      HS_CUDA(cudaStreamSynchronize(st));
      std::vector<double> hr(R);
      for (int r = 0; r < R; ++r) hr[r] = h[r].x;
      HS_CUDA(cudaMemcpyAsync(out, hr.data(), sizeof(double) * R, cudaMemcpyHostToDevice, st));
      HS_CUDA(cudaStreamSynchronize(st));
    };
    gmres_loop(K, nrhs, b, x, tol, maxit, restart, reports);
  });
}

extern "C" int hs_ddm_profile(hs_ddm* s, double* solve_seconds, int64_t* solve_launches, int64_t* subdomain_solves,
                              double* alg_bytes, double* alg_flops) {
  return guarded([&] {
    if (!s) config_error("profile: null handle");
    DdmHandle& H = s->h;
    if (H.nsweeps == 0) config_error("profile: no solve has run");
    HS_CUDA(cudaSetDevice(H.eng.device));
    HS_CUDA(cudaStreamSynchronize(H.eng.stream));
    const int nsub = H.geom.nsub;
    std::vector<rmask> nz(static_cast<size_t>(H.nsweeps) * nsub);
    std::vector<unsigned> tf(nz.size());
    HS_CUDA(cudaMemcpy(nz.data(), H.nzmask.p, nz.size() * sizeof(rmask), cudaMemcpyDeviceToHost));
    HS_CUDA(cudaMemcpy(tf.data(), H.tface.p, tf.size() * sizeof(unsigned), cudaMemcpyDeviceToHost));
    // the work the solve performs: the backward pass over every front, the forward pass over the
    // live fronts only (past sweep 1, fronts whose subtree holds no nonzero injection line have
    // T = z = V = 0 and are skipped; their packed entries are neither read nor multiplied)
    auto live_packed = [&](int cls, unsigned fm) {
      const ClassDev& cd = *H.eng.classes[cls];
      if (fm & 0x100u || cd.fbits.empty()) return static_cast<double>(cd.sym->packed_entries);
      double p = 0.0;
      for (size_t f = 0; f < cd.sym->fronts.size(); ++f) {
        if (!(cd.fbits[f] & fm & 0xFFu)) continue;
        const double m = cd.sym->fronts[f].m, k = cd.sym->fronts[f].k;
        p += m * k - k * (k - 1) / 2;
      }
      return p;
    };
    // ... and the backward pass over the fronts whose x the application reads back; of a front
    // the forward skipped (z = 0) only the boundary block W is multiplied
    auto needed_packed = [&](int sub, unsigned fm) {
      const ClassDev& cd = *H.eng.classes[H.subs[sub].cls];
      const unsigned* w = H.need_h.empty() ? nullptr : H.need_h.data() + static_cast<size_t>(sub) * H.need_words;
      const bool all = (fm & 0x100u) || cd.fbits.empty();
      double p = 0.0;
      for (size_t f = 0; f < cd.sym->fronts.size(); ++f) {
        if (w && !(w[f >> 5] >> (f & 31) & 1u)) continue;
        const double m = cd.sym->fronts[f].m, k = cd.sym->fronts[f].k;
        const bool zlive = all || (cd.fbits[f] & fm & 0xFFu);
        p += zlive ? m * k - k * (k - 1) / 2 : (m - k) * k;
      }
      return p;
    };
    double sec = 0.0, bytes = 0.0, flops = 0.0;
    int64_t launches = 0, solves = 0;
    const bool no_skip = std::getenv("HS_NO_GROUP_SKIP") != nullptr || H.eng.quad;
    float ms = 0.f;
    for (size_t m = 0; m < H.msteps.size(); ++m) {
      HS_CUDA(cudaEventElapsedTime(&ms, H.ev[1 + H.nsweeps + 2 * m], H.ev[2 + H.nsweeps + 2 * m]));
      sec += ms * 1e-3;
      launches += 2;  // forward + backward dataflow launches (the counter reset is a memset)
      for (const int2& t : H.msteps_own[m]) {  // this rank's solves
        if (nz[static_cast<size_t>(t.y - 1) * nsub + t.x] == 0) continue;
        const SymbolicClass& c = *H.eng.classes[H.subs[t.x].cls]->sym;
        // per 8-column group: the columns the items compute (RHS groups that are exactly zero for
        // the task are skipped, half-zero 16-column groups run as 8-column items) over the fronts
        // that are live for the group -- every front where the group holds part of the split source
        // (sweep 1, bits 16-23 of the face word), else the fronts of the receiving faces
        const unsigned fw = tf[static_cast<size_t>(t.y - 1) * nsub + t.x];
        const rmask m8 = nz[static_cast<size_t>(t.y - 1) * nsub + t.x];
        const double pf_all = live_packed(H.subs[t.x].cls, 0x100u), pb_all = needed_packed(t.x, 0x100u);
        const double pf_face = live_packed(H.subs[t.x].cls, fw & 0xFFu), pb_face = needed_packed(t.x, fw & 0xFFu);
        ++solves;
        double pmax = 0.0;
        int cols = 0;
        for (int g8 = 0; 8 * g8 < H.R; ++g8) {
          if (!no_skip && !((m8 >> (8 * g8)) & 0xFFull)) continue;
          const int w = std::min(8, H.R - 8 * g8);
          const bool all = (fw & 0x100u) || ((fw >> 16) >> g8 & 1u);
          const double p = all ? pf_all + pb_all : pf_face + pb_face;
          pmax = std::max(pmax, p);
          cols += w;
          flops += 8.0 * p * w;
        }
        bytes += pmax * 16 + 2.0 * cols * c.n * 16;
      }
    }
    if (solve_seconds) *solve_seconds = sec;
    if (solve_launches) *solve_launches = launches;
    if (subdomain_solves) *subdomain_solves = solves;
    if (alg_bytes) *alg_bytes = bytes;
    if (alg_flops) *alg_flops = flops;
  });
}

extern "C" int hs_route_trace(int dim, int rounds, int gen_sweep, int axis, int sign) {
  try {
    const std::vector<Vec3i> plan = sweep_plan(dim, rounds);
    if (gen_sweep < 1 || gen_sweep > static_cast<int>(plan.size()) || axis < 0 || axis >= dim) return -1;
    return route_trace(plan, dim, gen_sweep, axis, sign);
  } catch (...) {
    return -1;
  }
}

// global_direct_solve (src/harness.cpp:185-214): b = J f off the shell on the padded global grid,
// then the direct factorization of the global J-scaled operator (built on first use and kept).
extern "C" int hs_ddm_global_solve(hs_ddm* s, int nrhs, const double* f, double* u, hs_factor_stats* stats) {
  return guarded([&] {
    if (!s) config_error("global_direct_solve: null handle");
    DdmHandle& H = s->h;
    HS_CUDA(cudaSetDevice(H.eng.device));
    const std::int64_t n = H.ggrid.range.count();
    const std::int64_t guard = H.dim == 2 ? 4'500'000 : 450'000;  // src/harness.cpp:19-20
    if (n > guard)
      config_error("global_direct_solve: " + std::to_string(n) +
                   " nodes exceed the direct-solve memory guard; reduce the scale");
    if (!H.gfact) {
      Csr op = assemble(H.ggrid, H.gcoeffs, extend_to_subdomain(H.medium, H.interior, H.ggrid));
      H.gfact = make_factor(H.dim, H.ggrid.range, std::move(op.row_ptr), std::move(op.col), op.val, H.eng.device)
                    .release();
    }
    if (stats) *stats = H.gfact->h.stats;
    if (nrhs <= 0) return;
    const Complex* fi = reinterpret_cast<const Complex*>(f);
    Complex* bo = reinterpret_cast<Complex*>(u);
    parallel_for(nrhs, [&](long long r) {
      for (std::int64_t i = 0; i < n; ++i) {
        const Vec3i p = H.ggrid.range.unlinear(i);
        bo[r * n + i] = H.ggrid.on_shell(p) ? Complex(0.0) : H.gcoeffs.jacobian(p) * fi[r * n + i];
      }
    });
    FactorHandle& F = H.gfact->h;
    std::lock_guard<std::mutex> lk(F.mu);
    F.io.alloc(static_cast<size_t>(n) * nrhs);
    HS_CUDA(cudaMemcpyAsync(F.io.p, u, sizeof(double2) * n * nrhs, cudaMemcpyHostToDevice, F.eng.stream));
    factor_solve_device(F, nrhs, F.io.p, nullptr);
    HS_CUDA(cudaMemcpyAsync(u, F.io.p, sizeof(double2) * n * nrhs, cudaMemcpyDeviceToHost, F.eng.stream));
    HS_CUDA(cudaStreamSynchronize(F.eng.stream));
  });
}

namespace hsb {
std::string& last_error_ref() { return g_last_error; }  // shared with the on-disk format entry points (hs_io.cpp)
}  // namespace hsb

extern "C" int hs_ddm_memory(const hs_ddm* s, int64_t* factor_bytes, int64_t* state_bytes, int* max_batch) {
  if (!s) return kConfig;
  const DdmHandle& H = s->h;
  const Engine& E = H.eng;
  if (factor_bytes) *factor_bytes = static_cast<int64_t>(E.factor.n * sizeof(double2));
  if (state_bytes)
    *state_bytes = static_cast<int64_t>((E.x.n + E.x1.n + E.rb.n + E.vbuf.n) * sizeof(double2) + E.part.n * sizeof(double) +
                                        (H.mbox.n + H.bN.n + H.u.n + H.io.n) * sizeof(double2));
  if (max_batch) *max_batch = kMaxRhs;
  return kOk;
}

extern "C" int hs_ddm_schedule_info(hs_ddm* s, int rounds, int* macro_steps, int* max_width, int* sequential_steps,
                                    int* buffers) {
  return guarded([&] {
    if (!s) config_error("schedule_info: null handle");
    DdmHandle& H = s->h;
    HS_CUDA(cudaSetDevice(H.eng.device));
    H.ensure_state(H.R > 0 ? H.R : 1, rounds);
    if (macro_steps) *macro_steps = static_cast<int>(H.msteps.size());
    if (max_width) *max_width = H.max_width;
    if (sequential_steps) *sequential_steps = H.nsweeps * H.steps;
    if (buffers) *buffers = H.nbuf;
  });
}
