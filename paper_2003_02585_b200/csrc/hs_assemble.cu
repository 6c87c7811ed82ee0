// Subdomain setup on the device: extended wavenumber and the J-scaled PML
// operator's CSR values of every subdomain, computed by one thread per row
// (/root/reference/proj/src/media.cpp:203-217 extend_to_subdomain, src/operator.cpp:25-98
// assemble, include/helmsweep/pml.hpp:40-57 jacobian / coupling). The CSR structure is the
// symbolic class's; the 1-D PML tables alpha = 1 + i sigma at nodes and half-points
// (src/pml.cpp:19-52) are built on the host, O(n) per axis, since their std::pow has no
// bit-identical device counterpart.
//
// Bit-for-bit with the host: every operation is an explicitly rounded intrinsic (no FMA
// contraction), complex products are (ac - bd, ad + bc) as GCC lowers std::complex<double>
// multiplication, and complex division is libgcc's __divdc3 (ratio / denominator form, with the
// alternate order for a subnormal ratio).
#include "hs_assemble.cuh"

#include <atomic>

namespace hsb {

extern std::atomic<long long> g_kernel_launches;

namespace {

__device__ __forceinline__ double2 cmul_x(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
// libgcc __divdc3 for finite operands of moderate magnitude (its power-of-two rescalings of
// huge / tiny operands do not change the rounded result and are never taken here)
__device__ __forceinline__ double2 cdiv_x(double2 n, double2 dd) {
  const double a = n.x, b = n.y, c = dd.x, d = dd.y;
  double x, y;
  if (fabs(c) < fabs(d)) {
    const double ratio = __ddiv_rn(c, d);
    const double denom = __dadd_rn(__dmul_rn(c, ratio), d);
    if (fabs(ratio) > 2.2250738585072014e-308) {
      x = __ddiv_rn(__dadd_rn(__dmul_rn(a, ratio), b), denom);
      y = __ddiv_rn(__dsub_rn(__dmul_rn(b, ratio), a), denom);
    } else {
      x = __ddiv_rn(__dadd_rn(__dmul_rn(c, __ddiv_rn(a, d)), b), denom);
      y = __ddiv_rn(__dsub_rn(__dmul_rn(c, __ddiv_rn(b, d)), a), denom);
    }
  } else {
    const double ratio = __ddiv_rn(d, c);
    const double denom = __dadd_rn(__dmul_rn(d, ratio), c);
    if (fabs(ratio) > 2.2250738585072014e-308) {
      x = __ddiv_rn(__dadd_rn(__dmul_rn(b, ratio), a), denom);
      y = __ddiv_rn(__dsub_rn(b, __dmul_rn(a, ratio)), denom);
    } else {
      x = __ddiv_rn(__dadd_rn(a, __dmul_rn(d, __ddiv_rn(b, c))), denom);
      y = __ddiv_rn(__dsub_rn(b, __dmul_rn(d, __ddiv_rn(a, c))), denom);
    }
  }
  return make_double2(x, y);
}

// VelocityGrid::sample (src/media.cpp:30-56): multilinear interpolation of float samples
__device__ double sample_velocity(const AsmMedium& m, const double (&x)[3]) {
  int i0[3] = {0, 0, 0};
  double w[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < m.vdim; ++a) {
    double t = __ddiv_rn(__dsub_rn(x[a], m.vorg[a]), m.vsp[a]);
    const double hi = static_cast<double>(m.vn[a] - 1);
    t = t < 0.0 ? 0.0 : (hi < t ? hi : t);
    i0[a] = min(static_cast<int>(t), m.vn[a] - 2);
    w[a] = __dsub_rn(t, static_cast<double>(i0[a]));
  }
  double v = 0.0;
  const int kmax = m.vdim == 3 ? 1 : 0;
  for (int dk = 0; dk <= kmax; ++dk)
    for (int dj = 0; dj <= 1; ++dj)
      for (int di = 0; di <= 1; ++di) {
        double ww = __dmul_rn(di ? w[0] : __dsub_rn(1.0, w[0]), dj ? w[1] : __dsub_rn(1.0, w[1]));
        if (m.vdim == 3) ww = __dmul_rn(ww, dk ? w[2] : __dsub_rn(1.0, w[2]));
        long long id = i0[0] + di;
        id += static_cast<long long>(m.vn[0]) * (i0[1] + dj);
        if (m.vdim == 3) id += static_cast<long long>(m.vn[0]) * m.vn[1] * (i0[2] + dk);
        v = __dadd_rn(v, __dmul_rn(ww, static_cast<double>(m.vc[id])));
      }
  return v;
}

// eval_kappa (src/media.cpp:167-185); a non-positive gridded sample flags *bad
__device__ double eval_kappa_dev(const AsmMedium& m, const double (&x)[3], unsigned* bad) {
  switch (m.kind) {
    case 0:
      return m.kappa;
    case 1: {
      const double t = x[m.axis];
      if (t < m.eta) return m.kd;
      if (t > __dadd_rn(m.eta, m.eps) || m.eps == 0.0) return t == m.eta ? m.kd : m.ku;
      const double w = __ddiv_rn(__dsub_rn(t, m.eta), m.eps);
      return __dadd_rn(__dmul_rn(m.kd, __dsub_rn(1.0, w)), __dmul_rn(m.ku, w));
    }
    default: {
      const double c = sample_velocity(m, x);
      if (!(c > 0.0)) {
        atomicOr(bad, 1u);
        return 0.0;
      }
      return __ddiv_rn(m.omega, c);
    }
  }
}

__global__ void assemble_kernel(AsmArgs a) {
  const AsmSub& S = a.subs[blockIdx.y];
  const long long n = static_cast<long long>(S.size[0]) * S.size[1] * S.size[2];
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int dim = a.dim;
  int p[3], li[3];  // grid index, local index
  long long stride[3];
  {
    long long t = r, st = 1;
    for (int ax = 0; ax < 3; ++ax) {
      li[ax] = static_cast<int>(t % S.size[ax]);
      t /= S.size[ax];
      p[ax] = S.lo[ax] + li[ax];
      stride[ax] = st;
      st *= S.size[ax];
    }
  }
  bool shell = false;
  for (int ax = 0; ax < dim; ++ax) shell |= li[ax] == 0 || li[ax] == S.size[ax] - 1;
  const long long k0 = S.row_ptr[r], k1 = S.row_ptr[r + 1];
  double2* val = S.val;
  if (shell) {  // identity row (src/operator.cpp:44-49)
    val[k0] = make_double2(1.0, 0.0);
    atomicMax(S.maxabs, __double_as_longlong(1.0));
    return;
  }
  // extend_to_subdomain: kappa at the nearest point of the subdomain's cell (coordinates clamped)
  double x[3] = {0.0, 0.0, 0.0};
  for (int ax = 0; ax < dim; ++ax) {
    const double c = __dadd_rn(a.origin[ax], __dmul_rn(static_cast<double>(p[ax]), a.h[ax]));
    x[ax] = c < S.cell_lo[ax] ? S.cell_lo[ax] : (S.cell_hi[ax] < c ? S.cell_hi[ax] : c);
  }
  const double kap = eval_kappa_dev(a.med, x, a.bad);
  // diag = J kappa^2 - sum of the couplings, in the reference's (axis, side) order
  double2 J = make_double2(1.0, 0.0);
  for (int ax = 0; ax < dim; ++ax) J = cmul_x(J, S.anode[ax][li[ax]]);
  double2 diag = make_double2(__dmul_rn(J.x, kap), __dmul_rn(J.y, kap));
  diag = make_double2(__dmul_rn(diag.x, kap), __dmul_rn(diag.y, kap));
  double2 cpl[6];
  for (int ax = 0; ax < dim; ++ax)
    for (int s = 0; s < 2; ++s) {
      const int hl = s == 0 ? li[ax] - 1 : li[ax];  // the coupling sits at the lower node of the edge
      double2 v = make_double2(1.0, 0.0);
      for (int b = 0; b < dim; ++b)
        if (b != ax) v = cmul_x(v, S.anode[b][li[b]]);
      v = cdiv_x(v, S.ahalf[ax][hl]);
      const double hh = __dmul_rn(a.h[ax], a.h[ax]);
      v = make_double2(__ddiv_rn(v.x, hh), __ddiv_rn(v.y, hh));
      diag = make_double2(__dsub_rn(diag.x, v.x), __dsub_rn(diag.y, v.y));
      cpl[2 * ax + s] = v;
    }
  // the class's column order: ascending, diagonal in place, shell neighbours dropped
  double mx = 0.0;
  for (long long k = k0; k < k1; ++k) {
    const long long c = S.col[k];
    double2 v = diag;
    if (c != r)
      for (int ax = 0; ax < dim; ++ax) {
        if (c == r - stride[ax]) v = cpl[2 * ax];
        if (c == r + stride[ax]) v = cpl[2 * ax + 1];
      }
    val[k] = v;
    mx = fmax(mx, hypot(v.x, v.y));
  }
  atomicMax(S.maxabs, __double_as_longlong(mx));  // non-negative doubles order as their bit patterns
}

__device__ __forceinline__ int weight2_dev(const PlanGeom& g, int axis, int cell, int index) {
  const int lo = cell * g.w[axis], hi = (cell + 1) * g.w[axis];
  const int lo_ext = cell == 0 ? lo - g.pad : lo;
  const int hi_ext = cell == g.counts[axis] - 1 ? hi + g.pad : hi;
  if (index < lo_ext || index > hi_ext) return 0;
  if (index == lo && cell > 0) return 1;
  if (index == hi && cell < g.counts[axis] - 1) return 1;
  return 2;
}

struct PlanDirs {
  int d[8][3];
};

template <int E>
__global__ void acc_plan_kernel(PlanGeom g, int ndirs, PlanDirs dirs, int2* acc_ent) {
  const long long node = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= g.gn) return;
  int p[3] = {0, 0, 0}, cand[3][2], nc[3] = {1, 1, 1};
  {
    long long t = node;
    for (int a = 0; a < g.dim; ++a) {
      p[a] = g.glo[a] + static_cast<int>(t % g.gsize[a]);
      t /= g.gsize[a];
      int c = p[a] >= 0 ? p[a] / g.w[a] : 0;
      c = min(c, g.counts[a] - 1);
      nc[a] = 0;
      if (c > 0 && p[a] == c * g.w[a]) cand[a][nc[a]++] = c - 1;  // shared face: the lower cell first
      cand[a][nc[a]++] = c;
    }
  }
  int2 ent[E];
  int sub[E][3];
  int n = 0;
  // every combination of per-axis cells, in ascending flattened id (axis 0 fastest)
  const int n2 = g.dim > 2 ? nc[2] : 1;
  for (int i2 = 0; i2 < n2; ++i2)
    for (int i1 = 0; i1 < nc[1]; ++i1)
      for (int i0 = 0; i0 < nc[0]; ++i0) {
        const int s3[3] = {cand[0][i0], cand[1][i1], g.dim > 2 ? cand[2][i2] : 0};
        int num = 1;
        for (int a = 0; a < g.dim; ++a) num *= weight2_dev(g, a, s3[a], p[a]);
        if (num == 0) continue;
        const int id = s3[0] + g.counts[0] * (s3[1] + g.counts[1] * s3[2]);
        const DevClass& C = g.cls[g.sub_cls[id]];
        long long loc = 0, ls = 1;
        for (int a = 0; a < g.dim; ++a) {
          loc += static_cast<long long>(p[a] - (s3[a] * g.w[a] - g.pad)) * ls;
          ls *= C.size[a];
        }
        ent[n] = make_int2(static_cast<int>(g.n_base[id] + C.elim_of_local[loc]), (id << 4) | num);
        for (int a = 0; a < 3; ++a) sub[n][a] = s3[a];
        ++n;
      }
  for (int di = 0; di < ndirs; ++di) {
    long long key[E];
    int2 e2[E];
    for (int i = 0; i < n; ++i) {
      int st = 1;
      for (int a = 0; a < g.dim; ++a) st += dirs.d[di][a] == 1 ? sub[i][a] : g.counts[a] - 1 - sub[i][a];
      key[i] = (static_cast<long long>(st) << 32) | (ent[i].y >> 4);
      e2[i] = ent[i];
    }
    for (int i = 1; i < n; ++i)
      for (int j = i; j > 0 && key[j] < key[j - 1]; --j) {
        const long long tk = key[j];
        key[j] = key[j - 1];
        key[j - 1] = tk;
        const int2 te = e2[j];
        e2[j] = e2[j - 1];
        e2[j - 1] = te;
      }
    int2* dst = acc_ent + (static_cast<long long>(di) * g.gn + node) * E;
    for (int i = 0; i < E; ++i) dst[i] = i < n ? e2[i] : make_int2(-1, 0);
  }
}

__global__ void split_plan_kernel(PlanGeom g, int* split_gp, unsigned char* split_w) {
  const int id = blockIdx.y;
  const DevClass& C = g.cls[g.sub_cls[id]];
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= C.n) return;
  int s3[3];
  {
    int t = id;
    for (int a = 0; a < 3; ++a) {
      s3[a] = t % g.counts[a];
      t /= g.counts[a];
    }
  }
  long long loc = C.local_of_elim[e];
  bool shell = false;
  int num = 1;
  long long gl = 0, gs = 1;
  for (int a = 0; a < g.dim; ++a) {
    const int li = static_cast<int>(loc % C.size[a]);
    loc /= C.size[a];
    const int pa = s3[a] * g.w[a] - g.pad + li;
    shell |= li == 0 || li == C.size[a] - 1;
    num *= weight2_dev(g, a, s3[a], pa);
    gl += static_cast<long long>(pa - g.glo[a]) * gs;
    gs *= g.gsize[a];
  }
  const long long o = g.n_base[id] + e;
  const bool on = num != 0 && !shell;
  split_gp[o] = on ? static_cast<int>(gl) : 0;
  split_w[o] = on ? static_cast<unsigned char>(num) : 0;
}

}  // namespace

void launch_acc_plan(const PlanGeom& g, int ndirs, const int (*dvec)[3], int2* acc_ent, cudaStream_t s) {
  PlanDirs d{};
  for (int i = 0; i < ndirs && i < 8; ++i)
    for (int a = 0; a < 3; ++a) d.d[i][a] = dvec[i][a];
  const int threads = 128;
  const unsigned blocks = static_cast<unsigned>((g.gn + threads - 1) / threads);
  if (g.dim == 3)
    acc_plan_kernel<8><<<blocks, threads, 0, s>>>(g, ndirs, d, acc_ent);
  else
    acc_plan_kernel<4><<<blocks, threads, 0, s>>>(g, ndirs, d, acc_ent);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  HS_CUDA(cudaGetLastError());
}

void launch_split_plan(const PlanGeom& g, int nsub, long long max_n, int* split_gp, unsigned char* split_w,
                       cudaStream_t s) {
  const int threads = 128;
  const dim3 grid(static_cast<unsigned>((max_n + threads - 1) / threads), static_cast<unsigned>(nsub));
  split_plan_kernel<<<grid, threads, 0, s>>>(g, split_gp, split_w);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  HS_CUDA(cudaGetLastError());
}

void launch_assemble(const AsmArgs& a, long long max_rows, cudaStream_t s) {
  if (a.nsub <= 0 || max_rows <= 0) return;
  const int threads = 128;
  const dim3 grid(static_cast<unsigned>((max_rows + threads - 1) / threads), static_cast<unsigned>(a.nsub));
  assemble_kernel<<<grid, threads, 0, s>>>(a);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  HS_CUDA(cudaGetLastError());
}

}  // namespace hsb
