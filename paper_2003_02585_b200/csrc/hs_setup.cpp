// Host setup layer; see hs_setup.hpp for the reference lines each piece follows.
#include "hs_setup.hpp"

#include <algorithm>
#include <cmath>

namespace hsb {

Partition make_partition(const Box& interior, const Vec3i& intervals, const Vec3i& counts) {
  Partition p;
  p.dim = interior.dim;
  p.box = interior;
  for (int a = 0; a < 3; ++a) {
    p.counts[a] = a < p.dim ? counts[a] : 1;
    p.h[a] = a < p.dim ? interior.extent(a) / intervals[a] : 0.0;
  }
  for (int a = 0; a < p.dim; ++a) {
    if (intervals[a] < 1) config_error("UniformGrid: need at least one interval per axis");
    if (p.counts[a] < 1) config_error("partition_domain: counts must be >= 1");
    const int m = intervals[a];
    if (m % p.counts[a] != 0)
      config_error("partition_domain: grid intervals (" + std::to_string(m) +
                   ") not divisible by partition count (" + std::to_string(p.counts[a]) +
                   ") on axis " + std::to_string(a));
    const int w = m / p.counts[a];
    p.cuts[a].resize(p.counts[a] + 1);
    for (int c = 0; c <= p.counts[a]; ++c) p.cuts[a][c] = c * w;
  }
  return p;
}

GridRange Partition::owned(const Vec3i& s) const {
  GridRange r;
  r.dim = dim;
  for (int a = 0; a < dim; ++a) {
    r.lo[a] = cuts[a][s[a]];
    r.hi[a] = cuts[a][s[a] + 1];
  }
  return r;
}

Box Partition::cell(const Vec3i& s) const {
  Box b;
  b.dim = dim;
  for (int a = 0; a < dim; ++a) {
    b.lo[a] = box.lo[a] + cuts[a][s[a]] * h[a];
    b.hi[a] = box.lo[a] + cuts[a][s[a] + 1] * h[a];
  }
  return b;
}

int Weights::weight2(int axis, int cell, int index) const {
  const auto& cuts = p->cuts[axis];
  const int lo = cuts[cell], hi = cuts[cell + 1];
  const int lo_ext = cell == 0 ? lo - pad : lo;
  const int hi_ext = cell == p->counts[axis] - 1 ? hi + pad : hi;
  if (index < lo_ext || index > hi_ext) return 0;
  if (index == lo && cell > 0) return 1;
  if (index == hi && cell < p->counts[axis] - 1) return 1;
  return 2;
}

double Weights::weight(const Vec3i& sub, const Vec3i& node) const {
  int num = 1;
  for (int a = 0; a < p->dim; ++a) {
    num *= weight2(a, sub[a], node[a]);
    if (num == 0) return 0.0;
  }
  return num / static_cast<double>(1 << p->dim);
}

GridRange Weights::support(const Vec3i& sub) const {
  GridRange r = p->owned(sub);
  for (int a = 0; a < p->dim; ++a) {
    if (sub[a] == 0) r.lo[a] -= pad;
    if (sub[a] == p->counts[a] - 1) r.hi[a] += pad;
  }
  return r;
}

namespace {
double sigma_profile(const PmlSpec& spec, const Box& box, double h, int axis, double x) {
  const double scale = spec.width * h;
  double t = 0.0;
  if (x >= box.hi[axis])
    t = x - box.hi[axis];
  else if (x <= box.lo[axis])
    t = box.lo[axis] - x;
  else
    return 0.0;
  return spec.strength * std::pow(t / scale, spec.exponent);
}
}  // namespace

PmlCoefficients build_coefficients(const PmlSpec& spec, const Box& box, const LocalGrid& grid) {
  if (spec.width < 1) config_error("PmlSpec: width must be >= 1 layer");
  if (spec.strength <= 0.0) config_error("PmlSpec: strength must be positive");
  if (spec.exponent < 1) config_error("PmlSpec: exponent must be >= 1");
  PmlCoefficients c;
  c.dim = grid.dim;
  c.range = grid.range;
  c.h = grid.h;
  Box onset = box;
  for (int a = 0; a < grid.dim; ++a) {
    onset.lo[a] -= grid.h[a];
    onset.hi[a] += grid.h[a];
  }
  for (int a = 0; a < grid.dim; ++a) {
    const int n = grid.range.size(a);
    const double tol = 1e-9 * grid.h[a];
    if (grid.coord(a, grid.range.lo[a]) > box.lo[a] - spec.width * grid.h[a] + tol ||
        grid.coord(a, grid.range.hi[a]) < box.hi[a] + spec.width * grid.h[a] - tol)
      config_error("build_coefficients: grid does not cover the box plus " +
                   std::to_string(spec.width) + " pad layers on axis " + std::to_string(a));
    c.node[a].resize(n);
    c.half[a].resize(n - 1);
    for (int i = 0; i < n; ++i) {
      const double x = grid.coord(a, grid.range.lo[a] + i);
      c.node[a][i] = Complex(1.0, sigma_profile(spec, onset, grid.h[a], a, x));
    }
    for (int i = 0; i + 1 < n; ++i) {
      const double x = grid.coord(a, grid.range.lo[a] + i) + 0.5 * grid.h[a];
      c.half[a][i] = Complex(1.0, sigma_profile(spec, onset, grid.h[a], a, x));
    }
  }
  return c;
}

double VelocityGrid::sample(const Vec3d& x) const {
  Vec3i i0{0, 0, 0};
  Vec3d w{0.0, 0.0, 0.0};
  for (int a = 0; a < dim; ++a) {
    double t = (x[a] - origin[a]) / spacing[a];
    t = std::clamp(t, 0.0, static_cast<double>(n[a] - 1));
    i0[a] = std::min(static_cast<int>(t), n[a] - 2);
    w[a] = t - i0[a];
  }
  auto at = [&](int di, int dj, int dk) {
    std::int64_t id = i0[0] + di;
    id += static_cast<std::int64_t>(n[0]) * (i0[1] + dj);
    if (dim == 3) id += static_cast<std::int64_t>(n[0]) * n[1] * (i0[2] + dk);
    return static_cast<double>(c[id]);
  };
  double v = 0.0;
  const int kmax = dim == 3 ? 1 : 0;
  for (int dk = 0; dk <= kmax; ++dk)
    for (int dj = 0; dj <= 1; ++dj)
      for (int di = 0; di <= 1; ++di) {
        double ww = (di ? w[0] : 1 - w[0]) * (dj ? w[1] : 1 - w[1]);
        if (dim == 3) ww *= (dk ? w[2] : 1 - w[2]);
        v += ww * at(di, dj, dk);
      }
  return v;
}

double eval_kappa(const Medium& m, const Vec3d& x) {
  switch (m.kind) {
    case Medium::Constant:
      return m.kappa;
    case Medium::TwoLayered: {
      const double t = x[m.axis];
      if (t < m.eta) return m.kappa_down;
      if (t > m.eta + m.eps || m.eps == 0.0) return (t == m.eta) ? m.kappa_down : m.kappa_up;
      const double w = (t - m.eta) / m.eps;
      return m.kappa_down * (1.0 - w) + m.kappa_up * w;
    }
    case Medium::Gridded: {
      const double c = m.velocity.sample(x);
      if (!(c > 0.0)) data_error("eval_kappa: non-positive velocity sample");
      return m.omega / c;
    }
  }
  return 0.0;
}

std::vector<double> extend_to_subdomain(const Medium& m, const Box& cell, const LocalGrid& grid) {
  const std::int64_t count = grid.range.count();
  std::vector<double> kappa(count);
  for (std::int64_t id = 0; id < count; ++id) {
    const Vec3i p = grid.range.unlinear(id);
    Vec3d x{0.0, 0.0, 0.0};
    for (int a = 0; a < grid.dim; ++a) x[a] = std::clamp(grid.coord(a, p[a]), cell.lo[a], cell.hi[a]);
    kappa[id] = eval_kappa(m, x);
  }
  return kappa;
}

Csr assemble(const LocalGrid& grid, const PmlCoefficients& coeffs, const std::vector<double>& kappa) {
  if (static_cast<std::int64_t>(kappa.size()) != grid.range.count())
    config_error("assemble: kappa field size does not match grid");
  Csr op;
  op.n = grid.range.count();
  op.row_ptr.assign(op.n + 1, 0);
  const int stencil = 2 * grid.dim + 1;
  op.col.reserve(op.n * stencil);
  op.val.reserve(op.n * stencil);
  for (std::int64_t r = 0; r < op.n; ++r) {
    const Vec3i p = grid.range.unlinear(r);
    if (grid.on_shell(p)) {
      op.col.push_back(r);
      op.val.push_back(Complex(1.0, 0.0));
      op.row_ptr[r + 1] = static_cast<std::int64_t>(op.col.size());
      continue;
    }
    Complex diag = coeffs.jacobian(p) * kappa[r] * kappa[r];
    std::int64_t lc[6];
    Complex lv[6];
    int nl = 0;
    for (int a = 0; a < grid.dim; ++a)
      for (int s = -1; s <= 1; s += 2) {
        Vec3i q = p;
        q[a] += s;
        Vec3i half = p;
        if (s == -1) half[a] -= 1;
        const Complex c = coeffs.coupling(a, half);
        diag -= c;
        if (!grid.on_shell(q)) {
          lc[nl] = grid.range.linear(q);
          lv[nl] = c;
          ++nl;
        }
      }
    // insertion sort by column (at most 6 links)
    for (int i = 1; i < nl; ++i)
      for (int j = i; j > 0 && lc[j] < lc[j - 1]; --j) {
        std::swap(lc[j], lc[j - 1]);
        std::swap(lv[j], lv[j - 1]);
      }
    bool diag_done = false;
    for (int i = 0; i < nl; ++i) {
      if (!diag_done && lc[i] > r) {
        op.col.push_back(r);
        op.val.push_back(diag);
        diag_done = true;
      }
      op.col.push_back(lc[i]);
      op.val.push_back(lv[i]);
    }
    if (!diag_done) {
      op.col.push_back(r);
      op.val.push_back(diag);
    }
    op.row_ptr[r + 1] = static_cast<std::int64_t>(op.col.size());
  }
  return op;
}

std::vector<Vec3i> sweep_plan(int dim, int rounds) {
  if (dim != 2 && dim != 3) config_error("SweepPlan: dim must be 2 or 3");
  if (rounds < 1) config_error("SweepPlan: rounds must be >= 1");
  static const Vec3i o2[4] = {{1, 1, 1}, {-1, 1, 1}, {1, -1, 1}, {-1, -1, 1}};
  static const Vec3i o3[8] = {{1, 1, 1},  {-1, 1, 1},  {1, -1, 1},  {-1, -1, 1},
                              {1, 1, -1}, {-1, 1, -1}, {1, -1, -1}, {-1, -1, -1}};
  std::vector<Vec3i> plan;
  const int per = 1 << dim;
  for (int r = 0; r < rounds; ++r)
    for (int l = 0; l < per; ++l) plan.push_back(dim == 2 ? o2[l] : o3[l]);
  return plan;
}

namespace {
bool similar(int dim, const Vec3i& t, const Vec3i& s) {
  int dot = 0;
  for (int a = 0; a < dim; ++a) {
    dot += t[a] * s[a];
    if (dim == 3 && t[a] * s[a] < 0) return false;
  }
  return dot > 0;
}
bool opposite2(const Vec3i& a, const Vec3i& b) { return a[0] == -b[0] && a[1] == -b[1]; }
bool rule4(const Vec3i& t, const Vec3i& gen, const Vec3i& use) {
  for (int drop = 0; drop < 3; ++drop) {
    const int p = (drop + 1) % 3, q = (drop + 2) % 3;
    const int zeros = (t[p] == 0) + (t[q] == 0);
    if (zeros != 1) continue;
    if (gen[p] == -use[p] && gen[q] == -use[q]) return true;
  }
  return false;
}
}  // namespace

int route_trace(const std::vector<Vec3i>& plan, int dim, int gen_sweep, int axis, int sign) {
  Vec3i t{0, 0, 0};
  t[axis] = sign;
  const Vec3i gen = plan[gen_sweep - 1];
  for (int l = gen_sweep; l <= static_cast<int>(plan.size()); ++l) {
    const Vec3i use = plan[l - 1];
    if (!similar(dim, t, use)) continue;
    if (l == gen_sweep) return l;
    if (dim == 2) {
      if (opposite2(gen, use)) continue;
    } else if (rule4(t, gen, use)) {
      continue;
    }
    return l;
  }
  return 0;
}

int sweep_step_count(const Vec3i& counts, int dim) {
  int s = 1;
  for (int a = 0; a < dim; ++a) s += counts[a] - 1;
  return s;
}

int step_of(const Vec3i& counts, int dim, const Vec3i& d, const Vec3i& sub) {
  int s = 1;
  for (int a = 0; a < dim; ++a) s += d[a] == 1 ? sub[a] : counts[a] - 1 - sub[a];
  return s;
}

}  // namespace hsb
