// Symbolic nested dissection (see hs_symbolic.hpp).
#include "hs_symbolic.hpp"

#include <algorithm>
#include <numeric>

namespace hsb {

namespace {

struct Node {
  Vec3i blo{0, 0, 0}, bhi{0, 0, 0};
  int c0 = -1, c1 = -1;
  std::vector<int> sep, bnd;  // local linear ids
};

struct Builder {
  int dim;
  GridRange range;
  std::vector<Node> tree;

  void box_ids(const Vec3i& lo, const Vec3i& hi, std::vector<int>& out) const {
    for (int k = lo[2]; k <= hi[2]; ++k)
      for (int j = lo[1]; j <= hi[1]; ++j)
        for (int i = lo[0]; i <= hi[0]; ++i) out.push_back(static_cast<int>(range.linear({i, j, k})));
  }

  // src/direct.cpp:91-136
  int build_rec(Vec3i blo, Vec3i bhi) {
    Node nd;
    nd.blo = blo;
    nd.bhi = bhi;
    std::int64_t count = 1;
    int la = 0;
    for (int a = 0; a < dim; ++a) {
      count *= bhi[a] - blo[a] + 1;
      if (bhi[a] - blo[a] > bhi[la] - blo[la]) la = a;
    }
    const int id = static_cast<int>(tree.size());
    tree.push_back(nd);
    if (count <= kLeafNodes || bhi[la] - blo[la] < 2) {
      std::vector<int> s;
      box_ids(blo, bhi, s);
      tree[id].sep = std::move(s);
      return id;
    }
    const int mid = (blo[la] + bhi[la]) / 2;  // C++ truncation, as the reference
    Vec3i lhi = bhi, rlo = blo;
    lhi[la] = mid - 1;
    rlo[la] = mid + 1;
    int c0 = -1, c1 = -1;
    if (lhi[la] >= blo[la]) c0 = build_rec(blo, lhi);
    if (rlo[la] <= bhi[la]) c1 = build_rec(rlo, bhi);
    tree[id].c0 = c0;
    tree[id].c1 = c1;
    Vec3i slo = blo, shi = bhi;
    slo[la] = shi[la] = mid;
    std::vector<int> s;
    box_ids(slo, shi, s);
    tree[id].sep = std::move(s);
    return id;
  }

  // src/direct.cpp:138-155
  void compute_bnd(Node& nd) const {
    for (int a = 0; a < dim; ++a)
      for (int s = 0; s < 2; ++s) {
        const int plane = s == 0 ? nd.blo[a] - 1 : nd.bhi[a] + 1;
        if (plane < range.lo[a] || plane > range.hi[a]) continue;
        Vec3i lo = nd.blo, hi = nd.bhi;
        lo[a] = hi[a] = plane;
        box_ids(lo, hi, nd.bnd);
      }
  }
};

}  // namespace

std::unique_ptr<SymbolicClass> build_symbolic(int dim, const GridRange& range,
                                              const std::vector<std::int64_t>& row_ptr,
                                              const std::vector<std::int64_t>& col) {
  Builder b{dim, range, {}};
  Vec3i lo = range.lo, hi = range.hi;
  for (int a = dim; a < 3; ++a) lo[a] = hi[a] = 0;
  b.build_rec(lo, hi);
  for (auto& nd : b.tree) b.compute_bnd(nd);
  // postorder (src/direct.cpp:163-178)
  std::vector<int> post;
  {
    std::vector<std::pair<int, int>> stack{{0, 0}};
    while (!stack.empty()) {
      auto& [id, ph] = stack.back();
      if (ph == 0) {
        ph = 1;
        if (b.tree[id].c0 >= 0) stack.push_back({b.tree[id].c0, 0});
      } else if (ph == 1) {
        ph = 2;
        if (b.tree[id].c1 >= 0) stack.push_back({b.tree[id].c1, 0});
      } else {
        post.push_back(id);
        stack.pop_back();
      }
    }
  }
  auto sc = std::make_unique<SymbolicClass>();
  SymbolicClass& c = *sc;
  c.dim = dim;
  for (int a = 0; a < 3; ++a) c.size[a] = a < dim ? range.size(a) : 1;
  c.n = range.count();
  const int nf = static_cast<int>(post.size());
  std::vector<int> front_of_node(b.tree.size(), -1);
  for (int f = 0; f < nf; ++f) front_of_node[post[f]] = f;

  c.elim_of_local.assign(c.n, -1);
  c.local_of_elim.assign(c.n, -1);
  int pos = 0;
  c.fronts.resize(nf);
  for (int f = 0; f < nf; ++f) {
    const Node& nd = b.tree[post[f]];
    c.fronts[f].sep_off = pos;
    c.fronts[f].k = static_cast<int>(nd.sep.size());
    for (int g : nd.sep) {
      c.elim_of_local[g] = pos;
      c.local_of_elim[pos] = g;
      c.sep_local.push_back(g);
      ++pos;
    }
  }
  if (pos != c.n) throw Error(kInternal, "symbolic: elimination order does not cover the grid");

  // bnd sorted by elimination position (src/direct.cpp:205-206); tree links
  for (int f = 0; f < nf; ++f) {
    const Node& nd = b.tree[post[f]];
    FrontDesc& fd = c.fronts[f];
    std::vector<int> be;
    be.reserve(nd.bnd.size());
    for (int g : nd.bnd) be.push_back(c.elim_of_local[g]);
    std::sort(be.begin(), be.end());
    fd.bnd_off = static_cast<int>(c.bnd_elim.size());
    c.bnd_elim.insert(c.bnd_elim.end(), be.begin(), be.end());
    fd.m = fd.k + static_cast<int>(be.size());
    fd.child[0] = nd.c0 >= 0 ? front_of_node[nd.c0] : -1;
    fd.child[1] = nd.c1 >= 0 ? front_of_node[nd.c1] : -1;
    for (int ch : fd.child)
      if (ch >= 0) c.fronts[ch].parent = f;
    c.max_m = std::max(c.max_m, fd.m);
    c.max_k = std::max(c.max_k, fd.k);
  }
  // child -> parent position maps (the merge map of src/direct.cpp:245-252)
  for (int f = 0; f < nf; ++f) {
    FrontDesc& fd = c.fronts[f];
    for (int q = 0; q < 2; ++q) {
      const int ch = fd.child[q];
      fd.cmap_off[q] = static_cast<int>(c.child_map.size());
      if (ch < 0) continue;
      const FrontDesc& cd = c.fronts[ch];
      const int cb = cd.m - cd.k;
      for (int i = 0; i < cb; ++i) {
        const int e = c.bnd_elim[cd.bnd_off + i];
        int p;
        if (e >= fd.sep_off && e < fd.sep_off + fd.k) {
          p = e - fd.sep_off;
        } else {
          const int* bb = c.bnd_elim.data() + fd.bnd_off;
          const int* it = std::lower_bound(bb, bb + (fd.m - fd.k), e);
          if (it == bb + (fd.m - fd.k) || *it != e)
            throw Error(kInternal, "symbolic: child bnd not contained in parent front");
          p = fd.k + static_cast<int>(it - bb);
        }
        c.child_map.push_back(p);
      }
    }
  }
  // heights (children first in postorder) and depths
  for (int f = 0; f < nf; ++f) {
    int h = 0;
    for (int ch : c.fronts[f].child)
      if (ch >= 0) h = std::max(h, c.fronts[ch].height + 1);
    c.fronts[f].height = h;
    c.max_height = std::max(c.max_height, h);
  }
  for (int f = nf - 1; f >= 0; --f) {
    const int p = c.fronts[f].parent;
    c.fronts[f].depth = p >= 0 ? c.fronts[p].depth + 1 : 0;
    c.max_depth = std::max(c.max_depth, c.fronts[f].depth);
  }
  // original-entry scatter lists (src/direct.cpp:219-237), lower triangle only
  for (int f = 0; f < nf; ++f) {
    FrontDesc& fd = c.fronts[f];
    fd.orig_off = static_cast<int>(c.orig_fpos.size());
    for (int qi = 0; qi < fd.k; ++qi) {
      const int q = c.local_of_elim[fd.sep_off + qi];
      const int eq = fd.sep_off + qi;
      for (std::int64_t e = row_ptr[q]; e < row_ptr[q + 1]; ++e) {
        const int cc = static_cast<int>(col[e]);
        const int ec = c.elim_of_local[cc];
        if (ec < eq) continue;
        int ci;
        if (ec < fd.sep_off + fd.k) {
          ci = ec - fd.sep_off;
        } else {
          const int* bb = c.bnd_elim.data() + fd.bnd_off;
          const int* it = std::lower_bound(bb, bb + (fd.m - fd.k), ec);
          if (it == bb + (fd.m - fd.k) || *it != ec)
            throw Error(kInternal, "symbolic: coupling outside the front");
          ci = fd.k + static_cast<int>(it - bb);
        }
        c.orig_fpos.push_back(qi * fd.m + ci);  // column-major lower entry (ci >= qi)
        c.orig_eidx.push_back(static_cast<int>(e));
      }
    }
    fd.orig_cnt = static_cast<int>(c.orig_fpos.size()) - fd.orig_off;
  }
  // storage offsets and the reference's stats accounting
  long long fac = 0, v = 0, fw = 0, tt = 0;
  std::int64_t active = 0, peak = 0;
  for (int f = 0; f < nf; ++f) {
    FrontDesc& fd = c.fronts[f];
    fd.fac_off = fac;
    fac += front_block_elems(fd.m, fd.k);
    fd.v_off = v;
    v += fd.m - fd.k;
    fd.t_off = tt;
    tt += fd.m;
    fd.f_off = fw;
    fw += static_cast<long long>(fd.m) * fd.m;
    const std::int64_t m = fd.m, k = fd.k;
    c.factor_nnz += m * k;
    c.packed_entries += m * k - k * (k - 1) / 2;
    active += m * m * 16;
    peak = std::max(peak, active);
    for (int ch : fd.child)
      if (ch >= 0) {
        const std::int64_t cb = c.fronts[ch].m - c.fronts[ch].k;
        active -= cb * cb * 16;
      }
    if (m > k) active += (m - k) * (m - k) * 16;
    active -= m * m * 16;
    active += m * k * 16;
    peak = std::max(peak, active);
  }
  c.fac_total = fac;
  c.v_total = v;
  // Dense front workspaces (m x m each) live from their front's level (assembly, elimination)
  // to their parent's level (extend-add of the Schur complement), the device factorizing one tree
  // height at a time. Fronts whose lifetimes overlap get disjoint ranges: first fit, largest
  // first. The workspace is the peak over heights instead of the sum over all fronts (3D 57^3
  // subdomains: about 6x less), so more subdomains are factorized side by side.
  {
    std::vector<int> ord(nf);
    std::iota(ord.begin(), ord.end(), 0);
    auto sz = [&](int f) { return static_cast<long long>(c.fronts[f].m) * c.fronts[f].m; };
    auto life_hi = [&](int f) { return c.fronts[f].parent >= 0 ? c.fronts[c.fronts[f].parent].height : c.fronts[f].height; };
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return sz(a) > sz(b); });
    std::vector<int> placed;
    std::vector<std::pair<long long, long long>> busy;
    long long top = 0;
    for (int f : ord) {
      const int lo = c.fronts[f].height, hi = life_hi(f);
      busy.clear();
      for (int g : placed)
        if (c.fronts[g].height <= hi && lo <= life_hi(g)) busy.emplace_back(c.fronts[g].f_off, c.fronts[g].f_off + sz(g));
      std::sort(busy.begin(), busy.end());
      long long off = 0;
      for (const auto& iv : busy) {
        if (iv.first >= off + sz(f)) break;
        off = std::max(off, iv.second);
      }
      c.fronts[f].f_off = off;
      top = std::max(top, off + sz(f));
      placed.push_back(f);
    }
    fw = top;
  }
  c.f_total = fw;
  c.t_total = tt;
  c.peak_bytes = peak;
  // schedules
  c.order_up.resize(nf);
  std::iota(c.order_up.begin(), c.order_up.end(), 0);
  std::stable_sort(c.order_up.begin(), c.order_up.end(),
                   [&](int a, int bb) { return c.fronts[a].height < c.fronts[bb].height; });
  c.level_start_up.assign(c.max_height + 2, 0);
  for (int f = 0; f < nf; ++f) c.level_start_up[c.fronts[f].height + 1]++;
  for (int h = 0; h <= c.max_height; ++h) c.level_start_up[h + 1] += c.level_start_up[h];
  c.order_down.resize(nf);
  std::iota(c.order_down.begin(), c.order_down.end(), 0);
  std::stable_sort(c.order_down.begin(), c.order_down.end(),
                   [&](int a, int bb) { return c.fronts[a].depth < c.fronts[bb].depth; });
  c.csr_row_ptr = row_ptr;
  c.csr_col = col;
  return sc;
}

bool same_structure(const SymbolicClass& a, const SymbolicClass& b) {
  if (a.dim != b.dim || a.size != b.size || a.fronts.size() != b.fronts.size()) return false;
  for (size_t f = 0; f < a.fronts.size(); ++f) {
    const FrontDesc &x = a.fronts[f], &y = b.fronts[f];
    if (x.k != y.k || x.m != y.m || x.parent != y.parent || x.child[0] != y.child[0] ||
        x.child[1] != y.child[1])
      return false;
  }
  return a.sep_local == b.sep_local && a.bnd_elim == b.bnd_elim && a.csr_col == b.csr_col &&
         a.csr_row_ptr == b.csr_row_ptr;
}

}  // namespace hsb
