// Task-graph levels and subdomain ownership for partitioned solves (see hs_partition.hpp).
#include "hs_partition.hpp"

#include <algorithm>
#include <cstdint>
#include <numeric>

namespace hsb {

namespace {

Vec3i unflatten(const Vec3i& counts, int dim, int id) {
  Vec3i s{0, 0, 0};
  for (int a = 0; a < dim; ++a) {
    s[a] = id % counts[a];
    id /= counts[a];
  }
  return s;
}
int flatten(const Vec3i& counts, int dim, const Vec3i& s) {
  int id = 0;
  for (int a = dim - 1; a >= 0; --a) id = id * counts[a] + s[a];
  return id;
}
int cell_count(const Vec3i& counts, int dim) { return counts[0] * counts[1] * (dim == 3 ? counts[2] : 1); }

}  // namespace

std::vector<int> route_table(const std::vector<Vec3i>& plan, int dim, int nsweeps) {
  const int dirs = 2 * dim;
  std::vector<int> r(static_cast<size_t>(nsweeps) * dirs, 0);
  for (int l = 1; l <= nsweeps; ++l)
    for (int d = 0; d < dirs; ++d) r[(l - 1) * dirs + d] = route_trace(plan, dim, l, d / 2, (d & 1) ? 1 : -1);
  return r;
}

void task_levels(int dim, const Vec3i& counts, const std::vector<Vec3i>& plan, const std::vector<int>& route_h,
                 int nsweeps, int nbuf, std::vector<int>& level, std::vector<int>& accl) {
  const int nsub = cell_count(counts, dim), dirs = 2 * dim;
  level.assign(static_cast<size_t>(nsweeps) * nsub, 0);
  accl.assign(nsweeps + 1, 0);
  for (int l = 1; l <= nsweeps; ++l) {
    // within a sweep, in step order: a trace routed into the same sweep comes from an earlier step
    std::vector<int> order(nsub);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
      return step_of(counts, dim, plan[l - 1], unflatten(counts, dim, x)) <
             step_of(counts, dim, plan[l - 1], unflatten(counts, dim, y));
    });
    int done = 0;
    for (int id : order) {
      const Vec3i sub = unflatten(counts, dim, id);
      int lev = l > nbuf ? accl[l - nbuf] : 0;
      for (int ax = 0; ax < dim; ++ax)
        for (int sg = -1; sg <= 1; sg += 2) {
          Vec3i nb = sub;
          nb[ax] -= sg;  // the neighbour whose trace travels along (ax, sg) into id
          if (nb[ax] < 0 || nb[ax] >= counts[ax]) continue;
          const int nbid = flatten(counts, dim, nb);
          const int d = 2 * ax + (sg > 0 ? 1 : 0);
          for (int lp = 1; lp <= l; ++lp)
            if (route_h[(lp - 1) * dirs + d] == l) lev = std::max(lev, level[static_cast<size_t>(lp - 1) * nsub + nbid]);
        }
      level[static_cast<size_t>(l - 1) * nsub + id] = lev + 1;
      done = std::max(done, lev + 1);
    }
    accl[l] = std::max(done, accl[l - 1]);
  }
}

PartitionCost partition_cost(int dim, const Vec3i& counts, int rounds, int world, const std::vector<int>& owner,
                             int nbuf) {
  PartitionCost c;
  const int nsub = cell_count(counts, dim), dirs = 2 * dim;
  const std::vector<Vec3i> plan = sweep_plan(dim, rounds);
  const int nsweeps = static_cast<int>(plan.size());
  const std::vector<int> route_h = route_table(plan, dim, nsweeps);
  std::vector<int> level, accl;
  task_levels(dim, counts, plan, route_h, nsweeps, std::min(nbuf, nsweeps), level, accl);
  c.macro_steps = accl[nsweeps];
  std::vector<int> load(static_cast<size_t>(c.macro_steps) * world, 0);
  for (int l = 1; l <= nsweeps; ++l)
    for (int id = 0; id < nsub; ++id) ++load[static_cast<size_t>(level[(l - 1) * nsub + id] - 1) * world + owner[id]];
  for (int m = 0; m < c.macro_steps; ++m)
    c.makespan_tasks += *std::max_element(load.begin() + static_cast<long long>(m) * world,
                                          load.begin() + static_cast<long long>(m + 1) * world);
  c.traces.assign(static_cast<size_t>(world) * world, 0);
  for (int id = 0; id < nsub; ++id) {
    const Vec3i s = unflatten(counts, dim, id);
    for (int d = 0; d < dirs; ++d) {
      Vec3i t = s;
      t[d / 2] += (d & 1) ? 1 : -1;
      if (t[d / 2] < 0 || t[d / 2] >= counts[d / 2]) continue;
      const int tid = flatten(counts, dim, t);
      if (owner[tid] != owner[id] && (d & 1)) ++c.cross_faces;
      for (int l = 1; l <= nsweeps; ++l)
        if (route_h[(l - 1) * dirs + d] != 0) ++c.traces[static_cast<size_t>(owner[id]) * world + owner[tid]];
    }
  }
  return c;
}

std::vector<int> default_owners(int dim, const Vec3i& counts, int world, int nbuf) {
  const int nsub = cell_count(counts, dim);
  if (world <= 1) return std::vector<int>(nsub, 0);
  auto better = [](const PartitionCost& a, const PartitionCost& b) {
    return a.makespan_tasks != b.makespan_tasks ? a.makespan_tasks < b.makespan_tasks : a.cross_faces < b.cross_faces;
  };
  // candidates: cyclic along each axis with the other axes shifting the cycle (SURVEY.md §8(e):
  // owner = (i + N_1 (j mod ceil(G / N_1))) mod G in 2D), and plain cyclic over the flattened id
  std::vector<std::vector<int>> cand;
  for (int a = 0; a < dim; ++a)
    for (int shift = 0; shift <= 2; ++shift) {
      std::vector<int> o(nsub);
      for (int id = 0; id < nsub; ++id) {
        const Vec3i s = unflatten(counts, dim, id);
        const int reps = std::max(1, (world + counts[a] - 1) / counts[a]);
        long long v = s[a];
        int mul = counts[a];
        for (int b = 0; b < dim; ++b) {
          if (b == a) continue;
          v += shift == 0 ? static_cast<long long>(mul) * (s[b] % reps) : static_cast<long long>(shift) * s[b];
          mul *= reps;
        }
        o[id] = static_cast<int>(v % world);
      }
      cand.push_back(o);
    }
  {
    std::vector<int> o(nsub);
    for (int id = 0; id < nsub; ++id) o[id] = id % world;
    cand.push_back(o);
  }
  std::vector<int> best = cand[0];
  PartitionCost bc = partition_cost(dim, counts, 1, world, best, nbuf);
  for (size_t i = 1; i < cand.size(); ++i) {
    const PartitionCost c = partition_cost(dim, counts, 1, world, cand[i], nbuf);
    if (better(c, bc)) {
      bc = c;
      best = cand[i];
    }
  }
  // pairwise swaps (small partitions only; the cost is O(nsub^2) evaluations per pass)
  if (nsub <= 64) {
    for (int pass = 0; pass < 2; ++pass) {
      bool improved = false;
      for (int a = 0; a < nsub; ++a)
        for (int b = a + 1; b < nsub; ++b) {
          if (best[a] == best[b]) continue;
          std::swap(best[a], best[b]);
          const PartitionCost c = partition_cost(dim, counts, 1, world, best, nbuf);
          if (better(c, bc)) {
            bc = c;
            improved = true;
          } else {
            std::swap(best[a], best[b]);
          }
        }
      if (!improved) break;
    }
  }
  return best;
}

}  // namespace hsb
