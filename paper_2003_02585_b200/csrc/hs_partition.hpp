// Macro-step levels of the (sweep, subdomain) task graph and the subdomain ownership of a
// partitioned (multi-rank) solve. Host-only; shared by the device scheduler (hs_ddm.cu) and the
// pure-host C-ABI queries (hs_partition_owners / hs_partition_traffic).
#pragma once

#include <vector>

#include "hs_setup.hpp"

namespace hsb {

// Route table route_h[(l-1)*dirs + d] of sweep_plan(dim, rounds) (src/sweeper.cpp:58-73).
std::vector<int> route_table(const std::vector<Vec3i>& plan, int dim, int nsweeps);

// Levels of the task graph: task (l, id) runs at macro-step level[(l-1)*nsub + id] - 1, one
// after the latest of the tasks whose traces it consumes and the accumulate of sweep l - nbuf
// whose x buffer it reuses. accl[l] = macro-steps through sweep l (accumulate after accl[l]-1).
void task_levels(int dim, const Vec3i& counts, const std::vector<Vec3i>& plan, const std::vector<int>& route_h,
                 int nsweeps, int nbuf, std::vector<int>& level, std::vector<int>& accl);

// Balanced static ownership of the subdomains over `world` ranks: the candidate among
// axis-cyclic layouts with the smallest sum over macro-steps of the busiest
// rank's task count, ties broken by fewer cross-rank faces, then improved by pairwise swaps.
std::vector<int> default_owners(int dim, const Vec3i& counts, int world, int nbuf = 4);

struct PartitionCost {
  int macro_steps = 0;
  long long makespan_tasks = 0;   // sum over macro-steps of the busiest rank's task count
  long long cross_faces = 0;      // neighbour pairs with different owners
  std::vector<long long> traces;  // [src * world + dst]: routed traces per application
};
PartitionCost partition_cost(int dim, const Vec3i& counts, int rounds, int world, const std::vector<int>& owner,
                             int nbuf = 4);

}  // namespace hsb
