// The paper's cost model of pipelined multi-RHS sweeping (include/helmsweep/pipeline.hpp,
// src/pipeline.cpp:20-111), so GPU-measured subdomain solve times can be fed into it and the
// device scheduler compared with it. Host-only.
//
// Scenario: one unit-capacity processor per subdomain, n_rhs right-hand sides, n_iter DDM
// applications each (2^dim sweeps per application), every subdomain solve costing t0.
//   closed form   per RHS = 2^dim n_iter t0 + steps / n_rhs * t0, idle = steps / (2^dim n_iter n_rhs)
//   simulation    tasks (rhs, sweep, subdomain); (l, p) waits for every (l', q) whose trace toward
//                 p routes to sweep l (route_trace); each tick every processor starts its ready
//                 task with the smallest (rhs, sweep), completions release dependents at the tick
//                 boundary; makespan = ticks * t0.
#include <algorithm>
#include <cstdint>
#include <queue>
#include <vector>

#include "helmsweep_b200.h"
#include "hs_common.hpp"
#include "hs_setup.hpp"

namespace hsb {
std::string& last_error_ref();
}

namespace {

using hsb::Error;

struct Scenario {
  int dim;
  hsb::Vec3i counts;
  int n_rhs, n_iter;
  double t0;
  void validate() const {
    if (dim != 2 && dim != 3) hsb::config_error("PipelineScenario: dim must be 2 or 3");
    for (int a = 0; a < dim; ++a)
      if (counts[a] < 1) hsb::config_error("PipelineScenario: counts must be >= 1");
    if (n_rhs < 1 || n_iter < 1 || !(t0 > 0.0)) hsb::config_error("PipelineScenario: n_rhs, n_iter and t0 must be positive");
  }
  hsb::Vec3i cnt3() const {
    hsb::Vec3i c = counts;
    for (int a = dim; a < 3; ++a) c[a] = 1;
    return c;
  }
};

template <class F>
int pipe_guarded(F&& fn) {
  try {
    fn();
    return HS_OK;
  } catch (const Error& e) {
    hsb::last_error_ref() = e.what();
    return e.code;
  } catch (const std::exception& e) {
    hsb::last_error_ref() = e.what();
    return HS_ERR_INTERNAL;
  }
}

}  // namespace

extern "C" {

int hs_pipeline_cost(int dim, const int counts[3], int n_rhs, int n_iter, double t0, double* average_per_rhs,
                     double* idle_fraction) {
  return pipe_guarded([&] {
    const Scenario s{dim, {counts[0], counts[1], counts[2]}, n_rhs, n_iter, t0};
    s.validate();
    const double sweeps = static_cast<double>(1 << dim) * n_iter;
    const int steps = hsb::sweep_step_count(s.cnt3(), dim);
    if (average_per_rhs) *average_per_rhs = sweeps * t0 + static_cast<double>(steps) / n_rhs * t0;
    if (idle_fraction) *idle_fraction = steps / (sweeps * n_rhs);
  });
}

int hs_pipeline_simulate(int dim, const int counts[3], int n_rhs, int n_iter, double t0, double* completion_times,
                         double* makespan, double* average_per_rhs) {
  return pipe_guarded([&] {
    const Scenario s{dim, {counts[0], counts[1], counts[2]}, n_rhs, n_iter, t0};
    s.validate();
    const hsb::Vec3i c = s.cnt3();
    const int nsub = c[0] * c[1] * c[2];
    const int S = (1 << dim) * n_iter;  // sweeps per RHS
    const std::vector<hsb::Vec3i> plan = hsb::sweep_plan(dim, n_iter);
    // trace DAG, the same for every RHS: out[l0 * nsub + q] = tasks released by (l0, q); need = in-degrees
    std::vector<std::vector<int>> out(static_cast<size_t>(S) * nsub);
    std::vector<int> need(static_cast<size_t>(S) * nsub, 0);
    for (int lg = 1; lg <= S; ++lg)
      for (int ax = 0; ax < dim; ++ax)
        for (int sg = -1; sg <= 1; sg += 2) {
          const int lu = hsb::route_trace(plan, dim, lg, ax, sg);
          if (lu == 0) continue;
          for (int q = 0; q < nsub; ++q) {
            hsb::Vec3i pq{q % c[0], (q / c[0]) % c[1], q / (c[0] * c[1])};
            pq[ax] += sg;
            if (pq[ax] < 0 || pq[ax] >= c[ax]) continue;
            const int p = (pq[2] * c[1] + pq[1]) * c[0] + pq[0];
            out[static_cast<size_t>(lg - 1) * nsub + q].push_back((lu - 1) * nsub + p);
            ++need[static_cast<size_t>(lu - 1) * nsub + p];
          }
        }
    // per-processor ready sets ordered by (rhs, sweep) packed into one key
    using Key = std::int64_t;
    auto key = [&](int r, int l0) { return static_cast<Key>(r) * S + l0; };
    std::vector<std::priority_queue<Key, std::vector<Key>, std::greater<Key>>> ready(nsub);
    std::vector<int> left(static_cast<size_t>(n_rhs) * S * nsub);
    for (int r = 0; r < n_rhs; ++r)
      for (int t = 0; t < S * nsub; ++t) {
        left[static_cast<size_t>(r) * S * nsub + t] = need[t];
        if (need[t] == 0) ready[t % nsub].push(key(r, t / nsub));
      }
    std::vector<double> done_at(n_rhs, 0.0);
    std::vector<Key> run(nsub, -1);
    const std::int64_t total = static_cast<std::int64_t>(n_rhs) * S * nsub;
    std::int64_t finished = 0, tick = 0;
    while (finished < total) {
      ++tick;
      for (int p = 0; p < nsub; ++p) {
        run[p] = -1;
        if (!ready[p].empty()) {
          run[p] = ready[p].top();
          ready[p].pop();
        }
      }
      for (int p = 0; p < nsub; ++p) {
        if (run[p] < 0) continue;
        const int r = static_cast<int>(run[p] / S), l0 = static_cast<int>(run[p] % S);
        ++finished;
        done_at[r] = std::max(done_at[r], tick * t0);
        for (int t : out[static_cast<size_t>(l0) * nsub + p])
          if (--left[static_cast<size_t>(r) * S * nsub + t] == 0) ready[t % nsub].push(key(r, t / nsub));
      }
    }
    if (completion_times) std::copy(done_at.begin(), done_at.end(), completion_times);
    if (makespan) *makespan = tick * t0;
    if (average_per_rhs) *average_per_rhs = tick * t0 / n_rhs;
  });
}

}  // extern "C"
