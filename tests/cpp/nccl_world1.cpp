// C++ client of the C-ABI (include/helmsweep_b200.h) driving the native NCCL transport at world 1:
// hs_nccl_unique_id -> hs_ddm_create_nccl runs the partitioned machinery (ownership, home-node
// accumulation, ncclAllReduce of u / norms / counters on the solver stream, graph capture) over one
// rank, which must reproduce the plain solver bit for bit. Built and run by tests/test_gpu_nccl.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "helmsweep_b200.h"

static int fail(const char* what, int rc) {
  std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, hs_last_error());
  return 1;
}

int main() {
  int v = 0;
  if (int rc = hs_nccl_version(&v)) return fail("hs_nccl_version", rc);
  std::printf("nccl %d\n", v);
  hs_problem p;
  std::memset(&p, 0, sizeof(p));
  p.dim = 2;
  for (int a = 0; a < 3; ++a) {
    p.interior_lo[a] = 0.0;
    p.interior_hi[a] = 1.0;
    p.intervals[a] = a < 2 ? 48 : 1;
    p.counts[a] = a < 2 ? 3 : 1;
  }
  p.pml_width = 8;
  p.pml_strength = 2.0;
  p.pml_exponent = 2;
  p.medium_kind = 0;
  p.kappa = 9.0 * M_PI;
  p.workers = 1;
  hs_ddm *plain = nullptr, *nat = nullptr;
  int ps = -1;
  int64_t pi = -1;
  if (int rc = hs_ddm_create(&p, 0, &plain, &ps, &pi)) return fail("hs_ddm_create", rc);
  unsigned char id[128];
  if (int rc = hs_nccl_unique_id(id)) return fail("hs_nccl_unique_id", rc);
  if (int rc = hs_ddm_create_nccl(&p, 0, 0, 1, nullptr, id, &nat, &ps, &pi)) return fail("hs_ddm_create_nccl", rc);
  int64_t n = 0;
  hs_ddm_info(plain, nullptr, &n, nullptr, nullptr, nullptr, nullptr);
  const int R = 3, rounds = 2;
  std::vector<double> f(2 * n * R, 0.0), b(2 * n * R), u0(2 * n * R), u1(2 * n * R);
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  for (int r = 0; r < R; ++r)  // a few point-like sources per RHS
    for (int q = 0; q < 5; ++q) f[2 * (r * n + static_cast<int64_t>(std::abs(U(g)) * (n - 1)))] = U(g);
  if (int rc = hs_ddm_scale_source(plain, R, f.data(), b.data())) return fail("scale_source", rc);
  std::vector<hs_solve_report> r0(R), r1(R);
  if (int rc = hs_ddm_solve(plain, R, b.data(), u0.data(), rounds, 1, r0.data())) return fail("solve plain", rc);
  for (int rep = 0; rep < 2; ++rep)  // second call replays the captured graph
    if (int rc = hs_ddm_solve(nat, R, b.data(), u1.data(), rounds, 1, r1.data())) return fail("solve nccl", rc);
  if (std::memcmp(u0.data(), u1.data(), u0.size() * sizeof(double)) != 0) {
    std::fprintf(stderr, "u differs between the plain and the NCCL world-1 solver\n");
    return 1;
  }
  for (int r = 0; r < R; ++r) {
    if (r0[r].local_solves != r1[r].local_solves || r0[r].skipped_zero_solves != r1[r].skipped_zero_solves ||
        r0[r].traces_routed != r1[r].traces_routed || r0[r].traces_discarded != r1[r].traces_discarded) {
      std::fprintf(stderr, "counters differ for rhs %d\n", r);
      return 1;
    }
    for (int q = 0; q < rounds; ++q)
      if (r0[r].round_residuals[q] != r1[r].round_residuals[q]) {
        std::fprintf(stderr, "round residual differs for rhs %d round %d\n", r, q);
        return 1;
      }
  }
  int rk = -1, w = -1, owned = -1;
  int64_t sent = -1, msgs = -1;
  hs_ddm_partition_info(nat, &rk, &w, &owned, &sent, &msgs);
  std::printf("ok: %lld nodes, %d RHS, %d rounds, world %d owns %d subdomains, %lld doubles sent\n",
              static_cast<long long>(n), R, rounds, w, owned, static_cast<long long>(sent));
  hs_ddm_destroy(nat);
  hs_ddm_destroy(plain);
  return 0;
}
