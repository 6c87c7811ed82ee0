// Header-only C++ facade over the helmsweep_b200 C-ABI, mirroring the reference's hot-path
// classes so host callers (the reference's run_direct / run_precond, src/harness.cpp:269-305)
// switch by changing a namespace:
//
//   reference                                   B200 facade
//   helmsweep::factorize(op)        direct.hpp:40    helmsweep_b200::factorize(...)
//   Factorization::solve / solve_inplace :28-29  helmsweep_b200::Factorization::solve / ...
//   DdmSolver(setup)              sweeper.hpp:70  helmsweep_b200::DdmSolver(problem)
//   DdmSolver::ddm_solve(b, rounds, rep, tr) :84  DdmSolver::ddm_solve(...) (+ batched form)
//   gmres(op, pc, b, cfg)          krylov.hpp:35  DdmSolver::gmres(...)
//   global_direct_solve(cfg, f)   harness.cpp:185  DdmSolver::global_direct_solve(...)
//
// Errors are rethrown as ConfigError / DataError / SingularMatrixError(pivot_index) with the
// reference's meaning (include/helmsweep/common.hpp:18-35); CudaError when no device works.
#pragma once

#include <complex>
#include <cstdint>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "helmsweep_b200.h"

namespace helmsweep_b200 {

using Complex = std::complex<double>;
using CVector = std::vector<Complex>;

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SingularMatrixError : std::runtime_error {
  SingularMatrixError(const std::string& m, std::int64_t p) : std::runtime_error(m), pivot_index(p) {}
  std::int64_t pivot_index;
};

inline void check(int rc, std::int64_t pivot = -1) {
  if (rc == HS_OK) return;
  const std::string msg = hs_last_error();
  switch (rc) {
    case HS_ERR_CONFIG: throw ConfigError(msg);
    case HS_ERR_DATA: throw DataError(msg);
    case HS_ERR_SINGULAR: throw SingularMatrixError(msg, pivot);
    case HS_ERR_CUDA: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

inline double* dp(Complex* p) { return reinterpret_cast<double*>(p); }
inline const double* dp(const Complex* p) { return reinterpret_cast<const double*>(p); }

class Factorization {
 public:
  Factorization(int dim, const int lo[3], const int hi[3], const std::vector<std::int64_t>& row_ptr,
                const std::vector<std::int64_t>& col, const CVector& val, int device = 0) {
    std::int64_t pivot = -1;
    check(hs_factorize(dim, lo, hi, static_cast<std::int64_t>(row_ptr.size()) - 1, row_ptr.data(), col.data(),
                       dp(val.data()), device, &f_, &stats_, &pivot),
          pivot);
  }
  ~Factorization() { hs_factor_destroy(f_); }
  Factorization(const Factorization&) = delete;
  Factorization& operator=(const Factorization&) = delete;

  CVector solve(const CVector& rhs) const {
    CVector x(rhs);
    solve_inplace(x);
    return x;
  }
  void solve_inplace(CVector& x) const {
    if (static_cast<std::int64_t>(x.size()) != stats_.n) throw ConfigError("Factorization::solve: length mismatch");
    check(hs_factor_solve(f_, 1, dp(x.data())));
  }
  // nrhs vectors of length n, RHS-major
  void solve_batch(std::vector<CVector>& xs) const {
    CVector flat;
    for (auto& x : xs) flat.insert(flat.end(), x.begin(), x.end());
    check(hs_factor_solve(f_, static_cast<int>(xs.size()), dp(flat.data())));
    for (size_t r = 0; r < xs.size(); ++r)
      std::copy(flat.begin() + r * stats_.n, flat.begin() + (r + 1) * stats_.n, xs[r].begin());
  }
  const hs_factor_stats& stats() const { return stats_; }

 private:
  hs_factor* f_ = nullptr;
  hs_factor_stats stats_{};
};

class DdmSolver {
 public:
  explicit DdmSolver(const hs_problem& setup, int device = 0) {
    int sub = -1;
    std::int64_t pivot = -1;
    check(hs_ddm_create(&setup, device, &s_, &sub, &pivot), pivot);
    check(hs_ddm_info(s_, &dim_, &n_, &nsub_, &factor_seconds_, nullptr, nullptr));
  }
  // Subdomain-partitioned solver, one per rank (hs_ddm_create_partitioned): owner may be null
  // (hs_partition_owners); exchange / allreduce carry the messages (e.g. NCCL).
  DdmSolver(const hs_problem& setup, int device, int rank, int world, const int* owner, hs_exchange_fn exchange,
            hs_allreduce_fn allreduce, void* user) {
    int sub = -1;
    std::int64_t pivot = -1;
    check(hs_ddm_create_partitioned(&setup, device, rank, world, owner, exchange, allreduce, user, &s_, &sub, &pivot),
          pivot);
    check(hs_ddm_info(s_, &dim_, &n_, &nsub_, &factor_seconds_, nullptr, nullptr));
  }
  ~DdmSolver() { hs_ddm_destroy(s_); }
  DdmSolver(const DdmSolver&) = delete;
  DdmSolver& operator=(const DdmSolver&) = delete;

  std::int64_t global_n() const { return n_; }
  double factor_seconds() const { return factor_seconds_; }

  CVector scale_source(const CVector& f) const {
    CVector b(f.size());
    check(hs_ddm_scale_source(s_, 1, dp(f.data()), dp(b.data())));
    return b;
  }
  CVector ddm_solve(const CVector& b, int rounds, hs_solve_report* report = nullptr, bool track_residuals = false) {
    CVector u(b.size());
    check(hs_ddm_solve(s_, 1, dp(b.data()), dp(u.data()), rounds, track_residuals ? 1 : 0, report));
    return u;
  }
  // batched: b holds nrhs vectors back to back; reports (optional) nrhs entries
  CVector ddm_solve_batch(const CVector& b, int nrhs, int rounds, hs_solve_report* reports = nullptr,
                          bool track_residuals = false) {
    CVector u(b.size());
    check(hs_ddm_solve(s_, nrhs, dp(b.data()), dp(u.data()), rounds, track_residuals ? 1 : 0, reports));
    return u;
  }
  CVector apply_op(const CVector& x) {
    CVector y(x.size());
    check(hs_ddm_apply_op(s_, 1, dp(x.data()), dp(y.data())));
    return y;
  }
  // global_direct_solve (src/harness.cpp:185-214): A^-1 (J f) on the global grid, device LDL^T
  CVector global_direct_solve(const CVector& f, hs_factor_stats* stats = nullptr) {
    CVector u(f.size());
    check(hs_ddm_global_solve(s_, 1, dp(f.data()), dp(u.data()), stats));
    return u;
  }
  CVector gmres(const CVector& b, double tol, int maxit, int rounds, hs_gmres_report* report = nullptr) {
    CVector x(b.size());
    hs_gmres_report local{};
    check(hs_gmres(s_, 1, dp(b.data()), dp(x.data()), tol, maxit, rounds, report ? report : &local));
    return x;
  }
  // GMRES(restart) cycles up to maxit iterations (BASELINE config 4's GMRES(30))
  CVector gmres_restarted(const CVector& b, double tol, int maxit, int restart, int rounds,
                          hs_gmres_report* report = nullptr) {
    CVector x(b.size());
    hs_gmres_report local{};
    check(hs_gmres_restarted(s_, 1, dp(b.data()), dp(x.data()), tol, maxit, restart, rounds, report ? report : &local));
    return x;
  }

 private:
  hs_ddm* s_ = nullptr;
  int dim_ = 0, nsub_ = 0;
  std::int64_t n_ = 0;
  double factor_seconds_ = 0.0;
};

// gmres(op, pc, b, cfg) (include/helmsweep/krylov.hpp:30-36) for any pair of LinearOperators given
// as callables CVector -> CVector (pc may be empty: identity); the Krylov loop runs on `device`.
using LinearOperatorFn = std::function<CVector(const CVector&)>;
namespace detail {
struct LinopCtx {
  const LinearOperatorFn* op;
  const LinearOperatorFn* pc;
  std::size_t n;
};
inline int linop_apply(const LinearOperatorFn& f, std::size_t n, int nrhs, const double* x, double* y) {
  try {
    for (int r = 0; r < nrhs; ++r) {
      CVector v(n);
      std::memcpy(static_cast<void*>(v.data()), x + 2 * r * n, sizeof(Complex) * n);
      const CVector w = f(v);
      if (w.size() != n) return 1;
      std::memcpy(y + 2 * r * n, static_cast<const void*>(w.data()), sizeof(Complex) * n);
    }
    return 0;
  } catch (...) {
    return 1;
  }
}
inline int linop_op(void* u, int nrhs, const double* x, double* y, void*) {
  const LinopCtx& c = *static_cast<const LinopCtx*>(u);
  return linop_apply(*c.op, c.n, nrhs, x, y);
}
inline int linop_pc(void* u, int nrhs, const double* x, double* y, void*) {
  const LinopCtx& c = *static_cast<const LinopCtx*>(u);
  return linop_apply(*c.pc, c.n, nrhs, x, y);
}
}  // namespace detail
inline CVector gmres(const LinearOperatorFn& op, const LinearOperatorFn& pc, const CVector& b, double tol, int maxit,
                     hs_gmres_report* report = nullptr, int device = 0) {
  detail::LinopCtx ctx{&op, &pc, b.size()};
  CVector x(b.size());
  hs_gmres_report local{};
  check(hs_gmres_general(device, static_cast<std::int64_t>(b.size()), 1, detail::linop_op, pc ? detail::linop_pc : nullptr,
                         &ctx, 0, dp(b.data()), dp(x.data()), tol, maxit, maxit, report ? report : &local));
  return x;
}

}  // namespace helmsweep_b200
