// C-ABI driver around the UNMODIFIED reference sources (/root/reference/proj/src/*.cpp),
// compiled in place by oracle/Makefile into oracle/_ref/libhelmsweep_ref.so.
//
// TEST INFRASTRUCTURE ONLY. Used by tests/ (to pin the numpy restatement and to
// generate golden fixtures) and by bench.py's reference / cpu_baseline arm. The
// product (paper_2003_02585_b200/) never links or loads it.
//
// Every entry point goes through the reference's own public API:
//   DdmSolver / ddm_solve / scale_source   proj/include/helmsweep/sweeper.hpp:70-107
//   factorize / Factorization::solve        proj/include/helmsweep/direct.hpp:22-41
//   gmres                                   proj/include/helmsweep/krylov.hpp:30-36
//   sample_source / global_direct_solve     proj/include/helmsweep/harness.hpp:17-41
//   parse_config_text                       proj/include/helmsweep/config.hpp:55
//   write_velocity_grid / read_velocity_grid proj/include/helmsweep/media.hpp:22-27
//   write_field / read_field                proj/include/helmsweep/harness.hpp:10-16
#include <Eigen/Dense>  // the oracle shim (hsref_blas_active)
#include <chrono>
#include <cstdint>
#include <span>
#include <cstring>
#include <memory>
#include <string>

#include "helmsweep/harness.hpp"
#include "helmsweep/pipeline.hpp"

using namespace helmsweep;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const SingularMatrixError*>(&e)) return 3;
  if (dynamic_cast<const DataError*>(&e)) return 2;
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  return 5;
}

struct Solver {
  RunConfig cfg;
  std::unique_ptr<DdmSolver> ddm;
};

struct Fact {
  SparseOperator op;
  Factorization f;
};

Complex* cx(double* p) { return reinterpret_cast<Complex*>(p); }
const Complex* cx(const double* p) { return reinterpret_cast<const Complex*>(p); }
}  // namespace

extern "C" {

struct hsref_report {
  double factor_seconds, sweep_seconds_total, median_subdomain_solve_seconds;
  long long traces_generated, traces_routed, traces_discarded, local_solves, skipped_zero_solves;
  int n_sweeps, n_round_residuals;
};

const char* hsref_last_error() { return g_err.c_str(); }

// 1 when the Eigen-subset shim routes large dense products to OpenBLAS (shim/Eigen/Dense).
int hsref_blas_active() { return hsref_blas::active() ? 1 : 0; }

// Parses reference config text (key = value lines, src/config.cpp:90-196); an
// optional workers override (>0) replaces sweep.workers; builds DdmSolver
// (factorizes every subdomain).
int hsref_solver_create(const char* cfg_text, int workers, void** out) {
  try {
    auto s = std::make_unique<Solver>();
    s->cfg = parse_config_text(cfg_text);
    if (workers > 0) s->cfg.workers = workers;
    s->ddm = std::make_unique<DdmSolver>(s->cfg.setup());
    *out = s.release();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void hsref_solver_destroy(void* h) { delete static_cast<Solver*>(h); }

int hsref_solver_info(void* h, int* dim, long long* global_n, int* nsub, double* factor_seconds,
                      int lo[3], int hi[3], double hh[3], double origin[3]) {
  auto* s = static_cast<Solver*>(h);
  const LocalGrid& g = s->ddm->global_grid();
  *dim = g.dim;
  *global_n = g.node_count();
  *nsub = s->ddm->partition().cell_count();
  *factor_seconds = s->ddm->factor_seconds();
  for (int a = 0; a < 3; ++a) {
    lo[a] = g.range.lo[a];
    hi[a] = g.range.hi[a];
    hh[a] = g.h[a];
    origin[a] = g.origin[a];
  }
  return 0;
}

// Physical source f of the config on the padded global grid (harness.cpp:85-144).
int hsref_sample_source(void* h, double* f_out) {
  try {
    auto* s = static_cast<Solver*>(h);
    CVector f = sample_source(s->cfg.source, s->cfg.medium, s->ddm->global_grid(), s->cfg.interior);
    std::memcpy(f_out, f.data(), f.size() * sizeof(Complex));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int hsref_scale_source(void* h, const double* f, double* b_out) {
  try {
    auto* s = static_cast<Solver*>(h);
    const std::int64_t n = s->ddm->global_grid().node_count();
    CVector b = s->ddm->scale_source(std::span<const Complex>(cx(f), n));
    std::memcpy(b_out, b.data(), b.size() * sizeof(Complex));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// One ddm_solve (sweeper.cpp:176-334). Per-sweep arrays must hold rounds*2^dim
// doubles; round_res must hold `rounds` doubles.
int hsref_ddm_solve(void* h, const double* b, double* u_out, int rounds, int track,
                    hsref_report* rep, double* sweep_seconds, double* contrib_norm,
                    double* round_res) {
  try {
    auto* s = static_cast<Solver*>(h);
    const std::int64_t n = s->ddm->global_grid().node_count();
    SolveReport r;
    CVector u = s->ddm->ddm_solve(std::span<const Complex>(cx(b), n), rounds, &r, track != 0);
    std::memcpy(u_out, u.data(), u.size() * sizeof(Complex));
    if (rep) {
      rep->factor_seconds = r.factor_seconds;
      rep->sweep_seconds_total = r.sweep_seconds_total;
      rep->median_subdomain_solve_seconds = r.median_subdomain_solve_seconds;
      rep->traces_generated = r.traces_generated;
      rep->traces_routed = r.traces_routed;
      rep->traces_discarded = r.traces_discarded;
      rep->local_solves = r.local_solves;
      rep->skipped_zero_solves = r.skipped_zero_solves;
      rep->n_sweeps = static_cast<int>(r.sweep_seconds.size());
      rep->n_round_residuals = static_cast<int>(r.round_residuals.size());
    }
    for (size_t i = 0; i < r.sweep_seconds.size(); ++i) {
      if (sweep_seconds) sweep_seconds[i] = r.sweep_seconds[i];
      if (contrib_norm) contrib_norm[i] = r.sweep_contrib_norm[i];
    }
    if (round_res)
      for (size_t i = 0; i < r.round_residuals.size(); ++i) round_res[i] = r.round_residuals[i];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Subdomain state accessors (SubdomainState, sweeper.hpp:30-42).
int hsref_sub_info(void* h, int sub, int lo[3], int hi[3], int olo[3], int ohi[3],
                   long long* n, long long* nnz, long long* factor_nnz, long long* peak_bytes) {
  auto* s = static_cast<Solver*>(h);
  const SubdomainState& st = s->ddm->states().at(sub);
  for (int a = 0; a < 3; ++a) {
    lo[a] = st.grid.range.lo[a];
    hi[a] = st.grid.range.hi[a];
    olo[a] = st.owned.lo[a];
    ohi[a] = st.owned.hi[a];
  }
  *n = st.op.n;
  *nnz = static_cast<long long>(st.op.val.size());
  *factor_nnz = st.fact.stats().factor_nnz;
  *peak_bytes = st.fact.stats().peak_bytes;
  return 0;
}

int hsref_sub_csr(void* h, int sub, long long* row_ptr, long long* col, double* val) {
  auto* s = static_cast<Solver*>(h);
  const SparseOperator& op = s->ddm->states().at(sub).op;
  for (size_t i = 0; i < op.row_ptr.size(); ++i) row_ptr[i] = op.row_ptr[i];
  for (size_t i = 0; i < op.col.size(); ++i) col[i] = op.col[i];
  std::memcpy(val, op.val.data(), op.val.size() * sizeof(Complex));
  return 0;
}

int hsref_sub_solve(void* h, int sub, const double* rhs, double* x_out) {
  try {
    auto* s = static_cast<Solver*>(h);
    const SubdomainState& st = s->ddm->states().at(sub);
    CVector x = st.fact.solve(std::span<const Complex>(cx(rhs), st.op.n));
    std::memcpy(x_out, x.data(), x.size() * sizeof(Complex));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int hsref_global_csr_nnz(void* h, long long* nnz) {
  auto* s = static_cast<Solver*>(h);
  *nnz = static_cast<long long>(s->ddm->global_op().val.size());
  return 0;
}

int hsref_global_csr(void* h, long long* row_ptr, long long* col, double* val) {
  auto* s = static_cast<Solver*>(h);
  const SparseOperator& op = s->ddm->global_op();
  for (size_t i = 0; i < op.row_ptr.size(); ++i) row_ptr[i] = op.row_ptr[i];
  for (size_t i = 0; i < op.col.size(); ++i) col[i] = op.col[i];
  std::memcpy(val, op.val.data(), op.val.size() * sizeof(Complex));
  return 0;
}

// GMRES with the DDM preconditioner exactly as run_precond wires it
// (harness.cpp:285-305): op = global_op().apply, pc = ddm_solve(v, rounds).
int hsref_gmres(void* h, const double* b, double* x_out, double tol, int maxit, int rounds,
                int* iterations, int* converged, double* history /* maxit+1 */,
                int* n_history, double* final_res, double* true_res, double* seconds) {
  try {
    auto* s = static_cast<Solver*>(h);
    const std::int64_t n = s->ddm->global_grid().node_count();
    const SparseOperator& A = s->ddm->global_op();
    LinearMap apply_op = [&](std::span<const Complex> v) { return A.apply(v); };
    LinearMap apply_pc = [&](std::span<const Complex> v) {
      return s->ddm->ddm_solve(v, rounds, nullptr, false);
    };
    GmresConfig gc;
    gc.tol = tol;
    gc.max_iterations = maxit;
    const auto t0 = std::chrono::steady_clock::now();
    GmresResult g = gmres(apply_op, apply_pc, std::span<const Complex>(cx(b), n), gc);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(x_out, g.x.data(), g.x.size() * sizeof(Complex));
    *iterations = g.iterations;
    *converged = g.converged ? 1 : 0;
    *n_history = static_cast<int>(g.history.size());
    for (size_t i = 0; i < g.history.size(); ++i) history[i] = g.history[i];
    *final_res = g.final_residual;
    *true_res = g.true_residual;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int hsref_global_direct_solve(void* h, const double* f, double* u_out) {
  try {
    auto* s = static_cast<Solver*>(h);
    const std::int64_t n = s->ddm->global_grid().node_count();
    CVector u = global_direct_solve(s->cfg, std::span<const Complex>(cx(f), n), nullptr);
    std::memcpy(u_out, u.data(), u.size() * sizeof(Complex));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Sweep plan / routing (sweeper.cpp:10-73) and step groups (geometry.cpp:156-177).
int hsref_route(int dim, int rounds, int gen_sweep, int axis, int sign) {
  SweepPlan plan = SweepPlan::make(dim, rounds);
  return route_trace(plan, gen_sweep, Cardinal{axis, sign});
}

int hsref_step_of(int dim, const int counts[3], int sweep_index /*0-based in one round*/,
                  const int sub[3]) {
  SweepPlan plan = SweepPlan::make(dim, 1);
  Vec3i c{counts[0], counts[1], counts[2]}, s{sub[0], sub[1], sub[2]};
  return step_of(c, dim, plan.sweeps[sweep_index], s);
}

// Standalone factorization of a CSR on a grid range (direct.hpp:40) and solve.
int hsref_factorize(int dim, const int lo[3], const int hi[3], long long n,
                    const long long* row_ptr, const long long* col, const double* val,
                    void** out, long long* factor_nnz, long long* pivot_index) {
  auto fa = std::make_unique<Fact>();
  try {
    fa->op.grid.dim = dim;
    fa->op.grid.range.dim = dim;
    for (int a = 0; a < 3; ++a) {
      fa->op.grid.range.lo[a] = lo[a];
      fa->op.grid.range.hi[a] = hi[a];
      fa->op.grid.h[a] = 1.0;
    }
    fa->op.n = n;
    fa->op.row_ptr.assign(row_ptr, row_ptr + n + 1);
    fa->op.col.assign(col, col + row_ptr[n]);
    fa->op.val.assign(cx(val), cx(val) + row_ptr[n]);
    fa->f = factorize(fa->op);
    *factor_nnz = fa->f.stats().factor_nnz;
    *out = fa.release();
    return 0;
  } catch (const SingularMatrixError& e) {
    *pivot_index = e.pivot_index;
    return fail(e);
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int hsref_fact_solve(void* h, const double* rhs, double* x_out) {
  try {
    auto* fa = static_cast<Fact*>(h);
    CVector x = fa->f.solve(std::span<const Complex>(cx(rhs), fa->op.n));
    std::memcpy(x_out, x.data(), x.size() * sizeof(Complex));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void hsref_fact_destroy(void* h) { delete static_cast<Fact*>(h); }

// tests/test_direct.cpp:14-37 pml_operator: unit box, h=1/n, range [-pad, n+pad],
// PmlSpec{width=pad}, constant kappa, J-scaled assembly. Returns sizes first
// (val==nullptr) then fills.
int hsref_pml_operator(int dim, int n, int pad, double kappa, long long* rows, long long* nnz,
                       long long* row_ptr, long long* col, double* val) {
  try {
    Box box;
    box.dim = dim;
    box.lo = {0.0, 0.0, 0.0};
    box.hi = {1.0, 1.0, 1.0};
    LocalGrid g;
    g.dim = dim;
    g.range.dim = dim;
    for (int a = 0; a < dim; ++a) {
      g.h[a] = 1.0 / n;
      g.origin[a] = 0.0;
      g.range.lo[a] = -pad;
      g.range.hi[a] = n + pad;
    }
    PmlSpec spec;
    spec.width = pad;
    PmlCoefficients c = build_coefficients(spec, box, g);
    std::vector<double> kap(g.node_count(), kappa);
    SparseOperator op = assemble(g, c, kap, true);
    *rows = op.n;
    *nnz = static_cast<long long>(op.val.size());
    if (val) {
      for (size_t i = 0; i < op.row_ptr.size(); ++i) row_ptr[i] = op.row_ptr[i];
      for (size_t i = 0; i < op.col.size(); ++i) col[i] = op.col[i];
      std::memcpy(val, op.val.data(), op.val.size() * sizeof(Complex));
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}


// On-disk formats through the reference's own writers / readers (golden fixtures of the HSVG
// velocity grid and the HSFD field dump).
int hsref_write_velocity_grid(const char* path, int dim, const int n[3], const double origin[3],
                              const double spacing[3], const float* c) {
  try {
    VelocityGrid g;
    g.dim = dim;
    std::int64_t count = 1;
    for (int a = 0; a < 3; ++a) {
      g.n[a] = n[a];
      g.origin[a] = origin[a];
      g.spacing[a] = spacing[a];
    }
    for (int a = 0; a < dim; ++a) count *= n[a];
    g.c.assign(c, c + count);
    write_velocity_grid(path, g);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int hsref_read_velocity_grid(const char* path, int* dim, int n[3], double origin[3], double spacing[3],
                             float* c, long long cap, long long* count) {
  try {
    VelocityGrid g = read_velocity_grid(path);
    *dim = g.dim;
    for (int a = 0; a < 3; ++a) {
      n[a] = g.n[a];
      origin[a] = g.origin[a];
      spacing[a] = g.spacing[a];
    }
    *count = static_cast<long long>(g.c.size());
    if (c && cap >= *count) std::memcpy(c, g.c.data(), g.c.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int hsref_write_field(const char* path, int dim, const int lo[3], const int hi[3], const double h[3],
                      const double origin[3], const double* u) {
  try {
    LocalGrid g;
    g.dim = dim;
    g.range.dim = dim;
    for (int a = 0; a < 3; ++a) {
      g.range.lo[a] = lo[a];
      g.range.hi[a] = hi[a];
      g.h[a] = h[a];
      g.origin[a] = origin[a];
    }
    write_field(path, g, std::span<const Complex>(cx(u), static_cast<size_t>(g.node_count())));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}


// Pipeline cost model through the reference (src/pipeline.cpp:20-111).
int hsref_pipeline(int dim, const int counts[3], int n_rhs, int n_iter, double t0, double* avg_closed,
                   double* idle, double* makespan, double* avg_sim, double* completion) {
  try {
    PipelineScenario sc;
    sc.dim = dim;
    sc.counts = Vec3i{counts[0], counts[1], counts[2]};
    sc.n_rhs = n_rhs;
    sc.n_iter = n_iter;
    sc.t0 = t0;
    const PipelineCost c = average_time_per_rhs(sc);
    const PipelineSimulation sim = simulate_pipeline(sc);
    *avg_closed = c.average_per_rhs;
    *idle = c.idle_fraction;
    *makespan = sim.makespan;
    *avg_sim = sim.average_per_rhs;
    for (int r = 0; r < n_rhs; ++r) completion[r] = sim.completion_times[r];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
