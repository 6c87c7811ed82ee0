/*
 * helmsweep_b200 — C-ABI of the B200-native trace-transfer diagonal-sweeping DDM hot path
 * (arXiv 2003.02585). Plain pointers and sizes only; every complex128 array is interleaved
 * (re, im) doubles, and multi-RHS host/device arrays are RHS-major (nrhs consecutive vectors
 * of length n — each one exactly a reference CVector).
 *
 * Each entry point replaces one reference interface (paths relative to
 * /root/reference/proj):
 *
 *   hs_factorize / hs_factor_solve / hs_factor_stats / hs_factor_destroy
 *       factorize(const SparseOperator&)            include/helmsweep/direct.hpp:40
 *       Factorization::solve / solve_inplace         include/helmsweep/direct.hpp:28-29
 *       Factorization::stats / FactorStats           include/helmsweep/direct.hpp:10-17,31
 *   hs_ddm_create / hs_ddm_destroy / hs_ddm_info / hs_ddm_sub_stats
 *       DdmSolver::DdmSolver(const ProblemSetup&)    include/helmsweep/sweeper.hpp:70-71
 *       build_subdomain_states                       include/helmsweep/sweeper.hpp:111-114
 *   hs_ddm_scale_source
 *       DdmSolver::scale_source                      include/helmsweep/sweeper.hpp:88
 *   hs_ddm_solve / hs_ddm_solve_device
 *       DdmSolver::ddm_solve                         include/helmsweep/sweeper.hpp:84-85
 *       (batched over nrhs right-hand sides; one SolveReport per RHS)
 *   hs_ddm_apply_op
 *       SparseOperator::apply on DdmSolver::global_op include/helmsweep/operator.hpp:25,
 *                                                    include/helmsweep/sweeper.hpp:77
 *   hs_ddm_global_solve
 *       global_direct_solve(cfg, f)                  src/harness.cpp:185-214
 *   hs_read/write_velocity_grid, hs_read_velocity_csv, hs_write_field / hs_read_field
 *       read/write_velocity_grid, read_velocity_csv  include/helmsweep/media.hpp:22-27
 *       write_field / read_field                     include/helmsweep/harness.hpp:10-16
 *   hs_pipeline_cost / hs_pipeline_simulate
 *       average_time_per_rhs / simulate_pipeline     include/helmsweep/pipeline.hpp:27-44
 *   hs_gmres, hs_gmres_general
 *       gmres(op, precond, b, cfg) as wired by run_precond
 *                                                    include/helmsweep/krylov.hpp:30-36,
 *                                                    src/harness.cpp:285-305
 *
 * Status codes mirror the reference exception classes (include/helmsweep/common.hpp:18-35):
 * HS_ERR_CONFIG = ConfigError, HS_ERR_DATA = DataError, HS_ERR_SINGULAR =
 * SingularMatrixError (pivot index returned through an out-parameter). hs_last_error()
 * returns the message of the last failure on the calling thread.
 *
 * There is no CPU fallback: every numeric entry point runs on the CUDA device and fails
 * with HS_ERR_CUDA when none is usable.
 */
#ifndef HELMSWEEP_B200_H
#define HELMSWEEP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HS_OK = 0,
  HS_ERR_CONFIG = 1,
  HS_ERR_DATA = 2,
  HS_ERR_SINGULAR = 3,
  HS_ERR_CUDA = 4,
  HS_ERR_INTERNAL = 5
};

#define HS_MAX_SWEEPS 64
#define HS_MAX_ROUNDS 16
#define HS_MAX_GMRES_HISTORY 257

typedef struct hs_factor hs_factor;
typedef struct hs_ddm hs_ddm;

/* FactorStats (include/helmsweep/direct.hpp:10-17). */
typedef struct {
  int64_t n;
  int64_t matrix_nnz;
  int64_t factor_nnz; /* sum over fronts of m*k, the reference's convention */
  int64_t peak_bytes; /* reference active-front accounting */
  double factor_seconds;
} hs_factor_stats;

/* ProblemSetup (include/helmsweep/sweeper.hpp:58-65) with WaveNumberModel
 * (include/helmsweep/media.hpp:31-55) and PmlSpec (include/helmsweep/pml.hpp:8-18). */
typedef struct {
  int dim;
  double interior_lo[3], interior_hi[3];
  int intervals[3];
  int counts[3];
  int pml_width;
  double pml_strength;
  int pml_exponent;
  int medium_kind; /* 0 constant, 1 two_layered, 2 gridded */
  double kappa;
  double kappa_down, kappa_up;
  int interface_axis;
  double eta, eps;
  int vel_dim;
  int vel_n[3];
  double vel_origin[3], vel_spacing[3];
  const float* vel_c; /* gridded velocity samples, axis 0 fastest (copied) */
  double omega;
  int workers; /* accepted for ProblemSetup parity; the device schedules itself */
} hs_problem;

/* SolveReport (include/helmsweep/sweeper.hpp:44-56). Device timings are CUDA-event based
 * and describe the whole batched application the RHS belonged to. */
typedef struct {
  double factor_seconds;
  double sweep_seconds_total;
  double median_subdomain_solve_seconds;
  int64_t traces_generated, traces_routed, traces_discarded;
  int64_t local_solves, skipped_zero_solves;
  int n_sweeps;
  int n_round_residuals;
  double sweep_seconds[HS_MAX_SWEEPS];
  double sweep_contrib_norm[HS_MAX_SWEEPS];
  double round_residuals[HS_MAX_ROUNDS];
} hs_solve_report;

/* GmresResult (include/helmsweep/krylov.hpp:22-29), without x. */
typedef struct {
  int iterations;
  int converged;
  double final_residual;
  double true_residual;
  int n_history;
  double history[HS_MAX_GMRES_HISTORY];
} hs_gmres_report;

const char* hs_last_error(void);
int hs_device_count(void);

/* ---- Factorization ---------------------------------------------------------------- */
/* CSR of a J-scaled operator over the grid range [lo, hi] (dim axes). pivot_index (may be
 * NULL) receives the reference's grid node of a failing pivot on HS_ERR_SINGULAR. */
int hs_factorize(int dim, const int lo[3], const int hi[3], int64_t n, const int64_t* row_ptr,
                 const int64_t* col, const double* val, int device, hs_factor** out,
                 hs_factor_stats* stats, int64_t* pivot_index);
/* x: nrhs host vectors of length n, solved in place. */
int hs_factor_solve(hs_factor* f, int nrhs, double* x);
/* d_x: nrhs device vectors (RHS-major) solved in place on `stream` (cudaStream_t or NULL). */
int hs_factor_solve_device(hs_factor* f, int nrhs, double* d_x, void* stream);
int hs_factor_stats_get(const hs_factor* f, hs_factor_stats* stats);
void hs_factor_destroy(hs_factor* f);

/* ---- DdmSolver ------------------------------------------------------------------- */
/* Builds the padded global grid, partitions it and factorizes every subdomain on the GPU.
 * On HS_ERR_SINGULAR, pivot_sub / pivot_index name the subdomain and its grid node. */
int hs_ddm_create(const hs_problem* setup, int device, hs_ddm** out, int* pivot_sub,
                  int64_t* pivot_index);
void hs_ddm_destroy(hs_ddm* s);
/* global grid: dim, node count, subdomain count, factorization seconds, padded range. */
int hs_ddm_info(const hs_ddm* s, int* dim, int64_t* global_n, int* nsub, double* factor_seconds,
                int lo[3], int hi[3]);
int hs_ddm_sub_stats(const hs_ddm* s, int sub, hs_factor_stats* stats);
/* b = J f on non-shell nodes (nrhs RHS-major vectors, host). */
int hs_ddm_scale_source(const hs_ddm* s, int nrhs, const double* f, double* b);
/* One DDM application (rounds x 2^dim sweeps) for nrhs right-hand sides; host buffers.
 * reports (may be NULL) receives nrhs SolveReports. */
int hs_ddm_solve(hs_ddm* s, int nrhs, const double* b, double* u, int rounds, int track_residuals,
                 hs_solve_report* reports);
/* Same with device buffers (RHS-major), asynchronous on `stream` when reports == NULL. */
int hs_ddm_solve_device(hs_ddm* s, int nrhs, const double* d_b, double* d_u, int rounds,
                        int track_residuals, hs_solve_report* reports, void* stream);
/* y = A x with A the global J-scaled operator (host buffers, nrhs vectors). */
int hs_ddm_apply_op(hs_ddm* s, int nrhs, const double* x, double* y);
/* Right-preconditioned GMRES with the DDM preconditioner (rounds sweeps cycles), one
 * independent Krylov process per RHS, batched through the device. */
int hs_gmres(hs_ddm* s, int nrhs, const double* b, double* x, double tol, int maxit, int rounds,
             hs_gmres_report* reports);
/* GMRES(restart): cycles of at most `restart` Arnoldi steps from the current iterate (residual
 * b - A x recomputed, convergence still |g_{j+1}| / ||b|| <= tol) until tol or `maxit` total
 * iterations; BASELINE config 4 asks for GMRES(30). The reference's gmres never restarts
 * (include/helmsweep/krylov.hpp:32-34), which is hs_gmres (restart = maxit); the two agree
 * whenever the iteration count stays within `restart`. */
int hs_gmres_restarted(hs_ddm* s, int nrhs, const double* b, double* x, double tol, int maxit, int restart,
                       int rounds, hs_gmres_report* reports);

/* A LinearMap (include/helmsweep/krylov.hpp:30: CVector -> CVector) as a callback: y = Op x for nrhs
 * vectors of n complex128 each, RHS-major (each vector one reference CVector). With on_device = 0
 * x and y are host arrays and stream is NULL; with on_device = 1 they are device arrays and the
 * callback enqueues its work on `stream` (a cudaStream_t). Returns 0, or nonzero to abort the solve
 * (HS_ERR_DATA). */
typedef int (*hs_linop_fn)(void* user, int nrhs, const double* x, double* y, void* stream);
/* gmres(op, pc, b, cfg) (include/helmsweep/krylov.hpp:30-36, src/krylov.cpp:17-123) for any
 * operator and right preconditioner: the Krylov loop of hs_gmres (MGS Arnoldi, complex Givens,
 * breakdown and convergence tests, one process per RHS, vectors and reductions on the device) with
 * the caller's callbacks in place of the global operator and the DDM application. pc = NULL is the
 * identity. restart >= maxit is the reference's full GMRES. b, x: host buffers, nrhs RHS-major
 * vectors of n complex128. */
int hs_gmres_general(int device, int64_t n, int nrhs, hs_linop_fn op, hs_linop_fn pc, void* user, int on_device,
                     const double* b, double* x, double tol, int maxit, int restart, hs_gmres_report* reports);

/* global_direct_solve (src/harness.cpp:185-214): u = A^-1 (J f) on the padded global grid with
 * the device sparse-direct factorization of the global J-scaled operator (factorized on first
 * use and kept by the handle; stats, may be NULL, receives its FactorStats). Host buffers, nrhs
 * RHS-major vectors; HS_ERR_CONFIG above the reference's memory guard (4.5e6 nodes in 2D,
 * 4.5e5 in 3D). nrhs = 0 only factorizes. */
int hs_ddm_global_solve(hs_ddm* s, int nrhs, const double* f, double* u, hs_factor_stats* stats);

/* Device profile of the most recent timed hs_ddm_solve[_device] batch: total duration of the
 * multifrontal solve launches (forward + backward, CUDA events), their count, the subdomain
 * solves they executed, and the algorithmic bytes / flops of those solves (SURVEY.md §8(d):
 * per solve (P_f + P_b)*16 + 2*R*N_loc*16 bytes and 8*(P_f + P_b)*R flops over packed factor
 * entries: P_f those of the fronts the forward pass needs -- all of them in sweep 1, past it
 * only fronts whose subtree holds a nonzero injection line, the others being exactly zero --
 * and P_b those of the fronts whose subtree holds a position the application reads back,
 * accumulated with a nonzero weight or extracted as a trace). */
int hs_ddm_profile(hs_ddm* s, double* solve_seconds, int64_t* solve_launches, int64_t* subdomain_solves,
                   double* alg_bytes, double* alg_flops);
/* Route table of the reference's route_trace (src/sweeper.cpp:58-73): target sweep of a
 * trace generated in sweep gen_sweep (1-based) travelling along (axis, sign); 0 = discard. */
int hs_route_trace(int dim, int rounds, int gen_sweep, int axis, int sign);

/* ---- On-disk formats (byte-exact with the reference) -------------------------------- */
/* HSVG velocity grid (include/helmsweep/media.hpp:22-27, src/media.cpp:58-100): "HSVG", u32
 * version 1, u32 dim, u32 n[3], f64 origin[3], f64 spacing[3], f32 samples (axis 0 fastest).
 * Readers fill the header and, when c != NULL and cap >= *count, the samples (call once with
 * c = NULL to size the buffer). Errors: HS_ERR_DATA (open, magic, version, dims, truncation,
 * VelocityGrid::validate). */
int hs_read_velocity_grid(const char* path, int* dim, int n[3], double origin[3], double spacing[3], float* c,
                          int64_t cap, int64_t* count);
int hs_write_velocity_grid(const char* path, int dim, const int n[3], const double origin[3], const double spacing[3],
                           const float* c);
/* CSV fallback (src/media.cpp:102-130): "dim,n..,origin..,spacing.." then one sample per line. */
int hs_read_velocity_csv(const char* path, int* dim, int n[3], double origin[3], double spacing[3], float* c,
                         int64_t cap, int64_t* count);
/* HSFD field dump (src/harness.cpp:32-83): "HSFD", u32 version 1, u32 dim, u32 n[3], i32 lo[3],
 * f64 h[3], f64 origin[3], complex128 values over the grid range [lo, hi] (axis 0 fastest). */
int hs_write_field(const char* path, int dim, const int lo[3], const int hi[3], const double h[3],
                   const double origin[3], const double* u);
int hs_read_field(const char* path, int* dim, int lo[3], int hi[3], double h[3], double origin[3], double* u,
                  int64_t cap, int64_t* count);

/* Shape of the device sweep schedule for `rounds` rounds:
 * macro-steps (dependency levels of the (sweep, subdomain) task graph), the widest one, the
 * reference's sequential step count (sweeps x anti-diagonal steps) and the x buffers in flight. */
int hs_ddm_schedule_info(hs_ddm* s, int rounds, int* macro_steps, int* max_width, int* sequential_steps,
                         int* buffers);

/* ---- Subdomain-partitioned DdmSolver over several ranks ------------
 * The reference runs every subdomain in one process (src/sweeper.cpp:263-283); here each rank
 * (one process per GPU) factorizes and solves only the subdomains `owner` assigns to it. All
 * ranks call hs_ddm_solve / hs_ddm_solve_device collectively with the same b. After each
 * macro-step a rank sends the traces it deposited for other ranks' subdomains (mailbox slot +
 * presence word, src/transfer.cpp:24-36) and the values of its subdomain solutions on nodes
 * another rank accumulates (each global node is accumulated by one "home" rank in the
 * reference's order, src/transfer.cpp:91-102), so u and the counters equal the single-process
 * result bit for bit. The transport is the caller's: `exchange` moves one message to / from
 * each listed peer (device buffers, offsets and counts in doubles, ordered on `stream`, e.g.
 * NCCL send/recv pairs); `allreduce` sums `count` device doubles over all ranks (the home-node
 * u slices, sweep norms, counters). Both return 0 on success. */
typedef int (*hs_exchange_fn)(void* user, int npeers, const int* peers, const int64_t* send_off,
                              const int64_t* send_count, const int64_t* recv_off, const int64_t* recv_count,
                              const double* send_buf, double* recv_buf, void* stream);
typedef int (*hs_allreduce_fn)(void* user, double* buf, int64_t count, void* stream);
/* Balanced default ownership (host only): owner[nsub], subdomains in flattened id order
 * (axis 0 fastest, src/geometry.cpp:105-122). */
int hs_partition_owners(int dim, const int counts[3], int world, int* owner);
/* Cost of an ownership (host only): macro-steps, sum over macro-steps of the busiest rank's task
 * count, cross-rank faces, and traces[src * world + dst] routed per application. */
int hs_partition_traffic(int dim, const int counts[3], int rounds, int world, const int* owner, int* macro_steps,
                         int64_t* makespan_tasks, int64_t* cross_faces, int64_t* traces);
/* owner may be NULL (hs_partition_owners). world == 1 is the plain hs_ddm_create. */
int hs_ddm_create_partitioned(const hs_problem* setup, int device, int rank, int world, const int* owner,
                              hs_exchange_fn exchange, hs_allreduce_fn allreduce, void* user, hs_ddm** out,
                              int* pivot_sub, int64_t* pivot_index);
/* Native NCCL transport (libnccl loaded at run time; no caller callbacks). One rank calls
 * hs_nccl_unique_id and distributes the 128 bytes to every rank (any channel); every rank then
 * calls hs_ddm_create_nccl with them (collective: it builds the library's own communicator). The
 * per-macro-step exchange runs as ncclSend/ncclRecv groups and the reductions as ncclAllReduce on
 * the solver stream, so applications stay CUDA-graph captured. world == 1 runs the partitioned
 * machinery over one rank (every node home, no peers). HS_ERR_CUDA when libnccl is missing. */
int hs_nccl_unique_id(unsigned char id[128]);
int hs_nccl_version(int* version);
int hs_ddm_create_nccl(const hs_problem* setup, int device, int rank, int world, const int* owner,
                       const unsigned char id[128], hs_ddm** out, int* pivot_sub, int64_t* pivot_index);
/* Owned subdomains of this rank and the exchange volume (doubles sent per application, for the
 * last batch width and rounds solved). */
int hs_ddm_partition_info(const hs_ddm* s, int* rank, int* world, int* owned, int64_t* sent_doubles,
                          int64_t* messages);

/* ---- Pipeline cost model (include/helmsweep/pipeline.hpp, src/pipeline.cpp:20-111) ------ */
/* PipelineScenario {dim, counts, n_rhs, n_iter, t0}: closed form average_time_per_rhs and the
 * discrete-event simulate_pipeline (one unit-capacity processor per subdomain, trace-routing
 * precedence). completion_times (may be NULL) receives n_rhs values. HS_ERR_CONFIG on bad input. */
int hs_pipeline_cost(int dim, const int counts[3], int n_rhs, int n_iter, double t0, double* average_per_rhs,
                     double* idle_fraction);
int hs_pipeline_simulate(int dim, const int counts[3], int n_rhs, int n_iter, double t0, double* completion_times,
                         double* makespan, double* average_per_rhs);

/* CSR of one subdomain's J-scaled PML operator as the solver assembled it (on the device unless
 * HS_HOST_SETUP=1), in the reference's layout (include/helmsweep/operator.hpp:14-29; rows over
 * the subdomain's local grid, axis 0 fastest). Pass NULL arrays to query n / nnz first. */
int hs_ddm_sub_csr(const hs_ddm* s, int sub, int64_t* row_ptr, int64_t* col, double* val, int64_t* n, int64_t* nnz);
/* Device memory of a solver: bytes of resident solve factors (packed 8x8-block layout), bytes of
 * the solve state for the current batch width, and the RHS the device solves per batch (wider
 * requests run as consecutive batches). */
int hs_ddm_memory(const hs_ddm* s, int64_t* factor_bytes, int64_t* state_bytes, int* max_batch);

/* Number of kernel launches issued by this library since load (evidence counter). */
int64_t hs_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* HELMSWEEP_B200_H */
