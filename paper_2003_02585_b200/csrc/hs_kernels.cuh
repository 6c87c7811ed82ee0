// Launch wrappers for the sm_100a kernels of the helmsweep hot path (hs_kernels.cu).
#pragma once

#include "hs_device.cuh"

// Items spanning several (band, RHS group) units (host HS_MERGE, measured slower); 0: the solve
// kernel runs one unit per item and the host never merges
#ifndef HS_MERGE_UNITS
#define HS_MERGE_UNITS 0
#endif

namespace hsb {

struct SolveArgs {
  const SolveItem* items;
  const SolveJob* jobs;
  int nitems;
  int R;           // RHS per batch (row stride of x / x1 / V)
  int ngr;         // RHS groups of 8 (stride of the per-group arrival counters / partial tiles)
  int* done;       // per [slot * nf_max + front]: finalized (band, group) pairs of this pass
  int* arr;        // split-K arrivals per [(slot * arr_stride + arr_off + band) * ngr + group]
  long long arr_stride;
  double* part;    // split-K partial tiles (1024 doubles) per [(slot * part_stride + part_off + idx) * ngr + group]
  long long part_stride;
  unsigned* queue; // dynamic item counter, zeroed per launch
  unsigned long long* trace;  // optional per-item timestamps [4 * item]: dequeue, ready, done, smid
  int nf_max;
  double2* vbuf;           // update-vector slots
  long long vslot_stride;  // elements per slot
  const rmask* nzmask;     // per subdomain: RHS columns with a nonzero right-hand side
  const unsigned* tface;   // per task: faces with nonzero injected data (bits 0-7), 0x100 = every front live,
                           // bits 16-23 = 8-column groups for which every front is live (sweep 1: split source)
                           // (sweep 1); null = every front live
  int quad;                // items are listed in quads (four RHS groups of one band chunk, null-padded,
                           // nzi < 0) that one CTA dequeues together and streams through L1
  int m3;                  // complex products as 3 real DMMAs (3 CTAs / SM) instead of 4 (4 CTAs / SM)
  const unsigned* need;    // per subdomain bitset over fronts: x read back (backward pass); null = all
  int need_words;          // 32-bit words per subdomain in `need`
  int nsub;                // subdomains (task index nzi = (sweep - 1) * nsub + sub)
  int no_group_skip;       // 1: RHS groups that are all zero for a task are computed anyway (HS_NO_GROUP_SKIP, A/B)
  // per-slot buffers (slot = the task's position in its macro-step): the task's right-hand side
  // (forward input) and z = D^-1 L^-1 b (forward output, backward input), elimination order,
  // node-major x R; slot_stride elements apart
  double2* rbs;
  double2* x1s;
  long long slot_stride;
};

// Multifrontal forward (z = D^-1 L^-1 b) or backward (x = L^-T z) pass over the work items of
// one step group (src/direct.cpp:290-325); hs_solve.cu.
void launch_solve(const SolveArgs& a, bool fwd, cudaStream_t s);
// split-K bookkeeping shared by the host item builder and the kernels
int solve_fwd_chunks(int m, int k, int band, int kc);
int solve_bwd_chunks(int m, int k, int cband, int kr);

struct FactorArgs {
  const FactorTask* tasks;
  int ntasks;
  const DevClass* cls;
  const DevSub* subs;
  double2* work;                // dense front workspace (column-major m x m per front)
  double2* scratch;             // global panel scratch when a panel does not fit in smem
  unsigned long long* err_key;  // min over (sub << 32 | elimination position) of bad pivots
};
// Assembly + extend-add + partial LDL^T of every front at one tree height
// (src/direct.cpp:55-87, 181-281).
void launch_factor_level(const FactorArgs& a, int max_m, cudaStream_t s);
// The same with one thread-block cluster of kFactorCluster CTAs per front (large fronts); scratch
// must hold kFactorCluster * ntasks * 2 * max_m * kNB entries.
constexpr int kFactorCluster = 8;
constexpr int kFactorBigM = 640;  // fronts with m >= this go to the cluster path
void launch_factor_level_cluster(const FactorArgs& a, int max_m, cudaStream_t s);
// Blocked GEMM-phase factorization of large fronts, one cluster per front (hs_factor.cu); scratch
// must hold ntasks * factor_big_scratch(max_m) entries.
void launch_factor_big(const FactorArgs& a, int max_m, cudaStream_t s);
long long factor_big_scratch(int max_m);
size_t factor_smem_bytes(int max_m);

struct SweepArgs {
  DevGeom g;
  const DevClass* cls;
  const DevSub* subs;
  const int2* tasks;       // (subdomain, 1-based sweep) of every task of the macro-step
  int ntasks;
  int R;
  int nsweeps;
  int dirs;                // 2*dim
  int nbuf;                // x buffers: sweep l uses buffer (l-1) % nbuf
  long long xstride;       // elements between x buffers
  const double2* b;        // global rhs, node-major N x R
  double2* mbox;           // mailbox slots [target sub][generating sweep][dir][2][line][R]
  long long mbox_dir_stride;  // elements per (sub, sweep, dir) slot
  rmask* mpres;            // presence bitmask [target sub][generating sweep][dir]
  rmask* nzmask;           // [sweep][sub]
  unsigned* tface;         // [sweep][sub]: faces whose injection lines carry a nonzero value
  const int* route;        // [sweep][dir] target sweep (0 = discard)
  double2* rbs;            // per-slot right-hand sides (slot = task position in the macro-step)
  long long slot_stride;
  const int2* prev;        // per task: the previous occupant of its slot (class, 1 if it wrote the
                           // whole buffer) -- (-1, 0) when the slot is clean
};
// RHS of each subdomain task: split source (sweep 1) plus injected traces, and the
// exact-zero test (src/sweeper.cpp:189-251, src/transfer.cpp:68-89).
void launch_build_rhs(const SweepArgs& a, long long max_n, int max_line, cudaStream_t s);
// Trace extraction -> routing -> mailbox deposit (src/transfer.cpp:13-66, src/sweeper.cpp:295-307).
void launch_extract_deposit(const SweepArgs& a, int max_line, cudaStream_t s);

#define HS_MAX_ACC_SWEEPS 8
struct AccumArgs {
  DevGeom g;
  int R;
  int l;
  int dvec[3];               // sweep direction of sweep l
  long long xoff;            // offset of sweep l's x buffer (elements)
  const double2* x;          // x buffers of every subdomain (elimination order, node-major x R)
  const int2* acc_ent;       // this sweep direction's plan: per global node 2^dim entries in the
                             // reference's accumulation order (x position n_base[sub] + elim,
                             // sub << 4 | weight numerator); unused entries have position -1
  const rmask* nzmask;       // [sub] for sweep l
  double2* u;                // global solution, node-major N x R
  double* partial;           // per-block partial |contrib|^2 [nblocks][R]
  long long n0, n1;          // node range of this launch
};
// u += sum_sub w * u_local over the subdomain supports in the reference's order
// (src/transfer.cpp:91-102, src/sweeper.cpp:308-312); emits per-block norm partials.
int launch_accumulate(const AccumArgs& a, cudaStream_t s);  // nodes [a.n0, a.n1); returns its block count

// Every sweep of an application in one pass (all x buffers distinct): u = (((0 + c_1) + c_2) + ...)
// with c_l the sweep-l contribution, node by node in sweep order -- the same sums as L separate
// accumulates, one read of each x and one write of u; partials of |c_l|^2 per sweep.
struct AccumAllArgs {
  DevGeom g;
  int R, L;
  const int2* acc_ent[HS_MAX_ACC_SWEEPS];   // plan of sweep l's direction
  long long xoff[HS_MAX_ACC_SWEEPS];        // x buffer of sweep l
  const rmask* nzmask[HS_MAX_ACC_SWEEPS];
  const double2* x;
  double2* u;
  double* partial;     // sweep l's partials at partial + l * pstride
  long long pstride;
  // region: rows [row0, row0 + cnt / w) of gx nodes, columns [x0, x0 + w) (a stripe: x0 = 0, w = gx)
  long long row0, cnt;
  int gx, x0, w;
  // u after every completed round but the last (per-round residuals, src/sweeper.cpp:313-325):
  // uround + (q - 1) * rstride after sweep q * rlen; null: none
  double2* uround;
  long long rstride;
  int rlen;
};
int launch_accumulate_all(const AccumAllArgs& a, cudaStream_t s);
// Deterministic final reduction of per-block partials: out[r] = sum_b partial[b][r].
constexpr int kReducePad = 256;  // extra partial rows every partial buffer reserves (reduction scratch)
void launch_reduce_partials(double* partial, int nblocks, int R, double* out, cudaStream_t s);

// Cross-rank exchange of a partitioned solve: one segment per mailbox slot,
// presence word, ghost x run or nonzero word, copied between the solver's arrays and a flat
// message buffer of doubles (words travel as exactly representable doubles).
struct XSeg {
  int kind;        // 0 mailbox data, 1 presence word, 2 ghost x values, 3 nonzero word
  int count;       // complex values (kinds 0, 2), 1 for words
  long long a;     // mbox element / mpres slot / ghost position-table offset / nzmask index
  long long b;     // offset in the message buffer (doubles)
  long long c;     // kind 2: x buffer offset (elements)
};
void launch_pack_home(const double2* u, const int* list, long long count, int R, double2* out, cudaStream_t s);
void launch_unpack_home(const double2* in, const int* lists, long long max_home, int world, int R, double2* u,
                        cudaStream_t s);
void launch_xpack(const XSeg* segs, int nseg, bool pack, double* buf, double2* mbox, rmask* mpres, double2* x,
                  rmask* nzmask, const long long* gpos, int R, cudaStream_t s);

// Global CSR SpMV y = A x (x, y node-major N x R) (src/operator.cpp:7-17) and the
// residual partials |b - y|^2, |b|^2.
// The global operator in stencil form: every row's entries sit at row + off[q] (a 2 dim + 1 point
// stencil in CSR column order; absent entries hold zero), so a row's x loads need no row-pointer /
// column-index loads first. val = nullptr: not available (use the CSR arrays).
struct StencilOp {
  const double2* val = nullptr;  // [n][S]
  int S = 0;
  long long off[7] = {0, 0, 0, 0, 0, 0, 0};
};
// Builds the stencil form from CSR; *bad is set when some entry is off the stencil.
void launch_stencil_build(long long n, const std::int64_t* row_ptr, const int* col, const double2* val, StencilOp op,
                          double2* out, unsigned* bad, cudaStream_t s);
int launch_residual(long long n, const std::int64_t* row_ptr, const int* col, const double2* val,
                    const double2* x, const double2* b, int R, double* partial_num,
                    double* partial_den, cudaStream_t s, int gx = 0, StencilOp sop = StencilOp());
void launch_spmv(long long n, const std::int64_t* row_ptr, const int* col, const double2* val,
                 const double2* x, double2* y, int R, cudaStream_t s);

// RHS-major [R][N] <-> node-major [N][R] with optional per-column shell masking.
void launch_transpose_in(const double2* src, double2* dst, long long n, int R, cudaStream_t s, const int* perm = nullptr);
void launch_transpose_out(const double2* src, double2* dst, long long n, int R, cudaStream_t s, const int* perm = nullptr);
void launch_bump_epoch(unsigned* epoch, unsigned by, cudaStream_t s);
// node range [n0, n1) only (streamed host transfers)
void launch_transpose_in_range(const double2* src, double2* dst, long long n, int R, long long n0, long long n1,
                               cudaStream_t s);
void launch_transpose_in_tile(const double2* src, double2* dst, long long n, int R, int gx, int x0, int x1,
                              long long row0, long long row1, cudaStream_t s, const int* perm = nullptr);
void launch_transpose_out_tile(const double2* src, double2* dst, long long n, int R, int gx, int x0, int x1,
                               long long row0, long long row1, cudaStream_t s, const int* perm = nullptr);
// Column order of a batch (perm[j] = the caller's column held at internal position j): ascending
// Morton key of the subdomain cell at the centre of each column's nonzeros (bbox: 6 ints per column,
// scratch). rhs_order_key is the same key on the host (the streamed path samples b there).
void launch_rhs_order(const double2* b, long long n, int R, const DevGeom& g, int* bbox, int* perm, cudaStream_t s);
unsigned rhs_order_key(const DevGeom& g, const int* bbox6);
void launch_transpose_out_range(const double2* src, double2* dst, long long n, int R, long long n0, long long n1,
                                cudaStream_t s);

// Krylov vector kernels (src/krylov.cpp:9-13, 52-56, 109-111) on node-major N x R arrays.
int launch_dot_partials(const double2* a, const double2* b, long long n, int R, double2* partial,
                        cudaStream_t s);
void launch_reduce_cpartials(const double2* partial, int nblocks, int R, double2* out, cudaStream_t s);
void launch_axpy_cols(double2* y, const double2* x, const double2* alpha, int neg, long long n, int R,
                      cudaStream_t s);
void launch_scale_cols(double2* y, const double* inv, long long n, int R, cudaStream_t s);

}  // namespace hsb
