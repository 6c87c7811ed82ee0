// Device-visible descriptors shared by the sm_100a kernels (hs_kernels.cu) and the
// host orchestration (hs_ddm.cu). Plain PODs; complex128 is double2 (re, im).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hsb {

constexpr int kMaxDirs = 6;  // 2*dim cardinal faces
constexpr int kMaxRhs = 64;  // RHS per device batch (bitmask width)
using rmask = unsigned long long;  // one bit per RHS column of a batch

struct DevFront {
  int k, m, sep_off, bnd_off;
  int parent, child0, child1, cmap0, cmap1;
  int orig_off, orig_cnt;
  int arr_off;   // split-K arrival counters: first band / column band of this front
  int part_off;  // split-K partial tiles of this front (0 parts when no band is split)
  int pad_;
  long long fac_off, v_off, f_off, t_off;
};

struct DevClass {
  const DevFront* fronts;
  const int* bnd_elim;
  const int* child_map;
  const int2* pmap;           // per front position (offset t_off): update-vector row (v_off + i) of child0 / child1, -1 if none
  const int* orig_fpos;
  const int* orig_eidx;
  const int* elim_of_local;
  const int* local_of_elim;
  // trace line tables per direction d = 2*axis + (sign > 0), elimination positions
  const int* ext_u0[kMaxDirs];   // outgoing trace: interface line
  const int* ext_um1[kMaxDirs];  // outgoing trace: line one step toward the source
  const int* inj_p0[kMaxDirs];   // incoming trace: interface line (-1 on shell)
  const int* inj_pm[kMaxDirs];   // incoming trace: first source-side line (-1 on shell)
  int line_len[kMaxDirs];
  const unsigned char* on_line;  // per elimination position: on an injection line of some face
  int n, nfronts;
  int size[3];
};

struct DevSub {
  int cls;
  int sub[3];
  int lo[3];                  // local grid range lo (global index coordinates)
  double tol;                 // pivot tolerance 1e-14 * max|a_ij| (src/direct.cpp:191-193)
  double2* factor;            // panels (hs_symbolic.hpp)
  double2* dinv;              // 1/d, elimination order
  const double2* val;         // CSR values (factorization input)
  double2* x;                 // solve vector, elimination order, node-major x R (rhs -> solution)
  double2* x1;                // (unused: z and the right-hand side live in per-slot buffers,
  double2* rb;                //  SolveArgs / SweepArgs rbs, x1s)
  const double2* coef[kMaxDirs];  // injection couplings per incoming direction
  const int* split_gp;             // per elimination position: global node of the split source
  const unsigned char* split_w;    // its weight numerator over 2^dim (0 = shell or outside support)
};

// Global grid and partition geometry for split / accumulate kernels.
struct DevGeom {
  int dim;
  int glo[3], gsize[3];       // global padded range
  int counts[3];
  int pad;
  int cut_w[3];               // uniform cut width per axis (cuts[c] = c * w)
  int nsub;
  long long gn;               // global node count
};

// A solve work item (hs_solve.cu): forward band idx (32 padded rows of [M; W]) over
// column-block chunk `chunk`, or backward column band idx (32 separator columns) over
// block-row chunk `chunk`; RHS columns [r0, r0 + rw), rw <= 16. slot = position of the task
// in its macro-step; job = its (x buffer, subdomain, front) record; nzi = the task's entry in the
// per-(sweep, subdomain) nonzero masks.
// A merged item (idx1 > idx + 1 or r1 > r0 + rw) runs the unsplit units (band t in [idx, idx1)) x
// (RHS group r in [r0, r1), step gw) one after the other in one warp: one dependency wait, one
// ticket and one release for all of them (small fronts' units are only a few k-steps long).
struct SolveItem {
  int nzi, front, job, idx, slot, r0, rw, chunk;
  int idx1, r1;
  // the first factor range the item streams (L2 bulk prefetch issued by the warp that dequeues it,
  // as soon as it has the record, ahead of the item's dependency wait)
  const void* pf;
  unsigned pf_bytes;
  int pad_;
};

// Everything a solve item needs about its (subdomain, front), resolved on the host for the
// current RHS width so an item costs two dependent loads (item, job) before its loads start.
struct SolveJob {
  const double2* factor;  // solve-layout factor of the front
  const double2* dinv;    // 1/d of the separator (elimination order)
  double2* x;             // the subdomain's x (elimination order, node-major x R)
  double2* x1;            // (unused: z and the right-hand side are per slot, SolveArgs x1s / rbs)
  const double2* b;
  const int2* pm;         // extend-add source map of the front's positions
  const int* be;          // boundary elimination positions
  int k, m, sep_off, v_off;
  int child0, child1, tgt_c0, tgt_c1;      // children and their finalized-item counts (forward waits)
  int parent, tgt_p, arr_off, part_off;    // parent and its finalized-item count (backward waits)
  int kc, kr;                              // split-K chunk: column blocks (forward) / block rows (backward)
  int gw;                                  // RHS per item group (8 on the critical path, else 16)
  // Faces whose injection lines lie in the subtree of this front (bits 0-7), of child0 (8-15) and
  // child1 (16-23). Past sweep 1 a task's right-hand side is zero off the lines of the faces that
  // received traces, so a front whose subtree holds none of them has T = 0, z = 0 and V = 0.
  int act;
};

struct FactorTask {
  int sub, front;
  long long fbase;            // dense workspace base of this subdomain (elements)
};

}  // namespace hsb
