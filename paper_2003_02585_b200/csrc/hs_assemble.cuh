// Device subdomain setup (hs_assemble.cu): extended wavenumber + J-scaled PML CSR values.
#pragma once

#include <cstdint>

#include "hs_common.hpp"
#include "hs_device.cuh"

namespace hsb {

// WaveNumberModel on the device (include/helmsweep/media.hpp:31-55).
struct AsmMedium {
  int kind;  // 0 constant, 1 two-layered, 2 gridded
  double kappa, kd, ku, eta, eps, omega;
  int axis;
  int vdim;
  int vn[3];
  double vorg[3], vsp[3];
  const float* vc;  // gridded velocity samples (device)
};

// One grid to assemble (a subdomain's local grid, or the global grid).
struct AsmSub {
  int lo[3], size[3];             // range lo and extents (axis 0 fastest; unused axes size 1)
  double cell_lo[3], cell_hi[3];  // the box kappa is extended from (nearest point)
  const double2* anode[3];        // alpha at nodes, per axis (local index)
  const double2* ahalf[3];        // alpha at half-points, per axis
  const std::int64_t* row_ptr;    // CSR structure (the symbolic class's)
  const std::int64_t* col;
  double2* val;                   // output values
  unsigned long long* maxabs;     // max |a_ij| (bit pattern of a non-negative double), pre-zeroed
};

struct AsmArgs {
  int dim;
  double h[3], origin[3];
  AsmMedium med;
  const AsmSub* subs;
  int nsub;
  unsigned* bad;  // set when a velocity sample interpolates to <= 0
};

void launch_assemble(const AsmArgs& a, long long max_rows, cudaStream_t s);

// Partition geometry of the setup plans (src/geometry.cpp:105-154: uniform cuts c * w, supports
// extended by pad on the outer faces, weight numerators 1 or 2 per axis).
struct PlanGeom {
  int dim;
  int glo[3], gsize[3];  // global padded range
  long long gn;
  int counts[3], w[3], pad;
  const DevClass* cls;
  const int* sub_cls;          // per subdomain: symbolic class
  const long long* n_base;     // per subdomain: first position of its vectors
};
// Accumulate plan (src/transfer.cpp:91-102, src/sweeper.cpp:285-311): per global node and sweep
// direction, the (x position, sub << 4 | weight numerator) of every subdomain whose support holds
// the node, in the reference's order for that direction (step of the sweep, then ascending id);
// unused entries (-1, 0). acc_ent[(di * gn + node) * 2^dim + i].
void launch_acc_plan(const PlanGeom& g, int ndirs, const int (*dvec)[3], int2* acc_ent, cudaStream_t s);
// Split-source plan (src/sweeper.cpp:189-202): per (subdomain, elimination position), the global
// node and the weight numerator (0 on the local shell or outside the support).
void launch_split_plan(const PlanGeom& g, int nsub, long long max_n, int* split_gp, unsigned char* split_w,
                       cudaStream_t s);

}  // namespace hsb
