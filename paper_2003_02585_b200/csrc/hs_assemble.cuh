// Device subdomain setup (hs_assemble.cu): extended wavenumber + J-scaled PML CSR values.
#pragma once

#include <cstdint>

#include "hs_common.hpp"

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

}  // namespace hsb
