// Host-side problem setup for the B200 hot path: grids, checkerboard partition,
// partition-of-unity weights, PML stretching, wave-number media and the J-scaled
// operator assembly. This is the input producer of the GPU factorization; it
// reproduces the reference's formulas operation for operation so the operator
// handed to the device is bitwise the one the reference factorizes:
//   geometry   /root/reference/proj/src/geometry.cpp:28-177
//   PML        /root/reference/proj/src/pml.cpp:7-52, include/helmsweep/pml.hpp:35-58
//   media      /root/reference/proj/src/media.cpp:30-217
//   assembly   /root/reference/proj/src/operator.cpp:25-98
//   sweep plan /root/reference/proj/src/sweeper.cpp:10-73
#pragma once

#include "hs_common.hpp"

namespace hsb {

struct Box {
  int dim = 2;
  Vec3d lo{0.0, 0.0, 0.0};
  Vec3d hi{1.0, 1.0, 1.0};
  double extent(int a) const { return hi[a] - lo[a]; }
};

struct GridRange {
  int dim = 2;
  Vec3i lo{0, 0, 0};
  Vec3i hi{0, 0, 0};
  int size(int a) const { return hi[a] - lo[a] + 1; }
  std::int64_t count() const {
    std::int64_t c = 1;
    for (int a = 0; a < dim; ++a) c *= size(a);
    return c;
  }
  std::int64_t linear(const Vec3i& p) const {
    std::int64_t id = 0;
    for (int a = dim - 1; a >= 0; --a) id = id * size(a) + (p[a] - lo[a]);
    return id;
  }
  Vec3i unlinear(std::int64_t id) const {
    Vec3i p{0, 0, 0};
    for (int a = 0; a < dim; ++a) {
      p[a] = lo[a] + static_cast<int>(id % size(a));
      id /= size(a);
    }
    return p;
  }
  bool contains(const Vec3i& p) const {
    for (int a = 0; a < dim; ++a)
      if (p[a] < lo[a] || p[a] > hi[a]) return false;
    return true;
  }
};

struct LocalGrid {
  int dim = 2;
  GridRange range;
  Vec3d h{0.0, 0.0, 0.0};
  Vec3d origin{0.0, 0.0, 0.0};
  double coord(int a, int i) const { return origin[a] + i * h[a]; }
  bool on_shell(const Vec3i& p) const {
    for (int a = 0; a < dim; ++a)
      if (p[a] == range.lo[a] || p[a] == range.hi[a]) return true;
    return false;
  }
};

struct PmlSpec {
  int width = 30;
  double strength = 2.0;
  int exponent = 2;
};

struct Partition {
  int dim = 2;
  Vec3i counts{1, 1, 1};
  std::array<std::vector<int>, 3> cuts;
  Box box;  // interior box
  Vec3d h{0.0, 0.0, 0.0};
  int cell_count() const { return counts[0] * counts[1] * (dim == 3 ? counts[2] : 1); }
  int flatten(const Vec3i& s) const {
    int id = 0;
    for (int a = dim - 1; a >= 0; --a) id = id * counts[a] + s[a];
    return id;
  }
  Vec3i unflatten(int id) const {
    Vec3i s{0, 0, 0};
    for (int a = 0; a < dim; ++a) {
      s[a] = id % counts[a];
      id /= counts[a];
    }
    return s;
  }
  GridRange owned(const Vec3i& s) const;
  Box cell(const Vec3i& s) const;
  bool has_neighbor(const Vec3i& s, int axis, int sign) const {
    if (axis >= dim) return false;
    const int t = s[axis] + sign;
    return t >= 0 && t < counts[axis];
  }
};

Partition make_partition(const Box& interior, const Vec3i& intervals, const Vec3i& counts);

// Partition-of-unity weights (src/geometry.cpp:124-154).
struct Weights {
  const Partition* p = nullptr;
  int pad = 0;
  int weight2(int axis, int cell, int index) const;
  double weight(const Vec3i& sub, const Vec3i& node) const;
  GridRange support(const Vec3i& sub) const;
};

struct PmlCoefficients {
  int dim = 2;
  GridRange range;
  Vec3d h{0.0, 0.0, 0.0};
  std::array<CVector, 3> node, half;
  Complex alpha(int a, int gi) const { return node[a][gi - range.lo[a]]; }
  Complex jacobian(const Vec3i& p) const {
    Complex j = 1.0;
    for (int a = 0; a < dim; ++a) j *= alpha(a, p[a]);
    return j;
  }
  Complex coupling(int axis, const Vec3i& p) const {
    Complex v = 1.0;
    for (int b = 0; b < dim; ++b)
      if (b != axis) v *= alpha(b, p[b]);
    return v / half[axis][p[axis] - range.lo[axis]] / (h[axis] * h[axis]);
  }
};

PmlCoefficients build_coefficients(const PmlSpec& spec, const Box& box, const LocalGrid& grid);

struct VelocityGrid {
  int dim = 2;
  Vec3i n{2, 2, 1};
  Vec3d origin{0.0, 0.0, 0.0};
  Vec3d spacing{1.0, 1.0, 0.0};
  std::vector<float> c;
  double sample(const Vec3d& x) const;
};

struct Medium {
  enum Kind { Constant = 0, TwoLayered = 1, Gridded = 2 };
  Kind kind = Constant;
  double kappa = 0.0, kappa_up = 0.0, kappa_down = 0.0;
  int axis = 1;
  double eta = 0.0, eps = 0.0;
  VelocityGrid velocity;
  double omega = 0.0;
};

double eval_kappa(const Medium& m, const Vec3d& x);
std::vector<double> extend_to_subdomain(const Medium& m, const Box& cell, const LocalGrid& grid);

struct Csr {
  std::int64_t n = 0;
  std::vector<std::int64_t> row_ptr, col;
  CVector val;
};

Csr assemble(const LocalGrid& grid, const PmlCoefficients& coeffs, const std::vector<double>& kappa);

// Sweep plan and routing (src/sweeper.cpp:10-73, src/geometry.cpp:156-177).
std::vector<Vec3i> sweep_plan(int dim, int rounds);
int route_trace(const std::vector<Vec3i>& plan, int dim, int gen_sweep, int axis, int sign);
int sweep_step_count(const Vec3i& counts, int dim);
int step_of(const Vec3i& counts, int dim, const Vec3i& d, const Vec3i& sub);

}  // namespace hsb
