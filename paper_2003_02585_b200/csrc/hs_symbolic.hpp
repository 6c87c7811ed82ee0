// Symbolic layer: geometric nested-dissection tree of one subdomain grid and the
// integer tables the device kernels consume. The tree is the reference's exactly
// (/root/reference/proj/src/direct.cpp:91-179: longest axis with ties to the lowest,
// C++ truncating mid = (lo+hi)/2, leaves of <= 64 nodes or extent < 2, separator =
// mid plane, bnd = face-adjacent halo planes, postorder child0-child1-node), so the
// elimination order, factor_nnz and pivot indices match the reference.
//
// Device layout decisions:
//  * vectors are permuted once into elimination order, so a front's separator is
//    the contiguous slice [sep_off, sep_off+k) and RHS columns are node-major with the
//    RHS index fastest;
//  * a front's solve factor [M; W] is stored once in 8x8 complex blocks (front_block_elems),
//    read as DMMA A fragments by the forward and as transposed B fragments by the backward;
//  * forward-solve update vectors (the multifrontal "extend-add" of x[bnd] -= L21 t)
//    live in a per-front slot of m-k nodes, reduced into the parent in fixed order.
#pragma once

#include <memory>

#include "hs_setup.hpp"

namespace hsb {

constexpr int kLeafNodes = 64;   // src/direct.cpp:15
constexpr int kSolvePanel = 32;  // solve-kernel panel width (device layout)

// Solve-factor layout of one front (hs_solve.cu, written by the factorization kernel):
// [M; W] with rows [0, kp) = separator (kp = k rounded up to 8, rows >= k zero) followed by
// ceil8(m - k) boundary rows, columns [0, kp); cut into 8x8 complex blocks stored row-major
// (1 KB). Bands of 4 block rows; band t holds column blocks cb < min(kp/8, 4t + 4) (M is
// lower triangular), ordered [cb][block row in band]. Every band but the last is full, so
// the band base has a closed form (band_base).
inline int pad8(int v) { return (v + 7) & ~7; }
inline long long band_base(int t, int kb) {
  const int j0 = kb >> 2;
  const long long s = t <= j0 ? 2LL * t * (t + 1) : 2LL * j0 * (j0 + 1) + static_cast<long long>(t - j0) * kb;
  return s * 256;
}
inline long long front_block_elems(int m, int k) {
  const int kb = pad8(k) >> 3, nrb = kb + (pad8(m - k) >> 3), nband = (nrb + 3) >> 2;
  if (nband == 0) return 0;
  const int t = nband - 1, rbs = nrb - 4 * t, ncb = kb < 4 * t + 4 ? kb : 4 * t + 4;
  return band_base(t, kb) + static_cast<long long>(ncb) * rbs * 64;
}

struct FrontDesc {
  int k = 0, m = 0;
  int sep_off = 0;       // first elimination position of the separator
  int bnd_off = 0;       // offset into bnd_elim (m-k entries)
  int parent = -1;       // front index (postorder numbering)
  int child[2] = {-1, -1};
  int cmap_off[2] = {0, 0};  // offset into child_map for child c (m_c-k_c entries)
  int height = 0, depth = 0;
  int orig_off = 0, orig_cnt = 0;  // original-entry scatter list
  long long fac_off = 0;  // elements into the subdomain's factor block
  long long v_off = 0;    // nodes into the update-vector slot
  long long f_off = 0;    // elements into the dense factorization workspace
  long long t_off = 0;    // front positions (m per front) into the extend-add source map
};

// One symbolic class: subdomains whose local grids (and therefore trees, CSR
// structure and index tables) coincide share one of these on the device.
struct SymbolicClass {
  int dim = 2;
  Vec3i size{1, 1, 1};   // local grid extents
  std::int64_t n = 0;    // local node count
  std::vector<FrontDesc> fronts;        // postorder
  std::vector<int> elim_of_local;       // local linear -> elimination position
  std::vector<int> local_of_elim;       // inverse
  std::vector<int> sep_local;           // per front, separator local ids (elimination order)
  std::vector<int> bnd_elim;            // per front, bnd elimination positions
  std::vector<int> child_map;           // child bnd slot -> parent front position
  std::vector<int> orig_fpos;           // factorization scatter: lower F index (col*m+row)
  std::vector<int> orig_eidx;           // factorization scatter: CSR entry index
  std::vector<int> order_up;            // fronts sorted by (height, index)
  std::vector<int> order_down;          // fronts sorted by (depth, index)
  std::vector<int> level_start_up;      // order_up slice per height
  int max_height = 0, max_depth = 0;
  long long fac_total = 0;   // elements per subdomain factor block
  long long v_total = 0;     // update-vector nodes per slot
  long long f_total = 0;     // dense workspace elements
  long long t_total = 0;     // front positions per class (source-map entries)
  std::int64_t factor_nnz = 0;  // reference convention sum m*k (src/direct.cpp:271)
  std::int64_t packed_entries = 0;  // sum over fronts of m*k - k*(k-1)/2 (lower trapezoid incl. D)
  std::int64_t peak_bytes = 0;  // reference accounting (src/direct.cpp:216-279)
  int max_m = 0, max_k = 0;
  std::vector<std::int64_t> csr_row_ptr, csr_col;  // CSR structure shared by the class
};

// Builds the symbolic class of a grid range from the CSR structure assembled on it.
std::unique_ptr<SymbolicClass> build_symbolic(int dim, const GridRange& range,
                                              const std::vector<std::int64_t>& row_ptr,
                                              const std::vector<std::int64_t>& col);

bool same_structure(const SymbolicClass& a, const SymbolicClass& b);

}  // namespace hsb
