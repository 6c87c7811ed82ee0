// Common host/device types and error plumbing for the helmsweep B200 hot path.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <array>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>

namespace hsb {

using Complex = std::complex<double>;
using CVector = std::vector<Complex>;
using Vec3i = std::array<int, 3>;
using Vec3d = std::array<double, 3>;

// Status codes of the C-ABI (include/helmsweep_b200.h). They mirror the reference's
// exception classes (inc/common.hpp:18-35).
enum Status : int {
  kOk = 0,
  kConfig = 1,    // ConfigError
  kData = 2,      // DataError
  kSingular = 3,  // SingularMatrixError
  kCuda = 4,
  kInternal = 5,
};

struct Error : std::runtime_error {
  Status code;
  std::int64_t pivot_index = -1;
  int pivot_sub = -1;
  Error(Status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void config_error(const std::string& m) { throw Error(kConfig, m); }
[[noreturn]] inline void data_error(const std::string& m) { throw Error(kData, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw Error(kCuda, std::string(what) + ": " + cudaGetErrorString(e) + " at " + file + ":" +
                           std::to_string(line));
}
#define HS_CUDA(x) ::hsb::cuda_check((x), #x, __FILE__, __LINE__)

// Per-device cached launch setup. CUDA function attributes (the >48 KB dynamic shared memory
// opt-in) and occupancy-derived grid sizes belong to one device context, so they are set and
// cached per device ordinal, not once per process.
struct PerDevice {
  std::mutex mu;
  std::array<int, 64> val{};  // 0: not configured on that device yet
  template <class F>
  int get(F&& configure) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice", __FILE__, __LINE__);
    if (dev < 0 || dev >= static_cast<int>(val.size())) throw Error(kCuda, "device ordinal out of range");
    std::lock_guard<std::mutex> lk(mu);
    if (!val[dev]) val[dev] = configure(dev);
    return val[dev];
  }
};

}  // namespace hsb
